# usage: bash scripts/gpu_check.sh [pytest -k expr]   — GPU tests (no -x), smoke, bench lines of every config
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "from paper_2309_01906_b200 import build; build.build()" > gpurun_out/build.log 2>&1
K=${1:+-k "$1"}
timeout 2400 python -m pytest tests -m gpu -q -rf $K > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for c in ${CONFIGS:-c5 c2 c1 c3 c4 c6}; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
