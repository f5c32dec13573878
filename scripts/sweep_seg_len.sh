# C3: long-row segment length sweep (HPAR_SEG_SEG); parity at the smallest length first
mkdir -p gpurun_out
HPAR_SEG_SEG=2048 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "segmented" 2>&1 | tail -1
for i in 1 2; do for L in ${SWEEP:-8192 4096 2048 1024 16384}; do
  r=$(HPAR_SEG_SEG=$L timeout -s KILL 120 python bench.py --config c3 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))")
  echo "HPAR_SEG_SEG=$L $r"
done; done
