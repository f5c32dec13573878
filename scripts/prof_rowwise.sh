mkdir -p gpurun_out
python bench.py --config c2 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/std.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/std.json')); print('std', d['ms_per_step'], d['roofline']['frac'])"
python bench.py --config c2 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/std2.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/std2.json')); print('std2', d['ms_per_step'], d['roofline']['frac'])"
CMD="python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --clusters 296"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rowwise -s 3 -c 1 -o gpurun_out/prof_c2b $CMD > gpurun_out/ncu_full.log 2>&1; echo full=$?
