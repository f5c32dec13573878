mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "teams or c1" 2>&1 | tail -1
for cfg in "1024 0 8" "0 74 8" "0 148 8" "0 74 4" "0 148 4" "0 296 4" "1024 0 8" "0 74 8"; do
 set -- $cfg
 HPAR_C1_TEAMS=$1 timeout -s KILL 120 python bench.py --config c1 --steps 300 --no-cpu-baseline --no-e2e --clusters $2 --warps $3 > gpurun_out/sw1.json 2>gpurun_out/sw1.err
 python -c "import json; d=json.load(open('gpurun_out/sw1.json')); print('teams=$1 C=$2 W=$3', round(d['ms_per_step']*1000,2), 'us', d['config']['geometry'])" || tail -3 gpurun_out/sw1.err
done
