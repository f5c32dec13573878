mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests -m gpu -x -q -k "hist" 2>&1 | tail -2
for cfg in "74 4" "148 2" "148 4" "74 2" "222 2"; do
 set -- $cfg
 timeout -s KILL 120 python bench.py --config c4 --steps 20 --no-cpu-baseline --no-e2e --clusters $1 --warps $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
 python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('C=$1 W=$2', round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err
done
