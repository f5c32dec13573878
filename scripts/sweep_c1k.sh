# C1: CTAs per cluster K (1 = plain CTAs, no cluster barrier) x teams; 2 rounds
mkdir -p gpurun_out
for i in 1 2; do
for cfg in "2 148 8" "1 296 8" "1 148 8" "1 296 4" "2 148 4" "1 592 4"; do
 set -- $cfg
 HPAR_K=$1 timeout -s KILL 120 python bench.py --config c1 --steps 1000 --no-cpu-baseline --no-e2e --clusters $2 --warps $3 > gpurun_out/sw1.json 2>gpurun_out/sw1.err
 python -c "import json; d=json.load(open('gpurun_out/sw1.json')); print('K=$1 C=$2 W=$3', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw1.err
done; done
