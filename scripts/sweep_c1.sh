# C1 sweep: teams (1024 = the config's outer loop, 0 = C clusters x K) x warps; run under gpurun
mkdir -p gpurun_out
for cfg in "1024 0 8" "1024 0 4" "0 74 8" "0 74 4" "0 148 8" "0 148 4" "0 296 4" "0 37 8" "1024 0 8"; do
 set -- $cfg
 HPAR_C1_TEAMS=$1 timeout -s KILL 120 python bench.py --config c1 --steps 200 --no-cpu-baseline --no-e2e --clusters $2 --warps $3 > gpurun_out/sw1.json 2>gpurun_out/sw1.err
 python -c "import json; d=json.load(open('gpurun_out/sw1.json')); print('teams=$1 C=$2 W=$3', round(d['ms_per_step']*1000,2), 'us', d['config']['geometry'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw1.err
done
