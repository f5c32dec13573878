# C1: cluster size x warps at teams = 1024 (HPAR_K = CTAs per cluster); run under gpurun
mkdir -p gpurun_out
for cfg in "2 8" "1 8" "1 4" "4 8" "2 4" "1 2" "2 8"; do
 set -- $cfg
 HPAR_K=$1 timeout -s KILL 120 python bench.py --config c1 --steps 300 --no-cpu-baseline --no-e2e --warps $2 > gpurun_out/sw1.json 2>gpurun_out/sw1.err
 python -c "import json; d=json.load(open('gpurun_out/sw1.json')); print('K=$1 W=$2', round(d['ms_per_step']*1000,2), 'us', d['config']['geometry'])" || tail -3 gpurun_out/sw1.err
done
