mkdir -p gpurun_out
for cfg in "3 592 4" "3 592 4" "2 592 4" "2 740 4" "3 666 4" "4 518 4" "3 518 4" "2 888 4" "3 444 4" "2 1184 2" "3 592 8" "2 592 8"; do
 set -- $cfg
 HPAR_RW_STAGES=$1 timeout -s KILL 120 python bench.py --config c2 --steps 200 --no-cpu-baseline --no-e2e --clusters $2 --warps $3 > gpurun_out/sw.json 2>gpurun_out/sw.err
 python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('S=$1 C=$2 W=$3', round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err
done
