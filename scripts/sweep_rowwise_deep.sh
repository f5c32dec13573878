# C2: fewer, deeper streams vs the tuned many-shallow geometry (same box).  args: S C W
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "2 888 4" "8 74 8" "12 74 8" "16 74 4" "6 148 4" "4 296 4" "8 148 4" "3 444 4"; do
 set -- $cfg
 HPAR_RW_STAGES=$1 timeout -s KILL 120 python bench.py --config c2 --steps 200 --no-cpu-baseline --no-e2e --clusters $2 --warps $3 > gpurun_out/sw.json 2>gpurun_out/sw.err
 python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('S=$1 C=$2 W=$3', round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err
done; done
