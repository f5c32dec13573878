# C4 sweep over (clusters, warps, tile, lane-table regions); run under gpurun
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests -m gpu -x -q -k "hist" 2>&1 | tail -2
IFS_OLD=$IFS; [ -n "$SWEEP" ] && IFS="|"
for cfg in ${SWEEP:-"74 8 16384 2" "74 8 8192 2" "74 8 8192 3" "74 6 12288 2" "74 6 12288 3" "74 10 10240 2" "74 10 10240 3" "74 12 12288 2" "74 12 6144 3" "74 16 16384 2" "74 16 8192 3" "74 8 16384 2" "74 4 16384 2"}; do
 IFS=$IFS_OLD; set -- $cfg
 HPAR_C4_TILE=$3 HPAR_C4_REGIONS=$4 timeout -s KILL 120 python bench.py --config c4 --steps 20 --no-cpu-baseline --no-e2e --clusters $1 --warps $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
 python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('C=$1 W=$2 tile=$3 R=$4', round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err
done
