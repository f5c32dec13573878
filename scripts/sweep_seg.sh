# usage: bash scripts/sweep_seg.sh "LPL D DBG LONG CB" ... -- C3 segmented kernel variants
for v in "$@"; do
  set -- $v
  export HPAR_C3_LPL=$1 HPAR_SEG_D=$2 HPAR_SEG_DEBUG=$3 HPAR_SEG_LONG=$4 HPAR_SEG_CB=${5:-8}
  r=$(timeout -s KILL 120 python bench.py --config c3 --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))")
  t=$(HPAR_SEG_TIMES=1 timeout -s KILL 120 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "seg times" | tail -1)
  echo "LPL=$1 D=$2 dbg=$3 long=$4 cb=${5:-8}: $r | $t"
done
