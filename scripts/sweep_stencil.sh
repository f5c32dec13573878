# usage: bash scripts/sweep_stencil.sh "TY NST L2P" ...   -- c6 stencil kernel variants (env knobs)
for v in "$@"; do
  set -- $v
  r=$(HPAR_ST_TY=$1 HPAR_ST_NST=$2 HPAR_ST_L2P=$3 timeout -s KILL 120 python bench.py --config c6 --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))")
  echo "TY=$1 NST=$2 L2P=$3: $r"
done
