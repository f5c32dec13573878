# A/B timing on one box of two env settings for a config: bash scripts/ab_env.sh c6 "HPAR_ST_NW=8" "HPAR_ST_NW=16"
cfg=$1; A=$2; B=$3
for i in 1 2 3; do
  for v in "$A" "$B"; do
    r=$(env $v timeout -s KILL 120 python bench.py --config $cfg --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
    echo "$v $r"
  done
done
