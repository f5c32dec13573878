# A/B/C... timing on one box: bash scripts/ab_multi.sh <config> "ENV=a" "ENV=b" ...  (3 rounds, alternating)
cfg=$1; shift
for i in 1 2 3; do
  for v in "$@"; do
    r=$(env $v timeout -s KILL 120 python bench.py --config $cfg --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['clocks']['sm_mhz'])")
    echo "$v $r"
  done
done
