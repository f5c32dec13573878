# same-box A/B of experiment library builds: bash scripts/ab_lib.sh <config> <lib1> <lib2> ...  ("" = default build)
cfg=$1; shift
for i in 1 2; do for L in "$@"; do
  r=$(HPAR_LIB=$L timeout -s KILL 120 python bench.py --config $cfg --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))")
  echo "${L:-default} $r"
done; done
