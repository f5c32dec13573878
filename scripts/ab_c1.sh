# C1 A/B of libraries: bash scripts/ab_c1.sh lib1 lib2 ... (3 rounds, 1000-step graphs)
for i in 1 2 3; do for l in "$@"; do
 r=$(HPAR_LIB=$l timeout -s KILL 120 python bench.py --config c1 --steps 1000 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,3), 'us', d['clocks']['sm_mhz'])")
 echo "$l $r"; done; done
