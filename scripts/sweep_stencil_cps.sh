# stencil: CTAs per SM x ring stages x tile rows (same box).  HPAR_ST_CPS overrides the occupancy-derived grid.
mkdir -p gpurun_out
run() { r=$(env "$@" timeout 120 python bench.py --config c6 --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))"); echo "$* $r"; }
for rep in 1 2; do
run HPAR_ST_CPS=3 HPAR_ST_NST=2
run HPAR_ST_CPS=1 HPAR_ST_NST=4
run HPAR_ST_CPS=1 HPAR_ST_NST=5
run HPAR_ST_CPS=1 HPAR_ST_NST=2 HPAR_ST_TY=128
run HPAR_ST_CPS=1 HPAR_ST_NST=3 HPAR_ST_TY=128
done
