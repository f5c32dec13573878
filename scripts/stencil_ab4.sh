mkdir -p gpurun_out
for v in "1 4 32" "2 4 32" "4 2 32" "4 1 32" "1 8 32" "1 8 64"; do set -- $v
  HPAR_ST_IMPL=1 HPAR_ST_V=$1 HPAR_ST_PF=$2 HPAR_ST_RB=$3 timeout 600 python -m pytest tests/test_gpu_stencil.py -x -q 2>&1 | tail -1
done
for i in 1 2; do
for v in "HPAR_ST_IMPL=0 HPAR_ST_DEBUG=4" "HPAR_ST_IMPL=1 HPAR_ST_V=1 HPAR_ST_PF=4" "HPAR_ST_IMPL=1 HPAR_ST_V=2 HPAR_ST_PF=4" "HPAR_ST_IMPL=1 HPAR_ST_V=4 HPAR_ST_PF=2" "HPAR_ST_IMPL=1 HPAR_ST_V=4 HPAR_ST_PF=1" "HPAR_ST_IMPL=1 HPAR_ST_V=1 HPAR_ST_PF=8" "HPAR_ST_IMPL=1 HPAR_ST_V=1 HPAR_ST_PF=8 HPAR_ST_RB=64"; do
  r=$(env HPAR_C6_LDA=32 $v timeout -s KILL 120 python bench.py --config c6 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
  echo "$v $r ms"
done; done
