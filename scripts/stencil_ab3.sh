mkdir -p gpurun_out
HPAR_ST_IMPL=1 timeout 600 python -m pytest tests/test_gpu_stencil.py -x -q 2>&1 | tail -2
for i in 1 2; do
for v in "HPAR_ST_IMPL=0 HPAR_ST_DEBUG=4" "HPAR_ST_IMPL=1"; do
  r=$(env HPAR_C6_LDA=32 $v timeout -s KILL 120 python bench.py --config c6 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
  echo "$v $r ms"
done; done
