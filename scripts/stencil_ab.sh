# c6 A/B: row pitch (HPAR_C6_LDA floats) x store policy (HPAR_ST_DEBUG=4: default stores)
mkdir -p gpurun_out
for i in 1 2; do
for v in "HPAR_C6_LDA=4 HPAR_ST_DEBUG=0" "HPAR_C6_LDA=4 HPAR_ST_DEBUG=4" "HPAR_C6_LDA=32 HPAR_ST_DEBUG=0" "HPAR_C6_LDA=32 HPAR_ST_DEBUG=4" "HPAR_C6_LDA=32 HPAR_ST_DEBUG=1"; do
  r=$(env $v timeout -s KILL 120 python bench.py --config c6 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
  echo "$v $r ms"
done; done
