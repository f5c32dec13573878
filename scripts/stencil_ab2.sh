mkdir -p gpurun_out
for v in "HPAR_ST_TY=64 HPAR_ST_NST=2" "HPAR_ST_TY=32 HPAR_ST_NST=2" "HPAR_ST_TY=32 HPAR_ST_NST=3" "HPAR_ST_TY=32 HPAR_ST_NST=4" "HPAR_ST_TY=16 HPAR_ST_NST=4" "HPAR_ST_TY=64 HPAR_ST_NST=2 HPAR_ST_L2P=0"; do
  r=$(env HPAR_C6_LDA=32 HPAR_ST_DEBUG=4 $v timeout -s KILL 120 python bench.py --config c6 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
  echo "$v $r ms"
done
for T in 4096 8192 16384 65536; do
  r=$(HPAR_SEG_LONG=$T timeout -s KILL 120 python bench.py --config c3 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))")
  echo "HPAR_SEG_LONG=$T $r"
done
