# C3: split threshold sweep (rows longer than HPAR_SEG_LONG go to the segment queue); run under gpurun
mkdir -p gpurun_out
for T in ${SWEEP:-4096 2048 1024 512 256 4096}; do
  r=$(HPAR_SEG_LONG=$T timeout -s KILL 120 python bench.py --config c3 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))")
  echo "HPAR_SEG_LONG=$T $r"
done
