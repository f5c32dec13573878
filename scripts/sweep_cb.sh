# C3 CTA chunk (blocks per CTA claim) vs shard size
for G in 1 8; do
  for CB in 1 2 4 8; do
    r=$(HPAR_SEG_CB=$CB timeout -s KILL 120 python bench.py --config c3 --shard $G --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3))")
    echo "c3 G=$G CB=$CB $r"
  done
done
