# C3 split threshold (rows > LONG go to the segment queue) vs shard size
for G in 1 2 4 8; do
  for LG in 512 1024 2048 4096; do
    r=$(HPAR_SEG_LONG=$LG timeout -s KILL 120 python bench.py --config c3 --shard $G --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3))")
    echo "c3 G=$G LONG=$LG $r"
  done
done
