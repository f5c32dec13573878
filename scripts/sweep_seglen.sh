# C3 long-row segment length vs shard size (rank 0's shard on one GPU)
for G in 1 2 4 8; do
  for L in 4096 8192 16384; do
    r=$(HPAR_SEG_LEN_RT=$L timeout -s KILL 120 python bench.py --config c3 --shard $G --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3))")
    echo "c3 G=$G seg=$L $r"
  done
done
