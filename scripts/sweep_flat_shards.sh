# per-rank kernel time of the strong-scaled total configs (rank 0's shard on one GPU)
for G in 1 2 4 8; do
  for C in -1 0; do
    r=$(timeout -s KILL 300 python bench.py --config c5 --shard $G --clusters $C --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['config']['geometry'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")
    echo "c5 G=$G C=$C $r"
  done
  r=$(timeout -s KILL 300 python bench.py --config c4 --shard $G --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['config']['geometry'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")
  echo "c4 G=$G $r"
done
