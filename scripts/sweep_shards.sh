# per-rank kernel time of the strong-scaled keyed configs at G = 2..64 (rank 0's shard on one GPU; rotating inputs)
mkdir -p gpurun_out
for G in 1 2 4 8 16 32 64; do
  for C in -1 296 444; do
    r=$(timeout -s KILL 120 python bench.py --config c2 --shard $G --clusters $C --steps 200 --no-cpu-baseline --no-e2e $XARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3), d['config']['geometry'], d['config']['l2'])")
    echo "c2 G=$G C=$C $r"
  done
done
for G in 1 2 4 8; do
  r=$(timeout -s KILL 120 python bench.py --config c3 --shard $G --steps 200 --no-cpu-baseline --no-e2e $XARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3), d['config']['geometry'], d['config']['l2'])")
  echo "c3 G=$G $r"
done
python - <<'PY'
import torch
L2 = 126 * 2**20
for mb in (1074, 537, 268, 134, 67, 16):
    n = mb * 2**20 // 4
    k = max(1, -(-3 * L2 // (n * 4)) + 1)
    xs = [torch.empty(n, device="cuda") for _ in range(k)]
    ys = [torch.empty(n // 4096, device="cuda") for _ in range(k)]
    for i in range(5):
        torch.sum(xs[i % k].view(-1, 4096), dim=1, out=ys[i % k])
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for i, (a, b) in enumerate(ev):
        a.record(); torch.sum(xs[i % k].view(-1, 4096), dim=1, out=ys[i % k]); b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)[25]
    print(f"torch row-sum {mb} MB ({k} copies): {t*1e3:.1f} us = {mb * 2**20 / (t * 1e-3) / 1e9:.0f} GB/s")
PY
