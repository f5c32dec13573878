# c6 bounds: the same buffer copied by torch (read+write, no ghosts), and the
# stencil with timing knobs (HPAR_ST_DEBUG bit 1: box without ghost ring, bit 2: no stores)
mkdir -p gpurun_out
python - <<'PY'
import torch
n = 16386 * 16388
a = torch.rand(n, device="cuda"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize(); e0.record()
for _ in range(100): b.copy_(a)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 100
print(f"torch copy of the c6 buffer: {ms:.4f} ms = {2 * n * 4 / ms / 1e6:.0f} GB/s")
PY
for d in 0 1 2 3 0; do
  r=$(HPAR_ST_DEBUG=$d timeout -s KILL 120 python bench.py --config c6 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
  echo "HPAR_ST_DEBUG=$d $r ms"
done
