#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for c in 4 8 16 32; do
  CONV_HOST_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 3 --soak 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks $c e2e', d['e2e'])"
done
python - <<'PY'
import torch, time
a = torch.empty(69468160 // 4, dtype=torch.float32).pin_memory(); d = torch.empty_like(a, device='cuda')
b = torch.empty(51380224 // 4, dtype=torch.float32).pin_memory(); e = torch.empty_like(b, device='cuda')
for _ in range(3): d.copy_(a, non_blocking=True); b.copy_(e, non_blocking=True)
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); d.copy_(a, non_blocking=True); t1.record(); torch.cuda.synchronize(); print('H2D GB/s', 69468160 / t0.elapsed_time(t1) / 1e6)
t0.record(); b.copy_(e, non_blocking=True); t1.record(); torch.cuda.synchronize(); print('D2H GB/s', 51380224 / t0.elapsed_time(t1) / 1e6)
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(a, non_blocking=True)
with torch.cuda.stream(s2): b.copy_(e, non_blocking=True)
torch.cuda.synchronize(); print('both concurrent ms', (time.perf_counter() - t) * 1e3)
PY
