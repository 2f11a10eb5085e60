# e2e ramp sweep (dev tool, run under gpurun): host pipeline time per slot
for f in ${FIRSTS:-24 48 96}; do for c in ${CAPS:-8 12 16 24}; do
  ISINGLINK_PIPE_FIRST_DIV=$f ISINGLINK_PIPE_CAP_DIV=$c python - <<'PY' 2>&1 | grep -v Warn
import os, sys, time, torch
sys.path.insert(0, '.')
from paper_2510_01579_b200 import batched
from paper_2510_01579_b200.params import CacParams
from tools.parity_scale import batch
P = 45864
H, y, nv, seeds, _ = batch(16, 16, 20.0, P, 7)
Hh, yh, nvh, sh = (t.cpu().pin_memory() for t in (H, y, nv, seeds))
prm = CacParams()
batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm); torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    t0 = time.perf_counter(); batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm); torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(f"first_div={os.environ['ISINGLINK_PIPE_FIRST_DIV']} cap_div={os.environ['ISINGLINK_PIPE_CAP_DIV']}: {best*1e3:.3f} ms")
PY
done; done
