# streamed e2e (submit/wait, 2 slots in flight) vs chunk schedule (dev tool, under gpurun)
for f in ${FIRSTS:-48 16 8}; do for c in ${CAPS:-16 8 4}; do
  [ $f -lt $c ] && continue
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
outs = [batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm) for _ in range(2)]
torch.cuda.synchronize()
K = 10
t0 = time.perf_counter(); prev = None
for k in range(K):
    tk = batched.detect_cim_host_submit(Hh, yh, nvh, 16, sh, prm, out=outs[k % 2])
    if prev is not None: prev.wait()
    prev = tk
prev.wait()
ms = (time.perf_counter() - t0) * 1e3 / K
print(f"first_div={os.environ['ISINGLINK_PIPE_FIRST_DIV']} cap_div={os.environ['ISINGLINK_PIPE_CAP_DIV']}: streamed {ms:.3f} ms/slot")
PY
done; done
