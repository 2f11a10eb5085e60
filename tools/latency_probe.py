"""Per-call latency of the reference-shaped per-instance API and the kernel
plugin (dev tool): the drop-in granularity (one RE per call)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import isinglink_oracle as orc  # noqa: E402  (instance generator only)
from paper_2510_01579_b200 import _kernel_cuda, api  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402

H, y, s2, _ = orc.uplink_instance(1, 20.0, 0, 0, 16, 16, 16)
inst = api.MimoInstance(H=H, y=y, constellation=api.make_qam(16), noise_var=s2)
for prec in ("fp32", "fp64_exact"):
    prm = CacParams(precision=prec)
    api.detect_cim(inst, prm, 7)
    t0 = time.perf_counter()
    for _ in range(50):
        api.detect_cim(inst, prm, 7)
    print(f"api.detect_cim 16x16 ({prec}): {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms/call")
si = api.build_ising(inst, api.detect_mmse(inst).x_hard)
x0 = np.random.default_rng(0).uniform(-0.1, 0.1, (32, si.spin_count))
args = (si.G, si.g_diag, si.b, x0, 0.02, 1.5, 0.5, 1.0, si.eps_scale, 1e-6, 2, 128, 10.0)
_kernel_cuda.run_anneals(*args)
t0 = time.perf_counter()
for _ in range(50):
    _kernel_cuda.run_anneals(*args)
print(f"_kernel_cuda.run_anneals 16x16 x32: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms/call")
# device-tensor form: kernel time alone (CUDA events), no host copies
import torch  # noqa: E402
from paper_2510_01579_b200 import batched, _lib  # noqa: E402
Gd, gd, bd, xd = (torch.as_tensor(a, device="cuda") for a in (si.G, si.g_diag, si.b, x0))
batched.run_anneals(Gd, gd, bd, xd, *args[4:])
torch.cuda.synchronize()
_lib.profile_begin()
for _ in range(20):
    batched.run_anneals(Gd, gd, bd, xd, *args[4:])
pr = _lib.profile_end()
print(f"k_anneal_exact alone (1 RE x 32 anneals): {pr['anneal'][0] / 20:.3f} ms")
