"""Streamed slots must not grow device memory: the host pipeline reserves the
pool's working set at first use and every later call is served from it."""
import numpy as np
import pytest
import torch

from conftest import load_golden


@pytest.mark.gpu
def test_streamed_slots_keep_memory_flat(built_lib):
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("d16x16_16qam_20db.npz")
    reps = 120  # ~9k REs: the two-chunk and ramp paths both run
    H = torch.from_numpy(np.concatenate([d["H"]] * reps)).pin_memory()
    y = torch.from_numpy(np.concatenate([d["y"]] * reps)).pin_memory()
    s2 = torch.from_numpy(np.concatenate([d["noise_var"]] * reps)).pin_memory()
    seed = np.concatenate([d["seed"]] * reps)
    prm = CacParams(precision="fp32")

    def run(n):
        prev = None
        for k in range(n):
            m = len(seed) - (k % 3) * 1000
            tk = batched.detect_cim_host_submit(H[:m], y[:m], s2[:m], int(d["order"]), seed[:m], prm)
            if prev is not None:
                prev.wait()
            prev = tk
        prev.wait()

    run(6)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    run(30)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] >= free0 - (64 << 20)
