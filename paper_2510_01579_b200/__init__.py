"""isinglink-b200: B200-native hot path of MMGaP (arXiv 2510.01579).

Per-resource-element ML-MIMO uplink detection and vector-perturbation
downlink precoding, each cast as a structured Ising problem and solved by
many-replica CIM-CAC annealing, on hand-written sm_100a CUDA kernels behind
a C ABI (include/isinglink_b200.h).

Entry points:
  * ``_kernel_cuda``  — drop-in ``run_anneals`` plugin for the reference package
    (``install.install(isinglink)`` registers it as backend "cuda");
  * ``api``           — the reference's per-instance API (detect_cim, precode_vpp,
    build_ising, solve_batch, ...) running on the GPU;
  * ``batched``       — whole-slot device API (detect_cim_batch, precode_vpp_batch, ...);
  * ``shard``         — subcarrier sharding over GPUs with an NCCL gather of bits;
  * ``harness``       — the reference's sweeps / heatmap / bench report on the GPU.
"""

from . import _lib
from .channel import (Constellation, MimoInstance, bit_errors, from_indices, make_qam,
                      project_to_constellation, sample_channel, symbol_errors, to_indices,
                      transmit)
from .params import CacParams

__version__ = "0.1.0"

__all__ = [
    "CacParams", "Constellation", "MimoInstance", "bit_errors", "from_indices", "make_qam",
    "project_to_constellation", "sample_channel", "symbol_errors", "to_indices", "transmit",
]


def library_path() -> str:
    return _lib.LIB_PATH
