"""Solver configuration: the reference's ``CacParams`` (solver.py:87-124) plus
the B200 arithmetic mode.

``precision`` selects the anneal arithmetic:
  * ``"fp64_exact"`` — FP64 in the reference kernel's evaluation order, no
    FMA contraction: bit-identical to the reference "ext" backend;
  * ``"fp32"`` (default) — FP32 state, coupling product on tensor cores as a
    3-pass f16 hi/lo split (hi*hi + lo*hi + hi*lo, FP32 accumulate;
    FP32-accurate); the throughput mode;
  * ``"tf32"`` — single-pass f16 coupling product (11-bit significand, like
    TF32; fastest, least accurate);
  * ``"mixed"`` — ``"fp32"`` for the first 16 steps, then a 2-pass product
    (G split to FP32 accuracy, the state rounded to f16): the early steps,
    where the chaotic dynamics amplify rounding, keep FP32 accuracy.

``rng`` selects the initial states: ``"numpy"`` (default) replays the
reference's numpy streams bit for bit; ``"philox"`` draws them from a
counter-based Philox4x32-10 keyed by the same per-problem seeds (cheaper,
statistically equivalent; with ``precision="fp64_exact"`` it gives the FP64
reference dynamics on the same states).

Reference ``CacParams`` objects (no ``precision`` attribute) are accepted
everywhere and run in ``DEFAULT_PRECISION``.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

from ._lib import PREC, RNG, CacParamsC

DEFAULT_PRECISION = os.environ.get("ISINGLINK_B200_PRECISION", "fp32")
if DEFAULT_PRECISION not in PREC:
    raise ValueError(f"ISINGLINK_B200_PRECISION must be one of {sorted(PREC)}, "
                     f"not {DEFAULT_PRECISION!r}")


@dataclass(frozen=True)
class CacParams:
    p: float = 1.5
    a: float = 0.5
    zeta: float = 1.0
    eps: float | None = None
    dt: float = 0.02
    f_mvm: int = 2
    n_steps: int = 128
    n_anneals: int = 32
    diverge_threshold: float = 10.0
    e_floor: float = 1e-6
    init_amplitude: float = 0.1
    precision: str = DEFAULT_PRECISION
    rng: str = "numpy"

    def validate(self) -> None:
        """Same rules and messages as the reference (solver.py:109-124)."""
        if not self.dt > 0:
            raise ValueError("dt must be positive")
        if self.f_mvm < 1 or self.n_steps < 1 or self.n_anneals < 1:
            raise ValueError("f_mvm, n_steps and n_anneals must be >= 1")
        if not self.e_floor > 0:
            raise ValueError("e_floor must be positive")
        if self.init_amplitude <= 0:
            raise ValueError("init_amplitude must be positive")
        if self.eps is not None and not self.eps > 0:
            raise ValueError("eps must be positive or None for auto scaling")
        floor = math.sqrt(max(self.a, self.p - 1.0, 0.0))
        if not self.diverge_threshold > floor:
            raise ValueError(
                f"diverge_threshold must exceed sqrt(max(a, p - 1)) = {floor:.3g}")
        if self.precision not in PREC:
            raise ValueError(f"precision must be one of {sorted(PREC)}")
        if self.rng not in RNG:
            raise ValueError(f"rng must be one of {sorted(RNG)}")


def precision_of(params) -> str:
    return getattr(params, "precision", None) or DEFAULT_PRECISION


def to_c(params, precision: str | None = None) -> CacParamsC:
    """Validated il_cac_params from any CacParams-like object."""
    params.validate()
    prec = precision or precision_of(params)
    if prec not in PREC:
        raise ValueError(f"precision must be one of {sorted(PREC)}")
    eps = params.eps
    return CacParamsC(p=float(params.p), a=float(params.a), zeta=float(params.zeta),
                      eps=-1.0 if eps is None else float(eps), dt=float(params.dt),
                      f_mvm=int(params.f_mvm), n_steps=int(params.n_steps),
                      n_anneals=int(params.n_anneals), precision=PREC[prec],
                      diverge_threshold=float(params.diverge_threshold),
                      e_floor=float(params.e_floor),
                      init_amplitude=float(params.init_amplitude),
                      rng=RNG[getattr(params, "rng", "numpy") or "numpy"], reserved=0)
