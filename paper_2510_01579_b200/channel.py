"""Host-side data formats either side of the hot path (mirror of the
reference ``channel.py`` API: channel.py:24-180).

Symbols travel through the CUDA path as *level indices*: one uint8 per real
dimension, ``(re_idx, im_idx)`` per user, into the ascending PAM level list.
This module converts between those indices and complex symbol values, and
provides the reference's alphabet, projection, error-count and synthetic
channel helpers with identical semantics (they are pure functions of their
arguments and seeds, used to build inputs and score outputs).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

QAM_ORDERS = (4, 16, 64, 256)


@dataclass(frozen=True)
class Constellation:
    """Square product alphabet; ``points[i*m + q] = pam[i] + 1j*pam[q]``."""

    order: int
    points: np.ndarray = field(repr=False)
    pam_levels: np.ndarray = field(repr=False)
    spacing: float

    @property
    def bits_per_symbol(self) -> int:
        return int(round(math.log2(self.order)))

    @property
    def bits_per_dim(self) -> int:
        return int(round(math.log2(len(self.pam_levels))))


@dataclass(frozen=True)
class MimoInstance:
    """One detection problem (channel.py:61-85 semantics)."""

    H: np.ndarray
    y: np.ndarray
    constellation: Constellation
    noise_var: float
    truth: np.ndarray | None = None

    def __post_init__(self):
        if self.H.ndim != 2 or self.y.shape != (self.H.shape[0],):
            raise ValueError("channel/observation dimensions are inconsistent")
        if self.truth is not None and self.truth.shape != (self.H.shape[1],):
            raise ValueError("truth length must match the channel column count")
        if self.noise_var < 0:
            raise ValueError("noise_var must be nonnegative")

    @property
    def n_r(self) -> int:
        return self.H.shape[0]

    @property
    def n_t(self) -> int:
        return self.H.shape[1]


def make_qam(order: int) -> Constellation:
    """Unit-average-energy square QAM (channel.py:88-108)."""
    if order not in QAM_ORDERS:
        raise ValueError(f"unsupported QAM order {order}; expected one of {QAM_ORDERS}")
    m = math.isqrt(order)
    scale = math.sqrt(2.0 * (m * m - 1) / 3.0)
    pam = np.arange(-(m - 1), m, 2, dtype=np.float64) / scale
    pts = (pam[:, None] + 1j * pam[None, :]).reshape(-1)
    return Constellation(order=order, points=pts, pam_levels=pam, spacing=float(2.0 / scale))


def level_indices(values: np.ndarray, levels: np.ndarray) -> np.ndarray:
    """Nearest level per real value; exact midpoints go to the lower level."""
    mids = (levels[:-1] + levels[1:]) / 2.0
    return np.searchsorted(mids, values, side="left")


def to_indices(x: np.ndarray, c: Constellation) -> np.ndarray:
    """Complex symbols -> uint8 level indices [..., n, 2] (re, im)."""
    x = np.asarray(x)
    return np.stack([level_indices(x.real, c.pam_levels),
                     level_indices(x.imag, c.pam_levels)], axis=-1).astype(np.uint8)


def from_indices(idx: np.ndarray, c: Constellation) -> np.ndarray:
    """uint8 level indices [..., n, 2] -> complex symbols [..., n]."""
    idx = np.asarray(idx, dtype=np.int64)
    return c.pam_levels[idx[..., 0]] + 1j * c.pam_levels[idx[..., 1]]


def project_to_constellation(x_soft: np.ndarray, c: Constellation) -> np.ndarray:
    """Per-dimension nearest point; idempotent on the alphabet (channel.py:148-157)."""
    return from_indices(to_indices(x_soft, c), c)


def gray_label(idx: np.ndarray) -> np.ndarray:
    idx = np.asarray(idx)
    return idx ^ (idx >> 1)


_POP = np.array([bin(i).count("1") for i in range(256)], dtype=np.int64)


def symbol_errors(x_true: np.ndarray, x_hat: np.ndarray) -> int:
    return int(np.count_nonzero(np.asarray(x_true) != np.asarray(x_hat)))


def bit_errors(x_true: np.ndarray, x_hat: np.ndarray, c: Constellation) -> int:
    """Gray-coded bit errors per PAM dimension (channel.py:172-180)."""
    a = to_indices(x_true, c).astype(np.int64)
    b = to_indices(x_hat, c).astype(np.int64)
    return int(_POP[gray_label(a) ^ gray_label(b)].sum())


def sample_channel(n_r: int, n_t: int, rng_seed: int) -> np.ndarray:
    """i.i.d. CN(0, 1) channel, deterministic in the seed (channel.py:111-118)."""
    if not n_r >= n_t >= 1:
        raise ValueError(f"need n_r >= n_t >= 1, got ({n_r}, {n_t})")
    g = np.random.default_rng(rng_seed)
    re = g.standard_normal((n_r, n_t))
    im = g.standard_normal((n_r, n_t))
    return (re + 1j * im) * np.sqrt(0.5)


def transmit(H: np.ndarray, x: np.ndarray, snr_db: float, rng_seed: int):
    """y = Hx + n with sigma2 = n_t / 10^(snr/10) (channel.py:121-138)."""
    n_r, n_t = H.shape
    if x.shape != (n_t,):
        raise ValueError("transmit vector length must match channel columns")
    sigma2 = float(n_t / (10.0 ** (snr_db / 10.0)))
    g = np.random.default_rng(rng_seed)
    noise = (g.standard_normal(n_r) + 1j * g.standard_normal(n_r)) * math.sqrt(sigma2 / 2.0)
    return H @ x + noise, sigma2
