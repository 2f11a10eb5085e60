"""Batched device API: whole slots of resource elements per call.

All functions take torch CUDA tensors (or numpy arrays, which are copied to
the current device) and enqueue on the current torch stream; outputs are
torch CUDA tensors.  Shapes use P = number of problems (resource elements):

  H  complex128 [P, n_r, n_t]     y  complex128 [P, n_r]     noise_var f64 [P]
  x_idx  uint8 [P, n_t, 2]        level indices (re, im) of the decided symbols

These are the B200-native entry points the throughput benchmark drives; the
reference-shaped per-instance API in ``api.py`` is built on them.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .params import CacParams, to_c


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dev(x, dtype: torch.dtype) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x
    else:
        arr = np.ascontiguousarray(x)
        t = torch.from_numpy(arr)
    if t.device.type != "cuda":
        t = t.to("cuda", non_blocking=False)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def _seeds(seeds, P: int) -> torch.Tensor:
    if isinstance(seeds, torch.Tensor):
        s = seeds
    else:
        s = torch.from_numpy(np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(-1)))
    s = s.to("cuda").contiguous()
    if s.dtype not in (torch.uint64, torch.int64):
        raise TypeError("seeds must be uint64 (or int64 bit patterns)")
    if s.numel() != P:
        raise ValueError(f"expected {P} seeds, got {s.numel()}")
    return s


@dataclass
class DetectBatch:
    x_idx: torch.Tensor          # uint8 [P, n_t, 2]
    energy: torch.Tensor         # f64 [P]   ||y - H x||^2
    source: torch.Tensor         # int8 [P]  0 guess (MMSE), 1 anneal, -1 failed
    anneal_index: torch.Tensor   # int32 [P] winning anneal or -1
    diverged: torch.Tensor       # int32 [P] diverged anneal count
    bits: torch.Tensor | None = None  # uint8 [P, n_t, 2 bpd] Gray bits (host entries, bits=True)


def detect_cim_batch(H, y, noise_var, order: int, seeds, params=None,
                     precision: str | None = None) -> DetectBatch:
    """P x ``detect_cim`` (detector.py:57-82); seeds[p] is detect_cim's ``seed``."""
    params = params or CacParams()
    prm = to_c(params, precision)
    Hd = _dev(H, torch.complex128)
    if Hd.dim() != 3:
        raise ValueError("H must be [P, n_r, n_t]")
    P, n_r, n_t = Hd.shape
    yd = _dev(y, torch.complex128)
    sd = _dev(noise_var, torch.float64)
    if yd.shape != (P, n_r) or sd.shape != (P,):
        raise ValueError("y must be [P, n_r] and noise_var [P]")
    seed_t = _seeds(seeds, P)
    dev = Hd.device
    out = DetectBatch(
        x_idx=torch.empty((P, n_t, 2), dtype=torch.uint8, device=dev),
        energy=torch.empty(P, dtype=torch.float64, device=dev),
        source=torch.empty(P, dtype=torch.int8, device=dev),
        anneal_index=torch.empty(P, dtype=torch.int32, device=dev),
        diverged=torch.empty(P, dtype=torch.int32, device=dev),
    )
    _lib.call("il_detect_cim_batch", Hd.data_ptr(), yd.data_ptr(), sd.data_ptr(), P, n_r, n_t,
              int(order), seed_t.data_ptr(), prm, out.x_idx.data_ptr(), out.energy.data_ptr(),
              out.source.data_ptr(), out.anneal_index.data_ptr(), out.diverged.data_ptr(),
              _stream())
    return out


def _host(x, dtype: torch.dtype, shape) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    if t.device.type != "cpu":
        raise ValueError("detect_cim_host takes host (CPU) buffers")
    if t.dtype != dtype:
        t = t.to(dtype)
    t = t.contiguous()
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


class HostTicket:
    """A slot submitted with ``detect_cim_host_submit``: ``wait()`` returns
    its DetectBatch once the outputs are in host memory.  Holds the input
    and output buffers alive until then."""

    def __init__(self, handle, out, keep):
        self._handle, self.out, self._keep = handle, out, keep

    def wait(self) -> DetectBatch:
        if self._keep is not None:
            h, self._handle = self._handle, None
            self._keep_alive, self._keep = self._keep, None
            _lib.call("il_pipeline_wait", h)
            self._keep_alive = None
        return self.out

    def __del__(self):  # never release buffers a copy may still be using
        try:
            self.wait()
        except Exception:
            pass


def _host_seeds(seeds, P: int) -> torch.Tensor:
    """Seeds as a contiguous host tensor of P 64-bit words (the C pipelines
    copy 8 P bytes from it, so a narrower dtype is rejected, not read past)."""
    st = seeds if isinstance(seeds, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(-1)))
    if st.dtype not in (torch.uint64, torch.int64):
        raise TypeError("seeds must be uint64 (or int64 bit patterns)")
    return _host(st, st.dtype, (P,))


def detect_cim_host_submit(H, y, noise_var, order: int, seeds, params=None,
                           precision: str | None = None, n_chunks: int = 0,
                           out=None, bits: bool = False) -> HostTicket:
    """Streaming form of ``detect_cim_host`` (il_detect_cim_host_submit):
    enqueue the slot and return a ticket at once.  Slots submitted back to
    back overlap: the next slot's copies and first chunks run under this
    slot's tail.  bits=True also returns the Gray bits of the decisions,
    demapped on the device inside the pipeline (il_detect_cim_bits_host_submit)."""
    params = params or CacParams()
    prm = to_c(params, precision)
    Ht = H if isinstance(H, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(H))
    if Ht.dim() != 3:
        raise ValueError("H must be [P, n_r, n_t]")
    P, n_r, n_t = Ht.shape
    Hh = _host(Ht, torch.complex128, (P, n_r, n_t))
    yh = _host(y, torch.complex128, (P, n_r))
    sh = _host(noise_var, torch.float64, (P,))
    st = _host_seeds(seeds, P)
    pin = torch.cuda.is_available()
    if out is None:
        out = DetectBatch(x_idx=torch.empty((P, n_t, 2), dtype=torch.uint8, pin_memory=pin),
                          energy=torch.empty(P, dtype=torch.float64, pin_memory=pin),
                          source=torch.empty(P, dtype=torch.int8, pin_memory=pin),
                          anneal_index=torch.empty(P, dtype=torch.int32, pin_memory=pin),
                          diverged=torch.empty(P, dtype=torch.int32, pin_memory=pin))
    handle = ctypes.c_void_p()
    if bits:
        m = int(round(math.sqrt(int(order))))
        bpd = max(1, (m - 1).bit_length())
        if out.bits is None or tuple(out.bits.shape) != (P, n_t, 2 * bpd):
            out.bits = torch.empty((P, n_t, 2 * bpd), dtype=torch.uint8, pin_memory=pin)
        _lib.call("il_detect_cim_bits_host_submit", Hh.data_ptr(), yh.data_ptr(), sh.data_ptr(),
                  P, n_r, n_t, int(order), st.data_ptr(), prm, out.bits.data_ptr(),
                  out.x_idx.data_ptr(), out.energy.data_ptr(), out.source.data_ptr(),
                  out.anneal_index.data_ptr(), out.diverged.data_ptr(), int(n_chunks),
                  ctypes.byref(handle))
    else:
        _lib.call("il_detect_cim_host_submit", Hh.data_ptr(), yh.data_ptr(), sh.data_ptr(), P,
                  n_r, n_t, int(order), st.data_ptr(), prm, out.x_idx.data_ptr(),
                  out.energy.data_ptr(), out.source.data_ptr(), out.anneal_index.data_ptr(),
                  out.diverged.data_ptr(), int(n_chunks), ctypes.byref(handle))
    return HostTicket(handle, out, (Hh, yh, sh, st))


def detect_cim_host(H, y, noise_var, order: int, seeds, params=None,
                    precision: str | None = None, n_chunks: int = 0, out=None,
                    bits: bool = False) -> DetectBatch:
    """P x ``detect_cim`` from HOST buffers to HOST buffers.

    The slot is streamed through the GPU in chunks with H2D copy, detection
    and D2H copy overlapped (il_detect_cim_host).  Pass pinned CPU tensors
    (``tensor.pin_memory()``) for the overlap; ``out`` may hold preallocated
    (pinned) output tensors in DetectBatch layout."""
    return detect_cim_host_submit(H, y, noise_var, order, seeds, params, precision, n_chunks,
                                  out, bits).wait()


@dataclass
class PrecodeBatch:
    x: torch.Tensor              # complex128 [P, n_ant] power-normalised transmit vector
    v: torch.Tensor              # complex128 [P, n_u] perturbation (even Gaussian integers)
    unnormalized_power: torch.Tensor  # f64 [P]
    diverged: torch.Tensor       # int32 [P]


def precode_vpp_batch(H, u, power: float, tau: float, seeds, params=None, n_stages: int = 1,
                      precision: str | None = None) -> PrecodeBatch:
    """P x ``precode_vpp`` (precoder.py:93-146).  H [P, n_u, n_ant], u [P, n_u]."""
    params = params or CacParams()
    prm = to_c(params, precision)
    Hd = _dev(H, torch.complex128)
    P, n_u, n_ant = Hd.shape
    ud = _dev(u, torch.complex128)
    if ud.shape != (P, n_u):
        raise ValueError("u must be [P, n_u]")
    seed_t = _seeds(seeds, P)
    dev = Hd.device
    out = PrecodeBatch(
        x=torch.empty((P, n_ant), dtype=torch.complex128, device=dev),
        v=torch.empty((P, n_u), dtype=torch.complex128, device=dev),
        unnormalized_power=torch.empty(P, dtype=torch.float64, device=dev),
        diverged=torch.empty(P, dtype=torch.int32, device=dev),
    )
    _lib.call("il_precode_vpp_batch", Hd.data_ptr(), ud.data_ptr(), P, n_u, n_ant, float(power),
              float(tau), int(n_stages), seed_t.data_ptr(), prm, out.x.data_ptr(),
              out.v.data_ptr(), out.unnormalized_power.data_ptr(), out.diverged.data_ptr(),
              _stream())
    return out


def precode_vpp_host(H, u, power: float, tau: float, seeds, params=None, n_stages: int = 1,
                     precision: str | None = None, n_chunks: int = 0) -> PrecodeBatch:
    """P x ``precode_vpp`` from HOST buffers to HOST buffers, streamed through
    the GPU in chunks with copies overlapped (il_precode_vpp_host)."""
    params = params or CacParams()
    prm = to_c(params, precision)
    Ht = H if isinstance(H, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(H))
    if Ht.dim() != 3:
        raise ValueError("H must be [P, n_u, n_ant]")
    P, n_u, n_ant = Ht.shape
    Hh = _host(Ht, torch.complex128, (P, n_u, n_ant))
    uh = _host(u, torch.complex128, (P, n_u))
    st = _host_seeds(seeds, P)
    pin = torch.cuda.is_available()
    out = PrecodeBatch(x=torch.empty((P, n_ant), dtype=torch.complex128, pin_memory=pin),
                       v=torch.empty((P, n_u), dtype=torch.complex128, pin_memory=pin),
                       unnormalized_power=torch.empty(P, dtype=torch.float64, pin_memory=pin),
                       diverged=torch.empty(P, dtype=torch.int32, pin_memory=pin))
    _lib.call("il_precode_vpp_host", Hh.data_ptr(), uh.data_ptr(), P, n_u, n_ant, float(power),
              float(tau), int(n_stages), st.data_ptr(), prm, out.x.data_ptr(), out.v.data_ptr(),
              out.unnormalized_power.data_ptr(), out.diverged.data_ptr(), int(n_chunks))
    return out


def mmse_batch(H, y, noise_var, order: int):
    """P x ``detect_mmse`` (linear.py:55-75) -> (x_idx, energy, status)."""
    Hd = _dev(H, torch.complex128)
    P, n_r, n_t = Hd.shape
    yd = _dev(y, torch.complex128)
    sd = _dev(noise_var, torch.float64)
    x_idx = torch.empty((P, n_t, 2), dtype=torch.uint8, device=Hd.device)
    energy = torch.empty(P, dtype=torch.float64, device=Hd.device)
    status = torch.empty(P, dtype=torch.int8, device=Hd.device)
    _lib.call("il_mmse_batch", Hd.data_ptr(), yd.data_ptr(), sd.data_ptr(), P, n_r, n_t,
              int(order), x_idx.data_ptr(), energy.data_ptr(), status.data_ptr(), _stream())
    return x_idx, energy, status


def residual_batch(H, y, x) -> torch.Tensor:
    """||y - H x||^2 per problem (linear.py:44-47), x complex [P, n_t]."""
    Hd = _dev(H, torch.complex128)
    P, n_r, n_t = Hd.shape
    yd = _dev(y, torch.complex128)
    xd = _dev(x, torch.complex128)
    out = torch.empty(P, dtype=torch.float64, device=Hd.device)
    _lib.call("il_residual_batch", Hd.data_ptr(), yd.data_ptr(), xd.data_ptr(), P, n_r, n_t,
              out.data_ptr(), _stream())
    return out


def ml_batch(H, y, order: int):
    """P x ``detect_ml`` (linear.py:109-144) -> (x_idx, energy)."""
    Hd = _dev(H, torch.complex128)
    P, n_r, n_t = Hd.shape
    yd = _dev(y, torch.complex128)
    x_idx = torch.empty((P, n_t, 2), dtype=torch.uint8, device=Hd.device)
    energy = torch.empty(P, dtype=torch.float64, device=Hd.device)
    _lib.call("il_ml_batch", Hd.data_ptr(), yd.data_ptr(), P, n_r, n_t, int(order),
              x_idx.data_ptr(), energy.data_ptr(), _stream())
    return x_idx, energy


def ml_llr_batch(H, y, order: int, noise_var=None) -> torch.Tensor:
    """Max-log bit LLRs by exhaustive search -> [P, n_t, 2 * bits_per_dim]
    (bit order of ``gray_demap``; positive favours bit 0).  No reference
    counterpart: soft output is a non-goal of the reference."""
    Hd = _dev(H, torch.complex128)
    P, n_r, n_t = Hd.shape
    yd = _dev(y, torch.complex128)
    m = int(round(math.sqrt(order)))
    bpd = max(1, int(round(math.log2(m))))
    nv = None if noise_var is None else _dev(torch.as_tensor(noise_var, dtype=torch.float64)
                                              .reshape(-1).expand(P).contiguous(), torch.float64)
    llr = torch.empty((P, n_t, 2 * bpd), dtype=torch.float64, device=Hd.device)
    _lib.call("il_ml_llr_batch", Hd.data_ptr(), yd.data_ptr(), 0 if nv is None else nv.data_ptr(),
              P, n_r, n_t, int(order), llr.data_ptr(), _stream())
    return llr


def integrate_batch(G, g_diag, b, eps, seeds, params=None) -> dict:
    """P x ``integrate_anneal`` (solver.py:217-235), FP64-exact: problem p
    starts from default_rng(seeds[p]) with coupling eps[p]."""
    params = params or CacParams()
    prm = to_c(params, "fp64_exact")
    Gd = _dev(G, torch.float64)
    P, N, _ = Gd.shape
    gd = _dev(g_diag, torch.float64)
    bd = _dev(b, torch.float64)
    ed = _dev(eps, torch.float64).reshape(P)
    sd = _seeds(seeds, P)
    dev = Gd.device
    out = dict(spins=torch.empty((P, 2 * N + 1), dtype=torch.int8, device=dev),
               diverged=torch.empty(P, dtype=torch.uint8, device=dev),
               steps=torch.empty(P, dtype=torch.int64, device=dev),
               mvms=torch.empty(P, dtype=torch.int64, device=dev),
               energy=torch.empty(P, dtype=torch.float64, device=dev))
    _lib.call("il_integrate_batch", Gd.data_ptr(), gd.data_ptr(), bd.data_ptr(), ed.data_ptr(),
              sd.data_ptr(), P, N, prm, out["spins"].data_ptr(), out["diverged"].data_ptr(),
              out["steps"].data_ptr(), out["mvms"].data_ptr(), out["energy"].data_ptr(),
              _stream())
    return out


def mmse_sic_batch(H, y, noise_var, order: int):
    """P x ``detect_mmse_sic`` (linear.py:78-106) -> (x_idx, energy, status)."""
    Hd = _dev(H, torch.complex128)
    P, n_r, n_t = Hd.shape
    yd = _dev(y, torch.complex128)
    sd = _dev(noise_var, torch.float64)
    x_idx = torch.empty((P, n_t, 2), dtype=torch.uint8, device=Hd.device)
    energy = torch.empty(P, dtype=torch.float64, device=Hd.device)
    status = torch.empty(P, dtype=torch.int8, device=Hd.device)
    _lib.call("il_mmse_sic_batch", Hd.data_ptr(), yd.data_ptr(), sd.data_ptr(), P, n_r, n_t,
              int(order), x_idx.data_ptr(), energy.data_ptr(), status.data_ptr(), _stream())
    return x_idx, energy, status


CHAIN_CODES = {"mmse": 0, "mmse_sic": 1}


def detect_cim_multi_batch(H, y, noise_var, order: int, seeds, params=None, n_stages: int = 1,
                           chains=("mmse", "mmse_sic"),
                           precision: str | None = None) -> DetectBatch:
    """P x ``detect_cim_multi`` (MMGaP-E, detector.py:85-134).

    ``source``: 0 mmse, 1 anneal, 2 mmse_sic, -1 failed baseline."""
    params = params or CacParams()
    prm = to_c(params, precision)
    if n_stages < 1:
        raise ValueError("n_stages must be >= 1")
    codes = np.array([CHAIN_CODES[c] for c in chains], dtype=np.int32)
    Hd = _dev(H, torch.complex128)
    if Hd.dim() != 3:
        raise ValueError("H must be [P, n_r, n_t]")
    P, n_r, n_t = Hd.shape
    yd = _dev(y, torch.complex128)
    sd = _dev(noise_var, torch.float64)
    seed_t = _seeds(seeds, P)
    dev = Hd.device
    out = DetectBatch(
        x_idx=torch.empty((P, n_t, 2), dtype=torch.uint8, device=dev),
        energy=torch.empty(P, dtype=torch.float64, device=dev),
        source=torch.empty(P, dtype=torch.int8, device=dev),
        anneal_index=torch.empty(P, dtype=torch.int32, device=dev),
        diverged=torch.empty(P, dtype=torch.int32, device=dev),
    )
    _lib.call("il_detect_cim_multi_batch", Hd.data_ptr(), yd.data_ptr(), sd.data_ptr(), P, n_r,
              n_t, int(order), seed_t.data_ptr(), prm, int(n_stages), codes.ctypes.data,
              len(codes), out.x_idx.data_ptr(), out.energy.data_ptr(), out.source.data_ptr(),
              out.anneal_index.data_ptr(), out.diverged.data_ptr(), _stream())
    return out


def build_ising_batch(H, y, guess_idx, order: int) -> dict:
    """P x ``build_ising`` (transform.py:108-140) around level-index guesses.

    order > 0: unit-energy QAM; order < 0: VPP lattice of reach -order."""
    Hd = _dev(H, torch.complex128)
    P, n_r, n_t = Hd.shape
    yd = _dev(y, torch.complex128)
    gd = _dev(guess_idx, torch.uint8)
    N = 2 * n_t
    dev = Hd.device
    out = dict(G=torch.empty((P, N, N), dtype=torch.float64, device=dev),
               g_diag=torch.empty((P, N), dtype=torch.float64, device=dev),
               b=torch.empty((P, N), dtype=torch.float64, device=dev),
               offset=torch.empty(P, dtype=torch.float64, device=dev),
               eps_scale=torch.empty(P, dtype=torch.float64, device=dev))
    _lib.call("il_build_ising_batch", Hd.data_ptr(), yd.data_ptr(), gd.data_ptr(), P, n_r, n_t,
              int(order), out["G"].data_ptr(), out["g_diag"].data_ptr(), out["b"].data_ptr(),
              out["offset"].data_ptr(), out["eps_scale"].data_ptr(), _stream())
    return out


def run_anneals(G, g_diag, b, x0, dt, p, a, zeta, eps, e_floor, f_mvm, n_steps,
                diverge_threshold):
    """Device-tensor form of the kernel plugin (FP64-exact, _kernel.pyx:16-102)."""
    Gd = _dev(G, torch.float64)
    gd = _dev(g_diag, torch.float64)
    bd = _dev(b, torch.float64)
    xd = _dev(x0, torch.float64)
    nb, S = xd.shape
    n = Gd.shape[0]
    if S != 2 * n + 1:
        raise ValueError("x0 must be (n_anneals, 2N+1)")
    dev = xd.device
    spins = torch.empty((nb, S), dtype=torch.int8, device=dev)
    div = torch.empty(nb, dtype=torch.uint8, device=dev)
    steps = torch.empty(nb, dtype=torch.int64, device=dev)
    mvms = torch.empty(nb, dtype=torch.int64, device=dev)
    _lib.call("il_run_anneals", Gd.data_ptr(), gd.data_ptr(), bd.data_ptr(), xd.data_ptr(), n, nb,
              float(dt), float(p), float(a), float(zeta), float(eps), float(e_floor), int(f_mvm),
              int(n_steps), float(diverge_threshold), spins.data_ptr(), div.data_ptr(),
              steps.data_ptr(), mvms.data_ptr(), _stream())
    return spins, div.bool(), steps, mvms


def derive_seeds(parts) -> torch.Tensor:
    """Row-wise ``derive_seed(*parts[i])`` (solver.py:137-144) on the device."""
    arr = np.ascontiguousarray(np.asarray(parts, dtype=np.uint64))
    if arr.ndim == 1:
        arr = arr[:, None]
    n, k = arr.shape
    pd = torch.from_numpy(arr).to("cuda")
    out = torch.empty(n, dtype=torch.uint64, device="cuda")
    _lib.call("il_derive_seeds", pd.data_ptr(), k, n, out.data_ptr(), _stream())
    return out


def initial_states(seeds, S: int, amplitude: float) -> torch.Tensor:
    """``default_rng(seed).uniform(-amp, amp, S)`` per seed (solver.py:182-187)."""
    sd = _seeds(seeds, len(seeds) if not isinstance(seeds, torch.Tensor) else seeds.numel())
    out = torch.empty((sd.numel(), S), dtype=torch.float64, device="cuda")
    _lib.call("il_initial_states", sd.data_ptr(), sd.numel(), int(S), float(amplitude),
              out.data_ptr(), _stream())
    return out


def gray_demap(x_idx, bits_per_dim: int) -> torch.Tensor:
    """Level indices [..., 2] -> Gray bits [..., 2*bits_per_dim] (channel.py:160-180)."""
    xd = _dev(x_idx, torch.uint8)
    n_sym = xd.numel() // 2
    out = torch.empty(xd.shape[:-1] + (2 * bits_per_dim,), dtype=torch.uint8, device=xd.device)
    _lib.call("il_gray_demap", xd.data_ptr(), n_sym, int(bits_per_dim), out.data_ptr(), _stream())
    return out


def spin_energies(G, b, spins) -> torch.Tensor:
    """E(s) per spin row (solver.py:171-175).  G [P,N,N], b [P,N], spins [P,B,2N+1]."""
    Gd = _dev(G, torch.float64)
    bd = _dev(b, torch.float64)
    sd = _dev(spins, torch.int8)
    P, N = bd.shape
    B = sd.shape[1]
    out = torch.empty((P, B), dtype=torch.float64, device=Gd.device)
    _lib.call("il_spin_energies", Gd.data_ptr(), 0, bd.data_ptr(), sd.data_ptr(), P, B, N,
              out.data_ptr(), _stream())
    return out


@dataclass
class SolveBatch:
    best_spins: torch.Tensor     # int8 [P, 2N+1]
    best_energy: torch.Tensor    # f64 [P] Ising energy of the best survivor (inf if none)
    best_index: torch.Tensor     # int32 [P]; -1 where the reference returns None
    diverged: torch.Tensor       # int32 [P]
    steps: torch.Tensor | None = None  # int64 [P, B] (counts=True; every precision)
    mvms: torch.Tensor | None = None


def solve_batch(G, g_diag, b, offset, fallback_energy, eps, base_seeds, params=None,
                precision: str | None = None, counts: bool = False) -> SolveBatch:
    """P x ``solve_batch`` (solver.py:238-279) on given Ising problems."""
    params = params or CacParams()
    prm = to_c(params, precision)
    Gd = _dev(G, torch.float64)
    P, N, _ = Gd.shape
    gd = _dev(g_diag, torch.float64)
    bd = _dev(b, torch.float64)
    od = _dev(offset, torch.float64).reshape(P)
    fd = _dev(fallback_energy, torch.float64).reshape(P)
    ed = _dev(eps, torch.float64).reshape(P)
    sd = _seeds(base_seeds, P)
    dev = Gd.device
    B = int(params.n_anneals)
    out = SolveBatch(best_spins=torch.empty((P, 2 * N + 1), dtype=torch.int8, device=dev),
                     best_energy=torch.empty(P, dtype=torch.float64, device=dev),
                     best_index=torch.empty(P, dtype=torch.int32, device=dev),
                     diverged=torch.empty(P, dtype=torch.int32, device=dev))
    if counts:
        out.steps = torch.empty((P, B), dtype=torch.int64, device=dev)
        out.mvms = torch.empty((P, B), dtype=torch.int64, device=dev)
    _lib.call("il_solve_batch", Gd.data_ptr(), gd.data_ptr(), bd.data_ptr(), od.data_ptr(),
              fd.data_ptr(), ed.data_ptr(), sd.data_ptr(), P, N, prm,
              out.best_spins.data_ptr(), out.best_energy.data_ptr(), out.best_index.data_ptr(),
              out.diverged.data_ptr(), out.steps.data_ptr() if counts else None,
              out.mvms.data_ptr() if counts else None, _stream())
    return out
