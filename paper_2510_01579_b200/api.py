"""The reference's per-instance API, running on the GPU.

Same names, arguments and result types as the reference ``isinglink``
package (detector.py, precoder.py, solver.py, transform.py, linear.py), so a
caller can switch imports:

    from paper_2510_01579_b200 import api as isinglink
    res = isinglink.detect_cim(inst, isinglink.CacParams(), seed)

Every numerical stage of the hot path (MMSE, Ising reduction with
lambda_max, the anneals, energies, selection, decode) runs in the CUDA
library through the batched entry points with P = 1; only format
conversions (complex <-> level indices, SpinVector packing) happen on the
host.  Throughput callers should use ``batched`` directly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, batched
from .batched import _stream
from .channel import (Constellation, MimoInstance, from_indices, make_qam,  # noqa: F401
                      project_to_constellation, to_indices)
from .params import CacParams

# transform.py:46, precoder.py:41
EPS_GAIN = 32.0
VPP_EPS_GAIN = 0.0625


# ---------------------------------------------------------------------------
# result / problem types (same fields as the reference)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class DetectionResult:
    x_hard: np.ndarray
    energy: float
    source: str              # "mmse" | "anneal"
    anneal_index: int = -1
    diverged_count: int = 0


@dataclass(frozen=True)
class SpinVector:
    s_A: np.ndarray
    s_B: np.ndarray
    s_aux: int

    def to_array(self) -> np.ndarray:
        return np.concatenate([self.s_A, self.s_B, [self.s_aux]]).astype(np.float64)

    @classmethod
    def from_array(cls, s: np.ndarray) -> "SpinVector":
        arr = np.asarray(s)
        n = (len(arr) - 1) // 2
        return cls(s_A=arr[:n].astype(np.int8), s_B=arr[n:2 * n].astype(np.int8),
                   s_aux=int(arr[2 * n]))


@dataclass(frozen=True)
class StructuredIsing:
    n_dim: int
    G: np.ndarray = field(repr=False)
    g_diag: np.ndarray = field(repr=False)
    b: np.ndarray = field(repr=False)
    c: float
    offset: float
    x_guess: np.ndarray = field(repr=False)
    spin_count: int
    eps_scale: float


@dataclass(frozen=True)
class AnnealResult:
    spins: SpinVector = field(repr=False)
    energy: float
    diverged: bool
    anneal_index: int


@dataclass(frozen=True)
class PrecodeResult:
    x_transmit: np.ndarray = field(repr=False)
    v: np.ndarray = field(repr=False)
    unnormalized_power: float
    tau: float


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def derive_seed(*parts: int) -> int:
    """solver.py:137-144 (NumPy SeedSequence, the reference's own dependency)."""
    st = np.random.SeedSequence(tuple(int(p) for p in parts)).generate_state(2)
    return int(st[0]) | (int(st[1]) << 32)


def _order_code(c: Constellation) -> int:
    """Library alphabet code: QAM order, or -reach for the VPP integer lattice."""
    lv = np.asarray(c.pam_levels)
    if c.order in (4, 16, 64, 256) and np.array_equal(lv, make_qam(c.order).pam_levels):
        return int(c.order)
    reach = (len(lv) - 1) // 2
    if len(lv) % 2 == 1 and np.array_equal(lv, 4.0 * np.arange(-reach, reach + 1)):
        return -reach
    raise ValueError("the CUDA path supports unit-energy square QAM and the VPP lattice")


def _note(counters, diverged, steps, mvms):
    if counters is None:
        return
    counters["anneals"] = counters.get("anneals", 0) + int(np.size(steps))
    counters["diverged"] = counters.get("diverged", 0) + int(np.sum(diverged))
    counters["steps"] = counters.get("steps", 0) + int(np.sum(steps))
    counters["mvm_updates"] = counters.get("mvm_updates", 0) + int(np.sum(mvms))


def residual_energy(H: np.ndarray, y: np.ndarray, x: np.ndarray) -> float:
    """||y - Hx||^2 (linear.py:44-47) on the GPU, in the same arithmetic as
    the energies the detectors compute, so guess and decoded energies tie
    exactly when the decision is unchanged (strict test, detector.py:52)."""
    H = np.asarray(H, dtype=np.complex128)
    y = np.asarray(y, dtype=np.complex128)
    x = np.asarray(x, dtype=np.complex128)
    return float(batched.residual_batch(H[None], y[None], x[None])[0])


# ---------------------------------------------------------------------------
# linear front-end and Ising reduction
# ---------------------------------------------------------------------------
def _check_uplink(inst: MimoInstance) -> None:
    """linear.py:50-52, plus SciPy's check_finite of the Cholesky solve: the
    reference raises ValueError on non-finite H, y or noise variance."""
    if inst.n_r < inst.n_t:
        raise ValueError("uplink detection requires n_r >= n_t")
    if not (np.all(np.isfinite(inst.H)) and np.all(np.isfinite(inst.y))
            and np.isfinite(inst.noise_var)):
        raise ValueError("array must not contain infs or NaNs")


def detect_mmse(inst: MimoInstance) -> DetectionResult:
    """linear.py:69-75 on the GPU."""
    _check_uplink(inst)
    x_idx, energy, status = batched.mmse_batch(inst.H[None], inst.y[None],
                                               np.array([inst.noise_var]),
                                               _order_code(inst.constellation))
    if int(status[0]) != 0:
        raise np.linalg.LinAlgError("regularized normal matrix is not positive definite")
    x = from_indices(x_idx[0].cpu().numpy(), inst.constellation)
    return DetectionResult(x_hard=x, energy=float(energy[0]), source="mmse")


def detect_mmse_sic(inst: MimoInstance) -> DetectionResult:
    """linear.py:78-106 (ordered MMSE-SIC) on the GPU."""
    _check_uplink(inst)
    x_idx, energy, status = batched.mmse_sic_batch(inst.H[None], inst.y[None],
                                                   np.array([inst.noise_var]),
                                                   _order_code(inst.constellation))
    if int(status[0]) != 0:
        raise np.linalg.LinAlgError("regularized normal matrix is not positive definite")
    x = from_indices(x_idx[0].cpu().numpy(), inst.constellation)
    return DetectionResult(x_hard=x, energy=float(energy[0]), source="mmse_sic")


ML_MAX_BITS = 24  # linear.py:28


def detect_ml(inst: MimoInstance) -> DetectionResult:
    """linear.py:109-144: exhaustive ML on the GPU (ties to the smallest
    symbol-index vector, user 0 most significant)."""
    bits = inst.n_t * inst.constellation.bits_per_symbol
    if bits > ML_MAX_BITS:
        raise ValueError(f"ML search space of {bits} bits exceeds the {ML_MAX_BITS}-bit guard")
    x_idx, energy = batched.ml_batch(inst.H[None], inst.y[None], _order_code(inst.constellation))
    x = from_indices(x_idx[0].cpu().numpy(), inst.constellation)
    return DetectionResult(x_hard=x, energy=float(energy[0]), source="ml")


def ml_llr(inst: MimoInstance) -> np.ndarray:
    """Max-log bit LLRs of the exhaustive search, [n_t, bits_per_symbol] in
    the Gray-demapper bit order, (d1 - d0) / noise_var: positive favours bit 0.
    No reference counterpart (soft output is a reference non-goal,
    SPEC.md:153); the sign agrees with the bits of ``detect_ml``."""
    bits = inst.n_t * inst.constellation.bits_per_symbol
    if bits > ML_MAX_BITS:
        raise ValueError(f"ML search space of {bits} bits exceeds the {ML_MAX_BITS}-bit guard")
    if inst.H.shape[0] > 16:
        raise ValueError("ml_llr supports n_r <= 16")
    llr = batched.ml_llr_batch(inst.H[None], inst.y[None], _order_code(inst.constellation),
                               noise_var=[float(inst.noise_var)])
    return llr[0].cpu().numpy()


def build_ising(inst: MimoInstance, x_guess: np.ndarray) -> StructuredIsing:
    """transform.py:108-140 on the GPU, around a constellation-point guess."""
    x_guess = np.asarray(x_guess, dtype=complex)
    if not np.all(np.isfinite(x_guess.view(np.float64))):
        raise ValueError("x_guess must be finite")
    c = inst.constellation
    idx = to_indices(x_guess, c)
    if not np.array_equal(from_indices(idx, c), x_guess):
        raise ValueError("the CUDA build_ising takes a guess on the constellation grid")
    out = batched.build_ising_batch(inst.H[None], inst.y[None], idx[None], _order_code(c))
    N = 2 * inst.n_t
    return StructuredIsing(n_dim=N, G=out["G"][0].cpu().numpy(),
                           g_diag=out["g_diag"][0].cpu().numpy(), b=out["b"][0].cpu().numpy(),
                           c=c.spacing / 2.0, offset=float(out["offset"][0]), x_guess=x_guess,
                           spin_count=2 * N + 1, eps_scale=float(out["eps_scale"][0]))


def ising_energy(si: StructuredIsing, s: SpinVector) -> float:
    """transform.py:143-152 (FP64 on the GPU)."""
    if len(s.s_A) != si.n_dim or len(s.s_B) != si.n_dim:
        raise ValueError("spin vector does not match the problem dimension")
    e = batched.spin_energies(si.G[None], si.b[None], s.to_array().astype(np.int8)[None, None])
    return float(e[0, 0])


def spin_perturbation(si: StructuredIsing, s: SpinVector) -> np.ndarray:
    """transform.py:155-164: c * s_aux * (s_A + s_B), real dims then imaginary."""
    d = si.c * s.s_aux * (s.s_A.astype(np.float64) + s.s_B)
    nt = si.n_dim // 2
    return d[:nt] + 1j * d[nt:]


def decode_spins(si: StructuredIsing, s: SpinVector, c: Constellation) -> np.ndarray:
    """transform.py:167-169."""
    return project_to_constellation(si.x_guess + spin_perturbation(si, s), c)


def structured_mvm(si: StructuredIsing, x1, x2, xa: float) -> np.ndarray:
    """solver.py:147-168 (device matvec in FP64)."""
    x1 = np.asarray(x1, dtype=np.float64)
    x2 = np.asarray(x2, dtype=np.float64)
    if x1.shape != (si.n_dim,) or x2.shape != (si.n_dim,):
        raise ValueError("x1/x2 must have length n_dim")
    N = si.n_dim
    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = dict(dtype=torch.float64, device=dev)
    G = torch.as_tensor(np.ascontiguousarray(si.G, dtype=np.float64), **f64)
    g = torch.as_tensor(np.ascontiguousarray(si.g_diag, dtype=np.float64), **f64)
    b = torch.as_tensor(np.ascontiguousarray(si.b, dtype=np.float64), **f64)
    t1 = torch.as_tensor(x1, **f64)
    t2 = torch.as_tensor(x2, **f64)
    ta = torch.tensor([float(xa)], **f64)
    out = torch.empty(2 * N + 1, **f64)
    _lib.call("il_structured_mvm_batch", G.data_ptr(), g.data_ptr(), b.data_ptr(), t1.data_ptr(),
              t2.data_ptr(), ta.data_ptr(), 1, N, out.data_ptr(), _stream())
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# solver
# ---------------------------------------------------------------------------
def _resolved_eps(si: StructuredIsing, params) -> float:
    return si.eps_scale if params.eps is None else params.eps


def integrate_anneal(si: StructuredIsing, params=None, seed: int = 0, counters=None) -> AnnealResult:
    """solver.py:217-235: one anneal from default_rng(seed), FP64-exact kernel."""
    params = params or CacParams()
    params.validate()
    x0 = batched.initial_states(np.array([seed], np.uint64), si.spin_count, params.init_amplitude)
    spins, div, steps, mvms = batched.run_anneals(
        si.G, si.g_diag, si.b, x0, params.dt, params.p, params.a, params.zeta,
        _resolved_eps(si, params), params.e_floor, params.f_mvm, params.n_steps,
        params.diverge_threshold)
    e = batched.spin_energies(si.G[None], si.b[None], spins[None])
    _note(counters, div.cpu().numpy(), steps.cpu().numpy(), mvms.cpu().numpy())
    return AnnealResult(spins=SpinVector.from_array(spins[0].cpu().numpy()), energy=float(e[0, 0]),
                        diverged=bool(div[0]), anneal_index=0)


def solve_batch(si: StructuredIsing, params, fallback_energy: float, base_seed: int,
                counters=None):
    """solver.py:238-279: (AnnealResult | None, diverged_count)."""
    params = params or CacParams()
    params.validate()
    r = batched.solve_batch(si.G[None], si.g_diag[None], si.b[None], np.array([si.offset]),
                            np.array([fallback_energy], np.float64),
                            np.array([_resolved_eps(si, params)]),
                            np.array([base_seed], np.uint64), params, counts=counters is not None)
    ndiv = int(r.diverged[0])
    if counters is not None:
        counters["anneals"] = counters.get("anneals", 0) + int(params.n_anneals)
        counters["diverged"] = counters.get("diverged", 0) + ndiv
        counters["steps"] = counters.get("steps", 0) + int(r.steps.sum())
        counters["mvm_updates"] = counters.get("mvm_updates", 0) + int(r.mvms.sum())
    bi = int(r.best_index[0])
    if bi < 0:
        return None, ndiv
    return AnnealResult(spins=SpinVector.from_array(r.best_spins[0].cpu().numpy()),
                        energy=float(r.best_energy[0]), diverged=False, anneal_index=bi), ndiv


def _improve_guess(inst, guess, guess_energy, params, base_seed, counters, eps_gain=1.0):
    """detector.py:27-54."""
    si = build_ising(inst, guess)
    if params.eps is None and eps_gain != 1.0:
        from dataclasses import replace
        params = replace(params, eps=si.eps_scale * eps_gain)
    best, diverged = solve_batch(si, params, guess_energy, base_seed, counters=counters)
    if best is None:
        return guess, guess_energy, -1, diverged
    decoded = decode_spins(si, best.spins, inst.constellation)
    energy = residual_energy(inst.H, inst.y, decoded)
    if energy < guess_energy:
        return decoded, energy, best.anneal_index, diverged
    return guess, guess_energy, -1, diverged


# ---------------------------------------------------------------------------
# pipelines
# ---------------------------------------------------------------------------
def detect_cim(inst: MimoInstance, params=None, seed: int = 0, counters=None) -> DetectionResult:
    """detector.py:57-82.  Without counters this is one fused batched call."""
    params = params or CacParams()
    if counters is not None:
        mmse = detect_mmse(inst)
        x, energy, widx, diverged = _improve_guess(inst, mmse.x_hard, mmse.energy, params,
                                                   derive_seed(seed, 0, 0), counters)
        if widx < 0:
            return DetectionResult(x_hard=mmse.x_hard, energy=mmse.energy, source="mmse",
                                   diverged_count=diverged)
        return DetectionResult(x_hard=x, energy=energy, source="anneal", anneal_index=widx,
                               diverged_count=diverged)
    _check_uplink(inst)
    r = batched.detect_cim_batch(inst.H[None], inst.y[None], np.array([inst.noise_var]),
                                 _order_code(inst.constellation), np.array([seed], np.uint64),
                                 params)
    src = int(r.source[0])
    if src < 0:
        raise np.linalg.LinAlgError("regularized normal matrix is not positive definite")
    x = from_indices(r.x_idx[0].cpu().numpy(), inst.constellation)
    return DetectionResult(x_hard=x, energy=float(r.energy[0]),
                           source="anneal" if src == 1 else "mmse",
                           anneal_index=int(r.anneal_index[0]),
                           diverged_count=int(r.diverged[0]))


_SOURCES = {0: "mmse", 1: "anneal", 2: "mmse_sic"}


def detect_cim_multi(inst: MimoInstance, params=None, n_stages: int = 1, seed: int = 0,
                     chains: tuple = ("mmse", "mmse_sic"), counters=None,
                     stage_log: list | None = None) -> DetectionResult:
    """MMGaP-E, detector.py:85-134: one fused batched call (P = 1).

    ``counters`` / ``stage_log`` are the reference's instrumentation hooks;
    with either given the chains run stage by stage through the per-stage
    API so the hooks see every stage."""
    params = params or CacParams()
    if n_stages < 1:
        raise ValueError("n_stages must be >= 1")
    if counters is not None or stage_log is not None:
        fns = {"mmse": detect_mmse, "mmse_sic": detect_mmse_sic}
        baselines = [(name, fns[name](inst)) for name in chains]
        best = min(baselines, key=lambda kv: kv[1].energy)[1]
        total = 0
        for chain_id, (name, base) in enumerate(baselines):
            guess, energy, widx = base.x_hard, base.energy, -1
            for stage in range(n_stages):
                guess, energy, idx, div = _improve_guess(inst, guess, energy, params,
                                                         derive_seed(seed, chain_id, stage),
                                                         counters)
                total += div
                if idx >= 0:
                    widx = idx
                if stage_log is not None:
                    stage_log.append((name, stage, energy))
            if energy < best.energy:
                best = DetectionResult(x_hard=guess, energy=energy, source="anneal",
                                       anneal_index=widx)
        return DetectionResult(x_hard=best.x_hard, energy=best.energy, source=best.source,
                               anneal_index=best.anneal_index, diverged_count=total)
    _check_uplink(inst)
    r = batched.detect_cim_multi_batch(inst.H[None], inst.y[None], np.array([inst.noise_var]),
                                       _order_code(inst.constellation),
                                       np.array([seed], np.uint64), params, n_stages, chains)
    src = int(r.source[0])
    if src < 0:
        raise np.linalg.LinAlgError("regularized normal matrix is not positive definite")
    x = from_indices(r.x_idx[0].cpu().numpy(), inst.constellation)
    return DetectionResult(x_hard=x, energy=float(r.energy[0]), source=_SOURCES[src],
                           anneal_index=int(r.anneal_index[0]),
                           diverged_count=int(r.diverged[0]))


def zf_matrix(H: np.ndarray) -> np.ndarray:
    """precoder.py:54-60: W = H^H (H H^H)^-1 (FP64 on the GPU)."""
    n_r, n_t = H.shape
    if n_r > n_t:
        raise ValueError("downlink precoding requires n_r <= n_t")
    dev = torch.device("cuda", torch.cuda.current_device())
    Ht = torch.as_tensor(np.ascontiguousarray(H, dtype=np.complex128), device=dev)
    W = torch.empty((n_t, n_r), dtype=torch.complex128, device=dev)
    status = torch.empty(1, dtype=torch.int8, device=dev)
    _lib.call("il_zf_batch", Ht.data_ptr(), 1, n_r, n_t, W.data_ptr(), status.data_ptr(), _stream())
    if int(status.item()) != 0:
        raise np.linalg.LinAlgError("H H^H is not positive definite")
    return W.cpu().numpy()


def precode_zf(H: np.ndarray, u: np.ndarray, P: float) -> np.ndarray:
    """precoder.py:63-71."""
    if P <= 0:
        raise ValueError("P must be positive")
    w = zf_matrix(H) @ u
    norm = np.linalg.norm(w)
    return w if norm == 0.0 else math.sqrt(P) * w / norm


def default_tau(c: Constellation) -> float:
    """precoder.py:74-76."""
    return float(2.0 * (c.pam_levels[-1] + c.spacing / 2.0))


def precode_vpp(H: np.ndarray, u: np.ndarray, P: float, tau: float, params=None, seed: int = 0,
                n_stages: int = 1, counters=None) -> PrecodeResult:
    """precoder.py:93-146 on the GPU (one fused batched call)."""
    params = params or CacParams()
    if P <= 0:
        raise ValueError("P must be positive")
    r = batched.precode_vpp_batch(np.asarray(H, complex)[None], np.asarray(u, complex)[None],
                                  float(P), float(tau), np.array([seed], np.uint64), params,
                                  n_stages=n_stages)
    if counters is not None:
        counters["diverged"] = counters.get("diverged", 0) + int(r.diverged[0])
        counters["anneals"] = counters.get("anneals", 0) + n_stages * int(params.n_anneals)
    return PrecodeResult(x_transmit=r.x[0].cpu().numpy(), v=r.v[0].cpu().numpy(),
                         unnormalized_power=float(r.unnormalized_power[0]), tau=float(tau))


def effective_snr(H, u, v, tau, P, noise_var) -> float:
    """precoder.py:149-160."""
    W = zf_matrix(H)
    w = W @ u if v is None else W @ (u + tau * v)
    return float(P / (noise_var * np.real(np.vdot(w, w))))


def fold_mod_tau(z, tau):
    """precoder.py:163-168."""
    z = np.asarray(z)
    re = np.mod(z.real + tau / 2.0, tau) - tau / 2.0
    im = np.mod(z.imag + tau / 2.0, tau) - tau / 2.0
    return re + 1j * im
