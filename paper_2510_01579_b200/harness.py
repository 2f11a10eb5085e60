"""GPU experiment harness: the reference's paired sweeps, integration heatmap
and benchmark report (harness/sweeps.py, heatmap.py, bench.py) with every
detector, precoder and integration batched through the CUDA library.

Instances are generated exactly as the reference does (NumPy streams keyed
by ``derive_seed(seed, domain, grid point, trial, k)``, channel.py:111-138,
sweeps.py:85-96), so a sweep here and the reference's sweep see the same
problems.  Rather than one process per trial block, all trials of a grid
point go to the GPU in one batch; the per-row data columns are reduced in
trial order like the reference's concatenate-then-sum.  With
``precision="fp64_exact"`` (the default) the detections are the
reference's; ``"fp32"`` is the throughput mode.

Rows use the reference's ``SweepRow`` / ``HeatmapCell`` fields and the CSV
layout of ``write_csv`` (header, ``repr`` floats, ``# config_hash=`` footer)
with the same canonical config hash, so downstream tooling reads either.
The ``cfg`` argument is a reference ``ExperimentConfig`` (or any object with
the same fields).
"""

from __future__ import annotations

import csv
import dataclasses
import hashlib
import math
import time
from dataclasses import dataclass, fields

import numpy as np
import torch

from . import _lib, api, batched
from .channel import (bit_errors, make_qam, project_to_constellation, sample_channel,
                      symbol_errors, transmit)
from .params import CacParams

__all__ = ["ExperimentConfig", "CacConfig", "config_from_text", "SweepRow", "HeatmapCell",
           "write_csv", "format_config", "config_hash", "uplink_batch", "run_detection_sweep", "run_precoding_sweep",
           "run_integration_heatmap", "run_bench", "REFERENCE_DT", "REFERENCE_FMVM"]

# domain keys of derive_seed (sweeps.py:41-42, heatmap.py:27, bench.py:29)
DOM_UPLINK, DOM_DOWNLINK, DOM_HEATMAP, DOM_BENCH = 1, 2, 3, 4
REFERENCE_DT, REFERENCE_FMVM = 0.01, 1  # heatmap.py:29-30
_HASH_EXCLUDED = ("output_path", "n_workers")  # config.py:51


@dataclass(frozen=True)
class SweepRow:
    """sweeps.py:46-55."""
    snr_db: float
    detector: str
    ser: float
    ber: float
    mean_energy: float
    mean_diverged: float
    wall_time_s: float
    n_trials: int


@dataclass(frozen=True)
class HeatmapCell:
    """heatmap.py:34-40."""
    dt: float
    f_mvm: int
    p_diverge: float
    p_error_mean: float
    n_instances: int


# ---------------------------------------------------------------------------
# configuration (config.py:54-110): same fields, defaults and validation as
# the reference's ExperimentConfig, so hashes agree; reference configs are
# accepted too
# ---------------------------------------------------------------------------
MODES = ("uplink_sweep", "downlink_sweep", "heatmap", "bench")
DETECTOR_NAMES = ("mmse", "mmse_sic", "ml", "cim", "cim_multi")


@dataclass(frozen=True)
class CacConfig:
    """The reference CacParams fields (solver.py:97-107)."""
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

    def validate(self) -> None:
        CacParams(**dataclasses.asdict(self)).validate()


@dataclass(frozen=True)
class ExperimentConfig:
    mode: str = "uplink_sweep"
    n_r: int = 8
    n_t: int = 8
    modulation: int = 16
    snr_grid_db: tuple = (10.0, 15.0, 20.0, 25.0, 30.0)
    n_trials: int = 200
    detectors: tuple = ("mmse", "cim")
    n_stages: int = 1
    channel_model: str = "iid"
    power: float = 0.0
    n_workers: int = 1
    seed: int = 1
    output_path: str = ""
    dt_grid: tuple = (0.01, 0.02, 0.04, 0.08, 0.16)
    fmvm_grid: tuple = (1, 2, 4, 8)
    n_instances: int = 1000
    budget: float = 2.56
    batch_size: int = 4096
    worker_grid: tuple = (1, 2, 4)
    cac: CacConfig = dataclasses.field(default_factory=CacConfig)

    def validate(self) -> None:
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, not {self.mode!r}")
        if not (self.n_r >= 1 and self.n_t >= 1):
            raise ValueError("n_r and n_t must be >= 1")
        if not self.snr_grid_db:
            raise ValueError("snr_grid_db must be non-empty")
        if self.n_trials < 1 or self.n_instances < 1 or self.batch_size < 1:
            raise ValueError("trial/instance/batch counts must be >= 1")
        if not self.detectors:
            raise ValueError("detectors must be non-empty")
        for name in self.detectors:
            if name not in DETECTOR_NAMES:
                raise ValueError(f"unknown detector {name!r}; valid: {DETECTOR_NAMES}")
        if self.channel_model not in ("iid", "identity"):
            raise ValueError("channel_model must be iid or identity")
        if self.n_stages < 1:
            raise ValueError("n_stages must be >= 1")
        if self.n_workers < 1 or not self.worker_grid:
            raise ValueError("worker counts must be >= 1")
        if not self.dt_grid or not self.fmvm_grid:
            raise ValueError("heatmap grids must be non-empty")
        if self.budget <= 0:
            raise ValueError("budget must be positive")
        self.cac.validate()


def _coerce(example, raw: str):
    if isinstance(example, tuple):
        items = [t.strip() for t in raw.split(",") if t.strip()]
        kind = type(example[0]) if example else str
        return tuple(kind(t) for t in items)
    if example is None:
        return None if raw.lower() in ("auto", "none") else float(raw)
    if isinstance(example, bool):
        return raw.lower() in ("1", "true", "yes")
    return type(example)(raw)


def config_from_text(text: str) -> ExperimentConfig:
    """Parse 'key = value' lines (config.py:113-165), e.g. format_config output."""
    base = ExperimentConfig()
    kw, cac = {}, {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"line {lineno}: expected 'key = value', got {raw!r}")
        key, value = (t.strip() for t in line.split("=", 1))
        if key.startswith("cac."):
            cac[key[4:]] = _coerce(getattr(base.cac, key[4:]), value)
        else:
            kw[key] = _coerce(getattr(base, key), value)
    cfg = dataclasses.replace(base, cac=dataclasses.replace(base.cac, **cac), **kw)
    cfg.validate()
    return cfg


# ---------------------------------------------------------------------------
# formats (sweeps.py:58-74, config.py:168-196)
# ---------------------------------------------------------------------------
def _fmt(value) -> str:
    return repr(value) if isinstance(value, float) else str(value)


def write_csv(path: str, rows: list, cfg_hash: str) -> None:
    """Header, one line per row, ``# config_hash=...`` footer (sweeps.py:63-74)."""
    if not rows:
        raise ValueError("no rows to write")
    names = [f.name for f in fields(rows[0])]
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh, lineterminator="\n")
        writer.writerow(names)
        for row in rows:
            writer.writerow([_fmt(getattr(row, n)) for n in names])
        fh.write(f"# config_hash={cfg_hash}\n")


def _format_value(value) -> str:
    if value is None:
        return "auto"
    if isinstance(value, tuple):
        return ", ".join(_format_value(v) for v in value)
    if isinstance(value, float):
        return repr(value)
    return str(value)


def format_config(cfg, include_excluded: bool = True) -> str:
    """Canonical text form of an ExperimentConfig (config.py:179-190)."""
    lines = []
    for f in sorted(fields(cfg), key=lambda f: f.name):
        if f.name == "cac":
            continue
        if not include_excluded and f.name in _HASH_EXCLUDED:
            continue
        lines.append(f"{f.name} = {_format_value(getattr(cfg, f.name))}")
    for f in sorted(fields(cfg.cac), key=lambda f: f.name):
        lines.append(f"cac.{f.name} = {_format_value(getattr(cfg.cac, f.name))}")
    return "\n".join(lines) + "\n"


def config_hash(cfg) -> str:
    """SHA-256 of the canonical form minus output path and worker count."""
    return hashlib.sha256(format_config(cfg, include_excluded=False).encode()).hexdigest()


# ---------------------------------------------------------------------------
# instances
# ---------------------------------------------------------------------------
def _params(cfg) -> CacParams:
    c = cfg.cac
    return CacParams(p=c.p, a=c.a, zeta=c.zeta, eps=c.eps, dt=c.dt, f_mvm=c.f_mvm,
                     n_steps=c.n_steps, n_anneals=c.n_anneals,
                     diverge_threshold=c.diverge_threshold, e_floor=c.e_floor,
                     init_amplitude=c.init_amplitude)


def _seeds(rows) -> np.ndarray:
    """derive_seed per row of parts, on the device (bit-exact SeedSequence)."""
    return batched.derive_seeds(np.asarray(rows, dtype=np.uint64)).cpu().numpy()


def _channel_for(cfg, seed: int) -> np.ndarray:
    if cfg.channel_model == "identity":
        n = max(cfg.n_r, cfg.n_t)
        return np.eye(n, dtype=complex)[: cfg.n_r, : cfg.n_t]
    return sample_channel(cfg.n_r, cfg.n_t, seed)


def uplink_batch(cfg, snr_idx: int, trials) -> dict:
    """The reference's make_uplink_instance for many trials (sweeps.py:85-96).

    Returns H [T, n_r, n_t], y [T, n_r], noise_var [T], truth (level indices
    [T, n_t, 2]) and the detector seeds derive_seed(seed, 1, snr_idx, t, 3)."""
    trials = np.asarray(list(trials), dtype=np.int64)
    const = make_qam(cfg.modulation)
    base = [[cfg.seed, DOM_UPLINK, snr_idx, int(t)] for t in trials]
    s = _seeds([b + [k] for b in base for k in range(4)]).reshape(len(trials), 4)
    T = len(trials)
    H = np.empty((T, cfg.n_r, cfg.n_t), complex)
    y = np.empty((T, cfg.n_r), complex)
    nv = np.empty(T)
    truth = np.empty((T, cfg.n_t, 2), np.uint8)
    m = int(math.isqrt(cfg.modulation))
    for i in range(T):
        H[i] = _channel_for(cfg, int(s[i, 0]))
        d = np.random.default_rng(int(s[i, 1])).integers(0, const.order, cfg.n_t)
        x = const.points[d]
        y[i], nv[i] = transmit(H[i], x, cfg.snr_grid_db[snr_idx], int(s[i, 2]))
        truth[i, :, 0] = d // m
        truth[i, :, 1] = d % m
    return dict(H=H, y=y, noise_var=nv, truth=truth, seed=s[:, 3].astype(np.uint64))


def _errors(truth: torch.Tensor, x_idx: torch.Tensor, bpd: int):
    """Per-trial symbol and Gray-bit error counts (channel.py:167-180)."""
    sym = (truth != x_idx).any(-1).sum(-1)
    gt = batched.gray_demap(truth, bpd).view(truth.shape[0], -1)
    gx = batched.gray_demap(x_idx, bpd).view(truth.shape[0], -1)
    return sym, (gt != gx).sum(-1)


# ---------------------------------------------------------------------------
# uplink sweep (sweeps.py:99-192)
# ---------------------------------------------------------------------------
def _detect(name: str, b: dict, cfg, prm: CacParams):
    order = cfg.modulation
    if name == "mmse":
        x, e, st = batched.mmse_batch(b["H"], b["y"], b["noise_var"], order)
        return x, e, torch.zeros_like(e, dtype=torch.int32), st
    if name == "mmse_sic":
        x, e, st = batched.mmse_sic_batch(b["H"], b["y"], b["noise_var"], order)
        return x, e, torch.zeros_like(e, dtype=torch.int32), st
    if name == "ml":
        x, e = batched.ml_batch(b["H"], b["y"], order)
        return x, e, torch.zeros_like(e, dtype=torch.int32), None
    if name == "cim":
        r = batched.detect_cim_batch(b["H"], b["y"], b["noise_var"], order, b["seed"], prm)
    elif name == "cim_multi":
        r = batched.detect_cim_multi_batch(b["H"], b["y"], b["noise_var"], order, b["seed"], prm,
                                           cfg.n_stages)
    else:
        raise ValueError(f"unknown detector {name!r}")
    return r.x_idx, r.energy, r.diverged, r.source


def run_detection_sweep(cfg, precision: str = "fp64_exact", rng: str = "numpy") -> list:
    """Paired uplink sweep (sweeps.py:150-192), every detector on the GPU.
    ``rng="philox"`` draws the anneals' initial states from Philox4x32-10
    instead of the reference's numpy streams (statistical parity)."""
    cfg.validate()
    if cfg.mode != "uplink_sweep":
        raise ValueError(f"config mode is {cfg.mode!r}, expected uplink_sweep")
    const = make_qam(cfg.modulation)
    bpd = int(round(math.log2(int(math.isqrt(cfg.modulation)))))
    prm = dataclasses.replace(_params(cfg), precision=precision, rng=rng)
    n_sym = cfg.n_trials * cfg.n_t
    n_bit = n_sym * const.bits_per_symbol
    rows = []
    for snr_idx, snr_db in enumerate(cfg.snr_grid_db):
        b = uplink_batch(cfg, snr_idx, range(cfg.n_trials))
        truth = torch.from_numpy(b["truth"]).cuda()
        for det in cfg.detectors:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, e, dv, st = _detect(det, b, cfg, prm)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            if st is not None and bool((st < 0).any()):
                raise np.linalg.LinAlgError("regularized normal matrix is not positive definite")
            sym, bit = _errors(truth, x, bpd)
            energy = e.cpu().numpy()
            rows.append(SweepRow(
                snr_db=float(snr_db), detector=det,
                ser=float(np.sum(sym.cpu().numpy()) / n_sym),
                ber=float(np.sum(bit.cpu().numpy()) / n_bit),
                mean_energy=float(np.sum(energy) / cfg.n_trials),
                mean_diverged=float(np.sum(dv.cpu().numpy()) / cfg.n_trials),
                wall_time_s=float(wall), n_trials=cfg.n_trials))
    if cfg.output_path:
        write_csv(cfg.output_path, rows, config_hash(cfg))
    return rows


# ---------------------------------------------------------------------------
# downlink sweep (sweeps.py:195-279)
# ---------------------------------------------------------------------------
def run_precoding_sweep(cfg, precision: str = "fp64_exact", rng: str = "numpy") -> list:
    """Paired downlink sweep: ZF vs VPP through a modulo-tau receiver.

    VPP runs batched on the GPU (precoder.py:93-146); ZF and the receiver
    (scoring) follow sweeps.py:213-250 on the host."""
    cfg.validate()
    if cfg.mode != "downlink_sweep":
        raise ValueError(f"config mode is {cfg.mode!r}, expected downlink_sweep")
    if cfg.n_r > cfg.n_t:
        raise ValueError("downlink requires n_r <= n_t")
    const = make_qam(cfg.modulation)
    tau = api.default_tau(const)
    P = cfg.power if cfg.power > 0 else float(cfg.n_r)
    prm = dataclasses.replace(_params(cfg), precision=precision, rng=rng)
    n_sym = cfg.n_trials * cfg.n_r
    n_bit = n_sym * const.bits_per_symbol
    rows = []
    for snr_idx, snr_db in enumerate(cfg.snr_grid_db):
        sigma2 = 10.0 ** (-snr_db / 10.0)
        s = _seeds([[cfg.seed, DOM_DOWNLINK, snr_idx, t, k] for t in range(cfg.n_trials)
                    for k in range(4)]).reshape(cfg.n_trials, 4)
        Hs, us, noise = [], [], []
        for t in range(cfg.n_trials):
            H = _channel_for(cfg, int(s[t, 0]))
            rng = np.random.default_rng(int(s[t, 1]))
            u = const.points[rng.integers(0, const.order, cfg.n_r)]
            nz = (rng.standard_normal(cfg.n_r) + 1j * rng.standard_normal(cfg.n_r)) * np.sqrt(
                sigma2 / 2.0)
            Hs.append(H); us.append(u); noise.append(nz)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = batched.precode_vpp_batch(np.array(Hs), np.array(us), P, tau,
                                        s[:, 3].astype(np.uint64), prm, n_stages=cfg.n_stages)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        xv = res.x.cpu().numpy()
        pw = res.unnormalized_power.cpu().numpy()
        dvv = res.diverged.cpu().numpy()
        cells = {d: dict(sym=0, bit=0, energy=[]) for d in ("zf", "vpp")}
        for t in range(cfg.n_trials):
            H, u = Hs[t], us[t]
            W = api.zf_matrix(H)
            w_u = W @ u
            zf_power = float(np.real(np.vdot(w_u, w_u)))
            for det, x_tx, power in (("zf", np.sqrt(P) * w_u / np.linalg.norm(w_u), zf_power),
                                     ("vpp", xv[t], float(pw[t]))):
                gain = np.sqrt(P / power)
                z = api.fold_mod_tau((H @ x_tx + noise[t]) / gain, tau)
                u_hat = project_to_constellation(z, const)
                cells[det]["sym"] += symbol_errors(u, u_hat)
                cells[det]["bit"] += bit_errors(u, u_hat, const)
                cells[det]["energy"].append(power)
        for det in ("zf", "vpp"):
            c = cells[det]
            rows.append(SweepRow(
                snr_db=float(snr_db), detector=det, ser=float(c["sym"] / n_sym),
                ber=float(c["bit"] / n_bit),
                mean_energy=float(np.sum(np.array(c["energy"])) / cfg.n_trials),
                mean_diverged=float(np.sum(dvv) / cfg.n_trials) if det == "vpp" else 0.0,
                wall_time_s=float(wall) if det == "vpp" else 0.0, n_trials=cfg.n_trials))
    if cfg.output_path:
        write_csv(cfg.output_path, rows, config_hash(cfg))
    return rows


# ---------------------------------------------------------------------------
# integration heatmap (heatmap.py:47-108)
# ---------------------------------------------------------------------------
def _steps_for(budget: float, dt: float) -> int:
    return max(1, round(budget / dt))


def run_integration_heatmap(cfg) -> list:
    """(dt, f_mvm) fidelity grid against the (0.01, 1) reference run; every
    integration is one FP64-exact batched launch over all instances."""
    cfg.validate()
    if cfg.mode != "heatmap":
        raise ValueError(f"config mode is {cfg.mode!r}, expected heatmap")
    heat = dataclasses.replace(cfg, snr_grid_db=(cfg.snr_grid_db[0],))
    b = uplink_batch(heat, 0, range(cfg.n_instances))
    x_idx, _, _ = batched.mmse_batch(b["H"], b["y"], b["noise_var"], cfg.modulation)
    si = batched.build_ising_batch(b["H"], b["y"], x_idx, cfg.modulation)
    seeds = _seeds([[cfg.seed, DOM_HEATMAP, i] for i in range(cfg.n_instances)])
    base = _params(cfg)
    eps = (si["eps_scale"] if base.eps is None
           else torch.full_like(si["eps_scale"], float(base.eps)))

    def integrate(prm: CacParams):
        return batched.integrate_batch(si["G"], si["g_diag"], si["b"], eps, seeds, prm)

    ref = integrate(dataclasses.replace(base, dt=REFERENCE_DT, f_mvm=REFERENCE_FMVM,
                                        n_steps=_steps_for(cfg.budget, REFERENCE_DT)))
    ref_spins = ref["spins"].cpu().numpy()
    ref_div = ref["diverged"].cpu().numpy()
    rows = []
    for dt in cfg.dt_grid:
        for f in cfg.fmvm_grid:
            run = integrate(dataclasses.replace(base, dt=dt, f_mvm=f,
                                                n_steps=_steps_for(cfg.budget, dt)))
            sp = run["spins"].cpu().numpy()
            dv = run["diverged"].cpu().numpy()
            n_div, err_sum, err_n = 0, 0.0, 0
            for i in range(cfg.n_instances):  # instance order, as the reference sums
                if dv[i]:
                    n_div += 1
                elif not ref_div[i]:
                    err_sum += float(np.mean(sp[i] != ref_spins[i]))
                    err_n += 1
            rows.append(HeatmapCell(dt=float(dt), f_mvm=int(f),
                                    p_diverge=float(n_div / cfg.n_instances),
                                    p_error_mean=float(err_sum / err_n) if err_n else 1.0,
                                    n_instances=cfg.n_instances))
    if cfg.output_path:
        write_csv(cfg.output_path, rows, config_hash(cfg))
    return rows


# ---------------------------------------------------------------------------
# benchmark report (bench.py:147-203), GPU form
# ---------------------------------------------------------------------------
def kernel_comparison(isinglink, cfg, n_probe: int = 64) -> dict:
    """The reference's ``_kernel_comparison`` (harness/bench.py:117-144) with
    the CUDA plugin among the kernels.

    ``isinglink`` is the reference package with ``install(isinglink)`` done.
    Every available kernel ("cuda", "ext", "python") times ``detect_cim`` per
    instance through the reference's own code path on the reference bench's
    instances and seeds; each kernel's decisions are compared with "ext".
    The batched slot path (``batched.detect_cim_batch``, P = n_probe in one
    call, FP64-exact and FP32) is timed and compared beside them."""
    from isinglink.harness.bench import _DOM_BENCH, _bench_instances  # reference internals
    cfg.validate()
    instances = _bench_instances(cfg)[:n_probe]
    timings, outputs = {}, {}
    for name in sorted(isinglink.available_kernels()):
        with isinglink.use_kernel(name):
            t0 = time.perf_counter()
            res = [isinglink.detect_cim(inst, cfg.cac, isinglink.derive_seed(cfg.seed, _DOM_BENCH, i))
                   for i, inst in enumerate(instances)]
            timings[name] = (time.perf_counter() - t0) / len(instances)
            outputs[name] = np.array([r.x_hard for r in res])
    H = np.array([inst.H for inst in instances])
    y = np.array([inst.y for inst in instances])
    nv = np.array([inst.noise_var for inst in instances], dtype=np.float64)
    seeds = _seeds([[cfg.seed, _DOM_BENCH, i] for i in range(len(instances))])
    const = instances[0].constellation
    for prec in ("fp64_exact", "fp32"):
        prm = dataclasses.replace(_params(cfg), precision=prec)
        batched.detect_cim_batch(H, y, nv, len(const.points), seeds, prm)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = batched.detect_cim_batch(H, y, nv, len(const.points), seeds, prm)
        torch.cuda.synchronize()
        timings[f"cuda_batched_{prec}"] = (time.perf_counter() - t0) / len(instances)
        lv = torch.as_tensor(const.pam_levels)
        idx = r.x_idx.cpu().long()
        outputs[f"cuda_batched_{prec}"] = (lv[idx[..., 0]] + 1j * lv[idx[..., 1]]).numpy()
    ref = outputs["ext"]
    return {
        "per_instance_s": timings,
        "speedup_vs_ext": {k: timings["ext"] / v for k, v in timings.items()},
        "output_agreement_with_ext": {k: float(np.mean(np.all(v == ref, axis=1)))
                                      for k, v in outputs.items()},
        "n_probe": len(instances),
    }


def run_bench(cfg, precisions=("fp32", "tf32", "fp64_exact"), chunks=(1, 4)) -> dict:
    """Throughput report over a fixed detection batch (bench.py:147-203).

    The reference scales worker processes; here the batch is one launch
    sequence on one GPU, timed device-resident per precision and end to end
    through the chunked host-buffer pipeline (il_detect_cim_host) for each
    chunk count, with outputs compared bitwise across chunk counts (the
    reference's outputs_identical).  The kernel comparison reports the
    agreement of each throughput precision with the FP64-exact kernel."""
    import json
    cfg.validate()
    if cfg.mode != "bench":
        raise ValueError(f"config mode is {cfg.mode!r}, expected bench")
    bench_cfg = dataclasses.replace(cfg, snr_grid_db=(cfg.snr_grid_db[0],))
    b = uplink_batch(bench_cfg, 0, range(cfg.batch_size))
    seeds = _seeds([[cfg.seed, DOM_BENCH, i] for i in range(cfg.batch_size)])
    dev = {k: torch.from_numpy(np.ascontiguousarray(b[k])).cuda() for k in ("H", "y", "noise_var")}
    sd = torch.from_numpy(seeds.view(np.int64)).cuda()
    base = _params(cfg)
    throughput, outputs = {}, {}
    for prec in precisions:
        prm = dataclasses.replace(base, precision=prec)
        batched.detect_cim_batch(dev["H"], dev["y"], dev["noise_var"], cfg.modulation, sd, prm)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = batched.detect_cim_batch(dev["H"], dev["y"], dev["noise_var"], cfg.modulation, sd, prm)
        e1.record()
        torch.cuda.synchronize()
        throughput[prec] = cfg.batch_size / (e0.elapsed_time(e1) / 1e3)
        outputs[prec] = r.x_idx.cpu()
    prm = dataclasses.replace(base, precision=precisions[0])
    pinned = {k: torch.from_numpy(np.ascontiguousarray(b[k])).pin_memory()
              for k in ("H", "y", "noise_var")}
    e2e, host_out = [], []
    for n in chunks:
        batched.detect_cim_host(pinned["H"], pinned["y"], pinned["noise_var"], cfg.modulation,
                                seeds, prm, n_chunks=n)
        t0 = time.perf_counter()
        r = batched.detect_cim_host(pinned["H"], pinned["y"], pinned["noise_var"], cfg.modulation,
                                    seeds, prm, n_chunks=n)
        e2e.append({"n_chunks": n, "wall_time_s": time.perf_counter() - t0,
                    "detections_per_s": cfg.batch_size / (time.perf_counter() - t0)})
        host_out.append(r.x_idx.clone())
    identical = all(torch.equal(host_out[0], o) for o in host_out[1:]) and torch.equal(
        host_out[0], outputs[precisions[0]])
    # critical path: one problem, and one anneal (bench.py:109-126)
    inst = api.MimoInstance(H=b["H"][0], y=b["y"][0], constellation=make_qam(cfg.modulation),
                            noise_var=float(b["noise_var"][0]))
    t0 = time.perf_counter()
    for _ in range(8):
        api.detect_cim(inst, base, int(seeds[0]))
    per_instance = (time.perf_counter() - t0) / 8
    si = api.build_ising(inst, api.detect_mmse(inst).x_hard)
    t0 = time.perf_counter()
    for _ in range(8):
        api.integrate_anneal(si, base, int(seeds[0]))
    per_anneal = (time.perf_counter() - t0) / 8
    ref = outputs.get("fp64_exact")
    comparison = None
    if ref is not None:
        comparison = {f"{p}_decision_agreement_with_fp64_exact":
                      float(torch.all(outputs[p] == ref, dim=(1, 2)).float().mean())
                      for p in precisions if p != "fp64_exact"}
    report = {
        "config_hash": config_hash(cfg),
        "backend": "cuda",
        "device": torch.cuda.get_device_name(),
        "batch_size": cfg.batch_size,
        "n_anneals": cfg.cac.n_anneals,
        "device_detections_per_s": throughput,
        "e2e": e2e,
        "outputs_identical": bool(identical),
        "critical_path": {"per_instance_s": per_instance, "per_anneal_path_s": per_anneal,
                          "n_probe": 8},
        "kernel_comparison": comparison,
        "kernel_launches": _lib.kernel_launches(),
    }
    if cfg.output_path:
        with open(cfg.output_path, "w") as fh:
            json.dump(report, fh, indent=2)
    return report
