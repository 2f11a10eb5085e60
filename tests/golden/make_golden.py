"""Generate the golden fixtures from the REAL reference (build container only).

Run:  python tests/golden/make_golden.py          (needs /root/reference and
      `make -C oracle ref`, i.e. the compiled reference kernel in oracle/_ref)

Imports the reference package from /root/reference/pkg/src with its compiled
Cython kernel (oracle/_ref) injected as ``isinglink._kernel`` so the "ext"
backend is active, exactly as an installed reference would run.  The outputs
are small .npz files committed under tests/golden/; the GPU box never reads
/root/reference — it only reads these fixtures.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import isinglink_oracle as orc  # noqa: E402


def import_reference():
    mod = orc.ref_kernel_module()
    if mod is None:
        raise SystemExit("build the reference kernel first: make -C oracle ref")
    sys.modules["isinglink._kernel"] = mod
    sys.path.insert(0, "/root/reference/pkg/src")
    import isinglink  # noqa: F401
    assert isinglink.kernel_backend() == "ext"
    return isinglink


def level_idx(x, levels):
    x = np.asarray(x)
    return np.stack([orc.level_index(x.real, levels), orc.level_index(x.imag, levels)], -1)


def main():
    il = import_reference()
    from isinglink.harness.config import ExperimentConfig
    from isinglink.harness.sweeps import make_uplink_instance
    from isinglink import solver as ref_solver

    # ---- 1. seeds / PCG64 streams -------------------------------------
    parts = [(0,), (1,), (2**32 - 1,), (2**32,), (2**64 - 1,), (1, 2, 3), (7, 0, 0),
             (123456789012345, 5), (1, 1, 4, 17, 3), (2**40 + 3, 2**33, 0, 9),
             (0, 0, 0, 0, 0, 0), (1, 4, 0), (3, 2**31)]
    flat = np.zeros((len(parts), 8), np.uint64)
    lens = np.zeros(len(parts), np.int64)
    for i, p in enumerate(parts):
        flat[i, :len(p)] = p
        lens[i] = len(p)
    derived = np.array([il.derive_seed(*p) for p in parts], np.uint64)
    x0_seeds = np.array([0, 1, 2**32 - 1, 2**32, il.derive_seed(9, 0), il.derive_seed(1, 2, 3)],
                        np.uint64)
    x0 = np.stack([np.random.default_rng(int(s)).uniform(-0.1, 0.1, 65) for s in x0_seeds])
    raw64 = np.stack([np.random.default_rng(int(s)).bit_generator.random_raw(16)
                      for s in x0_seeds]).astype(np.uint64)
    np.savez_compressed(os.path.join(HERE, "seeds.npz"), parts=flat, lens=lens,
                        derived=derived, x0_seeds=x0_seeds, x0=x0, raw64=raw64)

    # ---- 2. run_anneals (ext backend) ----------------------------------
    from isinglink import CacParams, build_ising, detect_mmse
    rng = np.random.default_rng(2024)
    cases = []
    specs = [  # (n_r, n_t, order, snr, params overrides, n_batch)
        (8, 8, 16, 20.0, {}, 32),
        (4, 4, 4, 15.0, {}, 32),
        (16, 16, 16, 20.0, {}, 32),
        (16, 16, 64, 25.0, {}, 16),
        (8, 8, 16, 20.0, dict(dt=0.16, n_steps=16), 16),
        (8, 8, 16, 20.0, dict(dt=10.0, n_steps=64), 8),
        (8, 8, 16, 20.0, dict(f_mvm=3, n_steps=100), 8),
        (3, 3, 4, 10.0, dict(f_mvm=1, n_steps=40), 5),
        (8, 8, 16, 20.0, dict(p=1.0, a=0.0, diverge_threshold=0.001), 8),
        (8, 8, 16, 20.0, dict(e_floor=1e-4, n_steps=200), 4),
        (16, 16, 16, 20.0, dict(dt=0.01, f_mvm=1, n_steps=256), 8),
    ]
    for k, (nr, nt, order, snr, over, nb) in enumerate(specs):
        levels, spacing = orc.qam(order)
        H, y, s2, _ = orc.uplink_instance(77, snr, 0, k, nr, nt, order)
        inst = il.MimoInstance(H=H, y=y, constellation=il.make_qam(order), noise_var=s2)
        si = build_ising(inst, detect_mmse(inst).x_hard)
        prm = CacParams(**over)
        x0c = rng.uniform(-prm.init_amplitude, prm.init_amplitude, (nb, si.spin_count))
        out = ref_solver._impl.run_anneals(si.G, si.g_diag, si.b, x0c, prm.dt, prm.p, prm.a,
                                           prm.zeta, si.eps_scale, prm.e_floor, prm.f_mvm,
                                           prm.n_steps, prm.diverge_threshold)
        cases.append(dict(G=si.G, g=si.g_diag, b=si.b, x0=x0c,
                          prm=np.array([prm.dt, prm.p, prm.a, prm.zeta, si.eps_scale,
                                        prm.e_floor, prm.f_mvm, prm.n_steps,
                                        prm.diverge_threshold]),
                          spins=out[0], diverged=out[1], steps=out[2], mvms=out[3]))
    np.savez_compressed(os.path.join(HERE, "anneals.npz"),
                        **{f"c{k}_{name}": v for k, c in enumerate(cases) for name, v in c.items()},
                        n_cases=len(cases))

    # ---- 3. detection sets (sweep instances, ext backend) -----------------
    sets = [  # name, n_r, n_t, order, snr, n_trials
        ("d8x8_qpsk_10db", 8, 8, 4, 10.0, 96),
        ("d8x8_16qam_20db", 8, 8, 16, 20.0, 96),
        ("d16x16_16qam_20db", 16, 16, 16, 20.0, 64),
        ("d16x16_64qam_25db", 16, 16, 64, 25.0, 48),
    ]
    for name, nr, nt, order, snr, ntr in sets:
        cfg = ExperimentConfig(n_r=nr, n_t=nt, modulation=order, snr_grid_db=(snr,),
                               n_trials=ntr, seed=1)
        levels = il.make_qam(order).pam_levels
        Hs, ys, s2s, truth, seeds = [], [], [], [], []
        xm, em, Gs, bs, offs, epss = [], [], [], [], [], []
        xo, eo, src, aidx, ndiv = [], [], [], [], []
        for t in range(ntr):
            inst = make_uplink_instance(cfg, 0, t)
            seed = il.derive_seed(cfg.seed, 1, 0, t, 3)
            m = il.detect_mmse(inst)
            si = il.build_ising(inst, m.x_hard)
            r = il.detect_cim(inst, cfg.cac, seed)
            Hs.append(inst.H); ys.append(inst.y); s2s.append(inst.noise_var)
            truth.append(level_idx(inst.truth, levels)); seeds.append(seed)
            xm.append(level_idx(m.x_hard, levels)); em.append(m.energy)
            Gs.append(si.G); bs.append(si.b); offs.append(si.offset); epss.append(si.eps_scale)
            xo.append(level_idx(r.x_hard, levels)); eo.append(r.energy)
            src.append(1 if r.source == "anneal" else 0); aidx.append(r.anneal_index)
            ndiv.append(r.diverged_count)
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), H=np.array(Hs), y=np.array(ys),
            noise_var=np.array(s2s), truth=np.array(truth), seed=np.array(seeds, np.uint64),
            order=order, x_mmse=np.array(xm), e_mmse=np.array(em), G=np.array(Gs),
            b=np.array(bs), offset=np.array(offs), eps_scale=np.array(epss),
            x_hat=np.array(xo), energy=np.array(eo), source=np.array(src),
            anneal_index=np.array(aidx), diverged=np.array(ndiv))

    # ---- 4. VPP (downlink sweep instances, ext backend) --------------------
    nr, nt, order, ntr, snr_idx = 8, 8, 16, 64, 0
    const = il.make_qam(order)
    tau = il.default_tau(const)
    Hs, us, vs, pw, xs, seeds = [], [], [], [], [], []
    for t in range(ntr):
        H = il.sample_channel(nr, nt, il.derive_seed(1, 2, snr_idx, t, 0))
        rr = np.random.default_rng(il.derive_seed(1, 2, snr_idx, t, 1))
        u = const.points[rr.integers(0, const.order, nr)]
        seed = il.derive_seed(1, 2, snr_idx, t, 3)
        res = il.precode_vpp(H, u, P=float(nr), tau=tau, params=il.CacParams(), seed=seed)
        Hs.append(H); us.append(u); vs.append(res.v); pw.append(res.unnormalized_power)
        xs.append(res.x_transmit); seeds.append(seed)
    np.savez_compressed(os.path.join(HERE, "vpp8x8_16qam.npz"), H=np.array(Hs), u=np.array(us),
                        v=np.array(vs), power=np.array(pw), x=np.array(xs),
                        seed=np.array(seeds, np.uint64), tau=tau, P=float(nr), order=order)
    print("golden fixtures written to", HERE)


def main_multi():
    """MMGaP-E (detect_cim_multi, detector.py:85-134), MMSE-SIC
    (linear.py:78-106) and brute-force ML (linear.py:109-144) fixtures."""
    il = import_reference()
    from isinglink.harness.config import ExperimentConfig
    from isinglink.harness.sweeps import make_uplink_instance
    sets = [  # name, n_r, n_t, order, snr, n_trials, n_stages
        ("m8x8_16qam_15db", 8, 8, 16, 15.0, 48, 2),
        ("m16x16_16qam_20db", 16, 16, 16, 20.0, 32, 1),
    ]
    src_code = {"mmse": 0, "anneal": 1, "mmse_sic": 2}
    for name, nr, nt, order, snr, ntr, ns in sets:
        cfg = ExperimentConfig(n_r=nr, n_t=nt, modulation=order, snr_grid_db=(snr,),
                               n_trials=ntr, seed=3)
        levels = il.make_qam(order).pam_levels
        rec = {k: [] for k in ("H", "y", "noise_var", "seed", "x_sic", "e_sic", "x_hat",
                               "energy", "source", "anneal_index", "diverged")}
        for t in range(ntr):
            inst = make_uplink_instance(cfg, 0, t)
            seed = il.derive_seed(cfg.seed, 1, 0, t, 3)
            sic = il.detect_mmse_sic(inst)
            r = il.detect_cim_multi(inst, cfg.cac, n_stages=ns, seed=seed)
            rec["H"].append(inst.H); rec["y"].append(inst.y); rec["noise_var"].append(inst.noise_var)
            rec["seed"].append(seed)
            rec["x_sic"].append(level_idx(sic.x_hard, levels)); rec["e_sic"].append(sic.energy)
            rec["x_hat"].append(level_idx(r.x_hard, levels)); rec["energy"].append(r.energy)
            rec["source"].append(src_code[r.source]); rec["anneal_index"].append(r.anneal_index)
            rec["diverged"].append(r.diverged_count)
        out = {k: np.array(v) for k, v in rec.items() if k != "seed"}
        out["seed"] = np.array(rec["seed"], dtype=np.uint64)  # 64-bit ints, no float detour
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), order=order, n_stages=ns, **out)
    # brute-force ML (small search spaces)
    specs = [("ml4x4_qpsk_8db", 4, 4, 4, 8.0, 24), ("ml3x2_16qam_12db", 3, 2, 16, 12.0, 24)]
    for name, nr, nt, order, snr, ntr in specs:
        cfg = ExperimentConfig(n_r=nr, n_t=nt, modulation=order, snr_grid_db=(snr,),
                               n_trials=ntr, seed=4)
        levels = il.make_qam(order).pam_levels
        Hs, ys, xs, es = [], [], [], []
        for t in range(ntr):
            inst = make_uplink_instance(cfg, 0, t)
            r = il.detect_ml(inst)
            Hs.append(inst.H); ys.append(inst.y)
            xs.append(level_idx(r.x_hard, levels)); es.append(r.energy)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), H=np.array(Hs), y=np.array(ys),
                            x_ml=np.array(xs), e_ml=np.array(es), order=order)
    print("MMGaP-E / SIC / ML fixtures written to", HERE)


HARNESS_CASES = [  # (file stem, config overrides) -> reference CSV + config text
    ("sweep_up_4x4_qpsk", dict(mode="uplink_sweep", n_r=4, n_t=4, modulation=4,
                               snr_grid_db=(5.0, 15.0), n_trials=48, n_stages=2, seed=7,
                               detectors=("mmse", "mmse_sic", "ml", "cim", "cim_multi"))),
    ("sweep_up_8x8_16qam", dict(mode="uplink_sweep", n_r=8, n_t=8, modulation=16,
                                snr_grid_db=(15.0, 25.0), n_trials=32, seed=8,
                                detectors=("mmse", "mmse_sic", "cim", "cim_multi"))),
    ("sweep_down_4x4_16qam", dict(mode="downlink_sweep", n_r=4, n_t=4, modulation=16,
                                  snr_grid_db=(10.0, 20.0), n_trials=24, seed=9)),
    ("heatmap_8x8_16qam", dict(mode="heatmap", n_r=8, n_t=8, modulation=16,
                               snr_grid_db=(10.0,), n_instances=32, seed=10)),
]


def main_harness():
    """The reference's own sweep / heatmap CSVs (harness/sweeps.py, heatmap.py)."""
    import dataclasses
    import_reference()
    from isinglink.harness.config import ExperimentConfig, format_config
    from isinglink.harness.heatmap import run_integration_heatmap
    from isinglink.harness.sweeps import run_detection_sweep, run_precoding_sweep
    run = {"uplink_sweep": run_detection_sweep, "downlink_sweep": run_precoding_sweep,
           "heatmap": run_integration_heatmap}
    for stem, over in HARNESS_CASES:
        cfg = dataclasses.replace(ExperimentConfig(), output_path=os.path.join(HERE, stem + ".csv"),
                                  **over)
        run[cfg.mode](cfg)
        with open(os.path.join(HERE, stem + ".cfg"), "w") as fh:
            fh.write(format_config(dataclasses.replace(cfg, output_path="")))
    print("harness fixtures written to", HERE)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "harness":
        main_harness()
        raise SystemExit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "multi":
        main_multi()
    else:
        main()
        main_multi()
        main_harness()
