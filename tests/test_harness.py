"""The GPU harness (paper_2510_01579_b200/harness.py) against the reference's
own sweep / heatmap CSVs (tests/golden/*.csv, written by the reference's
harness via tests/golden/make_golden.py; the .cfg next to each is the
reference's canonical config text)."""

import csv
import os

import numpy as np
import pytest

from conftest import GOLDEN

CASES = ["sweep_up_4x4_qpsk", "sweep_up_8x8_16qam", "sweep_down_4x4_16qam", "heatmap_8x8_16qam"]


def _read(stem):
    with open(os.path.join(GOLDEN, stem + ".csv")) as fh:
        lines = fh.read().splitlines()
    footer = lines[-1]
    assert footer.startswith("# config_hash=")
    rows = list(csv.DictReader(lines[:-1]))
    with open(os.path.join(GOLDEN, stem + ".cfg")) as fh:
        cfg_text = fh.read()
    return rows, footer.split("=", 1)[1], cfg_text


@pytest.mark.parametrize("stem", CASES)
def test_config_hash_matches_reference(stem):
    from paper_2510_01579_b200 import harness
    _, want, text = _read(stem)
    cfg = harness.config_from_text(text)
    assert harness.config_hash(cfg) == want
    assert harness.format_config(cfg) == text


def test_config_validation():
    import dataclasses

    from paper_2510_01579_b200 import harness
    cfg = harness.ExperimentConfig()
    cfg.validate()
    for bad in (dict(mode="x"), dict(detectors=("foo",)), dict(n_stages=0), dict(budget=0.0)):
        with pytest.raises(ValueError):
            dataclasses.replace(cfg, **bad).validate()
    with pytest.raises(ValueError):
        harness.config_from_text("n_r 4")


def test_write_csv_layout(tmp_path):
    from paper_2510_01579_b200 import harness
    rows = [harness.SweepRow(10.0, "cim", 0.25, 0.125, 1.5, 0.0, 0.01, 8)]
    p = tmp_path / "x.csv"
    harness.write_csv(str(p), rows, "abc")
    assert p.read_text() == ("snr_db,detector,ser,ber,mean_energy,mean_diverged,wall_time_s,"
                             "n_trials\n10.0,cim,0.25,0.125,1.5,0.0,0.01,8\n# config_hash=abc\n")
    with pytest.raises(ValueError):
        harness.write_csv(str(p), [], "abc")


@pytest.mark.gpu
@pytest.mark.parametrize("stem", CASES)
def test_gpu_harness_reproduces_reference_csv(stem, tmp_path, built_lib):
    import dataclasses

    from paper_2510_01579_b200 import harness
    want, hash_, text = _read(stem)
    cfg = dataclasses.replace(harness.config_from_text(text), output_path=str(tmp_path / "o.csv"))
    fn = {"uplink_sweep": harness.run_detection_sweep,
          "downlink_sweep": harness.run_precoding_sweep,
          "heatmap": harness.run_integration_heatmap}[cfg.mode]
    fn(cfg)
    got, got_hash, _ = _read_path(str(tmp_path / "o.csv"))
    assert got_hash == hash_
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for k in w:
            if k == "wall_time_s":
                continue
            if k == "mean_energy":
                np.testing.assert_allclose(float(g[k]), float(w[k]), rtol=1e-12)
            else:
                assert g[k] == w[k], (k, g, w)


def _read_path(path):
    with open(path) as fh:
        lines = fh.read().splitlines()
    return list(csv.DictReader(lines[:-1])), lines[-1].split("=", 1)[1], None


@pytest.mark.gpu
def test_gpu_ml_matches_reference_fixtures(built_lib):
    from conftest import load_golden
    from paper_2510_01579_b200 import batched
    for name in ("ml4x4_qpsk_8db", "ml3x2_16qam_12db"):
        d = load_golden(f"{name}.npz")
        x, e = batched.ml_batch(d["H"], d["y"], int(d["order"]))
        assert np.array_equal(x.cpu().numpy(), d["x_ml"])
        np.testing.assert_allclose(e.cpu().numpy(), d["e_ml"], rtol=1e-12)


@pytest.mark.gpu
def test_gpu_bench_report(built_lib):
    import dataclasses

    from paper_2510_01579_b200 import harness
    cfg = dataclasses.replace(harness.ExperimentConfig(), mode="bench", batch_size=256,
                              snr_grid_db=(20.0,))
    rep = harness.run_bench(cfg, chunks=(1, 3))
    assert rep["outputs_identical"]
    assert rep["backend"] == "cuda" and rep["batch_size"] == 256
    assert all(v > 0 for v in rep["device_detections_per_s"].values())
    assert rep["kernel_comparison"]["fp32_decision_agreement_with_fp64_exact"] >= 0.9
