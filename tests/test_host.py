"""CPU: host-side logic of the package (parameters, alphabets, index formats,
sharding rule) against the oracle / the reference's documented rules."""

import dataclasses

import numpy as np
import pytest

from oracle import isinglink_oracle as orc
from paper_2510_01579_b200 import channel
from paper_2510_01579_b200.params import CacParams, to_c
from paper_2510_01579_b200.shard import partition_blocks, slot_shard


class TestCacParams:
    def test_defaults(self):
        p = CacParams()
        p.validate()
        assert p.dt * p.n_steps == pytest.approx(2.56)
        assert p.f_mvm == 2 and p.n_anneals == 32

    @pytest.mark.parametrize("kwargs", [
        {"dt": 0.0}, {"f_mvm": 0}, {"n_steps": 0}, {"n_anneals": 0}, {"e_floor": 0.0},
        {"init_amplitude": 0.0}, {"eps": -1.0}, {"diverge_threshold": 0.5},
        {"precision": "fp8"},
    ])
    def test_invalid(self, kwargs):
        with pytest.raises(ValueError):
            dataclasses.replace(CacParams(), **kwargs).validate()

    def test_tiny_threshold_legal_when_dynamics_allow(self):
        dataclasses.replace(CacParams(), p=1.0, a=0.0, diverge_threshold=0.001).validate()

    def test_c_struct(self):
        c = to_c(CacParams(eps=0.25, precision="fp64_exact"))
        assert c.eps == 0.25 and c.precision == 0 and c.n_anneals == 32
        assert to_c(CacParams()).eps < 0  # auto

    def test_accepts_reference_like_params(self):
        @dataclasses.dataclass(frozen=True)
        class Ref:
            p: float = 1.5
            a: float = 0.5
            zeta: float = 1.0
            eps: float = None
            dt: float = 0.02
            f_mvm: int = 2
            n_steps: int = 128
            n_anneals: int = 32
            diverge_threshold: float = 10.0
            e_floor: float = 1e-6
            init_amplitude: float = 0.1

            def validate(self):
                pass
        assert to_c(Ref()).precision in (0, 1, 2)


class TestChannel:
    @pytest.mark.parametrize("order", [4, 16, 64, 256])
    def test_qam_matches_oracle(self, order):
        c = channel.make_qam(order)
        lv, sp = orc.qam(order)
        assert np.array_equal(c.pam_levels, lv) and c.spacing == sp
        assert np.mean(np.abs(c.points) ** 2) == pytest.approx(1.0)

    def test_bad_order(self):
        with pytest.raises(ValueError):
            channel.make_qam(8)

    def test_index_roundtrip_and_projection(self, rng):
        c = channel.make_qam(64)
        x = rng.standard_normal(500) + 1j * rng.standard_normal(500)
        idx = channel.to_indices(x, c)
        assert idx.dtype == np.uint8 and idx.shape == (500, 2)
        assert np.array_equal(channel.from_indices(idx, c), orc.project(x, c.pam_levels))
        pts = channel.from_indices(idx, c)
        assert np.array_equal(channel.project_to_constellation(pts, c), pts)

    def test_midpoint_ties_go_down(self):
        c = channel.make_qam(16)
        mid = (c.pam_levels[1] + c.pam_levels[2]) / 2
        assert channel.to_indices(np.array([mid + 1j * mid]), c)[0].tolist() == [1, 1]

    def test_bit_errors_gray(self, rng):
        c = channel.make_qam(16)
        a = c.points[rng.integers(0, 16, 200)]
        b = c.points[rng.integers(0, 16, 200)]
        want = orc.bit_errors(channel.to_indices(a, c), channel.to_indices(b, c))
        assert channel.bit_errors(a, b, c) == want
        assert channel.symbol_errors(a, a) == 0

    def test_synthetic_generators_match_oracle(self):
        H, y, s2, truth = orc.uplink_instance(1, 20.0, 0, 3, 8, 8, 16)
        Hc = channel.sample_channel(8, 8, orc.seed_of(1, 1, 0, 3, 0))
        assert np.array_equal(H, Hc)
        c = channel.make_qam(16)
        x = channel.from_indices(truth, c)
        yc, s2c = channel.transmit(H, x, 20.0, orc.seed_of(1, 1, 0, 3, 2))
        assert np.array_equal(y, yc) and s2 == s2c


class TestSharding:
    def test_partition_rule(self):
        assert partition_blocks(10, 3) == [(0, 3), (3, 6), (6, 10)]
        assert partition_blocks(2, 5) == [(0, 1), (1, 2)]
        with pytest.raises(ValueError):
            partition_blocks(3, 0)

    @pytest.mark.parametrize("world", [1, 2, 4, 8])
    def test_slot_shards_tile_the_slot(self, world):
        shards = [slot_shard(273, r, world) for r in range(world)]
        assert shards[0].re_start == 0 and shards[-1].re_stop == 273 * 12 * 14
        for a, b in zip(shards, shards[1:]):
            assert a.re_stop == b.re_start
        assert sum(s.local_res for s in shards) == 45864
        if world == 8:
            assert [s.sc_stop - s.sc_start for s in shards] == [409] * 7 + [413]
