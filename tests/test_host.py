"""Host-side logic of the drop-in API (CPU only): generators identical to
the reference, CSR validation, config validation, model packing, records."""

import math

import numpy as np
import pytest

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import _lib, errors
from paper_2604_22092_b200.graph import Strategy, resolve_strategy
from paper_2604_22092_b200.models import model_descriptor
from tests._cases import MANIFEST, csr_sha, golden, graph


@pytest.mark.parametrize("name", list(MANIFEST["graphs"]))
def test_generators_bit_identical_to_reference(name):
    assert csr_sha(graph(name)) == MANIFEST["graphs"][name]["sha256"]


def test_build_csr_validation():
    with pytest.raises(errors.SelfLoopError):
        fs.build_csr([(0, 0, 1.0)], 2)
    with pytest.raises(errors.DuplicateEdgeError):
        fs.build_csr([(0, 1, 1.0), (0, 1, 2.0)], 2)
    with pytest.raises(errors.NegativeWeightError):
        fs.build_csr([(0, 1, -1.0)], 2)
    with pytest.raises(errors.IndexOutOfRangeError):
        fs.build_csr([(0, 5, 1.0)], 2)
    g = fs.build_csr([(2, 0, 1.0), (1, 0, 0.5), (0, 1, 2.0)], 3)
    assert list(g.row_offsets) == [0, 2, 3, 3] and list(g.col_indices) == [1, 2, 0]
    assert g.weights.tolist() == [0.5, 1.0, 2.0]
    e = fs.decompose(g)
    assert np.array_equal(fs.decompose(fs.build_csr(e, 3)), e)
    t = fs.transpose(g)
    assert np.array_equal(fs.transpose(t).col_indices, g.col_indices)


def test_strategy_dispatch_thresholds():
    S = fs.DegreeStats
    assert fs.select_strategy(S(10.0, 39, 3.9)) == Strategy.PER_NODE
    assert fs.select_strategy(S(10.0, 40, 4.0)) == Strategy.LANE_CHUNKED
    assert fs.select_strategy(S(10.0, 500, 50.0)) == Strategy.EDGE_MERGE
    assert resolve_strategy(graph("fixed_400"), Strategy.AUTO) == Strategy.PER_NODE
    assert resolve_strategy(graph("ba_2000"), Strategy.AUTO) == Strategy.LANE_CHUNKED  # rho 17.9
    assert resolve_strategy(graph("ba_1e4"), Strategy.AUTO) == Strategy.LANE_CHUNKED  # rho 44.6
    assert resolve_strategy(graph("ba_1e5"), Strategy.AUTO) == Strategy.EDGE_MERGE
    assert resolve_strategy(fs.build_csr([], 4), Strategy.AUTO) == Strategy.PER_NODE


def test_config_validation():
    with pytest.raises(ValueError):
        fs.RenewalConfig(epsilon=0.0)
    with pytest.raises(ValueError):
        fs.RenewalConfig(tau_max=0.0)
    with pytest.raises(ValueError):
        fs.RenewalConfig(steps_per_batch=0)
    with pytest.raises(ValueError):
        fs.RenewalConfig(rng="mt19937")
    assert fs.RenewalConfig(0.05, 0.2).epsilon == 0.05


def test_model_descriptor_packing():
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    d = model_descriptor(m)
    assert (d.num_compartments, d.edge_from, d.edge_to, d.infectious) == (4, 0, 1, 2)
    assert [d.comp[i].succ for i in range(4)] == [1, 2, 3, 3]
    assert [d.comp[i].terminal for i in range(4)] == [0, 0, 0, 1]
    assert [d.comp[i].hazard for i in range(4)] == [_lib.HZ_NONE, _lib.HZ_LOGNORMAL, _lib.HZ_LOGNORMAL, _lib.HZ_NONE]
    assert d.comp[1].p0 == pytest.approx(math.log(4.0)) and d.comp[1].p1 == pytest.approx(0.66805, abs=1e-5)
    w = model_descriptor(fs.seir_weibull_erlang(0.25))
    assert (w.comp[1].hazard, w.comp[2].hazard, w.comp[2].p0) == (_lib.HZ_WEIBULL, _lib.HZ_ERLANG, 3.0)
    s = model_descriptor(fs.sis_model(0.3, 0.1))
    assert (s.comp[1].hazard, s.comp[1].p0, s.comp[1].succ, s.comp[0].terminal) == (_lib.HZ_EXPONENTIAL, 0.1, 0, 0)


def test_weibull_moment_inversion():
    p = fs.weibull_from_mean_median(5.0, 4.0)
    assert p.k == pytest.approx(1.247568, abs=1e-5) and p.lam == pytest.approx(5.365966, abs=1e-5)
    assert p.mean == pytest.approx(5.0, rel=1e-9) and p.median == pytest.approx(4.0, rel=1e-9)


def test_derive_seed_host_matches_reference():
    for s, i, v in golden("rng")["derive"]:
        assert fs.derive_seed(int(s), int(i)) == int(v)


def test_make_record_last_value_interpolation():
    rec = fs.make_record([0.0, 1.0, 2.5], [[10, 0, 0], [6, 4, 0], [2, 3, 5]], ("S", "I", "R"), 10, 3.0, grid_points=7)
    assert np.allclose(rec.fractions.sum(axis=0), 1.0)
    assert rec.fraction_of("I").tolist() == [0.0, 0.0, 0.4, 0.4, 0.4, 0.3, 0.3]
    assert rec.summary["peak_I"] == 0.4 and rec.summary["peak_I_time"] == 1.0 and rec.summary["final_R"] == 0.5
