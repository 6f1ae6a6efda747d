"""The oracle (oracle/spreadsim_port.py) reproduces the reference's own
outputs bit for bit — pins the checker every GPU parity test relies on.
CPU only."""

import math

import numpy as np
import pytest
from scipy import special, stats

from oracle import spreadsim_port as O
from tests._cases import TRAJECTORY_CASES, golden, graph, trajectory_case


def test_uniform_matches_reference():
    z = golden("rng")
    for (s, k), row in zip(z["cases"], z["uniform"]):
        assert np.array_equal(O.uniform_array(int(s), int(k), z["streams"]), row)
    big = O.uniform_array(77, 5, np.arange(100_000, dtype=np.uint64))
    assert np.array_equal(big[:1000], z["uniform_77_5_head"])
    assert big.sum() == z["uniform_77_5_sum"][0]


def test_derive_seed_matches_reference():
    for s, i, v in golden("rng")["derive"]:
        assert O.derive_seed(int(s), int(i)) == int(v)


def test_erfcx_and_hazards_match_reference():
    z = golden("hazards")
    assert np.array_equal(O.erfcx_piecewise(z["z"]), z["erfcx"])
    assert np.array_equal(O.hazard_lognormal(z["tau"], *z["ei"]), z["h_ei"])
    assert np.array_equal(O.hazard_lognormal(z["tau"], *z["ir"]), z["h_ir"])


def test_shedding_matches_reference():
    import paper_2604_22092_b200 as fs

    z = golden("hazards")
    ir = fs.LogNormalParams(*z["ir"])
    assert np.array_equal(O.shedding_values(fs.Shedding.density_peak(ir), z["tau"]), z["shed_peak"])
    assert np.array_equal(O.shedding_values(fs.Shedding.lognormal_hazard(ir), z["tau"]), z["shed_haz"])


@pytest.mark.parametrize("name", ["er_400", "fixed_400", "ba_2000", "weighted"])
def test_pressure_fold_matches_reference(name):
    z = golden("pressure")
    g = graph(name)
    p = O.fold_pressure(g.row_offsets, g.col_indices, g.weights, z[f"{name}_inf"])
    assert np.array_equal(p, z[f"{name}_p"])


def run_oracle_case(name):
    meta, g, m, cfg, ref = trajectory_case(name)
    st = O.init_state(g, m, cfg, meta["seed"], meta["seed_count"], meta["seed_compartment"])
    cps = {}
    k = 0
    for _ in range(meta["batches"]):
        if not cfg.carry_tau:
            st.tau_prev = cfg.tau_max
        for _ in range(cfg.steps_per_batch):
            O.step(st, g, m, cfg, meta["seed"])
            k += 1
            if k in (1, 10, 50):
                cps[k] = (st.states.astype(np.int32).copy(), st.ages.astype(np.float32).copy())
    return st, cps, ref


@pytest.mark.parametrize("name", TRAJECTORY_CASES)
def test_oracle_trajectory_bit_exact(name):
    st, cps, ref = run_oracle_case(name)
    clocks = np.array([c for c, _, _ in st.log])
    taus = np.array([t for _, t, _ in st.log])
    counts = np.array([c for _, _, c in st.log])
    assert np.array_equal(counts, ref["counts"])
    assert np.array_equal(clocks, ref["clock"])
    assert np.array_equal(taus, ref["tau"])
    assert np.array_equal(st.states.astype(np.int32), ref["states"])
    assert np.array_equal(st.ages.astype(np.float32), ref["ages"])
    assert np.array_equal(st.infectivity.astype(np.float32), ref["infectivity"])
    assert np.array_equal(st.rates, ref["rates"])
    assert np.array_equal(st.pressure, ref["pressure"])
    for k, (s, a) in cps.items():
        assert np.array_equal(s, ref[f"cp{k}_states"]) and np.array_equal(a, ref[f"cp{k}_ages"])


# ---- unpinned extensions, pinned against independent references --------

PHILOX_KAT = [  # Random123 kat_vectors, philox4x32_10: (ctr, key, expected)
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,expected", PHILOX_KAT)
def test_philox_known_answers(ctr, key, expected):
    out = O.philox4x32_10(*(np.array([c], dtype=np.uint64) for c in ctr), *key)
    assert tuple(int(x[0]) for x in out) == expected


def test_philox_uniform_quality():
    u = O.philox_uniform_array(2024, 3, np.arange(200_000, dtype=np.uint64))
    assert abs(u.mean() - 0.5) < 0.003
    counts, _ = np.histogram(u, bins=256, range=(0, 1))
    e = u.size / 256
    assert stats.chi2.sf(((counts - e) ** 2 / e).sum(), 255) > 1e-6


def test_weibull_erlang_hazards_match_scipy():
    tau = np.linspace(0.05, 60.0, 500)
    k, lam = 1.247568, 5.365966
    hw = O.hazard_weibull(tau, k, lam)
    ref_w = stats.weibull_min.pdf(tau, k, scale=lam) / stats.weibull_min.sf(tau, k, scale=lam)
    assert np.allclose(hw, ref_w, rtol=1e-10)
    he = O.hazard_erlang(tau, 3, 0.4)
    ref_e = stats.gamma.pdf(tau, 3, scale=1 / 0.4) / stats.gamma.sf(tau, 3, scale=1 / 0.4)
    assert np.allclose(he, ref_e, rtol=1e-10)
    assert O.hazard_weibull(np.array([0.0]), k, lam)[0] == 0.0
    assert O.hazard_erlang(np.array([0.0]), 1, 0.4)[0] == 0.4
