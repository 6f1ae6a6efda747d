"""Full-size (BASELINE C2 / C3 shape, N = 1e6) checks on the GPU.

The oracle finishes a few steps at this size, so the first steps are
compared exactly; the long run is checked through size-independent
properties: conservation, monotone absorbing count, the tau cap invariant,
determinism, and strategy / encoding neutrality (identical states).
"""

import numpy as np
import pytest

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200.graph import Strategy
from oracle import spreadsim_port as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
N = 1_000_000


@pytest.fixture(scope="module")
def c2_graph():
    return fs.gen_fixed_degree(N, 10, seed=1)


def test_c2_first_steps_match_oracle(c2_graph):
    g, m = c2_graph, fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig()
    ref = O.init_state(g, m, cfg, 7)
    st = fs.init_renewal_state(g, m, cfg, 7)
    assert np.array_equal(st.states, ref.states)
    for _ in range(12):
        fs.renewal_step(st, g, m, cfg, 7)
        O.step(ref, g, m, cfg, 7)
    assert np.array_equal(st.counts, ref.counts)
    assert np.array_equal(st.states, ref.states)
    assert np.array_equal(st.ages, ref.ages)
    assert np.array_equal(st.pressure, ref.pressure)
    assert st.clock == ref.clock and st.tau_prev == ref.tau_prev


def test_c2_long_run_properties(c2_graph):
    g, m = c2_graph, fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig()
    finals = []
    for strategy in (Strategy.PER_NODE, Strategy.EDGE_MERGE):
        cfg_s = fs.RenewalConfig(strategy=strategy)
        st = fs.init_renewal_state(g, m, cfg_s, 7)
        last_r = 0
        for _ in range(8):
            rec = []
            fs.run_batch(st, g, m, cfg_s, 7, recorder=rec)
            counts = np.array([c for _, c in rec])
            assert (counts.sum(axis=1) == N).all()
            assert (np.diff(counts[:, 3]) >= 0).all() and counts[0, 3] >= last_r
            last_r = counts[-1, 3]
            assert float(st.rates.max()) * st.tau_prev <= cfg.epsilon + cfg.delta * cfg.tau_max + 1e-12
        finals.append((st.states.copy(), st.ages.copy(), st.counts.copy(), st.clock))
    assert np.array_equal(finals[0][0], finals[1][0]) and np.array_equal(finals[0][1], finals[1][1])
    assert finals[0][3] == finals[1][3]


def test_c3_ba_merge_vs_oracle():
    g = fs.gen_barabasi_albert(200_000, 5, seed=1)
    m = fs.seir_weibull_erlang(0.25)
    cfg = fs.RenewalConfig()
    assert fs.select_strategy(fs.degree_stats(g)) == Strategy.EDGE_MERGE
    ref = O.init_state(g, m, cfg, 7)
    st = fs.init_renewal_state(g, m, cfg, 7)
    for _ in range(60):
        O.step(ref, g, m, cfg, 7)
    fs.run_batch(st, g, m, fs.RenewalConfig(steps_per_batch=60), 7)
    assert np.array_equal(st.counts, ref.counts)
    assert np.array_equal(st.states.astype(np.int32), ref.states.astype(np.int32))
    assert np.allclose(st.ages, ref.ages, rtol=1e-5, atol=0)


@pytest.fixture(scope="module")
def c3_oracle():
    g = fs.gen_barabasi_albert(N, 5, seed=1)
    m = fs.seir_weibull_erlang(0.25)
    cfg = fs.RenewalConfig(steps_per_batch=20)
    ref = O.init_state(g, m, cfg, 7)
    for _ in range(3):
        O.run_batch(ref, g, m, cfg, 7)
    return g, m, ref


@pytest.mark.parametrize("gather", ["auto", "f32", "count"])
def test_c3_full_size_ba_weibull_erlang_vs_oracle(c3_oracle, gather):
    """BASELINE C3 at its own size: BA N=1e6, m=5, seed 1, Weibull/Erlang,
    60 steps (graph-replayed batches) against the oracle port, through the
    default incremental counts, the one-launch f32 edge-merge fold and the
    count-gather merge.  Counts per step, states, ages and clock exact."""
    g, m, ref = c3_oracle
    cfg = fs.RenewalConfig(steps_per_batch=20, gather=gather)
    assert fs.select_strategy(fs.degree_stats(g)) == Strategy.EDGE_MERGE
    st = fs.init_renewal_state(g, m, cfg, 7)
    counts = []
    for _ in range(3):
        rec = []
        fs.run_batch(st, g, m, cfg, 7, recorder=rec)
        counts += [c for _, c in rec]
    assert np.array_equal(np.array(counts), np.array([c for _, _, c in ref.log]))
    assert np.array_equal(st.states.astype(np.int32), ref.states.astype(np.int32))
    assert np.array_equal(st.ages, ref.ages)
    assert st.clock == ref.clock and st.tau_prev == ref.tau_prev


def _oracle_step_chunked(states, ages, inf32, ro, col, tau, k, m, seed, mixed, chunk=10_000_000):
    """One oracle step over all N nodes, computed in row chunks with
    oracle.step_rows (the partition oracle; same arithmetic as O.step) so
    the host temporaries stay ~1e8-edge sized at N = 1e8."""
    n = states.size
    s_out = np.empty_like(states)
    a_out = np.empty_like(ages)
    i_out = np.empty(n, np.float32)
    mx, delta = 0.0, np.zeros(m.num_compartments, np.int64)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        ro_l = ro[lo:hi + 1] - ro[lo]
        s, a, inf, mx_l, d = O.step_rows(states[lo:hi], ages[lo:hi], ro_l, col[ro[lo]:ro[hi]], inf32, lo, tau, k, m,
                                         seed, mixed)
        s_out[lo:hi], a_out[lo:hi], i_out[lo:hi] = s, a, inf
        mx, delta = max(mx, mx_l), delta + d
    return s_out, a_out, i_out, mx, delta


def test_c4_full_size_mixed_vs_oracle():
    """BASELINE C4 at its own size: the device uniform-degree graph at
    N = 1e8 (k = 10), mixed-precision storage, 3 steps against the oracle
    on the same CSR (copied to the host).  States, ages (f16), counts,
    clock and tau exact after every step (R/renewal.py:483-580, mixed
    storage :358-367, :567-575)."""
    n = 100_000_000
    g = fs.gen_fixed_degree_device(n, 10, seed=1)
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig(mixed_precision=True)
    st = fs.init_renewal_state(g, m, cfg, 7)
    ro, col = np.asarray(g.row_offsets, np.int64), g.col_indices
    ref = O.init_state(g, m, cfg, 7)
    assert np.array_equal(st.states, ref.states)
    states, ages, inf32 = ref.states, ref.ages, ref.infectivity.astype(np.float32)
    counts, tau = ref.counts.copy(), float(cfg.tau_max)
    clock = 0.0
    for k in range(3):
        fs.renewal_step(st, g, m, cfg, 7)
        clock += tau
        states, ages, inf32, mx, d = _oracle_step_chunked(states, ages, inf32, ro, col, tau, k, m, 7, True)
        counts = counts + d
        tau = min(cfg.tau_max, cfg.epsilon / (mx + cfg.delta))
        assert np.array_equal(st.counts, counts), k
        assert np.array_equal(st.states, states), k
        assert np.array_equal(st.ages.view(np.uint16), ages.view(np.uint16)), k
        assert st.clock == clock and st.tau_prev == tau, k
    assert counts[1] != ref.counts[1] or counts[2] != ref.counts[2]  # the epidemic moved


def test_c2_whole_run_matches_reference_record():
    """The reference's own full C2 run, `run_renewal(gen_fixed_degree(1e6,
    10, seed=1), seir_standard(...), RenewalConfig(), seed=7, t_final=50)`
    (1710 steps, tests/golden/make_c2_run_golden.py): the whole record —
    every grid fraction and the summary — bit for bit."""
    import json

    from tests._cases import GOLDEN, csr_sha, golden

    meta = json.loads((GOLDEN / "c2_run.json").read_text())
    z = golden("c2_run")
    g = fs.gen_fixed_degree(N, 10, seed=1)
    assert csr_sha(g) == meta["csr_sha256"]
    rec = fs.run_renewal(g, fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0), fs.RenewalConfig(), seed=7, t_final=50.0)
    assert np.array_equal(rec.grid, z["grid"])
    assert np.array_equal(rec.fractions, z["fractions"])
    s = z["summary"]
    assert (rec.summary["peak_I"], rec.summary["peak_I_time"], rec.summary["final_R"], rec.summary["step_count"]) == (
        s[0], s[1], s[2], int(s[3]))
    assert rec.summary["peak_I"] == 0.413512 and rec.summary["final_R"] == 0.973909 and rec.summary["step_count"] == 1710
