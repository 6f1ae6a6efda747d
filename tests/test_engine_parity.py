"""GPU engine vs the oracle / golden vectors (the parity gate).

Bar (BASELINE north_star): states, counts, clock and tau bit-exact given the
same uniforms; pressure bit-exact; rates / hazards within 1e-5 relative
(f64 hazards are expected to agree to a few ulp of f64, i.e. exact after the
f32 store, except when a libm ulp straddles an f32 rounding boundary).
"""

import numpy as np
import pytest
import torch

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import renewal as R
from paper_2604_22092_b200.graph import Strategy
from oracle import spreadsim_port as O
from tests._cases import TRAJECTORY_CASES, golden, graph, model, trajectory_case

pytestmark = pytest.mark.gpu
RATE_RTOL = 1e-5


def test_device_uniform_bit_exact():
    z = golden("rng")
    for (s, k), row in zip(z["cases"], z["uniform"]):
        assert np.array_equal(fs.uniform_array(int(s), int(k), z["streams"]), row)
    u = fs.uniform_array(77, 5, n=100_000).cpu().numpy()
    assert np.array_equal(u[:1000], z["uniform_77_5_head"]) and u.sum() == z["uniform_77_5_sum"][0]


def test_device_philox_matches_oracle():
    streams = np.concatenate([np.arange(5000, dtype=np.uint64), np.array([2**40 + 3, 2**63 + 9], dtype=np.uint64)])
    for seed, step in [(0, 0), (7, 199), (2**63 + 5, 2**33 + 1)]:
        assert np.array_equal(fs.uniform_array(seed, step, streams, rng="philox"),
                              O.philox_uniform_array(seed, step, streams))


def test_device_erfcx_and_lognormal_hazard():
    z = golden("hazards")
    assert np.allclose(fs.erfcx_stable(z["z"]), z["erfcx"], rtol=1e-13, atol=0)
    ei = fs.LogNormalParams(*z["ei"])
    ir = fs.LogNormalParams(*z["ir"])
    assert np.allclose(fs.lognormal_hazard(z["tau"], ei), z["h_ei"], rtol=1e-13, atol=0)
    assert np.allclose(fs.lognormal_hazard(z["tau"], ir), z["h_ir"], rtol=1e-13, atol=0)
    # the f32 rate actually stored by the engine: bit-identical almost everywhere
    f32_dev = fs.lognormal_hazard(z["tau"], ei).astype(np.float32)
    f32_ref = z["h_ei"].astype(np.float32)
    assert (f32_dev != f32_ref).sum() <= 2
    assert fs.erfcx_stable(0.0) == 1.0 and fs.lognormal_hazard(0.0, ei) == 0.0


def test_device_weibull_erlang_hazards():
    tau = np.concatenate([[0.0, 1e-6], np.linspace(0.01, 80.0, 3000)])
    w = fs.WeibullParams(1.247568, 5.365966)
    e = fs.ErlangParams(3, 0.4)
    assert np.allclose(fs.weibull_hazard(tau, w), O.hazard_weibull(tau, w.k, w.lam), rtol=1e-13, atol=0)
    assert np.allclose(fs.erlang_hazard(tau, e), O.hazard_erlang(tau, e.k, e.rate), rtol=1e-13, atol=0)


@pytest.mark.parametrize("name", ["er_400", "fixed_400", "ba_2000", "weighted"])
@pytest.mark.parametrize("strategy", [Strategy.PER_NODE, Strategy.LANE_CHUNKED, Strategy.EDGE_MERGE])
@pytest.mark.parametrize("epb", [4, 256, 1024])
def test_pressure_gather_bit_exact(name, strategy, epb):
    z = golden("pressure")
    g = graph(name)
    cfg = fs.RenewalConfig(edges_per_block=epb, lanes_per_node=8)
    p = fs.pressure_gather(g, z[f"{name}_inf"], strategy, cfg)
    assert p.dtype == np.float32 and np.array_equal(p, z[f"{name}_p"])


def test_pressure_gather_edge_cases():
    cfg = fs.RenewalConfig()
    g0 = fs.build_csr([], 1)
    assert np.array_equal(fs.pressure_gather(g0, np.zeros(1, np.float32), Strategy.AUTO, cfg), np.zeros(1, np.float32))
    chain = fs.build_csr([(0, 1, 1.0), (1, 2, 1.0)], 3)
    inf = np.array([0.25, 0.0, 0.0], np.float32)
    for s in (Strategy.PER_NODE, Strategy.LANE_CHUNKED, Strategy.EDGE_MERGE):
        assert np.array_equal(fs.pressure_gather(chain, inf, s, cfg), np.array([0.0, 0.25, 0.0], np.float32))


def run_engine_case(name, overrides=None, batches_via_graph=False):
    meta, g, m, cfg, ref = trajectory_case(name)
    if overrides:
        cfg = fs.RenewalConfig(**{**vars(cfg), **overrides})
    st = fs.init_renewal_state(g, m, cfg, meta["seed"], meta["seed_count"], meta["seed_compartment"])
    plan = R._build_plan(g, m, cfg, st.mixed_precision)
    clocks, taus, counts, cps = [], [], [], {}
    k = 0
    for _ in range(meta["batches"]):
        if batches_via_graph:
            rec = []
            _, total = fs.run_batch(st, g, m, cfg, meta["seed"], plan=plan, recorder=rec)
            for c, cnt in rec:
                clocks.append(c)
                counts.append(cnt)
            k += cfg.steps_per_batch
            continue
        R._begin_batch(st, g, cfg, plan)
        for _ in range(cfg.steps_per_batch):
            _, tau = fs.renewal_step(st, g, m, cfg, meta["seed"], plan=plan)
            k += 1
            clocks.append(st.clock)
            taus.append(tau)
            counts.append(st.counts.copy())
            if k in (1, 10, 50):
                cps[k] = (st.states.astype(np.int32), st.ages.astype(np.float32))
    return st, dict(clock=np.array(clocks), tau=np.array(taus), counts=np.array(counts)), cps, ref


def assert_matches(st, log, cps, ref, exact_ages=True):
    assert np.array_equal(log["counts"], ref["counts"]), "per-step compartment counts"
    assert np.array_equal(log["clock"], ref["clock"]), "per-step clock"
    if log["tau"].size:
        assert np.array_equal(log["tau"], ref["tau"]), "per-step tau"
    assert np.array_equal(st.states.astype(np.int32), ref["states"]), "final states"
    ages = st.ages.astype(np.float32)
    if exact_ages:
        assert np.array_equal(ages, ref["ages"]), "final ages"
    else:
        assert np.allclose(ages, ref["ages"], rtol=RATE_RTOL, atol=0)
    assert np.array_equal(st.pressure, ref["pressure"]), "pressure"
    assert np.allclose(st.rates, ref["rates"], rtol=RATE_RTOL, atol=0), "rates"
    assert np.array_equal(st.infectivity.astype(np.float32), ref["infectivity"]) or np.allclose(
        st.infectivity.astype(np.float32), ref["infectivity"], rtol=RATE_RTOL, atol=0)
    for k, (s, a) in cps.items():
        assert np.array_equal(s, ref[f"cp{k}_states"]), f"states at step {k}"
        assert np.array_equal(a, ref[f"cp{k}_ages"]), f"ages at step {k}"


@pytest.mark.parametrize("name", TRAJECTORY_CASES)
def test_trajectory_parity_stepwise(name):
    st, log, cps, ref = run_engine_case(name)
    assert_matches(st, log, cps, ref)


@pytest.mark.parametrize("name", ["c1", "c1_mixed", "er1000", "er1000_nocarry", "ba_merge", "sis", "shed_hazard", "weighted"])
def test_trajectory_parity_graph_replay(name):
    st, log, _, ref = run_engine_case(name, batches_via_graph=True)
    assert np.array_equal(log["counts"], ref["counts"])
    assert np.array_equal(log["clock"], ref["clock"])
    assert np.array_equal(st.states.astype(np.int32), ref["states"])
    assert np.array_equal(st.ages.astype(np.float32), ref["ages"])
    assert np.allclose(st.rates, ref["rates"], rtol=RATE_RTOL, atol=0)


@pytest.mark.parametrize("overrides", [
    {"strategy": Strategy.PER_NODE}, {"strategy": Strategy.LANE_CHUNKED}, {"strategy": Strategy.EDGE_MERGE},
    {"strategy": Strategy.EDGE_MERGE, "edges_per_block": 64}, {"compaction": True}, {"gather": "f32"},
    {"gather": "count"}, {"gather": "count", "strategy": Strategy.EDGE_MERGE}, {"gather": "incremental"},
    {"gather": "incremental", "compaction": True},
    {"chunk_skip": False, "hazard_chunk": 64},
])
@pytest.mark.parametrize("name", ["c1", "ba_merge"])
def test_variants_are_result_neutral(name, overrides):
    st, log, cps, ref = run_engine_case(name, overrides=overrides)
    assert_matches(st, log, cps, ref)


@pytest.mark.parametrize("env", [{}, {"FS_MERGE_UNFUSED": "1"}, {"FS_NO_F32_MASK": "1"}])
@pytest.mark.parametrize("overrides", [
    {"gather": "f32", "strategy": Strategy.EDGE_MERGE},           # fused edge-merge: hub pre-pass + tile sweep
    {"gather": "f32", "strategy": Strategy.EDGE_MERGE, "edges_per_block": 64},
    {"gather": "f32", "strategy": Strategy.PER_NODE},             # thread-per-node fold, mask prefilter
    {"gather": "f32", "strategy": Strategy.EDGE_MERGE, "compaction": True},
    {"gather": "count", "strategy": Strategy.EDGE_MERGE},         # one-launch edge-merge, count gather
    {"gather": "count", "strategy": Strategy.EDGE_MERGE, "compaction": True},
])
@pytest.mark.parametrize("name", ["ba_merge", "shed_hazard", "weighted", "c1_mixed"])
def test_gather_forms_bit_exact(name, overrides, env, monkeypatch):
    """Every form of the CSR gather — the f32 fold with and without the
    nonzero-infectivity mask, the count gather, the one-launch edge-merge and
    the two-launch one — against the reference goldens, stepwise and
    graph-replayed."""
    if overrides["gather"] == "count" and name in ("shed_hazard", "weighted"):
        pytest.skip("the count gather needs constant transmission and uniform weights")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    st, log, cps, ref = run_engine_case(name, overrides=overrides)
    assert_matches(st, log, cps, ref)
    st, log, _, ref = run_engine_case(name, overrides=overrides, batches_via_graph=True)
    assert np.array_equal(log["counts"], ref["counts"])
    assert np.array_equal(log["clock"], ref["clock"])
    assert np.array_equal(st.states.astype(np.int32), ref["states"])


@pytest.mark.parametrize("gather", ["incremental", "count"])
@pytest.mark.parametrize("name", ["c1", "ba_merge"])
def test_compaction_graph_replay_neutral(name, gather):
    st, log, _, ref = run_engine_case(name, overrides={"compaction": True, "gather": gather}, batches_via_graph=True)
    assert np.array_equal(log["counts"], ref["counts"])
    assert np.array_equal(st.states.astype(np.int32), ref["states"])
    assert np.array_equal(st.ages.astype(np.float32), ref["ages"])


def oracle_run(g, m, cfg, seed, steps, rng="splitmix", seed_count=None):
    st = O.init_state(g, m, cfg, seed, seed_count)
    for _ in range(steps):
        O.step(st, g, m, cfg, seed, rng)
    return st


@pytest.mark.parametrize("rng", ["splitmix", "philox"])
@pytest.mark.parametrize("mname,gname", [("seir_we", "ba_1e4"), ("seir", "fixed_1e4"), ("seir_we", "er_1000")])
def test_weibull_erlang_and_philox_vs_oracle(mname, gname, rng):
    g, m = graph(gname), model(mname)
    cfg = fs.RenewalConfig(rng=rng)
    steps = 150
    ref = oracle_run(g, m, cfg, 21, steps, rng)
    st = fs.init_renewal_state(g, m, cfg, 21)
    for _ in range(steps // cfg.steps_per_batch):
        fs.run_batch(st, g, m, cfg, 21)
    assert np.array_equal(st.counts, ref.counts)
    assert np.array_equal(st.states.astype(np.int32), ref.states.astype(np.int32))
    # f64 hazards: equal after the f32 store unless a libm ulp straddles an
    # f32 rounding boundary (p ~ 2^-28 per evaluation), so ages and clock exact
    assert np.array_equal(st.ages, ref.ages)
    assert np.allclose(st.rates, ref.rates, rtol=RATE_RTOL, atol=0)
    assert st.clock == ref.clock and st.tau_prev == ref.tau_prev


def test_host_edits_between_steps_are_seen():
    # T/test_renewal.py:112-134 — single E node at age 4.0
    g = fs.build_csr([], 1)
    m = model("seir")
    cfg = fs.RenewalConfig(tau_max=0.1)
    st = fs.init_renewal_state(g, m, cfg, seed=0, seed_count=1)
    st.states[0] = 1
    st.ages[0] = 4.0
    st.counts = np.array([0, 1, 0, 0], dtype=np.int64)
    _, elapsed = fs.renewal_step(st, g, m, cfg, seed=11)
    assert elapsed == 0.1
    u = float(O.uniform_array(11, 0, np.array([0], dtype=np.uint64))[0])
    rate = float(O.hazard_lognormal(np.array([4.0]), *m.nodal[1][1].params.__dict__.values())[0])
    q = -np.expm1(-np.float64(np.float32(rate)) * 0.1)
    assert q == pytest.approx(0.029418, abs=2e-5)
    if u < q:
        assert st.states[0] == 2 and st.ages[0] == 0.0
    else:
        assert st.states[0] == 1 and float(st.ages[0]) == np.float32(np.float32(4.0) + np.float32(0.1))
        assert float(st.rates[0]) == pytest.approx(rate, rel=1e-6)


def test_general_gather_switch_on_host_infectivity_edit():
    g, m = graph("er_300"), model("seir")
    cfg = fs.RenewalConfig()
    a = fs.init_renewal_state(g, m, cfg, seed=3)
    b = O.init_state(g, m, cfg, seed=3)
    for _ in range(20):
        fs.renewal_step(a, g, m, cfg, 3)
        O.step(b, g, m, cfg, 3)
    inf = np.random.default_rng(4).random(g.num_nodes).astype(np.float32) * 0.3
    a.infectivity = inf
    b.infectivity = inf.copy()
    for _ in range(30):
        fs.renewal_step(a, g, m, cfg, 3)
        O.step(b, g, m, cfg, 3)
    assert np.array_equal(a.states.astype(np.int32), b.states.astype(np.int32))
    assert np.array_equal(a.pressure, b.pressure)


def test_all_susceptible_and_all_absorbed():
    g = graph("er_200")
    m = model("seir")
    cfg = fs.RenewalConfig()
    st = fs.init_renewal_state(g, m, cfg, seed=3, seed_count=0)
    for _ in range(5):
        fs.renewal_step(st, g, m, cfg, seed=3)
    assert st.counts[0] == g.num_nodes and st.tau_prev == cfg.tau_max
    assert st.clock == pytest.approx(5 * cfg.tau_max)
    g2 = fs.build_csr([(0, 1, 1.0), (1, 0, 1.0)], 2)
    cfg2 = fs.RenewalConfig(compaction=True, steps_per_batch=5)
    st2 = fs.init_renewal_state(g2, m, cfg2, seed=0, seed_count=0)
    st2.states[:] = 3
    st2.counts = np.array([0, 0, 0, 2], dtype=np.int64)
    fs.run_batch(st2, g2, m, cfg2, seed=0)
    assert st2.clock == pytest.approx(5 * cfg2.tau_max) and st2.counts[3] == 2


def test_mixed_precision_toggle_and_lock():
    g = graph("er_200")
    m = model("seir")
    cfg = fs.RenewalConfig()
    s = fs.init_renewal_state(g, m, cfg, seed=1)
    ref = (s.states.copy(), s.ages.copy(), s.infectivity.copy())
    fs.set_mixed_precision(s, True)
    assert s.states.dtype == np.int8 and s.ages.dtype == np.float16 and s.infectivity.dtype.itemsize == 2
    fs.set_mixed_precision(s, False)
    assert all(np.array_equal(x, y) for x, y in zip((s.states, s.ages, s.infectivity), ref))
    fs.renewal_step(s, g, m, cfg, seed=1)
    with pytest.raises(fs.ReconfigureAfterStartError):
        fs.set_mixed_precision(s, True)


def test_refresh_active_examples():
    term = np.array([False, False, False, True])
    act = fs.refresh_active(np.array([0, 3, 1, 3, 2], dtype=np.int32), term, pad=4)
    assert act.num_active == 3 and list(act.ids) == [0, 2, 4] and act.active_nodes.size == 9
    assert np.all(act.active_nodes[3:] == 0)
    big = np.random.default_rng(0).integers(0, 4, 100_003).astype(np.int8)
    act = fs.refresh_active(big, term, pad=128)
    assert np.array_equal(act.ids, np.flatnonzero(big != 3))


def test_run_renewal_record_matches_reference():
    z = golden("record")
    g, m = graph("er_300"), model("seir")
    rec = fs.run_renewal(g, m, fs.RenewalConfig(), seed=77, t_final=20.0)
    assert np.array_equal(rec.fractions, z["fractions"]) and np.array_equal(rec.grid, z["grid"])
    s = z["summary"]
    assert (rec.summary["peak_I"], rec.summary["peak_I_time"], rec.summary["final_R"], rec.summary["step_count"]) == (
        s[0], s[1], s[2], int(s[3]))


@pytest.mark.parametrize("env", [
    {"FS_MEMO": "1"},                        # age-cohort hazard memo (default only at N >= 8M)
    {"FS_NO_STREAM": "1"},                   # incremental counts in the general kernel
    {"FS_NO_PDL": "1", "FS_MEMO": "1"},
])
@pytest.mark.parametrize("name", ["c1", "c1_mixed", "ba_merge", "sir", "shed_hazard", "weighted"])
def test_engine_variants_bit_exact(name, env, monkeypatch):
    """Kernel variants the engine selects by size or switch (read when an
    engine is created) against the reference goldens, stepwise and replayed."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    st, log, cps, ref = run_engine_case(name)
    assert_matches(st, log, cps, ref)
    st, log, _, ref = run_engine_case(name, batches_via_graph=True)
    assert np.array_equal(log["counts"], ref["counts"])
    assert np.array_equal(st.states.astype(np.int32), ref["states"])
    assert np.array_equal(st.ages.astype(np.float32), ref["ages"])


@pytest.mark.parametrize("gather", ["incremental", "count"])
@pytest.mark.parametrize("edit_inf", [False, True])
def test_host_state_edits_mid_run(gather, edit_inf):
    """States written between steps (T/test_renewal.py:118-120, 245-246 edit
    them): the next step still gathers the infectivity of the previous one
    (R/renewal.py:500-505), the step after sees the edited nodes — also with
    incremental counts, which must push the implied status changes."""
    g, m = graph("er_300"), model("sir")
    cfg = fs.RenewalConfig(gather=gather)
    st = fs.init_renewal_state(g, m, cfg, 5)
    ref = O.init_state(g, m, cfg, 5)
    for _ in range(30):
        fs.renewal_step(st, g, m, cfg, 5)
        O.step(ref, g, m, cfg, 5)
    s_nodes = np.flatnonzero(ref.states == 0)[:6]
    i_nodes = np.flatnonzero(ref.states == 1)[:2]
    for arr in (st.states, ref.states):
        arr[s_nodes] = 1  # S -> I by hand
        arr[i_nodes] = 2  # I -> R by hand
    c = np.bincount(ref.states.astype(np.int64), minlength=3)
    st.counts = c
    ref.counts = c.copy()
    if edit_inf:  # infectivity made consistent with the edit as well
        inf = np.where(ref.states == 1, np.float32(m.beta), np.float32(0.0)).astype(np.float32)
        st.infectivity = inf
        ref.infectivity = inf.copy()
    for _ in range(40):
        fs.renewal_step(st, g, m, cfg, 5)
        O.step(ref, g, m, cfg, 5)
        assert np.array_equal(st.counts, ref.counts)
    assert np.array_equal(st.states.astype(np.int32), ref.states.astype(np.int32))
    assert np.array_equal(st.pressure, ref.pressure)
    assert st.clock == ref.clock


def test_snapshot_restore_replays_the_same_steps():
    """bench.py times a step window twice (warm, then flushed) from one
    snapshot: after a restore the engine must replay exactly the same
    trajectory — counts, states, ages, clock — including its incremental
    counts and pending deltas (fs_engine_state_restored)."""
    meta, g, m, cfg, ref = trajectory_case("c1")
    st = fs.init_renewal_state(g, m, cfg, meta["seed"])
    plan = R._build_plan(g, m, cfg, st.mixed_precision)
    eng = st._bind(plan, meta["seed"], materialize=False)
    eng.step(10, False, False)
    snap = eng.snapshot()
    runs = []
    for _ in range(2):
        eng.restore(snap)
        eng.run_batch(False)   # a graph-replayed batch ...
        eng.step(37, False, False)  # ... and eager steps: 10 + 50 + 37 = 97 (odd parity)
        st._after_device()
        runs.append((st.states.copy(), st.ages.copy(), st.counts.copy(), st.clock))
    for a, b in zip(runs[0], runs[1]):
        assert np.array_equal(a, b)
    eng.restore(snap)
    eng.step(190, False, False)
    st._after_device()
    assert np.array_equal(st.states.astype(np.int32), ref["states"]) and np.array_equal(st.ages, ref["ages"])
    assert np.array_equal(st.counts, ref["counts"][199]) and st.clock == ref["clock"][199]


@pytest.mark.parametrize("mixed", [False, True])
def test_uniform_s_age_mode_and_reentry_edit(mixed):
    """SEIR never re-enters S, so the engine keeps the S age as one scalar
    (DESIGN.md §3.4): host reads of `ages` still see every S node's age, and
    an edit that puts a node back into S with a different age switches the
    mode off — the run stays exact against the oracle either way."""
    g, m = graph("er_300"), model("seir")
    cfg = fs.RenewalConfig(mixed_precision=mixed)
    st = fs.init_renewal_state(g, m, cfg, 5)
    ref = O.init_state(g, m, cfg, 5)
    for _ in range(60):
        fs.renewal_step(st, g, m, cfg, 5)
        O.step(ref, g, m, cfg, 5)
    assert st._engine.uniform_s_age()
    assert np.array_equal(st.ages, ref.ages)
    r_nodes = np.flatnonzero(ref.states == 3)[:3]
    e_nodes = np.flatnonzero(ref.states == 1)[:3]
    assert r_nodes.size and e_nodes.size
    for arr in (st.states, ref.states):
        arr[r_nodes] = 0  # R -> S, keeping the R node's own (different) age
        arr[e_nodes] = 0
    c = np.bincount(ref.states.astype(np.int64), minlength=4)
    st.counts = c
    ref.counts = c.copy()
    fs.renewal_step(st, g, m, cfg, 5)
    O.step(ref, g, m, cfg, 5)
    assert not st._engine.uniform_s_age()
    for _ in range(40):
        fs.renewal_step(st, g, m, cfg, 5)
        O.step(ref, g, m, cfg, 5)
    assert np.array_equal(st.counts, ref.counts) and np.array_equal(st.states, ref.states)
    assert np.array_equal(st.ages, ref.ages) and st.clock == ref.clock


@pytest.mark.parametrize("n,count", [(1, 1), (300, 0), (300, 1), (300, 299), (300, 300), (5000, 50),
                                     (200_000, 2000), (3_000_000, 30_000)])
def test_seed_selection_matches_reference_choice(n, count):
    """fs_seed_select (device radix select, several digit passes at the
    larger sizes) picks exactly the reference's _pick_seed_nodes set
    (R/renewal.py:162-169): the `count` smallest uniforms."""
    ids = R._pick_seed_nodes(n, 11, count, torch.device("cuda")).cpu().numpy()
    u = O.uniform_array(O.derive_seed(11, 0x5EEDC0DE), 0, np.arange(n, dtype=np.uint64))
    want = np.sort(np.argpartition(u, count - 1)[:count]) if count else np.empty(0, np.int64)
    assert np.array_equal(ids, want)


def test_symmetry_check_on_device():
    from paper_2604_22092_b200.renewal import device_graph

    assert device_graph(graph("ba_2000")).symmetric and device_graph(graph("er_300")).symmetric
    assert not device_graph(fs.build_csr([(0, 1, 1.0), (1, 2, 1.0)], 3)).symmetric  # directed chain
    # multiplicities must match too (a hand-built multigraph CSR): 0->1 twice, 1->0 once
    multi = fs.CsrGraph(2, 3, np.array([0, 1, 3]), np.array([1, 0, 0], np.int32), np.ones(3, np.float32))
    assert not device_graph(multi).symmetric
    multi2 = fs.CsrGraph(2, 4, np.array([0, 2, 4]), np.array([1, 1, 0, 0], np.int32), np.ones(4, np.float32))
    assert device_graph(multi2).symmetric
