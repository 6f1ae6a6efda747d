"""The drop-in accepts the reference's own objects (INTEGRATION
§3): a `spreadsim.renewal.RenewalConfig` (R/renewal.py:75-99) has none of
this package's three extra fields, and its `Strategy` is the reference's
enum (R/graph.py:61-67), not this package's.

* CPU, in the build container where /root/reference exists: the real
  reference objects go through the plan normalisation (config, strategy
  resolution, model descriptor) — skipped elsewhere.
* GPU: INTEGRATION §3's `_run_single` patch, verbatim, driven with a config
  object that carries exactly the reference's fields (recorded from the
  reference by tests/golden/make_reference_api.py) and the reference's
  Strategy enum shape, reproduces the reference's own record golden.
"""

import dataclasses
import enum
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200.graph import Strategy
from paper_2604_22092_b200.models import model_descriptor
from paper_2604_22092_b200.renewal import as_config
from tests._cases import GOLDEN, golden, graph, model

REF = Path("/root/reference/pkg/src")
API = json.loads((GOLDEN / "reference_api.json").read_text())

# reference-shaped stand-ins (exact field names, order, defaults)
RefStrategy = enum.Enum("Strategy", API["Strategy"])
RefRenewalConfig = dataclasses.make_dataclass(
    "RenewalConfig",
    [(f["name"], object, dataclasses.field(default=RefStrategy[f["default"]] if f["name"] == "strategy" else f["default"]))
     for f in API["RenewalConfig"]])


def test_reference_api_fixture_is_a_prefix_of_ours():
    ours = [f.name for f in dataclasses.fields(fs.RenewalConfig)]
    theirs = [f["name"] for f in API["RenewalConfig"]]
    assert ours[: len(theirs)] == theirs
    for f in API["RenewalConfig"]:
        d = getattr(fs.RenewalConfig(), f["name"])
        assert (d.name if isinstance(d, Strategy) else d) == f["default"], f["name"]
    assert {m.name: m.value for m in Strategy} == API["Strategy"]


@pytest.mark.parametrize("member", list(API["Strategy"]))
def test_foreign_strategy_and_config_normalise(member):
    cfg = as_config(RefRenewalConfig(strategy=RefStrategy[member], epsilon=0.05, compaction=True))
    assert isinstance(cfg, fs.RenewalConfig) and cfg.strategy == Strategy[member]
    assert (cfg.epsilon, cfg.compaction, cfg.rng, cfg.hazard_precision, cfg.gather) == (0.05, True, "splitmix", "f64", "auto")
    assert fs.graph.as_strategy(RefStrategy[member]) is Strategy[member]
    assert fs.graph.as_strategy(API["Strategy"][member]) is Strategy[member]
    assert as_config(None) == fs.RenewalConfig()


def test_foreign_auto_resolves_like_ours():
    for name in ("fixed_1e4", "ba_1e4"):
        g = graph(name)
        assert fs.graph.resolve_strategy(g, RefStrategy.AUTO) == fs.graph.resolve_strategy(g, Strategy.AUTO)
    assert fs.select_strategy(fs.degree_stats(graph("ba_1e4")), RefStrategy.AUTO) == Strategy.LANE_CHUNKED  # rho 44.6
    assert fs.select_strategy(fs.degree_stats(graph("ba_1e5")), RefStrategy.AUTO) == Strategy.EDGE_MERGE


@pytest.mark.skipif(not REF.exists(), reason="the reference is importable only in the build container")
def test_real_reference_objects_through_plan_normalisation():
    sys.path.insert(0, str(REF))
    try:
        import spreadsim as ss
        from spreadsim import renewal as RR
        from spreadsim.graph import Strategy as SS
    finally:
        sys.path.remove(str(REF))
    g = ss.gen_barabasi_albert(2000, 5, seed=3)
    m = ss.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    for s in SS:
        cfg = as_config(RR.RenewalConfig(strategy=s, steps_per_batch=7))
        assert cfg.strategy.value == s.value and cfg.steps_per_batch == 7
        assert fs.graph.resolve_strategy(g, cfg.strategy).value == RR._build_plan(g, m, RR.RenewalConfig(strategy=s),
                                                                                  False).strategy.value
    d_ref, d_ours = model_descriptor(m), model_descriptor(fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0))
    assert bytes(d_ref) == bytes(d_ours)
    # the graph object itself is accepted where the package reads a CsrGraph
    assert fs.degree_stats(g) == fs.degree_stats(fs.gen_barabasi_albert(2000, 5, seed=3))


# INTEGRATION.md §3, verbatim apart from the reference's other branches
def _run_single(engine, g, m, cfg, trial_seed, t_final, grid_points, seed_count, seed_compartment):
    if engine == "renewal-b200":
        from paper_2604_22092_b200 import run_renewal as run_renewal_b200
        return run_renewal_b200(g, m, cfg or RefRenewalConfig(), trial_seed, t_final, grid_points,
                                seed_count=seed_count, seed_compartment=seed_compartment)
    raise ValueError(f"unknown engine {engine!r}")


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [None, RefRenewalConfig(), RefRenewalConfig(strategy=RefStrategy.EDGE_MERGE),
                                 RefRenewalConfig(compaction=True)])
def test_run_single_patch_with_reference_config(cfg):
    z = golden("record")
    rec = _run_single("renewal-b200", graph("er_300"), model("seir"), cfg, 77, 20.0, 501, None, None)
    assert np.array_equal(rec.fractions, z["fractions"]) and np.array_equal(rec.grid, z["grid"])
    assert rec.summary["step_count"] == int(z["summary"][3])


@pytest.mark.gpu
def test_renewal_step_with_reference_config_and_active_set():
    """The reference's stepped driver (R/analysis.py:401-418) passes its own
    config and the active set `_begin_batch` returns."""
    from paper_2604_22092_b200 import renewal as R
    from tests._cases import trajectory_case

    meta, g, m, _, ref = trajectory_case("c1")
    cfg = RefRenewalConfig(compaction=True)
    st = fs.init_renewal_state(g, m, cfg, meta["seed"])
    plan = R._build_plan(g, m, cfg, st.mixed_precision)
    counts = []
    for _ in range(meta["batches"]):
        active = R._begin_batch(st, g, cfg, plan)
        assert active is not None
        for _ in range(cfg.steps_per_batch):
            fs.renewal_step(st, g, m, cfg, meta["seed"], plan=plan, active=active)
            counts.append(st.counts.copy())
    assert np.array_equal(np.array(counts), ref["counts"])
    assert np.array_equal(st.states.astype(np.int32), ref["states"])


@pytest.mark.gpu
def test_renewal_step_active_without_begin_batch_and_bad_subset():
    """a step given an ActiveSet before any batch boundary must
    still process the live nodes; a subset that is not the live set is
    refused rather than silently widened."""
    from oracle import spreadsim_port as O

    g, m = graph("er_300"), model("seir")
    cfg = fs.RenewalConfig(compaction=True)
    st = fs.init_renewal_state(g, m, cfg, 5)
    ref = O.init_state(g, m, cfg, 5)
    act = fs.refresh_active(st.states, m.terminal_mask())
    for _ in range(20):
        fs.renewal_step(st, g, m, cfg, 5, active=act)
        O.step(ref, g, m, cfg, 5)
    assert np.array_equal(st.counts, ref.counts) and np.array_equal(st.ages, ref.ages)
    bad = fs.refresh_active(st.states, m.terminal_mask())
    bad = type(bad)(active_nodes=bad.active_nodes[1:], num_active=bad.num_active - 1)
    with pytest.raises(ValueError):
        fs.renewal_step(st, g, m, cfg, 5, active=bad)
