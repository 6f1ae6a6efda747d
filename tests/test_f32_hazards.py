"""The `hazard_precision="f32"` path (north_star: hazards within 1e-5
relative in fp32).

The reference evaluates every nodal hazard in float64 and stores it as f32
(R/renewal.py:474-480; R/hazards.py:84-132); its own tolerance tests are
T/test_hazards.py:23-39.  The f32 kernel path evaluates the same piecewise
formulas in float (fs_device.cuh `hazard_*_f32`; the z < 0 erfcx reflection
rewritten as e^{-z^2} / (2 - e^{-z^2} erfcx(-z)) to stay finite).

Bounds asserted here:
  * h > 1e-6: relative error <= 1e-5 against the reference's f64 hazard,
    except within 1e-5 of z = 3.5, the reference's own erfcx branch point,
    where its 4-term asymptotic series jumps by 2.2e-4 and the f32 z may
    fall on the other side (bound there: 3e-4);
  * tau -> 0 tail (h <= 1e-6): absolute error <= 1e-8 (measured max
    3.4e-9) — a rate there fires with q <= 1e-7 per step, so the error moves
    q by <= 1e-9;
  * whole trajectories: per-step counts and states identical to the
    reference's f64 run on the C1 and BA-merge golden cases, clock / tau /
    ages within 1e-5 relative (tau moves only when the step's maximum rate
    is a hazard, not a pressure).
"""

import numpy as np
import pytest

import paper_2604_22092_b200 as fs
from oracle import spreadsim_port as O
from tests._cases import golden, trajectory_case

pytestmark = pytest.mark.gpu
REL = 1e-5
TAIL_ABS = 1e-8


def _check(h32, h64, skip=None):
    keep = np.ones(h64.shape, bool) if skip is None else ~skip
    big, tail = keep & (h64 > 1e-6), keep & (h64 <= 1e-6)
    rel = np.abs(h32[big] - h64[big]) / h64[big]
    assert rel.max() <= REL, (rel.max(), np.argmax(rel))
    assert np.abs(h32[tail] - h64[tail]).max(initial=0.0) <= TAIL_ABS
    assert np.isfinite(h32).all() and (h32 >= 0).all()


@pytest.mark.parametrize("which", ["ei", "ir"])
def test_f32_lognormal_against_reference_grid(which):
    z = golden("hazards")
    p = fs.LogNormalParams(*z[which])
    # the kernel evaluates at the f32 storage age; compare on the f32 grid
    tau = z["tau"].astype(np.float32).astype(np.float64)
    h32 = fs.lognormal_hazard(tau, p, precision="f32")
    _check(h32, O.hazard_lognormal(tau, p.mu, p.sigma))
    # and directly against the golden vector (f64 tau) where tau is exactly representable
    exact = z["tau"].astype(np.float32).astype(np.float64) == z["tau"]
    _check(h32[exact], z[f"h_{which}"][exact])


@pytest.mark.parametrize("which", ["ei", "ir"])
def test_f32_lognormal_all_three_erfcx_branches(which):
    """z < 0, 0 <= z <= 3.5 and z > 3.5 (the asymptotic series), dense."""
    z = golden("hazards")
    p = fs.LogNormalParams(*z[which])
    zz = np.concatenate([np.linspace(-6.0, -1e-3, 4001), np.linspace(0.0, 3.5, 4001), np.linspace(3.5001, 12.0, 4001)])
    tau = np.exp(p.mu + p.sigma * np.sqrt(2.0) * zz).astype(np.float32).astype(np.float64)
    h32, h64 = fs.lognormal_hazard(tau, p, precision="f32"), O.hazard_lognormal(tau, p.mu, p.sigma)
    # The reference's piecewise erfcx (R/hazards.py:84-105) switches to the
    # 4-term asymptotic series at z = 3.5, where the series is off by its
    # next term (105/16 z^-8 = 2.9e-4 relative): the function itself jumps
    # there.  z evaluated in f32 can land one ulp on the other side of 3.5
    # than the f64 z, so within 1e-5 of the switch the bound is that jump.
    z64 = (np.log(tau) - p.mu) / (p.sigma * np.sqrt(2.0))
    edge = np.abs(z64 - 3.5) < 1e-5
    _check(h32, h64, skip=edge)
    assert (np.abs(h32[edge] - h64[edge]) / h64[edge]).max(initial=0.0) <= 3e-4


def test_f32_weibull_erlang_against_oracle():
    tau = np.concatenate([[0.0, 1e-6, 1e-4], np.linspace(0.01, 80.0, 6000)]).astype(np.float32).astype(np.float64)
    w, e = fs.WeibullParams(1.247568, 5.365966), fs.ErlangParams(3, 0.4)
    _check(fs.weibull_hazard(tau, w, precision="f32"), O.hazard_weibull(tau, w.k, w.lam))
    _check(fs.erlang_hazard(tau, e, precision="f32"), O.hazard_erlang(tau, e.k, e.rate))
    assert fs.weibull_hazard(0.0, fs.WeibullParams(1.0, 2.0), precision="f32") == 0.5
    assert fs.erlang_hazard(0.0, fs.ErlangParams(1, 0.4), precision="f32") == np.float32(0.4)


@pytest.mark.parametrize("name", ["c1", "ba_merge", "c1_mixed"])
def test_f32_trajectory_against_reference_f64_run(name):
    meta, g, m, cfg, ref = trajectory_case(name)
    cfg = fs.RenewalConfig(**{**vars(cfg), "hazard_precision": "f32"})
    st = fs.init_renewal_state(g, m, cfg, meta["seed"], meta["seed_count"], meta["seed_compartment"])
    clocks, counts = [], []
    for _ in range(meta["batches"]):
        rec = []
        fs.run_batch(st, g, m, cfg, meta["seed"], recorder=rec)
        clocks += [c for c, _ in rec]
        counts += [c for _, c in rec]
    assert np.array_equal(np.array(counts), ref["counts"]), "per-step counts"
    assert np.array_equal(st.states.astype(np.int32), ref["states"]), "final states"
    assert np.allclose(np.array(clocks), ref["clock"], rtol=REL, atol=0)
    assert np.allclose(st.ages.astype(np.float32), ref["ages"], rtol=REL, atol=0)
    big = ref["rates"] > 1e-6
    assert np.allclose(st.rates[big], ref["rates"][big], rtol=10 * REL, atol=0)
