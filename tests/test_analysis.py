"""Trajectory records and ensemble analysis.

Golden vectors: tests/golden/make_analysis_golden.py runs the REFERENCE
make_record / ensemble_mean / quantile_band / fidelity on the synthetic logs
of tests/_analysis_cases.py.  CPU: the oracle restatement reproduces them
(bit for bit, bootstrap CIs to rounding).  GPU: csrc/fs_analysis.cu
reproduces them through the package API — records, means, quantile bands,
per-run errors and point metrics bit for bit; bootstrap CIs within
rtol 1e-12 (the reference's resample means are a BLAS product).
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import analysis_port as O
from tests._analysis_cases import CASES, ensemble_logs

G = np.load(Path(__file__).resolve().parent / "golden" / "analysis.npz")
CI_RTOL, CI_ATOL = 1e-12, 1e-15


def _stack_host(logs, name):
    comps, n, t_final, gp, *_ = CASES[name]
    return np.stack([O.make_record_arrays(t, c, n, t_final, gp)[1] for t, c in logs])


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_records_means_bands_match_reference(name):
    comps = CASES[name][0]
    la, _ = ensemble_logs(name)
    A = _stack_host(la, name)
    assert np.array_equal(A, G[f"{name}__frac_a"])
    assert np.array_equal(O.ensemble_mean(A), G[f"{name}__mean_a"])
    for ci, label in enumerate(comps):
        band = np.stack([O.quantile_linear(A[:, ci, :], 0.1), O.quantile_linear(A[:, ci, :], 0.9)])
        assert np.array_equal(band, G[f"{name}__band_{label}"])


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_fidelity_matches_reference(name):
    comps, *_, resamples, seed = CASES[name]
    la, lb = ensemble_logs(name)
    point, per_run, ci = O.fidelity(_stack_host(la, name), _stack_host(lb, name), comps, resamples, seed)
    ref = G[f"{name}__point"]
    got = [point["l_inf"], point["l2"], point.get("err_peak_i", 0.0), point.get("err_final_r", np.nan),
           per_run[0], np.nan if per_run[1] is None else per_run[1]]
    assert np.array_equal(np.array(got), ref, equal_nan=True)
    assert list(ci) == list(G[f"{name}__ci_keys"])
    np.testing.assert_allclose(np.array([ci[k] for k in ci]), G[f"{name}__ci"], rtol=CI_RTOL, atol=CI_ATOL)


def test_package_host_make_record_matches_reference():
    import paper_2604_22092_b200 as fs

    for name in CASES:
        comps, n, t_final, gp, *_ = CASES[name]
        la, _ = ensemble_logs(name)
        A = np.stack([fs.make_record(t, c, comps, n, t_final, gp).fractions for t, c in la])
        assert np.array_equal(A, G[f"{name}__frac_a"])


def test_fidelity_grid_mismatch_raises():
    import paper_2604_22092_b200 as fs
    from paper_2604_22092_b200.analysis import fidelity

    la, _ = ensemble_logs("sis")
    a = [fs.make_record(t, c, ("S", "I"), 2000, 20.0, 201) for t, c in la[:3]]
    b = [fs.make_record(t, c, ("S", "I"), 2000, 20.0, 101) for t, c in la[:3]]
    with pytest.raises(fs.errors.GridMismatchError):
        fidelity(a, b)
    with pytest.raises(fs.errors.GridMismatchError):
        fidelity([], b)


# ---------------------------------------------------------------- device --

def _device_records(name, logs):
    from paper_2604_22092_b200.analysis import make_records

    comps, n, t_final, gp, *_ = CASES[name]
    return make_records(logs, comps, n, t_final, gp)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_device_records_match_reference(name):
    import paper_2604_22092_b200 as fs

    comps, n, t_final, gp, *_ = CASES[name]
    la, _ = ensemble_logs(name)
    recs = _device_records(name, la)
    assert np.array_equal(np.stack([r.fractions for r in recs]), G[f"{name}__frac_a"])
    keys = list(G[f"{name}__summary_keys"])
    got = np.array([[r.summary[k] for k in keys] for r in recs]).reshape(len(recs), len(keys))
    assert np.array_equal(got, G[f"{name}__summary_a"])
    for r, (t, c) in zip(recs, la):  # and the package's host make_record, summary included
        h = fs.make_record(t, c, comps, n, t_final, gp)
        assert np.array_equal(r.grid, h.grid) and r.summary == h.summary


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_device_mean_and_bands_match_reference(name):
    from paper_2604_22092_b200.analysis import ensemble_mean, quantile_band

    comps = CASES[name][0]
    la, _ = ensemble_logs(name)
    recs = _device_records(name, la)
    assert np.array_equal(ensemble_mean(recs), G[f"{name}__mean_a"])
    for label in comps:
        lo, hi = quantile_band(recs, label, 0.1, 0.9)
        assert np.array_equal(np.stack([lo, hi]), G[f"{name}__band_{label}"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_device_fidelity_matches_reference(name):
    from paper_2604_22092_b200.analysis import fidelity

    *_, resamples, seed = CASES[name]
    la, lb = ensemble_logs(name)
    rep = fidelity(_device_records(name, la), _device_records(name, lb), resamples=resamples, seed=seed)
    got = [rep.l_inf, rep.l2, rep.err_peak_i, np.nan if rep.err_final_r is None else rep.err_final_r,
           rep.per_run_peak_err, np.nan if rep.per_run_final_err is None else rep.per_run_final_err]
    assert np.array_equal(np.array(got), G[f"{name}__point"], equal_nan=True)
    assert list(rep.ci) == list(G[f"{name}__ci_keys"])
    np.testing.assert_allclose(np.array([rep.ci[k] for k in rep.ci]), G[f"{name}__ci"], rtol=CI_RTOL, atol=CI_ATOL)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 31, 1000, 1025, 16384])
def test_device_column_quantiles_match_numpy(n):
    """Sizes around the bitonic padding, duplicates, negatives."""
    import torch

    from paper_2604_22092_b200.analysis import _column_quantiles

    rng = np.random.default_rng(n)
    x = np.round(rng.normal(size=(n, 5)), 2 if n > 100 else 6)
    qs = [0.0, 0.025000000000000022, 0.1, 0.5, 0.9, 0.975, 1.0]
    got = _column_quantiles(torch.from_numpy(x).cuda(), n, 5, 5, 1, qs)
    for k, q in enumerate(qs):
        assert np.array_equal(got[k], np.quantile(x, q, axis=0)), q


@pytest.mark.gpu
def test_ensemble_records_built_on_device_match_sequential():
    """run_ensemble builds all trial records in one fs_traj_records launch;
    each equals the host make_record of that trial's log."""
    import paper_2604_22092_b200 as fs

    g = fs.gen_fixed_degree(2000, 6, seed=3)
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    recs = fs.run_ensemble("renewal", g, m, fs.RenewalConfig(), 9, 15.0, 4, grid_points=301)
    for t, r in enumerate(recs):
        one = fs.run_renewal(g, m, fs.RenewalConfig(), fs.derive_seed(9, t), 15.0, grid_points=301)
        assert np.array_equal(r.fractions, one.fractions)
        assert {k: r.summary[k] for k in ("peak_I", "peak_I_time", "final_R", "step_count")} == \
               {k: one.summary[k] for k in ("peak_I", "peak_I_time", "final_R", "step_count")}
