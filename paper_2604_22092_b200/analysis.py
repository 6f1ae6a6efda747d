"""Device-side trajectory records and ensemble analysis.

Drop-ins for the consumers of the per-step log in the reference's
``spreadsim.analysis`` / ``spreadsim.trajectory``: ``make_records`` (a batch
``make_record``, R/trajectory.py:31-61), ``ensemble_mean``
(R/analysis.py:137-138), ``quantile_band`` (:141-148), ``fidelity`` and
``FidelityReport`` (:165-256).  The arithmetic runs in csrc/fs_analysis.cu:
the records, ensemble means, per-run deviations and quantile interpolation
are bit-identical to numpy; the bootstrap resample means (a matrix product
numpy hands to BLAS) agree to a few ulps.  The multinomial resample counts
are drawn on the host with the reference's own generator
(``np.random.default_rng(seed).multinomial``, R/analysis.py:153-157), so the
bootstrap sees the same resamples as the reference; everything computed from
them runs on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .errors import GridMismatchError, InvalidConfigError
from .trajectory import DEFAULT_GRID_POINTS, TrajectoryRecord

__all__ = ["make_records", "ensemble_mean", "quantile_band", "fidelity", "FidelityReport"]


def _dev():
    return _device.device()


def _stream():
    return _device.stream_handle(_dev())


def _to_dev(a: np.ndarray, dtype=torch.float64) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=_dev(), dtype=dtype)


def make_records(logs, compartments, num_nodes: int, t_final: float, grid_points: int = DEFAULT_GRID_POINTS,
                 extra_summaries=None) -> list[TrajectoryRecord]:
    """``make_record`` for many trajectories in one launch.  ``logs`` is a
    sequence of (times f64[S_t], counts int[S_t, M]) per trial, times from 0
    and non-decreasing; record t equals
    ``make_record(times_t, counts_t, compartments, num_nodes, t_final,
    grid_points, extra_summaries[t])`` bit for bit."""
    logs = list(logs)
    comps = tuple(compartments)
    m = len(comps)
    if not logs:
        return []
    lens = np.array([len(t) for t, _ in logs], dtype=np.int64)
    if lens.min() < 1:
        raise InvalidConfigError("make_records: every log needs at least the t=0 sample")
    smax = int(lens.max())
    times = np.full((len(logs), smax), np.inf)
    counts = np.zeros((len(logs), smax, m), dtype=np.int64)
    for k, (t, c) in enumerate(logs):
        times[k, : lens[k]] = t
        counts[k, : lens[k]] = np.asarray(c, dtype=np.int64).reshape(lens[k], m)
    grid = np.linspace(0.0, t_final, grid_points)
    i_idx = comps.index("I") if "I" in comps else -1
    r_idx = comps.index("R") if "R" in comps else -1
    d_t, d_c, d_l, d_g = _to_dev(times), _to_dev(counts, torch.int64), _to_dev(lens, torch.int64), _to_dev(grid)
    frac = torch.empty((len(logs), grid_points, m), dtype=torch.float64, device=_dev())
    summ = torch.zeros((len(logs), 3), dtype=torch.float64, device=_dev())
    lib = _lib.load()
    _lib.check(lib.fs_traj_records(_lib.ptr(d_t), _lib.ptr(d_c), _lib.ptr(d_l), len(logs), smax, m, _lib.ptr(d_g),
                                   grid_points, int(num_nodes), i_idx, r_idx, _lib.ptr(frac), _lib.ptr(summ),
                                   _stream()))
    frac_h, summ_h = frac.cpu().numpy(), summ.cpu().numpy()
    extra = list(extra_summaries) if extra_summaries is not None else [None] * len(logs)
    out = []
    for k in range(len(logs)):
        summary = dict(extra[k] or {})
        if i_idx >= 0:
            summary.setdefault("peak_I", float(summ_h[k, 0]))
            summary.setdefault("peak_I_time", float(summ_h[k, 1]))
        if r_idx >= 0:
            summary.setdefault("final_R", float(summ_h[k, 2]))
        # (C, G) in Fortran order, the layout of the reference's `counts[idx].T / N`
        out.append(TrajectoryRecord(grid=grid.copy(), fractions=frac_h[k].T, compartments=comps, summary=summary))
    return out


def _check_same_grid(a, b) -> None:
    """R/analysis.py:183-189."""
    if not a or not b:
        raise GridMismatchError("empty ensemble")
    if a[0].compartments != b[0].compartments:
        raise GridMismatchError("compartment sets differ")
    if not np.array_equal(a[0].grid, b[0].grid):
        raise GridMismatchError("sample grids differ")


def _stack_dev(records) -> torch.Tensor:
    """R/analysis.py:133-134 `_stack`, uploaded: (runs, C, G) f64."""
    return _to_dev(np.stack([r.fractions for r in records]).astype(np.float64, copy=False))


def _mean_dev(x: torch.Tensor) -> torch.Tensor:
    runs = x.shape[0]
    out = torch.empty(x.shape[1:], dtype=torch.float64, device=x.device)
    _lib.check(_lib.load().fs_ensemble_mean(_lib.ptr(x), runs, x[0].numel(), _lib.ptr(out), _stream()))
    return out


def ensemble_mean(records) -> np.ndarray:
    """R/analysis.py:137-138: the pointwise mean over runs, (C, G)."""
    if not records:
        raise GridMismatchError("empty ensemble")
    return _mean_dev(_stack_dev(records)).cpu().numpy()


def _quantile_plan(n: int, qs) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """numpy's "linear" virtual index, _get_indexes and _get_gamma
    (numpy/lib/_function_base_impl.py) for sample size n."""
    q = np.asarray(qs, dtype=np.float64)
    vi = (n - 1) * q
    prev = np.floor(vi)
    nxt = prev + 1
    above = vi >= n - 1
    prev[above] = -1
    nxt[above] = -1
    below = vi < 0
    prev[below] = 0
    nxt[below] = 0
    gamma = np.asarray(vi - prev, dtype=np.float64)
    return prev.astype(np.int64), nxt.astype(np.int64), gamma


def _column_quantiles(x: torch.Tensor, n: int, ncols: int, row_stride: int, col_stride: int, qs) -> np.ndarray:
    prev, nxt, gamma = _quantile_plan(n, qs)
    out = torch.empty((len(qs), ncols), dtype=torch.float64, device=x.device)
    _lib.check(_lib.load().fs_column_quantiles(_lib.ptr(x), n, ncols, row_stride, col_stride, len(qs),
                                               prev.ctypes.data, nxt.ctypes.data, gamma.ctypes.data, _lib.ptr(out),
                                               _stream()))
    return out.cpu().numpy()


def quantile_band(records, label: str, q_lo: float = 0.25, q_hi: float = 0.75) -> tuple[np.ndarray, np.ndarray]:
    """R/analysis.py:141-148: pointwise cross-run quantiles of one
    compartment's fraction."""
    ci = records[0].compartments.index(label)
    x = _stack_dev(records)
    runs, m, g = x.shape
    sub = x[:, ci, :]
    q = _column_quantiles(sub, runs, g, m * g, 1, [q_lo, q_hi])
    return q[0], q[1]


def _percentile_levels(level: float = 0.95) -> tuple[float, float]:
    lo = (1.0 - level) / 2.0  # R/analysis.py:160-162
    return lo, 1.0 - lo


@dataclass
class FidelityReport:
    """R/analysis.py:165-174."""

    l_inf: float
    l2: float
    err_peak_i: float
    err_final_r: float | None
    per_run_peak_err: float
    per_run_final_err: float | None
    ci: dict = field(default_factory=dict)


def fidelity(a, b, resamples: int = 1000, seed: int = 0) -> FidelityReport:
    """Trajectory and summary errors of ensemble a against ensemble b, with
    95% percentile bootstrap CIs over runs (R/analysis.py:192-256)."""
    _check_same_grid(a, b)
    comps = a[0].compartments
    A, B = _stack_dev(a), _stack_dev(b)
    na, m, g = A.shape
    nb = B.shape[0]
    i_idx = comps.index("I") if "I" in comps else None
    r_idx = comps.index("R") if "R" in comps else None
    lib = _lib.load()
    st = _stream()

    # the point metrics reduce in the memory order of the records' fractions
    # (numpy keeps it through _stack and mean; the reference's records are
    # Fortran order), so the means take that layout before np.mean
    mean_a, mean_b = np.empty_like(a[0].fractions, dtype=np.float64), np.empty_like(b[0].fractions, dtype=np.float64)
    mean_a[...] = _mean_dev(A).cpu().numpy()
    mean_b[...] = _mean_dev(B).cpu().numpy()

    def metrics(ma, mb):  # R/analysis.py:205-216, on the (C, G) means
        diff = ma - mb
        out = {"l_inf": float(np.abs(diff).max()), "l2": float(np.sqrt(np.mean(diff ** 2)))}
        if i_idx is not None:
            out["err_peak_i"] = float(abs(ma[i_idx].max() - mb[i_idx].max()))
        if r_idx is not None:
            out["err_final_r"] = float(abs(ma[r_idx, -1] - mb[r_idx, -1]))
        return out

    point = metrics(mean_a, mean_b)
    ref_peak = float(mean_b[i_idx].max()) if i_idx is not None else 0.0
    ref_final = float(mean_b[r_idx, -1]) if r_idx is not None else 0.0
    peak_dev = torch.empty(na, dtype=torch.float64, device=A.device)
    final_dev = torch.empty(na, dtype=torch.float64, device=A.device)
    _lib.check(lib.fs_run_deviation(_lib.ptr(A), na, m, g, -1 if i_idx is None else i_idx,
                                    -1 if r_idx is None else r_idx, ref_peak, ref_final, _lib.ptr(peak_dev),
                                    _lib.ptr(final_dev), st))

    rng = np.random.default_rng(seed)  # R/analysis.py:153-157, same draw order (a, then b)
    cnt_a = rng.multinomial(na, np.full(na, 1.0 / na), size=resamples)
    cnt_b = rng.multinomial(nb, np.full(nb, 1.0 / nb), size=resamples)
    d_ca, d_cb = _to_dev(cnt_a, torch.int64), _to_dev(cnt_b, torch.int64)
    scratch = torch.empty(resamples * (na + nb), dtype=torch.float64, device=A.device)
    samples = torch.zeros((6, resamples), dtype=torch.float64, device=A.device)
    _lib.check(lib.fs_bootstrap_metrics(_lib.ptr(A), na, _lib.ptr(B), nb, m, g, _lib.ptr(d_ca), _lib.ptr(d_cb),
                                        resamples, -1 if i_idx is None else i_idx, -1 if r_idx is None else r_idx,
                                        _lib.ptr(peak_dev), _lib.ptr(final_dev), _lib.ptr(scratch),
                                        _lib.ptr(samples), st))
    rows = [("l_inf", 0), ("l2", 1)]
    if i_idx is not None:
        rows.append(("err_peak_i", 2))
    if r_idx is not None:
        rows.append(("err_final_r", 3))
    if i_idx is not None:
        rows.append(("per_run_peak_err", 4))
    if r_idx is not None:
        rows.append(("per_run_final_err", 5))
    q = _column_quantiles(samples, resamples, 6, 1, resamples, list(_percentile_levels()))
    ci = {k: (float(q[0, j]), float(q[1, j])) for k, j in rows}

    prp = peak_dev.cpu().numpy() if i_idx is not None else None
    prf = final_dev.cpu().numpy() if r_idx is not None else None
    return FidelityReport(
        l_inf=point["l_inf"],
        l2=point["l2"],
        err_peak_i=point.get("err_peak_i", 0.0),
        err_final_r=point.get("err_final_r"),
        per_run_peak_err=float(prp.mean()) if prp is not None else 0.0,
        per_run_final_err=float(prf.mean()) if prf is not None else None,
        ci=ci,
    )
