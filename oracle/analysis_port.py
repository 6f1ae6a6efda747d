"""numpy restatement of the reference's trajectory / ensemble analysis
 — the checker for csrc/fs_analysis.cu.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Pinned against the
reference's own outputs: tests/golden/make_analysis_golden.py imports
/root/reference/pkg/src/spreadsim and writes tests/golden/analysis.npz;
tests/test_analysis.py asserts this module reproduces them (bit for bit
except the bootstrap resample means, which the reference computes as a BLAS
matrix product; here they are explicit sequential sums, as on the device).

R = /root/reference/pkg/src/spreadsim.
"""

from __future__ import annotations

import numpy as np


def make_record_arrays(times, counts, num_nodes: int, t_final: float, grid_points: int):
    """R/trajectory.py:48-53: (grid, fractions (C, G))."""
    t = np.asarray(times, dtype=np.float64)
    c = np.asarray(counts, dtype=np.float64)
    grid = np.linspace(0.0, t_final, grid_points)
    idx = np.clip(np.searchsorted(t, grid, side="right") - 1, 0, len(t) - 1)
    return grid, c[idx].T / float(num_nodes)


def ensemble_mean(stack: np.ndarray) -> np.ndarray:
    """R/analysis.py:137-138: mean over axis 0 = sequential sum in run order
    (numpy reduces an outer axis row by row), then / runs."""
    s = stack[0].copy(order="K")  # numpy keeps the records' memory order
    for i in range(1, stack.shape[0]):
        s = s + stack[i]
    return s / stack.shape[0]


def quantile_linear(x: np.ndarray, q: float) -> np.ndarray:
    """np.quantile(x, q, axis=0), method "linear" (numpy
    _function_base_impl._quantile / _get_indexes / _lerp), written out."""
    n = x.shape[0]
    s = np.sort(x, axis=0)
    vi = (n - 1) * q
    prev = int(np.floor(vi))
    nxt = prev + 1
    if vi >= n - 1:
        prev = nxt = -1
    if vi < 0:
        prev = nxt = 0
    gamma = vi - prev
    a, b = s[prev], s[nxt]
    d = b - a
    return b - d * (1 - gamma) if gamma >= 0.5 else a + d * gamma


def fidelity_samples(A: np.ndarray, B: np.ndarray, wa: np.ndarray, wb: np.ndarray, i_idx, r_idx,
                     per_run_peak, per_run_final) -> dict[str, np.ndarray]:
    """The per-resample metrics of R/analysis.py:226-240 with the resample
    means as explicit sums over runs."""
    ma = np.einsum("ri,ij->rj", wa, A.reshape(A.shape[0], -1), optimize=False).reshape(-1, *A.shape[1:])
    mb = np.einsum("ri,ij->rj", wb, B.reshape(B.shape[0], -1), optimize=False).reshape(-1, *B.shape[1:])
    d = ma - mb
    out = {"l_inf": np.abs(d).reshape(len(d), -1).max(axis=1), "l2": np.sqrt((d.reshape(len(d), -1) ** 2).mean(axis=1))}
    if i_idx is not None:
        out["err_peak_i"] = np.abs(ma[:, i_idx].max(axis=1) - mb[:, i_idx].max(axis=1))
    if r_idx is not None:
        out["err_final_r"] = np.abs(ma[:, r_idx, -1] - mb[:, r_idx, -1])
    if i_idx is not None:
        out["per_run_peak_err"] = wa @ per_run_peak
    if r_idx is not None:
        out["per_run_final_err"] = wa @ per_run_final
    return out


def fidelity(A: np.ndarray, B: np.ndarray, comps, resamples: int, seed: int):
    """R/analysis.py:192-256 on stacked ensembles: (point metrics dict,
    per_run means, ci dict)."""
    i_idx = comps.index("I") if "I" in comps else None
    r_idx = comps.index("R") if "R" in comps else None
    mean_a, mean_b = ensemble_mean(A), ensemble_mean(B)
    diff = mean_a - mean_b
    point = {"l_inf": float(np.abs(diff).max()), "l2": float(np.sqrt(np.mean(diff ** 2)))}
    if i_idx is not None:
        point["err_peak_i"] = float(abs(mean_a[i_idx].max() - mean_b[i_idx].max()))
    if r_idx is not None:
        point["err_final_r"] = float(abs(mean_a[r_idx, -1] - mean_b[r_idx, -1]))
    prp = np.abs(A[:, i_idx, :].max(axis=1) - mean_b[i_idx].max()) if i_idx is not None else None
    prf = np.abs(A[:, r_idx, -1] - mean_b[r_idx, -1]) if r_idx is not None else None
    rng = np.random.default_rng(seed)
    wa = rng.multinomial(A.shape[0], np.full(A.shape[0], 1.0 / A.shape[0]), size=resamples) / float(A.shape[0])
    wb = rng.multinomial(B.shape[0], np.full(B.shape[0], 1.0 / B.shape[0]), size=resamples) / float(B.shape[0])
    samples = fidelity_samples(A, B, wa, wb, i_idx, r_idx, prp, prf)
    lo = (1.0 - 0.95) / 2.0
    ci = {k: (float(quantile_linear(v, lo)), float(quantile_linear(v, 1.0 - lo))) for k, v in samples.items()}
    per_run = (float(prp.mean()) if prp is not None else 0.0, float(prf.mean()) if prf is not None else None)
    return point, per_run, ci
