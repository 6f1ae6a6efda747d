"""Deterministic synthetic trajectory logs for the analysis parity tests
(tests/test_analysis.py, tests/golden/make_analysis_golden.py).  Plain
numpy, counter-based (splitmix64 finaliser over (case, trial, step)), so the
golden script and the tests rebuild the same inputs without storing them."""

from __future__ import annotations

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _u(case: int, trial: int, k: np.ndarray, lane: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (np.uint64(case) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(trial) * np.uint64(0xD1B54A32D192ED03)
             + k.astype(np.uint64) * np.uint64(0xA24BAED4963EE407) + np.uint64(lane) * np.uint64(0x9FB21C651E98DF25))
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def trajectory_log(case: int, trial: int, compartments, n: int, t_final: float, shift: float = 0.0):
    """(times, counts) of one synthetic epidemic-shaped run: steps of
    random length from t=0 until past t_final, compartment counts that sum
    to n (an I bump, a monotone R; S / E take the rest)."""
    m = len(compartments)
    steps = 40 + int(_u(case, trial, np.array([0]), 7)[0] * 160)
    k = np.arange(steps)
    dt = (0.6 + 0.8 * _u(case, trial, k, 1)) * (t_final * 1.1 / steps)
    times = np.concatenate([[0.0], np.cumsum(dt)])
    ph = times / t_final
    noise = 0.85 + 0.3 * _u(case, trial, np.arange(steps + 1), 2)
    i_frac = np.clip(0.25 * np.sin(np.pi * np.clip(ph + shift, 0, 1)) ** 2 * noise, 0, 0.4)
    r_frac = np.clip(0.7 * np.clip(ph + shift, 0, 1) * (0.9 + 0.2 * _u(case, trial, np.array([1]), 3)[0]), 0, 0.55)
    counts = np.zeros((steps + 1, m), dtype=np.int64)
    rest = np.full(steps + 1, n, dtype=np.int64)
    for c, label in enumerate(compartments):
        if label == "I":
            counts[:, c] = np.floor(i_frac * n).astype(np.int64)
        elif label == "R":
            counts[:, c] = np.floor(r_frac * n).astype(np.int64)
        elif label == "E":
            counts[:, c] = np.floor(0.1 * n * _u(case, trial, np.arange(steps + 1), 4)).astype(np.int64)
    rest -= counts.sum(axis=1)
    s = compartments.index("S")
    counts[:, s] += rest
    return times, counts


CASES = {
    # name: (compartments, n, t_final, grid_points, runs_a, runs_b, shift_b, resamples, seed)
    "seir": (("S", "E", "I", "R"), 10_000, 30.0, 501, 48, 64, 0.02, 300, 5),
    "sis": (("S", "I"), 2_000, 20.0, 201, 33, 20, 0.0, 250, 1),
    "sir_small": (("S", "I", "R"), 997, 10.0, 101, 7, 9, -0.05, 120, 11),
    "se_only": (("S", "E"), 500, 5.0, 51, 12, 12, 0.0, 64, 3),
}


def ensemble_logs(name: str):
    comps, n, t_final, _, ra, rb, shift, _, _ = CASES[name]
    case = list(CASES).index(name) * 2
    a = [trajectory_log(case, t, comps, n, t_final) for t in range(ra)]
    b = [trajectory_log(case + 1, t, comps, n, t_final, shift) for t in range(rb)]
    return a, b
