"""Golden outputs of the REFERENCE trajectory / analysis functions.

    python tests/golden/make_analysis_golden.py

Imports /root/reference/pkg/src/spreadsim unmodified and evaluates
make_record (R/trajectory.py:31-61) on every synthetic log of
tests/_analysis_cases.py, then ensemble_mean (R/analysis.py:137-138),
quantile_band (:141-148) and fidelity (:192-256) on the two ensembles of
each case.  Written to tests/golden/analysis.npz; read by
tests/test_analysis.py.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
from spreadsim.analysis import ensemble_mean, fidelity, quantile_band  # noqa: E402
from spreadsim.trajectory import make_record  # noqa: E402

from tests._analysis_cases import CASES, ensemble_logs  # noqa: E402


def main() -> None:
    out = {}
    for name, (comps, n, t_final, gp, _, _, _, resamples, seed) in CASES.items():
        la, lb = ensemble_logs(name)
        ra = [make_record(t, c, comps, n, t_final, gp) for t, c in la]
        rb = [make_record(t, c, comps, n, t_final, gp) for t, c in lb]
        out[f"{name}__frac_a"] = np.stack([r.fractions for r in ra])
        keys = [k for k in ("peak_I", "peak_I_time", "final_R") if k in ra[0].summary]
        out[f"{name}__summary_keys"] = np.array(keys)
        out[f"{name}__summary_a"] = np.array([[r.summary[k] for k in keys] for r in ra]).reshape(len(ra), len(keys))
        out[f"{name}__mean_a"] = ensemble_mean(ra)
        for label in comps:
            lo, hi = quantile_band(ra, label, 0.1, 0.9)
            out[f"{name}__band_{label}"] = np.stack([lo, hi])
        rep = fidelity(ra, rb, resamples=resamples, seed=seed)
        out[f"{name}__point"] = np.array([rep.l_inf, rep.l2, rep.err_peak_i,
                                          np.nan if rep.err_final_r is None else rep.err_final_r,
                                          rep.per_run_peak_err,
                                          np.nan if rep.per_run_final_err is None else rep.per_run_final_err])
        out[f"{name}__ci_keys"] = np.array(list(rep.ci))
        out[f"{name}__ci"] = np.array([rep.ci[k] for k in rep.ci])
    np.savez_compressed(Path(__file__).resolve().parent / "analysis.npz", **out)
    print(sorted(k for k in out if k.endswith("ci_keys")), {k: v.shape for k, v in out.items() if "frac" in k})


if __name__ == "__main__":
    main()
