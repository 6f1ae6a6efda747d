"""Ensemble golden statistics from the REFERENCE implementation.

    python tests/golden/make_ensemble_golden.py

Runs, with the reference imported unmodified from /root/reference, the
ensembles of its acceptance suite (T/test_acceptance.py:34-79: ER N=1000,
d=8, seed 20250809, 100 runs, 10 E seeds, t_final=50):

  * "renewal" — the CPU tau-leaping engine, RenewalConfig() (eps = 0.03);
  * "exact"   — the exact next-reaction oracle gillespie_renewal_seir
                (R/exact.py:187-310).

and stores the per-run summaries (peak_I, peak_I_time, final_R, step_count)
and the ensemble-mean trajectories in tests/golden/ensemble.npz.  The GPU
test reproduces the tau-leap runs trajectory by trajectory (same per-trial
seeds derive_seed(seed, trial), R/analysis.py:61-74) and compares the
ensemble with the exact oracle within Monte Carlo error.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import spreadsim as ss  # noqa: E402
from spreadsim.analysis import run_ensemble  # noqa: E402
from spreadsim.renewal import RenewalConfig  # noqa: E402

ACC_SEED, RUNS, T_FINAL, SEEDS = 20250809, 100, 50.0, 10


def summaries(recs):
    return {k: np.array([r.summary[k] for r in recs], dtype=np.float64)
            for k in ("peak_I", "peak_I_time", "final_R", "step_count") if k in recs[0].summary}


def main() -> None:
    g = ss.gen_erdos_renyi(1000, 8.0, seed=ACC_SEED)
    m = ss.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    workers = len(os.sched_getaffinity(0))
    out, meta = {}, {"graph": ["gen_erdos_renyi", 1000, 8.0, ACC_SEED], "model": "seir_standard(0.25,5,4,7.5,5)",
                     "seed": ACC_SEED, "runs": RUNS, "t_final": T_FINAL, "seed_count": SEEDS}
    for engine, cfg in (("renewal", RenewalConfig()), ("exact", None)):
        t0 = time.time()
        recs = run_ensemble(engine, g, m, cfg, ACC_SEED, T_FINAL, RUNS, workers=workers, seed_count=SEEDS)
        for k, v in summaries(recs).items():
            out[f"{engine}__{k}"] = v
        out[f"{engine}__mean"] = np.mean([r.fractions for r in recs], axis=0)
        meta[f"{engine}_seconds"] = round(time.time() - t0, 1)
        print(engine, {k: float(v.mean()) for k, v in summaries(recs).items()}, meta[f"{engine}_seconds"], "s")
    out["grid"] = recs[0].grid
    np.savez_compressed(OUT / "ensemble.npz", **out)
    (OUT / "ensemble.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
