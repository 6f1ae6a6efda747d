"""Exact-oracle ensemble statistics for the Weibull / Erlang model of C3.

    python tests/golden/make_we_ensemble_golden.py      (~1 min)

The reference's exact next-reaction oracle, `gillespie_renewal_seir`
(R/exact.py:187-310), schedules every nodal event by sampling its holding
time once at entry (`_sample_holding`, R/exact.py:59-64).  It ships samplers
for log-normal and exponential holding times only, and routes to the
non-Markovian oracle only when `ModelSpec.age_dependent()` is true
(R/models.py:100-101, R/analysis.py:82-89).  This script imports the
reference unmodified from /root/reference and patches exactly those two
points, nothing else:

  * `_sample_holding`: Weibull(k, lam) by inverse CDF,
    lam * (-log1p(-u))**(1/k); Erlang(k, r) by `scipy.stats.gamma.ppf(u, k,
    scale=1/r)`; u is the oracle's own counter-based draw `_draw(seed,
    counter)` (one draw per scheduled event, as for the exponential);
  * `ModelSpec.age_dependent`: also true for "weibull" / "erlang".

The model is BASELINE C3's (E->I Weibull k=1.247568, lam=5.365966; I->R
Erlang k=3, r=0.4; beta=0.25), on the reference's acceptance
ensemble graphs.  Per-run summaries (peak_I, peak_I_time, final_R) go to
tests/golden/we_ensemble.npz; tests/test_ensemble.py compares the GPU
tau-leaping ensemble with them within Monte Carlo error.
"""

from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np
from scipy import stats

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import spreadsim as ss  # noqa: E402
from spreadsim import exact as X  # noqa: E402
from spreadsim import models as M  # noqa: E402
from spreadsim.analysis import _run_single  # noqa: E402
from spreadsim.rng import derive_seed  # noqa: E402

WEIBULL = SimpleNamespace(k=1.247568, lam=5.365966)
ERLANG = SimpleNamespace(k=3, rate=0.4)
SEED, RUNS, T_FINAL, SEEDS = 20250809, 200, 50.0, 10
GRAPHS = {"er1000": ("gen_erdos_renyi", (1000, 8.0)), "ba1000": ("gen_barabasi_albert", (1000, 5))}

_orig_sample = X._sample_holding
_orig_age_dep = M.ModelSpec.age_dependent


def _sample_holding(seed: int, counter: int, holding) -> float:
    if holding.kind == "weibull":
        u = X._draw(seed, counter)
        return holding.params.lam * (-math.log1p(-u)) ** (1.0 / holding.params.k)
    if holding.kind == "erlang":
        u = X._draw(seed, counter)
        return float(stats.gamma.ppf(u, holding.params.k, scale=1.0 / holding.params.rate))
    return _orig_sample(seed, counter, holding)


def _age_dependent(self) -> bool:
    return _orig_age_dep(self) or any(h.kind in ("weibull", "erlang") for _, h in self.nodal.values())


X._sample_holding = _sample_holding
M.ModelSpec.age_dependent = _age_dependent


def model() -> M.ModelSpec:
    return M.ModelSpec("seir-we", ("S", "E", "I", "R"), 0.25, 0, 1,
                       {1: (2, M.Holding(kind="weibull", params=WEIBULL)),
                        2: (3, M.Holding(kind="erlang", params=ERLANG))}, infectious=2)


def main() -> None:
    m = model()
    out, meta = {}, {"model": "seir_weibull_erlang(0.25): E->I Weibull(1.247568, 5.365966), I->R Erlang(3, 0.4)",
                     "seed": SEED, "runs": RUNS, "t_final": T_FINAL, "seed_count": SEEDS,
                     "oracle": "spreadsim.exact.gillespie_renewal_seir with _sample_holding/age_dependent patched"}
    for name, (fn, args) in GRAPHS.items():
        g = getattr(ss, fn)(*args, seed=SEED)
        t0 = time.time()
        recs = [_run_single("exact", g, m, None, derive_seed(SEED, t), T_FINAL, 501, SEEDS, None) for t in range(RUNS)]
        assert all(r.summary["engine"] == "exact" for r in recs)
        for k in ("peak_I", "peak_I_time", "final_R"):
            out[f"{name}__{k}"] = np.array([r.summary[k] for r in recs], dtype=np.float64)
        out[f"{name}__mean"] = np.mean([r.fractions for r in recs], axis=0)
        meta[name] = {"graph": [fn, *args, SEED], "seconds": round(time.time() - t0, 1),
                      **{k: float(out[f"{name}__{k}"].mean()) for k in ("peak_I", "peak_I_time", "final_R")}}
        print(name, meta[name])
    np.savez_compressed(OUT / "we_ensemble.npz", **out)
    (OUT / "we_ensemble.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
