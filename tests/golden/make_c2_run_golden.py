"""Whole-run golden for the headline configuration C2, from the REFERENCE.

    python tests/golden/make_c2_run_golden.py      (~6 min on one core)

Imports /root/reference/pkg/src/spreadsim unmodified and runs exactly the
call the bench's e2e leg makes:

    run_renewal(gen_fixed_degree(1_000_000, 10, seed=1),
                seir_standard(0.25, 5, 4, 7.5, 5), RenewalConfig(),
                seed=7, t_final=50)            (R/renewal.py:632-663)

and stores the whole TrajectoryRecord (f64 fractions on the 501-point grid,
R/trajectory.py:31-61) plus its summary in tests/golden/c2_run.npz.  The
CSR hash is stored too, so the GPU test can show it ran on the same graph.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import spreadsim as ss  # noqa: E402
from spreadsim import renewal as R  # noqa: E402


def main() -> None:
    t0 = time.time()
    g = ss.gen_fixed_degree(1_000_000, 10, seed=1)
    h = hashlib.sha256()
    for a in (g.row_offsets.astype(np.int64), g.col_indices.astype(np.int32), g.weights.astype(np.float32)):
        h.update(np.ascontiguousarray(a).tobytes())
    t1 = time.time()
    m = ss.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    rec = ss.run_renewal(g, m, R.RenewalConfig(), seed=7, t_final=50.0)
    t2 = time.time()
    s = rec.summary
    np.savez_compressed(OUT / "c2_run.npz", fractions=rec.fractions, grid=rec.grid,
                        summary=np.array([s["peak_I"], s["peak_I_time"], s["final_R"], s["step_count"]]))
    meta = {"graph": ["gen_fixed_degree", 1_000_000, 10, 1], "csr_sha256": h.hexdigest(),
            "model": "seir_standard(0.25,5,4,7.5,5)", "cfg": "RenewalConfig()", "seed": 7, "t_final": 50.0,
            "summary": {k: (float(v) if isinstance(v, (int, float, np.floating, np.integer)) else str(v))
                        for k, v in s.items()},
            "graph_seconds": round(t1 - t0, 1), "run_seconds": round(t2 - t1, 1)}
    (OUT / "c2_run.json").write_text(json.dumps(meta, indent=1))
    print(json.dumps(meta["summary"]), meta["run_seconds"], "s")


if __name__ == "__main__":
    main()
