"""Full run_renewal (t_final 50) device-time per step with / without the cohort
hazard table across N: where the table starts to pay (FS_NO_MEMO is read at
engine creation)."""
import os, sys, time
os.environ["FS_E2E_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_22092_b200 as fs
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
for n in (10_000, 30_000, 100_000, 300_000, 1_000_000):
    g = fs.gen_fixed_degree_device(n, 10, seed=1)
    out = []
    for flag in (None, "1"):
        if flag: os.environ["FS_NO_MEMO"] = flag
        else: os.environ.pop("FS_NO_MEMO", None)
        best = None
        for _ in range(3):
            rec = fs.run_renewal(g, m, fs.RenewalConfig(), 7, 50.0)
            bm = float(np.sum(rec.summary["batch_ms"]))
            best = bm if best is None else min(best, bm)
        out.append(round(best * 1e3 / rec.summary["step_count"], 2))
    print(n, "us/step memo on / off:", out)
