"""Per-batch wall times of one run_renewal (FS_E2E_TRACE) at C2, in 5 windows."""
import os, sys
os.environ["FS_E2E_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_22092_b200 as fs
g = fs.gen_fixed_degree(1_000_000, 10, seed=1)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
for rep in range(3):
    rec = fs.run_renewal(g, m, fs.RenewalConfig(), 7, 50.0)
    bm = np.array(rec.summary["batch_ms"])
    w = np.array_split(bm, 5)
    print(f"rep {rep}: total {bm.sum():.1f} ms, per-window us/step", [round(x.mean() * 1e3 / 50, 1) for x in w])
