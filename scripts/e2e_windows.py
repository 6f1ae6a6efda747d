"""Per-window step cost of one full run_renewal (FS_E2E_TRACE batch times) for a
bench workload: python scripts/e2e_windows.py c4 [windows]"""
import os, sys
os.environ["FS_E2E_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2604_22092_b200 as fs

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g, m = bench.build_inputs(w)
cfg = fs.RenewalConfig(mixed_precision=bool(w.get("mixed")))
for rep in range(2):
    rec = fs.run_renewal(g, m, cfg, bench.SIM_SEED, w.get("t_final", 50.0))
    bm = np.array(rec.summary["batch_ms"])
    print(f"rep {rep}: total {bm.sum():.1f} ms, per-window us/step",
          [round(x.mean() * 1e3 / cfg.steps_per_batch, 1) for x in np.array_split(bm, nw)])
