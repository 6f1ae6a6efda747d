"""bench-like e2e reps of run_renewal on a host graph, with per-batch wall times (FS_E2E_TRACE)."""
import os, sys, time
os.environ["FS_E2E_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2604_22092_b200 as fs
w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
g, m = bench.build_inputs(w)
cfg = fs.RenewalConfig()
for rep in range(5):
    g.__dict__.pop("_fs_device_cache", None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rec = fs.run_renewal(g, m, cfg, 7, 50.0)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    bm = np.array(rec.summary["batch_ms"])
    print(f"rep {rep}: wall {wall*1e3:.1f} ms setup {rec.summary['setup_s']*1e3:.1f} ms, batches {len(bm)} "
          f"record {rec.summary['record_ms']} unbind {rec.summary['unbind_ms']} ms, sum {bm.sum():.1f} median {np.median(bm):.2f} max {bm.max():.1f} at {int(bm.argmax())}; top: {sorted(bm)[-4:]}")
