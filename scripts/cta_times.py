"""Timeline of the streaming step kernel inside one CUDA-graph batch:
per step, first CTA start / last CTA work end / finish stamp, and the gap to
the next step.  Run with FS_DEBUG_TIMES=1 (optionally FS_NO_PDL=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import renewal as R, _lib
lib = _lib.load()
lib.fs_engine_debug_times.restype = ctypes.c_int
lib.fs_engine_debug_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
g = fs.gen_fixed_degree(1_000_000, 10, seed=1)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig(steps_per_batch=16)
st = fs.init_renewal_state(g, m, cfg, 7)
plan = R._build_plan(g, m, cfg, False)
eng = st._bind(plan, 7, False)
eng.run_batch(False)  # capture + warm
buf = np.zeros((16, 1024, 4), dtype=np.uint64)
lib.fs_engine_debug_times(eng.handle, buf.ctypes.data, 1024)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); eng.run_batch(False); e1.record(); torch.cuda.synchronize()
print(f"graph batch of 16 steps: {e0.elapsed_time(e1)*1e3/16:.1f} us/step (events)")
n = lib.fs_engine_debug_times(eng.handle, buf.ctypes.data, 1024)
b = buf[:, :n, :].astype(np.int64)
rows = []
for s in range(16):
    start = b[s, :, 0]; end = b[s, :, 1]; fin = b[s, :, 3]
    if start.min() == 0:
        continue
    rows.append((start.min(), np.median(start), start.max(), end.max(), fin.max()))
rows.sort()
t0 = rows[0][0]
for i, (smin, smed, smax, emax, fmax) in enumerate(rows):
    nxt = rows[i + 1][0] if i + 1 < len(rows) else None
    print(f"step {i:2d}: start {(smin-t0)/1e3:7.1f} (med +{(smed-smin)/1e3:4.1f}, max +{(smax-smin)/1e3:4.1f})  work end +{(emax-smin)/1e3:5.1f}"
          f"  finish +{(fmax-smin)/1e3:5.1f}  next start +{((nxt-smin)/1e3 if nxt else float('nan')):5.1f} us")
