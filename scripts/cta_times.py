"""Per-CTA start/end (globaltimer) of the step kernel — load-balance probe.
Run with FS_DEBUG_TIMES=1."""
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
cfg = fs.RenewalConfig()
st = fs.init_renewal_state(g, m, cfg, 7)
plan = R._build_plan(g, m, cfg, False)
eng = st._bind(plan, 7, False)
eng.step(20, False, False)
buf = np.zeros((1024, 4), dtype=np.uint64)
lib.fs_engine_debug_times(eng.handle, buf.ctypes.data, 1024)
for rep in range(3):
    eng.step(1, False, False)
    n = lib.fs_engine_debug_times(eng.handle, buf.ctypes.data, 1024)
    b = buf[:n].astype(np.int64)
    t0 = b[:, 0].min()
    start, end, sm = (b[:, 0] - t0) / 1e3, (b[:, 1] - t0) / 1e3, b[:, 2]
    order = np.argsort(-end)
    print(f"rep {rep}: ctas {n} kernel span {end.max():.1f} us; end p50 {np.median(end):.1f} p90 {np.percentile(end,90):.1f}; start max {start.max():.1f}")
    print("  slowest:", [(int(i), int(sm[i]), round(float(start[i]),1), round(float(end[i]),1)) for i in order[:8]])
    print("  fastest:", [(int(i), int(sm[i]), round(float(start[i]),1), round(float(end[i]),1)) for i in order[-4:]])
