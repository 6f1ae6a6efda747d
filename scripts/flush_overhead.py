"""Event-timed cost of a trivial kernel after the bench's L2 flush, next to
the step kernel: how much of the flushed 'value' is fixed overhead."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import renewal as R
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
x = torch.zeros(1, device="cuda")
def timed(fn, n=50, do_flush=True):
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if do_flush:
            flush.zero_(); flush_rd.max()
        a.record(); fn(); b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    return np.median([s.elapsed_time(e) * 1e3 for s, e in ts])
print("empty (x.add_) after flush: %.1f us" % timed(lambda: x.add_(1)))
print("empty (x.add_) no flush:    %.1f us" % timed(lambda: x.add_(1), do_flush=False))
g = fs.gen_fixed_degree(1_000_000, 10, seed=1)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
st = fs.init_renewal_state(g, m, cfg, 7)
eng = st._bind(R._build_plan(g, m, cfg, False), 7, False)
eng.step(10, False, False)
print("step after flush:           %.1f us" % timed(lambda: eng.step(1, False, False), n=50))
print("step no flush:              %.1f us" % timed(lambda: eng.step(1, False, False), n=50, do_flush=False))
print("2 steps after flush:        %.1f us" % timed(lambda: eng.step(2, False, False), n=25))
