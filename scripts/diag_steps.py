"""Per-step kernel time across the bench window (eager, no flush, and with
the bench's L2 flush), uniform-S-age status, for one workload."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_22092_b200 as fs  # noqa: E402
from paper_2604_22092_b200 import renewal as R  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g, m = bench.build_inputs(w)
cfg = fs.RenewalConfig(mixed_precision=bool(w.get("mixed")))
st = fs.init_renewal_state(g, m, cfg, 7)
plan = R._build_plan(g, m, cfg, st.mixed_precision)
eng = st._bind(plan, 7, materialize=False)
eng.step(10, False, False)
snap = eng.snapshot()
print("uni", eng.uniform_s_age())
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
for mode in ("eager", "flushed"):
    eng.restore(snap)
    print(mode, "uni after restore", eng.uniform_s_age())
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for k in range(steps):
        if mode == "flushed":
            flush.zero_()
            flush_rd.max()
        ev[k][0].record()
        eng.step(1, False, False)
        ev[k][1].record()
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in ev]
    print(mode, " ".join("%d:%.0f" % (k, t[k]) for k in range(0, steps, max(1, steps // 20))), "mean %.1f" % (sum(t) / steps))
s = eng.scalars()
print("counts", list(s.counts)[:4], "clock", s.clock)
