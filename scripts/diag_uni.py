"""Diagnostics for the uniform-S-age kernel: is it on, and per-step time of
the step kernel alone (CUDA events, L2 warm) for a workload."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_22092_b200 as fs  # noqa: E402
from paper_2604_22092_b200 import renewal as R  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
g, m = bench.build_inputs(w)
cfg = fs.RenewalConfig(mixed_precision=bool(w.get("mixed")))
st = fs.init_renewal_state(g, m, cfg, 7)
plan = R._build_plan(g, m, cfg, st.mixed_precision)
eng = st._bind(plan, 7, materialize=False)
print("uniform_s_age", eng.uniform_s_age(), "kernels/step", eng.kernels_per_step())
eng.step(10, False, False)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.step(20, False, False)
    e1.record()
    torch.cuda.synchronize()
    print("eager 20 steps: %.1f us/step" % (e0.elapsed_time(e1) * 1e3 / 20), "counts", st.counts.tolist())
