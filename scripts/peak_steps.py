"""Eager C2 steps from t = 0 into the epidemic peak (for an ncu capture of a
peak-window step: `ncu -k regex:^k_step_incr$ -s 800 -c 1 python scripts/peak_steps.py`)
and, without ncu, per-step event times across the run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import renewal as R

n_steps = int(sys.argv[1]) if len(sys.argv) > 1 else 850
g = fs.gen_fixed_degree(1_000_000, 10, seed=1)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
st = fs.init_renewal_state(g, m, cfg, 7)
plan = R._build_plan(g, m, cfg, False)
eng = st._bind(plan, 7, materialize=False)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_steps)]
for k in range(n_steps):
    ev[k][0].record()
    eng.step(1, False, False)
    ev[k][1].record()
torch.cuda.synchronize()
t = [a.elapsed_time(b) * 1e3 for a, b in ev]
w = max(1, n_steps // 17)
print("eager us/step by window of", w, ":", [round(sum(t[i:i + w]) / len(t[i:i + w]), 1) for i in range(0, n_steps, w)])
s = eng.scalars()
print("counts", list(s.counts)[:4], "clock", round(s.clock, 2))
