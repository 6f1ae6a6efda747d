"""Repeated run_renewal phases at C1 size, to find where e2e outliers go."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import renewal as R
g = fs.gen_fixed_degree(10_000, 10, seed=1)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
names = ["init", "plan", "bind", "batch1", "rest", "unbind"]
rows = []
for r in range(int(os.environ.get("REPS", "12"))):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    st = R.init_renewal_state(g, m, cfg, 7); t.append(time.perf_counter())
    plan = R._build_plan(g, m, cfg, st.mixed_precision); t.append(time.perf_counter())
    eng = st._bind(plan, 7, materialize=False); t.append(time.perf_counter())
    eng.run_batch(materialize=False); eng.read_log(0, 50); t.append(time.perf_counter())
    done, clock = 50, 0.0
    while clock < 50.0:
        eng.run_batch(materialize=False)
        c, _, _ = eng.read_log(done, 50)
        done += 50
        clock = float(c[-1])
    t.append(time.perf_counter())
    st._unbind(); torch.cuda.synchronize(); t.append(time.perf_counter())
    rows.append(np.diff(t) * 1e3)
rows = np.array(rows)
for i, n in enumerate(names):
    print(f"{n:7s} ms:", " ".join(f"{v:6.1f}" for v in rows[:, i]))
