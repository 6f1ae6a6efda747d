"""Where run_renewal's wall time goes at C2 (host phases, synchronised)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_22092_b200 as fs  # noqa: E402
from paper_2604_22092_b200 import renewal as R  # noqa: E402

g = fs.gen_fixed_degree(1_000_000, 10, seed=1)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
for rep in range(3):
    g.__dict__.pop("_fs_device_cache", None)
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    dg = R.device_graph(g, False)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    st = fs.init_renewal_state(g, m, cfg, 7)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    plan = R._build_plan(g, m, cfg, False)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    eng = st._bind(plan, 7, materialize=False)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    eng.run_batch(False)
    eng.read_log(0, 50)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    done, clock = 50, 0.0
    while clock < 50.0:
        eng.run_batch(False)
        clocks, _, _ = eng.read_log(done, 50)
        done += 50
        clock = float(clocks[-1])
    torch.cuda.synchronize(); t.append(time.perf_counter())
    st._unbind()
    names = ["upload+symmetry", "init_state", "plan", "engine", "first batch (capture)", f"remaining {done - 50} steps"]
    print(f"rep {rep}: " + ", ".join(f"{n} {1e3 * (b - a):.1f} ms" for n, a, b in zip(names, t[:-1], t[1:])),
          f"| per step {1e6 * (t[-1] - t[-2]) / (done - 50):.1f} us")
