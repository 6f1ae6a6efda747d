"""Host-side phase times of one lockstep run_ensemble call (ens workload):
init (states + engines + ensemble), the batch loop, close, records."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import ensemble as E
from paper_2604_22092_b200.renewal import _build_plan

g = fs.gen_erdos_renyi(1000, 8.0, seed=20250809)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
for rep in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    plan = _build_plan(g, m, cfg, False); torch.cuda.synchronize(); t.append(time.perf_counter())
    ls = E._Lockstep(list(range(100)), g, m, cfg, 20250809, 10, None, plan); torch.cuda.synchronize(); t.append(time.perf_counter())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ls.run_batch(); fin = False; nb = 1
    while not fin:
        ls.run_batch(); nb += 1
        fin = ls.collect(cfg.steps_per_batch, g.num_nodes, 50.0)
    ev1.record(); torch.cuda.synchronize(); t.append(time.perf_counter())
    ls.close(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"plan {d[0]:.2f} init {d[1]:.2f} loop {d[2]:.2f} (gpu span {ev0.elapsed_time(ev1):.2f}, {nb} batches) close {d[3]:.2f} ms")
