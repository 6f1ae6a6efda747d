"""Virtual ranks on one GPU (LocalPartitionedRun, N = 1e7, 4 ranks): per-step
time and remote pushes with the bulk (mailbox) exchange vs direct peer
atomics — on one device both transports are local memory, so this measures
the bulk path's own overhead (staging, flush, apply), not NVLink."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200.distributed import LocalPartitionedRun, partition_plan

n, k, world = 10_000_000, 10, 4
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
plan = partition_plan(n, world)
parts = [fs.gen_fixed_degree_device(n, k, seed=5, row_lo=lo, row_hi=hi) for lo, hi in plan.ranges]
for ex in ("bulk", "atomic", "bulk", "atomic"):
    run = LocalPartitionedRun(parts, m, cfg, 7, plan, exchange=ex)
    out = []
    for b in range(8):  # 400 steps: into the growth phase
        torch.cuda.synchronize(); t0 = time.perf_counter()
        run.run_batch()
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        rp = sum(int(p.remote_pushes(run.steps - 50, 50).sum()) for p in run.parts)
        out.append((round(dt * 1e6 / 50, 1), rp // 50))
    print(ex, "us/step, remote pushes/step per batch:", out)
    run.close()
