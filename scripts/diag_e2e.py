"""Break down run_renewal's end-to-end wall on a fresh host CsrGraph (the
bench e2e leg): pinning, H2D, host scans, symmetry check, engine creation,
batches."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_22092_b200 as fs  # noqa: E402
from paper_2604_22092_b200 import renewal as R  # noqa: E402
from paper_2604_22092_b200 import _lib  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
g0, m = bench.build_inputs(w)
cfg = fs.RenewalConfig()


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(3):
    g = fs.CsrGraph(g0.num_nodes, g0.num_edges, g0.row_offsets.copy(), g0.col_indices.copy(), g0.weights.copy())
    marks = {}
    t0 = t()
    ro = np.ascontiguousarray(g.row_offsets, dtype=np.int64)
    col = np.ascontiguousarray(g.col_indices, dtype=np.int32)
    marks["contig"] = t()
    lib = _lib.load()
    lib.fs_host_register(ro.ctypes.data, ro.nbytes)
    lib.fs_host_register(col.ctypes.data, col.nbytes)
    marks["register"] = t()
    lib.fs_host_unregister(ro.ctypes.data)
    lib.fs_host_unregister(col.ctypes.data)
    w32 = np.ascontiguousarray(g.weights, dtype=np.float32)
    _ = bool((w32 == w32[0]).all())
    marks["uniform_scan"] = t()
    _ = int(np.diff(ro).max())
    marks["dmax_scan"] = t()
    g = fs.CsrGraph(g0.num_nodes, g0.num_edges, g0.row_offsets.copy(), g0.col_indices.copy(), g0.weights.copy())
    t1 = t()
    st = fs.init_renewal_state(g, m, cfg, 7)
    marks["init_state"] = t()
    plan = R._build_plan(g, m, cfg, False)
    marks["build_plan(device_graph)"] = t()
    eng = st._bind(plan, 7, materialize=False)
    marks["bind(engine create)"] = t()
    done = 0
    clock = 0.0
    nb = 0
    while clock < 50.0:
        eng.run_batch(materialize=False)
        clocks, _, counts = eng.read_log(done, cfg.steps_per_batch)
        done += cfg.steps_per_batch
        clock = float(clocks[-1])
        nb += 1
    marks[f"{nb} batches"] = t()
    st._unbind()
    marks["unbind"] = t()
    prev = t0
    out = []
    for k, v in marks.items():
        if k == "init_state":
            prev = t1
        out.append(f"{k} {1e3 * (v - prev):.2f}")
        prev = v
    print(f"rep {rep}: " + ", ".join(out) + " ms")
