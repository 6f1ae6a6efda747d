"""Where run_renewal's setup goes on a fresh host CsrGraph (C2): each piece of
_DeviceGraph / init / engine creation timed separately (device synced)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import renewal as R, _lib, _device

g0 = fs.gen_fixed_degree(1_000_000, 10, seed=1)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
lib = _lib.load(); dev = _device.device(); st = _device.stream_handle(dev)
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(4):
    g = fs.CsrGraph(g0.num_nodes, g0.num_edges, g0.row_offsets.copy(), g0.col_indices.copy(), g0.weights.copy())
    t = {}; t0 = T()
    ro = np.ascontiguousarray(g.row_offsets, dtype=np.int64); col = np.ascontiguousarray(g.col_indices, dtype=np.int32)
    dro = torch.empty(ro.size, dtype=torch.int64, device=dev); t1 = T(); t["alloc"] = t1 - t0
    lib.fs_h2d_staged(_lib.ptr(dro), ro.ctypes.data, ro.nbytes, st); t2 = T(); t["h2d_ro"] = t2 - t1
    dcol = torch.empty(col.size + 4, dtype=torch.int32, device=dev)
    lib.fs_h2d_staged(_lib.ptr(dcol), col.ctypes.data, col.nbytes, st); t3 = T(); t["h2d_col"] = t3 - t2
    w32 = np.ascontiguousarray(g.weights, dtype=np.float32)
    dmax, flag, w0 = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_float()
    lib.fs_host_csr_scan(ro.ctypes.data, g.num_nodes, w32.ctypes.data, w32.size, ctypes.byref(dmax), ctypes.byref(flag), ctypes.byref(w0)); t4 = T(); t["host_scan"] = t4 - t3
    g2 = fs.CsrGraph(g0.num_nodes, g0.num_edges, g0.row_offsets.copy(), g0.col_indices.copy(), g0.weights.copy())
    t5 = T(); dg = R.device_graph(g2, False); t6 = T(); t["device_graph_total"] = t6 - t5
    s = fs.init_renewal_state(g2, m, cfg, 7); t7 = T(); t["init_state"] = t7 - t6
    plan = R._build_plan(g2, m, cfg, False); t8 = T(); t["build_plan_rest"] = t8 - t7
    e = s._bind(plan, 7, materialize=False); t9 = T(); t["bind"] = t9 - t8
    print(rep, {k: round(v * 1e3, 2) for k, v in t.items()})
