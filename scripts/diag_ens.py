"""Phase timings of the lockstep ensemble (ens workload): where the wall goes."""
import time, ctypes, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import ensemble as E, renewal as Rn, _lib

g = fs.gen_erdos_renyi(1000, 8.0, seed=20250809)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
for rep in range(3):
    torch.cuda.synchronize(); T = {}
    t = time.perf_counter()
    plan = Rn._build_plan(g, m, cfg, False); torch.cuda.synchronize(); T["plan"] = time.perf_counter() - t; t = time.perf_counter()
    seeds = [fs.derive_seed(20250809, k) for k in range(100)]
    states = Rn.init_renewal_states(g, m, cfg, seeds, 10); torch.cuda.synchronize(); T["states"] = time.perf_counter() - t; t = time.perf_counter()
    engs = [st._bind(plan, s, materialize=False) for st, s in zip(states, seeds)]; torch.cuda.synchronize(); T["bind"] = time.perf_counter() - t; t = time.perf_counter()
    lib = _lib.load()
    arr = (ctypes.c_void_p * 100)(*[e.handle.value for e in engs]); h = ctypes.c_void_p()
    _lib.check(lib.fs_ensemble_create(arr, 100, ctypes.byref(h))); T["create"] = time.perf_counter() - t; t = time.perf_counter()
    st = E._device.stream_handle(E._device.device())
    b = cfg.steps_per_batch; done = 0; nb = 0
    _lib.check(lib.fs_ensemble_run_batch(h, st))
    clocks = np.empty((100, b)); counts = np.empty((100, b, 4), dtype=np.int64)
    tw = 0.0
    while True:
        _lib.check(lib.fs_ensemble_run_batch(h, st))
        tq = time.perf_counter()
        _lib.check(lib.fs_ensemble_wait_log(h, done, b, clocks.ctypes.data, None, counts.ctypes.data))
        tw += time.perf_counter() - tq
        done += b; nb += 1
        if clocks[:, -1].min() >= 50.0: break
    T["loop"] = time.perf_counter() - t; T["loop_wait"] = tw; T["batches"] = nb; t = time.perf_counter()
    torch.cuda.synchronize(); lib.fs_ensemble_destroy(h)
    for e in engs: e.close()
    T["close"] = time.perf_counter() - t
    print({k: round(v * 1e3, 2) if isinstance(v, float) else v for k, v in T.items()})
# graph replay cost of one batch alone
