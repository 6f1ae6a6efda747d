"""Per-CTA timeline of k_step_incr for flushed single steps (the bench's
headline timing): entry spread, time to step constants, work end, finish,
next to the event-timed step.  Needs a library built with
`make NVFLAGS_EXTRA=-DFS_STEP_PROBE=1` and FS_DEBUG_TIMES=1 at run time.
%globaltimer is not aligned between the two dies, so cross-CTA stamps are
compared within a CTA (work duration = work end - constants ready)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_22092_b200 as fs
from paper_2604_22092_b200 import renewal as R, _lib
lib = _lib.load()
lib.fs_engine_debug_times.restype = ctypes.c_int
lib.fs_engine_debug_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
n = int(float(os.environ.get("N", "1e6")))
g = fs.gen_fixed_degree_device(n, 10, seed=1) if n > 2_000_000 else fs.gen_fixed_degree(n, 10, seed=1)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig(mixed_precision=n > 2_000_000)
st = fs.init_renewal_state(g, m, cfg, 7)
plan = R._build_plan(g, m, cfg, cfg.mixed_precision)
eng = st._bind(plan, 7, False)
eng.step(10, False, False)
buf = np.zeros(16 * 2048 * 36, dtype=np.uint64)
lib.fs_engine_debug_times(eng.handle, buf.ctypes.data, 2048)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
ev = []
for k in range(16):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.zero_(); flush_rd.max()
    a.record(); eng.step(1, False, False); b.record()
    ev.append((a, b))
torch.cuda.synchronize()
grid = lib.fs_engine_debug_times(eng.handle, buf.ctypes.data, 2048)
b = buf[: 16 * grid * 4].reshape(16, grid, 4).astype(np.int64)
wb = buf[16 * grid * 4: 16 * grid * 36].reshape(16, grid, 16, 2).astype(np.int64)
smid = (b[:, :, 0] >> 48)
b[:, :, 0] &= (1 << 48) - 1
ms = [x.elapsed_time(y) * 1e3 for x, y in ev]
print(f"N={n} grid={grid} event us/step median {np.median(ms):.1f}")
rows = []
for s in range(16):
    e, w, c, f = b[s, :, 0], b[s, :, 1], b[s, :, 2], b[s, :, 3]
    if e.min() == 0:
        continue
    t0 = e.min()
    rows.append([(np.median(e) - t0), (e.max() - t0), np.median(c - e), np.max(c - e), np.median(w - t0), (w.max() - t0),
                 np.median(f - w), (f.max() - t0)])
r = np.median(np.array(rows), axis=0) / 1e3
print("entry med %.2f max %.2f | consts-ready med %.2f max %.2f | work end med %.2f max %.2f | finish-work med %.2f | kernel %.2f us" % tuple(r))
# distribution of work end over CTAs (relative to the median entry), slowest CTAs
W = []
for s in range(16):
    e, w = b[s, :, 0], b[s, :, 1]
    if e.min() == 0:
        continue
    W.append((w - np.median(e)) / 1e3)
W = np.array(W)
print("work end percentiles (us) p0 %.2f p10 %.2f p50 %.2f p90 %.2f p99 %.2f p100 %.2f" %
      tuple(np.percentile(W, [0, 10, 50, 90, 99, 100])))
avg = W.mean(axis=0)
order = np.argsort(avg)
print("slowest CTAs (mean over steps):", [(int(i), round(float(avg[i]), 2)) for i in order[-12:]])
print("fastest CTAs:", [(int(i), round(float(avg[i]), 2)) for i in order[:6]])
print("per-CTA consistency: corr of work end between even/odd steps %.2f" % np.corrcoef(W[::2].mean(0), W[1::2].mean(0))[0, 1])

# offset-free: per-CTA work duration (work end - constants ready, same SM clock)
D = []
for s_ in range(16):
    if b[s_, :, 0].min() == 0:
        continue
    D.append((b[s_, :, 1] - b[s_, :, 2]) / 1e3)
D = np.array(D)
print("work duration percentiles (us) p0 %.2f p10 %.2f p50 %.2f p90 %.2f p100 %.2f" % tuple(np.percentile(D, [0, 10, 50, 90, 100])))
sm0 = smid[0]
dm = D.mean(0)
per_sm = {}
for i in range(len(dm)):
    per_sm.setdefault(int(sm0[i]), []).append(dm[i])
sms = sorted(per_sm)
print("SM ids %d..%d; mean duration by SM id decile:" % (sms[0], sms[-1]),
      [round(float(np.mean([np.mean(per_sm[x]) for x in sms[i:i + 15]])), 2) for i in range(0, len(sms), 15)])
print("slowest by duration:", [(int(i), int(sm0[i]), round(float(dm[i]), 2)) for i in np.argsort(dm)[-10:]])

# per warp: phase end relative to the CTA's constants-ready stamp, deferred nodes, drains
WE, WD, WN = [], [], []
for s_ in range(16):
    if b[s_, :, 0].min() == 0:
        continue
    WE.append((wb[s_, :, :, 0] - b[s_, :, 2][:, None]) / 1e3)
    WD.append(wb[s_, :, :, 1] >> 20)
    WN.append(wb[s_, :, :, 1] & 0xFFFFF)
WE, WD, WN = np.array(WE), np.array(WD), np.array(WN)
print("warp phase end (us after constants) p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(WE, [10, 50, 90, 100])))
print("deferred per warp p10 %d p50 %d p90 %d max %d; drains p50 %d max %d" % (*np.percentile(WD, [10, 50, 90, 100]), np.median(WN), WN.max()))
for d in range(int(WN.max()) + 1):
    sel = WN == d
    if sel.any():
        print(f"  drains={d}: warps {sel.mean()*100:.1f}%  phase end mean {WE[sel].mean():.2f} us")
cta_end = WE.max(axis=2)
slow = cta_end > np.percentile(cta_end, 90)
print("slowest-10%% CTAs: mean deferred/warp %.1f vs others %.1f; max drains/warp %.2f vs %.2f" % (
    WD.mean(axis=2)[slow].mean(), WD.mean(axis=2)[~slow].mean(), WN.max(axis=2)[slow].mean(), WN.max(axis=2)[~slow].mean()))
c = np.corrcoef(WE.reshape(-1), WD.reshape(-1))[0, 1]
print("corr(warp phase end, deferred) %.2f" % c)
