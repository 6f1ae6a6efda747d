"""numpy restatement of the reference's renewal hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the checker the GPU
engine is compared against, and the CPU baseline bench.py times.  It never
runs inside the product path.

Pinning.  The reference is Python and was importable when this file was
written, so every function here is checked against vectors produced by the
reference itself: tests/golden/make_golden.py imports
/root/reference/pkg/src/spreadsim and writes tests/golden/*.npz;
tests/test_oracle_golden.py asserts this module reproduces them bit for bit
(RNG streams, erfcx/hazard grids, pressure folds, 200-step trajectories in
fp32 and mixed precision, SIS/SIR, strategy variants).  The Weibull / Erlang
hazards and the Philox stream have no reference implementation: they are
"parity unpinned" against the reference and pinned instead against scipy
(weibull_min / gamma pdf/sf) and the Random123 known-answer vectors.

Each function cites the reference lines it restates
(R = /root/reference/pkg/src/spreadsim).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import erfc

# ----------------------------------------------------------------------
# counter-based uniforms — R/rng.py:31-67, 91-96
# ----------------------------------------------------------------------
_U = np.uint64
_MIX1, _MIX2 = _U(0xBF58476D1CE4E5B9), _U(0x94D049BB133111EB)
_STEP, _STREAM, _TRIAL = _U(0xA24BAED4963EE407), _U(0x9FB21C651E98DF25), _U(0xD6E8FEB86659FD93)


def _aval(x):
    x = (x ^ (x >> _U(30))) * _MIX1
    x = (x ^ (x >> _U(27))) * _MIX2
    return x ^ (x >> _U(31))


def uniform_array(seed: int, step: int, streams) -> np.ndarray:
    """R/rng.py:54-67: two avalanche rounds, top 53 bits."""
    s = np.asarray(streams, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = _aval(_U(seed) ^ (_U(step) * _STEP))
        bits = _aval(key ^ (s * _STREAM))
    return (bits >> _U(11)).astype(np.float64) * (2.0 ** -53)


def derive_seed(seed: int, index: int) -> int:
    """R/rng.py:91-96."""
    with np.errstate(over="ignore"):
        x = _aval(_U(seed) ^ (_U(index) * _TRIAL))
        return int(_aval(x + _MIX1))


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 (Salmon et al. 2011) on uint32 arrays; no reference
    counterpart — pinned by the Random123 known-answer vectors."""
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & np.uint64(0xFFFFFFFF) for x in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0 & 0xFFFFFFFF), np.uint64(k1 & 0xFFFFFFFF)
    mask = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + np.uint64(0x9E3779B9)) & mask
        k1 = (k1 + np.uint64(0xBB67AE85)) & mask
    return c0, c1, c2, c3


def philox_uniform_array(seed: int, step: int, streams) -> np.ndarray:
    """key = seed, counter = (stream lo, stream hi, step lo, step hi);
    u = top 53 bits of (x1 << 32 | x0) — the engine's FS_RNG_PHILOX."""
    s = np.asarray(streams, dtype=np.uint64)
    mask = np.uint64(0xFFFFFFFF)
    x0, x1, _, _ = philox4x32_10(s & mask, s >> np.uint64(32), np.full_like(s, step & 0xFFFFFFFF),
                                 np.full_like(s, (step >> 32) & 0xFFFFFFFF), seed & 0xFFFFFFFF, seed >> 32)
    bits = (x1 << np.uint64(32)) | x0
    return (bits >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


# ----------------------------------------------------------------------
# hazards — R/hazards.py:84-132 (+ Weibull / Erlang, unpinned)
# ----------------------------------------------------------------------
_SQRT_PI = math.sqrt(math.pi)
_SQRT_2_OVER_PI = math.sqrt(2.0 / math.pi)


def _erfcx_nonneg(z: np.ndarray) -> np.ndarray:
    """R/hazards.py:84-95."""
    out = np.empty_like(z)
    small = z <= 3.5
    zs = z[small]
    out[small] = np.exp(zs * zs) * erfc(zs)
    zb = z[~small]
    r = 1.0 / (zb * zb)
    out[~small] = (1.0 + r * (-0.5 + r * (0.75 + r * (-1.875)))) / (zb * _SQRT_PI)
    return out


def erfcx_piecewise(z) -> np.ndarray:
    """R/hazards.py:98-105 (reflection below 0)."""
    z = np.atleast_1d(np.asarray(z, dtype=np.float64))
    out = np.empty_like(z)
    neg = z < 0.0
    out[~neg] = _erfcx_nonneg(z[~neg])
    if neg.any():
        zn = z[neg]
        with np.errstate(over="ignore"):
            out[neg] = 2.0 * np.exp(zn * zn) - _erfcx_nonneg(-zn)
    return out


def hazard_lognormal(tau: np.ndarray, mu: float, sigma: float) -> np.ndarray:
    """R/hazards.py:122-132."""
    tau = np.asarray(tau, dtype=np.float64)
    out = np.zeros_like(tau)
    pos = tau > 0.0
    if pos.any():
        t = tau[pos]
        z = (np.log(t) - mu) / (sigma * math.sqrt(2.0))
        with np.errstate(over="ignore", divide="ignore"):
            d = t * sigma * erfcx_piecewise(z)
            out[pos] = np.where(np.isinf(d), 0.0, _SQRT_2_OVER_PI / d)
    return out


def hazard_weibull(tau: np.ndarray, k: float, lam: float) -> np.ndarray:
    """(k/lam)(tau/lam)^(k-1); h(0) = 1/lam if k == 1 else 0 (engine
    convention, like the log-normal h(0) = 0)."""
    tau = np.asarray(tau, dtype=np.float64)
    out = np.full_like(tau, (1.0 / lam) if k == 1.0 else 0.0)
    pos = tau > 0.0
    out[pos] = (k / lam) * np.power(tau[pos] / lam, k - 1.0)
    return out


def hazard_erlang(tau: np.ndarray, k: int, r: float) -> np.ndarray:
    """r (r t)^(k-1)/(k-1)! / sum_{n<k} (r t)^n/n! with the running term."""
    tau = np.asarray(tau, dtype=np.float64)
    out = np.full_like(tau, r if k == 1 else 0.0)
    pos = tau > 0.0
    x = r * tau[pos]
    term = np.ones_like(x)
    total = np.ones_like(x)
    for n in range(1, int(k)):
        term = (term * x) / float(n)
        total = total + term
    out[pos] = (r * term) / total
    return out


def lognormal_pdf(tau: np.ndarray, mu: float, sigma: float) -> np.ndarray:
    """R/hazards.py:149-158."""
    tau = np.atleast_1d(np.asarray(tau, dtype=np.float64))
    out = np.zeros_like(tau)
    pos = tau > 0.0
    if pos.any():
        t = tau[pos]
        zs = (np.log(t) - mu) / sigma
        out[pos] = np.exp(-0.5 * zs * zs) / (t * sigma * math.sqrt(2.0 * math.pi))
    return out


def shedding_values(tr, tau: np.ndarray) -> np.ndarray:
    """R/hazards.py:196-218 for a Shedding-like object (kind, params)."""
    tau = np.asarray(tau, dtype=np.float64)
    if tr.kind == "constant":
        return np.ones_like(tau)
    p = tr.params
    if tr.kind == "lognormal_hazard":
        return hazard_lognormal(tau, p.mu, p.sigma)
    mode = math.exp(p.mu - p.sigma ** 2)
    return lognormal_pdf(tau, p.mu, p.sigma) / lognormal_pdf(np.array([mode]), p.mu, p.sigma)[0]


def nodal_hazard(holding, age64: np.ndarray) -> np.ndarray:
    kind = holding.kind
    if kind == "lognormal":
        return hazard_lognormal(age64, holding.params.mu, holding.params.sigma)
    if kind == "weibull":
        return hazard_weibull(age64, holding.params.k, holding.params.lam)
    if kind == "erlang":
        return hazard_erlang(age64, int(holding.params.k), holding.params.rate)
    return np.full_like(age64, holding.rate)


# ----------------------------------------------------------------------
# pressure fold — R/renewal.py:264-313 (CSR-order f32 accumulation)
# ----------------------------------------------------------------------


try:  # the reference's optional compiled fold (R/renewal.py:57-68), same per-node order
    import numba

    @numba.njit("void(float32[::1], float32[::1], int64[::1], int64[::1], int64[::1])", cache=False)
    def _fold_seq(out, contrib, nodes, starts, degs):  # pragma: no cover
        for k in range(nodes.size):
            acc = np.float32(0.0)
            base = starts[k]
            for e in range(degs[k]):
                acc += contrib[base + e]
            out[nodes[k]] += acc

    _HAVE_NUMBA = True
except Exception:  # pragma: no cover
    _HAVE_NUMBA = False

_FOLD_SETS: dict = {}


def _fold_set(row_offsets: np.ndarray):
    """Degree-sorted node order, slice starts and degrees, built once per
    row_offsets array as the reference's plan does (R/renewal.py:177-195)."""
    key = (id(row_offsets), row_offsets.size, int(row_offsets[-1]) if row_offsets.size else 0)
    fs = _FOLD_SETS.get(key)
    if fs is None or fs[0] is not row_offsets:
        deg = np.diff(row_offsets)
        order = np.argsort(-deg, kind="stable")
        fs = (row_offsets, order, np.ascontiguousarray(row_offsets[:-1][order]), np.ascontiguousarray(deg[order]))
        if len(_FOLD_SETS) > 8:
            _FOLD_SETS.clear()
        _FOLD_SETS[key] = fs
    return fs[1:]


def fold_pressure(row_offsets: np.ndarray, col: np.ndarray, w32: np.ndarray, inf32: np.ndarray) -> np.ndarray:
    """p_i = f32 sequential sum over the slice of f32(inf[col]*w), in CSR
    order per node (R/renewal.py:60-68, 198-218): the reference's compiled
    fold when numba is importable, else its numpy position-major fold —
    bit-identical (T/test_renewal.py:74-87)."""
    n = row_offsets.size - 1
    out = np.zeros(n, dtype=np.float32)
    if col.size == 0:
        return out
    contrib = inf32.astype(np.float32, copy=False)[col]
    w = w32.astype(np.float32, copy=False)
    if not (w.size and w[0] == 1.0 and (w == 1.0).all()):
        contrib = contrib * w
    order, start, sdeg = _fold_set(row_offsets)
    if _HAVE_NUMBA:
        _fold_seq(out, np.ascontiguousarray(contrib, dtype=np.float32), order.astype(np.int64, copy=False),
                  start.astype(np.int64, copy=False), sdeg.astype(np.int64, copy=False))
        return out
    live = n
    for p in range(int(sdeg[0]) if n else 0):
        while live and sdeg[live - 1] <= p:
            live -= 1
        if not live:
            break
        nodes = order[:live]
        out[nodes] = out[nodes] + contrib[start[:live] + p]
    return out


# ----------------------------------------------------------------------
# engine state and step — R/renewal.py:370-410, 483-580
# ----------------------------------------------------------------------


@dataclass
class OracleState:
    states: np.ndarray
    ages: np.ndarray
    infectivity: np.ndarray
    pressure: np.ndarray
    rates: np.ndarray
    clock: float
    step_counter: int
    tau_prev: float
    counts: np.ndarray
    mixed_precision: bool
    log: list = field(default_factory=list)  # (clock, tau, counts) per step


def _bf16():
    import ml_dtypes

    return np.dtype(ml_dtypes.bfloat16)


def init_state(g, m, cfg, seed: int, seed_count: int | None = None, seed_compartment: int | None = None) -> OracleState:
    """R/renewal.py:370-410 with _pick_seed_nodes (162-169)."""
    n = int(g.num_nodes)
    if seed_count is None:
        seed_count = max(10, int(round(0.01 * n)))
    comp = m.edge_to if seed_compartment is None else seed_compartment
    mixed = bool(cfg.mixed_precision)
    states = np.full(n, m.edge_from, dtype=np.int8 if mixed else np.int32)
    if seed_count:
        u = uniform_array(derive_seed(seed, 0x5EEDC0DE), 0, np.arange(n, dtype=np.uint64))
        states[np.sort(np.argpartition(u, seed_count - 1)[:seed_count])] = comp
    ages = np.zeros(n, dtype=np.float16 if mixed else np.float32)
    inf32 = np.zeros(n, dtype=np.float32)
    imask = states == m.infectious
    if imask.any():
        inf32[imask] = np.float32(m.beta) * shedding_values(m.transmission, ages[imask].astype(np.float64)).astype(np.float32)
    counts = np.bincount(states.astype(np.int64), minlength=m.num_compartments).astype(np.int64)
    return OracleState(states, ages, inf32.astype(_bf16() if mixed else np.float32), np.zeros(n, np.float32),
                       np.zeros(n, np.float32), 0.0, 0, float(cfg.tau_max), counts, mixed)


def step(st: OracleState, g, m, cfg, seed: int, rng: str = "splitmix") -> float:
    """One synchronous Bernoulli tau-leap over all nodes (R/renewal.py:483-580)."""
    tau = st.tau_prev
    st.clock += tau
    w32 = np.asarray(g.weights, dtype=np.float32)
    if st.mixed_precision:
        w32 = w32.astype(_bf16()).astype(np.float32)
    inf32 = st.infectivity.astype(np.float32)
    pressure = fold_pressure(np.asarray(g.row_offsets, np.int64), np.asarray(g.col_indices), w32, inf32)
    st.pressure = pressure
    s = st.states
    age32 = st.ages.astype(np.float32)
    rates = np.zeros(s.size, dtype=np.float32)
    S = s == m.edge_from
    rates[S] = pressure[S]
    for c, (_, h) in sorted(m.nodal.items()):
        sel = s == c
        if sel.any():
            rates[sel] = nodal_hazard(h, age32[sel].astype(np.float64)).astype(np.float32)
    q = -np.expm1(-(rates.astype(np.float64)) * tau)
    ids = np.arange(s.size, dtype=np.uint64)
    u = uniform_array(seed, st.step_counter, ids) if rng == "splitmix" else philox_uniform_array(seed, st.step_counter, ids)
    fired = np.flatnonzero(u < q)
    succ = m.successor_array().astype(np.int64)
    term = m.terminal_mask()
    old = s[fired].astype(np.int64)
    new = succ[old]
    new_age = np.where(~term[s.astype(np.int64)], age32 + np.float32(tau), age32).astype(np.float32)
    new_age[fired] = 0.0
    s[fired] = new.astype(s.dtype)
    if fired.size:
        st.counts += np.bincount(new, minlength=m.num_compartments)
        st.counts -= np.bincount(old, minlength=m.num_compartments)
    assert int(st.counts.sum()) == s.size
    inf_new = np.zeros(s.size, dtype=np.float32)
    imask = s == m.infectious
    if imask.any():
        if m.transmission.kind == "constant":
            inf_new[imask] = np.float32(m.beta)
        else:
            inf_new[imask] = (m.beta * shedding_values(m.transmission, new_age[imask].astype(np.float64))).astype(np.float32)
    st.ages = new_age.astype(st.ages.dtype)
    st.infectivity = inf_new.astype(st.infectivity.dtype)
    st.rates = rates
    mx = float(rates.max()) if rates.size else 0.0
    st.tau_prev = min(cfg.tau_max, cfg.epsilon / (mx + cfg.delta))
    st.step_counter += 1
    st.log.append((st.clock, tau, st.counts.copy()))
    return tau


def step_rows(states, ages, ro_local, col_global, inf32_global, lo: int, tau: float, step_counter: int, m, seed: int,
              mixed: bool, rng: str = "splitmix"):
    """`step`'s per-node arithmetic on the rows [lo, lo+n) of a node
    partition: the incoming slices hold global column ids and
    read the global infectivity; the uniforms are keyed by global id.
    Returns (states', ages', infectivity' of the rows, local max rate, local
    count deltas) — the pieces a partitioned run exchanges.  Test oracle for
    paper_2604_22092_b200.distributed; same operations as `step`."""
    n = states.size
    w32 = np.ones(col_global.size, dtype=np.float32)
    pressure = fold_pressure(np.asarray(ro_local, np.int64), np.asarray(col_global), w32, inf32_global)
    s = states.copy()
    age32 = ages.astype(np.float32)
    rates = np.zeros(n, dtype=np.float32)
    S = s == m.edge_from
    rates[S] = pressure[S]
    for c, (_, h) in sorted(m.nodal.items()):
        sel = s == c
        if sel.any():
            rates[sel] = nodal_hazard(h, age32[sel].astype(np.float64)).astype(np.float32)
    q = -np.expm1(-(rates.astype(np.float64)) * tau)
    ids = np.arange(lo, lo + n, dtype=np.uint64)
    u = uniform_array(seed, step_counter, ids) if rng == "splitmix" else philox_uniform_array(seed, step_counter, ids)
    fired = np.flatnonzero(u < q)
    succ = m.successor_array().astype(np.int64)
    term = m.terminal_mask()
    old = s[fired].astype(np.int64)
    new = succ[old]
    new_age = np.where(~term[s.astype(np.int64)], age32 + np.float32(tau), age32).astype(np.float32)
    new_age[fired] = 0.0
    s[fired] = new.astype(s.dtype)
    delta = np.bincount(new, minlength=m.num_compartments) - np.bincount(old, minlength=m.num_compartments)
    inf_new = np.where(s == m.infectious, np.float32(m.beta), np.float32(0.0)).astype(np.float32)
    mx = float(rates.max()) if rates.size else 0.0
    return s, new_age.astype(np.float16 if mixed else np.float32), inf_new, mx, delta.astype(np.int64)


def run_batch(st: OracleState, g, m, cfg, seed: int, rng: str = "splitmix") -> float:
    """R/renewal.py:600-629 (compaction is result-neutral and omitted)."""
    if not cfg.carry_tau:
        st.tau_prev = cfg.tau_max
    total = 0.0
    for _ in range(cfg.steps_per_batch):
        total += step(st, g, m, cfg, seed, rng)
    return total


def run(g, m, cfg, seed: int, t_final: float, seed_count=None, seed_compartment=None, rng: str = "splitmix"):
    """R/renewal.py:632-663 without the grid: returns (times, counts, state)."""
    st = init_state(g, m, cfg, seed, seed_count, seed_compartment)
    times, rows = [0.0], [st.counts.copy()]
    while st.clock < t_final:
        run_batch(st, g, m, cfg, seed, rng)
    for clock, _, c in st.log:
        times.append(clock)
        rows.append(c)
    return np.asarray(times), np.asarray(rows), st
