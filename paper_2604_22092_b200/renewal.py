"""Drop-in for ``spreadsim.renewal`` backed by the sm_100a engine.

Same public names, signatures and semantics as the reference module
(/root/reference/pkg/src/spreadsim/renewal.py:39-51): ``RenewalConfig``,
``RenewalState``, ``ActiveSet``, ``init_renewal_state``, ``renewal_step``,
``run_batch``, ``run_renewal``, ``pressure_gather``, ``refresh_active``,
``set_mixed_precision``, ``default_seed_count`` and the private-but-called
``_build_plan`` / ``_begin_batch`` used by ``analysis._SteppedRun``
(analysis.py:401-418).

Where the data lives.  Per-node arrays (states, ages, infectivity, pressure,
rates) and the run scalars (clock, step counter, tau', counts) are
device-resident; the attributes of ``RenewalState`` download them on access
and any in-place edit of a downloaded array is pushed back before the next
step (the reference's tests edit ``state.states`` / ``ages`` / ``counts``
between steps, T/test_renewal.py:118-120, 245-246).  A step is one launch of
the fused kernel; ``run_batch`` is one CUDA-graph replay of
``steps_per_batch`` launches; the per-step (clock, counts) recorder comes
back as one small D2H copy per batch.  There is no CPU path: without the
shared library or a CUDA device every entry point raises
``FlashSpreadNativeError``.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, fields

import numpy as np
import torch

from . import _device, _lib
from .errors import InvalidConfigError, ReconfigureAfterStartError
from .graph import CsrGraph, DegreeStats, Strategy, as_strategy, resolve_strategy, select_strategy
from .models import ModelSpec, model_descriptor
from .rng import RNG_KINDS, derive_seed, uniform_array
from .trajectory import DEFAULT_GRID_POINTS, TrajectoryRecord, make_record

__all__ = [
    "RenewalConfig",
    "RenewalState",
    "ActiveSet",
    "init_renewal_state",
    "set_mixed_precision",
    "refresh_active",
    "pressure_gather",
    "renewal_step",
    "run_batch",
    "run_renewal",
    "default_seed_count",
    "as_config",
]

_SEED_PICK_SALT = 0x5EEDC0DE  # renewal.py:55
_STRATEGY_CODE = {Strategy.PER_NODE: _lib.PER_NODE, Strategy.LANE_CHUNKED: _lib.LANE,
                  Strategy.EDGE_MERGE: _lib.MERGE}
_PRECISION = {"f64": _lib.HAZ_F64, "f32": _lib.HAZ_F32}
_GATHER = {"auto": -1, "f32": 0, "count": 1, "incremental": 1}
_INCREMENTAL = {"auto": -1, "f32": 0, "count": 0, "incremental": 1}


@dataclass
class RenewalConfig:
    """renewal.py:75-99, plus three B200 options appended after the
    reference's fields (positional construction is unchanged):

    rng               "splitmix" (reference mixer, bit-exact parity) | "philox"
    hazard_precision  "f64" (the reference's float64 hazard) | "f32"
    gather            "auto" (exact count encodings when transmission is
                      constant and weights uniform: incremental counts when an
                      outgoing CSR is known, else the 1-bit mask gather) |
                      "f32" (the literal CSR-order fold) | "count" (mask gather
                      every step) | "incremental" (require incremental counts)
    """

    epsilon: float = 0.03
    tau_max: float = 0.1
    delta: float = 1e-9
    steps_per_batch: int = 50
    strategy: Strategy = Strategy.AUTO
    compaction: bool = False
    mixed_precision: bool = False
    lanes_per_node: int = 32
    edges_per_block: int = 1024
    hazard_chunk: int = 128
    chunk_skip: bool = True
    carry_tau: bool = True
    rng: str = "splitmix"
    hazard_precision: str = "f64"
    gather: str = "auto"

    def __post_init__(self) -> None:
        if not (0.0 < self.epsilon < 1.0):
            raise ValueError("epsilon must be in (0, 1)")
        if self.tau_max <= 0.0:
            raise ValueError("tau_max must be > 0")
        if self.steps_per_batch < 1:
            raise ValueError("steps_per_batch must be >= 1")
        if self.rng not in RNG_KINDS:
            raise ValueError(f"rng must be one of {sorted(RNG_KINDS)}")
        if self.hazard_precision not in _PRECISION:
            raise ValueError("hazard_precision must be 'f64' or 'f32'")
        if self.gather not in _GATHER:
            raise ValueError("gather must be 'auto', 'f32', 'count' or 'incremental'")


def as_config(cfg) -> RenewalConfig:
    """This package's RenewalConfig for `cfg`.

    Accepts None (defaults), a RenewalConfig, or the reference's own
    `spreadsim.renewal.RenewalConfig` (R/renewal.py:75-99) or any object with
    its fields: the reference fields are copied by name, its `Strategy`
    member is mapped by value, and the three B200 fields the reference does
    not have (`rng`, `hazard_precision`, `gather`) take their defaults —
    the reference's own arithmetic (splitmix, f64 hazards) with the exact
    gather encodings chosen automatically."""
    if cfg is None:
        return RenewalConfig()
    if isinstance(cfg, RenewalConfig):
        return cfg
    kw = {f.name: getattr(cfg, f.name) for f in fields(RenewalConfig) if hasattr(cfg, f.name)}
    if "strategy" in kw:
        kw["strategy"] = as_strategy(kw["strategy"])
    return RenewalConfig(**kw)


@dataclass
class ActiveSet:
    """Zero-padded sorted ids of non-absorbed nodes (renewal.py:102-111)."""

    active_nodes: np.ndarray
    num_active: int

    @property
    def ids(self) -> np.ndarray:
        return self.active_nodes[: self.num_active]


def default_seed_count(num_nodes: int) -> int:
    """max(10, 1% of N) (renewal.py:157-159)."""
    return max(10, int(round(0.01 * num_nodes)))


_BYTES = {torch.int8: 1, torch.uint8: 1, torch.int16: 2, torch.float16: 2, torch.bfloat16: 2, torch.int32: 4,
          torch.float32: 4, torch.int64: 8, torch.float64: 8}


_FILL_PATTERN: dict = {}


def _fill(t: torch.Tensor, value) -> torch.Tensor:
    """Fill a device buffer through the library (fs_fill) — torch only owns it."""
    if t.numel():
        key = (t.dtype, repr(value))  # repr: -0.0 and 0.0 are different patterns
        pat = _FILL_PATTERN.get(key)
        if pat is None:  # the element's bytes, once per (dtype, value)
            raw = torch.tensor([value], dtype=t.dtype).view(torch.uint8).numpy().tobytes()
            pat = _FILL_PATTERN[key] = int.from_bytes(raw, "little")
        _lib.check(_lib.load().fs_fill(_lib.ptr(t), t.numel(), _BYTES[t.dtype], pat, _device.stream_handle(t.device)))
    return t


def _node_buffer(n: int, dtype: torch.dtype, dev: torch.device, fill=0) -> torch.Tensor:
    """Per-node device array, allocated to a whole number of 128-node units
    (the streaming kernels read whole tiles / vectors, fs_state_buffers.padded)
    and returned as the [:n] view."""
    cap = (n + 127) // 128 * 128
    return _fill(torch.empty((cap,), dtype=dtype, device=dev), fill)[:n]


def _storage(mixed: bool):
    """(states, ages, infectivity) torch dtypes (renewal.py:358-367)."""
    if mixed:
        return torch.int8, torch.float16, torch.bfloat16
    return torch.int32, torch.float32, torch.float32


# ----------------------------------------------------------------------
# device graph + plan
# ----------------------------------------------------------------------


class _DeviceGraph:
    """CSR on the device, uploaded once per (graph, precision) and cached on
    the graph object.  Uniform weights (every generator's 1.0,
    graph.py:230) are passed as a scalar instead of an E-long stream."""

    def __init__(self, g, mixed: bool, dev: torch.device):
        self.num_nodes = int(g.num_nodes)
        self.num_edges = int(g.num_edges)
        ro = np.ascontiguousarray(g.row_offsets, dtype=np.int64)
        col_h = np.ascontiguousarray(g.col_indices, dtype=np.int32)
        lib = _lib.load()
        stream = _device.stream_handle(dev)
        # uploads through the library's page-locked staging slots (host
        # threads copy one slot while the previous one is in flight)
        self.row_offsets = torch.empty(ro.size, dtype=torch.int64, device=dev)
        _lib.check(lib.fs_h2d_staged(_lib.ptr(self.row_offsets), ro.ctypes.data, ro.nbytes, stream))
        # int32 copy for the hot kernels when every offset fits (halves the
        # offset stream; listed in DESIGN.md as an encoding).  Both the int32
        # offsets and the columns carry slack past the end for 16-byte TMA
        # bulk copies (fs_graph.padded).
        self.row_offsets32 = _narrow_offsets(self.row_offsets, self.num_nodes, self.num_edges, dev)
        col = torch.empty(self.num_edges + 4, dtype=torch.int32, device=dev)
        _lib.check(lib.fs_h2d_staged(_lib.ptr(col), col_h.ctypes.data, col_h.nbytes, stream))
        _fill(col[self.num_edges:], 0)
        self.col_indices = col[: self.num_edges]
        # host passes over the arrays (max degree, uniform weights) run once
        # per graph object, in parallel host threads, and are cached on it,
        # like the symmetry check below
        uni = g.__dict__.get("_fs_uniform")
        dm = g.__dict__.get("_fs_dmax")
        if uni is None or dm is None:
            w32 = np.ascontiguousarray(g.weights, dtype=np.float32)
            dmax, flag, w0 = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_float()
            _lib.check(lib.fs_host_csr_scan(ro.ctypes.data, self.num_nodes, w32.ctypes.data, w32.size,
                                            ctypes.byref(dmax), ctypes.byref(flag), ctypes.byref(w0)))
            uni = g.__dict__["_fs_uniform"] = (bool(flag.value), float(w0.value) if w32.size else 1.0)
            dm = g.__dict__["_fs_dmax"] = int(dmax.value)
        self.uniform = uni[0]
        if mixed:  # weights rounded to bf16 at plan time (renewal.py:330-331)
            import ml_dtypes

            self.uniform_weight = float(np.float32(np.array([uni[1]], np.float32).astype(ml_dtypes.bfloat16)[0]))
        else:
            self.uniform_weight = uni[1]
        self.weights = None
        if not self.uniform:
            w = np.ascontiguousarray(g.weights, dtype=np.float32)
            if mixed:
                import ml_dtypes

                w = w.astype(ml_dtypes.bfloat16)
            self.weights = _device.to_device(w, dev)
        self.weights_bf16 = mixed
        self.d_max = dm
        # cached on the host graph like the reference caches its transpose
        # (R/graph.py:187-191 build_outgoing): a property of the arrays
        sym = g.__dict__.get("_fs_symmetric")
        if sym is None:
            sym = g.__dict__["_fs_symmetric"] = _is_symmetric(self)
        self.symmetric = sym

    def view(self) -> _lib.FsGraph:
        v = self.__dict__.get("_view")
        if v is None:  # the device arrays never change: build the descriptor once
            v = self._view = self._make_view()
        return v

    def _make_view(self) -> _lib.FsGraph:
        return _lib.FsGraph(
            num_nodes=self.num_nodes,
            num_edges=self.num_edges,
            row_offsets=_lib.ptr(self.row_offsets),
            row_offsets32=_lib.ptr(self.row_offsets32),
            col_indices=_lib.ptr(self.col_indices),
            weights=_lib.ptr(self.weights),
            weights_dtype=_lib.BF16 if self.weights_bf16 else _lib.F32,
            weights_uniform=int(self.uniform),
            uniform_weight=self.uniform_weight,
            d_max=self.d_max,
            padded=1,
            # the outgoing CSR of a symmetric (undirected) graph is the incoming one
            out_row_offsets=_lib.ptr(self.row_offsets) if self.symmetric else None,
            out_col_indices=_lib.ptr(self.col_indices) if self.symmetric else None,
        )


    @classmethod
    def from_device(cls, g, dev: torch.device) -> "_DeviceGraph":
        """Wrap a DeviceCsrGraph (GPU-generated, uniform weights) without a
        host round trip."""
        self = cls.__new__(cls)
        self.num_nodes = int(g.num_rows)
        self.num_edges = int(g.num_edges)
        t = g.device_tensors()
        self.row_offsets = t["row_offsets"]
        self.row_offsets32 = _narrow_offsets(self.row_offsets, self.num_nodes, self.num_edges, dev)
        self.col_indices = t["col_buffer"][: self.num_edges]
        self.uniform = True
        self.uniform_weight = float(g.uniform_weight)
        self.weights = None
        self.weights_bf16 = False
        self.d_max = int(g.d_max)
        # fs_gen_regular graphs are undirected by construction: a row slice's
        # out-rows are its in-rows (global ids), which is all the pushes need
        self.symmetric = bool(getattr(g, "symmetric_global", False))
        return self


def _narrow_offsets(ro: torch.Tensor, n: int, e: int, dev: torch.device):
    """int32 offsets (+8 slack entries = E) when E < 2^31, else None."""
    if e >= 2**31:
        return None
    r32 = torch.empty(n + 1 + 8, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().fs_narrow_offsets(_lib.ptr(ro), n + 1, _lib.ptr(r32), _device.stream_handle(dev)))
    _fill(r32[n + 1:], e)
    return r32[: n + 1]


def _is_symmetric(dg) -> bool:
    """Is the incoming CSR its own transpose (an undirected graph, as every
    reference generator makes, R/graph.py:221-231)?  Decided on the device
    (fs_check_symmetric): every edge's multiplicity equals its reverse's."""
    if dg.num_edges == 0:
        return True
    out = ctypes.c_int32()
    _lib.check(_lib.load().fs_check_symmetric(_lib.ptr(dg.row_offsets), _lib.ptr(dg.row_offsets32),
                                              _lib.ptr(dg.col_indices), dg.num_nodes, dg.num_edges,
                                              ctypes.byref(out), _device.stream_handle(dg.row_offsets.device)))
    return bool(out.value)


def device_graph(g, mixed: bool = False) -> _DeviceGraph:
    dev = _device.device()
    if hasattr(g, "device_tensors"):  # DeviceCsrGraph: already on the device
        cache = g.__dict__.setdefault("_fs_device_cache", {})
        if dev.index not in cache:
            cache[dev.index] = _DeviceGraph.from_device(g, dev)
        return cache[dev.index]
    cache = g.__dict__.setdefault("_fs_device_cache", {})
    key = (bool(mixed), dev.index)
    if key not in cache:
        cache[key] = _DeviceGraph(g, mixed, dev)
    return cache[key]


@dataclass
class _EnginePlan:
    """Per-(graph, model, config) preparation (renewal.py:140-155, 321-355)."""

    strategy: Strategy
    graph: _DeviceGraph
    model: _lib.FsModel
    config: _lib.FsConfig
    succ: np.ndarray
    terminal: np.ndarray
    count_mode: bool
    mixed: bool
    num_compartments: int
    fold_active: None = None  # reference field; compaction lives in the engine

    @property
    def weights_f32(self) -> np.ndarray:  # reference field, host copy
        if self.graph.weights is None:
            return np.full(self.graph.num_edges, self.graph.uniform_weight, dtype=np.float32)
        return _device.to_host(self.graph.weights).astype(np.float32)


def _build_plan(g, m, cfg: RenewalConfig, mixed: bool) -> _EnginePlan:
    cfg = as_config(cfg)
    dg = device_graph(g, mixed)
    strategy = as_strategy(cfg.strategy)
    if strategy == Strategy.AUTO:  # degree_stats from the upload's own max-degree scan (no second host pass)
        strategy = (select_strategy(DegreeStats(d_avg=dg.num_edges / dg.num_nodes, d_max=dg.d_max,
                                                rho=dg.d_max / (dg.num_edges / dg.num_nodes)))
                    if dg.num_edges > 0 else Strategy.PER_NODE)
    count_mode = m.transmission.kind == "constant" and dg.uniform and cfg.gather != "f32"
    if cfg.gather in ("count", "incremental") and not count_mode:
        raise InvalidConfigError(f"gather={cfg.gather!r} needs constant transmission and uniform weights")
    c = _lib.FsConfig(
        epsilon=cfg.epsilon, tau_max=cfg.tau_max, delta=cfg.delta,
        steps_per_batch=cfg.steps_per_batch, strategy=_STRATEGY_CODE[strategy],
        compaction=int(cfg.compaction), mixed_precision=int(mixed),
        lanes_per_node=cfg.lanes_per_node, edges_per_block=cfg.edges_per_block,
        hazard_chunk=cfg.hazard_chunk, chunk_skip=int(cfg.chunk_skip), carry_tau=int(cfg.carry_tau),
        rng=RNG_KINDS[cfg.rng], hazard_precision=_PRECISION[cfg.hazard_precision],
        count_gather=1 if count_mode else 0,
        incremental=_INCREMENTAL[cfg.gather] if count_mode else 0,
    )
    return _EnginePlan(strategy=strategy, graph=dg, model=model_descriptor(m), config=c,
                       succ=m.successor_array(), terminal=m.terminal_mask(), count_mode=count_mode,
                       mixed=bool(mixed), num_compartments=m.num_compartments)


# ----------------------------------------------------------------------
# engine handle
# ----------------------------------------------------------------------


class _Engine:
    """Owns one fs_engine bound to a state's device buffers."""

    def __init__(self, state: "RenewalState", plan: _EnginePlan, scal: _lib.FsScalars, inf: torch.Tensor,
                 materialize: bool):
        self.lib = _lib.load()
        self.plan = plan
        self.state = state
        n = state._n
        dev = state._dev
        self.stream = _device.stream_handle(dev)
        _, _, it = _storage(state.mixed_precision)
        w = ((n + 31) // 32 + 1 + 3) // 4 * 4  # + a zero sentinel word, 16-byte multiple (TMA)
        # the infectious mask (count gather), or the nonzero-infectivity
        # bitmap kept next to the f32 infectivity (the f32 gather's prefilter):
        # both parities in one allocation
        masks = _fill(torch.empty((2, w), dtype=torch.int32, device=dev), 0)
        self.masks = [masks[0], masks[1]]
        if plan.count_mode:
            self.bufs = self.masks
        else:
            self.bufs = [_fill(torch.empty(n, dtype=it, device=dev), 0) for _ in range(2)]
        self.materialize = materialize
        if materialize:
            state._ensure_debug_buffers()
        b = _lib.FsStateBuffers()
        b.states = _lib.ptr(state._t["states"])
        b.ages = _lib.ptr(state._t["ages"])
        b.imask[0], b.imask[1] = _lib.ptr(self.masks[0]), _lib.ptr(self.masks[1])
        if not plan.count_mode:
            b.infectivity[0], b.infectivity[1] = _lib.ptr(self.bufs[0]), _lib.ptr(self.bufs[1])
        b.pressure = _lib.ptr(state._t.get("pressure"))
        b.rates = _lib.ptr(state._t.get("rates"))
        b.padded = 2  # states / ages come from _node_buffer (whole 128-node units)
        if state._fresh:  # untouched init_renewal_state: ages 0, infectivity {0, beta}
            b.padded |= _lib.FS_BUF_FRESH
        state._fresh = False
        self._buffers = b
        h = ctypes.c_void_p()
        _lib.check(self.lib.fs_engine_create(plan.graph.view(), plan.model, plan.config, b, scal,
                                             dev.index, ctypes.byref(h)))
        self.handle = h
        self.load_infectivity(inf)

    def close(self, sync: bool = True) -> None:
        """sync=False: the caller has already synchronised the engine's work."""
        if getattr(self, "handle", None):
            if sync:
                torch.cuda.current_stream().synchronize()
            self.lib.fs_engine_destroy(self.handle)
            self.handle = None

    def __del__(self) -> None:
        self.close()

    def sync_ages(self) -> None:
        """Uniform S age back into the ages array (before host reads / edits)."""
        _lib.check(self.lib.fs_engine_sync_ages(self.handle, self.stream))

    def uniform_s_age(self) -> bool:
        return bool(self.lib.fs_engine_uniform_s_age(self.handle))

    def kernels_per_step(self) -> int:
        return int(self.lib.fs_engine_kernels_per_step(self.handle))

    def scalars(self) -> _lib.FsScalars:
        s = _lib.FsScalars()
        _lib.check(self.lib.fs_engine_get_scalars(self.handle, ctypes.byref(s), self.stream))
        return s

    def set_scalars(self, s: _lib.FsScalars) -> None:
        _lib.check(self.lib.fs_engine_set_scalars(self.handle, ctypes.byref(s), self.stream))

    def load_infectivity(self, inf: torch.Tensor) -> None:
        rc = self.lib.fs_engine_load_infectivity(self.handle, _lib.ptr(inf), self.stream)
        if rc == _lib.FS_EREPR:
            raise _NeedsGeneralGather()
        _lib.check(rc)

    def store_infectivity(self) -> torch.Tensor:
        _, _, it = _storage(self.state.mixed_precision)
        out = torch.empty(self.state._n, dtype=it, device=self.state._dev)
        _lib.check(self.lib.fs_engine_store_infectivity(self.handle, _lib.ptr(out), self.stream))
        return out

    def step(self, nsteps: int, materialize: bool, use_active: bool) -> None:
        _lib.check(self.lib.fs_engine_step(self.handle, nsteps, int(materialize), int(use_active), self.stream))

    def begin_batch(self) -> None:
        _lib.check(self.lib.fs_engine_begin_batch(self.handle, self.stream))

    def run_batch(self, materialize: bool) -> None:
        _lib.check(self.lib.fs_engine_run_batch(self.handle, int(materialize), self.stream))

    def snapshot(self) -> tuple:
        """Device copies of everything a step mutates (states, ages, the
        infectivity / mask double buffer, scalars) — for benchmarking the
        same step window twice."""
        self.sync_ages()
        t = self.state._t
        return (t["states"].clone(), t["ages"].clone(), [b.clone() for b in self._mutable_bufs()], self.scalars())

    def _mutable_bufs(self) -> list:
        # the double buffers a step writes (f32 gather: infectivity and its bitmap)
        return self.bufs if self.plan.count_mode else self.bufs + self.masks

    def restore(self, snap: tuple) -> None:
        st, ag, bufs, sc = snap
        self.state._t["states"].copy_(st)
        self.state._t["ages"].copy_(ag)
        for dst, src in zip(self._mutable_bufs(), bufs):
            dst.copy_(src)
        self.set_scalars(sc)
        # incremental counts / pending deltas follow the restored mask, not
        # the steps run since the snapshot
        _lib.check(self.lib.fs_engine_state_restored(self.handle, self.stream))

    def states_edited(self) -> None:
        _lib.check(self.lib.fs_engine_states_edited(self.handle, self.stream))

    def reset_age_memo(self) -> None:
        fn = getattr(self.lib, "fs_engine_reset_age_memo", None)  # absent only in older A/B builds
        if fn is not None:
            _lib.check(fn(self.handle, self.stream))

    def wait_log(self, first_step: int, n: int):
        """Log of the replayed batch ending at first_step + n, waiting for that
        batch only (later batches may be running)."""
        M = self.plan.num_compartments
        clocks = np.empty(n, dtype=np.float64)
        taus = np.empty(n, dtype=np.float64)
        counts = np.empty((n, M), dtype=np.int64)
        _lib.check(self.lib.fs_engine_wait_log(self.handle, first_step, n, clocks.ctypes.data, taus.ctypes.data,
                                               counts.ctypes.data))
        return clocks, taus, counts

    def read_log(self, first_step: int, n: int):
        M = self.plan.num_compartments
        clocks = np.empty(n, dtype=np.float64)
        taus = np.empty(n, dtype=np.float64)
        counts = np.empty((n, M), dtype=np.int64)
        _lib.check(self.lib.fs_engine_read_log(self.handle, first_step, n, clocks.ctypes.data, taus.ctypes.data,
                                               counts.ctypes.data, self.stream))
        return clocks, taus, counts


class _NeedsGeneralGather(Exception):
    pass


# ----------------------------------------------------------------------
# state
# ----------------------------------------------------------------------

_ARRAYS = ("states", "ages", "infectivity", "pressure", "rates")


class RenewalState:
    """Device-resident counterpart of renewal.py:114-126.

    The reference's fields are properties: per-node arrays download on
    access (numpy, the reference's dtypes) and in-place edits are pushed back
    before the next device operation; scalar assignments are written through.
    ``device_tensors()`` exposes the device buffers without copies.
    """

    def __init__(self, n: int, M: int, mixed: bool, dev: torch.device, tensors: dict, counts: np.ndarray,
                 tau_prev: float):
        self._n, self._M, self._dev = n, M, dev
        self._mixed = bool(mixed)
        self._t = tensors  # states, ages, inf (canonical while no engine), [pressure, rates]
        self._host_scal = _lib.FsScalars(clock=0.0, tau_next=tau_prev, step=0, seed=0, last_max_rate=0.0, started=0)
        for i, c in enumerate(counts):
            self._host_scal.counts[i] = int(c)
        self._engine: _Engine | None = None
        self._plan_key = None
        self._plans: dict = {}
        self._mirror: dict[str, tuple[np.ndarray, np.ndarray]] = {}
        self._scal_cache: _lib.FsScalars | None = None
        self._fresh = False  # set by the initialisers; any host write clears it

    # ---- engine binding ------------------------------------------------
    def _scal(self) -> _lib.FsScalars:
        if self._scal_cache is None:
            self._scal_cache = self._engine.scalars() if self._engine else self._host_scal
        return self._scal_cache

    def _write_scal(self, **kw) -> None:
        self._fresh = False
        s = _lib.FsScalars()
        ctypes.memmove(ctypes.byref(s), ctypes.byref(self._scal()), ctypes.sizeof(s))
        for k, v in kw.items():
            if k == "counts":
                for i, c in enumerate(v):
                    s.counts[i] = int(c)
            else:
                setattr(s, k, v)
        if self._engine:
            self._engine.set_scalars(s)
            self._scal_cache = None
        else:
            self._host_scal = s
            self._scal_cache = None

    def _current_infectivity(self) -> torch.Tensor:
        return self._engine.store_infectivity() if self._engine else self._t["inf"]

    def _unbind(self) -> None:
        """Drop the engine, moving scalars and infectivity back to the state."""
        if self._engine is None:
            return
        s = self._engine.scalars()
        inf = self._engine.store_infectivity()
        self._engine.sync_ages()  # the state's ages array is authoritative without an engine
        self._engine.close()
        self._engine = None
        self._host_scal = s
        self._t["inf"] = inf
        self._scal_cache = None
        self._plan_key = None

    def _bind(self, plan: _EnginePlan, seed: int, materialize: bool) -> _Engine:
        self._push_host()
        key = id(plan)
        e = self._engine
        if e is not None and (self._plan_key != key or (materialize and not e.materialize)):
            self._unbind()
            e = None
        if e is None:
            if plan.mixed != self._mixed:
                raise InvalidConfigError("plan precision does not match the state's storage")
            s = self._host_scal
            s.seed = seed & ((1 << 64) - 1)
            inf = self._t["inf"]
            try:
                e = _Engine(self, plan, s, inf, materialize)
            except _NeedsGeneralGather:
                # host-edited infectivity outside {0, beta}: switch this state
                # to the general f32 gather (same results, wider buffers)
                plan.config.count_gather = 0
                plan.count_mode = False
                e = _Engine(self, plan, s, inf, materialize)
            self._engine, self._plan_key = e, key
            self._t.pop("inf", None)  # the engine now owns the current infectivity
        else:
            s = self._scal()
            if s.seed != (seed & ((1 << 64) - 1)):
                self._write_scal(seed=seed & ((1 << 64) - 1))
        self._plan_ref = plan  # keep the plan (and its device graph) alive
        self._scal_cache = None
        return e

    def _plan_for(self, g, m, cfg) -> _EnginePlan:
        key = (id(g), id(m), tuple(sorted(vars(cfg).items(), key=lambda kv: kv[0])), self._mixed)
        p = self._plans.get(key)
        if p is None:
            p = self._plans[key] = _build_plan(g, m, cfg, self._mixed)
        return p

    def _ensure_debug_buffers(self) -> None:
        for name in ("pressure", "rates"):
            if name not in self._t:
                self._t[name] = _fill(torch.empty(self._n, dtype=torch.float32, device=self._dev), 0.0)

    # ---- host mirror -----------------------------------------------------
    def _download(self, name: str) -> np.ndarray:
        if name == "infectivity":
            return _device.to_host(self._current_infectivity())
        if name in ("pressure", "rates") and name not in self._t:
            return np.zeros(self._n, dtype=np.float32)
        if name == "ages" and self._engine is not None:
            self._engine.sync_ages()
        return _device.to_host(self._t[name])

    def _view(self, name: str) -> np.ndarray:
        hit = self._mirror.get(name)
        if hit is None:
            arr = self._download(name)
            self._mirror[name] = hit = (arr, arr.copy())
        return hit[0]

    def _upload(self, name: str, arr: np.ndarray) -> None:
        self._fresh = False
        st, at, it = _storage(self._mixed)
        if name == "counts":
            self._write_scal(counts=np.asarray(arr, dtype=np.int64))
            return
        arr = np.asarray(arr)
        if arr.shape != (self._n,):
            raise ValueError(f"{name} must have shape ({self._n},)")
        if name == "infectivity":
            t = _device.to_device(_host_cast(arr, it), self._dev)
            if self._engine is None:
                self._t["inf"] = t
                return
            try:
                self._engine.load_infectivity(t)
            except _NeedsGeneralGather:
                plan = self._engine.plan
                self._unbind()
                plan.config.count_gather = 0
                plan.count_mode = False
                self._t["inf"] = t
            return
        dtype = {"states": st, "ages": at}.get(name, torch.float32)
        if name in ("pressure", "rates"):
            self._ensure_debug_buffers()
        if name == "states" and self._engine is not None:
            self._engine.sync_ages()  # untouched S nodes keep their true age in the array
        self._t[name].copy_(_device.to_device(_host_cast(arr, dtype), self._dev))
        if name == "states" and self._engine is not None:
            self._engine.states_edited()  # age cohorts, and the pushes of implied status changes
        elif name == "ages" and self._engine is not None:
            self._engine.reset_age_memo()  # host-written nodes no longer follow their age cohorts

    def _push_host(self) -> None:
        """Upload every downloaded array the caller edited in place."""
        if self._mirror:
            # infectivity first: its upload rebuilds the engine's counts, which
            # the pushes implied by edited states then build on
            order = {"infectivity": 0, "counts": 1, "states": 2}
            for name, (arr, snap) in sorted(self._mirror.items(), key=lambda kv: order.get(kv[0], 3)):
                if arr.shape != snap.shape or arr.tobytes() != snap.tobytes():
                    self._upload(name, arr)
            self._mirror.clear()
        self._scal_cache = None

    def _after_device(self) -> None:
        self._mirror.clear()
        self._scal_cache = None

    # ---- reference fields ----------------------------------------------
    def device_tensors(self) -> dict:
        """The live device buffers (no copies)."""
        self._fresh = False  # the caller may write them
        self._push_host()
        if self._engine is not None:
            self._engine.sync_ages()
        return dict(self._t)

    @property
    def num_nodes(self) -> int:
        return self._n

    @property
    def mixed_precision(self) -> bool:
        return self._mixed

    @property
    def counts(self) -> np.ndarray:
        hit = self._mirror.get("counts")
        if hit is None:
            arr = np.array(self._scal().counts[: self._M], dtype=np.int64)
            self._mirror["counts"] = hit = (arr, arr.copy())
        return hit[0]

    @counts.setter
    def counts(self, v) -> None:
        self._mirror.pop("counts", None)
        self._upload("counts", v)

    @property
    def clock(self) -> float:
        return float(self._scal().clock)

    @clock.setter
    def clock(self, v: float) -> None:
        self._write_scal(clock=float(v))

    @property
    def tau_prev(self) -> float:
        return float(self._scal().tau_next)

    @tau_prev.setter
    def tau_prev(self, v: float) -> None:
        self._write_scal(tau_next=float(v))

    @property
    def step_counter(self) -> int:
        return int(self._scal().step)

    @step_counter.setter
    def step_counter(self, v: int) -> None:
        self._write_scal(step=int(v))

    @property
    def started(self) -> bool:
        return bool(self._scal().started)

    @started.setter
    def started(self, v: bool) -> None:
        self._write_scal(started=int(bool(v)))


def _host_cast(arr: np.ndarray, dtype: torch.dtype) -> np.ndarray:
    if dtype == torch.bfloat16:
        import ml_dtypes

        return np.asarray(arr).astype(np.float32).astype(ml_dtypes.bfloat16)
    npd = {torch.int8: np.int8, torch.int32: np.int32, torch.float16: np.float16, torch.float32: np.float32}[dtype]
    return np.asarray(arr).astype(npd)


def _make_array_property(name: str):
    def get(self: RenewalState) -> np.ndarray:
        return self._view(name)

    def put(self: RenewalState, v) -> None:
        self._mirror.pop(name, None)
        self._upload(name, np.asarray(v))

    return property(get, put, doc=f"{name} (downloaded on access; edits are pushed back)")


for _name in _ARRAYS:
    setattr(RenewalState, _name, _make_array_property(_name))


# ----------------------------------------------------------------------
# public API
# ----------------------------------------------------------------------


def _seed_select(n: int, seed: int, count: int, dev: torch.device, states=None, comp: int = 0, inf=None,
                 inf_value: float = 0.0, flags=None) -> None:
    """fs_seed_select: the `count` nodes with the smallest
    u(derive_seed(seed, salt), 0, id) (renewal.py:162-169), marked on the device."""
    if not 0 <= count <= n:
        raise ValueError(f"seed count {count} outside [0, N]")
    st_dt = _lib.I8 if states is not None and states.dtype == torch.int8 else _lib.I32
    inf_dt = _lib.BF16 if inf is not None and inf.dtype == torch.bfloat16 else _lib.F32
    _lib.check(_lib.load().fs_seed_select(n, derive_seed(seed, _SEED_PICK_SALT) & ((1 << 64) - 1), count,
                                          _lib.ptr(states), st_dt, int(comp), _lib.ptr(inf), inf_dt,
                                          float(inf_value), _lib.ptr(flags), _device.stream_handle(dev)))


def _pick_seed_nodes(n: int, seed: int, count: int, dev: torch.device) -> torch.Tensor:
    """The `count` nodes with the smallest u(derive_seed(seed, salt), 0, id)
    (renewal.py:162-169), chosen on the device; sorted int64 ids."""
    if not 0 <= count <= n:
        raise ValueError(f"seed count {count} outside [0, N]")
    if count == 0:
        return torch.empty(0, dtype=torch.int64, device=dev)
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    _seed_select(n, seed, count, dev, flags=flags)
    ids = torch.empty(count, dtype=torch.int64, device=dev)
    got = ctypes.c_int64()
    _lib.check(_lib.load().fs_flags_to_ids(_lib.ptr(flags), n, _lib.ptr(ids), ctypes.byref(got),
                                           _device.stream_handle(dev)))
    if got.value != count:
        raise AssertionError(f"seed selection picked {got.value} nodes, expected {count}")
    return ids


def init_renewal_state(g, m, cfg: RenewalConfig, seed: int, seed_count: int | None = None,
                       seed_compartment: int | None = None) -> RenewalState:
    """Fresh device state: all nodes in S at age 0, `seed_count` nodes in
    `seed_compartment` (default the first infected successor), infectivity
    consistent with the seeded state (renewal.py:370-410)."""
    cfg = as_config(cfg)
    n = int(g.num_nodes)
    if seed_count is None:
        seed_count = default_seed_count(n)
    if not 0 <= seed_count <= n:
        raise ValueError(f"seed_count {seed_count} outside [0, N]")
    comp = m.edge_to if seed_compartment is None else int(seed_compartment)
    dev = _device.device()
    mixed = bool(cfg.mixed_precision)
    st, at, it = _storage(mixed)
    states = _node_buffer(n, st, dev, int(m.edge_from))
    ages = _node_buffer(n, at, dev)
    # infectivity beta * s(0): s(0) = 1 for constant transmission and 0 for
    # the hazard / density profiles (h(0) = 0, f(0) = 0)
    inf = _fill(torch.empty(n, dtype=it, device=dev), 0)
    seeded_inf = comp == m.infectious and m.transmission.kind == "constant"
    if seed_count:
        _seed_select(n, seed, seed_count, dev, states=states, comp=comp, inf=inf if seeded_inf else None,
                     inf_value=float(np.float32(m.beta)))
    counts = np.zeros(m.num_compartments, dtype=np.int64)
    counts[m.edge_from] += n - seed_count
    counts[comp] += seed_count
    st = RenewalState(n, m.num_compartments, mixed, dev, {"states": states, "ages": ages, "inf": inf},
                      counts, cfg.tau_max)
    st._fresh = True
    return st


def init_renewal_states(g, m, cfg: RenewalConfig, seeds, seed_count: int | None = None,
                        seed_compartment: int | None = None) -> list[RenewalState]:
    """init_renewal_state for many seeds (an ensemble's trials) at once: for
    graphs of up to 4096 nodes one batched device allocation and one seed-
    selection launch for every trial (fs_seed_select_batch); each state is
    exactly init_renewal_state(g, m, cfg, seed, ...)."""
    cfg = as_config(cfg)
    seeds = list(seeds)
    n = int(g.num_nodes)
    if n > 4096 or len(seeds) < 2:
        return [init_renewal_state(g, m, cfg, s, seed_count, seed_compartment) for s in seeds]
    if seed_count is None:
        seed_count = default_seed_count(n)
    if not 0 <= seed_count <= n:
        raise ValueError(f"seed_count {seed_count} outside [0, N]")
    comp = m.edge_to if seed_compartment is None else int(seed_compartment)
    dev = _device.device()
    mixed = bool(cfg.mixed_precision)
    st_t, at_t, it_t = _storage(mixed)
    R = len(seeds)
    cap = (n + 127) // 128 * 128
    states = _fill(torch.empty((R, cap), dtype=st_t, device=dev), int(m.edge_from))
    ages = _fill(torch.empty((R, cap), dtype=at_t, device=dev), 0)
    inf = _fill(torch.empty((R, cap), dtype=it_t, device=dev), 0)
    seeded_inf = comp == m.infectious and m.transmission.kind == "constant"
    keys = np.array([derive_seed(s, _SEED_PICK_SALT) & ((1 << 64) - 1) for s in seeds], dtype=np.uint64)
    if seed_count:
        _lib.check(_lib.load().fs_seed_select_batch(
            n, R, keys.ctypes.data, seed_count, _lib.ptr(states), cap, _lib.I8 if mixed else _lib.I32, comp,
            _lib.ptr(inf) if seeded_inf else None, _lib.BF16 if mixed else _lib.F32, float(np.float32(m.beta)),
            _device.stream_handle(dev)))
    counts = np.zeros(m.num_compartments, dtype=np.int64)
    counts[m.edge_from] += n - seed_count
    counts[comp] += seed_count
    out = []
    for r in range(R):
        st = RenewalState(n, m.num_compartments, mixed, dev,
                          {"states": states[r, :n], "ages": ages[r, :n], "inf": inf[r, :n]}, counts, cfg.tau_max)
        st._fresh = True
        out.append(st)
    return out


def set_mixed_precision(state: RenewalState, on: bool) -> RenewalState:
    """Re-encode the storage of a not-yet-started state (renewal.py:413-423)."""
    if state.started:
        raise ReconfigureAfterStartError("cannot change precision after the first step")
    if bool(on) == state.mixed_precision:
        return state
    state._push_host()
    state._unbind()
    st, at, it = _storage(bool(on))
    for name, dt in (("states", st), ("ages", at)):
        buf = _node_buffer(state._n, dt, state._dev)
        buf.copy_(state._t[name].to(dt))
        state._t[name] = buf
    state._t["inf"] = state._t["inf"].to(torch.float32).to(it)
    state._mixed = bool(on)
    state._plans.clear()
    state._after_device()
    return state


def refresh_active(states, terminal, pad: int = 128) -> ActiveSet:
    """Sorted ids of non-absorbed nodes, zero-padded to N + pad (renewal.py:426-432)."""
    lib = _lib.load()
    dev = _device.device()
    term = np.ascontiguousarray(np.asarray(terminal, dtype=np.uint8))
    if isinstance(states, torch.Tensor):
        s_t = states.to(dev)
    else:
        a = np.asarray(states)
        s_t = torch.from_numpy(np.ascontiguousarray(a.astype(np.int8 if a.dtype == np.int8 else np.int32))).to(dev)
    n = s_t.numel()
    dt = _lib.I8 if s_t.dtype == torch.int8 else _lib.I32
    if dt == _lib.I32 and s_t.dtype != torch.int32:
        s_t = s_t.to(torch.int32)
    out = torch.empty(n + pad, dtype=torch.int32, device=dev)
    num = ctypes.c_int64()
    _lib.check(lib.fs_refresh_active(_lib.ptr(s_t), dt, n, term.ctypes.data, term.size, _lib.ptr(out), n + pad,
                                     ctypes.byref(num), _device.stream_handle(dev)))
    return ActiveSet(active_nodes=out.cpu().numpy(), num_active=int(num.value))


def pressure_gather(g, infectivity, strategy: Strategy, cfg: RenewalConfig, active: ActiveSet | None = None, *,
                    plan: _EnginePlan | None = None):
    """p_i = sum_j inf[j] w_ji over incoming edges, folded in CSR order with
    an f32 accumulator, bit-identical across strategies (renewal.py:264-313).

    numpy in -> numpy out; a CUDA tensor in -> CUDA tensor out.
    """
    cfg = as_config(cfg)
    lib = _lib.load()
    dev = _device.device()
    strategy = resolve_strategy(g, strategy)
    mixed = plan.mixed if plan is not None else False
    dg = plan.graph if plan is not None else device_graph(g, mixed)
    on_device = isinstance(infectivity, torch.Tensor)
    if on_device:
        inf_t = infectivity.to(dev)
    else:
        a = np.asarray(infectivity)
        inf_t = _device.to_device(a if a.dtype.name == "bfloat16" else a.astype(np.float32), dev)
    if inf_t.dtype not in (torch.float32, torch.bfloat16):
        inf_t = inf_t.to(torch.float32)
    out = torch.empty(dg.num_nodes, dtype=torch.float32, device=dev)
    _lib.check(lib.fs_pressure_gather(dg.view(), _lib.ptr(inf_t), _lib.BF16 if inf_t.dtype == torch.bfloat16 else _lib.F32,
                                      _lib.ptr(out), _STRATEGY_CODE[strategy], cfg.lanes_per_node,
                                      cfg.edges_per_block, _device.stream_handle(dev)))
    if active is not None and strategy != Strategy.EDGE_MERGE:
        keep = torch.zeros(dg.num_nodes, dtype=torch.bool, device=dev)
        keep[torch.from_numpy(active.ids.astype(np.int64)).to(dev)] = True
        out = torch.where(keep, out, torch.zeros_like(out))
    return out if on_device else out.cpu().numpy()


def _check_conservation(counts: np.ndarray, n: int) -> None:
    bad = np.flatnonzero(counts.sum(axis=-1) != n)
    if bad.size:
        raise AssertionError(f"compartment counts no longer sum to N={n} (renewal.py:554)")


def _check_active(state: RenewalState, plan: _EnginePlan, active: ActiveSet) -> None:
    """The reference steps exactly `active.ids` (renewal.py:509-520); its
    callers pass the set `_begin_batch` returned — the nodes not absorbed at
    the batch start, `refresh_active(states, terminal)`, a superset of the
    nodes live now — and absorbed nodes do not change in a step, so
    processing that set is processing every node.  The fused
    kernel works on whole 32-node tiles of that set (rebuilt from the
    current states when the engine's list is stale, fs_engine_step); a
    different subset (which would freeze the ages of the left-out live
    nodes) is refused instead of being silently widened."""
    live = refresh_active(state._t["states"], plan.terminal, pad=0).ids.astype(np.int64)
    if not np.isin(live, np.asarray(active.ids, dtype=np.int64), assume_unique=True).all():
        raise InvalidConfigError(
            "renewal_step(active=...) must contain every live node (the set _begin_batch / refresh_active(states, "
            "terminal) returns); a subset that leaves live nodes out is not supported")


def renewal_step(state: RenewalState, g, m, cfg: RenewalConfig, seed: int, *, plan: _EnginePlan | None = None,
                 active: ActiveSet | None = None) -> tuple[RenewalState, float]:
    """One fused tau-leap (renewal.py:483-580): one kernel launch (two under
    EDGE_MERGE), pressure / rates materialised for inspection.

    With an active set (compaction) the step is exact for the nodes it
    processes, but the materialised `state.pressure` is specified only for
    the listed nodes (the values the step uses): terminal nodes inside an
    active 32-node tile may carry their gathered pressure and, under
    EDGE_MERGE, nodes outside the active tiles read 0, where the reference
    writes 0 for every unlisted node under PER_NODE / LANE and keeps the
    whole-graph merge gather under EDGE_MERGE (R/renewal.py:276-302).
    States, ages, infectivity, counts and the clock are bit-exact either
    way."""
    cfg = as_config(cfg)
    if plan is None:
        plan = state._plan_for(g, m, cfg)
    eng = state._bind(plan, seed, materialize=True)
    if active is not None:
        _check_active(state, plan, active)
    before = eng.scalars()
    eng.step(1, materialize=True, use_active=active is not None and bool(cfg.compaction))
    state._after_device()
    _check_conservation(state.counts[None, :], state._n)
    return state, float(before.tau_next)


def _begin_batch(state: RenewalState, g, cfg: RenewalConfig, plan: _EnginePlan) -> ActiveSet | None:
    """Batch boundary (renewal.py:583-597): tau reset unless carry_tau;
    under compaction rates are zeroed and the active list refreshed."""
    cfg = as_config(cfg)
    eng = state._bind(plan, state._scal().seed, materialize=True)
    eng.begin_batch()
    state._after_device()
    if not cfg.compaction:
        return None
    return refresh_active(state._t["states"], plan.terminal, pad=cfg.hazard_chunk)


def run_batch(state: RenewalState, g, m, cfg: RenewalConfig, seed: int, *, plan: _EnginePlan | None = None,
              recorder: list | None = None) -> tuple[RenewalState, float]:
    """steps_per_batch fused steps as one CUDA-graph replay (renewal.py:600-629)."""
    cfg = as_config(cfg)
    if plan is None:
        plan = state._plan_for(g, m, cfg)
    eng = state._bind(plan, seed, materialize=True)
    first = int(eng.scalars().step)
    eng.run_batch(materialize=True)
    b = cfg.steps_per_batch
    clocks, taus, counts = eng.read_log(first, b)
    state._after_device()
    _check_conservation(counts, state._n)
    if recorder is not None:
        for k in range(b):
            recorder.append((float(clocks[k]), counts[k].copy()))
    total = 0.0
    for t in taus:
        total += float(t)
    return state, total


def run_renewal(g, m, cfg: RenewalConfig, seed: int, t_final: float, grid_points: int = DEFAULT_GRID_POINTS,
                seed_count: int | None = None, seed_compartment: int | None = None) -> TrajectoryRecord:
    """Whole batches until clock >= t_final, sampled onto the grid
    (renewal.py:632-663).  One graph replay and one log read per batch."""
    cfg = as_config(cfg)
    t0 = time.perf_counter()
    state = init_renewal_state(g, m, cfg, seed, seed_count, seed_compartment)
    plan = _build_plan(g, m, cfg, state.mixed_precision)
    eng = state._bind(plan, seed, materialize=False)
    setup = time.perf_counter() - t0
    b = cfg.steps_per_batch
    times = [0.0]
    rows = [state.counts.copy()]
    done, clock = 0, 0.0
    trace = [] if os.environ.get("FS_E2E_TRACE") else None  # per-batch wall times (diagnostics)
    # pipelined: batch j+1 is queued before batch j's log is read, so the GPU
    # never waits for the host; the loop stops at the first batch whose clock
    # reaches t_final, exactly as the reference's (the one batch launched past
    # it only advances this function's private state)
    eng.run_batch(materialize=False)
    while clock < t_final:
        tb = time.perf_counter()
        eng.run_batch(materialize=False)
        clocks, _, counts = eng.wait_log(done, b)
        _check_conservation(counts, state._n)
        times.extend(clocks.tolist())
        rows.extend(counts)
        done += b
        clock = float(clocks[-1])
        if trace is not None:
            trace.append(round((time.perf_counter() - tb) * 1e3, 2))
    wall = time.perf_counter() - t0
    t_arr = np.asarray(times)
    steps = min(int(np.searchsorted(t_arr, t_final, side="left")), done)
    rec = make_record(t_arr, np.asarray(rows), m.compartments, g.num_nodes, t_final, grid_points,
                      extra_summary={"step_count": steps, "wall_clock": wall, "engine": "renewal", "setup_s": setup})
    if trace is not None:
        rec.summary["batch_ms"] = trace
        tu = time.perf_counter()
    state._unbind()
    if trace is not None:
        rec.summary["record_ms"] = round((tu - t0 - wall) * 1e3, 2)
        rec.summary["unbind_ms"] = round((time.perf_counter() - tu) * 1e3, 2)
    return rec
