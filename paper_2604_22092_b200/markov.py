"""Drop-in for ``spreadsim.markov`` (the Markovian tau-leaping engine,
R/markov.py) backed by csrc/fs_markov.cu — SURVEY.md §8f row 3.

Same names and semantics as the reference (R/markov.py:23-31):
``MarkovConfig``, ``MarkovState``, ``init_markov_state``,
``influence_gather``, ``inertial_update``, ``markov_step``, ``run_markov``.
A step is four kernels (rates, the pairwise-sum leaves, the sum tree + tau,
fire + pushes); ``run_markov`` replays them as CUDA-graph batches.  Results
are bit-identical to the reference given the same seed: the uniforms are the
reference's, the total rate is summed in numpy's pairwise order, and the
influence is an integer count (Control and Inertial mode agree exactly, so
``rebuild_every`` / ``inertial_threshold`` are accepted and have no effect on
the results).  Scope: constant transmission, exponential holding times (as
the reference requires, R/markov.py:59-65) and uniform edge weights.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .errors import InvalidConfigError
from .models import model_descriptor
from .renewal import _node_buffer, _pick_seed_nodes, device_graph
from .trajectory import TrajectoryRecord, make_record

__all__ = ["MarkovConfig", "MarkovState", "init_markov_state", "influence_gather", "inertial_update",
           "markov_step", "run_markov"]


@dataclass
class MarkovConfig:
    """R/markov.py:34-46 (+ ``steps_per_batch``: steps per CUDA-graph replay)."""

    theta: float = 0.01
    p_max: float = 0.1
    tau_max: float = 0.1
    rebuild_every: int = 200
    inertial_threshold: float = 8.0
    steps_per_batch: int = 50

    def __post_init__(self) -> None:
        if not (0.0 < self.p_max < 1.0):
            raise ValueError("p_max must be in (0, 1)")
        if self.theta <= 0.0 or self.tau_max <= 0.0:
            raise ValueError("theta and tau_max must be > 0")


def _check_markovian(m) -> None:
    """R/markov.py:59-65."""
    for _, holding in m.nodal.values():
        if holding.kind != "exponential":
            raise ValueError("the Markovian engine requires exponential holding times")
    if m.transmission.kind != "constant":
        raise ValueError("the Markovian engine requires constant transmission")


class MarkovState:
    """Device-backed R/markov.py:48-56: ``states`` / ``rates`` / ``influence``
    download on access (edits to ``states`` are pushed back before the next
    step); ``clock``, ``step_counter``, ``counts`` are the engine scalars."""

    def __init__(self, g, m, states: torch.Tensor, counts: np.ndarray):
        self._g, self._m = g, m
        self._n = int(g.num_nodes)
        self._states = states
        self._rates = torch.zeros(self._n, dtype=torch.float64, device=states.device)
        self._host = _lib.FsScalars(clock=0.0, tau_next=0.0, step=0, seed=0, last_max_rate=0.0, started=0)
        for i, c in enumerate(counts):
            self._host.counts[i] = int(c)
        self._eng = None
        self._key = None
        self._mirror = None
        self.events_since_rebuild = 0

    # engine ---------------------------------------------------------------
    def _bind(self, cfg: MarkovConfig, seed: int):
        key = (cfg.theta, cfg.p_max, cfg.tau_max, cfg.steps_per_batch)
        self._push_host()
        if self._eng is not None and self._key != key:
            self._unbind()
        seed64 = seed & ((1 << 64) - 1)
        if self._eng is None:
            dg = device_graph(self._g, False)
            if not dg.uniform:
                raise InvalidConfigError("the B200 Markov engine needs uniform edge weights (exact influence)")
            if not dg.symmetric:
                raise InvalidConfigError("the B200 Markov engine needs the outgoing CSR (undirected graph)")
            self._dg = dg
            lib = _lib.load()
            c = _lib.FsMarkovConfig(theta=cfg.theta, p_max=cfg.p_max, tau_max=cfg.tau_max,
                                    steps_per_batch=cfg.steps_per_batch)
            self._host.seed = seed64
            h = ctypes.c_void_p()
            _lib.check(lib.fs_markov_create(dg.view(), model_descriptor(self._m), c, _lib.ptr(self._states),
                                            _lib.ptr(self._rates), self._host, self._states.device.index,
                                            ctypes.byref(h)))
            self._eng, self._key, self._lib = h, key, lib
            self._stream = _device.stream_handle(self._states.device)
        elif self._scal().seed != seed64:
            s = self._scal()
            s.seed = seed64
            self._set(s)
        return self._eng

    def _unbind(self) -> None:
        if self._eng is not None:
            self._host = self._scal()
            torch.cuda.current_stream().synchronize()
            self._lib.fs_markov_destroy(self._eng)
            self._eng = None

    __del__ = _unbind

    def _scal(self) -> _lib.FsScalars:
        if self._eng is None:
            return self._host
        s = _lib.FsScalars()
        _lib.check(self._lib.fs_markov_get_scalars(self._eng, ctypes.byref(s), self._stream))
        return s

    def _set(self, s: _lib.FsScalars) -> None:
        if self._eng is None:
            self._host = s
        else:
            _lib.check(self._lib.fs_markov_set_scalars(self._eng, ctypes.byref(s), self._stream))

    def _push_host(self) -> None:
        if self._mirror is not None:
            arr, snap = self._mirror
            self._mirror = None
            if arr.tobytes() != snap.tobytes():
                self._states.copy_(torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32)).to(self._states.device))
                self._set(self._scal())  # rebuild the counts from the edited states

    # reference fields -------------------------------------------------------
    @property
    def states(self) -> np.ndarray:
        if self._mirror is None:
            a = self._states.cpu().numpy()
            self._mirror = (a, a.copy())
        return self._mirror[0]

    @states.setter
    def states(self, v) -> None:
        self._mirror = (np.asarray(v, dtype=np.int32).copy(), np.full(self._n, -1, dtype=np.int32))

    @property
    def rates(self) -> np.ndarray:
        self._push_host()
        if self._eng is not None:
            _lib.check(self._lib.fs_markov_refresh_rates(self._eng, self._stream))
        return self._rates.cpu().numpy()

    @rates.setter
    def rates(self, v) -> None:  # the engine recomputes rates from states and influence each step
        self._rates.copy_(torch.as_tensor(np.asarray(v, dtype=np.float64)))

    @property
    def influence(self) -> np.ndarray:
        self._push_host()
        if self._eng is None:
            return influence_gather(self._g, self._states, self._m)
        out = np.empty(self._n, dtype=np.float64)
        _lib.check(self._lib.fs_markov_influence(self._eng, out.ctypes.data, self._stream))
        return out

    @influence.setter
    def influence(self, v) -> None:  # derived from states (R/markov.py influence is a cache of it)
        pass

    @property
    def clock(self) -> float:
        return float(self._scal().clock)

    @clock.setter
    def clock(self, v: float) -> None:
        s = self._scal()
        s.clock = float(v)
        self._set(s)

    @property
    def step_counter(self) -> int:
        return int(self._scal().step)

    @step_counter.setter
    def step_counter(self, v: int) -> None:
        s = self._scal()
        s.step = int(v)
        self._set(s)

    @property
    def counts(self) -> np.ndarray:
        return np.array(self._scal().counts[: len(self._m.compartments)], dtype=np.int64)

    @counts.setter
    def counts(self, v) -> None:
        s = self._scal()
        for i, c in enumerate(np.asarray(v, dtype=np.int64)):
            s.counts[i] = int(c)
        self._set(s)


def influence_gather(g, states, m) -> np.ndarray:
    """Infectious in-degree (weighted) of every node, f64 (R/markov.py:68-81),
    computed on the device; exact for uniform weights."""
    from .renewal import pressure_gather, resolve_strategy  # noqa: F401

    dg = device_graph(g, False)
    if not dg.uniform:
        raise InvalidConfigError("influence_gather on the device needs uniform edge weights")
    dev = _device.device()
    st = states if isinstance(states, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(states)).to(dev)
    flags = (st.to(dev) == m.infectious).to(torch.float32)
    from .graph import Strategy
    from .renewal import RenewalConfig

    p = pressure_gather(g, flags, Strategy.PER_NODE, RenewalConfig())  # exact integer counts (< 2^24) * 1.0
    return (p.to(torch.float64) * dg.uniform_weight).cpu().numpy() if dg.uniform_weight != 1.0 else \
        p.to(torch.float64).cpu().numpy()


def init_markov_state(g, m, seed_nodes) -> MarkovState:
    """R/markov.py:98-119: all S, `seed_nodes` infectious."""
    _check_markovian(m)
    dev = _device.device()
    n = int(g.num_nodes)
    states = _node_buffer(n, torch.int32, dev, int(m.edge_from))
    ids = np.asarray(seed_nodes, dtype=np.int64)
    if ids.size:
        states[torch.from_numpy(ids).to(dev)] = int(m.infectious)
    counts = np.zeros(len(m.compartments), dtype=np.int64)
    counts[m.edge_from] = n - ids.size
    counts[m.infectious] += ids.size
    return MarkovState(g, m, states, counts)


def inertial_update(state: MarkovState, transitioned, g, m) -> MarkovState:
    """R/markov.py:122-140.  The engine applies the same sparse updates (as
    integer pushes) inside every step, so the influence is always current:
    nothing to do here."""
    return state


def markov_step(state: MarkovState, g, m, cfg: MarkovConfig, seed: int) -> tuple[MarkovState, float]:
    """One adaptive tau-leap (R/markov.py:143-181); returns (state, tau)."""
    eng = state._bind(cfg, seed)
    _lib.check(state._lib.fs_markov_step(eng, 1, state._stream))
    s = state._scal()
    return state, float(s.tau_next)


def run_markov(g, m, cfg: MarkovConfig, seed: int, t_final: float, grid_points: int = 101, seed_count: int = 10,
               seed_compartment: int | None = None) -> TrajectoryRecord:
    """R/markov.py:184-228: CUDA-graph batches until clock >= t_final."""
    t0 = time.perf_counter()
    _check_markovian(m)
    dev = _device.device()
    comp = m.infectious if seed_compartment is None else seed_compartment
    picked = _pick_seed_nodes(int(g.num_nodes), seed, seed_count, dev).cpu().numpy()
    state = init_markov_state(g, m, picked)
    if comp != m.infectious and picked.size:
        state._states[torch.from_numpy(picked).to(dev)] = int(comp)
        counts = np.zeros(len(m.compartments), dtype=np.int64)
        counts[m.edge_from] = g.num_nodes - picked.size
        counts[comp] += picked.size
        state.counts = counts
    eng = state._bind(cfg, seed)
    lib, b = state._lib, cfg.steps_per_batch
    times, rows = [0.0], [state.counts.copy()]
    done, clock = 0, 0.0
    clocks = np.empty(b)
    counts = np.empty((b, len(m.compartments)), dtype=np.int64)
    while clock < t_final:
        _lib.check(lib.fs_markov_run_batch(eng, state._stream))
        _lib.check(lib.fs_markov_read_log(eng, done, b, clocks.ctypes.data, None, counts.ctypes.data, state._stream))
        # the reference stops at the first step with clock >= t_final
        stop = int(np.searchsorted(clocks, t_final, side="left"))
        take = b if stop >= b else stop + 1
        times.extend(clocks[:take].tolist())
        rows.extend(counts[:take].copy())
        done += b
        clock = float(clocks[take - 1])
    wall = time.perf_counter() - t0
    t_arr = np.asarray(times)
    steps = int(np.searchsorted(t_arr, t_final, side="left"))
    rec = make_record(t_arr, np.asarray(rows), m.compartments, g.num_nodes, t_final, grid_points,
                      extra_summary={"step_count": steps, "wall_clock": wall, "engine": "markov"})
    state._unbind()
    return rec
