"""GPU ensembles of independent renewal trajectories.

The reference runs ensembles as a process pool of CPU trajectories,
`run_ensemble(engine, g, m, cfg, seed, t_final, runs, ...)` with per-trial
seeds `derive_seed(seed, trial)` and results ordered by trial
(R/analysis.py:97-130).  Here the trials of the "renewal" engine run on one
GPU at the same time: every trial owns an engine on its own CUDA stream,
the graph's device copy is shared, and the host loop keeps `concurrency`
trials in flight, launching one CUDA-graph batch per trial per round and
reading each trial's per-batch log as it lands (one batch queued ahead of the one read, so the
GPU never waits for the host); the trajectory records
of all trials are built by one device launch (analysis.make_records).  Each trial is exactly
`run_renewal(g, m, cfg, derive_seed(seed, trial), ...)` (same kernels, same
per-trial RNG keys), so the ensemble is bit-identical to the sequential one
and to the reference's CPU ensemble (tests/test_ensemble.py).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np
import torch

from . import _device, _lib
from .renewal import RenewalConfig, _build_plan, as_config, _check_conservation, init_renewal_state, init_renewal_states
from .rng import derive_seed
from .analysis import make_records
from .trajectory import DEFAULT_GRID_POINTS, TrajectoryRecord

__all__ = ["run_ensemble"]


class _Trial:
    def __init__(self, trial: int, g, m, cfg, seed: int, seed_count, seed_compartment, stream, plan):
        self.trial, self.stream = trial, stream
        self.seed = derive_seed(seed, trial)
        self.t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            self.state = init_renewal_state(g, m, cfg, self.seed, seed_count, seed_compartment)
            self.eng = self.state._bind(plan, self.seed, materialize=False)
        self.times = [0.0]
        self.rows = [self.state.counts.copy()]
        self.done, self.clock = 0, 0.0

    def launch(self) -> None:
        self.eng.run_batch(materialize=False)

    def collect(self, b: int, n: int) -> None:
        clocks, _, counts = self.eng.wait_log(self.done, b)  # this batch only; the next may be running
        _check_conservation(counts, n)
        self.times.extend(clocks.tolist())
        self.rows.extend(counts)
        self.done += b
        self.clock = float(clocks[-1])

    def finish(self, t_final: float):
        """(times, counts, summary) of the finished trial; the record itself
        is built with every other trial's by one device launch."""
        wall = time.perf_counter() - self.t0
        t_arr = np.asarray(self.times)
        steps = min(int(np.searchsorted(t_arr, t_final, side="left")), self.done)
        with torch.cuda.stream(self.stream):
            self.state._unbind()
        self.stream.synchronize()
        return t_arr, np.asarray(self.rows), {"step_count": steps, "wall_clock": wall, "engine": "renewal"}


class _Lockstep:
    """A group of trials stepped by one grid per step (fs_ensemble): every
    trial is an ordinary engine; the ensemble launches the step of all of them
    at once and keeps their logs in one ring, read back once per batch."""

    def __init__(self, trials: list[int], g, m, cfg, seed: int, seed_count, seed_compartment, plan):
        self.lib = _lib.load()
        self.trials = trials
        self.seeds = [derive_seed(seed, t) for t in trials]
        self.states = init_renewal_states(g, m, cfg, self.seeds, seed_count, seed_compartment)
        self.c0 = np.stack([st.counts for st in self.states])  # host scalars: read before the engines own them
        self.engines = [st._bind(plan, s, materialize=False) for st, s in zip(self.states, self.seeds)]
        arr = (ctypes.c_void_p * len(trials))(*[e.handle.value for e in self.engines])
        h = ctypes.c_void_p()
        rc = self.lib.fs_ensemble_create(arr, len(trials), ctypes.byref(h))
        self.handle = h if rc == 0 else None
        self.rc = rc
        self.stream = _device.stream_handle(_device.device())
        self.M = len(m.compartments)
        self.clk = []   # per batch: clocks [R, b] and counts [R, b, M] of every trial
        self.cnt = []
        self.end = np.zeros(len(trials), dtype=np.int64)  # batches a single run would have taken (0: running)
        self.done = 0

    def run_batch(self) -> None:
        _lib.check(self.lib.fs_ensemble_run_batch(self.handle, self.stream))

    def collect(self, b: int, n: int, t_final: float) -> bool:
        R = len(self.trials)
        clocks = np.empty((R, b), dtype=np.float64)
        counts = np.empty((R, b, self.M), dtype=np.int64)
        _lib.check(self.lib.fs_ensemble_wait_log(self.handle, self.done, b, clocks.ctypes.data, None,
                                                 counts.ctypes.data))
        self.done += b
        live = self.end == 0  # past its own stopping batch a single run would have stopped
        _check_conservation(counts[live], n)
        self.clk.append(clocks)
        self.cnt.append(counts)
        self.end[live & (clocks[:, -1] >= t_final)] = len(self.clk)
        return bool((self.end > 0).all())

    def logs(self, r: int):
        """(times, counts) of trial r over its own batches, the t = 0 sample first."""
        k = int(self.end[r])
        times = np.concatenate([[0.0]] + [c[r] for c in self.clk[:k]])
        rows = np.concatenate([self.c0[r:r + 1]] + [c[r] for c in self.cnt[:k]])
        return times, rows

    def close(self) -> None:
        torch.cuda.current_stream().synchronize()  # once for the ensemble and every member
        if self.handle is not None:
            self.lib.fs_ensemble_destroy(self.handle)
            self.handle = None
        for e in self.engines:  # the trial states are dropped with their engines
            e.close(sync=False)


def _run_lockstep(g, m, cfg, seed, t_final, runs, seed_count, seed_compartment, plan, group: int):
    """Trials in lockstep groups of `group`; None when the engines cannot form
    an ensemble (e.g. a model or graph that needs the general gather)."""
    b = cfg.steps_per_batch
    out = []
    t0 = time.perf_counter()
    for lo in range(0, runs, group):
        ls = _Lockstep(list(range(lo, min(runs, lo + group))), g, m, cfg, seed, seed_count, seed_compartment, plan)
        try:
            if ls.handle is None:
                if lo == 0:
                    return None
                _lib.check(ls.rc)
            ls.run_batch()
            finished = False
            while not finished:
                ls.run_batch()  # one batch queued ahead of the one read
                finished = ls.collect(b, g.num_nodes, t_final)
        finally:
            ls.close()
        wall = time.perf_counter() - t0
        for r in range(len(ls.trials)):
            t_arr, rows = ls.logs(r)
            steps = min(int(np.searchsorted(t_arr, t_final, side="left")), int(ls.end[r]) * b)
            out.append((t_arr, rows, {"step_count": steps, "wall_clock": wall, "engine": "renewal"}))
    return out


def run_ensemble(engine: str, g, m, cfg, seed: int, t_final: float, runs: int,
                 grid_points: int = DEFAULT_GRID_POINTS, workers: int = 1, seed_count=None, seed_compartment=None,
                 concurrency: int = 32, lockstep: bool = True) -> list[TrajectoryRecord]:
    """R/analysis.py:97-130 for the renewal engine, every trial on the GPU
    (`workers` is accepted for signature compatibility).  Records are ordered
    by trial index.

    lockstep (default): groups of trials advance together, one step launch
    for the whole group (fs_ensemble), as many trials per group as fit
    ~2^27 nodes; trials whose engines cannot share a launch run as below.
    lockstep=False: one engine per trial on its own CUDA stream, `concurrency`
    trials in flight."""
    if engine != "renewal":
        raise ValueError(f"the B200 ensemble runs the renewal engine only (got {engine!r})")
    cfg = as_config(cfg)
    _device.device()
    b = cfg.steps_per_batch
    if lockstep and runs > 0:
        plan = _build_plan(g, m, cfg, bool(cfg.mixed_precision))
        torch.cuda.current_stream().synchronize()
        group = max(1, min(runs, (1 << 27) // max(1, g.num_nodes)))
        res = _run_lockstep(g, m, cfg, seed, t_final, runs, seed_count, seed_compartment, plan, group)
        if res is not None:
            return make_records([(t, c) for t, c, _ in res], m.compartments, g.num_nodes, t_final, grid_points,
                                [s for _, _, s in res])
    free = [torch.cuda.Stream() for _ in range(max(1, min(concurrency, runs)))]
    plan = _build_plan(g, m, cfg, bool(cfg.mixed_precision))  # one device copy of the graph for every trial
    out: list[tuple | None] = [None] * runs
    pending = list(range(runs))
    live: list[_Trial] = []
    torch.cuda.current_stream().synchronize()  # the graph upload precedes the trial streams
    while pending or live:
        while pending and free:
            tr = _Trial(pending.pop(0), g, m, cfg, seed, seed_count, seed_compartment, free.pop(), plan)
            tr.launch()  # pipelined: every live trial keeps one batch queued ahead of the one collected
            live.append(tr)
        for tr in live:
            tr.launch()
        still = []
        for tr in live:
            tr.collect(b, g.num_nodes)
            if tr.clock < t_final:
                still.append(tr)
            else:
                out[tr.trial] = tr.finish(t_final)
                free.append(tr.stream)
        live = still
    return make_records([(t, c) for t, c, _ in out], m.compartments, g.num_nodes, t_final, grid_points,
                        [s for _, _, s in out])
