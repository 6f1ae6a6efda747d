"""Node-partitioned renewal runs across GPUs.

The reference has no multi-GPU path (its only parallelism is the
ProcessPool of independent trajectories, R/analysis.py:97-130; the paper
lists multi-GPU as future work).  Here one process per GPU
owns a contiguous range of global node ids:

* rank r owns nodes [r*chunk, min(N, (r+1)*chunk)), chunk a multiple of 1024
  nodes, so its slice of the 1-bit infectious mask is the word range
  [r*chunk/32, (r+1)*chunk/32) — equal-size segments for an in-place
  all-gather;
* its CSR rows (global column ids) come from ``gen_fixed_degree_device(...,
  row_lo, row_hi)`` — no exchange is needed to build the graph;
* states / ages are local; the infectious mask is replicated;
* after every step the engine runs one NCCL group (count-delta all-reduce,
  max-rate all-reduce, mask all-gather) on its stream, inside the batch CUDA
  graph.

The RNG is keyed by the global node id (R/rng.py:5-7), the max and the
integer counts are order-free, so a partitioned run is bit-identical to the
single-GPU run of the same graph (tests/test_distributed.py).

``LocalPartitionedRun`` runs P partitions inside one process on one device
(shared mask buffers, accumulators combined by ``fs_engines_exchange_local``):
the same kernels and the same exchange semantics without the transport, so
the partitioned path is parity-tested on a single GPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .errors import InvalidConfigError
from .graph import resolve_strategy
from .models import model_descriptor
from .renewal import (
    _PRECISION,
    _STRATEGY_CODE,
    RenewalConfig,
    _check_conservation,
    as_config,
    _DeviceGraph,
    _node_buffer,
    _pick_seed_nodes,
    _storage,
    default_seed_count,
)
from .rng import RNG_KINDS
from .trajectory import DEFAULT_GRID_POINTS, make_record

__all__ = ["PartitionPlan", "partition_plan", "LocalPartitionedRun", "DistributedRun", "run_renewal_distributed"]

ALIGN = 1024  # nodes per alignment unit: 32 mask words = 128 B segments


@dataclass(frozen=True)
class PartitionPlan:
    num_nodes: int      # N of the whole graph
    world: int
    chunk: int          # nodes per rank (multiple of ALIGN); the last rank may own fewer
    ranges: tuple       # ((lo, hi), ...) per rank
    balanced: bool = False  # ranges cut at edge quantiles (unequal node counts)

    @property
    def bounds(self) -> np.ndarray:
        """world + 1 node boundaries of the ranges."""
        return np.array([lo for lo, _ in self.ranges] + [self.ranges[-1][1]], dtype=np.int64)

    @property
    def mask_segment_words(self) -> int:
        return self.chunk // 32

    @property
    def mask_words(self) -> int:
        """Words of each replicated mask buffer: every segment, the zero
        sentinel word past the last tile, rounded to 16 bytes."""
        w = max(self.world * self.mask_segment_words, (self.num_nodes + 31) // 32 + 1)
        return (w + 3) // 4 * 4


def partition_plan(num_nodes: int, world: int, align: int = ALIGN, row_offsets=None) -> PartitionPlan:
    """Contiguous node ranges, each a multiple of `align` nodes so no mask
    word straddles two ranks.  Equal node counts by default (the regular
    graphs of C4/C5 are edge-balanced by node count); with `row_offsets`
    (the incoming CSR's, global) the boundaries are cut at the edge
    quantiles instead, so the hubs of a scale-free graph do not
    load one rank — the partitioned engine then needs incremental counts."""
    if world < 1 or num_nodes < world:
        raise ValueError("need 1 <= world <= num_nodes")
    if align % 32:
        raise ValueError("align must be a multiple of 32")
    if row_offsets is not None and world > 1:
        ro = np.asarray(row_offsets, dtype=np.int64)
        if ro.size != num_nodes + 1:
            raise ValueError("row_offsets must have N + 1 entries")
        e = int(ro[-1])
        cuts = [0]
        for r in range(1, world):
            b = int(np.searchsorted(ro, (r * e) // world, side="left"))
            b = max(cuts[-1] + align, (b + align // 2) // align * align)
            cuts.append(min(b, num_nodes))
        cuts.append(num_nodes)
        ranges = tuple((cuts[r], cuts[r + 1]) for r in range(world))
        if any(hi <= lo for lo, hi in ranges):
            raise ValueError(f"N={num_nodes} too small for {world} edge-balanced ranks of {align}-node granularity")
        chunk = max(hi - lo for lo, hi in ranges)
        chunk = -(-chunk // align) * align
        return PartitionPlan(num_nodes, world, chunk, ranges, balanced=True)
    chunk = -(-num_nodes // world)
    chunk = -(-chunk // align) * align
    ranges = []
    for r in range(world):
        lo = min(num_nodes, r * chunk)
        hi = min(num_nodes, (r + 1) * chunk)
        ranges.append((lo, hi))
    if any(hi <= lo for lo, hi in ranges):
        raise ValueError(f"N={num_nodes} too small for {world} ranks of {align}-node granularity")
    return PartitionPlan(num_nodes, world, chunk, tuple(ranges))


def _config(cfg: RenewalConfig, strategy, incremental: int) -> _lib.FsConfig:
    cfg = as_config(cfg)
    return _lib.FsConfig(
        epsilon=cfg.epsilon, tau_max=cfg.tau_max, delta=cfg.delta, steps_per_batch=cfg.steps_per_batch,
        strategy=_STRATEGY_CODE[strategy], compaction=int(cfg.compaction), mixed_precision=int(cfg.mixed_precision),
        lanes_per_node=cfg.lanes_per_node, edges_per_block=cfg.edges_per_block, hazard_chunk=cfg.hazard_chunk,
        chunk_skip=int(cfg.chunk_skip), carry_tau=int(cfg.carry_tau), rng=RNG_KINDS[cfg.rng],
        hazard_precision=_PRECISION[cfg.hazard_precision], count_gather=1, incremental=incremental)


def _initial_mask(plan: PartitionPlan, seed_ids: torch.Tensor, infectious: bool, dev) -> torch.Tensor:
    m = torch.zeros(plan.mask_words, dtype=torch.int32, device=dev)
    if infectious and seed_ids.numel():
        words = (seed_ids >> 5).to(torch.int64)
        bits = torch.ones_like(seed_ids, dtype=torch.int64) << (seed_ids & 31).to(torch.int64)
        acc = torch.zeros(plan.mask_words, dtype=torch.int64, device=dev)
        acc.index_add_(0, words, bits)  # distinct ids: sums are disjoint ors
        m = torch.where(acc >= 2**31, acc - 2**32, acc).to(torch.int32)  # same 32-bit pattern
    return m


class _Partition:
    """One rank's engine: local rows, global mask buffers (owned or shared)."""

    def __init__(self, g_local, m, cfg: RenewalConfig, seed: int, plan: PartitionPlan, rank: int,
                 seed_ids: torch.Tensor, masks: list, comm, dev):
        cfg = as_config(cfg)
        if m.transmission.kind != "constant":
            raise InvalidConfigError("partitioned runs need constant transmission (count gather)")
        lo, hi = plan.ranges[rank]
        if g_local.num_nodes != hi - lo:
            raise ValueError(f"rank {rank}: graph slice has {g_local.num_nodes} rows, partition owns {hi - lo}")
        self.lib = _lib.load()
        self.lo, self.hi, self.rank = lo, hi, rank
        self.n = hi - lo
        self.M = m.num_compartments
        self.stream = _device.stream_handle(dev)
        mixed = bool(cfg.mixed_precision)
        st_t, at_t, _ = _storage(mixed)
        comp = m.edge_to
        self.states = _node_buffer(self.n, st_t, dev, int(m.edge_from))
        local = seed_ids[(seed_ids >= lo) & (seed_ids < hi)] - lo
        if local.numel():
            self.states[local] = comp
        self.ages = _node_buffer(self.n, at_t, dev)
        self.masks = masks
        self.dg = _DeviceGraph.from_device(g_local, dev) if hasattr(g_local, "device_tensors") else None
        if self.dg is None:
            from .renewal import device_graph

            self.dg = device_graph(g_local, mixed)
        strategy = resolve_strategy(g_local, cfg.strategy)
        counts = np.zeros(self.M, dtype=np.int64)
        counts[m.edge_from] = plan.num_nodes - seed_ids.numel()
        counts[comp] += seed_ids.numel()
        scal = _lib.FsScalars(clock=0.0, tau_next=cfg.tau_max, step=0, seed=seed & ((1 << 64) - 1),
                              last_max_rate=0.0, started=0)
        for i, c in enumerate(counts):
            scal.counts[i] = int(c)
        b = _lib.FsStateBuffers()
        b.states, b.ages = _lib.ptr(self.states), _lib.ptr(self.ages)
        b.imask[0], b.imask[1] = _lib.ptr(masks[0]), _lib.ptr(masks[1])
        b.padded = 2  # _node_buffer: whole 128-node units (the streaming step kernel)
        self._b = b
        self._bounds = plan.bounds if plan.balanced else None  # kept alive for the create call
        part = _lib.FsPartition(node_base=lo, num_nodes_global=plan.num_nodes,
                                mask_segment_words=plan.mask_segment_words, rank=rank, world=plan.world,
                                comm=comm,
                                range_bounds=self._bounds.ctypes.data if self._bounds is not None else None)
        h = ctypes.c_void_p()
        incr = {"auto": -1, "incremental": 1}.get(cfg.gather, 0) if self.dg.symmetric else 0
        _lib.check(self.lib.fs_engine_create_partitioned(self.dg.view(), model_descriptor(m),
                                                          _config(cfg, strategy, incr), b, scal, dev.index, part,
                                                          ctypes.byref(h)))
        self.handle = h
        bufs = (ctypes.c_void_p * 2)()
        self.incremental = self.lib.fs_engine_delta_buffers(self.handle, bufs) == 0
        self.delta_buffers = (bufs[0], bufs[1]) if self.incremental else None
        mb = ctypes.c_void_p()
        self.mailbox = mb.value if (plan.world > 1 and self.incremental and
                                    self.lib.fs_engine_mailbox(self.handle, ctypes.byref(mb), None) == 0) else None

    def link_peers(self, table) -> None:
        """table[parity][rank] = device address of that rank's delta buffer
        (own entries: this engine's buffers)."""
        world = len(table[0])
        arr = (ctypes.c_void_p * (2 * world))(*[table[par][r] for par in range(2) for r in range(world)])
        _lib.check(self.lib.fs_engine_set_peer_deltas(self.handle, arr))

    def link_mailboxes(self, table) -> None:
        """table[rank] = device address of that rank's mailbox: the bulk
        exchange of remote pushes."""
        arr = (ctypes.c_void_p * len(table))(*table)
        _lib.check(self.lib.fs_engine_set_peer_mailboxes(self.handle, arr))

    def apply_mailbox(self) -> None:
        _lib.check(self.lib.fs_engine_apply_mailbox(self.handle, self.stream))

    def sync_ages(self) -> None:
        """The uniform S age back into `ages` (the engine keeps it as one
        scalar while every S node shares it): call before
        reading `ages`."""
        _lib.check(self.lib.fs_engine_sync_ages(self.handle, self.stream))

    def close(self) -> None:
        if getattr(self, "handle", None):
            if torch is not None and torch.cuda is not None:  # (interpreter teardown)
                torch.cuda.current_stream().synchronize()
            self.lib.fs_engine_destroy(self.handle)
            self.handle = None

    __del__ = close

    def step(self, nsteps: int = 1) -> None:
        _lib.check(self.lib.fs_engine_step(self.handle, nsteps, 0, 0, self.stream))

    def run_batch(self) -> None:
        _lib.check(self.lib.fs_engine_run_batch(self.handle, 0, self.stream))

    def scalars(self) -> _lib.FsScalars:
        s = _lib.FsScalars()
        _lib.check(self.lib.fs_engine_get_scalars(self.handle, ctypes.byref(s), self.stream))
        return s

    def remote_pushes(self, first: int, n: int) -> np.ndarray:
        """Per-step count of the pushes this rank sent to other ranks."""
        out = np.zeros(n, dtype=np.uint32)
        _lib.check(self.lib.fs_engine_read_remote_pushes(self.handle, first, n, out.ctypes.data, self.stream))
        return out

    def read_log(self, first: int, n: int):
        clocks = np.empty(n, dtype=np.float64)
        taus = np.empty(n, dtype=np.float64)
        counts = np.empty((n, self.M), dtype=np.int64)
        _lib.check(self.lib.fs_engine_read_log(self.handle, first, n, clocks.ctypes.data, taus.ctypes.data,
                                               counts.ctypes.data, self.stream))
        return clocks, taus, counts


def _seed_ids(m, num_nodes: int, seed: int, seed_count, dev) -> torch.Tensor:
    count = default_seed_count(num_nodes) if seed_count is None else int(seed_count)
    return _pick_seed_nodes(num_nodes, seed, count, dev)  # the same global choice on every rank


class LocalPartitionedRun:
    """P partitions of one graph on one device, stepped in lockstep with the
    exchange done in place (shared mask buffers + fs_engines_exchange_local).
    `graph_parts[r]` holds rows plan.ranges[r] with global column ids."""

    def __init__(self, graph_parts, m, cfg: RenewalConfig, seed: int, plan: PartitionPlan, seed_count=None,
                 exchange: str = "bulk"):
        """exchange "bulk": pushes to other partitions staged and written to
        their mailboxes in bulk; "atomic": one peer atomic per push."""
        if exchange not in ("bulk", "atomic"):
            raise ValueError("exchange must be 'bulk' or 'atomic'")
        dev = _device.device()
        self.plan, self.cfg, self.M = plan, cfg, m.num_compartments
        ids = _seed_ids(m, plan.num_nodes, seed, seed_count, dev)
        mask0 = _initial_mask(plan, ids, m.edge_to == m.infectious, dev)
        self.masks = [mask0, mask0.clone()]
        self.parts = [_Partition(graph_parts[r], m, cfg, seed, plan, r, ids, self.masks, None, dev)
                      for r in range(plan.world)]
        if plan.world > 1 and self.parts[0].incremental:
            table = [[p.delta_buffers[par] for p in self.parts] for par in range(2)]
            for p in self.parts:
                p.link_peers(table)
            if exchange == "bulk":
                boxes = [p.mailbox for p in self.parts]
                for p in self.parts:
                    p.link_mailboxes(boxes)
        self._arr = (ctypes.c_void_p * len(self.parts))(*[p.handle.value for p in self.parts])
        self.steps = 0

    def step(self) -> None:
        for p in self.parts:
            p.step(1)
        _lib.check(_lib.load().fs_engines_exchange_local(self._arr, len(self.parts), self.parts[0].stream))
        self.steps += 1

    def run_batch(self):
        first = self.steps
        for _ in range(self.cfg.steps_per_batch):
            self.step()
        return self.parts[0].read_log(first, self.cfg.steps_per_batch)

    def gather(self) -> dict:
        """Whole-graph states / ages (concatenated partitions) and scalars."""
        for p in self.parts:
            p.sync_ages()
        s = self.parts[0].scalars()
        return {"states": torch.cat([p.states for p in self.parts]).cpu().numpy(),
                "ages": torch.cat([p.ages for p in self.parts]).cpu().numpy(),
                "counts": np.array(s.counts[: self.M], dtype=np.int64), "clock": s.clock, "tau_prev": s.tau_next,
                "step": s.step, "scalars": [p.scalars() for p in self.parts]}

    def close(self) -> None:
        for p in self.parts:
            p.close()


class DistributedRun:
    """This rank's share of a node-partitioned run over NCCL (one process per
    GPU).  `graph_local` holds the rows of plan.ranges[rank]; `pg` is the
    torch.distributed group used once, to broadcast the NCCL unique id."""

    def __init__(self, graph_local, m, cfg: RenewalConfig, seed: int, plan: PartitionPlan, rank: int,
                 seed_count=None, pg=None, transport: str = "nccl", exchange: str = "bulk"):
        """transport "nccl": the per-step all-reduce is an NCCL group inside
        the engine's launches (and CUDA graphs); "host": eager steps only, the
        accumulator is all-reduced through `pg` (any torch.distributed
        backend) — lets several processes share one GPU in tests."""
        import torch.distributed as dist

        dev = _device.device()
        lib = _lib.load()
        self.plan, self.cfg, self.M, self.rank = plan, cfg, m.num_compartments, rank
        self.transport, self.pg = transport, pg
        comm = ctypes.c_void_p()
        if transport == "nccl":
            buf = (ctypes.c_uint8 * 256)()
            if rank == 0:
                nb = _lib.check(lib.fs_comm_unique_id(buf, 256))
                payload = [bytes(buf)[:nb]]
            else:
                payload = [None]
            if plan.world > 1:
                dist.broadcast_object_list(payload, src=0, group=pg)
            idb = (ctypes.c_uint8 * 256).from_buffer_copy(payload[0].ljust(256, b"\0"))
            _lib.check(lib.fs_comm_init(plan.world, rank, idb, dev.index, ctypes.byref(comm)))
        elif transport != "host":
            raise ValueError("transport must be 'nccl' or 'host'")
        self.comm = comm
        ids = _seed_ids(m, plan.num_nodes, seed, seed_count, dev)
        mask0 = _initial_mask(plan, ids, m.edge_to == m.infectious, dev)
        self.masks = [mask0, mask0.clone()]
        self.part = _Partition(graph_local, m, cfg, seed, plan, rank, ids, self.masks, comm.value or None, dev)
        self.steps = 0
        self._opened = []
        if transport == "host" and plan.world > 1 and not self.part.incremental:
            raise InvalidConfigError("the host transport needs the incremental-count mode (no mask exchange)")
        if exchange not in ("bulk", "atomic"):
            raise ValueError("exchange must be 'bulk' or 'atomic'")
        self.exchange = exchange
        if plan.world > 1 and self.part.incremental:
            self._link_peers_ipc(dev, pg)

    def _link_peers_ipc(self, dev, pg) -> None:
        """Map every rank's pending-delta buffers into this process (CUDA IPC
        over NVLink) so the step kernel can push into them directly."""
        import torch.distributed as dist

        lib = _lib.load()
        mine = []
        bulk = self.exchange == "bulk" and self.part.mailbox is not None
        for ptr in list(self.part.delta_buffers) + ([self.part.mailbox] if bulk else []):
            h = (ctypes.c_uint8 * 128)()
            nb = _lib.check(lib.fs_ipc_get_handle(ptr, h, 128))
            mine.append(bytes(h)[:nb])
        allh = [None] * self.plan.world
        dist.all_gather_object(allh, mine, group=pg)
        table = [[None] * self.plan.world for _ in range(2)]
        for r in range(self.plan.world):
            for par in range(2):
                if r == self.rank:
                    table[par][r] = self.part.delta_buffers[par]
                    continue
                buf = (ctypes.c_uint8 * 128).from_buffer_copy(allh[r][par].ljust(128, b"\0"))
                out = ctypes.c_void_p()
                _lib.check(lib.fs_ipc_open_handle(buf, dev.index, ctypes.byref(out)))
                self._opened.append(out)
                table[par][r] = out.value
        self.part.link_peers(table)
        if bulk:  # every rank's mailbox, for the bulk exchange
            boxes = [None] * self.plan.world
            for r in range(self.plan.world):
                if r == self.rank:
                    boxes[r] = self.part.mailbox
                    continue
                buf = (ctypes.c_uint8 * 128).from_buffer_copy(allh[r][2].ljust(128, b"\0"))
                out = ctypes.c_void_p()
                _lib.check(lib.fs_ipc_open_handle(buf, dev.index, ctypes.byref(out)))
                self._opened.append(out)
                boxes[r] = out.value
            self.part.link_mailboxes(boxes)
        dist.barrier(group=pg)  # every rank linked before anyone pushes

    def exchange_us(self, iters: int = 200) -> float | None:
        """Mean device time of one per-step NCCL exchange on this rank's
        stream (the count / max all-reduce group, plus the mask all-gather
        when the engine exchanges the mask)."""
        if not self.comm.value:
            return None
        us = ctypes.c_float()
        seg = 0 if self.part.incremental else self.plan.mask_segment_words
        _lib.check(_lib.load().fs_comm_time_exchange(self.comm, self.rank, seg, iters, self.part.stream,
                                                     ctypes.byref(us)))
        return float(us.value)

    def run_batch(self):
        first = self.steps
        if self.transport == "host":
            self.step(self.cfg.steps_per_batch)
        else:
            self.part.run_batch()
            self.steps += self.cfg.steps_per_batch
        return self.part.read_log(first, self.cfg.steps_per_batch)

    def step(self, nsteps: int = 1) -> None:
        if self.transport == "nccl":
            self.part.step(nsteps)
            self.steps += nsteps
            return
        import torch.distributed as dist

        lib = _lib.load()
        acc = np.zeros(17, dtype=np.uint64)
        for _ in range(nsteps):
            self.part.step(1)
            _lib.check(lib.fs_engine_acc_get(self.part.handle, acc.ctypes.data, self.part.stream))
            d = torch.from_numpy(acc[:16].view(np.int64).copy())
            mx = torch.tensor([int(acc[16])], dtype=torch.int64)
            dist.all_reduce(d, op=dist.ReduceOp.SUM, group=self.pg)  # two's complement sums
            dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=self.pg)  # rates >= 0: bits order like values
            acc[:16] = d.numpy().view(np.uint64)
            acc[16] = np.uint64(mx.item())
            _lib.check(lib.fs_engine_acc_set(self.part.handle, acc.ctypes.data, self.part.stream))
            self.part.apply_mailbox()  # after every rank's step (the all-reduce above is the barrier)
            self.steps += 1

    def close(self) -> None:
        lib = _lib.load()
        for h in getattr(self, "_opened", []):
            lib.fs_ipc_close(h)
        self._opened = []
        self.part.close()
        if getattr(self, "comm", None) and self.comm.value:
            _lib.load().fs_comm_destroy(self.comm)
            self.comm = None


def run_renewal_distributed(graph_local, m, cfg: RenewalConfig, seed: int, t_final: float, plan: PartitionPlan,
                            rank: int, grid_points: int = DEFAULT_GRID_POINTS, seed_count=None, pg=None):
    """`run_renewal` (R/renewal.py:632-663) over a node partition: whole
    batches until clock >= t_final.  Every rank returns the same record
    (clock and counts are global after each step's exchange)."""
    import time

    t0 = time.perf_counter()
    run = DistributedRun(graph_local, m, cfg, seed, plan, rank, seed_count=seed_count, pg=pg)
    s = run.part.scalars()
    times, rows = [0.0], [np.array(s.counts[: run.M], dtype=np.int64)]
    clock, done = 0.0, 0
    while clock < t_final:
        clocks, _, counts = run.run_batch()
        _check_conservation(counts, plan.num_nodes)
        times.extend(clocks.tolist())
        rows.extend(counts)
        done += cfg.steps_per_batch
        clock = float(clocks[-1])
    wall = time.perf_counter() - t0
    t_arr = np.asarray(times)
    steps = min(int(np.searchsorted(t_arr, t_final, side="left")), done)
    rec = make_record(t_arr, np.asarray(rows), m.compartments, plan.num_nodes, t_final, grid_points,
                      extra_summary={"step_count": steps, "wall_clock": wall, "engine": "renewal-partitioned",
                                     "world": plan.world})
    run.close()
    return rec
