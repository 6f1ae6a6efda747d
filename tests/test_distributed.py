"""Node-partitioned runs (paper_2604_22092_b200.distributed).

CPU (gloo, world size 2): the partition plan, and the partitioned algorithm
itself — the oracle stepped on each rank's rows with the per-step exchange
(infectivity all-gather, max / count all-reduce) done by torch.distributed —
reproduces the single-process oracle bit for bit.  GPU: P virtual ranks on
one device (the partitioned kernels, shared mask buffers, in-place exchange)
and a world-1 NCCL run both reproduce the single-engine trajectory.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200.distributed import partition_plan


def test_partition_plan_properties():
    for n, world in [(10_000, 2), (1_000_000, 8), (1_000_000_000, 8), (5000, 3), (4096, 4)]:
        p = partition_plan(n, world)
        assert p.ranges[0][0] == 0 and p.ranges[-1][1] == n
        for (lo, hi), (lo2, _) in zip(p.ranges[:-1], p.ranges[1:]):
            assert hi == lo2 and lo % 1024 == 0 and (hi - lo) == p.chunk
        assert p.chunk % 1024 == 0 and p.mask_segment_words * 32 == p.chunk
        assert p.mask_words >= world * p.mask_segment_words and p.mask_words >= (n + 31) // 32 + 1
        assert p.mask_words % 4 == 0
    with pytest.raises(ValueError):
        partition_plan(2048, 3)  # third rank would be empty


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _partitioned_oracle_worker(rank: int, world: int, port: int, steps: int, out_q) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import spreadsim_port as O

    g = fs.gen_fixed_degree(6000, 10, seed=4)
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig()
    seed = 7
    plan = partition_plan(g.num_nodes, world)
    lo, hi = plan.ranges[rank]
    full = O.init_state(g, m, cfg, seed)  # every rank derives the same global seeds
    states, ages = full.states[lo:hi].copy(), full.ages[lo:hi].copy()
    ro = g.row_offsets[lo:hi + 1] - g.row_offsets[lo]
    col = g.col_indices[g.row_offsets[lo]:g.row_offsets[hi]]
    inf = full.infectivity.astype(np.float32)
    counts = full.counts.copy()
    tau, clock = cfg.tau_max, 0.0
    for k in range(steps):
        clock += tau
        states, ages, inf_loc, mx, delta = O.step_rows(states, ages, ro, col, inf, lo, tau, k, m, seed, False)
        # the exchange: infectivity segments all-gathered, max and deltas all-reduced
        pad = np.zeros(plan.chunk, dtype=np.float32)
        pad[: hi - lo] = inf_loc
        parts = [torch.zeros(plan.chunk) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(pad))
        inf = torch.cat(parts).numpy()[: g.num_nodes]
        t = torch.tensor([mx], dtype=torch.float32)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        d = torch.from_numpy(delta)
        dist.all_reduce(d, op=dist.ReduceOp.SUM)
        counts = counts + d.numpy()
        tau = min(cfg.tau_max, cfg.epsilon / (float(t.item()) + cfg.delta))
    out_q.put((rank, states, ages, counts, clock, tau))
    dist.destroy_process_group()


def test_partitioned_oracle_matches_single_process_gloo():
    from oracle import spreadsim_port as O

    steps, world = 60, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_partitioned_oracle_worker, args=(r, world, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = fs.gen_fixed_degree(6000, 10, seed=4)
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig()
    ref = O.init_state(g, m, cfg, 7)
    for _ in range(steps):
        O.step(ref, g, m, cfg, 7)
    states = np.concatenate([res[r][0] for r in range(world)])
    ages = np.concatenate([res[r][1] for r in range(world)])
    assert np.array_equal(states, ref.states)
    assert np.array_equal(ages.view(np.uint32), ref.ages.view(np.uint32))
    for r in range(world):
        assert np.array_equal(res[r][2], ref.counts)
        assert res[r][3] == ref.clock and res[r][4] == ref.tau_prev


@pytest.mark.gpu
@pytest.mark.parametrize("world,mixed,exchange,cap", [
    (3, False, "bulk", None), (2, True, "bulk", None), (4, False, "bulk", None),
    (3, False, "atomic", None),
    (4, False, "bulk", "8"),  # mailboxes overflow every step: the rest goes as direct peer atomics
])
def test_virtual_ranks_match_single_engine(world, mixed, exchange, cap, monkeypatch):
    """P partitions on one device, pushes to other partitions through their
    mailboxes (bulk) or as direct peer atomics: bit-identical to one engine."""
    from paper_2604_22092_b200.distributed import LocalPartitionedRun

    if cap:
        monkeypatch.setenv("FS_MBOX_CAP", cap)
    n, k = 50_000, 10
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig(mixed_precision=mixed)
    plan = partition_plan(n, world)
    whole = fs.gen_fixed_degree_device(n, k, seed=2)
    parts = [fs.gen_fixed_degree_device(n, k, seed=2, row_lo=lo, row_hi=hi) for lo, hi in plan.ranges]
    run = LocalPartitionedRun(parts, m, cfg, 7, plan, exchange=exchange)
    st = fs.init_renewal_state(whole, m, cfg, 7)
    for _ in range(3):
        clocks, _, counts = run.run_batch()
        rec = []
        fs.run_batch(st, whole, m, cfg, 7, recorder=rec)
        assert np.array_equal(counts, np.array([c for _, c in rec]))
        assert np.array_equal(clocks, np.array([t for t, _ in rec]))
    got = run.gather()
    assert np.array_equal(got["states"].astype(np.int32), st.states.astype(np.int32))
    assert np.array_equal(got["ages"].view(np.uint16 if mixed else np.uint32),
                          st.ages.view(np.uint16 if mixed else np.uint32))
    assert np.array_equal(got["counts"], st.counts)
    assert got["clock"] == st.clock and got["tau_prev"] == st.tau_prev
    run.close()


def _nccl_world1_worker(port: int, out_q) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    from paper_2604_22092_b200.distributed import run_renewal_distributed

    n = 40_000
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig()
    plan = partition_plan(n, 1)
    g = fs.gen_fixed_degree_device(n, 10, seed=3)
    rec = run_renewal_distributed(g, m, cfg, 7, 20.0, plan, 0)
    ref = fs.run_renewal(g, m, cfg, 7, 20.0)
    out_q.put((np.array_equal(rec.fractions, ref.fractions), rec.summary["step_count"], ref.summary["step_count"]))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_world1_matches_single_engine():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1_worker, args=(_free_port(), q))
    p.start()
    same, s1, s2 = q.get(timeout=600)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert same and s1 == s2


def _ipc_worker(rank: int, world: int, port: int, steps: int, out_q, exchange: str = "bulk") -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2604_22092_b200.distributed import DistributedRun

    n = 30_000
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    plan = partition_plan(n, world)
    lo, hi = plan.ranges[rank]
    g = fs.gen_fixed_degree_device(n, 10, seed=2, row_lo=lo, row_hi=hi)
    run = DistributedRun(g, m, fs.RenewalConfig(), 7, plan, rank, transport="host", exchange=exchange)
    assert run.part.incremental
    run.step(steps)
    s = run.part.scalars()
    run.part.sync_ages()
    out_q.put((rank, run.part.states.cpu().numpy(), run.part.ages.cpu().numpy(),
               np.array(s.counts[:4], dtype=np.int64), s.clock))
    dist.barrier()
    run.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["bulk", "atomic"])
def test_two_processes_push_through_cuda_ipc(exchange):
    """Two ranks as two processes on the one GPU: the step kernels push into
    each other's pending-delta arrays through CUDA IPC mappings (the
    multi-GPU path's transport, minus NVLink), the accumulator is all-reduced
    over gloo; the result equals the single-engine run bit for bit."""
    steps, world = 60, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, steps, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=600) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 30_000
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig()
    whole = fs.gen_fixed_degree_device(n, 10, seed=2)
    st = fs.init_renewal_state(whole, m, cfg, 7)
    for _ in range(steps):
        fs.renewal_step(st, whole, m, cfg, 7)
    assert np.array_equal(np.concatenate([res[r][0] for r in range(world)]), st.states)
    assert np.array_equal(np.concatenate([res[r][1] for r in range(world)]).view(np.uint32), st.ages.view(np.uint32))
    for r in range(world):
        assert np.array_equal(res[r][2], st.counts) and res[r][3] == st.clock


def test_edge_balanced_partition_plan():
    g = fs.gen_barabasi_albert(20_000, 5, seed=3)
    for world in (2, 3, 4):
        p = partition_plan(g.num_nodes, world, row_offsets=g.row_offsets)
        assert p.balanced and p.ranges[0][0] == 0 and p.ranges[-1][1] == g.num_nodes
        assert all(lo % 1024 == 0 and lo < hi for lo, hi in p.ranges)
        assert all(p.ranges[r][1] == p.ranges[r + 1][0] for r in range(world - 1))
        e = [int(g.row_offsets[hi] - g.row_offsets[lo]) for lo, hi in p.ranges]
        # within one alignment unit's worth of edges of the even split
        assert max(e) - min(e) <= 2 * 1024 * 40, e
        eq = partition_plan(g.num_nodes, world)
        e_eq = [int(g.row_offsets[hi] - g.row_offsets[lo]) for lo, hi in eq.ranges]
        assert max(e) - min(e) < max(e_eq) - min(e_eq)  # hubs are the low ids: equal node ranges are skewed
    assert not partition_plan(g.num_nodes, 2).balanced


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_edge_balanced_virtual_ranks_match_single_engine(world):
    """Unequal (edge-balanced) node ranges of a Barabasi-Albert graph: the
    pushes find their owner by range boundaries; bit-identical to one engine,
    and the per-step remote-push counters see the cross-rank traffic."""
    from paper_2604_22092_b200.distributed import LocalPartitionedRun

    g = fs.gen_barabasi_albert(30_000, 5, seed=4)
    m = fs.seir_weibull_erlang(0.25)
    cfg = fs.RenewalConfig()
    plan = partition_plan(g.num_nodes, world, row_offsets=g.row_offsets)
    parts = []
    for lo, hi in plan.ranges:
        ro = g.row_offsets[lo:hi + 1] - g.row_offsets[lo]
        col = g.col_indices[g.row_offsets[lo]:g.row_offsets[hi]]
        parts.append(fs.CsrGraph(hi - lo, int(ro[-1]), ro, col, np.ones(col.size, np.float32)))
    # a row slice of an undirected graph: its out-rows are its in-rows (global ids)
    for p in parts:
        p.__dict__["_fs_symmetric"] = True
    run = LocalPartitionedRun(parts, m, cfg, 7, plan)
    assert run.parts[0].incremental
    st = fs.init_renewal_state(g, m, cfg, 7)
    for _ in range(3):
        clocks, _, counts = run.run_batch()
        rec = []
        fs.run_batch(st, g, m, cfg, 7, recorder=rec)
        assert np.array_equal(counts, np.array([c for _, c in rec]))
    got = run.gather()
    assert np.array_equal(got["states"].astype(np.int32), st.states.astype(np.int32))
    assert np.array_equal(got["ages"].view(np.uint32), st.ages.view(np.uint32))
    remote = sum(int(p.remote_pushes(run.steps - 150, 150).sum()) for p in run.parts)
    assert remote > 0
    run.close()


@pytest.mark.gpu
@pytest.mark.slow
def test_virtual_ranks_at_1e7():
    """SURVEY §8e at scale: 4 virtual ranks over a 1e7-node uniform-degree
    graph, bit-identical to one engine over 100 steps."""
    from paper_2604_22092_b200.distributed import LocalPartitionedRun

    n, k, world = 10_000_000, 10, 4
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    cfg = fs.RenewalConfig()
    plan = partition_plan(n, world)
    parts = [fs.gen_fixed_degree_device(n, k, seed=5, row_lo=lo, row_hi=hi) for lo, hi in plan.ranges]
    run = LocalPartitionedRun(parts, m, cfg, 7, plan)
    for _ in range(2):
        clocks, _, counts = run.run_batch()
    got = run.gather()
    remote = [int(p.remote_pushes(run.steps - 100, 100).sum()) for p in run.parts]
    run.close()
    del parts, run
    whole = fs.gen_fixed_degree_device(n, k, seed=5)
    st = fs.init_renewal_state(whole, m, cfg, 7)
    rec = []
    for _ in range(2):
        fs.run_batch(st, whole, m, cfg, 7, recorder=rec)
    assert np.array_equal(counts, np.array([c for _, c in rec[-50:]]))
    assert np.array_equal(got["states"].astype(np.int32), st.states.astype(np.int32))
    assert np.array_equal(got["ages"].view(np.uint32), st.ages.view(np.uint32))
    assert got["clock"] == st.clock
    # with random edges ~3/4 of the pushes of a status change cross ranks
    assert min(remote) > 0
