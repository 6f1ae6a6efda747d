#!/usr/bin/env python
"""Throughput of the fused renewal tau-leap (BASELINE.json metric: Giga-NUPS).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c1]
  python bench.py --impl reference ...      # the reference path on the host CPU

A "step" is one synchronous tau-leap over every node of the workload graph.
Default workload = BASELINE config C2 (configs[1]): SEIR with log-normal
holding times on a uniform-degree (k=10) random graph, N = 1e6, fp32
storage, CUDA-graph-capturable engine.  Synthetic inputs: the reference's
own generator with graph seed 1, simulation seed 7.

value     device NUPS: K single steps, each bracketed by CUDA events on the
          launch stream, with L2 flushed (a 512 MiB write) before every step
          so the graph/state stream from HBM; max over ranks.
e2e       the public API end to end: run_renewal() from a host CsrGraph —
          CSR upload, device init, CUDA-graph batches to t_final, per-batch
          log download, trajectory record — NUPS = N * steps / wall
          (the reference's `spreadsim bench` definition, cli.py:563-573).
roofline  B_alg = 112 B per node-update (fp32 reference layout)
          x N / mean step time, against MEASURED_PEAKS.json hbm_gbs.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

B_ALG = {False: 112.0, True: 78.0}  # bytes per node-update, fp32 / mixed
WORKLOADS = {
    "c1": dict(desc="C1: SEIR log-normal, uniform-degree k=10, N=1e4", kind="fixed", n=10_000, k=10, model="seir"),
    "c2": dict(desc="C2: SEIR log-normal, uniform-degree k=10, N=1e6, CUDA graph", kind="fixed", n=1_000_000, k=10,
               model="seir"),
    "c3": dict(desc="C3: SEIR Weibull/Erlang, Barabasi-Albert m=5, N=1e6 (rho 421.7: merge strategy selected)",
               kind="ba", n=1_000_000, k=5, model="seir_we"),
    # the real gather paths: every step folds the CSR
    "c2s": dict(desc="C2 with age-dependent shedding s(tau) = lognormal hazard (IR): SEIR log-normal, uniform-degree "
                     "k=10, N=1e6 — f32 CSR-order fold of beta*s(age) every step",
                kind="fixed", n=1_000_000, k=10, model="seir_shed"),
    "c3f": dict(desc="C3 graph and model, gather='f32': edge-merge f32 fold of the CSR every step (EDGE_MERGE)",
                kind="ba", n=1_000_000, k=5, model="seir_we", gather="f32"),
    "c3c": dict(desc="C3 graph and model, gather='count': 1-bit infectious-mask gather of the CSR every step "
                     "(EDGE_MERGE)", kind="ba", n=1_000_000, k=5, model="seir_we", gather="count"),
    "c5": dict(desc="C5: SEIR log-normal, uniform-degree k=10, N=1e9, node-partitioned across the GPUs "
                    "(cross-rank pushes to peer mailboxes over NVLink + one 17-word NCCL all-reduce per step)",
               kind="regular_dev", n=1_000_000_000, k=10, model="seir", cpu_n=10_000_000, t_final=10.0),
    "m2": dict(desc="M2 (SURVEY §8f row 3): Markovian SIR (beta 0.25, gamma 0.15), uniform-degree k=10, N=1e6",
               kind="fixed", n=1_000_000, k=10, model="sir_markov", engine="markov"),
    "c2w": dict(desc="C2 per GPU, weak scaling: SEIR log-normal, uniform-degree k=10, N=1e6 nodes per GPU, "
                     "node-partitioned (peer pushes + NCCL all-reduce per step)",
                kind="regular_dev", n=1_000_000, k=10, model="seir", per_gpu=True),
    # the reference's acceptance ensemble (T/test_acceptance.py:34-79)
    "ens": dict(desc="ensemble: run_ensemble('renewal', ER N=1000 d=8 seed 20250809, SEIR log-normal, 100 runs, "
                     "10 E seeds, t_final=50) — R/analysis.py:97-130",
                kind="er", n=1000, k=8.0, model="seir", ensemble=dict(runs=100, seed=20250809, t_final=50.0,
                                                                      seed_count=10)),
    "c4": dict(desc="C4: SEIR log-normal, uniform-degree k=10, N=1e8, bf16/fp16 mixed-precision storage",
               kind="regular_dev", n=100_000_000, k=10, model="seir", mixed=True, cpu_n=10_000_000),
}
GRAPH_SEED, SIM_SEED = 1, 7


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def build_inputs(w):
    import paper_2604_22092_b200 as fs

    if w["kind"] == "fixed":
        g = fs.gen_fixed_degree(w["n"], w["k"], seed=GRAPH_SEED)
    elif w["kind"] == "er":
        g = fs.gen_erdos_renyi(w["n"], w["k"], seed=w["ensemble"]["seed"])
    elif w["kind"] == "regular_dev":  # GPU generator (the CPU one does not scale to 1e8)
        g = fs.gen_fixed_degree_device(w["n"], w["k"], seed=GRAPH_SEED)
    else:
        g = fs.gen_barabasi_albert(w["n"], w["k"], seed=GRAPH_SEED)
    if w["model"] == "seir":
        m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    elif w["model"] == "seir_shed":
        ir = fs.lognormal_from_mean_median(7.5, 5.0)
        m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0, transmission=fs.Shedding.lognormal_hazard(ir))
    elif w["model"] == "sir_markov":
        m = fs.sir_model(0.25, 0.15)
    else:
        m = fs.seir_weibull_erlang(0.25)
    return g, m


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,clocks.mem,power.draw,"
         "power.limit,temperature.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        extra = {"mem_mhz": [], "power_w": [], "power_limit_w": [], "temp_c": []}
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            for key, v in zip(extra, parts[6:10]):
                try:
                    extra[key].append(float(v))
                except ValueError:
                    pass
        # memory clock / power / temperature: the box-to-box spread of the
        # HBM-bound numbers shows up here, not in the SM clock
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
               "samples": len(sm)}
        for key, vals in extra.items():
            out[key] = (max(vals) if key == "power_w" else statistics.median(vals)) if vals else None
        return out


def roofline_block(achieved: float, pk: dict, ncu: dict, ms_per_step: float, b_alg: float) -> dict:
    """`achieved` counts the reference layout's B_alg bytes per node-update
     over the measured step time.  The physical picture comes
    from the dominant kernel's ncu capture (profiles/ncu_summary.json):
    `traffic` = its DRAM bytes per launch, `frac_physical` = those bytes over
    its ncu duration against the same peak, and `traffic_frac` the same bytes
    over this run's step time.  `ncu_same_build` says whether the capture ran
    the library this run loaded.  The encodings move fewer
    bytes than B_alg, which is why frac can exceed 1 while the physical
    fractions cannot."""
    traffic = ncu.get("dram_bytes_per_launch")
    out = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
           "traffic": traffic, "bytes_per_update": b_alg, "peak_source": pk["source"]}
    if traffic:
        out["traffic_gbs"] = traffic / (ms_per_step / 1e3) / 1e9
        out["traffic_frac"] = out["traffic_gbs"] / pk["hbm_gbs"]
        if ncu.get("gpu_time_us"):
            out["frac_physical"] = traffic / (ncu["gpu_time_us"] * 1e-6) / 1e9 / pk["hbm_gbs"]
            out["ncu_kernel"] = ncu.get("kernel")
            out["ncu_gpu_time_us"] = ncu["gpu_time_us"]
        out["ncu_same_build"] = ncu.get("lib_sha16") is not None and ncu.get("lib_sha16") == lib_sha16()
    return out


def lib_sha16() -> str | None:
    import hashlib

    p = ROOT / "paper_2604_22092_b200" / "libflashspread_b200.so"
    return hashlib.sha256(p.read_bytes()).hexdigest()[:16] if p.exists() else None


def ncu_entry(workload: str) -> dict:
    """The dominant kernel's ncu capture for this workload
    (profiles/ncu_summary.json, written by scripts/ncu_to_summary.py from a
    `ncu --set full` run of `bench.py --workload W`): DRAM bytes and duration
    per launch, and the sha of the library the capture ran."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return {}
    return json.loads(p.read_text()).get(workload, {})


def workload_config(w: dict, n: int, world: int = 1) -> dict:
    """`config` of both arms (same keys and values: the workload, not the
    implementation; the edge count and the CPU sample size are reported
    beside it)."""
    return {"workload": w["desc"], "n": n, "graph_seed": GRAPH_SEED, "sim_seed": SIM_SEED,
            "precision": "mixed (states i8, ages f16, infectivity bf16)" if w.get("mixed") else "fp32 storage",
            "gather_option": w.get("gather", "auto"),
            "l2": ("inputs larger than L2; steps timed back to back as CUDA-graph batches"
                   if world > 1 and not w.get("per_gpu") else
                   "flushed before every timed step (512 MiB write + 512 MiB read of another buffer)")}


def dtype_of(w: dict) -> str:
    return "i8/f16/bf16 storage, f32 rates, f64 hazard/q" if w.get("mixed") else "f32 (f64 hazard/q)"


def data_of(w: dict) -> str:
    if w["kind"] == "regular_dev":
        return "synthetic (GPU uniform-degree generator fs_gen_regular, graph seed 1, sim seed 7)"
    if w.get("ensemble"):
        return f"synthetic (reference generator gen_erdos_renyi, seed {w['ensemble']['seed']}; trial seeds derive_seed)"
    return "synthetic (reference generators, graph seed 1, sim seed 7)"


def port_vs_reference() -> dict | None:
    """Per-core speed of the oracle port against the reference's own
    renewal_step on the same C2 graph, measured in the build container where
    the reference is importable (scripts/port_vs_reference.py)."""
    p = ROOT / "profiles" / "port_vs_reference.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())["c2"]
    return {"port_mnups_per_core": round(d["port_mnups_per_core"], 3),
            "reference_mnups_per_core": round(d["reference_mnups_per_core"], 3),
            "port_over_reference_time": round(d["port_over_reference_time"], 3),
            "where": "build container, 1 thread each, C2 graph, states checked equal (profiles/port_vs_reference.json)"}


def _cpu_worker(args):
    """One trajectory of the oracle port (numpy restatement of the
    reference's renewal_step) on the shared graph: `warm` untimed steps, then
    `steps` timed ones.  Runs in a forked worker (the graph is inherited)."""
    trial, warm, steps = args
    import paper_2604_22092_b200 as fs
    from oracle import spreadsim_port as O

    g, m, cfg = _CPU_INPUTS
    seed = O.derive_seed(SIM_SEED, trial)  # run_ensemble's per-trial seed (analysis.py:61-74)
    st = O.init_state(g, m, cfg, seed)
    for _ in range(warm):
        O.step(st, g, m, cfg, seed)
    t0 = time.perf_counter()
    for _ in range(steps):
        O.step(st, g, m, cfg, seed)
    return time.perf_counter() - t0


_CPU_INPUTS = None


def cpu_ensemble(g, m, warm: int, steps: int, workers: int | None = None, mixed: bool = False) -> dict:
    """The reference's multi-core mode: independent trajectories in a process
    pool, one per host core (analysis.py:97-130 `run_ensemble`), each stepping
    the same graph.  Aggregate NUPS = workers * N * steps / slowest worker."""
    import multiprocessing as mp

    global _CPU_INPUTS
    import paper_2604_22092_b200 as fs

    _CPU_INPUTS = (g, m, fs.RenewalConfig(mixed_precision=mixed))
    cores = workers or len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        walls = pool.map(_cpu_worker, [(t, warm, steps) for t in range(cores)])
    wall = max(walls)
    return {"value": cores * g.num_nodes * steps / wall / 1e9, "unit": "G-NUPS", "cores": cores, "kind": "port",
            "wall_s": wall, "per_core_value": g.num_nodes * steps / (sum(walls) / len(walls)) / 1e9,
            "sample": f"{cores} independent trajectories (one per host core, run_ensemble style) x {steps} timed "
                      f"steps after {warm} warm-up, N={g.num_nodes}; oracle/spreadsim_port.py (numpy restatement "
                      f"of renewal_step with the reference's numba CSR fold, pinned to the reference's golden "
                      f"vectors)",
            "port_vs_reference": port_vs_reference()}


def _ens_worker(trial):
    from oracle import spreadsim_port as O

    g, m, cfg, e = _CPU_INPUTS
    times, rows, st = O.run(g, m, cfg, O.derive_seed(e["seed"], trial), e["t_final"], seed_count=e["seed_count"])
    return len(times) - 1  # steps run (whole batches)


def cpu_ensemble_trials(g, m, e: dict, runs: int) -> dict:
    """The reference's run_ensemble on the host cores: a process pool of
    trajectories of the oracle port (R/analysis.py:97-130)."""
    import multiprocessing as mp

    import paper_2604_22092_b200 as fs

    global _CPU_INPUTS
    _CPU_INPUTS = (g, m, fs.RenewalConfig(), e)
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        steps = pool.map(_ens_worker, range(runs))
    wall = time.perf_counter() - t0
    return {"value": g.num_nodes * sum(steps) / wall / 1e9, "unit": "G-NUPS", "cores": cores, "kind": "port",
            "wall_s": wall, "trajectories_per_s": runs / wall,
            "sample": f"{runs} trajectories to t_final={e['t_final']} in a process pool of {cores} workers "
                      f"(oracle/spreadsim_port.py, run_ensemble style)", "port_vs_reference": port_vs_reference()}


def run_ensemble_bench(args, w) -> None:
    """run_ensemble on the GPU (trials in lockstep, one launch per step for
    all of them, one graph upload, pipelined batches, device records):
    node-updates of every trial
    (whole batches, as run) over the call's wall time, max of `steps` calls
    after `warmup` untimed calls; host graph already built."""
    import torch

    import paper_2604_22092_b200 as fs

    g, m = build_inputs(w)
    e = w["ensemble"]
    cfg = fs.RenewalConfig()
    runs = e["runs"]

    def once(lockstep=True):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        recs = fs.run_ensemble("renewal", g, m, cfg, e["seed"], e["t_final"], runs, seed_count=e["seed_count"],
                               lockstep=lockstep)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, recs

    for _ in range(max(1, args.warmup // 3)):
        once()
    walls = []
    with ClockSampler(0) as clk:
        for _ in range(max(1, args.steps // 40)):
            wall, recs = once()
            walls.append(wall)
    wall = statistics.median(walls)
    b = cfg.steps_per_batch
    steps = sum(int(np.ceil(r.summary["step_count"] / b) * b) for r in recs)
    value = g.num_nodes * steps / wall / 1e9
    # lockstep: one launch per step for all trials, until the slowest trial ends
    lock_steps = max(int(np.ceil(r.summary["step_count"] / b) * b) for r in recs) + b  # + the batch queued ahead
    launches = lock_steps + 2 * (lock_steps // b)
    # the per-trial-stream runner (one engine and one launch per trial per step) on the same call, for comparison
    once(False)
    s_walls = [once(False)[0] for _ in range(max(1, args.steps // 40))]
    s_wall = statistics.median(s_walls)
    out = {
        "metric": "Giga-NUPS (node updates/s)", "value": value, "unit": "G-NUPS", "n_gpus": 1,
        "steps": len(walls), "warmup": args.warmup, "ms_per_step": wall * 1e3 / (steps / runs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(w), "data": data_of(w),
        "config": workload_config(w, w["n"]), "edges": g.num_edges,
        "engine": {"runner": "run_ensemble lockstep: every trial stepped by one grid per step (fs_ensemble, "
                             "k_step_incr_multi), CUDA-graph batches, one 2-D log copy per batch, records by one "
                             "device launch",
                   "trials": runs, "trajectories_per_s": runs / wall, "wall_s": walls, "lib_sha16": lib_sha16(),
                   "streams_runner": {"what": "run_ensemble(lockstep=False): one engine per trial on 32 CUDA streams",
                                      "value": g.num_nodes * steps / s_wall / 1e9, "wall_s": s_walls}},
        "roofline": None, "gpu_launches": launches, "clocks": clk.summary(),
        "e2e": {"value": value, "unit": "G-NUPS", "h2d_bytes_per_step": (g.row_offsets.nbytes + g.col_indices.nbytes)
                / (steps / runs), "d2h_bytes_per_step": 8 * (2 + m.num_compartments) * runs,
                "what": "the whole run_ensemble call from a host graph (graph upload, 100 trials, records)"},
        "cpu_baseline": cpu_ensemble_trials(g, m, e, runs) if args.cpu_steps > 0 else None,
    }
    print(json.dumps(out))


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    if w.get("ensemble"):
        g, m = build_inputs(w)
        cb = cpu_ensemble_trials(g, m, w["ensemble"], w["ensemble"]["runs"])
        print(json.dumps({"impl": "reference", "metric": "Giga-NUPS (node updates/s)", "value": cb["value"],
                          "unit": "G-NUPS", "n_gpus": world, "steps": 1, "warmup": 0,
                          "ms_per_step": cb["wall_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": dtype_of(w), "data": data_of(w),
                          "config": workload_config(w, w["n"], world), "cpu_baseline": cb,
                          "e2e": {"value": cb["value"], "unit": "G-NUPS", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return
    if w.get("engine") == "markov":
        print(json.dumps({"impl": "reference", "unavailable": "the CPU oracle port restates the renewal path only"}))
        return
    if "cpu_n" in w or w.get("per_gpu"):  # bounded sample of a workload too large for host RAM
        import paper_2604_22092_b200 as fs

        g = fs.gen_fixed_degree_device(w.get("cpu_n", w["n"]), w["k"], seed=GRAPH_SEED).to_host()
        m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    else:
        g, m = build_inputs(w)
    cb = cpu_ensemble(g, m, args.warmup, args.steps, mixed=bool(w.get("mixed", False)))
    v = cb["value"]
    print(json.dumps({
        "impl": "reference", "metric": "Giga-NUPS (node updates/s)", "value": v, "unit": "G-NUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["wall_s"] / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak" if (world == 1 or w.get("per_gpu")) else "strong",
        "vs_baseline": None, "dtype": dtype_of(w), "data": data_of(w),
        "config": workload_config(w, w["n"] * (world if w.get("per_gpu") else 1), world),
        "edges": g.num_edges if "cpu_n" not in w else None,
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "G-NUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def run_markov_bench(args, w) -> None:
    """The Markovian engine (R/markov.py) on the same graph family: each of
    the K steps (two kernels) timed alone after an L2 flush; e2e =
    run_markov to t_final from the host graph.  No CPU baseline: the oracle
    port restates the renewal path only."""
    import torch

    import paper_2604_22092_b200 as fs
    from paper_2604_22092_b200 import _lib
    from paper_2604_22092_b200.renewal import _pick_seed_nodes

    g, m = build_inputs(w)
    cfg = fs.MarkovConfig()
    n = g.num_nodes
    picked = _pick_seed_nodes(n, SIM_SEED, 10, torch.device("cuda")).cpu().numpy()
    st = fs.init_markov_state(g, m, picked)
    eng = st._bind(cfg, SIM_SEED)
    lib = st._lib
    _lib.check(lib.fs_markov_step(eng, args.warmup, st._stream))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush_rd = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        for k in range(args.steps):
            flush.zero_()
            flush_rd.max()
            starts[k].record()
            _lib.check(lib.fs_markov_step(eng, 1, st._stream))
            ends[k].record()
        torch.cuda.synchronize()
    total_ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    st._unbind()
    e2e = None
    if not args.no_e2e:
        walls = []
        for _ in range(5):  # median of 5 (host-side stalls, see the renewal e2e)
            g.__dict__.pop("_fs_device_cache", None)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rec = fs.run_markov(g, m, cfg, SIM_SEED, 50.0)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        wall = statistics.median(walls)
        steps_run = rec.summary["step_count"]
        e2e = {"value": n * steps_run / wall / 1e9, "unit": "G-NUPS",
               "h2d_bytes_per_step": (g.row_offsets.nbytes + g.col_indices.nbytes) / steps_run,
               "d2h_bytes_per_step": 8 * (1 + m.num_compartments), "steps": steps_run, "wall_s": wall,
               "walls_s": walls,
               "what": "run_markov(t_final=50) from a host CsrGraph: CSR H2D + init + CUDA-graph batches + log D2H; "
                       "median of 5 runs"}
    ms = total_ms / args.steps
    print(json.dumps({
        "metric": "Giga-NUPS (node updates/s)", "value": n / (ms / 1e3) / 1e9, "unit": "G-NUPS", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 rates, integer influence",
        "data": "synthetic (reference generators, graph seed 1, sim seed 7)",
        "config": {"workload": w["desc"], "n": n, "edges": g.num_edges, "engine": "markov (2 kernels per step)",
                   "l2": "flushed before every timed step (512 MiB write + 512 MiB read of another buffer)"},
        "roofline": None, "gpu_launches": 2 * args.steps, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": None,
    }))


def run_partitioned(args, w, rank: int, world: int, local: int) -> None:
    """Node-partitioned run over `world` GPUs: each rank
    generates its own rows of the graph, owns that node range, and exchanges
    the infectious mask + max rate + count deltas with NCCL after every step.
    Strong scaling: the graph (w["n"] nodes) is fixed as the GPU count grows.
    Inputs are far larger than L2, so the K steps are timed as back-to-back
    CUDA-graph batches (no flush needed), max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2604_22092_b200 as fs
    from paper_2604_22092_b200.distributed import DistributedRun, partition_plan, run_renewal_distributed

    weak = bool(w.get("per_gpu"))
    n_total = w["n"] * world if weak else w["n"]
    plan = partition_plan(n_total, world)
    lo, hi = plan.ranges[rank]
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    mixed = bool(w.get("mixed", False))
    cfg = fs.RenewalConfig(mixed_precision=mixed)
    g = fs.gen_fixed_degree_device(n_total, w["k"], seed=GRAPH_SEED, row_lo=lo, row_hi=hi)
    edges = torch.tensor([g.num_edges], dtype=torch.int64, device="cuda")
    dist.all_reduce(edges)
    run = DistributedRun(g, m, cfg, SIM_SEED, plan, rank)
    run.step(args.warmup)
    run.run_batch()  # capture the batch graph (NCCL inside) outside the timed region
    if weak:
        # per-GPU inputs fit in L2: each step timed alone after an L2 flush
        steps = args.steps
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        flush_rd = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            for k in range(steps):
                flush.zero_()
                flush_rd.max()
                starts[k].record()
                run.step(1)
                ends[k].record()
            torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(starts, ends))], dtype=torch.float64, device="cuda")
    else:
        nb = max(1, args.steps // cfg.steps_per_batch)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            e0.record()
            for _ in range(nb):
                run.part.run_batch()
            e1.record()
            torch.cuda.synchronize()
        dist.barrier()
        steps = nb * cfg.steps_per_batch
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    # transport evidence: pushes this rank sent to other ranks per timed step
    # (read from the engine's per-step ring), and the exchange's own time
    k_rp = min(steps, 200)
    rp = run.part.remote_pushes(run.steps - k_rp, k_rp).astype(np.float64)
    rp_t = torch.tensor([rp.mean(), rp.max()], dtype=torch.float64, device="cuda")
    dist.all_reduce(rp_t, op=dist.ReduceOp.MAX)
    xus = run.exchange_us(100)
    xus_t = torch.tensor([xus or 0.0], dtype=torch.float64, device="cuda")
    dist.all_reduce(xus_t, op=dist.ReduceOp.MAX)
    run.close()
    del g
    torch.cuda.empty_cache()
    e2e = None
    if not args.no_e2e:
        t_final = float(w.get("t_final", 50.0))
        dist.barrier()
        t0 = time.perf_counter()
        g = fs.gen_fixed_degree_device(n_total, w["k"], seed=GRAPH_SEED, row_lo=lo, row_hi=hi)
        rec = run_renewal_distributed(g, m, cfg, SIM_SEED, t_final, plan, rank)
        torch.cuda.synchronize()
        wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        dist.all_reduce(wall, op=dist.ReduceOp.MAX)
        wall = float(wall.item())
        steps_run = int(np.ceil(rec.summary["step_count"] / cfg.steps_per_batch) * cfg.steps_per_batch)
        d2h = 8 * (2 + m.num_compartments) * steps_run
        e2e = {"value": n_total * steps_run / wall / 1e9, "unit": "G-NUPS", "h2d_bytes_per_step": 0.0,
               "d2h_bytes_per_step": d2h / steps_run, "steps": steps_run, "wall_s": wall,
               "what": f"run_renewal_distributed(t_final={t_final}) on {world} ranks: per-rank graph generation on the "
                       f"device + NCCL setup + {steps_run} steps in CUDA-graph batches + per-batch log D2H + record",
               "final_R": rec.summary["final_R"], "peak_I": rec.summary["peak_I"]}
    if rank != 0:
        return
    pk = peaks()
    ms_per_step = total_ms / steps
    achieved = B_ALG[mixed] * n_total / (ms_per_step / 1e3) / 1e9
    print(json.dumps({
        "metric": "Giga-NUPS (node updates/s)", "value": n_total * steps / (total_ms / 1e3) / 1e9, "unit": "G-NUPS",
        "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None,
        "dtype": dtype_of(w), "data": data_of(w),
        "config": workload_config(w, n_total, world),
        "edges": int(edges.item()),
        "engine": {"strategy": "per-node",
                   "gather": "incremental counts, cross-rank pushes into peer memory (CUDA IPC / NVLink)",
                   "parallelism": f"node-partitioned x{world} (peer pushes + NCCL all-reduce of 17 words per step)",
                   "steps_from": f"t=0 after {args.warmup} warm-up steps", "lib_sha16": lib_sha16(),
                   "remote_pushes_per_step": {"mean_max_over_ranks": float(rp_t[0]), "max": float(rp_t[1]),
                                              "steps": k_rp},
                   "exchange_us_max_over_ranks": float(xus_t[0])},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"] * world, "unit": "GB/s",
                     "frac": achieved / (pk["hbm_gbs"] * world), "traffic": None,
                     "bytes_per_update": B_ALG[mixed], "peak_source": pk["source"] + f" x {world} GPUs"},
        "gpu_launches": steps,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": None,
        "scaling_t1": scaling_t1(args.workload, weak),
    }))


def scaling_t1(workload: str, weak: bool) -> dict | None:
    """The one-GPU point of this scaling line: the same workload's committed
    single-GPU bench line (strong scaling: C5 N = 1e9 on one GPU; weak: C2),
    so the efficiency value_N / (N x T1) compares like with like — the
    driver's own N = 1 run is the headline C2, a different workload."""
    name = {"c5": "c5", "c2w": "c2"}.get(workload)
    p = ROOT / "profiles" / f"r2_bench_{name}.json" if name else None
    if not p or not p.exists():
        return None
    d = json.loads(p.read_text())
    return {"workload": d["config"]["workload"], "value": d["value"], "unit": d["unit"],
            "scaling": "weak" if weak else "strong", "source": str(p.relative_to(ROOT))}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: c2 on one GPU (the headline config), c5 (N=1e9 partitioned) on several")
    ap.add_argument("--cpu-steps", type=int, default=30)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the node-partitioned (NCCL) path even on one GPU (checks the multi-GPU code path)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload is None:
        # N=1: the headline C2; N>1: BASELINE C5, N_total = 1e9 node-partitioned
        # over the GPUs (strong scaling, north_star's >= 70 % at 8 GPUs; its
        # T_1 is `--workload c5` on one GPU).  `--workload c2w` is the weak-
        # scaling alternative (1e6 nodes per GPU).
        args.workload = "c2" if world == 1 else "c5"
    if world > 1:
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return

    torch.cuda.set_device(local)
    import paper_2604_22092_b200 as fs
    from paper_2604_22092_b200 import renewal as R

    if world > 1 or args.partitioned:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            dist.init_process_group("nccl", rank=0, world_size=1)
        run_partitioned(args, WORKLOADS[args.workload], rank, world, local)
        dist.destroy_process_group()
        return
    if WORKLOADS[args.workload].get("engine") == "markov":
        run_markov_bench(args, WORKLOADS[args.workload])
        return
    if WORKLOADS[args.workload].get("ensemble"):
        run_ensemble_bench(args, WORKLOADS[args.workload])
        return

    w = WORKLOADS[args.workload]
    g, m = build_inputs(w)
    mixed = bool(w.get("mixed", False))
    cfg = fs.RenewalConfig(mixed_precision=mixed, gather=w.get("gather", "auto"))
    n = g.num_nodes
    device_graph = hasattr(g, "device_tensors")

    # ---------------- device throughput (value) ----------------
    st = fs.init_renewal_state(g, m, cfg, SIM_SEED)
    plan = R._build_plan(g, m, cfg, st.mixed_precision)
    eng = st._bind(plan, SIM_SEED, materialize=False)
    strategy_name, count_mode = plan.strategy.value, plan.count_mode
    incremental = count_mode and plan.config.incremental != 0 and plan.graph.symmetric
    kernels_per_step = eng.kernels_per_step()
    snap0 = eng.snapshot()
    for _ in range(6):  # captures the batch CUDA graphs (every step-parity variant) outside any timed region
        eng.run_batch(False)
    eng.restore(snap0)
    eng.step(args.warmup, False, False)
    snap = eng.snapshot()
    # L2-warm: the same K steps back to back as CUDA-graph batches (no flush)
    nb = max(1, args.steps // cfg.steps_per_batch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(nb):
        eng.run_batch(False)
    e1.record()
    torch.cuda.synchronize()
    warm_ms = e0.elapsed_time(e1) / (nb * cfg.steps_per_batch)
    eng.restore(snap)
    # headline: each of the K steps timed alone after an L2 flush: a 512 MiB
    # write, then a 512 MiB read of another buffer, so the step starts with
    # none of its inputs in L2 and without the flush's dirty lines pending
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush_rd = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            flush_rd.max()
            starts[k].record()
            eng.step(1, False, False)
            ends[k].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    uni_on = eng.uniform_s_age()
    per_step = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = torch.tensor([sum(per_step)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    total_ms = float(total_ms.item())
    ms_per_step = total_ms / args.steps
    value = world * n * args.steps / (total_ms / 1e3) / 1e9
    sim = st.step_counter
    st._unbind()

    # ---------------- end to end through the public API ----------------
    e2e = None
    if not args.no_e2e:
        t_final = float(w.get("t_final", 50.0))
        # host graphs: median of 5 end-to-end runs — single runs on the pool's
        # boxes occasionally stall 0.1-0.8 s on the host (scripts/e2e_trace.py:
        # neither in the batches nor in setup), which a median of 3 let through
        reps = 1 if device_graph else 5
        if device_graph:
            del st, eng, plan, snap, snap0
        walls, setups = [], []
        for _ in range(reps):
            torch.cuda.synchronize()
            if device_graph:
                del g
                torch.cuda.empty_cache()
                t0 = time.perf_counter()
                g = fs.gen_fixed_degree_device(w["n"], w["k"], seed=GRAPH_SEED)
                h2d = 0
                src = "a graph generated on the device (fs_gen_regular, inside the timed region)"
            else:
                # a fresh CsrGraph (new arrays, nothing cached on it) for every
                # run: the symmetry check, degree scan, page-locking and upload
                # are all inside the timed region, as on a user's first call
                g_run = fs.CsrGraph(g.num_nodes, g.num_edges, g.row_offsets.copy(), g.col_indices.copy(),
                                    g.weights.copy())
                t0 = time.perf_counter()
                h2d = g_run.row_offsets.nbytes + g_run.col_indices.nbytes
                src = "a fresh host CsrGraph per run (no cached device copy or scans; CSR H2D inside the timed region)"
            rec = fs.run_renewal(g if device_graph else g_run, m, cfg, SIM_SEED, t_final)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
            setups.append(rec.summary.get("setup_s"))
        wall = statistics.median(walls)
        steps_run = int(np.ceil(rec.summary["step_count"] / cfg.steps_per_batch) * cfg.steps_per_batch)
        d2h = 8 * (2 + m.num_compartments) * steps_run
        e2e = {"value": n * steps_run / wall / 1e9, "unit": "G-NUPS", "h2d_bytes_per_step": h2d / steps_run,
               "d2h_bytes_per_step": d2h / steps_run, "steps": steps_run, "wall_s": wall, "walls_s": walls,
               "setup_s": setups,
               "what": f"run_renewal(t_final={t_final}) from {src}: init + {steps_run} steps in "
                       f"CUDA-graph batches + per-batch log D2H + record; median of {reps} runs",
               "final_R": rec.summary["final_R"], "peak_I": rec.summary["peak_I"]}

    pk = peaks()
    achieved = B_ALG[mixed] * n / (ms_per_step / 1e3) / 1e9
    out = {
        "metric": "Giga-NUPS (node updates/s)",
        "value": value,
        "unit": "G-NUPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": dtype_of(w),
        "data": data_of(w),
        "config": workload_config(w, n, world),
        "edges": g.num_edges,
        "engine": {"strategy": strategy_name,
                   "gather": ("incremental counts (pushes along the outgoing CSR)" if incremental else
                              "count (1-bit mask)" if count_mode else "f32 CSR-order fold"),
                   "kernels_per_step": kernels_per_step, "uniform_s_age": uni_on, "parallelism": f"replicas x{world}",
                   "steps_from": f"t=0 after {args.warmup} warm-up steps", "lib_sha16": lib_sha16()},
        "roofline": roofline_block(achieved, pk, ncu_entry(args.workload), ms_per_step, B_ALG[mixed]),
        "value_l2_warm": {"value": n / (warm_ms / 1e3) / 1e9, "ms_per_step": warm_ms,
                          "what": f"the same {nb * cfg.steps_per_batch} steps replayed as {nb} back-to-back "
                                  f"CUDA-graph batches, no flush (engine state restored in between)"},
        "gpu_launches": args.steps * kernels_per_step,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if rank == 0 and world == 1 or rank == 0:
        out["cpu_baseline"] = None
        if world == 1 and args.cpu_steps > 0:
            if "cpu_n" in w:  # bounded sample: the same generator at a size the host handles
                gs = fs.gen_fixed_degree_device(w["cpu_n"], w["k"], seed=GRAPH_SEED).to_host()
                cb = cpu_ensemble(gs, m, 1, max(1, args.cpu_steps // 10), workers=2, mixed=mixed)
                cb["sample"] = "N=%d slice of the same workload family (" % w["cpu_n"] + cb["sample"] + ")"
            else:
                cb = cpu_ensemble(g, m, 2, args.cpu_steps, mixed=mixed)
            out["cpu_baseline"] = cb
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
