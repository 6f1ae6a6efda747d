"""Generate golden vectors from the REFERENCE implementation.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/spreadsim (unmodified, read-only) and
writes small .npz fixtures next to this file.  The fixtures travel with the
repo; nothing on the GPU box reads /root/reference.  Graph inputs are
recorded by generator arguments plus a SHA-256 of the CSR arrays, because
paper_2604_22092_b200.graph reproduces the reference generators bit for bit
(tests/test_graph.py checks the hashes).
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import spreadsim as ss  # noqa: E402
from spreadsim import renewal as R  # noqa: E402
from spreadsim.graph import Strategy  # noqa: E402
from spreadsim.hazards import Shedding  # noqa: E402


def csr_sha(g) -> str:
    h = hashlib.sha256()
    for a in (g.row_offsets.astype(np.int64), g.col_indices.astype(np.int32), g.weights.astype(np.float32)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


GRAPHS = {
    "fixed_1e4": ("gen_fixed_degree", (10_000, 10), 1),
    "er_1000": ("gen_erdos_renyi", (1000, 8.0), 20250809),
    "er_400": ("gen_erdos_renyi", (400, 8.0), 5),
    "er_300": ("gen_erdos_renyi", (300, 8.0), 4),
    "er_200": ("gen_erdos_renyi", (200, 8.0), 17),
    "fixed_400": ("gen_fixed_degree", (400, 8), 5),
    "ba_1e4": ("gen_barabasi_albert", (10_000, 5), 1),
    "ba_2000": ("gen_barabasi_albert", (2000, 5), 3),
    "ba_1e5": ("gen_barabasi_albert", (100_000, 5), 2),
}


def make_graph(name):
    fn, args, seed = GRAPHS[name]
    return getattr(ss, fn)(*args, seed=seed)


def weighted_graph():
    """ER(300, 8) with random weights in [0.1, 1.5) (general gather)."""
    base = make_graph("er_300")
    e = ss.graph.decompose(base)
    e[:, 2] = np.random.default_rng(99).uniform(0.1, 1.5, size=e.shape[0])
    return ss.build_csr(e, base.num_nodes), e


def rng_vectors():
    out = {}
    streams = np.array([0, 1, 5, 42, 10**9, 2**40, 2**63 + 7], dtype=np.uint64)
    cases = [(0, 0), (7, 0), (7, 199), (12345, 3), (2**63 + 11, 2**40)]
    out["streams"] = streams
    out["cases"] = np.array(cases, dtype=np.uint64)
    out["uniform"] = np.stack([ss.rng.uniform_array(s, k, streams) for s, k in cases])
    big = ss.rng.uniform_array(77, 5, np.arange(100_000, dtype=np.uint64))
    out["uniform_77_5_head"] = big[:1000]
    out["uniform_77_5_sum"] = np.array([big.sum()])
    out["derive"] = np.array([[s, i, ss.derive_seed(s, i)] for s in (0, 7, 99, 20250809) for i in (0, 1, 5, 0x5EEDC0DE, 0x6EA9)],
                             dtype=np.uint64)
    return out


def hazard_vectors():
    z = np.linspace(-9.0, 30.0, 10_001)
    z = np.concatenate([z, [0.0, 3.5, 3.5 + 1e-9, 3.5 - 1e-9, -3.5, 20.0, -26.0, -27.0, 100.0]])
    tau = np.concatenate([[0.0, 1e-6, 1e-3, 0.01, 0.1, 4.0, 5.0], np.linspace(0.05, 60.0, 2000), [80.0, 110.0, 450.0, 1e4]])
    ei = ss.lognormal_from_mean_median(5.0, 4.0)
    ir = ss.lognormal_from_mean_median(7.5, 5.0)
    return {
        "z": z, "erfcx": ss.erfcx_stable(z),
        "tau": tau,
        "h_ei": ss.lognormal_hazard(tau, ei), "h_ir": ss.lognormal_hazard(tau, ir),
        "ei": np.array([ei.mu, ei.sigma]), "ir": np.array([ir.mu, ir.sigma]),
        "shed_peak": ss.shedding(Shedding.density_peak(ir), tau),
        "shed_haz": ss.shedding(Shedding.lognormal_hazard(ir), tau),
    }


def pressure_vectors():
    out = {}
    for name in ("er_400", "fixed_400", "ba_2000"):
        g = make_graph(name)
        inf = (np.random.default_rng(0).random(g.num_nodes) * 0.25).astype(np.float32)
        out[f"{name}_inf"] = inf
        out[f"{name}_p"] = R.pressure_gather(g, inf, Strategy.PER_NODE, R.RenewalConfig())
    g, _ = weighted_graph()
    inf = np.random.default_rng(1).random(g.num_nodes).astype(np.float32)
    out["weighted_inf"] = inf
    out["weighted_p"] = R.pressure_gather(g, inf, Strategy.PER_NODE, R.RenewalConfig())
    return out


def trajectory(g, m, cfg, seed, batches, seed_count=None, seed_compartment=None, checkpoints=(1, 10, 50)):
    st = R.init_renewal_state(g, m, cfg, seed, seed_count, seed_compartment)
    plan = R._build_plan(g, m, cfg, st.mixed_precision)
    clocks, taus, counts, cps = [], [], [], {}
    k = 0
    for _ in range(batches):
        R._begin_batch(st, g, cfg, plan)
        for _ in range(cfg.steps_per_batch):
            _, tau = R.renewal_step(st, g, m, cfg, seed, plan=plan)
            k += 1
            clocks.append(st.clock)
            taus.append(tau)
            counts.append(st.counts.copy())
            if k in checkpoints:
                cps[f"cp{k}_states"] = st.states.astype(np.int32).copy()
                cps[f"cp{k}_ages"] = st.ages.astype(np.float32).copy()
    return dict(
        clock=np.array(clocks), tau=np.array(taus), counts=np.array(counts),
        states=st.states.astype(np.int32), ages=st.ages.astype(np.float32),
        infectivity=st.infectivity.astype(np.float32), rates=st.rates.copy(), pressure=st.pressure.copy(),
        tau_prev=np.array([st.tau_prev]), **cps,
    )


SEIR = ss.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)


def trajectory_cases():
    ir = ss.lognormal_from_mean_median(7.5, 5.0)
    wg, _ = weighted_graph()
    cases = {
        # name: (graph, model, cfg kwargs, seed, batches, seed_count, seed_compartment)
        "c1": ("fixed_1e4", "seir", {}, 7, 4, None, None),
        "c1_mixed": ("fixed_1e4", "seir", {"mixed_precision": True}, 7, 4, None, None),
        "er1000": ("er_1000", "seir", {}, 3, 6, 10, None),
        "er1000_nocarry": ("er_1000", "seir", {"carry_tau": False, "steps_per_batch": 7}, 5, 20, 10, None),
        "ba_merge": ("ba_1e4", "seir", {"strategy": "EDGE_MERGE"}, 11, 2, None, None),
        "ba_auto": ("ba_1e5", "seir", {}, 13, 2, None, None),
        "ba_lane": ("ba_1e4", "seir", {"strategy": "LANE_CHUNKED"}, 11, 1, None, None),
        "sis": ("er_200", "sis", {}, 5, 4, 10, None),
        "sir": ("er_300", "sir", {}, 3, 4, 10, None),
        "shed_hazard": ("er_300", "seir_shed", {}, 5, 3, None, None),
        "shed_peak_iseed": ("er_300", "seir_peak", {}, 8, 3, 12, 2),
        "weighted": ("weighted", "seir", {}, 9, 3, 20, None),
        "eps05": ("er_300", "seir", {"epsilon": 0.05, "tau_max": 0.2}, 1, 6, None, None),
    }
    models = {
        "seir": SEIR,
        "sis": ss.sis_model(0.25, 0.15),
        "sir": ss.sir_model(0.25, 0.15),
        "seir_shed": ss.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0, transmission=Shedding.lognormal_hazard(ir)),
        "seir_peak": ss.seir_standard(0.4, 5.0, 4.0, 7.5, 5.0, transmission=Shedding.density_peak(ir)),
    }
    out, meta = {}, {}
    for name, (gname, mname, kw, seed, batches, sc, scomp) in cases.items():
        g = wg if gname == "weighted" else make_graph(gname)
        kw = dict(kw)
        if "strategy" in kw:
            kw["strategy"] = Strategy[kw["strategy"]]
        cfg = R.RenewalConfig(**kw)
        res = trajectory(g, models[mname], cfg, seed, batches, sc, scomp)
        for k, v in res.items():
            out[f"{name}__{k}"] = v
        meta[name] = dict(graph=gname, model=mname, cfg={k: (v.name if isinstance(v, Strategy) else v) for k, v in kw.items()},
                          seed=seed, batches=batches, seed_count=sc, seed_compartment=scomp)
    return out, meta


def record_vectors():
    g = make_graph("er_300")
    rec = ss.run_renewal(g, SEIR, R.RenewalConfig(), seed=77, t_final=20.0)
    return {"fractions": rec.fractions, "grid": rec.grid,
            "summary": np.array([rec.summary["peak_I"], rec.summary["peak_I_time"], rec.summary["final_R"],
                                 rec.summary["step_count"]])}


def main():
    np.savez_compressed(OUT / "rng.npz", **rng_vectors())
    np.savez_compressed(OUT / "hazards.npz", **hazard_vectors())
    np.savez_compressed(OUT / "pressure.npz", **pressure_vectors())
    traj, meta = trajectory_cases()
    np.savez_compressed(OUT / "trajectories.npz", **traj)
    np.savez_compressed(OUT / "record.npz", **record_vectors())
    wg, _ = weighted_graph()
    graphs = {name: {"fn": fn, "args": list(args), "seed": seed, "sha256": csr_sha(make_graph(name))}
              for name, (fn, args, seed) in GRAPHS.items()}
    graphs["weighted"] = {"fn": "weighted_er_300", "sha256": csr_sha(wg)}
    (OUT / "manifest.json").write_text(json.dumps({"graphs": graphs, "trajectories": meta,
                                                   "reference": "spreadsim 0.1.0 @ /root/reference/pkg"}, indent=1))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
