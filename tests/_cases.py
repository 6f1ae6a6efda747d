"""Shared fixtures: golden vectors, graphs and models rebuilt from the
manifest with this package's (reference-identical) generators."""

from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200.graph import Strategy

GOLDEN = Path(__file__).resolve().parent / "golden"
MANIFEST = json.loads((GOLDEN / "manifest.json").read_text())


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def csr_sha(g) -> str:
    h = hashlib.sha256()
    for a in (g.row_offsets.astype(np.int64), g.col_indices.astype(np.int32), g.weights.astype(np.float32)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@lru_cache(maxsize=None)
def graph(name: str):
    if name == "weighted":
        base = graph("er_300")
        e = fs.decompose(base)
        e[:, 2] = np.random.default_rng(99).uniform(0.1, 1.5, size=e.shape[0])
        return fs.build_csr(e, base.num_nodes)
    spec = MANIFEST["graphs"][name]
    return getattr(fs, spec["fn"])(*spec["args"], seed=spec["seed"])


def model(name: str):
    ir = fs.lognormal_from_mean_median(7.5, 5.0)
    return {
        "seir": fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0),
        "sis": fs.sis_model(0.25, 0.15),
        "sir": fs.sir_model(0.25, 0.15),
        "seir_shed": fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0, transmission=fs.Shedding.lognormal_hazard(ir)),
        "seir_peak": fs.seir_standard(0.4, 5.0, 4.0, 7.5, 5.0, transmission=fs.Shedding.density_peak(ir)),
        "seir_we": fs.seir_weibull_erlang(0.25),
    }[name]


def config(kw: dict) -> fs.RenewalConfig:
    kw = dict(kw)
    if "strategy" in kw and isinstance(kw["strategy"], str):
        kw["strategy"] = Strategy[kw["strategy"]]
    return fs.RenewalConfig(**kw)


def trajectory_case(name: str):
    meta = MANIFEST["trajectories"][name]
    traj = golden("trajectories")
    ref = {k.split("__", 1)[1]: v for k, v in traj.items() if k.startswith(name + "__")}
    return meta, graph(meta["graph"]), model(meta["model"]), config(meta["cfg"]), ref


TRAJECTORY_CASES = tuple(MANIFEST["trajectories"])
