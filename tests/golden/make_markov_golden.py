"""Golden vectors of the REFERENCE Markovian engine (R/markov.py).

    python tests/golden/make_markov_golden.py

Imports /root/reference/pkg/src/spreadsim unmodified and records, per case,
run_markov's initial state (R/markov.py:184-212) followed by `steps`
markov_step calls (R/markov.py:143-181): per-step clock, tau and counts, and
the final states, influence and rates; plus one run_markov record.  Written
to tests/golden/markov.npz + markov.json; read by tests/test_markov.py.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
import spreadsim as ss  # noqa: E402
from spreadsim.graph import build_outgoing  # noqa: E402
from spreadsim.markov import MarkovConfig, init_markov_state, influence_gather, markov_step, run_markov  # noqa: E402
from spreadsim.models import Holding, ModelSpec  # noqa: E402
from spreadsim.renewal import _pick_seed_nodes  # noqa: E402


def seir_exp():
    return ModelSpec(name="seir-exp", compartments=("S", "E", "I", "R"), beta=0.25, edge_from=0, edge_to=1,
                     nodal={1: (2, Holding.exponential(0.2)), 2: (3, Holding.exponential(1.0 / 7.5))}, infectious=2)


CASES = {
    "sir_er": (["gen_erdos_renyi", 1000, 8.0, 3], "sir", {}, 11, 10, 400),
    "sis_reg": (["gen_fixed_degree", 2000, 6, 2], "sis", {}, 5, 20, 400),
    "seir_ba": (["gen_barabasi_albert", 3000, 4, 7], "seir_exp", {"theta": 0.02}, 9, 15, 300),
    "sir_er_pmax": (["gen_erdos_renyi", 1500, 6.0, 4], "sir", {"p_max": 0.05, "tau_max": 0.2}, 13, 10, 300),
}
MODELS = {"sir": lambda: ss.sir_model(0.25, 0.15), "sis": lambda: ss.sis_model(0.25, 0.15), "seir_exp": seir_exp}


def main() -> None:
    out, meta = {}, {}
    for name, (gspec, mname, cfgkw, seed, seed_count, steps) in CASES.items():
        g = getattr(ss, gspec[0])(*gspec[1:3], seed=gspec[3])
        build_outgoing(g)
        m = MODELS[mname]()
        cfg = MarkovConfig(**cfgkw)
        picked = _pick_seed_nodes(g.num_nodes, seed, seed_count)
        st = init_markov_state(g, m, picked)
        clocks, taus, counts = [], [], []
        for _ in range(steps):
            _, tau = markov_step(st, g, m, cfg, seed)
            clocks.append(st.clock)
            taus.append(tau)
            counts.append(st.counts.copy())
        out[f"{name}__clock"] = np.array(clocks)
        out[f"{name}__tau"] = np.array(taus)
        out[f"{name}__counts"] = np.array(counts)
        out[f"{name}__states"] = st.states.copy()
        out[f"{name}__influence"] = st.influence.copy()
        out[f"{name}__rates"] = st.rates.copy()
        assert np.array_equal(st.influence, influence_gather(g, st.states, m))
        rec = run_markov(g, m, cfg, seed, 30.0, seed_count=seed_count)
        out[f"{name}__record"] = rec.fractions
        out[f"{name}__record_steps"] = np.array(rec.summary["step_count"])
        meta[name] = {"graph": gspec, "model": mname, "cfg": cfgkw, "seed": seed, "seed_count": seed_count,
                      "steps": steps, "t_final": 30.0}
    np.savez_compressed(OUT / "markov.npz", **out)
    (OUT / "markov.json").write_text(json.dumps(meta, indent=1))
    print({k: v.shape for k, v in out.items() if k.endswith("counts")})


if __name__ == "__main__":
    main()
