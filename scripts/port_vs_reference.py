"""Per-core speed of the oracle port (bench.py's CPU arm) against the
reference's own renewal_step, on the same graph, in the build container
(the only place the reference is importable).  Writes
profiles/port_vs_reference.json, which bench.py quotes next to
cpu_baseline.

    python scripts/port_vs_reference.py [N] [steps]
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(1, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import spreadsim as ss  # noqa: E402
from spreadsim import renewal as RR  # noqa: E402

from oracle import spreadsim_port as O  # noqa: E402


def main() -> None:
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    out = {}
    for name, gen, model in (("c2", lambda: ss.gen_fixed_degree(n, 10, seed=1), lambda: ss.seir_standard(0.25, 5, 4, 7.5, 5)),):
        g, m = gen(), model()
        cfg = RR.RenewalConfig()
        st = RR.init_renewal_state(g, m, cfg, 7)
        plan = RR._build_plan(g, m, cfg, False)
        for _ in range(3):
            RR.renewal_step(st, g, m, cfg, 7, plan=plan)
        t0 = time.perf_counter()
        for _ in range(steps):
            RR.renewal_step(st, g, m, cfg, 7, plan=plan)
        t_ref = (time.perf_counter() - t0) / steps
        ost = O.init_state(g, m, cfg, 7)
        for _ in range(3):
            O.step(ost, g, m, cfg, 7)
        t0 = time.perf_counter()
        for _ in range(steps):
            O.step(ost, g, m, cfg, 7)
        t_port = (time.perf_counter() - t0) / steps
        assert np.array_equal(ost.states, st.states) and np.array_equal(ost.ages, st.ages)
        out[name] = {"n": n, "steps": steps, "reference_s_per_step": t_ref, "port_s_per_step": t_port,
                     "reference_mnups_per_core": n / t_ref / 1e6, "port_mnups_per_core": n / t_port / 1e6,
                     "port_over_reference_time": t_port / t_ref, "reference_numba_fold": bool(RR._HAVE_NUMBA)}
        print(name, json.dumps(out[name]))
    (ROOT / "profiles" / "port_vs_reference.json").write_text(json.dumps(
        {**out, "where": "build container (8-core Xeon), single thread each, same graph/seed, states checked equal"},
        indent=1))


if __name__ == "__main__":
    main()
