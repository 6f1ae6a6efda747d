"""Fold `ncu --set full` captures of bench.py workloads into
profiles/ncu_summary.json (the file bench.py's roofline block reads).

    python scripts/ncu_to_summary.py TAG W1 [W2 ...]           (here, from reports)
    OUT=gpurun_out python scripts/ncu_to_summary.py TAG W1 ...  (on the GPU box)

reads gpurun_out/prof_TAG_W.ncu-rep (scripts/gpu_evidence_r2.sh) and
gpurun_out/lib_sha16_TAG.txt (the sha of the library the capture ran) and
writes, per workload: kernel, DRAM bytes per launch, ncu duration, into
$OUT/ncu_summary.json (default profiles/) and the text summary into
$OUT/TAG_W_ncu_full.txt.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def metrics(rep: Path) -> dict:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, r = rows[0], rows[1], rows[2]

    def val(name):
        i = h.index(name)
        x = float(r[i].replace(",", ""))
        unit = u[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "usecond": 1, "us": 1,
                 "msecond": 1e3, "ms": 1e3}.get(unit, 1)
        return x * scale

    return {"kernel": r[h.index("Kernel Name")], "gpu_time_us": round(val("gpu__time_duration.sum"), 3),
            "dram_bytes_per_launch": int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))}


def main() -> None:
    tag, works = sys.argv[1], sys.argv[2:]
    import os

    out_dir = ROOT / os.environ.get("OUT", "profiles")
    out_p = out_dir / "ncu_summary.json"
    summary = json.loads(out_p.read_text()) if out_p.exists() else {}
    sha_p = ROOT / "gpurun_out" / f"lib_sha16_{tag}.txt"
    sha = sha_p.read_text().strip() if sha_p.exists() else None
    for w in works:
        rep = ROOT / "gpurun_out" / f"prof_{tag}_{w}.ncu-rep"
        if not rep.exists():
            print("missing", rep)
            continue
        m = metrics(rep)
        m.update(lib_sha16=sha, source=f"ncu --set full of `bench.py --workload {w}` (capture {tag}), "
                                        f"summary profiles/{tag}_{w}_ncu_full.txt")
        summary[w] = m
        txt = subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_summary.py"), str(rep)],
                             capture_output=True, text=True).stdout
        (out_dir / f"{tag}_{w}_ncu_full.txt").write_text(txt)
        print(w, m)
    out_p.write_text(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
