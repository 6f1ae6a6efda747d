"""bench.py's JSON contract on CPU: the reference arm's line (C1, the
oracle port on the host cores), the roofline block, the nvidia-smi clock
parser and the workload table."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line_c1():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "2",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert BASE_KEYS <= set(line) and line["impl"] == "reference"
    assert line["metric"] == "Giga-NUPS (node updates/s)" and line["unit"] == "G-NUPS" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"] and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "G-NUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("C1")


def test_roofline_block_fields():
    pk = {"hbm_gbs": 6537.6, "source": "measured"}
    ncu = {"dram_bytes_per_launch": 12_000_000, "gpu_time_us": 20.0, "kernel": "k", "lib_sha16": "x"}
    r = bench.roofline_block(3000.0, pk, ncu, 0.025, 112.0)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] == 6537.6
    assert r["frac"] == pytest.approx(3000.0 / 6537.6)
    assert r["traffic"] == 12_000_000 and r["bytes_per_update"] == 112.0
    assert r["traffic_gbs"] == pytest.approx(12_000_000 / 0.025e-3 / 1e9)
    assert r["frac_physical"] == pytest.approx(12_000_000 / 20e-6 / 1e9 / 6537.6)
    assert r["ncu_same_build"] is False  # the sha does not match the built library
    assert "frac_physical" not in bench.roofline_block(3000.0, pk, {}, 0.025, 112.0)


def test_both_arms_share_the_workload_config():
    for name, w in bench.WORKLOADS.items():
        for world in (1, 8):
            a = bench.workload_config(w, w["n"], world)
            assert a == bench.workload_config(w, w["n"], world)
            assert set(a) == {"workload", "n", "graph_seed", "sim_seed", "precision", "gather_option", "l2"}


def test_clock_sampler_parses_reasons_and_memory_clock():
    c = bench.ClockSampler(0)
    c.lines = ["1965, 1965, Not Active, Not Active, Not Active, Active, 3996, 700.5, 1000.00, 50",
               "1950, 1965, Not Active, Not Active, Not Active, Not Active, 3996, 650.0, 1000.00, 51",
               "garbage"]
    s = c.summary()
    assert s["sm_mhz"] == pytest.approx(1957.5) and s["sm_max_mhz"] == 1965.0 and s["samples"] == 2
    assert s["reasons"] == ["sw_power_cap"]
    assert s["mem_mhz"] == 3996.0 and s["power_w"] == 700.5 and s["power_limit_w"] == 1000.0


def test_workload_table():
    for name, w in bench.WORKLOADS.items():
        assert "desc" in w, name
    assert {"c1", "c2", "c3", "c4", "c5", "m2"} <= set(bench.WORKLOADS)
