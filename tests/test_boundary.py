"""The C-ABI boundary (CPU only): the shared library loads, exports every
function include/flashspread.h declares, the ctypes mirrors have the C
layouts, and the product package never reaches into oracle/."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2604_22092_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "flashspread.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTED_SYMBOLS, f"{name} declared in the header but not bound in _lib.py"
    assert lib.fs_abi_version() == _lib.ABI_VERSION
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    for name in names:
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported"


def test_ctypes_layouts_match_c(tmp_path):
    src = tmp_path / "layout.c"
    structs = ["fs_graph", "fs_compartment", "fs_model", "fs_config", "fs_scalars", "fs_state_buffers", "fs_partition",
               "fs_markov_config"]
    body = "\n".join(f'printf("{s} %zu\\n", sizeof({s}));' for s in structs)
    offs = {
        "fs_model": ["beta", "shedding", "shed_mu", "shed_peak", "comp"],
        "fs_scalars": ["step", "seed", "last_max_rate", "started", "counts"],
        "fs_graph": ["row_offsets", "weights_dtype", "uniform_weight", "d_max"],
        "fs_config": ["steps_per_batch", "count_gather"],
        "fs_partition": ["num_nodes_global", "mask_segment_words", "rank", "world", "comm"],
        "fs_markov_config": ["p_max", "tau_max", "steps_per_batch"],
    }
    for s, fields in offs.items():
        for f in fields:
            body += f'\nprintf("{s}.{f} %zu\\n", offsetof({s}, {f}));'
    src.write_text(f'#include <stdio.h>\n#include <stddef.h>\n#include "{HEADER}"\nint main(void){{{body} return 0;}}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    cls = {"fs_graph": _lib.FsGraph, "fs_compartment": _lib.FsCompartment, "fs_model": _lib.FsModel,
           "fs_config": _lib.FsConfig, "fs_scalars": _lib.FsScalars, "fs_state_buffers": _lib.FsStateBuffers,
           "fs_partition": _lib.FsPartition, "fs_markov_config": _lib.FsMarkovConfig}
    for s, c in cls.items():
        assert int(got[s]) == ctypes.sizeof(c), s
    for key, v in got.items():
        if "." in key:
            s, f = key.split(".")
            assert getattr(cls[s], f).offset == int(v), key


def test_product_never_imports_the_oracle():
    pkg = ROOT / "paper_2604_22092_b200"
    for p in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = p.read_text()
        assert not re.search(r"^\s*(from|import)\s+(oracle|spreadsim)\b", text, flags=re.M), p
        assert not re.search(r"import_module\(|__import__\(|sys\.path", text), p
        assert not re.search(r'#include\s*"[^"]*oracle', text), p


def test_errors_map_to_reference_types():
    from paper_2604_22092_b200 import errors

    assert issubclass(errors.InvalidConfigError, ValueError)
    for name in ("GraphError", "IndexOutOfRangeError", "DuplicateEdgeError", "SelfLoopError",
                 "InfeasibleDegreeSequenceError", "InvalidMomentsError", "ReconfigureAfterStartError"):
        assert issubclass(getattr(errors, name), errors.SpreadSimError)
