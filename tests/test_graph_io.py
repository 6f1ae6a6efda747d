"""FSPG v1 graph files (R/graph.py:373-425), byte-compatible with files the
reference wrote (tests/golden/make_fspg_golden.py)."""

import numpy as np
import pytest

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200.errors import GraphFileError
from tests._cases import GOLDEN


def _same(a, b):
    assert a.num_nodes == b.num_nodes and a.num_edges == b.num_edges
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(a.weights, b.weights)


def test_reads_reference_file_and_writes_identical_bytes(tmp_path):
    ref = fs.load_graph(GOLDEN / "ba300.fspg")
    _same(ref, fs.gen_barabasi_albert(300, 3, seed=5))
    out = tmp_path / "ours.fspg"
    fs.save_graph(ref, out)
    assert out.read_bytes() == (GOLDEN / "ba300.fspg").read_bytes()


def test_edge_list_matches_reference(tmp_path):
    g = fs.read_edge_list(GOLDEN / "edges.txt")
    out = tmp_path / "e.fspg"
    fs.save_graph(g, out)
    assert out.read_bytes() == (GOLDEN / "edges.fspg").read_bytes()
    assert g.weights.tolist() == [2.0, 1.0, 1.0, 0.5]  # slices of node 0, 1, 1, 2


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXX" + b[4:], "bad magic"),
    (lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:], "version"),
    (lambda b: b[:-4], "truncated"),
    (lambda b: b + b"\0\0\0\0", "oversized"),
])
def test_malformed_files_raise(tmp_path, mutate, msg):
    p = tmp_path / "bad.fspg"
    p.write_bytes(mutate((GOLDEN / "ba300.fspg").read_bytes()))
    with pytest.raises(GraphFileError, match=msg):
        fs.load_graph(p)


def test_round_trip_generated_graphs(tmp_path):
    for g in (fs.gen_fixed_degree(2000, 10, seed=1), fs.gen_erdos_renyi(500, 4.0, seed=2)):
        p = tmp_path / "g.fspg"
        fs.save_graph(g, p)
        _same(fs.load_graph(p), g)
