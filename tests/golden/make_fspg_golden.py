"""FSPG v1 graph files written by the REFERENCE (R/graph.py:373-381, 409-425).

    python tests/golden/make_fspg_golden.py

Imports /root/reference/pkg/src/spreadsim unmodified; the two small files it
writes are committed next to this script and read by tests/test_graph_io.py.
"""
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
import spreadsim as ss  # noqa: E402
from spreadsim.graph import save_graph  # noqa: E402

save_graph(ss.gen_barabasi_albert(300, 3, seed=5), OUT / "ba300.fspg")
(OUT / "edges.txt").write_text("# src dst [w]\n0 1\n1 2 0.5\n2 0 2.0\n3 1\n")
save_graph(ss.read_edge_list(OUT / "edges.txt"), OUT / "edges.fspg")
