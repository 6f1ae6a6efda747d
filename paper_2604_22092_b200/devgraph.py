"""Device-resident CSR graphs produced on the GPU.

The reference's generators (R/graph.py:252-365) are CPU code; at the
N = 1e8 / 1e9 configurations (BASELINE configs 4 and 5) the configuration
model needs ~100 GB / ~1 TB of host memory.
``gen_fixed_degree_device`` builds a random uniform-degree graph directly in
HBM with ``fs_gen_regular`` (csrc/fs_graphgen.cu: union of keyed random
Hamiltonian cycles), optionally only the rows
[row_lo, row_hi) a rank of a node-partitioned run owns.
``gen_barabasi_albert_device`` / ``gen_erdos_renyi_device`` do the same for
the reference's other two models (csrc/fs_gen_random.cu).

``DeviceCsrGraph`` quacks like ``CsrGraph`` for the renewal API: the engine
uses the device arrays as they are, and the host attributes
(``row_offsets``, ``col_indices``, ``weights``) download on first access so the
oracle can run on small instances.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _device, _lib
from .errors import InfeasibleDegreeSequenceError, IndexOutOfRangeError
from .graph import MAX_NODES, DegreeStats

__all__ = ["DeviceCsrGraph", "gen_fixed_degree_device", "gen_barabasi_albert_device", "gen_erdos_renyi_device",
           "regular_row_host"]


class DeviceCsrGraph:
    """Rows [row_lo, row_lo + num_rows) of an incoming CSR over `num_nodes`
    global nodes, held on the device.  Column ids are global; weights are
    the uniform 1.0 of the reference generators (R/graph.py:230)."""

    def __init__(self, num_nodes: int, row_lo: int, num_rows: int, num_edges: int, row_offsets: torch.Tensor,
                 col_buffer: torch.Tensor, d_max: int, weight: float = 1.0):
        self.num_nodes_global = int(num_nodes)
        self.row_lo = int(row_lo)
        self.num_rows = int(num_rows)
        self.num_edges = int(num_edges)
        self.uniform_weight = float(weight)
        self._ro = row_offsets            # int64[num_rows + 1]
        self._col_buffer = col_buffer     # int32[>= num_edges + 4] (bulk-copy slack)
        self.d_max = int(d_max)
        self.symmetric_global = True  # fs_gen_regular graphs are undirected: out-rows == in-rows
        self._host: dict[str, np.ndarray] = {}
        self.outgoing = None

    # CsrGraph surface ------------------------------------------------------
    @property
    def num_nodes(self) -> int:
        """Rows this object holds (== the graph's N when unpartitioned)."""
        return self.num_rows

    @property
    def partitioned(self) -> bool:
        return self.num_rows != self.num_nodes_global

    @property
    def row_offsets(self) -> np.ndarray:
        if "ro" not in self._host:
            self._host["ro"] = self._ro.cpu().numpy()
        return self._host["ro"]

    @property
    def col_indices(self) -> np.ndarray:
        if "col" not in self._host:
            self._host["col"] = self._col_buffer[: self.num_edges].cpu().numpy()
        return self._host["col"]

    @property
    def weights(self) -> np.ndarray:
        return np.full(self.num_edges, self.uniform_weight, dtype=np.float32)

    def in_degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def device_degree_stats(self) -> DegreeStats:
        d_avg = self.num_edges / max(1, self.num_rows)
        return DegreeStats(d_avg=d_avg, d_max=self.d_max, rho=self.d_max / d_avg if d_avg else float("inf"))

    def to_host(self):
        """A host ``CsrGraph`` with the same arrays (small instances)."""
        from .graph import CsrGraph

        if self.partitioned:
            raise ValueError("to_host() of a partition slice is not a graph")
        return CsrGraph(self.num_nodes, self.num_edges, self.row_offsets.copy(), self.col_indices.copy(),
                        self.weights)

    # device views -----------------------------------------------------------
    def device_tensors(self) -> dict:
        return {"row_offsets": self._ro, "col_buffer": self._col_buffer}


def gen_fixed_degree_device(N: int, d: int, seed: int, row_lo: int = 0, row_hi: int | None = None) -> DeviceCsrGraph:
    """Random d-regular graph on the device (rows [row_lo, row_hi) only when
    partitioned).  Same argument checks as the reference's gen_fixed_degree
    (R/graph.py:289-303)."""
    if N < 2 or N > MAX_NODES:
        raise IndexOutOfRangeError("need 2 <= N <= 2^31-1")
    if d < 0 or d >= N:
        raise InfeasibleDegreeSequenceError(f"degree {d} infeasible for N={N}")
    if (N * d) % 2 != 0:
        raise InfeasibleDegreeSequenceError("N * d must be even")
    if d >= 2 and N < 3:
        raise InfeasibleDegreeSequenceError("N >= 3 needed")
    row_hi = N if row_hi is None else int(row_hi)
    if not 0 <= row_lo <= row_hi <= N:
        raise IndexOutOfRangeError("bad row range")
    lib = _lib.load()
    dev = _device.device()
    rows = row_hi - row_lo
    ro = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    cap = rows * d
    col = torch.zeros(cap + 4, dtype=torch.int32, device=dev)
    e = ctypes.c_int64()
    _lib.check(lib.fs_gen_regular(N, d, seed & ((1 << 64) - 1), row_lo, row_hi, _lib.ptr(ro), _lib.ptr(col), cap,
                                  ctypes.byref(e), _device.stream_handle(dev)))
    ne = int(e.value)
    d_max = int((ro[1:] - ro[:-1]).max().item()) if rows else 0
    return DeviceCsrGraph(N, row_lo, rows, ne, ro, col, d_max)


def regular_row_host(N: int, d: int, seed: int, node: int) -> np.ndarray:
    """One row of the same construction evaluated on the host (tests)."""
    lib = _lib.load()
    out = np.zeros(max(1, d), dtype=np.int32)
    k = _lib.check(lib.fs_gen_regular_row_host(N, d, seed & ((1 << 64) - 1), node, out.ctypes.data))
    return out[:k].copy()


def _sized_generate(fn, args, N: int, row_lo: int, row_hi: int | None) -> DeviceCsrGraph:
    """Sizing call (offsets + edge count), then the fill call."""
    row_hi = N if row_hi is None else int(row_hi)
    if not 0 <= row_lo <= row_hi <= N:
        raise IndexOutOfRangeError("bad row range")
    dev = _device.device()
    st = _device.stream_handle(dev)
    rows = row_hi - row_lo
    ro = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    e = ctypes.c_int64()
    _lib.check(fn(*args, row_lo, row_hi, _lib.ptr(ro), None, 0, ctypes.byref(e), st))
    ne = int(e.value)
    col = torch.zeros(ne + 4, dtype=torch.int32, device=dev)
    _lib.check(fn(*args, row_lo, row_hi, _lib.ptr(ro), _lib.ptr(col), ne, ctypes.byref(e), st))
    d_max = int((ro[1:] - ro[:-1]).max().item()) if rows else 0
    return DeviceCsrGraph(N, row_lo, rows, ne, ro, col, d_max)


def gen_barabasi_albert_device(N: int, m: int, seed: int, row_lo: int = 0, row_hi: int | None = None) -> DeviceCsrGraph:
    """Preferential attachment from an m-clique (the model of the reference's
    gen_barabasi_albert, R/graph.py:331-365; same argument checks), built on
    the device by fs_gen_barabasi_albert.  Same law, not the same numpy draw
    stream: the graph differs from the reference's for the same seed."""
    if N < 2 or N > MAX_NODES:
        raise IndexOutOfRangeError("need 2 <= N <= 2^31-1")
    if not (1 <= m < N):
        raise InfeasibleDegreeSequenceError(f"need 1 <= m < N, got m={m}")
    lib = _lib.load()
    return _sized_generate(lib.fs_gen_barabasi_albert, (N, m, seed & ((1 << 64) - 1)), N, row_lo, row_hi)


def gen_erdos_renyi_device(N: int, d_avg: float, seed: int, row_lo: int = 0, row_hi: int | None = None) -> DeviceCsrGraph:
    """G(N, p), p = min(d_avg / (N-1), 1) (the model of the reference's
    gen_erdos_renyi, R/graph.py:252-286; same argument checks), built on the
    device by fs_gen_erdos_renyi."""
    if N < 2 or N > MAX_NODES:
        raise IndexOutOfRangeError("need N >= 2")
    if d_avg < 0:
        raise ValueError("d_avg must be >= 0")
    lib = _lib.load()
    return _sized_generate(lib.fs_gen_erdos_renyi, (N, float(d_avg), seed & ((1 << 64) - 1)), N, row_lo, row_hi)
