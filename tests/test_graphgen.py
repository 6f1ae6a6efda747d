"""GPU uniform-degree generator (csrc/fs_graphgen.cu).

CPU tests evaluate the construction row by row through the library's host
entry point (no device): degree, sortedness, no self-loops, symmetry.  GPU
tests check the device CSR against the host rows, partition slices against
the whole graph, and run the engine on a generated graph bit-exactly
against the oracle.
"""

import numpy as np
import pytest

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200.devgraph import regular_row_host


@pytest.mark.parametrize("n,k", [(1000, 10), (1001, 10), (1000, 7), (64, 4), (5, 2), (2, 1), (4098, 3)])
def test_regular_rows_host_properties(n, k):
    rows = [regular_row_host(n, k, 11, i) for i in range(n)]
    deg = np.array([r.size for r in rows])
    assert deg.max() <= k and deg.min() >= max(0, k - 4)
    assert (deg == k).mean() > (0.9 if n > 100 else 0.0)
    for i, r in enumerate(rows):
        assert (np.diff(r) > 0).all()          # sorted, no duplicates
        assert not (r == i).any()              # no self-loops
        assert r.min(initial=0) >= 0 and r.max(initial=0) < n
    adj = {(i, int(j)) for i, r in enumerate(rows) for j in r}
    assert all((j, i) in adj for i, j in adj)  # undirected: symmetric


def test_regular_rows_depend_on_seed():
    a = [regular_row_host(5000, 10, 1, i) for i in range(50)]
    b = [regular_row_host(5000, 10, 2, i) for i in range(50)]
    assert sum(np.array_equal(x, y) for x, y in zip(a, b)) < 5


def test_regular_argument_checks():
    with pytest.raises(fs.errors.InfeasibleDegreeSequenceError):
        fs.gen_fixed_degree_device(11, 3, seed=1)      # N*d odd
    with pytest.raises(fs.errors.InfeasibleDegreeSequenceError):
        fs.gen_fixed_degree_device(10, 10, seed=1)     # d >= N


@pytest.mark.gpu
@pytest.mark.parametrize("n,k", [(20_000, 10), (4098, 3), (1000, 7)])
def test_device_generator_matches_host_rows(n, k):
    g = fs.gen_fixed_degree_device(n, k, seed=5)
    h = g.to_host()
    h.validate()
    assert g.num_edges == h.row_offsets[-1]
    for i in list(range(50)) + list(range(n - 50, n)):
        assert np.array_equal(h.col_indices[h.row_offsets[i]:h.row_offsets[i + 1]], regular_row_host(n, k, 5, i))
    # the transpose of an undirected graph is itself
    t = fs.transpose(h)
    assert np.array_equal(t.row_offsets, h.row_offsets) and np.array_equal(t.col_indices, h.col_indices)


@pytest.mark.gpu
def test_device_generator_partition_slices():
    n, k = 30_000, 10
    whole = fs.gen_fixed_degree_device(n, k, seed=9).to_host()
    cuts = [0, 7_168, 19_456, n]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        part = fs.gen_fixed_degree_device(n, k, seed=9, row_lo=lo, row_hi=hi)
        ro = part.row_offsets
        assert np.array_equal(ro + whole.row_offsets[lo], whole.row_offsets[lo:hi + 1])
        assert np.array_equal(part.col_indices, whole.col_indices[whole.row_offsets[lo]:whole.row_offsets[hi]])


@pytest.mark.gpu
def test_engine_on_generated_graph_matches_oracle():
    from oracle import spreadsim_port as O

    g = fs.gen_fixed_degree_device(20_000, 10, seed=3)
    h = g.to_host()
    m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
    for mixed in (False, True):
        cfg = fs.RenewalConfig(mixed_precision=mixed)
        st = fs.init_renewal_state(g, m, cfg, 7)
        ref = O.init_state(h, m, cfg, 7)
        fs.run_batch(st, g, m, cfg, 7)
        O.run_batch(ref, h, m, cfg, 7)
        assert np.array_equal(st.counts, ref.counts)
        assert np.array_equal(st.states.astype(np.int32), ref.states.astype(np.int32))
        assert np.array_equal(st.ages.view(np.uint16 if mixed else np.uint32),
                              ref.ages.view(np.uint16 if mixed else np.uint32))
        assert st.clock == ref.clock
