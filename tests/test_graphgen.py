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


# ---------------------------------------------------- BA and G(N, p) (fs_gen_random.cu) --

def _structure_checks(h, n):
    ro, col = h.row_offsets, h.col_indices
    src = np.repeat(np.arange(n), np.diff(ro))
    assert np.all(col >= 0) and np.all(col < n)
    assert not np.any(src == col)                                         # no self-loops
    for i in range(0, n, max(1, n // 500)):                               # sorted, no duplicates
        r = col[ro[i]:ro[i + 1]]
        assert np.all(r[1:] > r[:-1])
    fwd = src.astype(np.int64) * n + col
    bwd = col.astype(np.int64) * n + src
    assert np.array_equal(np.sort(fwd), np.sort(bwd))                     # symmetric
    return src, col


@pytest.mark.gpu
@pytest.mark.parametrize("n,m", [(20_000, 5), (3_000, 1), (500, 3), (2, 1), (64, 63)])
def test_ba_device_structure(n, m):
    g = fs.gen_barabasi_albert_device(n, m, seed=4)
    h = g.to_host()
    assert g.num_edges == 2 * ((n - m) * m + m * (m - 1) // 2)           # the reference's edge count
    src, col = _structure_checks(h, n)
    earlier = np.bincount(src[col < src], minlength=n)                   # each new node attaches to m
    assert np.all(earlier[m:] == m)
    assert np.all(earlier[:m] == np.arange(m))                           # the m-clique seed
    again = fs.gen_barabasi_albert_device(n, m, seed=4).to_host()
    assert np.array_equal(again.col_indices, h.col_indices)              # deterministic for a seed


@pytest.mark.gpu
def test_ba_device_degree_law_matches_reference_generator():
    """Same attachment law as the reference's generator (host port):
    degree-m fraction (BA theory 2/(m+2)), mean log-degree, hub sizes."""
    n, m = 20_000, 5
    dev = np.diff(fs.gen_barabasi_albert_device(n, m, seed=1).row_offsets)
    ref = np.diff(fs.gen_barabasi_albert(n, m, seed=1).row_offsets)
    assert dev.sum() == ref.sum() and dev.min() == ref.min() == m
    assert abs(np.mean(dev == m) - np.mean(ref == m)) < 0.02
    assert abs(np.mean(np.log(dev)) - np.mean(np.log(ref))) < 0.02
    top_d, top_r = np.sort(dev)[-20:].mean(), np.sort(ref)[-20:].mean()
    assert 0.5 < top_d / top_r < 2.0
    # CCDF tail exponent ~ 2 for both (P(k >= x) ~ x^-2)
    for d in (dev, ref):
        f1, f2 = np.mean(d >= 20), np.mean(d >= 80)
        assert 10 < f1 / f2 < 24


@pytest.mark.gpu
@pytest.mark.parametrize("n,d", [(20_000, 8.0), (3_001, 2.5), (50, 100.0), (10, 0.0), (1_000, 999.0)])
def test_er_device_structure_and_law(n, d):
    g = fs.gen_erdos_renyi_device(n, d, seed=6)
    h = g.to_host()
    p = min(d / (n - 1), 1.0)
    pairs = n * (n - 1) // 2
    if p >= 1.0:
        assert g.num_edges == 2 * pairs
    elif p == 0.0:
        assert g.num_edges == 0
    else:
        mu, sd = pairs * p, np.sqrt(pairs * p * (1 - p))
        assert abs(g.num_edges / 2 - mu) < 6 * sd
    if g.num_edges:
        _structure_checks(h, n)
    if 0 < p < 1 and n >= 3000:
        deg = np.diff(h.row_offsets)
        assert abs(deg.var() / deg.mean() - (1 - p)) < 0.1                # binomial degrees
    again = fs.gen_erdos_renyi_device(n, d, seed=6).to_host()
    assert np.array_equal(again.col_indices, h.col_indices)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["ba", "er"])
def test_random_generators_partition_slices(kind):
    n = 30_000
    gen = (lambda **kw: fs.gen_barabasi_albert_device(n, 5, seed=2, **kw)) if kind == "ba" else \
          (lambda **kw: fs.gen_erdos_renyi_device(n, 10.0, seed=2, **kw))
    whole = gen().to_host()
    cuts = [0, 7_168, 19_456, n]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        part = gen(row_lo=lo, row_hi=hi)
        assert np.array_equal(part.row_offsets + whole.row_offsets[lo], whole.row_offsets[lo:hi + 1])
        assert np.array_equal(part.col_indices, whole.col_indices[whole.row_offsets[lo]:whole.row_offsets[hi]])


@pytest.mark.gpu
def test_engine_on_device_ba_graph_matches_oracle():
    """C3's graph family built on the device: the merge-strategy engine
    (hub rows) is bit-exact against the oracle on it."""
    from oracle import spreadsim_port as O

    g = fs.gen_barabasi_albert_device(20_000, 5, seed=1)
    h = g.to_host()
    m = fs.seir_weibull_erlang(0.25)
    cfg = fs.RenewalConfig()
    st = fs.init_renewal_state(g, m, cfg, 7)
    ref = O.init_state(h, m, cfg, 7)
    for _ in range(2):
        fs.run_batch(st, g, m, cfg, 7)
        O.run_batch(ref, h, m, cfg, 7)
    assert np.array_equal(st.counts, ref.counts)
    assert np.array_equal(st.states.astype(np.int32), ref.states.astype(np.int32))
    assert np.array_equal(st.ages.view(np.uint32), ref.ages.view(np.uint32))
    assert st.clock == ref.clock


@pytest.mark.parametrize("fn,args", [("gen_barabasi_albert_device", (10, 10)), ("gen_barabasi_albert_device", (10, 0)),
                                     ("gen_barabasi_albert_device", (1, 1)), ("gen_erdos_renyi_device", (1, 2.0)),
                                     ("gen_erdos_renyi_device", (10, -1.0))])
def test_random_generator_argument_checks(fn, args):
    with pytest.raises((fs.errors.GraphError, ValueError)):
        getattr(fs, fn)(*args, seed=0)
