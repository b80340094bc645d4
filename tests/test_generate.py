"""The synthetic-input generator's law, on its host restatement (oracle.synth_graph_host).

graph.synth_graph_device (csrc/generate.cu) builds the benchmark graphs in HBM;
oracle.synth_graph_host rebuilds the same arrays bit for bit on the host
(tests/test_gpu_generate.py checks the equality on a B200).  These CPU tests
check that those arrays follow the reference's synth_graph law
(graph.py:252-280): a Pareto(a = exponent - 1) degree sequence with mean
avg_degree, stubs paired uniformly (configuration model, self loops and
multi-edges kept), every pair stored in both directions; features uniform
[-1, 1] rounded to fp16 (graph.py:283-292); labels uniform (graph.py:295-298).
"""

import numpy as np
import pytest

import oracle as O
from paper_2110_08450_b200 import synth_graph


@pytest.fixture(scope="module")
def g200k():
    return O.synth_graph_host(200_000, 14.55, 3.0, seed=5, num_features=100, num_classes=47,
                              nthreads=4)


def owners(indptr):
    return np.repeat(np.arange(len(indptr) - 1, dtype=np.int64), np.diff(indptr))


def test_deterministic_and_seeded():
    a = O.synth_graph_host(1000, 10, 3.0, seed=7)
    b = O.synth_graph_host(1000, 10, 3.0, seed=7, nthreads=3)
    c = O.synth_graph_host(1000, 10, 3.0, seed=8)
    assert np.array_equal(a["indptr"], b["indptr"]) and np.array_equal(a["indices"], b["indices"])
    assert not (np.array_equal(a["indptr"], c["indptr"]) and
                np.array_equal(a["indices"], c["indices"]))


def test_edge_count_like_reference():
    # reference test_graph.py:121-124
    g = O.synth_graph_host(1000, 10, 3.0, seed=7)
    pairs = g["indptr"][-1] / 2
    assert abs(pairs - 5000) / 5000 < 0.05


def test_csr_valid_and_in_range(g200k):
    ip, ind = g200k["indptr"], g200k["indices"]
    assert ip[0] == 0 and ip[-1] == len(ind) and ip[-1] % 2 == 0
    assert np.all(np.diff(ip) >= 0)
    assert ind.min() >= 0 and ind.max() < 200_000
    # mean degree (slots per node) within 3 % of avg_degree (Pareto a = 2: slow mean convergence)
    assert abs(ip[-1] / 200_000 - 14.55) / 14.55 < 0.03


def test_pairing_is_a_symmetric_matching(g200k):
    """Every stored slot (u -> v) has its mirror (v -> u): the directed slot
    multiset equals its transpose (make_undirected=True, graph.py:279)."""
    ip, ind = g200k["indptr"], g200k["indices"].astype(np.int64)
    u = owners(ip)
    n = 200_000
    fwd = np.sort(u * n + ind)
    rev = np.sort(ind * n + u)
    assert np.array_equal(fwd, rev)


def test_degree_law_chi2(g200k):
    """Degrees against the exact law: P(deg <= k) = 1 - (scale / (k + 1/2))^a."""
    from scipy import stats
    n, avg, a = 200_000, 14.55, 2.0
    scale = avg * (a - 1.0) / a
    deg = np.diff(g200k["indptr"])
    edges = np.array([0, 8, 9, 10, 11, 12, 14, 16, 19, 23, 30, 45, 80, 200, 10**9], dtype=np.float64)
    cdf = lambda k: np.where(k + 0.5 > scale, 1.0 - (scale / (k + 0.5)) ** a, 0.0)
    # bin j holds degrees in (edges[j], edges[j+1]]
    p = np.diff(cdf(edges))
    p[0] += cdf(edges[0])
    obs = np.histogram(deg, bins=np.concatenate([[-1], edges[1:]]) + 0.5)[0]
    exp = p / p.sum() * n
    chi2 = ((obs - exp) ** 2 / exp).sum()
    assert stats.chi2.sf(chi2, len(obs) - 1) > 1e-4, (obs, exp.round())


def test_degree_law_ks_vs_reference_generator():
    """Two-sample KS of the degree sequence against the reference's own
    synth_graph (graph.synth_graph reproduces it bit for bit, test_host)."""
    from scipy import stats
    ref = np.diff(synth_graph(100_000, 14.55, 3.0, seed=11).indptr)
    ours = np.diff(O.synth_graph_host(100_000, 14.55, 3.0, seed=11)["indptr"])
    assert stats.ks_2samp(ref, ours).pvalue > 1e-3


def test_pairing_uniform_between_degree_classes(g200k):
    """Configuration model: slots of u land on v's stubs with probability
    d_v / (2m - 1).  Edges between the low- and high-degree halves of the stubs
    match d_lo d_hi / 2m; self-loops match sum C(d, 2) / (2m - 1)."""
    ip, ind = g200k["indptr"], g200k["indices"].astype(np.int64)
    deg = np.diff(ip)
    u = owners(ip)
    two_m = float(ip[-1])
    hi = deg >= np.median(deg[deg > 0]) + 3
    s_hi = deg[hi].sum()
    s_lo = two_m - s_hi
    cross = np.count_nonzero(hi[u] & ~hi[ind])
    expect = s_hi * s_lo / two_m
    assert abs(cross - expect) / expect < 0.02
    loops = np.count_nonzero(u == ind) / 2
    exp_loops = float((deg * (deg - 1) / 2).sum()) / (two_m - 1)
    assert abs(loops - exp_loops) < 6 * np.sqrt(exp_loops) + 5


def test_features_uniform_fp16(g200k):
    x = g200k["features"]
    assert x.shape == (200_000, 104) and x.dtype == np.float16   # host default stride
    assert not np.any(x[:, 100:])                     # padding columns stay zero
    v = x[:, :100].astype(np.float32)
    assert v.min() >= -1.0 and v.max() <= 1.0
    assert abs(v.mean()) < 2e-3 and abs(v.var() - 1.0 / 3.0) < 2e-3
    # fp16 rounding of the host restatement = numpy's round-to-nearest-even
    rng = np.random.default_rng(0)
    for f in np.concatenate([rng.uniform(-1, 1, 2000), rng.standard_normal(2000) * 1e-5,
                             [2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26, 65504.0, 1e-8, -1.0]]
                            ).astype(np.float32):
        assert O.f32_to_f16_bits(float(f)) == int(np.float32(f).astype(np.float16).view(np.uint16))


def test_labels_uniform(g200k):
    y = g200k["labels"]
    assert y.min() >= 0 and y.max() < 47
    cnt = np.bincount(y, minlength=47)
    from scipy import stats
    assert stats.chisquare(cnt).pvalue > 1e-4
