"""Host-side logic of the package (no GPU): generators, plans, configs, keys."""
import numpy as np
import pytest

from conftest import golden
from paper_2110_08450_b200 import (FanoutSpec, PrepConfig, SamplerVariant, SeedBatch,
                                   from_edge_list, list_variants, make_epoch_plan, size_hint_for,
                                   stream_key, synth_graph)
from paper_2110_08450_b200.sampler import (CounterRng, HopStream, _fmix, _fmix_inverse,
                                           hop_key_prefix)


def test_synth_graph_reproduces_reference_checksums():
    z = golden("graphs")
    for (n, seed, ne, ck, maxdeg), (avg, ex) in zip(z["spec_int"], z["spec_float"]):
        if n > 20000:
            continue  # the large specs are covered by test_oracle / GPU tests
        g = synth_graph(int(n), float(avg), float(ex), seed=int(seed))
        assert g.num_edges == ne and g.checksum() == ck and g.max_degree() == maxdeg


def test_small_graph_arrays(small_graph):
    z = golden("graphs")
    assert np.array_equal(small_graph.indptr, z["small_indptr"])
    assert np.array_equal(small_graph.indices, z["small_indices"])


def test_three_node_path_csr():
    g = from_edge_list([(0, 1), (1, 2)], 3, make_undirected=True)
    assert list(g.indptr) == [0, 1, 3, 4]
    assert list(g.indices) == [1, 0, 2, 1]


def test_bad_endpoint_reports_index():
    with pytest.raises(ValueError, match="edge 1"):
        from_edge_list([(0, 1), (0, 5)], 3)


def test_multi_edges_and_self_loops_preserved():
    g = from_edge_list([(0, 1), (0, 1), (2, 2)], 3)
    assert list(g.neighbors(0)) == [1, 1]
    assert list(g.neighbors(2)) == [2]


def test_stream_keys_match_reference():
    z = golden("rng")
    for q, k, p in zip(z["quad"], z["keys"], z["prefixes"]):
        assert stream_key(*map(int, q)) == int(k)
        assert HopStream(int(q[0]), int(q[1]), int(q[2])).key_prefix == int(p)
    for k, draws in zip(z["keys"], z["draws"]):
        r = CounterRng(int(k))
        assert [r.next_u64() for _ in range(8)] == [int(d) for d in draws]


def test_fmix_inverse():
    rng = np.random.default_rng(0)
    for z in rng.integers(0, 2**63, size=200, dtype=np.int64).tolist() + [0, 2**64 - 1]:
        assert _fmix(_fmix_inverse(z)) == z
        assert _fmix_inverse(_fmix(z)) == z


def test_epoch_plan_matches_reference():
    z = golden("prep_small")
    plan = make_epoch_plan(np.arange(1000), 128, 5)
    assert np.array_equal(np.concatenate([b.dst_ids for b in plan.batches]), z["plan_perm"])
    assert [b.batch_id for b in plan.batches] == list(range(8))


def test_epoch_plan_chunking_and_empty():
    plan = make_epoch_plan(np.arange(10), 4, shuffle_seed=0)
    assert [len(b) for b in plan.batches] == [4, 4, 2]
    assert len(make_epoch_plan([], 4, 0)) == 0
    with pytest.raises(ValueError):
        make_epoch_plan([1, 2], 0, 0)


def test_config_validation():
    with pytest.raises(ValueError):
        PrepConfig(num_workers=0)
    with pytest.raises(ValueError):
        PrepConfig(num_workers=1, delivery="whenever")
    with pytest.raises(ValueError):
        FanoutSpec(())
    with pytest.raises(ValueError):
        FanoutSpec((3, -1))
    with pytest.raises(ValueError):
        SeedBatch(0, np.array([1, 1, 2]))
    assert PrepConfig(num_workers=2).queue_capacity == 8
    # batches in flight: two per worker stream, inside the reference's pool bound
    assert PrepConfig(num_workers=1).depth == 2
    assert PrepConfig(num_workers=8).depth == 16
    assert PrepConfig(num_workers=1, queue_capacity=1).depth == 1
    assert PrepConfig(num_workers=3, queue_capacity=2).depth == 4


def test_variants():
    vs = list_variants()
    assert len(vs) == 18 and len({v.descriptor for v in vs}) == 18
    assert "flat_probing/vector_set/fused" in {v.descriptor for v in vs}
    for v in vs:
        assert SamplerVariant.from_descriptor(v.descriptor) == v
    with pytest.raises(ValueError):
        SamplerVariant.from_descriptor("nope")
    with pytest.raises(ValueError):
        SamplerVariant.from_descriptor("std_hash/hash_set/maybe")


def test_size_hint():
    assert size_hint_for(1024, FanoutSpec((15, 10, 5)), 10**9) == 1024 * 6 * 11 * 16
    assert size_hint_for(1024, FanoutSpec((15, 10, 5)), 5000) == 5000


def test_hop_key_prefix_host_matches_capi():
    from paper_2110_08450_b200 import _lib
    L = _lib.lib()
    for s, b, h in [(0, 0, 0), (1, 5, 2), (2**63 + 5, 1171, 7)]:
        assert L.sal_hop_key_prefix(s, b, h) == hop_key_prefix(s, b, h)
