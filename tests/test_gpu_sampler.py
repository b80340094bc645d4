"""GPU parity of the sampler / MFG construction against reference goldens + oracle."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import assert_mfg_equal, golden, golden_mfg
from paper_2110_08450_b200 import (DeviceGraph, FanoutSpec, HopStream, IdMap, SamplerVariant,
                                   SeedBatch, from_edge_list, list_variants, make_epoch_plan,
                                   multihop_mfg, one_hop_mfg, sample_neighbors, synth_graph)
from paper_2110_08450_b200.sampler import CounterRng, stream_key

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dg_small(small_graph):
    return DeviceGraph.from_host(small_graph)


def _host(mfg):
    gids, layers = mfg.to_host()
    return gids, layers


@pytest.mark.parametrize("case", list("abcdef"))
def test_multihop_bit_exact_vs_reference(case, mfg_small, dg_small):
    z = mfg_small
    seeds = SeedBatch(int(z[f"{case}_batch"]), z[f"{case}_seeds"])
    mfg = multihop_mfg(dg_small, seeds, FanoutSpec(tuple(z[f"{case}_fan"])),
                       int(z[f"{case}_gseed"]), SamplerVariant())
    want_g, want_l = golden_mfg(z, f"{case}_")
    assert_mfg_equal(*_host(mfg), want_g, want_l)
    assert mfg.digest() == str(z[f"{case}_digest"])


def test_all_variants_accepted_and_equal(mfg_small, dg_small):
    z = mfg_small
    seeds = SeedBatch(0, z["a_seeds"])
    digests = {multihop_mfg(dg_small, seeds, FanoutSpec((15, 10, 5)), 9, v).digest()
               for v in list_variants()}
    assert digests == {str(z["a_digest"])}


def test_one_hop_tiny_example():
    g = from_edge_list([(7, 2), (7, 9)], 10)
    seeds = SeedBatch(0, np.array([7]))
    idm = IdMap(SamplerVariant())
    idm.insert(seeds.dst_ids)
    layer = one_hop_mfg(g, seeds, 5, HopStream(0, 0, 0), SamplerVariant(), idm)
    assert idm.global_ids.tolist() == [7, 2, 9]
    assert layer.num_dst == 1 and layer.num_src == 3
    assert layer.indptr.tolist() == [0, 2]
    assert layer.src_local.tolist() == [1, 2]


def test_one_hop_isolated_dst():
    g = from_edge_list([(0, 1)], 3)
    idm = IdMap(SamplerVariant())
    idm.insert(np.array([2]))
    layer = one_hop_mfg(g, SeedBatch(0, np.array([2])), 4, HopStream(0, 0, 0),
                        SamplerVariant(), idm)
    assert layer.num_dst == 1 and layer.num_edges == 0


def test_multi_edge_slots_can_repeat_neighbor():
    g = from_edge_list([(0, 1), (0, 1)], 2)
    idm = IdMap(SamplerVariant())
    idm.insert(np.array([0]))
    layer = one_hop_mfg(g, SeedBatch(0, np.array([0])), 5, HopStream(0, 0, 0),
                        SamplerVariant(), idm)
    assert layer.src_local.tolist() == [1, 1]


def test_one_hop_prefix_mismatch_raises(dg_small):
    idm = IdMap(SamplerVariant())
    idm.insert(np.array([1, 2, 3]))
    with pytest.raises(ValueError, match="prefix"):
        one_hop_mfg(dg_small, SeedBatch(0, np.array([2, 1])), 3, HopStream(0, 0, 0),
                    SamplerVariant(), idm)
    with pytest.raises(ValueError, match="exceeds"):
        one_hop_mfg(dg_small, 5, 3, HopStream(0, 0, 0), SamplerVariant(), idm)


def test_single_hop_chain_equals_one_hop(dg_small, mfg_small):
    z = mfg_small
    seeds = SeedBatch(0, z["seeds64"])
    mfg = multihop_mfg(dg_small, seeds, FanoutSpec((4,)), 5, SamplerVariant())
    idm = IdMap(SamplerVariant())
    idm.insert(seeds.dst_ids)
    layer = one_hop_mfg(dg_small, seeds, 4, HopStream(5, 0, 0), SamplerVariant(), idm)
    assert mfg.layers[0].structurally_equal(layer)
    assert torch.equal(mfg.id_map.global_ids, idm.global_ids)


def test_idmap_insert_duplicates_matches_reference(mfg_small):
    idm = IdMap(SamplerVariant())
    idm.insert(np.array([5, 9, 5, 3]))
    idm.insert(np.array([3, 11, 9, 12, 11]))
    assert idm.global_ids.tolist() == mfg_small["idmap_globals"].tolist()
    assert idm.local_of(12) == 4 and idm.global_of(1) == 9


def test_idmap_growth_rehash():
    idm = IdMap(SamplerVariant(), size_hint=1)
    keys = np.random.default_rng(0).permutation(5000)[:3000]
    for chunk in np.array_split(keys, 7):
        idm.insert(chunk)
    assert idm.global_ids.cpu().numpy().tolist() == keys.tolist()
    idm.insert(keys[::-1])
    assert idm.size == 3000


def test_idmap_insert_many_tiles_of_duplicates():
    """One insert spanning hundreds of scan tiles whose first occurrences sit in earlier
    tiles (the chain's last relabel resolves in its scan launch, waiting on the tile that
    holds each first occurrence): new locals in first-occurrence order, and the slots
    finalized for the next insert."""
    rng = np.random.default_rng(3)
    idm = IdMap(SamplerVariant())
    pre = rng.permutation(20000)[:700]
    idm.insert(pre)
    keys = rng.integers(0, 20000, 300_000)
    keys[:50] = keys[-50:]             # the last tile's keys first seen in tile 0
    idm.insert(keys)
    _, first = np.unique(keys, return_index=True)
    order = keys[np.sort(first)]
    want = np.concatenate([pre, order[~np.isin(order, pre)]])
    got = idm.global_ids.cpu().numpy()
    assert got.tolist() == want.tolist()
    for k in (int(keys[-1]), int(keys[150_000]), int(pre[3])):
        assert idm.local_of(k) == int(np.flatnonzero(want == k)[0])
    idm.insert(keys[::-3])
    assert idm.size == len(want)


def test_injected_positions_reproduce_hop(dg_small, mfg_small):
    """Sampling driven by the reference's own pos_all (hop_kernel two-pass)."""
    z = mfg_small
    seeds = SeedBatch(0, z["seeds64"])
    idm = IdMap(SamplerVariant())
    idm.insert(seeds.dst_ids)
    # a wrong key proves the positions come from the injection, not the draws
    layer = one_hop_mfg(dg_small, seeds, 5, HopStream(12345, 9, 3), SamplerVariant(), idm,
                        inject_pos=z["inject_pos"])
    assert layer.indptr.cpu().numpy().tolist() == z["inject_indptr"].tolist()
    assert layer.src_local.cpu().numpy().tolist() == z["inject_src"].tolist()


def test_sample_neighbors_vs_reference_oracle(small_graph, dg_small):
    z = golden("rng")
    for v in range(0, 300, 7):
        key = stream_key(42, 0, 0, v)
        rng = CounterRng(key)
        got = sample_neighbors(dg_small, v, 3, rng)
        want = O.sample_positions(key, small_graph.degree(v), 3)
        assert got.tolist() == want
        if small_graph.degree(v) <= 3:
            assert rng.counter == 0
        else:
            # replaying the host stream for rng.counter draws gives the same set
            h = CounterRng(key)
            draws = [h.next_below(small_graph.degree(v)) for _ in range(rng.counter)]
            assert set(draws) == set(want) and draws[-1] == want[-1]


def test_sample_neighbors_continues_an_advanced_stream(small_graph, dg_small):
    """Several calls on one CounterRng (reference sampler.py:253-273): each call picks
    up the stream where the previous one left it, exactly like the host loop."""
    def host_sample(deg, d, rng):   # the reference's sequential rejection sampler
        if deg <= d:
            return list(range(deg))
        seen, out = set(), []
        while len(out) < d:
            pos = rng.next_below(deg)
            if pos not in seen:
                seen.add(pos)
                out.append(pos)
        return out

    for v in (v for v in range(0, 400, 3) if small_graph.degree(v) > 3):
        key = stream_key(7, 1, 2, v)
        dev, host = CounterRng(key), CounterRng(key)
        for _ in range(3):
            got = sample_neighbors(dg_small, v, 3, dev)
            assert got.tolist() == host_sample(small_graph.degree(v), 3, host)
            assert dev.counter == host.counter


def test_large_fanout_path(dg_small, small_graph):
    """fanout > 32 (global-memory accepted set) vs oracle."""
    seeds = SeedBatch(4, np.arange(0, 1000, 9))
    for fan in [(40, 33), (64,), (100, 2)]:
        mfg = multihop_mfg(dg_small, seeds, FanoutSpec(fan), 77, SamplerVariant())
        gids, layers = O.multihop(small_graph.indptr, small_graph.indices, 1000, seeds.dst_ids,
                                  fan, 77, 4)
        assert_mfg_equal(*_host(mfg), gids, layers)


def test_fanout_zero_and_unbounded(dg_small, small_graph):
    seeds = SeedBatch(0, np.arange(10))
    m0 = multihop_mfg(dg_small, seeds, FanoutSpec((0, 0)), 1, SamplerVariant())
    assert m0.num_nodes == 10 and m0.num_edges == 0
    d = small_graph.max_degree()
    mb = multihop_mfg(dg_small, seeds, FanoutSpec((d, d, d)), 1, SamplerVariant())
    gids, layers = O.multihop(small_graph.indptr, small_graph.indices, 1000, seeds.dst_ids,
                              (d, d, d), 1, 0)
    assert_mfg_equal(*_host(mb), gids, layers)


def test_empty_seed_batch(dg_small):
    m = multihop_mfg(dg_small, SeedBatch(0, np.array([], dtype=np.int64)), FanoutSpec((3, 2)),
                     1, SamplerVariant())
    assert m.num_nodes == 0 and m.num_edges == 0
    assert all(l.num_dst == 0 for l in m.layers)


def test_config1_batches_bit_exact():
    """BASELINE config 1 (100K / 991K slots), batch 1024, (15,10,5), 5 reference batches."""
    z = golden("config1")
    g = synth_graph(100_000, 10, 3.0, seed=1)
    assert g.checksum() == int(z["checksum"])
    dg = DeviceGraph.from_host(g)
    plan = make_epoch_plan(np.arange(100_000), 1024, 1)
    picks = list(plan.batches[:4]) + [plan.batches[-1]]
    for b, want in zip(picks, z["mfg_digests"]):
        assert multihop_mfg(dg, b, FanoutSpec((15, 10, 5)), 1).digest() == str(want)
    m0 = multihop_mfg(dg, plan.batches[0], FanoutSpec((15, 10, 5)), 1)
    gids, layers = m0.to_host()
    assert np.array_equal(gids, z["b0_global_ids"].astype(np.int64))
    for i, l in enumerate(layers):
        assert np.array_equal(l["indptr"], z[f"b0_l{i}_indptr"].astype(np.int64))
        assert np.array_equal(l["src_local"], z[f"b0_l{i}_src"].astype(np.int64))
    for tag, fan in (("paper", (5, 10, 15)), ("infer", (20, 20, 20))):
        assert multihop_mfg(dg, plan.batches[0], FanoutSpec(fan), 1).digest() == \
            str(z[f"{tag}_digest"])


def test_philox_policy_invariants(dg_small, small_graph):
    """Philox policy: fanout bound exact, positions distinct, deterministic."""
    seeds = SeedBatch(3, np.arange(0, 1000, 4))
    fan = FanoutSpec((15, 10, 5))
    a = multihop_mfg(dg_small, seeds, fan, 11, rng_policy="philox")
    b = multihop_mfg(dg_small, seeds, fan, 11, rng_policy="philox")
    assert a.digest() == b.digest()
    gids, layers = a.to_host()
    deg = np.diff(small_graph.indptr)
    for lay, f in zip(layers, fan.per_hop):
        indeg = np.diff(lay["indptr"])
        assert np.array_equal(indeg, np.minimum(deg[gids[:lay["num_dst"]]], f))


def test_philox_uniform_without_replacement():
    """Per-node statistical test: star node of degree 40, fanout 10, 4000 batches.

    Each slot must be chosen with probability f/deg = 0.25; chi-square over
    the 40 slots (39 dof) must pass at p > 1e-4, and no slot repeats.
    """
    deg, f, trials = 40, 10, 4000
    edges = [(0, 1 + k) for k in range(deg)]
    g = DeviceGraph.from_host(from_edge_list(edges, deg + 1))
    counts = np.zeros(deg, dtype=np.int64)
    for t in range(trials):
        m = multihop_mfg(g, SeedBatch(t, np.array([0])), FanoutSpec((f,)), 5,
                         rng_policy="philox")
        gids, layers = m.to_host()
        nb = gids[layers[0]["src_local"]] - 1
        assert len(set(nb.tolist())) == f
        counts[nb] += 1
    expected = trials * f / deg
    chi2 = float(((counts - expected) ** 2 / expected).sum())
    # chi-square(39) upper 1e-4 quantile ~ 83.3 (fpc makes the statistic smaller)
    assert chi2 < 83.3, (chi2, counts)


@pytest.mark.parametrize("fan", [(15, 10, 5), (4, 3), (6,)])
def test_last_hop_edges_only_matches_full_sample(fan):
    """SAL_MFG_LAST_HOP_EDGES: hops 0..L-2 identical to the full sample, the last
    hop's edges identical as global ids (against the reference-exact full MFG),
    sizes[L] = -1."""
    from paper_2110_08450_b200.sampler import MfgWorkspace
    g = synth_graph(100_000, 10, 3.0, seed=1)
    dg = DeviceGraph.from_host(g)
    plan = make_epoch_plan(np.arange(100_000), 1024, 1)
    spec = FanoutSpec(fan)
    full = MfgWorkspace(dg.num_nodes, spec, 1024)
    edg = MfgWorkspace(dg.num_nodes, spec, 1024, last_hop_edges=True)
    assert edg.plan.table_cap <= full.plan.table_cap
    L = len(fan)
    for b in (plan.batches[0], plan.batches[-1]):
        for ws in (full, edg):
            ws.load_seeds(b)
            ws.run(dg, ws.seeds, ws.desc, 1)
        torch.cuda.synchronize()
        sf, ef = full.read_extents()
        se, ee = edg.read_extents()
        assert se[:L] == sf[:L] and ee == ef and se[L] == -1
        assert torch.equal(edg.globals[:sf[L - 1]], full.globals[:sf[L - 1]])
        for h in range(L):
            assert torch.equal(edg.dst_indptr[h][:sf[h] + 1], full.dst_indptr[h][:sf[h] + 1])
        for h in range(L - 1):
            assert torch.equal(edg.src_local[h][:ef[h]], full.src_local[h][:ef[h]])
        want = full.globals[full.src_local[L - 1][:ef[L - 1]].long()]
        assert torch.equal(edg.src_glob[:ef[L - 1]], want)
        with pytest.raises(ValueError):
            edg.to_mfg(b)


def _star_forest(k: int, degs: np.ndarray):
    """k hubs (ids 0..k-1), hub i linked to degs[i] private leaves, as a device CSR."""
    n = k + int(degs.sum())
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:k + 1] = np.cumsum(degs)
    indptr[k + 1:] = indptr[k]
    indices = (k + np.arange(int(degs.sum()))).astype(np.int32)
    return DeviceGraph(n, torch.from_numpy(indptr).cuda(), torch.from_numpy(indices).cuda()), indptr


def _sampled_positions(dg, indptr, k, f, policy, batch_id=0, seed=5):
    """Slot positions sampled for hubs 0..k-1 in one hop (one batch of k seeds)."""
    m = multihop_mfg(dg, SeedBatch(batch_id, np.arange(k)), FanoutSpec((f,)), seed,
                     rng_policy=policy)
    gids, layers = m.to_host()
    ip, src = layers[0]["indptr"], gids[layers[0]["src_local"]]
    pos = src - k - indptr[np.repeat(np.arange(k), np.diff(ip))]
    return [pos[ip[i]:ip[i + 1]] for i in range(k)]


@pytest.mark.parametrize("policy", ["philox", "splitmix"])
def test_subset_frequencies_chi2(policy):
    """Joint uniformity, not just marginals: 20,000 nodes of degree 6 at fanout 3 —
    each of the C(6,3) = 20 subsets must come up equally often (chi-square, 19 dof,
    p > 1e-4), and each node's sample is 3 distinct positions.  A sampler drawing a
    random contiguous window (uniform marginals) fails this."""
    from itertools import combinations
    from scipy import stats
    k, d, f = 20_000, 6, 3
    dg, indptr = _star_forest(k, np.full(k, d))
    idx = {c: i for i, c in enumerate(combinations(range(d), f))}
    counts = np.zeros(len(idx), dtype=np.int64)
    for p in _sampled_positions(dg, indptr, k, f, policy):
        assert len(set(p.tolist())) == f
        counts[idx[tuple(sorted(p.tolist()))]] += 1
    assert stats.chisquare(counts).pvalue > 1e-4, counts


@pytest.mark.parametrize("policy", ["philox", "splitmix"])
def test_pairwise_inclusion_by_degree(policy):
    """Pairwise inclusion over nodes of degree 4..12 at fanout 3: P(i and j both
    sampled) = f(f-1) / (d(d-1)) for every pair of slots (uniform sampling without
    replacement); chi-square per degree over the C(d,2) pair counts, plus the
    first-order rate f/d per slot."""
    from scipy import stats
    f, per = 3, 3000
    degs = np.repeat(np.arange(4, 13), per)
    k = len(degs)
    dg, indptr = _star_forest(k, degs)
    samples = _sampled_positions(dg, indptr, k, f, policy, batch_id=3, seed=9)
    for d in range(4, 13):
        pair = np.zeros((d, d), dtype=np.int64)
        single = np.zeros(d, dtype=np.int64)
        for i in np.nonzero(degs == d)[0]:
            p = np.sort(samples[i])
            single[p] += 1
            for a in range(f):
                for b in range(a + 1, f):
                    pair[p[a], p[b]] += 1
        iu = np.triu_indices(d, 1)
        obs = pair[iu]
        assert obs.sum() == per * f * (f - 1) // 2
        assert stats.chisquare(obs).pvalue > 1e-4, (d, obs)
        assert stats.chisquare(single).pvalue > 1e-4, (d, single)


@pytest.mark.parametrize("fused", [False, True])
def test_sample_mfg_next_equals_plan_next_then_sample(fused):
    """sal_sample_mfg_next (the plan cursor folded into the seed-insertion kernel) gives
    the descriptor, cursor and MFG of sal_plan_next followed by sal_sample_mfg, step
    after step, including the empty batch past the end of the plan."""
    from paper_2110_08450_b200 import _lib
    from paper_2110_08450_b200.graph import synth_graph_device
    from paper_2110_08450_b200.sampler import MfgWorkspace
    g = synth_graph_device(50_000, 12.0, 3.0, seed=3, num_features=16, num_classes=4,
                           feature_seed=3, label_seed=3)
    rng = np.random.default_rng(5)
    perm = torch.from_numpy(rng.permutation(g.num_nodes)[:3000].astype(np.int64)).cuda()
    desc_all = torch.tensor([[7, 0, 1024], [3, 1024, 1024], [9, 2048, 952]],
                            dtype=torch.int64, device="cuda")
    fan = FanoutSpec((15, 10, 5))
    kw = dict(device="cuda", last_hop_fused=fused)
    a, b = MfgWorkspace(g.num_nodes, fan, 1024, **kw), MfgWorkspace(g.num_nodes, fan, 1024, **kw)
    ca = torch.zeros(1, dtype=torch.int64, device="cuda")
    cb = torch.zeros(1, dtype=torch.int64, device="cuda")
    da = torch.zeros(3, dtype=torch.int64, device="cuda")
    db = torch.zeros(3, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    for step in range(4):
        _lib.check(L.sal_plan_next(desc_all.data_ptr(), 3, ca.data_ptr(), da.data_ptr(),
                                   _lib.stream_ptr()), "plan_next")
        a.run(g, perm, da, 11, 0)
        b.run_next(g, perm, desc_all, 3, cb, db, 11, 0)
        assert torch.equal(da, db) and int(cb.item()) == step + 1 == int(ca.item())
        assert torch.equal(a.sizes, b.sizes) and torch.equal(a.etot, b.etot)
        h = a.num_hops - (1 if fused else 0)
        for k in range(h):
            n, e = int(a.sizes[k].item()), int(a.etot[k].item())
            assert torch.equal(a.dst_indptr[k][:n + 1], b.dst_indptr[k][:n + 1])
            if not (fused and k == h - 1):   # hops 0..L-2 relabelled in the chain
                assert torch.equal(a.src_local[k][:e], b.src_local[k][:e])
        n = int(a.sizes[h].item())
        assert torch.equal(a.globals[:n], b.globals[:n])
    assert db.tolist() == [-1, 0, 0] and int(b.sizes[0].item()) == 0
