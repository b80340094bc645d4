"""Pin the CPU oracle (oracle/) against golden vectors made by the reference.

These run without a GPU.  The oracle is the checker for every GPU parity
test, so it must reproduce the reference bit-for-bit first.
"""
import numpy as np
import pytest

import oracle as O
from conftest import assert_mfg_equal, golden, golden_mfg


def test_stream_keys_and_draws():
    z = golden("rng")
    for q, k, p in zip(z["quad"], z["keys"], z["prefixes"]):
        assert O.stream_key(*map(int, q)) == int(k)
        assert O.hop_prefix(int(q[0]), int(q[1]), int(q[2])) == int(p)


def test_sample_positions_vs_reference_oracle():
    z = golden("rng")
    off = 0
    for (deg, d, key), n in zip(z["cases"], z["pos_len"]):
        want = z["pos_flat"][off:off + n].tolist()
        off += n
        assert O.sample_positions(int(key), int(deg), int(d)) == want


@pytest.mark.parametrize("case", list("abcdef"))
def test_multihop_matches_reference(case, mfg_small, g_small):
    z = mfg_small
    gids, layers = O.multihop(g_small["small_indptr"], g_small["small_indices"], 1000,
                              z[f"{case}_seeds"], tuple(z[f"{case}_fan"]), int(z[f"{case}_gseed"]),
                              int(z[f"{case}_batch"]))
    want_g, want_l = golden_mfg(z, f"{case}_")
    assert_mfg_equal(gids, layers, want_g, want_l)
    assert O.mfg_digest(gids, layers) == str(z[f"{case}_digest"])


def test_gather_f16_specials(prep_small):
    z = prep_small
    data = z["specials"].view(np.float16).reshape(4, 4)
    out = O.gather_features(data, z["specials_ids"])
    assert np.array_equal(out.view(np.uint32), z["specials_out"])


def test_prepared_batch_digest(prep_small, g_small):
    """prepare_batch digest of plan batch 0 with f16 features (prep.py:132-137)."""
    from paper_2110_08450_b200.graph import generate_features, generate_labels
    z = prep_small
    fm = generate_features(1000, 8, "f16", seed=13)
    y = generate_labels(1000, 7, seed=13)
    seeds = z["plan_perm"][:128]
    gids, layers = O.multihop(g_small["small_indptr"], g_small["small_indices"], 1000, seeds,
                              (15, 10, 5), 42, 0)
    feats = O.gather_features(fm.data, gids)
    labels = O.gather_labels(y.values, seeds)
    assert np.array_equal(feats, z["pb_features"])
    assert np.array_equal(labels, z["pb_labels"])
    assert O.batch_digest(O.mfg_digest(gids, layers), feats, labels) == str(z["pb_digest"])


def test_epoch_digests_match_reference(prep_small, g_small):
    from paper_2110_08450_b200.graph import generate_features, generate_labels
    z = prep_small
    perm = z["plan_perm"]
    y = generate_labels(1000, 7, seed=13)
    for dt, key in (("f32", "digests32"), ("f16", "digests16")):
        fm = generate_features(1000, 8, dt, seed=13)
        digs = []
        for b in range(8):
            seeds = perm[128 * b:128 * (b + 1)]
            gids, layers = O.multihop(g_small["small_indptr"], g_small["small_indices"], 1000,
                                      seeds, (15, 10, 5), 42, b)
            digs.append(O.batch_digest(O.mfg_digest(gids, layers),
                                       O.gather_features(fm.data, gids),
                                       O.gather_labels(y.values, seeds)))
        assert digs == [str(d) for d in z[key]]


def test_mfg_forward_matches_reference(prep_small, g_small):
    z = prep_small
    seeds = z["plan_perm"][:128]
    gids, layers = O.multihop(g_small["small_indptr"], g_small["small_indices"], 1000, seeds,
                              (15, 10, 5), 42, 0)
    ws = [tuple(z["fwd_w0"])] + [tuple(w) for w in z["fwd_w"]]
    out = O.mfg_forward(layers, z["pb_features"], ws)
    assert np.max(np.abs(out - z["fwd"])) <= 1e-6


def test_config1_batches_match_reference():
    """BASELINE config 1 (100K nodes, 128-d f16): digests of 5 reference batches."""
    from paper_2110_08450_b200.graph import synth_graph
    from paper_2110_08450_b200.prep import make_epoch_plan
    z = golden("config1")
    g = synth_graph(100_000, 10, 3.0, seed=1)
    assert g.checksum() == int(z["checksum"])
    plan = make_epoch_plan(np.arange(100_000), 1024, 1)
    picks = list(plan.batches[:4]) + [plan.batches[-1]]
    for b, want, st in zip(picks, z["mfg_digests"], z["stats"]):
        gids, layers = O.multihop(g.indptr, g.indices, g.num_nodes, b.dst_ids, (15, 10, 5), 1,
                                  b.batch_id)
        assert O.mfg_digest(gids, layers) == str(want)
        assert int(st[0]) == b.batch_id
        assert [x for l in layers for x in (l["num_dst"], l["num_src"], len(l["src_local"]))] \
            == st[1:].tolist()
    for tag, fan in (("paper", (5, 10, 15)), ("infer", (20, 20, 20))):
        gids, layers = O.multihop(g.indptr, g.indices, g.num_nodes, plan.batches[0].dst_ids, fan,
                                  1, 0)
        assert O.mfg_digest(gids, layers) == str(z[f"{tag}_digest"])


def test_epoch_prep_threads_agree(g_small):
    """The timed CPU baseline: identical per-batch results for 1 and 4 threads."""
    from paper_2110_08450_b200.graph import generate_features
    fm = generate_features(1000, 8, "f16", seed=13)
    perm = np.random.default_rng(5).permutation(1000)
    batches = [(i, perm[i * 100:(i + 1) * 100]) for i in range(10)]
    r1 = O.epoch_prep(g_small["small_indptr"], g_small["small_indices"], 1000, fm.data, None,
                      batches, (15, 10, 5), 3, 1)
    r4 = O.epoch_prep(g_small["small_indptr"], g_small["small_indices"], 1000, fm.data, None,
                      batches, (15, 10, 5), 3, 4)
    assert np.array_equal(r1[1][:, :2], r4[1][:, :2])
    assert np.array_equal(r1[2], r4[2])
    for b, (bid, seeds) in enumerate(batches):
        gids, layers = O.multihop(g_small["small_indptr"], g_small["small_indices"], 1000, seeds,
                                  (15, 10, 5), 3, bid)
        assert r1[1][b, 0] == len(gids)
        assert r1[1][b, 1] == sum(len(l["src_local"]) for l in layers)
