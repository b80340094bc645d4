"""Generate golden vectors from the REFERENCE implementation (mfgprep).

Run here (the reference is importable in this container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports /root/reference/pkg/src/mfgprep read-only and writes small .npz
fixtures next to this file.  Those fixtures travel with the repo; nothing at
test/bench time reads /root/reference.  Every fixture records the reference
call that produced it.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
REF_SRC = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)

import mfgprep as M  # noqa: E402
from mfgprep import _kernels as K  # noqa: E402
from mfgprep.reference import sample_positions_oracle  # noqa: E402
from mfgprep.rng import stream_key, stream_u64  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items()})


def mfg_arrays(prefix, mfg):
    d = {f"{prefix}global_ids": mfg.id_map.global_ids.astype(np.int64),
         f"{prefix}digest": np.array(mfg.digest())}
    for i, l in enumerate(mfg.layers):
        d[f"{prefix}l{i}_meta"] = np.array([l.num_dst, l.num_src, l.num_edges], dtype=np.int64)
        d[f"{prefix}l{i}_indptr"] = l.indptr.astype(np.int64)
        d[f"{prefix}l{i}_src"] = l.src_local.astype(np.int64)
    return d


def gen_rng():
    # (seed, batch, hop, pos) -> stream key and the first draws
    rng = np.random.default_rng(0)
    quad = rng.integers(0, 2**31, size=(64, 4), dtype=np.int64)
    quad[0] = (0, 0, 0, 0)
    quad[1] = (42, 0, 0, 1)
    keys = np.array([stream_key(*map(int, q)) for q in quad], dtype=np.uint64)
    draws = np.array([[stream_u64(int(k), c) for c in range(8)] for k in keys], dtype=np.uint64)
    prefixes = np.array([M.HopStream(int(q[0]), int(q[1]), int(q[2])).key_prefix for q in quad],
                        dtype=np.uint64)
    # sample_positions_oracle cases (reference.py:21-34)
    cases = []
    pos = []
    for i in range(400):
        deg = int(rng.integers(1, 300))
        d = int(rng.integers(0, 40))
        key = int(rng.integers(0, 2**63))
        p = sample_positions_oracle(deg, d, key)
        cases.append((deg, d, key))
        pos.append(p)
    lens = np.array([len(p) for p in pos], dtype=np.int64)
    flat = np.array([x for p in pos for x in p], dtype=np.int64)
    save("rng", quad=quad, keys=keys, draws=draws, prefixes=prefixes,
         cases=np.array(cases, dtype=np.uint64), pos_len=lens, pos_flat=flat)


def gen_graphs():
    specs = [(1000, 8, 3.0, 13), (800, 6, 3.0, 3), (4000, 8, 3.0, 5), (20000, 10, 2.5, 7),
             (100_000, 10, 3.0, 1), (169_343, 1_166_243 / 169_343, 3.0, 1), (500, 6, float("inf"), 2)]
    rows = []
    for n, avg, ex, seed in specs:
        g = M.synth_graph(n, avg, ex, seed=seed)
        rows.append((n, avg, ex, seed, g.num_edges, g.checksum(), g.max_degree()))
    arr = np.array([(r[0], r[3], r[4], r[5], r[6]) for r in rows], dtype=np.int64)
    fl = np.array([(r[1], r[2]) for r in rows], dtype=np.float64)
    g = M.synth_graph(1000, 8, 3.0, seed=13)
    save("graphs", spec_int=arr, spec_float=fl, small_indptr=g.indptr, small_indices=g.indices)


def gen_small_mfgs():
    g = M.synth_graph(1000, 8, 3.0, seed=13)
    seeds64 = M.SeedBatch(0, np.random.default_rng(99).choice(1000, size=64, replace=False))
    out = {"seeds64": seeds64.dst_ids}
    v = M.SamplerVariant()
    cases = {
        "a": ((15, 10, 5), 9, seeds64),
        "b": ((5, 10, 15), 42, seeds64),
        "c": ((4,), 5, seeds64),
        "d": ((g.max_degree(),) * 3, 0, seeds64),
        "e": ((3, 2), 77, M.SeedBatch(17, seeds64.dst_ids[:5])),
        "f": ((40, 33), 123, M.SeedBatch(3, seeds64.dst_ids[:16])),
    }
    for name, (fan, gs, sb) in cases.items():
        mfg = M.multihop_mfg(g, sb, M.FanoutSpec(fan), gs, v)
        out.update(mfg_arrays(f"{name}_", mfg))
        out[f"{name}_fan"] = np.array(fan, dtype=np.int64)
        out[f"{name}_gseed"] = np.array(gs, dtype=np.int64)
        out[f"{name}_batch"] = np.array(sb.batch_id, dtype=np.int64)
        out[f"{name}_seeds"] = sb.dst_ids
    # injection: two-pass hop_kernel pos_all for hop 0 of case a (edge order)
    idm = M.IdMap(v)
    idm.insert(seeds64.dst_ids)
    n_dst = idm.size
    fan = 5
    budget = int(K.hop_budget(g.indptr, idm._globals, n_dst, fan))
    idm.ensure_capacity(budget)
    src_out = np.empty(budget, dtype=np.int64)
    dptr = np.empty(n_dst + 1, dtype=np.int64)
    pos_scratch = np.empty(fan, dtype=np.int64)
    set_scratch = np.empty(16, dtype=np.int64)
    pos_all = np.empty(budget, dtype=np.int64)
    K.hop_kernel(g.indptr, g.indices, idm._globals, idm.size, idm._heads, idm._nxt, idm._table,
                 idm.map_code, K.SET_VECTOR, False, n_dst, fan,
                 np.uint64(M.HopStream(9, 0, 0).key_prefix), src_out, dptr, pos_scratch,
                 set_scratch, pos_all)
    out["inject_pos"] = pos_all
    out["inject_src"] = src_out
    out["inject_indptr"] = dptr
    # IdMap.insert with duplicates / existing keys (insert_keys)
    idm2 = M.IdMap(v)
    idm2.insert(np.array([5, 9, 5, 3]))
    idm2.insert(np.array([3, 11, 9, 12, 11]))
    out["idmap_globals"] = idm2.global_ids.copy()
    save("mfg_small", **out)


def gen_prep_small():
    g = M.synth_graph(1000, 8, 3.0, seed=13)
    fm32 = M.generate_features(1000, 8, "f32", seed=13)
    fm16 = M.generate_features(1000, 8, "f16", seed=13)
    y = M.generate_labels(1000, 7, seed=13)
    plan = M.make_epoch_plan(np.arange(1000), 128, 5)
    cfg = M.PrepConfig(num_workers=2, fanouts=M.FanoutSpec((15, 10, 5)))
    digests32 = [b.digest() for b in M.run_epoch_prep(g, fm32, y, plan, cfg, 42)]
    digests16 = [b.digest() for b in M.run_epoch_prep(g, fm16, y, plan, cfg, 42)]
    pb = M.prepare_batch(g, fm16, y, plan.batches[0], M.FanoutSpec((15, 10, 5)),
                         M.SamplerVariant(), 42)
    # special f16 values through slice_features
    specials = np.array([0x0000, 0x8000, 0x0001, 0x03FF, 0x0400, 0x3C00, 0xBC00, 0x7BFF, 0x7C00,
                         0xFC00, 0x7E00, 0x7C01, 0xFE00, 0x3555, 0x8001, 0xC000], dtype=np.uint16)
    sp = M.FeatureMatrix(rows=4, cols=4, data=specials.view(np.float16).reshape(4, 4))
    idm = M.IdMap(M.SamplerVariant())
    idm.insert(np.array([3, 1, 2, 0, 1]))
    buf = np.empty(16, dtype=np.float32)
    sp_out = M.slice_features(sp, idm, buf)
    # mfg_forward on the prepared batch (mpnn.py:68-83)
    ws = M.init_weights(8, 16, 3, seed=3)
    fwd = M.mfg_forward(pb.mfg, pb.features, ws)
    save("prep_small", plan_perm=np.concatenate([b.dst_ids for b in plan.batches]),
         digests32=np.array(digests32), digests16=np.array(digests16),
         pb_features=pb.features, pb_labels=pb.labels, pb_digest=np.array(pb.digest()),
         pb_byte_size=np.array(pb.byte_size), specials=specials,
         specials_ids=idm.global_ids.copy(), specials_out=sp_out.view(np.uint32).copy(),
         fwd=fwd, fwd_w=np.stack([np.stack([w.w_self, w.w_neigh]) for w in ws[1:]]),
         fwd_w0=np.stack([ws[0].w_self, ws[0].w_neigh]))


def gen_config1():
    """BASELINE config 1: 100K nodes / ~1M slots, 128-d f16, (15,10,5), batch 1024."""
    n = 100_000
    g = M.synth_graph(n, 10, 3.0, seed=1)
    fm = M.generate_features(n, 128, "f16", seed=1)
    y = M.generate_labels(n, 172, seed=1)
    plan = M.make_epoch_plan(np.arange(n), 1024, 1)
    out = {"checksum": np.array(g.checksum(), dtype=np.int64), "num_edges": np.array(g.num_edges)}
    digs, pdigs, stats = [], [], []
    for b in plan.batches[:4] + plan.batches[-1:]:
        pb = M.prepare_batch(g, fm, y, b, M.FanoutSpec((15, 10, 5)), M.SamplerVariant(), 1)
        digs.append(pb.mfg.digest())
        pdigs.append(pb.digest())
        stats.append([b.batch_id] + [x for s in pb.stats for x in s])
    out["mfg_digests"] = np.array(digs)
    out["batch_digests"] = np.array(pdigs)
    out["stats"] = np.array(stats, dtype=np.int64)
    # paper-order fanouts and inference fanouts on batch 0
    for tag, fan in (("paper", (5, 10, 15)), ("infer", (20, 20, 20))):
        m = M.multihop_mfg(g, plan.batches[0], M.FanoutSpec(fan), 1, M.SamplerVariant())
        out[f"{tag}_digest"] = np.array(m.digest())
        out[f"{tag}_stats"] = np.array([[l.num_dst, l.num_src, l.num_edges] for l in m.layers])
    # full arrays of batch 0 (int32 to keep the fixture small)
    m0 = M.multihop_mfg(g, plan.batches[0], M.FanoutSpec((15, 10, 5)), 1, M.SamplerVariant())
    out["b0_global_ids"] = m0.id_map.global_ids.astype(np.int32)
    for i, l in enumerate(m0.layers):
        out[f"b0_l{i}_indptr"] = l.indptr.astype(np.int32)
        out[f"b0_l{i}_src"] = l.src_local.astype(np.int32)
    save("config1", **out)


def _malformed_cases(good: bytes, magic: bytes):
    """(tag, bytes) variants of one good file: bad magic, bad version, and a
    truncation inside every field (magic, version, counts/shape, payloads)."""
    cases = [("badmagic", b"XXXX" + good[4:]),
             ("badversion", good[:4] + (2).to_bytes(4, "little") + good[8:])]
    for cut in (2, 6, 12, 30, len(good) - 1):
        if cut < len(good):
            cases.append((f"trunc{cut}", good[:cut]))
    return cases


def gen_files():
    """f2 loaders: small MFGC / FEAT / LABL files written by the reference's own
    writers (graph.py:194-240), the arrays its loaders return, and the
    exception class + message its loaders raise on malformed variants."""
    import tempfile
    d = OUT / "files"
    d.mkdir(exist_ok=True)
    g = M.synth_graph(700, 6, 3.0, seed=5)
    fh = M.generate_features(700, 20, "f16", seed=5)
    ff = M.generate_features(700, 7, "f32", seed=5)
    y = M.generate_labels(700, 13, seed=5)
    M.save_csr(g, d / "g.mfgc")
    M.save_features(fh, d / "x16.feat")
    M.save_features(ff, d / "x32.feat")
    M.save_labels(y, d / "y.labl")
    out = {"indptr": M.load_csr(d / "g.mfgc").indptr, "indices": M.load_csr(d / "g.mfgc").indices,
           "num_nodes": np.array(g.num_nodes),
           "x16": M.load_features(d / "x16.feat").data, "x32": M.load_features(d / "x32.feat").data,
           "y": M.load_labels(d / "y.labl").values,
           "num_classes": np.array(M.load_labels(d / "y.labl").num_classes)}
    errs = []
    loaders = {"g.mfgc": M.load_csr, "x16.feat": M.load_features, "y.labl": M.load_labels}
    with tempfile.TemporaryDirectory() as td:
        for name, fn in loaders.items():
            good = (d / name).read_bytes()
            for tag, data in _malformed_cases(good, good[:4]):
                p = Path(td) / f"{tag}_{name}"
                p.write_bytes(data)
                try:
                    fn(p)
                    errs.append((name, tag, "", ""))
                except Exception as e:  # noqa: BLE001 — recording the reference's behaviour
                    errs.append((name, tag, type(e).__name__, str(e)))
        # semantic faults the loaders' validation catches (graph.py:58-65, 96-100)
        good = bytearray((d / "g.mfgc").read_bytes())
        n, e = g.num_nodes, g.num_edges
        ip0 = 4 + 4 + 16
        ix0 = ip0 + 8 * (n + 1)
        sem = {}
        b = bytearray(good); b[ix0 + 4 * (e - 1): ix0 + 4 * e] = int(n).to_bytes(4, "little")
        sem["badindex_g.mfgc"] = b
        b = bytearray(good); b[ip0 + 8 * 5: ip0 + 8 * 6] = int(e + 3).to_bytes(8, "little")
        sem["decreasing_g.mfgc"] = b
        b = bytearray(good); b[ip0 + 8 * n: ip0 + 8 * (n + 1)] = int(e - 1).to_bytes(8, "little")
        sem["endpoint_g.mfgc"] = b
        b = bytearray(good); b[ip0: ip0 + 8] = int(1).to_bytes(8, "little")
        sem["start_g.mfgc"] = b
        lb = bytearray((d / "y.labl").read_bytes())
        lb[8 + 12 + 4 * 9: 8 + 12 + 4 * 10] = (13).to_bytes(4, "little")
        sem["badlabel_y.labl"] = lb
        for key, data in sem.items():
            tag, name = key.split("_", 1)
            p = Path(td) / key
            p.write_bytes(bytes(data))
            (d / key).write_bytes(bytes(data))
            try:
                loaders[name](p)
                errs.append((name, tag, "", ""))
            except Exception as ex:  # noqa: BLE001
                errs.append((name, tag, type(ex).__name__, str(ex)))
    out["errors"] = np.array(errs)
    save("files", **out)


def gen_trace():
    """f3 hop replay: a TRCE file written by the reference's record_trace
    (bench.py:46-79), the digest its replay_variant computes (bench.py:104-139)
    and the errors load_trace raises on malformed copies."""
    import tempfile
    from mfgprep import bench as RB
    d = OUT / "files"
    d.mkdir(exist_ok=True)
    g = M.synth_graph(5000, 9, 3.0, seed=8)
    batches = M.make_epoch_plan(np.arange(0, 5000, 3), 128, 2).batches[:4]

    class _Plan:  # record_trace only reads plan.batches
        pass
    p = _Plan()
    p.batches = batches
    tr = RB.record_trace(g, p, M.FanoutSpec((15, 10, 5)), 11, path=d / "trace.trce")
    rep = RB.replay_variant(tr, g, M.SamplerVariant(), repetitions=1, warmup=False)
    good = (d / "trace.trce").read_bytes()
    errs = []
    with tempfile.TemporaryDirectory() as td:
        for tag, data in (("badmagic", b"XXXX" + good[4:]),
                          ("badversion", good[:4] + (2).to_bytes(4, "little") + good[8:]),
                          ("trunc10", good[:10]), ("trunc40", good[:40]),
                          ("trunc60", good[:60]), ("truncm1", good[:-1])):
            q = Path(td) / tag
            q.write_bytes(data)
            try:
                RB.load_trace(q)
                errs.append((tag, "", ""))
            except Exception as e:  # noqa: BLE001
                errs.append((tag, type(e).__name__, str(e)))
    save("trace", digest=np.array(rep.digest), checksum=np.array(g.checksum(), dtype=np.int64),
         indptr=g.indptr, indices=g.indices.astype(np.int32),
         batch_ids=np.array([b.batch_id for b in batches]),
         seeds=np.concatenate([b.dst_ids for b in batches]),
         nrec=np.array(len(tr.records)), errors=np.array(errs))


if __name__ == "__main__":
    gen_trace()
    gen_files()
    gen_rng()
    gen_graphs()
    gen_small_mfgs()
    gen_prep_small()
    gen_config1()
