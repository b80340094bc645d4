"""Mean aggregation kernels vs the numpy oracle (mpnn.py semantics) and autograd."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2110_08450_b200 import (DeviceGraph, FanoutSpec, LayerWeights, SamplerVariant,
                                   SeedBatch, full_forward, init_weights, make_epoch_plan,
                                   mfg_forward, multihop_mfg, prepare_batch, synth_graph,
                                   from_edge_list, generate_features, generate_labels)
from paper_2110_08450_b200.mpnn import segment_mean

pytestmark = pytest.mark.gpu


def test_segment_mean_bit_exact_fp32():
    rng = np.random.default_rng(0)
    for f in (1, 3, 8, 128, 256, 100):
        n_dst, n_src = 300, 900
        deg = rng.integers(0, 40, size=n_dst)
        indptr = np.zeros(n_dst + 1, dtype=np.int64)
        indptr[1:] = np.cumsum(deg)
        src = rng.integers(0, n_src, size=indptr[-1])
        h = rng.standard_normal((n_src, f)).astype(np.float32)
        want = O.mean_neighbors(h, indptr, src, n_dst)
        got = segment_mean(torch.from_numpy(indptr.astype(np.int32)).cuda(),
                           torch.from_numpy(src.astype(np.int32)).cuda(),
                           torch.from_numpy(h).cuda(), n_dst)
        assert np.array_equal(got.cpu().numpy(), want), f


@pytest.mark.parametrize("f,n_pad", [(128, 256), (104, 256), (24, 256), (128, 200000),
                                     (256, 256)])
def test_segment_mean_fp16_input_and_padding(f, n_pad):
    """16-bit rows: the warp-row kernels (pipelined for the training layer-0 shape,
    plain otherwise), including rows of 13 vectors on 16 lanes (products' 104)."""
    rng = np.random.default_rng(1)
    n_dst, n_src = 200, 500
    deg = rng.integers(0, 20, size=n_dst)
    indptr = np.zeros(n_dst + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(deg)
    src = rng.integers(0, n_src, size=indptr[-1])
    h = rng.uniform(-1, 1, (n_src, f)).astype(np.float16)
    want = O.mean_neighbors(h.astype(np.float32), indptr, src, n_dst)
    nd = torch.tensor([n_dst], dtype=torch.int64, device="cuda")
    got = segment_mean(torch.from_numpy(indptr.astype(np.int32)).cuda(),
                       torch.from_numpy(src.astype(np.int32)).cuda(),
                       torch.from_numpy(h).cuda(), n_dst, n_pad=n_pad, n_dst_dev=nd)
    # 16-bit rows take the warp-row kernel: per-lane-group partial sums, so the
    # fp32 summation order differs from strict edge order (tolerance, not bits)
    assert np.allclose(got[:n_dst].cpu().numpy(), want, rtol=1e-6, atol=1e-6)
    assert not got[n_dst:].any()


def test_neighbor_mean_example():
    g = from_edge_list([(0, 1), (1, 2)], 3, make_undirected=True)
    X = np.array([[1.0], [100.0], [3.0]], dtype=np.float32)
    mfg = multihop_mfg(g, SeedBatch(0, np.array([1])), FanoutSpec((2,)), 0)
    ws = [LayerWeights(w_self=np.zeros((1, 1), np.float32), w_neigh=np.eye(1, dtype=np.float32))]
    out = mfg_forward(mfg, X[mfg.id_map.global_ids.cpu().numpy()], ws)
    assert out.tolist() == [[2.0]]


def test_full_forward_hand_computed():
    g = from_edge_list([(0, 1), (1, 2)], 3, make_undirected=True)
    X = np.array([[1.0], [2.0], [4.0]], dtype=np.float32)
    ws = [LayerWeights(w_self=np.array([[2.0]], np.float32), w_neigh=np.array([[1.0]], np.float32))]
    assert full_forward(g, X, ws, [0, 1, 2]).tolist() == [[4.0], [6.5], [10.0]]


def test_mfg_forward_matches_reference(prep_small):
    z = prep_small
    g = synth_graph(1000, 8, 3.0, seed=13)
    fm = generate_features(1000, 8, "f16", seed=13)
    y = generate_labels(1000, 7, seed=13)
    plan = make_epoch_plan(np.arange(1000), 128, 5)
    pb = prepare_batch(g, fm, y, plan.batches[0], FanoutSpec((15, 10, 5)), SamplerVariant(), 42)
    ws = init_weights(8, 16, 3, seed=3)
    assert np.array_equal(ws[0].w_self, z["fwd_w0"][0])
    got = mfg_forward(pb.mfg, pb.features, ws).cpu().numpy()
    assert np.max(np.abs(got - z["fwd"])) <= 1e-6
    # the global-index path (reference mpnn.py:86-111) agrees with the golden too
    from paper_2110_08450_b200 import sampled_reference_forward
    glob = sampled_reference_forward(pb.mfg, fm.data.astype(np.float32), ws).cpu().numpy()
    assert np.max(np.abs(glob - z["fwd"])) <= 1e-6
    assert np.max(np.abs(glob - got)) <= 1e-6


def test_unbounded_fanout_matches_full_forward():
    g = synth_graph(1000, 8, 3.0, seed=13)
    X = generate_features(1000, 8, "f32", seed=13).data
    seeds = SeedBatch(0, np.random.default_rng(99).choice(1000, size=64, replace=False))
    d = g.max_degree()
    mfg = multihop_mfg(g, seeds, FanoutSpec((d, d)), 0)
    ws = init_weights(8, 16, 2, seed=3)
    got = mfg_forward(mfg, X[mfg.id_map.global_ids.cpu().numpy()], ws)
    want = full_forward(g, X, ws, seeds.dst_ids)
    assert torch.max(torch.abs(got - want)).item() <= 1e-5


def test_segment_mean_backward_vs_autograd():
    from paper_2110_08450_b200.model import SegmentMean
    rng = np.random.default_rng(3)
    n_dst, n_src, f = 150, 400, 256
    deg = rng.integers(0, 12, size=n_dst)
    indptr = torch.from_numpy(np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)).cuda()
    src = torch.from_numpy(rng.integers(0, n_src, size=int(deg.sum())).astype(np.int32)).cuda()
    h = torch.randn(n_src, f, device="cuda", requires_grad=True)
    out = SegmentMean.apply(h, indptr, src, n_dst, None, torch.float32)
    g = torch.randn_like(out)
    (out * g).sum().backward()
    # reference: dense mean matrix
    M = torch.zeros(n_dst, n_src, device="cuda", dtype=torch.float64)
    ip = indptr.cpu().numpy()
    sc = src.cpu().numpy()
    for d in range(n_dst):
        for e in range(ip[d], ip[d + 1]):
            M[d, sc[e]] += 1.0 / (ip[d + 1] - ip[d])
    want = M.T @ g.double()
    assert torch.allclose(h.grad.double(), want, atol=1e-5)
    assert torch.allclose(out.double(), M @ h.detach().double(), atol=1e-5)


@pytest.mark.parametrize("f,n_pad", [(128, 512), (104, 512), (128, 200000), (256, 512)])
def test_segment_mean_no_pad_fill_leaves_padding(f, n_pad):
    """sal_segment_mean_fwd_ex(SAL_SEG_NO_PAD_FILL): rows [n_dst, n_pad) keep what
    the buffer held; rows below n_dst equal the zero-filling call."""
    from paper_2110_08450_b200 import _lib
    rng = np.random.default_rng(2)
    n_dst, n_src = 300, 700
    deg = rng.integers(0, 16, size=n_dst)
    indptr = np.zeros(n_dst + 1, dtype=np.int32)
    indptr[1:] = np.cumsum(deg)
    src = rng.integers(0, n_src, size=int(indptr[-1])).astype(np.int32)
    h = torch.from_numpy(rng.uniform(-1, 1, (n_src, f)).astype(np.float16)).cuda()
    ip, sr = torch.from_numpy(indptr).cuda(), torch.from_numpy(src).cuda()
    nd = torch.tensor([n_dst], dtype=torch.int64, device="cuda")
    L = _lib.lib()
    outs = []
    for flags in (0, _lib.SAL_SEG_NO_PAD_FILL):
        out = torch.full((n_pad, f), 7.0, dtype=torch.bfloat16, device="cuda")
        _lib.check(L.sal_segment_mean_fwd_ex(ip.data_ptr(), sr.data_ptr(), nd.data_ptr(), n_pad,
                                             h.data_ptr(), _lib.SAL_F16, h.stride(0), f,
                                             out.data_ptr(), _lib.SAL_BF16, out.stride(0),
                                             flags, _lib.stream_ptr()), "segment_mean_fwd_ex")
        outs.append(out)
    torch.cuda.synchronize()
    assert torch.equal(outs[0][:n_dst], outs[1][:n_dst])
    assert (outs[0][n_dst:] == 0).all() and (outs[1][n_dst:] == 7.0).all()
