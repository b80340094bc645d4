"""Fused last hop (sal_sample_aggregate) against the two-kernel path it replaces.

The unfused path — the last hop materialised as global source ids
(SAL_MFG_LAST_HOP_EDGES, bit-exact with the reference sampler: test_gpu_sampler),
then the layer-0 mean over them and the destination rows gathered — is the
comparator: the fused kernel must draw the same sample and sum it in the same
order, so the [mean | self] buffer must be bit-identical.  The mean is also
checked against the oracle's full MFG (reference multihop_mfg +
_mean_neighbors, mpnn.py:57-65) within fp32 tolerance.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2110_08450_b200 import _lib
from paper_2110_08450_b200.graph import synth_graph_device
from paper_2110_08450_b200.prep import gather_rows
from paper_2110_08450_b200.sampler import FanoutSpec, MfgWorkspace, RNG_POLICIES

pytestmark = pytest.mark.gpu


def _two_kernel(dg, fan, seeds, desc, gseed, policy, out_dtype, f_model):
    ws = MfgWorkspace(dg.num_nodes, fan, len(seeds), device="cuda", last_hop_edges=True)
    ws.run(dg, seeds, desc, gseed, policy)
    h = ws.num_hops - 1
    x = dg.features
    out = torch.zeros((ws.node_cap[h], 2 * f_model), dtype=out_dtype, device="cuda")
    L = _lib.lib()
    _lib.check(L.sal_segment_mean_fwd_ex(
        ws.dst_indptr[h].data_ptr(), ws.src_glob.data_ptr(), ws.sizes[h:h + 1].data_ptr(),
        ws.node_cap[h], x.data_ptr(), _lib.SAL_F16, x.stride(0), x.shape[1], out.data_ptr(),
        _lib.dtype_code(out_dtype), out.stride(0), _lib.SAL_SEG_NO_PAD_FILL,
        _lib.stream_ptr()), "segment_mean_fwd_ex")
    gather_rows(x, ws.globals, out[:, f_model:f_model + x.shape[1]], n=ws.node_cap[h],
                n_dev=ws.sizes[h:h + 1])
    n = int(ws.sizes[h].item())
    return out, n, ws


def _fused(dg, fan, seeds, desc, gseed, policy, out_dtype, f_model):
    ws = MfgWorkspace(dg.num_nodes, fan, len(seeds), device="cuda", last_hop_fused=True)
    ws.run(dg, seeds, desc, gseed, policy)
    h = ws.num_hops - 1
    out = torch.zeros((ws.node_cap[h], 2 * f_model), dtype=out_dtype, device="cuda")
    ws.aggregate(dg, dg.features, out, f_model, desc, gseed, policy)
    return out, int(ws.sizes[h].item()), ws


@pytest.fixture(scope="module")
def g128():
    return synth_graph_device(200_000, 14.0, 3.0, seed=5, num_features=128, num_classes=10,
                              feature_seed=5, label_seed=5)


@pytest.fixture(scope="module")
def g104():  # rows of 13 16-byte vectors: 100 fp16 columns at a 104-column stride
    g = synth_graph_device(100_000, 25.0, 3.0, seed=6, num_features=100, num_classes=10,
                           feature_seed=6, label_seed=6)
    g.features = g.features[:, :104].contiguous()   # tables are stored at 128 now
    return g


@pytest.mark.parametrize("fan", [(15, 10, 5), (5, 10, 15), (20, 20, 20), (3, 4), (32,)])
@pytest.mark.parametrize("policy", ["splitmix", "philox"])
def test_fused_equals_two_kernel_path(g128, fan, policy):
    rng = np.random.default_rng(len(fan) * 7 + fan[0])
    seeds = torch.from_numpy(rng.choice(g128.num_nodes, 1024, replace=False)).cuda()
    desc = torch.tensor([11, 0, 1024], dtype=torch.int64, device="cuda")
    pol = RNG_POLICIES[policy]
    a, na, _ = _two_kernel(g128, FanoutSpec(fan), seeds, desc, 3, pol, torch.bfloat16, 128)
    b, nb, ws = _fused(g128, FanoutSpec(fan), seeds, desc, 3, pol, torch.bfloat16, 128)
    assert na == nb > 0
    assert torch.equal(a[:na].view(torch.int16), b[:nb].view(torch.int16))
    assert not b[nb:].any()                       # rows past the count are not written
    assert int(ws.sizes[ws.num_hops].item()) == -1  # the last hop's size is unknown


def test_fused_narrow_rows_and_fp16_out(g104):
    rng = np.random.default_rng(9)
    seeds = torch.from_numpy(rng.choice(g104.num_nodes, 512, replace=False)).cuda()
    desc = torch.tensor([2, 0, 512], dtype=torch.int64, device="cuda")
    for dt in (torch.bfloat16, torch.float16):
        a, na, _ = _two_kernel(g104, FanoutSpec((15, 10, 5)), seeds, desc, 1, 0, dt, 128)
        b, nb, _ = _fused(g104, FanoutSpec((15, 10, 5)), seeds, desc, 1, 0, dt, 128)
        assert na == nb
        assert torch.equal(a[:na].view(torch.int16), b[:nb].view(torch.int16))
        assert not b[:, 104:128].any() and not b[:, 232:].any()   # padding columns untouched


def test_fused_mean_matches_oracle(g128):
    """Against the reference's own algorithm on host copies: the oracle's full MFG
    (multihop_mfg) -> numpy mean of the last hop's rows (mpnn.py:57-65)."""
    import shape_parity as parity
    host = parity.host_copy(g128)
    rng = np.random.default_rng(4)
    ids = rng.choice(g128.num_nodes, 700, replace=False)
    seeds = torch.from_numpy(ids).cuda()
    desc = torch.tensor([5, 0, len(ids)], dtype=torch.int64, device="cuda")
    fan = FanoutSpec((15, 10, 5))
    out, n, ws = _fused(g128, fan, seeds, desc, 2, 0, torch.bfloat16, 128)
    gids, layers = O.multihop(host["indptr"], host["indices"], g128.num_nodes, ids,
                              list(fan.per_hop), 2, 5)
    lay0 = layers[0]             # consumption order: layer 0 = the last expansion hop
    assert lay0["num_dst"] == n
    x16 = host["features"][:, :128]
    x = x16.astype(np.float32)
    want = O.mean_neighbors(x[gids[:lay0["num_src"]]], lay0["indptr"], lay0["src_local"], n)
    got = out[:n, :128].float().cpu().numpy()
    # fp32 sums, bf16 output: within one bf16 rounding of the fp32 mean
    assert np.allclose(got, want, rtol=2 ** -8, atol=1e-6)
    want_self = torch.from_numpy(x[gids[:n]]).to(torch.bfloat16)
    assert torch.equal(out[:n, 128:].cpu().view(torch.int16), want_self.view(torch.int16))


def test_fused_rejects_bad_arguments(g128):
    ws = MfgWorkspace(g128.num_nodes, FanoutSpec((15, 10, 5)), 64, device="cuda",
                      last_hop_edges=True)
    out = torch.zeros((ws.node_cap[2], 256), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        ws.aggregate(g128, g128.features, out, 128, ws.desc, 1)
    ws2 = MfgWorkspace(g128.num_nodes, FanoutSpec((40, 2)), 64, device="cuda",
                       last_hop_fused=True)
    with pytest.raises(RuntimeError, match="fanout 40 > 32"):
        ws2.aggregate(g128, g128.features, out, 128, ws2.desc, 1)


def test_fused_special_values_bit_exact():
    """-0, +-inf, NaN and subnormal fp16 values: the self rows must equal the row
    gather's conversion bit for bit, the means the pipe kernel's."""
    from paper_2110_08450_b200.graph import DeviceGraph
    rng = np.random.default_rng(17)
    n = 5000
    deg = rng.integers(0, 40, size=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(deg)
    indices = rng.integers(0, n, size=indptr[-1]).astype(np.int32)
    bits = rng.integers(0, 1 << 16, size=(n, 128), dtype=np.uint32).astype(np.uint16)
    specials = np.array([0x8000, 0x7C00, 0xFC00, 0x7E00, 0x0001, 0x83FF, 0x0000], np.uint16)
    pick = rng.random((n, 128)) < 0.3
    bits[pick] = specials[rng.integers(0, len(specials), size=pick.sum())]
    x = torch.from_numpy(bits.view(np.float16)).cuda()
    dg = DeviceGraph(n, torch.from_numpy(indptr).cuda(), torch.from_numpy(indices).cuda(),
                     features=x)
    seeds = torch.from_numpy(rng.choice(n, 300, replace=False)).cuda()
    desc = torch.tensor([1, 0, 300], dtype=torch.int64, device="cuda")
    a, na, _ = _two_kernel(dg, FanoutSpec((15, 10)), seeds, desc, 9, 0, torch.bfloat16, 128)
    b, nb, _ = _fused(dg, FanoutSpec((15, 10)), seeds, desc, 9, 0, torch.bfloat16, 128)
    assert na == nb
    assert torch.equal(a[:na].view(torch.int16), b[:nb].view(torch.int16))


def test_reset_in_aggregate_reuses_the_workspace(g128):
    """sal_mfg_plan.reset_in_aggregate: run() skips the table/scan resets and the fused
    kernel leaves them reset, so one workspace serves batch after batch exactly like
    fresh workspaces (and like the unfused two-kernel path)."""
    fan = FanoutSpec((15, 10, 5))
    ws = MfgWorkspace(g128.num_nodes, fan, 1024, device="cuda", last_hop_fused=True,
                      reset_in_aggregate=True)
    assert ws.plan.reset_in_aggregate == 1
    h = ws.num_hops - 1
    rng = np.random.default_rng(21)
    for b in range(4):
        seeds = torch.from_numpy(rng.choice(g128.num_nodes, 1024, replace=False)).cuda()
        desc = torch.tensor([b, 0, 1024], dtype=torch.int64, device="cuda")
        want, n, _ = _two_kernel(g128, fan, seeds, desc, 4, 0, torch.bfloat16, 128)
        ws.run(g128, seeds, desc, 4, 0)
        out = torch.zeros_like(want)
        ws.aggregate(g128, g128.features, out, 128, desc, 4, 0)
        assert int(ws.sizes[h].item()) == n
        assert torch.equal(out[:n].view(torch.int16), want[:n].view(torch.int16)), b
        assert bool((ws.table == -1).all())          # left reset for the next batch


@pytest.mark.parametrize("fan", [(15, 10, 5), (20, 20, 20), (3, 4), (2, 3, 4, 5)])
def test_resolve_in_aggregate_gives_the_same_mfg(g128, fan):
    """sal_mfg_plan.resolve_in_aggregate: hop L-2's relabel second pass runs inside the
    fused kernel (from the table words flag_scan kept).  After aggregate() the MFG of
    hops 0..L-2 (sizes, indptr, local ids, globals) and the [mean | self] buffer equal
    the in-chain resolve's, batch after batch on one workspace."""
    fan = FanoutSpec(fan)
    kw = dict(device="cuda", last_hop_fused=True, reset_in_aggregate=True)
    ref = MfgWorkspace(g128.num_nodes, fan, 1024, **kw)
    ws = MfgWorkspace(g128.num_nodes, fan, 1024, resolve_in_aggregate=True, **kw)
    assert ws.plan.resolve_in_aggregate == 1 and ref.plan.resolve_in_aggregate == 0
    h = ws.num_hops - 1
    rng = np.random.default_rng(len(fan) + 31)
    for b in range(3):
        seeds = torch.from_numpy(rng.choice(g128.num_nodes, 1024, replace=False)).cuda()
        desc = torch.tensor([b, 0, 1024], dtype=torch.int64, device="cuda")
        outs = []
        for w in (ref, ws):
            w.src_local[h - 1].fill_(-7)
            w.run(g128, seeds, desc, 5, 0)
            out = torch.zeros((w.node_cap[h], 256), dtype=torch.bfloat16, device="cuda")
            w.aggregate(g128, g128.features, out, 128, desc, 5, 0)
            outs.append(out)
        assert torch.equal(ref.sizes[:h + 1], ws.sizes[:h + 1])
        n = int(ws.sizes[h].item())
        assert torch.equal(ref.globals[:n], ws.globals[:n])
        for k in range(h):
            e = int(ws.etot[k].item())
            assert torch.equal(ref.dst_indptr[k][:int(ws.sizes[k].item()) + 1],
                               ws.dst_indptr[k][:int(ws.sizes[k].item()) + 1]), (b, k)
            assert torch.equal(ref.src_local[k][:e], ws.src_local[k][:e]), (b, k)
            assert int(ws.src_local[k][:e].min()) >= 0
        assert torch.equal(outs[0][:n].view(torch.int16), outs[1][:n].view(torch.int16))
        assert bool((ws.table == -1).all())
