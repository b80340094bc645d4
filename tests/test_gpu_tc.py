"""tcgen05 GEMM kernels (layer-0 SAGEConv) vs torch fp32 references."""
import pytest
import torch

from paper_2110_08450_b200 import _lib

pytestmark = pytest.mark.gpu


def _fwd(A, W, p=0.0, relu=True, seed=7, salt=None, out_cols=256, m_dev=None, fill=0.0):
    M = A.shape[0]
    Y = torch.full((M, 2 * out_cols), fill, dtype=torch.bfloat16, device="cuda")[:, out_cols:]
    mask = torch.full((M * 256 // 8,), 255 if fill else 0, dtype=torch.uint8, device="cuda")
    L = _lib.lib()
    _lib.check(L.sal_tc_sage_fwd(A.data_ptr(), A.stride(0), M, _lib.ptr(m_dev), W.data_ptr(),
                                 256, A.shape[1],
                                 Y.data_ptr(), Y.stride(0), mask.data_ptr(), p, seed,
                                 _lib.ptr(salt), int(relu), _lib.stream_ptr()), "tc_sage_fwd")
    torch.cuda.synchronize()
    return Y, mask


@pytest.mark.parametrize("M,K", [(128, 256), (1000, 256), (67584, 256), (128, 512),
                                 (1000, 512), (6144, 512)])
def test_tc_fwd_matches_torch(M, K):
    """K = 256: the layer-0 shape; K = 512: a hidden layer's [mean | h] (two
    128-column blocks per row tile, grid.y)."""
    g = torch.Generator(device="cuda").manual_seed(M)
    A = (torch.randn(M, 2 * K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)[:, :K]
    W = (torch.randn(256, K, device="cuda", generator=g) * 0.06).to(torch.bfloat16)
    Y, mask = _fwd(A, W, p=0.0, relu=False)
    want = A.float() @ W.float().t()
    err = (Y.float() - want).norm() / want.norm()
    assert err < 1e-2, err
    Y2, mask2 = _fwd(A, W, p=0.0, relu=True)
    want2 = torch.relu(want)
    assert ((Y2.float() - want2).norm() / want2.norm()) < 1e-2
    # relu bits agree except where the fp32 value sits within bf16 rounding of 0
    bits = torch.stack([(mask2 >> j) & 1 for j in range(8)], 1).reshape(M, 256).bool()
    agree = (bits == (want > 0)) | (want.abs() < 1e-2)
    assert agree.all()


@pytest.mark.parametrize("K", [256, 512])
def test_tc_fwd_dropout_matches_unfused_kernels(K):
    M = 4096
    g = torch.Generator(device="cuda").manual_seed(1)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = (torch.randn(256, K, device="cuda", generator=g) * 0.06).to(torch.bfloat16)
    salt = torch.tensor([5], dtype=torch.int64, device="cuda")
    Y, mask = _fwd(A, W, p=0.5, relu=True, seed=123, salt=salt)
    # unfused: torch GEMM -> library relu_dropout with the same seed/salt
    z = (A.float() @ W.float().t()).to(torch.bfloat16)
    y_ref = torch.empty_like(z)
    m_ref = torch.empty(M * 32, dtype=torch.uint8, device="cuda")
    L = _lib.lib()
    _lib.check(L.sal_relu_dropout_fwd(z.data_ptr(), z.stride(0), y_ref.data_ptr(),
                                      y_ref.stride(0), M, 256, _lib.SAL_BF16, m_ref.data_ptr(),
                                      0.5, 123, salt.data_ptr(), _lib.stream_ptr()), "relu")
    torch.cuda.synchronize()
    same = (mask == m_ref).float().mean().item()
    assert same > 0.995, same  # differences only where z ~ 0 (accumulation order)
    keep = torch.stack([(mask >> j) & 1 for j in range(8)], 1).reshape(M, 256).float()
    frac = keep.sum() / ((z.float() > 0).float().sum())
    assert 0.45 < frac.item() < 0.55


@pytest.mark.parametrize("M,N,K", [(64, 256, 256), (1000, 256, 256), (67584, 256, 256),
                                   (6144, 256, 512), (777, 128, 384)])
def test_tc_wgrad_matches_torch(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M + 1)
    dz = (torch.randn(M, N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    A = (torch.randn(M, 2 * K, device="cuda", generator=g)).to(torch.bfloat16)[:, :K]
    dW = torch.full((N, K), 7.0, device="cuda")
    L = _lib.lib()
    _lib.check(L.sal_tc_sage_wgrad(dz.data_ptr(), dz.stride(0), A.data_ptr(), A.stride(0), M,
                                   None, N, K, dW.data_ptr(), dW.stride(0), 0, _lib.stream_ptr()),
               "tc_sage_wgrad")
    # accumulate mode adds into dW (the trainer's Adam leaves the gradient zeroed)
    dW2 = torch.full((N, K), 0.5, device="cuda")
    _lib.check(L.sal_tc_sage_wgrad(dz.data_ptr(), dz.stride(0), A.data_ptr(), A.stride(0), M,
                                   None, N, K, dW2.data_ptr(), dW2.stride(0), 1, _lib.stream_ptr()),
               "tc_sage_wgrad(accumulate)")
    torch.cuda.synchronize()
    want = dz.float().t() @ A.float()
    assert ((dW2 - 0.5 - want).norm() / want.norm()).item() < 1e-3
    err = (dW - want).norm() / want.norm()
    assert err < 1e-3, err


@pytest.mark.parametrize("K", [256, 512])
@pytest.mark.parametrize("m_true", [0, 1, 300, 1000, 4096])
def test_tc_fwd_true_row_count_zero_fills_padding(m_true, K):
    """Static shapes pad to M; rows past *m_dev come out zero (Y and mask) and the
    rows before it equal the full computation."""
    M = 4096
    g = torch.Generator(device="cuda").manual_seed(9)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = (torch.randn(256, K, device="cuda", generator=g) * 0.06).to(torch.bfloat16)
    salt = torch.tensor([3], dtype=torch.int64, device="cuda")
    Yf, mf = _fwd(A, W, p=0.5, relu=True, seed=11, salt=salt)
    md = torch.tensor([m_true], dtype=torch.int64, device="cuda")
    Yp, mp = _fwd(A, W, p=0.5, relu=True, seed=11, salt=salt, m_dev=md, fill=7.0)
    tile_end = min(M, -(-m_true // 128) * 128)   # whole 128-row tiles are computed
    assert torch.equal(Yp[:tile_end], Yf[:tile_end])
    assert torch.equal(mp[:tile_end * 32], mf[:tile_end * 32])
    assert (Yp[tile_end:] == 0).all() and (mp[tile_end * 32:] == 0).all()


@pytest.mark.parametrize("m_true", [0, 100, 3000, 4096])
def test_tc_wgrad_true_row_count(m_true):
    """With *m_dev the split-K ranges cover only the first m_true rows (in whole
    64-row chunks: the contract is that dz rows past m_true are zero, as the
    trainer's padding rows are)."""
    M, N, K = 4096, 256, 256
    g = torch.Generator(device="cuda").manual_seed(17)
    dz = (torch.randn(M, N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    dz[m_true:] = 0
    dz[-(-m_true // 64) * 64:] = float("nan")   # chunks past the last partial one: never read
    A = (torch.randn(M, K, device="cuda", generator=g)).to(torch.bfloat16)
    dW = torch.full((N, K), 3.0, device="cuda")
    md = torch.tensor([m_true], dtype=torch.int64, device="cuda")
    L = _lib.lib()
    _lib.check(L.sal_tc_sage_wgrad(dz.data_ptr(), dz.stride(0), A.data_ptr(), A.stride(0), M,
                                   md.data_ptr(), N, K, dW.data_ptr(), dW.stride(0), 0,
                                   _lib.stream_ptr()), "tc_sage_wgrad(m_dev)")
    torch.cuda.synchronize()
    want = dz[:m_true].float().t() @ A[:m_true].float()
    if m_true == 0:
        assert (dW == 0).all()
    else:
        assert ((dW - want).norm() / want.norm()).item() < 1e-3


@pytest.mark.parametrize("m_true,parts", [(0, 2), (100, 2), (3000, 3), (4096, 4), (1000, 8),
                                          (4000, 5)])
def test_tc_wgrad_parts_sum_to_whole(m_true, parts):
    """sal_tc_sage_wgrad_part over parts 0..P-1 (the first zeroing dW) equals the
    whole weight gradient; no part reads a row past the 64-row chunk holding
    the last live row."""
    M, N, K = 4096, 256, 256
    g = torch.Generator(device="cuda").manual_seed(19)
    dz = (torch.randn(M, N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    dz[m_true:] = 0
    dz[-(-m_true // 64) * 64:] = float("nan")
    A = (torch.randn(M, K, device="cuda", generator=g)).to(torch.bfloat16)
    dW = torch.full((N, K), 3.0, device="cuda")
    md = torch.tensor([m_true], dtype=torch.int64, device="cuda")
    L = _lib.lib()
    for k in range(parts):
        _lib.check(L.sal_tc_sage_wgrad_part(dz.data_ptr(), dz.stride(0), A.data_ptr(),
                                            A.stride(0), M, md.data_ptr(), k, parts, N, K,
                                            dW.data_ptr(), dW.stride(0), 1 if k else 0,
                                            _lib.stream_ptr()), "tc_sage_wgrad_part")
    torch.cuda.synchronize()
    want = dz[:m_true].float().t() @ A[:m_true].float()
    if m_true == 0:
        assert (dW == 0).all()
    else:
        assert ((dW - want).norm() / want.norm()).item() < 1e-3
