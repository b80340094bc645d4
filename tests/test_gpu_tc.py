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


@pytest.mark.parametrize("N", [176, 48, 256])
def test_tc_wgrad_output_layer_rows(N):
    """The output layer's dW [c_pad, 2f]: N a multiple of 16 but not of 128 — dz
    columns past N are read as zero (TMA) and dW rows past N are not written."""
    M, K, m_true = 1024, 512, 1000
    g = torch.Generator(device="cuda").manual_seed(23)
    dz = (torch.randn(M, N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    dz[m_true:] = 0
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    A[-(-m_true // 64) * 64:] = float("nan")   # padding rows past the last chunk: never read
    dW = torch.full((N + 16, K), 3.0, device="cuda")
    md = torch.tensor([m_true], dtype=torch.int64, device="cuda")
    L = _lib.lib()
    _lib.check(L.sal_tc_sage_wgrad(dz.data_ptr(), dz.stride(0), A.data_ptr(), A.stride(0), M,
                                   md.data_ptr(), N, K, dW.data_ptr(), dW.stride(0), 1,
                                   _lib.stream_ptr()), "tc_sage_wgrad(N)")
    torch.cuda.synchronize()
    want = dz[:m_true].float().t() @ A[:m_true].float() + 3.0
    assert ((dW[:N] - want).norm() / want.norm()).item() < 1e-3
    assert (dW[N:] == 3.0).all()


def _gemm_nn(A, B, m_dev=None, pad_fill=1, fill=7.0):
    M, K = A.shape
    N = B.shape[1]
    C = torch.full((M, N), fill, dtype=torch.bfloat16, device="cuda")
    L = _lib.lib()
    _lib.check(L.sal_tc_gemm_nn(A.data_ptr(), A.stride(0), M, _lib.ptr(m_dev), K, B.data_ptr(),
                                B.stride(0), N, C.data_ptr(), C.stride(0), pad_fill,
                                _lib.stream_ptr()), "tc_gemm_nn")
    torch.cuda.synchronize()
    return C


@pytest.mark.parametrize("M,K,N", [(1024, 176, 512), (6144, 256, 512), (100, 256, 512),
                                   (67584, 256, 256), (1000, 48, 128), (300, 512, 384)])
def test_tc_gemm_nn_matches_torch(M, K, N):
    """dA = dz @ W_cat: the output layer's (K = c_pad = 176) and the hidden layers'
    (K = 256) input-gradient shapes; K not a multiple of 64 reads zero columns."""
    g = torch.Generator(device="cuda").manual_seed(M + K)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    B = (torch.randn(K, N, device="cuda", generator=g) * 0.06).to(torch.bfloat16)
    C = _gemm_nn(A, B)
    want = A.float() @ B.float()
    assert ((C.float() - want).norm() / want.norm()).item() < 1e-2


@pytest.mark.parametrize("m_true", [0, 1, 127, 128, 1000])
def test_tc_gemm_nn_true_row_count(m_true):
    """Tiles past ceil128(m_true) are zero-filled (pad_fill) or left alone; A rows
    in those tiles are never read."""
    M, K, N = 1024, 256, 512
    g = torch.Generator(device="cuda").manual_seed(5)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    end = min(M, -(-m_true // 128) * 128)
    A[end:] = float("nan")
    B = (torch.randn(K, N, device="cuda", generator=g) * 0.06).to(torch.bfloat16)
    md = torch.tensor([m_true], dtype=torch.int64, device="cuda")
    C = _gemm_nn(A, B, md, pad_fill=1)
    want = A[:end].float() @ B.float()
    if end:
        assert ((C[:end].float() - want).norm() / want.norm()).item() < 1e-2
    assert (C[end:] == 0).all()
    C2 = _gemm_nn(A, B, md, pad_fill=0, fill=7.0)
    assert (C2[end:] == 7.0).all() and torch.equal(C2[:end], C[:end])


def _logits_ref(A, W, C):
    return (A.float() @ W.float().t())[:, :C]


@pytest.mark.parametrize("M,K,C,c_pad", [(1024, 512, 172, 176), (1000, 512, 47, 48),
                                         (300, 128, 40, 48), (2048, 256, 10, 16),
                                         (1024, 512, 192, 192), (700, 256, 100, 112)])
def test_tc_head_matches_torch(M, K, C, c_pad):
    """sal_tc_sage_head = logits, log_softmax + NLL (mean over labels >= 0), dlogits,
    dA = dlogits @ W and dW += dlogits^T @ A in one kernel, against torch in fp32
    (dlogits rounded to bf16 as the kernel's tensor-core operand)."""
    g = torch.Generator(device="cuda").manual_seed(M + C)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = torch.zeros(c_pad, K, device="cuda", dtype=torch.bfloat16)
    W[:C] = (torch.randn(C, K, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    labels = torch.randint(0, C, (M,), device="cuda", generator=g)
    labels[::7] = -1
    m_true = M - 37
    labels[m_true:] = -1
    md = torch.tensor([m_true], dtype=torch.int64, device="cuda")
    loss = torch.full((), 0.25, device="cuda")
    dlog = torch.full((M, c_pad), 9.0, dtype=torch.bfloat16, device="cuda")
    dA = torch.full((M, K), 9.0, dtype=torch.bfloat16, device="cuda")
    dW = torch.full((c_pad, K), 2.0, device="cuda")
    L = _lib.lib()
    ws = torch.full((L.sal_tc_sage_head_ws_bytes(M, K, c_pad),), 255, dtype=torch.uint8,
                    device="cuda")
    _lib.check(L.sal_tc_sage_head(A.data_ptr(), A.stride(0), M, md.data_ptr(), K, W.data_ptr(),
                                  W.stride(0), c_pad, C, labels.data_ptr(), M, loss.data_ptr(),
                                  dlog.data_ptr(), dlog.stride(0), dA.data_ptr(), dA.stride(0),
                                  dW.data_ptr(), dW.stride(0), ws.data_ptr(), ws.numel(),
                                  _lib.stream_ptr()), "tc_sage_head")
    torch.cuda.synchronize()
    z = _logits_ref(A, W, C).requires_grad_(True)
    keep = labels >= 0
    ref = torch.nn.functional.nll_loss(torch.log_softmax(z, -1)[keep], labels[keep])
    ref.backward()
    assert abs(loss.item() - 0.25 - ref.item()) < 1e-4 * max(1.0, ref.item())
    got = dlog.float()
    assert torch.allclose(got[:, :C], z.grad, atol=2e-4, rtol=1e-2)
    assert (got[:, C:] == 0).all()
    tile_end = min(M, -(-m_true // 128) * 128)
    assert (got[tile_end:] == 0).all()
    gb = got.to(torch.bfloat16).float()               # the operand the kernel multiplies
    want_dA = gb @ W.float()
    assert ((dA.float() - want_dA).norm() / want_dA.norm()).item() < 1e-2
    assert (dA[tile_end:] == 0).all()
    want_dW = gb.t() @ A.float() + 2.0
    assert ((dW - want_dW).norm() / (want_dW - 2.0).norm()).item() < 1e-3


@pytest.mark.parametrize("M,K,C,c_pad", [(1024, 512, 172, 176), (500, 128, 40, 48)])
def test_tc_logits_argmax_matches_torch(M, K, C, c_pad):
    g = torch.Generator(device="cuda").manual_seed(M)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = torch.zeros(c_pad, K, device="cuda", dtype=torch.bfloat16)
    W[:C] = (torch.randn(C, K, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    z = _logits_ref(A, W, C)
    labels = z.argmax(-1)
    labels[::3] = torch.randint(0, C, (labels[::3].numel(),), device="cuda", generator=g)
    labels[::11] = -1
    counts = torch.zeros(2, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    ws = torch.empty(L.sal_tc_sage_head_ws_bytes(M, K, c_pad), dtype=torch.uint8, device="cuda")
    _lib.check(L.sal_tc_sage_logits_argmax(A.data_ptr(), A.stride(0), M, None, K, W.data_ptr(),
                                           W.stride(0), c_pad, C, labels.data_ptr(), M,
                                           counts.data_ptr(), ws.data_ptr(), ws.numel(),
                                           _lib.stream_ptr()), "argmax")
    torch.cuda.synchronize()
    keep = labels >= 0
    want_ok = int((z.argmax(-1)[keep] == labels[keep]).sum())
    assert int(counts[1]) == int(keep.sum())
    # near-ties between the fp32 TMEM logits and the reference's summation order
    top2 = z.topk(2, -1).values
    ties = int(((top2[:, 0] - top2[:, 1]) < 1e-3)[keep].sum())
    assert abs(int(counts[0]) - want_ok) <= ties
