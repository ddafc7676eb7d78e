"""tcgen05 GEMM (K5) vs a plain PyTorch fp32 reference of the same contraction."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(a, b, a_mn, b_mn):
    A = a.float().t() if a_mn else a.float()
    B = b.float() if b_mn else b.float().t()
    return A @ B


SHAPES = [(128, 128, 64), (256, 512, 128), (200, 136, 72), (1000, 776, 264), (384, 2304, 768),
          (130, 256, 4096), (64, 64, 8)]


FORCES = ["", "256,1,1", "128,1,1", "256,2,1"]


@pytest.fixture(params=FORCES)
def force(request, monkeypatch):
    if request.param:
        monkeypatch.setenv("B2S_GEMM_FORCE", request.param)
    else:
        monkeypatch.delenv("B2S_GEMM_FORCE", raising=False)
    return request.param


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_layouts(cuda, a_mn, b_mn, shape, force):
    from paper_2602_08387_b200 import ops

    M, N, K = shape
    if a_mn and M % 8:
        pytest.skip("MN-major A needs M % 8 == 0 (row stride alignment)")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    a = torch.randn((K, M) if a_mn else (M, K), device=cuda, generator=g).bfloat16()
    b = torch.randn((K, N) if b_mn else (N, K), device=cuda, generator=g).bfloat16()
    ref = _ref(a, b, a_mn, b_mn)
    c32 = ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=K, out_f32=True)
    torch.testing.assert_close(c32, ref, rtol=1e-4, atol=1e-3 * K ** 0.5)
    c16 = ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=K)
    torch.testing.assert_close(c16.float(), ref, rtol=1e-2, atol=1e-2 * K ** 0.5)


def test_gemm_epilogues(cuda, force):
    from paper_2602_08387_b200 import ops

    M, N, K = 300, 520, 192
    x = torch.randn(M, K, device=cuda).bfloat16()
    w = torch.randn(N, K, device=cuda).bfloat16() * 0.1
    bias = torch.randn(N, device=cuda).bfloat16()
    pre = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    y = ops.linear(x, w, bias=bias, act=1, aux=pre)
    ref_pre = x.float() @ w.float().t() + bias.float()
    torch.testing.assert_close(pre.float(), ref_pre, rtol=1e-2, atol=2e-2)
    torch.testing.assert_close(y.float(), torch.nn.functional.gelu(pre.float(), approximate="tanh"),
                               rtol=1e-2, atol=2e-2)
    # dgelu epilogue: dh = (dy @ w2) * gelu'(pre)
    w2 = torch.randn(K, N, device=cuda).bfloat16() * 0.1
    dy = torch.randn(M, K, device=cuda).bfloat16()
    dh = ops.linear_dgrad(dy, w2, act=2, aux=pre)
    p = pre.float().requires_grad_()
    torch.nn.functional.gelu(p, approximate="tanh").backward(dy.float() @ w2.float())
    torch.testing.assert_close(dh.float(), p.grad, rtol=2e-2, atol=5e-2)
    # act 5 / 6: the forward stores gelu'(z) instead of z, the backward multiplies by it
    gd = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    y5 = ops.linear(x, w, bias=bias, act=5, aux=gd)
    z = ref_pre.requires_grad_()
    gz = torch.nn.functional.gelu(z, approximate="tanh")
    torch.testing.assert_close(y5.float(), gz.detach(), rtol=1e-2, atol=2e-2)
    gz.backward(torch.ones_like(gz))
    torch.testing.assert_close(gd.float(), z.grad, rtol=1e-2, atol=2e-2)
    dh6 = ops.linear_dgrad(dy, w2, act=6, aux=gd)
    torch.testing.assert_close(dh6.float(), (dy.float() @ w2.float()) * gd.float(), rtol=1e-2, atol=2e-2)
    torch.testing.assert_close(dh6.float(), p.grad, rtol=2e-2, atol=5e-2)
    # dgrad with the bias-gradient column sums from the epilogue (rows not a multiple of 32)
    for act_, aux_ in ((0, None), (6, gd)):
        cs = torch.full((N,), 0.5, device=cuda)
        dhc = ops.linear_dgrad(dy, w2, act=act_, aux=aux_, colsum_out=cs)
        ref_dh = ops.linear_dgrad(dy, w2, act=act_, aux=aux_)
        assert torch.equal(dhc, ref_dh)
        torch.testing.assert_close(cs, 0.5 + ref_dh.float().sum(0), rtol=1e-4, atol=1e-3)
    # accumulate (fp32 and bf16) and wgrad
    acc = torch.randn(N, K, device=cuda)
    ref = acc + dy.new_tensor(0).float() + (torch.randn(0, device=cuda).sum())
    dw = acc.clone()
    dyy = torch.randn(M, N, device=cuda).bfloat16()
    ops.linear_wgrad(dyy, x, out=dw, accumulate=True)
    torch.testing.assert_close(dw, acc + dyy.float().t() @ x.float(), rtol=1e-4, atol=1e-2)
    res = torch.randn(M, N, device=cuda).bfloat16()
    out = res.clone()
    ops.linear(x, w, out=out, accumulate=True)
    torch.testing.assert_close(out.float(), res.float() + x.float() @ w.float().t(), rtol=1e-2, atol=3e-2)


@pytest.mark.parametrize("force_split", ["256,1,4", "256,2,4", "128,1,8"])
def test_gemm_split_k(cuda, monkeypatch, force_split):
    from paper_2602_08387_b200 import ops

    monkeypatch.setenv("B2S_GEMM_FORCE", force_split)
    M, N, K = 768, 2304, 4096  # wgrad-like: few output tiles, long K
    a = torch.randn(K, M, device=cuda).bfloat16()
    b = torch.randn(K, N, device=cuda).bfloat16()
    c = torch.randn(M, N, device=cuda)
    ref = c + a.float().t() @ b.float()
    ops.gemm(a, b, a_mn=True, b_mn=True, M=M, N=N, K=K, out=c, accumulate=True)
    torch.testing.assert_close(c, ref, rtol=1e-4, atol=5e-2)


@pytest.mark.parametrize("force", ["", "256,2,1", "256,2,4", "128,1,8"])
def test_gemm_overwrite_mode(cuda, monkeypatch, force):
    """accumulate=OVERWRITE writes the product whatever C held: a plain store unsplit, a memset
    then the split-K add-reduce when split (the weight-gradient path; C starts as garbage)."""
    from paper_2602_08387_b200 import ops

    if force:
        monkeypatch.setenv("B2S_GEMM_FORCE", force)
    M, N, K = 768, 2304, 4096
    a = torch.randn(K, M, device=cuda).bfloat16()
    b = torch.randn(K, N, device=cuda).bfloat16()
    c = torch.full((M, N), float("nan"), device=cuda)
    ref = a.float().t() @ b.float()
    ops.gemm(a, b, a_mn=True, b_mn=True, M=M, N=N, K=K, out=c, accumulate=ops.OVERWRITE)
    torch.testing.assert_close(c, ref, rtol=1e-4, atol=5e-2)
    # a strided destination (rows of a wider buffer): the memset must touch only the view
    big = torch.full((M, N + 64), 7.0, device=cuda)
    ops.gemm(a, b, a_mn=True, b_mn=True, M=M, N=N, K=K, out=big[:, :N], accumulate=ops.OVERWRITE)
    torch.testing.assert_close(big[:, :N], ref, rtol=1e-4, atol=5e-2)
    assert torch.all(big[:, N:] == 7.0)


@pytest.mark.parametrize("M,F,K", [(2048, 512, 256), (1000, 384, 200), (16384, 8192, 2048)])
def test_swiglu_fused_gemms_match_unfused(cuda, M, F, K):
    """The SwiGLU forward / backward fused into the GEMM epilogues give the unfused chain's bits."""
    from paper_2602_08387_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(M + F)
    x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
    w13 = (torch.randn(2 * F, K, device=cuda, generator=g) * K ** -0.5).bfloat16()
    gu_ref = ops.linear(x, w13)
    h_ref = ops.swiglu_fwd(gu_ref)
    gu = torch.empty_like(gu_ref)
    h = torch.empty_like(h_ref)
    ops.linear_swiglu(x, w13, gu, h)
    assert torch.equal(gu, gu_ref)
    torch.testing.assert_close(h.float(), h_ref.float(), rtol=8e-3, atol=1e-6)  # <= 1 bf16 ulp
    d = 256
    dy = torch.randn(M, d, device=cuda, generator=g).bfloat16()
    w2 = (torch.randn(d, F, device=cuda, generator=g) * d ** -0.5).bfloat16()
    dh = ops.linear_dgrad(dy, w2)
    dgu_ref = ops.swiglu_bwd(gu_ref, dh)
    dgu = torch.empty_like(gu_ref)
    ops.linear_dgrad_swiglu(dy, w2, gu_ref, dgu)
    torch.testing.assert_close(dgu.float(), dgu_ref.float(), rtol=8e-3, atol=1e-5)


@pytest.mark.parametrize("raster", ["1", "3", "-1", "-2", "-5", "mfast"])
@pytest.mark.parametrize("shape", [(1000, 776, 264), (1792, 1280, 192), (384, 2304, 768)])
@pytest.mark.parametrize("force", ["256,2,1", "128,1,1", "256,1,2"])
def test_gemm_rasters(cuda, monkeypatch, raster, shape, force):
    """Every tile raster (gemm.cu tile_mn: M- / N-grouped, partial last groups, split-K) covers
    each output tile exactly once: same result as the fp32 reference."""
    from paper_2602_08387_b200 import ops

    monkeypatch.setenv("B2S_GEMM_RASTER", raster)
    monkeypatch.setenv("B2S_GEMM_FORCE", force)
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    ref = a.float() @ b.float().t()
    c = torch.randn(M, N, device=cuda)
    want = c + ref
    ops.gemm(a, b, a_mn=False, b_mn=False, M=M, N=N, K=K, out=c, accumulate=True)
    torch.testing.assert_close(c, want, rtol=1e-4, atol=1e-3 * K ** 0.5)
