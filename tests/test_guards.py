"""Out-of-bounds and determinism guards for the CUDA kernels (GPU).

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset), so the
memcheck / racecheck coverage it would give is approximated here:
  * every output buffer sits between two 64 KB canary regions filled with a byte pattern; a
    kernel that writes outside its output (a bad tile bound, a wrong stride, a mask off by one)
    changes a canary byte;
  * kernels whose reduction order is fixed are run twice on the same inputs and must agree
    bit for bit (a shared-memory race or a missing barrier shows up as run-to-run noise).
Shapes include ragged edges (M, N not multiples of the tile) where the kernels support them.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

PAD = 1 << 16  # canary bytes on each side
PATTERN = 0xA5


def guarded(shape, dtype):
    """A tensor of `shape` inside a byte buffer with canaries on both sides; returns (t, check)."""
    n = 1
    for s in shape:
        n *= s
    es = torch.empty((), dtype=dtype).element_size()
    raw = torch.full((2 * PAD + n * es,), PATTERN, dtype=torch.uint8, device="cuda")
    t = raw[PAD:PAD + n * es].view(dtype).view(*shape)

    def check(name=""):
        torch.cuda.synchronize()
        lo, hi = raw[:PAD], raw[PAD + n * es:]
        bad_lo = int((lo != PATTERN).sum())
        bad_hi = int((hi != PATTERN).sum())
        assert bad_lo == 0 and bad_hi == 0, f"{name}: {bad_lo} bytes below, {bad_hi} above the output changed"

    return t, check


def _r(*shape, dtype=torch.bfloat16, scale=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(dtype)


@pytest.mark.parametrize("M,N,K", [(1000, 776, 264), (16384, 3072, 2048), (200, 136, 72)])
@pytest.mark.parametrize("force", ["", "256,2,1", "128,1,1", "256,1,4"])
def test_gemm_bounds_and_determinism(cuda, monkeypatch, M, N, K, force):
    from paper_2602_08387_b200 import ops

    if force:
        monkeypatch.setenv("B2S_GEMM_FORCE", force)
    a, b = _r(M, K, seed=1), _r(N, K, seed=2, scale=K ** -0.5)
    c, check = guarded((M, N), torch.bfloat16)
    ops.gemm(a, b, a_mn=False, b_mn=False, M=M, N=N, K=K, out=c)
    check("gemm bf16")
    c1 = c.clone()
    ops.gemm(a, b, a_mn=False, b_mn=False, M=M, N=N, K=K, out=c)
    assert torch.equal(c, c1), "bf16 GEMM not deterministic"
    acc, check32 = guarded((M, N), torch.float32)
    acc.zero_()
    ops.gemm(a, b, a_mn=False, b_mn=False, M=M, N=N, K=K, out=acc, accumulate=True)
    check32("gemm f32 accumulate / split-K")


def test_gemm_rope_swiglu_bounds(cuda):
    from paper_2602_08387_b200 import ops
    from paper_2602_08387_b200.model import PRESETS, rope_tables

    cfg = PRESETS["tiny-llama"]
    M, d, F = 512, cfg.d_model, cfg.d_ff
    x = _r(M, d, seed=3)
    w = _r(cfg.qkv_dim, d, seed=4, scale=d ** -0.5)
    cos, sin = rope_tables(cfg, 256, cuda)
    out, check = guarded((M, cfg.qkv_dim), torch.bfloat16)
    ops.linear_rope(x, w, out, 256, cfg.head_dim, (cfg.n_head + cfg.n_kv_head) * cfg.head_dim, cos, sin)
    check("gemm_rope")
    w13 = _r(2 * F, d, seed=5, scale=d ** -0.5)
    gu, cg = guarded((M, 2 * F), torch.bfloat16)
    h, ch = guarded((M, F), torch.bfloat16)
    ops.linear_swiglu(x, w13, gu, h)
    cg("swiglu gu")
    ch("swiglu h")
    w2 = _r(d, F, seed=6, scale=F ** -0.5)
    dgu, cd = guarded((M, 2 * F), torch.bfloat16)
    ops.linear_dgrad_swiglu(_r(M, d, seed=7), w2, gu, dgu)
    cd("swiglu bwd")


@pytest.mark.parametrize("B,T,Hq,Hkv,dh", [(2, 256, 4, 2, 64), (1, 384, 3, 3, 64), (1, 256, 2, 1, 128),
                                           (1, 1024, 8, 2, 64)])
def test_attention_bounds_and_determinism(cuda, B, T, Hq, Hkv, dh):
    from paper_2602_08387_b200 import ops

    qkv = _r(B * T, (Hq + 2 * Hkv) * dh, seed=8)
    o, co = guarded((B * T, Hq * dh), torch.bfloat16)
    lse, cl = guarded((B, Hq, T), torch.float32)
    ops.attn_fwd(qkv, B, T, Hq, Hkv, dh, o=o, lse=lse)
    co("attn o")
    cl("attn lse")
    o1, l1 = o.clone(), lse.clone()
    ops.attn_fwd(qkv, B, T, Hq, Hkv, dh, o=o, lse=lse)
    assert torch.equal(o, o1) and torch.equal(lse, l1), "attention forward not deterministic"
    do = _r(B * T, Hq * dh, seed=9)
    dqkv, cq = guarded((B * T, (Hq + 2 * Hkv) * dh), torch.bfloat16)
    ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh, dqkv=dqkv)
    cq("attn dqkv")


def test_bandwidth_kernels_bounds(cuda):
    from paper_2602_08387_b200 import ops

    M, D = 777, 768
    x = _r(M, D, dtype=torch.float32, seed=10)
    g, b = torch.ones(D, device=cuda).bfloat16(), torch.zeros(D, device=cuda).bfloat16()
    y, cy = guarded((M, D), torch.bfloat16)
    mean, cm = guarded((M,), torch.float32)
    rstd, cr = guarded((M,), torch.float32)
    ops.layernorm_fwd(x, g, b, 1e-5, y, mean, rstd)
    cy("layernorm y")
    cm("layernorm mean")
    cr("layernorm rstd")
    y2 = y.clone()
    ops.layernorm_fwd(x, g, b, 1e-5, y, mean, rstd)
    assert torch.equal(y, y2)
    dx, cdx = guarded((M, D), torch.float32)
    dx.zero_()
    dxb, cdb = guarded((M, D), torch.bfloat16)
    dg, cdg = guarded((D,), torch.float32)
    dbb, cbb = guarded((D,), torch.float32)
    dg.zero_()
    dbb.zero_()
    ops.layernorm_bwd(x, _r(M, D, seed=11), g, mean, rstd, dx, dxb, dg, dbb)
    for c, n in ((cdx, "dx"), (cdb, "dxb"), (cdg, "dgamma"), (cbb, "dbeta")):
        c("layernorm bwd " + n)
    V, ld = 1000, 1008
    logits, cx = guarded((M, ld), torch.bfloat16)
    logits.copy_(_r(M, ld, seed=12))
    loss, cls_ = guarded((M,), torch.float32)
    tgt = torch.randint(0, V, (M,), device=cuda)
    ops.cross_entropy(logits, V, tgt, loss, grad_scale=1.0 / M)
    cx("cross-entropy dlogits")
    cls_("cross-entropy loss rows")
    n = 1_000_003 // 4 * 4
    p, m_, v_, gr = (torch.randn(n, device=cuda) for _ in range(4))
    pb, cp = guarded((n,), torch.bfloat16)
    ops.adamw(p, m_, v_, gr, pb, 3, 1e-3, 0.9, 0.95, 1e-8, 0.1)
    cp("adamw bf16 shard")


def test_gather_bounds(cuda, tmp_path):
    import numpy as np

    from paper_2602_08387_b200 import _lib
    from paper_2602_08387_b200.packed import DevicePackedStream, PackedWriter, open_packed

    path = str(tmp_path / "g.cfpk")
    with PackedWriter(path, 2) as w:
        w.write_stream(np.random.default_rng(0).integers(0, 4096, size=100_003), 1000)
    r = open_packed(path)
    ds = DevicePackedStream(r, torch.device("cuda"))
    B, L = 7, 333
    ids = torch.tensor([0, 5, 299, 17, 3, 150, 298], dtype=torch.int64, device=cuda)
    inp, ci = guarded((B, L), torch.int64)
    tg, ct = guarded((B, L), torch.int64)
    _lib.call("b2s_gather_samples", ds.payload.data_ptr(), ds.token_width, ds.token_count, ids.data_ptr(), B, L,
              inp.data_ptr(), tg.data_ptr(), ds.status.data_ptr(), _lib.stream_ptr())
    ci("gather inputs")
    ct("gather targets")
