"""Parity of the production bf16 tcgen05 path at the headline shapes (BASELINE configs[1]/[2]/[3]).

The bench times GPT-2 124M at T=2048 and Llama-1B / Llama-8B at T=4096; these tests check the
same kernels at exactly those shapes against plain PyTorch fp32 references on the GPU (true
fp32: TF32 disabled), and a 2-layer model of each headline width end to end against the fp32
oracle (oracle/model_oracle.py) on identical weights and samples (packed_data.py:196-203 feed).

Tolerances (bf16 operands, fp32 accumulation):
  * attention: our error against the fp32 reference must be within 2x (+ a small floor) of the
    error torch's own bf16 SDPA kernel makes on the same inputs -- the bf16 rounding of P / O
    is the floor both pay;
  * GEMMs: fp32 output within 2e-5 * max|ref| (accumulation order only), bf16 output within
    1e-2 * max|ref| (one bf16 rounding);
  * 2-layer steps: loss within 5e-3 relative, every parameter gradient cosine >= 0.995.
"""

import math
from dataclasses import replace

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _true_fp32():
    old = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = old


# ----------------------------------------------------------------------------- attention
ATTN = [  # (B, T, Hq, Hkv, dh): GPT-2 124M, Llama-1B (GQA 32/8), Llama-8B (GQA 32/8, dh 128)
    (2, 2048, 12, 12, 64),
    (1, 4096, 32, 8, 64),
    (1, 4096, 32, 8, 128),
]


def _split(qkv, B, T, Hq, Hkv, dh):
    x = qkv.view(B, T, Hq + 2 * Hkv, dh)
    return (x[:, :, :Hq].transpose(1, 2), x[:, :, Hq:Hq + Hkv].transpose(1, 2),
            x[:, :, Hq + Hkv:].transpose(1, 2))


def _ref_attn(qkv32, B, T, Hq, Hkv, dh):
    """fp32 causal attention (explicit softmax) -> (o [B*T, Hq*dh], lse [B, Hq, T])."""
    q, k, v = _split(qkv32, B, T, Hq, Hkv, dh)
    g = Hq // Hkv
    k, v = k.repeat_interleave(g, 1), v.repeat_interleave(g, 1)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(dh)
    mask = torch.ones(T, T, device=qkv32.device, dtype=torch.bool).tril()
    s = s.masked_fill(~mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ v
    return o.transpose(1, 2).reshape(B * T, Hq * dh), lse


def _sdpa(qkv, B, T, Hq, Hkv, dh):
    q, k, v = _split(qkv, B, T, Hq, Hkv, dh)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=Hq != Hkv)
    return o.transpose(1, 2).reshape(B * T, Hq * dh)


def _inputs(B, T, Hq, Hkv, dh, mode, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(B, T, Hq + 2 * Hkv, dh, device="cuda", generator=g)
    if mode == "peaky":  # scores ~ N(0, 4^2): sharp rows, large maxima
        x = x * 2.0
    elif mode == "ramp":  # key norms grow along the sequence: the running max keeps jumping, so the
        # lazy O rescale (threshold 2^8, attn.cu) fires on many rows
        ramp = torch.linspace(0.5, 3.0, T, device="cuda")[None, :, None, None]
        x[:, :, Hq:Hq + Hkv] *= ramp
        x[:, :, :Hq] *= 1.5
    return x.reshape(B * T, -1).bfloat16()


def _rel(a, b):
    return float((a.float() - b).abs().max() / b.abs().max())


@pytest.mark.parametrize("mode", ["unit", "peaky", "ramp"])
@pytest.mark.parametrize("B,T,Hq,Hkv,dh", ATTN)
def test_attn_fwd_headline(cuda, B, T, Hq, Hkv, dh, mode):
    from paper_2602_08387_b200 import ops

    qkv = _inputs(B, T, Hq, Hkv, dh, mode, seed=T + Hq + dh)
    o, lse = ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
    ro, rl = _ref_attn(qkv.float(), B, T, Hq, Hkv, dh)
    so = _sdpa(qkv, B, T, Hq, Hkv, dh)
    err, sdpa_err = _rel(o, ro), _rel(so, ro)
    assert err <= 2 * sdpa_err + 2e-3, (err, sdpa_err)
    torch.testing.assert_close(lse, rl, rtol=2e-4, atol=2e-3)


@pytest.mark.parametrize("mode", ["unit", "ramp"])
@pytest.mark.parametrize("B,T,Hq,Hkv,dh", ATTN)
def test_attn_bwd_headline(cuda, B, T, Hq, Hkv, dh, mode):
    from paper_2602_08387_b200 import ops

    qkv = _inputs(B, T, Hq, Hkv, dh, mode, seed=T + Hq + dh + 7)
    o, lse = ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
    g = torch.Generator(device="cuda").manual_seed(11)
    do = torch.randn(B * T, Hq * dh, device="cuda", generator=g).bfloat16()
    dqkv = ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh)
    # fp32 reference gradient (same bf16 inputs and dO)
    x = qkv.float().requires_grad_()
    ro, _ = _ref_attn(x, B, T, Hq, Hkv, dh)
    ro.backward(do.float())
    ref = x.grad.view(B * T, Hq + 2 * Hkv, dh)
    # yardstick: torch's bf16 SDPA backward on the same inputs
    xs = qkv.clone().requires_grad_()
    _sdpa(xs, B, T, Hq, Hkv, dh).backward(do)
    sd = xs.grad.view(B * T, Hq + 2 * Hkv, dh)
    got = dqkv.view(B * T, Hq + 2 * Hkv, dh)
    for name, sl in (("dq", slice(0, Hq)), ("dk", slice(Hq, Hq + Hkv)), ("dv", slice(Hq + Hkv, Hq + 2 * Hkv))):
        err, sdpa_err = _rel(got[:, sl], ref[:, sl]), _rel(sd[:, sl], ref[:, sl])
        assert err <= 2 * sdpa_err + 5e-3, (name, err, sdpa_err)
        cos = torch.nn.functional.cosine_similarity(got[:, sl].reshape(-1).double(), ref[:, sl].reshape(-1).double(),
                                                    dim=0)
        assert cos > 0.9995, (name, float(cos))


# ----------------------------------------------------------------------------- GEMMs
def step_gemms(cfg, M):
    """Every (M, N, K, a_mn, b_mn, out, accumulate, bias, act) GEMM the bf16 step launches
    (model.DecoderLM.forward_backward), plus the fused SwiGLU entry points."""
    d, f, V, qkv, hd = cfg.d_model, cfg.d_ff, cfg.padded_vocab, cfg.qkv_dim, cfg.n_head * cfg.head_dim
    g = []
    gpt2 = cfg.arch == "gpt2"
    # forward: qkv, o-proj, (fc | gate-up), (fc2 | down), head
    g += [(M, qkv, d, 0, 0, "bf16", 0, gpt2, 0), (M, d, hd, 0, 0, "bf16", 0, gpt2, 0)]
    if gpt2:
        g += [(M, f, d, 0, 0, "bf16", 0, 1, 5), (M, d, f, 0, 0, "bf16", 0, 1, 0)]
    else:
        g += [("swiglu_fwd", M, f, d), (M, d, f, 0, 0, "bf16", 0, 0, 0)]
    g += [(M, V, d, 0, 0, "bf16", 0, 0, 0)]
    # backward: head wgrad / dgrad, then per block (weight gradients in overwrite mode: acc 2)
    g += [(V, d, M, 1, 1, "f32", 2, 0, 0), (M, d, V, 0, 1, "bf16", 0, 0, 0)]
    if gpt2:
        g += [(d, f, M, 1, 1, "f32", 2, 0, 0), ("colsum", M, f, d, 6), (f, d, M, 1, 1, "f32", 2, 0, 0),
              (M, d, f, 0, 1, "bf16", 0, 0, 0)]
    else:
        g += [(d, f, M, 1, 1, "f32", 2, 0, 0), ("swiglu_bwd", M, f, d), (2 * f, d, M, 1, 1, "f32", 2, 0, 0),
              (M, d, 2 * f, 0, 1, "bf16", 0, 0, 0)]
    g += [(d, hd, M, 1, 1, "f32", 2, 0, 0), (M, hd, d, 0, 1, "bf16", 0, 0, 0),
          (qkv, d, M, 1, 1, "f32", 2, 0, 0), (M, d, qkv, 0, 1, "bf16", 0, 0, 0)]
    out = []
    for x in g:
        if x not in out:
            out.append(x)
    return out


def _headline_cfgs():
    from paper_2602_08387_b200.model import PRESETS

    return {"gpt2-124m": (PRESETS["gpt2-124m"], 8 * 2048), "llama-1b": (PRESETS["llama-1b"], 4 * 4096),
            "llama-8b": (PRESETS["llama-8b"], 2 * 4096)}


def _gemm_cases():
    from paper_2602_08387_b200.model import PRESETS

    cases = []
    for name, M in (("gpt2-124m", 8 * 2048), ("llama-1b", 4 * 4096), ("llama-8b", 2 * 4096)):
        for sh in step_gemms(PRESETS[name], M):
            cases.append(pytest.param(name, sh, id=f"{name}-" + "-".join(str(v) for v in sh)))
    return cases


def _rnd(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).bfloat16()


@pytest.mark.parametrize("name,shape", _gemm_cases())
def test_step_gemm_headline(cuda, name, shape):
    from paper_2602_08387_b200 import ops

    torch.cuda.empty_cache()
    if shape[0] == "swiglu_fwd":
        _, M, F, K = shape
        x, w = _rnd((M, K), 1), _rnd((2 * F, K), 2, K ** -0.5)
        gu = torch.empty(M, 2 * F, device=cuda, dtype=torch.bfloat16)
        h = torch.empty(M, F, device=cuda, dtype=torch.bfloat16)
        ops.linear_swiglu(x, w, gu, h)
        ref = x.float() @ w.float().t()
        assert _rel(gu, ref) < 1e-2
        rh = torch.nn.functional.silu(gu[:, :F].float()) * gu[:, F:].float()  # from the stored bf16 gate / up
        assert _rel(h, rh) < 1e-2
        return
    if shape[0] == "swiglu_bwd":
        _, M, F, K = shape
        dy, w2 = _rnd((M, K), 3), _rnd((K, F), 4, K ** -0.5)
        gu = _rnd((M, 2 * F), 5)
        dgu = torch.empty(M, 2 * F, device=cuda, dtype=torch.bfloat16)
        ops.linear_dgrad_swiglu(dy, w2, gu, dgu)
        dh = dy.float() @ w2.float()
        gt, up = gu[:, :F].float(), gu[:, F:].float()
        sg = torch.sigmoid(gt)
        ref_dg = dh * up * sg * (1 + gt * (1 - sg))
        ref_du = dh * gt * sg
        assert _rel(dgu[:, :F], ref_dg) < 1.5e-2 and _rel(dgu[:, F:], ref_du) < 1.5e-2
        return
    if shape[0] == "colsum":  # fc2 dgrad with the gelu' product (act 6) and the fc_b column sums
        _, M, F, K, act = shape
        dy, w = _rnd((M, K), 6), _rnd((K, F), 7, K ** -0.5)
        aux = (torch.rand(M, F, device=cuda) * 1.2).bfloat16()  # gelu'(z) values
        colsum = torch.zeros(F, device=cuda)
        dh = ops.linear_dgrad(dy, w, act=act, aux=aux, colsum_out=colsum)
        ref = (dy.float() @ w.float()) * aux.float()
        assert _rel(dh, ref) < 1e-2
        assert _rel(colsum, dh.float().sum(0)) < 1e-4  # bias grad = column sums of the stored dh
        return
    M, N, K, a_mn, b_mn, dt, acc, bias, act = shape
    a = _rnd((K, M) if a_mn else (M, K), 8)
    b = _rnd((K, N) if b_mn else (N, K), 9, K ** -0.5)
    ref = (a.float().t() if a_mn else a.float()) @ (b.float() if b_mn else b.float().t())
    bv = _rnd((N,), 10) if bias else None
    if bv is not None:
        ref = ref + bv.float()
    if dt == "f32":
        init = torch.randn(M, N, device=cuda) if acc else None
        out = init.clone() if acc else torch.empty(M, N, device=cuda)
        ops.gemm(a, b, a_mn=bool(a_mn), b_mn=bool(b_mn), M=M, N=N, K=K, out=out, accumulate=acc, bias=bv)
        want = ref + init if acc == 1 else ref  # acc 2 (overwrite): whatever C held is replaced
        assert _rel(out, want) < (2e-5 if acc == 1 else 5e-5), _rel(out, want)  # acc 2: relative to the bare product
        return
    if act == 5:  # bias + GELU(tanh); aux = gelu'(z)
        aux = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
        y = ops.gemm(a, b, a_mn=False, b_mn=False, M=M, N=N, K=K, bias=bv, act=5, aux=aux)
        z = ref
        assert _rel(y, torch.nn.functional.gelu(z, approximate="tanh")) < 1e-2
        zz = z.clone().requires_grad_()
        torch.nn.functional.gelu(zz, approximate="tanh").sum().backward()
        assert _rel(aux, zz.grad) < 1e-2
        return
    y = ops.gemm(a, b, a_mn=bool(a_mn), b_mn=bool(b_mn), M=M, N=N, K=K, bias=bv)
    assert _rel(y, ref) < 1e-2, _rel(y, ref)


@pytest.mark.parametrize("name", ["gpt2-124m", "llama-1b"])
def test_step_gemm_list_is_complete(cuda, tmp_path, name):
    """The GEMM list above is exactly what a (2-layer, full-width) bf16 step launches."""
    from paper_2602_08387_b200 import ops

    cfg, M = _headline_cfgs()[name]
    cfg2 = replace(cfg, n_layer=2)
    B, T = (8, 2048) if name == "gpt2-124m" else (4, 4096)
    tr = _trainer(tmp_path, cfg2, B, T)
    x, y = tr.dataloader.batch(0)
    with ops.KernelTimer() as kt:
        tr.engine.begin_step()
        tr.model.forward_backward(x, y, hooks=tr.engine)
    got = {(d[0], d[1], d[2]) for (kind, d), *_ in kt.detail() if kind == "gemm"}
    want = set()
    for s in step_gemms(cfg, M):
        if s[0] == "swiglu_fwd":
            want.add((s[1], 2 * s[2], s[3]))
        elif s[0] in ("swiglu_bwd", "colsum"):
            want.add((s[1], s[2], s[3]))
        else:
            want.add(tuple(s[:3]))
    assert got == want, (sorted(got - want), sorted(want - got))


# ----------------------------------------------------------------------------- 2-layer steps
def _trainer(tmp_path, cfg, B, T, init_device="cpu"):
    from paper_2602_08387_b200.data import PackedDataLoader, Sampler, make_synthetic_packed
    from paper_2602_08387_b200.model import DecoderLM
    from paper_2602_08387_b200.optim import AdamWConfig
    from paper_2602_08387_b200.packed import open_packed
    from paper_2602_08387_b200.trainer import SPMDTrainer

    path = str(tmp_path / "data.cfpk")
    make_synthetic_packed(path, 8 * B * (T + 1), cfg.vocab_size, kind="uniform", seed=3)
    dl = PackedDataLoader(open_packed(path), B, T, Sampler(shuffle=True, seed=2))
    return SPMDTrainer(DecoderLM(cfg), AdamWConfig(), dl, seed=0, init_device=init_device).setup()


@pytest.mark.parametrize("name,B,T", [("gpt2-124m", 2, 2048), ("llama-1b", 1, 4096)])
def test_two_layer_headline_step_matches_oracle(cuda, tmp_path, name, B, T):
    """2-layer GPT-2-124M-width (T=2048) and Llama-1B-width (T=4096, GQA 32/8, vocab 128256)
    bf16 steps vs the fp32 oracle on the GPU: loss within 5e-3, every gradient cosine >= 0.995."""
    from oracle.model_oracle import OracleModel
    from paper_2602_08387_b200.model import init_params

    cfg = replace(_headline_cfgs()[name][0], n_layer=2)
    tr = _trainer(tmp_path, cfg, B, T)
    x, y = tr.dataloader.batch(0)
    tr.engine.begin_step()
    loss = float(tr.model.forward_backward(x, y, hooks=tr.engine).item())
    torch.cuda.synchronize()
    gpu = tr.params.grads_full_fp32()
    del tr
    torch.cuda.empty_cache()
    om = OracleModel(cfg, init_params(cfg, 0)).to(cuda)
    oloss = om(x, y)
    oloss.backward()
    assert abs(loss - oloss.item()) / oloss.item() < 5e-3, (loss, oloss.item())
    for k, p in om.params.items():
        key = k.replace("__", ".")
        g = p.grad
        gg = gpu[key].to(cuda)[: g.shape[0]] if g.dim() else gpu[key].to(cuda)
        cos = torch.nn.functional.cosine_similarity(gg.reshape(-1).double(), g.reshape(-1).double(), dim=0)
        assert cos >= 0.995, (key, float(cos))


# ----------------------------------------------------------------------------- fused RoPE
@pytest.mark.parametrize("name,M,T", [("llama-1b", 4 * 4096, 4096), ("llama-8b", 2 * 4096, 4096),
                                      ("tiny-llama", 2 * 256, 256)])
def test_qkv_gemm_rope_epilogue(cuda, name, M, T):
    """b2s_gemm_rope (RoPE in the QKV GEMM epilogue) == b2s_gemm then b2s_rope, at the step shapes."""
    from paper_2602_08387_b200 import ops
    from paper_2602_08387_b200.model import PRESETS, rope_tables

    cfg = PRESETS[name]
    d, H, Hkv, dh = cfg.d_model, cfg.n_head, cfg.n_kv_head, cfg.head_dim
    N = cfg.qkv_dim
    x, w = _rnd((M, d), 21), _rnd((N, d), 22, d ** -0.5)
    cos, sin = rope_tables(cfg, T, cuda)
    ref = ops.linear(x, w)
    ops.rope(ref, T, H + Hkv, dh, cos, sin)
    out = torch.empty_like(ref)
    ops.linear_rope(x, w, out, T, dh, (H + Hkv) * dh, cos, sin)
    # same bf16 input to the same fp32 rotation: equal up to one bf16 rounding of a contraction
    diff = (out.float() - ref.float()).abs()
    assert float(diff.max()) <= 2 ** -7 * float(ref.float().abs().max()), float(diff.max())
    assert float((diff > 0).float().mean()) < 1e-3
    torch.testing.assert_close(out[:, (H + Hkv) * dh:], ref[:, (H + Hkv) * dh:], rtol=0, atol=0)  # v untouched


@pytest.mark.parametrize("B,T,Hq,Hkv,dh", [(1, 4096, 32, 8, 64), (1, 4096, 32, 8, 128), (2, 256, 4, 2, 64)])
def test_attn_bwd_rope(cuda, B, T, Hq, Hkv, dh):
    """b2s_attn_bwd_rope == b2s_attn_bwd followed by the inverse rotation of the q and k heads."""
    from dataclasses import replace as _r

    from paper_2602_08387_b200 import ops
    from paper_2602_08387_b200.model import PRESETS, rope_tables

    cfg = _r(PRESETS["llama-1b"], d_model=Hq * dh, n_head=Hq, n_kv_head=Hkv)
    cos, sin = rope_tables(cfg, T, cuda)
    qkv = _inputs(B, T, Hq, Hkv, dh, "unit", seed=5)
    o, lse = ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
    g = torch.Generator(device="cuda").manual_seed(6)
    do = torch.randn(B * T, Hq * dh, device="cuda", generator=g).bfloat16()
    ref = ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh).clone()
    ops.rope(ref, T, Hq + Hkv, dh, cos, sin, inverse=True)
    got = ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh, rope=(cos, sin))
    # dq: the fused path rotates the fp32 accumulator (one bf16 rounding instead of two)
    scale = float(ref.float().abs().max())
    assert float((got.float() - ref.float()).abs().max()) <= 2 ** -7 * scale
    torch.testing.assert_close(got[:, Hq * dh:], ref[:, Hq * dh:], rtol=0, atol=0)  # dk (same kernel), dv
