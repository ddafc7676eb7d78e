"""fp32 mode (north star: per-step losses and gradients within 1e-4 relative of the CPU fp32 reference).

Kernel level: the true-fp32 SIMT GEMM / attention against float64 torch of
the same op. Step level: the whole training step in fp32 mode against the CPU
fp32 oracle (oracle/model_oracle.py) on the same weights and samples, at
BASELINE.json configs[0] exactly (tiny GPT-2: 2 layers, d 128, 4 heads -> head
dim 32, seq 256, vocab 4096, 20 steps, batch 8) and at the tiny Llama.
"""

import math

import numpy as np
import pytest
import torch

from oracle import packed_oracle as orc
from oracle.model_oracle import OracleTrainer

pytestmark = pytest.mark.gpu

TOL = 1e-4  # BASELINE.json north_star: "within 1e-4 relative in fp32 mode"


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(128, 128, 16), (200, 136, 72), (1000, 776, 264), (33, 4096, 128), (7, 5, 3)])
def test_gemm_f32_layouts(cuda, a_mn, b_mn, shape):
    from paper_2602_08387_b200 import ops

    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M + 7 * N + 13 * K)
    a = torch.randn((K, M) if a_mn else (M, K), device=cuda, generator=g)
    b = torch.randn((K, N) if b_mn else (N, K), device=cuda, generator=g)
    A = a.double().t() if a_mn else a.double()
    Bm = b.double() if b_mn else b.double().t()
    ref = A @ Bm
    c = ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=K)
    assert c.dtype == torch.float32
    torch.testing.assert_close(c.double(), ref, rtol=1e-5, atol=1e-5 * math.sqrt(K))


def test_gemm_f32_epilogues(cuda):
    from paper_2602_08387_b200 import ops

    M, N, K = 300, 264, 96
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(M, K, device=cuda, generator=g)
    w = torch.randn(N, K, device=cuda, generator=g)
    bias = torch.randn(N, device=cuda, generator=g)
    pre_ref = x.double() @ w.double().t() + bias.double()
    aux = torch.empty(M, N, device=cuda)
    y = ops.linear(x, w, bias=bias, act=1, aux=aux)
    torch.testing.assert_close(aux.double(), pre_ref, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(y.double(), torch.nn.functional.gelu(pre_ref, approximate="tanh"), rtol=1e-5,
                               atol=1e-4)
    # accumulate + bias into an fp32 residual
    r0 = torch.randn(M, N, device=cuda, generator=g)
    r = r0.clone()
    ops.linear(x, w, bias=bias, out=r, accumulate=True)
    torch.testing.assert_close(r.double(), r0.double() + pre_ref, rtol=1e-5, atol=1e-4)


def test_gemm_f32_dgelu(cuda):
    from paper_2602_08387_b200 import ops

    M, N, K = 256, 192, 160  # dy [M, N], W [N, K] -> dx [M, K] scaled by GELU'(aux [M, K])
    g = torch.Generator(device="cuda").manual_seed(4)
    dy = torch.randn(M, N, device=cuda, generator=g)
    w = torch.randn(N, K, device=cuda, generator=g)
    aux = torch.randn(M, K, device=cuda, generator=g)
    d = ops.linear_dgrad(dy, w, act=2, aux=aux)
    pre = aux.double().requires_grad_()
    torch.nn.functional.gelu(pre, approximate="tanh").backward(torch.ones_like(pre))
    ref = (dy.double() @ w.double()) * pre.grad
    torch.testing.assert_close(d.double(), ref, rtol=1e-5, atol=1e-4)


def _attn_ref(qkv, B, T, Hq, Hkv, dh):
    x = qkv.view(B, T, Hq + 2 * Hkv, dh)
    q = x[:, :, :Hq].transpose(1, 2)
    k = x[:, :, Hq:Hq + Hkv].transpose(1, 2).repeat_interleave(Hq // Hkv, 1)
    v = x[:, :, Hq + Hkv:].transpose(1, 2).repeat_interleave(Hq // Hkv, 1)
    s = q @ k.transpose(-1, -2) / math.sqrt(dh)
    mask = torch.ones(T, T, device=qkv.device, dtype=torch.bool).tril()
    s = s.masked_fill(~mask, float("-inf"))
    return (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(B * T, Hq * dh), torch.logsumexp(s, -1)


@pytest.mark.parametrize("dh", [32, 64, 128])
@pytest.mark.parametrize("B,T,Hq,Hkv", [(1, 1, 1, 1), (2, 100, 4, 2), (1, 256, 3, 3), (2, 130, 8, 2)])
def test_attn_f32(cuda, dh, B, T, Hq, Hkv):
    from paper_2602_08387_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(B * T + Hq + dh)
    qkv = torch.randn(B * T, (Hq + 2 * Hkv) * dh, device=cuda, generator=g)
    o, lse = ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
    x = qkv.double().requires_grad_()
    ro, rl = _attn_ref(x, B, T, Hq, Hkv, dh)
    torch.testing.assert_close(o.double(), ro, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(lse.double(), rl, rtol=1e-5, atol=1e-5)
    do = torch.randn(B * T, Hq * dh, device=cuda, generator=g)
    dqkv = ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh)
    ro.backward(do.double())
    torch.testing.assert_close(dqkv.double(), x.grad, rtol=1e-5, atol=1e-5)


# ---------------------------------------------------------------------------- whole step


def _trainer(tmp_path, preset, B=8, T=256, steps=20):
    from paper_2602_08387_b200.data import PackedDataLoader, Sampler, make_synthetic_packed
    from paper_2602_08387_b200.model import PRESETS, DecoderLM
    from paper_2602_08387_b200.optim import AdamWConfig
    from paper_2602_08387_b200.packed import open_packed
    from paper_2602_08387_b200.trainer import SPMDTrainer

    cfg = PRESETS[preset]
    path = str(tmp_path / "data.cfpk")
    make_synthetic_packed(path, 1 << 19, cfg.vocab_size, kind="markov", seed=1)
    dl = PackedDataLoader(open_packed(path), B, T, Sampler(shuffle=True, seed=5))
    tr = SPMDTrainer(DecoderLM(cfg, precision="fp32"), AdamWConfig(lr=1e-3, warmup_steps=5), dl, steps=steps)
    return cfg, tr, path


def _oracle_batch(path, ids, T):
    buf = open(path, "rb").read()
    width, count, _, _ = orc.parse_header(buf, len(buf))
    payload = np.frombuffer(buf, {1: "<u1", 2: "<u2", 4: "<u4"}[width], count, 40)
    x, y = orc.batch_windows(payload, ids, T)
    return torch.from_numpy(x), torch.from_numpy(y)


@pytest.mark.parametrize("preset", ["tiny-gpt2", "tiny-llama"])
def test_fp32_first_step_grads(cuda, tmp_path, preset):
    from paper_2602_08387_b200.model import init_params

    cfg, tr, path = _trainer(tmp_path, preset)
    tr.setup()
    x, y = tr.dataloader.batch(0)
    tr.engine.begin_step()
    loss = float(tr.model.forward_backward(x, y, hooks=tr.engine).item())
    gpu = tr.params.grads_full_fp32()
    ox, oy = _oracle_batch(path, tr.dataloader.sample_ids(0), 256)
    ot = OracleTrainer(cfg, init_params(cfg, 0))
    oloss = ot.model(ox, oy)
    oloss.backward()
    assert abs(loss - oloss.item()) / oloss.item() < TOL, (loss, oloss.item())
    worst = 0.0
    for k, g in ot.grads().items():
        gg = gpu[k][: g.shape[0]] if g.dim() else gpu[k]
        rel = float((gg.double() - g.double()).norm() / (g.double().norm() + 1e-30))
        worst = max(worst, rel)
        assert rel < TOL, (k, rel)
    print(f"{preset}: loss rel {abs(loss - oloss.item()) / oloss.item():.2e}, worst grad rel {worst:.2e}")


@pytest.mark.parametrize("preset", ["tiny-gpt2", "tiny-llama"])
def test_fp32_loss_curve_20_steps(cuda, tmp_path, preset):
    """configs[0]: 20 steps, batch 8, seq 256 -- every step's loss within 1e-4 of the oracle."""
    from paper_2602_08387_b200.model import init_params

    cfg, tr, path = _trainer(tmp_path, preset, steps=20)
    gpu = tr.run()
    ot = OracleTrainer(cfg, init_params(cfg, 0), lr=1e-3, warmup_steps=5)
    ref = []
    for s in range(20):
        ox, oy = _oracle_batch(path, tr.dataloader.sample_ids(s), 256)
        ref.append(ot.step(ox, oy))
    rel = [abs(a - b) / b for a, b in zip(gpu, ref)]
    assert max(rel) < TOL, list(zip(gpu, ref, rel))
    print(f"{preset}: 20-step max loss rel {max(rel):.2e}, loss {gpu[0]:.4f} -> {gpu[-1]:.4f}")
    assert gpu[-1] < gpu[0] - 0.1


def test_fp32_gpt2_124m_first_step_matches_oracle(cuda, tmp_path):
    """BASELINE configs[1]'s model (GPT-2 124M, vocab 50257) in fp32 mode: the first step's loss
    and every parameter gradient within 1e-4 of the CPU fp32 oracle (1 sequence of 1024 tokens)."""
    from paper_2602_08387_b200.data import PackedDataLoader, Sampler, make_synthetic_packed
    from paper_2602_08387_b200.model import PRESETS, DecoderLM, init_params
    from paper_2602_08387_b200.optim import AdamWConfig
    from paper_2602_08387_b200.packed import open_packed
    from paper_2602_08387_b200.trainer import SPMDTrainer

    cfg = PRESETS["gpt2-124m"]
    path = str(tmp_path / "data.cfpk")
    make_synthetic_packed(path, 1 << 16, cfg.vocab_size, kind="markov", seed=4)
    dl = PackedDataLoader(open_packed(path), 1, 1024, Sampler(shuffle=True, seed=2))
    tr = SPMDTrainer(DecoderLM(cfg, precision="fp32"), AdamWConfig(), dl).setup()
    x, y = tr.dataloader.batch(0)
    tr.engine.begin_step()
    loss = float(tr.model.forward_backward(x, y, hooks=tr.engine).item())
    gpu = tr.params.grads_full_fp32()
    ox, oy = _oracle_batch(path, tr.dataloader.sample_ids(0), 1024)
    ot = OracleTrainer(cfg, init_params(cfg, 0))
    oloss = ot.model(ox, oy)
    oloss.backward()
    assert abs(loss - oloss.item()) / oloss.item() < TOL, (loss, oloss.item())
    worst = 0.0
    for k, g in ot.grads().items():
        gg = gpu[k][: g.shape[0]] if g.dim() else gpu[k]
        rel = float((gg.double() - g.double()).norm() / (g.double().norm() + 1e-30))
        worst = max(worst, rel)
        assert rel < TOL, (k, rel)
    print(f"gpt2-124m fp32: loss rel {abs(loss - oloss.item()) / oloss.item():.2e}, worst grad rel {worst:.2e}")


def test_fp32_llama1b_shape_first_step_matches_oracle(cuda, tmp_path):
    """The Llama-1B block and vocabulary shapes (d 2048, GQA 32/8, FFN 8192, vocab 128256, tied)
    with 2 layers, fp32 mode: first-step loss and gradients within 1e-4 of the CPU oracle."""
    from dataclasses import replace

    from paper_2602_08387_b200.data import PackedDataLoader, Sampler, make_synthetic_packed
    from paper_2602_08387_b200.model import PRESETS, DecoderLM, init_params
    from paper_2602_08387_b200.optim import AdamWConfig
    from paper_2602_08387_b200.packed import open_packed
    from paper_2602_08387_b200.trainer import SPMDTrainer

    cfg = replace(PRESETS["llama-1b"], n_layer=2)
    path = str(tmp_path / "data.cfpk")
    make_synthetic_packed(path, 1 << 16, cfg.vocab_size, kind="markov", seed=6)
    dl = PackedDataLoader(open_packed(path), 1, 512, Sampler(shuffle=True, seed=3))
    tr = SPMDTrainer(DecoderLM(cfg, precision="fp32"), AdamWConfig(), dl).setup()
    x, y = tr.dataloader.batch(0)
    tr.engine.begin_step()
    loss = float(tr.model.forward_backward(x, y, hooks=tr.engine).item())
    gpu = tr.params.grads_full_fp32()
    ox, oy = _oracle_batch(path, tr.dataloader.sample_ids(0), 512)
    ot = OracleTrainer(cfg, init_params(cfg, 0))
    oloss = ot.model(ox, oy)
    oloss.backward()
    assert abs(loss - oloss.item()) / oloss.item() < TOL, (loss, oloss.item())
    worst = 0.0
    for k, g in ot.grads().items():
        gg = gpu[k][: g.shape[0]] if g.dim() else gpu[k]
        rel = float((gg.double() - g.double()).norm() / (g.double().norm() + 1e-30))
        worst = max(worst, rel)
        assert rel < TOL, (k, rel)
    print(f"llama-1b shape fp32: loss rel {abs(loss - oloss.item()) / oloss.item():.2e}, worst grad rel {worst:.2e}")
