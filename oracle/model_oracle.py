"""ORACLE — test infrastructure only (tests/, smoke(), bench.py's reference/cpu_baseline leg).

CPU fp32 restatement of the training step the product runs on the GPU:
GPT-2 / Llama-style decoder forward, autograd backward, global-norm clipping
and AdamW, in plain PyTorch eager (torch.nn.functional, torch.optim.AdamW).

Why this is the oracle: the reference (arxiv/paper_2602_08387 as mounted)
contains no model, optimizer or training loop -- SPEC.md:12 puts "actual
distributed training execution (FSDP/TP/PP kernels, the gym loop,
checkpointing)" out of its scope -- so the arithmetic lives in the
third-party dependency the paper's framework builds on: PyTorch (container
pin 2.11.0+cu128). This module restates that published algorithm; its
forward is cross-checked against Hugging Face transformers 5.5.0
GPT2LMHeadModel / LlamaForCausalLM on identical weights (tests/test_oracle.py).
Parity of the model arithmetic with the *reference* is therefore "parity
unpinned" (no reference test or golden vector exists for it); the packed
data path (oracle/packed_oracle.py) is pinned to reference goldens.

Parameters use the product's flat naming 'unit.param' (model.unit_specs).
The module is device-agnostic: the headline-shape tests move it to the GPU and
run it in true fp32 (TF32 off) as the fp32 reference of the bf16 step, where the
CPU would take minutes per step.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


class OracleModel(torch.nn.Module):
    def __init__(self, cfg, tensors: dict):
        super().__init__()
        self.cfg = cfg
        self.params = torch.nn.ParameterDict(
            {k.replace(".", "__"): torch.nn.Parameter(v.detach().clone().float()) for k, v in tensors.items()})

    def P(self, key):
        return self.params[key.replace(".", "__")]

    def forward(self, tok, tgt):
        c = self.cfg
        B, T = tok.shape
        V, d, H, Hkv = c.vocab_size, c.d_model, c.n_head, c.n_kv_head
        dh = d // H
        gpt2 = c.arch == "gpt2"
        wte = self.P("embed.wte")[:V]
        x = wte[tok]
        if gpt2:
            x = x + self.P("embed.wpe")[:T][None]
        else:
            inv = 1.0 / (c.rope_theta ** (torch.arange(0, dh, 2, dtype=torch.float64) / dh))
            ang = torch.arange(T, dtype=torch.float64)[:, None] * inv[None]
            cos, sin = ang.cos().float().to(tok.device), ang.sin().float().to(tok.device)

        def rope(t):  # t [B, h, T, dh], rotate-half pairing
            t1, t2 = t[..., : dh // 2], t[..., dh // 2:]
            return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], -1)

        def rms(t, g):
            return t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + c.norm_eps) * g

        mask = torch.ones(T, T, dtype=torch.bool, device=tok.device).tril()
        for i in range(c.n_layer):
            u = f"block{i}."
            if gpt2:
                a = F.layer_norm(x, (d,), self.P(u + "ln1_g"), self.P(u + "ln1_b"), c.norm_eps)
                qkv = a @ self.P(u + "qkv_w").t() + self.P(u + "qkv_b")
            else:
                a = rms(x, self.P(u + "attn_norm"))
                qkv = a @ self.P(u + "wqkv").t()
            qkv = qkv.view(B, T, H + 2 * Hkv, dh)
            q = qkv[:, :, :H].transpose(1, 2)
            k = qkv[:, :, H:H + Hkv].transpose(1, 2)
            v = qkv[:, :, H + Hkv:].transpose(1, 2)
            if not gpt2:
                q, k = rope(q), rope(k)
            k = k.repeat_interleave(H // Hkv, 1)
            v = v.repeat_interleave(H // Hkv, 1)
            s = (q @ k.transpose(-1, -2)) / math.sqrt(dh)
            s = s.masked_fill(~mask, float("-inf"))
            o = (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(B, T, H * dh)
            if gpt2:
                x = x + o @ self.P(u + "proj_w").t() + self.P(u + "proj_b")
                a = F.layer_norm(x, (d,), self.P(u + "ln2_g"), self.P(u + "ln2_b"), c.norm_eps)
                h = F.gelu(a @ self.P(u + "fc_w").t() + self.P(u + "fc_b"), approximate="tanh")
                x = x + h @ self.P(u + "fc2_w").t() + self.P(u + "fc2_b")
            else:
                x = x + o @ self.P(u + "wo").t()
                a = rms(x, self.P(u + "mlp_norm"))
                gu = a @ self.P(u + "w13").t()
                g_, up = gu[..., : c.d_ff], gu[..., c.d_ff:]
                x = x + (F.silu(g_) * up) @ self.P(u + "w2").t()
        if gpt2:
            x = F.layer_norm(x, (d,), self.P("head.lnf_g"), self.P("head.lnf_b"), c.norm_eps)
        else:
            x = rms(x, self.P("head.lnf_g"))
        w = wte if c.tie_embeddings else self.P("head.lm_head")[:V]
        logits = x @ w.t()
        return F.cross_entropy(logits.view(-1, V), tgt.reshape(-1))


def decay_flags(cfg) -> dict:
    """'unit.param' -> weight decay applies (matrices and embeddings; not norms/biases)."""
    from paper_2602_08387_b200.model import unit_specs  # spec table only (names/shapes), no compute

    return {f"{u.name}.{p.name}": p.decay for u in unit_specs(cfg) for p in u.params}


class OracleTrainer:
    """fp32 CPU training loop with the product's optimizer semantics."""

    def __init__(self, cfg, tensors: dict, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1,
                 grad_clip=1.0, warmup_steps=10):
        self.model = OracleModel(cfg, tensors)
        flags = decay_flags(cfg)
        dec, nodec = [], []
        for k, p in self.model.params.items():
            (dec if flags[k.replace("__", ".")] else nodec).append(p)
        self.opt = torch.optim.AdamW([{"params": dec, "weight_decay": weight_decay},
                                      {"params": nodec, "weight_decay": 0.0}], lr=lr, betas=betas, eps=eps)
        self.lr, self.warmup, self.clip = lr, warmup_steps, grad_clip
        self.step_count = 0

    def step(self, tok, tgt) -> float:
        self.step_count += 1
        s = self.step_count
        lr = self.lr * s / self.warmup if self.warmup and s <= self.warmup else self.lr
        for g in self.opt.param_groups:
            g["lr"] = lr
        self.opt.zero_grad(set_to_none=True)
        loss = self.model(tok, tgt)
        loss.backward()
        if self.clip > 0:
            torch.nn.utils.clip_grad_norm_(list(self.model.params.values()), self.clip)
        self.opt.step()
        return float(loss.detach())

    def grads(self) -> dict:
        return {k.replace("__", "."): p.grad.detach().clone() for k, p in self.model.params.items()
                if p.grad is not None}
