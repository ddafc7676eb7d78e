"""Pin the CPU fp32 model oracle to an independent implementation: Hugging Face
transformers GPT2LMHeadModel / LlamaForCausalLM with the same weights (CPU, fp32)."""

import pytest
import torch
import torch.nn.functional as F

from oracle.model_oracle import OracleModel
from paper_2602_08387_b200.model import PRESETS, init_params

transformers = pytest.importorskip("transformers")


def _batch(cfg, B=2, T=64, seed=0):
    g = torch.Generator().manual_seed(seed)
    x = torch.randint(0, cfg.vocab_size, (B, T + 1), generator=g)
    return x[:, :T], x[:, 1:]


def _hf_gpt2(cfg, p):
    from transformers import GPT2Config, GPT2LMHeadModel

    hc = GPT2Config(vocab_size=cfg.vocab_size, n_positions=cfg.max_seq_len, n_embd=cfg.d_model, n_layer=cfg.n_layer,
                    n_head=cfg.n_head, n_inner=cfg.d_ff, activation_function="gelu_new",
                    layer_norm_epsilon=cfg.norm_eps, resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0)
    m = GPT2LMHeadModel(hc).eval()
    sd = {"transformer.wte.weight": p["embed.wte"][: cfg.vocab_size], "transformer.wpe.weight": p["embed.wpe"],
          "transformer.ln_f.weight": p["head.lnf_g"], "transformer.ln_f.bias": p["head.lnf_b"]}
    for i in range(cfg.n_layer):
        b, u = f"transformer.h.{i}.", f"block{i}."
        sd.update({b + "ln_1.weight": p[u + "ln1_g"], b + "ln_1.bias": p[u + "ln1_b"],
                   b + "attn.c_attn.weight": p[u + "qkv_w"].t(), b + "attn.c_attn.bias": p[u + "qkv_b"],
                   b + "attn.c_proj.weight": p[u + "proj_w"].t(), b + "attn.c_proj.bias": p[u + "proj_b"],
                   b + "ln_2.weight": p[u + "ln2_g"], b + "ln_2.bias": p[u + "ln2_b"],
                   b + "mlp.c_fc.weight": p[u + "fc_w"].t(), b + "mlp.c_fc.bias": p[u + "fc_b"],
                   b + "mlp.c_proj.weight": p[u + "fc2_w"].t(), b + "mlp.c_proj.bias": p[u + "fc2_b"]})
    sd["lm_head.weight"] = sd["transformer.wte.weight"]
    missing, unexpected = m.load_state_dict({k: v.contiguous() for k, v in sd.items()}, strict=False)
    assert not [k for k in missing if "attn.bias" not in k and "masked_bias" not in k], missing
    return m


def _hf_llama(cfg, p):
    from transformers import LlamaConfig, LlamaForCausalLM

    H, Hkv, dh, Fd = cfg.n_head, cfg.n_kv_head, cfg.head_dim, cfg.d_ff
    hc = LlamaConfig(vocab_size=cfg.vocab_size, hidden_size=cfg.d_model, intermediate_size=Fd,
                     num_hidden_layers=cfg.n_layer, num_attention_heads=H, num_key_value_heads=Hkv,
                     max_position_embeddings=cfg.max_seq_len, rms_norm_eps=cfg.norm_eps, rope_theta=cfg.rope_theta,
                     tie_word_embeddings=cfg.tie_embeddings, attention_bias=False, mlp_bias=False, head_dim=dh)
    m = LlamaForCausalLM(hc).eval()
    sd = {"model.embed_tokens.weight": p["embed.wte"][: cfg.vocab_size], "model.norm.weight": p["head.lnf_g"]}
    for i in range(cfg.n_layer):
        b, u = f"model.layers.{i}.", f"block{i}."
        w = p[u + "wqkv"]
        sd.update({b + "self_attn.q_proj.weight": w[: H * dh], b + "self_attn.k_proj.weight": w[H * dh:(H + Hkv) * dh],
                   b + "self_attn.v_proj.weight": w[(H + Hkv) * dh:], b + "self_attn.o_proj.weight": p[u + "wo"],
                   b + "mlp.gate_proj.weight": p[u + "w13"][:Fd], b + "mlp.up_proj.weight": p[u + "w13"][Fd:],
                   b + "mlp.down_proj.weight": p[u + "w2"], b + "input_layernorm.weight": p[u + "attn_norm"],
                   b + "post_attention_layernorm.weight": p[u + "mlp_norm"]})
    sd["lm_head.weight"] = sd["model.embed_tokens.weight"]
    missing, unexpected = m.load_state_dict({k: v.contiguous() for k, v in sd.items()}, strict=False)
    assert not [k for k in missing if "rotary" not in k], missing
    return m


@pytest.mark.parametrize("preset", ["tiny-gpt2", "tiny-gpt2-dh64", "tiny-llama"])
def test_oracle_matches_hf(preset):
    torch.manual_seed(0)
    cfg = PRESETS[preset]
    p = init_params(cfg, 0)
    # randomise norms/biases too so they are exercised
    g = torch.Generator().manual_seed(1)
    for k, v in p.items():
        if v.dim() == 1:
            p[k] = v + 0.1 * torch.randn(v.shape, generator=g)
    x, y = _batch(cfg)
    orc = OracleModel(cfg, p)
    loss = orc(x, y)
    hf = _hf_gpt2(cfg, p) if cfg.arch == "gpt2" else _hf_llama(cfg, p)
    logits = hf(input_ids=x).logits
    ref = F.cross_entropy(logits.reshape(-1, cfg.vocab_size), y.reshape(-1))
    assert abs(loss.item() - ref.item()) < 1e-5 * ref.item(), (loss.item(), ref.item())
    # gradients of a block matrix agree too
    loss.backward()
    ref.backward()
    if cfg.arch == "gpt2":
        a, b = orc.P("block1.fc_w").grad, hf.transformer.h[1].mlp.c_fc.weight.grad.t()
    else:
        a, b = orc.P("block1.w2").grad, hf.model.layers[1].mlp.down_proj.weight.grad
    torch.testing.assert_close(a, b, rtol=1e-4, atol=1e-7)
