"""GPT-2 / Llama-style decoder with an explicit, buffer-planned forward+backward.

The reference fixes the model interface to ``nn.Module`` and has
no model code, so this module is the B200-native decoder the
registered ``model`` component builds. It is an ``nn.Module`` for the
interface, but the training step does not run autograd: ``forward_backward``
is a fixed sequence of C-ABI kernel launches over activation buffers that are
allocated once per (batch, seq) shape, which keeps the step CUDA-graph
capturable and lets the backward write weight gradients straight into the
FSDP flat gradient buffers (see fsdp.py).

Numerics (``precision``):
  "bf16"  bf16 weights/activations into tcgen05 GEMMs and attention with fp32
          accumulation; the residual stream, its gradient, norm statistics,
          the loss and all parameter gradients are fp32 (the training mode).
  "fp32"  every tensor fp32; GEMMs and attention on the true-fp32 SIMT kernels
          (f32.cu), the bandwidth kernels in their fp32 instantiation -- the
          north star's "fp32 mode" (per-step losses and gradients within 1e-4
          relative of the CPU fp32 reference). Same call sequence, same
          buffers, only the element type changes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import torch

from . import ops

ALIGN = 64  # parameter offsets inside a flat unit, in elements (128 B of bf16)
PRECISIONS = {"bf16": torch.bfloat16, "fp32": torch.float32}


@dataclass(frozen=True)
class ModelConfig:
    arch: str  # "gpt2" | "llama"
    n_layer: int
    d_model: int
    n_head: int
    n_kv_head: int
    d_ff: int
    vocab_size: int
    max_seq_len: int
    tie_embeddings: bool = True
    norm_eps: float = 1e-5
    rope_theta: float = 500000.0
    init_std: float = 0.02

    def __post_init__(self):
        if self.arch not in ("gpt2", "llama"):
            raise ValueError(f"arch must be gpt2 or llama, got {self.arch!r}")
        if self.d_model % self.n_head or self.n_head % self.n_kv_head:
            raise ValueError("d_model % n_head and n_head % n_kv_head must be 0")
        if self.arch == "gpt2" and self.n_kv_head != self.n_head:
            raise ValueError("gpt2 uses multi-head attention (n_kv_head == n_head)")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_head

    @property
    def padded_vocab(self) -> int:
        return (self.vocab_size + 127) // 128 * 128

    @property
    def qkv_dim(self) -> int:
        return (self.n_head + 2 * self.n_kv_head) * self.head_dim

    def matmul_params(self) -> int:
        """Parameters that take part in matmuls (incl. the LM head, excl. embeddings/norms)."""
        d, f = self.d_model, self.d_ff
        per = d * self.qkv_dim + d * d + (2 if self.arch == "gpt2" else 3) * d * f
        return self.n_layer * per + d * self.vocab_size

    def flops_per_token(self, seq_len: int) -> float:
        """Training FLOPs per token: 6 * N_matmul + 12 * L * d * T (PaLM/nanoGPT convention)."""
        return 6.0 * self.matmul_params() + 12.0 * self.n_layer * self.d_model * seq_len

    def num_params(self) -> int:
        """Trainable parameters (padded vocabulary rows excluded)."""
        n = sum(int(torch.Size(p.shape).numel()) for u in unit_specs(self) for p in u.params)
        pad_rows = (self.padded_vocab - self.vocab_size) * self.d_model
        return n - pad_rows * (1 if self.tie_embeddings else 2)


PRESETS = {
    # BASELINE.json configs[0]: the CPU-runnable oracle case
    "tiny-gpt2": ModelConfig("gpt2", 2, 128, 4, 4, 512, 4096, 256),
    # GPU parity configs (head dim 64, the attention kernel's tile): tiny GPT-2 / tiny Llama
    "tiny-gpt2-dh64": ModelConfig("gpt2", 2, 256, 4, 4, 1024, 4096, 256),
    "tiny-llama": ModelConfig("llama", 2, 256, 4, 2, 512, 4096, 256),
    "tiny-llama-dh128": ModelConfig("llama", 2, 256, 2, 1, 512, 4096, 256),  # the 8B's head dim / GQA path
    # configs[1]
    "gpt2-124m": ModelConfig("gpt2", 12, 768, 12, 12, 3072, 50257, 2048),
    # configs[2]: Llama-3.2-1B-like (tied head, GQA 32/8, dh 64)
    "llama-1b": ModelConfig("llama", 16, 2048, 32, 8, 8192, 128256, 4096),
    # configs[3]: Llama-3-8B-like (untied head, GQA 32/8, dh 128)
    "llama-8b": ModelConfig("llama", 32, 4096, 32, 8, 14336, 128256, 4096, tie_embeddings=False),
}


@dataclass(frozen=True)
class ParamSpec:
    name: str
    shape: tuple
    init: str  # normal | resid | zeros | ones
    decay: bool


@dataclass
class UnitSpec:
    name: str
    params: list
    offsets: dict = field(default_factory=dict)
    numel: int = 0

    def layout(self):
        off = 0
        for p in self.params:
            self.offsets[p.name] = off
            n = int(torch.Size(p.shape).numel())
            off += (n + ALIGN - 1) // ALIGN * ALIGN
        self.numel = off
        return self


def unit_specs(cfg: ModelConfig) -> list:
    """FSDP units in execution order: embedding, one per block, final norm (+ head)."""
    d, f, Vp = cfg.d_model, cfg.d_ff, cfg.padded_vocab
    units = []
    emb = [ParamSpec("wte", (Vp, d), "normal", True)]
    if cfg.arch == "gpt2":
        emb.append(ParamSpec("wpe", (cfg.max_seq_len, d), "normal", True))
    units.append(UnitSpec("embed", emb))
    for i in range(cfg.n_layer):
        if cfg.arch == "gpt2":
            ps = [ParamSpec("ln1_g", (d,), "ones", False), ParamSpec("ln1_b", (d,), "zeros", False),
                  ParamSpec("qkv_w", (cfg.qkv_dim, d), "normal", True), ParamSpec("qkv_b", (cfg.qkv_dim,), "zeros", False),
                  ParamSpec("proj_w", (d, d), "resid", True), ParamSpec("proj_b", (d,), "zeros", False),
                  ParamSpec("ln2_g", (d,), "ones", False), ParamSpec("ln2_b", (d,), "zeros", False),
                  ParamSpec("fc_w", (f, d), "normal", True), ParamSpec("fc_b", (f,), "zeros", False),
                  ParamSpec("fc2_w", (d, f), "resid", True), ParamSpec("fc2_b", (d,), "zeros", False)]
        else:
            ps = [ParamSpec("attn_norm", (d,), "ones", False),
                  ParamSpec("wqkv", (cfg.qkv_dim, d), "normal", True),
                  ParamSpec("wo", (d, cfg.n_head * cfg.head_dim), "resid", True),
                  ParamSpec("mlp_norm", (d,), "ones", False),
                  ParamSpec("w13", (2 * f, d), "normal", True),
                  ParamSpec("w2", (d, f), "resid", True)]
        units.append(UnitSpec(f"block{i}", ps))
    head = [ParamSpec("lnf_g", (d,), "ones", False)]
    if cfg.arch == "gpt2":
        head.append(ParamSpec("lnf_b", (d,), "zeros", False))
    if not cfg.tie_embeddings:
        head.append(ParamSpec("lm_head", (Vp, d), "normal", True))
    units.append(UnitSpec("head", head))
    return [u.layout() for u in units]


def init_params(cfg: ModelConfig, seed: int = 0) -> dict:
    """fp32 CPU initial weights, generated in unit/param order from one seeded generator.

    N(0, std) for matrices, N(0, std/sqrt(2L)) for residual output projections,
    ones/zeros for norms and biases; padded vocabulary rows are zero.
    """
    g = torch.Generator().manual_seed(seed)
    out = {}
    resid_std = cfg.init_std / math.sqrt(2 * cfg.n_layer)
    for u in unit_specs(cfg):
        for p in u.params:
            key = f"{u.name}.{p.name}"
            if p.init == "ones":
                t = torch.ones(p.shape)
            elif p.init == "zeros":
                t = torch.zeros(p.shape)
            else:
                t = torch.empty(p.shape).normal_(0.0, resid_std if p.init == "resid" else cfg.init_std, generator=g)
            if p.name in ("wte", "lm_head") and cfg.padded_vocab > cfg.vocab_size:
                t[cfg.vocab_size:] = 0
            out[key] = t
    return out


def param_initializer(cfg: ModelConfig, seed: int = 0, device="cpu"):
    """Returns get(key) -> fp32 initial tensor for 'unit.param'.

    device='cpu' replays init_params (one sequential CPU generator: the oracle
    reproduces it exactly). Any other device generates each tensor on that
    device from its own generator seeded by (seed, crc32(key)) -- identical on
    every rank, no host-memory copy of the whole model (used for 1B/8B).
    """
    if str(device) == "cpu":
        tensors = init_params(cfg, seed)
        return tensors.__getitem__
    import zlib

    specs = {f"{u.name}.{p.name}": p for u in unit_specs(cfg) for p in u.params}
    resid_std = cfg.init_std / math.sqrt(2 * cfg.n_layer)

    def get(key):
        p = specs[key]
        if p.init == "ones":
            return torch.ones(p.shape, device=device)
        if p.init == "zeros":
            return torch.zeros(p.shape, device=device)
        g = torch.Generator(device=device).manual_seed((seed * 1_000_003 + zlib.crc32(key.encode())) & 0x7FFFFFFF)
        t = torch.empty(p.shape, device=device).normal_(0.0, resid_std if p.init == "resid" else cfg.init_std,
                                                        generator=g)
        if p.name in ("wte", "lm_head") and cfg.padded_vocab > cfg.vocab_size:
            t[cfg.vocab_size:] = 0
        return t

    return get


def rope_tables(cfg: ModelConfig, T: int, device):
    dh = cfg.head_dim
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, dh, 2, dtype=torch.float64) / dh))
    ang = torch.arange(T, dtype=torch.float64)[:, None] * inv[None]
    return ang.cos().float().contiguous().to(device), ang.sin().float().contiguous().to(device)


class _Slot:
    """The forward buffers of one transformer block (see _Acts)."""

    __slots__ = ("xa", "xb", "xn", "ln_a", "mean_a", "rstd_a", "ln_b", "mean_b", "rstd_b", "qkv", "o", "lse",
                 "ya", "yb", "hpre", "gu", "h")


class _Acts:
    """Activation buffers for one (B, T): saved forward tensors + backward scratch.

    Residual stream (fp32): the attention output projection writes its result y1
    (bf16, bias included) and the next norm kernel forms xb = xa + y1 while it
    normalises; likewise the MLP output y2 is added into xn (= the next block's
    xa) by the next block's first norm (or the final norm). The fp32 residual
    is therefore written once per sublayer by a norm kernel instead of being
    read-modify-written by a TMA add-reduce in the GEMM epilogue.

    Without checkpointing every block owns its slot (all saved). With
    ``checkpoint`` only the block inputs xa (L + 1 fp32 [M, d] buffers) are
    kept; every other per-block buffer is one shared slot that the backward
    refills by recomputing the block's forward.
    """

    def __init__(self, cfg: ModelConfig, B: int, T: int, device, act_dtype=torch.bfloat16, checkpoint=False):
        M, d, f, L = B * T, cfg.d_model, cfg.d_ff, cfg.n_layer
        bf, f32 = act_dtype, torch.float32
        e = lambda *s, dt=bf: torch.empty(*s, device=device, dtype=dt)  # noqa: E731
        self.B, self.T, self.M = B, T, M
        self.checkpoint = checkpoint
        self.xin = [e(M, d, dt=f32) for _ in range(L + 1)]  # block inputs; xin[L] enters the head
        self.ya, self.yb = e(M, d), e(M, d)  # attention / MLP sublayer outputs (bias added)

        def slot(i, xb=None):
            sl = _Slot()
            sl.xa, sl.xn = self.xin[i], self.xin[i + 1]
            sl.xb = e(M, d, dt=f32) if xb is None else xb
            sl.ln_a, sl.ln_b = e(M, d), e(M, d)
            sl.mean_a, sl.rstd_a, sl.mean_b, sl.rstd_b = (e(M, dt=f32) for _ in range(4))
            sl.qkv = e(M, cfg.qkv_dim)
            sl.o = e(M, cfg.n_head * cfg.head_dim)
            sl.lse = e(B, cfg.n_head, T, dt=f32)
            sl.ya, sl.yb = self.ya, self.yb  # sublayer outputs: consumed by the next norm, shared
            sl.hpre = e(M, f) if cfg.arch == "gpt2" else None
            sl.gu = e(M, 2 * f) if cfg.arch == "llama" else None
            sl.h = e(M, f)
            return sl

        if checkpoint:
            shared = slot(0)
            self.slots = []
            for i in range(L):
                sl = _Slot()
                for k in _Slot.__slots__:
                    setattr(sl, k, getattr(shared, k))
                sl.xa, sl.xn = self.xin[i], self.xin[i + 1]
                self.slots.append(sl)
        else:
            self.slots = [slot(i) for i in range(L)]
        self.ln_f = e(M, d)
        self.mean_f, self.rstd_f = e(M, dt=f32), e(M, dt=f32)
        self.logits = e(M, cfg.padded_vocab)
        self.loss_rows = e(M, dt=f32)
        self.loss = e(1, dt=f32)
        # backward scratch (reused across layers)
        self.dx = e(M, d, dt=f32)
        # low-precision copy of dx for the GEMMs; in fp32 mode dx itself
        self.dxb = self.dx if bf == f32 else e(M, d)
        self.dln = e(M, d)
        self.do = e(M, cfg.n_head * cfg.head_dim)
        self.dqkv = e(M, cfg.qkv_dim)
        self.dh = e(M, f)
        if cfg.arch == "llama":
            self.dgu = e(M, 2 * f)
        self.attn_work = e(ops._lib.load().b2s_attn_bwd_work_floats(B, T, cfg.n_head, cfg.head_dim), dt=f32)


class DecoderLM(torch.nn.Module):
    """Decoder-only LM whose parameters live in FSDP flat units (see fsdp.FlatParams)."""

    def __init__(self, cfg: ModelConfig, precision: str = "bf16", activation_checkpointing: bool = False):
        super().__init__()
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}, got {precision!r}")
        if precision == "bf16" and cfg.head_dim not in (64, 128):
            raise ValueError(f"bf16 attention kernels implement head dims 64 and 128 (got {cfg.head_dim}); "
                             "use precision='fp32' for other head dims")
        self.cfg = cfg
        self.precision = precision
        # GELU epilogues: bf16 stores gelu'(z) as the aux (act 5 / 6); fp32 keeps z (act 1 / 2)
        gd = precision != "fp32"
        self._act_fwd, self._act_bwd = (5, 6) if gd else (1, 2)
        self.dtype = PRECISIONS[precision]
        self.activation_checkpointing = bool(activation_checkpointing)
        self.units = unit_specs(cfg)
        self._acts = {}
        self._rope = {}
        self.params = None  # fsdp.FlatParams, attached by the trainer

    def attach(self, flat_params) -> None:
        self.params = flat_params

    def overwritten_grads(self) -> set:
        """Parameter names whose gradient one weight-gradient GEMM writes whole each step
        (``ops.OVERWRITE``), so the step need not zero them first (fsdp.FlatParams.grad_zero_ranges).
        The tied GPT-2 wte is written by the head's wgrad before the embedding backward adds to it."""
        names = {"qkv_w", "proj_w", "fc_w", "fc2_w"} if self.cfg.arch == "gpt2" else {"wqkv", "wo", "w13", "w2"}
        names.add("wte" if self.cfg.tie_embeddings else "lm_head")
        return names

    def acts(self, B, T, device) -> _Acts:
        key = (B, T)
        if key not in self._acts:
            self._acts.clear()
            self._acts[key] = _Acts(self.cfg, B, T, device, self.dtype, self.activation_checkpointing)
        return self._acts[key]

    def rope(self, T, device):
        if T not in self._rope:
            self._rope[T] = rope_tables(self.cfg, T, device)
        return self._rope[T]

    # ------------------------------------------------------------------ step
    def _block_forward(self, i, S, T, rope, pending=None, with_output=True):
        """Block i's forward over slot S. ``pending`` = (x, y) of the previous sublayer: the
        first norm forms S.xa = x + y while normalising (None: S.xa is already the input).
        Leaves (S.xb, S.yb) pending for the next norm; with_output=False (the checkpoint
        recompute) skips the MLP output GEMM, whose result the backward does not need."""
        cfg, U = self.cfg, self.params.unit(i + 1)
        M, d = S.xa.shape
        B = M // T
        H, Hkv, dh, eps = cfg.n_head, cfg.n_kv_head, cfg.head_dim, cfg.norm_eps
        gpt2 = cfg.arch == "gpt2"
        if gpt2:
            if pending is None:
                ops.layernorm_fwd(S.xa, U.p("ln1_g"), U.p("ln1_b"), eps, S.ln_a, S.mean_a, S.rstd_a)
            else:
                ops.layernorm_fwd_res(pending[0], pending[1], U.p("ln1_g"), U.p("ln1_b"), eps, S.ln_a, S.mean_a,
                                      S.rstd_a, S.xa)
            ops.linear(S.ln_a, U.p("qkv_w"), bias=U.p("qkv_b"), out=S.qkv)
        else:
            if pending is None:
                ops.rmsnorm_fwd(S.xa, U.p("attn_norm"), eps, S.ln_a, S.rstd_a)
            else:
                ops.rmsnorm_fwd_res(pending[0], pending[1], U.p("attn_norm"), eps, S.ln_a, S.rstd_a, S.xa)
            if self.dtype == torch.bfloat16:  # RoPE on q / k in the projection's epilogue
                ops.linear_rope(S.ln_a, U.p("wqkv"), S.qkv, T, dh, (H + Hkv) * dh, *rope)
            else:
                ops.linear(S.ln_a, U.p("wqkv"), out=S.qkv)
                ops.rope(S.qkv, T, H + Hkv, dh, *rope)
        ops.attn_fwd(S.qkv, B, T, H, Hkv, dh, o=S.o, lse=S.lse)
        # y1 = o @ Wo^T (+ bias); the next norm adds it into the residual: xb = xa + y1
        ops.gemm(S.o, U.p("proj_w" if gpt2 else "wo"), a_mn=False, b_mn=False, M=M, N=d, K=H * dh, out=S.ya,
                 bias=U.p("proj_b") if gpt2 else None)
        if gpt2:
            ops.layernorm_fwd_res(S.xa, S.ya, U.p("ln2_g"), U.p("ln2_b"), eps, S.ln_b, S.mean_b, S.rstd_b, S.xb)
            # bf16: the epilogue stores gelu'(z) in hpre (act 5) so the backward multiplies by it
            # (act 6); fp32 mode keeps z itself (act 1 / 2 on the SIMT kernel)
            ops.linear(S.ln_b, U.p("fc_w"), bias=U.p("fc_b"), out=S.h, act=self._act_fwd, aux=S.hpre)
            if with_output:
                ops.gemm(S.h, U.p("fc2_w"), a_mn=False, b_mn=False, M=M, N=d, K=cfg.d_ff, out=S.yb,
                         bias=U.p("fc2_b"))
        else:
            ops.rmsnorm_fwd_res(S.xa, S.ya, U.p("mlp_norm"), eps, S.ln_b, S.rstd_b, S.xb)
            if self.dtype == torch.bfloat16:  # gate|up GEMM with the SwiGLU in its epilogue
                ops.linear_swiglu(S.ln_b, U.p("w13"), S.gu, S.h)
            else:
                ops.linear(S.ln_b, U.p("w13"), out=S.gu)
                ops.swiglu_fwd(S.gu, S.h)
            if with_output:
                ops.gemm(S.h, U.p("w2"), a_mn=False, b_mn=False, M=M, N=d, K=cfg.d_ff, out=S.yb)
        return (S.xb, S.yb)

    def forward_backward(self, tokens, targets, hooks=None, compute_grad: bool = True):
        """One training forward + backward over int64 tokens/targets [B, T].

        Writes fp32 parameter gradients into the flat grad buffers -- the weight matrices'
        (overwritten_grads()) whole, the rest accumulated into buffers the caller zeroed -- and
        returns the device scalar mean loss.
        ``hooks`` (fsdp.Engine) is told when each unit's parameters are needed
        and when each unit's gradients are complete. With activation
        checkpointing each block's forward is re-run (into the shared slot)
        right before its backward.
        """
        cfg, P = self.cfg, self.params
        B, T = tokens.shape
        dev = tokens.device
        A = self.acts(B, T, dev)
        M, d, L = A.M, cfg.d_model, cfg.n_layer
        H, Hkv, dh = cfg.n_head, cfg.n_kv_head, cfg.head_dim
        gpt2 = cfg.arch == "gpt2"
        tok = tokens.reshape(-1)
        tgt = targets.reshape(-1)
        hk = hooks
        pre = (lambda u: hk.before_forward(u)) if hk else (lambda u: None)
        post = (lambda u: hk.after_backward(u)) if hk else (lambda u: None)
        eps = cfg.norm_eps
        rope = None if gpt2 else self.rope(T, dev)

        # ---------------- forward
        pre(0)
        E = P.unit(0)
        ops.embedding_fwd(tok, E.p("wte"), E.p("wpe") if gpt2 else None, T, out=A.xin[0])
        pending = None
        for i in range(L):
            pre(i + 1)
            pending = self._block_forward(i, A.slots[i], T, rope, pending)
        pre(L + 1)
        Hd = P.unit(L + 1)
        xf = A.xin[L]  # = the last block's xb + its MLP output, formed by the final norm
        if gpt2:
            ops.layernorm_fwd_res(pending[0], pending[1], Hd.p("lnf_g"), Hd.p("lnf_b"), eps, A.ln_f, A.mean_f,
                                  A.rstd_f, xf)
        else:
            ops.rmsnorm_fwd_res(pending[0], pending[1], Hd.p("lnf_g"), eps, A.ln_f, A.rstd_f, xf)
        w_head = E.p("wte") if cfg.tie_embeddings else Hd.p("lm_head")
        ops.linear(A.ln_f, w_head, out=A.logits)
        ops.cross_entropy(A.logits, cfg.vocab_size, tgt, A.loss_rows, grad_scale=1.0 / M, write_grad=compute_grad)
        ops.sum_(A.loss_rows, A.loss, scale=1.0 / M)
        if not compute_grad:
            return A.loss

        # ---------------- backward
        # head: dlogits (in A.logits) -> d ln_f, dW_head
        g_head = E.g("wte") if cfg.tie_embeddings else Hd.g("lm_head")
        ops.linear_wgrad(A.logits, A.ln_f, out=g_head, accumulate=ops.OVERWRITE)  # first writer (tied wte too)
        ops.linear_dgrad(A.logits, w_head, out=A.dln)
        ops.zero_(A.dx)
        if gpt2:
            # the updated dx is the output gradient of the last block's fc2 -> its bias grad
            ops.layernorm_bwd(xf, A.dln, Hd.p("lnf_g"), A.mean_f, A.rstd_f, A.dx, A.dxb,
                              Hd.g("lnf_g"), Hd.g("lnf_b"), dxsum=P.unit(L).g("fc2_b"))
        else:
            ops.rmsnorm_bwd(xf, A.dln, Hd.p("lnf_g"), A.rstd_f, A.dx, A.dxb, Hd.g("lnf_g"))
        post(L + 1)
        for i in reversed(range(L)):
            U = P.unit(i + 1)
            S = A.slots[i]
            if A.checkpoint:
                self._block_forward(i, S, T, rope, with_output=False)
            # --- MLP (its output gradient is the residual gradient dx, bf16 copy in dxb)
            if gpt2:  # fc2_b's grad was summed by the norm backward that produced dx
                ops.linear_wgrad(A.dxb, S.h, out=U.g("fc2_w"), accumulate=ops.OVERWRITE)
                # fc_b's gradient = colsum(dh), from the dgrad epilogue's per-32-row partials
                ops.linear_dgrad(A.dxb, U.p("fc2_w"), out=A.dh, act=self._act_bwd, aux=S.hpre, colsum_out=U.g("fc_b"))
                ops.linear_wgrad(A.dh, S.ln_b, out=U.g("fc_w"), accumulate=ops.OVERWRITE)
                ops.linear_dgrad(A.dh, U.p("fc_w"), out=A.dln)
                ops.layernorm_bwd(S.xb, A.dln, U.p("ln2_g"), S.mean_b, S.rstd_b, A.dx, A.dxb,
                                  U.g("ln2_g"), U.g("ln2_b"), dxsum=U.g("proj_b"))
            else:
                ops.linear_wgrad(A.dxb, S.h, out=U.g("w2"), accumulate=ops.OVERWRITE)
                if self.dtype == torch.bfloat16 and cfg.d_ff % 128 == 0:
                    # dh = dy W2 with the SwiGLU backward in the epilogue (gate / up tiles by TMA):
                    # dh never reaches HBM (0.68 -> 0.61 ms per Llama-1B layer)
                    ops.linear_dgrad_swiglu(A.dxb, U.p("w2"), S.gu, A.dgu)
                else:
                    ops.linear_dgrad(A.dxb, U.p("w2"), out=A.dh)
                    ops.swiglu_bwd(S.gu, A.dh, A.dgu)
                ops.linear_wgrad(A.dgu, S.ln_b, out=U.g("w13"), accumulate=ops.OVERWRITE)
                ops.linear_dgrad(A.dgu, U.p("w13"), out=A.dln)
                ops.rmsnorm_bwd(S.xb, A.dln, U.p("mlp_norm"), S.rstd_b, A.dx, A.dxb, U.g("mlp_norm"))
            # --- attention
            wo = "proj_w" if gpt2 else "wo"
            ops.linear_wgrad(A.dxb, S.o, out=U.g(wo), accumulate=ops.OVERWRITE)
            ops.linear_dgrad(A.dxb, U.p(wo), out=A.do)
            if not gpt2 and self.dtype == torch.bfloat16:  # dq / dk rotated back inside (b2s_attn_bwd_rope)
                ops.attn_bwd(S.qkv, S.o, A.do, S.lse, B, T, H, Hkv, dh, dqkv=A.dqkv, work=A.attn_work, rope=rope)
            else:
                ops.attn_bwd(S.qkv, S.o, A.do, S.lse, B, T, H, Hkv, dh, dqkv=A.dqkv, work=A.attn_work)
                if not gpt2:
                    ops.rope(A.dqkv, T, H + Hkv, dh, *rope, inverse=True)
            wq = "qkv_w" if gpt2 else "wqkv"
            if gpt2:
                ops.colsum_accumulate(A.dqkv, U.g("qkv_b"))
            ops.linear_wgrad(A.dqkv, S.ln_a, out=U.g(wq), accumulate=ops.OVERWRITE)
            ops.linear_dgrad(A.dqkv, U.p(wq), out=A.dln)
            if gpt2:
                prev_fc2_b = P.unit(i).g("fc2_b") if i > 0 else None
                ops.layernorm_bwd(S.xa, A.dln, U.p("ln1_g"), S.mean_a, S.rstd_a, A.dx, A.dxb,
                                  U.g("ln1_g"), U.g("ln1_b"), dxsum=prev_fc2_b)
            else:
                ops.rmsnorm_bwd(S.xa, A.dln, U.p("attn_norm"), S.rstd_a, A.dx, A.dxb, U.g("attn_norm"))
            post(i + 1)
        ops.embedding_bwd(tok, A.dx, E.g("wte"), E.g("wpe") if gpt2 else None, B, T)
        post(0)
        return A.loss
