"""Thin Python wrappers over the C-ABI kernels (one call = one kernel launch).

Every function takes/returns torch CUDA tensors, launches on torch's current
stream and raises :class:`_lib.B2SError` on a failed status. There is no CPU
path: calling an op on a CPU tensor is an error.
"""

from __future__ import annotations

import torch

from . import _lib

_call = _lib.call
_sp = _lib.stream_ptr


class KernelTimer:
    """CUDA-event timing of selected kernel classes on the launching stream.

    While active (``with KernelTimer() as kt``), every gemm / attention launch
    is bracketed by events and its algorithmic FLOPs recorded; ``summary()``
    (after a synchronize) returns per-class launches, FLOPs and milliseconds.
    """

    active = None

    def __init__(self):
        self.records = []

    def __enter__(self):
        KernelTimer.active = self
        return self

    def __exit__(self, *exc):
        KernelTimer.active = None

    def start(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def stop(self, kind, flops, start, detail=None):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.records.append((kind, flops, start, e, detail))

    def detail(self):
        """Per (kind, detail) launches / ms / TFLOP/s, sorted by time."""
        torch.cuda.synchronize()
        out = {}
        for kind, flops, s, e, det in self.records:
            d = out.setdefault((kind, det), [0, 0.0, 0.0])
            d[0] += 1
            d[1] += s.elapsed_time(e)
            d[2] += flops
        return sorted(((k, n, ms, fl / (ms / 1e3) / 1e12 if ms else 0) for k, (n, ms, fl) in out.items()),
                      key=lambda r: -r[2])

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for kind, flops, s, e, _ in self.records:
            d = out.setdefault(kind, {"launches": 0, "flops": 0.0, "ms": 0.0})
            d["launches"] += 1
            d["flops"] += flops
            d["ms"] += s.elapsed_time(e)
        return out


def _timed(kind, flops, fn, detail=None):
    kt = KernelTimer.active
    if kt is None:
        return fn()
    s = kt.start()
    r = fn()
    kt.stop(kind, flops, s, detail)
    return r


def _dev(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("b2s ops run on CUDA tensors only (no CPU fallback)")


def _ptr(t):
    return 0 if t is None else t.data_ptr()


def zero_(t):
    """t.zero_() as a cudaMemsetAsync on the current stream (no fill kernel in the step)."""
    _dev(t)
    assert t.is_contiguous()
    _call("b2s_memset_async", t.data_ptr(), 0, t.numel() * t.element_size(), _sp())
    return t


# ---------------------------------------------------------------------------- GEMM


def gemm(a, b, *, a_mn: bool, b_mn: bool, M: int, N: int, K: int, out=None, out_f32=False,
         accumulate=False, bias=None, act=0, aux=None):
    """C[M,N] = act(sum_k A(m,k) B(n,k) + bias) on the tcgen05 kernel.

    ``a_mn``/``b_mn`` say whether the operand's M/N dimension (rather than K) is
    the contiguous one: A is [M][K] (a_mn=False) or [K][M] (a_mn=True); B is
    [N][K] (b_mn=False) or [K][N] (b_mn=True). ``out`` may be a strided view
    whose rows are contiguous.
    """
    _dev(a, b, out, bias, aux)
    if a.dtype == torch.float32:
        return _gemm_f32(a, b, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=K, out=out, accumulate=accumulate, bias=bias,
                         act=act, aux=aux)
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    if out is None:
        out = torch.empty(M, N, device=a.device, dtype=torch.float32 if out_f32 else torch.bfloat16)
    assert out.stride(-1) == 1 and a.stride(-1) == 1 and b.stride(-1) == 1
    lda, ldb, ldc = a.stride(0), b.stride(0), out.stride(0)
    ld_aux = aux.stride(0) if aux is not None else 0
    _timed("gemm", 2.0 * M * N * K, lambda: _call(
        "b2s_gemm", a.data_ptr(), int(a_mn), lda, b.data_ptr(), int(b_mn), ldb, out.data_ptr(), ldc,
        int(out.dtype == torch.float32), M, N, K, int(accumulate), _ptr(bias), act, _ptr(aux), ld_aux, _sp()),
        detail=(M, N, K, "MN" if a_mn else "K", "MN" if b_mn else "K", "f32" if out.dtype == torch.float32 else "bf16",
                "acc" if accumulate else "", "bias" if bias is not None else "", act))
    return out


def _gemm_f32(a, b, *, a_mn, b_mn, M, N, K, out=None, accumulate=False, bias=None, act=0, aux=None):
    """fp32 mode: the same contract on the true-fp32 SIMT kernel (fp32 operands and output)."""
    assert b.dtype == torch.float32 and (bias is None or bias.dtype == torch.float32)
    if out is None:
        out = torch.empty(M, N, device=a.device, dtype=torch.float32)
    assert out.dtype == torch.float32 and out.stride(-1) == 1 and a.stride(-1) == 1 and b.stride(-1) == 1
    ld_aux = aux.stride(0) if aux is not None else 0
    _timed("gemm", 2.0 * M * N * K, lambda: _call(
        "b2s_gemm_f32", a.data_ptr(), int(a_mn), a.stride(0), b.data_ptr(), int(b_mn), b.stride(0), out.data_ptr(),
        out.stride(0), M, N, K, int(accumulate == 1 or accumulate is True), _ptr(bias), act, _ptr(aux), ld_aux,
        _sp()))
    return out


def _sfx(t):
    """C-ABI entry-point suffix for the element type of an activation tensor."""
    return "_f32" if t.dtype == torch.float32 else ""


def linear(x, w, bias=None, out=None, act=0, aux=None, accumulate=False):
    """y = x @ w^T (+ bias): x [M,K], w [N,K] (nn.Linear layout)."""
    M, K = x.shape
    N = w.shape[0]
    return gemm(x, w, a_mn=False, b_mn=False, M=M, N=N, K=K, out=out, bias=bias, act=act, aux=aux,
                accumulate=accumulate)


def linear_dgrad(dy, w, out=None, act=0, aux=None, accumulate=False, colsum_out=None):
    """dx = dy @ w: dy [M,N], w [N,K] -> [M,K].

    colsum_out (fp32 [K], bf16 path): also ``colsum_out += dx.sum(0)`` (the bias gradient of
    the layer whose output gradient dx is), from per-32-row partial sums the GEMM epilogue
    writes -- dx is not read back."""
    M, N = dy.shape
    K = w.shape[1]
    if colsum_out is None or dy.dtype != torch.bfloat16 or accumulate:
        out = gemm(dy, w, a_mn=False, b_mn=True, M=M, N=K, K=N, out=out, act=act, aux=aux,
                   accumulate=accumulate)
        if colsum_out is not None:
            colsum_accumulate(out, colsum_out)
        return out
    _dev(dy, w, out, aux, colsum_out)
    if out is None:
        out = torch.empty(M, K, device=dy.device, dtype=torch.bfloat16)
    rb = (M + 31) // 32
    part = _colsum_part(rb * K, dy.device)[: rb * K].view(rb, K)
    ld_aux = aux.stride(0) if aux is not None else 0
    _timed("gemm", 2.0 * M * N * K, lambda: _call(
        "b2s_gemm_colsum", dy.data_ptr(), 0, dy.stride(0), w.data_ptr(), 1, w.stride(0), out.data_ptr(), out.stride(0),
        M, K, N, act, _ptr(aux), ld_aux, part.data_ptr(), _sp()),
        detail=(M, K, N, "K", "MN", "bf16", "", "", act))
    colsum_accumulate(part, colsum_out)
    return out


_colsum_part_cache = {}


def _colsum_part(n, device):
    """Per-(device, stream) scratch for the GEMM-epilogue column-sum partials."""
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _colsum_part_cache.get(key)
    if buf is None or buf.numel() < n:
        buf = torch.empty(n, device=device, dtype=torch.float32)
        _colsum_part_cache[key] = buf
    return buf


def linear_swiglu(x, w13, gu, h):
    """gu = x @ w13^T ([M, 2F] gate | up) and h = silu(gate) * up ([M, F]) in one GEMM."""
    _dev(x, w13, gu, h)
    M, K = x.shape
    F = w13.shape[0] // 2
    _timed("gemm", 2.0 * M * 2 * F * K, lambda: _call(
        "b2s_gemm_swiglu_fwd", x.data_ptr(), x.stride(0), w13.data_ptr(), w13.stride(0), gu.data_ptr(), gu.stride(0),
        h.data_ptr(), h.stride(0), M, F, K, _sp()), detail=(M, 2 * F, K, "K", "K", "bf16", "", "", "swiglu"))
    return gu, h


def linear_rope(x, w, out, T, dh, rope_cols, cos, sin):
    """out = x @ w^T with the rotary embedding applied to columns [0, rope_cols) in the epilogue
    (the Llama QKV projection: q and k heads rotated, v heads as is)."""
    _dev(x, w, out, cos, sin)
    M, K = x.shape
    N = w.shape[0]
    _timed("gemm", 2.0 * M * N * K, lambda: _call(
        "b2s_gemm_rope", x.data_ptr(), x.stride(0), w.data_ptr(), w.stride(0), out.data_ptr(), out.stride(0), M, N, K,
        cos.data_ptr(), sin.data_ptr(), T, dh, rope_cols, _sp()), detail=(M, N, K, "K", "K", "bf16", "", "", "rope"))
    return out


def linear_dgrad_swiglu(dy, w2, gu, dgu):
    """dgu = SwiGLU backward of dh = dy @ w2 (dy [M, d], w2 [d, F]) without materialising dh."""
    _dev(dy, w2, gu, dgu)
    M, K = dy.shape
    F = w2.shape[1]
    _timed("gemm", 2.0 * M * F * K, lambda: _call(
        "b2s_gemm_swiglu_bwd", dy.data_ptr(), dy.stride(0), w2.data_ptr(), w2.stride(0), gu.data_ptr(), gu.stride(0),
        dgu.data_ptr(), dgu.stride(0), M, F, K, _sp()), detail=(M, F, K, "K", "MN", "bf16", "", "", "dswiglu"))
    return dgu


OVERWRITE = 2  # gemm accumulate mode: C is written whatever it held (see b2s_gemm)


def linear_wgrad(dy, x, out=None, accumulate=False, out_f32=True):
    """dw = dy^T @ x: dy [M,N], x [M,K] -> [N,K] (fp32 by default).

    accumulate: False (store), True (add into out) or OVERWRITE (fp32: store, or zero + split-K
    add-reduce -- a weight gradient's single writer in a step needs no pre-zeroed buffer)."""
    M, N = dy.shape
    K = x.shape[1]
    return gemm(dy, x, a_mn=True, b_mn=True, M=N, N=K, K=M, out=out, out_f32=out_f32,
                accumulate=accumulate)


# ---------------------------------------------------------------------------- norms


def _f32(M, D, dev):
    return torch.empty(M, D, device=dev, dtype=torch.float32)


_work_cache: dict = {}


def _work(n_floats: int, device):
    """Reusable scratch for the deterministic reductions, one per (device, stream): kernels
    on different streams (the backward's weight-gradient side stream) never share it."""
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _work_cache.get(key)
    if buf is None or buf.numel() < n_floats:
        buf = torch.empty(max(n_floats, 1 << 20), device=device, dtype=torch.float32)
        _work_cache[key] = buf
    return buf


def layernorm_fwd(x, g, b, eps=1e-5, y=None, mean=None, rstd=None, x_copy=None):
    _dev(x)
    M, D = x.shape
    y = torch.empty(M, D, device=x.device, dtype=torch.bfloat16) if y is None else y
    mean = torch.empty(M, device=x.device) if mean is None else mean
    rstd = torch.empty(M, device=x.device) if rstd is None else rstd
    _call("b2s_layernorm_fwd" + _sfx(y), x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
          rstd.data_ptr(), _ptr(x_copy), M, D, eps, _sp())
    return y, mean, rstd


def rmsnorm_fwd(x, g, eps=1e-5, y=None, rstd=None, x_copy=None):
    _dev(x)
    M, D = x.shape
    y = torch.empty(M, D, device=x.device, dtype=torch.bfloat16) if y is None else y
    rstd = torch.empty(M, device=x.device) if rstd is None else rstd
    _call("b2s_rmsnorm_fwd" + _sfx(y), x.data_ptr(), g.data_ptr(), y.data_ptr(), rstd.data_ptr(), _ptr(x_copy), M, D,
          eps, _sp())
    return y, rstd


def layernorm_fwd_res(x, res, g, b, eps, y, mean, rstd, x_out):
    """x_out = x + res (the residual add of the previous sublayer), y = LayerNorm(x_out)."""
    M, D = x.shape
    _call("b2s_layernorm_fwd_res" + _sfx(y), x.data_ptr(), res.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(),
          mean.data_ptr(), rstd.data_ptr(), x_out.data_ptr(), M, D, eps, _sp())


def rmsnorm_fwd_res(x, res, g, eps, y, rstd, x_out):
    """x_out = x + res, y = RMSNorm(x_out)."""
    M, D = x.shape
    _call("b2s_rmsnorm_fwd_res" + _sfx(y), x.data_ptr(), res.data_ptr(), g.data_ptr(), y.data_ptr(),
          rstd.data_ptr(), x_out.data_ptr(), M, D, eps, _sp())


def layernorm_bwd(x, dy, g, mean, rstd, dx, dx_bf16=None, dg=None, db=None, dxsum=None):
    """dx += LN backward; dg/db (fp32) accumulated; dxsum += colsum(updated dx)."""
    M, D = x.shape
    work = _work(_lib.load().b2s_norm_work_floats(D), x.device)
    if dx_bf16 is dx:  # fp32 mode: the GEMM operand is dx itself
        dx_bf16 = None
    _call("b2s_layernorm_bwd" + _sfx(dy), x.data_ptr(), dy.data_ptr(), g.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
          dx.data_ptr(), _ptr(dx_bf16), _ptr(dg), _ptr(db), _ptr(dxsum), work.data_ptr(), M, D, _sp())


def rmsnorm_bwd(x, dy, g, rstd, dx, dx_bf16=None, dg=None, dxsum=None):
    M, D = x.shape
    work = _work(_lib.load().b2s_norm_work_floats(D), x.device)
    if dx_bf16 is dx:
        dx_bf16 = None
    _call("b2s_rmsnorm_bwd" + _sfx(dy), x.data_ptr(), dy.data_ptr(), g.data_ptr(), rstd.data_ptr(), dx.data_ptr(),
          _ptr(dx_bf16), _ptr(dg), _ptr(dxsum), work.data_ptr(), M, D, _sp())


def colsum_accumulate(x, out):
    """out[c] += sum_r x[r, c]   (bias gradient)."""
    M, N = x.shape
    work = _work(_lib.load().b2s_colsum_work_floats(N), x.device)
    _call("b2s_colsum_accumulate", x.data_ptr(), int(x.dtype == torch.float32), M, N, x.stride(0),
          out.data_ptr(), work.data_ptr(), _sp())


# ---------------------------------------------------------------------------- misc


def embedding_fwd(tok, wte, wpe, T, out=None):
    M = tok.numel()
    D = wte.shape[1]
    out = torch.empty(M, D, device=tok.device) if out is None else out
    _call("b2s_embedding_fwd" + _sfx(wte), tok.data_ptr(), wte.data_ptr(), _ptr(wpe), out.data_ptr(), M, T, D, _sp())
    return out


def embedding_bwd(tok, dx, dwte, dwpe, B, T):
    _call("b2s_embedding_bwd", tok.data_ptr(), dx.data_ptr(), dwte.data_ptr(), _ptr(dwpe), B, T, dx.shape[1],
          _sp())


def rope(qkv, T, nheads, dh, cos, sin, inverse=False):
    M = qkv.shape[0]
    _call("b2s_rope" + _sfx(qkv), qkv.data_ptr(), M, T, qkv.stride(0), nheads, dh, cos.data_ptr(), sin.data_ptr(),
          int(inverse), _sp())


def swiglu_fwd(gu, h=None):
    M, F2 = gu.shape
    h = torch.empty(M, F2 // 2, device=gu.device, dtype=gu.dtype) if h is None else h
    _call("b2s_swiglu_fwd" + _sfx(gu), gu.data_ptr(), h.data_ptr(), M, F2 // 2, _sp())
    return h


def swiglu_bwd(gu, dh, dgu=None):
    M, F2 = gu.shape
    dgu = torch.empty_like(gu) if dgu is None else dgu
    _call("b2s_swiglu_bwd" + _sfx(gu), gu.data_ptr(), dh.data_ptr(), dgu.data_ptr(), M, F2 // 2, _sp())
    return dgu


def cross_entropy(logits, V, target, loss_rows=None, grad_scale=1.0, write_grad=True):
    M = logits.shape[0]
    loss_rows = torch.empty(M, device=logits.device) if loss_rows is None else loss_rows
    _call("b2s_cross_entropy" + _sfx(logits), logits.data_ptr(), logits.stride(0), V, target.data_ptr(), loss_rows.data_ptr(),
          grad_scale, M, int(write_grad), _sp())
    return loss_rows


def sum_(x, out, squares=False, scale=1.0):
    _call("b2s_sum", x.data_ptr(), x.numel(), int(squares), out.data_ptr(), scale, _sp())
    return out


def sumsq_partial(x, part):
    _call("b2s_sumsq_partial", x.data_ptr(), x.numel(), part.data_ptr(), part.numel(), _sp())


def sumsq_partial_multi(table, nseg, part):
    """table: int64 device tensor [2, nseg] = (fp32 buffer addresses, element counts)."""
    _call("b2s_sumsq_partial_multi", table[0].data_ptr(), table[1].data_ptr(), nseg, part.data_ptr(), part.numel(),
          _sp())


def adamw(p, m, v, g, p_bf16, step, lr, beta1, beta2, eps, wd, gn2=None, max_norm=0.0, wd_mask=None):
    """p_bf16: the compute copy written after the update (bf16 or fp32), or None / p itself (fp32 mode)."""
    if p_bf16 is p:
        p_bf16 = None
    name = "b2s_adamw_f32" if p_bf16 is None or p_bf16.dtype == torch.float32 else "b2s_adamw"
    _call(name, p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), _ptr(p_bf16), _ptr(wd_mask),
          p.numel(), _ptr(gn2), max_norm, lr, beta1, beta2, eps, wd, step, _sp())


def f32_to_bf16(x, y, scale=1.0):
    _call("b2s_f32_to_bf16", x.data_ptr(), y.data_ptr(), x.numel(), scale, _sp())
    return y


def scale_f32(x, scale):
    _call("b2s_scale_f32", x.data_ptr(), x.numel(), scale, _sp())


# ---------------------------------------------------------------------------- attention


def attn_fwd(qkv, B, T, Hq, Hkv, dh, o=None, lse=None):
    """Causal attention over the fused [B*T, (Hq+2Hkv)*dh] projection output."""
    _dev(qkv)
    o = torch.empty(B * T, Hq * dh, device=qkv.device, dtype=qkv.dtype) if o is None else o
    lse = torch.empty(B, Hq, T, device=qkv.device, dtype=torch.float32) if lse is None else lse
    flops = 4.0 * B * Hq * dh * T * T / 2  # algorithmic causal FLOPs: QK^T and PV, lower triangle
    _timed("attn_fwd", flops, lambda: _call("b2s_attn_fwd" + _sfx(qkv), qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T,
                                            Hq, Hkv, dh, _sp()))
    return o, lse


def attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh, dqkv=None, work=None, rope=None):
    """dq/dk/dv of causal attention, written into a [B*T, (Hq+2Hkv)*dh] buffer.

    rope=(cos, sin) (bf16 path): q / k carried the rotary embedding, so dq and dk are rotated
    back (the gradient w.r.t. the projection output) by b2s_attn_bwd_rope."""
    dqkv = torch.empty_like(qkv) if dqkv is None else dqkv
    n = _lib.load().b2s_attn_bwd_work_floats(B, T, Hq, dh)
    work = _work(n, qkv.device) if work is None else work
    flops = 10.0 * B * Hq * dh * T * T / 2  # S, dP, dV, dK, dQ over the lower triangle
    if rope is not None:
        assert qkv.dtype == torch.bfloat16
        cos, sin = rope
        _timed("attn_bwd", flops, lambda: _call("b2s_attn_bwd_rope", qkv.data_ptr(), o.data_ptr(), do.data_ptr(),
                                                lse.data_ptr(), dqkv.data_ptr(), work.data_ptr(), B, T, Hq, Hkv, dh,
                                                cos.data_ptr(), sin.data_ptr(), _sp()))
        return dqkv
    _timed("attn_bwd", flops, lambda: _call("b2s_attn_bwd" + _sfx(qkv), qkv.data_ptr(), o.data_ptr(), do.data_ptr(),
                                            lse.data_ptr(), dqkv.data_ptr(), work.data_ptr(), B, T, Hq, Hkv, dh,
                                            _sp()))
    return dqkv
