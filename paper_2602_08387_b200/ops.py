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


def _dev(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("b2s ops run on CUDA tensors only (no CPU fallback)")


def _ptr(t):
    return 0 if t is None else t.data_ptr()


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
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    if out is None:
        out = torch.empty(M, N, device=a.device, dtype=torch.float32 if out_f32 else torch.bfloat16)
    assert out.stride(-1) == 1 and a.stride(-1) == 1 and b.stride(-1) == 1
    lda, ldb, ldc = a.stride(0), b.stride(0), out.stride(0)
    ld_aux = aux.stride(0) if aux is not None else 0
    _call("b2s_gemm", a.data_ptr(), int(a_mn), lda, b.data_ptr(), int(b_mn), ldb, out.data_ptr(), ldc,
          int(out.dtype == torch.float32), M, N, K, int(accumulate), _ptr(bias), act, _ptr(aux), ld_aux,
          _sp())
    return out


def linear(x, w, bias=None, out=None, act=0, aux=None, accumulate=False):
    """y = x @ w^T (+ bias): x [M,K], w [N,K] (nn.Linear layout)."""
    M, K = x.shape
    N = w.shape[0]
    return gemm(x, w, a_mn=False, b_mn=False, M=M, N=N, K=K, out=out, bias=bias, act=act, aux=aux,
                accumulate=accumulate)


def linear_dgrad(dy, w, out=None, act=0, aux=None, accumulate=False):
    """dx = dy @ w: dy [M,N], w [N,K] -> [M,K]."""
    M, N = dy.shape
    K = w.shape[1]
    return gemm(dy, w, a_mn=False, b_mn=True, M=M, N=K, K=N, out=out, act=act, aux=aux,
                accumulate=accumulate)


def linear_wgrad(dy, x, out=None, accumulate=False, out_f32=True):
    """dw = dy^T @ x: dy [M,N], x [M,K] -> [N,K] (fp32 by default)."""
    M, N = dy.shape
    K = x.shape[1]
    return gemm(dy, x, a_mn=True, b_mn=True, M=N, N=K, K=M, out=out, out_f32=out_f32,
                accumulate=accumulate)
