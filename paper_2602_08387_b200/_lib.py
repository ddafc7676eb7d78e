"""ctypes binding of the C-ABI library ``libb2s.so`` (declared in include/b2s.h).

This is the only way the package reaches its CUDA kernels. There is no CPU
fallback: if the library is missing the import of any op raises
:class:`NativeLibraryMissing` instead of silently computing on the host.
"""

from __future__ import annotations

import ctypes
import os
import re
from ctypes import POINTER, c_char_p, c_int, c_int32, c_int64, c_uint64, c_void_p, c_float

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B2S_LIB") or os.path.join(_HERE, "libb2s.so")  # B2S_LIB: experiment builds
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "b2s.h")

B2S_OK = 0
B2S_EINVAL = -1
B2S_ERANGE = -2
B2S_ECUDA = -3
B2S_EUNSUPPORTED = -4


class NativeLibraryMissing(RuntimeError):
    """libb2s.so was not built; run ``__graft_entry__.build()``."""


class B2SError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


_lib = None

# Argument signatures of every exported function, keyed by name. `p` = pointer
# (device or host; passed as int), `i` = int, `l` = int64, `u` = uint64, `f` = float.
_SIGS = {
    "b2s_abi_version": "",
    "b2s_memset_async": "piup",
    "b2s_graph_capture_begin": "p",
    "b2s_graph_capture_end": "pp",
    "b2s_graph_launch": "pp",
    "b2s_graph_destroy": "p",
    "b2s_token_width_for_vocab": "up",
    "b2s_sample_count": "ulp",
    "b2s_splitmix64": "uup",
    "b2s_make_permutation": "uup",
    "b2s_chunk_bounds": "uup",
    "b2s_gather_samples": "piupilpppp",
    "b2s_unpack_windows": "piilppp",
    "b2s_gather_documents": "pippplpp",
    "b2s_newline_count": "puupip",
    "b2s_newline_positions": "puupiupp",
    "b2s_tokenizer_encode": "pplplp",
    "b2s_tokenize_corpus": "pplppiiiipp",
    "b2s_gemm": "pilpilpliiiiipiplp",
    "b2s_gemm_colsum": "pilpilpliiiiplpp",
    "b2s_gemm_swiglu_fwd": "plplplpliiip",
    "b2s_gemm_swiglu_bwd": "plplplpliiip",
    "b2s_gemm_rope": "plplpliiippiiip",
    "b2s_layernorm_fwd": "ppppppplifp",
    "b2s_rmsnorm_fwd": "ppppplifp",
    "b2s_layernorm_fwd_res": "pppppppplifp",
    "b2s_rmsnorm_fwd_res": "pppppplifp",
    "b2s_layernorm_fwd_res_f32": "pppppppplifp",
    "b2s_rmsnorm_fwd_res_f32": "pppppplifp",
    "b2s_layernorm_bwd": "ppppppppppplip",
    "b2s_rmsnorm_bwd": "ppppppppplip",
    "b2s_colsum_accumulate": "pililppp",
    "b2s_embedding_fwd": "ppppliip",
    "b2s_embedding_bwd": "ppppiiip",
    "b2s_rope": "pliliippip",
    "b2s_swiglu_fwd": "pplip",
    "b2s_swiglu_bwd": "ppplip",
    "b2s_cross_entropy": "plippflip",
    "b2s_sum": "plipfp",
    "b2s_sumsq_partial": "plpip",
    "b2s_sumsq_partial_multi": "ppipip",
    "b2s_adamw": "pppppplpffffffip",
    "b2s_f32_to_bf16": "pplfp",
    "b2s_scale_f32": "plfp",
    "b2s_attn_fwd": "pppiiiiip",
    "b2s_attn_bwd": "ppppppiiiiip",
    "b2s_attn_bwd_rope": "ppppppiiiiippp",
    # fp32 mode (same argument order as the bf16 entry points)
    "b2s_gemm_f32": "pilpilpliiiipiplp",
    "b2s_layernorm_fwd_f32": "ppppppplifp",
    "b2s_rmsnorm_fwd_f32": "ppppplifp",
    "b2s_layernorm_bwd_f32": "ppppppppppplip",
    "b2s_rmsnorm_bwd_f32": "ppppppppplip",
    "b2s_embedding_fwd_f32": "ppppliip",
    "b2s_rope_f32": "pliliippip",
    "b2s_swiglu_fwd_f32": "pplip",
    "b2s_swiglu_bwd_f32": "ppplip",
    "b2s_cross_entropy_f32": "plippflip",
    "b2s_adamw_f32": "pppppplpffffffip",
    "b2s_attn_fwd_f32": "pppiiiiip",
    "b2s_attn_bwd_f32": "ppppppiiiiip",
}
# functions returning int64 sizes (not statuses): name -> argument signature
_SIZE_FNS = {"b2s_launch_count": "", "b2s_norm_work_floats": "i", "b2s_colsum_work_floats": "i", "b2s_attn_bwd_work_floats": "iiii"}

_CT = {"p": c_void_p, "i": c_int, "l": c_int64, "u": c_uint64, "f": c_float}


def load():
    """Load libb2s.so once and attach argtypes. Raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found: the CUDA path has no fallback; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    lib.b2s_last_error.restype = c_char_p
    lib.b2s_last_error.argtypes = []
    for name, sig in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = c_int
        fn.argtypes = [_CT[c] for c in sig]
    lib.b2s_tokenizer_create.restype = c_void_p
    lib.b2s_tokenizer_create.argtypes = [c_int, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64]
    lib.b2s_tokenizer_destroy.restype = None
    lib.b2s_tokenizer_destroy.argtypes = [c_void_p]
    for name, sig in _SIZE_FNS.items():
        fn = getattr(lib, name)
        fn.restype = c_int64
        fn.argtypes = [_CT[c] for c in sig]
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke ``name``; raise :class:`B2SError` on a non-zero status."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != B2S_OK:
        raise B2SError(name, rc, lib.b2s_last_error().decode(errors="replace"))


_replayed = 0


def count_replayed_launches(n: int) -> None:
    """Kernels launched by replaying a captured CUDA graph (the library's own
    counter only sees host-side launches)."""
    global _replayed
    _replayed += n


def launch_count() -> int:
    """Library kernels launched so far: direct launches + CUDA-graph replays."""
    return int(load().b2s_launch_count()) + _replayed


def last_error() -> str:
    return load().b2s_last_error().decode(errors="replace")


def declared_symbols() -> list[str]:
    """Function names declared in include/b2s.h (used by the ABI export test)."""
    with open(HEADER_PATH) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(b2s_[a-z0-9_]+)\s*\(", text)))


def stream_ptr(stream=None) -> int:
    """cudaStream_t of ``stream`` (default: torch's current stream) as an int."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
