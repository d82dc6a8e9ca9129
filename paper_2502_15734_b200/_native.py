"""ctypes binding of the C ABI in include/cachecraft_b200.h.

The library is built in-tree (``paper_2502_15734_b200/_lib/libcc_b200.so``,
see ``csrc/Makefile`` / ``__graft_entry__.build``).  There is no CPU fallback:
if the library or a GPU is missing, every compute entry point raises
``NativeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ArgumentError, NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libcc_b200.so")

F64, F32, BF16 = 0, 1, 2
EPI_STORE, EPI_RESID_ADD, EPI_SWIGLU, EPI_GELU = 0, 1, 2, 3
OK, E_ARG, E_CUDA, E_UNSUP = 0, -1, -2, -3

_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
_sz = ctypes.c_size_t

_SIGS = {
    "cc_abi_version": ([], _i32),
    "cc_last_error": ([], ctypes.c_char_p),
    "cc_sm_count": ([_i32], _i32),
    "cc_bf16_simt_launches": ([], ctypes.c_longlong),
    "cc_rope_table": ([_vp, _vp, _i32, _i32, _i32, _vp], _i32),
    "cc_rope_apply_f64": ([_vp, _vp, _vp, _i32, _i32, _i32, _vp, _i32, _vp], _i32),
    "cc_gather_rope_kv": ([_vp, _i64, _i64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp], _i32),
    "cc_rope_scatter_qkv": ([_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_embed_rows": ([_vp, _vp, _vp, _i32, _i32, _i32, _vp], _i32),
    "cc_rmsnorm": ([_vp, _vp, _vp, _i32, _i32, _f64, _i32, _vp], _i32),
    "cc_gemm": ([_vp, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_gemm_qkv_rope": ([_vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32,
                          _vp], _i32),
    "cc_attention": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_attention_probs": ([_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_segment_mass": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _i32, _vp, _i32, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_chunk_stats": ([_vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp], _i32),
    "cc_topk_select": ([_vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp], _i32),
    "cc_logits_argmax": ([_vp, _vp, _f64, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_extract_to_pool": ([_vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _i64, _i64, _i32, _i32, _vp], _i32),
    "cc_add_f32": ([_vp, _vp, _i64, _vp], _i32),
    "cc_flush_l2": ([_vp, _sz, _vp], _i32),
    "cc_prefetch_l2": ([_vp, _sz, _vp], _i32),
    "cc_gemv": ([_vp, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_decode_attention": ([_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_rope_rows": ([_vp, _vp, _i64, _i32, _i32, _vp, _vp, _i32, _i32, _vp], _i32),
    "cc_decode_attention_dev": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp], _i32),
    "cc_decode_attention_qkv": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _i32, _i32, _i32, _i32,
                                 _vp], _i32),
    "cc_decode_advance": ([_vp, _vp, _vp, _vp], _i32),
    "cc_set_pdl": ([_i32], _i32),
    "cc_set_stream_k": ([_i32], _i32),
    "cc_tp_push_gemm": ([_vp, _i64, _vp, _i64, _i32, _i32, _i32, _vp, _vp], _i32),
    "cc_tp_reduce": ([_vp, _i32, _i32, _vp], _i32),
    "cc_tp_wait": ([_vp, _i64, _vp], _i32),
    "cc_ipc_get_handle": ([_vp, _vp, _vp], _i32),
    "cc_ipc_open_handle": ([_vp, _vp], _i32),
    "cc_gemv_rmsnorm": ([_vp, _i64, _vp, _f64, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp], _i32),
}

_lib = None
_lock = threading.Lock()
# per-entry-point call counters and the number of kernels those calls launched
calls: dict[str, int] = {}
kernels_launched = 0


def library_loaded() -> bool:
    return _lib is not None


def lib():
    """Load (once) and return the native library; raise NativeError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(
                    f"native library {LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "or `make -C paper_2502_15734_b200/csrc`"
                )
            handle = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = res
            if handle.cc_abi_version() != 1:
                raise NativeError("native library ABI mismatch")
            _lib = handle
    return _lib


def check(rc: int, what: str):
    if rc == OK:
        return
    msg = lib().cc_last_error().decode("utf-8", "replace")
    if rc == E_ARG:
        raise ArgumentError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args):
    """Invoke a native entry point, count it and map its status."""
    global kernels_launched
    fn = getattr(lib(), name)
    rc = fn(*args)
    calls[name] = calls.get(name, 0) + 1
    # cc_logits_argmax with an argmax output runs GEMV + two argmax stages;
    # cc_decode_attention runs the split-KV partials + the combine
    kernels_launched += 3 if (name == "cc_logits_argmax" and args[5] is not None) else (
        2 if name in ("cc_decode_attention", "cc_decode_attention_dev") else 1)
    check(rc, name)
    return rc


def bf16_simt_launches() -> int:
    """SIMT kernel launches made on bf16 data (0 in the product path)."""
    return int(lib().cc_bf16_simt_launches())


def assert_tensor_core_only(before: int = 0):
    """Fail loudly if any bf16 work since ``before`` ran on a SIMT kernel."""
    n = bf16_simt_launches() - before
    if n:
        raise NativeError(f"{n} bf16 launches ran on SIMT kernels instead of tcgen05")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeError("a CUDA device is required: the B200 path has no CPU fallback")
    lib()
