"""ctypes binding of the C ABI in include/mxb200.h (libmxb200.so, in-tree).

The shared library is plain C ABI (no torch types), built for sm_100a by
``__graft_entry__.build()`` / ``python -m paper_2411_09510_b200.build``.
There is no fallback: if the library or a CUDA device is missing, every
compute entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeUnavailable, raise_for_status

LIB_NAME = "libmxb200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

MX_F32, MX_F16, MX_BF16, MX_F64 = 0, 1, 2, 3

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_vp = ctypes.c_void_p
c_i64p = ctypes.POINTER(ctypes.c_int64)


class MxScheme(ctypes.Structure):
    """mx_scheme_t"""

    _fields_ = [("kind", c_i32), ("exponent_bits", c_i32), ("mantissa_bits", c_i32),
                ("scale_bits", c_i32), ("block_size", c_i64)]


_SP = ctypes.POINTER(MxScheme)

# name -> (restype, argtypes); every symbol include/mxb200.h declares
SIGNATURES = {
    "mx_abi_version": (c_i32, []),
    "mx_last_error": (ctypes.c_char_p, []),
    "mx_scheme_check": (c_i32, [_SP]),
    "mx_stream_nbytes": (c_i32, [c_i64, _SP, c_i64p, c_i64p]),
    "mx_shard_layout": (c_i32, [c_i64, _SP, c_i64p, c_i64p, c_i64p]),
    "mx_workspace_bytes": (c_i32, [c_i64, _SP, c_i64p]),
    "mx_requant_workspace_bytes": (c_i32, [c_i64, _SP, c_i64p]),
    "mx_quantize": (c_i32, [c_vp, c_i32, c_i64, _SP, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "mx_dequantize": (c_i32, [c_vp, c_vp, c_i64, _SP, c_vp, c_i32, c_vp]),
    "mx_quantize_chunks": (c_i32, [c_vp, c_i32, c_i64, c_i64, _SP, c_vp, c_i64, c_vp, c_vp,
                                   c_i64, c_vp]),
    "mx_dequant_sum": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_i64, c_i64, _SP, c_vp, c_i32, c_vp]),
    "mx_dequant_sum_residual": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_i64, c_i64, _SP, c_vp, c_vp,
                                        c_i32, c_vp]),
    "mx_dequant_sum_requant": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_i64, _SP, c_vp, c_vp, c_vp,
                                       c_i64, c_vp]),
    "mx_allreduce_fused": (c_i32, [c_vp, c_i32, c_i32, c_i64, _SP, c_vp, c_i64, c_vp, c_i32,
                                   c_vp, c_vp, c_vp]),
    "mx_symm_twoshot_layout": (c_i32, [c_i64, _SP, c_i32, c_i64p, c_i64p, c_i64p, c_i64p,
                                       c_i64p]),
    "mx_allreduce_symm_twoshot": (c_i32, [c_vp, c_i32, c_i64, _SP, c_vp, c_vp, c_i32, c_i32,
                                          c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mx_symm_layout": (c_i32, [c_i64, _SP, c_i32, c_i64p, c_i64p, c_i64p, c_i64p]),
    "mx_allreduce_symm": (c_i32, [c_vp, c_i32, c_i64, _SP, c_vp, c_vp, c_i32, c_i32, c_i64, c_vp,
                                  c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mx_unpack_codes": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "mx_pack_codes": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "mx_chanint_compress": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_i64,
                                    c_vp, c_vp]),
    "mx_chanint_decompress": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_i32, c_vp]),
    "mx_topk_workspace_bytes": (c_i32, [c_i64, c_i64p]),
    "mx_topk_compress": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "mx_topk_decompress": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i32, c_vp]),
    "mx_gemm_quantize": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, _SP, c_vp, c_vp, c_vp, c_vp,
                                 c_vp]),
    "mx_gemm_quantize_chunks": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, _SP, c_vp, c_i64,
                                        c_vp, c_vp, c_vp]),
    "mx_memset_async": (c_i32, [c_vp, c_i32, c_i64, c_vp]),
    "mx_serialize": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "mx_push_layout": (c_i32, [c_i64, _SP, c_i32, c_i64p, c_i64p, c_i64p, c_i64p]),
    "mx_push2_layout": (c_i32, [c_i64, _SP, c_i32, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p]),
    "mx_gemm_reducescatter_push": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, _SP, c_vp, c_i32,
                                           c_i32, c_vp, c_vp, c_vp]),
    "mx_push2_requant": (c_i32, [c_vp, c_i64, _SP, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                 c_vp]),
    "mx_push2_decode": (c_i32, [c_vp, c_i64, _SP, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp,
                                c_vp]),
    "mx_gemm_allgather_push": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, _SP, c_vp, c_i32, c_i32,
                                       c_vp, c_vp, c_vp]),
    "mx_push_dequant_sum": (c_i32, [c_vp, c_i64, _SP, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                    c_i32, c_vp, c_vp]),
    "mx_copy_bytes": (c_i32, [c_vp, c_i64, c_vp, c_vp]),
    "mx_nonfinite_reset": (c_i32, [c_vp, c_vp]),
}

ABI_VERSION = 1

_lock = threading.Lock()
_lib = None


class _StrictLib:
    """The loaded CDLL with an exact-arity check on every declared entry
    point: ctypes silently accepts surplus arguments (it treats them as C
    varargs), which would turn an ABI drift into a mis-bound stream pointer."""

    def __init__(self, lib: ctypes.CDLL):
        self._cdll = lib
        for name, (_res, args) in SIGNATURES.items():
            setattr(self, name, self._strict(name, getattr(lib, name), len(args)))

    @staticmethod
    def _strict(name, fn, arity):
        def call(*a):
            if len(a) != arity:
                raise TypeError(f"{name} takes {arity} arguments, got {len(a)}")
            return fn(*a)

        call.__name__ = name
        return call

    def __getattr__(self, name):  # undeclared helpers (mx_abi_version, mx_last_error)
        return getattr(self._cdll, name)


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libmxb200.so and bind every exported symbol (raises if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError = ABI drift, fail loudly
            fn.restype = res
            fn.argtypes = args
        if lib.mx_abi_version() != ABI_VERSION:
            raise NativeUnavailable(f"{path}: ABI {lib.mx_abi_version()} != {ABI_VERSION}")
        _lib = _StrictLib(lib)
        return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _lib.mx_last_error().decode(errors="replace") if _lib is not None else ""
        raise_for_status(rc, f"{what}: {msg}")


def scheme_ptr(c_scheme: MxScheme):
    return ctypes.byref(c_scheme)


def stream_nbytes(n: int, cs: MxScheme) -> tuple[int, int]:
    lib = load()
    a, b = c_i64(), c_i64()
    check(lib.mx_stream_nbytes(n, ctypes.byref(cs), ctypes.byref(a), ctypes.byref(b)),
          "mx_stream_nbytes")
    return a.value, b.value


def shard_layout(n: int, cs: MxScheme) -> tuple[int, int, int]:
    lib = load()
    a, b, c = c_i64(), c_i64(), c_i64()
    check(lib.mx_shard_layout(n, ctypes.byref(cs), ctypes.byref(a), ctypes.byref(b),
                              ctypes.byref(c)), "mx_shard_layout")
    return a.value, b.value, c.value


def workspace_bytes(n: int, cs: MxScheme, requant: bool = False) -> int:
    lib = load()
    a = c_i64()
    fn = lib.mx_requant_workspace_bytes if requant else lib.mx_workspace_bytes
    check(fn(n, ctypes.byref(cs), ctypes.byref(a)), "mx_workspace_bytes")
    return a.value


def symm_layout(n: int, cs: MxScheme, nranks: int) -> tuple[int, int, int, int]:
    """(slot_stride, flags_offset, buffer_bytes, ctas) of the symmetric-memory collective."""
    lib = load()
    a, b, c, d = c_i64(), c_i64(), c_i64(), c_i64()
    check(lib.mx_symm_layout(n, ctypes.byref(cs), nranks, ctypes.byref(a), ctypes.byref(b),
                             ctypes.byref(c), ctypes.byref(d)), "mx_symm_layout")
    return a.value, b.value, c.value, d.value


def push_layout(n: int, cs: MxScheme, nranks: int) -> tuple[int, int, int, int]:
    """(slot_stride, shard_stride, flags_offset, buffer_bytes) of the GEMM +
    all-gather push (mx_push_layout)."""
    lib = load()
    v = [c_i64() for _ in range(4)]
    check(lib.mx_push_layout(n, ctypes.byref(cs), nranks, *[ctypes.byref(x) for x in v]),
          "mx_push_layout")
    return tuple(x.value for x in v)


def push2_layout(n: int, cs: MxScheme, nranks: int) -> tuple[int, int, int, int, int]:
    """(chunk_values, slot_stride, shard_stride, flags_offset, buffer_bytes)
    of the two-shot GEMM push (mx_push2_layout)."""
    lib = load()
    v = [c_i64() for _ in range(5)]
    check(lib.mx_push2_layout(n, ctypes.byref(cs), nranks, *[ctypes.byref(x) for x in v]),
          "mx_push2_layout")
    return tuple(x.value for x in v)


def symm_twoshot_layout(n: int, cs: MxScheme, nranks: int):
    """(slot_stride, shard_stride, flags_offset, buffer_bytes, ctas) of the
    two-shot symmetric-memory collective."""
    lib = load()
    v = [c_i64() for _ in range(5)]
    check(lib.mx_symm_twoshot_layout(n, ctypes.byref(cs), nranks, *[ctypes.byref(x) for x in v]),
          "mx_symm_twoshot_layout")
    return tuple(x.value for x in v)


def require_cuda():
    """The product path runs on the GPU or not at all."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the MX codec runs only on the sm_100a kernels")
    load()
