"""ctypes binding of libpa.so (include/pa.h).  Argument marshalling only.

Every function below has the name and argument order of its C counterpart;
pointers are passed as Python ints (e.g. ``tensor.data_ptr()``) and streams as
``torch.cuda.Stream.cuda_stream`` ints (0 = legacy default stream).  Non-OK
statuses raise :class:`PaError` carrying the library's ``pa_last_error()``.
There is no fallback: if the shared library is missing this module raises at
import time.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PA_LIB", os.path.join(HERE, "libpa.so"))

PA_OK = 0
PA_ERR_INVALID_ARG = 1
PA_ERR_UNSUPPORTED = 2
PA_ERR_NOMEM = 3
PA_ERR_CUDA = 4
PA_ERR_PRECISION = 5
STATUS_NAMES = {0: "PA_OK", 1: "PA_ERR_INVALID_ARG", 2: "PA_ERR_UNSUPPORTED", 3: "PA_ERR_NOMEM",
                4: "PA_ERR_CUDA", 5: "PA_ERR_PRECISION"}

PA_ROUTE_AUTO = 0
PA_ROUTE_TRANSFORM = 1
PA_ROUTE_BITPACKED = 2
PA_ARITH_AUTO, PA_ARITH_FP64, PA_ARITH_NTT32, PA_ARITH_NTT64 = 0, 1, 2, 3
PA_PLAN_MODEL, PA_PLAN_MEASURE = 0, 1
PA_RESIDUAL_LIMIT = 0.25

EXPORTED = ["pa_options_init", "pa_create", "pa_create_ex", "pa_hash", "pa_hash_batch",
            "pa_hash_host", "pa_create_u64", "pa_hash_u64", "pa_residual", "pa_get_info",
            "pa_destroy", "pa_last_error", "pa_status_string", "pa_version", "pa_profile_enable",
            "pa_profile_read", "pa_plan", "pa_set_seed", "pa_xor_fold", "pa_hash_host_async", "pa_hash_blocked", "pa_hash_blocked_host",
            "pa_workspace_size", "pa_create_ws", "pa_hash_fresh_batch", "pa_seed_from_paper_eq1",
            "pa_hash_host_batch", "pa_xor_fold_peers", "pa_peer_alloc", "pa_peer_free", "pa_peer_export",
            "pa_peer_open", "pa_peer_close", "pa_hash_blocked_release", "pa_blocked_plan"]


class PaError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")


class pa_peer_handle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 64)]


class pa_options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("route", ctypes.c_int32),
                ("seed_bit_offset", ctypes.c_uint64), ("allow_wide", ctypes.c_uint32),
                ("batch_keys", ctypes.c_uint32), ("max_transform_len", ctypes.c_uint64),
                ("arith", ctypes.c_int32), ("device", ctypes.c_int32), ("plan_mode", ctypes.c_uint32)]


class pa_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("m", ctypes.c_uint64), ("route", ctypes.c_int32),
                ("device", ctypes.c_int32), ("transform_len", ctypes.c_uint64),
                ("n1", ctypes.c_uint64), ("n2", ctypes.c_uint64), ("cols_per_cta", ctypes.c_uint64),
                ("workspace_bytes", ctypes.c_uint64), ("kernels_per_hash", ctypes.c_uint64),
                ("column_blocks", ctypes.c_uint64), ("k3_cols_per_cta", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class pa_kernel_time(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64), ("total_ms", ctypes.c_double)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1805_02372_b200.build` "
                      "(nvcc, sm_100a).  There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)
_u64, _p, _st = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
_H = ctypes.c_void_p
_sig = {
    "pa_options_init": (_st, [ctypes.POINTER(pa_options)]),
    "pa_create": (_st, [ctypes.POINTER(_H), _u64, _u64, _p, _p]),
    "pa_create_ex": (_st, [ctypes.POINTER(_H), _u64, _u64, _p, ctypes.POINTER(pa_options), _p]),
    "pa_hash": (_st, [_H, _p, _p, _p]),
    "pa_hash_batch": (_st, [_H, _p, _u64, _p, _u64, ctypes.c_uint32, _p]),
    "pa_hash_host": (_st, [_H, _p, _p, _p]),
    "pa_hash_host_async": (_st, [_H, _p, _p, _p]),
    "pa_hash_host_batch": (_st, [_H, _p, _u64, _p, _u64, ctypes.c_uint32, _p]),
    "pa_hash_blocked": (_st, [_u64, _u64, _p, _p, _p, _u64, _p]),
    "pa_hash_blocked_host": (_st, [_u64, _u64, _p, _p, _p, _u64, _u64, _p]),
    "pa_create_u64": (_st, [ctypes.POINTER(_H), _u64, _u64, _p, _p]),
    "pa_hash_u64": (_st, [_H, _p, _p, _p]),
    "pa_residual": (_st, [_H, ctypes.POINTER(ctypes.c_double), _p]),
    "pa_get_info": (_st, [_H, ctypes.POINTER(pa_info)]),
    "pa_destroy": (None, [_H]),
    "pa_last_error": (ctypes.c_char_p, []),
    "pa_status_string": (ctypes.c_char_p, [_st]),
    "pa_version": (ctypes.c_uint32, []),
    "pa_profile_enable": (_st, [_H, ctypes.c_int]),
    "pa_plan": (_st, [_u64, _u64, ctypes.POINTER(pa_info)]),
    "pa_set_seed": (_st, [_H, _p, _p]),
    "pa_workspace_size": (_st, [_u64, _u64, ctypes.POINTER(pa_options), ctypes.POINTER(_u64)]),
    "pa_create_ws": (_st, [ctypes.POINTER(_H), _u64, _u64, _p, ctypes.POINTER(pa_options), _p, _u64, _p]),
    "pa_hash_fresh_batch": (_st, [_H, _p, _u64, _p, _u64, _p, _u64, ctypes.c_uint32, _p]),
    "pa_seed_from_paper_eq1": (_st, [_p, _p, _u64, _u64, _p]),
    "pa_xor_fold": (_st, [_p, _p, _u64, ctypes.c_uint32, _u64, _p]),
    "pa_xor_fold_peers": (_st, [_p, _p, ctypes.c_uint32, _u64, _u64, _p]),
    "pa_peer_alloc": (_st, [_u64, ctypes.POINTER(_p)]),
    "pa_peer_free": (_st, [_p]),
    "pa_peer_export": (_st, [_p, ctypes.POINTER(pa_peer_handle)]),
    "pa_peer_open": (_st, [ctypes.POINTER(pa_peer_handle), ctypes.POINTER(_p)]),
    "pa_peer_close": (_st, [_p]),
    "pa_hash_blocked_release": (None, []),
    "pa_blocked_plan": (_st, [_u64, _u64, _u64, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64),
                              ctypes.POINTER(_u64)]),
    "pa_profile_read": (_st, [_H, ctypes.POINTER(pa_kernel_time), ctypes.c_uint32,
                              ctypes.POINTER(ctypes.c_uint32)]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def _check(status: int) -> None:
    if status != PA_OK:
        raise PaError(status, _lib.pa_last_error().decode(errors="replace"))


def pa_version() -> int:
    return int(_lib.pa_version())


def pa_last_error() -> str:
    return _lib.pa_last_error().decode(errors="replace")


def pa_status_string(status: int) -> str:
    return _lib.pa_status_string(status).decode()


def pa_options_init() -> pa_options:
    o = pa_options()
    _check(_lib.pa_options_init(ctypes.byref(o)))
    return o


def pa_create(n: int, m: int, seed_ptr: int, stream: int = 0) -> int:
    h = _H()
    _check(_lib.pa_create(ctypes.byref(h), n, m, seed_ptr, stream))
    return h.value


def pa_create_ex(n: int, m: int, seed_ptr: int, opt: pa_options | None, stream: int = 0) -> int:
    h = _H()
    _check(_lib.pa_create_ex(ctypes.byref(h), n, m, seed_ptr,
                             ctypes.byref(opt) if opt is not None else None, stream))
    return h.value


def pa_create_u64(n: int, m: int, seed_ptr: int, stream: int = 0) -> int:
    h = _H()
    _check(_lib.pa_create_u64(ctypes.byref(h), n, m, seed_ptr, stream))
    return h.value


def pa_hash(h: int, key_ptr: int, out_ptr: int, stream: int = 0) -> None:
    _check(_lib.pa_hash(h, key_ptr, out_ptr, stream))


def pa_hash_u64(h: int, key_ptr: int, out_ptr: int, stream: int = 0) -> None:
    _check(_lib.pa_hash_u64(h, key_ptr, out_ptr, stream))


def pa_hash_batch(h: int, keys_ptr: int, key_stride_words: int, outs_ptr: int,
                  out_stride_words: int, count: int, stream: int = 0) -> None:
    _check(_lib.pa_hash_batch(h, keys_ptr, key_stride_words, outs_ptr, out_stride_words, count, stream))


def pa_hash_host(h: int, key_host_ptr: int, out_host_ptr: int, stream: int = 0) -> None:
    _check(_lib.pa_hash_host(h, key_host_ptr, out_host_ptr, stream))


def pa_hash_host_async(h: int, key_host_ptr: int, out_host_ptr: int, stream: int = 0) -> None:
    _check(_lib.pa_hash_host_async(h, key_host_ptr, out_host_ptr, stream))


def pa_residual(h: int, stream: int = 0) -> float:
    r = ctypes.c_double()
    _check(_lib.pa_residual(h, ctypes.byref(r), stream))
    return r.value


def pa_get_info(h: int) -> dict:
    info = pa_info()
    _check(_lib.pa_get_info(h, ctypes.byref(info)))
    return info.as_dict()


def pa_destroy(h: int) -> None:
    _lib.pa_destroy(h)


def pa_profile_enable(h: int, enable: bool) -> None:
    _check(_lib.pa_profile_enable(h, 1 if enable else 0))


def pa_profile_read(h: int) -> dict:
    """{kernel name: (launches, total_ms)} accumulated since the last read."""
    arr = (pa_kernel_time * 8)()
    n = ctypes.c_uint32()
    _check(_lib.pa_profile_read(h, arr, 8, ctypes.byref(n)))
    return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(n.value)}


def pa_plan(n: int, m: int) -> dict:
    """Host-only: the plan pa_create would choose for (n, m)."""
    info = pa_info()
    _check(_lib.pa_plan(n, m, ctypes.byref(info)))
    return info.as_dict()


def pa_set_seed(h: int, seed_ptr: int, stream: int = 0) -> None:
    _check(_lib.pa_set_seed(h, seed_ptr, stream))


def pa_xor_fold(dst_ptr: int, src_ptr: int, words: int, count: int, src_stride_words: int,
                stream: int = 0) -> None:
    _check(_lib.pa_xor_fold(dst_ptr, src_ptr, words, count, src_stride_words, stream))


def pa_hash_blocked(n: int, m: int, seed_ptr: int, key_ptr: int, out_ptr: int, max_block_bits: int = 0,
                    stream: int = 0) -> None:
    _check(_lib.pa_hash_blocked(n, m, seed_ptr, key_ptr, out_ptr, max_block_bits, stream))


def pa_hash_blocked_host(n: int, m: int, seed_host_ptr: int, key_host_ptr: int, out_host_ptr: int,
                         max_block_bits: int = 0, device_budget_bytes: int = 0, stream: int = 0) -> None:
    _check(_lib.pa_hash_blocked_host(n, m, seed_host_ptr, key_host_ptr, out_host_ptr, max_block_bits,
                                     device_budget_bytes, stream))


def pa_workspace_size(n: int, m: int, opt: pa_options | None = None) -> int:
    """Host-only: exact device bytes pa_create_ws needs for (n, m, opt)."""
    b = _u64()
    _check(_lib.pa_workspace_size(n, m, ctypes.byref(opt) if opt is not None else None, ctypes.byref(b)))
    return int(b.value)


def pa_create_ws(n: int, m: int, seed_ptr: int, opt: pa_options | None, workspace_ptr: int,
                 workspace_bytes: int, stream: int = 0) -> int:
    h = _H()
    _check(_lib.pa_create_ws(ctypes.byref(h), n, m, seed_ptr, ctypes.byref(opt) if opt is not None else None,
                             workspace_ptr, workspace_bytes, stream))
    return h.value


def pa_hash_fresh_batch(h: int, seeds_ptr: int, seed_stride_words: int, keys_ptr: int, key_stride_words: int,
                        outs_ptr: int, out_stride_words: int, count: int, stream: int = 0) -> None:
    _check(_lib.pa_hash_fresh_batch(h, seeds_ptr, seed_stride_words, keys_ptr, key_stride_words, outs_ptr,
                                    out_stride_words, count, stream))


def pa_seed_from_paper_eq1(s_ptr: int, t_ptr: int, n: int, m: int, stream: int = 0) -> None:
    _check(_lib.pa_seed_from_paper_eq1(s_ptr, t_ptr, n, m, stream))


def pa_hash_host_batch(h: int, keys_host_ptr: int, key_stride_words: int, outs_host_ptr: int,
                       out_stride_words: int, count: int, stream: int = 0) -> None:
    _check(_lib.pa_hash_host_batch(h, keys_host_ptr, key_stride_words, outs_host_ptr, out_stride_words, count,
                                   stream))


def pa_xor_fold_peers(dst_ptr: int, srcs_dev_ptr: int, count: int, first_word: int, words: int,
                      stream: int = 0) -> None:
    _check(_lib.pa_xor_fold_peers(dst_ptr, srcs_dev_ptr, count, first_word, words, stream))


def pa_peer_alloc(nbytes: int) -> int:
    p = _p()
    _check(_lib.pa_peer_alloc(nbytes, ctypes.byref(p)))
    return int(p.value)


def pa_peer_free(ptr: int) -> None:
    _check(_lib.pa_peer_free(ptr))


def pa_peer_export(ptr: int) -> bytes:
    h = pa_peer_handle()
    _check(_lib.pa_peer_export(ptr, ctypes.byref(h)))
    return bytes(h.bytes)


def pa_peer_open(handle: bytes) -> int:
    h = pa_peer_handle()
    ctypes.memmove(h.bytes, handle, 64)
    p = _p()
    _check(_lib.pa_peer_open(ctypes.byref(h), ctypes.byref(p)))
    return int(p.value)


def pa_peer_close(ptr: int) -> None:
    _check(_lib.pa_peer_close(ptr))


def pa_blocked_plan(n: int, m: int, max_block_bits: int = 0, device_budget_bytes: int = 0) -> dict:
    """The block shape pa_hash_blocked(_host) would use: {"nb", "mb", "blocks"} (host-only)."""
    nb, mb, blocks = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _check(_lib.pa_blocked_plan(n, m, max_block_bits, device_budget_bytes, ctypes.byref(nb), ctypes.byref(mb),
                                ctypes.byref(blocks)))
    return {"nb": nb.value, "mb": mb.value, "blocks": blocks.value}


def pa_hash_blocked_release() -> None:
    _lib.pa_hash_blocked_release()
