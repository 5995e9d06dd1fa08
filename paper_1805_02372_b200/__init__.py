"""paper_1805_02372_b200 -- bit-exact Toeplitz-hash privacy amplification on B200.

The hot path of arXiv 1805.02372 (length-compatible privacy amplification for
CV-QKD): y = T x over GF(2), T the m x n Toeplitz matrix of an (n+m-1)-bit
seed, x the n-bit corrected key (Sec. 2.1 Eq. (1), Sec. 2.3, Sec. 3).
All arithmetic runs in the sm_100a kernels of ``libpa.so`` (C ABI in
``include/pa.h``); this package only marshals torch CUDA tensors into it.

    import torch, paper_1805_02372_b200 as pa
    h = pa.Hasher(n, m, seed_words_cuda)     # pa_create
    y = h.hash(key_words_cuda)               # pa_hash -> int32 words, LSB-first
    h.close()                                # pa_destroy

Bit strings are LSB-first in 32-bit words (any integer dtype is accepted; its
bytes are reinterpreted).  torch is used for device memory and streams only.
"""
from __future__ import annotations

import torch  # loads the CUDA runtime that libpa.so binds to

from . import _lib
from ._lib import (PA_ARITH_AUTO, PA_ARITH_FP64, PA_ARITH_NTT32, PA_ARITH_NTT64, PA_PLAN_MEASURE,  # noqa: F401
                   PA_PLAN_MODEL,
                   PA_ERR_CUDA, PA_ERR_INVALID_ARG, PA_ERR_NOMEM, PA_ERR_PRECISION,  # noqa: F401
                   PA_ERR_UNSUPPORTED, PA_OK, PA_RESIDUAL_LIMIT, PA_ROUTE_AUTO, PA_ROUTE_BITPACKED,
                   PA_ROUTE_TRANSFORM, PaError, pa_create, pa_create_ex, pa_create_u64, pa_destroy,
                   pa_get_info, pa_hash, pa_hash_batch, pa_hash_blocked, pa_hash_blocked_host, pa_hash_host, pa_hash_host_async, pa_hash_u64, pa_last_error,
                   pa_options_init, pa_plan, pa_profile_enable, pa_profile_read, pa_set_seed, pa_xor_fold, pa_residual, pa_status_string,
                   pa_version, pa_workspace_size, pa_create_ws, pa_hash_fresh_batch, pa_seed_from_paper_eq1,
                   pa_hash_host_batch, pa_xor_fold_peers, pa_peer_alloc, pa_peer_free, pa_peer_export,
                   pa_peer_open, pa_peer_close, pa_hash_blocked_release, pa_blocked_plan)

ROUTES = {"auto": PA_ROUTE_AUTO, "transform": PA_ROUTE_TRANSFORM, "bitpacked": PA_ROUTE_BITPACKED}


def words32(nbits: int) -> int:
    return (nbits + 31) // 32


def _nbits(t: torch.Tensor) -> int:
    return t.numel() * t.element_size() * 8


def _stream_ptr(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _need_cuda(t: torch.Tensor, name: str, nbits: int) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (use Hasher.hash_host for host buffers)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if _nbits(t) < nbits:
        raise ValueError(f"{name} holds {_nbits(t)} bits, {nbits} required")


def make_options(route: str = "auto", seed_bit_offset: int = 0, allow_wide: bool = False, batch_keys: int = 0,
                 max_transform_len: int = 0, device: int = -1, arith: int = PA_ARITH_AUTO, plan: str = "model"):
    """pa_options from keyword arguments (see include/pa.h for each field); plan = "model" or
    "measure" (PA_PLAN_MEASURE: time the planner's best candidates at create)."""
    opt = pa_options_init()
    opt.plan_mode = {"model": PA_PLAN_MODEL, "measure": PA_PLAN_MEASURE}[plan]
    opt.device = int(device)
    opt.arith = int(arith)
    opt.route = ROUTES[route]
    opt.seed_bit_offset = int(seed_bit_offset)
    opt.allow_wide = 1 if allow_wide else 0
    opt.batch_keys = int(batch_keys)
    opt.max_transform_len = int(max_transform_len)
    return opt


def workspace_size(n: int, m: int, **options) -> int:
    """Device bytes a Hasher(n, m, ..., workspace=...) needs (pa_workspace_size)."""
    return pa_workspace_size(int(n), int(m), make_options(**options))


def seed_from_paper_eq1(t_words: torch.Tensor, n: int, m: int, out: torch.Tensor | None = None,
                        stream=None) -> torch.Tensor:
    """Eq. (1)-ordered seed t -> this library's diagonal order (pa_seed_from_paper_eq1)."""
    L = n + m - 1
    _need_cuda(t_words, "t_words", L)
    if out is None:
        out = torch.empty(((words32(L) + 3) // 4 * 4,), dtype=torch.int32, device=t_words.device)
    _need_cuda(out, "out", L)
    with torch.cuda.device(t_words.device):
        pa_seed_from_paper_eq1(out.data_ptr(), t_words.data_ptr(), int(n), int(m), _stream_ptr(stream))
    return out


class Hasher:
    """One pa_handle: fixed (n, m, seed); hash any number of n-bit keys.

    workspace: optional CUDA tensor (>= workspace_size(n, m, ...) bytes, 256-byte
    aligned) that holds all of the handle's device memory (pa_create_ws); the
    Hasher keeps a reference to it.  max_transform_len forces the Eq. (4)
    column split, batch_keys the keys per launch (include/pa.h pa_options)."""

    def __init__(self, n: int, m: int, seed: torch.Tensor, route: str = "auto",
                 seed_bit_offset: int = 0, stream=None, allow_wide: bool = False, batch_keys: int = 0,
                 max_transform_len: int = 0, workspace: torch.Tensor | None = None, plan: str = "model"):
        _need_cuda(seed, "seed", seed_bit_offset + n + m - 1)
        self.n, self.m = int(n), int(m)
        self.seed_bit_offset = int(seed_bit_offset)
        self.device = seed.device
        opt = make_options(route, seed_bit_offset, allow_wide, batch_keys, max_transform_len,
                           device=seed.device.index if seed.device.index is not None else -1, plan=plan)
        self._ws = workspace
        with torch.cuda.device(self.device):
            if workspace is None:
                self._h = pa_create_ex(self.n, self.m, seed.data_ptr(), opt, _stream_ptr(stream))
            else:
                if not workspace.is_cuda or not workspace.is_contiguous():
                    raise ValueError("workspace must be a contiguous CUDA tensor")
                self._h = pa_create_ws(self.n, self.m, seed.data_ptr(), opt, workspace.data_ptr(),
                                       workspace.numel() * workspace.element_size(), _stream_ptr(stream))
        self.info = pa_get_info(self._h)

    @property
    def handle(self) -> int:
        return self._h

    @property
    def route(self) -> str:
        return {PA_ROUTE_TRANSFORM: "transform", PA_ROUTE_BITPACKED: "bitpacked"}[self.info["route"]]

    def new_out(self, count: int | None = None) -> torch.Tensor:
        w = words32(self.m)
        w4 = (w + 3) // 4 * 4
        shape = (w4,) if count is None else (count, w4)
        return torch.empty(shape, dtype=torch.int32, device=self.device)

    def hash(self, key: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        _need_cuda(key, "key", self.n)
        if out is None:
            out = self.new_out()
        _need_cuda(out, "out", self.m)
        with torch.cuda.device(self.device):
            pa_hash(self._h, key.data_ptr(), out.data_ptr(), _stream_ptr(stream))
        return out

    def hash_batch(self, keys: torch.Tensor, outs: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """keys: (count, words) CUDA tensor, one key per row."""
        if keys.dim() != 2:
            raise ValueError("keys must be 2-D (count, words)")
        count = keys.shape[0]
        if outs is None:
            outs = self.new_out(count)
        _need_cuda(keys, "keys", self.n * count)
        _need_cuda(outs, "outs", self.m * count)
        kstride = keys.stride(0) * keys.element_size() // 4
        ostride = outs.stride(0) * outs.element_size() // 4
        with torch.cuda.device(self.device):
            pa_hash_batch(self._h, keys.data_ptr(), kstride, outs.data_ptr(), ostride, count,
                          _stream_ptr(stream))
        return outs

    def hash_host(self, key_host: torch.Tensor, out_host: torch.Tensor, stream=None) -> torch.Tensor:
        """End-to-end: host (preferably pinned) key in, host output words out."""
        if key_host.is_cuda or out_host.is_cuda:
            raise ValueError("hash_host takes CPU tensors")
        if _nbits(key_host) < self.n or _nbits(out_host) < 32 * words32(self.m):
            raise ValueError("host buffers too small")
        with torch.cuda.device(self.device):
            pa_hash_host(self._h, key_host.data_ptr(), out_host.data_ptr(), _stream_ptr(stream))
        return out_host

    def hash_fresh_batch(self, seeds: torch.Tensor, keys: torch.Tensor, outs: torch.Tensor | None = None,
                         stream=None) -> torch.Tensor:
        """Key k hashed with its own seed k (pa_hash_fresh_batch): seeds (count, words),
        keys (count, words).  The handle keeps the last seed."""
        if keys.dim() != 2 or seeds.dim() != 2 or seeds.shape[0] != keys.shape[0]:
            raise ValueError("seeds and keys must be 2-D with one row per key")
        count = keys.shape[0]
        if outs is None:
            outs = self.new_out(count)
        _need_cuda(keys, "keys", self.n * count)
        _need_cuda(seeds, "seeds", (self.seed_bit_offset + self.n + self.m - 1) * count)
        _need_cuda(outs, "outs", self.m * count)
        st = [t.stride(0) * t.element_size() // 4 for t in (seeds, keys, outs)]
        with torch.cuda.device(self.device):
            pa_hash_fresh_batch(self._h, seeds.data_ptr(), st[0], keys.data_ptr(), st[1], outs.data_ptr(), st[2],
                                count, _stream_ptr(stream))
        return outs

    def hash_host_batch(self, keys_host: torch.Tensor, outs_host: torch.Tensor, stream=None) -> torch.Tensor:
        """Host (pinned) keys (count, words) in, host outputs (count, words) out, one transfer each
        way and one batched hash (pa_hash_host_batch)."""
        if keys_host.is_cuda or outs_host.is_cuda or keys_host.dim() != 2 or outs_host.dim() != 2:
            raise ValueError("hash_host_batch takes 2-D CPU tensors (count, words)")
        count = keys_host.shape[0]
        if outs_host.shape[0] < count or keys_host.stride(1) != 1 or outs_host.stride(1) != 1:
            raise ValueError("outs_host needs a row per key; rows must be contiguous")
        ks = keys_host.stride(0) * keys_host.element_size() // 4
        os_ = outs_host.stride(0) * outs_host.element_size() // 4
        with torch.cuda.device(self.device):
            pa_hash_host_batch(self._h, keys_host.data_ptr(), ks, outs_host.data_ptr(), os_, count,
                               _stream_ptr(stream))
        return outs_host

    def set_seed(self, seed: torch.Tensor, stream=None) -> None:
        """Fresh seed for the next hashes (pa_set_seed; same n, m, seed_bit_offset)."""
        _need_cuda(seed, "seed", self.seed_bit_offset + self.n + self.m - 1)
        with torch.cuda.device(self.device):
            pa_set_seed(self._h, seed.data_ptr(), _stream_ptr(stream))

    def hash_host_async(self, key_host: torch.Tensor, out_host: torch.Tensor, stream=None) -> torch.Tensor:
        """As hash_host but without the final synchronisation (pinned buffers; the
        output is valid once `stream` reaches this call)."""
        if key_host.is_cuda or out_host.is_cuda:
            raise ValueError("hash_host_async takes CPU tensors")
        if _nbits(key_host) < self.n or _nbits(out_host) < 32 * words32(self.m):
            raise ValueError("host buffers too small")
        with torch.cuda.device(self.device):
            pa_hash_host_async(self._h, key_host.data_ptr(), out_host.data_ptr(), _stream_ptr(stream))
        return out_host

    def residual(self, stream=None) -> float:
        with torch.cuda.device(self.device):
            return pa_residual(self._h, _stream_ptr(stream))

    def close(self) -> None:
        if getattr(self, "_h", None):
            pa_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
