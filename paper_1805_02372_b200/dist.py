"""Multi-GPU partitioning of one Toeplitz hash (one process per GPU, torch.distributed).

Three exact decompositions of y = T x (Eq. (1)):

* Output-row split (BASELINE.json configs[3]): rank g owns rows [r0, r1) and its
  own handle on the seed window s[r0 : r1 + n - 1] (pa_options.seed_bit_offset
  = r0), hashes the whole key, and the m-bit result is assembled with one NCCL
  all-gather (every rank ends with all of y).
* Input-column split (the paper's Eq. (4) block division, with the
  Eq. (7) modulo-2 merge): rank g owns key bits [c0, c1) and the seed
  window s[n - c1 : n - c0 + m - 1]; partial m-bit hashes are XOR-reduced.  NCCL
  has no XOR reduction (nccl.h: Sum/Prod/Max/Min/Avg), so the merge is a
  reduce-scatter built from all_to_all_single + libpa's XOR-fold kernel, then an
  all-gather (exact, order-free).
* Independent keys (configs[4]): keys are dealt round-robin; no collective on
  the data path.

The split arithmetic (`row_ranges`, `col_ranges`, window offsets, bit packing of
shard keys) is host logic; all hashing runs in libpa on each rank's GPU.  With
the gloo backend and CPU tensors the same driver runs in CI through an injected
`hash_fn` (see tests/test_dist_cpu.py) -- never on the product path.
"""
from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

WORD = 32


def split_even(total: int, parts: int) -> list[tuple[int, int]]:
    """[a, b) ranges covering [0, total) in `parts` nearly equal contiguous pieces."""
    q, r = divmod(total, parts)
    out, a = [], 0
    for g in range(parts):
        b = a + q + (1 if g < r else 0)
        out.append((a, b))
        a = b
    return out


def row_ranges(m: int, world: int) -> list[tuple[int, int]]:
    """Output rows per rank, each a multiple of 32 except the last (word-aligned
    gather: every rank's slice starts on a uint32 boundary of y)."""
    words = (m + WORD - 1) // WORD
    out = []
    for a, b in split_even(words, world):
        out.append((min(m, a * WORD), min(m, b * WORD)))
    return out


def row_seed_offset(r0: int) -> int:
    """Row block [r0, r1) uses seed bits [r0, r1 + n - 1): T[i][j] = s[i-j+n-1]."""
    return r0


def col_ranges(n: int, m: int, world: int) -> list[tuple[int, int]]:
    """Key-bit blocks per rank (n_g may be < m: the handles use pa_options.allow_wide)."""
    return split_even(n, world)


def col_seed_offset(n: int, c0: int, c1: int) -> int:
    """Key block [c0, c1) (n_g = c1 - c0 bits) uses seed bits [n - c1, n - c0 + m - 1)."""
    return n - c1


def extract_bits(words: np.ndarray, start: int, count: int) -> np.ndarray:
    """Bits [start, start+count) of an LSB-first uint32/uint64 array, repacked into uint32
    words starting at bit 0 (host-side shard preparation)."""
    b = np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")[start:start + count]
    pad = np.zeros(((count + WORD - 1) // WORD) * WORD, np.uint8)
    pad[:count] = b
    return np.packbits(pad, bitorder="little").view(np.uint32)


def _words4(nbits: int) -> int:
    w = (nbits + WORD - 1) // WORD
    return (w + 3) // 4 * 4


class _LibpaHash:
    """hash_fn backed by libpa on this rank's GPU (the product path)."""

    def __init__(self):
        from . import Hasher
        self._Hasher = Hasher
        self._cache = {}

    def __call__(self, n, m, seed_t, seed_off, key_t):
        k = (n, m, seed_t.data_ptr(), seed_off)
        h = self._cache.get(k)
        if h is None:
            h = self._Hasher(n, m, seed_t, seed_bit_offset=seed_off, allow_wide=m > n)
            self._cache[k] = h
        return h.hash(key_t)

    def close(self):
        for h in self._cache.values():
            h.close()
        self._cache.clear()


def hash_rows(n: int, m: int, seed_t: torch.Tensor, key_t: torch.Tensor, group=None,
              hash_fn: Callable | None = None) -> torch.Tensor:
    """Output-row split: returns all ceil(m/32) words of y on every rank."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    ranges = row_ranges(m, world)
    r0, r1 = ranges[rank]
    hf = hash_fn or _LibpaHash()
    span = (ranges[0][1] - ranges[0][0]) // WORD  # words per slice (all but the last equal)
    span = max(span, max((b - a + WORD - 1) // WORD for a, b in ranges))
    mine = torch.zeros(span, dtype=torch.int32, device=key_t.device)
    if r1 > r0:
        part = hf(n, r1 - r0, seed_t, row_seed_offset(r0), key_t)
        w = (r1 - r0 + WORD - 1) // WORD
        mine[:w] = part[:w]
    gathered = torch.empty(world * span, dtype=torch.int32, device=key_t.device)
    dist.all_gather_into_tensor(gathered, mine, group=group)
    words = (m + WORD - 1) // WORD
    out = torch.zeros(words, dtype=torch.int32, device=key_t.device)
    for g, (a, b) in enumerate(ranges):
        if b > a:
            wa, wb = a // WORD, (b + WORD - 1) // WORD
            out[wa:wb] = gathered[g * span: g * span + (wb - wa)]
    if hash_fn is None:
        hf.close()
    return out


def _xor_fold_libpa(parts: torch.Tensor) -> torch.Tensor:
    """XOR of the rows of `parts` ((G, words) int32, CUDA) with libpa's k_xor_fold."""
    from . import pa_xor_fold
    G, words = parts.shape
    out = torch.empty(words, dtype=torch.int32, device=parts.device)
    pa_xor_fold(out.data_ptr(), parts.data_ptr(), words, G, parts.stride(0),
                torch.cuda.current_stream(parts.device).cuda_stream)
    return out


def _xor_fold_host(parts: torch.Tensor) -> torch.Tensor:
    """CPU tensors (gloo tests): the same fold with torch bitwise ops."""
    out = parts[0].clone()
    for g in range(1, parts.shape[0]):
        out ^= parts[g]
    return out


def hash_cols(n: int, m: int, seed_t: torch.Tensor, key_words: np.ndarray, group=None,
              hash_fn: Callable | None = None, device=None, xor_fn: Callable | None = None) -> torch.Tensor:
    """Input-column split with the Eq. (7) XOR merge; returns all ceil(m/32) words of y on
    every rank.  key_words: the full key (host, LSB-first); each rank uploads its block.

    Merge = XOR reduce-scatter + all-gather: the packed partial (words padded to a
    multiple of 4*G) is cut into G slices, one all_to_all_single sends slice g to rank g,
    rank g XOR-folds the G copies of its slice (libpa k_xor_fold), and one
    all_gather_into_tensor assembles y -- 2 * m/8 bytes per rank on the wire."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    c0, c1 = col_ranges(n, m, world)[rank]
    words = (m + WORD - 1) // WORD
    dev = device if device is not None else seed_t.device
    hf = hash_fn or _LibpaHash()
    fold = xor_fn or (_xor_fold_libpa if dev.type == "cuda" else _xor_fold_host)
    slice_w = ((words + world - 1) // world + 3) // 4 * 4
    mine = torch.zeros(world * slice_w, dtype=torch.int32, device=dev)
    if c1 > c0:
        blk = extract_bits(key_words, c0, c1 - c0)
        kt = torch.zeros(_words4(c1 - c0), dtype=torch.int32)
        kt[:blk.size] = torch.from_numpy(blk.view(np.int32))
        part = hf(c1 - c0, m, seed_t, col_seed_offset(n, c0, c1), kt.to(dev))
        mine[:words] = part[:words]
    recv = torch.empty_like(mine)
    dist.all_to_all_single(recv, mine, group=group)
    myslice = fold(recv.view(world, slice_w))
    gathered = torch.empty(world * slice_w, dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(gathered, myslice, group=group)
    if hash_fn is None:
        hf.close()
    return gathered[:words].clone()


def hash_keys(n: int, m: int, seed_t: torch.Tensor, keys: torch.Tensor, group=None,
              hash_fn: Callable | None = None) -> tuple[list[int], torch.Tensor]:
    """Independent keys: rank g hashes keys g, g+W, g+2W, ... of `keys` ((count, words)).
    Returns (indices, outputs) for this rank; no data-path collective."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    idx = list(range(rank, keys.shape[0], world))
    hf = hash_fn or _LibpaHash()
    outs = torch.zeros((len(idx), _words4(m)), dtype=torch.int32, device=keys.device)
    for i, k in enumerate(idx):
        o = hf(n, m, seed_t, 0, keys[k].contiguous())
        outs[i, :o.numel()] = o[: outs.shape[1]]
    if hash_fn is None:
        hf.close()
    return idx, outs


# ---------------------------------------------------------------- persistent sharded hashers
def _world_rank(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


class RowSplit:
    """Output-row split of one (n, m) hash (BASELINE configs[3], "output rows sharded with NCCL
    gather"): this rank owns rows row_ranges(m, W)[rank] and keeps a handle on the seed window
    at offset r0 (n + m_g - 1 bits, P:88-92 per row block); each call hashes the full key
    (device words, every rank holds it) and one all_gather_into_tensor assembles y.  Per-rank
    transform >= n + m/W - 1: it barely shrinks."""

    def __init__(self, n: int, m: int, seed_t: torch.Tensor, group=None):
        from . import Hasher
        self.n, self.m, self.group = n, m, group
        self.world, self.rank = _world_rank(group)
        self.ranges = row_ranges(m, self.world)
        r0, r1 = self.ranges[self.rank]
        self.span = max((b - a + WORD - 1) // WORD for a, b in self.ranges)
        self.h = Hasher(n, r1 - r0, seed_t, seed_bit_offset=row_seed_offset(r0), allow_wide=True) if r1 > r0 else None
        dev = seed_t.device
        self.mine = torch.zeros(self.span, dtype=torch.int32, device=dev)
        self.gathered = torch.empty(self.world * self.span, dtype=torch.int32, device=dev)
        self.out = torch.zeros((m + WORD - 1) // WORD, dtype=torch.int32, device=dev)

    def __call__(self, key_t: torch.Tensor) -> torch.Tensor:
        if self.h is not None:
            part = self.h.hash(key_t)
            w = min(self.span, part.numel())
            self.mine[:w] = part[:w]
        if self.world == 1:
            return self.mine[: self.out.numel()]
        dist.all_gather_into_tensor(self.gathered, self.mine, group=self.group)
        for g, (a, b) in enumerate(self.ranges):
            if b > a:
                wa, wb = a // WORD, (b + WORD - 1) // WORD
                self.out[wa:wb] = self.gathered[g * self.span: g * self.span + (wb - wa)]
        return self.out

    def close(self):
        if self.h is not None:
            self.h.close()


class ColSplit:
    """Input-column split (the paper's Eq. (4) key blocks, with the Eq. (7) modulo-2
    merge): this rank owns key bits col_ranges(n, m, W)[rank] -- the layout when each
    GPU already holds its own decoded key segment -- and keeps a handle on the seed
    window at offset n - c1.  Each call hashes this rank's key block (device words, see
    key_block) and merges: XOR reduce-scatter (one all_to_all_single + libpa's pa_xor_fold; NCCL
    has no XOR op) then one all_gather_into_tensor.  Per-rank transform >= n/W + m - 1."""

    def __init__(self, n: int, m: int, seed_t: torch.Tensor, group=None):
        from . import Hasher
        self.n, self.m, self.group = n, m, group
        self.world, self.rank = _world_rank(group)
        self.c0, self.c1 = col_ranges(n, m, self.world)[self.rank]
        ng = self.c1 - self.c0
        self.h = Hasher(ng, m, seed_t, seed_bit_offset=col_seed_offset(n, self.c0, self.c1),
                        allow_wide=m > ng) if ng > 0 else None
        dev = seed_t.device
        self.words = (m + WORD - 1) // WORD
        self.slice_w = ((self.words + self.world - 1) // self.world + 3) // 4 * 4
        self.mine = torch.zeros(self.world * self.slice_w, dtype=torch.int32, device=dev)
        self.recv = torch.empty_like(self.mine)
        self.gathered = torch.empty(self.world * self.slice_w, dtype=torch.int32, device=dev)

    def key_block(self, key_words: np.ndarray, device) -> torch.Tensor:
        """This rank's key bits [c0, c1) as word-aligned device words (host-side extraction)."""
        ng = self.c1 - self.c0
        blk = extract_bits(key_words, self.c0, ng)
        kt = torch.zeros(_words4(ng), dtype=torch.int32)
        kt[:blk.size] = torch.from_numpy(blk.view(np.int32))
        return kt.to(device)

    def __call__(self, key_block_t: torch.Tensor) -> torch.Tensor:
        if self.h is not None:
            part = self.h.hash(key_block_t)
            self.mine[: self.words] = part[: self.words]
        if self.world == 1:
            return self.mine[: self.words]
        dist.all_to_all_single(self.recv, self.mine, group=self.group)
        myslice = _xor_fold_libpa(self.recv.view(self.world, self.slice_w))
        dist.all_gather_into_tensor(self.gathered, myslice, group=self.group)
        return self.gathered[: self.words]

    def close(self):
        if self.h is not None:
            self.h.close()
