"""Multi-GPU partitioning of one Toeplitz hash (one process per GPU, torch.distributed).

Three exact decompositions of y = T x (Eq. (1)):

* Output-row split (BASELINE.json configs[3]): rank g owns rows [r0, r1) and its
  own handle on the seed window s[r0 : r1 + n - 1] (pa_options.seed_bit_offset
  = r0), hashes the whole key (broadcast from the source rank), and the m-bit
  result is assembled with one NCCL all-gather (every rank ends with all of y).
* Input-column split (the paper's Eq. (4) block division, with the
  Eq. (7) modulo-2 merge): rank g owns key bits [c0, c1) (scattered
  from the source rank, or already resident: P:107) and the seed window
  s[n - c1 : n - c0 + m - 1]; partial m-bit hashes are XOR-reduced.  NCCL has no
  XOR reduction (nccl.h: Sum/Prod/Max/Min/Avg), so the merge is a reduce-scatter
  built from all_to_all_single + libpa's XOR-fold kernel, then an all-gather -- or,
  fused (ColSplit(fused=True)), K3 leaves each partial in a
  peer-mappable buffer and one kernel (pa_xor_fold_peers) folds this rank's slice
  of every partial straight from the peers' memory over NVLink, then an all-gather.
* Independent keys (configs[4]): keys are dealt round-robin, hashed in batches
  (pa_hash_batch); no collective on the data path.

`choose_split` is the cost model that picks the row or the column split for one
key: per-GPU transform length (rows: n + m/G - 1, cols: n/G + m - 1) against the
merge traffic (rows: one all-gather of m/8 bytes; cols: reduce-scatter +
all-gather).  At C4 (n = 10^8, m = 2*10^7) it picks the column split for G >= 2.

The split arithmetic (`row_ranges`, `col_ranges`, window offsets, key blocks) is
host logic; all hashing runs in libpa on each rank's GPU.  With the gloo backend
and CPU tensors the same classes run in CI through an injected hash factory (see
tests/test_dist_cpu.py: the CPU oracle) -- never on the product path.
"""
from __future__ import annotations

import math
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

WORD = 32
COL_ALIGN = 128  # key blocks start on 16-byte boundaries of the packed key (no bit shifting)


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
    return [(min(m, a * WORD), min(m, b * WORD)) for a, b in split_even(words, world)]


def row_seed_offset(r0: int) -> int:
    """Row block [r0, r1) uses seed bits [r0, r1 + n - 1): T[i][j] = s[i-j+n-1]."""
    return r0


def col_ranges(n: int, m: int, world: int, align: int = COL_ALIGN) -> list[tuple[int, int]]:
    """Key-bit blocks per rank, starting at multiples of `align` bits (n_g may be < m: the
    handles use pa_options.allow_wide; trailing ranks may be empty when n < world * align)."""
    units = (n + align - 1) // align
    return [(min(n, a * align), min(n, b * align)) for a, b in split_even(units, world)]


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


def _world_rank(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


# ---------------------------------------------------------------- cost model
def choose_split(n: int, m: int, world: int, ns_per_point: float = 0.0196, link_gbs: float = 300.0,
                 coll_us: float = 20.0) -> str:
    """'rows' or 'cols' for one (n, m) key over `world` GPUs: modelled step time =
    per-GPU transform (ns_per_point x real length, the measured C4 rate) + merge (bytes over
    NVLink + a fixed latency per collective).  world == 1 -> 'rows' (no split)."""
    if world <= 1:
        return "rows"
    ybytes = m / 8.0
    t_rows = ns_per_point * (n + math.ceil(m / world) - 1) * 1e-3 + coll_us + ybytes / link_gbs * 1e-3
    t_cols = (ns_per_point * (math.ceil(n / world) + m - 1) * 1e-3 + 2 * coll_us
              + 2 * ybytes / link_gbs * 1e-3)
    return "cols" if t_cols < t_rows else "rows"


# ---------------------------------------------------------------- hash factories
class LibpaFactory:
    """Per-shard handles from libpa on this rank's GPU (the product path)."""

    def __call__(self, n, m, seed_t, seed_off, allow_wide):
        from . import Hasher
        return Hasher(n, m, seed_t, seed_bit_offset=seed_off, allow_wide=allow_wide)


class FnFactory:
    """Wraps a plain hash_fn(n, m, seed_t, seed_off, key_t) -> words (test injection)."""

    class _H:
        def __init__(self, fn, n, m, seed_t, seed_off):
            self.fn, self.n, self.m, self.seed_t, self.seed_off = fn, n, m, seed_t, seed_off

        def hash(self, key_t):
            return self.fn(self.n, self.m, self.seed_t, self.seed_off, key_t)

        def close(self):
            pass

    def __init__(self, fn: Callable):
        self.fn = fn

    def __call__(self, n, m, seed_t, seed_off, allow_wide):
        return FnFactory._H(self.fn, n, m, seed_t, seed_off)


def _factory(factory=None, hash_fn=None):
    if factory is not None:
        return factory
    return FnFactory(hash_fn) if hash_fn is not None else LibpaFactory()


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


def distribute_seed(seed_t: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Create-time seed distribution: the source rank's seed words are broadcast in place
    (every shard window is a slice of them; the seed is bound once)."""
    w, _ = _world_rank(group)
    if w > 1:
        dist.broadcast(seed_t, src, group=group)
    return seed_t


# ---------------------------------------------------------------- persistent sharded hashers
class RowSplit:
    """Output-row split of one (n, m) hash (BASELINE configs[3], "output rows sharded with NCCL
    gather"): this rank owns rows row_ranges(m, W)[rank] and keeps a handle on the seed window
    at offset r0 (n + m_g - 1 bits, P:88-92 per row block); each call hashes the full key
    (device words; with src set it is first broadcast from rank src) and one
    all_gather_into_tensor assembles y.  Per-rank transform >= n + m/W - 1."""

    def __init__(self, n: int, m: int, seed_t: torch.Tensor, group=None, factory=None, hash_fn=None):
        self.n, self.m, self.group = n, m, group
        self.world, self.rank = _world_rank(group)
        self.ranges = row_ranges(m, self.world)
        r0, r1 = self.ranges[self.rank]
        self.span = max((b - a + WORD - 1) // WORD for a, b in self.ranges)
        fac = _factory(factory, hash_fn)
        self.h = fac(n, r1 - r0, seed_t, row_seed_offset(r0), True) if r1 > r0 else None
        dev = seed_t.device
        self.mine = torch.zeros(self.span, dtype=torch.int32, device=dev)
        self.gathered = torch.empty(self.world * self.span, dtype=torch.int32, device=dev)
        self.out = torch.zeros((m + WORD - 1) // WORD, dtype=torch.int32, device=dev)

    def __call__(self, key_t: torch.Tensor, src: int | None = None) -> torch.Tensor:
        if src is not None and self.world > 1:
            dist.broadcast(key_t, src, group=self.group)  # every rank hashes the whole key
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
    merge): this rank owns key bits col_ranges(n, m, W)[rank] (128-bit aligned) -- the
    layout when each GPU already holds its own decoded key segment, or scattered from a
    source rank each step (scatter_key) -- and keeps a handle on the seed window at offset
    n - c1.  Each call hashes this rank's key block and merges: XOR reduce-scatter (one
    all_to_all_single + an XOR fold; NCCL has no XOR op) then one all_gather_into_tensor.
    Per-rank transform >= n/W + m - 1."""

    def __init__(self, n: int, m: int, seed_t: torch.Tensor, group=None, factory=None, hash_fn=None,
                 xor_fn: Callable | None = None, fused: bool = False):
        self.n, self.m, self.group = n, m, group
        self.fused = fused
        self.world, self.rank = _world_rank(group)
        self.ranges = col_ranges(n, m, self.world)
        self.c0, self.c1 = self.ranges[self.rank]
        ng = self.c1 - self.c0
        fac = _factory(factory, hash_fn)
        self.h = fac(ng, m, seed_t, col_seed_offset(n, self.c0, self.c1), m > ng) if ng > 0 else None
        dev = seed_t.device
        self.device = dev
        self.fold = xor_fn or (_xor_fold_libpa if dev.type == "cuda" else _xor_fold_host)
        self.words = (m + WORD - 1) // WORD
        self.slice_w = ((self.words + self.world - 1) // self.world + 3) // 4 * 4
        self.mine = torch.zeros(self.world * self.slice_w, dtype=torch.int32, device=dev)
        self.recv = torch.empty_like(self.mine)
        self.gathered = torch.empty(self.world * self.slice_w, dtype=torch.int32, device=dev)
        # key scatter: equal chunks of blk_w words (the widest block), block g at word c0_g / 32
        self.blk_w = max(_words4(b - a) for a, b in self.ranges)
        self.blk = torch.zeros(self.blk_w, dtype=torch.int32, device=dev)
        self._opened, self.part_ptr = [], None
        if fused:
            self._setup_peers(dev)

    def _setup_peers(self, dev):
        """Fused merge: this rank's partial lives in a peer-mappable buffer
        (pa_peer_alloc); the buffers' IPC handles are exchanged once (all_gather_object) and the
        peers' partials mapped (pa_peer_open), so the Eq. (7) fold reads them over NVLink."""
        from . import pa_peer_alloc, pa_peer_export, pa_peer_open
        if self.h is None or not hasattr(self.h, "handle"):
            raise ValueError("the fused column split needs libpa handles on CUDA devices")
        self.part_ptr = pa_peer_alloc(4 * self.world * self.slice_w)
        handles = [None] * self.world
        mine = pa_peer_export(self.part_ptr)
        if self.world > 1:
            dist.all_gather_object(handles, mine, group=self.group)
        else:
            handles = [mine]
        ptrs, err = [], None
        try:
            for g, hd in enumerate(handles):
                if g == self.rank:
                    ptrs.append(self.part_ptr)
                else:
                    p = pa_peer_open(hd)
                    self._opened.append(p)
                    ptrs.append(p)
        except Exception as e:  # noqa: BLE001 - any mapping failure: every rank falls back together
            err = e
        if self.world > 1:
            # all ranks agree on the merge: one rank that cannot map a peer's partial must not leave
            # the others waiting in a collective the fused path would enter
            ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
            agreed = bool(ok.item())
        else:
            agreed = err is None
        if not agreed:
            import warnings
            warnings.warn(f"fused column split unavailable ({err or 'a peer could not map'}): NCCL merge")
            self._release_peers()
            self.fused = False
            return
        self.ptrs_dev = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        self.myslice = torch.zeros(self.slice_w, dtype=torch.int32, device=dev)
        self.tick = torch.zeros(1, dtype=torch.float32, device=dev)
        self.valid = max(0, min(self.slice_w, self.words - self.rank * self.slice_w))

    def _fused_call(self, key_block_t: torch.Tensor) -> torch.Tensor:
        """K3 leaves this rank's partial in its peer-visible buffer; one stream-ordered barrier
        (a one-element NCCL all-reduce); pa_xor_fold_peers folds this rank's slice of all G
        partials straight from the peers' memory (the reduce-scatter and the XOR in one kernel);
        one all-gather of the slices.  The all-gather also orders the next step's hash (which
        rewrites the partial) after every peer's fold."""
        from . import _lib
        st = torch.cuda.current_stream(self.device).cuda_stream
        _lib.pa_hash(self.h.handle, key_block_t.data_ptr(), self.part_ptr, st)
        if self.world > 1:
            dist.all_reduce(self.tick, group=self.group)
        if self.valid:
            _lib.pa_xor_fold_peers(self.myslice.data_ptr(), self.ptrs_dev.data_ptr(), self.world,
                                   self.rank * self.slice_w, self.valid, st)
        if self.world == 1:
            return self.myslice[: self.words]
        dist.all_gather_into_tensor(self.gathered, self.myslice, group=self.group)
        return self.gathered[: self.words]

    def key_block(self, key_words: np.ndarray, device) -> torch.Tensor:
        """This rank's key bits [c0, c1) as device words (host-side extraction)."""
        ng = self.c1 - self.c0
        blk = extract_bits(key_words, self.c0, ng)
        kt = torch.zeros(max(4, _words4(ng)), dtype=torch.int32)
        kt[:blk.size] = torch.from_numpy(blk.view(np.int32))
        return kt.to(device)

    def scatter_key(self, key_t: torch.Tensor | None, src: int = 0) -> torch.Tensor:
        """Per-step key distribution for the column split: rank src holds the whole key (device
        words, >= ceil(n/32)); every rank receives its block (blocks start on 128-bit
        boundaries, so a block is a word slice; bits past c1 are ignored by the handle)."""
        if self.world == 1:
            return key_t
        chunks = None
        if self.rank == src:
            chunks = []
            for a, b in self.ranges:
                c = torch.zeros(self.blk_w, dtype=torch.int32, device=self.device)
                if b > a:
                    wa, wb = a // WORD, min(key_t.numel(), (b + WORD - 1) // WORD)
                    c[: wb - wa] = key_t[wa:wb]
                chunks.append(c)
        dist.scatter(self.blk, chunks, src=src, group=self.group)
        return self.blk

    def __call__(self, key_block_t: torch.Tensor) -> torch.Tensor:
        if self.fused:
            return self._fused_call(key_block_t)
        if self.h is not None:
            part = self.h.hash(key_block_t)
            self.mine[: self.words] = part[: self.words]
        if self.world == 1:
            return self.mine[: self.words]
        dist.all_to_all_single(self.recv, self.mine, group=self.group)
        myslice = self.fold(self.recv.view(self.world, self.slice_w))
        dist.all_gather_into_tensor(self.gathered, myslice, group=self.group)
        return self.gathered[: self.words]

    def _release_peers(self):
        """Unmap the peers' partials and free this rank's (local only: no collective)."""
        from . import pa_peer_close, pa_peer_free
        for p in self._opened:
            pa_peer_close(p)
        if self.part_ptr:
            pa_peer_free(self.part_ptr)
        self._opened, self.part_ptr = [], None

    def close(self):
        if self._opened or self.part_ptr:
            torch.cuda.synchronize(self.device)
            if self.world > 1:
                dist.barrier(group=self.group)  # no peer still reads this rank's partial
            self._release_peers()
        if self.h is not None:
            self.h.close()


class KeyDeal:
    """Independent keys (BASELINE configs[4]): this rank hashes keys rank, rank + W, ... of a
    batch in one pa_hash_batch (shared seed spectrum per GPU); no data-path collective."""

    def __init__(self, n: int, m: int, seed_t: torch.Tensor, group=None, factory=None, hash_fn=None):
        self.n, self.m = n, m
        self.world, self.rank = _world_rank(group)
        self.h = _factory(factory, hash_fn)(n, m, seed_t, 0, False)

    def indices(self, count: int) -> list[int]:
        return list(range(self.rank, count, self.world))

    def __call__(self, keys: torch.Tensor, outs: torch.Tensor | None = None) -> torch.Tensor:
        """keys: this rank's keys, (count_mine, words) -- already dealt."""
        if hasattr(self.h, "hash_batch"):
            return self.h.hash_batch(keys, outs)
        res = torch.zeros((keys.shape[0], _words4(self.m)), dtype=torch.int32, device=keys.device)
        for i in range(keys.shape[0]):
            o = self.h.hash(keys[i].contiguous())
            res[i, :min(o.numel(), res.shape[1])] = o[: res.shape[1]]
        return res

    def close(self):
        self.h.close()


# ---------------------------------------------------------------- one-shot entry points
def hash_rows(n: int, m: int, seed_t: torch.Tensor, key_t: torch.Tensor, group=None,
              hash_fn: Callable | None = None, factory=None, src: int | None = None) -> torch.Tensor:
    """Output-row split: returns all ceil(m/32) words of y on every rank."""
    sh = RowSplit(n, m, seed_t, group, factory, hash_fn)
    try:
        return sh(key_t, src).clone()
    finally:
        sh.close()


def hash_cols(n: int, m: int, seed_t: torch.Tensor, key_words: np.ndarray | None, group=None,
              hash_fn: Callable | None = None, device=None, xor_fn: Callable | None = None, factory=None,
              key_t: torch.Tensor | None = None, src: int | None = None) -> torch.Tensor:
    """Input-column split with the Eq. (7) XOR merge; returns all ceil(m/32) words of y on
    every rank.  The key block comes from key_words (the full key on the host, each rank
    extracts its block) or, with src set, is scattered from rank src's device key_t."""
    dev = device if device is not None else seed_t.device
    sh = ColSplit(n, m, seed_t, group, factory, hash_fn, xor_fn)
    try:
        blk = sh.scatter_key(key_t, src) if src is not None else sh.key_block(key_words, dev)
        return sh(blk).clone()
    finally:
        sh.close()


def hash_keys(n: int, m: int, seed_t: torch.Tensor, keys: torch.Tensor, group=None,
              hash_fn: Callable | None = None, factory=None) -> tuple[list[int], torch.Tensor]:
    """Independent keys: rank g hashes keys g, g+W, g+2W, ... of `keys` ((count, words)) as one
    batch.  Returns (indices, outputs) for this rank; no data-path collective."""
    kd = KeyDeal(n, m, seed_t, group, factory, hash_fn)
    try:
        idx = kd.indices(keys.shape[0])
        if not idx:
            return idx, torch.zeros((0, _words4(m)), dtype=torch.int32, device=keys.device)
        return idx, kd(keys[idx].contiguous())
    finally:
        kd.close()


def hash(n: int, m: int, seed_t: torch.Tensor, key_t: torch.Tensor, group=None, split: str = "auto",
         src: int = 0, factory=None, hash_fn: Callable | None = None, xor_fn: Callable | None = None,
         fused: bool = False):
    """One key over all ranks of `group`, the split chosen by choose_split (or forced):
    rank src holds the key (device words); returns (split, y words) on every rank."""
    world, _ = _world_rank(group)
    if split == "auto":
        split = choose_split(n, m, world)
    if split == "rows":
        return split, hash_rows(n, m, seed_t, key_t, group, hash_fn, factory, src=src)
    if fused:
        sh = ColSplit(n, m, seed_t, group, factory, hash_fn, xor_fn, fused=True)
        try:
            return split, sh(sh.scatter_key(key_t, src)).clone()
        finally:
            sh.close()
    return split, hash_cols(n, m, seed_t, None, group, hash_fn, key_t.device, xor_fn, factory,
                            key_t=key_t, src=src)
