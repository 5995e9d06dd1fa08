"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no Toeplitz products, no
transforms, no parity).  It only draws bit strings and names the workloads,
so both ``oracle/`` and ``paper_1805_02372_b200`` consumers (tests, bench)
can feed byte-identical inputs to both sides.

Generator: SplitMix64 (Steele, Lea, Flood 2014), counter form
    state_k = stream + (k+1) * 0x9E3779B97F4A7C15   (mod 2^64)
    z = state_k; z = (z ^ (z>>30)) * 0xBF58476D1CE4E5B9
                 z = (z ^ (z>>27)) * 0x94D049BB133111EB;  word_k = z ^ (z>>31)
Words are LSB-first bit strings (bit b -> word b//64, bit b%64); bits past the
requested length are zero.  i.i.d. Bernoulli(1/2) bits are the paper's
distribution: the seed is "a uniform string" and a reconciled
key is near-uniform.  Stream ids follow SURVEY.md Sec. 8(d):
    key(c, k)  = 0x5041_0000_0000_0000 ^ (c << 32) ^ k
    seed(c)    = 0x5345_4544_0000_0000 ^ (c << 32)
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# Workloads of BASELINE.json "configs" (C1..C5).  m = floor(ratio * n); C5's
# ratio is not stated in BASELINE.json, 0.1 is the paper's.
CONFIGS = {
    "C1": dict(n=4096, m=1024, keys=1, desc="n=4096, m=1024, 5119-bit seed, single key"),
    "C2": dict(n=1_000_003, m=250_000, keys=1, desc="n=1,000,003, m/n=0.25, single B200"),
    "C3": dict(n=10_000_000, m=1_000_000, keys=1, desc="n=10^7, m/n=0.1, single B200"),
    "C4": dict(n=100_000_000, m=20_000_000, keys=1, desc="n=10^8, m/n=0.2, rows sharded"),
    "C5a": dict(n=1 << 20, m=(1 << 20) // 10, keys=1024, desc="batched, n=2^20"),
    "C5b": dict(n=3_000_000, m=300_000, keys=1024, desc="batched, n=3e6"),
    "C5c": dict(n=(1 << 24) + 17, m=((1 << 24) + 17) // 10, keys=1024, desc="batched, n=2^24+17"),
    "C5d": dict(n=50_000_000, m=5_000_000, keys=1024, desc="batched, n=5e7"),
}
CONFIG_INDEX = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5a": 51, "C5b": 52, "C5c": 53, "C5d": 54}


def key_stream(c: int, k: int = 0) -> int:
    return (0x5041_0000_0000_0000 ^ (c << 32) ^ k) & 0xFFFF_FFFF_FFFF_FFFF


def seed_stream(c: int) -> int:
    return (0x5345_4544_0000_0000 ^ (c << 32)) & 0xFFFF_FFFF_FFFF_FFFF


def splitmix64(stream: int, nwords: int, start: int = 0) -> np.ndarray:
    """nwords SplitMix64 outputs of the counter stream `stream`, from index start."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + nwords + 1, dtype=np.uint64)
        z = np.uint64(stream) + k * GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def mask_tail(words: np.ndarray, nbits: int) -> np.ndarray:
    """Zero every bit at position >= nbits (in place) and return words."""
    nw = words.size
    full = nbits // 64
    if full < nw:
        r = nbits % 64
        if r:
            words[full] &= np.uint64((1 << r) - 1)
            words[full + 1:] = 0
        else:
            words[full:] = 0
    return words


def random_bits(stream: int, nbits: int) -> np.ndarray:
    """nbits i.i.d. uniform bits, LSB-first in ceil(nbits/64) uint64 words."""
    nw = (nbits + 63) // 64
    return mask_tail(splitmix64(stream, nw), nbits)


def sparse_bits(stream: int, nbits: int, k: int) -> tuple[np.ndarray, np.ndarray]:
    """A key with k distinct set bits at seeded positions -> (words, positions)."""
    rng = np.random.default_rng(stream & 0xFFFF_FFFF)
    pos = np.sort(rng.choice(nbits, size=min(k, nbits), replace=False)).astype(np.int64)
    w = np.zeros((nbits + 63) // 64, dtype=np.uint64)
    np.bitwise_or.at(w, pos // 64, np.left_shift(np.uint64(1), (pos % 64).astype(np.uint64)))
    return w, pos


def ones_bits(nbits: int) -> np.ndarray:
    return mask_tail(np.full((nbits + 63) // 64, np.uint64(0xFFFF_FFFF_FFFF_FFFF)), nbits)


def zero_bits(nbits: int) -> np.ndarray:
    return np.zeros((nbits + 63) // 64, dtype=np.uint64)


def unit_bits(nbits: int, j: int) -> np.ndarray:
    w = zero_bits(nbits)
    w[j // 64] = np.uint64(1) << np.uint64(j % 64)
    return w


def as_u32(words64: np.ndarray) -> np.ndarray:
    """Same bits viewed as uint32 words (little-endian), no copy semantics implied."""
    return np.ascontiguousarray(words64).view(np.uint32)


def _s64(u: int) -> int:
    """A uint64 constant as the int64 with the same bits (torch has no uint64 arithmetic)."""
    return u - (1 << 64) if u >= (1 << 63) else u


def random_bits_torch(streams, nbits: int, device, words32: int | None = None):
    """The same SplitMix64 words as random_bits(stream, nbits), generated where they are used
    (e.g. on the GPU: 1024 C5d keys are 6.4 GB) with torch int64 ops (two's-complement
    wrap-around multiply, logical shifts by masking).  streams: a list of stream ids.
    Returns a (len(streams), W) int32 tensor, W = words32 or ceil(nbits/32) rounded up to a
    multiple of 4 (16-byte rows), bits past nbits zero.  No method arithmetic here either."""
    import torch
    nw64 = (nbits + 63) // 64
    nw32 = (nbits + 31) // 32
    W = words32 if words32 is not None else (nw32 + 3) // 4 * 4
    out = torch.zeros((len(streams), W), dtype=torch.int32, device=device)
    k = torch.arange(1, nw64 + 1, dtype=torch.int64, device=device)
    g, m1, m2 = _s64(int(GAMMA)), _s64(int(_M1)), _s64(int(_M2))
    st = torch.tensor([_s64(int(x) & 0xFFFF_FFFF_FFFF_FFFF) for x in streams], dtype=torch.int64, device=device)

    def lsr(z, s):  # logical shift right of int64 bits
        return (z >> s) & ((1 << (64 - s)) - 1)
    rows = max(1, (1 << 25) // max(1, nw64))  # streams per chunk (bounded temporaries)
    for i in range(0, len(streams), rows):
        z = (k * g).unsqueeze(0) + st[i:i + rows].unsqueeze(1)
        z = (z ^ lsr(z, 30)) * m1
        z = (z ^ lsr(z, 27)) * m2
        z = z ^ lsr(z, 31)
        w32 = z.view(torch.int32)[:, :nw32]
        out[i:i + rows, :nw32] = w32
    r = nbits % 32
    if r:
        out[:, nw32 - 1] &= (1 << r) - 1
    return out


def config_inputs(name: str, key_index: int = 0) -> tuple[int, int, np.ndarray, np.ndarray]:
    """(n, m, seed_words, key_words) for a named config, seeded per SURVEY 8(d)."""
    cfg = CONFIGS[name]
    c = CONFIG_INDEX[name]
    n, m = cfg["n"], cfg["m"]
    return n, m, random_bits(seed_stream(c), n + m - 1), random_bits(key_stream(c, key_index), n)
