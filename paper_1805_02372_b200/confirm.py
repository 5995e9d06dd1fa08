"""Key-confirmation digest -- a step beside the hot path.

After privacy amplification Alice and Bob compare a short digest of their l-bit secret keys
to detect a mismatch without revealing key bits (the paper only says an authentication is
performed before use).  The digest is a second, independently seeded Toeplitz hash of
the secret key down to tag_bits >= 64 bits -- the same primitive (libpa kernels), so:

  * identical keys give identical digests;
  * keys differing in a set D of bits give digests differing by XOR_{j in D} (column j of
    the tag matrix) = a window of the tag seed, which is zero with probability 2^(-tag_bits)
    over the seed (GF(2) linearity): a one-bit mismatch is missed only if its
    seed window is all zeros.
"""
from __future__ import annotations

import torch

from . import Hasher

MIN_TAG_BITS = 64


def confirmation_digest(secret_key: torch.Tensor, l: int, tag_seed: torch.Tensor, tag_bits: int = 64,
                        stream=None) -> torch.Tensor:
    """tag_bits-bit digest of the l-bit key (CUDA int32 words, LSB-first), with the
    (l + tag_bits - 1)-bit tag seed; returns ceil(tag_bits/32) int32 words (padded to 4)."""
    if tag_bits < MIN_TAG_BITS:
        raise ValueError(f"tag_bits = {tag_bits}: the confirmation digest needs >= {MIN_TAG_BITS} bits (SPEC S:383)")
    with Hasher(int(l), int(tag_bits), tag_seed, allow_wide=tag_bits > l, stream=stream) as h:
        return h.hash(secret_key, stream=stream)


def digests_match(a: torch.Tensor, b: torch.Tensor, tag_bits: int = 64) -> bool:
    """Compare two digests on their tag_bits bits (host round trip: a protocol decision)."""
    w = (tag_bits + 31) // 32
    return bool(torch.equal(a.reshape(-1)[:w].cpu(), b.reshape(-1)[:w].cpu()))
