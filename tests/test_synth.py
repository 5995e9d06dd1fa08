"""pa_synth: the torch (device-side) SplitMix64 generator draws exactly the numpy streams, so
inputs generated on the GPU (bench C5 batches of 1024 distinct keys) are the ones the oracle
checks against."""
import numpy as np
import pytest
import torch

import pa_synth as syn


@pytest.mark.parametrize("nbits", [1, 31, 32, 33, 63, 64, 65, 1000, 4096, 100_003])
def test_torch_generator_matches_numpy(nbits):
    streams = [syn.key_stream(54, 3), syn.seed_stream(4), 0xFFFF_FFFF_FFFF_FFFF, 0]
    got = syn.random_bits_torch(streams, nbits, "cpu")
    assert got.shape[1] % 4 == 0
    for i, st in enumerate(streams):
        want = syn.random_bits(st, nbits).view(np.uint32)[: (nbits + 31) // 32]
        row = got[i].numpy().view(np.uint32)
        assert np.array_equal(row[: want.size], want)
        assert not row[want.size:].any()
