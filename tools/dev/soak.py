"""One-off soak: many random (n, m) shapes through route (a) (and (b) where cheap) vs the
oracle (full output when affordable, else sampled rows).  Prints failures; exit 1 on any."""
import os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import test_parity_gpu as T
import pa_synth as syn
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
count = int(sys.argv[1]) if len(sys.argv) > 1 else 300
bad = 0
for i in range(count):
    n = int(np.exp(rng.uniform(0, np.log(2e7))))
    m = int(rng.integers(1, n + 1)) if rng.random() < 0.7 else max(1, n // int(rng.integers(10, 10000)))
    sw = syn.random_bits(syn.seed_stream(1000 + i), n + m - 1)
    kw = syn.random_bits(syn.key_stream(1000 + i, 0), n)
    try:
        got, info = T.check(n, m, sw, kw, "transform")
        if n * m <= 2e9:
            got_b, _ = T.check(n, m, sw, kw, "bitpacked", full=False)
            assert np.array_equal(got, got_b), "routes disagree"
    except Exception as e:  # noqa: BLE001
        bad += 1
        print(f"FAIL n={n} m={m}: {str(e)[:200]}", flush=True)
print(f"soak: {count} shapes, {bad} failures", flush=True)
sys.exit(1 if bad else 0)
