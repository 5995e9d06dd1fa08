"""Quick per-config check after a kernel change: ms/hash (L2 flushed), per-kernel launch times,
sampled rows vs the oracle, FP64 residual.  Batched configs (C5x*K) use K distinct keys.

    python tools/dev/kcheck.py C2 C3 C4 C5d*32
    PA_LIB=$PWD/paper_1805_02372_b200/libpa_dev.so PA_K1P=0 python tools/dev/kcheck.py C4
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import pa_synth as syn  # noqa: E402
import paper_1805_02372_b200 as pa  # noqa: E402


def words(w):
    w = np.ascontiguousarray(w).view(np.int32)
    w = np.concatenate([w, np.zeros((-w.size) % 4, np.int32)])
    return torch.from_numpy(w.copy()).cuda()


def main(specs, iters=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for spec in specs:
        name, count = (spec.split("*") + ["1"])[:2]
        count = int(count)
        n, m, sw, kw = syn.config_inputs(name)
        h = pa.Hasher(n, m, words(sw))
        if count == 1:
            key = words(kw)
            out = h.new_out()
            fn = lambda: h.hash(key, out)  # noqa: E731
        else:
            keys = syn.random_bits_torch([syn.key_stream(syn.CONFIG_INDEX[name], k) for k in range(count)], n, "cuda")
            outs = h.new_out(count)
            fn = lambda: h.hash_batch(keys, outs)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        pa.pa_profile_enable(h.handle, True)
        pa.pa_profile_read(h.handle)
        for _ in range(5):
            flush.zero_()
            fn()
        kern = pa.pa_profile_read(h.handle)
        pa.pa_profile_enable(h.handle, False)
        torch.cuda.synchronize()
        rows = np.unique(np.concatenate([np.arange(min(m, 64)), np.arange(max(0, m - 64), m),
                                         np.random.default_rng(3).integers(0, m, 256)])).astype(np.uint64)
        if count == 1:
            got = oracle.unpack(out.cpu().numpy().view(np.uint32), m)[rows.astype(np.int64)]
            ok = np.array_equal(got, oracle.toeplitz_rows(n, m, sw, kw, rows))
        else:
            ok = True
            for k in (0, count - 1):
                kk = syn.random_bits(syn.key_stream(syn.CONFIG_INDEX[name], k), n)
                got = oracle.unpack(outs[k].cpu().numpy().view(np.uint32), m)[rows.astype(np.int64)]
                ok &= np.array_equal(got, oracle.toeplitz_rows(n, m, sw, kk, rows))
        t = float(np.median(ts)) / count
        ks = " ".join(f"{k.split('_')[0]}={v[1] / v[0] * 1e3 / count:.1f}" for k, v in kern.items())
        print(f"{spec:8s} {t * 1e3:9.2f} us/key {n / t / 1e6:7.2f} Gbit/s  [{ks}] ok={ok} resid={h.residual():.1e} "
              f"plan={h.info['n1']}x{h.info['n2']} C={h.info['cols_per_cta']}", flush=True)
        h.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3", "C4"])
