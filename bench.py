#!/usr/bin/env python
"""bench.py -- Toeplitz privacy-amplification throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]
                    [--split rows|cols|auto] [--no-sweep] [--no-cpu] [--selftest-cpu]

One step = one pass of the whole hot path (pa_hash: y = T x over GF(2), every kernel of
route (a)) over one synthetic n-bit key against a seed bound at pa_create, inputs resident
in HBM.  Workload: BASELINE.json configs[3], C4 (n = 10^8 key bits, m = 2*10^7 output bits,
m/n = 0.2), the largest configuration that fits one GPU; at N = 1 it is the G = 1 point of
its 1/2/4/8 curve.  For N > 1 (one process per GPU; the driver's torchrun, or --gpus N
re-executes this script under torch.distributed.run) the same key is split across the ranks
by output rows as configured ("output rows sharded ... with NCCL gather", --split rows; the
column split and the cost-model choice are measured beside it), and the C5 batches are
dealt across the ranks (keys pre-distributed, no collective).

Timing: W untimed warm-up steps, then K steps, each timed with CUDA events on the launching
stream; before every step a 256 MiB buffer (> the 126 MB L2) is zeroed outside the events
(the C4 working set, 2 GB, exceeds L2 anyway).  value = n * keys / sum of step times
(decimal Gbit/s of input key), max over ranks.  A second pass of K steps with libpa's
per-launch event profiling gives each kernel's launch time behind `roofline`.  `e2e` is
the same metric through the public API with host buffers (pinned key in, host output out,
copies inside the timed region).  `cpu_baseline` is the CPU oracle (oracle/, OpenMP) on a
bounded sample of the same workload, all host cores and one core.  --impl reference times
that oracle as the reference arm.  --selftest-cpu runs the multi-rank plumbing (gloo, the
CPU oracle injected as the per-rank hash) and prints a check line -- not a measurement.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import pa_synth as syn  # noqa: E402

METRIC = "PA throughput, input Gbit/s vs input length n, 1/2/4/8 B200; % of HBM roofline"
FLUSH_BYTES = 256 << 20
C5_KEYS = 1024


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(syn.CONFIGS),
                    help="headline workload (default C4, BASELINE configs[3])")
    ap.add_argument("--split", default="rows", choices=["rows", "cols", "auto"],
                    help="N > 1: how the key is split (rows = configured; auto = dist.choose_split)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the other-config side measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-oracle baseline")
    ap.add_argument("--side-smoke", action="store_true",
                    help="N = 1: also run the N > 1 side measurements (splits, fused merge, key dealing) "
                         "over a one-rank NCCL group -- a code-path check, not a scaling number")
    ap.add_argument("--selftest-cpu", action="store_true",
                    help="multi-rank plumbing check on CPU (gloo, oracle as the per-rank hash)")
    return ap.parse_args()


def config_dict(name, n, m):
    """The workload, identical in both arms' lines (the driver compares them)."""
    return {"workload": workload_desc(name), "n": n, "m": m,
            "l2": "GPU arm: L2 flushed before every timed step (256 MiB memset, untimed) and the C4 "
                  "working set (2 GB) exceeds L2"}


def workload_desc(name):
    c = syn.CONFIGS[name]
    return f"{name}: {c['desc']} (n={c['n']}, m={c['m']})"


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def respawn(args):
    """--gpus N without a torchrun environment: run N ranks of this script under
    torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML while the timed region runs."""
    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks",
            0x10: "sync_boost", 0x1: "gpu_idle"}

    def __init__(self, torch_device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(torch_device).uuid)
            try:
                self._h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU-") else uuid)
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(torch_device)
            self._nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.error = repr(e)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for b, name in self.BITS.items():
                    if r & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._h is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._h is not None:
            self._t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- helpers
def peak_hbm():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_kernel(config, kernel):
    """The committed `ncu --set full` summary of `kernel` (profiles/ncu_<config>.json)."""
    path = os.path.join(ROOT, "profiles", f"ncu_{config}.json")

    def base(name):  # k2_rows_t<16, 16> / k1p_fwd_columns<3, 8, 0> -> k2_rows / k1_fwd_columns
        name = name.split("<", 1)[0].strip()
        name = name[:-2] if name.endswith("_t") else name
        return {"k1p_fwd_columns": "k1_fwd_columns"}.get(name, name)
    try:
        for d in json.load(open(path)):
            if base(d.get("kernel", "")) == kernel:
                return d
    except Exception:
        pass
    return None


def alg_bytes(kernel, info):
    """Algorithmic HBM bytes of one launch (DESIGN.md Sec. 5 / SURVEY 8(d)), M = n1 * n2 complex
    doubles (16 bytes each) per key."""
    M = info["n1"] * info["n2"]
    n, m = info["n"], info["m"]
    return {"k0_bits_transpose": n / 8.0 + M / 4.0,          # key bits in, 2M bits of streams out
            "k1_fwd_columns": M / 4.0 + 16 * M,             # bit streams in, work array out
            "k2_rows": 48 * M,                              # row in, spectrum in, row out
            "k3_inv_columns": 16 * M + m / 8.0}.get(kernel)  # work array in, output bits out


def hash_bytes(n, m, M):
    """SURVEY 8(d) route (a) FP64 model per hash: 40 N + (n+m)/8 bytes, N = 2M real points."""
    return 80.0 * M + (n + m) / 8.0


def dev_words(torch, w64, device):
    w = np.ascontiguousarray(w64).view(np.int32)
    pad = (-w.size) % 4
    if pad:
        w = np.concatenate([w, np.zeros(pad, np.int32)])
    return torch.from_numpy(w.copy()).to(device)


def time_steps(torch, fn, steps, flush, stream=None):
    """Per-step CUDA-event times (ms) on the launching stream, L2 flushed before each step."""
    st = stream or torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for e0, e1 in ev:
        flush.zero_()
        e0.record(st)
        fn()
        e1.record(st)
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) for e0, e1 in ev]


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores():
    """Logical CPUs this process may run on (torchrun sets OMP_NUM_THREADS=1; the oracle's
    thread count is passed explicitly instead)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def sampled_rows(m, k=128, seed=1):
    return np.unique(np.concatenate([np.arange(min(m, 32)), np.arange(max(0, m - 32), m),
                                     np.random.default_rng(seed).integers(0, m, k)])).astype(np.uint64)


def verify_rows(n, m, seed_w, key_w, out_words_np, rows):
    import oracle
    got = oracle.unpack(out_words_np.view(np.uint32), m)[rows.astype(np.int64)]
    return bool(np.array_equal(got, oracle.toeplitz_rows(n, m, seed_w, key_w, rows)))


def roofline(kern, info, name, steps_per_launch=1):
    """Per-kernel roofline from libpa's per-launch event times: achieved = algorithmic bytes per
    launch / average launch time vs the measured HBM copy bandwidth; `traffic` = ncu DRAM bytes
    of that kernel (committed capture profiles/ncu_<config>.json)."""
    peak, peak_src = peak_hbm()
    per = {k: v[1] / max(1, v[0]) for k, v in kern.items()}  # ms per launch
    if not per:
        return None
    kernels = {}
    for k, t in per.items():
        b = alg_bytes(k, info)
        nk = ncu_kernel(name, k) or {}
        tr = (float(nk["dram_read"] + nk["dram_write"]) * 1e9) if nk else None
        kernels[k] = {"avg_launch_us": t * 1e3, "alg_bytes_per_launch": b,
                      "achieved": (b / (t * 1e-3) / 1e9) if b else None,
                      "frac": (b / (t * 1e-3) / 1e9 / peak) if b else None, "traffic": tr,
                      "fp64_pipe_frac_ncu": (nk.get("fp64_pipe_pct") or 0) / 100 or None,
                      "issue_active_frac_ncu": (nk.get("issue_pct") or 0) / 100 or None}
    top = max(per, key=per.get)
    if top == "k_toeplitz_bitpacked":
        bp = float(info["n"]) * info["m"]
        achieved = bp / (per[top] * 1e-3) / 1e12
        alu_peak = 1024 * 148 * 1965e6 / 1e12
        return {"kernel": top, "bound": "alu", "achieved": achieved, "peak": alu_peak,
                "unit": "Tbit-products/s", "frac": achieved / alu_peak, "traffic": None,
                "peak_source": "derived (DESIGN.md Sec. 6): 148 SMs x 64 ALU lanes/clk x 16 bit-products "
                               "per op (SHF + LOP3 per 32) x 1.965 GHz", "kernels": kernels}
    k = kernels[top]
    M = info["n1"] * info["n2"]
    tot_ms = sum(per.values())
    hb = hash_bytes(info["n"], info["m"], M)
    return {"kernel": top, "bound": "hbm", "achieved": k["achieved"], "peak": peak, "unit": "GB/s",
            "frac": k["frac"], "traffic": k["traffic"], "alg_bytes_per_launch": k["alg_bytes_per_launch"],
            "avg_launch_us": k["avg_launch_us"], "peak_source": peak_src, "kernels": kernels,
            "whole_hash": {"alg_bytes": hb, "sum_launch_us": tot_ms * 1e3,
                           "achieved": hb / (tot_ms * 1e-3) / 1e9, "frac": hb / (tot_ms * 1e-3) / 1e9 / peak},
            "note": "achieved = algorithmic HBM bytes (SURVEY 8(d): K1 16M+M/4, K2 48M, K3 16M+m/8 per key, "
                    "M complex points) / CUDA-event launch time (libpa pa_profile, events on the launch "
                    "stream) vs the measured copy bandwidth; fp64/issue fractions from the committed ncu "
                    "capture (DESIGN.md Sec. 9)"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1805_02372_b200 as pa
    from paper_1805_02372_b200 import dist as pd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    elif args.side_smoke:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    name = args.config
    n, m, sw, kw = syn.config_inputs(name)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    seed_t = dev_words(torch, sw, dev)
    key = dev_words(torch, kw, dev)  # resident on every rank (the device-timed value)
    split = "none" if world == 1 else (pd.choose_split(n, m, world) if args.split == "auto" else args.split)
    res = {}
    if world == 1:
        h = pa.Hasher(n, m, seed_t)
        out = h.new_out()
        res["out"] = out

        def step():
            h.hash(key, out)
        sh = None
    else:
        sh = pd.RowSplit(n, m, seed_t) if split == "rows" else pd.ColSplit(n, m, seed_t)
        blk = key if split == "rows" else sh.key_block(kw, dev)
        h = sh.h

        def step():
            res["out"] = sh(blk)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = time_steps(torch, step, args.steps, flush)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tot_ms = float(sum(ms))
    verified = None
    if rank == 0:
        verified = verify_rows(n, m, sw, kw, res["out"].cpu().numpy(), sampled_rows(m, 256))

    # profiled pass: per-kernel CUDA-event times of the same K steps (rank 0's handle)
    kern = {}
    if h is not None:
        pa.pa_profile_enable(h.handle, True)
        pa.pa_profile_read(h.handle)
        time_steps(torch, step, args.steps, flush)
        kern = pa.pa_profile_read(h.handle)
        pa.pa_profile_enable(h.handle, False)

    # end to end through the public API with host buffers: every step copies the key from
    # pinned host memory and reads the output back.  N = 1: pa_hash_host_async (one CUDA graph:
    # pinned key -> copy kernel -> K0..K3 -> copy kernel -> pinned output).  N > 1: rank 0's
    # pinned key H2D, broadcast (row split) / scatter (column split) to the ranks, the sharded
    # hash with its collectives, y D2H on rank 0.
    out_h = torch.empty(pa.words32(m), dtype=torch.int32).pin_memory()
    key_h = torch.from_numpy(np.ascontiguousarray(kw).view(np.int32).copy()).pin_memory()
    e2e_steps = max(3, min(args.steps, 50))
    if world == 1:
        e2e_fn = lambda: h.hash_host_async(key_h, out_h)  # noqa: E731
        h2d = 4 * key_h.numel()
    else:
        src_key = torch.zeros_like(key)

        def e2e_fn():
            if rank == 0:
                src_key[: key_h.numel()].copy_(key_h, non_blocking=True)
            if split == "rows":
                y = sh(src_key, src=0)
            else:
                y = sh(sh.scatter_key(src_key if rank == 0 else None, src=0))
            if rank == 0:
                out_h.copy_(y[: out_h.numel()], non_blocking=True)
        h2d = 4 * key_h.numel()
    for _ in range(3):
        e2e_fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = time_steps(torch, e2e_fn, e2e_steps, flush)
    e2e_ok = None
    if rank == 0:
        e2e_ok = bool(np.array_equal(out_h.numpy().view(np.uint32),
                                     res["out"].cpu().numpy().view(np.uint32)[: out_h.numel()]))
    # streaming end to end (N = 1): E distinct keys in pinned host memory through one
    # pa_hash_host_batch call -- every key's H2D and every output's D2H inside the timed region,
    # the copies of neighbouring chunks on the copy engines under the hashes
    stream_e2e = None
    if world == 1:
        E = max(4, min(args.steps, 16))
        c = syn.CONFIG_INDEX[name]
        kw4 = (pa.words32(n) + 3) // 4 * 4
        keys_h = torch.zeros((E, kw4), dtype=torch.int32)
        for k in range(E):
            keys_h[k, : pa.words32(n)] = torch.from_numpy(
                syn.random_bits(syn.key_stream(c, 1000 + k), n).view(np.int32)[: pa.words32(n)])
        keys_h = keys_h.pin_memory()
        outs_h = torch.zeros((E, pa.words32(m)), dtype=torch.int32).pin_memory()
        h.hash_host_batch(keys_h, outs_h)
        torch.cuda.synchronize()
        st_ms = float(np.mean(time_steps(torch, lambda: h.hash_host_batch(keys_h, outs_h), 2, flush)))
        kE = syn.random_bits(syn.key_stream(c, 1000 + E - 1), n)
        stream_e2e = {"keys": E, "ms_per_key": st_ms / E, "value": n * E / (st_ms * 1e-3) / 1e9,
                      "verified_rows": verify_rows(n, m, sw, kE, outs_h[E - 1].numpy(), sampled_rows(m, 64))}
        del keys_h, outs_h

    # N > 1: the other split and the cost model's choice, and C5 key dealing, same protocol
    side = {}
    if world > 1 or args.side_smoke:
        try:
            side = multi_gpu_side(args, torch, dist, pa, pd, dev, rank, world, flush,
                                  split if world > 1 else "cols", name)
        except Exception as e:  # noqa: BLE001 - the headline above stands; report the side failure
            side = {"error": f"{type(e).__name__}: {e}"[:300]}

    t = torch.tensor([tot_ms, float(np.mean(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, e2e_mean = float(t[0]), float(t[1])

    line = None
    if rank == 0:
        info = h.info
        value = n * args.steps / (tot_ms * 1e-3) / 1e9
        roof = roofline(kern, info, name)
        parallelism = {
            "none": "one key on 1 GPU (the G = 1 point of the configured 1/2/4/8 curve)",
            "rows": f"one key, output rows split over {world} GPUs (configured): per-rank seed window at "
                    "offset r0, NCCL all_gather_into_tensor",
            "cols": f"one key, Eq. (4) key blocks over {world} GPUs: XOR reduce-scatter (all_to_all_single "
                    "+ pa_xor_fold) + all_gather"}[split]
        line = {
            "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None,
            "dtype": "f64" if info["route"] == 1 else "u32",
            "data": "synthetic: SplitMix64 i.i.d. Bernoulli(1/2) key and seed bits (SURVEY 8(d) streams)",
            # config: the same keys as the reference arm's line (the workload); how it ran is in
            # "plan" / "parallelism"
            "config": config_dict(name, n, m),
            "plan": {"route": h.route, "transform_len": info["transform_len"], "n1": info["n1"], "n2": info["n2"],
                     "cols_per_cta": info["cols_per_cta"], "split": split,
                     "l2": "flushed before every step (256 MiB memset, untimed); working set > L2",
                     "verified_rows": verified},
            "parallelism": parallelism,
            "roofline": roof,
            "kernels_us": {k: v[1] / max(1, v[0]) * 1e3 for k, v in kern.items()},
            "e2e": {"value": stream_e2e["value"] if stream_e2e else n / (e2e_mean * 1e-3) / 1e9,
                    "unit": "Gbit/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 4 * pa.words32(m), "steps": stream_e2e["keys"] if stream_e2e else e2e_steps,
                    "verified": e2e_ok and (stream_e2e["verified_rows"] if stream_e2e else True),
                    "how": "a stream of distinct keys in pinned host memory through pa_hash_host_batch (each "
                           "key's H2D and output D2H timed; chunks pipelined: copy engines move chunk i+1 in "
                           "and chunk i-1 out while chunk i hashes); CUDA events around the call"
                    if world == 1 else
                    "rank 0: pinned key H2D, NCCL broadcast (rows) / scatter of key blocks (cols), sharded "
                    "hash and merge collectives, y D2H; CUDA events, max over ranks",
                    "single_call": {"value": n / (float(np.median(e2e_ms)) * 1e-3) / 1e9,
                                    "mean_value": n / (e2e_mean * 1e-3) / 1e9, "steps": e2e_steps,
                                    "how": "one key per pa_hash_host_async call (CUDA graph: pinned host key -> "
                                           "copy kernel -> K0..K3 -> copy kernel -> pinned host output), "
                                           "CUDA events around each step; value from the median step, "
                                           "mean_value from the mean"} if world == 1 else None},
            "gpu_launches": args.steps * (info["kernels_per_hash"] + (1 if split == "cols" else 0)),
            "clocks": clk.result(),
        }
        if side:
            line["multi_gpu"] = side
    if sh is not None:
        sh.close()
    else:
        h.close()
    if world > 1 or args.side_smoke:
        dist.barrier()
        dist.destroy_process_group()
    return line


def c5_keys(torch, name, count, dev, first=0):
    """`count` distinct keys of C5 sub-config `name` (streams key(c, first..first+count-1)),
    generated on the device with the pa_synth counter generator."""
    c = syn.CONFIG_INDEX[name]
    n = syn.CONFIGS[name]["n"]
    return syn.random_bits_torch([syn.key_stream(c, k) for k in range(first, first + count)], n, dev)


def time_batch(torch, h, keys, outs, flush, reps=2):
    h.hash_batch(keys, outs)
    torch.cuda.synchronize()
    return float(np.mean(time_steps(torch, lambda: h.hash_batch(keys, outs), reps, flush)))


def multi_gpu_side(args, torch, dist, pa, pd, dev, rank, world, flush, split, name):
    """N > 1 side measurements: the other split of the same key, the cost model's pick, and C5
    batches dealt across the ranks (each rank generates its own keys: pre-distributed)."""
    out = {"choose_split": pd.choose_split(syn.CONFIGS[name]["n"], syn.CONFIGS[name]["m"], world)}
    n, m, sw, kw = syn.config_inputs(name)
    seed_t = dev_words(torch, sw, dev)
    other = "cols" if split == "rows" else "rows"
    sh = pd.RowSplit(n, m, seed_t) if other == "rows" else pd.ColSplit(n, m, seed_t)
    blk = dev_words(torch, kw, dev) if other == "rows" else sh.key_block(kw, dev)
    for _ in range(3):
        y = sh(blk)
    torch.cuda.synchronize()
    dist.barrier()
    steps = max(5, min(args.steps, 30))
    t = float(sum(time_steps(torch, lambda: sh(blk), steps, flush)))
    tt = torch.tensor([t], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ok = None
    if rank == 0:
        ok = verify_rows(n, m, sw, kw, y.cpu().numpy(), sampled_rows(m, 64))
    out[f"{other}_split"] = {"gbit_s": n * steps / (float(tt[0]) * 1e-3) / 1e9,
                             "ms_per_hash": float(tt[0]) / steps, "verified_rows": ok}
    sh.close()
    # the column split with the fused Eq. (7) merge (NEXT-1): partials folded straight from the
    # peers' memory (pa_xor_fold_peers over CUDA IPC mappings) + one all-gather
    sh = pd.ColSplit(n, m, seed_t, fused=True)
    blk = sh.key_block(kw, dev)
    for _ in range(3):
        y = sh(blk)
    torch.cuda.synchronize()
    dist.barrier()
    t = float(sum(time_steps(torch, lambda: sh(blk), steps, flush)))
    tt = torch.tensor([t], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ok = verify_rows(n, m, sw, kw, y.cpu().numpy(), sampled_rows(m, 64)) if rank == 0 else None
    out["cols_fused_split"] = {"gbit_s": n * steps / (float(tt[0]) * 1e-3) / 1e9,
                               "ms_per_hash": float(tt[0]) / steps, "verified_rows": ok,
                               "merge": "pa_xor_fold_peers over CUDA-IPC-mapped peer partials + all_gather"}
    sh.close()
    for cname in ("C5a", "C5b", "C5c", "C5d"):
        cn, cm, csw, _ = syn.config_inputs(cname)
        idx = list(range(rank, C5_KEYS, world))
        total = len(idx) * world
        c = syn.CONFIG_INDEX[cname]
        keys = syn.random_bits_torch([syn.key_stream(c, k) for k in idx], cn, dev)
        kd = pd.KeyDeal(cn, cm, dev_words(torch, csw, dev))
        outs = kd.h.new_out(len(idx))
        kd(keys, outs)
        torch.cuda.synchronize()
        dist.barrier()
        ms = float(np.mean(time_steps(torch, lambda: kd(keys, outs), 2, flush)))
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        out[f"{cname}_dealt"] = {"keys": total, "keys_per_rank": len(idx),
                                 "gbit_s": cn * total / (float(tt[0]) * 1e-3) / 1e9}
        kd.close()
        del keys, outs
    return out


def sweep(torch, pa, dev, steps=10):
    """Side measurements (rank 0, N = 1), same protocol: C1 latency and 2^16 distinct keys
    batched (route b), C2 / C3 single keys, the C5 batches of 1024 distinct keys, fresh seeds, host-buffer batches.  Each transform entry carries its
    whole-hash HBM fraction (SURVEY 8(d) model bytes / time / measured peak)."""
    import oracle  # noqa: F401  (sampled-row checks below)
    peak, _ = peak_hbm()
    res = {}
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    for name in ("C1", "C2", "C3"):
        n, m, sw, kw = syn.config_inputs(name)
        h = pa.Hasher(n, m, dev_words(torch, sw, dev))
        key = dev_words(torch, kw, dev)
        out = h.new_out()
        for _ in range(3):
            h.hash(key, out)
        ms = time_steps(torch, lambda: h.hash(key, out), max(steps, 20), flush)
        t = float(np.mean(ms))
        info = h.info
        e = {"n": n, "m": m, "route": h.route, "ms_per_hash": t, "gbit_s": n / (t * 1e-3) / 1e9,
             "transform_len": info["transform_len"], "residual": h.residual(),
             "verified_rows": verify_rows(n, m, sw, kw, out.cpu().numpy(), sampled_rows(m))}
        if info["route"] == 1:
            hb = hash_bytes(n, m, info["n1"] * info["n2"])
            e["hbm_frac_whole_hash"] = hb / (t * 1e-3) / 1e9 / peak
        res[name] = e
        h.close()
    # the metric's curve, Gbit/s vs input length n (m = n/10, the paper's ratio): single
    # keys, arbitrary non-power-of-two lengths from 10^6 to 10^8 bits
    curve = {}
    # (each length planned by the cost model and by measurement, PA_PLAN_MEASURE)
    for n in (1_000_003, 2_999_999, 10_000_019, 29_999_999, 53_164_100, 100_000_007):
        m = n // 10 if n != 53_164_100 else n // 5
        sw = syn.random_bits(syn.seed_stream(70), n + m - 1)
        kw = syn.random_bits(syn.key_stream(70, n % 1000), n)
        key = dev_words(torch, kw, dev)
        e = {"m": m}
        for plan in ("model", "measure"):
            h = pa.Hasher(n, m, dev_words(torch, sw, dev), plan=plan)
            out = h.new_out()
            for _ in range(3):
                h.hash(key, out)
            t = float(np.mean(time_steps(torch, lambda: h.hash(key, out), max(steps, 10), flush)))
            info = h.info
            e[plan] = {"ms_per_hash": t, "gbit_s": n / (t * 1e-3) / 1e9,
                       "hbm_frac_whole_hash": hash_bytes(n, m, info["n1"] * info["n2"]) / (t * 1e-3) / 1e9 / peak,
                       "plan": f"{info['n1']}x{info['n2']} C={info['cols_per_cta']}",
                       "verified_rows": verify_rows(n, m, sw, kw, out.cpu().numpy(), sampled_rows(m, 32))}
            h.close()
        curve[str(n)] = e
    res["length_curve"] = curve
    # C5 (BASELINE configs[4]): distinct keys against one seed through pa_hash_batch
    for name in ("C5a", "C5b", "C5c", "C5d"):
        n, m, sw, _ = syn.config_inputs(name)
        count = C5_KEYS
        h = pa.Hasher(n, m, dev_words(torch, sw, dev))
        keys = c5_keys(torch, name, count, dev)
        outs = h.new_out(count)
        t = time_batch(torch, h, keys, outs, flush) / count
        info = h.info
        ok = True
        for k in (0, count - 1):
            kw = syn.random_bits(syn.key_stream(syn.CONFIG_INDEX[name], k), n)
            ok &= verify_rows(n, m, sw, kw, outs[k].cpu().numpy(), sampled_rows(m, 32, seed=k))
        res[name + "_batched"] = {"n": n, "m": m, "keys": count, "distinct_keys": True, "ms_per_key": t,
                                  "gbit_s": n / (t * 1e-3) / 1e9, "transform_len": info["transform_len"],
                                  "hbm_frac_whole_hash": hash_bytes(n, m, info["n1"] * info["n2"])
                                  / (t * 1e-3) / 1e9 / peak, "verified_rows": ok}
        h.close()
        del keys, outs
    # C1: one key's latency is launch-bound; throughput over 2^16 distinct keys (route b)
    n, m, sw, _ = syn.config_inputs("C1")
    count = 1 << 16
    h = pa.Hasher(n, m, dev_words(torch, sw, dev))
    keys = c5_keys(torch, "C1", count, dev)
    outs = h.new_out(count)
    t = time_batch(torch, h, keys, outs, flush, reps=3) / count
    ok = True
    for k in (0, 65534, count - 1):  # both launches of the batch (65535 keys per grid)
        kw = syn.random_bits(syn.key_stream(syn.CONFIG_INDEX["C1"], k), n)
        ok &= verify_rows(n, m, sw, kw, outs[k].cpu().numpy(), np.arange(m, dtype=np.uint64))
    res["C1_batched"] = {"n": n, "m": m, "keys": count, "distinct_keys": True, "route": h.route,
                         "us_per_key": t * 1e3, "gbit_s": n / (t * 1e-3) / 1e9, "verified_rows": ok}
    h.close()
    # C5a end to end from pinned host memory (pa_hash_host_batch: H2D / batched hash / D2H of
    # neighbouring chunks overlapped), 1024 distinct keys
    n, m, sw, _ = syn.config_inputs("C5a")
    h = pa.Hasher(n, m, dev_words(torch, sw, dev))
    kh = c5_keys(torch, "C5a", C5_KEYS, dev).cpu().pin_memory()
    oh = torch.empty((C5_KEYS, pa.words32(m)), dtype=torch.int32).pin_memory()
    h.hash_host_batch(kh, oh)
    ms = time_steps(torch, lambda: h.hash_host_batch(kh, oh), 2, flush)
    t = float(np.mean(ms)) / C5_KEYS
    res["C5a_batched_e2e"] = {"n": n, "m": m, "keys": C5_KEYS, "ms_per_key": t, "gbit_s": n / (t * 1e-3) / 1e9,
                              "note": "pa_hash_host_batch: pinned host keys in, host outputs out"}
    h.close()
    # fresh seed per key (NEXT-2): seed transform + hash per key, C2 and C4 shapes
    for cname, count in (("C2", 64), ("C4", 4)):
        n, m, sw, kw = syn.config_inputs(cname)
        ci = syn.CONFIG_INDEX[cname]
        seeds = syn.random_bits_torch([syn.seed_stream(900 + k) for k in range(count)], n + m - 1, dev)
        keys = syn.random_bits_torch([syn.key_stream(ci, k) for k in range(count)], n, dev)
        h = pa.Hasher(n, m, seeds[0])
        outs = h.new_out(count)
        h.hash_fresh_batch(seeds, keys, outs)
        ms = time_steps(torch, lambda: h.hash_fresh_batch(seeds, keys, outs), 3, flush)
        t = float(np.mean(ms)) / count
        res[f"{cname}_fresh_seed"] = {
            "n": n, "m": m, "keys": count, "ms_per_key": t, "gbit_s": n / (t * 1e-3) / 1e9,
            "note": "pa_hash_fresh_batch: a distinct seed per key (each seed's forward half fused into "
                    "the hash's K2, its spectrum row held in TMEM)"}
        h.close()
        del seeds, keys, outs
    # create time (SURVEY 8(d) timing protocol: pa_create timed separately): C4 seed transform
    n, m, sw, _ = syn.config_inputs("C4")
    seed_t = dev_words(torch, sw, dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h = pa.Hasher(n, m, seed_t)
    torch.cuda.synchronize()
    e0.record()
    h.set_seed(seed_t)
    e1.record()
    torch.cuda.synchronize()
    res["C4_set_seed_ms"] = e0.elapsed_time(e1)
    h.close()
    # NEXT-3: a 10^9-bit key (m = n/10, the paper's ratio) hashed from pinned HOST memory
    # through pa_hash_blocked_host under a 16 GiB device budget (blocks streamed in)
    n, m = 10**9, 10**8
    sw = syn.random_bits(syn.seed_stream(60), n + m - 1)
    kw = syn.random_bits(syn.key_stream(60, 0), n)
    sh_, kh_ = torch.from_numpy(sw.view(np.int32)).pin_memory(), torch.from_numpy(kw.view(np.int32)).pin_memory()
    oh_ = torch.zeros(pa.words32(m), dtype=torch.int32).pin_memory()
    budget = 16 << 30
    ts = []
    for i in range(6):  # the first calls pay one-time costs (pinned-page mappings, the block handle)
        t0 = time.perf_counter()
        pa.pa_hash_blocked_host(n, m, sh_.data_ptr(), kh_.data_ptr(), oh_.data_ptr(), 0, budget, 0)
        if i >= 3:
            ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    pa.pa_hash_blocked_release()
    res["NEXT3_host_1e9"] = {"n": n, "m": m, "s_per_hash": t, "gbit_s": n / t / 1e9, "device_budget_gib": 16,
                             "verified_rows": verify_rows(n, m, sw, kw, oh_.numpy(), sampled_rows(m, 16)),
                             "note": "pa_hash_blocked_host: key and seed in pinned host memory, row x column blocks "
                                     "streamed through two staging slots, Eq. (7) XOR merge; host wall clock "
                                     "(the call synchronises)"}
    del sh_, kh_, oh_
    return res


def cpu_oracle_baseline(name, budget_s=12.0):
    """The CPU oracle (as it stands) on a bounded sample of the workload's rows (every row costs
    the same: n/64 word products), all host cores and one core; extrapolated to a full hash."""
    import oracle
    n, m, sw, kw = syn.config_inputs(name)
    cores = host_cores()

    def rate(threads, budget):
        probe = np.arange(min(m, 256), dtype=np.uint64)
        t0 = time.perf_counter()
        oracle.toeplitz_rows(n, m, sw, kw, probe, threads=threads)
        per_row = (time.perf_counter() - t0) / probe.size
        rows = np.arange(min(m, max(256, int(budget / 3 / max(per_row, 1e-12)))), dtype=np.uint64)
        t0, reps = time.perf_counter(), 0
        while True:
            oracle.toeplitz_rows(n, m, sw, kw, rows, threads=threads)
            reps += 1
            el = time.perf_counter() - t0
            if el >= budget or reps >= 50:
                break
        return el / (reps * rows.size) * m, rows.size, reps, el
    t_all, r_all, reps_all, el_all = rate(cores, budget_s)
    t_one, r_one, reps_one, el_one = rate(1, budget_s * 0.6)
    return {"value": n / t_all / 1e9, "unit": "Gbit/s", "cores": cores, "kind": "oracle",
            "sample": f"{name}: rows [0,{r_all}) of m={m} x {reps_all} repeats ({el_all:.1f} s, word-level direct "
                      f"GF(2) product, OpenMP {cores} threads); every row costs the same, value extrapolated "
                      f"to the full hash (x{m / r_all:.0f})",
            "seconds_per_hash": t_all, "cpu_model": cpu_model(),
            "one_core": {"value": n / t_one / 1e9, "cores": 1, "seconds_per_hash": t_one,
                         "sample": f"rows [0,{r_one}) x {reps_one} ({el_one:.1f} s)"}}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle
    name = args.config
    n, m, sw, kw = syn.config_inputs(name)
    cores = host_cores()
    # size each step so the whole run takes ~1-2 minutes: estimate one row's cost
    probe = np.arange(min(m, 512), dtype=np.uint64)
    t0 = time.perf_counter()
    oracle.toeplitz_rows(n, m, sw, kw, probe, threads=cores)
    per_row = (time.perf_counter() - t0) / probe.size
    budget = 90.0 / max(1, args.steps + args.warmup)
    nrows = int(max(64, min(m, budget / max(per_row, 1e-9))))
    rows = np.arange(nrows, dtype=np.uint64)
    for _ in range(args.warmup):
        oracle.toeplitz_rows(n, m, sw, kw, rows, threads=cores)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.toeplitz_rows(n, m, sw, kw, rows, threads=cores)
        ts.append(time.perf_counter() - t0)
    t_full = float(np.sum(ts)) / args.steps * (m / nrows)
    value = n / t_full / 1e9
    sample = (f"{name}: rows [0,{nrows}) of m={m} per step (full hash extrapolated x{m / nrows:.0f}; every row "
              f"costs the same), word-level direct GF(2) oracle, OpenMP {cores} threads ({cpu_model()})")
    return {"metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "u64",
            "impl": "reference",
            "data": "synthetic: SplitMix64 i.i.d. Bernoulli(1/2) key and seed bits",
            "config": config_dict(name, n, m),
            "cpu_baseline": {"value": value, "unit": "Gbit/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------------------- CPU plumbing check
def run_selftest_cpu(args):
    """The multi-rank path without a GPU: gloo process group, the CPU oracle injected as each
    rank's hash (paper_1805_02372_b200.dist factories) -- rank spawning, row split with key
    broadcast, column split with key scatter + XOR merge, key dealing, cost model.  Prints a
    check line (not a measurement)."""
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1805_02372_b200 import dist as pd
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    n, m = 3001, 700
    sw = syn.random_bits(syn.seed_stream(91), n + m - 1)
    kw = syn.random_bits(syn.key_stream(91, 0), n)

    def ohash(nn, mm, seed_t, off, key_t):
        s = pd.extract_bits(seed_t.numpy().view(np.uint32), off, nn + mm - 1)
        k = pd.extract_bits(key_t.numpy().view(np.uint32), 0, nn)
        return torch.from_numpy(oracle.toeplitz_words(nn, mm, s, k).view(np.int32)[: (mm + 31) // 32].copy())
    seed_t = torch.from_numpy(sw.view(np.int32).copy())
    pd.distribute_seed(seed_t)
    key_t = torch.from_numpy(kw.view(np.int32).copy()) if rank == 0 else torch.zeros(
        (kw.size * 2,), dtype=torch.int32)
    want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    ok = {}
    for split in ("rows", "cols"):
        _, y = pd.hash(n, m, seed_t, key_t, split=split, hash_fn=ohash, xor_fn=pd._xor_fold_host)
        ok[split] = bool(np.array_equal(oracle.unpack(y.numpy().view(np.uint32), m), want))
    flags = torch.tensor([int(ok["rows"]), int(ok["cols"])])
    if world > 1:
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        dist.destroy_process_group()
    if rank == 0:
        return {"selftest": "cpu-gloo multi-rank plumbing (not a measurement)", "n_gpus": world,
                "rows_split_ok": bool(flags[0]), "cols_split_ok": bool(flags[1]),
                "choose_split_C4": pd.choose_split(10**8, 2 * 10**7, world)}
    return None


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(respawn(args))
    if args.selftest_cpu:
        line = run_selftest_cpu(args)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if args.impl == "reference":
        line = run_reference(args)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    line = run_ours(args)
    if line is None:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1:
        import torch

        import paper_1805_02372_b200 as pa
        if not args.no_sweep:
            line["sweep"] = sweep(torch, pa, torch.device("cuda", 0))
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_oracle_baseline(args.config)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
