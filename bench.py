#!/usr/bin/env python
"""bench.py -- key-candidate fitness evaluations / second (BASELINE.json metric).

Workload (BASELINE.json configs[1], SURVEY.md 8d "C2"): a batch of 10,000 MAS
ciphertexts, lengths L_i = default_rng(2).integers(100, 501), windows of the in-sample
corpus (tests/golden/data.npz, frozen from the reference's pkg/data/corpus.txt) at
offsets default_rng(seed).integers(0, len - L), keys WorkerRng(100000 + i, KEYGEN).
Each ciphertext gets 64 workers x 10,000 climbings (the acceptance #07 shape), bigram
table = the reference's english_bigrams.txt.  One step = one full batch: 640,000 worker
climbs = 6.4e9 fitness evaluations (one swap_delta each, mas.py:181-210), all executed.

value: device-resident inputs (ccg_mas_climb_dev), CUDA events on the engine's stream,
  L2 flushed between steps (a 256 MiB write; the inputs are ~16 MB < L2).
e2e:   the public batch API (engine.mas_climb) from pinned host buffers: H2D of the step's
  inputs, kernel, group argmax, D2H of scores + letter maps, wall clock per step.
cpu_baseline / --impl reference: the CPU oracle (a C port of the reference algorithm,
  oracle/cc_oracle.c) on every host core over a bounded sample of the same workload.

Multi-GPU (torchrun): weak scaling -- rank r solves its own 10,000-ciphertext batch
(key seeds offset by r * n_ciphers); no data-path collective; time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

KEYGEN_STREAM = 2**32 - 2
# Algorithmic shared-memory bytes of the D-form kernel (ccg_mas_dform.cu):
DFORM_BYTES_PER_TRY = 16         # exact delta of the proposal: T[a][b], T[b][a] (2 B each),
                                 # N[a][b], N[b][a], ks[a][b] (4 B each)
DFORM_BYTES_PER_ACCEPT = 6812    # N update 5408 + T row/column swap 416 + u,v 208 + S factors
                                 # 416 + saved rows 208 + diagonal refresh 156
DFORM_BYTES_PER_CIPHER = 12168   # once per ciphertext (dform_init_kernel): N from scratch 8112
                                 # + score 4056 (+8 B per bigram for the count matrix)
DFORM_BYTES_PER_WORKER = 5356    # each worker copies the ciphertext's T, N (5200) + diagonals 156
REF_LOOKUP_BYTES_PER_EVAL = 208 * 4    # reference-equivalent: 208 table lookups


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ciphers", type=int, default=10_000)
    ap.add_argument("--workers", type=int, default=64)
    ap.add_argument("--climbings", type=int, default=10_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true", help="one warm-up + one step (for ncu)")
    return ap.parse_args()


# ------------------------------------------------------------------ workload
def reference_permutation(seed: int, stream: int, n: int) -> np.ndarray:
    """WorkerRng(seed, stream).permutation(n) (rng.py:91-97) via numpy's own Philox."""
    from numpy.random import Generator, Philox

    from paper_2103_13937_b200.rng import philox_key

    u = Generator(Philox(key=list(philox_key(seed, stream)))).random(max(0, n - 1))
    perm = np.arange(n, dtype=np.int64)
    for t, i in enumerate(range(n - 1, 0, -1)):
        j = int(u[t] * (i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def make_workload(n_ciphers: int, rank: int = 0):
    with np.load(ROOT / "tests" / "golden" / "data.npz") as z:
        corpus = z["corpus"].astype(np.int64)
        scores = z["english_scores"].astype(np.int64)
    lengths = np.random.default_rng(2).integers(100, 501, n_ciphers)
    plains, ciphers = [], []
    for i, L in enumerate(lengths):
        gi = rank * n_ciphers + i
        off = int(np.random.default_rng(100000 + gi).integers(0, corpus.size - L))
        p = corpus[off:off + L]
        key = reference_permutation(100000 + gi, KEYGEN_STREAM, 26)
        plains.append(p)
        ciphers.append(key[p])
    return plains, ciphers, scores, lengths


def worker_keys(n_ciphers, workers, rank):
    """Philox key of worker w of ciphertext i: WorkerRng(7000 + gi, (0 << 32) | w)."""
    from paper_2103_13937_b200.rng import philox_key

    keys = np.empty((n_ciphers * workers, 2), dtype=np.uint64)
    for i in range(n_ciphers):
        k0, _ = philox_key(7000 + rank * n_ciphers + i, 0)
        keys[i * workers:(i + 1) * workers, 0] = k0
        keys[i * workers:(i + 1) * workers, 1] = np.arange(workers, dtype=np.uint64)
    return keys


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, which: str):
        """Record the host time the timed region starts ("begin") or ends ("end")."""
        setattr(self, "t_" + which, time.time())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.3)  # let the sample covering the end of the timed region arrive
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        t0, t1 = getattr(self, "t_begin", 0.0), getattr(self, "t_end", float("inf"))
        window = [ln for t, ln in self.lines if t0 - 0.1 <= t <= t1 + 0.15]
        for ln in window or [ln for _, ln in self.lines]:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names[1:], f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        load = [v for v in sm if v > 300] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ distributed plumbing
def dist_init(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist

        backend = "nccl" if os.environ.get("CCG_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        dist.init_process_group(backend)
        return dist.get_rank(), world, int(os.environ.get("LOCAL_RANK", "0"))
    return 0, 1, 0


def barrier_max(value: float, world: int, device: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([value], dtype=torch.float64, device=f"cuda:{device}" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ------------------------------------------------------------------ CPU legs
def cpu_sample(ciphers, scores, workers, climbings, seconds, rank=0):
    """Time the C oracle on all host cores over a prefix of the workload, growing the
    prefix until the run takes >= `seconds` (or the whole batch is used)."""
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    m = max(1, min(len(ciphers), threads // max(1, workers) + 1))
    while True:
        n = m * workers
        cof = np.repeat(np.arange(m, dtype=np.int32), workers)
        seeds = [7000 + rank * len(ciphers) + i for i in range(m) for _ in range(workers)]
        streams = [w for _ in range(m) for w in range(workers)]
        t0 = time.perf_counter()
        sc, maps = O.mas_workers(ciphers[:m], cof, seeds, streams, scores, climbings,
                                 threads=threads)
        dt = time.perf_counter() - t0
        if dt >= seconds or m >= len(ciphers):
            evals = n * climbings
            best = [int(np.argmax(sc[i * workers:(i + 1) * workers])) for i in range(m)]
            return {"value": evals / dt, "unit": "evals/s", "cores": threads, "kind": "port",
                    "sample": f"{m} ciphertexts x {workers} workers x {climbings} climbings "
                              f"({evals:.3g} evals, {dt:.1f} s) of the bench workload, "
                              "C oracle (oracle/cc_oracle.c), one pthread per core",
                    "best_maps": [maps[i * workers + b] for i, b in enumerate(best)]}
        m = min(len(ciphers), max(m + 1, int(m * max(2.0, 1.3 * seconds / max(dt, 1e-3)))))


def run_reference(args):
    rank, world, local = dist_init(args.gpus)
    if rank != 0:
        return
    plains, ciphers, scores, lengths = make_workload(args.ciphers, 0)
    samples = []
    for s in range(args.warmup + args.steps):
        r = cpu_sample(ciphers, scores, args.workers, args.climbings,
                       seconds=3.0 if s < args.warmup else args.cpu_seconds)
        if s >= args.warmup:
            samples.append(r)
    value = float(np.mean([r["value"] for r in samples]))
    # success rate vs length over the reference arm's own sample (same seeds as our arm)
    maps = samples[-1].pop("best_maps")
    for r in samples[:-1]:
        r.pop("best_maps", None)
    m = len(maps)
    rec = np.array([np.array_equal(maps[i][ciphers[i]], plains[i]) for i in range(m)])
    bins = (lengths[:m] // 50) * 50
    line = {
        "impl": "reference", "metric": "key-candidate fitness evals/sec", "value": value,
        "unit": "evals/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (corpus windows of the reference's pkg/data, reference key recipe)",
        "config": config_block(args, world),
        "cpu_baseline": {**samples[-1], "value": value},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "success_by_len": {f"{b}-{b + 49}": round(float(rec[bins == b].mean()), 4)
                           for b in sorted(set(bins.tolist()))},
        "success_sample": f"first {m} ciphertexts of the workload",
    }
    print(json.dumps(line), flush=True)


def config_block(args, world):
    return {"workload": "C2: MASC batch, 10k ciphertexts of 100-500 letters, bigram, "
                        "64 workers x 10k climbings each",
            "n_ciphers_per_gpu": args.ciphers, "workers_per_cipher": args.workers,
            "climbings": args.climbings, "table": "english_bigrams (reference pkg/data)",
            "l2": "flushed between steps (256 MiB write); inputs ~16 MB",
            "parallelism": f"restart/ciphertext sharding, {world} process(es), one GPU each"}


# ------------------------------------------------------------------ GPU leg
def issue_roofline(evals_per_s: float, clk: dict) -> dict | None:
    """Warp instructions issued per second vs the issue peak (4 per SM per clock), using the
    warp instructions per evaluation measured by ncu on this kernel (profiles/r1i_ncu.txt)."""
    prof = ROOT / "profiles" / "r1f_ncu.txt"
    try:
        import re

        inst = float(re.search(r"warp instructions per try = ([0-9.]+)", prof.read_text()).group(1))
    except Exception:  # noqa: BLE001
        return None
    mhz = clk.get("sm_mhz") or 1965.0
    peak = 4 * 148 * mhz * 1e6
    achieved = evals_per_s * inst
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp-inst/s",
            "frac": achieved / peak, "inst_per_eval": inst,
            "source": "ncu smsp__inst_executed.sum / tries (profiles/r1i_ncu.txt); peak = "
                      "4 issue slots x 148 SMs x the median SM clock during the timed steps"}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.profile:
        args.steps, args.warmup, args.no_e2e, args.no_cpu = 1, 1, True, True
    rank, world, local = dist_init(args.gpus)

    import ctypes as C

    import torch

    from paper_2103_13937_b200 import _lib, engine

    device = local if world > 1 else 0
    # CCG_BENCH_SHARE_GPU=1 (testing only, with CCG_BENCH_BACKEND=gloo): ranks share the
    # visible GPUs round-robin, so the multi-rank path can be exercised on a 1-GPU box
    if os.environ.get("CCG_BENCH_SHARE_GPU") == "1":
        device = local % torch.cuda.device_count()
    torch.cuda.set_device(device)
    engine.set_devices([device])
    ctx = _lib.context(device)
    L = _lib.load()

    plains, ciphers, scores, lengths = make_workload(args.ciphers, rank)
    W, K = args.workers, args.climbings
    n_workers = len(ciphers) * W
    keys = worker_keys(len(ciphers), W, rank)
    flat, off = _lib.ragged(ciphers)
    cof = np.repeat(np.arange(len(ciphers), dtype=np.int32), W)
    evals_per_step = n_workers * K

    # ---- device-resident inputs
    def dev(arr):
        p = ctx.dev_alloc(max(1, arr.nbytes))
        ctx.h2d(p, np.ascontiguousarray(arr))
        return p

    d_flat, d_off, d_cof, d_keys, d_tab = dev(flat), dev(off), dev(cof), dev(keys), dev(scores)
    d_scores = ctx.dev_alloc(n_workers * 8)
    d_maps = ctx.dev_alloc(n_workers * 26)
    d_best = ctx.dev_alloc(len(ciphers) * 8)
    d_acc = ctx.dev_alloc(n_workers * 8)
    a = _lib.MasClimbArgs()
    a.ciphers, a.offsets, a.n_ciphers = d_flat, d_off, len(ciphers)
    a.cipher_of, a.keys, a.skips = d_cof, d_keys, None
    a.n_workers, a.climbings, a.table = n_workers, K, d_tab
    a.scores, a.maps = d_scores, d_maps
    a.group_size, a.group_best = W, d_best
    a.max_len, a.table_max = int(lengths.max()), int(scores.max())
    a.flags = 0
    a.accepts = d_acc
    ctx.synchronize()

    stream = torch.cuda.ExternalStream(ctx.stream(), device=f"cuda:{device}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{device}")

    smem_bw = C.c_double(0.0)
    _lib.check(L.ccg_bench_smem_bandwidth(ctx.handle, C.byref(smem_bw)), "smem bench")

    def step():
        _lib.check(L.ccg_mas_climb_dev(ctx.handle, a), "mas_climb_dev")

    clocks = ClockSampler(device)
    clocks.start()  # running before the warm-up so that it samples the whole timed region
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step()
    ctx.synchronize()

    barrier(world)
    torch.cuda.synchronize()
    clocks.mark("begin")
    launches0 = ctx.launches()
    evs = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        step()
        with torch.cuda.stream(stream):
            e1.record(stream)
        evs.append((e0, e1))
    ctx.synchronize()
    torch.cuda.synchronize()
    clocks.mark("end")
    barrier(world)
    clk = clocks.stop()
    launches = ctx.launches() - launches0
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    total_s = barrier_max(sum(step_ms) / 1e3, world, device)
    value = evals_per_step * args.steps * world / total_s

    # per-launch duration of the dominant kernel (mas_climb; the group argmax is ~us)
    kernel_s = float(np.mean(step_ms)) / 1e3
    smem_peak = smem_bw.value / 1e9
    acc = np.empty(n_workers, dtype=np.int64)
    ctx.d2h(acc, d_acc)
    ctx.synchronize()
    n_accepts = int(acc.sum())
    worker_bytes = sum(W * DFORM_BYTES_PER_WORKER + DFORM_BYTES_PER_CIPHER + 8 * (int(L) - 1)
                       for L in lengths)
    launch_bytes = (DFORM_BYTES_PER_TRY * evals_per_step + DFORM_BYTES_PER_ACCEPT * n_accepts
                    + worker_bytes)
    bytes_per_eval = launch_bytes / evals_per_step
    achieved = launch_bytes / kernel_s / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        try:
            t = json.loads(tfile.read_text())
            if t.get("n_workers") == n_workers and t.get("climbings") == K:
                traffic = t.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # correctness spot-check of this run: recovered plaintexts, scores consistent
    sc = np.empty(n_workers, dtype=np.int64)
    ctx.d2h(sc, d_scores)
    ctx.synchronize()

    # ---- e2e through the public batch API, pinned host buffers
    e2e = None
    success = None
    if not args.no_e2e:
        def pinned(arr):
            p = C.c_void_p()
            _lib.check(L.ccg_host_alloc(arr.nbytes, C.byref(p)), "host_alloc")
            buf = (C.c_uint8 * arr.nbytes).from_address(p.value)
            out = np.frombuffer(buf, dtype=arr.dtype).reshape(arr.shape)
            out[...] = arr
            return out

        # the step's inputs in pinned host memory: the packed ciphertext batch (uint8 letters
        # + offsets, the C ABI's input format), worker keys and cipher indices; results come
        # back into pinned host buffers
        p_keys = pinned(keys)
        p_cof = pinned(cof)
        p_batch = _lib.Packed.__new__(_lib.Packed)
        p_batch.flat, p_batch.offsets = pinned(flat), pinned(off)
        res = engine.ClimbResult(scores=pinned(np.zeros(n_workers, np.int64)),
                                 keys=pinned(np.zeros((n_workers, 26), np.uint8)),
                                 group_best=pinned(np.zeros(len(ciphers), np.int64)),
                                 draws_used=None, last_accept=None, tries_done=None, launches=0)
        e2e_ms = []
        for i in range(1 + min(args.steps, 3)):
            barrier(world)
            t0 = time.perf_counter()
            engine.mas_climb(p_batch, p_cof, p_keys, scores, K, group_size=W, out=res)
            dt = time.perf_counter() - t0
            if i > 0:
                e2e_ms.append(dt * 1e3)
        e2e_s = barrier_max(float(np.mean(e2e_ms)) / 1e3, world, device)
        h2d = flat.nbytes + off.nbytes + cof.nbytes + keys.nbytes + scores.nbytes
        d2h = n_workers * 8 + n_workers * 26 + len(ciphers) * 8
        e2e = {"value": evals_per_step * world / e2e_s, "unit": "evals/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_s * 1e3,
               "api": "paper_2103_13937_b200.engine.mas_climb (packed batch + results in "
                      "pinned host memory)"}
        assert np.array_equal(res.scores, sc), "e2e and device-resident runs disagree"
        # success rate vs length (the C2 quality metric), 50-letter bins
        rec = np.array([np.array_equal(res.keys[i * W + int(res.group_best[i])].astype(np.int64)
                                       [ciphers[i]], plains[i]) for i in range(len(ciphers))])
        bins = (lengths // 50) * 50
        success = {f"{b}-{b + 49}": round(float(rec[bins == b].mean()), 4)
                   for b in sorted(set(bins.tolist()))}

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_sample(ciphers, scores, W, K, args.cpu_seconds)
        cpu_maps = cpu.pop("best_maps")
        # the same per-ciphertext outcome as the CPU port on its whole sample (bit-exact parity)
        if e2e is not None:
            cpu["agrees_with_gpu"] = all(
                np.array_equal(res.keys[i * W + int(res.group_best[i])].astype(np.int64)[ciphers[i]],
                               cpu_maps[i][ciphers[i]]) for i in range(len(cpu_maps)))

    if rank == 0:
        line = {
            "metric": "key-candidate fitness evals/sec",
            "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int32",
            "data": "synthetic (corpus windows of the reference's pkg/data, reference key recipe)",
            "config": config_block(args, world),
            "e2e": e2e,
            "roofline": {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                         "frac": achieved / smem_peak, "traffic": traffic,
                         "kernel": "mas_climb_dform_kernel<false>",
                         "bytes_per_eval": bytes_per_eval,
                         "accepts_per_eval": n_accepts / evals_per_step,
                         "peak_source": "measured on this GPU by ccg_bench_smem_bandwidth "
                                        "(128-bit conflict-free LDS, full occupancy)",
                         "ref_equiv_achieved": evals_per_step * REF_LOOKUP_BYTES_PER_EVAL
                         / kernel_s / 1e9,
                         "note": "algorithmic shared-memory bytes of the D-form algorithm "
                                 "(DESIGN.md 3.1); the kernel is issue-bound, see "
                                 "issue_roofline"},
            # the binding resource: warp-instruction issue (4 schedulers per SM), with the
            # instructions per evaluation of the committed ncu capture of this kernel
            "issue_roofline": issue_roofline(value / world, clk),
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
            "evals_per_step": evals_per_step,
            "success_by_len": success,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
