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

Multi-GPU: weak scaling -- rank r solves its own 10,000-ciphertext batch (key seeds offset
by r * n_ciphers); no data-path collective; time = max over ranks (all-reduce MAX).  Under
torchrun one rank per GPU; a plain `python bench.py --gpus N` re-launches itself under
torch.distributed.run with N ranks (and fails loudly if fewer than N GPUs are visible).

configs: BASELINE.json's other configurations (C1, C1d, C3, C4, C5) and time-to-recover on
the reference's acceptance recipes #07/#08, bounded to about a minute, each with the GPU
rate, the CPU port's rate and a bit-exact parity sample (tests/tools/bench_configs.py);
rank 0 at N=1 only.
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
    ap.add_argument("--cpu-ciphers", type=int, default=None,
                    help="ciphertexts the CPU port checks (default: the whole batch)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the bounded C1/C1d/C3/C4/C5/TTR block")
    ap.add_argument("--profile", action="store_true", help="one warm-up + one step (for ncu)")
    return ap.parse_args()


# ------------------------------------------------------------------ launcher
def visible_gpus() -> int:
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def maybe_relaunch(args) -> None:
    """`python bench.py --gpus N` without torchrun: re-run this script under
    torch.distributed.run with N ranks, one per GPU (the driver's multi-GPU launch), so both
    launchers measure N GPUs.  Fails loudly when fewer than N GPUs are visible (except in
    the CCG_BENCH_SHARE_GPU=1 test mode, where ranks share the visible GPUs over gloo)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    share = os.environ.get("CCG_BENCH_SHARE_GPU") == "1"
    if args.impl == "ours" and not share:
        n = visible_gpus()
        if n < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but only {n} CUDA "
                             "device(s) are visible; refusing to report a smaller run\n")
            sys.exit(2)
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def check_world(args, world: int, share: bool) -> None:
    if world != args.gpus and world > 1:
        sys.stderr.write(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}\n")
        sys.exit(2)
    if args.impl == "ours" and not share and world > 1 and visible_gpus() < world:
        sys.stderr.write(f"bench.py: {world} ranks but only {visible_gpus()} visible GPUs\n")
        sys.exit(2)


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
def cpu_port(ciphers, scores, workers, climbings, idx, rank=0, n_ciphers=None):
    """Run the C oracle (a port of stochastic_worker, mas.py:218-244) on every worker of the
    ciphertexts `idx`, one pthread per host core.  Returns (seconds, {i: best letter map}),
    the best map of ciphertext i being its first-maximum worker's (search.py:19-25)."""
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    n_ciphers = len(ciphers) if n_ciphers is None else n_ciphers
    idx = list(idx)
    best, seconds = {}, 0.0
    for lo in range(0, len(idx), 1000):  # chunks bound the host memory of the outputs
        part = idx[lo:lo + 1000]
        cof = np.repeat(np.arange(len(part), dtype=np.int32), workers)
        seeds = [7000 + rank * n_ciphers + i for i in part for _ in range(workers)]
        streams = [w for _ in part for w in range(workers)]
        t0 = time.perf_counter()
        sc, maps = O.mas_workers([ciphers[i] for i in part], cof, seeds, streams, scores,
                                 climbings, threads=threads)
        seconds += time.perf_counter() - t0
        for j, i in enumerate(part):
            best[i] = maps[j * workers + int(np.argmax(sc[j * workers:(j + 1) * workers]))]
    return seconds, best


def success_curve(recovered, lengths) -> dict:
    """Fraction of ciphertexts whose best key decrypts to the plaintext, 50-letter bins."""
    rec = np.asarray(recovered, dtype=bool)
    bins = (np.asarray(lengths) // 50) * 50
    return {f"{b}-{b + 49}": round(float(rec[bins == b].mean()), 4)
            for b in sorted(set(bins.tolist()))}


def run_reference(args):
    """The reference arm: the CPU port of the reference algorithm on all host cores.  Step s
    runs the s-th of `steps` contiguous slices of the 10,000-ciphertext batch (all 64
    workers x 10,000 climbings of each), so the timed steps together cover the whole
    workload and the success curve is over exactly the GPU arm's ciphertexts."""
    if int(os.environ.get("RANK", "0")) != 0:  # under torchrun rank 0 alone runs the port
        return
    plains, ciphers, scores, lengths = make_workload(args.ciphers, 0)
    W, K = args.workers, args.climbings
    threads = os.cpu_count() or 1
    for s in range(args.warmup):  # warm-up: one ciphertext per step
        cpu_port(ciphers, scores, W, K, [s % len(ciphers)])
    chunks = [c.tolist() for c in np.array_split(np.arange(len(ciphers)), max(1, args.steps))]
    seconds, best = 0.0, {}
    for ch in chunks:
        dt, b = cpu_port(ciphers, scores, W, K, ch)
        seconds += dt
        best.update(b)
    evals = len(ciphers) * W * K
    value = evals / seconds
    rec = [np.array_equal(best[i][ciphers[i]], plains[i]) for i in range(len(ciphers))]
    sample = (f"all {len(ciphers)} ciphertexts x {W} workers x {K} climbings ({evals:.3g} "
              f"evals, {seconds:.1f} s), {args.steps} slices, C oracle (oracle/cc_oracle.c), "
              "one pthread per core")
    line = {
        "impl": "reference", "metric": "key-candidate fitness evals/sec", "value": value,
        "unit": "evals/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": seconds / max(1, args.steps) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (corpus windows of the reference's pkg/data, reference key recipe)",
        "config": config_block(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "success_by_len": success_curve(rec, lengths),
        "success_sample": f"all {len(ciphers)} ciphertexts of the workload (the GPU arm's set)",
        "recovered": int(sum(rec)),
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
# The committed ncu --set full capture of the headline kernel (update with the kernel):
DFORM_PROFILE = "profiles/r2h_dform_ncu.txt"


def read_ncu_summary(rel: str) -> dict | None:
    """The counters this line derives from, read from a committed profiles/*_ncu.txt."""
    import re

    try:
        txt = (ROOT / rel).read_text()
    except OSError:
        return None

    def num(pat):
        m = re.search(pat + r"\s+([0-9.eE+]+)", txt)
        return float(m.group(1)) if m else None

    tries = num(r"tries in the captured launch:")
    out = {"file": rel, "tries": tries,
           "inst": num(r"smsp__inst_executed\.sum"),
           "smem_wavefronts": num(r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum"),
           "smem_conflicts": num(r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum"),
           "smem_pipe_pct": num(r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum\.pct_of_peak_sustained_elapsed"),
           "issue_pct": num(r"smsp__issue_active\.avg\.pct_of_peak_sustained_active")}
    if not tries or not out["inst"]:
        return None
    return out


def issue_roofline(evals_per_s: float, clk: dict) -> dict | None:
    """Warp instructions issued per second vs the issue peak (4 per SM per clock), with the
    warp instructions per evaluation of the committed ncu capture DFORM_PROFILE."""
    prof = read_ncu_summary(DFORM_PROFILE)
    if prof is None:
        return None
    inst = prof["inst"] / prof["tries"]
    mhz = clk.get("sm_mhz") or 1965.0
    peak = 4 * 148 * mhz * 1e6
    achieved = evals_per_s * inst
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp-inst/s",
            "frac": achieved / peak, "inst_per_eval": inst,
            "ncu_issue_active_pct": prof["issue_pct"],
            "source": f"ncu smsp__inst_executed.sum / tries ({DFORM_PROFILE}) x this run's "
                      "evals/s; peak = 4 issue slots x 148 SMs x the median SM clock during "
                      "the timed steps"}


def smem_pipe_roofline(evals_per_s: float, clk: dict) -> dict | None:
    """Shared-memory pipe occupancy: wavefronts (including bank-conflict replays) per
    evaluation from the committed ncu capture x this run's evals/s, against one wavefront
    per SM per clock -- the counter-based companion of the algorithmic-bytes fraction."""
    prof = read_ncu_summary(DFORM_PROFILE)
    if prof is None or not prof["smem_wavefronts"]:
        return None
    wpe = prof["smem_wavefronts"] / prof["tries"]
    mhz = clk.get("sm_mhz") or 1965.0
    peak = 148 * mhz * 1e6
    achieved = evals_per_s * wpe
    return {"bound": "smem-pipe", "achieved": achieved, "peak": peak, "unit": "wavefronts/s",
            "frac": achieved / peak, "wavefronts_per_eval": wpe,
            "conflict_wavefronts_per_eval": (prof["smem_conflicts"] or 0.0) / prof["tries"],
            "ncu_pct_of_peak": prof["smem_pipe_pct"],
            "source": f"ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum / tries "
                      f"({DFORM_PROFILE}) x this run's evals/s; peak = 1 wavefront per SM per "
                      "clock at the median SM clock during the timed steps"}


def run_configs() -> dict | None:
    """BASELINE.json's other configurations, bounded (tests/tools/bench_configs.py)."""
    sys.path.insert(0, str(ROOT / "tests" / "tools"))
    try:
        import bench_configs
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"}
    t0 = time.perf_counter()
    out = bench_configs.run_all(bounded=True)
    out["wall_s"] = round(time.perf_counter() - t0, 1)
    return out


def main():
    args = parse_args()
    maybe_relaunch(args)
    share = os.environ.get("CCG_BENCH_SHARE_GPU") == "1"
    if args.impl == "reference":
        run_reference(args)
        return
    if args.profile:
        args.steps, args.warmup, args.no_e2e, args.no_cpu = 1, 1, True, True
        args.no_configs = True
    rank, world, local = dist_init(args.gpus)
    check_world(args, world, share)

    import ctypes as C

    import torch

    from paper_2103_13937_b200 import _lib, engine

    device = local if world > 1 else 0
    # CCG_BENCH_SHARE_GPU=1 (testing only, with CCG_BENCH_BACKEND=gloo): ranks share the
    # visible GPUs round-robin, so the multi-rank path can be exercised on a 1-GPU box
    if share:
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
        gpu_best = [res.keys[i * W + int(res.group_best[i])].astype(np.int64)
                    for i in range(len(ciphers))]
        success = success_curve([np.array_equal(gpu_best[i][ciphers[i]], plains[i])
                                 for i in range(len(ciphers))], lengths)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the CPU port over the whole batch (or --cpu-ciphers of it): the CPU baseline and
        # the key-recovery agreement of every ciphertext
        m = len(ciphers) if args.cpu_ciphers is None else min(len(ciphers), args.cpu_ciphers)
        dt, cpu_best = cpu_port(ciphers, scores, W, K, range(m))
        evals = m * W * K
        cpu = {"value": evals / dt, "unit": "evals/s", "cores": os.cpu_count() or 1,
               "kind": "port",
               "sample": f"{m} ciphertexts x {W} workers x {K} climbings ({evals:.3g} evals, "
                         f"{dt:.1f} s) of the bench workload, C oracle (oracle/cc_oracle.c), "
                         "one pthread per core"}
        if e2e is not None:
            agree = sum(bool(np.array_equal(gpu_best[i][ciphers[i]], cpu_best[i][ciphers[i]]))
                        for i in range(m))
            cpu["agrees_with_gpu"] = agree == m
            cpu["agreement"] = f"{agree}/{m} ciphertexts: identical best decryption"
            cpu["success_by_len"] = success_curve(
                [np.array_equal(cpu_best[i][ciphers[i]], plains[i]) for i in range(m)],
                lengths[:m])

    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = run_configs()

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
            "smem_pipe_roofline": smem_pipe_roofline(value / world, clk),
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
            "evals_per_step": evals_per_step,
            "success_by_len": success,
            "configs": configs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
