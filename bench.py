#!/usr/bin/env python
"""Benchmark of the GNND hot path on B200 (BASELINE.json metric:
"kNN-graph build sec at recall@10>=0.95 (SIFT1M, DEEP100M shape)").

One step = one complete knng_build (init + all iterations + export, every
SURVEY.md section 8(a) row of the build) over the SIFT1M-shaped workload
(BASELINE.json configs[1]: 1M x 128 fp32, k = 32, L2), vectors resident in
HBM.  The vectors (512 MB) exceed the 126 MB L2, so no L2 flush is needed
between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): every rank builds its own
SIFT1M-shaped shard (independent problems, no collective; "scaling": weak).
--impl reference times the oracle (oracle/, plain C, single thread) on a
bounded sample of the same workload on the host CPU (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "kNN-graph build sec at recall@10>=0.95 (SIFT1M, DEEP100M shape), 1/2/4/8 B200"
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # derived


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", dest="n", type=int, default=1_000_000,
                    help="rows per GPU (C2: 10^6)")
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--recall-nodes", type=int, default=10_000)
    ap.add_argument("--cpu-sample", type=int, default=20_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--merge-iters", default="6",
                    help="GGM refine iterations: one count, or one per tree level (N>1); the N=1 GGM "
                         "line uses the first")
    ap.add_argument("--no-ggm", action="store_true", help="skip the N=1 GGM measurement")
    ap.add_argument("--deep-rows", type=int, default=50_000_000,
                    help="N=1 DEEP-shaped (continuous fp32, d=96) line: rows (0 = skip)")
    ap.add_argument("--deep-iters", type=int, default=8)
    ap.add_argument("--deep-steps", type=int, default=2)
    ap.add_argument("--deep-warmup", type=int, default=1)
    ap.add_argument("--ooc-rows", type=int, default=4_000_000,
                    help="N=1 out-of-memory all-pairs line (knng_build_ooc, P:298-302): rows (0 = skip)")
    ap.add_argument("--ooc-shards", type=int, default=4)
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload(args, rank, world=1):
    """N=1: the C2 SIFT1M-shaped set.  N>1: shard `rank` of an N x 1M
    SIFT-shaped set (one mixture of 1000 components, rows from the stream
    (1, rank)) -- the sharded build's weak-scaling workload.  Every shard
    holds ~1000 rows of every component, as the C2 set does: the GGM merge
    navigates the shard graphs from random cross seeds and needs components
    that are not split into tiny per-shard islands (D38)."""
    import datagen
    if world == 1:
        return datagen.make("sift", args.n, seed=1)
    return datagen.make("sift", args.n, seed=1, part=rank, components=1000)


def host_info() -> dict:
    """CPU model and core count of the host the oracle runs on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_baseline(args, X) -> dict:
    """The oracle as it stands, single thread pinned to core 0 (the
    process affinity is set to {0} around the call: `taskset -c 0`), on a
    bounded sample of the same workload: the first `cpu_sample` rows, same
    k/p/iters/seed; build seconds extrapolated linearly in n (GNND's
    per-iteration work is per-node: sample, 2p-bounded join, bounded
    update).  A full-size oracle build of C2 is tools/oracle_full_c2.py."""
    import oracle.oracle as orc
    ns = min(args.cpu_sample, X.shape[0])
    Xs = np.ascontiguousarray(X[:ns])
    old = None
    try:
        old = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {0})
    except Exception:
        old = None
    try:
        t0 = time.perf_counter()
        orc.build(Xs, args.k, args.p, args.iters, args.seed)
        dt = time.perf_counter() - t0
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    info = host_info()
    return {"value": dt * (X.shape[0] / ns), "unit": "s", "cores": 1, "kind": "oracle",
            "sample": f"oracle GNND build of the first {ns} rows of the same SIFT1M-shaped workload "
                      f"(k={args.k}, p={args.p}, iters={args.iters}) took {dt:.2f} s on 1 host core (affinity "
                      f"{{0}}); value = that x {X.shape[0]}/{ns} (linear in n)",
            "pinned_core": 0 if old is not None else None, **info, "sample_seconds": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    X = workload(args, 0)
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up state; warm-up steps are not repeated on the CPU
    times = []
    res = None
    for _ in range(args.steps):
        res = cpu_baseline(args, X)
        times.append(res["value"])
    v = statistics.median(times)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1000.0, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic GMM-LR SIFT-shaped (datagen 'sift', seed 1)",
            "config": {"workload": "C2 SIFT1M-shaped", "n": args.n, "d": 128, "k": args.k,
                       "sample_size": args.p, "iters": args.iters, "metric": "l2"},
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "oracle", "sample": res["sample"]},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def recall_at_10(K, Xd, dists, nodes, ids=None):
    """recall@10 (Eq. 4) on `nodes` sampled nodes against the exact k-NN
    (knng_bruteforce), with the D27 tie rule: entry j of the first 10 counts
    iff d(i, j) <= d_true,10(i).  When the ids are given, the graph is first
    checked independently of its own reported distances: on the sampled rows
    every id is a valid non-self node, no id repeats, and every stored
    distance equals the distance recomputed in float64 from the two vectors
    (within 1e-5 relative, BASELINE.json north_star); the tie rule then uses
    the verified distances."""
    import torch

    import datagen
    q = datagen.sample_nodes(Xd.shape[0], nodes)
    qt = torch.from_numpy(q).cuda().long()
    _, gd = K.knng_bruteforce(Xd, torch.from_numpy(q), 10)
    mine = dists[qt, :10]
    if ids is not None:
        gi = ids[qt].long()
        assert (gi >= 0).all() and (gi < Xd.shape[0]).all(), "graph id out of range"
        assert (gi != qt[:, None]).all(), "self-loop in the graph"
        srt = gi.sort(dim=1).values
        assert (srt[:, 1:] != srt[:, :-1]).all(), "duplicate id in a list"
        x = Xd[qt].double()
        for j in range(gi.shape[1]):
            ref = ((Xd[gi[:, j]].double() - x) ** 2).sum(1)
            got = dists[qt, j].double()
            assert ((got - ref).abs() <= 1e-5 * ref.abs().clamp_min(1e-30)).all(), "stored distance != recomputed"
    return float((mine <= gd[:, 9:10]).float().mean().item()), len(q)


def measure_ggm(args, K, Xd, stream):
    """GGM (Alg. 3) on the bench workload split in two halves:
    knng_build per half, then knng_merge timed with CUDA events on the
    launch stream."""
    import torch
    n, d = Xd.shape
    h = n // 2
    XA, XB = Xd[:h], Xd[h:]  # contiguous: knng_merge uses them in place
    ia, da = K.knng_build(XA, args.k, args.iters, args.p, args.seed, stream=stream)
    ib, db = K.knng_build(XB, args.k, args.iters, args.p, args.seed + 1, stream=stream)
    ws = torch.empty(K.lib().knng_merge_workspace_bytes(K.KNNG_F32, h, n - h, d, args.k, args.p, 0),
                     dtype=torch.uint8, device="cuda")

    def merge():
        return K.knng_merge(XA, ia, da, XB, ib, db, args.k, args.merge_iters[0], args.p, seed=args.seed, level=0,
                            workspace=ws, stream=stream)

    for _ in range(2):
        merge()
    torch.cuda.synchronize()
    K.knng_set_timing(True)
    K.knng_reset_timing()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, args.steps)
    e0.record(stream)
    for _ in range(reps):
        mi, md = merge()
    e1.record(stream)
    torch.cuda.synchronize()
    K.knng_set_timing(False)
    ms = e0.elapsed_time(e1) / reps
    join_ms, join_launches = K.knng_kernel_time("k_join")
    kernels = {}
    for nm in ["k_ggm_seed", "k_merge_sample", "k_rev_scatter", "k_rev_select", "k_join", "k_ggm_finalize",
               "k_check_u8", "k_to_u8", "k_export"]:
        t, c = K.knng_kernel_time(nm)
        if c:
            kernels[nm] = round(t / reps, 3)
    st = K.knng_last_stats()
    rec, nq = recall_at_10(K, Xd, md, args.recall_nodes)
    return {"workload": f"C2 split into 2 x {h} (knng_build per half, seeds {args.seed}/{args.seed + 1}), "
                        f"then knng_merge", "merge_iters": args.merge_iters[0], "ms_per_merge": ms,
            "recall_at_10": rec, "recall_nodes": nq,
            "join_ms_per_launch": join_ms / max(1, join_launches),
            "dist_evals": sum(s["dist_evals"] for s in st), "accepted": sum(s["accepted"] for s in st),
            "dist_evals_per_s": sum(s["dist_evals"] for s in st) / (ms * 1e-3),
            "kernel_ms_per_merge": kernels,
            # device time of the merge's own kernels (the events above also
            # see the host between the blocking calls)
            "kernel_sum_ms_per_merge": round(sum(kernels.values()), 3)}


FP32_ISSUE_PEAK = None  # set from the SM count and the sampled clock


def measure_ooc(args, K):
    """the paper's out-of-memory scheme from host
    memory to host memory -- GNND per shard, GGM of every pair of sub-graphs,
    running top-k lists; one resident and two streamed shards on the GPU.
    Wall clock around the (blocking) call: its host copies are part of the
    method here (the "disk" traffic overlapped with the merges)."""
    import torch
    import datagen
    n, S = args.ooc_rows, args.ooc_shards
    Xd = datagen.make_device("sift", n, seed=3, components=max(1, n // 1000)).to(torch.uint8)
    Xh = np.ascontiguousarray(Xd.cpu().numpy())
    ids = np.empty((n, args.k), np.uint32)
    dists = np.empty((n, args.k), np.float32)
    mi = int(args.merge_iters[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K.knng_build_ooc(Xh, args.k, 8, mi, args.p, S, seed=args.seed, out_ids=ids, out_dists=dists)
    wall = time.perf_counter() - t0
    nodes = datagen.sample_nodes(n, args.recall_nodes)
    _, td = K.knng_bruteforce(Xd, torch.from_numpy(nodes).cuda(), 10)
    t10 = td.cpu().numpy()[:, 9]
    rec = float((dists[nodes, :10] <= t10[:, None]).sum()) / (10 * len(nodes))
    del Xd
    torch.cuda.empty_cache()
    return {"workload": f"SIFT-shaped {n} x 128 uint8 in HOST memory (10^3 rows per mixture component), "
                        f"{S} shards, GNND per shard (8 iterations) + GGM of all {S * (S - 1) // 2} pairs "
                        f"({mi} refine iterations), host buffers in and out (knng_build_ooc)",
            "value": wall, "unit": "s", "recall_at_10": rec, "recall_nodes": len(nodes),
            "h2d_bytes": int(Xh.nbytes), "d2h_bytes": int(ids.nbytes + dists.nbytes), "timing": "wall clock"}


def measure_deep(args, K, stream, clk_ghz):
    """The metric's second shape: DEEP-shaped continuous fp32 rows (d = 96,
    L2-normalised GMM-LR, 10^4 components; BASELINE.json configs[3] shape)
    at the largest direct single-GPU size the bench budget allows, built with
    knng_build (the float path: k_join_ws, no exact-u8 shortcut).  Device
    time with CUDA events; recall@10 on 10k sampled nodes vs brute force."""
    import torch

    import datagen
    n, d = args.deep_rows, 96
    X = datagen.make_device("deep", n, seed=2)
    torch.cuda.synchronize()
    ws = torch.empty(K.knng_build_workspace_bytes(K.KNNG_F32, n, d, args.k, args.p), dtype=torch.uint8, device="cuda")
    ids = torch.empty((n, args.k), dtype=torch.int32, device="cuda")
    dists = torch.empty((n, args.k), dtype=torch.float32, device="cuda")

    def step():
        K.knng_build(X, args.k, args.deep_iters, args.p, args.seed, "l2", ids, dists, ws, stream)

    for _ in range(max(1, args.deep_warmup)):
        step()
    torch.cuda.synchronize()
    K.knng_set_timing(True)
    K.knng_reset_timing()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    hist = []
    for _ in range(args.deep_steps):
        step()
        hist.extend(K.knng_last_stats())
    e1.record(stream)
    torch.cuda.synchronize()
    K.knng_set_timing(False)
    ms = e0.elapsed_time(e1) / args.deep_steps
    exact_u8 = bool(K.knng_get_option("last_exact_u8"))
    join_ms, join_launches = K.knng_kernel_time("k_join")
    kernels = {}
    for nm in ["k_init", "k_merge_sample", "k_scan_reduce", "k_rev_scatter", "k_rev_select", "k_join", "k_merge",
               "k_export"]:
        t, c = K.knng_kernel_time(nm)
        if c:
            kernels[nm] = round(t / args.deep_steps, 3)
    rec, nq = recall_at_10(K, X, dists, args.recall_nodes, ids)
    evals = sum(s["dist_evals"] for s in hist)
    rows = sum(s["rows"] for s in hist)
    L = max(1, join_launches)
    join_avg = join_ms / L
    # ALU roofline of the canonical fp32 tile (D5): FADD + FFMA per dimension
    # and pair, against the FP32 pipe (148 SMs x 128 lanes x clock)
    fp_instr = evals * d * 2 / L
    fp_peak = 148 * 128 * clk_ghz * 1e9
    achieved = fp_instr / (join_avg * 1e-3)
    hbm_peak, _ = peaks()
    gbs = rows * (d * 4 + 4) / L / (join_avg * 1e-3) / 1e9
    return {"workload": f"DEEP-shaped {n} x {d} continuous fp32 (BASELINE.json configs[3] row shape; GMM-LR "
                        f"10^4 components, L2-normalised, generated on the GPU), direct knng_build on one B200",
            "metric": METRIC, "value": ms / 1000.0, "unit": "s", "ms_per_step": ms, "steps": args.deep_steps,
            "warmup": max(1, args.deep_warmup), "higher_is_better": False, "dtype": "u8" if exact_u8 else "f32",
            "config": {"n": n, "d": d, "k": args.k, "sample_size": args.p, "iters": args.deep_iters, "metric": "l2",
                       "l2_flush": f"inputs ({n * d * 4 / 1e9:.1f} GB) larger than L2"},
            "recall_at_10": rec, "recall_nodes": nq,
            "roofline": {"bound": "alu", "kernel": "k_join (k_join_ws, canonical fp32 tile)",
                         "achieved": achieved / 1e9, "peak": fp_peak / 1e9, "unit": "G fp32-instr/s",
                         "frac": achieved / fp_peak, "instr_per_dim_pair": 2, "sm_clock_ghz": clk_ghz,
                         "avg_launch_ms": join_avg, "launches": join_launches,
                         "share_of_step": join_ms / args.deep_steps / ms if ms > 0 else None,
                         "hbm_view": {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                                      "alg_bytes_per_launch": rows * (d * 4 + 4) / L}},
            "throughput": {"dist_evals_per_s": evals / args.deep_steps / (ms * 1e-3)},
            "kernel_ms_per_build": kernels}


def main():
    args = parse()
    args.merge_iters = [int(m) for m in str(args.merge_iters).split(",")]
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2103_15386_b200.knng as K
    from paper_2103_15386_b200.sharded import CudaOps, knng_build_sharded_nccl, nccl_comm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # KNNG_BENCH_BACKEND=gloo (testing only): several ranks sharing one GPU;
    # the product exchange is NCCL.
    backend = os.environ.get("KNNG_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        nccl_comm()  # libknng's own NCCL communicator (unique id broadcast by torch)
    coll_dev = "cuda" if backend == "nccl" else "cpu"

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather_rows(t):
        """all ranks' row blocks concatenated (for the recall check only)."""
        parts = [torch.empty_like(t, device=coll_dev) for _ in range(world)]
        dist.all_gather(parts, t.to(coll_dev))
        return torch.cat(parts).cuda()

    X = workload(args, rank, world)
    n, d = X.shape
    Xd = torch.from_numpy(X).cuda()
    stream = torch.cuda.current_stream()
    ws = torch.empty(K.knng_build_workspace_bytes(K.KNNG_F32, n, d, args.k, args.p), dtype=torch.uint8,
                     device="cuda")
    ids = torch.empty((n, args.k), dtype=torch.int32, device="cuda")
    dists = torch.empty((n, args.k), dtype=torch.float32, device="cuda")

    class Ops(CudaOps):
        """The product compute, recording each call's iteration counters."""

        def __init__(self, stream=None):
            super().__init__(stream=stream)
            self.history = []

        def build(self, *a):
            r = super().build(*a)
            self.history.extend(K.knng_last_stats())
            return r

        def merge(self, *a):
            r = super().merge(*a)
            self.history.extend(K.knng_last_stats())
            return r

    ops = Ops(stream=stream)
    out = {}
    levels = max(0, world.bit_length() - 1)  # log2(world) tree levels (world a power of two)
    level_iters = [args.merge_iters[min(i, len(args.merge_iters) - 1)] for i in range(levels)]

    def step():
        if world == 1:
            K.knng_build(Xd, args.k, args.iters, args.p, args.seed, "l2", ids, dists, ws, stream)
            ops.history.extend(K.knng_last_stats())
        else:  # one shard per GPU; every tree level merged by all GPUs of its group (C ABI, NCCL)
            out["g"] = knng_build_sharded_nccl(Xd, args.k, args.iters, level_iters, args.p, args.seed,
                                               stream=stream)
            ops.history.extend(K.knng_last_stats())

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: device time with CUDA events on the launch stream
    K.knng_set_timing(True)
    K.knng_reset_timing()
    ops.history.clear()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = K.knng_launch_count()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = K.knng_launch_count() - launches0
    clk = clocks.stop()
    K.knng_set_timing(False)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    join_ms, join_launches = K.knng_kernel_time("k_join")
    history = list(ops.history)
    stats = K.knng_last_stats()
    exact_u8 = bool(K.knng_get_option("last_exact_u8"))

    # ---- quality: recall@10 on sampled nodes vs exact brute force (GPU)
    if world > 1:
        my_i, my_d = out["g"]
        Xall = gather_rows(Xd)
        Dall = gather_rows(my_d.contiguous())
        recall, nq = recall_at_10(K, Xall, Dall, args.recall_nodes) if rank == 0 else (None, 0)
        del Xall, Dall
    else:
        recall, nq = recall_at_10(K, Xd, dists, args.recall_nodes, ids)

    # ---- end to end through the public API (pinned host buffers, copies timed)
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(X).pin_memory()
        ih = torch.empty((n, args.k), dtype=torch.int32).pin_memory()
        dh = torch.empty((n, args.k), dtype=torch.float32).pin_memory()
        lib = K.lib()

        def e2e_step():
            if world == 1:
                st = lib.knng_build_host(Xh.data_ptr(), K.KNNG_F32, n, d, args.k, K.KNNG_L2SQ, args.iters, args.p,
                                         args.seed, ih.data_ptr(), dh.data_ptr(), stream.cuda_stream)
                if st != 0:
                    raise RuntimeError(K.knng_last_error())
            else:
                Xd.copy_(Xh, non_blocking=True)
                gi, gd = knng_build_sharded_nccl(Xd, args.k, args.iters, level_iters, args.p, args.seed,
                                                 stream=stream)
                ih.copy_(gi, non_blocking=True)
                dh.copy_(gd, non_blocking=True)
                torch.cuda.synchronize()

        e2e_step()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
        barrier()
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(X.nbytes),
               "d2h_bytes_per_step": int(n * args.k * 8),
               "api": "knng_build_host" if world == 1 else "knng_build_sharded over NCCL (per-rank H2D/D2H)"}

    # ---- roofline of the dominant kernel (k_join), DESIGN.md section 6:
    # HBM view (primary): algorithmic gather bytes = rows x (d x element + 4
    # id bytes) per launch / launch time.  Tensor view (the exact-u8 tile is
    # an int8 Gram matrix on tcgen05): the method's int8 multiply-adds,
    # dist_evals x d x 2 ops, against the int8 dense peak (the measured bf16
    # burst peak x 2, the guide's nominal int8:bf16 ratio).  Issue view: the
    # measured issue-active fraction of the same kernel from the committed
    # ncu capture (profiles/join_traffic.json).
    esz = 1 if exact_u8 else 4
    rows = sum(s["rows"] for s in history)
    evals = sum(s["dist_evals"] for s in history)
    accepted = sum(s["accepted"] for s in history)
    launches_in_hist = max(1, join_launches)
    alg_bytes_per_launch = rows * (d * esz + 4) / launches_in_hist
    join_avg_ms = join_ms / launches_in_hist
    achieved_gbs = alg_bytes_per_launch / (join_avg_ms * 1e-3) / 1e9 if join_avg_ms > 0 else 0.0
    peak, peak_kind = peaks()
    clk_ghz = (clk.get("sm_mhz") or 1965.0) / 1000.0
    traffic, ncu_issue = None, None
    try:  # dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "join_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get("u8" if exact_u8 else "f32")
        ncu_issue = tj.get("issue_active_u8" if exact_u8 else "issue_active_f32")
    except Exception:
        pass
    views = {}
    if exact_u8:
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                bf16 = float(json.load(f)["bf16_tflops"])
            i8_src = "measured bf16 burst x 2"
        except Exception:
            bf16, i8_src = 2250.0, "nominal bf16 2250 TF/s x 2 (fallback)"
        ops = evals * d * 2 / launches_in_hist
        tops = ops / (join_avg_ms * 1e-3) / 1e12 if join_avg_ms > 0 else 0.0
        views["tensor"] = {"bound": "tensor", "achieved": tops, "peak": 2 * bf16, "unit": "TOPS int8",
                           "frac": tops / (2 * bf16), "peak_source": i8_src,
                           "note": "method's multiply-adds only; the 128x128 Gram tile computes ~8x more"}
    else:
        fp_instr = evals * d * 2 / launches_in_hist
        ach = fp_instr / (join_avg_ms * 1e-3) if join_avg_ms > 0 else 0.0
        fpk = 148 * 128 * clk_ghz * 1e9
        views["alu"] = {"bound": "alu", "achieved": ach / 1e9, "peak": fpk / 1e9, "unit": "G fp32-instr/s",
                        "frac": ach / fpk, "instr_per_dim_pair": 2}
    if ncu_issue is not None:
        views["issue"] = {"issue_active": ncu_issue, "source": "profiles/join_traffic.json (ncu --set full)"}
    roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                "frac": achieved_gbs / peak, "traffic": traffic, "peak_source": peak_kind,
                "kernel": "k_join", "avg_launch_ms": join_avg_ms, "launches": join_launches,
                "share_of_step": join_ms / args.steps / ms if ms > 0 else None,
                "alg_bytes_per_launch": alg_bytes_per_launch, "element_bytes": esz, "views": views}
    throughput = {"dist_evals_per_s": evals / args.steps / (ms * 1e-3),
                  "accepted_updates_per_s": accepted / args.steps / (ms * 1e-3), "per": "rank 0"}

    ggm = None
    if world == 1 and not args.no_ggm:
        ggm = measure_ggm(args, K, Xd, stream)

    deep = None
    if world == 1 and args.deep_rows > 0:
        deep = measure_deep(args, K, stream, clk_ghz)

    ooc = None
    if world == 1 and args.ooc_rows > 0:
        ooc = measure_ooc(args, K)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, X)
        cpu.pop("sample_seconds", None)

    if rank == 0:
        if world == 1:
            cfg = {"workload": "C2 SIFT1M-shaped (BASELINE.json configs[1])", "n": n, "d": d, "k": args.k,
                   "sample_size": args.p, "iters": args.iters, "metric": "l2",
                   "l2_flush": "inputs (512 MB) larger than L2"}
        else:
            cfg = {"workload": f"sharded SIFT-shaped {world} x {n} (one {n}-row shard per GPU, GNND per shard + "
                               f"log-depth GGM tree, every level merged by all GPUs of its group with records "
                               f"exchanged over NCCL (knng_build_sharded): the C4/C5 scheme at C2 shard size)",
                   "n": world * n, "n_per_gpu": n,
                   "d": d, "k": args.k, "sample_size": args.p, "iters": args.iters,
                   "merge_iters": level_iters, "shards": world, "metric": "l2",
                   "l2_flush": "inputs (512 MB per GPU) larger than L2"}
        line = {"metric": METRIC, "value": ms / 1000.0, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "u8" if exact_u8 else "f32",
                "data": "synthetic GMM-LR SIFT-shaped (datagen 'sift'), integer-valued fp32 input"
                        + ("; built on the exact uint8 path (option exact_u8: graph bit-identical to fp32)"
                           if exact_u8 else ""),
                "config": cfg, "recall_at_10": recall, "recall_nodes": nq,
                "roofline": roofline, "throughput": throughput, "ggm": ggm, "shapes": {"deep": deep}, "ooc": ooc,
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk, "iter_stats": stats}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
