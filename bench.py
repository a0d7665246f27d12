"""bench.py -- one step of the MicroMix hot path on B200, timed.

A STEP is one pass of the whole hot path over one batch of synthetic input:
    mm_reorder_quantize_act(X)  (fused gather + MX block quantization, rows R1-R5)
    mm_mixed_gemm_bf16(A, W)    (3-segment block-scaled tcgen05 GEMM, rows R7-R8)
against offline-calibrated, offline-quantized weights (rows R0, R6; untimed).

Default workload at N=1 (BASELINE.json configs[1]): Llama-3.1-8B q_proj, M=2048
K=4096 N=4096, calibrated plan.  Default at N>1 (BASELINE.json configs[3], the
north star's multi-GPU case): the Llama-3.1-70B down_proj (M=8192 K=28672 N=8192)
N-sharded over the N ranks -- each rank quantizes the replicated activation and
computes its N/G output channels, and the library's NCCL all-gather assembles the
BF16 Y on every rank (strong scaling); the fused all-gather epilogue (peer stores
over NVLink) is timed on the same ranks and reported in `fused_allgather`.
`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N local ranks (127.0.0.1 rendezvous).

Timing: the K timed steps run back to back, split into R = min(5, K) chunks with
one CUDA event between chunks; `value`/`ms_per_step` come from the whole region,
`ms_per_step_stats` gives the median / p10 / p90 over the chunks.  Per-kernel
durations: R passes of K back-to-back launches of that kernel alone.

L2 policy: every step reads a different one of `nsets` rotating input sets
(activations, quantized weights, outputs) whose total exceeds 2x the 126 MB L2,
so no step finds its operands L2-resident from the previous one.

`--impl reference` times the CPU oracle (oracle/, the deliberately slow
reference of this tier) on a bounded row sample of the same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "mixed MX GEMM TFLOPS (% mix-weighted peak); reorder-quantize HBM GB/s"
UNIT = "TFLOP/s"

CONFIGS = {
    # name: (M, K, N, workload text)
    "q_proj": (2048, 4096, 4096, "Llama-3.1-8B q_proj M=2048 K=4096 N=4096, calibrated thresholds"),
    "llama70b_down": (8192, 28672, 8192,
                      "Llama-3.1-70B down_proj M=8192 K=28672 N=8192, calibrated, N-sharded + BF16 all-gather"),
    "cfg1": (16, 256, 256, "single linear M=16 K=256 N=256, fixed split 128/64/64, 4 outlier channels"),
}


# ----------------------------------------------------------------------------- helpers
def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written), else the
    fallback in B200_PROFILING.md.  FP8/FP6 and FP4 dense peaks are the measured
    bf16 peak x the nominal ratios 2x and 4x (2.25 -> 4.5 -> 9 PF)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    src = "measured"
    try:
        with open(path) as f:
            p = json.load(f)
        hbm, bf16 = float(p["hbm_gbs"]), float(p["bf16_tflops"])
        bf16_s = float(p.get("bf16_tflops_sustained", bf16))
    except Exception:
        hbm, bf16, bf16_s, src = 6650.0, 1590.0, 1400.0, "fallback"
    return dict(hbm_gbs=hbm, bf16=bf16, bf16_sustained=bf16_s, fp8=2 * bf16, fp4=4 * bf16, src=src)


def mix_peak_tflops(n, pk):
    """P_mix = K / (n4/P_FP4 + (n6+n8)/P_FP8) (FP6 runs at the FP8 rate)."""
    K = sum(n)
    return K / (n[0] / pk["fp4"] + (n[1] + n[2]) / pk["fp8"])


def rq_bytes(M, n):
    """Algorithmic reorder-quantize bytes: BF16 read + packed codes + E8M0 scales (no padding)."""
    K = sum(n)
    return 2 * M * K + M * (n[0] // 2 + 3 * n[1] // 4 + n[2]) + M * K // 32


def host_facts():
    """CPU model, sockets and usable threads of this host (for cpu_baseline)."""
    model, sockets = None, set()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name") and model is None:
                    model = line.split(":", 1)[1].strip()
                elif line.startswith("physical id"):
                    sockets.add(line.split(":", 1)[1].strip())
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count()
    return {"cpu_model": model, "sockets": max(1, len(sockets)), "cpu_count": os.cpu_count(),
            "usable_threads": usable}


def pct(vals, q):
    return float(np.percentile(np.asarray(vals, dtype=np.float64), q)) if vals else None


def stats(vals):
    return {"median": pct(vals, 50), "p10": pct(vals, 10), "p90": pct(vals, 90), "n": len(vals)}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms in the background."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # NCCL's init log shows the N ranks (kept off stdout, which carries the JSON line)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    from paper_2508_02343_b200.dist import max_over_ranks as mor
    return mor(v, device="cuda") if world > 1 else v


# ----------------------------------------------------------------------------- oracle (CPU) arm
def calib_rows_for(K):
    """Calibration rows of BOTH arms (the GPU arm's plan and the oracle's are equal)."""
    return 16384 if K <= 8192 else 2048


_ORACLE_PLAN = {}


def oracle_plan(K, seed_layer=0):
    """The oracle's calibration of the same calibration draw the GPU arm uses."""
    from oracle import calib as ocal
    from synth import bf16_bits, gen_act
    key = (K, seed_layer)
    if key not in _ORACLE_PLAN:
        cal = ocal.calibrate(bf16_bits(gen_act(calib_rows_for(K), K, 1000 + seed_layer, 2000 + 10 * seed_layer)))
        _ORACLE_PLAN[key] = (cal["perm"], cal["n"])
    return _ORACLE_PLAN[key]


def oracle_cpu_rate(M, K, N, budget_s=15.0, seed_layer=0, threads=None):
    """Time the CPU oracle (as it stands) on a bounded row sample of the workload:
    reorder-quantize of the sampled activation rows + fp64 GEMM of the dequantized
    operands against all N output channels.  The weight quantization is offline for
    both arms and is done before timing.  threads=1 limits BLAS and OpenMP to one
    thread.  Returns (TFLOP/s, sample text, threads used, rows/s, n4_n6_n8)."""
    import contextlib

    from oracle import mx as omx
    from synth import bf16_bits, gen_act, gen_weight
    perm, n = oracle_plan(K, seed_layer)
    omx.encode(np.zeros(1), 0)            # load the OpenMP encoder so threadpoolctl sees it
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        ctx = threadpool_limits(limits=threads) if threads else contextlib.nullcontext()
    except Exception:
        threadpool_info, ctx = None, contextlib.nullcontext()
    with ctx:
        try:
            used = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
        except Exception:
            used = threads or os.cpu_count()
        return _oracle_loop(M, K, N, budget_s, seed_layer, perm, n, omx, bf16_bits, gen_act, gen_weight) + (used, n)


ORACLE_MAX_WEIGHT_ELEMS = 1 << 26   # bound the oracle's offline weight quantization (host RAM / time)


def _oracle_loop(M, K, N, budget_s, seed_layer, perm, n, omx, bf16_bits, gen_act, gen_weight):
    # large layers (70B down_proj: 235 M weights): the oracle's FLOP rate is measured
    # against a bounded subset of the output channels (same K, same per-element work)
    n_cols = N if N * K <= ORACLE_MAX_WEIGHT_ELEMS else max(256, ORACLE_MAX_WEIGHT_ELEMS // K // 256 * 256)
    w_bits = bf16_bits(gen_weight(n_cols, K, 3000 + seed_layer))
    n_all, N = N, n_cols
    wc, wsf, _ = omx.reorder_quantize(w_bits, perm, n)
    Wd = omx.dequantize_segments(wc, wsf)
    # run row batches of the workload (cycling over the M rows) for ~budget_s of CPU time
    rows = 64
    total_rows, t_total = 0, 0.0
    while t_total < budget_s:
        x_bits = bf16_bits(gen_act(rows, K, 1000 + seed_layer, 5000 + (total_rows % M)))
        t0 = time.perf_counter()
        ac, asf, _ = omx.reorder_quantize(x_bits, perm, n)
        y = omx.dequantize_segments(ac, asf) @ Wd.T
        _ = omx.bf16_rne(y)
        dt = time.perf_counter() - t0
        total_rows += rows
        t_total += dt
        rows = max(64, min(M, int(rows * max(1.0, min(4.0, (budget_s - t_total) / max(dt, 1e-3) / 2)))))
    tflops = 2.0 * total_rows * N * K / t_total / 1e12
    sample = (f"{total_rows} activation rows ({total_rows / M:.2f} x the M={M} batch; reorder-quantize + fp64 "
              f"GEMM vs {'all ' if N == n_all else ''}{N}{'' if N == n_all else f' of the {n_all}'} output channels) "
              f"in {t_total:.1f} s; weights quantized offline (untimed)")
    return tflops, sample, total_rows / t_total


def run_reference(args, rank, world):
    if rank != 0:
        return
    M, K, N, text = CONFIGS[args.config]
    vals = []
    sample = ""
    threads = 1
    per = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    n = None
    for i in range(args.warmup + args.steps):
        v, sample, _, threads, n = oracle_cpu_rate(M, K, N, budget_s=per)
        if i >= args.warmup:
            vals.append(v)
    v = statistics.median(vals)
    ms = 2.0 * M * N * K / (v * 1e12) * 1e3
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong" if world > 1 and args.config == "llama70b_down" else "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": text, "M": M, "K": K, "N": N, "n4_n6_n8": [int(c) for c in n],
                      "calibration_rows": calib_rows_for(K)},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                            "host": host_facts(), "per_step_tflops": stats(vals)},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def build_layer(M, K, N, n_sets, device, layer=0, calib_rows=16384, n_shard=None, rank=0, world=1):
    """Offline part (untimed): calibrate on a calibration draw, quantize n_sets
    distinct weight matrices, allocate n_sets activation / output buffers."""
    import paper_2508_02343_b200 as mm
    from synth import gen_act, gen_weight
    # calibration draw generated on the host (the oracle arm calibrates on the very same
    # BF16 rows, so both arms quantize with the same plan)
    cal_x = gen_act(calib_rows, K, 1000 + layer, 2000 + 10 * layer).to(device)
    plan = mm.mm_calibrate_thresholds(cal_x)
    del cal_x
    Ns = N if n_shard is None else N // world
    sets = []
    for i in range(n_sets):
        x = gen_act(M, K, 1000 + layer, 2001 + 10 * layer + 100 * i, device=device)
        w = gen_weight(N, K, 3000 + layer + 100 * i, device=device)
        if n_shard is not None:
            w = w[rank * Ns:(rank + 1) * Ns].contiguous()
        wq = mm.mm_quantize_weight_offline(w, plan)
        del w
        a = mm.MXTensor(plan, M, device)
        y = torch.empty(M, N if n_shard is not None else Ns, dtype=torch.bfloat16, device=device)
        sets.append(dict(x=x, wq=wq, a=a, y=y))
    torch.cuda.synchronize()
    return plan, sets


LEAD = int(os.environ.get("BENCH_LEAD", "64"))
HOST = {}


def timed_chunks(stream, n_steps, fn, sleep_ms, lead=None, mark=None):
    """n_steps calls of fn(i) back to back on `stream`, split into R = min(5, n_steps)
    chunks with one event between chunks, pre-queued behind a device sleep so the
    events time device execution.  `lead` untimed calls run between the sleep and the
    first event: the SM clock drops during the one-thread sleep kernel and needs ~1-2 ms
    of load to come back, which a short timed region would otherwise absorb.
    `mark()` (if given) runs between the lead-in and the timed calls.
    Returns (total ms, [ms per step of each chunk])."""
    lead = LEAD if lead is None else lead
    R = max(1, min(5, n_steps))
    bounds = [lead + round(j * n_steps / R) for j in range(R + 1)]
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(R + 1)]
    torch.cuda._sleep(int((sleep_ms + 0.3 * lead) * 1e-3 * 1.9e9))
    for i in range(lead):
        fn(i)
    if mark is not None:
        mark()
    t0 = time.perf_counter()
    evs[0].record(stream)
    for j in range(R):
        for i in range(bounds[j], bounds[j + 1]):
            fn(i)
        evs[j + 1].record(stream)
    HOST["enqueue_us_per_step"] = (time.perf_counter() - t0) * 1e6 / max(1, n_steps)
    torch.cuda.synchronize()
    per = [evs[j].elapsed_time(evs[j + 1]) / max(1, bounds[j + 1] - bounds[j]) for j in range(R)]
    return evs[0].elapsed_time(evs[R]), per


def kernel_passes(stream, steps, fn, reps=5):
    """`reps` passes of `steps` back-to-back launches of ONE kernel (fn(i)), each
    bracketed by two events -> average launch duration per pass (ms)."""
    out = []
    for _ in range(reps):
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(min(400.0, 1.0 + 0.2 * (steps + LEAD)) * 1e-3 * 1.9e9))
        for i in range(LEAD):   # untimed lead-in launches (clock ramp, see timed_chunks)
            fn(i)
        k0.record(stream)
        for i in range(LEAD, LEAD + steps):
            fn(i)
        k1.record(stream)
        torch.cuda.synchronize()
        out.append(k0.elapsed_time(k1) / steps)
    return out


def measure_shape(M, K, N, dev, stream, pk, launches=10, layer=0):
    """Extra driver-observed single-GPU shape: RQ and GEMM alone, 5 passes of
    `launches` back-to-back launches over 2 rotating sets (each set > L2)."""
    import paper_2508_02343_b200 as mm
    plan, sets = build_layer(M, K, N, 2, dev, layer=layer, calib_rows=calib_rows_for(K))
    with torch.cuda.stream(stream):
        for st in sets:
            mm.mm_reorder_quantize_act(st["x"], plan, out=st["a"], stream=stream)
            mm.mm_mixed_gemm_bf16(st["a"], st["wq"], plan, out=st["y"], stream=stream)
        torch.cuda.synchronize()
        rq = kernel_passes(stream, launches, lambda i: mm.mm_reorder_quantize_act(
            sets[i % 2]["x"], plan, out=sets[i % 2]["a"], stream=stream))
        gm = kernel_passes(stream, launches, lambda i: mm.mm_mixed_gemm_bf16(
            sets[i % 2]["a"], sets[i % 2]["wq"], plan, out=sets[i % 2]["y"], stream=stream))
    n = plan.n
    rq_ms, gm_ms = statistics.median(rq), statistics.median(gm)
    rq_gbs = rq_bytes(M, n) / (rq_ms * 1e-3) / 1e9
    tf = 2.0 * M * N * K / (gm_ms * 1e-3) / 1e12
    pmix = mix_peak_tflops(n, pk)
    del sets
    torch.cuda.empty_cache()
    return {"M": M, "K": K, "N": N, "n4_n6_n8": list(n), "rq_us": rq_ms * 1e3, "rq_gbs": rq_gbs,
            "rq_frac_hbm": rq_gbs / pk["hbm_gbs"], "gemm_us": gm_ms * 1e3, "gemm_tflops": tf,
            "gemm_frac_mix_peak": tf / pmix, "rq_us_stats": stats([v * 1e3 for v in rq]),
            "gemm_us_stats": stats([v * 1e3 for v in gm])}


def run_gpu(args, rank, world, local):
    import paper_2508_02343_b200 as mm
    M, K, N, text = CONFIGS[args.config]
    dev = torch.device("cuda", local)
    if args.gemm_bn or args.gemm_stages:
        mm.mm_set_gemm_config(args.gemm_bn, args.gemm_stages, 0)
    pk = peaks()
    nshard = args.config == "llama70b_down" and (world > 1 or args.comm == "peer")
    use_peer = nshard and args.comm == "peer"
    comm = win = y_peer = None
    fused_err = None
    if nshard:
        from paper_2508_02343_b200.dist import exchange_unique_id
        comm = mm.mm_comm_init(rank, world, exchange_unique_id(mm.nccl_unique_id)) if world > 1 else \
            mm.mm_comm_init(0, 1, mm.nccl_unique_id())
    if nshard and (use_peer or (world > 1 and not args.no_fused)):
        # fused all-gather epilogue: tiles stored into every rank's Y over NVLink
        if world > 1:
            from paper_2508_02343_b200.dist import open_peer_window
            try:
                win, y_peer = open_peer_window(M, N)   # collective; fails on every rank together
            except RuntimeError as e_:
                if use_peer:
                    raise
                win, y_peer, fused_err = None, None, str(e_)
        else:
            buf = mm.peer_buffer(M, N, device=dev)
            win, y_peer = mm.PeerWindow.from_ptrs(0, 1, [buf], M, N), mm.peer_y(buf, M, N)
    if win is not None:
        win.set_timeout(60.0)   # a rank that never arrives must not hang the box
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    # bytes touched per step (for the L2 rotation count)
    Ns = N // world if nshard else N
    per_set = 2 * M * K + M * K + Ns * K + 2 * M * N
    n_sets = max(2, min(16, -(-3 * l2 // per_set)))
    if args.config == "cfg1":
        n_sets = 2
    plan, sets = build_layer(M, K, N, n_sets, dev, n_shard=(True if nshard else None), rank=rank, world=world,
                             calib_rows=calib_rows_for(K))
    n = plan.n
    stage = torch.empty(M * N, dtype=torch.bfloat16, device=dev) if nshard else None
    stream = torch.cuda.Stream(dev)

    def gemm(st, y=None, peer=use_peer):
        if nshard and peer:
            mm.mm_mixed_gemm_bf16_nshard_peerstore(st["a"], st["wq"], plan, N, win, barrier=True, stream=stream)
        elif nshard:
            mm.mm_mixed_gemm_bf16_nshard_allgather(st["a"], st["wq"], plan, N, comm, out=st["y"] if y is None else y,
                                                   stage=stage, stream=stream)
        else:
            mm.mm_mixed_gemm_bf16(st["a"], st["wq"], plan, out=st["y"] if y is None else y, stream=stream)

    def step(i, peer=use_peer):
        s = sets[i % n_sets]
        mm.mm_reorder_quantize_act(s["x"], plan, out=s["a"], stream=stream)
        gemm(s, peer=peer)

    sleep_ms = min(400.0, 1.0 + 0.3 * args.steps) * (20.0 if nshard else 1.0)
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
        # keep the clocks honest: ~0.3 s of identical steps just before the timed region,
        # sampled together with it
        sampler = ClockSampler(local)
        sampler.start()
        t_end = time.time() + 0.3
        i = 0
        while time.time() < t_end:
            step(i)
            i += 1
            if i % 64 == 0:
                stream.synchronize()
        stream.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        lc = {}
        # K steps back to back (only chunk-boundary events in the stream, so consecutive
        # kernels keep their programmatic-dependent-launch overlap)
        total_ms, chunk_ms = timed_chunks(stream, args.steps, step, min(400.0, sleep_ms),
                                          mark=lambda: lc.setdefault("l0", mm.launch_count()))
        barrier(world)
        launches = mm.launch_count() - lc["l0"]
        host_us = HOST.get("enqueue_us_per_step")
        # per-kernel passes: that kernel's average launch duration over the same rotation
        rq_pass = kernel_passes(stream, args.steps, lambda i: mm.mm_reorder_quantize_act(
            sets[i % n_sets]["x"], plan, out=sets[i % n_sets]["a"], stream=stream))
        gemm_pass = kernel_passes(stream, args.steps, lambda i: gemm(sets[i % n_sets]))
        extra_nshard = {}
        if nshard and world > 1:
            # the N-shard GEMM alone (no exchange) and the bare collective on the same bytes
            gemm_only = kernel_passes(stream, args.steps, lambda i: mm.mm_mixed_gemm_bf16(
                sets[i % n_sets]["a"], sets[i % n_sets]["wq"], plan, out=stage[: M * Ns].view(M, Ns), stream=stream))
            import torch.distributed as dist
            src = stage[rank * M * Ns:(rank + 1) * M * Ns]
            ag = []
            for _ in range(5):
                barrier(world)
                e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0_.record(stream)
                for _i in range(args.steps):
                    dist.all_gather_into_tensor(stage, src)
                e1_.record(stream)
                torch.cuda.synchronize()
                ag.append(e0_.elapsed_time(e1_) / args.steps)
            ag_ms = max_over_ranks(statistics.median(ag), world)
            extra_nshard = {
                "gemm_shard_us": max_over_ranks(statistics.median(gemm_only), world) * 1e3,
                "allgather_us": ag_ms * 1e3,
                "allgather_busbw_gbs": (world - 1) / world * (2 * M * N) / (ag_ms * 1e-3) / 1e9,
                "allgather_bytes": 2 * M * N,
                "allgather_note": "torch.distributed all_gather_into_tensor (NCCL) of the same BF16 bytes, "
                                  "busbw = (G-1)/G x bytes / time"}
            mwin, nvls_err = None, None
            if mm.mc_supported():   # NVLS: each element written once via multimem.st, switch replicates
                try:
                    mwin = mm.McWindow.create(M, N)   # collective; fails on every rank together
                    mwin.set_timeout(60.0)
                except mm.MMError as e_:
                    nvls_err = str(e_)
            if mwin is not None:
                try:
                    def nvls_step(i):
                        st_ = sets[i % n_sets]
                        mm.mm_reorder_quantize_act(st_["x"], plan, out=st_["a"], stream=stream)
                        mm.mm_mixed_gemm_bf16_nshard_nvls(st_["a"], st_["wq"], plan, N, mwin, barrier=True,
                                                          stream=stream)
                    for i in range(args.warmup):
                        nvls_step(i)
                    barrier(world)
                    torch.cuda.synchronize()
                    v_total, _ = timed_chunks(stream, args.steps, nvls_step, min(400.0, sleep_ms))
                    barrier(world)
                    v_ms = max_over_ranks(v_total, world) / args.steps
                    extra_nshard["nvls_allgather"] = {
                        "value": 2.0 * M * N * K / (v_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": v_ms,
                        "what": "RQ + GEMM whose epilogue writes each element once through a multicast object "
                                "(multimem.st over NVLink SHARP) + multimem.red flag barrier"}
                finally:
                    torch.cuda.synchronize()
                    barrier(world)
                    mwin.close()
            else:
                extra_nshard["nvls_allgather"] = "unavailable: " + (nvls_err or "this GPU cannot create multicast objects")
            if win is None:
                extra_nshard["fused_allgather"] = "unavailable: " + (fused_err or "not run")
            if win is not None:   # the fused all-gather epilogue on the same ranks
                barrier(world)
                torch.cuda.synchronize()
                f_total, f_chunks = timed_chunks(stream, args.steps, lambda i: step(i, peer=True),
                                                 min(400.0, sleep_ms))
                barrier(world)
                f_ms = max_over_ranks(f_total, world) / args.steps
                extra_nshard["fused_allgather"] = {
                    "value": 2.0 * M * N * K / (f_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": f_ms,
                    "what": "RQ + GEMM with every tile TMA-stored into every rank's Y over peer memory + flag "
                            "barrier (mm_mixed_gemm_bf16_nshard_peerstore)"}
        clocks = sampler.stop()
    total_ms = max_over_ranks(total_ms, world)
    ms = total_ms / args.steps
    flops_rank = 2.0 * M * Ns * K
    units = flops_rank * world * args.steps                       # all ranks' useful FLOPs
    value = units / (total_ms * 1e-3) / 1e12
    rq_ms, gemm_ms = statistics.median(rq_pass), statistics.median(gemm_pass)
    gemm_tflops = flops_rank / (gemm_ms * 1e-3) / 1e12
    kpad = sum(plan.padded_cols(g) for g in range(3))
    pmix = mix_peak_tflops(n, pk)
    rqb = rq_bytes(M, n)
    rq_gbs = rqb / (rq_ms * 1e-3) / 1e9

    # ---- end to end through the public API with host buffers --------------------------
    # Every step copies its X from pinned host memory, runs RQ + GEMM and copies Y back.
    # The copies run on their own streams, double-buffered over two device slots, so
    # step i's H2D, step i-1's compute and step i-2's D2H overlap (PCIe is full duplex);
    # the peer-store path has one Y window and runs the steps serially.
    x_host = sets[0]["x"].cpu().pin_memory()
    y_hosts = [torch.empty(M, N, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    pipelined = not use_peer
    slots = [sets[0], sets[1 % n_sets]] if pipelined else [sets[0]]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("in", "rq", "comp", "out")}

    def e2e_step(i):
        b = i % len(slots)
        st = slots[b]
        y_dev = y_peer if use_peer else st["y"]
        if not pipelined:
            with torch.cuda.stream(stream):
                st["x"].copy_(x_host, non_blocking=True)
                mm.mm_reorder_quantize_act(st["x"], plan, out=st["a"], stream=stream)
                gemm(st, y_dev)
                y_hosts[0].copy_(y_dev[:, :N] if y_dev.shape[1] != N else y_dev, non_blocking=True)
            return
        s_in.wait_event(ev["rq"][b])                  # X slot consumed by the RQ of step i-2
        with torch.cuda.stream(s_in):
            st["x"].copy_(x_host, non_blocking=True)
        ev["in"][b].record(s_in)
        stream.wait_event(ev["in"][b])
        mm.mm_reorder_quantize_act(st["x"], plan, out=st["a"], stream=stream)
        ev["rq"][b].record(stream)
        stream.wait_event(ev["out"][b])               # Y slot read back by the D2H of step i-2
        gemm(st, y_dev)
        ev["comp"][b].record(stream)
        s_out.wait_event(ev["comp"][b])
        with torch.cuda.stream(s_out):
            y_hosts[b].copy_(y_dev, non_blocking=True)
        ev["out"][b].record(s_out)

    for k in ev:
        for e_ in ev[k]:
            e_.record(stream)
    for i in range(max(3, args.warmup)):
        e2e_step(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    e0.record(stream)
    s_in.wait_event(e0)
    s_out.wait_event(e0)
    for i in range(args.steps):
        e2e_step(i)
    stream.wait_stream(s_out)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    e2e_val = units / (e2e_ms * 1e-3) / 1e12
    if comm is not None:
        mm.mm_comm_destroy(comm)
    if win is not None:
        barrier(world)   # no rank unmaps while a peer may still store into it
        win.close()

    large = None
    large_more = []
    if world == 1 and args.large and args.config == "q_proj":
        M3, K3, N3 = 16384, 14336, 4096
        large = measure_shape(M3, K3, N3, dev, stream, pk, layer=1)
        large["workload"] = "Llama-3.1-8B down_proj at batch 8 x seq 2048 (BASELINE configs[2], b8 down)"
        # the other BASELINE shapes the driver can observe on one GPU: b8 q/o (configs[2])
        # and the north-star 70B down_proj unsharded (configs[3] at N = 1)
        for (Mx, Kx, Nx, layer, what) in ((16384, 4096, 4096, 2, "Llama-3.1-8B q/o_proj at batch 8 x seq 2048 "
                                                                  "(BASELINE configs[2], b8 q/o)"),
                                          (8192, 28672, 8192, 3, "Llama-3.1-70B down_proj, 1 GPU (BASELINE "
                                                                 "configs[3] unsharded)")):
            r = measure_shape(Mx, Kx, Nx, dev, stream, pk, layer=layer)
            r["workload"] = what
            large_more.append(r)

    if rank != 0:
        return
    # ---- CPU baseline (oracle as it stands, bounded sample) -----------------------------
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, sample, _, threads, _ = oracle_cpu_rate(M, K, N, budget_s=args.cpu_seconds)
        v1, sample1, _, _, _ = oracle_cpu_rate(M, K, N, budget_s=max(3.0, args.cpu_seconds / 2), threads=1)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
               "host": host_facts(), "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "sample": sample1}}

    traffic_src = None
    tr = {}
    if args.traffic:
        try:
            with open(os.path.join(ROOT, args.traffic)) as f:
                tr = json.load(f)
            traffic_src = (f"{args.traffic}: ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per "
                           f"launch, captured {tr.get('captured', '?')} at commit {tr.get('commit', '?')} "
                           f"(static file, not re-measured by this run)")
        except Exception:
            tr = {}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if nshard else "weak", "vs_baseline": None,
        "dtype": "mxfp4/mxfp6(e3m2)/mxfp8(e4m3) x e8m0, fp32 accum, bf16 out", "data": "synthetic",
        "config": {"workload": text, "M": M, "K": K, "N": N, "n4_n6_n8": list(n),
                   "calibration_rows": calib_rows_for(K),
                   "parallelism": ((f"N-shard x{world} + NCCL all-gather" if not use_peer else
                                    f"N-shard x{world}, all-gather fused into the GEMM epilogue (peer stores)")
                                   if nshard else
                                   ("replicas" if world > 1 else "1 GPU")),
                   "l2": f"{n_sets} rotating input/weight/output sets, {n_sets * per_set / 1e6:.0f} MB > L2 "
                         f"{l2 / 1e6:.0f} MB (inputs differ from step to step; no L2 flush)",
                   "timing": "CUDA events on the launching stream; steps pre-queued behind a device sleep "
                             f"and {LEAD} untimed lead-in steps (the SM clock drops during the one-thread sleep "
                             "kernel and takes ~1-2 ms of load to recover) "
                             "(device time; host enqueue cost is in e2e); value/ms_per_step from the whole region "
                             "(R <= 5 chunks, one event between chunks); per-kernel durations (breakdown, roofline) "
                             "= median of 5 passes of K back-to-back launches of that kernel alone"},
        "ms_per_step_stats": stats(chunk_ms),
        "breakdown": {"rq_us": rq_ms * 1e3, "gemm_us": gemm_ms * 1e3,
                      "rq_us_stats": stats([v * 1e3 for v in rq_pass]),
                      "gemm_us_stats": stats([v * 1e3 for v in gemm_pass]),
                      "rq_gbs": rq_gbs, "rq_frac_hbm": rq_gbs / pk["hbm_gbs"],
                      "gemm_tflops": gemm_tflops, "gemm_tflops_padded_k": gemm_tflops * kpad / K,
                      "k_padded": kpad, "gemm_mix_peak_tflops": pmix,
                      "gemm_frac_mix_peak": gemm_tflops / pmix,
                      "peaks": f"{pk['src']}: HBM {pk['hbm_gbs']:.0f} GB/s, bf16 {pk['bf16']:.0f} TF/s "
                               f"(fp8 = 2x, fp4 = 4x)"},
        "roofline": {"bound": "tensor", "achieved": gemm_tflops, "peak": pmix, "unit": "TFLOP/s",
                     "frac": gemm_tflops / pmix, "traffic": tr.get("mixgemm"), "traffic_source": traffic_src,
                     "kernel": "mixgemm2_kernel (CTA-pair tcgen05; algorithmic 2*M*N*K per launch; "
                               "mix-weighted MXFP4/FP8 peak)" + ("; N-shard: GEMM + all-gather + layout" if nshard
                                                                else "")},
        "rq_roofline": {"bound": "hbm", "achieved": rq_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": rq_gbs / pk["hbm_gbs"], "traffic": tr.get("rq"), "traffic_source": traffic_src,
                        "kernel": "rq_kernel (algorithmic BF16 read + packed codes + scales)"},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 2 * M * K,
                "d2h_bytes_per_step": 2 * M * N,
                "pipeline": ("H2D, RQ + GEMM and D2H on three streams over two device slots (copies of "
                             "neighbouring steps overlap compute)" if pipelined else "serial")},
        "gpu_launches": launches,
        "host_enqueue_us_per_step": host_us,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    if extra_nshard:
        out["nshard"] = extra_nshard
    if large is not None:
        out["large_shape"] = large
    if large_more:
        out["more_shapes"] = large_more
    print(json.dumps(out), flush=True)


def relaunch_under_torchrun(n):
    """`--gpus N` (N > 1) without a torch.distributed environment: run this same
    command under torch.distributed.run with N local ranks and exit with its code."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=dict(os.environ)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="micromix", choices=["micromix", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: q_proj at N=1 (configs[1]), llama70b_down N-shard at N>1 (configs[3])")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "peer"],
                    help="N-shard output exchange of the headline value: NCCL all-gather, or the fused "
                         "peer-store epilogue")
    ap.add_argument("--no-fused", action="store_true", help="N>1: skip timing the fused all-gather epilogue")
    ap.add_argument("--large", type=int, default=1, help="N=1: also time the b8 down_proj shape (1/0)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gemm-bn", type=int, default=0, help="GEMM tile N override (tuning)")
    ap.add_argument("--gemm-stages", type=int, default=0, help="GEMM pipeline stages override (tuning)")
    ap.add_argument("--traffic", default="profiles/traffic_r02l.json",
                    help="ncu dram bytes per launch (written from an ncu --set full capture)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        relaunch_under_torchrun(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config is None:
        args.config = "llama70b_down" if max(world, args.gpus if args.impl == "reference" else 1) > 1 else "q_proj"
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, rank, world)
        return
    rank, world, local = dist_init()
    run_gpu(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
