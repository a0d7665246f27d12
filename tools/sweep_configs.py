"""Measure every BASELINE.json config on one GPU (tuning / reporting aid):

  C1  single linear M=16 K=256 N=256, fixed 128/64/64 split (latency-bound; CUDA-graph timed)
  C2  Llama-3.1-8B q_proj M=2048 K=4096 N=4096, calibrated
  C3  Llama-3.1-8B prefill linear set (qkv 4096->6144, o 4096->4096, gate_up 4096->28672,
      down 14336->4096) at batch 1/8/32 x seq 2048; one RQ per distinct input (qkv and
      gate_up share theirs)
  C4  Llama-3.1-70B down_proj M=8192 K=28672 N=8192 on 1 GPU (the N-shard rows are
      measured by bench.py --config llama70b_down under torchrun)
  C5  Qwen2.5-32B MLP (gate_up fused K=5120 N=55296, down K=27648 N=5120) at M=8192 over
      the precision-mix sweep all-FP4 -> all-FP8 (counts rounded to 128) plus a non-128 split

Every kernel time = K back-to-back launches of that kernel over >= 2 rotating input sets
(> L2 for all but C1/C2-sized layers, which use 8 sets) / K, CUDA events.  Prints one JSON
line per measurement and writes profiles/configs_<tag>.md.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
from synth import gen_act, gen_perm, gen_weight  # noqa: E402

sys.path.insert(0, ROOT)
from bench import mix_peak_tflops, peaks, rq_bytes  # noqa: E402

PK = peaks()
L2 = None


def n_sets_for(bytes_per_set):
    return max(2, min(8, -(-3 * L2 // max(bytes_per_set, 1))))


def time_loop(fn, n, reps):
    for i in range(3):
        fn(i % n)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e6))
    e0.record()
    for i in range(reps):
        fn(i % n)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


def measure_layer(name, M, K, N, plan, reps=20, sets=None, shared_a=None):
    """RQ of X[M, K] and GEMM vs W[N, K]; returns dict."""
    per_set = 2 * M * K + M * K + N * K + 2 * M * N
    ns = n_sets_for(per_set) if sets is None else sets
    xs, ws, aa, ys = [], [], [], []
    for i in range(ns):
        xs.append(gen_act(M, K, 1000, 2001 + 100 * i, device="cuda"))
        w = gen_weight(N, K, 3000 + 100 * i, device="cuda")
        ws.append(mm.mm_quantize_weight_offline(w, plan))
        del w
        aa.append(mm.MXTensor(plan, M))
        ys.append(torch.empty(M, N, dtype=torch.bfloat16, device="cuda"))
    rq_us = time_loop(lambda i: mm.mm_reorder_quantize_act(xs[i], plan, out=aa[i]), ns, reps)
    gemm_us = time_loop(lambda i: mm.mm_mixed_gemm_bf16(aa[i], ws[i], plan, out=ys[i]), ns, reps)
    n = plan.n
    flops = 2.0 * M * N * K
    pm = mix_peak_tflops(n, PK)
    r = {"layer": name, "M": M, "K": K, "N": N, "n4_n6_n8": list(n), "sets": ns,
         "rq_us": rq_us, "rq_gbs": rq_bytes(M, n) / (rq_us * 1e-6) / 1e9,
         "rq_frac_hbm": rq_bytes(M, n) / (rq_us * 1e-6) / 1e9 / PK["hbm_gbs"],
         "gemm_us": gemm_us, "gemm_tflops": flops / (gemm_us * 1e-6) / 1e12, "mix_peak_tflops": pm}
    r["gemm_frac_mix_peak"] = r["gemm_tflops"] / pm
    del xs, ws, aa, ys
    torch.cuda.empty_cache()
    print(json.dumps(r), flush=True)
    return r


def calibrated_plan(K, layer=0, rows=None):
    rows = rows or (16384 if K <= 8192 else 4096)
    x = gen_act(rows, K, 1000 + layer, 2000 + 10 * layer, device="cuda")
    p = mm.mm_calibrate_thresholds(x)
    del x
    return p


def fixed_plan(K, p4, p6, seed=7, round_to=128):
    n4 = int(round(K * p4 / round_to)) * round_to
    n6 = int(round(K * p6 / round_to)) * round_to
    n8 = K - n4 - n6
    if n8 < 0:
        n6 += n8
        n8 = 0
    return mm.mm_plan_init(K, (n4, n6, n8), gen_perm(K, seed))


def c1():
    plan = mm.mm_plan_init(256, (128, 64, 64), gen_perm(256, 11))
    x = gen_act(16, 256, 1000, 2001, device="cuda")
    w = mm.mm_quantize_weight_offline(gen_weight(256, 256, 3000, device="cuda"), plan)
    a = mm.MXTensor(plan, 16)
    y = torch.empty(16, 256, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    # CUDA-graph the step (latency-bound at this size)
    with torch.cuda.stream(s):
        for _ in range(3):
            mm.mm_reorder_quantize_act(x, plan, out=a, stream=s)
            mm.mm_mixed_gemm_bf16(a, w, plan, out=y, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        mm.mm_reorder_quantize_act(x, plan, out=a, stream=s)
        mm.mm_mixed_gemm_bf16(a, w, plan, out=y, stream=s)
    us = time_loop(lambda i: g.replay(), 1, 200)
    r = {"layer": "C1 M=16 K=256 N=256 (graph: RQ + GEMM)", "step_us": us}
    print(json.dumps(r), flush=True)
    return [r]


def c2():
    plan = calibrated_plan(4096)
    return [measure_layer("C2 Llama-3.1-8B q_proj", 2048, 4096, 4096, plan)]


def c6():
    """Decode-like small M (NEXT F3 small-M path): Llama-3.1-8B q_proj and down_proj
    at M = 1 / 16 / 32 / 128 (W read once from HBM is the bound)."""
    out = []
    plan_h = calibrated_plan(4096, layer=0)
    plan_d = calibrated_plan(14336, layer=2)
    for M in (1, 16, 32, 128):
        out.append(measure_layer(f"C6 decode q_proj M={M}", M, 4096, 4096, plan_h, sets=8))
        out.append(measure_layer(f"C6 decode down M={M}", M, 14336, 4096, plan_d, sets=8))
    return out


def c3(batches=(1, 8, 32)):
    out = []
    plan_h = calibrated_plan(4096, layer=0)      # input of qkv and gate_up (post-norm hidden)
    plan_o = calibrated_plan(4096, layer=1)      # input of o_proj (attention output)
    plan_d = calibrated_plan(14336, layer=2)     # input of down_proj (MLP activation)
    for b in batches:
        M = 2048 * b
        reps = 20 if b < 32 else 5
        out.append(measure_layer(f"C3 b{b} qkv", M, 4096, 6144, plan_h, reps=reps, sets=2 if b > 1 else None))
        out.append(measure_layer(f"C3 b{b} o", M, 4096, 4096, plan_o, reps=reps, sets=2 if b > 1 else None))
        out.append(measure_layer(f"C3 b{b} gate_up", M, 4096, 28672, plan_h, reps=reps, sets=2 if b > 1 else None))
        out.append(measure_layer(f"C3 b{b} down", M, 14336, 4096, plan_d, reps=reps, sets=2 if b > 1 else None))
    return out


def c4():
    plan = calibrated_plan(28672, layer=3, rows=2048)
    return [measure_layer("C4 Llama-3.1-70B down_proj (1 GPU)", 8192, 28672, 8192, plan, reps=10, sets=2)]


def c5():
    out = []
    mixes = [(1, 0, 0), (.75, .125, .125), (.5, .25, .25), (.25, .375, .375), (0, 1, 0), (0, .5, .5), (0, 0, 1)]
    for (K, N, nm) in ((5120, 55296, "gate_up"), (27648, 5120, "down")):
        for p4, p6, p8 in mixes:
            plan = fixed_plan(K, p4, p6)
            out.append(measure_layer(f"C5 Qwen2.5-32B {nm} mix=({p4},{p6},{p8})", 8192, K, N, plan, reps=5, sets=2))
        plan = calibrated_plan(K, layer=4)
        out.append(measure_layer(f"C5 Qwen2.5-32B {nm} calibrated (non-128 split)", 8192, K, N, plan, reps=5, sets=2))
    return out


def main():
    global L2
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c1", "c2", "c3", "c4", "c5", "c6"]
    torch.cuda.set_device(0)
    L2 = torch.cuda.get_device_properties(0).L2_cache_size
    res = []
    t0 = time.time()
    for w in which:
        res += globals()[w]()
    lines = [f"# Config sweep {tag} (1 x B200)", "",
             "Produced by `python tools/sweep_configs.py`; kernel time = back-to-back launches of that kernel",
             "over rotating input sets / count, CUDA events.  Peaks: " + PK["src"] +
             f" HBM {PK['hbm_gbs']:.0f} GB/s, bf16 {PK['bf16']:.0f} TF/s (FP8/FP6 = 2x, FP4 = 4x).", "",
             "| layer | M | K | N | n4/n6/n8 | RQ us | RQ GB/s (% HBM) | GEMM us | GEMM TF/s | % mix peak |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in res:
        if "step_us" in r:
            lines.append(f"| {r['layer']} | | | | | | | {r['step_us']:.1f} (step) | | |")
            continue
        lines.append(f"| {r['layer']} | {r['M']} | {r['K']} | {r['N']} | {'/'.join(map(str, r['n4_n6_n8']))} | "
                     f"{r['rq_us']:.1f} | {r['rq_gbs']:.0f} ({100 * r['rq_frac_hbm']:.0f}%) | {r['gemm_us']:.1f} | "
                     f"{r['gemm_tflops']:.0f} | {100 * r['gemm_frac_mix_peak']:.0f}% |")
    lines.append("")
    lines.append(f"wall {time.time() - t0:.0f} s")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "profiles",
                           f"configs_{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
