"""Library context for the mixed GEMM: cuBLASLt block-scaled MXFP8 / MXFP4 GEMMs
(torch.nn.functional.scaled_mm, BlockWise1x32 E8M0 scales, 32_4_4 swizzle) on the
BASELINE shapes, timed like tools/sweep_configs.py (back-to-back launches over
rotating operand sets > L2, CUDA events).  These are the single-format library
GEMMs the paper's decoupled design would call per segment; our kernel
runs all three segments in one K loop.  Not a product path; prints a markdown
table (also written to gpurun_out/cublas_mx.md).

    python tools/cublas_mx_baseline.py
"""
from __future__ import annotations

import json
import os
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SHAPES = [
    ("C2 Llama-3.1-8B q_proj", 2048, 4096, 4096),
    ("C3 b1 gate_up", 2048, 4096, 28672),
    ("C3 b8 o", 16384, 4096, 4096),
    ("C3 b8 down", 16384, 14336, 4096),
    ("C4 Llama-3.1-70B down_proj", 8192, 28672, 8192),
    ("C5 Qwen2.5-32B gate_up", 8192, 5120, 55296),
]


def peaks():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        p = json.load(f)
    return 2 * float(p["bf16_tflops"]), 4 * float(p["bf16_tflops"])


def scales(rows, K, dev):
    r = (rows + 127) // 128 * 128
    c = (K // 32 + 3) // 4 * 4
    return torch.full((r * c,), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)


def operands(fmt, M, K, N, dev):
    if fmt == "fp8":
        a = (torch.randn(M, K, device=dev) * 0.5).to(torch.float8_e4m3fn)
        b = (torch.randn(N, K, device=dev) * 0.5).to(torch.float8_e4m3fn)
    else:
        a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
    return a, b, scales(M, K, dev), scales(N, K, dev)


def run(fmt, M, K, N, dev, iters=20):
    bw = F.ScalingType.BlockWise1x32
    sw = F.SwizzleType.SWIZZLE_32_4_4
    per = M * K + N * K + 2 * M * N
    nsets = max(1, min(8, int(3 * 126e6 // per) + 1))
    sets = [operands(fmt, M, K, N, dev) for _ in range(nsets)]
    outs = []

    def call(i):
        a, b, sa, sb = sets[i % nsets]
        return F.scaled_mm(a, b.t(), sa, bw, sb, bw, swizzle_a=sw, swizzle_b=sw, output_dtype=torch.bfloat16)

    for i in range(3):
        outs.append(call(i))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        call(i)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    return us, 2.0 * M * N * K / (us * 1e-6) / 1e12


def run_ours(fmt, M, K, N, dev, iters=20):
    """Our mixed GEMM with a single-format plan (all-FP8 E4M3 or all-FP4), same timing."""
    sys.path.insert(0, ROOT)
    import paper_2508_02343_b200 as mm
    from synth import gen_act, gen_perm, gen_weight
    n = (0, 0, K) if fmt == "fp8" else (K, 0, 0)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 5))
    per = M * K + N * K + 2 * M * N
    nsets = max(1, min(8, int(3 * 126e6 // per) + 1))
    aa = [mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2001 + i, device=dev), plan) for i in range(nsets)]
    ws = [mm.mm_quantize_weight_offline(gen_weight(N, K, 3000 + i, device=dev), plan) for i in range(nsets)]
    ys = [torch.empty(M, N, dtype=torch.bfloat16, device=dev) for _ in range(nsets)]
    for i in range(3):
        mm.mm_mixed_gemm_bf16(aa[i % nsets], ws[i % nsets], plan, out=ys[i % nsets])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        mm.mm_mixed_gemm_bf16(aa[i % nsets], ws[i % nsets], plan, out=ys[i % nsets])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    return us, 2.0 * M * N * K / (us * 1e-6) / 1e12


def main():
    dev = torch.device("cuda:0")
    p8, p4 = peaks()
    lines = ["| layer | M | K | N | cuBLASLt MXFP8 us | ours all-FP8 us | cuBLASLt MXFP4 us | ours all-FP4 us |",
             "|---|---|---|---|---|---|---|---|"]
    for name, M, K, N in SHAPES:
        row = [name, str(M), str(K), str(N)]
        for fmt, pk in (("fp8", p8), ("fp4", p4)):
            for fn in (run, run_ours):
                try:
                    us, tf = fn(fmt, M, K, N, dev)
                    row += [f"{us:.1f} ({100 * tf / pk:.0f}%)"]
                except Exception as e:  # report, do not hide
                    row += [f"n/a ({type(e).__name__}: {str(e).splitlines()[0][:60]})"]
        lines.append("| " + " | ".join(row) + " |")
        print(lines[-1], flush=True)
    txt = (f"peaks: FP8 {p8:.0f} TF/s, FP4 {p4:.0f} TF/s (2x / 4x measured bf16); (%) = share of that peak\n\n"
           + "\n".join(lines) + "\n")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "cublas_mx.md"), "w") as f:
        f.write(txt)
    print(txt)


if __name__ == "__main__":
    sys.exit(main())
