"""Time mm_mixed_gemm_bf16 alone for several segment splits at one shape (tuning aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
from synth import gen_act, gen_perm, gen_weight  # noqa: E402


def time_gemm(M, N, n, reps=20):
    K = sum(n)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 1))
    x = gen_act(M, K, 1000, 2001, device="cuda")
    w = gen_weight(N, K, 3000, device="cuda")
    a = mm.mm_reorder_quantize_act(x, plan)
    wq = mm.mm_quantize_weight_offline(w, plan)
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        mm.mm_mixed_gemm_bf16(a, wq, plan, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # pre-queue a device sleep so the host enqueue of all reps hides behind it: the
    # events then time device execution only (small-M launches are shorter than the
    # Python + tensor-map encode cost per call)
    torch.cuda._sleep(int(2e-3 * 1.9e9))
    e0.record()
    for _ in range(reps):
        mm.mm_mixed_gemm_bf16(a, wq, plan, out=y)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    return us, 2.0 * M * N * K / (us * 1e-6) / 1e12


if __name__ == "__main__":
    M, N = int(sys.argv[1]), int(sys.argv[2])
    mm.mm_set_gemm_config(int(os.environ.get("BN", "0")), int(os.environ.get("STAGES", "0")),
                          int(os.environ.get("MAXCTAS", "0")))
    splits = [tuple(int(v) for v in a.split(",")) for a in sys.argv[3:]] or [
        (4096, 0, 0), (0, 4096, 0), (0, 0, 4096), (2240, 1184, 672)]
    for n in splits:
        us, tf = time_gemm(M, N, n)
        print(f"M={M} N={N} n={n}: {us:8.1f} us  {tf:7.0f} TFLOP/s  dbg={os.environ.get('MM_GEMM_DEBUG', '0')}",
              flush=True)
