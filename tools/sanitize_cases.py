"""Small launches of every kernel for compute-sanitizer (SURVEY §4.2 tier T3):
racecheck / synccheck / memcheck / initcheck over the RQ (plain and fused RMSNorm),
the CTA-pair GEMM (config 1, 256^3 and the balanced schedule; W scales multicast across
the pair), the single-CTA tile GEMM, the small-M
split-K GEMM (arrival counters), the opt-in stream-K schedule (per-warp flags) and
the fused all-gather epilogue with 2 virtual ranks + the flag barrier.
Run: compute-sanitizer --tool <t> python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
from synth import gen_act, gen_perm, gen_uniform_bf16, gen_weight  # noqa: E402


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print(f"case ok: {name}", flush=True)


def gemm(M, N, n, bn=0, env=None):
    K = sum(n)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 5))
    if env:
        os.environ.update(env)
    mm.mm_set_gemm_config(bn, 0, 0)
    try:
        a = mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2001).cuda(), plan)
        w = mm.mm_quantize_weight_offline(gen_weight(N, K, 3000).cuda(), plan)
        mm.mm_mixed_gemm_bf16(a, w, plan)
        mm.mm_mixed_gemm_bf16(a, w, plan)     # second call re-uses the zeroed counters/flags
    finally:
        mm.mm_set_gemm_config(0, 0, 0)
        if env:
            for k in env:
                os.environ.pop(k)


def rq_norm():
    K = 4096
    plan = mm.mm_plan_init(K, (2240, 1184, 672), gen_perm(K, 6))
    g = gen_uniform_bf16((K,), 0.5, 1.5, 7).cuda()
    mm.mm_rmsnorm_reorder_quantize_act(gen_act(64, K, 1000, 2002).cuda(), g, 1e-5, plan)


def peerstore():
    M, Ns, G, n = 300, 256, 2, (256, 128, 128)
    K = sum(n)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 8))
    a = mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2001).cuda(), plan)
    w = gen_weight(Ns * G, K, 3000).cuda()
    shards = [mm.mm_quantize_weight_offline(w[r * Ns:(r + 1) * Ns].contiguous(), plan) for r in range(G)]
    bufs = [mm.peer_buffer(M, Ns * G) for _ in range(G)]
    wins = [mm.PeerWindow.from_ptrs(r, G, bufs, M, Ns * G) for r in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    try:
        for r in range(G):
            mm.mm_mixed_gemm_bf16_nshard_peerstore(a, shards[r], plan, Ns * G, wins[r], barrier=False)
        ev = torch.cuda.Event()
        ev.record()
        for r in range(G):
            streams[r].wait_event(ev)
            mm.mm_peer_barrier(wins[r], stream=streams[r])
        torch.cuda.synchronize()
    finally:
        for wn in wins:
            wn.close()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    case("rq cfg1 M=16 K=256", lambda: mm.mm_reorder_quantize_act(
        gen_act(16, 256, 1000, 2001).cuda(), mm.mm_plan_init(256, (128, 64, 64), gen_perm(256, 4))))
    case("rq M=300 K=4096 (2-row tiles)", lambda: mm.mm_reorder_quantize_act(
        gen_act(300, 4096, 1000, 2001).cuda(), mm.mm_plan_init(4096, (2240, 1184, 672), gen_perm(4096, 4))))
    case("rq M=40 K=28672 (1-row tiles)", lambda: mm.mm_reorder_quantize_act(
        gen_act(40, 28672, 1000, 2001).cuda(), mm.mm_plan_init(28672, (16384, 8192, 4096), gen_perm(28672, 4))))
    case("rmsnorm+rq M=64 K=4096", rq_norm)
    case("pair GEMM cfg1-shape M=16 N=256 K=256 (forced)", lambda: gemm(16, 256, (128, 64, 64), bn=512))
    case("pair GEMM 256^3", lambda: gemm(256, 256, (128, 64, 64)))
    case("pair GEMM M=300 N=784 K=4096", lambda: gemm(300, 784, (2240, 1184, 672)))
    case("tile GEMM bn=256 M=100 N=512", lambda: gemm(100, 512, (256, 128, 128), bn=256))
    case("small-M split-K M=16 N=4096 K=4096", lambda: gemm(16, 4096, (2240, 1184, 672)))
    case("stream-K M=2560 N=2048 K=256", lambda: gemm(2560, 2048, (128, 64, 64), env={"MM_GEMM_STREAMK": "1"}))
    case("balanced schedule M=2560 N=2048 K=256 (64-column items)", lambda: gemm(2560, 2048, (128, 64, 64)))
    case("balanced schedule M=2048 N=4096 K=256 (192-column items, SFB offset)", lambda: gemm(2048, 4096, (128, 64, 64)))
    case("peer-store 2 virtual ranks + barrier", peerstore)
    print("all cases ok")
