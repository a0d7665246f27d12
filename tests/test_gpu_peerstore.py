"""GPU tests of the fused GEMM + all-gather epilogue over peer memory
(mm_mixed_gemm_bf16_nshard_peerstore).

A test box has one GPU, so the G ranks are VIRTUAL: G peer buffers on the one
device, one window per virtual rank (mm_peer_window_from_ptrs), each rank's GEMM
run with its own weight shard; every rank's kernel stores its tiles into all G
buffers exactly as it would over NVLink, and the flag barriers of all ranks run
concurrently on G streams.  Every buffer must then hold the full 1-GPU output bit
for bit (same tiles, same K order), columns beyond n_total untouched.  The CUDA
IPC path (mm_ipc_get_handle / mm_peer_window_open) is exercised at world size 1
and for the handle's sub-allocation offset; the world-2 handle exchange runs on
CPU in tests/test_dist_gloo.py."""
import numpy as np
import pytest
import torch

import paper_2508_02343_b200 as mm
from synth import bf16_bits, gen_act, gen_perm, gen_weight

from accuracy import ref_and_abs, report

pytestmark = pytest.mark.gpu


def _setup(M, Ns, G, n, seed=31, with_inputs=False):
    K = sum(n)
    N = Ns * G
    plan = mm.mm_plan_init(K, n, gen_perm(K, seed))
    x = gen_act(M, K, 1000, 2001)
    a = mm.mm_reorder_quantize_act(x.cuda(), plan)
    w = gen_weight(N, K, 3000).cuda()
    w_full = mm.mm_quantize_weight_offline(w, plan)
    shards = [mm.mm_quantize_weight_offline(w[r * Ns:(r + 1) * Ns].contiguous(), plan) for r in range(G)]
    y_ref = mm.mm_mixed_gemm_bf16(a, w_full, plan)
    if with_inputs:
        return plan, a, shards, y_ref, x, w.cpu()
    return plan, a, shards, y_ref


def _oracle_check(y, x, w, plan, rows):
    """Sampled rows of a gathered Y against the fp64 oracle (tests/accuracy.py bars)."""
    from oracle.formats import E2M3, E3M2, E4M3, E5M2
    f6 = {mm.MM_E3M2: E3M2, mm.MM_E2M3: E2M3}[plan.fmt6]
    f8 = {mm.MM_E4M3: E4M3, mm.MM_E5M2: E5M2}[plan.fmt8]
    yref, S = ref_and_abs(bf16_bits(x)[rows], bf16_bits(w), plan.perm_host().numpy(), plan.n, f6, f8, plan.rule)
    r = report(bf16_bits(y.cpu())[rows], yref, S, sum(plan.n))
    assert r["bound_violations"] == 0 and r["rel_fro"] <= 2e-3, r


def _virtual_ranks(plan, a, shards, M, Ns, G, ldy, iters=2):
    N = Ns * G
    bufs = [mm.peer_buffer(M, ldy) for _ in range(G)]
    wins = [mm.PeerWindow.from_ptrs(r, G, bufs, M, ldy) for r in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    try:
        for _ in range(iters):     # a second round re-uses the flags (next epoch)
            for r in range(G):
                mm.mm_mixed_gemm_bf16_nshard_peerstore(a, shards[r], plan, N, wins[r], barrier=False)
            ev = torch.cuda.Event()
            ev.record()
            for r in range(G):
                streams[r].wait_event(ev)
                mm.mm_peer_barrier(wins[r], stream=streams[r])
            torch.cuda.synchronize()
    finally:
        for wn in wins:
            wn.close()
    return [mm.peer_y(b, M, ldy) for b in bufs], bufs


@pytest.mark.parametrize("M,Ns,G,n", [(300, 256, 2, (256, 128, 128)), (256, 144, 4, (2240, 1184, 672)),
                                      (520, 512, 8, (512, 256, 256)), (64, 96, 2, (128, 64, 64)),
                                      (2048, 512, 8, (2240, 1184, 672)), (130, 272, 3, (0, 256, 0))])
def test_peerstore_virtual_ranks_equal_1gpu(M, Ns, G, n):
    plan, a, shards, y_ref, x, w = _setup(M, Ns, G, n, with_inputs=True)
    N = Ns * G
    ldy = N + 8                        # a column beyond n_total must stay untouched
    ys, _ = _virtual_ranks(plan, a, shards, M, Ns, G, ldy)
    for r, y in enumerate(ys):
        assert torch.equal(y[:, :N].view(torch.int16), y_ref.view(torch.int16)), f"rank {r} Y differs"
        assert not y[:, N:].view(torch.int16).any(), f"rank {r}: columns past n_total written"
    # the gathered output against the oracle (every 5th row, all N columns)
    _oracle_check(ys[-1][:, :N].contiguous(), x, w, plan, np.arange(0, M, 5))


def test_peerstore_world1_ipc_window():
    M, Ns, n = 200, 512, (256, 128, 128)
    plan, a, shards, y_ref = _setup(M, Ns, 1, n)
    buf = mm.peer_buffer(M, Ns)
    h = mm.ipc_handle(buf)
    assert len(h) == mm.lib().mm_ipc_handle_bytes() == 72
    win = mm.PeerWindow.open(0, 1, buf, [h], M, Ns)
    try:
        mm.mm_mixed_gemm_bf16_nshard_peerstore(a, shards[0], plan, Ns, win, barrier=True)
        torch.cuda.synchronize()
    finally:
        win.close()
    assert torch.equal(mm.peer_y(buf, M, Ns).view(torch.int16), y_ref.view(torch.int16))


def test_ipc_handle_records_suballocation_offset():
    big = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    sub = big[4096:]
    off = int.from_bytes(mm.ipc_handle(sub)[64:], "little")
    off0 = int.from_bytes(mm.ipc_handle(big)[64:], "little")
    assert off - off0 == 4096


def test_peerstore_rejects_bad_arguments():
    M, Ns, G, n = 64, 128, 2, (128, 64, 64)
    plan, a, shards, _ = _setup(M, Ns, G, n)
    bufs = [mm.peer_buffer(M, Ns * G) for _ in range(G)]
    with pytest.raises(mm.MMError):
        mm.PeerWindow.from_ptrs(0, 9, (bufs * 5)[:9], M, Ns * G)   # world > 8
    with pytest.raises(mm.MMError):
        mm.PeerWindow.from_ptrs(2, 2, bufs, M, Ns * G)              # rank >= world
    win = mm.PeerWindow.from_ptrs(0, G, bufs, M, Ns * G)
    try:
        with pytest.raises(mm.MMError):
            mm.mm_mixed_gemm_bf16_nshard_peerstore(a, shards[0], plan, Ns * G + 16, win, barrier=False)
        a2 = mm.mm_reorder_quantize_act(gen_act(M + 16, sum(n), 1000, 2002).cuda(), plan)
        with pytest.raises(mm.MMError):                              # rows != window M
            mm.mm_mixed_gemm_bf16_nshard_peerstore(a2, shards[0], plan, Ns * G, win, barrier=False)
    finally:
        win.close()
