"""Real multi-device runs of the N-sharded layer (SURVEY §4.2 tier T2, §8(e);
VERDICT r1 "next" #5): one process per GPU (torch.multiprocessing.spawn), world
sizes 2 / 4 / 8 where torch.cuda.device_count() allows, skipped otherwise (the
pool's test boxes have one GPU; the same code runs on an 8 x B200 node).

Each rank quantizes ITS shard of W's rows with the shared plan, runs the
replicated activation's reorder-quantize and then
  * mm_mixed_gemm_bf16_nshard_allgather (library-owned NCCL communicator, id
    exchanged through the torch process group), and
  * mm_mixed_gemm_bf16_nshard_peerstore (fused all-gather epilogue: every tile
    TMA-stored into every rank's Y over CUDA-IPC peer mappings, flag barrier),
  * mm_mixed_gemm_bf16_nshard_nvls (the same through one multicast object: each
    element written once with multimem.st, replicated by the switch) where supported,
and checks both gathered outputs (a) bit-equal to the 1-GPU GEMM of the full W on
its own device (each element's K order does not depend on the N offset, DESIGN.md
§8) and (b) against the fp64 oracle on sampled rows (tests/accuracy.py bars)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, N, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2508_02343_b200 as mm
        from paper_2508_02343_b200 import dist as mmdist
        from synth import bf16_bits, gen_act, gen_perm, gen_weight

        K = sum(n)
        plan = mm.mm_plan_init(K, n, gen_perm(K, 41))
        x = gen_act(M, K, 1000, 2001)
        w = gen_weight(N, K, 3000)
        a = mm.mm_reorder_quantize_act(x.cuda(), plan)
        w_shard = mm.mm_quantize_weight_offline(mmdist.shard_weight(w, world, rank).cuda(), plan)
        y_full = mm.mm_mixed_gemm_bf16(a, mm.mm_quantize_weight_offline(w.cuda(), plan), plan)
        # NCCL all-gather path
        uid = mmdist.exchange_unique_id(mm.nccl_unique_id)
        comm = mm.mm_comm_init(rank, world, uid)
        try:
            y_nccl = mm.mm_mixed_gemm_bf16_nshard_allgather(a, w_shard, plan, N, comm)
            torch.cuda.synchronize()
        finally:
            mm.mm_comm_destroy(comm)
        # fused peer-store path (two steps: the second re-uses the flags)
        win, y_peer = mmdist.open_peer_window(M, N)
        try:
            for _ in range(2):
                mm.mm_mixed_gemm_bf16_nshard_peerstore(a, w_shard, plan, N, win, barrier=True)
            torch.cuda.synchronize()
            dist.barrier()
        finally:
            win.close()
        ok_nccl = torch.equal(y_nccl.view(torch.int16), y_full.view(torch.int16))
        ok_peer = torch.equal(y_peer.view(torch.int16), y_full.view(torch.int16))
        if mm.mc_supported():   # NVLS: multimem stores through a multicast object over all ranks
            mwin = mm.McWindow.create(M, N)
            try:
                mwin.set_timeout(60.0)
                for _ in range(2):
                    mm.mm_mixed_gemm_bf16_nshard_nvls(a, w_shard, plan, N, mwin, barrier=True)
                torch.cuda.synchronize()
                dist.barrier()
                ok_peer = ok_peer and torch.equal(mwin.y().view(torch.int16), y_full.view(torch.int16)) \
                    and not mwin.timed_out()
            finally:
                mwin.close()
        rep = None
        if rank == 0:
            import sys
            sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
            from accuracy import ref_and_abs, report
            from oracle.formats import E3M2, E4M3
            rows = np.arange(0, M, 7)
            yref, S = ref_and_abs(bf16_bits(x)[rows], bf16_bits(w), plan.perm_host().numpy(), plan.n,
                                  E3M2, E4M3, plan.rule)
            rep = report(bf16_bits(y_peer.cpu())[rows], yref, S, K)
        q.put((rank, ok_nccl, ok_peer, rep))
    except Exception as e:   # report instead of hanging the parent
        q.put((rank, False, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_nshard_multidevice(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, have {torch.cuda.device_count()}")
    M, N, n = 520, 1024 * world // 2, (2240, 1184, 672)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), M, N, n, q), nprocs=world, join=True)
    res = sorted(q.get(timeout=60) for _ in range(world))
    for rank, ok_nccl, ok_peer, rep in res:
        assert ok_nccl and ok_peer, (rank, ok_nccl, ok_peer, rep)
    rep0 = res[0][3]
    assert rep0["bound_violations"] == 0 and rep0["rel_fro"] <= 2e-3, rep0
