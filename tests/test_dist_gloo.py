"""World-size-2 gloo tests (CPU) of the N-sharded layer's host logic.

Each rank computes the oracle's mixed GEMM for ITS shard of W's rows (the same
plan on every rank, the activation replicated), the shards are all-gathered in
the library's [G][M][N/G] staging layout and permuted to [M][N]; the result must
equal the unsharded oracle bit for bit (each output element's K order does not
depend on the N offset -- DESIGN.md §8).  Also: the NCCL unique-id exchange
through the process group and the max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_02343_b200 import dist as mmdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import calib as ocal
        from oracle import gemm as ogemm
        from synth import bf16_bits, gen_act, gen_weight

        M, K, N = 40, 512, 96
        cal = ocal.calibrate(bf16_bits(gen_act(512, K, 1000, 2000)))
        x = bf16_bits(gen_act(M, K, 1000, 2001))
        w = gen_weight(N, K, 3000)
        w_shard = mmdist.shard_weight(w, world, rank)
        _, ybf = ogemm.mixed_linear_ref(x, bf16_bits(w_shard), cal["perm"], cal["n"])
        mine = torch.from_numpy(np.ascontiguousarray(ybf))
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        stage = torch.stack(parts)                       # [G][M][N/G]
        y = mmdist.gathered_to_row_major(stage, world, M, N // world)
        uid = mmdist.exchange_unique_id(lambda: bytes(range(128)))
        t = mmdist.max_over_ranks(1.0 + rank)
        # peer-window handle exchange (fused all-gather epilogue): rank order kept
        hs = mmdist.exchange_handles(bytes([rank + 1]) * 72)
        hs_ok = hs == [bytes([r + 1]) * 72 for r in range(world)]
        try:   # a rank with a malformed handle makes every rank fail loudly
            mmdist.exchange_handles(bytes([rank + 1]) * (72 if rank == 0 else 8))
            bad_ok = False
        except RuntimeError:
            bad_ok = True
        if rank == 0:
            _, full = ogemm.mixed_linear_ref(x, bf16_bits(w), cal["perm"], cal["n"])
            q.put(("ok", bool(np.array_equal(y.numpy(), full)), uid == bytes(range(128)), t, hs_ok and bad_ok))
        else:
            q.put(("rank1", uid == bytes(range(128)), t, hs_ok and bad_ok))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_nshard_allgather_equals_unsharded_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in res if r[0] == "err"]
    assert not errs, errs
    r0 = [r for r in res if r[0] == "ok"][0]
    r1 = [r for r in res if r[0] == "rank1"][0]
    assert r0[1], "sharded + gathered Y differs from the unsharded oracle"
    assert r0[2] and r1[1], "unique id not exchanged"
    assert r0[3] == 2.0 and r1[2] == 2.0
    assert r0[4] and r1[3], "peer handle exchange lost rank order or accepted a malformed handle"


def test_shard_rows():
    assert mmdist.shard_rows(8192, 8, 3) == (3072, 4096)
    assert mmdist.shard_rows(8192, 1, 0) == (0, 8192)
    with pytest.raises(ValueError):
        mmdist.shard_rows(8192, 3, 0)
    with pytest.raises(ValueError):
        mmdist.shard_rows(96, 8, 0)            # 12-row shards are not a multiple of 16
    spans = [mmdist.shard_rows(4096, 4, r) for r in range(4)]
    assert spans[0][0] == 0 and spans[-1][1] == 4096
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
