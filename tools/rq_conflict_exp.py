"""Experiment: cost of shared-memory bank conflicts in the RQ gather.  Same segment
sizes, three permutations: random (like a calibrated plan), 'conflict-free' (every
gather step of a warp reads 32 channels in 32 distinct banks) and identity (16-way
conflicts under the kernel's lane mapping).  python tools/rq_conflict_exp.py M:K ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
import sweep_configs as sc  # noqa: E402
from bench import rq_bytes  # noqa: E402
from synth import gen_act  # noqa: E402


def conflict_free(K, n):
    """position (chunk c, lane l, step q) of each segment -> channel 32*q + l of a
    512-channel window (bank = l for 4-byte slots)."""
    perm = np.empty(K, dtype=np.int64)
    chans = np.arange(K)
    off = 0
    pos = 0
    for g in range(3):
        for j in range(n[g]):
            p = j % 512
            c0 = j - p
            lane_blk, w = divmod(p, 32)          # block inside the chunk, position inside the block
            h, q = divmod(w, 16)
            l = 2 * lane_blk + h
            perm[off + j] = off + c0 + 32 * q + l if c0 + 512 <= n[g] else off + j
        off += n[g]
    assert sorted(perm.tolist()) == list(range(K))
    return perm


L2 = torch.cuda.get_device_properties(0).L2_cache_size
hbm = sc.PK["hbm_gbs"]
for arg in sys.argv[1:]:
    M, K = map(int, arg.split(":"))
    base = sc.calibrated_plan(K, layer=2)
    n = base.n
    perms = {"random": np.random.default_rng(0).permutation(K), "conflict_free": conflict_free(K, n),
             "identity": np.arange(K)}
    nset = max(2, min(8, -(-3 * L2 // (2 * M * K))))
    xs = [gen_act(M, K, 1000, 2001 + 100 * i, device="cuda") for i in range(nset)]
    res = []
    for name, p in perms.items():
        plan = mm.mm_plan_init(K, n, p)
        outs = [mm.mm_reorder_quantize_act(x, plan) for x in xs]
        us = sc.time_loop(lambda i: mm.mm_reorder_quantize_act(xs[i], plan, out=outs[i]), nset, 40)
        res.append(f"{name}:{us:.2f}us/{rq_bytes(M, n) / us / 1e3 / hbm:.3f}")
        del outs
    print(f"M={M} K={K} n={n} " + " ".join(res), flush=True)
    del xs
    torch.cuda.empty_cache()
