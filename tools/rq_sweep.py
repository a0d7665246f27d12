"""RQ tuning sweep (GPU box): for each M:K, time the reorder-quantize with every
consumer-group width MM_RQ_GW in a list (and the automatic choice), same process.
MM_RQ_ROWS is read once per process: run once per rows value.
    MM_RQ_ROWS=2 python tools/rq_sweep.py 2048:4096 16384:4096"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
import sweep_configs as sc  # noqa: E402
from bench import rq_bytes  # noqa: E402
from synth import gen_act  # noqa: E402

L2 = torch.cuda.get_device_properties(0).L2_cache_size
hbm = sc.PK["hbm_gbs"]
GWS = [int(g) for g in os.environ.get("GWS", "0,1,2,3,4,5,6,8,10,12,19").split(",")]
for arg in sys.argv[1:]:
    M, K = map(int, arg.split(":"))
    plan = sc.calibrated_plan(K, layer=2)
    n = max(2, min(8, -(-3 * L2 // (2 * M * K))))
    xs = [gen_act(M, K, 1000, 2001 + 100 * i, device="cuda") for i in range(n)]
    outs = [mm.mm_reorder_quantize_act(x, plan) for x in xs]
    b = rq_bytes(M, plan.n)
    res = []
    for gw in GWS:
        if gw:
            os.environ["MM_RQ_GW"] = str(gw)
        else:
            os.environ.pop("MM_RQ_GW", None)
        try:
            us = sc.time_loop(lambda i: mm.mm_reorder_quantize_act(xs[i], plan, out=outs[i]), n, 40)
        except Exception as e:  # e.g. too many threads for the variant
            res.append(f"gw={gw}:ERR")
            continue
        res.append(f"gw={gw or 'auto'}:{us:.2f}us/{b / us / 1e3 / hbm:.3f}")
    os.environ.pop("MM_RQ_GW", None)
    print(f"M={M} K={K} rows={os.environ.get('MM_RQ_ROWS', 'auto')} " + " ".join(res), flush=True)
    del xs, outs
    torch.cuda.empty_cache()
