"""GPU debugging probe for the mixed GEMM: one scenario per process (run each under
`timeout`), prints the relative Frobenius error vs the oracle and, for the
one-hot scenarios, which reordered column the tensor core decoded per row.

usage: python tools/gemm_probe.py <seg-split e.g. 0,0,256> [M N bn stages onehot]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
from oracle import gemm as ogemm  # noqa: E402
from oracle import mx as omx  # noqa: E402
from synth import bf16_bits, bits_to_bf16, gen_act, gen_perm, gen_weight  # noqa: E402


def main():
    n = tuple(int(v) for v in sys.argv[1].split(","))
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    bn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    st = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    onehot = len(sys.argv) > 6 and sys.argv[6] == "onehot"
    K = sum(n)
    mm.mm_set_gemm_config(bn, st, 0)
    if onehot:
        rng = np.random.default_rng(0)
        perm = np.arange(K)
        jsel = rng.integers(0, K, size=M)
        xa = np.zeros((M, K))
        xa[np.arange(M), jsel] = 1.0
        wa = rng.choice([1.0, 2.0, 3.0, 4.0], size=(N, K))
        g = 0 if n[0] else (1 if n[1] else 2)
        wa[:, ::32] = (6.0, 28.0, 256.0)[g]
        x = bits_to_bf16(omx.bf16_rne_bits(xa))
        w = bits_to_bf16(omx.bf16_rne_bits(wa))
    else:
        perm = gen_perm(K, 11).numpy()
        x = gen_act(M, K, 1000, 2001)
        w = gen_weight(N, K, 3000)
    plan = mm.mm_plan_init(K, n, perm)
    a = mm.mm_reorder_quantize_act(x.cuda(), plan)
    wq = mm.mm_quantize_weight_offline(w.cuda(), plan)
    torch.cuda.synchronize()
    print("RQ done", flush=True)
    y = mm.mm_mixed_gemm_bf16(a, wq, plan)
    torch.cuda.synchronize()
    print("GEMM done", flush=True)
    yref, _ = ogemm.mixed_linear_ref(bf16_bits(x), bf16_bits(w), perm, n)
    yg = y.double().cpu().numpy()
    print(f"n={n} M={M} N={N} rel_fro={ogemm.rel_fro(yg, yref):.3e} |y|={np.linalg.norm(yg):.4e} "
          f"|ref|={np.linalg.norm(yref):.4e}")
    if onehot:
        bad = [(m, int(jsel[m]), int(np.argmin(np.abs(wa.T - yg[m][None, :]).sum(axis=1))))
               for m in range(M) if not np.array_equal(yg[m], wa[:, jsel[m]])]
        print(f"one-hot: {len(bad)} of {M} rows decoded the wrong column; first: {bad[:12]}")
        print("row0 y[:8]", yg[0, :8], "expect", wa[:8, jsel[0]])


if __name__ == "__main__":
    main()
