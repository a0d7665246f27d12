"""MicroMix CPU oracle -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously correct statement of what the hot
path computes, written from PAPER.md (arXiv 2508.02343) in the paper's order:

  formats.py  MX element formats from their bit fields (Appendix A, Table 6)
  mx.py       Eq. 1 block quantization; §3.2 fused reorder-and-quantize semantics
  calib.py    Definition 1 / Eq. 5-7 / Eq. 17 thresholds, counts, ordering
  gemm.py     Eq. 2 mixed GEMM of the dequantized operands in fp64
  norm.py     RMSNorm in front of the RQ (Fig. 7 integration, F2; R27)
  encode.c    the brute-force nearest-code search (only loop too slow for numpy)

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import or execute anything under oracle/.  The product
(paper_2508_02343_b200/) never imports it, and this package never imports the
product: the two share no code, headers, tables or helpers.  Inputs come from
synth/ (random numbers only).

Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".  Nothing
here is "parity unpinned" except the two points DESIGN.md lists under
"Unpinned readings" (the paper's own choice of scale offset and of element-
vs channel-level proportions, which no printed number in the paper fixes).
"""
from . import calib, formats, gemm, mx, norm  # noqa: F401
from .formats import E2M1, E2M3, E3M2, E4M3, E5M2, FORMATS, fmt  # noqa: F401
from .mx import RULE_OCP, RULE_PAPER  # noqa: F401
