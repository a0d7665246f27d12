"""Instruction mix + stall samples of an ncu --page source --csv (SASS) export.
usage: python tools/sass_mix.py file_src.csv [min_count]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 0
h = rows[1]
i_src, i_ex, i_s, i_a = h.index("Source"), h.index("Instructions Executed"), \
    h.index("Warp Stall Sampling (All Samples)"), h.index("Address")
op, st = collections.Counter(), collections.Counter()
tot = stot = 0
for r in rows[2:]:
    toks = r[i_src].split()
    o = toks[1] if toks[0].startswith("@") else toks[0]
    o = o.split(".")[0]
    n, sm = int(r[i_ex] or 0), int(r[i_s] or 0)
    op[o] += n; st[o] += sm; tot += n; stot += sm
    if thr and n >= thr:
        print(r[i_a][-5:], f"{n:8d} {sm:6d}", r[i_src][:90])
print("total warp instructions", tot, "stall samples", stot)
for o, n in op.most_common(30):
    print(f"{o:10s} {n:10d} {100 * n / tot:5.1f}%  stall {100 * st[o] / max(stot, 1):5.1f}%")
