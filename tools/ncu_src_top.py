"""Summarise an ncu `--page source --csv --print-source sass` export: top stall
instructions and executed-instruction totals (run here, on the CPU side)."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    i_src = hdr.index("Source")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        if len(r) <= i_s:
            continue
        data.append((int(r[i_s] or 0), int(r[0], 16) & 0xFFFF, r[i_src], int(r[i_e] or 0)))
    tot = sum(d[0] for d in data)
    ins = sum(d[3] for d in data)
    print(f"samples {tot}  warp-instructions executed {ins}")
    for d in sorted(data, reverse=True)[:top]:
        print(f"{d[0]:7d} {100 * d[0] / max(tot, 1):5.1f}% {d[1]:#06x} {d[2][:90]:90s} exec={d[3]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)


def by_reason(path, reason="stall_long_sb", top=15):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    i_src = hdr.index("Source")
    i_r = hdr.index(reason)
    data = [(int(r[i_r] or 0), int(r[0], 16) & 0xFFFF, r[i_src]) for r in rows[2:] if len(r) > i_r]
    tot = sum(d[0] for d in data)
    print(f"{reason}: {tot} samples")
    for d in sorted(data, reverse=True)[:top]:
        print(f"  {d[0]:6d} {d[1]:#06x} {d[2][:100]}")
