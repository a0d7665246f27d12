"""Summarise an ncu run of tools/profile.sh into profiles/ (tracked):

  profiles/<tag>_launches.csv   kernel, launches, mean/total device time, share of the step
  profiles/<tag>_kernels.md     per hot kernel: duration, DRAM bytes, L2/tensor/issue utilisation
  profiles/traffic_<tag>.json   dram bytes per launch (read + write) for bench.py's roofline.traffic

usage: python tools/ncu_summary.py gpurun_out/prof_r01 r01
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RAW_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__ops_path_tensor_op_utcomma_src_fp4_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "MXF4 (UTCOMMA) ops % of peak"),
    ("sm__ops_path_tensor_op_utcqmma_src_fp4_fp6_fp8_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "MXF8F6F4 (UTCQMMA) ops % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->L1/smem read bytes"),
]


def read_raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v) * scale


def main(src, tag):
    out = os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    # ---- launch list ------------------------------------------------------------------
    lpath = os.path.join(src, "launches.csv")
    agg = defaultdict(lambda: [0, 0.0])
    seq = []   # (kernel, ns) in launch order
    if os.path.exists(lpath):
        lines = [l for l in open(lpath) if l.startswith('"')]
        rdr = csv.reader(lines)
        hdr = next(rdr)
        i_name, i_metric, i_val = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        for r in rdr:
            if r[i_metric] != "gpu__time_duration.sum":
                continue
            name = r[i_name].split("(")[0].replace("void ", "").split("::")[-1]
            ns = float(r[i_val].replace(",", ""))
            agg[name][0] += 1
            agg[name][1] += ns
            seq.append((name, ns))
        # step shares: every step launches one RQ then one GEMM; the RQ launches before
        # the first GEMM are the offline weight quantizations and are excluded
        first_gemm = next((i for i, (k, _) in enumerate(seq) if "mixgemm" in k), len(seq))
        step_rq = [ns for i, (k, ns) in enumerate(seq) if "rq_kernel" in k and i >= first_gemm - 1]
        step_gemm = [ns for k, ns in seq if "mixgemm" in k]
        mean_rq = sum(step_rq) / max(len(step_rq), 1)
        mean_gemm = sum(step_gemm) / max(len(step_gemm), 1)
        with open(os.path.join(out, f"{tag}_launches.csv"), "w") as f:
            f.write("kernel,launches,total_ns,mean_ns\n")
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"{k},{n},{t:.0f},{t / n:.0f}\n")
            f.write(f"# step launches only: rq mean {mean_rq:.0f} ns over {len(step_rq)}, gemm mean "
                    f"{mean_gemm:.0f} ns over {len(step_gemm)}; gemm share of the step "
                    f"{mean_gemm / max(mean_rq + mean_gemm, 1):.3f}\n")
    # ---- full captures -------------------------------------------------------------------
    traffic = {}
    md = [f"# ncu summary {tag}", "",
          "Source: `ncu --set full --clock-control none` (one launch after warm-up, cold-cache replay;",
          "serialised, so compare shares with the bench, not absolute times). Produced by",
          "`tools/profile.sh` + `tools/ncu_summary.py`.", ""]
    for key, label in (("mixgemm", "mixed GEMM"), ("rq_kernel", "reorder-quantize")):
        path = os.path.join(src, f"full_{key}_raw.csv")
        if not os.path.exists(path):
            continue
        raw = read_raw(path)
        kname = raw.get("Kernel Name", ("?", ""))[0]
        md += [f"## {label}: `{kname[:90]}`", "", "| metric | value |", "|---|---|"]
        for m, lab in RAW_METRICS:
            if m in raw:
                v, u = raw[m]
                md.append(f"| {lab} (`{m}`) | {v} {u} |")
        rd = to_bytes(*raw["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in raw else None
        wr = to_bytes(*raw["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in raw else None
        if rd is not None and wr is not None:
            traffic["mixgemm" if key == "mixgemm" else "rq"] = rd + wr
            md.append(f"| DRAM traffic per launch (read + write) | {rd + wr:.4g} B |")
        md.append("")
    with open(os.path.join(out, f"{tag}_kernels.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    import datetime
    import subprocess
    try:
        commit = subprocess.check_output(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"], text=True).strip()
    except Exception:
        commit = None
    traffic["captured"] = f"{tag} ({datetime.date.today().isoformat()})"
    traffic["commit"] = commit
    with open(os.path.join(out, f"traffic_{tag}.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
