"""Summarise ncu reports (.ncu-rep from `ncu --set full`) or launch lists (CSV from
`ncu --metrics gpu__time_duration.sum --csv`) into small JSON files for profiles/.

    python scripts/ncu_summary.py rep gpurun_out/ncu_x.ncu-rep ... --out profiles/r1_ncu_kernels.json
    python scripts/ncu_summary.py launches gpurun_out/launches.csv --out profiles/r1_bench_launches.json
"""

import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True, check=False).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize_rep(path):
    rows = ncu_csv(["-i", path, "--page", "raw", "--csv"])
    if len(rows) < 3:
        return {"error": "no data"}
    h, v = rows[0], rows[2]
    out = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
    for m in METRICS:
        if m in h:
            out[m] = v[h.index(m)]
    src = ncu_csv(["-i", path, "--page", "source", "--csv", "--print-source", "sass"])
    if len(src) > 2 and "Warp Stall Sampling (All Samples)" in src[1]:
        hh = src[1]
        si = hh.index("Warp Stall Sampling (All Samples)")
        data = [r for r in src[2:] if len(r) > si and r[si].isdigit()]
        tot = sum(int(r[si]) for r in data) or 1
        top = sorted(data, key=lambda r: -int(r[si]))[:12]
        out["top_stall_sass"] = [{"share": round(int(r[si]) / tot, 3), "sass": r[1].strip()[:90]}
                                 for r in top]
    return out


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, ni, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[ni] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, {"launches": 0, "ns": 0.0})
        a["launches"] += 1
        a["ns"] += float(r[vi].replace(",", ""))
    total = sum(a["ns"] for a in agg.values()) or 1.0
    return {"total_ns": total, "kernels": [
        {"kernel": k, "launches": a["launches"], "ns": a["ns"], "share": round(a["ns"] / total, 4)}
        for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"])]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["rep", "launches"])
    ap.add_argument("paths", nargs="+")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    if args.mode == "rep":
        res = {os.path.basename(p).replace(".ncu-rep", ""): summarize_rep(p) for p in args.paths}
    else:
        res = summarize_launches(args.paths[0])
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    sys.exit(main())
