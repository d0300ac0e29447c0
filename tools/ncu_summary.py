"""Summarise an ncu --set full report into profiles/ (markdown + traffic.json).

    python tools/ncu_summary.py gpurun_out/prof_fill.ncu-rep profiles/r01_ncu_fill.md [key-prefix]

traffic.json maps a kernel key (fill_e<E>, fused, scan, ...) to
dram__bytes_read.sum + dram__bytes_write.sum per launch, which bench.py reports
as roofline.traffic.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy (IMAD) pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math-pipe throttle"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall dispatch"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not selected"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(v.replace(",", "")) * scale


def main():
    rep, out_md = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary: `{os.path.basename(rep)}`", "",
             "| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " |",
             "|---" * (len(METRICS) + 1) + "|"]
    tpath = os.path.join(os.path.dirname(out_md), "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for d in data:
        name = d[idx["Kernel Name"]]
        short = re.sub(r"\(.*", "", name).replace("void ", "")
        cells = []
        for m, _ in METRICS:
            cells.append(f"{d[idx[m]]} {units[idx[m]]}".strip() if m in idx else "n/a")
        lines.append(f"| `{short}` | " + " | ".join(cells) + " |")
        rd = to_bytes(d[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
        wr = to_bytes(d[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
        mt = re.search(r"k_fill_fast\w*<(\d+),", name)
        if mt:
            traffic[f"fill_e{mt.group(1)}"] = rd + wr
        elif "k_fused" in name:
            traffic["fused"] = rd + wr
        elif "k_scan_sieve" in name:
            traffic["scan_sieve"] = rd + wr
        elif "k_setup" in name:
            traffic["setup"] = rd + wr
    with open(out_md, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(tpath, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
