"""ncu launch list (--metrics gpu__time_duration.sum --csv) of a bench.py run ->
markdown: every kernel of the run with its launch count and times, and for
the config-2 step (the four k_fill_fast<E, 2, 0, 1> fills, E = 3, 5, 17,
65537) each fill's share of the device step.

    python tools/launch_summary.py gpurun_out/launches.csv profiles/r02_launches_bench.md "python bench.py ..."
"""
import collections
import csv
import re
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
STEP_FILLS = ("rsa::k_fill_fast<3, 2, 0, 1>", "rsa::k_fill_fast<5, 2, 0, 1>",
              "rsa::k_fill_fast<17, 2, 0, 1>", "rsa::k_fill_fast<65537, 2, 0, 1>")


def main():
    src, out = sys.argv[1], sys.argv[2]
    cmd = sys.argv[3] if len(sys.argv) > 3 else "python bench.py"
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    idx = {h: i for i, h in enumerate(rows[0])}
    per = collections.OrderedDict()
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[idx["Kernel Name"]]).replace("void ", "")
        name = re.sub(r"(\d+)u\b", r"\1", name).replace("false", "0").replace("true", "1")
        ms = float(r[idx["Metric Value"]].replace(",", "")) * SCALE[r[idx["Metric Unit"]]]
        per.setdefault(name, []).append(ms)
    lines = [f"# Launch list of `{cmd}` under ncu (gpu__time_duration.sum, --clock-control none)", "",
             f"Source: `{src.split('/')[-1]}`.  ncu serialises launches with cold caches: absolute times are "
             "not bench values; the shares within a step are what this list evidences.", ""]
    fills = {k: per[k] for k in STEP_FILLS if k in per}
    if len(fills) == 4:
        step = sum(sum(v) / len(v) for v in fills.values())
        lines += ["## config 2 step (the bench's `value`)", "",
                  "| kernel | launches | mean ms | share of the step |", "|---|---|---|---|"]
        for k, v in fills.items():
            m = sum(v) / len(v)
            lines.append(f"| `{k}` | {len(v)} | {m:.3f} | {100 * m / step:.1f}% |")
        lines += ["", f"Sum of the four means: {step:.2f} ms per step under ncu.", ""]
    lines += ["## every kernel of the run", "", "| kernel | launches | mean ms | total ms |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.4f} | {sum(v):.3f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
