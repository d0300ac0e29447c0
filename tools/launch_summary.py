"""ncu launch list (--metrics gpu__time_duration.sum --csv) of `bench.py` ->
markdown: per fill kernel the launch times and its share of the device step.

    python tools/launch_summary.py gpurun_out/launches.csv profiles/r01_launches_bench.md
"""
import collections
import csv
import re
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main():
    src, out = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    idx = {h: i for i, h in enumerate(rows[0])}
    per = collections.OrderedDict()
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[idx["Kernel Name"]]).replace("void ", "")
        ms = float(r[idx["Metric Value"]].replace(",", "")) * SCALE[r[idx["Metric Unit"]]]
        per.setdefault(name, []).append(ms)
    fills = {k: v for k, v in per.items() if k.startswith("rsa::k_fill_fast")}
    step = sum(sum(v) / len(v) for v in fills.values())
    lines = [f"# Launch list of `python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu` under ncu "
             "(gpu__time_duration.sum, --clock-control none)", "",
             f"Source: `{src.split('/')[-1]}` copied next to this file.  The device-timed step is the four "
             "full 2^30-value fills (1 warm-up + 2 timed launches each); `k_probe_imad` is the in-run "
             "roofline probe, the scan/setup/init launches build the stream parameters before timing.", "",
             "| kernel | launches (ms) | mean ms | share of the device step |", "|---|---|---|---|"]
    for k, v in fills.items():
        m = sum(v) / len(v)
        lines.append(f"| `{k}` | {', '.join(f'{x:.3f}' for x in v)} | {m:.3f} | {100 * m / step:.1f}% |")
    lines += ["", f"Sum of the four means: {step:.2f} ms per step under ncu (cold caches, serialised).", "",
              "Other launches (count, mean ms):", ""]
    for k, v in per.items():
        if k not in fills:
            lines.append(f"- `{k}`: {len(v)} x {sum(v) / len(v):.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
