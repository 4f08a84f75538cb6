"""Summarise an ncu launch list (CSV) and a full capture (.ncu-rep) of the pole kernel into
profiles/<tag>_summary.md and profiles/pole_kernel_traffic.json (run here, on CPU).

    python tools/summarize_profile.py <tag> <config>_<variant> [bench.log]
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag):
    path = os.path.join(OUT, f"{tag}_launches.csv")
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    gi = hdr.index("Grid Size")
    agg = OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki]
        v = float(r[vi].replace(",", ""))
        if r[ui] == "us":
            v *= 1e3
        elif r[ui] == "ms":
            v *= 1e6
        agg.setdefault(name, []).append((v, r[gi]))
    return agg


def raw_metrics(tag, names):
    rep = os.path.join(OUT, f"{tag}_pole.ncu-rep")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for n in names:
        if n in hdr:
            i = hdr.index(n)
            res[n] = (vals[i], units[i])
    return res


def main():
    tag, key = sys.argv[1], sys.argv[2]
    bench = sys.argv[3] if len(sys.argv) > 3 else None
    agg = launches(tag)
    per_kernel = []
    for name, lst in agg.items():
        ns = [v for v, _ in lst]
        per_kernel.append((name, len(ns), sum(ns) / len(ns), sum(ns), lst[0][1]))
    # one step = one pole-kernel launch and its neighbours: share of the per-step sum
    ours = [k for k in per_kernel if "rexi::" in k[0]]
    step_ns = sum(avg for _, _, avg, _, _ in ours)
    m = raw_metrics(tag, [
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"])
    lines = [f"# Profile summary `{tag}` ({key})", "",
             "Source: `ncu --metrics gpu__time_duration.sum --clock-control none` launch list of "
             "`python bench.py --steps 3 --warmup 3 --no-cpu-baseline` (cold-cache, serialised: "
             "compare shares, not absolutes) and one `ncu --set full` capture of the pole kernel.", "",
             "## Launch list (per launch, ns)", "",
             "| kernel | launches | avg ns | grid | share of one step |", "|---|---|---|---|---|"]
    for name, n, avg, tot, grid in per_kernel:
        share = f"{100 * avg / step_ns:.1f} %" if "rexi::" in name else "(not ours)"
        lines.append(f"| `{name[:70]}` | {n} | {avg:,.0f} | {grid} | {share} |")
    lines += ["", "## Pole kernel, full capture", "", "| metric | value |", "|---|---|"]
    for k, (v, u) in m.items():
        lines.append(f"| `{k}` | {v} {u} |")
    traffic = None
    try:
        rb = float(m["dram__bytes_read.sum"][0].replace(",", ""))
        wb = float(m["dram__bytes_write.sum"][0].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic = rb * scale[m["dram__bytes_read.sum"][1]] + wb * scale[m["dram__bytes_write.sum"][1]]
        lines.append(f"| dram read + write per launch | {traffic / 1e6:.2f} MB |")
    except Exception:
        pass
    if bench and os.path.exists(bench):
        lines += ["", "## bench.py line", "", "```", open(bench).read().strip().splitlines()[-1], "```"]
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tj = os.path.join(PROF, "pole_kernel_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    if traffic is not None:
        d[key] = traffic
        json.dump(d, open(tj, "w"), indent=1)
    # keep the raw launch list too
    src = os.path.join(OUT, f"{tag}_launches.csv")
    with open(src) as fi, open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as fo:
        fo.write(fi.read())
    print("\n".join(lines))


if __name__ == "__main__":
    main()
