"""Summarise ncu outputs into markdown under profiles/ (run in the build container).

    python tools/summarize_ncu.py --launches gpurun_out/launches_r1.csv \
        --report gpurun_out/prof_fp32_r3.ncu-rep --out profiles/r1_fp32.md --title "..."
"""

import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_active.avg", "SM active cycles"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA-pipe inst issued % (FFMA2 = 1 inst, 2 cycles)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) inst %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU inst %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe cycles active %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "TC pipe cycles active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
]


def launches_table(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        ns = float(r["Metric Value"])
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    total = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {ns / 1e6:.3f} | {100 * ns / total:.1f}% |")
    return "\n".join(out), len(rows)


def report_table(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        out.append(f"\n#### `{d.get('Kernel Name', '?')[:110]}`\n")
        out.append("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                out.append(f"| {label} (`{k}`) | {d[k]} {units.get(k, '')} |")
        stalls = []
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    v = float(d[k])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls.append((v, k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        if stalls:
            out.append("\nstalls per issued instruction: " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)))
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--notes", default="")
    a = ap.parse_args()
    parts = [f"# {a.title}\n", a.notes]
    if a.launches:
        tab, n = launches_table(a.launches)
        parts.append(f"\n## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, cold and serialised: compare shares)\n\n{tab}\n")
    if a.report:
        parts.append(f"\n## `ncu --set full` capture ({a.report.split('/')[-1]})\n" + report_table(a.report))
    open(a.out, "w").write("\n".join(parts) + "\n")
    print(open(a.out).read())
