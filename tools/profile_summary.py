"""Summarise ncu captures into profiles/*.md and profiles/traffic.json.
    python tools/profile_summary.py <report.ncu-rep> <name> [traffic-key]
    python tools/profile_summary.py --launches <launches.csv> <name>"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(REPO, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (of active cycles)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem -> tensor-core pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__cycles_active.avg", "SM active cycles"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def stalls(rep, kernel, n=14):
    """Stall samples of one kernel of the report, by reason and by CUDA source line."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kernel}"], capture_output=True, text=True).stdout.splitlines()
    fname, hdr = "?", None
    reasons = defaultdict(float)
    lines = {}
    tot = 0.0
    for r in csv.reader(out):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        try:
            ln = int(r[0])
            smp = float(r[4] or 0)
        except ValueError:
            continue
        tot += smp
        lines[(fname, ln)] = (smp, r[1].strip()[:90])
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    reasons[h] += float(r[i] or 0)
                except ValueError:
                    pass
    if not tot:
        return None
    top = sorted(reasons.items(), key=lambda x: -x[1])[:n]
    hot = sorted(lines.items(), key=lambda x: -x[1][0])[:n]
    return top, [(v[0] / tot * 100, f"{k[0]}:{k[1]}", v[1]) for k, v in hot], tot


def summarise(rep, name, key=None):
    hdr, units, rows = raw(rep)
    lines = [f"# ncu summary: {name}", "", f"source: `{os.path.basename(rep)}` (ncu --set full --clock-control none)", ""]
    for r in rows:
        kname = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines += [f"## {kname[:100]}", "", "| metric | value |", "|---|---|"]
        vals = {}
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                vals[m] = r[i]
                lines.append(f"| {label} (`{m}`) | {r[i]} {units[i]} |")
        lines.append("")
        short = kname.split("(")[0].split("::")[-1]
        if key and "dram__bytes_read.sum" in vals:
            def to_bytes(m):
                i = hdr.index(m)
                u = units[i].lower()
                mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
                return float(r[i].replace(",", "")) * mult
            traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
            tpath = os.path.join(PROF, "traffic.json")
            data = json.load(open(tpath)) if os.path.exists(tpath) else {}
            data[f"{key}:{short}"] = traffic
            json.dump(data, open(tpath, "w"), indent=1)
            lines.append(f"DRAM traffic per launch: {traffic / 1e9:.3f} GB (recorded as `{key}:{short}` in traffic.json)")
            lines.append("")
        st = stalls(rep, short)
        if st:
            top, hot, tot = st
            lines += ["### warp stall reasons (all samples)", "", "| reason | share |", "|---|---|"]
            for k, v in top:
                lines.append(f"| {k} | {v / tot * 100:.1f}% |")
            lines += ["", "### hottest source lines (share of stall samples)", "", "```"]
            lines += [f"{p:5.1f}%  {loc:22s} {src}" for p, loc, src in hot]
            lines += ["```", ""]
    os.makedirs(PROF, exist_ok=True)
    out = os.path.join(PROF, f"{name}.md")
    open(out, "w").write("\n".join(lines))
    print("wrote", out)


def launches(path, name):
    rows = list(csv.reader(open(path)))
    while rows and "Kernel Name" not in rows[0]:
        rows = rows[1:]
    hdr, data = rows[0], rows[1:]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    per = defaultdict(lambda: [0, 0.0])
    for r in data:
        if r[im] != "gpu__time_duration.sum":
            continue
        k = r[ik].split("(")[0]
        per[k][0] += 1
        per[k][1] += float(r[iv].replace(",", ""))
    tot = sum(v[1] for v in per.values()) or 1
    unit = [r for r in data if r[im] == "gpu__time_duration.sum"][0][hdr.index("Metric Unit")] if data else ""
    lines = [f"# launch list: {name}", "", f"source: `{os.path.basename(path)}` (ncu --metrics gpu__time_duration.sum "
             "--clock-control none; cold-cache, serialised: compare shares, not absolutes)", "",
             f"| kernel | launches | total ({unit}) | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {n} | {t:.1f} | {t / tot * 100:.1f}% |")
    out = os.path.join(PROF, f"{name}.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        summarise(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
