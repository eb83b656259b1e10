"""Summarise ncu outputs into text files under profiles/.

    python scripts/ncu_summary.py report  <x.ncu-rep> <out.txt>   # --set full capture
    python scripts/ncu_summary.py launches <launches.csv> <out.txt>  # gpu__time_duration list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__warps_eligible.avg.per_cycle_active",
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(rep, dst):
    lines = [f"ncu --set full summary of {rep}", ""]
    raw = ncu_csv(["-i", rep, "--page", "raw"])
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        lines.append(f"kernel: {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:70s} {d[k]:>20s} {u.get(k, '')}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        lines.append("  top stall reasons (warps per issue-active cycle):")
        for v, k in sorted(stalls, reverse=True)[:8]:
            lines.append(f"    {k:30s} {v:.3f}")
    src = ncu_csv(["-i", rep, "--page", "source", "--print-source", "sass"])
    if len(src) > 2:
        h = src[1]
        ix, isrc = h.index("Instructions Executed"), h.index("Source")
        by, tot = collections.Counter(), 0
        for r in src[2:]:
            try:
                n = int(r[ix])
            except (ValueError, IndexError):
                continue
            t = r[isrc].split()
            op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
            by[op] += n
            tot += n
        lines.append("")
        lines.append(f"dynamic SASS mix ({tot} warp-instructions):")
        for op, n in by.most_common(24):
            lines.append(f"  {op:24s} {100.0 * n / tot:6.2f}%")
    open(dst, "w").write("\n".join(lines) + "\n")


def launches(path, dst):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iname, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > iv and r[iname] == "gpu__time_duration.sum":
            per[r[ik].split("(")[0]].append(float(r[iv].replace(",", "")))
    tot = sum(sum(v) for v in per.values())
    lines = [f"launch list of {path} (gpu__time_duration.sum, --clock-control none; cold, serialised)",
             f"{'kernel':60s} {'launches':>8s} {'total':>14s} {'share':>7s}"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:60]:60s} {len(v):8d} {sum(v):14.0f} {100 * sum(v) / tot:6.2f}%")
    open(dst, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
