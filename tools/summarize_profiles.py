"""Turn an ncu launch list (CSV) and a --set full report of k_lane into the committed
summaries under profiles/ and refresh profiles/traffic.json (read by bench.py).

usage: python tools/summarize_profiles.py TAG LAUNCHES.csv REPORT.ncu-rep "COMMAND"
"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "smsp__inst_executed_op_shared_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
    "launch__grid_size", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(tag, path, command):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    seq = []
    for r in data:
        v = float(r[vi].replace(",", ""))
        ns = v * 1e6 if r[ui] == "msecond" else v * 1e3 if r[ui] == "usecond" else v
        seq.append((r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", ""), ns))
    first = [i for i, (n, _) in enumerate(seq) if n.startswith("k_lane")][0]
    agg = collections.OrderedDict()
    fillers = collections.Counter()
    for n, ns in seq[first:]:
        if "spin_kernel" in n:  # torch.cuda._sleep: bench.py's queue filler before the roofline pass
            fillers[n] += 1
            continue
        agg.setdefault(n, []).append(ns)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# {tag} ncu launch list (gpu__time_duration.sum, --clock-control none), command:", f"#   {command}",
             "# cold-cache serialised per-launch times; shares over the launches from the first histogram on",
             f"{'kernel':40s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}"]
    for n, v in agg.items():
        lines.append(f"{n[:40]:40s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / tot:6.3f}")
    if fillers:
        lines.append(f"# excluded from the shares (untimed queue filler of the roofline pass): {dict(fillers)}")
    setup = collections.Counter(n for n, _ in seq[:first])
    lines.append(f"# setup before the first histogram launch (input generation, untimed): {dict(setup)}")
    out = ROOT / "profiles" / f"{tag}_launches_summary.txt"
    out.write_text("\n".join(lines) + "\n")
    return out


def full(tag, report, command):
    raw = subprocess.run(["ncu", "-i", str(report), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "k_lane"
    lines = [f"# {tag} ncu --set full of {name}", f"# command: {command}", "# values of the first captured launch"]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"{k:90s} {vals[i]:>16s} {units[i]}")
    out = ROOT / "profiles" / f"{tag}_k_lane_ncu_full.txt"
    out.write_text("\n".join(lines) + "\n")
    rd = float(vals[hdr.index("dram__bytes_read.sum")].replace(",", "")) * SCALE[units[hdr.index("dram__bytes_read.sum")]]
    wr = float(vals[hdr.index("dram__bytes_write.sum")].replace(",", "")) * SCALE[units[hdr.index("dram__bytes_write.sum")]]
    (ROOT / "profiles" / "traffic.json").write_text(json.dumps({
        "k_lane_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": 1 << 30,
        "source": f"profiles/{out.name} (dram__bytes_read.sum + dram__bytes_write.sum)"}, indent=1) + "\n")
    return out


if __name__ == "__main__":
    tag, lcsv, rep, cmd = sys.argv[1:5]
    print(launches(tag, lcsv, cmd).read_text())
    print(full(tag, rep, cmd).read_text())
