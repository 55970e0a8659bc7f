"""Summarise one kernel of an ncu --set full report into a short text file.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.txt [algorithmic_bytes]

Prints duration, DRAM read/write bytes (the roofline ``traffic``), DRAM / L2 /
SM throughput, occupancy, registers and the warp stall breakdown.  When the
algorithmic bytes per launch are given, the achieved algorithmic bandwidth
and the traffic/algorithmic ratio are added.
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("dram__bytes_read.sum.per_second", "dram read rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
            "Tbyte": 1e12}.get(u, None)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    algo = float(sys.argv[3]) if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(raw.splitlines()) if r]
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    name = get.get("Kernel Name", ("", "?"))[1]
    lines = [f"kernel: {name}"]
    for k, label in KEYS:
        if k in get:
            u, v = get[k]
            lines.append(f"{label:24s} {v} {u}  ({k})")
    stalls = []
    for h, (u, v) in get.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and \
                h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), h[len("smsp__average_warps_issue_"
                                               "stalled_"):-len(
                    "_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    lines.append("stalls per issue: " + ", ".join(
        f"{n} {v:.2f}" for v, n in stalls[:8]))
    try:
        rb = float(get["dram__bytes_read.sum"][1]) * \
            unit_scale(get["dram__bytes_read.sum"][0])
        wb = float(get["dram__bytes_write.sum"][1]) * \
            unit_scale(get["dram__bytes_write.sum"][0])
        dur = float(get["gpu__time_duration.sum"][1]) * \
            {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}[get["gpu__time_duration.sum"][0]]
        lines.append(f"traffic (dram r+w) bytes  {rb + wb:.0f}")
        lines.append(f"dram r+w rate GB/s        {(rb + wb) / dur / 1e9:.1f}")
        if algo:
            lines.append(f"algorithmic bytes         {algo:.0f}")
            lines.append(f"algorithmic GB/s (ncu)    {algo / dur / 1e9:.1f}")
            lines.append(f"traffic / algorithmic     {(rb + wb) / algo:.3f}")
    except (KeyError, TypeError, ValueError):
        pass
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
