"""Summarise an ncu --set full report (one kernel launch) into a small text block for profiles/.

    python tools/ncu_summary.py report.ncu-rep [title]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor (tc) pipe active % (per active SM)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(f"== {title}")
    print(f"kernel: {vals[hdr.index('Kernel Name')][:120]}")
    for key, label in KEYS:
        if key in hdr:
            i = hdr.index(key)
            print(f"  {label:45s} {vals[i]} {units[i]}")
    stall = [(float(vals[i] or 0), h) for i, h in enumerate(hdr)
             if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    stall.sort(reverse=True)
    print("  top stall reasons (warps per issue): " + ", ".join(
        f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
        for v, h in stall[:5]))


if __name__ == "__main__":
    main()
