"""One-screen summary of an `ncu --set full` report (the numbers DESIGN.md and bench.py quote).

    python tools/ncu_summary.py report.ncu-rep "title" > profiles/rNN_name.txt
"""
import csv
import subprocess
import sys

METRICS = [
    ("duration", "gpu__time_duration.sum"),
    ("dram read", "dram__bytes_read.sum"),
    ("dram write", "dram__bytes_write.sum"),
    ("dram throughput % of peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor (tc) pipe active % (per active SM)", "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("tcgen05 UTC issue % (per active SM)", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"),
    ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("L2 hit rate %", "lts__t_sector_hit_rate.pct"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("registers/thread", "launch__registers_per_thread"),
    ("dynamic smem/block", "launch__shared_mem_per_block_dynamic"),
    ("warp instructions", "smsp__inst_executed.sum"),
]


def main():
    rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        idx = {h: i for i, h in enumerate(head)}
        print(f"== {title}")
        print(f"kernel: {r[idx['Kernel Name']]}" if "Kernel Name" in idx else "")
        for label, m in METRICS:
            if m in idx:
                print(f"  {label:<45} {r[idx[m]]} {units[idx[m]]}")
        stalls = []
        for h, i in idx.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = ", ".join(f"{n}={100 * v / tot:.1f}%" for v, n in sorted(stalls, reverse=True)[:6])
        print(f"  top stall reasons (share of samples): {top}")


if __name__ == "__main__":
    main()
