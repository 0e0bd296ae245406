"""Summarise an ncu --set full report (raw page) into the metrics we track."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__pcsamp_sample_count"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for row in rows[2:]:
        name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"## {name[:60]}")
        for i, k in enumerate(h):
            if k in WANT:
                print(f"{k} = {row[i]} {units[i]}")
        stalls = [(k, row[i]) for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("_not_issued")]
        tot = sum(float(v or 0) for _, v in stalls)
        print("stall samples (top):")
        for k, v in sorted(stalls, key=lambda kv: -float(kv[1] or 0))[:10]:
            print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {float(v or 0) / max(tot, 1):.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
