"""Summarise an ncu --set full capture of k_mcmc into profiles/ (metric,value,unit)."""
import csv, subprocess, sys

KEEP = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "l1tex__t_sector_hit_rate.pct",
        "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep, out, header):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    names, units, vals = rows[0], rows[1], rows[2]
    with open(out, "w") as fh:
        fh.write(header.rstrip("\n") + "\n")
        for i, n in enumerate(names):
            if n in KEEP or n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                fh.write(f"{n},{vals[i]},{units[i]}\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
