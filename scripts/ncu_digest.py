"""Print the key counters (and the pc-sampling stall split) of an .ncu-rep.
usage: python scripts/ncu_digest.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__waves_per_multiprocessor", "sm__maximum_warps_per_active_cycle_pct"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("----")
        for w in WANT:
            if w in h:
                print(f"{w:60s} {r[h.index(w)]} {units[h.index(w)]}")
        st = {k[len('smsp__pcsamp_warps_issue_stalled_'):]: float(r[i] or 0)
              for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("_not_issued")}
        tot = sum(st.values()) or 1
        top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
        print("stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
