#!/usr/bin/env python
"""Summarise ncu --set full reports: duration, DRAM bytes/throughput, smem
wavefronts, issue activity, top stall reasons.  usage: ncu_summary.py REP..."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__cycles_active.avg", "sm_active_cyc"),
    ("gpc__cycles_elapsed.max", "elapsed_cyc"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_%elapsed"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_conflicts"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn"),
    ("launch__occupancy_limit_shared_mem", "occ_lim_smem"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
]
# tensor-pipe counters (names differ across architectures: every raw metric
# mentioning the tensor / tcgen05 pipes is printed)
TENSOR_HINTS = ("pipe_tensor", "pipe_tc", "tcgen05", "umma", "tmem")


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    for rep in sys.argv[1:]:
        h, units, data = rows(rep)
        for row in data:
            name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            print(f"== {rep}: {name[:90]}")
            for k, lab in KEYS:
                if k in h:
                    i = h.index(k)
                    print(f"  {lab:18s} {row[i]:>14s} {units[i]}")
            for i, k in enumerate(h):
                if any(t in k for t in TENSOR_HINTS) and (k.endswith(".sum") or "pct" in k):
                    print(f"  {k[:60]:60s} {row[i]:>14s} {units[i]}")
            st = []
            for i, k in enumerate(h):
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(row[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            print("  stalls/issue      " + ", ".join(f"{n} {v:.2f}" for v, n in st[:7]))


if __name__ == "__main__":
    main()
