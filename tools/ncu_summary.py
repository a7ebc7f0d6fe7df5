"""Summarise an ncu --set full report (one or more kernels): time, pipes, stalls, memory."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "occ limit regs"),
    ("launch__occupancy_limit_shared_mem", "occ limit smem"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local ld inst"),
    ("smsp__sass_inst_executed_op_local_st.sum", "local st inst"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("sm__cycles_elapsed.avg", "cycles"),
]
STALLS = ["wait", "mio_throttle", "short_scoreboard", "long_scoreboard", "math_pipe_throttle", "not_selected",
          "selected", "barrier", "branch_resolving", "lg_throttle", "no_instruction", "dispatch_stall"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d.get("Kernel Name", "?")[:90])
        for k, name in KEYS:
            if k in d:
                print(f"   {name:28s} {d[k]} {units[hdr.index(k)]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d and d[k]:
                st.append(f"{s}={float(d[k]):.2f}")
        print("   stalls/issue:", " ".join(st))
        # flop counts (DFMA = 2 flop)
        f = {}
        for op in ("dfma", "dadd", "dmul", "ffma", "fadd", "fmul"):
            k = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum"
            if k in d and d[k]:
                f[op] = float(d[k])
        if f:
            print("   thread-inst:", f)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
