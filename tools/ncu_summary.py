"""Key counters of one or more ncu reports side by side (development):
    python tools/ncu_summary.py a.ncu-rep [b.ncu-rep ...] [--per N]   (--per: divide counts by N units)"""
import csv, subprocess, sys
args = [a for a in sys.argv[1:] if not a.startswith("--")]
per = 1.0
if "--per" in sys.argv:
    per = float(sys.argv[sys.argv.index("--per") + 1]); args = [a for a in args if a != sys.argv[sys.argv.index("--per") + 1]]
KEYS = [
    ("gpu__time_duration.sum", "time (us)", 1e-3, False),
    ("smsp__inst_executed.sum", "warp-instr", 1, True),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1, False),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %", 1, False),
    ("sm__inst_executed_pipe_fp64.sum", "fp64-pipe instr", 1, True),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts", 1, True),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts", 1, True),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefront %", 1, False),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1, False),
    ("launch__registers_per_thread", "regs", 1, False),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard", 1, False),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait", 1, False),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard", 1, False),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle", 1, False),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_throttle", 1, False),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected", 1, False),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "stall branch_resolving", 1, False),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier", 1, False),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall dispatch", 1, False),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "stall no_instruction", 1, False),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg_throttle", 1, False),
    ("dram__bytes_read.sum", "dram read B", 1, False),
    ("dram__bytes_write.sum", "dram write B", 1, False),
]
vals = []
for rep in args:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[-1]
    d = {}
    for i, n in enumerate(h):
        try:
            d[n] = float(v[i].replace(",", ""))
        except ValueError:
            pass
    vals.append(d)
print("%-26s" % "metric" + "".join("%18s" % a.split("/")[-1][:17] for a in args))
for k, name, sc, isc in KEYS:
    row = []
    for d in vals:
        x = d.get(k)
        if x is None:
            row.append("%18s" % "-")
        else:
            x = x * sc / (per if isc else 1.0)
            row.append("%18.4g" % x)
    print("%-26s" % name + "".join(row))
