"""Key counters from `ncu --page raw --csv` dumps: python tools/ncu_rawcsv.py a_raw.csv [b_raw.csv ...]"""
import csv, sys
KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h = rows[0]
    print("==", path)
    for v in rows[2:]:
        d = dict(zip(h, v))
        print("kernel:", d.get("Kernel Name", "?")[:90])
        for k in KEYS:
            if k in d:
                print(f"  {k:75s} {d[k]} {rows[1][h.index(k)]}")
        st = sorted(((float(d[k].replace(',', '')), k) for k in h if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio") and d[k]), reverse=True)
        for x, k in st[:6]:
            print(f"  stall {k.split('stalled_')[1].split('_per_issue')[0]:30s} {x:.2f}")
