import csv, subprocess, sys
WANT = ['Kernel Name','Grid Size','Block Size','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','launch__occupancy_limit_shared_mem',
        'smsp__average_warp_latency_issue_stalled_long_scoreboard','smsp__pcsamp_warps_issue_stalled_long_scoreboard',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct']
for f in sys.argv[1:]:
    out = subprocess.run(['ncu','-i',f,'--page','raw','--csv'],capture_output=True,text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f)
        for w in WANT:
            if w in hdr:
                i = hdr.index(w); print(f"   {w} [{units[i]}] = {r[i][:90]}")
