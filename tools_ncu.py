import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[0]; units=rows[1]; data=rows[2:]
keys=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','sm__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sectors.sum','lts__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__t_sector_hit_rate.pct','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','launch__grid_size','smsp__inst_executed.sum','smsp__thread_inst_executed_per_inst_executed.ratio','l1tex__throughput.avg.pct_of_peak_sustained_elapsed']
for r in data[: int(sys.argv[2]) if len(sys.argv)>2 else 1]:
    for k in keys:
        if k in h: print(f"{k}: {r[h.index(k)]} {units[h.index(k)]}")
    st=[(h[i], r[i]) for i in range(len(h)) if 'smsp__average_warp_latency_issue_stalled' in h[i] and h[i].endswith('ratio')]
    st=[(a,float(b)) for a,b in st if b]
    for a,b in sorted(st,key=lambda x:-x[1])[:8]: print('  stall',a.replace('smsp__average_warp_latency_issue_stalled_',''),round(b,2))
    pipes=[(h[i], r[i]) for i in range(len(h)) if h[i].startswith('sm__inst_executed_pipe_') and h[i].endswith('.avg.pct_of_peak_sustained_active')]
    for a,b in sorted([(a,float(b)) for a,b in pipes if b],key=lambda x:-x[1])[:5]: print('  pipe',a,round(b,2))
