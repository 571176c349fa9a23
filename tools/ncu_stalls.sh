# summary of an ncu report: duration, occupancy, issue, stall reasons per kernel (here, no GPU)
rep=$1
ncu -i $rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
want=['gpu__time_duration.sum','sm__warps_active.avg.pct_of_peak_sustained_active','sm__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__thread_inst_executed_per_inst_executed.ratio','launch__registers_per_thread','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    d=dict(zip(h,r))
    print(d['Kernel Name'][:60])
    for w in want:
        if w in d: print('   ',w,d[w])
    st=[(k.replace('smsp__average_warp_latency_issue_stalled_','').replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''),float(v)) for k,v in d.items() if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio') and v not in ('','n/a')]
    st.sort(key=lambda x:-x[1])
    print('    stalls/issue:', ', '.join('%s %.2f'%(k,v) for k,v in st[:8]))
"
