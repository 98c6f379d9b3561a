import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout.splitlines()
r=list(csv.reader(out)); hdr=r[0]; vals=r[2]
d=dict(zip(hdr,vals))
keys=['gpu__time_duration.sum','sm__inst_executed.sum','sm__inst_executed.sum.per_cycle_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','sm__warps_active.avg.per_cycle_active','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','launch__registers_per_thread','launch__occupancy_limit_shared_mem']
for k in keys: print(k.ljust(70), d.get(k))
for k,v in d.items():
    if 'average_warps_issue_stalled' in k and 'per_issue_active' in k:
        try:
            if float(v)>0.02: print(k.replace('smsp__average_warps_issue_stalled_','stall_').ljust(70), v)
        except: pass
