import csv, sys, subprocess, io
rep = sys.argv[1]
raw = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(raw)))
hdr=rows[0]; units=rows[1]; data=rows[2:]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_tensor_subpipe_dmma.sum','lts__t_requests_op_red.sum','lts__t_sectors_op_red.sum','lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum']
for d in data:
    print('----', d[hdr.index('Kernel Name')][:70])
    for w in want:
        if w in hdr:
            i=hdr.index(w); print(f"  {w:75s} {d[i]} {units[i]}")
    st=[(hdr[i],float(d[i])) for i in range(len(hdr)) if hdr[i].startswith('smsp__average_warps_issue_stalled_') and hdr[i].endswith('_per_issue_active.ratio') and d[i] not in ('','n/a')]
    st=[(k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''),round(v,2)) for k,v in st if v>0.3]
    st.sort(key=lambda x:-x[1]); print('  stalls', st[:8])
