"""Side-by-side ncu summary (time, registers, issue, DMMA pipe, shared-memory
wavefronts and bank conflicts, top stall reasons) of one kernel per report:
the DMMA DGEMM against cuBLAS's DGEMM (dev tool; prints JSON with --json)."""
import csv, subprocess, sys
keys = ['gpu__time_duration.sum','launch__registers_per_thread','smsp__issue_active.avg.pct_of_peak_sustained_active',
 'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum',
 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
 'dram__bytes_read.sum','lts__t_bytes.sum']
as_json = '--json' in sys.argv
result = {}
for rep in [a for a in sys.argv[1:] if a != '--json']:
    out = subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    for row in r[2:]:
        ent = result.setdefault(rep, {"kernel": row[h.index('Kernel Name')]})
        for k in keys:
            if k in h: ent[k] = row[h.index(k)]
        st = [(h[i], row[i]) for i in range(len(h)) if h[i].startswith('smsp__average_warps_issue_stalled_') and h[i].endswith('_per_issue_active.ratio')]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:10]
        ent["stalls_per_issue"] = {k.replace('smsp__average_warps_issue_stalled_', '').replace(
            '_per_issue_active.ratio', ''): v for k, v in st}
import json  # noqa: E402
print(json.dumps(result, indent=1))
