"""Print the key metrics of every kernel in an ncu report (raw page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'smsp__inst_executed.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__sass_inst_executed_op_global_ld.sum',
        'smsp__sass_inst_executed_op_shared_ld.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    print(r[hdr.index('Kernel Name')][:60])
    print('   ' + ' | '.join(f"{w.split('.')[0].replace('smsp__sass_inst_executed_op_','').replace('launch__','')}={r[hdr.index(w)]}" for w in want if w in hdr))
    st = [(hdr[i], float(r[i])) for i in range(len(hdr)) if hdr[i].startswith('smsp__average_warps_issue_stalled_')
          and hdr[i].endswith('_per_issue_active.ratio') and r[i] not in ('', 'n/a')]
    st.sort(key=lambda x: -x[1])
    print('   stalls: ' + ' '.join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for k, v in st[:6]))
