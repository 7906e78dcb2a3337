"""Print key metrics + top stall reasons for every kernel in an .ncu-rep."""
import csv, io, subprocess, sys
raw = open(sys.argv[1]).read() if sys.argv[1].endswith(".csv") else \
    subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__issue_active.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__cycles_elapsed.avg.per_second', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem']
for r in rows[2:]:
    print('---', r[h.index('Kernel Name')][:100])
    print('   ' + '; '.join(f"{k.split('.')[0].replace('__','.')}={r[h.index(k)]}{u[h.index(k)]}" for k in keys if k in h))
    st = [(float(r[i]), h[i]) for i in range(len(h)) if h[i].startswith('smsp__average_warps_issue_stalled')
          and h[i].endswith('per_issue_active.ratio') and r[i] not in ('', 'n/a')]
    st.sort(reverse=True)
    print('   stalls: ' + ', '.join(f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for v, n in st[:7]))
