"""Brief per-launch summary from an .ncu-rep: python tools/ncu_brief.py file.ncu-rep [...]"""
import csv, subprocess, sys
KEYS = ['gpu__time_duration.sum', 'launch__registers_per_thread', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__icc_request_hit_rate.pct',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum']
for f in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', f, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    print('==', f)
    for r in rows[2:]:
        name = r[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else ''
        print('--', name[:60])
        for k in KEYS:
            if k in hdr:
                print(f'   {k:78s} {r[hdr.index(k)]}')
        st = {h.split('issue_stalled_')[1].replace('_per_issue_active.ratio', ''): float(r[i]) for i, h in enumerate(hdr)
              if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio') and r[i]}
        tot = sum(st.values())
        print('   stalls/issue:', ', '.join(f'{k} {v:.2f}' for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]), f'(sum {tot:.2f})')
