"""Summarise an ncu report: key throughput metrics + SASS opcode mix per kernel."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__occupancy_limit_shared_mem', 'sm__warps_active.avg.per_cycle_active',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg.per_second']
STALL = 'smsp__average_warps_issue_stalled_'
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')]
    print('==', name[:90])
    for w in WANT:
        if w in hdr:
            print(f'   {w:65s} {r[hdr.index(w)]}')
    st = sorted(((float(r[i]), h[len(STALL):]) for i, h in enumerate(hdr)
                 if h.startswith(STALL) and h.endswith('per_issue_active.ratio') and r[i]),
                reverse=True)[:7]
    print('   stalls/issue:', ', '.join(f'{n.replace("_per_issue_active.ratio", "")}={v:.2f}' for v, n in st))
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                          '-k', 'regex:' + name.split('<')[0].split('(')[0].split()[-1]],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        h2 = srows[1]
        ie, sc = h2.index('Instructions Executed'), h2.index('Source')
        ops = collections.Counter()
        tot = 0
        for x in srows[2:]:
            try:
                n = int(x[ie])
            except (ValueError, IndexError):
                continue
            toks = x[sc].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith('@') else toks[0]
            ops[op.split('.')[0]] += n
            tot += n
        print('   opcode mix:', ', '.join(f'{o}={100 * n / tot:.1f}%' for o, n in ops.most_common(14)))
