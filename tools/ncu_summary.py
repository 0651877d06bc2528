"""Summarise an ncu report (raw page) for the metrics we track."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg']
STALLS = ['barrier', 'long_scoreboard', 'short_scoreboard', 'mio_throttle', 'math_pipe_throttle', 'wait',
          'not_selected', 'lg_throttle', 'dispatch_stall', 'no_instruction', 'branch_resolving']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    for d in data:
        print('=====', d[idx['Kernel Name']][:110])
        for w in WANT:
            if w in idx:
                print(f'  {w:70s} {d[idx[w]]:>18s} {units[idx[w]]}')
        st = []
        for s in STALLS:
            k = f'smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio'
            if k in idx:
                st.append(f'{s}={float(d[idx[k]]):.2f}')
        print('  stalls/issue:', ' '.join(st))


if __name__ == '__main__':
    main(sys.argv[1])
