"""Summarise an ncu --set full report: duration, issue, occupancy, top stalls,
memory traffic (reads `ncu -i REP --page raw --csv`)."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'smsp__inst_executed.sum',
        'sm__issue_active.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block_dynamic',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active']


def summary(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units, v = r[0], r[1], r[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    lines = [f"kernel {d.get('Kernel Name', '?')[:90]}"]
    for k in KEYS:
        lines.append(f"  {k} = {d.get(k)} {u.get(k, '')}")
    st = []
    for k in h:
        if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio'):
            try:
                st.append((float(d[k]), k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
            except ValueError:
                pass
    st.sort(reverse=True)
    lines.append('  stalls/issue: ' + ', '.join(f'{n} {x:.2f}' for x, n in st[:8]))
    return '\n'.join(lines)


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        print(summary(rep))
