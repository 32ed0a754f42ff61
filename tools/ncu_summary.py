"""Summarise an ncu report: headline metrics, stall totals, hottest SASS lines (dev tool)."""
import collections
import csv
import io
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers']


def ncu(rep, *args):
    return subprocess.run(['ncu', '-i', rep, *args], capture_output=True, text=True).stdout


def main(rep, ntop=30, kernel_idx=0):
    raw = list(csv.reader(io.StringIO(ncu(rep, '--page', 'raw', '--csv'))))
    h, v = raw[0], raw[2 + kernel_idx]
    for i, n in enumerate(h):
        if n in WANT:
            print(f'{n:75s} {v[i]}')
    for i, n in enumerate(h):
        if n.startswith('smsp__average_warps_issue_stalled') and n.endswith('per_issue_active.ratio'):
            try:
                if float(v[i]) > 0.1:
                    print(f'  {n[34:-29]:40s} {v[i]}')
            except ValueError:
                pass
    src = list(csv.reader(io.StringIO(ncu(rep, '--page', 'source', '--csv', '--print-source', 'sass'))))
    hdr, rows = src[1], src[2:]
    si = hdr.index('Warp Stall Sampling (All Samples)')
    ie = hdr.index('Instructions Executed')
    names = [x for x in hdr if x.startswith('stall_') and 'Not Issued' not in x]
    tot = sum(int(r[si]) for r in rows if r[si].isdigit())
    print('samples', tot)
    top = sorted([(int(r[si]), i) for i, r in enumerate(rows) if r[si].isdigit()], reverse=True)[:ntop]
    for c, i in top:
        r = rows[i]
        st = sorted([(int(r[hdr.index(n)]), n[6:]) for n in names if r[hdr.index(n)].isdigit()], reverse=True)[:3]
        print(f'{c:5d} {i:5d} {r[ie]:>9s} {r[1].strip()[:60]:60s} {st}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
