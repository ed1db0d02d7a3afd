"""Summarise an ncu --set full report: key section metrics, stall mix, and the
hottest CUDA source lines by warp-stall samples.
usage: python tools/ncu_report.py REPORT.ncu-rep [nlines]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 25
SECTIONS = ('GPU Speed Of Light Throughput', 'Memory Workload Analysis', 'Scheduler Statistics',
            'Warp State Statistics', 'Compute Workload Analysis', 'Occupancy', 'Launch Statistics')
KEEP = ('Duration', 'Memory Throughput', 'DRAM Throughput', 'L1/TEX Cache Throughput', 'L2 Cache Throughput',
        'Compute (SM) Throughput', 'Executed Ipc Active', 'Issue Slots Busy', 'L2 Hit Rate', 'L1/TEX Hit Rate',
        'Eligible Warps Per Scheduler', 'Active Warps Per Scheduler', 'Warp Cycles Per Issued Instruction',
        'Achieved Occupancy', 'Registers Per Thread', 'Avg. Active Threads Per Warp', 'Dynamic Shared Memory Per Block')


def run(*a):
    return subprocess.run(['ncu', '-i', rep, *a], capture_output=True, text=True).stdout


r = list(csv.reader(io.StringIO(run('--page', 'details', '--csv'))))
h = r[0]
si, mi, vi, ui = h.index('Section Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
print(r[1][h.index('Kernel Name')][:100])
for x in r[1:]:
    if x[si] in SECTIONS and x[mi] in KEEP:
        print(f"  {x[mi]:40s} {x[vi]} {x[ui]}")
r = list(csv.reader(io.StringIO(run('--page', 'raw', '--csv'))))
h, u, v = r[0], r[1], r[2]
for k, name in enumerate(h):
    if name in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
                'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__inst_executed.sum',
                'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
                'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum', 'gpu__time_duration.sum'):
        print(f"  {name:55s} {v[k]} {u[k]}")
r = list(csv.reader(io.StringIO(run('--page', 'source', '--csv', '--print-source', 'sass,cuda'))))
hi = [i for i, x in enumerate(r) if x and x[0] == 'Line No'][0]
h = r[hi]
ws = h.index('Warp Stall Sampling (All Samples)')
stall = [k for k, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
agg = []
for x in r[hi + 1:]:
    if len(x) > ws and x[0].strip().isdigit() and x[ws] not in ('', '0', '-'):
        try:
            float(x[ws])
        except ValueError:
            continue
        mix = sorted(((float(x[k]) if x[k].replace('.', '', 1).isdigit() else 0.0, h[k][6:]) for k in stall),
                     reverse=True)[:2]
        agg.append((float(x[ws]), int(x[0]), x[1].strip()[:80], mix))
tot = sum(a[0] for a in agg) or 1
tot_mix = {}
for x in r[hi + 1:]:
    if len(x) > ws and x[0].strip().isdigit():
        for k in stall:
            try:
                tot_mix[h[k][6:]] = tot_mix.get(h[k][6:], 0) + float(x[k])
            except ValueError:
                pass
T = sum(tot_mix.values()) or 1
print('  stalls:', ', '.join(f"{k} {100 * v / T:.0f}%" for k, v in sorted(tot_mix.items(), key=lambda kv: -kv[1])[:7]))
for s_, l, src, mix in sorted(agg, reverse=True)[:nl]:
    print(f"  {100 * s_ / tot:5.1f}% L{l}: {src}   [{', '.join(f'{n} {100 * a / s_:.0f}%' for a, n in mix)}]")
