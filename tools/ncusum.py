"""Key metrics of every launch in an .ncu-rep (ncu --set full):
python tools/ncusum.py X.ncu-rep"""
import csv
import subprocess
import sys

KEYS = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_warps', 'launch__grid_size',
        'sm__inst_executed_pipe_fp64.sum', 'sm__inst_executed_pipe_alu.sum',
        'sm__inst_executed_pipe_fma.sum', 'sm__inst_executed_pipe_lsu.sum',
        'sm__inst_executed_pipe_xu.sum', 'sm__inst_executed_pipe_cbu.sum',
        'sm__inst_executed_pipe_adu.sum', 'sm__inst_executed_pipe_uniform.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__thread_inst_executed_per_inst_executed.ratio']


def main(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        for k in KEYS:
            if k in d:
                print(k, d[k], units[hdr.index(k)])
        for k in hdr:
            if 'average_warps_issue_stalled' in k and k.endswith('per_issue_active.ratio'):
                if float(d[k] or 0) > 0.05:
                    print('  stall', k.split('stalled_')[1].split('_per_issue')[0], d[k])
        print('----')


if __name__ == '__main__':
    main(sys.argv[1])
