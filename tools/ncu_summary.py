"""Summarise an ncu report: key throughput counters + top stall reasons + hottest SASS."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum', 'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic', 'launch__grid_size',
        'launch__block_size', 'sm__cycles_elapsed.avg.per_second',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2]


def main(rep, top=12):
    h, u, v = raw(rep)
    res = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            res[k] = f"{v[i]} {u[i]}"
            print(f"{k:70s} {v[i]} {u[i]}")
    stalls = []
    for i, n in enumerate(h):
        if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued'):
            try:
                stalls.append((float(v[i].replace(',', '')), n.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    print("stalls:", ", ".join(f"{n} {s / tot * 100:.0f}%" for s, n in sorted(stalls, reverse=True)[:6]))
    return res


if __name__ == "__main__":
    main(sys.argv[1])
