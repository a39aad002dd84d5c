"""Summaries of an ncu report read here (no GPU): per-kernel key metrics and the top stall lines.
usage: python scripts/ncu_summary.py REPORT.ncu-rep [--source N]"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'lts__t_requests_srcunit_tex_op_read.sum', 'lts__t_requests_srcunit_tex_op_red.sum',
        'lts__t_requests_srcunit_tex_op_atom.sum', 'lts__t_requests_srcunit_tex_op_write.sum',
        'launch__registers_per_thread', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']
STALLS = ['long_scoreboard', 'short_scoreboard', 'barrier', 'mio_throttle', 'lg_throttle', 'wait',
          'math_pipe_throttle', 'not_selected', 'selected', 'no_instruction', 'branch_resolving',
          'dispatch_stall', 'drain', 'membar', 'sleeping', 'tex_throttle', 'imc_miss', 'misc']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        res.append(d)
    return res


def main():
    rep = sys.argv[1]
    for d in raw(rep):
        print(d.get('Kernel Name', '')[:70])
        for k in KEYS:
            if k in d:
                print(f"   {k:60s} {d[k]}")
        st = []
        for s in STALLS:
            k = f'smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio'
            if k in d and d[k] not in ('', 'n/a'):
                st.append((float(d[k]), s))
        print('   stalls/issue:', ', '.join(f'{s}={v:.2f}' for v, s in sorted(st, reverse=True)[:8]))
    if '--source' in sys.argv:
        n = int(sys.argv[sys.argv.index('--source') + 1])
        out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address']
        for j, h0 in enumerate(hi):
            h = rows[h0]
            iS, iW = h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
            iI, iT = h.index('Instructions Executed'), h.index('Avg. Threads Executed')
            end = hi[j + 1] - 1 if j + 1 < len(hi) else len(rows)
            data = []
            for r in rows[h0 + 1:end]:
                try:
                    data.append((r[iS], int(r[iW] or 0), int(r[iI] or 0), float(r[iT] or 0)))
                except (ValueError, IndexError):
                    pass
            print(f'--- kernel {j}: warp instr {sum(x[2] for x in data)}, samples {sum(x[1] for x in data)}')
            for s_, w, i, t in sorted(data, key=lambda x: -x[1])[:n]:
                print(f'{i:>12} {w:>7} {t:5.1f}  {s_[:90]}')


if __name__ == '__main__':
    main()
