"""Summarise an ncu report (raw page) into the metrics we track; usage: ncu_summary.py rep [rep...]"""
import csv, subprocess, sys, io
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size', 'smsp__inst_executed.sum',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__cycles_elapsed.avg.per_second']
STALL = 'smsp__pcsamp_warps_issue_stalled_'
for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"== {rep} :: {vals[hdr.index('Kernel Name')][:80]}")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w:70s} {vals[i]} {units[i]}")
        st = [(hdr[i][len(STALL):], vals[i]) for i in range(len(hdr)) if hdr[i].startswith(STALL) and not hdr[i].endswith('not_issued')]
        st = sorted(((n, float(v.replace(',', ''))) for n, v in st if v.replace(',', '').replace('.', '').isdigit()), key=lambda t: -t[1])
        tot = sum(v for _, v in st) or 1
        print("  stalls:", ", ".join(f"{n}={100*v/tot:.0f}%" for n, v in st[:8]))
