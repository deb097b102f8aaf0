"""Top stall sites of an ncu report (SASS view) with a window of surrounding instructions."""
import csv, subprocess, sys, io
rep = sys.argv[1]; ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
si = hdr.index('Warp Stall Sampling (All Samples)')
ie = hdr.index('Instructions Executed') if 'Instructions Executed' in hdr else None
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(float(r[si] or 0) for r in data)
idx = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:ntop]
for i in idx:
    r = data[i]
    st = sorted(((hdr[c][6:], float(r[c] or 0)) for c in stall_cols), key=lambda t: -t[1])[:2]
    print(f"{100*float(r[si])/tot:5.1f}% [{i:5d}] {r[1][:70]:70s} {st}")
