"""Stall samples per CUDA source line of an ncu report (needs -lineinfo + --import-source):
usage src_stalls.py rep [ntop]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
res = []
fname, hdr = None, None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == 'File Path':
        fname = row[1].split('/')[-1]; hdr = None; continue
    if row[0] == 'Line No':
        hdr = row
        si = hdr.index('Warp Stall Sampling (All Samples)')
        sc = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
        continue
    if hdr is None or len(row) <= si or row[si] in ('', '-'):
        continue
    try:
        v = float(row[si])
    except ValueError:
        continue
    if v > 0:
        st = sorted(((hdr[c][6:], float(row[c] or 0)) for c in sc if row[c] not in ('', '-')), key=lambda t: -t[1])[:3]
        res.append((v, fname, row[0], row[1].strip()[:60], st))
tot = sum(r[0] for r in res) or 1
for v, f, ln, src, st in sorted(res, key=lambda r: -r[0])[:ntop]:
    print(f"{100*v/tot:5.1f}% {f}:{ln:5s} {src:60s} {[(n, int(x)) for n, x in st]}")
