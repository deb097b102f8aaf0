"""Shared-memory wavefronts per CUDA source line of an ncu report (--set full, -lineinfo):
actual vs ideal (the excess is bank conflicts), per tile of the two-level engine if --tiles N.
usage: smem_wavefronts.py rep [ntop] [tiles]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tiles = float(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
res, fname, hdr, line = {}, None, None, None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == 'File Path':
        fname = row[1].split('/')[-1]; continue
    if row[0] == 'Line No':
        hdr = row; iw = hdr.index('L1 Wavefronts Shared'); ii = hdr.index('L1 Wavefronts Shared Ideal'); continue
    if hdr is None:
        continue
    if row[0] != '':
        line = (fname, row[0], row[1][:60]); continue
    if not row[2].startswith('0x'):
        continue
    try:
        w = float(row[iw].replace(',', '')); wi = float(row[ii].replace(',', ''))
    except ValueError:
        continue
    if w == 0:
        continue
    r = res.setdefault(line, [0.0, 0.0, set()])
    r[0] += w; r[1] += wi; r[2].add(row[3].split()[0])
tot = sum(v[0] for v in res.values()) or 1
toti = sum(v[1] for v in res.values())
sc = (1.0 / tiles) if tiles else 1.0
print(f"total shared wavefronts {tot:.3e} ({tot*sc:.0f} per tile), ideal {toti:.3e} (excess {100*(tot-toti)/tot:.0f}%)")
for (f, ln, src), (w, wi, ops) in sorted(res.items(), key=lambda t: -t[1][0])[:ntop]:
    print(f"{100*w/tot:5.1f}% {w*sc:8.0f} ideal {wi*sc:8.0f}  {f}:{ln:4s} {','.join(sorted(ops)):14s} {src}")
