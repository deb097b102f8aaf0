"""ncu --metrics gpu__time_duration.sum --csv launch list -> per-launch ms + each kernel's share.
usage: launch_list.py <launches.csv> <header line>"""
import csv, io, sys, collections
rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = list(csv.reader(io.StringIO("".join(rows))))
hdr = r[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
print("# " + sys.argv[2])
tot = collections.Counter()
for v in r[1:]:
    ms = float(v[vi].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}[v[ui]]
    print(f"{ms:10.4f} ms  {v[ki][:90]}")
    tot[v[ki].split("(")[0]] += ms
s = sum(tot.values())
print("# share of device time:")
for k, t in tot.most_common():
    print(f"#   {100 * t / s:6.2f}%  {k}")
