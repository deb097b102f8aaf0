"""Record the DRAM traffic of one kernel launch from an ncu --set full report into
profiles/ncu_traffic.json, keyed by bench.py's "<workload>|<variant>|<profiled kernel name>" and
stamped with the sha of the CUDA sources it was captured on (bench.py reuses a figure only
for the same key and the same sources).
usage: ncu_traffic.py <report.ncu-rep> <key> [kernel-name-regex]"""
import csv, io, json, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import csrc_sha  # noqa: E402

rep, key = sys.argv[1], sys.argv[2]
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
best = None
for v in rows[2:]:
    name = v[hdr.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    def val(m):
        i = hdr.index(m)
        x = float(v[i].replace(",", ""))
        u = units[i].lower()
        return x * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}.get(u, 1)
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    best = {"bytes_per_launch": rd + wr, "read": rd, "write": wr, "kernel": name[:120],
            "csrc_sha": csrc_sha(), "source": os.path.basename(rep)}
    break
if best is None:
    raise SystemExit("no matching kernel in " + rep)
p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
d = json.load(open(p)) if os.path.exists(p) else {}
d = {k: e for k, e in d.items() if isinstance(e, dict)}  # drop round-1 bare numbers
d[key] = best
json.dump(d, open(p, "w"), indent=1, sort_keys=True)
print(key, best)
