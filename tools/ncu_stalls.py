"""Stall-reason breakdown of an ncu report's source page, overall and for the
instructions of given SASS opcodes.  python tools/ncu_stalls.py rep.ncu-rep"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hi]; ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
def f(r, k):
    try: return float(r[ix[k]].replace(",", ""))
    except Exception: return 0.0
tot = collections.Counter(); byop = collections.defaultdict(collections.Counter)
for r in data:
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    for k in reasons:
        v = f(r, k); tot[k] += v; byop[op][k] += v
T = sum(tot.values())
print("overall:", ", ".join(f"{k[6:]} {v / T:.1%}" for k, v in tot.most_common(10)))
for op, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:16]:
    s = sum(c.values())
    print(f"{op:10s} {s / T:6.1%}: " + ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in c.most_common(4)))
