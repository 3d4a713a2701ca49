"""Stall samples of an ncu report aggregated by source line (via nvdisasm -g of the
kernel's cubin).  python tools/ncu_lines.py rep.ncu-rep mangled_kernel_name [N] [min_exec max_exec]"""
import csv, io, subprocess, collections, re, sys, os, tempfile
rep, kname = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lo, hi = (float(sys.argv[4]), float(sys.argv[5])) if len(sys.argv) > 5 else (-1, 1e18)
so = os.path.join(os.path.dirname(__file__), "..", "paper_2504_02658_b200", "lib", "libmilo_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(txt) if l.startswith(".text." + kname + ":"))
lines, cur = {}, None
for l in txt[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        lines[int(m.group(1), 16)] = cur
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]; ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
def f(r, k):
    try: return float(r[ix[k]].replace(",", ""))
    except Exception: return 0.0
S, I = "Warp Stall Sampling (All Samples)", "Instructions Executed"
base = min(int(r[ix["Address"]], 16) for r in data)
tot = sum(f(r, S) for r in data)
agg = collections.defaultdict(lambda: [0.0, 0.0])
for r in data:
    if not (lo <= f(r, I) <= hi):
        continue
    ln = lines.get(int(r[ix["Address"]], 16) - base)
    agg[ln][0] += f(r, S); agg[ln][1] += f(r, I)
srcs = {}
for ln, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    t = ""
    if ln:
        p = os.path.join(os.path.dirname(__file__), "..", "paper_2504_02658_b200", "csrc", ln[0])
        if os.path.exists(p):
            srcs.setdefault(p, open(p).read().split("\n")); t = srcs[p][ln[1] - 1].strip()[:80]
    print(f"{str(ln):34s} {s / tot:6.1%} inst={i:10.0f} {t}")
