"""Hot SASS instructions of an ncu report (source page): python tools/ncu_hot.py rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
def f(r, k):
    try: return float(r[ix[k]].replace(",", ""))
    except: return 0.0
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_i = sum(f(r, "Instructions Executed") for r in data)
print(f"total samples {tot_s:.0f}, warp instr {tot_i:.0f}")
data.sort(key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for r in data[:N]:
    top = sorted(((f(r, k), k) for k in stalls), reverse=True)[:2]
    print(f"{r[ix['Address']]:>6} {f(r,'Warp Stall Sampling (All Samples)')/tot_s:6.1%} inst={f(r,'Instructions Executed'):9.0f} {r[ix['Source']][:60]:60s} {top[0][1]}={top[0][0]:.0f} {top[1][1]}={top[1][0]:.0f}")
