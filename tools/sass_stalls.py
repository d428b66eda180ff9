"""Top stall sites of one kernel in an ncu report (source page, SASS view): python tools/sass_stalls.py rep [n]"""
import csv, subprocess, sys, io
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
idx = h.index("Warp Stall Sampling (All Samples)")
ex = h.index("Instructions Executed")
sc = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[idx]) for r in data if r[idx].isdigit())
agg = {}
for r in data:
    for i in sc:
        if r[i].isdigit():
            agg[h[i]] = agg.get(h[i], 0) + int(r[i])
print("samples", tot, {k: v for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]})
for r in sorted(data, key=lambda r: -int(r[idx]) if r[idx].isdigit() else 0)[:n]:
    st = sorted(((h[i], int(r[i])) for i in sc if r[i].isdigit() and int(r[i]) > 0), key=lambda x: -x[1])[:2]
    print(r[0][-5:], r[idx].rjust(5), r[ex].rjust(8), r[1].strip()[:70], st)
