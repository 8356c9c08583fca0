"""Hot SASS instructions of an ncu --page source --csv --print-source sass dump,
with their dominant stall reasons, plus context lines around one of them."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data)
agg = {s: sum(int(d[s]) for d in data) for s in stalls}
print("total samples", tot)
print("  ", sorted(((v, k) for k, v in agg.items()), reverse=True)[:8])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
idx = sorted(range(len(data)), key=lambda i: -int(data[i]["Warp Stall Sampling (All Samples)"]))[:n]
for i in idx:
    d = data[i]
    top = sorted(((int(d[s]), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{i:5d} {d['Address'][-5:]} {int(d['Warp Stall Sampling (All Samples)']):6d} "
          f"{d['Source'].strip()[:60]:60s} {top}")
if len(sys.argv) > 3:
    c = int(sys.argv[3])
    for j in range(max(0, c - 25), min(len(data), c + 8)):
        d = data[j]
        print(f"{j:5d} {int(d['Warp Stall Sampling (All Samples)']):6d} {d['Source'].strip()[:90]}")
