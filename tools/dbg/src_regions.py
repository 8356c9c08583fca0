"""Region breakdown (instructions / stall samples) of an ncu source-page CSV
holding several kernels: tools/dbg/src_regions.py <csv> <kernel index> [block]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ki = int(sys.argv[2])
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 60
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
sec = rows[starts[ki]:starts[ki + 1]]
print(sec[0][1][:120])
hdr = sec[1]
data = [dict(zip(hdr, r)) for r in sec[2:] if len(r) == len(hdr)]
ti = sum(int(d["Instructions Executed"]) for d in data)
ts = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = sorted(((sum(int(d[s]) for d in data), s) for s in stalls), reverse=True)[:8]
print("instrs", ti, "samples", ts, [(s[6:], round(100 * v / ts, 1)) for v, s in agg])
for i in range(0, len(data), blk):
    b = data[i:i + blk]
    ie = sum(int(d["Instructions Executed"]) for d in b)
    ss = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in b)
    if ie * 200 < ti and ss * 200 < ts:
        continue
    ops = {}
    for d in b:
        t = d["Source"].split()
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op] = ops.get(op, 0) + 1
    top = sorted(ops.items(), key=lambda x: -x[1])[:5]
    st = sorted(((sum(int(d[s]) for d in b), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{i:5d} {100 * ie / ti:5.1f}% instr {100 * ss / ts:5.1f}% stall {st} {top}")
