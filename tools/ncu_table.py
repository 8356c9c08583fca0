"""Summarise an ncu --csv launch list: one line per launch (name, metrics)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"].split("(")[0][:70])
        out.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for (i, name), m in sorted(out.items()):
    t = m.get("gpu__time_duration.sum", 0) / 1e6
    rd = m.get("dram__bytes_read.sum", 0) / 1e9
    wr = m.get("dram__bytes_write.sum", 0) / 1e9
    bw = (rd + wr) / (t * 1e-3) if t else 0
    print(f"{i:3d} {name:72s} {t:7.3f} ms  rd {rd:6.2f} GB  wr {wr:6.2f} GB  {bw:7.0f} GB/s")
