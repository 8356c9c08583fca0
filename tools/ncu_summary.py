"""Markdown summary of full ncu captures (raw page CSVs + source page CSVs):
time, DRAM traffic and throughput, issue/occupancy, smem conflicts, top
stall reasons. usage: ncu_summary.py <tag> k1 k2 ... (files gpurun_out/<tag>_<k>_*.csv)"""
import csv
import sys

tag, kernels = sys.argv[1], sys.argv[2:]
# the raw page's second row carries the units (ms, Gbyte, ...); values as given
keys = [
    ("gpu__time_duration.sum", "time", 1),
    ("dram__bytes_read.sum", "DRAM read", 1),
    ("dram__bytes_write.sum", "DRAM write", 1),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)", 1),
    ("smsp__inst_executed.sum", "warp instructions", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (% of max)", 1),
    ("launch__registers_per_thread", "registers/thread", 1),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA", 1),
    ("launch__grid_size", "CTAs", 1),
    ("launch__block_size", "threads/CTA", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts", 1),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate (%)", 1),
]
rows, units = {}, {}
for k in kernels:
    r = list(csv.reader(open(f"gpurun_out/{tag}_{k}_raw.csv")))
    rows[k] = dict(zip(r[0], r[2]))
    units = dict(zip(r[0], r[1]))
print("| metric | " + " | ".join(kernels) + " |")
print("|---|" + "---|" * len(kernels))
for key, label, scale in keys:
    vals = []
    for k in kernels:
        v = rows[k].get(key, "")
        try:
            vals.append(f"{float(v.replace(',', '')) * scale:.3g}")
        except ValueError:
            vals.append(v or "-")
    u = units.get(key, "")
    print(f"| {label}{' (' + u + ')' if u else ''} | " + " | ".join(vals) + " |")
# traffic-derived bandwidth (units: time ms, bytes Gbyte as ncu prints them)
scale_t = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}
scale_b = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}
bw = []
for k in kernels:
    d = rows[k]
    t = float(d["gpu__time_duration.sum"].replace(",", "")) * scale_t.get(units["gpu__time_duration.sum"], 1)
    b = sum(float(d[x].replace(",", "")) * scale_b.get(units[x], 1)
            for x in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    bw.append(f"{b / t / 1e9:.0f}")
print("| DRAM GB/s (read+write / time) | " + " | ".join(bw) + " |")
print()
for k in kernels:
    r = list(csv.reader(open(f"gpurun_out/{tag}_{k}_src.csv")))
    hdr = r[1]
    data = [dict(zip(hdr, x)) for x in r[2:] if len(x) == len(hdr)]
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data)
    agg = sorted(((sum(int(d[s]) for d in data), s[6:]) for s in stalls), reverse=True)[:6]
    print(f"* `{k}` stall samples: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in agg))
