"""Per-kernel summary of an ncu --csv --metrics launch list (mean over launches)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, defaultdict(lambda: defaultdict(list))
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg[d["Kernel Name"][:70]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
for k, m in agg.items():
    t = m.get("gpu__time_duration.sum", [0])
    rd, wr = m.get("dram__bytes_read.sum", [0]), m.get("dram__bytes_write.sum", [0])
    tm = sum(t) / len(t)
    gb = (sum(rd) / len(rd) + sum(wr) / len(wr)) / 1e9
    print(f"{len(t):3d}x {tm / 1e3:9.1f} us  dram {gb:6.3f} GB  {gb / (tm * 1e-9) / 1e3 if tm else 0:6.2f} TB/s  {k}")
