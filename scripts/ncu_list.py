"""Summarise an `ncu --csv --metrics ...` launch list: one line per launch."""
import csv
import sys
from collections import defaultdict

for fn in sys.argv[1:]:
    lines = [ln for ln in open(fn) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[int(r[ix["ID"]])][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        names[int(r[ix["ID"]])] = r[ix["Kernel Name"]].split("(")[0]
    print(fn)
    for i in sorted(per):
        m = per[i]
        t = m.get("gpu__time_duration.sum", 0) * 1e-9
        rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
        print(f"  {i:3d} {names[i]:22s} {t*1e3:8.3f} ms  R {rd/1e9:6.2f} GB  W {wr/1e9:6.2f} GB  "
              f"{(rd+wr)/t/1e12 if t else 0:5.2f} TB/s  inst {m.get('smsp__inst_executed.sum',0)/1e6:7.1f}M  "
              f"clk {m.get('sm__cycles_elapsed.avg.per_second',0)/1e9:4.2f} GHz")
