"""Table of an ncu launch list of the split passes (scripts/traffic_sweep*.sh):
time, DRAM read/write bytes against the algorithmic bytes, L2 read hit rate.

    python scripts/traffic_table.py <n_complex> <n_real> gpurun_out/tr_x.csv ...
"""
import csv
import sys
from collections import defaultdict

N = 13984256   # free edges of `large`
nc, nr = int(sys.argv[1]), int(sys.argv[2])
units = nc * 16 + nr * 8   # bytes of one value of every active shift
RD = {"k_sweep<3, 12>": 2, "k_sweep<4, 12>": 3, "k_delta<0, 12>": 1}
WR = {"k_sweep<3, 12>": 2, "k_sweep<4, 12>": 3, "k_delta<0, 12>": 0}
for fn in sys.argv[3:]:
    lines = [ln for ln in open(fn) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    ix = {k: i for i, k in enumerate(rows[0])}
    per, names = defaultdict(dict), {}
    for r in rows[1:]:
        per[int(r[ix["ID"]])][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        names[int(r[ix["ID"]])] = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
    print(fn)
    for i in sorted(per):
        m, k = per[i], names[i]
        t = m["gpu__time_duration.sum"] * 1e-9
        rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
        ar, aw = RD[k] * units * N, WR[k] * units * N
        hit = (m.get("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", 0)
               / max(1.0, m.get("lts__t_sectors_srcunit_tex_op_read.sum", 1.0)))
        print(f"  {k:16s} {t * 1e3:7.3f} ms  R {rd / 1e9:6.3f} GB (alg {ar / 1e9:6.3f}, x{rd / ar:5.3f})  "
              f"W {wr / 1e9:6.3f} GB  DRAM {(rd + wr) / t / 1e12:5.2f} TB/s  algorithmic "
              f"{(ar + aw) / t / 1e12:5.2f} TB/s  L2 tex read hit {hit:.2f}  inst {m.get('smsp__inst_executed.sum', 0) / 1e6:7.1f}M")
