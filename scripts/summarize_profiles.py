#!/usr/bin/env python
"""Summarise ncu outputs into profiles/<round>/ (run here, no GPU needed).

    python scripts/summarize_profiles.py launches gpurun_out/launches.csv profiles/r01/launches_summary.csv
    python scripts/summarize_profiles.py full gpurun_out/prof.ncu-rep profiles/r01/ncu_full_summary.json

`launches`: per-kernel launch counts, summed device time and share of the
first N launches of `ncu --metrics gpu__time_duration.sum` (cold-cache,
serialised: compare shares, not absolutes).
`full`: the roofline-relevant metrics and the top stall reasons of an
`ncu --set full` capture, one record per profiled launch.
"""
import collections
import csv
import json
import os
import subprocess
import sys

FULL_METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
    "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
]


def launches(src, dst):
    rows = list(csv.DictReader(l for l in open(src) if not l.startswith("==")))
    agg = collections.OrderedDict()
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        t = float(r["Metric Value"])
        a = agg.setdefault(name, [0, 0.0, r["Grid Size"], r["Block Size"]])
        a[0] += 1
        a[1] += t
    tot = sum(a[1] for a in agg.values())
    out = [f"# ncu launch list ({len(rows)} launches): {src}",
           "# cold-cache, serialised per-launch times: compare SHARES, not absolutes",
           "kernel,launches,total_ms,mean_us,share,grid,block"]
    for k, (n, t, g, b) in agg.items():
        out.append(f"{k},{n},{t / 1e6:.3f},{t / n / 1e3:.1f},{t / tot:.3f},\"{g}\",\"{b}\"")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def full(src, dst):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {w: (r[hdr.index(w)] + " " + units[hdr.index(w)]).strip() for w in FULL_METRICS if w in hdr}
        items = [(h, v) for h, v in zip(hdr, r)
                 if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")]
        vals = [(h, float(v)) for h, v in items if v.replace(".", "").isdigit()]
        tot = sum(v for _, v in vals) or 1.0
        d["top_stalls"] = ", ".join(
            f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v / tot * 100:.0f}%"
            for h, v in sorted(vals, key=lambda x: -x[1])[:6])
        try:
            t = float(r[hdr.index("gpu__time_duration.sum")])
            unit = units[hdr.index("gpu__time_duration.sum")]
            ms = t if unit == "ms" else t / 1e3 if unit == "us" else t / 1e6
            rd = float(r[hdr.index("dram__bytes_read.sum")])
            wr = float(r[hdr.index("dram__bytes_write.sum")])
            bu = units[hdr.index("dram__bytes_read.sum")]
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "byte": 1.0, "Kbyte": 1e3}.get(bu, 1.0)
            d["dram_GBps"] = round((rd + wr) * scale / (ms * 1e-3) / 1e9, 1)
        except (ValueError, IndexError):
            pass
        recs.append(d)
    json.dump(recs, open(dst, "w"), indent=1)
    for d in recs:
        print("---")
        for k, v in d.items():
            print(f"  {k}: {v}")


def _bytes(v):
    x, unit = v.split()
    return float(x) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[unit]


def traffic(src, dst):
    """profiles/traffic.json `split` entry from a `full` summary of the split
    passes on the bench workload (`large`, library poles: 10 complex + 4 real
    shifts, all active): DRAM bytes per COCG iteration = mean of an even and an
    odd pass 1 plus pass 2, against the algorithmic bytes."""
    recs = json.load(open(src))
    per = {}
    for r in recs:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("tem::", "")
        name = name.replace("(int)", "").replace("(bool)", "")
        per.setdefault(name, []).append(_bytes(r["dram__bytes_read.sum"]) + _bytes(r["dram__bytes_write.sum"]))
    per = {k: sum(v) / len(v) for k, v in per.items()}
    ev = next(v for k, v in per.items() if k.startswith("k_sweep<3"))
    od = next(v for k, v in per.items() if k.startswith("k_sweep<4"))
    de = next(v for k, v in per.items() if k.startswith("k_delta"))
    n_unknowns, n_complex, n_real = 13984256, 10, 4
    alg = 96.0 * n_unknowns * n_complex + 48.0 * n_unknowns * n_real
    out = json.load(open(dst)) if os.path.exists(dst) else {}
    out["split"] = {
        "source": src + " (ncu --set full, `large`, library poles: 10 complex + 4 real shifts, all active)",
        "workload": "large", "poles": "fit",
        "traffic_bytes_per_iteration": 0.5 * (ev + od) + de,
        "algorithmic_bytes_per_iteration": alg,
        "bytes_per_complex_sui": (0.5 * (ev + od) + de) / (n_unknowns * (n_complex + 0.5 * n_real)),
        "algorithmic_bytes_per_complex_sui": 96.0,
        "per_kernel_bytes": per,
        "iteration": "mean of an even (k_sweep<3,12>) and an odd (k_sweep<4,12>) pass 1, plus k_delta",
    }
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out["split"], indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](sys.argv[2], sys.argv[3])
