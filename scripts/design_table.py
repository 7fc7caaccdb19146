"""Print the DESIGN.md "Measured, round 2" table from profiles/r02/bench_*.json."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
print("| config | unknowns | systems | wall time to all channels (ms) | plain 1e-10 solve (ms) | SUI/s | "
      "roofline frac | e2e SUI/s | max channel error | outside COCG (ms) | clocks |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for c in ("tiny", "block", "layered", "hetero", "large"):
    d = json.load(open(os.path.join(ROOT, "profiles", "r02", f"bench_{c}.json")))
    g = d["config"]
    clk = f"{d['clocks']['sm_mhz']:.0f} MHz" + (", " + ", ".join(d["clocks"]["reasons"]) if d["clocks"]["reasons"] else "")
    sys_ = f"{g['shifts']}" + (f" ({g['real_shifts']} real)" if g["real_shifts"] else "")
    print(f"| {c} | {g['unknowns']:,} | {sys_} | {d['ms_per_step']:.4g} | {g['plain_solve']['ms']:.4g} | "
          f"{d['value']:.3g} | {d['roofline']['frac']:.3f} | {d['e2e']['value']:.3g} | "
          f"{g['field_accuracy']['max_channel_rel_l2_conducting']:.1e} | {g['outside_cocg_ms_per_step']:.3g} | {clk} |")
