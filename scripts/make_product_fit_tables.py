#!/usr/bin/env python
"""Write data/rational/<config>_fit.json: the PRODUCT's own shared-pole
family (tem_fit_family, host C++; what `bench.py --poles fit` computes at
run time) for each BASELINE config, so that the oracle arm of bench.py
(`--impl reference`, `cpu_baseline`) times the oracle on exactly the
shifted systems the GPU arm solves without running product code itself.
Deterministic: tests/test_product_fit.py checks the files against a fresh
fit.

    python scripts/make_product_fit_tables.py [config ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2506_11657_b200 import RationalTable  # noqa: E402
from workloads import CONFIG_NAMES, make_workload  # noqa: E402

for name in sys.argv[1:] or CONFIG_NAMES:
    wl = make_workload(name)
    tab = RationalTable.fit(wl.times, wl.n_poles)
    rec = tab.to_json()
    rec.update({"paper_ref": "PAPER.md §3.2 eq:ratfam/eq:rkfit/eq:rmj; fitted by tem_fit_family (product)",
                "degree": int(wl.n_poles), "config": name})
    path = os.path.join(ROOT, "data", "rational", f"{name}_fit.json")
    with open(path, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(path, tab.n_shift, "systems", int((~tab.is_pair).sum()), "real")
