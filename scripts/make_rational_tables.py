#!/usr/bin/env python
"""Write data/rational/<config>.json: the shared poles and residue table of
PAPER.md §3.2 (eq:ratfam, fitted by RKFIT per eq:rkfit) for each BASELINE
config's time channels and degree.

This script calls only ``oracle/`` (oracle.rkfit).  The tables are INPUTS to
both sides -- "poles and residues computed once on the host from the paper's
construction" (BASELINE.json north star) -- exactly as the conductivity and
source are.  Re-run after any change to oracle/rkfit.py:

    python scripts/make_rational_tables.py            # all configs
    python scripts/make_rational_tables.py tiny block
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import rkfit  # noqa: E402
from workloads import CONFIG_NAMES, make_workload  # noqa: E402

OUT = os.path.join(ROOT, "data", "rational")


def _c(a):
    a = np.asarray(a, dtype=np.complex128)
    return [[float(z.real), float(z.imag)] for z in a.ravel()]


def table_for(times, degree):
    fam = rkfit.fit_family(times, degree)
    poles_x, res_x, is_pair = fam.physical()
    errs = rkfit.channel_errors(fam)
    return {
        "paper_ref": "PAPER.md §3.2 eq:ratfam/eq:rkfit/eq:rmj; fitted by oracle/rkfit.py",
        "degree": int(degree),
        "t_max": float(fam.t_max),
        "times": [float(t) for t in fam.times],
        "weights": [float(w) for w in fam.weights],
        "poles_normalised": _c(fam.poles),
        "residues_normalised": [_c(fam.residues[i]) for i in range(fam.degree)],
        # physical variable x (1/s): u(t_j) = sum_i w_i Re(alpha_ij (K - xi_i M)^-1 f)
        "shifts": _c(-poles_x),               # s_i = -xi_i: (K + s_i M) x_i = f
        "residues": [_c(res_x[i]) for i in range(poles_x.size)],   # (n_shift, K)
        "is_pair": [bool(b) for b in is_pair],
        "channel_errors": [float(e) for e in errs],
        "uniform_error": float(np.max(fam.weights * errs)),
    }


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for name in names:
        wl = make_workload(name)
        tab = table_for(wl.times, wl.n_poles)
        tab["config"] = name
        path = os.path.join(OUT, f"{name}.json")
        with open(path, "w") as fh:
            json.dump(tab, fh, indent=1)
        print(f"{name}: degree {tab['degree']}, {len(tab['shifts'])} shifted systems, "
              f"uniform error {tab['uniform_error']:.2e} -> {path}")


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIG_NAMES))
