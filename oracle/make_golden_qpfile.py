"""Generate tests/golden/qpfile.npz with the REAL reference's QP file dialect.

TEST INFRASTRUCTURE ONLY (build container, reference read-only at
/root/reference):  python oracle/make_golden_qpfile.py

For seeded problems of every file-representable Hessian kind (the reference
test generator oracles.random_problem) plus hand-written documents (nulls,
duplicate COO entries, missing optional members), it records the document
text the reference writes (cli.qp_document, json.dumps) and the arrays the
reference's parser (cli.parse_qp_document) builds from it, and the device-IPM
reference answer of the reference's solve() on each parsed problem.
tests/test_qpfile.py checks paper_2308_00637_b200.qpfile against them.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
ROOT = Path(__file__).resolve().parents[1]

import qpipm.cli as ref_cli  # noqa: E402
import qpipm.ipm as ref_ipm  # noqa: E402
from oracles import random_problem  # noqa: E402

OUT = ROOT / "tests" / "golden"


def docs():
    out = []
    for seed, kind in enumerate(["diagonal", "sparse", "bfgs", "diagonal", "sparse", "bfgs"]):
        p = random_problem(np.random.default_rng(500 + seed), hessian_kind=kind)
        out.append((f"random_{kind}_{seed}", json.dumps(ref_cli.qp_document(p))))
    # hand-written: nulls, duplicate COO entries (summed), optional members absent
    out.append(("handwritten_dups", json.dumps({
        "n": 3, "hessian": {"kind": "coo", "rows": [0, 1, 2, 0, 1], "cols": [0, 1, 2, 0, 0],
                            "vals": [1.0, 2.0, 3.0, 0.5, 0.25]},
        "p": [1, -1, 0.5], "A": {"rows": [0, 0, 1, 0], "cols": [0, 2, 1, 0], "vals": [1, 1, 1, 2]},
        "l": [None, -1.0], "u": [4.0, None], "lx": [0, None, -2], "ux": [None, 3, 2]})))
    out.append(("handwritten_minimal", json.dumps({"n": 2, "hessian": {"kind": "diagonal", "d": [1, 2]},
                                                    "p": [0, 0], "lx": [0, 0]})))
    return out


def main():
    rec, names = {}, []
    for name, text in docs():
        prob = ref_cli.parse_qp_document(json.loads(text))
        p = name + "_"
        names.append(name)
        rec[p + "text"] = np.array(text)
        for mname in ("a", "c"):
            m = getattr(prob, mname)
            rec[p + mname + "_ro"] = np.asarray(m.row_offsets, dtype=np.int64)
            rec[p + mname + "_ci"] = np.asarray(m.col_indices, dtype=np.int64)
            rec[p + mname + "_v"] = np.asarray(m.values, dtype=np.float64)
        for f in ("p", "b"):
            rec[p + f] = np.asarray(getattr(prob, f), dtype=np.float64)
        rec[p + "bounds"] = np.stack([prob.lin_bounds.lower, prob.lin_bounds.upper]) if len(prob.lin_bounds) \
            else np.zeros((2, 0))
        rec[p + "vbounds"] = np.stack([prob.var_bounds.lower, prob.var_bounds.upper])
        h = prob.hessian
        kind = type(h).__name__
        rec[p + "hkind"] = np.array(kind)
        if kind == "DiagonalHessian":
            rec[p + "h_d"] = h.d
        elif kind == "SparseHessian":
            rec[p + "h_ro"], rec[p + "h_ci"], rec[p + "h_v"] = h.m.row_offsets, h.m.col_indices, h.m.values
        else:
            rec[p + "h_h0"], rec[p + "h_u"], rec[p + "h_w"] = h.h0_diag, h.u, h.w
        rep = ref_ipm.solve(prob)
        rec[p + "x"] = rep.x
        rec[p + "status"] = np.array(rep.status.value)
        rec[p + "objective"] = np.float64(rep.objective)
        print(name, kind, rep.status.value, rep.iterations)
    rec["names"] = np.array(names)
    np.savez_compressed(OUT / "qpfile.npz", **rec)


if __name__ == "__main__":
    main()
