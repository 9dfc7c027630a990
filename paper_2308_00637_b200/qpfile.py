"""The reference's QP file dialect (JSON), read into this package's problem types.

Mirrors ``qpipm/cli.py:37-183`` -- the format the reference's ``solve-qp``
command reads -- with the same member names, defaults (``l``/``u``/``lx``/
``ux`` null = unbounded, missing ``A``/``C`` = empty), COO sparse matrices
(duplicates summed), Hessian kinds ``diagonal`` / ``coo`` / ``bfgs``, and the
same ``QpFileError`` messages naming the offending member:

* ``parse_qp_document(doc)``  cli.py:117-136
* ``load_qp_file(path)``      cli.py:139-147
* ``qp_document(problem)``    cli.py:162-183 (round-trip safe writer)

``solve_file(path, cfg)`` loads a file and runs the device-resident IPM
(``ipm.solve``) on it.  Host-side parsing only; nothing here computes on the
hot path.
"""

from __future__ import annotations

import json

import numpy as np

from .problem import (Bounds, DiagonalHessian, QpProblem, QuasiNewtonHessian, SparseHessian,
                      SparseMatrix)


class QpFileError(ValueError):
    """Problem file is malformed; the message names the offending member."""


def _member(doc: dict, name: str, default=None, required: bool = False):
    if name in doc:
        return doc[name]
    if required:
        raise QpFileError(f"missing member '{name}'")
    return default


def _real_array(raw, name: str, allow_null: bool = False) -> np.ndarray:
    if not isinstance(raw, list):
        raise QpFileError(f"member '{name}' must be an array")
    out = np.empty(len(raw))
    for i, v in enumerate(raw):
        if v is None:
            if not allow_null:
                raise QpFileError(f"member '{name}' contains null at position {i}")
            out[i] = np.nan
        elif isinstance(v, bool) or not isinstance(v, (int, float)):
            raise QpFileError(f"member '{name}' contains non-numeric entry at position {i}")
        else:
            out[i] = float(v)
    return out


def _bounds(doc: dict, lname: str, uname: str) -> Bounds:
    lo = _real_array(doc.get(lname, []), lname, allow_null=True)
    hi = _real_array(doc.get(uname, []), uname, allow_null=True)
    if len(lo) != len(hi):
        raise QpFileError(f"members '{lname}' and '{uname}' have different lengths")
    return Bounds(np.where(np.isnan(lo), -np.inf, lo), np.where(np.isnan(hi), np.inf, hi))


def _coo(doc, name: str, n_rows: int, n_cols: int) -> SparseMatrix:
    if doc is None:
        return SparseMatrix.empty(n_rows, n_cols)
    missing = [k for k in ("rows", "cols", "vals") if k not in doc]
    if missing:
        raise QpFileError(f"member '{name}' is missing '{missing[0]}'")
    vals = _real_array(doc["vals"], f"{name}.vals")
    rows, cols = doc["rows"], doc["cols"]
    if not (len(rows) == len(cols) == len(vals)):
        raise QpFileError(f"member '{name}': rows/cols/vals lengths differ")
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if len(rows) and (rows.min() < 0 or rows.max() >= n_rows or cols.min() < 0 or cols.max() >= n_cols):
        raise QpFileError(f"member '{name}': coordinate index out of range")
    return _from_coo(n_rows, n_cols, rows, cols, vals)


def _from_coo(n_rows, n_cols, rows, cols, vals) -> SparseMatrix:
    """CSR with duplicates summed and columns sorted per row (model.py:53-63)."""
    key = rows * max(n_cols, 1) + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    uniq, start = np.unique(key, return_index=True)
    summed = np.add.reduceat(vals, start) if len(vals) else vals
    r, c = (uniq // max(n_cols, 1)), (uniq % max(n_cols, 1))
    ro = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(ro, r + 1, 1)
    return SparseMatrix(n_rows, n_cols, np.cumsum(ro), c, summed)


def _hessian(doc, n: int):
    if not isinstance(doc, dict) or "kind" not in doc:
        raise QpFileError("member 'hessian' must be an object with a 'kind'")
    kind = doc["kind"]
    if kind == "diagonal":
        d = _real_array(_member(doc, "d", required=True), "hessian.d")
        if len(d) != n:
            raise QpFileError("member 'hessian.d' has wrong length")
        return DiagonalHessian(d)
    if kind == "coo":
        return SparseHessian(_coo(doc, "hessian", n, n))
    if kind == "bfgs":
        h0 = _real_array(_member(doc, "h0_diag", required=True), "hessian.h0_diag")
        w = _real_array(_member(doc, "w", required=True), "hessian.w")
        u_rows = _member(doc, "u", required=True)
        if not isinstance(u_rows, list) or len(u_rows) != n:
            raise QpFileError("member 'hessian.u' must be an n-row array of arrays")
        u = np.array([_real_array(row, "hessian.u") for row in u_rows]) if n else np.zeros((0, len(w)))
        if u.shape != (n, len(w)):
            raise QpFileError("member 'hessian.u' has inconsistent row lengths")
        return QuasiNewtonHessian(h0, u, w)
    raise QpFileError(f"member 'hessian.kind' has unknown value '{kind}'")


def parse_qp_document(doc) -> QpProblem:
    if not isinstance(doc, dict):
        raise QpFileError("document root must be an object")
    n = _member(doc, "n", required=True)
    if isinstance(n, bool) or not isinstance(n, int) or n < 0:
        raise QpFileError("member 'n' must be a nonnegative integer")
    p = _real_array(_member(doc, "p", required=True), "p")
    lin_bounds = _bounds(doc, "l", "u")
    var_bounds = _bounds({"lx": doc.get("lx", [None] * n), "ux": doc.get("ux", [None] * n)}, "lx", "ux")
    b = _real_array(doc.get("b", []), "b")
    hessian = _hessian(_member(doc, "hessian", required=True), n)
    return QpProblem(n=n, hessian=hessian, p=p, a=_coo(doc.get("A"), "A", len(lin_bounds), n),
                     lin_bounds=lin_bounds, c=_coo(doc.get("C"), "C", len(b), n), b=b, var_bounds=var_bounds)


def load_qp_file(path: str) -> QpProblem:
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except OSError as exc:
        raise QpFileError(f"cannot read '{path}': {exc}") from exc
    except json.JSONDecodeError as exc:
        raise QpFileError(f"'{path}' is not valid JSON: {exc}") from exc
    return parse_qp_document(doc)


def _bounds_json(bounds: Bounds):
    return ([None if not np.isfinite(v) else float(v) for v in bounds.lower],
            [None if not np.isfinite(v) else float(v) for v in bounds.upper])


def _coo_json(m: SparseMatrix):
    rows = np.repeat(np.arange(m.n_rows), np.diff(m.row_offsets))
    return {"rows": rows.tolist(), "cols": np.asarray(m.col_indices).tolist(), "vals": np.asarray(m.values).tolist()}


def qp_document(problem) -> dict:
    """Serialise a problem to the file dialect (round-trip safe)."""
    h = problem.hessian
    kind = type(h).__name__
    if kind == "DiagonalHessian":
        hdoc = {"kind": "diagonal", "d": np.asarray(h.d).tolist()}
    elif kind == "SparseHessian":
        hdoc = {"kind": "coo", **_coo_json(h.m)}
    elif kind == "QuasiNewtonHessian":
        hdoc = {"kind": "bfgs", "h0_diag": np.asarray(h.h0_diag).tolist(),
                "u": [row.tolist() for row in np.asarray(h.u)], "w": np.asarray(h.w).tolist()}
    else:
        raise QpFileError("dense Hessians have no file representation")
    l, u = _bounds_json(problem.lin_bounds)
    lx, ux = _bounds_json(problem.var_bounds)
    return {"n": int(problem.n), "hessian": hdoc, "p": np.asarray(problem.p).tolist(),
            "A": _coo_json(problem.a), "l": l, "u": u, "C": _coo_json(problem.c),
            "b": np.asarray(problem.b).tolist(), "lx": lx, "ux": ux}


def solve_file(path: str, cfg=None, device: int = 0):
    """load_qp_file + the device-resident IPM (ipm.solve)."""
    from .ipm import solve
    return solve(load_qp_file(path), cfg, device=device)
