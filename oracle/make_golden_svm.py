"""Generate tests/golden/svm.npz by running the REAL reference SVM frontend here.

TEST INFRASTRUCTURE ONLY.  Run in the build container (reference mounted
read-only at /root/reference):

    python oracle/make_golden_svm.py

For a few seeded datasets (written as LIBSVM text with round-trip float
formatting, then parsed by the reference's own ``parse_libsvm``) it records the
reference's ``build_svm_dual`` Hessian, its IPM solution (``solve`` with the
default IpmConfig), the model (``extract_model``: bias, support vectors), the
training accuracy and ``predict`` scores of probe samples.  The GPU frontend
(paper_2308_00637_b200/svm.py) is checked against these on the GPU box
(tests/test_gpu_svm.py) and the CPU restatement (oracle/svm_oracle.py) here
(tests/test_oracle_golden.py).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import qpipm.ipm as ref_ipm  # noqa: E402
import qpipm.svm as ref_svm  # noqa: E402

from oracle.svm_oracle import synthetic_dataset  # noqa: E402

OUT = ROOT / "tests" / "golden"


def libsvm_text(x, y):
    lines = []
    for row, lab in zip(x, y):
        feats = " ".join(f"{j + 1}:{float(v)!r}" for j, v in enumerate(row) if v != 0.0)
        lines.append(f"{'+1' if lab > 0 else '-1'} {feats}".rstrip())
    return "\n".join(lines) + "\n"


def datasets():
    out = [("two_point", np.array([[1.0, 0.0], [0.0, 1.0]]), np.array([1.0, -1.0]), 1.0, 10.0)]
    x, y = synthetic_dataset(11, 40, 5, sep=4.0)
    out.append(("syn40", x, y, 1.0, 1.0))
    x, y = synthetic_dataset(12, 120, 20, sep=6.0)
    out.append(("syn120", x, y, 20.0, 0.5))
    x, y = synthetic_dataset(15, 400, 30, sep=3.0)
    out.append(("syn400", x, y, 10.0, 1.0))
    x, y = synthetic_dataset(13, 64, 12, sep=5.0)
    x[np.random.default_rng(14).random(x.shape) < 0.5] = 0.0        # LIBSVM-sparse samples
    out.append(("sparse64", x, y, 0.8, 2.0))
    return out


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rec = {}
    names = []
    for name, x, y, sigma, c in datasets():
        t0 = time.perf_counter()
        text = libsvm_text(x, y)
        data = ref_svm.parse_libsvm(text)
        cfg = ref_svm.SvmConfig(sigma=sigma, c=c)
        prob = ref_svm.build_svm_dual(data, cfg)
        rep = ref_ipm.solve(prob)
        model = ref_svm.extract_model(data, cfg, rep.x)
        probes = [ref_svm.SparseVector(np.arange(data.n_features), row) for row in
                  np.random.default_rng(99).standard_normal((3, data.n_features))]
        scores = [ref_svm.predict(model, pv) for pv in probes]
        p = name + "_"
        names.append(name)
        rec[p + "text"] = np.array(text)
        rec[p + "x"] = data.dense_matrix()
        rec[p + "y"] = data.labels
        rec[p + "sigma_c"] = np.array([sigma, c])
        rec[p + "H"] = prob.hessian.m
        rec[p + "alpha"] = rep.x
        rec[p + "status"] = np.array(rep.status.value)
        rec[p + "objective"] = np.float64(rep.objective)
        rec[p + "iterations"] = np.int64(rep.iterations)
        rec[p + "bias"] = np.float64(model.bias)
        rec[p + "support"] = np.asarray(model.support_indices, dtype=np.int64)
        rec[p + "decision"] = ref_svm._decision_values(data, cfg, rep.x)
        rec[p + "accuracy"] = np.float64(ref_svm.training_accuracy(model))
        rec[p + "probes"] = np.array([pv.values for pv in probes])
        rec[p + "probe_scores"] = np.array([s for s, _ in scores])
        rec[p + "probe_labels"] = np.array([lab for _, lab in scores], dtype=np.int64)
        print(name, rep.status.value, rep.iterations, f"obj {rep.objective:.12e}", f"bias {model.bias:.6f}",
              f"acc {rec[p + 'accuracy']:.3f}", f"{time.perf_counter() - t0:.1f}s")
    rec["names"] = np.array(names)
    np.savez_compressed(OUT / "svm.npz", **rec)


if __name__ == "__main__":
    main()
