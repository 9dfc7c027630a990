"""Parity criteria shared by the GPU tests (enforceable contract).

* operator apply / Jacobi: ||y_gpu - y_ref|| / ||y_ref|| <= 1e-12 (and Jacobi
  element-wise relative 1e-12, test_kkt.py:190-199).
* PCG residual histories: relative difference <= max(1e-8, 10 x env_k) at
  every iteration k, where env_k is the running maximum of the CPU-reorder
  envelope: the reference itself re-run with mathematically identical but
  reordered sums (operator and dot products, 4 orderings).  Before K_env (the
  first iteration where env leaves 1e-8) this is the north star's literal
  1e-8; beyond it the histories are chaotic for ANY reordering and the GPU
  must stay within 10x what reordering the CPU does.  Compared only while
  rnorm_k / rnorm_0 > 1e-13.
"""

import numpy as np
import scipy.sparse as sp

from oracle import qp_oracle as orc

APPLY_TOL = 1e-12
HIST_TOL = 1e-8


def rel_err(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def reordered_apply(op, seed=0):
    """Same operator, different summation order: column-permuted B for B u,
    row-permuted B for B' z (SURVEY.md Appendix A probe)."""
    c, a_l, a_u = orc.b_blocks(op)
    b = sp.vstack([c, a_l, -a_u]).tocsr() if op.m else sp.csr_matrix((0, op.n))
    rng = np.random.default_rng(seed)
    cperm = rng.permutation(op.n)
    rperm = rng.permutation(op.m)
    b_c = b[:, cperm].tocsr()
    bt_r = b[rperm, :].T.tocsr()
    h = op.problem.hessian

    def apply(v):
        u, w = v[:op.n], v[op.n:]
        t = b_c @ u[cperm]
        z = 2.0 * t / op.d_diag + w
        hu = orc.hessian_apply(h, u)
        top = (hu + op.q_diag_extra * u) + bt_r @ z[rperm]
        return np.concatenate([top, t + op.d_diag * w])

    return apply


def reordered_pcg(apply_op, apply_prec, rhs, cfg, perm, callback):
    """linalg.py:66-133 with every dot product / norm summed in permuted order
    (a legitimate reordering, like the apply's)."""
    def dot(a, b):
        return float(a[perm] @ b[perm])

    x = np.zeros_like(rhs)
    r = rhs.copy()
    rnorm = np.sqrt(dot(r, r))
    threshold = cfg.tol * (np.sqrt(dot(rhs, rhs)) if cfg.tol_is_relative else 1.0)
    if rnorm <= threshold:
        return
    z = apply_prec(r)
    p = z.copy()
    rz = dot(r, z)
    for k in range(1, cfg.max_iters + 1):
        y = apply_op(p)
        pap = dot(p, y)
        if pap <= 0:
            return
        alpha = rz / pap
        x += alpha * p
        r -= alpha * y
        rnorm = np.sqrt(dot(r, r))
        callback(k, x, rnorm)
        if rnorm <= threshold:
            true_r = rhs - apply_op(x)
            if np.sqrt(dot(true_r, true_r)) <= threshold:
                return
            r = true_r
            z = apply_prec(r)
            p = z.copy()
            rz = dot(r, z)
            continue
        z = apply_prec(r)
        rz_next = dot(r, z)
        beta = rz_next / rz
        rz = rz_next
        p = z + beta * p


def envelope(op, rhs, cfg, ref_hist, seeds=(0, 1, 2, 3)):
    """Per-iteration max over several reorderings (operator sums and PCG dot
    products) of |h_reordered - h_ref| / h_ref."""
    inv = 1.0 / orc.jacobi_diagonal(op)
    env = None
    for seed in seeds:
        hist = [np.linalg.norm(rhs)]
        perm = np.random.default_rng(1000 + seed).permutation(len(rhs))
        reordered_pcg(reordered_apply(op, seed), lambda v: inv * v, rhs, cfg, perm,
                      lambda k, x, rn: hist.append(rn))
        k = min(len(hist), len(ref_hist))
        e = np.abs(np.array(hist[:k]) - ref_hist[:k]) / ref_hist[:k]
        if env is None:
            env = e
        else:
            j = min(len(env), len(e))
            env = np.maximum(env[:j], e[:j])
    return env


def check_history(gpu_hist, ref_hist, env):
    """Returns (ok, message)."""
    k = min(len(gpu_hist), len(ref_hist), len(env))
    ref = np.asarray(ref_hist[:k])
    env = np.asarray(env[:k])
    live = ref / ref[0] > 1e-13
    dev = np.abs(np.asarray(gpu_hist[:k]) - ref) / ref
    over = np.nonzero(env > HIST_TOL)[0]
    k_env = int(over[0]) if len(over) else k
    run_env = np.maximum.accumulate(env)
    bound = np.maximum(10.0 * run_env, HIST_TOL)
    bad = np.nonzero(live & (dev > bound))[0]
    if len(bad):
        j = int(bad[0])
        return False, f"iteration {j}: dev {dev[j]:.3e} > bound {bound[j]:.3e} (K_env={k_env})"
    return True, f"K_env={k_env}, max dev before K_env {dev[:k_env][live[:k_env]].max(initial=0):.2e}"
