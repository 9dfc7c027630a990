"""Multi-GPU path on CPU: world_size 2, gloo.

The device kernels cannot run here, so each rank executes the SAME sharded
algorithm the library runs per slot (qpk_engine.cuh: every rank owns a slice
of the replicated top block and of the Hessian rows, rank-local B rows, one all-reduce of
[y_top partial | scalars] and one of [r'r, r'z]) with numpy on its shard, the
collectives going through torch.distributed/gloo.  The result must equal the
oracle's single-process operator apply and PCG (bit-for-bit is not expected:
the all-reduce reorders sums).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import qp_oracle as orc
from paper_2308_00637_b200 import sharded, workloads
from paper_2308_00637_b200.problem import build_operator


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _allreduce(x):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


class ShardEmulation:
    """numpy restatement of one rank of the sharded slot engine."""

    def __init__(self, op, rank, world):
        p = op.problem
        self.n = p.n
        segs = sharded.b_row_segments(p, op.bmap)
        self.lo, self.hi = sharded.partition_rows(sharded.b_row_nnz(segs), world)[rank]
        c, a_l, a_u = orc.b_blocks(op)
        import scipy.sparse as sp
        b = sp.vstack([c, a_l, -a_u]).tocsr() if op.m else sp.csr_matrix((0, p.n))
        self.b_loc = b[self.lo:self.hi]
        self.d_loc = op.d_diag[self.lo:self.hi]
        self.q = op.q_diag_extra
        self.h = p.hessian
        # the replicated top block is split into owned slices: rank r alone adds
        # diag(Q) u and the dot-product terms of [t_lo, t_hi), and applies a
        # contiguous, nnz-balanced slice of the sparse Hessian's non-empty rows
        # (the library slices them in RCM order; any fixed sequence partitions H)
        self.t_lo, self.t_hi = p.n * rank // world, p.n * (rank + 1) // world
        self.hrows = None
        if type(self.h).__name__ == "SparseHessian":
            hm = orc._csr(self.h.m)
            lens = np.diff(hm.indptr)
            seq = np.nonzero(lens)[0]
            pre = np.concatenate([[0], np.cumsum(lens[seq])])
            cut = lambda r: int(np.searchsorted(pre, pre[-1] * r // world, side="left"))  # noqa: E731
            lo = 0 if rank == 0 else cut(rank)
            hi = len(seq) if rank == world - 1 else cut(rank + 1)
            self.hrows = seq[lo:max(lo, hi)]
            self.hm = hm
        self.h_owner = rank == 0                      # dense / low-rank H: one owner

    def apply(self, v_loc):
        """K v restricted to this rank: y_top (global after the all-reduce), local y_bottom."""
        u, w = v_loc[:self.n], v_loc[self.n:]
        t = self.b_loc @ u
        z = 2.0 * t / self.d_loc + w
        top = self.b_loc.T @ z
        sl = slice(self.t_lo, self.t_hi)
        top[sl] += self.q[sl] * u[sl]
        kind = type(self.h).__name__
        if kind == "DiagonalHessian":
            top[sl] += self.h.d[sl] * u[sl]
        elif kind == "SparseHessian":
            top[self.hrows] += self.hm[self.hrows] @ u
        elif self.h_owner:
            top = top + orc.hessian_apply(self.h, u)
        top = _allreduce(top)
        return np.concatenate([top, t + self.d_loc * w])

    def dot(self, a, b):
        """Global dot of two local vectors: the replicated top counted once."""
        own = float(a[self.t_lo:self.t_hi] @ b[self.t_lo:self.t_hi])
        return float(_allreduce(np.array([own + float(a[self.n:] @ b[self.n:])]))[0])

    def jacobi(self):
        acc = _allreduce(np.asarray(self.b_loc.multiply(self.b_loc).T @ (1.0 / self.d_loc)).ravel())
        top = orc.hessian_diagonal(self.h) + self.q + 2.0 * acc
        return np.concatenate([top, self.d_loc])


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = {}
        for name, (fn, kw) in {
            "cfg5": (workloads.random_sweep, dict(seed=5, m=3000, n=800)),
            "cfg3": (workloads.rt_like, dict(seed=3, n_vox=2000, n_beam=300, density=0.03)),
            "cfg2": (workloads.svm_primal, dict(seed=2, d=20, n_samples=300)),
        }.items():
            problem, state, meta = fn(**kw)
            op = build_operator(problem, state)
            em = ShardEmulation(op, rank, world)
            rng = np.random.default_rng(11)
            v = rng.standard_normal(op.dim)
            sl = np.concatenate([v[:op.n], v[op.n + em.lo:op.n + em.hi]])
            y_loc = em.apply(sl)
            parts = [None] * world
            dist.all_gather_object(parts, y_loc[op.n:])
            y = np.concatenate([y_loc[:op.n]] + parts)
            jac_loc = em.jacobi()
            dist.all_gather_object(parts, jac_loc[op.n:])
            jac = np.concatenate([jac_loc[:op.n]] + parts)
            # sharded PCG (fixed 25 iterations, the reference recurrence)
            rhs = rng.standard_normal(op.dim)
            rl = np.concatenate([rhs[:op.n], rhs[op.n + em.lo:op.n + em.hi]])
            minv = 1.0 / jac_loc
            x = np.zeros_like(rl)
            r = rl.copy()
            z = minv * r
            p = z.copy()
            rz = em.dot(r, z)
            hist = [np.sqrt(em.dot(r, r))]
            for _ in range(25):
                yv = em.apply(p)
                alpha = rz / em.dot(p, yv)
                x += alpha * p
                r -= alpha * yv
                hist.append(np.sqrt(em.dot(r, r)))
                z = minv * r
                rzn = em.dot(r, z)
                p = z + (rzn / rz) * p
                rz = rzn
            dist.all_gather_object(parts, x[op.n:])
            xg = np.concatenate([x[:op.n]] + parts)
            results[name] = (y, jac, np.array(hist), xg, em.lo, em.hi)
        if rank == 0:
            out.put(results)
    finally:
        dist.destroy_process_group()


def test_partition_rows_is_balanced_and_contiguous():
    nnz = np.random.default_rng(0).integers(0, 40, size=1001)
    for world in (1, 2, 3, 8):
        parts = sharded.partition_rows(nnz, world)
        assert parts[0][0] == 0 and parts[-1][1] == len(nnz)
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        work = [int((nnz[lo:hi] + 1).sum()) for lo, hi in parts]
        assert max(work) - min(work) <= 2 * (nnz.max() + 1)


@pytest.mark.timeout(300)
def test_two_rank_sharded_algorithm_matches_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name, (fn, kw) in {
        "cfg5": (workloads.random_sweep, dict(seed=5, m=3000, n=800)),
        "cfg3": (workloads.rt_like, dict(seed=3, n_vox=2000, n_beam=300, density=0.03)),
        "cfg2": (workloads.svm_primal, dict(seed=2, d=20, n_samples=300)),
    }.items():
        problem, state, meta = fn(**kw)
        op = build_operator(problem, state)
        y, jac, hist, x, lo, hi = results[name]
        rng = np.random.default_rng(11)
        v = rng.standard_normal(op.dim)
        y_ref = orc.apply_doubly_augmented(op, v)
        assert np.linalg.norm(y - y_ref) <= 1e-12 * np.linalg.norm(y_ref), name
        jac_ref = orc.jacobi_diagonal(op)
        assert np.max(np.abs(jac - jac_ref) / jac_ref) <= 1e-12, name
        rhs = rng.standard_normal(op.dim)
        ref_hist = []
        ref = orc.pcg_direction(op, rhs, orc.PcgConfig(tol=1e-300, max_iters=25),
                                callback=lambda k, xk, rn: ref_hist.append(rn))
        h_ref = np.array([np.linalg.norm(rhs)] + ref_hist)
        # early iterations agree to reorder precision
        assert np.max(np.abs(hist[:8] - h_ref[:8]) / h_ref[:8]) <= 1e-8, name
