"""Row-sharded multi-GPU Jacobi-PCG (one process per GPU).

B = (C; A_l; -A_u) is split into contiguous, nnz-balanced row blocks, one per
rank; every bottom vector (w, D, r, p, x, ...) is split the
same way and the top block (n) is replicated, every rank owning a slice of
its terms.  Inside the library each PCG iteration all-reduces
[y_top partial | slot scalars] over NCCL on the solver's own stream
(`qpk_shard_init`) -- in the tile format that one all-reduce also carries
[r'r, r'z]; torch.distributed is only the plumbing that broadcasts the NCCL id
and gathers the solution.

`ShardedKkt` mirrors `direction.GpuKkt` with global-sized inputs and outputs,
so `sharded_direction(op, rhs, cfg)` is a drop-in `DirectionSolver` for an
SPMD caller (every rank calls it with the same op and rhs).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .direction import _csr_arrays, _dim
from .pcg import result_types


def b_row_segments(problem, bmap):
    """The reference's B row order (kkt.py:177, 206-207) as segments
    (matrix, selected rows or None, sign)."""
    segs = []
    if problem.c.n_rows:
        segs.append((problem.c, None, 1.0))
    lin_lower = np.asarray(bmap.lin_lower, dtype=np.int64)
    lin_upper = np.asarray(bmap.lin_upper, dtype=np.int64)
    if len(lin_lower):
        segs.append((problem.a, lin_lower, 1.0))
    if len(lin_upper):
        segs.append((problem.a, lin_upper, -1.0))
    return segs


def b_row_nnz(segs):
    parts = []
    for mat, rows, _ in segs:
        lens = np.diff(np.asarray(mat.row_offsets, dtype=np.int64))
        parts.append(lens if rows is None else lens[rows])
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def partition_rows(row_nnz, world: int):
    """Contiguous row ranges [(lo, hi)] with balanced work (nnz + 1 per row)."""
    m = len(row_nnz)
    if world == 1:
        return [(0, m)]
    work = np.concatenate([[0], np.cumsum(np.asarray(row_nnz, dtype=np.int64) + 1)])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(work, work[-1] * r / world, side="left")))
    cuts.append(m)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, m))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(world)]


def _dist():
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("sharded solver needs an initialised torch.distributed process group")
    return dist


class ShardedKkt:
    """This rank's shard of the device-resident doubly augmented operator."""

    def __init__(self, problem, bmap, device: int = 0, scatter: int = _native.QPK_SCATTER_AUTO, group=None):
        dist = _dist()
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n = int(problem.n)
        segs = b_row_segments(problem, bmap)
        self.m = int(sum(len(r) if r is not None else m.n_rows for m, r, _ in segs))
        self.dim = self.n + self.m
        self.bounds = partition_rows(b_row_nnz(segs), self.world)
        self.lo, self.hi = self.bounds[self.rank]
        self.ctx = _native.Context(device)
        lib = _native.load_library()
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            _native.check("qpk_nccl_get_unique_id", lib.qpk_nccl_get_unique_id(ctypes.addressof(uid)))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (ctypes.c_ubyte * 128).from_buffer_copy(box[0])
        self.ctx.call("qpk_shard_init", self.world, self.rank, ctypes.addressof(uid))
        m_loc = self.hi - self.lo
        self.ctx.call("qpk_problem_begin", self.n, 0, m_loc, 0)
        # rows [lo, hi) of the global B, segment by segment
        base = 0
        for mat, rows, sign in segs:
            count = mat.n_rows if rows is None else len(rows)
            a, b = max(self.lo, base), min(self.hi, base + count)
            if a < b:
                sel = (np.arange(a - base, b - base, dtype=np.int64) if rows is None
                       else np.ascontiguousarray(rows[a - base:b - base]))
                ro, ci, v = _csr_arrays(mat)
                self.ctx.call("qpk_problem_add_rows", int(mat.n_rows), _native.ptr(ro), _native.ptr(ci),
                              _native.ptr(v), _native.ptr(sel), len(sel), float(sign))
            base += count
        from .direction import GpuKkt
        GpuKkt._set_hessian(self, problem.hessian)
        self.ctx.call("qpk_problem_finalize", int(scatter))

    # -- per IPM iteration (global-sized arguments) --------------------------
    def set_diagonals(self, d_diag, q_extra):
        d = np.ascontiguousarray(d_diag, dtype=np.float64)
        q = np.ascontiguousarray(q_extra, dtype=np.float64)
        _dim(len(d), self.m, "d_diag")
        _dim(len(q), self.n, "q_diag_extra")
        d_loc = np.ascontiguousarray(d[self.lo:self.hi])
        self.ctx.call("qpk_set_diagonals", _native.ptr(d_loc), _native.ptr(q))

    def local(self, v):
        v = np.asarray(v, dtype=np.float64)
        _dim(len(v), self.dim, "vector")
        return np.ascontiguousarray(np.concatenate([v[:self.n], v[self.n + self.lo:self.n + self.hi]]))

    def gather(self, v_loc):
        """Global vector from the ranks' (replicated top, local bottom) pieces:
        one all_gather of equal-sized (padded) tensors on the group's backend
        (device tensors under NCCL, host tensors under gloo)."""
        import torch
        dist = _dist()
        sizes = [hi - lo for lo, hi in self.bounds]
        width = max(max(sizes), 1)
        on_gpu = dist.get_backend(self.group) == "nccl"
        piece = torch.zeros(width, dtype=torch.float64)
        piece[:sizes[self.rank]] = torch.from_numpy(np.ascontiguousarray(v_loc[self.n:]))
        if on_gpu:
            piece = piece.to(f"cuda:{self.ctx.device}")
        out = torch.empty(self.world * width, dtype=torch.float64, device=piece.device)
        dist.all_gather_into_tensor(out, piece, group=self.group)
        out = out.cpu().numpy().reshape(self.world, width)
        return np.concatenate([v_loc[:self.n]] + [out[r, :sizes[r]] for r in range(self.world)])

    def jacobi(self):
        out = np.empty(self.n + self.hi - self.lo)
        self.ctx.call("qpk_jacobi", _native.ptr(out))
        return self.gather(out)

    def apply(self, v):
        v_loc = self.local(v)
        y = np.empty(len(v_loc))
        self.ctx.call("qpk_apply", _native.ptr(v_loc), _native.ptr(y))
        return self.gather(y)

    def pcg(self, rhs, tol: float, max_iters: int, tol_is_relative: bool = True, history: bool = False):
        rhs_loc = self.local(rhs)
        x = np.empty(len(rhs_loc))
        info = _native.PcgInfo()
        hist = np.full(int(max_iters) + 1, np.nan) if history else None
        self.ctx.call("qpk_pcg", _native.ptr(rhs_loc), float(tol), int(bool(tol_is_relative)), int(max_iters),
                      _native.ptr(x), ctypes.byref(info), _native.ptr(hist) if history else None)
        if history:
            hist = hist[: info.iterations + 1]
        return self.gather(x), info, hist

    def close(self):
        self.ctx.close()


_CACHE: dict = {}


def sharded_direction(op, rhs, cfg, device: int | None = None, group=None):
    """DirectionSolver for an SPMD caller (all ranks, same op and rhs).  The
    device operator is cached per (problem, bound map), as direction.operator_for
    does; a replaced entry is closed at once -- on every rank at the same call,
    so the NCCL communicators are destroyed in the same order everywhere."""
    from .direction import _bmap_key
    PcgResult, PcgBreakdownError = result_types()
    key = id(op.problem)
    entry = _CACHE.get(key)
    fresh = entry is None or entry[0] is not op.problem
    if not fresh:
        same = entry[3][0] is op.bmap.lin_lower and entry[3][1] is op.bmap.lin_upper
        fresh = not (same or entry[2] == _bmap_key(op.bmap))
    if fresh:
        if device is None:
            import torch
            device = torch.cuda.current_device()
        for old in list(_CACHE.values()):
            old[1].close()
        _CACHE.clear()
        entry = (op.problem, ShardedKkt(op.problem, op.bmap, device=device, group=group), _bmap_key(op.bmap),
                 (op.bmap.lin_lower, op.bmap.lin_upper))
        _CACHE[key] = entry
    sk = entry[1]
    sk.set_diagonals(op.d_diag, op.q_diag_extra)
    x, info, _ = sk.pcg(rhs, cfg.tol, cfg.max_iters, cfg.tol_is_relative)
    result = PcgResult(x, int(info.iterations), float(info.final_residual_norm), bool(info.converged))
    if info.status == _native.QPK_PCG_BREAKDOWN:
        raise PcgBreakdownError(result)
    return result
