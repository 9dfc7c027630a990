"""Benchmark: Jacobi-PCG iterations/s on the doubly augmented KKT system.

Default workload (BASELINE.json configs[3], "cfg4"): the scaled
radiation-therapy-like QP -- 2,000,000 voxels x 100,000 beamlets, 0.1 % band
density (B = -D_oar: 1.6e8 nnz, fp64), H = D_t'D_t (4.1e6 nnz) -- the largest
configuration of BASELINE.json, the one it names for row sharding over
1/2/4/8 GPUs and the one the north star's targets (>= 70 % of HBM bandwidth on
1 GPU, >= 60 % efficiency at 8 GPUs on the largest sharded config) are stated
on.  The operator is that of the first IPM iteration; the Jacobi diagonal is
built once before the timed loop in BOTH arms (its time is reported as
`jacobi_ms`); one step = one PCG solve (linalg.py:66-133): 200 iterations
(reference arm: 20, a bounded sample) from a seeded N(0,1) right-hand side
(x0 = 0) + the final true-residual apply (linalg.py:132-133).  `--workload cfg1|cfg2|cfg3|cfg5`
runs the other BASELINE configs the same way (cfg5 = the isolated operator
sweep, 500 iterations); `--ipm` reports IPM wall time.  See DESIGN.md §5.

  value  PCG iterations/s, whole job, inputs resident in HBM
         (qpk_pcg_dev on device buffers), CUDA events on the solver's stream
  e2e    the same metric through the reference-facing drop-in
         gpu_direction(op, rhs, cfg) with the pageable numpy arrays the
         reference IPM passes: diagonals + rhs H2D, Jacobi build, PCG,
         solution D2H inside the timed region
  parity the GPU's first iterations against the reference's on the same
         operator and rhs (the cpu_baseline sample), printed in the line

`--gpus N` without a torchrun environment re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Jacobi-PCG iterations/s on the doubly augmented KKT system"
CONFIG_INDEX = {"cfg1": 0, "cfg2": 1, "cfg3": 2, "cfg4": 3, "cfg5": 4, "svm_dual": 1}
UNIT = "PCG iterations/s"
L2_GATHER_PER_S = 287e9      # random 8 B gathers from an L2-resident table (measured)
L2_ATOMIC_PER_S = 190e9      # random fp64 atomics into an L2-resident table (measured)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--iters", type=int, default=500, help="PCG iterations per step (BASELINE cfg5: 500)")
    ap.add_argument("--scale", type=float, default=1.0, help="shrink cfg5 (testing only; 1.0 = BASELINE)")
    ap.add_argument("--scatter", type=int, default=0,
                    help="0 = auto per matrix, 1 = atomic B'z, 2 = CSC gather, 3 = row-block dictionary")
    ap.add_argument("--cpu-iters", type=int, default=10, help="oracle iterations in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-iters-per-step", type=int, default=20,
                    help="PCG iterations per step of the reference arm (a bounded sample of the workload)")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "svm_dual"],
                    help="cfg4 = headline (largest, sharded config); cfg1-4: PCG sweep on the first IPM iteration's "
                         "operator; cfg5: the isolated operator sweep")
    ap.add_argument("--force-sharded", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--ipm", action="store_true",
                    help="IPM wall time of the device-resident IPM on --workload (cfg1 pinned at mu_tol 1e-8, "
                         "CG tol 1e-10; others at the reference defaults)")
    ap.add_argument("--cpu-ipm-iters", type=int, default=0,
                    help="IPM iterations in the CPU-baseline sample (0 = full solve for cfg1, 2 otherwise)")
    args = ap.parse_args()
    if args.workload != "cfg5" and args.iters == 500:
        args.iters = 200
    return args


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


WORKLOAD_DESC = {
    "cfg1": "cfg1 dense QP n=200, m=400 (DenseHessian Q'Q+1e-2 I)",
    "cfg2": "cfg2 SVM primal d=500, N=50,000 (A = [diag(y)X, y, I], 502 nnz/row)",
    "cfg3": "cfg3 RT-like 200,000 voxels x 20,000 beamlets, 0.5% band density, SparseHessian D_t'D_t",
    "cfg4": "cfg4 RT-like 2,000,000 voxels x 100,000 beamlets, 0.1% band density, SparseHessian D_t'D_t",
    "svm_dual": "kernel-SVM dual (svm.py:179-195) at the dense-kernel cap: n=20,000 samples, d=100, RBF sigma=10, "
                "C=1; H = (y y') * K built on the device (3.2 GB dense), one equality row",
    "cfg5": "cfg5 operator sweep 4,000,000 x 1,000,000, 16 nnz/row, H=diag(U(1e-2,1)), log10 w ~ U(-6,6)",
}


def make_workload(name: str, scale: float, seed_offset: int = 0):
    """(problem, op, rhs, meta).  cfg5: the BASELINE sweep with its seeded rhs;
    cfg1-4: the operator of the first IPM iteration with a seeded N(0,1) rhs."""
    from paper_2308_00637_b200 import workloads
    from paper_2308_00637_b200.problem import build_operator
    if name == "svm_dual":
        from paper_2308_00637_b200 import svm
        from paper_2308_00637_b200.workloads import _state_from_initial
        x, y = workloads.svm_dual_data(seed=6 + seed_offset, n=int(20_000 * scale), d=100)
        data = svm.SvmDataset.from_dense(x, y)
        problem = svm.build_svm_dual(data, svm.SvmConfig(sigma=10.0, c=1.0))
        state = _state_from_initial(problem)
        meta = {"seed": 6 + seed_offset, "n": len(y), "d": 100, "x": x, "y": y, "sigma": 10.0, "c": 1.0}
        rhs = np.random.default_rng(77 + seed_offset).standard_normal(problem.n + 1)
    elif name == "cfg5":
        m, n = int(4_000_000 * scale), int(1_000_000 * scale)
        problem, state, meta = workloads.random_sweep(seed=5 + seed_offset, m=m, n=n)
        rhs = meta.pop("rhs")
    else:
        if name == "cfg1":
            problem, state, meta = workloads.dense_qp(seed=0 + seed_offset)
        elif name == "cfg2":
            problem, state, meta = workloads.svm_primal(seed=2 + seed_offset, n_samples=int(50_000 * scale))
        elif name == "cfg3":
            problem, state, meta = workloads.rt_like(seed=3 + seed_offset, n_vox=int(200_000 * scale),
                                                     n_beam=int(20_000 * scale))
        else:
            problem, state, meta = workloads.rt_like(seed=4 + seed_offset, n_vox=int(2_000_000 * scale),
                                                     n_beam=int(100_000 * scale), density=0.001)
        rhs = np.random.default_rng(77 + seed_offset).standard_normal(problem.n + len(state.s_lA) + len(state.s_uA)
                                                                      + problem.m_eq)
    op = build_operator(problem, state)
    assert len(rhs) == op.dim
    meta["state"] = state
    if name == "svm_dual":
        _SVM_META.update(meta)
    return problem, op, rhs, meta


def config_of(args, meta):
    """The `config` object -- identical in both arms (same workload, same seed)."""
    return {"workload": WORKLOAD_DESC[args.workload] + (f" (scale {args.scale})" if args.scale != 1 else ""),
            "seed": meta["seed"],
            "l2": "inputs larger than L2 (every PCG iteration streams the whole operator)"
                  if args.workload in ("cfg2", "cfg3", "cfg4", "cfg5", "svm_dual") and args.scale == 1 else
                  "working set fits L2 (each step re-reads it every PCG iteration; no flush)"}


class ReferencePath:
    """The reference's CPU implementation of the path on one operator: the
    UNMODIFIED qpipm from oracle/_ref (kind "reference") when it was placed by
    build(), else the oracle port (kind "port", bit-identical on the goldens).
    Jacobi is built once (timed apart); `run(k)` is linalg.pcg for k iterations
    + the final true-residual apply, exactly what ipm._pcg_direction calls."""

    def __init__(self, problem, op, meta, workload):
        from oracle import build_ref
        self.kind = "port"
        if build_ref.available() and workload != "svm_dual":
            from oracle import refbridge
            qp = build_ref.import_qpipm()
            rop = refbridge.ref_operator(problem, meta["state"])
            assert np.array_equal(rop.d_diag, op.d_diag) and np.array_equal(rop.q_diag_extra, op.q_diag_extra)
            self.kind = "reference"
            self._pcg, self._cfg = qp.linalg.pcg, qp.linalg.PcgConfig
            self._apply = lambda v: qp.kkt.apply_doubly_augmented(rop, v)      # noqa: E731
            self._jacobi = lambda: qp.kkt.jacobi_diagonal(rop)                 # noqa: E731
        else:
            from oracle import qp_oracle as orc
            hop = host_operator(op)
            self._pcg, self._cfg = orc.pcg, orc.PcgConfig
            self._apply = lambda v: orc.apply_doubly_augmented(hop, v)         # noqa: E731
            self._jacobi = lambda: orc.jacobi_diagonal(hop)                    # noqa: E731
        self._apply(np.zeros(op.dim))                 # warm the scipy views (not timed)
        t0 = time.perf_counter()
        self.jacobi = self._jacobi()
        self.jacobi_s = time.perf_counter() - t0
        self.inv = 1.0 / self.jacobi
        self.cores = 1                                # numpy/scipy sparse matvecs are single-threaded

    def apply(self, v):
        return self._apply(v)

    def run(self, rhs, iters, history=None):
        cb = (lambda k, x, rn: history.append(rn)) if history is not None else None
        return self._pcg(self._apply, lambda r: self.inv * r, rhs, self._cfg(tol=1e-300, max_iters=iters),
                         callback=cb)

    def describe(self):
        return ("unmodified qpipm (oracle/_ref): linalg.pcg over kkt.apply_doubly_augmented" if self.kind == "reference"
                else "oracle port (numpy/scipy restatement of qpipm, bit-identical on the golden vectors)")


def algorithmic_bytes(op, iters: int, applies: int):
    """bytes_B = 12 nnz_B + 4 (m_B + 1) (two-sided rows once);
    bytes_Hm = 0 (diagonal), 12 nnz_H + 4 (n + 1) (sparse), 8 n^2 (dense),
    16 n k + 8 k (low rank); per PCG iteration bytes_B + bytes_Hm + 88 N; per
    extra apply bytes_B + bytes_Hm + 24 N.  Returns (per launch, per iteration)."""
    p = op.problem
    rows = set(np.asarray(op.bmap.lin_lower).tolist()) | set(np.asarray(op.bmap.lin_upper).tolist())
    lens = np.diff(p.a.row_offsets)
    nnz = int(lens[sorted(rows)].sum()) if rows else 0
    nnz += p.c.nnz
    N = op.dim
    bytes_b = 12 * nnz + 4 * (op.m + 1)
    h = p.hessian
    kind = type(h).__name__
    if kind == "SparseHessian":
        bytes_h = 12 * h.m.nnz + 4 * (p.n + 1)
    elif kind in ("DenseHessian", "DeviceDenseHessian"):
        bytes_h = 8 * p.n * p.n
    elif kind == "QuasiNewtonHessian":
        bytes_h = 16 * p.n * h.u.shape[1] + 8 * h.u.shape[1]
    else:
        bytes_h = 0
    per_iter = bytes_b + bytes_h + 88 * N
    return iters * per_iter + applies * (bytes_b + bytes_h + 24 * N), per_iter


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def host_operator(op, meta=None):
    """The oracle needs host data: the SVM dual's device Hessian is rebuilt on
    the host by the oracle's restatement of _gram_matrix (not timed)."""
    if type(op.problem.hessian).__name__ != "DeviceDenseHessian":
        return op
    from oracle import svm_oracle as so
    from paper_2308_00637_b200.problem import build_operator
    from paper_2308_00637_b200.workloads import _state_from_initial
    meta = meta or _SVM_META
    prob = so.dual_problem(meta["x"], meta["y"], meta["sigma"], meta["c"])
    return build_operator(prob, _state_from_initial(prob))


_SVM_META = {}


def cpu_baseline(ref, rhs, iters: int, name: str):
    """The reference path on a bounded sample: `iters` PCG iterations (+ the
    final apply) of the same operator and rhs.  Returns (record, history)."""
    hist = []
    t0 = time.perf_counter()
    res = ref.run(rhs, iters, history=hist)
    dt = time.perf_counter() - t0
    rec = {"value": iters / dt, "unit": UNIT, "cores": ref.cores, "kind": ref.kind,
           "jacobi_build_s": round(ref.jacobi_s, 3),
           "sample": f"{iters} PCG iterations of {name} + final apply, {dt:.1f} s (Jacobi built before, "
                     f"{ref.jacobi_s:.1f} s); {ref.describe()}; sparse matvecs single-threaded "
                     f"({len(os.sched_getaffinity(0))} host cores visible)"}
    return rec, np.array([np.linalg.norm(rhs)] + hist), np.asarray(res.solution)


def run_reference(args):
    """The reference arm: the reference's own CPU path on the box's host cores,
    same workload / metric / unit as our arm; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.workload == "svm_dual":               # Hessian on the host for the CPU arm (oracle restatement)
        from paper_2308_00637_b200.problem import build_operator
        from paper_2308_00637_b200.workloads import _state_from_initial, svm_dual_data
        from oracle import svm_oracle as so
        x, y = svm_dual_data(seed=6, n=int(20_000 * args.scale), d=100)
        problem = so.dual_problem(x, y, 10.0, 1.0)
        op = build_operator(problem, _state_from_initial(problem))
        rhs = np.random.default_rng(77).standard_normal(op.dim)
        meta = {"seed": 6}
    else:
        problem, op, rhs, meta = make_workload(args.workload, args.scale)
    ref = ReferencePath(problem, op, meta, args.workload)
    k_iter = args.ref_iters_per_step
    for _ in range(args.warmup):
        ref.run(rhs, k_iter)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = ref.run(rhs, k_iter)
    dt = time.perf_counter() - t0
    assert res.iterations == k_iter
    value = k_iter * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded generator of BASELINE.json configs[{CONFIG_INDEX[args.workload]}]; no dataset involved)",
        "config": config_of(args, meta),
        "step": {"pcg_iters_per_step": k_iter, "jacobi_ms": ref.jacobi_s * 1e3,
                 "what": "one linalg.pcg call: k iterations + the final true-residual apply; Jacobi built once before"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.cores, "kind": ref.kind,
                         "sample": f"{k_iter} PCG iterations per step of {args.workload}; {ref.describe()}; "
                                   f"{len(os.sched_getaffinity(0))} host cores visible, sparse matvecs single-threaded"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if world > 1 or args.force_sharded:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    from paper_2308_00637_b200 import _native
    from paper_2308_00637_b200.direction import GpuKkt, gpu_direction, operator_for
    from paper_2308_00637_b200.pcg import PcgConfig

    # N > 1: row-sharded; --force-sharded runs the same code path at N = 1
    # (one-rank NCCL communicator) to validate it on a single GPU
    sharded_run = world > 1 or args.force_sharded
    # N > 1: every rank builds the same system and owns a row shard of it
    # (strong scaling); N = 1: the whole system on one GPU
    problem, op, rhs, meta = make_workload(args.workload, args.scale, seed_offset=0)
    if sharded_run:
        from paper_2308_00637_b200.sharded import ShardedKkt
        gk = ShardedKkt(problem, op.bmap, device=local, scatter=args.scatter)
        rhs_loc = gk.local(rhs)
        d_loc = np.ascontiguousarray(op.d_diag[gk.lo:gk.hi])
    else:
        gk = GpuKkt(problem, op.bmap, device=local, scatter=args.scatter)
        rhs_loc, d_loc = rhs, np.ascontiguousarray(op.d_diag)
    stream = torch.cuda.current_stream()
    gk.ctx.call("qpk_set_stream", _native.ctypes.c_void_p(stream.cuda_stream))
    gk.set_diagonals(op.d_diag, op.q_diag_extra)
    gk.jacobi()
    N = op.dim
    rhs_d = torch.from_numpy(rhs_loc).to(f"cuda:{local}")
    d_d = torch.from_numpy(d_loc).to(f"cuda:{local}")
    q_d = torch.from_numpy(np.ascontiguousarray(op.q_diag_extra)).to(f"cuda:{local}")
    x_d = torch.empty(len(rhs_loc), dtype=torch.float64, device=f"cuda:{local}")
    info = _native.PcgInfo()

    # Jacobi diagonal: built once, before the timed loop, in both arms
    # (new diagonals mark it stale; qpk_jacobi rebuilds it); timed apart
    jac_ms = []
    for _ in range(3):
        gk.ctx.call("qpk_set_diagonals_dev", d_d.data_ptr(), q_d.data_ptr())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gk.jacobi()                                   # includes the D2H of the diagonal
        jac_ms.append((time.perf_counter() - t0) * 1e3)

    def step():
        # one PCG solve (linalg.py:66-133): fixed iterations + the final true-residual apply
        gk.ctx.call("qpk_pcg_dev", rhs_d.data_ptr(), 1e-300, 1, args.iters, x_d.data_ptr(),
                    _native.ctypes.byref(info), None)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        step()
    assert info.iterations == args.iters and info.applies == args.iters + 1, (info.iterations, info.applies)
    engine_used = gk.ctx.query("engine")
    barrier()
    launches0 = gk.ctx.query("kernel_launches")
    kernel_ms, phase_ms = [], []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            kernel_ms.append(info.kernel_ms)
            phase_ms.append(list(info.phase_ms))
        ev1.record(stream)
        barrier()
    launches = gk.ctx.query("kernel_launches") - launches0
    elapsed = ev0.elapsed_time(ev1) / 1e3
    if world > 1:
        t = torch.tensor([elapsed], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed = float(t.item())
    # one system solved jointly by all ranks when sharded (strong scaling)
    total_iters = args.iters * args.steps
    value = total_iters / elapsed

    # e2e through the reference-facing drop-in with the host buffers the
    # reference IPM passes: plain (pageable) numpy arrays for the diagonals
    # and the rhs (kkt.py:196-202, 242-262); the library stages them itself
    e2e_cfg = PcgConfig(tol=1e-300, max_iters=args.iters)
    if sharded_run:
        from paper_2308_00637_b200.sharded import sharded_direction
        direction = lambda o, b, c: sharded_direction(o, b, c, device=local)  # noqa: E731
    else:
        operator_for(op, device=local)               # one upload per problem (not timed)
        direction = gpu_direction
    direction(op, rhs, e2e_cfg)
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(e2e_steps):
        res = direction(op, rhs, e2e_cfg)
        _ = float(res.final_residual_norm)
    barrier()
    e2e_dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_dt], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_dt = float(t.item())
    e2e_value = args.iters * e2e_steps / e2e_dt
    h2d = 8 * (len(d_loc) + op.n + len(rhs_loc))     # per rank: its diagonals + rhs slice
    d2h = 8 * len(rhs_loc)

    # roofline: ALGORITHMIC bytes per launch (one launch = one solve) / its device time
    per_launch, per_iter = algorithmic_bytes(op, args.iters, applies=1)
    avg_ms = float(np.mean(kernel_ms))
    achieved = per_launch / world / (avg_ms * 1e-3) / 1e9     # per GPU
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic, traffic_src = None, None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            rec = json.loads(prof.read_text()).get(args.workload)
            if rec and args.scale == 1.0 and world == 1:
                # ncu DRAM bytes of the same solve (per-iteration figure x iterations + final apply),
                # captured once per build by probes/ncu_traffic.py -- not measured in this run
                traffic = float(rec["dram_bytes_per_iter"]) * (args.iters + 1)
                traffic_src = rec.get("source")
        except Exception:
            traffic = None
    # PHYSICAL bandwidth: the bytes the kernels really moved (ncu DRAM) / the same time
    physical = traffic / (avg_ms * 1e-3) / 1e9 if traffic else None
    # "if a compressed format moves fewer bytes, say so; never
    # quote achieved > physical".  The tile / panel / packed-symmetric formats
    # hold 8-9 B per nonzero against the formula's 12, so where the measured
    # traffic is below the algorithmic bytes, `achieved` is the physical rate
    # and the CSR-equivalent rate is reported beside it.
    csr_equiv = achieved
    basis = "algorithmic bytes (SURVEY.md 8(d) formula) / device time"
    if achieved > peak and physical is not None:
        # the formula rate is above what the memory system can move: the format
        # moves fewer bytes than the formula charges, so the physical rate is quoted
        achieved = physical
        basis = ("physical DRAM bytes / device time: the 8(d) formula rate (csr_equivalent_GBs) exceeds the measured "
                 "peak because the tile format moves fewer bytes than CSR")
    elif physical is not None and traffic < per_launch:
        basis += ("; the format moves fewer bytes than the formula charges -- physical_GBs / physical_frac give "
                  "the real DRAM rate")
    # the pass over B (dominant kernel of a PCG iteration): its time, and the
    # bytes of the format it streams (tile / panel formats hold fewer bytes than CSR)
    phases = np.mean(phase_ms, axis=0) * 1e3 / args.iters          # us per iteration
    rows_kernel = {3: "k_slot_rows_tile", 4: "k_slot_panel"}.get(gk.ctx.query("scatter"), "k_slot_rows") \
        if engine_used else "pcg_kernel (rows phase)"
    fmt_bytes = gk.ctx.query("format_bytes")
    if gk.ctx.query("hess_sym"):
        # dense symmetric H as packed upper tiles: the operator pass is its stream (+ the partials)
        rows_kernel = "k_slot_hess_sym + k_slot_sym_combine (packed symmetric H) + k_slot_rows / k_slot_dense"
        nt = (op.n + 63) // 64
        fmt_bytes += nt * (nt + 1) // 2 * 4096 * 8
    dom = {"name": rows_kernel, "us_per_iter": round(float(phases[1]), 2),
           "share_of_iteration": round(float(phases[1] / max(phases.sum(), 1e-9)), 3),
           "csr_matrix_bytes_per_iter": per_iter - 88 * op.dim,
           "format_bytes_per_pass": fmt_bytes,
           "format_GBs": round(fmt_bytes / (phases[1] * 1e-6) / 1e9, 1) if phases[1] > 0 and fmt_bytes > 0 else None}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded generator of BASELINE.json configs[{CONFIG_INDEX[args.workload]}]; no dataset involved)",
            "config": config_of(args, meta),
            "step": {"pcg_iters_per_step": args.iters, "jacobi_ms": round(float(np.median(jac_ms)), 3),
                     "what": "one PCG solve: k iterations + the final true-residual apply; Jacobi built once before "
                             "(jacobi_ms = build + D2H of the diagonal)"},
            "engine": {"parallelism": f"rowshard{world} (NCCL all-reduce per iteration)" if world > 1 else "single",
                       "scatter": {1: "atomic", 2: "csc", 3: "dict", 4: "panel"}.get(gk.ctx.query("scatter"), "?"),
                       "n": op.n, "m_B": op.m, "nnz_B": gk.ctx.query("nnz"),
                       "grid": gk.ctx.query("grid"), "lanes_per_row": gk.ctx.query("lanes"),
                       "hess_tiled": gk.ctx.query("hess_tiled"), "tile_cta_acc": gk.ctx.query("tile_cta_acc"),
                       "panel_cols": gk.ctx.query("panel_cols"),
                       "kind": "slot engine (per-phase kernels, CUDA graph)" if engine_used else
                               ("one thread-block cluster" if gk.ctx.query("cluster") else "persistent cooperative kernel")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "achieved_basis": basis, "csr_equivalent_GBs": csr_equiv,
                         "physical_GBs": physical, "physical_frac": physical / peak if physical else None,
                         "algorithmic_bytes_per_launch": per_launch, "algorithmic_bytes_per_iter": per_iter,
                         "kernel": (f"slot engine: {rows_kernel} + top / combine / update kernels per iteration "
                                    "(achieved = the whole solve's algorithmic bytes / its device time)"
                                    if engine_used else
                                    f"pcg_kernel<{gk.ctx.query('lanes')},{'true' if gk.ctx.query('scatter') == 2 else 'false'}>"
                                    " (one launch = the whole solve)"),
                         "dominant_kernel": dom,
                         "kernel_ms_avg": avg_ms,
                         "phase_us_per_iter": dict(zip(["direction_top", "rows_B_Bt", "residual_update",
                                                        "combine_Bt_partials" if engine_used else "other"],
                                                       [round(v * 1e3 / args.iters, 2) for v in np.mean(phase_ms, axis=0)])),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "gpu_direction(op, rhs, PcgConfig): pageable numpy inputs as the reference IPM passes them; "
                            "diagonals + rhs H2D, Jacobi build, PCG, solution D2H"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if args.workload == "cfg5" and gk.ctx.query("scatter") == 1 and phases[1] > 0:
            # random B (cfg5): each nonzero costs one random u gather and one
            # random fp64 atomic in L2; their measured ceilings on B200
            # (probes/random_probe.cu, profiles/r01_probe_random_access2.txt)
            # bound the rows phase before HBM does
            nnz = gk.ctx.query("nnz") / world
            floor_us = (nnz / L2_GATHER_PER_S + nnz / L2_ATOMIC_PER_S) * 1e6
            line["roofline"]["l2_request_bound"] = {
                "gathers_per_iter": nnz, "atomics_per_iter": nnz,
                "gather_rate_per_s": L2_GATHER_PER_S, "atomic_rate_per_s": L2_ATOMIC_PER_S,
                "floor_us_per_iter": round(floor_us, 1), "rows_phase_us_per_iter": round(float(phases[1]), 1),
                "frac": round(floor_us / float(phases[1]), 3),
                "source": "profiles/r01_probe_random_access2.txt (8 MB table, 148 SMs)"}
        if world == 1 and not args.no_cpu_baseline:
            try:
                # the reference on the same operator and rhs: the CPU baseline AND the
                # parity check of this very run (first iterations of the benchmarked path)
                ref = ReferencePath(problem, op, meta, args.workload)
                line["cpu_baseline"], ref_hist, ref_x = cpu_baseline(ref, rhs, args.cpu_iters, args.workload)
                v = np.random.default_rng(1234).standard_normal(op.dim)
                y_ref = ref.apply(v)
                gk2 = operator_for(op, device=local)
                gk2.set_diagonals(op.d_diag, op.q_diag_extra)
                apply_err = float(np.linalg.norm(gk2.apply(v) - y_ref) / np.linalg.norm(y_ref))
                jac_err = float(np.max(np.abs(gk2.jacobi() - ref.jacobi) / np.abs(ref.jacobi)))
                gx, ginfo, ghist = gk2.pcg(rhs, 1e-300, args.cpu_iters, True, history=True)
                hist_dev = float(np.max(np.abs(ghist - ref_hist) / ref_hist))
                x_err = float(np.linalg.norm(gx - ref_x) / max(np.linalg.norm(ref_x), 1e-300))
                hist_ok, hist_note = hist_dev <= 1e-8, "literal 1e-8"
                if not hist_ok:
                    # ill-conditioned operator (the SVM dual's residual swings by 1e4 per step): the
                    # histories are chaotic for ANY summation order; gate as the parity tests do, within
                    # 10x the envelope of the CPU reference re-run with reordered sums (tests/parity.py)
                    sys.path.insert(0, str(ROOT / "tests"))
                    import parity as tparity
                    from oracle import qp_oracle as orc
                    hop = host_operator(op)
                    env = tparity.envelope(hop, rhs, orc.PcgConfig(tol=1e-300, max_iters=args.cpu_iters), ref_hist)
                    hist_ok, hist_note = tparity.check_history(ghist, ref_hist, env)
                    hist_note = "CPU-reorder envelope (tests/parity.py): " + hist_note
                    if not hist_ok and float(np.max(env)) > 1e-2 and x_err <= 1e-6:
                        # reordering the CPU sums alone moves single residuals by > 1 %: the per-iteration
                        # norms are not comparable there; the iterates are (criterion-1 shape, <= 1e-6)
                        hist_ok = True
                        hist_note += (f"; envelope itself reaches {float(np.max(env)):.2e} (chaotic), gated on the "
                                      f"solution after {int(ginfo.iterations)} iterations instead")
                line["parity"] = {"apply_rel_err": apply_err, "jacobi_rel_err": jac_err, "hist_dev": hist_dev,
                                  "x_rel_err": x_err, "iterations_compared": int(ginfo.iterations), "against": ref.kind,
                                  "hist_gate": hist_note,
                                  "ok": bool(apply_err <= 1e-12 and jac_err <= 1e-12 and hist_ok),
                                  "gates": "apply, Jacobi <= 1e-12 relative; residual history <= 1e-8 relative, or within "
                                           "10x the CPU-reorder envelope where reordering alone exceeds 1e-8, or -- where "
                                           "that envelope itself exceeds 1e-2 -- the iterate after the compared iterations "
                                           "<= 1e-6 relative"}
            except Exception as exc:     # the measured line must still be printed
                line.setdefault("cpu_baseline", {"error": f"{type(exc).__name__}: {exc}"})
                line.setdefault("parity", {"ok": False, "error": f"{type(exc).__name__}: {exc}"})
        print(json.dumps(line), flush=True)
    gk.close()
    if world > 1 or args.force_sharded:
        torch.distributed.destroy_process_group()


def ipm_problem(name):
    from paper_2308_00637_b200 import workloads
    from paper_2308_00637_b200.ipm import IpmConfig
    from paper_2308_00637_b200.pcg import PcgConfig
    if name == "cfg1":
        problem, _, _ = workloads.dense_qp(seed=0)
        return problem, IpmConfig(mu_tol=1e-8, pcg=PcgConfig(tol=1e-10))
    if name == "cfg2":
        problem, _, _ = workloads.svm_primal(seed=2)
    elif name == "cfg3":
        problem, _, _ = workloads.rt_like(seed=3)
    elif name == "cfg4":
        problem, _, _ = workloads.rt_like(seed=4, n_vox=2_000_000, n_beam=100_000, density=0.001)
    elif name == "svm_dual":
        problem, _, _, _ = make_workload("svm_dual", 1.0)
    else:
        raise SystemExit("--ipm needs --workload cfg1..cfg4 (cfg5 is a fixed-iteration PCG sweep)")
    return problem, IpmConfig()


def run_ipm(args):
    """IPM wall time: the whole interior-point solve with the device-resident IPM."""
    import torch
    from paper_2308_00637_b200.ipm import DeviceIpm, solve as dev_solve
    rank, world, local = dist_env()
    if world > 1 and rank != 0:
        return                       # single-GPU measurement (replicas would be identical)
    torch.cuda.set_device(local)
    problem, cfg = ipm_problem(args.workload)
    dev = DeviceIpm(problem, device=local)
    launches0 = dev.kkt.ctx.query("kernel_launches")
    for _ in range(max(args.warmup, 3)):
        rep = dev.solve(cfg)
    walls = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            rep = dev.solve(cfg)
            walls.append(rep.wall_time)
    launches = (dev.kkt.ctx.query("kernel_launches") - launches0) // (args.steps + max(args.warmup, 3))
    dev.close()
    # e2e: problem upload + solve + x back, through the public solve()
    t0 = time.perf_counter()
    rep_e2e = dev_solve(problem, cfg, device=local)
    e2e = time.perf_counter() - t0
    line = {
        "metric": "IPM wall time (device-resident IPM + Jacobi-PCG direction solver)", "value": float(np.mean(walls)),
        "unit": "s", "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": float(np.mean(walls)) * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE generator; no dataset)",
        "config": {"workload": WORKLOAD_DESC[args.workload], "ipm": {"mu_tol": cfg.mu_tol, "cg_tol": cfg.pcg.tol,
                   "cg_max_iters": cfg.pcg.max_iters}, "status": rep.status.value, "ipm_iterations": rep.iterations,
                   "cg_iterations": rep.cg_total, "objective": rep.objective,
                   "l2": "each step re-solves the resident problem"},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": 8 * problem.n,
                "path": "paper_2308_00637_b200.ipm.solve(problem, cfg): upload + solve + x D2H"},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and args.workload != "svm_dual":
        # the drop-in as a reference user runs it: the reference's OWN IPM loop (host scipy code)
        # with gpu_direction as its direction_solver (ipm.py:185-212)
        from oracle import build_ref
        try:
            ref_ok = build_ref.available()
        except Exception:
            ref_ok = False
        if ref_ok:
            from oracle import refbridge
            from paper_2308_00637_b200.direction import gpu_direction
            qp = build_ref.import_qpipm()
            rcfg = qp.ipm.IpmConfig(gamma=cfg.gamma, mu_init=cfg.mu_init, mu_tol=cfg.mu_tol, mu_shrink=cfg.mu_shrink,
                                    max_iters=cfg.max_iters,
                                    pcg=qp.linalg.PcgConfig(tol=cfg.pcg.tol, max_iters=cfg.pcg.max_iters))
            rrep = qp.ipm.solve(refbridge.ref_problem(problem), rcfg, direction_solver=gpu_direction)
            line["reference_loop"] = {
                "value": rrep.wall_time, "unit": "s", "status": rrep.status.value, "ipm_iterations": rrep.iterations,
                "objective": rrep.objective,
                "path": "qpipm.ipm.solve(problem, cfg, direction_solver=gpu_direction): the reference's host loop "
                        "(residuals, rhs, recovery, step in scipy) around the GPU direction solve; upload included"}
    if not args.no_cpu_baseline:
        from oracle import qp_oracle as orc
        k = args.cpu_ipm_iters or (cfg.max_iters if args.workload == "cfg1" else 2)
        ocfg = orc.IpmConfig(gamma=cfg.gamma, mu_init=cfg.mu_init, mu_tol=cfg.mu_tol, mu_shrink=cfg.mu_shrink,
                             max_iters=k, pcg=orc.PcgConfig(tol=cfg.pcg.tol, max_iters=cfg.pcg.max_iters))
        if args.workload == "svm_dual":            # the oracle needs the Hessian on the host
            from oracle import svm_oracle as so
            problem = so.dual_problem(_SVM_META["x"], _SVM_META["y"], _SVM_META["sigma"], _SVM_META["c"])
        orep = orc.solve(problem, ocfg)
        full = orep.status == "converged"
        line["cpu_baseline"] = {
            "value": orep.wall_time if full else orep.wall_time / max(orep.iterations, 1),
            "unit": "s" if full else "s per IPM iteration", "cores": 1, "kind": "port",
            "sample": (f"full CPU IPM ({orep.iterations} IPM / {sum(t['cg_iters'] for t in orep.trace)} CG "
                       f"iterations, status {orep.status})" if full else
                       f"first {orep.iterations} IPM iterations ({sum(t['cg_iters'] for t in orep.trace)} CG)")
                      + "; oracle = numpy/scipy restatement of qpipm, bit-identical on the golden vectors"}
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` outside torchrun: re-launch as N ranks, one per
    GPU, exactly as the driver would (127.0.0.1 rendezvous on a free port)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    raise SystemExit(subprocess.run(cmd).returncode)


def main():
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.ipm:
        relaunch_under_torchrun(args)
    if args.launch_check:                 # launcher test (CPU): what each rank sees
        rank, world, local = dist_env()
        print(json.dumps({"launch_check": True, "rank": rank, "world": world, "local_rank": local,
                          "gpus": args.gpus}), flush=True)
        return
    if args.impl == "ours" and not args.ipm and dist_env()[1] != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={dist_env()[1]}")
    if args.ipm and args.impl != "reference":
        run_ipm(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
