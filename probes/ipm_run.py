"""Device IPM wall time on the BASELINE configs (GPU box)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_00637_b200 import workloads
from paper_2308_00637_b200.ipm import DeviceIpm, IpmConfig
from paper_2308_00637_b200.pcg import PcgConfig

for name in sys.argv[1].split(","):
    t0 = time.time()
    if name == "cfg1":
        problem, _, _ = workloads.dense_qp(seed=0); cfg = IpmConfig(mu_tol=1e-8, pcg=PcgConfig(tol=1e-10))
    elif name == "cfg2":
        problem, _, _ = workloads.svm_primal(seed=2); cfg = IpmConfig()
    elif name == "cfg3":
        problem, _, _ = workloads.rt_like(seed=3); cfg = IpmConfig()
    else:
        problem, _, _ = workloads.rt_like(seed=4, n_vox=2_000_000, n_beam=100_000, density=0.001); cfg = IpmConfig()
    gen = time.time() - t0
    dev = DeviceIpm(problem)
    t1 = time.time()
    rep = dev.solve(cfg, verbose="-v" in sys.argv)
    print(f"{name}: gen {gen:.1f}s upload {t1 - t0 - gen:.1f}s  status {rep.status.value} IPM {rep.iterations} "
          f"CG {rep.cg_total} wall {rep.wall_time:.3f}s objective {rep.objective:.12e}", flush=True)
    dev.close()
