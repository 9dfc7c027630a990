"""Kernel-SVM dual end to end on the device (GPU box): Gram Hessian build,
device IPM, model; prints timings and the IPM trace summary.
  python probes/svm_train.py [n] [d] [sigma] [C]"""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
from paper_2308_00637_b200 import svm
from paper_2308_00637_b200.ipm import DeviceIpm, IpmConfig
from paper_2308_00637_b200.workloads import svm_dual_data

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 100
sigma = float(sys.argv[3]) if len(sys.argv) > 3 else 10.0
C = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
x, y = svm_dual_data(seed=6, n=n, d=d)
data = svm.SvmDataset.from_dense(x, y)
cfg = svm.SvmConfig(sigma=sigma, c=C)
svm.rbf_hessian_device(data, sigma)                 # warm-up (module load, allocator)
torch.cuda.synchronize()
t0 = time.perf_counter()
prob = svm.build_svm_dual(data, cfg)
torch.cuda.synchronize()
t_gram = time.perf_counter() - t0
dev = DeviceIpm(prob)
t1 = time.perf_counter()
rep = dev.solve(IpmConfig())
t_ipm = time.perf_counter() - t1
dev.close()
print(f"n={n} d={d}: Gram+upload {t_gram * 1e3:.1f} ms; IPM {rep.status.value} in {rep.iterations} iterations, "
      f"{rep.cg_total} CG, wall {rep.wall_time:.2f} s (host {t_ipm:.2f} s), objective {rep.objective:.10e}")
for t in rep.trace[:: max(1, len(rep.trace) // 12)]:
    print(f"  it {t.iter:3d} mu {t.mu:.0e} cg {t.cg_iters:5d} primal {t.primal_inf:.2e} dual {t.dual_inf:.2e}")
svm._remember(data, sigma, 0, prob.hessian.m_dev)
model = svm.extract_model(data, cfg, rep.x)
print(f"bias {model.bias:.6f}, support vectors {len(model.support_indices)}, "
      f"training accuracy {svm.training_accuracy(model):.4f}")
