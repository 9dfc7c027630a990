// qpk_ipm.cuh -- the interior-point loop on the device (SURVEY.md 8(f) rows
// 1-2): per-IPM-iteration KKT work and the loop's scalars, around the PCG
// direction solver.  Restates qpipm/ipm.py:73-240 and kkt.py:113-143,
// 190-202, 242-284 with the iterate resident in HBM.
//
// Layout: B-row ("bottom") vectors follow B = (C; A_l; -A_u): the e rows
// [0, m_e), l rows [m_e, m_e + m_l), u rows [m_e + m_l, m_B).  So
//   slacks  s_B  = (unused, s_lA, s_uA),   multipliers lam_B = (lam_e, lam_lA, lam_uA),
//   bounds  bnd_B = (b, l_A, u_A),         t = B x = (C x, A_l x, -A_u x).
// Variable-bound families lx / ux live on index lists vlo / vhi.
#pragma once
#include "qpk_device.cuh"

namespace qpk {

struct IpmDev {
  int n, m, me, ml, mu_rows;     // m = me + ml + mu_rows
  int nl, nu;                    // variable-bound families
  const int* vlo; const int* vhi;
  const double* lx; const double* ux;   // bound values on those families
  const double* bnd;             // bottom order: b | l_A | u_A
  const double* pvec;            // linear term p (n)
  // iterate
  double* x;                     // n
  double* sB; double* lamB;      // m
  double* slx; double* sux; double* llx; double* lux;   // nl / nu
  // residuals
  double* rH;                    // n
  double* rB;                    // m: r_e | r_lA | r_uA
  double* rcB;                   // m: (unused for e) | r_c1 | r_c2
  double* rlx; double* rux; double* rc3; double* rc4;
  // direction
  double* dsB; double* dlamB;    // m (ds unused for e rows)
  double* dslx; double* dsux; double* dllx; double* dlux;
  // scratch
  double* hx;                    // H x (n)
  double* t;                     // B x (m)
  double* btl;                   // B' lam_B (n)
  double* part;                  // block partials
  int G;
};

__device__ __forceinline__ int row_family(const IpmDev& P, int i) {
  return i < P.me ? 0 : (i < P.me + P.ml ? 1 : 2);
}

// x0 and slacks (ipm.py:73-104); t = B x0 already computed
__global__ void k_ipm_init_x(IpmDev P) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.n; j += gridDim.x * blockDim.x) P.x[j] = 0.0;
}
// box midpoints / lower+1 / upper-1: families are index lists; a variable in
// both lists gets the midpoint.  Runs after k_ipm_init_x, one thread per entry.
__global__ void k_ipm_init_x_bounds(IpmDev P, const unsigned char* has_lo, const unsigned char* has_hi,
                                    const double* lo_full, const double* hi_full) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.n; j += gridDim.x * blockDim.x) {
    const bool l = has_lo[j], h = has_hi[j];
    double v = 0.0;
    if (l && h) v = 0.5 * (lo_full[j] + hi_full[j]);
    else if (l) v = lo_full[j] + 1.0;
    else if (h) v = hi_full[j] - 1.0;
    P.x[j] = v;
  }
}
__global__ void k_ipm_init_state(IpmDev P, double mu) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int i = tid; i < P.m; i += nth) {
    const int f = row_family(P, i);
    double s = 0.0, lam = 1.0;
    if (f == 0) { lam = 0.0; }
    else if (f == 1) s = fmax(1.0, fabs(P.t[i] - P.bnd[i]));          // A_l x - l_A
    else s = fmax(1.0, fabs(P.bnd[i] + P.t[i]));                        // u_A - A_u x  (t = -A_u x)
    P.sB[i] = s;
    P.lamB[i] = lam;
  }
  for (int k = tid; k < P.nl; k += nth) { P.slx[k] = fmax(1.0, fabs(P.x[P.vlo[k]] - P.lx[k])); P.llx[k] = 1.0; }
  for (int k = tid; k < P.nu; k += nth) { P.sux[k] = fmax(1.0, fabs(P.ux[k] - P.x[P.vhi[k]])); P.lux[k] = 1.0; }
}

// d_diag = (mu | s_lA/lam_lA | s_uA/lam_uA) and q_extra (kkt.py:190-202)
__global__ void k_ipm_diagonals(IpmDev P, double mu, double* d, double* q) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int i = tid; i < P.m; i += nth) d[i] = (i < P.me) ? mu : P.sB[i] / P.lamB[i];
  for (int j = tid; j < P.n; j += nth) q[j] = 0.0;
}
__global__ void k_ipm_qextra_lo(IpmDev P, double* q) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.nl; k += gridDim.x * blockDim.x)
    q[P.vlo[k]] += P.llx[k] / P.slx[k];
}
__global__ void k_ipm_qextra_hi(IpmDev P, double* q) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.nu; k += gridDim.x * blockDim.x)
    q[P.vhi[k]] += P.lux[k] / P.sux[k];
}

// residual blocks (kkt.py:113-143); needs hx = H x, t = B x, btl = B' lam_B.
// Partials (slot-major): 0 primal^2, 1 dual^2, 2 compl^2, 3 r_e^2, 4 non-finite count.
__global__ void __launch_bounds__(QPK_BLOCK) k_ipm_residuals(IpmDev P, double mu) {
  __shared__ double red[32];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  double pr = 0.0, co = 0.0, re = 0.0, bad = 0.0;
  for (int j = tid; j < P.n; j += nth) {
    const double v = (P.hx[j] + P.pvec[j]) - P.btl[j];
    P.rH[j] = v;
  }
  for (int i = tid; i < P.m; i += nth) {
    const int f = row_family(P, i);
    double rb, rc = 0.0;
    if (f == 0) {
      rb = (P.t[i] - P.bnd[i]) + mu * P.lamB[i];                          // r_e = C x - b + mu lam_e
      re += rb * rb;
    } else if (f == 1) {
      rb = (P.t[i] - P.sB[i]) - P.bnd[i];                                 // r_lA = A_l x - s - l_A
      rc = P.lamB[i] * P.sB[i] - mu;
    } else {
      rb = (P.bnd[i] + P.t[i]) - P.sB[i];                                 // r_uA = u_A - A_u x - s
      rc = P.lamB[i] * P.sB[i] - mu;
    }
    P.rB[i] = rb;
    P.rcB[i] = rc;
    if (f) { pr += rb * rb; co += rc * rc; }
    if (!isfinite(rb) || !isfinite(rc)) bad += 1.0;
  }
  for (int k = tid; k < P.nl; k += nth) {
    const double r = (P.x[P.vlo[k]] - P.slx[k]) - P.lx[k];
    const double c = P.llx[k] * P.slx[k] - mu;
    P.rlx[k] = r; P.rc3[k] = c;
    pr += r * r; co += c * c;
    if (!isfinite(r) || !isfinite(c)) bad += 1.0;
  }
  for (int k = tid; k < P.nu; k += nth) {
    const double r = (P.ux[k] - P.x[P.vhi[k]]) - P.sux[k];
    const double c = P.lux[k] * P.sux[k] - mu;
    P.rux[k] = r; P.rc4[k] = c;
    pr += r * r; co += c * c;
    if (!isfinite(r) || !isfinite(c)) bad += 1.0;
  }
  double t = block_sum(pr, red);
  if (threadIdx.x == 0) P.part[0 * P.G + blockIdx.x] = t;
  t = block_sum(co, red);
  if (threadIdx.x == 0) P.part[2 * P.G + blockIdx.x] = t;
  t = block_sum(re, red);
  if (threadIdx.x == 0) P.part[3 * P.G + blockIdx.x] = t;
  t = block_sum(bad, red);
  if (threadIdx.x == 0) P.part[4 * P.G + blockIdx.x] = t;
}
// variable-bound multipliers enter r_H after the elementwise part (kkt.py:294-295)
__global__ void k_ipm_rh_lo(IpmDev P) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.nl; k += gridDim.x * blockDim.x)
    P.rH[P.vlo[k]] -= P.llx[k];
}
__global__ void k_ipm_rh_hi(IpmDev P) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.nu; k += gridDim.x * blockDim.x)
    P.rH[P.vhi[k]] += P.lux[k];
}
__global__ void __launch_bounds__(QPK_BLOCK) k_ipm_dual_norm(IpmDev P) {
  __shared__ double red[32];
  double du = 0.0, bad = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.n; j += gridDim.x * blockDim.x) {
    const double v = P.rH[j];
    du += v * v;
    if (!isfinite(v)) bad += 1.0;
  }
  double t = block_sum(du, red);
  if (threadIdx.x == 0) P.part[1 * P.G + blockIdx.x] = t;
  t = block_sum(bad, red);
  if (threadIdx.x == 0) P.part[5 * P.G + blockIdx.x] = t;
}

// right-hand side (kkt.py:242-257): rhs_bottom = r2, w2 = 2 r2 / d (for the
// B' product), rhs_top = -r_H (+ bound terms, below) -- B' w2 added after.
__global__ void k_ipm_rhs(IpmDev P, const double* d, double* rhs, double* w2) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int j = tid; j < P.n; j += nth) rhs[j] = -P.rH[j];
  for (int i = tid; i < P.m; i += nth) {
    const int f = row_family(P, i);
    const double r2 = (f == 0) ? -P.rB[i] : (-P.rB[i] - P.rcB[i] / P.lamB[i]);
    rhs[P.n + i] = r2;
    w2[i] = 2.0 * r2 / d[i];
  }
}
__global__ void k_ipm_rhs_lo(IpmDev P, double* rhs) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.nl; k += gridDim.x * blockDim.x)
    rhs[P.vlo[k]] += -P.rc3[k] / P.slx[k] - (P.llx[k] / P.slx[k]) * P.rlx[k];
}
__global__ void k_ipm_rhs_hi(IpmDev P, double* rhs) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.nu; k += gridDim.x * blockDim.x)
    rhs[P.vhi[k]] += P.rc4[k] / P.sux[k] + (P.lux[k] / P.sux[k]) * P.rux[k];
}
__global__ void k_ipm_rhs_top(IpmDev P, double* rhs, const double* btw, double* bad_part) {
  __shared__ double red[32];
  double bad = 0.0;
  const int N = P.n + P.m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (i < P.n) rhs[i] = rhs[i] + btw[i];
    if (!isfinite(rhs[i])) bad += 1.0;
  }
  const double t = block_sum(bad, red);
  if (threadIdx.x == 0) bad_part[blockIdx.x] = t;
}

// direction recovery (kkt.py:260-284) + ratio-test partial minima
// (ipm.py:107-132).  sol = (dx, d_lam_B).  Partials: 0 min slack ratio,
// 1 min multiplier ratio, 2 non-finite count.
__device__ __forceinline__ void ratio(double v, double dv, double& m) {
  if (dv < 0.0) m = fmin(m, -v / dv);
}
__global__ void __launch_bounds__(QPK_BLOCK) k_ipm_recover(IpmDev P, const double* sol) {
  __shared__ double red[32];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  double ms = INFINITY, ml = INFINITY, bad = 0.0;
  const double* dx = sol;
  const double* dl = sol + P.n;
  for (int j = tid; j < P.n; j += nth) if (!isfinite(dx[j])) bad += 1.0;
  for (int i = tid; i < P.m; i += nth) {
    const int f = row_family(P, i);
    const double dlam = dl[i];
    P.dlamB[i] = dlam;
    if (!isfinite(dlam)) bad += 1.0;
    if (f == 0) continue;
    const double rc = P.rcB[i];
    const double ds = -(rc + P.sB[i] * dlam) / P.lamB[i];                // ds_lA / ds_uA
    P.dsB[i] = ds;
    if (!isfinite(ds)) bad += 1.0;
    ratio(P.sB[i], ds, ms);
    ratio(P.lamB[i], dlam, ml);
  }
  for (int k = tid; k < P.nl; k += nth) {
    const double ds = dx[P.vlo[k]] + P.rlx[k];
    const double dlam = -(P.rc3[k] + P.llx[k] * ds) / P.slx[k];
    P.dslx[k] = ds; P.dllx[k] = dlam;
    if (!isfinite(ds) || !isfinite(dlam)) bad += 1.0;
    ratio(P.slx[k], ds, ms);
    ratio(P.llx[k], dlam, ml);
  }
  for (int k = tid; k < P.nu; k += nth) {
    const double ds = P.rux[k] - dx[P.vhi[k]];
    const double dlam = -(P.rc4[k] + P.lux[k] * ds) / P.sux[k];
    P.dsux[k] = ds; P.dlux[k] = dlam;
    if (!isfinite(ds) || !isfinite(dlam)) bad += 1.0;
    ratio(P.sux[k], ds, ms);
    ratio(P.lux[k], dlam, ml);
  }
  // block minima (tree of fmin through shared memory)
  __shared__ double mins[2][QPK_BLOCK / 32];
  for (int o = 16; o > 0; o >>= 1) {
    ms = fmin(ms, __shfl_xor_sync(0xffffffffu, ms, o));
    ml = fmin(ml, __shfl_xor_sync(0xffffffffu, ml, o));
  }
  if ((threadIdx.x & 31) == 0) { mins[0][threadIdx.x >> 5] = ms; mins[1][threadIdx.x >> 5] = ml; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = INFINITY, b = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a = fmin(a, mins[0][w]); b = fmin(b, mins[1][w]); }
    P.part[0 * P.G + blockIdx.x] = a;
    P.part[1 * P.G + blockIdx.x] = b;
  }
  const double t = block_sum(bad, red);
  if (threadIdx.x == 0) P.part[2 * P.G + blockIdx.x] = t;
}

// move x and slacks by alpha_x, multipliers by alpha_lam (ipm.py:135-153);
// partial: min over the updated slacks / multipliers
__global__ void __launch_bounds__(QPK_BLOCK) k_ipm_step(IpmDev P, const double* dx, double ax, double al) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  double mn = INFINITY;
  for (int j = tid; j < P.n; j += nth) P.x[j] = P.x[j] + ax * dx[j];
  for (int i = tid; i < P.m; i += nth) {
    const double lam = P.lamB[i] + al * P.dlamB[i];
    P.lamB[i] = lam;
    if (i >= P.me) {
      const double s = P.sB[i] + ax * P.dsB[i];
      P.sB[i] = s;
      mn = fmin(mn, fmin(s, lam));
    }
  }
  for (int k = tid; k < P.nl; k += nth) {
    P.slx[k] = P.slx[k] + ax * P.dslx[k];
    P.llx[k] = P.llx[k] + al * P.dllx[k];
    mn = fmin(mn, fmin(P.slx[k], P.llx[k]));
  }
  for (int k = tid; k < P.nu; k += nth) {
    P.sux[k] = P.sux[k] + ax * P.dsux[k];
    P.lux[k] = P.lux[k] + al * P.dlux[k];
    mn = fmin(mn, fmin(P.sux[k], P.lux[k]));
  }
  __shared__ double mins[QPK_BLOCK / 32];
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) mins[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a = fmin(a, mins[w]);
    P.part[0 * P.G + blockIdx.x] = a;
  }
}

// objective partial: x'(H x) / 2 + p'x (model.py:257-258)
__global__ void __launch_bounds__(QPK_BLOCK) k_ipm_objective(IpmDev P) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.n; j += gridDim.x * blockDim.x) {
    a += P.x[j] * P.hx[j];
    b += P.pvec[j] * P.x[j];
  }
  double t = block_sum(a, red);
  if (threadIdx.x == 0) P.part[0 * P.G + blockIdx.x] = t;
  t = block_sum(b, red);
  if (threadIdx.x == 0) P.part[1 * P.G + blockIdx.x] = t;
}

// ---- sparse products used by the IPM (not on the PCG hot path) ----
// t = B u, one row per thread group of 4 lanes over the padded CSR
__global__ void __launch_bounds__(QPK_BLOCK) k_spmv_b(Op op, const double* u, double* t) {
  const int lane = threadIdx.x & 3;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < 4LL * ((op.m + 7) / 8 * 8);
       g += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(g >> 2);
    double s = 0.0;
    if (r < op.m) {
      const int b = __ldg(op.rp + r), e = __ldg(op.rp + r + 1);
      for (int k = b + lane; k < e; k += 4) {
        const int c = __ldg(op.ci + k);
        if (c >= 0) s = fma(__ldg(op.bv + k), u[c], s);
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (r < op.m && lane == 0) t[r] = s;
  }
}
// y += B' w (atomic scatter; y zeroed by the caller)
__global__ void __launch_bounds__(QPK_BLOCK) k_spmv_bt(Op op, const double* w, double* y) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < op.m;
       r += (long long)gridDim.x * blockDim.x) {
    const double wr = w[r];
    if (wr == 0.0) continue;
    const int b = __ldg(op.rp + r), e = __ldg(op.rp + r + 1);
    for (int k = b; k < e; ++k) {
      const int c = __ldg(op.ci + k);
      if (c >= 0) atomicAdd(y + c, __ldg(op.bv + k) * wr);
    }
  }
}

}  // namespace qpk
