// qpk.cu -- libqpk.so: B200-native Jacobi-PCG on the doubly augmented KKT
// system, behind the C ABI declared in include/qpk.h.
//
// Kernels
//   pcg_kernel<L, CSC>   persistent cooperative kernel running the whole PCG
//                        solve of linalg.py:66-133 on the device (one launch
//                        per solve, grid.sync between phases, no host round
//                        trips); L = lanes per row of B, CSC = gather-only
//                        (deterministic) B'z.
//   k_prep / k_rows / k_finish   the same phases as standalone launches, for
//                        qpk_apply (apply_doubly_augmented, kkt.py:211-221)
//   k_jac_*              jacobi_diagonal (kkt.py:224-239) + inv_diag (ipm.py:180)
//   k_hdiag_*            hessian_diagonal (model.py:179-186), once per problem
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <dlfcn.h>

#include "../../include/qpk.h"
#include "qpk_device.cuh"
#include "qpk_engine.cuh"
#include "qpk_tma.cuh"
#include "qpk_panel.cuh"
#include "qpk_cluster.cuh"
#include "qpk_ipm.cuh"
#include "qpk_svm.cuh"
#include <chrono>

namespace cg = cooperative_groups;
using namespace qpk;

// =========================================================== device code ===
struct PcgOut {
  int iterations, converged, status, restarts, applies, result_buf;
  double final_norm, threshold, rhs_norm;
  unsigned long long phase_ns[4];
};


// per-phase wall time as seen by block 0 (includes waiting for the slowest block)
struct PhaseClock {
  unsigned long long last = 0, acc[4] = {0, 0, 0, 0};
  __device__ void start() { last = globaltimer_ns(); }
  __device__ void lap(int phase) { const unsigned long long t = globaltimer_ns(); acc[phase] += t - last; last = t; }
};

struct PcgParams {
  Op op;
  const double* rhs;
  double* x0; double* x1; double* x2;
  double* r; double* p; double* y; double* zb;
  const double* minv;
  double* part; int G;
  double tol; int rel; long long max_iters;
  double* hist;
  PcgOut* out;
};

__device__ __forceinline__ void write_out(const PcgParams& P, long long iters, int conv, int status,
                                          int restarts, int applies, int buf, double fin, double thr,
                                          double rhs_norm, PhaseClock& pc) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    pc.lap(3);
    for (int i = 0; i < 4; ++i) P.out->phase_ns[i] = pc.acc[i];
    P.out->iterations = (int)iters; P.out->converged = conv; P.out->status = status;
    P.out->restarts = restarts; P.out->applies = applies; P.out->result_buf = buf;
    P.out->final_norm = fin; P.out->threshold = thr; P.out->rhs_norm = rhs_norm;
  }
}

// Top half of the direction update, with the lazy x update and the prep of
// the next apply:  x_t <- x_t + alpha_prev p_t ;  z = minv r ;
// p_t <- z (+ beta p_t) ;  y_t <- diag-part(Q) p_t.
// Partial sums: SLOT_AUX = r'z (top), SLOT_PREP = p'(diag Q)p, SLOT_S.. = U'p.
__device__ void phase_top(const PcgParams& P, const RowFuse& f, double* red) {
  const Op& op = P.op;
  const int G = P.G;
  double rz = 0.0, acc = 0.0;
  double sacc[QPK_KMAX];
  const bool lr = op.H.kind == HESS_LOWRANK;
  if (lr) for (int kk = 0; kk < op.H.k; ++kk) sacc[kk] = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < op.n; j += gridDim.x * blockDim.x) {
    const double pold = P.p[j];
    if (f.xupd) f.xdst[j] = __dadd_rn(f.xsrc[j], __dmul_rn(f.alpha_prev, pold));
    const double rj = P.r[j];
    const double zj = __dmul_rn(__ldg(P.minv + j), rj);
    rz += rj * zj;
    const double pn = f.restart ? zj : __dadd_rn(zj, __dmul_rn(f.beta, pold));
    P.p[j] = pn;
    acc += prep_elem(op, j, pn, P.y);
    if (lr) lowrank_accum(op, j, pn, sacc);
  }
  double t = block_sum(rz, red);
  if (threadIdx.x == 0) P.part[SLOT_AUX * G + blockIdx.x] = t;
  t = block_sum(acc, red);
  if (threadIdx.x == 0) P.part[SLOT_PREP * G + blockIdx.x] = t;
  if (lr) lowrank_flush(op, sacc, P.part, G, red);
}

// r <- r - alpha y ; partial r'r and r'z (z = minv r).  Atomic mode: y is final,
// vectorised over pairs; CSC mode: top entries of y completed by the gather.
template <bool CSC>
__device__ void phase_update(const PcgParams& P, double alpha, double* red) {
  const Op& op = P.op;
  const int N = op.n + op.m, G = P.G;
  double rr = 0.0, rz = 0.0;
  if (!CSC) {
    const int np = N >> 1;
    double2* r2 = reinterpret_cast<double2*>(P.r);
    const double2* y2 = reinterpret_cast<const double2*>(P.y);
    const double2* m2 = reinterpret_cast<const double2*>(P.minv);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
      double2 ri = r2[i];
      const double2 yi = y2[i];
      const double2 mi = __ldg(m2 + i);
      ri.x = __dsub_rn(ri.x, __dmul_rn(alpha, yi.x));
      ri.y = __dsub_rn(ri.y, __dmul_rn(alpha, yi.y));
      r2[i] = ri;
      rr += ri.x * ri.x + ri.y * ri.y;
      rz += ri.x * __dmul_rn(mi.x, ri.x) + ri.y * __dmul_rn(mi.y, ri.y);
    }
    if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const int i = N - 1;
      const double ri = __dsub_rn(P.r[i], __dmul_rn(alpha, P.y[i]));
      P.r[i] = ri;
      rr += ri * ri;
      rz += ri * __dmul_rn(__ldg(P.minv + i), ri);
    }
  } else {
    for_each_final<true>(op, P.y, P.zb, [&](int i, double yi) {
      const double ri = __dsub_rn(P.r[i], __dmul_rn(alpha, yi));
      P.r[i] = ri;
      rr += ri * ri;
      rz += ri * __dmul_rn(__ldg(P.minv + i), ri);
    });
  }
  double t = block_sum(rr, red);
  if (threadIdx.x == 0) P.part[SLOT_RR * G + blockIdx.x] = t;
  t = block_sum(rz, red);
  if (threadIdx.x == 0) P.part[SLOT_RZ * G + blockIdx.x] = t;
}

__device__ __forceinline__ int spare_buffer(int cur, int best) {
  return (cur != best) ? 3 - cur - best : (cur + 1) % 3;
}

// explicit residual r = rhs - K x (linalg.py:113-114, 132); partial ||r||^2 -> SLOT_RR
template <int L, bool CSC>
__device__ double true_residual(const PcgParams& P, double* x, bool store_r, double* red, double* s_lr) {
  cg::grid_group grid = cg::this_grid();
  const Op& op = P.op;
  const int G = P.G;
  phase_prep(op, x, P.y, P.part, G, red);
  grid.sync();
  RowFuse none{};
  phase_rows<L, CSC, false>(op, x, P.y, P.zb, P.part, G, red, s_lr, none);
  grid.sync();
  double rr = 0.0;
  for_each_final<CSC>(op, P.y, P.zb, [&](int i, double yi) {
    const double ri = __dsub_rn(__ldg(P.rhs + i), yi);
    if (store_r) P.r[i] = ri;
    rr += ri * ri;
  });
  const double t = block_sum(rr, red);
  if (threadIdx.x == 0) P.part[SLOT_RR * G + blockIdx.x] = t;
  grid.sync();
  return sqrt(grid_total(P.part + SLOT_RR * G, G, red));
}

template <int L, bool CSC>
__global__ void __launch_bounds__(QPK_BLOCK, QPK_PCG_MIN_BLOCKS) pcg_kernel(PcgParams P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  __shared__ double s_lr[QPK_KMAX];
  const Op& op = P.op;
  const int N = op.n + op.m, G = P.G;
  double* xs[3] = {P.x0, P.x1, P.x2};
  const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
  PhaseClock pc;
  if (writer) pc.start();

  // x = 0, r = rhs (linalg.py:85-87), ||rhs||
  {
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
      const double b = __ldg(P.rhs + i);
      P.x0[i] = 0.0;
      P.r[i] = b;
      acc += b * b;
    }
    const double t = block_sum(acc, red);
    if (threadIdx.x == 0) P.part[SLOT_AUX * G + blockIdx.x] = t;
  }
  grid.sync();
  const double rhs_norm = sqrt(grid_total(P.part + SLOT_AUX * G, G, red));
  const double thr = P.rel ? P.tol * rhs_norm : P.tol;          // linalg.py:83
  double rnorm = rhs_norm, best_rnorm = rhs_norm;
  int cur = 0, best = 0, xn = 0, restarts = 0, applies = 0;
  if (writer && P.hist) P.hist[0] = rnorm;
  if (rnorm <= thr) {                                               // linalg.py:93-94
    write_out(P, 0, 1, QPK_PCG_OK, 0, 0, 0, rnorm, thr, rhs_norm, pc);
    return;
  }
  // f carries the pending state: restart (p = z), beta, lazy x update
  RowFuse f{};
  f.r = P.r;
  f.restart = 1;
  f.xupd = 0;
  double rz = 0.0;

  for (long long k = 1; k <= P.max_iters; ++k) {
    f.xsrc = xs[cur];
    f.xdst = xs[xn];
    // p <- z (+ beta p) and x <- x + alpha p (top half), y_top init
    phase_top(P, f, red);
    grid.sync();
    if (writer) pc.lap(0);
    // y = K p; bottom half of the direction/x update fused in
    phase_rows<L, CSC, true>(op, P.p, P.y, P.zb, P.part, G, red, s_lr, f);
    ++applies;
    grid.sync();
    if (writer) pc.lap(1);
    if (f.xupd) { cur = xn; f.xupd = 0; }
    if (f.restart) rz = grid_total(P.part + SLOT_AUX * G, G, red) + grid_total(P.part + SLOT_AUX2 * G, G, red);
    const double pap = grid_total(P.part + SLOT_ROWS * G, G, red) + grid_total(P.part + SLOT_PREP * G, G, red);
    if (pap <= 0.0) {                                               // linalg.py:102-103
      write_out(P, k - 1, 0, QPK_PCG_BREAKDOWN, restarts, applies, best, best_rnorm, thr, rhs_norm, pc);
      return;
    }
    const double alpha = rz / pap;
    phase_update<CSC>(P, alpha, red);                               // r -= alpha y
    grid.sync();
    if (writer) pc.lap(2);
    rnorm = sqrt(grid_total(P.part + SLOT_RR * G, G, red));
    if (writer && P.hist) P.hist[k] = rnorm;
    // x_k = x_{k-1} + alpha p is pending; it will land in buffer xn
    xn = spare_buffer(cur, best);
    f.xupd = 1;
    f.alpha_prev = alpha;
    if (rnorm < best_rnorm) { best = xn; best_rnorm = rnorm; }      // linalg.py:110-111
    if (rnorm <= thr) {
      // materialise x_k, then the explicit residual (linalg.py:112-116)
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
        xs[xn][i] = __dadd_rn(xs[cur][i], __dmul_rn(alpha, P.p[i]));
      grid.sync();
      cur = xn;
      f.xupd = 0;
      const double true_norm = true_residual<L, CSC>(P, xs[cur], true, red, s_lr);
      ++applies;
      if (true_norm <= thr) {
        write_out(P, k, 1, QPK_PCG_OK, restarts, applies, cur, true_norm, thr, rhs_norm, pc);
        return;
      }
      // recurrence drifted: restart from the explicit residual (linalg.py:117-125)
      ++restarts;
      rnorm = true_norm;
      if (rnorm < best_rnorm) { best = cur; best_rnorm = rnorm; }
      f.restart = 1;
      continue;
    }
    const double rz_next = grid_total(P.part + SLOT_RZ * G, G, red);  // linalg.py:126-130
    f.beta = rz_next / rz;
    f.restart = 0;
    rz = rz_next;
  }
  // iteration cap: materialise the pending iterate, then the true residual of
  // the best one (linalg.py:132-133)
  if (f.xupd) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
      xs[xn][i] = __dadd_rn(xs[cur][i], __dmul_rn(f.alpha_prev, P.p[i]));
    grid.sync();
    cur = xn;
  }
  const double true_norm = true_residual<L, CSC>(P, xs[best], false, red, s_lr);
  ++applies;
  write_out(P, P.max_iters, true_norm <= thr ? 1 : 0, QPK_PCG_OK, restarts, applies, best, true_norm, thr,
            rhs_norm, pc);
}

// ---------------------------------------------------- standalone phases ---
// y += H' u for the non-diagonal Hessian kinds (after k_prep with q = 0)
__global__ void __launch_bounds__(QPK_BLOCK) k_hess(Op op, const double* u, double* y, double* part, int G) {
  __shared__ double red[32];
  __shared__ double s_lr[QPK_KMAX];
  if (op.H.kind == HESS_DENSE && op.H.sym) hess_sym(op, u, y);
  else hess_rows(op, u, y, part, G, red, s_lr);
}

// the packed symmetric H's partials into y (after k_hess), fixed order
__global__ void __launch_bounds__(QPK_SYMC_BLOCK) k_sym_combine(Op op, const double* u, double* y) {
  __shared__ double sh[QPK_SYMC_BLOCK];
  sym_combine(op, u, y, sh);
}

// dense symmetric H -> its upper 64 x 64 tiles, tile (I, J >= I) at
// I*nt - I*(I-1)/2 + (J - I), zero padded past n
__global__ void __launch_bounds__(256) k_pack_sym(const double* __restrict__ Hd, long long n, int nt,
                                                 double* __restrict__ out) {
  const int I = blockIdx.y, J = blockIdx.x;
  if (J < I) return;
  const size_t t = (size_t)I * nt - (size_t)I * (I - 1) / 2 + (J - I);
  double* dst = out + t * 4096;
  for (int e = threadIdx.x; e < 4096; e += 256) {
    const long long r = (long long)I * 64 + e / 64, col = (long long)J * 64 + e % 64;
    dst[e] = (r < n && col < n) ? Hd[r * n + col] : 0.0;
  }
}

// H == H' bit for bit?  (the packed upper-tile apply mirrors the upper triangle;
// the reference's hessian_apply, model.py:165-176, multiplies whatever it is given)
__global__ void __launch_bounds__(256) k_sym_check(const double* __restrict__ Hd, long long n, int* __restrict__ bad) {
  const int I = blockIdx.y, J = blockIdx.x;
  if (J < I) return;
  int mism = 0;
  for (int e = threadIdx.x; e < 4096; e += 256) {
    const long long r = (long long)I * 64 + e / 64, col = (long long)J * 64 + e % 64;
    if (r < n && col < n && col > r)
      mism |= __double_as_longlong(Hd[r * n + col]) != __double_as_longlong(Hd[col * n + r]);
  }
  if (mism) atomicOr(bad, 1);
}

__global__ void __launch_bounds__(QPK_BLOCK) k_prep(Op op, const double* v, double* y, double* part, int G) {
  __shared__ double red[32];
  phase_prep(op, v, y, part, G, red);
}

template <int L, bool CSC>
__global__ void __launch_bounds__(QPK_BLOCK) k_rows(Op op, const double* v, double* y, double* zb, double* part, int G) {
  __shared__ double red[32];
  __shared__ double s_lr[QPK_KMAX];
  RowFuse none{};
  phase_rows<L, CSC, false>(op, const_cast<double*>(v), y, zb, part, G, red, s_lr, none);
}

__global__ void __launch_bounds__(QPK_BLOCK) k_finish_csc(Op op, double* y, const double* zb) {
  for_each_final<true>(op, y, zb, [&](int i, double yi) { if (i < op.n) y[i] = yi; });
}

// Jacobi: acc_j = sum_r B_rj^2 * (1/d_r)
template <int L>
__global__ void __launch_bounds__(QPK_BLOCK) k_jac_rows(Op op, double* acc) {
  const int lane = threadIdx.x & (L - 1);
  const long long sub = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / L;
  const long long nsub = ((long long)gridDim.x * blockDim.x) / L;
  for (long long r = sub; r < op.m; r += nsub) {
    const double dinv = 1.0 / __ldg(op.d + r);
    const int b = __ldg(op.rp + r), e = __ldg(op.rp + r + 1);
    for (int k = b + 4 * lane; k < e; k += 4 * L) {
      int4 c = ld_stream_i4(op.ci + k);
      double2 a0 = ld_stream_d2(op.bv + k), a1 = ld_stream_d2(op.bv + k + 2);
      if (c.x >= 0) atomicAdd(acc + c.x, __dmul_rn(a0.x, a0.x) * dinv);
      if (c.y >= 0) atomicAdd(acc + c.y, __dmul_rn(a0.y, a0.y) * dinv);
      if (c.z >= 0) atomicAdd(acc + c.z, __dmul_rn(a1.x, a1.x) * dinv);
      if (c.w >= 0) atomicAdd(acc + c.w, __dmul_rn(a1.y, a1.y) * dinv);
    }
  }
}

__global__ void __launch_bounds__(QPK_BLOCK) k_jac_cols(Op op, double* acc) {
  const int LC = op.csc_lanes, lc = threadIdx.x & (LC - 1);
  const int per = 32 / LC, sw = (threadIdx.x & 31) / LC;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
  for (long long jb = (long long)gwarp * per; jb < op.n; jb += (long long)nwarp * per) {
    const int j = (int)jb + sw;
    double s = 0.0;
    if (j < op.n) {
      const int b = __ldg(op.cp + j), e = __ldg(op.cp + j + 1);
      for (int k = b + 4 * lc; k < e; k += 4 * LC) {
        const int4 c = ld_stream_i4(op.ri + k);
        const double2 a0 = ld_stream_d2(op.cv + k), a1 = ld_stream_d2(op.cv + k + 2);
        if (c.x >= 0) s += __dmul_rn(a0.x, a0.x) * (1.0 / __ldg(op.d + c.x));
        if (c.y >= 0) s += __dmul_rn(a0.y, a0.y) * (1.0 / __ldg(op.d + c.y));
        if (c.z >= 0) s += __dmul_rn(a1.x, a1.x) * (1.0 / __ldg(op.d + c.z));
        if (c.w >= 0) s += __dmul_rn(a1.y, a1.y) * (1.0 / __ldg(op.d + c.w));
      }
    }
    for (int o = LC / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (j < op.n && lc == 0) acc[j] = s;
  }
}

// jac = (diag(H) + q_extra) + 2 acc ; D   and   minv = 1 / jac
__global__ void k_jac_finish(Op op, const double* hdiag, const double* acc, double* jac, double* minv) {
  const int N = op.n + op.m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    double v;
    if (i < op.n) v = __dadd_rn(__dadd_rn(__ldg(hdiag + i), __ldg(op.q + i)), __dmul_rn(2.0, acc[i]));
    else v = __ldg(op.d + (i - op.n));
    jac[i] = v;
    minv[i] = 1.0 / v;
  }
}

// diag(H) once per problem (model.py:179-186)
__global__ void k_hdiag(Hess H, int n, double* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double v = 0.0;
    if (H.kind == HESS_DIAG) v = H.h[j];
    else if (H.kind == HESS_DENSE) v = H.dense[(size_t)j * n + j];
    else if (H.kind == HESS_CSR) {
      for (int k = H.rp[j]; k < H.rp[j + 1]; ++k)
        if (H.ci[k] == j) { v = H.v[k]; break; }
    } else {
      double s = 0.0;
      const double* urow = H.U + (size_t)j * H.k;
      for (int kk = 0; kk < H.k; ++kk) s += H.w[kk] * (urow[kk] * urow[kk]);
      v = H.h[j] + s;
    }
    out[j] = v;
  }
}

// ============================================================= host side ===
struct QpkNcclId { char internal[128]; };

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) return fail(QPK_E_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                  \
  } while (0)

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() { if (p) cudaFree(p); p = nullptr; n = 0; }
  cudaError_t alloc(size_t count) {
    if (count <= n && p) return cudaSuccess;
    release();
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) n = count; else p = nullptr;
    return e;
  }
  size_t bytes() const { return n * sizeof(T); }
};

int pow2_clamp(long long v, int lo, int hi) {
  int p = 1;
  while (p < v && p < hi) p <<= 1;
  return std::max(lo, std::min(hi, p));
}

// ---- NCCL, loaded at run time (the process's own libnccl.so.2: torch's when
// torch is loaded, so only one NCCL is ever in the process) ----
struct NcclApi {
  bool tried = false, ok = false;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, QpkNcclId, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*errStr)(int) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.getUniqueId = (int (*)(void*))dlsym(h, "ncclGetUniqueId");
  api.commInitRank = (int (*)(void**, int, QpkNcclId, int))dlsym(h, "ncclCommInitRank");
  api.allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclAllReduce");
  api.groupStart = (int (*)())dlsym(h, "ncclGroupStart");
  api.groupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
  api.commDestroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
  api.errStr = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.groupStart && api.groupEnd && api.commDestroy;
  return api;
}

// Host threads for the format builders (the box has far more cores than the
// one a serial build uses; the result does not depend on the thread count)
static int host_threads() {
  if (const char* ev = getenv("QPK_HOST_THREADS")) return std::max(1, std::min(64, atoi(ev)));
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(16u, hc ? hc : 4u));
}

template <typename F>
static void parallel_chunks(int nchunks, F fn) {
  const int T = std::min(host_threads(), nchunks);
  if (T <= 1) { for (int k = 0; k < nchunks; ++k) fn(k); return; }
  std::atomic<int> next(0);
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&] { for (int k = next++; k < nchunks; k = next++) fn(k); });
  for (auto& t : th) t.join();
}

struct SetupTimer {
  bool on = getenv("QPK_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[qpk setup] %-12s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

constexpr int NCCL_FLOAT64 = 8, NCCL_SUM = 0;

}  // namespace

// Test-only stand-in for the communicator (qpk_multi_create_emulated): the
// ranks are contexts of ONE process, each driven by its own host thread; an
// all-reduce synchronises the rank's stream, meets the other ranks at a host
// barrier and sums the buffers in rank order on the host.  No kernel ever
// waits on another rank, so several ranks can share one GPU.
struct HostComm {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<std::vector<double>> bufs;
  bool broken = false;
  // false when a rank never shows up (it failed): the others give up instead of hanging
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const long long g = gen;
    if (++arrived == n) { arrived = 0; ++gen; cv.notify_all(); return true; }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct qpk_ctx {
  int device = 0;
  int sms = 0;
  cudaStream_t own = nullptr, stream = nullptr;
  long long launches = 0;

  // problem staging
  bool building = false, finalized = false;
  long long n = 0, m = 0, m_e = 0, m_l = 0, m_u = 0;
  std::vector<int> h_rp;
  std::vector<int> h_ci;
  std::vector<double> h_v;
  long long nnz = 0;

  int hkind = -1;
  long long hk = 0;
  std::vector<double> h_h;               // diag d / low-rank h0
  std::vector<int> h_hrp, h_hci; std::vector<double> h_hv;
  std::vector<double> h_dense, h_U, h_w;
  const double* h_dense_dev = nullptr;  // dense H given as a device matrix (copied at finalize)

  int scatter = QPK_SCATTER_ATOMIC;
  int lanes = 4, csc_lanes = 8, h_lanes = 8;

  // device problem
  DBuf<int> rp, ci, cp, ri, hrp, hci, seg_ptr, seg_beg;
  DBuf<double> seg_sum;
  int n_seg = 0, seg_lanes = 8;
  // row-block dictionaries
  DBuf<int> dcols, col_ptr, col_pos, comb_beg, comb_col;
  DBuf<double> comb_sum;
  int comb_lanes = 8, comb_nseg = 0;
  DBuf<TileDescD> tiles;
  DBuf<int> hperm;                // Hessian tile row q -> H row hperm[q] (RCM order)
  // CTA-level accumulation of the tile partials (Dict::cacc)
  bool cacc = false;
  int tile_grid = 0;
  bool h_symmetric = true;
  DBuf<int> hown;                 // sharded, CSR H: the H rows this rank applies (RCM order)
  std::vector<int> h_own;
  bool h_own_set = false;
  DBuf<int> tile_beg, cta_off, tslot, col_ptr2, col_pos2, comb_beg2, comb_col2;
  DBuf<double> cpart;
  int comb_lanes2 = 8, comb_nseg2 = 0, comb_max2 = 0;   // max CTA partials of one column
  DBuf<double> tval;
  DBuf<double> bpart;
  int nblk = 0;
  bool have_dict = false, h_tiled = false;
  double dict_reuse = 0.0;        // tile density: nonzeros / dense tile slots
  DBuf<double> bv, cv, hh, hv, hdense, U, w, hdiag;
  DBuf<double> hsym;             // dense H as packed upper tiles (large dense H)
  DBuf<double> cdense;           // the leading dense rows of B as dense n-vectors
  int n_dense = 0;
  DBuf<int4> hchunks;
  int h_nchunks = 0;
  DBuf<double> hsymp;            // partial sums of the packed symmetric apply
  DBuf<int> hrowchunk;
  bool have_csc = false;
  // dense column panel (QPK_SCATTER_PANEL)
  bool have_panel = false;
  int panel_kp = 0, panel_q = 0, panel_ew = 0, panel_direct = 0, panel_grid = 0, panel_kd = 0;
  DBuf<double> panel_P, panel_ev, panel_part, panel_ue, panel_yrem;
  DBuf<int> panel_cols, panel_eci, panel_cpos;

  // per IPM iteration
  DBuf<double> d, q, jac, minv;
  bool diag_set = false, jac_ready = false;

  // work
  DBuf<double> x[3], r, p, y, zb, rhs, part, hist, vin;
  DBuf<PcgOut> out;
  int grid_pcg = 0, grid_std = 0;
  // small systems: the whole solve in one thread-block cluster (qpk_cluster.cuh)
  int cl_C = 0;                    // 0: not used
  size_t cl_smem = 0;
  DBuf<ClCta> cl_ctas;
  DBuf<unsigned char> cl_blob;
  DBuf<long long> cl_off;

  // device-resident IPM (qpk_ipm_*)
  bool ipm_ready = false;
  long long nl = 0, nu = 0;
  DBuf<int> vlo, vhi;
  DBuf<double> ipm_lx, ipm_ux, ipm_bnd, ipm_p, ipm_x, ipm_sB, ipm_lamB, ipm_slx, ipm_sux, ipm_llx, ipm_lux;
  DBuf<double> ipm_rH, ipm_rB, ipm_rcB, ipm_rlx, ipm_rux, ipm_rc3, ipm_rc4;
  DBuf<double> ipm_dsB, ipm_dlamB, ipm_dslx, ipm_dsux, ipm_dllx, ipm_dlux;
  DBuf<double> ipm_hx, ipm_t, ipm_btl, ipm_part, ipm_rhs, ipm_sol, ipm_w2, ipm_tmp, ipm_zero;
  DBuf<double> ipm_lofull, ipm_hifull;
  DBuf<unsigned char> ipm_haslo, ipm_hashi;

  // row sharding over ranks (one process per GPU)
  int world = 1, rank = 0;
  bool sharded = false;
  void* comm = nullptr;
  HostComm* hostcomm = nullptr;   // test-only host-mediated all-reduce (emulated ranks)
  bool fold_all = false;          // every rank can run the folded (one all-reduce) slot
  DBuf<double> gscal, lscal2, abuf;

  // slot engine
  int engine = -1;               // -1 auto, 0 persistent kernel, 1 slot engine
  int grid_eng = 0;
  DBuf<Ctrl> ctrl;
  DBuf<unsigned int> counter;
  DBuf<EngineCfg> ecfg;
  int* pinned_mode = nullptr;    // [2] host-mapped poll flags
  cudaEvent_t poll_ev[2] = {nullptr, nullptr};
  cudaEvent_t time_ev[2] = {nullptr, nullptr};   // solve timing (created once, reused)
  cudaGraphExec_t graph = nullptr;
  int graph_slots = 0;
  bool graph_failed = false;
  int attr_scatter = -1, attr_kp = -1;

  Op op() const {
    Op o;
    o.n = (int)n; o.m = (int)m;
    o.rp = rp.p; o.ci = ci.p; o.bv = bv.p;
    o.cp = cp.p; o.ri = ri.p; o.cv = cv.p; o.csc_lanes = csc_lanes;
    o.H.kind = hkind; o.H.h = hh.p; o.H.rp = hrp.p; o.H.ci = hci.p; o.H.v = hv.p; o.H.lanes = h_lanes;
    o.H.dense = hdense.p; o.H.U = U.p; o.H.w = w.p; o.H.k = (int)hk;
    o.H.sym = hsym.p; o.H.chunks = hchunks.p; o.H.nchunks = h_nchunks;
    o.H.symp = hsymp.p; o.H.rowchunk = hrowchunk.p;
    o.H.rows = h_own_set ? hown.p : nullptr; o.H.nrows = h_own_set ? (int)h_own.size() : 0;
    o.d = d.p; o.q = q.p;
    o.top_owner = rank == 0 ? 1 : 0;
    o.t_lo = (int)(n * rank / world); o.t_hi = (int)(n * (rank + 1) / world);   // this rank's top slice
    o.r0 = 0; o.ndense = 0; o.cdense = nullptr;        // dense-row split: slot engine only (make_engine)
    return o;
  }
  long long N() const { return n + m; }
};

template <typename T>
static cudaError_t upload(DBuf<T>& dst, const std::vector<T>& src, cudaStream_t s) {
  cudaError_t e = dst.alloc(src.size());
  if (e != cudaSuccess || src.empty()) return e;
  return cudaMemcpyAsync(dst.p, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s);
}

// src followed by `pad` copies of `fill`, without a padded host copy of src
// (pageable sources: the copies return once the host buffer is staged)
template <typename T>
static cudaError_t upload_padded(DBuf<T>& dst, const std::vector<T>& src, size_t pad, T fill, cudaStream_t s) {
  cudaError_t e = dst.alloc(src.size() + pad);
  if (e != cudaSuccess) return e;
  if (!src.empty()) {
    e = cudaMemcpyAsync(dst.p, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
  }
  const std::vector<T> tail(pad, fill);
  return cudaMemcpyAsync(dst.p + src.size(), tail.data(), pad * sizeof(T), cudaMemcpyHostToDevice, s);
}

#ifndef QPK_SYM_MIN_N
#define QPK_SYM_MIN_N 512      // dense H at least this large is applied from packed symmetric tiles
#endif
#define QPK_SYM_CHUNK 2        // tiles per hess_sym work unit
#ifndef QPK_DENSE_ROW_MIN
#define QPK_DENSE_ROW_MIN 2048 // a leading B row this long (and >= n/4) is applied as a dense vector
#endif

static int engine_setup(qpk_ctx* c);
static Engine make_engine(qpk_ctx* c);
static size_t tile_smem() { return sizeof(DTileSmem) + (size_t)QPK_TILE_GROUPS * QPK_TILE_UMAX * sizeof(double); }

// ---------------------------------------------------------- dispatchers ---
template <int L, bool CSC>
static const void* pcg_fn() { return (const void*)pcg_kernel<L, CSC>; }

static const void* pcg_kernel_for(int lanes, bool csc) {
  switch (lanes) {
    case 1: return csc ? pcg_fn<1, true>() : pcg_fn<1, false>();
    case 2: return csc ? pcg_fn<2, true>() : pcg_fn<2, false>();
    case 4: return csc ? pcg_fn<4, true>() : pcg_fn<4, false>();
    case 8: return csc ? pcg_fn<8, true>() : pcg_fn<8, false>();
    case 16: return csc ? pcg_fn<16, true>() : pcg_fn<16, false>();
    default: return csc ? pcg_fn<32, true>() : pcg_fn<32, false>();
  }
}

template <bool CSC>
static void launch_rows(int lanes, int grid, cudaStream_t s, const Op& o, const double* v, double* y, double* zb,
                        double* part, int G) {
  switch (lanes) {
    case 1: k_rows<1, CSC><<<grid, QPK_BLOCK, 0, s>>>(o, v, y, zb, part, G); break;
    case 2: k_rows<2, CSC><<<grid, QPK_BLOCK, 0, s>>>(o, v, y, zb, part, G); break;
    case 4: k_rows<4, CSC><<<grid, QPK_BLOCK, 0, s>>>(o, v, y, zb, part, G); break;
    case 8: k_rows<8, CSC><<<grid, QPK_BLOCK, 0, s>>>(o, v, y, zb, part, G); break;
    case 16: k_rows<16, CSC><<<grid, QPK_BLOCK, 0, s>>>(o, v, y, zb, part, G); break;
    default: k_rows<32, CSC><<<grid, QPK_BLOCK, 0, s>>>(o, v, y, zb, part, G); break;
  }
}

static void launch_jac_rows(int lanes, int grid, cudaStream_t s, const Op& o, double* acc) {
  switch (lanes) {
    case 1: k_jac_rows<1><<<grid, QPK_BLOCK, 0, s>>>(o, acc); break;
    case 2: k_jac_rows<2><<<grid, QPK_BLOCK, 0, s>>>(o, acc); break;
    case 4: k_jac_rows<4><<<grid, QPK_BLOCK, 0, s>>>(o, acc); break;
    case 8: k_jac_rows<8><<<grid, QPK_BLOCK, 0, s>>>(o, acc); break;
    case 16: k_jac_rows<16><<<grid, QPK_BLOCK, 0, s>>>(o, acc); break;
    default: k_jac_rows<32><<<grid, QPK_BLOCK, 0, s>>>(o, acc); break;
  }
}

// Kernel launch with programmatic dependent launch (PDL) allowed: the kernel
// may be scheduled while its stream predecessor drains (qpk_device.cuh,
// pdl_wait / pdl_trigger); plain launch when pdl is false
template <typename... KArgs, typename... Args>
static void launch_k(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid; lc.blockDim = block; lc.dynamicSmemBytes = smem; lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at; lc.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&lc, k, args...);
}

static const int kPanelQ[] = {1, 2, 4, 6, 8, 12, 16};


template <int Q>
static void launch_panel_t(const qpk_ctx* c, cudaStream_t s, const Engine& E, int par, bool pdl) {
  launch_k(pdl, k_slot_panel<Q>, dim3(c->panel_grid), dim3(QPK_PANEL_CW * 32),
           panel_smem_bytes(c->panel_kp, c->panel_ew), s, E, par);
}
template <int Q>
static void launch_jac_panel_t(const qpk_ctx* c, cudaStream_t s, const Engine& E) {
  k_jac_panel<Q><<<c->panel_grid, QPK_PANEL_CW * 32, (size_t)QPK_PANEL_CW * c->panel_kp * sizeof(double), s>>>(E);
}
template <int Q>
static cudaError_t panel_attr_t(const qpk_ctx* c) {
  cudaError_t e = cudaFuncSetAttribute(k_slot_panel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)panel_smem_bytes(c->panel_kp, c->panel_ew));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_jac_panel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(QPK_PANEL_CW * c->panel_kp * sizeof(double)));
}
#define QPK_PANEL_DISPATCH(FN, ...)                   \
  switch (c->panel_q) {                               \
    case 1: FN<1>(__VA_ARGS__); break;                \
    case 2: FN<2>(__VA_ARGS__); break;                \
    case 4: FN<4>(__VA_ARGS__); break;                \
    case 6: FN<6>(__VA_ARGS__); break;                \
    case 8: FN<8>(__VA_ARGS__); break;                \
    case 12: FN<12>(__VA_ARGS__); break;              \
    default: FN<16>(__VA_ARGS__); break;              \
  }

static cudaError_t panel_attr(const qpk_ctx* c) {
  switch (c->panel_q) {
    case 1: return panel_attr_t<1>(c);
    case 2: return panel_attr_t<2>(c);
    case 4: return panel_attr_t<4>(c);
    case 6: return panel_attr_t<6>(c);
    case 8: return panel_attr_t<8>(c);
    case 12: return panel_attr_t<12>(c);
    default: return panel_attr_t<16>(c);
  }
}

// ------------------------------------------------------------------ ABI ---
extern "C" {

int qpk_abi_version(void) { return QPK_ABI_VERSION; }
const char* qpk_last_error(void) { return g_err.c_str(); }

int qpk_create(int device, qpk_ctx** out) {
  if (!out) return fail(QPK_E_ARG, "qpk_create: out is NULL");
  int count = 0;
  CUDA_TRY(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(QPK_E_ARG, "qpk_create: device %d of %d", device, count);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (!prop.cooperativeLaunch) return fail(QPK_E_UNSUPPORTED, "device %d lacks cooperative launch", device);
  qpk_ctx* c = new (std::nothrow) qpk_ctx();
  if (!c) return fail(QPK_E_NOMEM, "qpk_create: host allocation failed");
  c->device = device;
  c->sms = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete c; return fail(QPK_E_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e)); }
  c->stream = c->own;
  if (c->out.alloc(1) != cudaSuccess) { delete c; return fail(QPK_E_NOMEM, "qpk_create: device alloc"); }
  *out = c;
  return QPK_OK;
}

int qpk_destroy(qpk_ctx* c) {
  if (!c) return QPK_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->comm && nccl().ok) nccl().commDestroy(c->comm);
  for (auto& e : c->poll_ev) if (e) cudaEventDestroy(e);
  for (auto& e : c->time_ev) if (e) cudaEventDestroy(e);
  if (c->pinned_mode) cudaFreeHost(c->pinned_mode);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
  return QPK_OK;
}

int qpk_set_stream(qpk_ctx* c, void* stream) {
  if (!c) return fail(QPK_E_ARG, "null context");
  c->stream = stream ? (cudaStream_t)stream : c->own;
  return QPK_OK;
}

int qpk_synchronize(qpk_ctx* c) {
  if (!c) return fail(QPK_E_ARG, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return QPK_OK;
}

int qpk_nccl_get_unique_id(unsigned char* id) {
  if (!id) return fail(QPK_E_ARG, "qpk_nccl_get_unique_id: null buffer");
  if (!nccl().ok) return fail(QPK_E_UNSUPPORTED, "libnccl.so.2 not loadable");
  const int rc = nccl().getUniqueId(id);
  if (rc != 0) return fail(QPK_E_CUDA, "ncclGetUniqueId failed (%d)", rc);
  return QPK_OK;
}

int qpk_shard_init(qpk_ctx* c, int world, int rank, const unsigned char* id) {
  if (!c || world < 1 || rank < 0 || rank >= world || !id) return fail(QPK_E_ARG, "qpk_shard_init: bad arguments");
  if (c->building || c->finalized) return fail(QPK_E_STATE, "qpk_shard_init must precede qpk_problem_begin");
  if (!nccl().ok) return fail(QPK_E_UNSUPPORTED, "libnccl.so.2 not loadable");
  CUDA_TRY(cudaSetDevice(c->device));
  QpkNcclId uid;
  memcpy(uid.internal, id, sizeof uid.internal);
  const int rc = nccl().commInitRank(&c->comm, world, uid, rank);
  if (rc != 0) return fail(QPK_E_CUDA, "ncclCommInitRank failed: %s", nccl().errStr ? nccl().errStr(rc) : "?");
  c->world = world;
  c->rank = rank;
  c->sharded = true;
  return QPK_OK;
}

// Test hook: this context behaves as rank `rank` of `world` WITHOUT a
// communicator -- it holds its row shard, owns its slice of the top block and
// of the Hessian rows, and qpk_apply / qpk_jacobi return its un-reduced share
// (the caller sums the shares of all ranks on the host).  Lets one GPU check
// the partition logic of the N > 1 layout rank by rank, with no kernel of one
// rank ever waiting on another.
int qpk_shard_emulate(qpk_ctx* c, int world, int rank) {
  if (!c || world < 1 || rank < 0 || rank >= world) return fail(QPK_E_ARG, "qpk_shard_emulate: bad arguments");
  if (c->building || c->finalized) return fail(QPK_E_STATE, "qpk_shard_emulate must precede qpk_problem_begin");
  c->world = world;
  c->rank = rank;
  c->sharded = false;
  return QPK_OK;
}

int qpk_problem_begin(qpk_ctx* c, int64_t n, int64_t m_e, int64_t m_l, int64_t m_u) {
  if (!c) return fail(QPK_E_ARG, "null context");
  if (n < 1 || m_e < 0 || m_l < 0 || m_u < 0)
    return fail(QPK_E_ARG, "qpk_problem_begin: bad sizes n=%lld m_e=%lld m_l=%lld m_u=%lld", (long long)n,
                (long long)m_e, (long long)m_l, (long long)m_u);
  if (n + m_e + m_l + m_u >= (1LL << 31) - 64) return fail(QPK_E_UNSUPPORTED, "dimension exceeds int32 range");
  c->building = true; c->finalized = false; c->diag_set = false; c->jac_ready = false; c->have_csc = false;
  c->graph_failed = false; c->h_symmetric = true;
  c->n = n; c->m_e = m_e; c->m_l = m_l; c->m_u = m_u; c->m = 0;
  c->h_rp.assign(1, 0); c->h_ci.clear(); c->h_v.clear(); c->nnz = 0;
  c->hkind = -1; c->hk = 0;
  return QPK_OK;
}

int qpk_problem_add_rows(qpk_ctx* c, int64_t n_rows, const int64_t* ro, const int64_t* ci, const double* vals,
                         const int64_t* rows, int64_t n_sel, double sign) {
  if (!c || !c->building) return fail(QPK_E_STATE, "qpk_problem_add_rows: no problem being built");
  if (n_rows < 0 || !ro || (n_rows > 0 && (!ci && ro[n_rows] > 0)))
    return fail(QPK_E_ARG, "qpk_problem_add_rows: bad CSR");
  const int64_t count = rows ? n_sel : n_rows;
  const long long mB = c->m_e + c->m_l + c->m_u;
  if (c->m + count > mB) return fail(QPK_E_ARG, "qpk_problem_add_rows: more rows than m_B=%lld", mB);
  // validate the selection and lay the rows out (padded to 4 entries), then
  // convert them on the host threads
  std::vector<size_t> at((size_t)count + 1, c->h_ci.size());
  for (int64_t s = 0; s < count; ++s) {
    const int64_t i = rows ? rows[s] : s;
    if (i < 0 || i >= n_rows) return fail(QPK_E_ARG, "qpk_problem_add_rows: row index %lld out of range", (long long)i);
    if (ro[i + 1] < ro[i]) return fail(QPK_E_ARG, "row_offsets must be nondecreasing");
    at[s + 1] = at[s] + (size_t)((ro[i + 1] - ro[i] + 3) & ~3LL);
    c->nnz += ro[i + 1] - ro[i];
  }
  if (at[count] >= (size_t)(1LL << 31) - 64) return fail(QPK_E_UNSUPPORTED, "nnz exceeds int32 range");
  c->h_ci.resize(at[count], -1);
  c->h_v.resize(at[count], 0.0);
  const size_t rp0 = c->h_rp.size();
  c->h_rp.resize(rp0 + (size_t)count);
  const int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(256, count / 4096));
  std::atomic<long long> bad_col(-1);
  int* hci = c->h_ci.data();
  double* hv = c->h_v.data();
  int* hrp = c->h_rp.data() + rp0;
  const int64_t ncols = c->n;
  parallel_chunks(nchunks, [&](int k) {
    const int64_t s0 = count * k / nchunks, s1 = count * (k + 1) / nchunks;
    for (int64_t s = s0; s < s1; ++s) {
      const int64_t i = rows ? rows[s] : s;
      size_t o = at[s];
      for (int64_t e = ro[i]; e < ro[i + 1]; ++e, ++o) {
        const int64_t col = ci[e];
        if (col < 0 || col >= ncols) { bad_col = col; return; }
        hci[o] = (int)col;
        hv[o] = sign * vals[e];
      }
      hrp[s] = (int)at[s + 1];
    }
  });
  if (bad_col.load() != -1) return fail(QPK_E_ARG, "column index %lld out of range", bad_col.load());
  c->m += count;
  return QPK_OK;
}

int qpk_set_hessian_diag(qpk_ctx* c, const double* dd) {
  if (!c || !c->building || !dd) return fail(QPK_E_STATE, "qpk_set_hessian_diag: bad state/arg");
  c->hkind = QPK_HESS_DIAG;
  c->h_h.assign(dd, dd + c->n);
  return QPK_OK;
}

int qpk_set_hessian_csr(qpk_ctx* c, const int64_t* ro, const int64_t* ci, const double* v) {
  if (!c || !c->building || !ro) return fail(QPK_E_STATE, "qpk_set_hessian_csr: bad state/arg");
  const int64_t nnz = ro[c->n];
  if (nnz >= (1LL << 31)) return fail(QPK_E_UNSUPPORTED, "Hessian nnz exceeds int32 range");
  c->hkind = QPK_HESS_CSR;
  c->h_hrp.resize(c->n + 1);
  for (long long j = 0; j <= c->n; ++j) c->h_hrp[j] = (int)ro[j];
  c->h_hci.resize(nnz);
  c->h_hv.assign(v, v + nnz);
  for (int64_t k = 0; k < nnz; ++k) {
    if (ci[k] < 0 || ci[k] >= c->n) return fail(QPK_E_ARG, "Hessian column out of range");
    c->h_hci[k] = (int)ci[k];
  }
  // lanes per H row from the NON-EMPTY rows (RT Hessians: most beamlets never
  // touch the target, the rest have hundreds of entries), ~5 entries per lane
  long long nonempty = 0;
  for (long long j = 0; j < c->n; ++j) nonempty += ro[j + 1] > ro[j];
  c->h_lanes = pow2_clamp((nnz + std::max<long long>(nonempty, 1) - 1) / std::max<long long>(nonempty, 1) / 5, 1, 32);
  return QPK_OK;
}

int qpk_set_hessian_dense(qpk_ctx* c, const double* mm) {
  if (!c || !c->building || !mm) return fail(QPK_E_STATE, "qpk_set_hessian_dense: bad state/arg");
  c->hkind = QPK_HESS_DENSE;
  c->h_dense.assign(mm, mm + c->n * c->n);
  return QPK_OK;
}

int qpk_set_hessian_dense_dev(qpk_ctx* c, const double* mm) {
  if (!c || !c->building || !mm) return fail(QPK_E_STATE, "qpk_set_hessian_dense_dev: bad state/arg");
  c->hkind = QPK_HESS_DENSE;
  std::vector<double>().swap(c->h_dense);
  c->h_dense_dev = mm;
  return QPK_OK;
}

int qpk_rbf_hessian_dev(qpk_ctx* c, const double* X, int64_t n, int64_t d, const double* y, double sigma,
                        double* H) {
  if (!c || !X || !y || !H || n < 1 || d < 0) return fail(QPK_E_ARG, "qpk_rbf_hessian_dev: bad argument");
  if (!(sigma > 0.0)) return fail(QPK_E_ARG, "qpk_rbf_hessian_dev: sigma must be positive");
  if ((n + QPK_GRAM_T - 1) / QPK_GRAM_T > 65535) return fail(QPK_E_ARG, "qpk_rbf_hessian_dev: n too large");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  double* sq = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&sq, n * sizeof(double), s));
  k_rowsq<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(X, n, d, sq);
  const unsigned T = (unsigned)((n + QPK_GRAM_T - 1) / QPK_GRAM_T);
  k_rbf_hessian<<<dim3(T, T), 256, 0, s>>>(X, n, d, y, sq, 1.0 / (2.0 * sigma), H);
  c->launches += 2;
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(sq, s));
  return QPK_OK;
}

int qpk_set_hessian_lowrank(qpk_ctx* c, const double* h0, int64_t k, const double* u, const double* w) {
  if (!c || !c->building || !h0 || k < 0) return fail(QPK_E_STATE, "qpk_set_hessian_lowrank: bad state/arg");
  if (k > QPK_KMAX) return fail(QPK_E_UNSUPPORTED, "low-rank Hessian with k=%lld > %d", (long long)k, QPK_KMAX);
  c->hkind = QPK_HESS_LOWRANK;
  c->hk = k;
  c->h_h.assign(h0, h0 + c->n);
  c->h_U.assign(u, u + c->n * k);
  c->h_w.assign(w, w + k);
  return QPK_OK;
}

// B' as CSC, every column padded to a multiple of 4 entries (row -1, value 0);
// rows inside a column ascend (deterministic gather order)
static int build_csc(qpk_ctx* c, const std::vector<int>& h_rp, const std::vector<int>& h_ci,
                     const std::vector<double>& h_v) {
  const long long n = c->n;
  std::vector<long long> cnt(n, 0);
  for (int col : h_ci) if (col >= 0) cnt[col]++;
  std::vector<int> cp(n + 1, 0);
  long long tot = 0;
  for (long long j = 0; j < n; ++j) {
    cp[j] = (int)tot;
    tot += (cnt[j] + 3) & ~3LL;
    if (tot >= (1LL << 31) - 64) return fail(QPK_E_UNSUPPORTED, "padded CSC exceeds int32 range");
  }
  cp[n] = (int)tot;
  std::vector<int> ri(tot, -1);
  std::vector<double> cv(tot, 0.0);
  std::vector<int> pos(cp.begin(), cp.end() - 1);
  for (long long r = 0; r < c->m; ++r)
    for (int k = h_rp[r]; k < h_rp[r + 1]; ++k) {
      const int col = h_ci[k];
      if (col < 0) continue;
      const int at = pos[col]++;
      ri[at] = (int)r;
      cv[at] = h_v[k];
    }
  // column segments for the engine's B'z pass: LS lanes x 8 entries each
  {
    const long long avg = tot / std::max<long long>(n, 1);
    c->seg_lanes = pow2_clamp((avg + 7) / 8, 1, 32);
    if (const char* ev = getenv("QPK_SEG_LANES")) c->seg_lanes = pow2_clamp(atoi(ev), 1, 32);
    const int seg = 8 * c->seg_lanes;
    std::vector<int> sp(n + 1), sb;
    sb.reserve(tot / seg + n + 1);
    for (long long j = 0; j < n; ++j) {
      sp[j] = (int)sb.size();
      for (int b = cp[j]; b < cp[j + 1]; b += seg) sb.push_back(b);
    }
    sp[n] = (int)sb.size();
    sb.push_back(cp[n]);
    c->n_seg = sp[n];
    // each segment ends where the next one (or the next column) begins
    CUDA_TRY(upload(c->seg_ptr, sp, c->stream));
    CUDA_TRY(upload(c->seg_beg, sb, c->stream));
    CUDA_TRY(c->seg_sum.alloc(std::max(c->n_seg, 1)));
  }
  CUDA_TRY(upload(c->cp, cp, c->stream));
  CUDA_TRY(upload(c->ri, ri, c->stream));
  CUDA_TRY(upload(c->cv, cv, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  // lanes per column: ~16 entries (4 chunks) per lane
  c->csc_lanes = pow2_clamp((tot / std::max<long long>(n, 1) + 15) / 16, 1, 32);
  if (const char* ev = getenv("QPK_CSC_LANES")) c->csc_lanes = pow2_clamp(atoi(ev), 1, 32);
  c->have_csc = true;
  return QPK_OK;
}

// Reverse Cuthill-McKee order of a symmetric sparsity pattern (rows of H):
// BFS from a pseudo-peripheral vertex of each component, neighbours by
// increasing degree, reversed.  Returns perm[new position] = old row.
static std::vector<int> rcm_order(long long n, const std::vector<int>& rp, const std::vector<int>& ci) {
  std::vector<int> order, deg(n), level(n, -1), nb;
  order.reserve(n);
  for (long long i = 0; i < n; ++i) deg[i] = rp[i + 1] - rp[i];
  std::vector<char> done(n, 0);
  auto bfs_last = [&](int s) {                       // farthest vertex from s (level structure)
    std::vector<int> q{s};
    level[s] = 0;
    int last = s;
    for (size_t h = 0; h < q.size(); ++h) {
      const int x = q[h];
      last = x;
      for (int k = rp[x]; k < rp[x + 1]; ++k) {
        const int y = ci[k];
        if (y >= 0 && y < n && level[y] < 0) { level[y] = level[x] + 1; q.push_back(y); }
      }
    }
    for (int x : q) level[x] = -1;
    return last;
  };
  std::vector<int> idx(n);
  for (long long i = 0; i < n; ++i) idx[i] = (int)i;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return deg[a] < deg[b]; });
  for (int s0 : idx) {
    if (done[s0]) continue;
    const int s = bfs_last(bfs_last(s0));
    const size_t head0 = order.size();
    order.push_back(s);
    done[s] = 1;
    for (size_t h = head0; h < order.size(); ++h) {
      const int x = order[h];
      nb.clear();
      for (int k = rp[x]; k < rp[x + 1]; ++k) {
        const int y = ci[k];
        if (y >= 0 && y < n && !done[y]) { done[y] = 1; nb.push_back(y); }
      }
      std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] < deg[b]; });
      for (int y : nb) order.push_back(y);
    }
  }
  std::reverse(order.begin(), order.end());
  return order;
}

struct TileOut {
  std::vector<TileDescD> tiles;
  std::vector<int> cols;
  std::vector<double> tval;
  long long slots = 0;
  bool too_wide = false;        // a single row does not fit a tile
};

// Tile the rows [q0, q1) of a CSR matrix (tile row q is matrix row perm[q], or
// q): consecutive rows grouped while (rows x padded distinct columns) fits
// QPK_TILE_DOUBLES, each tile a dense block over its sorted column list.
// d0 / v0 of the descriptors are offsets into o.cols / o.tval.
static void tile_range(const int* rp, const int* ci, const double* v, const int* perm, long long q0, long long q1,
                       int kind, std::vector<int>& mark, int& stamp, TileOut& o) {
  auto r4 = [](long long x) { return (x + 3) & ~3LL; };
  auto R = [&](long long q) -> long long { return perm ? perm[q] : q; };
  std::vector<int> cur;
  cur.reserve(QPK_TILE_DMAX);
  long long r = q0;
  while (r < q1) {
    const long long ra = r;
    cur.clear();
    ++stamp;
    while (r < q1) {
      long long fresh = 0;
      for (int k = rp[R(r)]; k < rp[R(r) + 1]; ++k)
        if (ci[k] >= 0 && mark[ci[k]] != stamp) ++fresh;
      const long long nd = (long long)cur.size() + fresh, rows = r - ra + 1;
      if (r4(nd) > QPK_TILE_DMAX || rows * (r4(nd) | 1) > QPK_TILE_DOUBLES || rows > QPK_TILE_ROWS) {
        if (r == ra) { o.too_wide = true; return; }
        break;
      }
      for (int k = rp[R(r)]; k < rp[R(r) + 1]; ++k)
        if (ci[k] >= 0 && mark[ci[k]] != stamp) { mark[ci[k]] = stamp; cur.push_back(ci[k]); }
      ++r;
    }
    std::sort(cur.begin(), cur.end());
    const int ndp = (int)r4((long long)cur.size());
    const int pitch = ndp | 1;                        // odd row pitch: conflict-free column reads
    TileDescD td;
    td.ra = (int)ra; td.rb = (int)r; td.d0 = (int)o.cols.size(); td.ndp = ndp;
    td.v0 = (int)((o.tval.size() + 1) & ~(size_t)1);  // 16-byte aligned block start
    td.pad0 = pitch; td.pad1 = kind; td.pad2 = 0;
    if ((long long)td.v0 + (r - ra) * pitch >= (1LL << 31) - 64) { o.too_wide = true; return; }
    for (int col : cur) o.cols.push_back(col);
    for (int i = (int)cur.size(); i < ndp; ++i) o.cols.push_back(-1);
    const size_t base = td.v0;
    o.tval.resize(base + (size_t)(r - ra) * pitch, 0.0);
    for (long long rr = ra; rr < r; ++rr)
      for (int k = rp[R(rr)]; k < rp[R(rr) + 1]; ++k) {
        if (ci[k] < 0) continue;
        const int pos = (int)(std::lower_bound(cur.begin(), cur.end(), ci[k]) - cur.begin());
        o.tval[base + (size_t)(rr - ra) * pitch + pos] = v[k];
      }
    o.slots += (r - ra) * pitch;
    o.tiles.push_back(td);
  }
}

// The rows [0, nrows) tiled in nnz-balanced chunks on the host threads (tiles
// end at chunk boundaries; the chunking depends on the matrix only), appended
// to tiles / cols / tval.  Returns the dense slots, or -1 (a row too wide, or
// the tile storage would exceed the int32 offsets).
static long long tile_rows_parallel(const int* rp, const int* ci, const double* v, const int* perm, long long nrows,
                                    int kind, long long n, std::vector<TileDescD>& tiles, std::vector<int>& cols,
                                    std::vector<double>& tval, size_t reserve_extra = 0) {
  if (nrows <= 0) return 0;
  const int C = (int)std::max<long long>(1, std::min<long long>(512, nrows / 2048));
  std::vector<long long> cut(C + 1, 0);
  cut[C] = nrows;
  for (int k = 1; k < C; ++k) {
    if (perm) { cut[k] = nrows * k / C; continue; }   // permuted rows: equal row counts
    const long long want = (long long)rp[0] + ((long long)rp[nrows] - rp[0]) * k / C;
    cut[k] = std::max(cut[k - 1], (long long)(std::lower_bound(rp, rp + nrows, (int)want) - rp));
  }
  std::vector<TileOut> outs(C);
  {
    const int T = std::min(host_threads(), C);
    std::vector<std::vector<int>> marks(T);
    std::atomic<int> next(0), slot(0);
    auto work = [&] {
      const int me = slot++;
      marks[me].assign(n, 0);
      int stamp = 0;
      for (int k = next++; k < C; k = next++)
        tile_range(rp, ci, v, perm, cut[k], cut[k + 1], kind, marks[me], stamp, outs[k]);
    };
    if (T <= 1) {
      work();
    } else {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t) th.emplace_back(work);
      for (auto& t : th) t.join();
    }
  }
  long long slots = 0;
  std::vector<size_t> cb(C + 1, cols.size()), vb(C + 1, (tval.size() + 1) & ~(size_t)1), tb(C + 1, tiles.size());
  for (int k = 0; k < C; ++k) {
    if (outs[k].too_wide) return -1;
    slots += outs[k].slots;
    cb[k + 1] = cb[k] + outs[k].cols.size();
    vb[k + 1] = vb[k] + ((outs[k].tval.size() + 1) & ~(size_t)1);
    tb[k + 1] = tb[k] + outs[k].tiles.size();
  }
  if (vb[C] >= (size_t)(1LL << 31) - 64 || cb[C] >= (size_t)(1LL << 31) - 64) return -1;
  // (room for what the caller appends next -- the Hessian tiles -- so the
  // 1.4 GB value array of cfg4 is not reallocated and copied)
  cols.reserve(cb[C] + reserve_extra + 64);
  tval.reserve(vb[C] + reserve_extra + 64);
  cols.resize(cb[C]);
  tval.resize(vb[C], 0.0);
  tiles.resize(tb[C]);
  parallel_chunks(C, [&](int k) {
    TileOut& o = outs[k];
    if (!o.cols.empty()) memcpy(cols.data() + cb[k], o.cols.data(), o.cols.size() * sizeof(int));
    if (!o.tval.empty()) memcpy(tval.data() + vb[k], o.tval.data(), o.tval.size() * sizeof(double));
    for (size_t t = 0; t < o.tiles.size(); ++t) {
      TileDescD td = o.tiles[t];
      td.d0 += (int)cb[k];
      td.v0 += (int)vb[k];
      tiles[tb[k] + t] = td;
    }
    std::vector<double>().swap(o.tval);
    std::vector<int>().swap(o.cols);
  });
  return slots;
}

// Dense row tiles for clustered B (and a sparse Hessian).  have_dict = false
// when a single row is too wide.  probe = true (AUTO selection): give up when
// the first 64k rows tile sparsely (random B: a tile is ~3 % nonzeros, and the
// full dense-tile copy would be ~16 GB on cfg5 only to be rejected)
static int build_dict(qpk_ctx* c, bool probe) {
  c->have_dict = false;
  c->h_tiled = false;
  const long long n = c->n, m = c->m;
  std::vector<TileDescD> tiles;
  std::vector<int> cols;
  std::vector<double> tval;
  if (probe && m > 65536) {
    TileOut o;
    std::vector<int> mark(n, 0);
    int stamp = 0;
    tile_range(c->h_rp.data(), c->h_ci.data(), c->h_v.data(), nullptr, 0, 65536, 0, mark, stamp, o);
    if (o.too_wide) return QPK_OK;
    if ((double)c->h_rp[65536] < 0.3 * (double)o.slots) {
      c->dict_reuse = (double)c->h_rp[65536] / (double)o.slots;       // estimate from the probed rows
      return QPK_OK;
    }
  }
  auto tile_rows = [&](const int* rp, const int* ci, const double* v, long long nrows, int kind,
                       const int* perm) -> long long {
    return tile_rows_parallel(rp, ci, v, perm, nrows, kind, n, tiles, cols, tval,
                              kind == 0 && c->hkind == QPK_HESS_CSR ? 2 * c->h_hci.size() + 65536 : 0);
  };
  SetupTimer tm;
  const long long slots = tile_rows(c->h_rp.data(), c->h_ci.data(), c->h_v.data(), m, 0, nullptr);
  if (slots < 0) return QPK_OK;                       // a row wider than a tile
  tm.lap("  B tiles");
  int tid = (int)tiles.size();
  const size_t n_bcols = cols.size();
  const int n_btiles = tid;
  // the sparse Hessian's rows as dense tiles too (top-block rows, no B'z part),
  // when they are dense enough.  Sharded: every rank takes a contiguous,
  // nnz-balanced slice of the tile-row sequence (the decision to tile is taken
  // on the whole H, so all ranks agree; H is replicated and small next to B)
  if (c->hkind == QPK_HESS_CSR && !c->h_hci.empty()) {
    const size_t t0 = tiles.size(), c0 = cols.size(), v0 = tval.size();
    // rows in reverse Cuthill-McKee order: a Hessian like D_t'D_t of randomly
    // numbered band columns is banded in that order, so consecutive rows share
    // their columns and the tiles come out dense (tile row q is H row hperm[q])
    std::vector<int> hperm = rcm_order(n, c->h_hrp, c->h_hci);
    // empty rows (columns that never meet the objective block) need no tile
    hperm.erase(std::remove_if(hperm.begin(), hperm.end(),
                               [&](int j) { return c->h_hrp[j + 1] == c->h_hrp[j]; }), hperm.end());
    long long hs = tile_rows(c->h_hrp.data(), c->h_hci.data(), c->h_hv.data(), (long long)hperm.size(), 1,
                             hperm.data());
    const bool tile_h = hs > 0 && (double)c->h_hci.size() / (double)hs >= 0.5;
    if (tile_h && c->h_own_set) {
      // keep only the rows this rank applies (its slice of the same sequence), re-tiled on their own
      tiles.resize(t0); cols.resize(c0); tval.resize(v0); tid = n_btiles;
      hperm = c->h_own;
      if (!hperm.empty())
        hs = tile_rows(c->h_hrp.data(), c->h_hci.data(), c->h_hv.data(), (long long)hperm.size(), 1, hperm.data());
    }
    if (tile_h) {
      c->h_tiled = true;
      hperm.resize(hperm.size() + 4, 0);               // the tile kernel bulk-copies 16-byte windows
      CUDA_TRY(upload(c->hperm, hperm, c->stream));
    } else {
      tiles.resize(t0); cols.resize(c0); tval.resize(v0); tid = n_btiles;
    }
  }
  tid = (int)tiles.size();
  tm.lap("  H tiles");
  // column -> its B-tile-partial positions, in tile order
  std::vector<int> col_ptr(n + 1, 0), col_pos;
  for (size_t p = 0; p < n_bcols; ++p) if (cols[p] >= 0) col_ptr[cols[p] + 1]++;
  for (long long j = 0; j < n; ++j) col_ptr[j + 1] += col_ptr[j];
  col_pos.resize(col_ptr[n]);
  {
    std::vector<int> at(col_ptr.begin(), col_ptr.end() - 1);
    for (size_t p = 0; p < n_bcols; ++p) if (cols[p] >= 0) col_pos[at[cols[p]]++] = (int)p;
  }
  {
    // combine segments: each column's partial list in chunks of <= QPK_COMB_CHUNK
    std::vector<int> cseg(n + 1, 0), cbeg;
    for (long long j = 0; j < n; ++j) {
      cseg[j] = (int)cbeg.size();
      for (int b = col_ptr[j]; b < col_ptr[j + 1]; b += QPK_COMB_CHUNK) cbeg.push_back(b);
    }
    cseg[n] = (int)cbeg.size();
    cbeg.push_back(col_ptr[n]);
    c->comb_nseg = cseg[n];
    const long long avg = (long long)col_pos.size() / std::max<long long>(c->comb_nseg, 1);
    c->comb_lanes = pow2_clamp((avg + 3) / 4, 1, 32);
    CUDA_TRY(upload(c->comb_col, cseg, c->stream));
    CUDA_TRY(upload(c->comb_beg, cbeg, c->stream));
    CUDA_TRY(c->comb_sum.alloc(std::max(c->comb_nseg, 1)));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  tm.lap("  col index");
  // CTA-level accumulation: CTA b runs a consecutive, slot-balanced range of
  // tiles and sums their partials per column of the range's union in shared
  // memory; the combine then reads ~one partial per (CTA, column)
  c->cacc = false;
  if (!getenv("QPK_NO_CACC")) {
    int G = std::max(1, std::min(c->sms, tid));
    // test switch: fewer CTAs -> long per-CTA tile streams on small problems
    // (ring-stage reuse, descriptor refill, L2 prefetch; tests/test_gpu_fullscale.py)
    if (const char* ev = getenv("QPK_TILE_GRID")) G = std::max(1, std::min(G, atoi(ev)));
    // weight = dense slots + a fixed per-tile cost (barriers, copies) of ~2k slots
    auto weight = [&](int t) { return (long long)(tiles[t].rb - tiles[t].ra) * tiles[t].pad0 + 2048; };
    auto split = [&](int t0, int t1, std::vector<int>& beg) {        // [t0, t1) into G weight-balanced runs
      std::vector<long long> pre(t1 - t0 + 1, 0);
      for (int t = t0; t < t1; ++t) pre[t - t0 + 1] = pre[t - t0] + weight(t);
      beg.assign(G + 1, t0);
      for (int b = 1; b < G; ++b)
        beg[b] = t0 + (int)(std::lower_bound(pre.begin(), pre.end(), pre.back() * b / G) - pre.begin());
      beg[G] = t1;
      for (int b = 1; b <= G; ++b) beg[b] = std::max(beg[b], beg[b - 1]);
    };
    std::vector<int> tbeg(G + 1, 0);
    if (n_btiles < tid && !getenv("QPK_TILE_NO_HSPREAD")) {
      // Hessian tiles (they write y directly and use no accumulator slots, so
      // any CTA may run them) are spread over the CTAs: CTA b runs its run of
      // B tiles, then its run of Hessian tiles -- B work and H work are each
      // balanced, instead of the last few CTAs running Hessian tiles only
      std::vector<int> bb, hb;
      split(0, n_btiles, bb);
      split(n_btiles, tid, hb);
      std::vector<TileDescD> re;
      re.reserve(tiles.size());
      for (int b = 0; b < G; ++b) {
        tbeg[b] = (int)re.size();
        re.insert(re.end(), tiles.begin() + bb[b], tiles.begin() + bb[b + 1]);
        re.insert(re.end(), tiles.begin() + hb[b], tiles.begin() + hb[b + 1]);
      }
      tbeg[G] = (int)re.size();
      tiles.swap(re);
    } else {
      split(0, tid, tbeg);
    }
    std::vector<int> seen(n, -1), slot_of(n, 0), off(G + 1, 0), ucols, tsl(cols.size(), -1);
    bool ok = true;
    for (int b = 0; b < G && ok; ++b) {
      int cnt = 0;
      for (int t = tbeg[b]; t < tbeg[b + 1]; ++t) {
        if (tiles[t].pad1) continue;                      // Hessian tiles write y directly
        for (int cc = 0; cc < tiles[t].ndp; ++cc) {
          const int col = cols[tiles[t].d0 + cc];
          if (col < 0) continue;
          if (seen[col] != b) { seen[col] = b; slot_of[col] = cnt++; ucols.push_back(col); }
          tsl[tiles[t].d0 + cc] = slot_of[col];
        }
      }
      if (cnt > QPK_TILE_UMAX) ok = false;
      off[b + 1] = off[b] + cnt;
    }
    if (ok) {
      // column j -> its CTA partial positions, in CTA order
      std::vector<int> cp2(n + 1, 0), cpos2((size_t)off[G]);
      for (int col : ucols) cp2[col + 1]++;
      for (long long j = 0; j < n; ++j) cp2[j + 1] += cp2[j];
      std::vector<int> at(cp2.begin(), cp2.end() - 1);
      for (int q = 0; q < off[G]; ++q) cpos2[at[ucols[q]]++] = q;
      c->comb_max2 = 0;
      for (long long j = 0; j < n; ++j) c->comb_max2 = std::max(c->comb_max2, cp2[j + 1] - cp2[j]);
      std::vector<int> cseg(n + 1, 0), cbeg;
      for (long long j = 0; j < n; ++j) {
        cseg[j] = (int)cbeg.size();
        for (int b = cp2[j]; b < cp2[j + 1]; b += QPK_COMB_CHUNK) cbeg.push_back(b);
      }
      cseg[n] = (int)cbeg.size();
      cbeg.push_back(cp2[n]);
      c->comb_nseg2 = cseg[n];
      const long long avg = (long long)cpos2.size() / std::max<long long>(c->comb_nseg2, 1);
      c->comb_lanes2 = pow2_clamp((avg + 3) / 4, 1, 32);
      tsl.resize(tsl.size() + 16, -1);
      CUDA_TRY(upload(c->tile_beg, tbeg, c->stream));
      CUDA_TRY(upload(c->cta_off, off, c->stream));
      CUDA_TRY(upload(c->tslot, tsl, c->stream));
      CUDA_TRY(upload(c->col_ptr2, cp2, c->stream));
      CUDA_TRY(upload(c->col_pos2, cpos2, c->stream));
      CUDA_TRY(upload(c->comb_col2, cseg, c->stream));
      CUDA_TRY(upload(c->comb_beg2, cbeg, c->stream));
      CUDA_TRY(c->cpart.alloc(std::max(off[G], 1)));
      CUDA_TRY(c->comb_sum.alloc(std::max(std::max(c->comb_nseg, c->comb_nseg2), 1)));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      c->cacc = true;
      c->tile_grid = G;
    }
  }
  tm.lap("  CTA slots");
  cols.resize(cols.size() + 16, -1);                  // bulk copies read 16-byte windows
  tval.resize(tval.size() + 16, 0.0);
  cudaStream_t s = c->stream;
  CUDA_TRY(upload(c->tiles, tiles, s));
  CUDA_TRY(upload(c->dcols, cols, s));
  CUDA_TRY(upload(c->tval, tval, s));
  CUDA_TRY(upload(c->col_ptr, col_ptr, s));
  CUDA_TRY(upload(c->col_pos, col_pos, s));
  CUDA_TRY(c->bpart.alloc(std::max<size_t>(cols.size(), 1)));
  CUDA_TRY(cudaStreamSynchronize(s));
  tm.lap("  tile upload");
  c->nblk = tid;
  c->dict_reuse = slots ? (double)c->nnz / (double)slots : 0.0;
  c->have_dict = true;
  return QPK_OK;
}

// Dense column panel: the columns present in at least half of the rows,
// stored as a dense row-major m x kp block (kp = 64 Q); every row's other
// entries as an ELL strip of width ew <= 32, plus their CSC (Jacobi, and B'z
// when a remainder column has several entries).  Chosen when the panel holds
// >= 70 % of the nonzeros (the SVM primal: [diag(y)X, y | I]).
static int build_panel(qpk_ctx* c, bool force) {
  c->have_panel = false;
  const long long n = c->n, m = c->m;
  if (m == 0 || n == 0) return QPK_OK;
  std::vector<long long> cnt(n, 0);
  for (int col : c->h_ci) if (col >= 0) cnt[col]++;
  std::vector<int> pos(n, -1), pcols;
  long long pnnz = 0;
  for (long long j = 0; j < n; ++j)
    if (cnt[j] > 0 && 2 * cnt[j] >= m) { pos[j] = (int)pcols.size(); pcols.push_back((int)j); pnnz += cnt[j]; }
  const long long kd = (long long)pcols.size();
  if (kd == 0 || (!force && (kd < 32 || 10 * pnnz < 7 * c->nnz))) return QPK_OK;
  int Q = 0;
  for (int q : kPanelQ) if (64LL * q >= kd) { Q = q; break; }
  if (!Q) return QPK_OK;
  const int kp = 64 * Q;
  // remainder: row widths and per-column counts
  int ew = 0;
  std::vector<int> rcnt(n, 0);
  for (long long r = 0; r < m; ++r) {
    int w = 0;
    for (int k = c->h_rp[r]; k < c->h_rp[r + 1]; ++k) {
      const int col = c->h_ci[k];
      if (col >= 0 && pos[col] < 0) { ++w; ++rcnt[col]; }
    }
    ew = std::max(ew, w);
  }
  if (ew > 32 || panel_smem_bytes(kp, ew) > 220 * 1024) return QPK_OK;
  size_t fr = 0, tot = 0;
  CUDA_TRY(cudaMemGetInfo(&fr, &tot));
  if ((double)m * kp * 8.0 > 0.4 * (double)fr) return QPK_OK;
  bool direct = true;
  for (long long j = 0; j < n; ++j) if (rcnt[j] > 1) { direct = false; break; }
  const int ewa = std::max(ew, 1);
  std::vector<double> P((size_t)m * kp, 0.0), ev((size_t)m * ewa, 0.0);
  std::vector<int> eci((size_t)m * ewa, -1);
  std::vector<int> rrp(m + 1, 0), rci;
  std::vector<double> rv;
  for (long long r = 0; r < m; ++r) {
    int w = 0;
    for (int k = c->h_rp[r]; k < c->h_rp[r + 1]; ++k) {
      const int col = c->h_ci[k];
      if (col < 0) continue;
      if (pos[col] >= 0) {
        P[(size_t)r * kp + pos[col]] = c->h_v[k];
      } else {
        eci[(size_t)r * ewa + w] = col;
        ev[(size_t)r * ewa + w] = c->h_v[k];
        ++w;
        rci.push_back(col);
        rv.push_back(c->h_v[k]);
      }
    }
    rrp[r + 1] = (int)rci.size();
  }
  pcols.resize(kp, -1);
  ev.resize(ev.size() + 8, 0.0);                  // bulk copies read 16-byte windows
  eci.resize(eci.size() + 8, -1);
  std::vector<int> cpos;
  if (direct) {
    cpos.assign(n, -1);
    for (size_t p = 0; p < (size_t)m * ewa; ++p) if (eci[p] >= 0) cpos[eci[p]] = (int)p;
  }
  cudaStream_t s = c->stream;
  if (direct && ew > 0) {
    CUDA_TRY(upload(c->panel_cpos, cpos, s));
    CUDA_TRY(c->panel_ue.alloc((size_t)m * ewa + 8));
    CUDA_TRY(c->panel_yrem.alloc((size_t)m * ewa + 8));
    CUDA_TRY(cudaMemsetAsync(c->panel_ue.p, 0, ((size_t)m * ewa + 8) * sizeof(double), s));
  }
  CUDA_TRY(upload(c->panel_P, P, s));
  CUDA_TRY(upload(c->panel_cols, pcols, s));
  CUDA_TRY(upload(c->panel_eci, eci, s));
  CUDA_TRY(upload(c->panel_ev, ev, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  int rc = build_csc(c, rrp, rci, rv);        // the remainder's CSC (Jacobi; B'z when not direct)
  if (rc) return rc;
  c->panel_kp = kp;
  c->panel_q = Q;
  c->panel_ew = ew;
  c->panel_kd = (int)kd;
  c->panel_direct = direct ? 1 : 0;
  c->have_panel = true;
  return QPK_OK;
}

// Small systems: split B's rows and H's rows over C CTAs of one cluster and
// pack each CTA's slice (CSR + CSC of its B rows, CSR of its H rows) into a
// blob the kernel copies to shared memory.  Eligible when every slice fits
// (QPK_CL_SMEM) and H is diagonal, sparse or dense.
static int build_cluster(qpk_ctx* c) {
  c->cl_C = 0;
  if (getenv("QPK_NO_CLUSTER") || c->sharded || c->hkind == QPK_HESS_LOWRANK) return QPK_OK;
  const long long n = c->n, m = c->m;
  if (n > 16384 || (long long)c->h_ci.size() > 4000000) return QPK_OK;
  if (c->hkind == QPK_HESS_DENSE && c->h_dense.size() != (size_t)(n * n)) return QPK_OK;   // device-given H
  // H as full CSR rows
  std::vector<int> hrp(n + 1, 0), hci;
  std::vector<double> hv;
  if (c->hkind == QPK_HESS_DIAG) {
    for (long long j = 0; j < n; ++j) { hci.push_back((int)j); hv.push_back(c->h_h[j]); hrp[j + 1] = (int)hci.size(); }
  } else if (c->hkind == QPK_HESS_DENSE) {
    for (long long j = 0; j < n; ++j) {
      for (long long k = 0; k < n; ++k) { hci.push_back((int)k); hv.push_back(c->h_dense[j * n + k]); }
      hrp[j + 1] = (int)hci.size();
    }
  } else {
    hrp = c->h_hrp; hci = c->h_hci; hv = c->h_hv;
  }
  auto align16 = [](size_t b) { return (b + 15) & ~(size_t)15; };
  int C = m >= 128 ? 16 : std::max(2, pow2_clamp((m + 7) / 8, 2, 16));
  for (; C <= QPK_CL_MAXC; C *= 2) {
    // contiguous splits balanced by nonzeros (B rows) and by nonzeros (H rows)
    std::vector<int> rsp(C + 1, 0), hsp(C + 1, 0);
    const long long nzb = c->h_rp[m];
    for (int k = 1; k < C; ++k) {
      long long target = nzb * k / C;
      rsp[k] = (int)(std::lower_bound(c->h_rp.begin(), c->h_rp.begin() + m + 1, (int)target) - c->h_rp.begin());
      rsp[k] = std::max(rsp[k], rsp[k - 1]);
      const long long nzh = hrp[n];
      target = nzh * k / C;
      hsp[k] = (int)(std::lower_bound(hrp.begin(), hrp.end(), (int)target) - hrp.begin());
      hsp[k] = std::max(hsp[k], hsp[k - 1]);
    }
    rsp[C] = (int)m; hsp[C] = (int)n;
    std::vector<ClCta> ctas(C);
    std::vector<unsigned char> blob;
    std::vector<long long> off(C);
    size_t worst = 0;
    for (int k = 0; k < C; ++k) {
      ClCta& t = ctas[k];
      t.r0 = rsp[k]; t.r1 = rsp[k + 1]; t.h0 = hsp[k]; t.h1 = hsp[k + 1];
      const int mr = t.r1 - t.r0, nh = t.h1 - t.h0;
      // B slice CSR (skip the padding entries of the padded CSR)
      std::vector<int> brp(mr + 1, 0), bci, ccp(n + 1, 0), cri;
      std::vector<double> bv, cv;
      for (int r = t.r0; r < t.r1; ++r) {
        for (int q = c->h_rp[r]; q < c->h_rp[r + 1]; ++q)
          if (c->h_ci[q] >= 0) { bci.push_back(c->h_ci[q]); bv.push_back(c->h_v[q]); }
        brp[r - t.r0 + 1] = (int)bci.size();
      }
      for (int col : bci) ccp[col + 1]++;
      for (long long j = 0; j < n; ++j) ccp[j + 1] += ccp[j];
      cri.resize(bci.size()); cv.resize(bci.size());
      {
        std::vector<int> at(ccp.begin(), ccp.end() - 1);
        for (int rr = 0; rr < mr; ++rr)
          for (int q = brp[rr]; q < brp[rr + 1]; ++q) { const int a = at[bci[q]]++; cri[a] = rr; cv[a] = bv[q]; }
      }
      const int nnzh = hrp[t.h1] - hrp[t.h0];
      std::vector<int> lhrp(nh + 1);
      for (int j = 0; j <= nh; ++j) lhrp[j] = hrp[t.h0 + j] - hrp[t.h0];
      t.nnzb = (int)bci.size(); t.nnzh = nnzh;
      size_t o = 0;
      auto place = [&](size_t bytes) { const size_t at = o; o = align16(o + bytes); return (int)at; };
      t.o_brp = place((mr + 1) * 4); t.o_bci = place(bci.size() * 4); t.o_bv = place(bv.size() * 8);
      t.o_ccp = place((n + 1) * 4); t.o_cri = place(cri.size() * 4); t.o_cv = place(cv.size() * 8);
      t.o_hrp = place((nh + 1) * 4); t.o_hci = place((size_t)nnzh * 4); t.o_hv = place((size_t)nnzh * 8);
      t.bytes = (int)align16(o); t.pad = 0;
      const size_t need = cl_layout((int)n, mr, nh, t.bytes).bytes;
      worst = std::max(worst, need);
      if (need > QPK_CL_SMEM) break;
      off[k] = (long long)blob.size();
      blob.resize(blob.size() + t.bytes, 0);
      unsigned char* b = blob.data() + off[k];
      auto put = [&](int at, const void* src, size_t bytes) { if (bytes) memcpy(b + at, src, bytes); };
      put(t.o_brp, brp.data(), brp.size() * 4); put(t.o_bci, bci.data(), bci.size() * 4);
      put(t.o_bv, bv.data(), bv.size() * 8); put(t.o_ccp, ccp.data(), ccp.size() * 4);
      put(t.o_cri, cri.data(), cri.size() * 4); put(t.o_cv, cv.data(), cv.size() * 8);
      put(t.o_hrp, lhrp.data(), lhrp.size() * 4); put(t.o_hci, hci.data() + hrp[t.h0], (size_t)nnzh * 4);
      put(t.o_hv, hv.data() + hrp[t.h0], (size_t)nnzh * 8);
    }
    if (worst > QPK_CL_SMEM) continue;
    // can the device co-schedule a cluster of C CTAs with this much shared memory?
    if (C > 8) cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, QPK_CL_SMEM);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(C); lc.blockDim = dim3(QPK_CL_THREADS); lc.dynamicSmemBytes = worst;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (void*)k_pcg_cluster, &lc) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      return QPK_OK;                                   // larger clusters will not fit either
    }
    blob.resize(blob.size() + 16, 0);
    CUDA_TRY(upload(c->cl_ctas, ctas, c->stream));
    CUDA_TRY(upload(c->cl_blob, blob, c->stream));
    CUDA_TRY(upload(c->cl_off, off, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->cl_C = C;
    c->cl_smem = worst;
    return QPK_OK;
  }
  return QPK_OK;
}

// QPK_TIMING=1: host setup phases of qpk_problem_finalize on stderr
static int allreduce_sum(qpk_ctx* c, double* buf, size_t count, cudaStream_t s);

int qpk_problem_finalize(qpk_ctx* c, int scatter) {
  SetupTimer tm;
  if (!c || !c->building) return fail(QPK_E_STATE, "qpk_problem_finalize: no problem being built");
  const long long mB = c->m_e + c->m_l + c->m_u;
  if (c->m != mB) return fail(QPK_E_ARG, "qpk_problem_finalize: %lld rows added, m_B=%lld", c->m, mB);
  if (c->hkind < 0) return fail(QPK_E_STATE, "qpk_problem_finalize: Hessian not set");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  // pad: the TMA tiles read aligned windows that may extend past the end
  CUDA_TRY(upload_padded(c->rp, c->h_rp, 16, c->h_rp.back(), s));
  CUDA_TRY(upload_padded(c->ci, c->h_ci, 32, -1, s));
  CUDA_TRY(upload_padded(c->bv, c->h_v, 32, 0.0, s));
  if (c->hkind == QPK_HESS_DIAG || c->hkind == QPK_HESS_LOWRANK) CUDA_TRY(upload(c->hh, c->h_h, s));
  if (c->hkind == QPK_HESS_CSR) {
    CUDA_TRY(upload(c->hrp, c->h_hrp, s));
    CUDA_TRY(upload(c->hci, c->h_hci, s));
    CUDA_TRY(upload(c->hv, c->h_hv, s));
  }
  if (c->hkind == QPK_HESS_DENSE && c->h_dense_dev) {
    CUDA_TRY(c->hdense.alloc((size_t)c->n * c->n));
    CUDA_TRY(cudaMemcpyAsync(c->hdense.p, c->h_dense_dev, (size_t)c->n * c->n * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
    c->h_dense_dev = nullptr;
  } else if (c->hkind == QPK_HESS_DENSE) {
    CUDA_TRY(upload(c->hdense, c->h_dense, s));
  }
  if (c->hkind == QPK_HESS_LOWRANK) {
    CUDA_TRY(upload(c->U, c->h_U, s));
    CUDA_TRY(upload(c->w, c->h_w, s));
  }
  const long long N = c->N();
  CUDA_TRY(c->hdiag.alloc(c->n));
  CUDA_TRY(c->d.alloc(c->m + 8));
  CUDA_TRY(c->q.alloc(c->n));
  CUDA_TRY(c->jac.alloc(N));
  CUDA_TRY(c->minv.alloc(N));
  for (auto& b : c->x) CUDA_TRY(b.alloc(N + 8));
  CUDA_TRY(c->r.alloc(N + 8));
  CUDA_TRY(c->p.alloc(N + 8));
  CUDA_TRY(c->y.alloc(N + 8));
  CUDA_TRY(c->rhs.alloc(N + 8));
  CUDA_TRY(c->vin.alloc(N + 8));
  CUDA_TRY(c->zb.alloc(std::max<long long>(c->m, 1)));

  tm.lap("upload");
  // lanes per row: ~3 chunks of 4 nonzeros per lane keeps several gathers in flight
  c->lanes = pow2_clamp((c->nnz + std::max<long long>(c->m, 1) - 1) / std::max<long long>(c->m, 1) / 12, 4, 32);
  if (const char* ev = getenv("QPK_LANES")) c->lanes = pow2_clamp(atoi(ev), 1, 32);
  // B'z strategy.  AUTO: the row-block dictionary when blocks reuse their
  // columns (banded / clustered B: RT, SVM, dense), else one-pass atomics
  // (random B, where no blocking creates reuse).  CSC and DICT are
  // deterministic; DICT falls back to CSC when a row is wider than a dictionary.
  if (const char* ev = getenv("QPK_SCATTER")) if (scatter == QPK_SCATTER_AUTO) scatter = atoi(ev);
  // Sharded, sparse H: H is replicated; rank r applies a contiguous, nnz-balanced
  // slice of its non-empty rows in reverse Cuthill-McKee order (the order the
  // Hessian tiles use), whatever apply format each rank ends up with
  c->h_own_set = false;
  c->h_own.clear();
  if (c->world > 1 && c->hkind == QPK_HESS_CSR) {
    std::vector<int> seq = rcm_order(c->n, c->h_hrp, c->h_hci);
    seq.erase(std::remove_if(seq.begin(), seq.end(), [&](int j) { return c->h_hrp[j + 1] == c->h_hrp[j]; }), seq.end());
    std::vector<long long> pre(seq.size() + 1, 0);
    for (size_t q = 0; q < seq.size(); ++q) pre[q + 1] = pre[q] + (c->h_hrp[seq[q] + 1] - c->h_hrp[seq[q]]);
    auto cut = [&](int r) {
      return (size_t)(std::lower_bound(pre.begin(), pre.end(), pre.back() * r / c->world) - pre.begin());
    };
    const size_t q_lo = c->rank == 0 ? 0 : cut(c->rank);
    const size_t q_hi = c->rank == c->world - 1 ? seq.size() : cut(c->rank + 1);
    c->h_own.assign(seq.begin() + q_lo, seq.begin() + std::max(q_lo, q_hi));
    c->h_own_set = true;
    std::vector<int> up = c->h_own;
    up.resize(up.size() + 4, 0);
    CUDA_TRY(upload(c->hown, up, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  c->scatter = QPK_SCATTER_ATOMIC;
  // a dense column panel (large systems in AUTO) comes first
  if (c->m > 0 && (scatter == QPK_SCATTER_PANEL || (scatter == QPK_SCATTER_AUTO && c->N() >= 50000))) {
    tm.lap("row tiles");
    int rc = build_panel(c, scatter == QPK_SCATTER_PANEL);
    if (rc) return rc;
    tm.lap("panel");
    if (c->have_panel) scatter = QPK_SCATTER_PANEL;
    else if (scatter == QPK_SCATTER_PANEL) scatter = QPK_SCATTER_CSC;     // no panel structure
  }
  if (scatter == QPK_SCATTER_PANEL) {
    c->scatter = QPK_SCATTER_PANEL;
  } else if ((scatter == QPK_SCATTER_AUTO || scatter == QPK_SCATTER_DICT) && c->m > 0) {
    tm.lap("pre-dict");
    int rc = build_dict(c, scatter == QPK_SCATTER_AUTO);
    if (rc) return rc;
    tm.lap("dict");
    // Dense tiles pay off when they are mostly nonzeros (banded / clustered
    // B: RT, SVM, dense).  Such B makes fp64 atomics contend, so small
    // systems of that kind take the CSC gather (in the single-launch
    // persistent kernel) instead; random B (cfg5) keeps the one-pass atomics.
    const bool dense_tiles = c->have_dict && c->dict_reuse >= 0.5;
    if (c->have_dict && (scatter == QPK_SCATTER_DICT || (dense_tiles && c->N() >= 50000)))
      c->scatter = QPK_SCATTER_DICT;
    else if (scatter == QPK_SCATTER_DICT || dense_tiles)
      scatter = QPK_SCATTER_CSC;
  }
  if (scatter == QPK_SCATTER_CSC && c->m > 0) {
    int rc = build_csc(c, c->h_rp, c->h_ci, c->h_v);
    if (rc) return rc;
    c->scatter = QPK_SCATTER_CSC;
    tm.lap("csc");
  }

  // grid sizes: persistent kernel = all co-resident blocks (capped by work)
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, pcg_kernel_for(c->lanes, c->scatter == QPK_SCATTER_CSC), QPK_BLOCK, 0));
  if (per_sm < 1) return fail(QPK_E_UNSUPPORTED, "PCG kernel cannot be resident");
  const long long work = std::max<long long>((long long)c->h_ci.size() / 1024, N / 512);
  c->grid_pcg = (int)std::max<long long>(1, std::min<long long>((long long)per_sm * c->sms, work));
  if (const char* ev = getenv("QPK_GRID")) c->grid_pcg = std::max(1, std::min(per_sm * c->sms, atoi(ev)));
  c->grid_std = c->grid_pcg;
  {
    int eng_per_sm = c->scatter == QPK_SCATTER_DICT ? 3 : 4;
    long long ework = std::max<long long>((long long)c->h_ci.size() / 512, N / 256);
    // panel mode: the engine grid only runs the vector kernels (top, update),
    // which are latency-bound -- fewer, fuller blocks
    if (c->scatter == QPK_SCATTER_PANEL) ework = std::max<long long>(2 * c->sms, N / 1024);
    if (const char* ev = getenv("QPK_ENGINE_GRID")) ework = atoi(ev);
    c->grid_eng = (int)std::max<long long>(1, std::min<long long>((long long)eng_per_sm * c->sms, ework));
    // the partial-sum stride E.G must cover every kernel's blocks (tile CTAs included)
    if (c->scatter == QPK_SCATTER_DICT && c->cacc) c->grid_eng = std::max(c->grid_eng, c->tile_grid);
    if (c->sharded) c->grid_eng = std::max(c->grid_eng, QPK_FOLD_BLOCKS);   // the folded slot's fixed top geometry
  }
  if (c->scatter == QPK_SCATTER_PANEL) {
    c->panel_grid = std::max(1, std::min(c->sms, c->grid_eng));      // one CTA per SM
    CUDA_TRY(c->panel_part.alloc((size_t)c->panel_grid * c->panel_kp));
  }
  CUDA_TRY(c->part.alloc((size_t)NSLOTS * std::max(c->grid_pcg, c->grid_eng)));
  if (c->graph) { cudaGraphExecDestroy(c->graph); c->graph = nullptr; }

  {
    int rc = build_cluster(c);
    if (rc) return rc;
  }
  // large dense H (the SVM dual's Gram Hessian): keep its upper tiles packed,
  // half the bytes per apply (hess_sym); the row-major copy stays for diag(H)
  c->h_nchunks = 0;
  if (c->hkind == QPK_HESS_DENSE && c->cl_C == 0 && !c->sharded && c->n >= QPK_SYM_MIN_N && !getenv("QPK_NO_SYM")) {
    const int nt = (int)((c->n + 63) / 64);
    // only a bitwise symmetric H may be packed; any other DenseHessian keeps
    // the row-major apply (h.m @ v for whatever m is, as the reference)
    DBuf<int> bad;
    CUDA_TRY(bad.alloc(1));
    CUDA_TRY(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    k_sym_check<<<dim3(nt, nt), 256, 0, s>>>(c->hdense.p, c->n, bad.p);
    c->launches++;
    int h_bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->h_symmetric = h_bad == 0;
  }
  if (c->hkind == QPK_HESS_DENSE && c->cl_C == 0 && !c->sharded && c->n >= QPK_SYM_MIN_N && !getenv("QPK_NO_SYM") &&
      c->h_symmetric) {
    const int nt = (int)((c->n + 63) / 64);
    const size_t tiles = (size_t)nt * (nt + 1) / 2;
    CUDA_TRY(c->hsym.alloc(tiles * 4096));
    k_pack_sym<<<dim3(nt, nt), 256, 0, s>>>(c->hdense.p, c->n, nt, c->hsym.p);
    c->launches++;
    std::vector<int4> ch;
    std::vector<int> rowchunk(nt + 1, 0);
    for (int I = 0; I < nt; ++I) {
      const int base = (int)((size_t)I * nt - (size_t)I * (I - 1) / 2);
      rowchunk[I] = (int)ch.size();
      for (int J0 = I; J0 < nt; J0 += QPK_SYM_CHUNK)
        ch.push_back(make_int4(I, J0, std::min(J0 + QPK_SYM_CHUNK, nt), base + (J0 - I)));
    }
    rowchunk[nt] = (int)ch.size();
    CUDA_TRY(upload(c->hchunks, ch, s));
    CUDA_TRY(upload(c->hrowchunk, rowchunk, s));
    CUDA_TRY(c->hsymp.alloc((ch.size() + tiles) * 64));
    c->h_nchunks = (int)ch.size();
  }
  // leading dense rows of B (the SVM dual's y' alpha = 0): as dense vectors,
  // applied outside the row pass by the slot engine (one warp per row would
  // serialise n entries)
  c->n_dense = 0;
  if (!c->sharded && !getenv("QPK_NO_DENSE_ROWS") &&
      (c->scatter == QPK_SCATTER_ATOMIC || c->scatter == QPK_SCATTER_CSC)) {
    const long long thr = std::max<long long>(QPK_DENSE_ROW_MIN, c->n / 4);
    int k = 0;
    while (k < QPK_DENSE_ROWS_MAX && k < c->m && c->h_rp[k + 1] - c->h_rp[k] >= thr) ++k;
    if (k > 0) {
      std::vector<double> cd((size_t)k * c->n, 0.0);
      for (int r = 0; r < k; ++r)
        for (int e = c->h_rp[r]; e < c->h_rp[r + 1]; ++e)
          if (c->h_ci[e] >= 0) cd[(size_t)r * c->n + c->h_ci[e]] = c->h_v[e];
      CUDA_TRY(upload(c->cdense, cd, s));
      c->n_dense = k;
    }
  }
  Op o = c->op();
  k_hdiag<<<std::max(1, std::min(c->sms * 4, (int)((c->n + 255) / 256))), 256, 0, s>>>(o.H, (int)c->n, c->hdiag.p);
  c->launches++;
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(s));
  // host staging no longer needed
  std::vector<int>().swap(c->h_ci);
  std::vector<double>().swap(c->h_v);
  std::vector<int>().swap(c->h_rp);
  std::vector<double>().swap(c->h_dense);
  std::vector<double>().swap(c->h_U);
  std::vector<int>().swap(c->h_hci);
  std::vector<double>().swap(c->h_hv);
  c->building = false;
  c->finalized = true;
  // Sharded: the ranks must agree on the collectives a slot issues.  The folded
  // slot (one all-reduce of n + 10 values) needs the tile format with CTA
  // accumulation on EVERY rank; each rank picks its format from its own shard,
  // so the choice is settled by one all-reduce here.
  c->fold_all = false;
  if (c->sharded) {
    DBuf<double> flag;
    CUDA_TRY(flag.alloc(1));
    const double mine = (c->scatter == QPK_SCATTER_DICT && c->cacc) ? 1.0 : 0.0;
    CUDA_TRY(cudaMemcpyAsync(flag.p, &mine, sizeof mine, cudaMemcpyHostToDevice, s));
    int rcf = allreduce_sum(c, flag.p, 1, s);
    if (rcf) return rcf;
    double all = 0.0;
    CUDA_TRY(cudaMemcpyAsync(&all, flag.p, sizeof all, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->fold_all = all > c->world - 0.5;
  }
  tm.lap("finish");
  return QPK_OK;
}

static int set_diagonals(qpk_ctx* c, const double* dd, const double* qq, cudaMemcpyKind kind) {
  if (!c || !c->finalized) return fail(QPK_E_STATE, "qpk_set_diagonals: problem not finalized");
  if ((c->m && !dd) || !qq) return fail(QPK_E_ARG, "qpk_set_diagonals: null vector");
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->m) CUDA_TRY(cudaMemcpyAsync(c->d.p, dd, c->m * sizeof(double), kind, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->q.p, qq, c->n * sizeof(double), kind, c->stream));
  c->diag_set = true;
  c->jac_ready = false;
  return QPK_OK;
}

int qpk_set_diagonals(qpk_ctx* c, const double* dd, const double* qq) {
  return set_diagonals(c, dd, qq, cudaMemcpyHostToDevice);
}
int qpk_set_diagonals_dev(qpk_ctx* c, const double* dd, const double* qq) {
  return set_diagonals(c, dd, qq, cudaMemcpyDeviceToDevice);
}

// in-place sum over ranks on the context's stream (sharded mode only)
static int allreduce_sum(qpk_ctx* c, double* buf, size_t count, cudaStream_t s) {
  if (!c->sharded || count == 0) return QPK_OK;
  if (c->hostcomm) {
    HostComm* hc = c->hostcomm;
    std::vector<double>& mine = hc->bufs[c->rank];
    mine.resize(count);
    CUDA_TRY(cudaMemcpyAsync(mine.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (!hc->barrier()) return fail(QPK_E_STATE, "emulated all-reduce: a rank did not arrive");
    std::vector<double> sum(count, 0.0);
    for (int r = 0; r < hc->n; ++r) {
      if (hc->bufs[r].size() != count) return fail(QPK_E_STATE, "emulated all-reduce: ranks disagree on the count");
      for (size_t i = 0; i < count; ++i) sum[i] += hc->bufs[r][i];
    }
    if (!hc->barrier()) return fail(QPK_E_STATE, "emulated all-reduce: a rank did not arrive");   // all have read
    CUDA_TRY(cudaMemcpyAsync(buf, sum.data(), count * sizeof(double), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return QPK_OK;
  }
  const int rc = nccl().allReduce(buf, buf, count, NCCL_FLOAT64, NCCL_SUM, c->comm, s);
  if (rc != 0) return fail(QPK_E_CUDA, "ncclAllReduce failed: %s", nccl().errStr ? nccl().errStr(rc) : "?");
  return QPK_OK;
}

static int build_jacobi(qpk_ctx* c) {
  Op o = c->op();
  const int G = c->grid_std;
  cudaStream_t s = c->stream;
  if (c->scatter == QPK_SCATTER_PANEL) {
    // remainder columns through their CSC (writes every column, 0 for the
    // panel's), then the panel columns from the per-CTA partials
    int rc = engine_setup(c);
    if (rc) return rc;
    Engine E = make_engine(c);
    k_jac_cols<<<G, QPK_BLOCK, 0, s>>>(o, c->y.p);
    QPK_PANEL_DISPATCH(launch_jac_panel_t, c, s, E);
    k_panel_comb<<<c->panel_kp / 32, 1024, 0, s>>>(E, c->y.p, 1, -1);     // panel columns only
    int rc2 = allreduce_sum(c, c->y.p, c->n, s);
    if (rc2) return rc2;
    k_jac_finish<<<G, QPK_BLOCK, 0, s>>>(o, c->hdiag.p, c->y.p, c->jac.p, c->minv.p);
    c->launches += 4;
    CUDA_TRY(cudaGetLastError());
    c->jac_ready = true;
    return QPK_OK;
  }
  if (c->scatter == QPK_SCATTER_DICT) {
    int rc = engine_setup(c);
    if (rc) return rc;
    Engine E = make_engine(c);
    // per-tile partials (strided tiles) and their combine structures
    E.dict.cacc = 0;
    E.dict.col_ptr = c->col_ptr.p; E.dict.col_pos = c->col_pos.p;
    E.dict.comb_lanes = c->comb_lanes; E.dict.nseg = c->comb_nseg;
    E.dict.seg_beg = c->comb_beg.p; E.dict.col_seg = c->comb_col.p;
    k_jac_tile<<<c->grid_eng, QPK_BLOCK, 0, s>>>(E);
    // column sums of the tile partials (sharded: summed over ranks), then the common finish
    k_comb_seg<<<G, QPK_BLOCK, 0, s>>>(E, -1);
    k_comb_col<<<G, QPK_BLOCK, 0, s>>>(E, c->y.p, 0, -1);
    int rc2 = allreduce_sum(c, c->y.p, c->n, s);
    if (rc2) return rc2;
    k_jac_finish<<<G, QPK_BLOCK, 0, s>>>(o, c->hdiag.p, c->y.p, c->jac.p, c->minv.p);
    c->launches += 2;
    CUDA_TRY(cudaGetLastError());
    c->jac_ready = true;
    return QPK_OK;
  }
  CUDA_TRY(cudaMemsetAsync(c->y.p, 0, c->n * sizeof(double), s));
  if (c->m) {
    if (c->have_csc) k_jac_cols<<<G, QPK_BLOCK, 0, s>>>(o, c->y.p);
    else launch_jac_rows(c->lanes, G, s, o, c->y.p);
    c->launches++;
  }
  {
    int rc2 = allreduce_sum(c, c->y.p, c->n, s);       // sharded: sum the ranks' B^2/D partials
    if (rc2) return rc2;
  }
  k_jac_finish<<<G, QPK_BLOCK, 0, s>>>(o, c->hdiag.p, c->y.p, c->jac.p, c->minv.p);
  c->launches++;
  CUDA_TRY(cudaGetLastError());
  c->jac_ready = true;
  return QPK_OK;
}

int qpk_jacobi(qpk_ctx* c, double* diag_out) {
  if (!c || !c->diag_set) return fail(QPK_E_STATE, "qpk_jacobi: diagonals not set");
  CUDA_TRY(cudaSetDevice(c->device));
  int rc = build_jacobi(c);
  if (rc) return rc;
  if (diag_out) {
    CUDA_TRY(cudaMemcpyAsync(diag_out, c->jac.p, c->N() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return QPK_OK;
}

static int apply_engine(qpk_ctx* c, const double* v_dev, double* y_dev);

static int apply_impl(qpk_ctx* c, const double* v_dev, double* y_dev) {
  if (c->scatter == QPK_SCATTER_DICT || c->scatter == QPK_SCATTER_PANEL) return apply_engine(c, v_dev, y_dev);
  Op o = c->op();
  const int G = c->grid_std;
  cudaStream_t s = c->stream;
  const bool csc = c->scatter == QPK_SCATTER_CSC;
  k_prep<<<G, QPK_BLOCK, 0, s>>>(o, v_dev, y_dev, c->part.p, G);
  if (csc) launch_rows<true>(c->lanes, G, s, o, v_dev, y_dev, c->zb.p, c->part.p, G);
  else launch_rows<false>(c->lanes, G, s, o, v_dev, y_dev, c->zb.p, c->part.p, G);
  c->launches += 2;
  if (csc) { k_finish_csc<<<G, QPK_BLOCK, 0, s>>>(o, y_dev, c->zb.p); c->launches++; }
  if (c->h_nchunks) {
    k_hess<<<G, QPK_BLOCK, 0, s>>>(o, v_dev, y_dev, c->part.p, G);
    k_sym_combine<<<G, QPK_SYMC_BLOCK, 0, s>>>(o, v_dev, y_dev);
    c->launches += 2;
  }
  CUDA_TRY(cudaGetLastError());
  return allreduce_sum(c, y_dev, c->n, s);          // sharded: y_top = sum of the ranks' partials
}

int qpk_apply(qpk_ctx* c, const double* v, double* y) {
  if (!c || !c->diag_set) return fail(QPK_E_STATE, "qpk_apply: diagonals not set");
  if (!v || !y) return fail(QPK_E_ARG, "qpk_apply: null vector");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t bytes = c->N() * sizeof(double);
  CUDA_TRY(cudaMemcpyAsync(c->vin.p, v, bytes, cudaMemcpyHostToDevice, c->stream));
  int rc = apply_impl(c, c->vin.p, c->y.p);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(y, c->y.p, bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return QPK_OK;
}

// out = H v with the problem's Hessian (hessian_apply, model.py:165-176,
// without q_extra); dense and diagonal H
__global__ void k_diag_mul(const double* h, const double* v, double* out, long long n) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    out[j] = h[j] * v[j];
}

int qpk_hessian_apply_dev(qpk_ctx* c, const double* v, double* out) {
  if (!c || !c->finalized) return fail(QPK_E_STATE, "qpk_hessian_apply_dev: problem not finalized");
  if (!v || !out) return fail(QPK_E_ARG, "qpk_hessian_apply_dev: null vector");
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->hkind == QPK_HESS_DENSE) {
    k_dense_gemv<<<c->sms * 8, 256, 0, c->stream>>>(c->hdense.p, c->n, v, out);
  } else if (c->hkind == QPK_HESS_DIAG) {
    k_diag_mul<<<c->sms * 4, 256, 0, c->stream>>>(c->hh.p, v, out, c->n);
  } else {
    return fail(QPK_E_UNSUPPORTED, "qpk_hessian_apply_dev: dense and diagonal Hessians only");
  }
  c->launches++;
  CUDA_TRY(cudaGetLastError());
  return QPK_OK;
}

int qpk_dense_gemv_dev(qpk_ctx* c, const double* Hm, int64_t n, const double* v, double* out) {
  if (!c || !Hm || !v || !out || n < 1) return fail(QPK_E_ARG, "qpk_dense_gemv_dev: bad argument");
  CUDA_TRY(cudaSetDevice(c->device));
  k_dense_gemv<<<c->sms * 8, 256, 0, c->stream>>>(Hm, n, v, out);
  c->launches++;
  CUDA_TRY(cudaGetLastError());
  return QPK_OK;
}

int qpk_apply_dev(qpk_ctx* c, const double* v, double* y) {
  if (!c || !c->diag_set) return fail(QPK_E_STATE, "qpk_apply_dev: diagonals not set");
  if (!v || !y) return fail(QPK_E_ARG, "qpk_apply_dev: null vector");
  CUDA_TRY(cudaSetDevice(c->device));
  return apply_impl(c, v, y);
}

}  // extern "C"

// ------------------------------------------------------------ slot engine ---
template <int L, bool CSC>
static void launch_slot_rows_t(const qpk_ctx* c, int grid, cudaStream_t s, const Engine& E, int par) {
  k_slot_rows<L, CSC><<<grid, QPK_BLOCK, 0, s>>>(E, par);
}

// PDL on the tile / panel slot chains (top -> pass over B -> combine -> update)
static bool slot_pdl(const qpk_ctx* c) {
  const int env = getenv("QPK_PDL") ? atoi(getenv("QPK_PDL")) : 1;
  return env != 0 && !c->sharded &&
         (c->scatter == QPK_SCATTER_DICT || (c->scatter == QPK_SCATTER_PANEL && c->panel_direct));
}

// CTA-accumulation mode with few partials per column: one combine launch
static bool comb_direct(const qpk_ctx* c) { return c->scatter == QPK_SCATTER_DICT && c->cacc && c->comb_max2 <= 16; }

// tile mode, single-level combine: the CTA partials are summed inside the
// update kernel (top_value<3>, same order as k_comb_direct), one launch less
static bool comb_fused(const qpk_ctx* c) {
  const int env = getenv("QPK_FUSE_COMB") ? atoi(getenv("QPK_FUSE_COMB")) : 1;
  return env != 0 && comb_direct(c);      // (sharded: summed inside k_shard_reduce<3> instead)
}

// sharded tile format: the residual scalars [r'r, r'z] ride in the slot's one
// all-reduce (k_slot_update has the algebra); QPK_SHARD_FOLD=0 keeps the
// second all-reduce + decision kernel
static bool slot_fold(const qpk_ctx* c) {
  const int env = getenv("QPK_SHARD_FOLD") ? atoi(getenv("QPK_SHARD_FOLD")) : 1;
  return env != 0 && c->sharded && c->fold_all && c->scatter == QPK_SCATTER_DICT && c->cacc;
}

// does the slot finish B'z with a CSC gather pass (k_slot_csc + seg sums)?
static bool slot_csc(const qpk_ctx* c) {
  return c->scatter == QPK_SCATTER_CSC || (c->scatter == QPK_SCATTER_PANEL && !c->panel_direct);
}

static int slot_launches(const qpk_ctx* c) {
  int k = 2;                                                    // top, update
  if (c->scatter == QPK_SCATTER_DICT)
    k += (comb_fused(c) ? 1 : comb_direct(c) ? 2 : 3) + ((c->hkind != QPK_HESS_DIAG && !c->h_tiled) ? 1 : 0) +
         (c->h_nchunks ? 1 : 0);
  else if (c->scatter == QPK_SCATTER_PANEL)
    k += 2 + (c->hkind != QPK_HESS_DIAG ? 1 : 0) + (slot_csc(c) ? 1 : 0) + (c->h_nchunks ? 1 : 0);
  else k += 1 + (slot_csc(c) ? 1 : 0) + (c->h_nchunks ? 2 : 0) + (c->n_dense ? 1 : 0);
  if (c->sharded) k += slot_fold(c) ? 1 : 2;
  return k;
}

// the operator part of a slot: top, the pass over B (+ its B'z completion
// into y_top, except the CSC segment sums, which the consumer adds)
static void launch_slot_apply(qpk_ctx* c, const Engine& E, int par, cudaStream_t s) {
  const bool csc = slot_csc(c);
  const int G = c->grid_eng;
  const bool pdl = slot_pdl(c);
  launch_k(pdl, k_slot_top, dim3(G), dim3(QPK_BLOCK), 0, s, E, par);
  if (c->scatter == QPK_SCATTER_PANEL) {
    QPK_PANEL_DISPATCH(launch_panel_t, c, s, E, par, pdl);
    // y_P += B'z (CTA partials); direct remainder: y[col] += yrem
    const int rem_blocks = (c->panel_direct && c->panel_ew > 0)
                               ? (int)std::min<long long>(2 * c->sms, (c->m * c->panel_ew + 1023) / 1024) : 0;
    launch_k(pdl, k_panel_comb, dim3(c->panel_kp / 32 + rem_blocks), dim3(1024), 0, s, E, c->y.p, 1, par);
    if (c->hkind != QPK_HESS_DIAG) k_slot_hess<<<G, QPK_BLOCK, 0, s>>>(E, par);
    if (c->h_nchunks) k_slot_sym_combine<<<G, QPK_SYMC_BLOCK, 0, s>>>(E, par);
    if (csc) k_slot_csc<<<c->sms * 8, QPK_BLOCK, 0, s>>>(E, par);
  } else if (c->scatter == QPK_SCATTER_DICT) {
    launch_k(pdl, k_slot_rows_tile, dim3(E.G_rows),
             dim3((QPK_TILE_GROUPS * QPK_TILE_GWARPS + 1 + QPK_TILE_GATHER_WARPS) * 32), tile_smem(), s, E, par);
    if (comb_fused(c)) {
      // y_top's B'z partials are summed by the update kernel (k_slot_update<3>)
    } else if (comb_direct(c)) {                               // y_top += B'z (CTA partials)
      launch_k(pdl, k_comb_direct, dim3(std::max(1, std::min(G, (int)((c->n + QPK_BLOCK - 1) / QPK_BLOCK)))),
               dim3(QPK_BLOCK), 0, s, E, c->y.p, 1, par);
    } else {
      launch_k(pdl, k_comb_seg, dim3(G), dim3(QPK_BLOCK), 0, s, E, par);     // y_top += B'z (tile partials)
      launch_k(pdl, k_comb_col, dim3(G), dim3(QPK_BLOCK), 0, s, E, c->y.p, 1, par);
    }
    if (c->hkind != QPK_HESS_DIAG && !c->h_tiled) k_slot_hess<<<G, QPK_BLOCK, 0, s>>>(E, par);
    if (c->h_nchunks) k_slot_sym_combine<<<G, QPK_SYMC_BLOCK, 0, s>>>(E, par);
  } else {
    switch (c->lanes * 2 + (csc ? 1 : 0)) {
      case 2: launch_slot_rows_t<1, false>(c, G, s, E, par); break;
      case 3: launch_slot_rows_t<1, true>(c, G, s, E, par); break;
      case 4: launch_slot_rows_t<2, false>(c, G, s, E, par); break;
      case 5: launch_slot_rows_t<2, true>(c, G, s, E, par); break;
      case 8: launch_slot_rows_t<4, false>(c, G, s, E, par); break;
      case 9: launch_slot_rows_t<4, true>(c, G, s, E, par); break;
      case 16: launch_slot_rows_t<8, false>(c, G, s, E, par); break;
      case 17: launch_slot_rows_t<8, true>(c, G, s, E, par); break;
      case 32: launch_slot_rows_t<16, false>(c, G, s, E, par); break;
      case 33: launch_slot_rows_t<16, true>(c, G, s, E, par); break;
      case 64: launch_slot_rows_t<32, false>(c, G, s, E, par); break;
      default: launch_slot_rows_t<32, true>(c, G, s, E, par); break;
    }
    if (c->n_dense) {                                                  // dense rows of B, before the CSC gather
      if (csc) k_slot_dense<true><<<G, QPK_BLOCK, 0, s>>>(E, par);
      else k_slot_dense<false><<<G, QPK_BLOCK, 0, s>>>(E, par);
    }
    if (csc) k_slot_csc<<<c->sms * 8, QPK_BLOCK, 0, s>>>(E, par);
    if (c->h_nchunks) {                                                // packed symmetric dense H
      k_slot_hess_sym<<<QPK_SYM_MINB * c->sms, QPK_BLOCK, 0, s>>>(E, par);
      k_slot_sym_combine<<<G, QPK_SYMC_BLOCK, 0, s>>>(E, par);
    }
  }
}

static void launch_slot(qpk_ctx* c, const Engine& E, int par, cudaStream_t s) {
  const bool csc = slot_csc(c);
  const int G = c->grid_eng;
  launch_slot_apply(c, E, par, s);
  if (!c->sharded) {
    if (csc) k_slot_update<2><<<G, QPK_BLOCK, 0, s>>>(E, par);
    else if (comb_fused(c)) launch_k(slot_pdl(c), k_slot_update<3>, dim3(G), dim3(QPK_BLOCK), 0, s, E, par);
    else launch_k(slot_pdl(c), k_slot_update<1>, dim3(G), dim3(QPK_BLOCK), 0, s, E, par);
    return;
  }
  // sharded: finish the local top block and scalars, one grouped all-reduce
  // of [y_top | scalars], the update on the now-global y, an all-reduce of
  // r'r and r'z, and the control decision.
  if (csc) k_shard_reduce<2><<<G, QPK_BLOCK, 0, s>>>(E, par);
  else if (comb_fused(c)) k_shard_reduce<3><<<G, QPK_BLOCK, 0, s>>>(E, par);   // + the CTA-partial combine
  else k_shard_reduce<1><<<G, QPK_BLOCK, 0, s>>>(E, par);
  const bool fold = slot_fold(c);
  if (!c->hostcomm) nccl().groupStart();
  allreduce_sum(c, c->y.p, c->n, s);
  allreduce_sum(c, c->gscal.p, fold ? 10 : 4, s);
  if (!c->hostcomm) nccl().groupEnd();
  k_slot_update<1><<<G, QPK_BLOCK, 0, s>>>(E, par);
  if (fold) return;                                  // the update kernel's last block decided
  allreduce_sum(c, c->lscal2.p, 2, s);
  k_slot_decide<<<1, 32, 0, s>>>(E, par);
}

// K v through the same kernels a PCG slot runs (tile / panel modes): v goes
// to x[0] and the slot runs as the explicit-residual apply (MODE_CHECK) of it
static int apply_engine(qpk_ctx* c, const double* v_dev, double* y_dev) {
  int rc = engine_setup(c);
  if (rc) return rc;
  cudaStream_t s = c->stream;
  Ctrl h;
  memset(&h, 0, sizeof h);
  h.mode = MODE_CHECK;
  CUDA_TRY(cudaMemcpyAsync(c->x[0].p, v_dev, c->N() * sizeof(double), cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(c->ctrl.p, &h, sizeof h, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaStreamSynchronize(s));          // h is a stack object
  Engine E = make_engine(c);
  launch_slot_apply(c, E, 0, s);
  if (slot_csc(c)) k_apply_finish<2><<<c->grid_eng, QPK_BLOCK, 0, s>>>(E, y_dev);
  else if (comb_fused(c)) k_apply_finish<3><<<c->grid_eng, QPK_BLOCK, 0, s>>>(E, y_dev);
  else k_apply_finish<1><<<c->grid_eng, QPK_BLOCK, 0, s>>>(E, y_dev);
  c->launches += slot_launches(c) - 1;
  CUDA_TRY(cudaGetLastError());
  return allreduce_sum(c, y_dev, c->n, s);
}

static Engine make_engine(qpk_ctx* c) {
  Engine E;
  E.op = c->op();
  E.rhs = c->rhs.p;
  for (int i = 0; i < 3; ++i) E.x[i] = c->x[i].p;
  E.r = c->r.p; E.p = c->p.p; E.y = c->y.p; E.zb = c->zb.p; E.minv = c->minv.p;
  E.part = c->part.p; E.G = c->grid_eng;
  E.G_rows = c->scatter == QPK_SCATTER_DICT ? std::min(c->sms, c->grid_eng) : c->grid_eng;
  if (c->scatter == QPK_SCATTER_PANEL) E.G_rows = c->panel_grid;
  E.panel.kp = c->panel_kp; E.panel.ew = c->panel_ew; E.panel.direct = c->panel_direct; E.panel.G = c->panel_grid;
  E.panel.P = c->panel_P.p; E.panel.pcols = c->panel_cols.p; E.panel.eci = c->panel_eci.p; E.panel.ev = c->panel_ev.p;
  E.panel.ppart = c->panel_part.p;
  const bool pdir = c->scatter == QPK_SCATTER_PANEL && c->panel_direct && c->panel_ew > 0;
  E.panel.cpos = pdir ? c->panel_cpos.p : nullptr;
  E.panel.ue = c->panel_ue.p; E.panel.yrem = c->panel_yrem.p;
  E.ctrl = c->ctrl.p; E.counter = c->counter.p; E.cfg = c->ecfg.p;
  E.seg_ptr = c->seg_ptr.p; E.seg_beg = c->seg_beg.p; E.seg_sum = c->seg_sum.p;
  E.n_seg = c->n_seg; E.seg_lanes = c->seg_lanes;
  E.scatter = c->scatter;
  E.sharded = c->sharded ? 1 : 0;
  E.fold = slot_fold(c) ? 1 : 0;
  if (c->n_dense && (c->scatter == QPK_SCATTER_ATOMIC || c->scatter == QPK_SCATTER_CSC)) {
    E.op.r0 = c->n_dense; E.op.ndense = c->n_dense; E.op.cdense = c->cdense.p;
  }
  E.gscal = c->gscal.p; E.lscal2 = c->lscal2.p; E.abuf = c->abuf.p;
  E.dict.nblk = c->nblk; E.dict.tiles = c->tiles.p; E.dict.cols = c->dcols.p; E.dict.tval = c->tval.p;
  E.dict.bpart = c->bpart.p; E.dict.col_ptr = c->col_ptr.p; E.dict.col_pos = c->col_pos.p;
  E.dict.comb_lanes = c->comb_lanes;
  E.dict.nseg = c->comb_nseg; E.dict.seg_beg = c->comb_beg.p; E.dict.col_seg = c->comb_col.p;
  E.dict.seg_sum = c->comb_sum.p;
  E.dict.hperm = c->h_tiled ? c->hperm.p : nullptr;
  E.dict.cacc = 0;
  E.dict.l2pf = 0;
  if (c->scatter == QPK_SCATTER_DICT && c->cacc) {
    E.dict.cacc = 1;
    E.dict.tile_beg = c->tile_beg.p; E.dict.cta_off = c->cta_off.p; E.dict.tslot = c->tslot.p;
    E.dict.cpart = c->cpart.p;
    // long per-CTA tile streams (cfg4: ~380 tiles per CTA) gain from an L2
    // prefetch 3 tiles beyond the ring (+3 %); short ones (cfg3: ~37) lose
    // (A/B in DESIGN.md §4.3).  QPK_TILE_L2PF overrides.
    // (with the evict-first stream the prefetch no longer pays: cfg4 297 us
    // without it, 307 us with 3 tiles; kept as a switch)
    E.dict.l2pf = 0;
    if (const char* ev = getenv("QPK_TILE_L2PF")) E.dict.l2pf = std::max(0, std::min(31, atoi(ev)));
    E.dict.col_ptr = c->col_ptr2.p; E.dict.col_pos = c->col_pos2.p;
    E.dict.comb_lanes = c->comb_lanes2; E.dict.nseg = c->comb_nseg2;
    E.dict.seg_beg = c->comb_beg2.p; E.dict.col_seg = c->comb_col2.p;
    E.G_rows = c->tile_grid;
  }
  return E;
}

static int engine_setup(qpk_ctx* c) {
  // per-format kernel attributes: a context may be re-finalized with another
  // problem (qpk_problem_begin again), so these are set for the current format
  if (c->attr_scatter != c->scatter || c->attr_kp != c->panel_kp) {
    CUDA_TRY(cudaFuncSetAttribute(k_slot_rows_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_smem()));
    if (c->scatter == QPK_SCATTER_PANEL) CUDA_TRY(panel_attr(c));
    c->attr_scatter = c->scatter; c->attr_kp = c->panel_kp;
  }
  if (c->ctrl.p) return QPK_OK;
  CUDA_TRY(c->ctrl.alloc(2));
  CUDA_TRY(c->gscal.alloc(10));
  CUDA_TRY(c->lscal2.alloc(2));
  CUDA_TRY(c->abuf.alloc(2));
  CUDA_TRY(c->counter.alloc(1));
  CUDA_TRY(c->ecfg.alloc(1));
  CUDA_TRY(cudaMemsetAsync(c->counter.p, 0, sizeof(unsigned int), c->stream));
  CUDA_TRY(cudaMemsetAsync(c->ctrl.p, 0, 2 * sizeof(Ctrl), c->stream));
  CUDA_TRY(cudaHostAlloc((void**)&c->pinned_mode, 2 * sizeof(int), cudaHostAllocDefault));
  for (auto& e : c->poll_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return QPK_OK;
}

// capture `slots` identical slots (slots even: parity pattern repeats) as a graph
static int engine_graph(qpk_ctx* c, int slots) {
  if (c->graph && c->graph_slots == slots) return QPK_OK;
  if (c->graph) { cudaGraphExecDestroy(c->graph); c->graph = nullptr; }
  if (c->graph_failed || c->hostcomm) return QPK_OK;   // (host-mediated collectives cannot be captured)
  Engine E = make_engine(c);
  cudaStream_t cs = c->own;
  cudaGraph_t g = nullptr;
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { c->graph_failed = true; cudaGetLastError(); return QPK_OK; }
  for (int s = 0; s < slots; ++s) launch_slot(c, E, s & 1, cs);
  if (cudaStreamEndCapture(cs, &g) != cudaSuccess || !g) { c->graph_failed = true; cudaGetLastError(); return QPK_OK; }
  if (cudaGraphInstantiate(&c->graph, g, 0) != cudaSuccess) { c->graph = nullptr; c->graph_failed = true; cudaGetLastError(); }
  cudaGraphDestroy(g);
  c->graph_slots = slots;
  return QPK_OK;
}

static int pcg_engine(qpk_ctx* c, double tol, int rel, int64_t max_iters, double* hist_dev, PcgOut* out) {
  int rc = engine_setup(c);
  if (rc) return rc;
  const int CH = 16;
  rc = engine_graph(c, CH);
  if (rc) return rc;
  cudaStream_t s = c->stream;
  EngineCfg hc;
  hc.tol = tol; hc.max_iters = max_iters; hc.rel = rel ? 1 : 0; hc.pad = 0; hc.hist = hist_dev;
  CUDA_TRY(cudaMemcpyAsync(c->ecfg.p, &hc, sizeof hc, cudaMemcpyHostToDevice, s));
  Engine E = make_engine(c);
  k_engine_init<<<c->grid_eng, QPK_BLOCK, 0, s>>>(E);
  c->launches++;
  if (c->sharded) {
    rc = allreduce_sum(c, c->lscal2.p, 1, s);      // ||rhs||^2 over ranks
    if (rc) return rc;
    k_engine_init2<<<1, 32, 0, s>>>(E);
    c->launches++;
  }
  CUDA_TRY(cudaGetLastError());
  // upper bound on slots: every iteration may be followed by a check, + final
  const long long max_slots = 2 * max_iters + 4;
  long long slots = 0;
  int chunk = 0;
  for (;;) {
    if (c->graph) {
      CUDA_TRY(cudaGraphLaunch(c->graph, s));
    } else {
      for (int k = 0; k < CH; ++k) launch_slot(c, E, k & 1, s);
    }
    c->launches += (long long)slot_launches(c) * CH;
    slots += CH;
    const int b = chunk & 1;
    CUDA_TRY(cudaMemcpyAsync(&c->pinned_mode[b], &c->ctrl.p[0].mode, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(c->poll_ev[b], s));
    if (chunk > 0) {
      CUDA_TRY(cudaEventSynchronize(c->poll_ev[b ^ 1]));
      if (c->pinned_mode[b ^ 1] == MODE_DONE) break;
    }
    if (slots > max_slots + 2 * CH) return fail(QPK_E_STATE, "slot engine did not terminate");
    ++chunk;
  }
  Ctrl fin;
  CUDA_TRY(cudaMemcpyAsync(&fin, c->ctrl.p, sizeof fin, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  if (fin.mode != MODE_DONE) return fail(QPK_E_STATE, "slot engine: final state not DONE");
  out->iterations = fin.k; out->converged = fin.converged; out->status = fin.status;
  out->restarts = fin.restarts; out->applies = fin.applies; out->result_buf = fin.result;
  out->final_norm = fin.final_norm; out->threshold = fin.thr; out->rhs_norm = fin.rhs_norm;
  out->phase_ns[0] = fin.ph[0]; out->phase_ns[1] = fin.ph[1]; out->phase_ns[2] = fin.ph[2]; out->phase_ns[3] = fin.ph[3];
  return QPK_OK;
}

extern "C" {

static bool use_engine(qpk_ctx* c) {
  if (c->scatter == QPK_SCATTER_DICT || c->scatter == QPK_SCATTER_PANEL || c->sharded || c->h_nchunks ||
      c->n_dense)
    return true;                                 // tile / panel / packed-H kernels, collectives: engine only
  if (c->engine >= 0) return c->engine == 1;
  const char* env = getenv("QPK_ENGINE");
  if (env) return atoi(env) == 1;
  // small systems: one cooperative launch wins on latency; the random-B atomic
  // path is as fast in the persistent kernel; the CSC path needs the engine's
  // balanced column segments
  return c->scatter == QPK_SCATTER_CSC && c->N() >= 50000;
}

static int pcg_impl(qpk_ctx* c, const double* rhs_dev, double tol, int rel, int64_t max_iters, double* x_dev,
                    qpk_pcg_info* info, double* hist_dev) {
  if (!(tol > 0.0)) return fail(QPK_E_ARG, "tol must be positive");
  if (max_iters < 1) return fail(QPK_E_ARG, "max_iters must be at least 1");
  if (max_iters > (1LL << 30)) return fail(QPK_E_ARG, "max_iters too large");
  if (!c->jac_ready) { int rc = build_jacobi(c); if (rc) return rc; }
  if (rhs_dev != c->rhs.p)
    CUDA_TRY(cudaMemcpyAsync(c->rhs.p, rhs_dev, c->N() * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  for (auto& e : c->time_ev) if (!e) CUDA_TRY(cudaEventCreate(&e));
  cudaEvent_t e0 = c->time_ev[0], e1 = c->time_ev[1];
  CUDA_TRY(cudaEventRecord(e0, c->stream));
  PcgOut o;
  if (use_engine(c)) {
    int rc = pcg_engine(c, tol, rel, max_iters, hist_dev, &o);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(e1, c->stream));
  } else if (c->cl_C > 0) {
    ClParams P;
    P.n = (int)c->n; P.m = (int)c->m; P.C = c->cl_C;
    P.ctas = c->cl_ctas.p; P.blob = c->cl_blob.p; P.blob_off = c->cl_off.p;
    P.q = c->q.p; P.d = c->d.p; P.minv = c->minv.p; P.rhs = c->rhs.p;
    P.x_out = c->x[0].p; P.hist = hist_dev;
    P.tol = tol; P.rel = rel ? 1 : 0; P.max_iters = max_iters;
    P.out = c->out.p;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(c->cl_C); lc.blockDim = dim3(QPK_CL_THREADS); lc.dynamicSmemBytes = c->cl_smem;
    lc.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->cl_C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&lc, k_pcg_cluster, P));
    c->launches++;
    CUDA_TRY(cudaEventRecord(e1, c->stream));
    CUDA_TRY(cudaMemcpyAsync(&o, c->out.p, sizeof o, cudaMemcpyDeviceToHost, c->stream));
  } else {
    PcgParams P;
    P.op = c->op();
    P.rhs = c->rhs.p;
    P.x0 = c->x[0].p; P.x1 = c->x[1].p; P.x2 = c->x[2].p;
    P.r = c->r.p; P.p = c->p.p; P.y = c->y.p; P.zb = c->zb.p; P.minv = c->minv.p;
    P.part = c->part.p; P.G = c->grid_pcg;
    P.tol = tol; P.rel = rel ? 1 : 0; P.max_iters = max_iters;
    P.hist = hist_dev;
    P.out = c->out.p;
    void* args[] = {&P};
    CUDA_TRY(cudaLaunchCooperativeKernel(pcg_kernel_for(c->lanes, c->scatter == QPK_SCATTER_CSC),
                                         dim3(c->grid_pcg), dim3(QPK_BLOCK), args, 0, c->stream));
    c->launches++;
    CUDA_TRY(cudaEventRecord(e1, c->stream));
    CUDA_TRY(cudaMemcpyAsync(&o, c->out.p, sizeof o, cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  const double* res = c->x[o.result_buf].p;
  CUDA_TRY(cudaMemcpyAsync(x_dev, res, c->N() * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if (info) {
    info->iterations = o.iterations; info->converged = o.converged; info->status = o.status;
    info->restarts = o.restarts; info->applies = o.applies; info->reserved = 0;
    info->final_residual_norm = o.final_norm; info->threshold = o.threshold; info->rhs_norm = o.rhs_norm;
    info->kernel_ms = ms;
    for (int i = 0; i < 4; ++i) info->phase_ms[i] = o.phase_ns[i] * 1e-6;
  }
  return QPK_OK;
}

int qpk_pcg_dev(qpk_ctx* c, const double* rhs, double tol, int rel, int64_t max_iters, double* x,
                qpk_pcg_info* info, double* hist) {
  if (!c || !c->diag_set) return fail(QPK_E_STATE, "qpk_pcg_dev: diagonals not set");
  if (!rhs || !x) return fail(QPK_E_ARG, "qpk_pcg_dev: null vector");
  CUDA_TRY(cudaSetDevice(c->device));
  int rc = pcg_impl(c, rhs, tol, rel, max_iters, x, info, hist);
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return QPK_OK;
}

int qpk_pcg(qpk_ctx* c, const double* rhs, double tol, int rel, int64_t max_iters, double* x, qpk_pcg_info* info,
            double* hist) {
  if (!c || !c->diag_set) return fail(QPK_E_STATE, "qpk_pcg: diagonals not set");
  if (!rhs || !x) return fail(QPK_E_ARG, "qpk_pcg: null vector");
  if (max_iters < 1) return fail(QPK_E_ARG, "max_iters must be at least 1");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t bytes = c->N() * sizeof(double);
  // the Jacobi build first: its kernels run while the host stages the (pageable) rhs
  if (!c->jac_ready) { int rcj = build_jacobi(c); if (rcj) return rcj; }
  CUDA_TRY(cudaMemcpyAsync(c->rhs.p, rhs, bytes, cudaMemcpyHostToDevice, c->stream));
  double* hist_dev = nullptr;
  if (hist) {
    CUDA_TRY(c->hist.alloc(max_iters + 1));
    hist_dev = c->hist.p;
  }
  int rc = pcg_impl(c, c->rhs.p, tol, rel, max_iters, c->vin.p, info, hist_dev);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(x, c->vin.p, bytes, cudaMemcpyDeviceToHost, c->stream));
  if (hist) {
    const long long cnt = (info ? info->iterations : max_iters) + 1;
    CUDA_TRY(cudaMemcpyAsync(hist, hist_dev, std::min<long long>(cnt, max_iters + 1) * sizeof(double),
                             cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return QPK_OK;
}

// ------------------------------------------------------------ device IPM ---
int qpk_ipm_set_bounds(qpk_ctx* c, const double* p, const double* bnd, int64_t nl, const int64_t* vlo,
                       const double* lx, int64_t nu, const int64_t* vhi, const double* ux) {
  if (!c || !c->finalized) return fail(QPK_E_STATE, "qpk_ipm_set_bounds: problem not finalized");
  if (c->sharded) return fail(QPK_E_UNSUPPORTED, "device IPM is single-GPU");
  if (!p || (c->m && !bnd) || nl < 0 || nu < 0 || nl > c->n || nu > c->n)
    return fail(QPK_E_ARG, "qpk_ipm_set_bounds: bad arguments");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const long long n = c->n, m = c->m, N = c->N();
  std::vector<int> lo(nl), hi(nu);
  std::vector<unsigned char> haslo(n, 0), hashi(n, 0);
  std::vector<double> lof(n, 0.0), hif(n, 0.0);
  for (long long k = 0; k < nl; ++k) {
    if (vlo[k] < 0 || vlo[k] >= n) return fail(QPK_E_ARG, "variable bound index out of range");
    lo[k] = (int)vlo[k]; haslo[vlo[k]] = 1; lof[vlo[k]] = lx[k];
  }
  for (long long k = 0; k < nu; ++k) {
    if (vhi[k] < 0 || vhi[k] >= n) return fail(QPK_E_ARG, "variable bound index out of range");
    hi[k] = (int)vhi[k]; hashi[vhi[k]] = 1; hif[vhi[k]] = ux[k];
  }
  c->nl = nl; c->nu = nu;
  CUDA_TRY(upload(c->vlo, lo, s));
  CUDA_TRY(upload(c->vhi, hi, s));
  CUDA_TRY(upload(c->ipm_haslo, haslo, s));
  CUDA_TRY(upload(c->ipm_hashi, hashi, s));
  CUDA_TRY(upload(c->ipm_lofull, lof, s));
  CUDA_TRY(upload(c->ipm_hifull, hif, s));
  const std::vector<double> vlx(lx, lx + nl), vux(ux, ux + nu), vbnd(bnd, bnd + m), vp(p, p + n);
  CUDA_TRY(upload(c->ipm_lx, vlx, s));
  CUDA_TRY(upload(c->ipm_ux, vux, s));
  CUDA_TRY(upload(c->ipm_bnd, vbnd, s));
  CUDA_TRY(upload(c->ipm_p, vp, s));
  for (DBuf<double>* b : {&c->ipm_x, &c->ipm_rH, &c->ipm_hx, &c->ipm_btl, &c->ipm_tmp, &c->ipm_zero})
    CUDA_TRY(b->alloc(n + 8));
  for (DBuf<double>* b : {&c->ipm_sB, &c->ipm_lamB, &c->ipm_rB, &c->ipm_rcB, &c->ipm_dsB, &c->ipm_dlamB,
                          &c->ipm_t, &c->ipm_w2})
    CUDA_TRY(b->alloc(m + 8));
  for (DBuf<double>* b : {&c->ipm_slx, &c->ipm_llx, &c->ipm_rlx, &c->ipm_rc3, &c->ipm_dslx, &c->ipm_dllx})
    CUDA_TRY(b->alloc(nl + 8));
  for (DBuf<double>* b : {&c->ipm_sux, &c->ipm_lux, &c->ipm_rux, &c->ipm_rc4, &c->ipm_dsux, &c->ipm_dlux})
    CUDA_TRY(b->alloc(nu + 8));
  CUDA_TRY(c->ipm_rhs.alloc(N + 8));
  CUDA_TRY(c->ipm_sol.alloc(N + 8));
  CUDA_TRY(c->ipm_part.alloc(8 * (size_t)c->grid_std));
  CUDA_TRY(cudaMemsetAsync(c->ipm_zero.p, 0, (n + 8) * sizeof(double), s));
  CUDA_TRY(cudaStreamSynchronize(s));
  c->ipm_ready = true;
  return QPK_OK;
}

static IpmDev ipm_dev(qpk_ctx* c) {
  IpmDev P;
  P.n = (int)c->n; P.m = (int)c->m; P.me = (int)c->m_e; P.ml = (int)c->m_l; P.mu_rows = (int)c->m_u;
  P.nl = (int)c->nl; P.nu = (int)c->nu;
  P.vlo = c->vlo.p; P.vhi = c->vhi.p; P.lx = c->ipm_lx.p; P.ux = c->ipm_ux.p; P.bnd = c->ipm_bnd.p; P.pvec = c->ipm_p.p;
  P.x = c->ipm_x.p; P.sB = c->ipm_sB.p; P.lamB = c->ipm_lamB.p;
  P.slx = c->ipm_slx.p; P.sux = c->ipm_sux.p; P.llx = c->ipm_llx.p; P.lux = c->ipm_lux.p;
  P.rH = c->ipm_rH.p; P.rB = c->ipm_rB.p; P.rcB = c->ipm_rcB.p; P.rlx = c->ipm_rlx.p; P.rux = c->ipm_rux.p;
  P.rc3 = c->ipm_rc3.p; P.rc4 = c->ipm_rc4.p;
  P.dsB = c->ipm_dsB.p; P.dlamB = c->ipm_dlamB.p; P.dslx = c->ipm_dslx.p; P.dsux = c->ipm_dsux.p;
  P.dllx = c->ipm_dllx.p; P.dlux = c->ipm_dlux.p;
  P.hx = c->ipm_hx.p; P.t = c->ipm_t.p; P.btl = c->ipm_btl.p; P.part = c->ipm_part.p; P.G = c->grid_std;
  return P;
}

// H x into ipm_hx (prep with q = 0 gives the diagonal part, k_hess the rest)
static void ipm_hess_apply(qpk_ctx* c, const double* xv, double* out) {
  Op o = c->op();
  o.q = c->ipm_zero.p;
  o.top_owner = 1;
  const int G = c->grid_std;
  k_prep<<<G, QPK_BLOCK, 0, c->stream>>>(o, xv, out, c->part.p, G);
  k_hess<<<G, QPK_BLOCK, 0, c->stream>>>(o, xv, out, c->part.p, G);
  if (c->h_nchunks) { k_sym_combine<<<G, QPK_SYMC_BLOCK, 0, c->stream>>>(o, xv, out); c->launches++; }
  c->launches += 2;
}

static void ipm_bt(qpk_ctx* c, const double* w, double* out) {
  const int G = c->grid_std;
  cudaMemsetAsync(out, 0, c->n * sizeof(double), c->stream);
  if (c->m) k_spmv_bt<<<G, QPK_BLOCK, 0, c->stream>>>(c->op(), w, out);
  c->launches++;
}

// partial sums (sum or min) of `slots` slots, on the host
static int ipm_read(qpk_ctx* c, int slots, std::vector<double>& h) {
  const int G = c->grid_std;
  h.resize((size_t)slots * G);
  CUDA_TRY(cudaMemcpyAsync(h.data(), c->ipm_part.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return QPK_OK;
}
static double slot_sum(const std::vector<double>& h, int slot, int G) {
  double s = 0.0;
  for (int i = 0; i < G; ++i) s += h[(size_t)slot * G + i];
  return s;
}
static double slot_min(const std::vector<double>& h, int slot, int G) {
  double s = INFINITY;
  for (int i = 0; i < G; ++i) s = std::min(s, h[(size_t)slot * G + i]);
  return s;
}

// residuals at the current iterate; returns (primal, dual, compl, full) norms
static int ipm_residuals(qpk_ctx* c, double mu, double out[4], bool* finite) {
  IpmDev P = ipm_dev(c);
  const int G = c->grid_std;
  cudaStream_t s = c->stream;
  ipm_hess_apply(c, P.x, P.hx);
  if (c->m) k_spmv_b<<<G, QPK_BLOCK, 0, s>>>(c->op(), P.x, P.t);
  ipm_bt(c, P.lamB, P.btl);
  k_ipm_residuals<<<G, QPK_BLOCK, 0, s>>>(P, mu);
  k_ipm_rh_lo<<<G, QPK_BLOCK, 0, s>>>(P);
  k_ipm_rh_hi<<<G, QPK_BLOCK, 0, s>>>(P);
  k_ipm_dual_norm<<<G, QPK_BLOCK, 0, s>>>(P);
  c->launches += 5;
  CUDA_TRY(cudaGetLastError());
  std::vector<double> h;
  int rc = ipm_read(c, 6, h);
  if (rc) return rc;
  const double pr = slot_sum(h, 0, G), du = slot_sum(h, 1, G), co = slot_sum(h, 2, G), re = slot_sum(h, 3, G);
  out[0] = sqrt(pr); out[1] = sqrt(du); out[2] = sqrt(co); out[3] = sqrt(pr + du + co + re);
  *finite = slot_sum(h, 4, G) == 0.0 && slot_sum(h, 5, G) == 0.0;
  return QPK_OK;
}

int qpk_ipm_solve(qpk_ctx* c, const qpk_ipm_config* cfg, double* x_out, qpk_ipm_trace* trace,
                  qpk_ipm_result* res) {
  if (!c || !c->ipm_ready) return fail(QPK_E_STATE, "qpk_ipm_solve: call qpk_ipm_set_bounds first");
  if (!cfg || !res) return fail(QPK_E_ARG, "qpk_ipm_solve: null config/result");
  if (!(cfg->gamma > 0.0 && cfg->gamma < 1.0)) return fail(QPK_E_ARG, "gamma must lie in (0, 1)");
  if (cfg->mu_init <= 0 || cfg->mu_tol <= 0 || cfg->mu_shrink <= 1.0) return fail(QPK_E_ARG, "bad barrier parameters");
  CUDA_TRY(cudaSetDevice(c->device));
  const auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = c->stream;
  IpmDev P = ipm_dev(c);
  const int G = c->grid_std;
  const long long n = c->n, m = c->m;
  // initialize (ipm.py:73-104)
  k_ipm_init_x_bounds<<<G, QPK_BLOCK, 0, s>>>(P, c->ipm_haslo.p, c->ipm_hashi.p, c->ipm_lofull.p, c->ipm_hifull.p);
  if (m) k_spmv_b<<<G, QPK_BLOCK, 0, s>>>(c->op(), P.x, P.t);
  k_ipm_init_state<<<G, QPK_BLOCK, 0, s>>>(P, cfg->mu_init);
  c->launches += 3;
  double mu = cfg->mu_init;
  double nrm[4];
  bool finite = true;
  int rc = ipm_residuals(c, mu, nrm, &finite);
  if (rc) return rc;
  if (!finite) return fail(QPK_E_STATE, "non-finite residual encountered");
  res->status = 1;                      // iteration_limit
  res->iterations = 0;
  res->cg_total = 0;
  for (long long it = 1; it <= cfg->max_iters; ++it) {
    // operator diagonals (kkt.py:190-202)
    k_ipm_diagonals<<<G, QPK_BLOCK, 0, s>>>(P, mu, c->d.p, c->q.p);
    k_ipm_qextra_lo<<<G, QPK_BLOCK, 0, s>>>(P, c->q.p);
    k_ipm_qextra_hi<<<G, QPK_BLOCK, 0, s>>>(P, c->q.p);
    c->diag_set = true;
    c->jac_ready = false;
    // right-hand side (kkt.py:242-257)
    k_ipm_rhs<<<G, QPK_BLOCK, 0, s>>>(P, c->d.p, c->ipm_rhs.p, c->ipm_w2.p);
    k_ipm_rhs_lo<<<G, QPK_BLOCK, 0, s>>>(P, c->ipm_rhs.p);
    k_ipm_rhs_hi<<<G, QPK_BLOCK, 0, s>>>(P, c->ipm_rhs.p);
    ipm_bt(c, c->ipm_w2.p, c->ipm_tmp.p);
    k_ipm_rhs_top<<<G, QPK_BLOCK, 0, s>>>(P, c->ipm_rhs.p, c->ipm_tmp.p, c->ipm_part.p);
    c->launches += 7;
    CUDA_TRY(cudaGetLastError());
    {
      std::vector<double> h;
      rc = ipm_read(c, 1, h);
      if (rc) return rc;
      if (slot_sum(h, 0, G) != 0.0) return fail(QPK_E_STATE, "non-finite right-hand side");
    }
    // direction (ipm.py:205-212): a breakdown returns the best iterate, as the
    // reference's except-branch does
    qpk_pcg_info info;
    rc = pcg_impl(c, c->ipm_rhs.p, cfg->pcg_tol, cfg->pcg_tol_is_relative, cfg->pcg_max_iters, c->ipm_sol.p,
                  &info, nullptr);
    if (rc) return rc;
    res->cg_total += info.iterations;
    k_ipm_recover<<<G, QPK_BLOCK, 0, s>>>(P, c->ipm_sol.p);
    c->launches++;
    std::vector<double> h;
    rc = ipm_read(c, 3, h);
    if (rc) return rc;
    if (slot_sum(h, 2, G) != 0.0) { res->status = 2; break; }   // LINEAR_SOLVER_FAILURE
    const double ax = std::min(1.0, cfg->gamma * slot_min(h, 0, G));
    const double al = std::min(1.0, cfg->gamma * slot_min(h, 1, G));
    k_ipm_step<<<G, QPK_BLOCK, 0, s>>>(P, c->ipm_sol.p, ax, al);
    c->launches++;
    rc = ipm_read(c, 1, h);
    if (rc) return rc;
    if (!(slot_min(h, 0, G) > 0.0)) return fail(QPK_E_STATE, "step left the strict interior");
    rc = ipm_residuals(c, mu, nrm, &finite);
    if (rc) return rc;
    if (!finite) return fail(QPK_E_STATE, "non-finite residual encountered");
    if (trace) {
      qpk_ipm_trace& tr = trace[it - 1];
      tr.iter = (int)it; tr.cg_iters = info.iterations; tr.mu = mu;
      tr.primal_inf = nrm[0]; tr.dual_inf = nrm[1]; tr.compl_inf = nrm[2];
      tr.cg_resid = info.final_residual_norm; tr.alpha_x = ax; tr.alpha_lam = al;
    }
    res->iterations = (int)it;
    if (cfg->verbose)
      fprintf(stderr, "iter %4lld  mu %9.3e  primal %9.3e  dual %9.3e  compl %9.3e  cg %5d  alpha (%.3f, %.3f)\n",
              it, mu, nrm[0], nrm[1], nrm[2], info.iterations, ax, al);
    // barrier update (ipm.py:166-173, 229-235)
    if (nrm[3] < mu) {
      if (mu < cfg->mu_tol) { res->status = 0; break; }
      mu = mu / cfg->mu_shrink;
      rc = ipm_residuals(c, mu, nrm, &finite);
      if (rc) return rc;
    }
  }
  // objective at the final x (residuals left H x in ipm_hx)
  ipm_hess_apply(c, P.x, P.hx);
  k_ipm_objective<<<G, QPK_BLOCK, 0, s>>>(P);
  c->launches++;
  std::vector<double> h;
  rc = ipm_read(c, 2, h);
  if (rc) return rc;
  res->objective = 0.5 * slot_sum(h, 0, G) + slot_sum(h, 1, G);
  if (x_out) {
    CUDA_TRY(cudaMemcpyAsync(x_out, P.x, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  res->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return QPK_OK;
}

int64_t qpk_query(qpk_ctx* c, const char* key) {
  if (!c || !key) return -1;
  std::string k(key);
  if (k == "n") return c->n;
  if (k == "m") return c->m;
  if (k == "nnz") return c->nnz;
  if (k == "nnz_padded") return (int64_t)(c->ci.n);
  if (k == "lanes") return c->lanes;
  if (k == "csc_lanes") return c->csc_lanes;
  if (k == "scatter") return c->scatter;
  if (k == "grid") return c->grid_pcg;
  if (k == "grid_engine") return c->grid_eng;
  if (k == "engine") return use_engine(c) ? 1 : 0;
  if (k == "world") return c->world;
  if (k == "rank") return c->rank;
  if (k == "dict_blocks") return c->nblk;
  if (k == "tile_density_x100") return (int64_t)(c->dict_reuse * 100);
  if (k == "hess_tiled") return c->h_tiled ? 1 : 0;
  if (k == "hess_sym") return c->h_nchunks > 0 ? 1 : 0;
  if (k == "hess_symmetric") return c->h_symmetric ? 1 : 0;
  if (k == "dense_rows") return c->n_dense;
  if (k == "cluster") return c->cl_C;
  if (k == "tile_cta_acc") return c->cacc ? 1 : 0;
  if (k == "tile_grid") return c->tile_grid;
  if (k == "format_bytes") {
    // bytes of the chosen apply format that one pass over B (and a tiled H) streams
    if (c->scatter == QPK_SCATTER_DICT)
      return (int64_t)(c->tval.bytes() + c->dcols.bytes() + (c->cacc ? c->tslot.bytes() : 0) + c->tiles.bytes());
    if (c->scatter == QPK_SCATTER_PANEL)
      return (int64_t)(c->panel_P.bytes() + c->panel_ev.bytes() + c->panel_eci.bytes());
    const int64_t csr = (int64_t)(c->ci.bytes() + c->bv.bytes() + c->rp.bytes());
    return c->scatter == QPK_SCATTER_CSC ? csr + (int64_t)(c->ri.bytes() + c->cv.bytes() + c->cp.bytes()) : csr;
  }
  if (k == "tile_l2pf") return (c->scatter == QPK_SCATTER_DICT && c->cacc) ? make_engine(c).dict.l2pf : 0;
  if (k == "panel_kp") return c->panel_kp;
  if (k == "panel_cols") return c->panel_kd;
  if (k == "panel_ew") return c->panel_ew;
  if (k == "panel_direct") return c->panel_direct;
  if (k == "panel_grid") return c->panel_grid;
  if (k == "block") return QPK_BLOCK;
  if (k == "sms") return c->sms;
  if (k == "hess_kind") return c->hkind;
  if (k == "kernel_launches") return c->launches;
  if (k == "device_bytes") {
    size_t b = c->rp.bytes() + c->ci.bytes() + c->bv.bytes() + c->cp.bytes() + c->ri.bytes() + c->cv.bytes() +
               c->hh.bytes() + c->hrp.bytes() + c->hci.bytes() + c->hv.bytes() + c->hdense.bytes() + c->U.bytes() +
               c->w.bytes() + c->hdiag.bytes() + c->d.bytes() + c->q.bytes() + c->jac.bytes() + c->minv.bytes() +
               c->r.bytes() + c->p.bytes() + c->y.bytes() + c->zb.bytes() + c->rhs.bytes() + c->part.bytes() +
               c->vin.bytes() + c->hist.bytes() + c->panel_P.bytes() + c->panel_ev.bytes() + c->panel_eci.bytes() +
               c->panel_part.bytes() + c->tval.bytes() + c->bpart.bytes();
    for (auto& x : c->x) b += x.bytes();
    return (int64_t)b;
  }
  return -1;
}

}  // extern "C"

#include "qpk_multi.cuh"
