// qpk_cluster.cuh -- small systems (BASELINE cfg1, the reference's own test
// problems): the whole Jacobi-PCG solve of linalg.py:66-133 in ONE
// thread-block cluster, with the operator resident in shared memory.
//
// CTA c of the C-CTA cluster owns a contiguous slice of B's rows and of H's
// rows, stored in its shared memory as CSR (for t = B u, H u) and, for B, as
// CSC over the same rows (for the B'z partial, thread per column, no
// atomics).  The top block (n entries) is replicated: every CTA runs the top
// vector updates on identical data in identical order, so its copies stay
// bitwise equal and every scalar decision agrees without communication.  Per
// PCG iteration there are exactly two cluster barriers:
//   #1  each CTA has published its B'z + H u partial of y_top and its scalar
//       partials of p'Kp (and r'z after a restart); every CTA then sums the C
//       partials in CTA order through distributed shared memory (ld.shared::cluster);
//   #2  each CTA has published its rows' r'r / r'z partials.
// No global memory is touched inside the loop except the residual history.
#pragma once
#include <cooperative_groups.h>
#include "qpk_device.cuh"

#define QPK_CL_MAXC 16
#define QPK_CL_THREADS 512
#define QPK_CL_SMEM (220 * 1024)

namespace qpk {

// per-CTA slice descriptor; blob byte offsets are relative to the CTA's blob
struct ClCta {
  int r0, r1;                  // own B rows
  int h0, h1;                  // own H rows (top indices)
  int nnzb, nnzh;
  int o_brp, o_bci, o_bv;      // CSR of own B rows: local row ptr, global column, value
  int o_ccp, o_cri, o_cv;      // CSC of own B rows: column ptr (n + 1), local row, value
  int o_hrp, o_hci, o_hv;      // CSR of own H rows (full rows, diagonal included)
  int bytes;                   // blob bytes (multiple of 16)
  int pad;
};

struct ClParams {
  int n, m, C;
  const ClCta* ctas;
  const unsigned char* blob;   // concatenated CTA blobs
  const long long* blob_off;   // [C]
  const double* q;             // q_diag_extra (n)
  const double* d;             // d_diag (m)
  const double* minv;          // Jacobi inverse (N)
  const double* rhs;           // N
  double* x_out;               // N: the returned iterate
  double* hist;                // nullable, max_iters + 1
  double tol;
  int rel;
  long long max_iters;
  void* out;                   // PcgOut*
};

// shared-memory layout (doubles first, then ints), built identically on host
// and device from (n, own rows, own H rows, nnz)
struct ClLayout {
  int pub, scal, red;                                       // exchanged / scratch (offsets depend on n only)
  int p_t, r_t, mi_t, x_t, xb_t, q_t, rhs_t, y_t;          // n each
  int p_b, r_b, mi_b, x_b, xb_b, d_b, rhs_b, z_b, y_b;     // mr each
  int hu;                                                   // nh
  int blob;                                                 // byte offset of the operator blob
  int bytes;
};
__host__ __device__ __forceinline__ ClLayout cl_layout(int n, int mr, int nh, int blob_bytes) {
  ClLayout L;
  int o = 0;
  auto take = [&](int cnt) { const int at = o; o += (cnt + 1) & ~1; return at; };
  // everything read remotely (pub, scal) sits at offsets that depend on n only
  L.pub = take(n); L.scal = take(32); L.red = take(128);
  L.p_t = take(n); L.r_t = take(n); L.mi_t = take(n); L.x_t = take(n); L.xb_t = take(n);
  L.q_t = take(n); L.rhs_t = take(n); L.y_t = take(n);
  L.p_b = take(mr); L.r_b = take(mr); L.mi_b = take(mr); L.x_b = take(mr); L.xb_b = take(mr);
  L.d_b = take(mr); L.rhs_b = take(mr); L.z_b = take(mr); L.y_b = take(mr);
  L.hu = take(nh);
  L.blob = o * 8;
  L.bytes = L.blob + blob_bytes;
  return L;
}

__device__ __forceinline__ double cl_block_sum(double v, double* red) { return block_sum(v, red); }

// four block sums in one pass (fixed tree: deterministic); red needs 4 * 32 doubles
__device__ __forceinline__ void block_sum4(double& a, double& b, double& c, double& d, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
    d += __shfl_xor_sync(0xffffffffu, d, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) { red[warp] = a; red[32 + warp] = b; red[64 + warp] = c; red[96 + warp] = d; }
  __syncthreads();
  double ta = lane < nw ? red[lane] : 0.0, tb = lane < nw ? red[32 + lane] : 0.0;
  double tc = lane < nw ? red[64 + lane] : 0.0, td = lane < nw ? red[96 + lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ta += __shfl_xor_sync(0xffffffffu, ta, o);
    tb += __shfl_xor_sync(0xffffffffu, tb, o);
    tc += __shfl_xor_sync(0xffffffffu, tc, o);
    td += __shfl_xor_sync(0xffffffffu, td, o);
  }
  a = ta; b = tb; c = tc; d = td;
}

// DSMEM read of CTA `rank`'s copy of a shared-memory double
__device__ __forceinline__ double ld_remote(const double* local, unsigned rank) {
  unsigned a = (unsigned)__cvta_generic_to_shared(local), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(r));
  return v;
}

// K v for the CTA's slice: top entries of v in vt (replicated), bottom own
// rows in vb.  Writes z_b, y_b (own rows), publishes pub[j] (B'z over own rows
// + (H v)_j on own H rows) and returns this CTA's partial of
// sum_r (z_r t_r + v_r y_r) + sum_{own j} v_j (H v)_j   (v'Kv minus the q term).
__device__ double cl_apply(const ClParams& P, const ClCta& me, const ClLayout& L, double* sm, const double* vt,
                           const double* vb) {
  const int n = P.n, mr = me.r1 - me.r0, nh = me.h1 - me.h0;
  const unsigned char* bl = reinterpret_cast<const unsigned char*>(sm) + L.blob;
  const int* brp = reinterpret_cast<const int*>(bl + me.o_brp);
  const int* bci = reinterpret_cast<const int*>(bl + me.o_bci);
  const double* bv = reinterpret_cast<const double*>(bl + me.o_bv);
  const int* ccp = reinterpret_cast<const int*>(bl + me.o_ccp);
  const int* cri = reinterpret_cast<const int*>(bl + me.o_cri);
  const double* cv = reinterpret_cast<const double*>(bl + me.o_cv);
  const int* hrp = reinterpret_cast<const int*>(bl + me.o_hrp);
  const int* hci = reinterpret_cast<const int*>(bl + me.o_hci);
  const double* hv = reinterpret_cast<const double*>(bl + me.o_hv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double acc = 0.0;
  // rows of B (warp per row): t, z = 2t/d + v_b, y_b = t + d v_b
  for (int rr = warp; rr < mr; rr += nw) {
    double s0 = 0.0, s1 = 0.0;
    int k = brp[rr] + lane;
    const int e = brp[rr + 1];
    for (; k + 32 < e; k += 64) {
      s0 = fma(bv[k], vt[bci[k]], s0);
      s1 = fma(bv[k + 32], vt[bci[k + 32]], s1);
    }
    if (k < e) s0 = fma(bv[k], vt[bci[k]], s0);
    double t = subwarp_sum<32>(s0 + s1);
    const double dr = sm[L.d_b + rr], wr = vb[rr];
    const double z = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, t), dr), wr);
    const double yb = __dadd_rn(t, __dmul_rn(dr, wr));
    if (lane == 0) {
      sm[L.z_b + rr] = z;
      sm[L.y_b + rr] = yb;
      acc += t * z + wr * yb;
    }
  }
  // rows of H (warp per row): (H v)_j on own rows
  for (int hh = warp; hh < nh; hh += nw) {
    double s0 = 0.0, s1 = 0.0;
    int k = hrp[hh] + lane;
    const int e = hrp[hh + 1];
    for (; k + 32 < e; k += 64) {
      s0 = fma(hv[k], vt[hci[k]], s0);
      s1 = fma(hv[k + 32], vt[hci[k + 32]], s1);
    }
    if (k < e) s0 = fma(hv[k], vt[hci[k]], s0);
    const double hu = subwarp_sum<32>(s0 + s1);
    if (lane == 0) {
      sm[L.hu + hh] = hu;
      acc += vt[me.h0 + hh] * hu;
    }
  }
  __syncthreads();
  // B'z partial over own rows (thread per column, CSC, fixed order) + own H rows
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    int k = ccp[j];
    const int e = ccp[j + 1];
    for (; k + 1 < e; k += 2) {
      s0 = fma(cv[k], sm[L.z_b + cri[k]], s0);
      s1 = fma(cv[k + 1], sm[L.z_b + cri[k + 1]], s1);
    }
    if (k < e) s0 = fma(cv[k], sm[L.z_b + cri[k]], s0);
    double pj = s0 + s1;
    if (j >= me.h0 && j < me.h1) pj += sm[L.hu + j - me.h0];
    sm[L.pub + j] = pj;
  }
  return acc;
}

// y_top = sum over CTAs (rank order) of the published partials + q v_t;
// returns sum_j v_j q_j v_j (identical in every CTA)
__device__ double cl_gather_top(const ClParams& P, const ClLayout& L, double* sm, const double* vt, double* red) {
  double acc = 0.0;
  for (int j = threadIdx.x; j < P.n; j += blockDim.x) {
    double v[QPK_CL_MAXC];
#pragma unroll
    for (int c = 0; c < QPK_CL_MAXC; ++c) v[c] = c < P.C ? ld_remote(sm + L.pub + j, (unsigned)c) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < QPK_CL_MAXC; ++c) s += v[c];           // CTA order (zeros past C)
    const double qv = __dmul_rn(sm[L.q_t + j], vt[j]);
    sm[L.y_t + j] = __dadd_rn(s, qv);
    acc += vt[j] * qv;
  }
  return cl_block_sum(acc, red);
}

// sums over the cluster (CTA order) of published scalar slots a and b: warp 0
// loads one value per lane and adds them in lane order; the totals go through
// this CTA's own shared memory (scal[8 + slot]) to every thread
__device__ __forceinline__ void cl_sum_scal2(const ClParams& P, const ClLayout& L, double* sm, int a, int b,
                                             double& sa, double& sb) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const double va = lane < P.C ? ld_remote(sm + L.scal + a, (unsigned)lane) : 0.0;
    const double vb = lane < P.C ? ld_remote(sm + L.scal + b, (unsigned)lane) : 0.0;
    double ta = 0.0, tb = 0.0;
    for (int c = 0; c < P.C; ++c) {
      ta += __shfl_sync(0xffffffffu, va, c);
      tb += __shfl_sync(0xffffffffu, vb, c);
    }
    if (lane == 0) { sm[L.scal + 8 + a] = ta; sm[L.scal + 8 + b] = tb; }
  }
  __syncthreads();
  sa = sm[L.scal + 8 + a];
  sb = sm[L.scal + 8 + b];
}
__device__ __forceinline__ double cl_sum_scal(const ClParams& P, const ClLayout& L, double* sm, int slot) {
  double a, b;
  cl_sum_scal2(P, L, sm, slot, slot, a, b);
  return a;
}

// explicit residual r = rhs - K x; returns ||r|| (identical in every CTA).
// store: keep it as the new r (restart) or only its norm (final).
__device__ double cl_true_residual(const ClParams& P, const ClCta& me, const ClLayout& L, double* sm,
                                   const double* xt, const double* xb, bool store) {
  namespace cgx = cooperative_groups;
  double* red = sm + L.red;
  const int mr = me.r1 - me.r0;
  const double pa = cl_apply(P, me, L, sm, xt, xb);
  (void)pa;
  cgx::this_cluster().sync();                                   // partials published
  cl_gather_top(P, L, sm, xt, red);
  double rrb = 0.0, rrt = 0.0;
  for (int i = threadIdx.x; i < mr; i += blockDim.x) {
    const double ri = __dsub_rn(sm[L.rhs_b + i], sm[L.y_b + i]);
    if (store) sm[L.r_b + i] = ri;
    rrb += ri * ri;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < P.n; j += blockDim.x) {
    const double ri = __dsub_rn(sm[L.rhs_t + j], sm[L.y_t + j]);
    if (store) sm[L.r_t + j] = ri;
    rrt += ri * ri;
  }
  rrb = cl_block_sum(rrb, red);
  rrt = cl_block_sum(rrt, red);
  if (threadIdx.x == 0) sm[L.scal + 4] = rrb;
  cgx::this_cluster().sync();                                   // norms published
  return sqrt(rrt + cl_sum_scal(P, L, sm, 4));
}

struct ClOut {
  int iterations, converged, status, restarts, applies, result_buf;
  double final_norm, threshold, rhs_norm;
  unsigned long long phase_ns[4];
};

__global__ void __launch_bounds__(QPK_CL_THREADS, 1) k_pcg_cluster(ClParams P) {
  namespace cgx = cooperative_groups;
  extern __shared__ __align__(16) double sm[];
  const unsigned rank = cgx::this_cluster().block_rank();
  const ClCta me = P.ctas[rank];
  const int n = P.n, mr = me.r1 - me.r0, nh = me.h1 - me.h0;
  const ClLayout L = cl_layout(n, mr, nh, me.bytes);
  double* red = sm + L.red;
  // ---- load: operator blob, diagonals, rhs; x = 0, r = rhs (linalg.py:85-87)
  {
    const int4* src = reinterpret_cast<const int4*>(P.blob + P.blob_off[rank]);
    int4* dst = reinterpret_cast<int4*>(reinterpret_cast<unsigned char*>(sm) + L.blob);
    for (int i = threadIdx.x; i < me.bytes / 16; i += blockDim.x) dst[i] = src[i];
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double b = P.rhs[j];
      sm[L.rhs_t + j] = b; sm[L.r_t + j] = b; sm[L.x_t + j] = 0.0; sm[L.xb_t + j] = 0.0;
      sm[L.q_t + j] = P.q[j]; sm[L.mi_t + j] = P.minv[j]; sm[L.p_t + j] = 0.0;
    }
    for (int i = threadIdx.x; i < mr; i += blockDim.x) {
      const double b = P.rhs[n + me.r0 + i];
      sm[L.rhs_b + i] = b; sm[L.r_b + i] = b; sm[L.x_b + i] = 0.0; sm[L.xb_b + i] = 0.0;
      sm[L.d_b + i] = P.d[me.r0 + i]; sm[L.mi_b + i] = P.minv[n + me.r0 + i]; sm[L.p_b + i] = 0.0;
    }
  }
  __syncthreads();
  ClOut* out = reinterpret_cast<ClOut*>(P.out);
  const bool writer = rank == 0 && threadIdx.x == 0;
  // ||rhs||: the top part is replicated (counted locally), the bottom rows owned
  double rr_t = 0.0, rr_b = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) rr_t += sm[L.rhs_t + j] * sm[L.rhs_t + j];
  for (int i = threadIdx.x; i < mr; i += blockDim.x) rr_b += sm[L.rhs_b + i] * sm[L.rhs_b + i];
  rr_t = cl_block_sum(rr_t, red);
  rr_b = cl_block_sum(rr_b, red);
  if (threadIdx.x == 0) sm[L.scal + 4] = rr_b;
  cgx::this_cluster().sync();
  const double rhs_norm = sqrt(rr_t + cl_sum_scal(P, L, sm, 4));
  const double thr = P.rel ? P.tol * rhs_norm : P.tol;           // linalg.py:83
  double rnorm = rhs_norm, best_rnorm = rhs_norm;
  int restarts = 0, applies = 0, status = 0, conv = 0;
  long long iters = 0;
  if (writer && P.hist) P.hist[0] = rnorm;
  bool done = false;
  if (rnorm <= thr) { conv = 1; done = true; }                      // linalg.py:93-94
  bool restart = true;
  double rz = 0.0, beta = 0.0;
  for (long long k = 1; !done && k <= P.max_iters; ++k) {
    // ---- direction: z = M^-1 r, p = z (+ beta p); top replicated, bottom owned
    double rzt = 0.0, rzb = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double rj = sm[L.r_t + j];
      const double zj = __dmul_rn(sm[L.mi_t + j], rj);
      rzt += rj * zj;
      sm[L.p_t + j] = restart ? zj : __dadd_rn(zj, __dmul_rn(beta, sm[L.p_t + j]));
    }
    for (int i = threadIdx.x; i < mr; i += blockDim.x) {
      const double ri = sm[L.r_b + i];
      const double zi = __dmul_rn(sm[L.mi_b + i], ri);
      rzb += ri * zi;
      sm[L.p_b + i] = restart ? zi : __dadd_rn(zi, __dmul_rn(beta, sm[L.p_b + i]));
    }
    if (restart) {
      rzt = cl_block_sum(rzt, red);
      rzb = cl_block_sum(rzb, red);
    }
    __syncthreads();
    // ---- y = K p (linalg.py:100)
    double part = cl_apply(P, me, L, sm, sm + L.p_t, sm + L.p_b);
    ++applies;
    part = cl_block_sum(part, red);
    if (threadIdx.x == 0) { sm[L.scal + 0] = part; sm[L.scal + 1] = rzb; }
    cgx::this_cluster().sync();                                     // barrier #1
    const double pq = cl_gather_top(P, L, sm, sm + L.p_t, red);
    double s_pap, s_rzb;
    cl_sum_scal2(P, L, sm, 0, 1, s_pap, s_rzb);
    if (restart) rz = rzt + s_rzb;
    const double pap = pq + s_pap;
    if (pap <= 0.0) {                                               // linalg.py:102-103
      status = QPK_PCG_BREAKDOWN; iters = k - 1; rnorm = best_rnorm; done = true;
      break;
    }
    const double alpha = rz / pap;
    // ---- x += alpha p; r -= alpha y; r'r, r'z
    double rrt = 0.0, rrb = 0.0, rzt2 = 0.0, rzb2 = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      sm[L.x_t + j] = __dadd_rn(sm[L.x_t + j], __dmul_rn(alpha, sm[L.p_t + j]));
      const double ri = __dsub_rn(sm[L.r_t + j], __dmul_rn(alpha, sm[L.y_t + j]));
      sm[L.r_t + j] = ri;
      rrt += ri * ri;
      rzt2 += ri * __dmul_rn(sm[L.mi_t + j], ri);
    }
    for (int i = threadIdx.x; i < mr; i += blockDim.x) {
      sm[L.x_b + i] = __dadd_rn(sm[L.x_b + i], __dmul_rn(alpha, sm[L.p_b + i]));
      const double ri = __dsub_rn(sm[L.r_b + i], __dmul_rn(alpha, sm[L.y_b + i]));
      sm[L.r_b + i] = ri;
      rrb += ri * ri;
      rzb2 += ri * __dmul_rn(sm[L.mi_b + i], ri);
    }
    block_sum4(rrt, rzt2, rrb, rzb2, red);
    if (threadIdx.x == 0) { sm[L.scal + 2] = rrb; sm[L.scal + 3] = rzb2; }
    cgx::this_cluster().sync();                                     // barrier #2
    double s_rr, s_rz;
    cl_sum_scal2(P, L, sm, 2, 3, s_rr, s_rz);
    rnorm = sqrt(rrt + s_rr);
    const double rz_next = rzt2 + s_rz;
    iters = k;
    if (writer && P.hist) P.hist[k] = rnorm;
    if (rnorm < best_rnorm) {                                       // linalg.py:110-111
      best_rnorm = rnorm;
      for (int j = threadIdx.x; j < n; j += blockDim.x) sm[L.xb_t + j] = sm[L.x_t + j];
      for (int i = threadIdx.x; i < mr; i += blockDim.x) sm[L.xb_b + i] = sm[L.x_b + i];
    }
    if (rnorm <= thr) {                                             // linalg.py:112-125
      __syncthreads();
      const double tn = cl_true_residual(P, me, L, sm, sm + L.x_t, sm + L.x_b, true);
      ++applies;
      if (tn <= thr) { conv = 1; rnorm = tn; done = true; break; }
      ++restarts;
      rnorm = tn;
      if (rnorm < best_rnorm) {
        best_rnorm = rnorm;
        for (int j = threadIdx.x; j < n; j += blockDim.x) sm[L.xb_t + j] = sm[L.x_t + j];
        for (int i = threadIdx.x; i < mr; i += blockDim.x) sm[L.xb_b + i] = sm[L.x_b + i];
      }
      restart = true;
      __syncthreads();
      continue;
    }
    beta = rz_next / rz;                                            // linalg.py:126-130
    rz = rz_next;
    restart = false;
    __syncthreads();
  }
  // result buffer: 0 = x (converged), 1 = best iterate (cap / breakdown)
  int result = 0;
  if (!done) {
    // iteration cap: the true residual of the best iterate (linalg.py:132-133)
    __syncthreads();
    const double tn = cl_true_residual(P, me, L, sm, sm + L.xb_t, sm + L.xb_b, false);
    ++applies;
    rnorm = tn;
    conv = tn <= thr ? 1 : 0;
    iters = P.max_iters;
    result = 1;
  } else if (status == QPK_PCG_BREAKDOWN) {
    result = 1;
  }
  __syncthreads();
  const double* rt = sm + (result ? L.xb_t : L.x_t);
  const double* rb = sm + (result ? L.xb_b : L.x_b);
  if (rank == 0)
    for (int j = threadIdx.x; j < n; j += blockDim.x) P.x_out[j] = rt[j];
  for (int i = threadIdx.x; i < mr; i += blockDim.x) P.x_out[n + me.r0 + i] = rb[i];
  if (writer) {
    out->iterations = (int)iters; out->converged = conv; out->status = status;
    out->restarts = restarts; out->applies = applies; out->result_buf = 0;   // x_out is x[0]
    out->final_norm = rnorm; out->threshold = thr; out->rhs_norm = rhs_norm;
    for (int i = 0; i < 4; ++i) out->phase_ns[i] = 0;
  }
  cgx::this_cluster().sync();                                       // no CTA exits while others read its smem
}

}  // namespace qpk
