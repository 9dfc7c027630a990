// qpk_device.cuh -- device-side phases of the doubly augmented KKT operator
// and of Jacobi-PCG, shared by the persistent cooperative solver kernel and
// the standalone apply / Jacobi kernels (qpk.cu).
//
// Data layout in HBM:
//   B      literal reference B = (C; A_l; -A_u) (kkt.py:177-184, 206-207),
//          CSR with int32 columns, fp64 values, every row start padded to a
//          multiple of 4 elements (padding: column -1, value 0) so a lane
//          reads one int4 + two double2 per chunk of 4 nonzeros.
//   B^T    optional CSC copy (int32 rows, fp64 values) for the deterministic,
//          gather-only B'z pass.
//   vectors of length N = n + m_B, top (n) first then bottom (m_B), exactly
//          the reference's concatenation order (kkt.py:221).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define QPK_BLOCK 256
#define QPK_KMAX 64
#ifndef QPK_PCG_MIN_BLOCKS
#define QPK_PCG_MIN_BLOCKS 4
#endif

namespace qpk {

enum { HESS_DIAG = 0, HESS_CSR = 1, HESS_DENSE = 2, HESS_LOWRANK = 3 };

struct Hess {
  int kind;
  const double* h;                      // DIAG: d ; LOWRANK: h0
  const int* rp; const int* ci; const double* v; int lanes;  // CSR (full symmetric storage)
  const int* rows; int nrows;           // CSR, sharded: the H rows this rank applies (null: all n rows)
  const double* dense;                  // n x n row-major
  const double* sym;                    // dense H as packed upper 64 x 64 tiles (null: not built)
  const int4* chunks;                   // sym work units {I, J0, J1, tile of (I, J0)}
  int nchunks;
  double* symp;                         // sym partials, 64 doubles each: [unit ch] its tile-row sums, then
                                        // [nchunks + tile t] the column sums of off-diagonal tile t
  const int* rowchunk;                  // units of tile row I: [rowchunk[I], rowchunk[I+1])
  const double* U; const double* w; int k;                  // LOWRANK: U n x k row-major
};

struct Op {
  int n, m;
  const int* rp; const int* ci; const double* bv;           // padded CSR of B
  const int* cp; const int* ri; const double* cv; int csc_lanes;  // CSC of B (may be null)
  Hess H;
  const double* d;                      // d_diag, m
  const double* q;                      // q_diag_extra, n
  int top_owner;                        // rank 0: applies a dense / low-rank H (one owner; single GPU: 1)
  // Sharded runs replicate the top block (n) on every rank.  Each rank OWNS
  // the slice [t_lo, t_hi) of it: it alone adds diag(Q) p, the sparse-H rows
  // and the dot-product terms of those entries, so every replicated term is
  // counted exactly once by the all-reduce -- and the work is spread over the
  // ranks instead of sitting on rank 0.  Single GPU: [0, n).
  int t_lo, t_hi;
  // slot engine only: the first ndense rows of B are dense (e.g. the SVM dual's
  // y' alpha = 0 row, n entries) and are handled as dense vectors outside the
  // row pass (dot partials in the top kernel, k_slot_dense); r0 = ndense rows
  // are skipped by phase_rows.  Zero everywhere else.
  int r0, ndense;
  const double* cdense;                 // ndense x n row-major
};

// partial-sum slots (slot-major: part[slot * G + cta])
#define QPK_DENSE_ROWS_MAX 4
enum { SLOT_ROWS = 0, SLOT_PREP = 1, SLOT_RR = 2, SLOT_RZ = 3, SLOT_AUX = 4, SLOT_AUX2 = 5, SLOT_S = 6,
       SLOT_DR = SLOT_S + QPK_KMAX, SLOT_F = SLOT_DR + QPK_DENSE_ROWS_MAX, NSLOTS = SLOT_F + 6 };
// SLOT_F .. SLOT_F+5 (sharded tile format, one all-reduce per iteration): this rank's bottom-block
// sums  sum r^2, sum r y, sum y^2  and the same weighted by M^-1 = 1/d -- see k_slot_update

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- loads ----
// Streaming loads of matrix data (read once per pass, far larger than L2):
// no L1 allocation and an L2 evict-first policy, so the stream does not flush
// the vectors (u, y, z, ...) the same pass gathers from and scatters into.
__device__ __forceinline__ unsigned long long stream_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));   // pure: hoisted out of loops
  return pol;
}
__device__ __forceinline__ int4 ld_stream_i4(const int* p) {
  int4 r;
#ifndef QPK_NO_STREAM_HINT
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(stream_policy()));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#endif
  return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const double* p) {
  double2 r;
#ifndef QPK_NO_STREAM_HINT
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(stream_policy()));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
#endif
  return r;
}

// ------------------------------------------------ programmatic launch ----
// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialisation attribute may be scheduled while its predecessor
// drains; it must not touch the predecessor's outputs before pdl_wait().  A
// kernel triggers its dependent only after its own pdl_wait(), so code before
// pdl_wait() may read anything produced two or more kernels back.  Both are
// no-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ----------------------------------------------------------- reductions ----
// Sum over the calling block; result broadcast to every thread.  Fixed tree:
// deterministic for a fixed blockDim.
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();                       // protect red[] from a previous use
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// Sum of one partial slot over all G blocks, in a fixed order: every block
// computes a bitwise identical value, so scalar control decisions (alpha,
// beta, convergence, breakdown) agree across the grid without another sync.
__device__ __forceinline__ double grid_total(const double* part, int G, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < G; i += blockDim.x) s += part[i];
  return block_sum(s, red);
}

// Two slot totals in one pass (one block reduction instead of two; each total
// keeps the fixed order of grid_total, so results are bitwise those of two
// grid_total calls).
__device__ __forceinline__ void grid_total2(const double* pa, int ga, const double* pb, int gb, double* red,
                                            double& ta, double& tb) {
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < ga; i += blockDim.x) a += pa[i];
  for (int i = threadIdx.x; i < gb; i += blockDim.x) b += pb[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) { red[warp] = a; red[16 + warp] = b; }
  __syncthreads();
  a = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
  b = (lane < (int)(blockDim.x >> 5)) ? red[16 + lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  ta = a;
  tb = b;
}

template <int L>
__device__ __forceinline__ double subwarp_sum(double s) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// entry i of an N-vector is counted by this rank in a dot product: every
// bottom entry it holds, and the top entries of its slice
__device__ __forceinline__ bool owns(const Op& op, int i) { return i >= op.n || (i >= op.t_lo && i < op.t_hi); }

// ------------------------------------------------------------ prep(v) ------
// y_top = Q_diag-part * v (the part of Q u = H u + q_extra*u that is diagonal)
// for element j, returns its contribution v_j * y_j to v'Kv.
__device__ __forceinline__ double prep_elem(const Op& op, int j, double vj, double* y) {
  if (j < op.t_lo || j >= op.t_hi) { y[j] = 0.0; return 0.0; }     // not this rank's slice: B'z partial only
  const int kind = op.H.kind;
  double qv = __dmul_rn(__ldg(op.q + j), vj);
  double t;
  if (kind == HESS_DIAG || kind == HESS_LOWRANK)
    t = __dadd_rn(__dmul_rn(__ldg(op.H.h + j), vj), qv);     // hessian_apply + q*u (kkt.py:186-187)
  else
    t = qv;                                                 // H u added in the rows phase
  y[j] = t;
  return vj * t;
}

// accumulate the low-rank projection s = U' v over this thread's elements
__device__ __forceinline__ void lowrank_accum(const Op& op, int j, double vj, double* sacc) {
  const double* urow = op.H.U + (size_t)j * op.H.k;
  for (int kk = 0; kk < op.H.k; ++kk) sacc[kk] += urow[kk] * vj;
}

__device__ __forceinline__ void lowrank_flush(const Op& op, double* sacc, double* part, int G, double* red) {
  for (int kk = 0; kk < op.H.k; ++kk) {
    double t = block_sum(sacc[kk], red);
    if (threadIdx.x == 0) part[(SLOT_S + kk) * G + blockIdx.x] = t;
  }
}

// prep phase over the top block: y_top = diag part of Q v; partial v'(diag Q)v
__device__ void phase_prep(const Op& op, const double* v, double* y, double* part, int G, double* red) {
  double acc = 0.0;
  double sacc[QPK_KMAX];
  const bool lr = op.H.kind == HESS_LOWRANK;
  if (lr) for (int kk = 0; kk < op.H.k; ++kk) sacc[kk] = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < op.n; j += gridDim.x * blockDim.x) {
    double vj = v[j];
    acc += prep_elem(op, j, vj, y);
    if (lr) lowrank_accum(op, j, vj, sacc);
  }
  double t = block_sum(acc, red);
  if (threadIdx.x == 0) part[SLOT_PREP * G + blockIdx.x] = t;
  if (lr) lowrank_flush(op, sacc, part, G, red);
}

// ------------------------------------------------------------ rows(v) ------
// Bottom-half work of the PCG direction update, fused into the rows pass
// (which is bound by random L2 requests, so this streaming is nearly free):
//   x_b <- x_b + alpha_prev p_b      (lazy x update of the previous iteration)
//   p_b <- (1/d) r_b (+ beta p_b)    (z = M^-1 r with M_bottom = D, linalg.py:126-130)
struct RowFuse {
  const double* r;
  const double* xsrc;
  double* xdst;
  double alpha_prev, beta;
  int restart, xupd;
};

// One pass over B: t = B u; z = 2 t / d + w; y_bottom = t + d w (kkt.py:217-220);
// B' z either scattered with fp64 atomics into y_top (CSC == false) or z
// stored for the gather pass (CSC == true).  Then the non-diagonal Hessian
// part H u (CSR / dense / low-rank) is added to y_top.  Accumulates
// t z + w y_bottom (+ u'H u) so that v'Kv is known after this phase:
//   v'Kv = u'Q u + sum_r z_r t_r + sum_r w_r y_r   (since u'B'z = t'z).
// Non-diagonal Hessian part of Q u (CSR / dense / low-rank), atomically added
// to y_top; returns this thread's share of u'H'u (H' = H minus its diagonal
// part handled in prep).  Grid-stride over the rows of H.
__device__ __forceinline__ double hess_rows(const Op& op, const double* u, double* y, const double* part, int G,
                                            double* red, double* s_lr) {
  double acc = 0.0;
  const int kind = op.H.kind;
  if (kind != HESS_CSR && !op.top_owner) return 0.0;  // dense / low-rank H: one owner rank
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  if (kind == HESS_CSR) {
    // the H rows this rank applies (sharded: its row list; single GPU: all rows)
    const int LH = op.H.lanes;                       // power of two <= 32
    const int lh = threadIdx.x & (LH - 1);
    const int per = 32 / LH, sw = (threadIdx.x & 31) / LH;
    const int nr = op.H.rows ? op.H.nrows : op.n;
    for (long long jb = (long long)gwarp * per; jb < nr; jb += (long long)nwarp * per) {
      const int q = (int)jb + sw;
      const int j = q < nr ? (op.H.rows ? __ldg(op.H.rows + q) : q) : 0;
      double s = 0.0;
      if (q < nr) {
        const int b = __ldg(op.H.rp + j), e = __ldg(op.H.rp + j + 1);
        for (int kk = b + lh; kk < e; kk += LH) s = fma(__ldg(op.H.v + kk), u[__ldg(op.H.ci + kk)], s);
      }
      for (int o = LH / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (q < nr && lh == 0) { atomicAdd(y + j, s); acc += u[j] * s; }
    }
  } else if (kind == HESS_DENSE && op.H.sym) {
    return 0.0;                                        // packed symmetric tiles: hess_sym (own launch)
  } else if (kind == HESS_DENSE) {
    const int ln = threadIdx.x & 31;
    for (int j = gwarp; j < op.n; j += nwarp) {
      const double* row = op.H.dense + (size_t)j * op.n;
      double s = 0.0;
      if ((op.n & 1) == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0) {
        // 16-byte loads, four independent chains (SVM dual: H is the whole operator)
        const double2* r2 = reinterpret_cast<const double2*>(row);
        const double2* u2 = reinterpret_cast<const double2*>(u);
        const int h = op.n >> 1;
        double s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int c = ln;
        for (; c + 32 < h; c += 64) {
          const double2 a = __ldg(r2 + c), b = __ldg(r2 + c + 32);
          const double2 x = u2[c], z = u2[c + 32];
          s = fma(a.x, x.x, s); s1 = fma(a.y, x.y, s1);
          s2 = fma(b.x, z.x, s2); s3 = fma(b.y, z.y, s3);
        }
        for (; c < h; c += 32) {
          const double2 a = __ldg(r2 + c), x = u2[c];
          s = fma(a.x, x.x, s); s1 = fma(a.y, x.y, s1);
        }
        s = (s + s1) + (s2 + s3);
      } else {
        for (int c = ln; c < op.n; c += 32) s = fma(__ldg(row + c), u[c], s);
      }
      s = subwarp_sum<32>(s);
      if (ln == 0) { atomicAdd(y + j, s); acc += u[j] * s; }
    }
  } else if (kind == HESS_LOWRANK) {
    // s = U'u was accumulated in the prep phase; fold w in and apply U
    const int k = op.H.k;
    for (int kk = 0; kk < k; ++kk) {
      double t = grid_total(part + (SLOT_S + kk) * G, G, red);
      if (threadIdx.x == 0) s_lr[kk] = t;
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double e2 = 0.0;
      for (int kk = 0; kk < k; ++kk) e2 += op.H.w[kk] * s_lr[kk] * s_lr[kk];
      acc += e2;                                      // u'U diag(w) U'u
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < op.n; j += gridDim.x * blockDim.x) {
      const double* urow = op.H.U + (size_t)j * k;
      double s = 0.0;
      for (int kk = 0; kk < k; ++kk) s += urow[kk] * (op.H.w[kk] * s_lr[kk]);
      atomicAdd(y + j, s);
    }
  }
  return acc;
}

// H u for a dense SYMMETRIC H stored as its upper 64 x 64 tiles (half the
// bytes of the row-major matrix).  One warp per work unit (a run of <= 2 tiles
// of one tile row I): lane l holds columns 2l, 2l+1 of each 512-byte tile row
// (one coalesced 16-byte load per lane per row, 32 in flight), so
//   columns:  (H_IJ' u_I)_c accumulates in registers  -> y_J  (J != I)
//   rows:     (H_IJ u_J)_r needs a sum over lanes: 32 rows at a time, a
//             transposed butterfly (31 shuffles) leaves row r0+l in lane l;
//             accumulated over the unit's tiles -> y_I
// No atomics: every unit stores its 64 row sums and every off-diagonal tile its
// 64 column sums as partials (op.H.symp); sym_combine adds them into y in a
// fixed order (bitwise reproducible) and returns u'H u.
template <int RG>
__device__ __forceinline__ double hess_sym_t(const Op& op, const double* u, double* y) {
  if (!op.top_owner) return 0.0;
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
  const int n = op.n;
  double acc = 0.0;
  for (int ch = gwarp; ch < op.H.nchunks; ch += nwarp) {
    const int4 cd = __ldg(op.H.chunks + ch);
    const int rI = cd.x * 64;
    const double uI0 = (rI + lane < n) ? u[rI + lane] : 0.0;
    const double uI1 = (rI + 32 + lane < n) ? u[rI + 32 + lane] : 0.0;
    double ry0 = 0.0, ry1 = 0.0;
    for (int J = cd.y, t = cd.w; J < cd.z; ++J, ++t) {
      const double2* tile = reinterpret_cast<const double2*>(op.H.sym + (size_t)t * 4096);
      const int cJ = J * 64 + 2 * lane;
      const double uJx = cJ < n ? u[cJ] : 0.0, uJy = cJ + 1 < n ? u[cJ + 1] : 0.0;
      double cz0 = 0.0, cz1 = 0.0;
#pragma unroll
      for (int g = 0; g < 64 / RG; ++g) {
        double p[RG];
        double2 a[RG];
#pragma unroll
        for (int k = 0; k < RG; ++k) a[k] = __ldg(tile + (g * RG + k) * 32 + lane);
        const double uIg = (g * RG < 32) ? uI0 : uI1;
#pragma unroll
        for (int k = 0; k < RG; ++k) {
          p[k] = fma(a[k].x, uJx, a[k].y * uJy);
          const double ur = __shfl_sync(0xffffffffu, uIg, (g * RG + k) & 31);
          cz0 = fma(a[k].x, ur, cz0);
          cz1 = fma(a[k].y, ur, cz1);
        }
        // transposed butterfly: row g*RG + (lane % RG) ends in p[0]
        if (RG < 32) {
#pragma unroll
          for (int k = 0; k < RG; ++k) p[k] += __shfl_xor_sync(0xffffffffu, p[k], 16);
        }
#pragma unroll
        for (int o = RG / 2; o >= 1; o >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int k = 0; k < o; ++k) {
            const double send = up ? p[k] : p[k + o];
            const double keep = up ? p[k + o] : p[k];
            p[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        // lane l holds row g*RG + (l % RG): keep it in the lane that owns that row
        const int row = g * RG + (lane % RG);
        if (row == lane) ry0 += p[0];
        else if (row == 32 + lane) ry1 += p[0];
      }
      if (J != cd.x)                                   // column sums of tile (I, J): slot J (J - 1) / 2 + I
        reinterpret_cast<double2*>(op.H.symp + ((size_t)op.H.nchunks + (size_t)J * (J - 1) / 2 + cd.x) * 64)[lane] =
            make_double2(cz0, cz1);
    }
    double* rp_ = op.H.symp + (size_t)ch * 64;
    rp_[lane] = ry0;
    rp_[32 + lane] = ry1;
  }
  return acc;
}

// y_j += (H u)_j from the partials of hess_sym_t, in a fixed order.  One block
// per tile column J (grid-stride): its items are the units of tile row J (row
// sums) followed by the tiles (I, J), I = 0 .. J-1 (column sums); thread
// (cc = tid % 64, part = tid / 64) adds the items part, part + P, ... for
// output 64 J + cc, the P parts are then added in order.  Returns this thread's
// share of u'H u.  `sh` holds blockDim.x doubles.
__device__ __forceinline__ double sym_combine(const Op& op, const double* u, double* y, double* sh) {
  const int n = op.n, nt = (n + 63) >> 6;
  const int cc = threadIdx.x & 63, part = threadIdx.x >> 6, P = blockDim.x >> 6;
  const double* rowp = op.H.symp + cc;
  const double* colp = op.H.symp + (size_t)op.H.nchunks * 64 + cc;
  double acc = 0.0;
  for (int J = blockIdx.x; J < nt; J += gridDim.x) {
    // two contiguous runs of 64-double partials: the units of tile row J, then
    // the tiles (0 .. J-1, J) (stored by tile column: slot J (J - 1) / 2 + I)
    const int c0 = __ldg(op.H.rowchunk + J), nrow = __ldg(op.H.rowchunk + J + 1) - c0;
    const double* run[2] = {rowp + (size_t)c0 * 64, colp + (size_t)J * (J - 1) / 2 * 64};
    const int len[2] = {nrow, J};
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const double* q = run[w];
      int k = part;
      for (; k + 3 * P < len[w]; k += 4 * P) {
        const double a0 = q[(size_t)k * 64], a1 = q[(size_t)(k + P) * 64], a2 = q[(size_t)(k + 2 * P) * 64],
                     a3 = q[(size_t)(k + 3 * P) * 64];
        s += a0; s += a1; s += a2; s += a3;
      }
      for (; k < len[w]; k += P) s += q[(size_t)k * 64];
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    if (part == 0) {
      double t = s;
      for (int q = 1; q < P; ++q) t += sh[q * 64 + cc];
      const int j = J * 64 + cc;
      if (j < n) { y[j] += t; acc += u[j] * t; }
    }
    __syncthreads();
  }
  return acc;
}

#ifndef QPK_SYM_RG
#define QPK_SYM_RG 32          // tile rows per transposed reduction (32 loads in flight per lane)
#endif
__device__ __noinline__ double hess_sym(const Op& op, const double* u, double* y) {
  return hess_sym_t<QPK_SYM_RG>(op, u, y);
}

template <int L>
__device__ __forceinline__ void load_chunk(const Op& op, int k, int e, int4& c, double2& v0, double2& v1) {
  c = make_int4(-1, -1, -1, -1);
  v0 = make_double2(0.0, 0.0);
  v1 = v0;
  if (k < e) { c = ld_stream_i4(op.ci + k); v0 = ld_stream_d2(op.bv + k); v1 = ld_stream_d2(op.bv + k + 2); }
}

// B-row loop, software-pipelined: while step i's gathers are in flight the
// index/value chunk of step i+1 and the row pointers of step i+2 load.
// Returns this thread's partial of t z + w y_b; *rzb gets r_b z_b (FUSE).
template <int L, bool CSC, bool FUSE>
__device__ __forceinline__ double rows_loop_pipelined(const Op& op, double* v, double* y, double* zb,
                                                      const RowFuse& f, double* rzb_out) {
  const double* u = v;
  double* w = v + op.n;
  double acc = 0.0, rzb = 0.0;
  const int lane = threadIdx.x & (L - 1);
  constexpr int RPW = 32 / L;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  const int sub = (threadIdx.x & 31) / L;
  const long long step = (long long)nwarp * RPW;
  long long rb = op.r0 + (long long)gwarp * RPW;
  int r = (int)rb + sub;
  bool act = rb < op.m && r < op.m;
  int b = 0, e = 0;
  if (act) { b = __ldg(op.rp + r); e = __ldg(op.rp + r + 1); }
  int4 c0; double2 v0, v1;
  load_chunk<L>(op, b + 4 * lane, e, c0, v0, v1);
  long long rb1 = rb + step;
  int r1 = (int)rb1 + sub;
  bool act1 = rb1 < op.m && r1 < op.m;
  int b1 = 0, e1 = 0;
  if (act1) { b1 = __ldg(op.rp + r1); e1 = __ldg(op.rp + r1 + 1); }
  for (; rb < op.m; rb += step) {
    int4 cn; double2 vn0, vn1;
    load_chunk<L>(op, b1 + 4 * lane, e1, cn, vn0, vn1);
    const long long rb2 = rb1 + step;
    const int r2 = (int)rb2 + sub;
    const bool act2 = rb2 < op.m && r2 < op.m;
    int b2 = 0, e2 = 0;
    if (act2) { b2 = __ldg(op.rp + r2); e2 = __ldg(op.rp + r2 + 1); }
    double dr = 1.0, wr = 0.0, rres = 0.0, xs = 0.0;
    if (act) {
      dr = __ldg(op.d + r);
      wr = w[r];
      if (FUSE) {
        rres = f.r[op.n + r];
        if (f.xupd && lane == 0) xs = f.xsrc[op.n + r];
      }
    }
    double s = 0.0;
    if (c0.x >= 0) s = fma(v0.x, u[c0.x], s);
    if (c0.y >= 0) s = fma(v0.y, u[c0.y], s);
    if (c0.z >= 0) s = fma(v1.x, u[c0.z], s);
    if (c0.w >= 0) s = fma(v1.y, u[c0.w], s);
    for (int k = b + 4 * lane + 4 * L; k < e; k += 4 * L) {
      int4 c = ld_stream_i4(op.ci + k);
      double2 a0 = ld_stream_d2(op.bv + k), a1 = ld_stream_d2(op.bv + k + 2);
      if (c.x >= 0) s = fma(a0.x, u[c.x], s);
      if (c.y >= 0) s = fma(a0.y, u[c.y], s);
      if (c.z >= 0) s = fma(a1.x, u[c.z], s);
      if (c.w >= 0) s = fma(a1.y, u[c.w], s);
    }
    const double t = subwarp_sum<L>(s);
    if (act) {
      if (FUSE) {
        const double zr = __dmul_rn(1.0 / dr, rres);
        if (f.xupd && lane == 0) f.xdst[op.n + r] = __dadd_rn(xs, __dmul_rn(f.alpha_prev, wr));
        const double pn = f.restart ? zr : __dadd_rn(zr, __dmul_rn(f.beta, wr));
        if (lane == 0) { w[r] = pn; rzb += rres * zr; }
        wr = pn;
      }
      const double z = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, t), dr), wr);
      const double yb = __dadd_rn(t, __dmul_rn(dr, wr));
      if (lane == 0) {
        y[op.n + r] = yb;
        acc += t * z + wr * yb;
        if (CSC) zb[r] = z;
      }
      if (!CSC) {
        if (c0.x >= 0) atomicAdd(y + c0.x, z * v0.x);
        if (c0.y >= 0) atomicAdd(y + c0.y, z * v0.y);
        if (c0.z >= 0) atomicAdd(y + c0.z, z * v1.x);
        if (c0.w >= 0) atomicAdd(y + c0.w, z * v1.y);
        for (int k = b + 4 * lane + 4 * L; k < e; k += 4 * L) {
          int4 c = *reinterpret_cast<const int4*>(op.ci + k);
          double2 a0 = *reinterpret_cast<const double2*>(op.bv + k);
          double2 a1 = *reinterpret_cast<const double2*>(op.bv + k + 2);
          if (c.x >= 0) atomicAdd(y + c.x, z * a0.x);
          if (c.y >= 0) atomicAdd(y + c.y, z * a0.y);
          if (c.z >= 0) atomicAdd(y + c.z, z * a1.x);
          if (c.w >= 0) atomicAdd(y + c.w, z * a1.y);
        }
      }
    }
    r = r1; act = act1; b = b1; e = e1; c0 = cn; v0 = vn0; v1 = vn1;
    rb1 = rb2; r1 = r2; act1 = act2; b1 = b2; e1 = e2;
  }
  *rzb_out = rzb;
  return acc;
}

template <int L, bool CSC, bool FUSE, bool PIPE = false>
__device__ void phase_rows(const Op& op, double* v, double* y, double* zb,
                           double* part, int G, double* red, double* s_lr, const RowFuse& f) {
  const double* u = v;
  double* w = v + op.n;
  double acc = 0.0, rzb = 0.0;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  if (PIPE) acc = rows_loop_pipelined<L, CSC, FUSE>(op, v, y, zb, f, &rzb);
  else {
  const int lane = threadIdx.x & (L - 1);
  constexpr int RPW = 32 / L;                       // rows per warp step
  const int sub_in_warp = (threadIdx.x & 31) / L;
  for (long long rb = op.r0 + (long long)gwarp * RPW; rb < op.m; rb += (long long)nwarp * RPW) {
    const int r = (int)rb + sub_in_warp;
    const bool active = r < op.m;
    int b = 0, e = 0;
    double dr = 1.0, wr = 0.0;
    if (active) {
      b = __ldg(op.rp + r); e = __ldg(op.rp + r + 1);
      dr = __ldg(op.d + r);
      wr = w[r];
      if (FUSE) {
        // every lane of the row computes the same values; lane 0 stores
        const double rr = f.r[op.n + r];
        const double zr = __dmul_rn(1.0 / dr, rr);
        if (f.xupd && lane == 0) f.xdst[op.n + r] = __dadd_rn(f.xsrc[op.n + r], __dmul_rn(f.alpha_prev, wr));
        const double pn = f.restart ? zr : __dadd_rn(zr, __dmul_rn(f.beta, wr));
        if (lane == 0) { w[r] = pn; rzb += rr * zr; }
        wr = pn;
      }
    }
    const int k0 = b + 4 * lane;
    int4 c0 = make_int4(-1, -1, -1, -1);
    double2 v0 = make_double2(0.0, 0.0), v1 = make_double2(0.0, 0.0);
    if (k0 < e) { c0 = ld_stream_i4(op.ci + k0); v0 = ld_stream_d2(op.bv + k0); v1 = ld_stream_d2(op.bv + k0 + 2); }
    double s = 0.0;
    if (c0.x >= 0) s = fma(v0.x, u[c0.x], s);
    if (c0.y >= 0) s = fma(v0.y, u[c0.y], s);
    if (c0.z >= 0) s = fma(v1.x, u[c0.z], s);
    if (c0.w >= 0) s = fma(v1.y, u[c0.w], s);
#pragma unroll 4
    for (int k = k0 + 4 * L; k < e; k += 4 * L) {   // rows longer than 4L nonzeros
      int4 c = ld_stream_i4(op.ci + k);
      double2 a0 = ld_stream_d2(op.bv + k), a1 = ld_stream_d2(op.bv + k + 2);
      if (c.x >= 0) s = fma(a0.x, u[c.x], s);
      if (c.y >= 0) s = fma(a0.y, u[c.y], s);
      if (c.z >= 0) s = fma(a1.x, u[c.z], s);
      if (c.w >= 0) s = fma(a1.y, u[c.w], s);
    }
    const double t = subwarp_sum<L>(s);
    if (!active) continue;
    const double z = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, t), dr), wr);
    const double yb = __dadd_rn(t, __dmul_rn(dr, wr));
    if (lane == 0) {
      y[op.n + r] = yb;
      acc += t * z + wr * yb;
      if (CSC) zb[r] = z;
    }
    if (!CSC) {
      if (c0.x >= 0) atomicAdd(y + c0.x, z * v0.x);
      if (c0.y >= 0) atomicAdd(y + c0.y, z * v0.y);
      if (c0.z >= 0) atomicAdd(y + c0.z, z * v1.x);
      if (c0.w >= 0) atomicAdd(y + c0.w, z * v1.y);
      for (int k = k0 + 4 * L; k < e; k += 4 * L) {
        int4 c = *reinterpret_cast<const int4*>(op.ci + k);
        double2 a0 = *reinterpret_cast<const double2*>(op.bv + k);
        double2 a1 = *reinterpret_cast<const double2*>(op.bv + k + 2);
        if (c.x >= 0) atomicAdd(y + c.x, z * a0.x);
        if (c.y >= 0) atomicAdd(y + c.y, z * a0.y);
        if (c.z >= 0) atomicAdd(y + c.z, z * a1.x);
        if (c.w >= 0) atomicAdd(y + c.w, z * a1.y);
      }
    }
  }
  }
  if (FUSE) {
    const double t2 = block_sum(rzb, red);
    if (threadIdx.x == 0) part[SLOT_AUX2 * G + blockIdx.x] = t2;
  }

  acc += hess_rows(op, u, y, part, G, red, s_lr);
  double tot = block_sum(acc, red);
  if (threadIdx.x == 0) part[SLOT_ROWS * G + blockIdx.x] = tot;
}

// CSC gather of (B'z)_j for column j by a group of LC lanes (all lanes get
// the sum).  Columns are padded to multiples of 4 entries (row index -1), so a
// lane reads one int4 of row indices + two double2 of values per chunk and has
// 4 independent z gathers in flight per chunk (two chunks per loop trip).
__device__ __forceinline__ double csc_col_sum(const Op& op, const double* zb, int j, bool valid, int lc, int LC) {
  double s0 = 0.0, s1 = 0.0;
  if (valid) {
    const int b = __ldg(op.cp + j), e = __ldg(op.cp + j + 1);
    int k = b + 4 * lc;
    for (; k + 4 * LC < e; k += 8 * LC) {
      const int4 c = ld_stream_i4(op.ri + k), d = ld_stream_i4(op.ri + k + 4 * LC);
      const double2 a0 = ld_stream_d2(op.cv + k), a1 = ld_stream_d2(op.cv + k + 2);
      const double2 b0 = ld_stream_d2(op.cv + k + 4 * LC), b1 = ld_stream_d2(op.cv + k + 4 * LC + 2);
      if (c.x >= 0) s0 = fma(a0.x, zb[c.x], s0);
      if (c.y >= 0) s0 = fma(a0.y, zb[c.y], s0);
      if (c.z >= 0) s0 = fma(a1.x, zb[c.z], s0);
      if (c.w >= 0) s0 = fma(a1.y, zb[c.w], s0);
      if (d.x >= 0) s1 = fma(b0.x, zb[d.x], s1);
      if (d.y >= 0) s1 = fma(b0.y, zb[d.y], s1);
      if (d.z >= 0) s1 = fma(b1.x, zb[d.z], s1);
      if (d.w >= 0) s1 = fma(b1.y, zb[d.w], s1);
    }
    if (k < e) {
      const int4 c = ld_stream_i4(op.ri + k);
      const double2 a0 = ld_stream_d2(op.cv + k), a1 = ld_stream_d2(op.cv + k + 2);
      if (c.x >= 0) s0 = fma(a0.x, zb[c.x], s0);
      if (c.y >= 0) s0 = fma(a0.y, zb[c.y], s0);
      if (c.z >= 0) s0 = fma(a1.x, zb[c.z], s0);
      if (c.w >= 0) s0 = fma(a1.y, zb[c.w], s0);
    }
  }
  double s = s0 + s1;
  for (int o = LC / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Visit every element i of the N-vector with its final K v value y_i.  In
// CSC mode the top entries are completed here by the gather pass.  f(i, yi)
// is called exactly once per element (by one lane).
template <bool CSC, typename F>
__device__ __forceinline__ void for_each_final(const Op& op, const double* y, const double* zb, F f) {
  const int N = op.n + op.m;
  if (!CSC) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) f(i, y[i]);
    return;
  }
  const int LC = op.csc_lanes;
  const int lc = threadIdx.x & (LC - 1);
  const int per = 32 / LC, sw = (threadIdx.x & 31) / LC;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  for (long long jb = (long long)gwarp * per; jb < op.n; jb += (long long)nwarp * per) {
    const int j = (int)jb + sw;
    const bool valid = j < op.n;
    const double yj = valid ? y[j] : 0.0;
    const double s = csc_col_sum(op, zb, j, valid, lc, LC);
    if (valid && lc == 0) f(j, yj + s);
  }
  for (int i = op.n + blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) f(i, y[i]);
}

}  // namespace qpk
