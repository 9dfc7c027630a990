// qpk_tma.cuh -- TMA-fed row-block dictionary kernel (the one-pass, atomic-
// free operator apply for banded / clustered B: the RT and SVM configs).
//
// Per CTA: 1 producer warp + QPK_DICT_WARPS consumer warps.  The producer's
// elected lane streams, tile by tile, the tile's 16-bit dictionary indices and
// fp64 values of B, its row pointers and the per-row vectors it needs (d, w =
// p_B or x_B, r_B, x_B) from HBM into a QPK_TMA_STAGES-deep ring of shared-
// memory stages with 1-D bulk async copies (cp.async.bulk ... complete_tx on
// an mbarrier; SASS UBLKCP).  Consumers wait on the stage's "full" barrier,
// process the rows from shared memory (u gathered from the block's
// dictionary copy in shared memory, B'z accumulated into per-warp shared-
// memory dictionaries, no atomics), and release the stage on its "empty"
// barrier.  Only the per-row outputs go back to HBM.
#pragma once
#include "qpk_engine.cuh"

#ifndef QPK_TMA_STAGES
#define QPK_TMA_STAGES 4
#endif
#define QPK_TILE_E 2048          // max padded entries per tile
#define QPK_TILE_R 256           // max rows per tile

namespace qpk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"r"(QPK_DICT_WARPS * 32) : "memory");
}

// tile descriptor written by the producer into its stage (visible to the
// consumers through the mbarrier's release/acquire)
struct TileDesc {
  int ra, rb;           // rows
  int e0;               // first entry copied for lci (multiple of 8)
  int e1;               // first entry copied for values (multiple of 2)
  int p0;               // first row pointer copied (multiple of 4)
  int v0;               // first row copied for d (multiple of 2)
  int w0;               // first element copied of the bottom vectors (n + row, multiple of 2)
};

struct alignas(16) TileStage {
  unsigned short lci[QPK_TILE_E + 16];
  double val[QPK_TILE_E + 8];
  int rp[QPK_TILE_R + 8];
  double d[QPK_TILE_R + 4];
  double w[QPK_TILE_R + 4];
  double r[QPK_TILE_R + 4];
  double x[QPK_TILE_R + 4];
  TileDesc t;
};

struct TmaSmem {
  TileStage st[QPK_TMA_STAGES];
  unsigned long long full[QPK_TMA_STAGES], empty[QPK_TMA_STAGES];
  double us[QPK_DICT_MAX];
  double acc[QPK_DICT_WARPS][QPK_DICT_MAX];
  double red[32];
  double s_lr[QPK_KMAX];
};

// tiles of the row blocks: tile t covers rows [tile_row[t], tile_row[t+1]);
// block b owns tiles [blk_tile[b], blk_tile[b+1])
struct Tiles {
  const int* tile_row;
  const int* blk_tile;
  const int4* tile_desc;      // (first row, end row, first entry, end entry) per tile
};

__device__ __forceinline__ uint32_t round_up16(uint32_t b) { return b == 0u ? 16u : (b + 15u) & ~15u; }

__global__ void __launch_bounds__((QPK_DICT_WARPS + 1) * 32, 1) k_slot_rows_tma(Engine E, Tiles T, int par) {
  extern __shared__ __align__(128) unsigned char smraw[];
  TmaSmem& S = *reinterpret_cast<TmaSmem*>(smraw);
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_rows = globaltimer_ns();
  const bool fuse = c.mode == MODE_NORMAL || c.mode == MODE_RESTART;
  double* v = fuse ? E.p : E.x[c.mode == MODE_CHECK ? c.xn : c.best];
  const Op& op = E.op;
  const Dict& D = E.dict;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < QPK_TMA_STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], QPK_DICT_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double pacc = 0.0, rzb = 0.0;
  if (warp == QPK_DICT_WARPS) {
    // ---------------------------------------------------------- producer ----
    // The whole warp fetches the tile descriptors of a block (lane i holds
    // tile t0 + i) one block ahead; lane 0 issues the bulk copies.
    int it = 0;
    const double* wsrc = v;                          // bottom vector w lives at v[n + r]
    const double* xsrc = E.x[c.cur];
    int blk = blockIdx.x;
    int t0 = 0, t1 = 0;
    int4 dsc = make_int4(0, 0, 0, 0);
    if (blk < D.nblk) {
      t0 = __ldg(T.blk_tile + blk); t1 = __ldg(T.blk_tile + blk + 1);
      if (t0 + lane < t1) dsc = __ldg(T.tile_desc + t0 + lane);
    }
    while (blk < D.nblk) {
      // prefetch the next block's descriptors
      const int nblk2 = blk + gridDim.x;
      int u0 = 0, u1 = 0;
      int4 ndsc = make_int4(0, 0, 0, 0);
      if (nblk2 < D.nblk) {
        u0 = __ldg(T.blk_tile + nblk2); u1 = __ldg(T.blk_tile + nblk2 + 1);
        if (u0 + lane < u1) ndsc = __ldg(T.tile_desc + u0 + lane);
      }
      for (int tb = t0; tb < t1; tb += 32) {
        if (tb != t0) dsc = (tb + lane < t1) ? __ldg(T.tile_desc + tb + lane) : make_int4(0, 0, 0, 0);
        const int cnt = min(32, t1 - tb);
        for (int i = 0; i < cnt; ++i, ++it) {
          const int ra = __shfl_sync(0xffffffffu, dsc.x, i), rb = __shfl_sync(0xffffffffu, dsc.y, i);
          const int ea = __shfl_sync(0xffffffffu, dsc.z, i), eb = __shfl_sync(0xffffffffu, dsc.w, i);
          const int s = it % QPK_TMA_STAGES;
          const uint32_t ph = (it / QPK_TMA_STAGES) & 1;
          mbar_wait(&S.empty[s], ph ^ 1);
          if (lane == 0) {
            TileStage& st = S.st[s];
            TileDesc td;
            td.ra = ra; td.rb = rb;
            td.e0 = ea & ~7;
            td.e1 = ea & ~1;
            td.p0 = ra & ~3;
            td.v0 = ra & ~1;
            td.w0 = (op.n + ra) & ~1;
            st.t = td;
            const uint32_t b_lci = round_up16((uint32_t)(((eb + 7) & ~7) - td.e0) * 2u);
            const uint32_t b_val = round_up16((uint32_t)(((eb + 1) & ~1) - td.e1) * 8u);
            const uint32_t b_rp = round_up16((uint32_t)(((rb + 1 + 3) & ~3) - td.p0) * 4u);
            const uint32_t b_d = round_up16((uint32_t)(((rb + 1) & ~1) - td.v0) * 8u);
            const uint32_t b_w = round_up16((uint32_t)(((op.n + rb + 1) & ~1) - td.w0) * 8u);
            const uint32_t bytes = b_lci + b_val + b_rp + b_d + b_w + (fuse ? 2 * b_w : 0u);
            mbar_expect_tx(&S.full[s], bytes);
            bulk_g2s(st.lci, D.lci + td.e0, b_lci, &S.full[s]);
            bulk_g2s(st.val, op.bv + td.e1, b_val, &S.full[s]);
            bulk_g2s(st.rp, op.rp + td.p0, b_rp, &S.full[s]);
            bulk_g2s(st.d, op.d + td.v0, b_d, &S.full[s]);
            bulk_g2s(st.w, wsrc + td.w0, b_w, &S.full[s]);
            if (fuse) {
              bulk_g2s(st.r, E.r + td.w0, b_w, &S.full[s]);
              bulk_g2s(st.x, xsrc + td.w0, b_w, &S.full[s]);
            }
          }
          __syncwarp();
        }
      }
      blk = nblk2; t0 = u0; t1 = u1; dsc = ndsc;
    }
  } else {
    // ---------------------------------------------------------- consumers ---
    const double* u = v;
    double* w = v + op.n;
    double* aw = S.acc[warp];
    const int ctid = threadIdx.x;                    // 0 .. 32*W-1
    int it = 0;
    for (int blk = blockIdx.x; blk < D.nblk; blk += gridDim.x) {
      const int d0 = __ldg(D.blk_dict + blk), nd = __ldg(D.blk_dict + blk + 1) - d0;
      for (int k = ctid; k < nd; k += QPK_DICT_WARPS * 32) {
        S.us[k] = u[__ldg(D.cols + d0 + k)];
#pragma unroll
        for (int ww = 0; ww < QPK_DICT_WARPS; ++ww) S.acc[ww][k] = 0.0;
      }
      consumer_bar();
      const int t0 = __ldg(T.blk_tile + blk), t1 = __ldg(T.blk_tile + blk + 1);
      for (int t = t0; t < t1; ++t, ++it) {
        const int s = it % QPK_TMA_STAGES;
        const uint32_t ph = (it / QPK_TMA_STAGES) & 1;
        mbar_wait(&S.full[s], ph);
        const TileStage& st = S.st[s];
        const TileDesc td = st.t;
        // RB rows per warp step, their gathers/reductions interleaved for ILP;
        // the scatters run one row after the other (lanes of a row hold
        // distinct columns, so the plain read-modify-write is race-free)
        constexpr int RB = 4;
        for (int r0 = td.ra + warp; r0 < td.rb; r0 += RB * QPK_DICT_WARPS) {
          int b[RB], e[RB];
          double dr[RB], wr[RB], sacc[RB];
          int tmax = 0;
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const int r = r0 + q * QPK_DICT_WARPS;
            b[q] = 0; e[q] = 0; dr[q] = 1.0; wr[q] = 0.0; sacc[q] = 0.0;
            if (r < td.rb) {
              b[q] = st.rp[r - td.p0]; e[q] = st.rp[r + 1 - td.p0];
              dr[q] = st.d[r - td.v0];
              wr[q] = st.w[op.n + r - td.w0];
              tmax = max(tmax, e[q] - b[q]);
            }
          }
          for (int j = lane; j < tmax; j += 32) {
#pragma unroll
            for (int q = 0; q < RB; ++q) {
              const int k = b[q] + j;
              if (k < e[q]) {
                const unsigned short l = st.lci[k - td.e0];
                if (l != 0xFFFF) sacc[q] = fma(st.val[k - td.e1], S.us[l], sacc[q]);
              }
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int q = 0; q < RB; ++q) sacc[q] += __shfl_xor_sync(0xffffffffu, sacc[q], o);
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const int r = r0 + q * QPK_DICT_WARPS;
            if (r >= td.rb) break;
            const double tt = sacc[q];
            double wv = wr[q];
            if (fuse) {
              const double rres = st.r[op.n + r - td.w0];
              const double zr = __dmul_rn(1.0 / dr[q], rres);
              if (c.xupd && lane == 0)
                E.x[c.xn][op.n + r] = __dadd_rn(st.x[op.n + r - td.w0], __dmul_rn(c.alpha_prev, wv));
              const double pn = (c.mode == MODE_RESTART) ? zr : __dadd_rn(zr, __dmul_rn(c.beta, wv));
              if (lane == 0) { w[r] = pn; rzb += rres * zr; }
              wv = pn;
            }
            const double z = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, tt), dr[q]), wv);
            const double yb = __dadd_rn(tt, __dmul_rn(dr[q], wv));
            if (lane == 0) {
              E.y[op.n + r] = yb;
              pacc += tt * z + wv * yb;
            }
            for (int k = b[q] + lane; k < e[q]; k += 32) {
              const unsigned short l = st.lci[k - td.e0];
              if (l != 0xFFFF) aw[l] += z * st.val[k - td.e1];
            }
            __syncwarp();
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
      }
      consumer_bar();
      for (int k = ctid; k < nd; k += QPK_DICT_WARPS * 32) {
        double sum = 0.0;
#pragma unroll
        for (int ww = 0; ww < QPK_DICT_WARPS; ++ww) sum += S.acc[ww][k];
        D.bpart[d0 + k] = sum;
      }
      consumer_bar();
    }
  }
  __syncthreads();
  pacc += hess_rows(op, v, E.y, E.part, E.G, S.red, S.s_lr);
  double t = block_sum(pacc, S.red);
  if (threadIdx.x == 0) E.part[SLOT_ROWS * E.G + blockIdx.x] = t;
  t = block_sum(rzb, S.red);
  if (threadIdx.x == 0) E.part[SLOT_AUX2 * E.G + blockIdx.x] = t;
}

// ---------------------------------------------------------------------------
// TMA-fed CSR rows kernel (random / general B): the producer streams tiles of
// the padded CSR (int32 columns + values) and the tile's per-row vectors into
// shared memory; consumer sub-warps (L lanes per row, RB rows in flight per
// sub-warp) read their indices from shared memory, so the u gathers -- the
// random L2 requests that bound this kernel -- issue back to back instead of
// waiting on a DRAM round trip for the indices.  CSC == true stores z_B for
// the gather pass (deterministic); otherwise B'z is scattered with atomics.
#define QPK_CSR_WARPS 16

struct alignas(16) CsrStage {
  int ci[QPK_TILE_E + 8];
  double val[QPK_TILE_E + 8];
  int rp[QPK_TILE_R + 8];
  double d[QPK_TILE_R + 4];
  double w[QPK_TILE_R + 4];
  double r[QPK_TILE_R + 4];
  double x[QPK_TILE_R + 4];
  TileDesc t;
};

struct CsrSmem {
  CsrStage st[QPK_TMA_STAGES];
  unsigned long long full[QPK_TMA_STAGES], empty[QPK_TMA_STAGES];
  double red[32];
  double s_lr[QPK_KMAX];
};

template <int L, bool CSC>
__global__ void __launch_bounds__((QPK_CSR_WARPS + 1) * 32, 1)
k_slot_rows_tma_csr(Engine E, const int4* __restrict__ tdesc, int ntiles, int par) {
  extern __shared__ __align__(128) unsigned char smraw[];
  CsrSmem& S = *reinterpret_cast<CsrSmem*>(smraw);
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_rows = globaltimer_ns();
  const bool fuse = c.mode == MODE_NORMAL || c.mode == MODE_RESTART;
  double* v = fuse ? E.p : E.x[c.mode == MODE_CHECK ? c.xn : c.best];
  const Op& op = E.op;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < QPK_TMA_STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], QPK_CSR_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double pacc = 0.0, rzb = 0.0;
  const int my_tiles = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (warp == QPK_CSR_WARPS) {
    const double* wsrc = v;
    const double* xsrc = E.x[c.cur];
    for (int base = 0; base < my_tiles; base += 32) {
      int4 dsc = make_int4(0, 0, 0, 0);
      if (base + lane < my_tiles) dsc = __ldg(tdesc + blockIdx.x + (size_t)(base + lane) * gridDim.x);
      const int cnt = min(32, my_tiles - base);
      for (int i = 0; i < cnt; ++i) {
        const int it = base + i;
        const int ra = __shfl_sync(0xffffffffu, dsc.x, i), rb = __shfl_sync(0xffffffffu, dsc.y, i);
        const int ea = __shfl_sync(0xffffffffu, dsc.z, i), eb = __shfl_sync(0xffffffffu, dsc.w, i);
        const int s = it % QPK_TMA_STAGES;
        mbar_wait(&S.empty[s], ((it / QPK_TMA_STAGES) & 1) ^ 1);
        if (lane == 0) {
          CsrStage& st = S.st[s];
          TileDesc td;
          td.ra = ra; td.rb = rb;
          td.e0 = ea & ~3;
          td.e1 = ea & ~1;
          td.p0 = ra & ~3;
          td.v0 = ra & ~1;
          td.w0 = (op.n + ra) & ~1;
          st.t = td;
          const uint32_t b_ci = round_up16((uint32_t)(((eb + 3) & ~3) - td.e0) * 4u);
          const uint32_t b_val = round_up16((uint32_t)(((eb + 1) & ~1) - td.e1) * 8u);
          const uint32_t b_rp = round_up16((uint32_t)(((rb + 1 + 3) & ~3) - td.p0) * 4u);
          const uint32_t b_d = round_up16((uint32_t)(((rb + 1) & ~1) - td.v0) * 8u);
          const uint32_t b_w = round_up16((uint32_t)(((op.n + rb + 1) & ~1) - td.w0) * 8u);
          mbar_expect_tx(&S.full[s], b_ci + b_val + b_rp + b_d + b_w + (fuse ? 2 * b_w : 0u));
          bulk_g2s(st.ci, op.ci + td.e0, b_ci, &S.full[s]);
          bulk_g2s(st.val, op.bv + td.e1, b_val, &S.full[s]);
          bulk_g2s(st.rp, op.rp + td.p0, b_rp, &S.full[s]);
          bulk_g2s(st.d, op.d + td.v0, b_d, &S.full[s]);
          bulk_g2s(st.w, wsrc + td.w0, b_w, &S.full[s]);
          if (fuse) {
            bulk_g2s(st.r, E.r + td.w0, b_w, &S.full[s]);
            bulk_g2s(st.x, xsrc + td.w0, b_w, &S.full[s]);
          }
        }
        __syncwarp();
      }
    }
  } else {
    const double* u = v;
    double* w = v + op.n;
    constexpr int RPW = 32 / L;                      // rows per warp per step
    constexpr int RB = 2;                            // steps in flight per sub-warp
    const int sub = lane / L, ln = lane & (L - 1);
    for (int it = 0; it < my_tiles; ++it) {
      const int s = it % QPK_TMA_STAGES;
      mbar_wait(&S.full[s], (it / QPK_TMA_STAGES) & 1);
      const CsrStage& st = S.st[s];
      const TileDesc td = st.t;
      for (int r0 = td.ra + warp * RPW + sub; r0 - sub < td.rb; r0 += RB * QPK_CSR_WARPS * RPW) {
        int b[RB], e[RB];
        double sacc[RB];
        int tmax = 0;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          const int r = r0 + q * QPK_CSR_WARPS * RPW;
          b[q] = 0; e[q] = 0; sacc[q] = 0.0;
          if (r < td.rb) { b[q] = st.rp[r - td.p0]; e[q] = st.rp[r + 1 - td.p0]; tmax = max(tmax, e[q] - b[q]); }
        }
        // uniform trip count across the warp (shuffles below need every lane)
        for (int o = L; o < 32; o <<= 1) tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        for (int j = ln; j < tmax; j += L) {
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const int k = b[q] + j;
            if (k < e[q]) {
              const int col = st.ci[k - td.e0];
              if (col >= 0) sacc[q] = fma(st.val[k - td.e1], u[col], sacc[q]);
            }
          }
        }
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1)
#pragma unroll
          for (int q = 0; q < RB; ++q) sacc[q] += __shfl_xor_sync(0xffffffffu, sacc[q], o);
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          const int r = r0 + q * QPK_CSR_WARPS * RPW;
          if (r >= td.rb) continue;
          const double tt = sacc[q];
          const double dr = st.d[r - td.v0];
          double wv = st.w[op.n + r - td.w0];
          if (fuse) {
            const double rres = st.r[op.n + r - td.w0];
            const double zr = __dmul_rn(1.0 / dr, rres);
            if (c.xupd && ln == 0)
              E.x[c.xn][op.n + r] = __dadd_rn(st.x[op.n + r - td.w0], __dmul_rn(c.alpha_prev, wv));
            const double pn = (c.mode == MODE_RESTART) ? zr : __dadd_rn(zr, __dmul_rn(c.beta, wv));
            if (ln == 0) { w[r] = pn; rzb += rres * zr; }
            wv = pn;
          }
          const double z = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, tt), dr), wv);
          const double yb = __dadd_rn(tt, __dmul_rn(dr, wv));
          if (ln == 0) {
            E.y[op.n + r] = yb;
            pacc += tt * z + wv * yb;
            if (CSC) E.zb[r] = z;
          }
          if (!CSC) {
            for (int k = b[q] + ln; k < e[q]; k += L) {
              const int col = st.ci[k - td.e0];
              if (col >= 0) atomicAdd(E.y + col, z * st.val[k - td.e1]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[s]);
    }
  }
  __syncthreads();
  pacc += hess_rows(op, v, E.y, E.part, E.G, S.red, S.s_lr);
  double t = block_sum(pacc, S.red);
  if (threadIdx.x == 0) E.part[SLOT_ROWS * E.G + blockIdx.x] = t;
  t = block_sum(rzb, S.red);
  if (threadIdx.x == 0) E.part[SLOT_AUX2 * E.G + blockIdx.x] = t;
}

}  // namespace qpk
