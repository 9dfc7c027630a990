// qpk_tma.cuh -- TMA-fed kernels: 1-D bulk async copies (cp.async.bulk ...
// mbarrier::complete_tx; SASS UBLKCP) from HBM into a ring of shared-memory
// stages, filled by one producer lane and drained by consumer warps.
//   k_slot_rows_tile     dense-tile apply for clustered B (one pass, no atomics)
#pragma once
#include "qpk_engine.cuh"


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

// the same copy with an L2 evict-first policy: data streamed once per pass
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, unsigned long long* bar,
                                                unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint32_t round_up16(uint32_t b) { return b == 0u ? 16u : (b + 15u) & ~15u; }

// ---------------------------------------------------------------------------
// Dense-tile kernel (the one-pass, atomic-free apply for clustered B).
// Producer warp: one elected lane streams each tile's dense block, its
// column list and the tile's per-row vectors into a 4-stage ring with
// cp.async.bulk (UBLKCP) + mbarrier complete_tx.  Consumers (8 warps):
//   u_dict[c] = u[cols[c]]  (gathered one tile ahead, from registers)
//   rows:    t_r = A_r . u_dict  (warp per row), z_r, y_B, fused bottom update
//   columns: bpart[c] = sum_r A[r][c] z_r  (thread per column, no atomics)
#define QPK_TILE_WARPS 8
#ifndef QPK_TILE_STAGES
#define QPK_TILE_STAGES 6        // ring stages (3 groups consume, 3 in flight)
#endif

struct alignas(16) DTileStage {
  double a[QPK_TILE_DOUBLES + 2];
  double ud[QPK_TILE_DMAX];        // u[cols], gathered by the gather warp
  int cols[QPK_TILE_DMAX];
  double d[QPK_TILE_ROWS + 4];
  double w[QPK_TILE_ROWS + 4];
  double r[QPK_TILE_ROWS + 4];
  double x[QPK_TILE_ROWS + 4];
  TileDescD t;
  int v0, w0, pad0, pad1;
};

#ifndef QPK_TILE_GROUPS
#define QPK_TILE_GROUPS 3        // consumer groups working on tiles round robin
#endif
#ifndef QPK_TILE_GWARPS
#define QPK_TILE_GWARPS 4        // warps per consumer group
#endif
#ifndef QPK_TILE_GATHER_WARPS
#define QPK_TILE_GATHER_WARPS 3  // warps gathering u[cols] for landed tiles (must divide QPK_TILE_STAGES)
#endif
// a ring stage is always reused by the warp / group that used it last, so an
// mbarrier parity wait can never be satisfied by a phase two uses old
static_assert(QPK_TILE_STAGES % QPK_TILE_GATHER_WARPS == 0, "gather warps must divide the ring stages");
static_assert(QPK_TILE_STAGES % QPK_TILE_GROUPS == 0, "consumer groups must divide the ring stages");
#ifndef QPK_TILE_UMAX
#define QPK_TILE_UMAX 1024       // CTA-accumulator capacity (distinct columns of a CTA's tiles)
#endif

struct DTileSmem {
  DTileStage st[QPK_TILE_STAGES];
  unsigned long long full[QPK_TILE_STAGES], empty[QPK_TILE_STAGES], uready[QPK_TILE_STAGES];
  double rpart[QPK_TILE_GROUPS][QPK_TILE_GWARPS][QPK_TILE_ROWS];
  alignas(16) double zs[QPK_TILE_GROUPS][QPK_TILE_ROWS];
  double red[32];
};

__device__ __forceinline__ void tile_group_bar(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(QPK_TILE_GWARPS * 32) : "memory");
}

// Tile layout: rows of the dense block have an odd pitch (ndp | 1 doubles,
// TileDescD::pad0) so that 32 lanes reading one column of consecutive rows
// hit distinct banks.  QPK_TILE_GROUPS groups of QPK_TILE_GWARPS consumer
// warps take the tiles round robin (so the groups' barrier-separated passes
// overlap: with 3 groups and 6 stages, 3 tiles are in flight while 3 are
// consumed -- measured best of 2-4 groups x 2-7 stages x 16-32 KB tiles on
// cfg3/cfg4); per tile a group runs three regular shared-memory passes: row
// slices (warp w, lane = row), row finish (thread per row), columns (thread
// per column).
__global__ void __launch_bounds__((QPK_TILE_GROUPS * QPK_TILE_GWARPS + 1 + QPK_TILE_GATHER_WARPS) * 32, 1)
k_slot_rows_tile(Engine E, int par) {
  extern __shared__ __align__(128) unsigned char smraw[];
  DTileSmem& S = *reinterpret_cast<DTileSmem*>(smraw);
  double* cacc = reinterpret_cast<double*>(smraw + sizeof(DTileSmem));   // [GROUPS][UMAX] (cacc mode)
  constexpr int CW = QPK_TILE_GROUPS * QPK_TILE_GWARPS;   // consumer warps
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_rows = globaltimer_ns();
  const bool fuse = c.mode == MODE_NORMAL || c.mode == MODE_RESTART;
  double* v = fuse ? E.p : E.x[c.mode == MODE_CHECK ? c.xn : c.best];
  const Op& op = E.op;
  const Dict& D = E.dict;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < QPK_TILE_STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.uready[s], 1);
      mbar_init(&S.empty[s], QPK_TILE_GWARPS);       // a stage is drained by one group
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // tiles of this CTA: consecutive (cacc) or strided
  const int tb = D.cacc ? __ldg(D.tile_beg + blockIdx.x) : (int)blockIdx.x;
  const int tstep = D.cacc ? 1 : (int)gridDim.x;
  const int my = D.cacc ? __ldg(D.tile_beg + blockIdx.x + 1) - tb
                        : ((D.nblk > (int)blockIdx.x) ? (D.nblk - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0);
  const int nu = D.cacc ? __ldg(D.cta_off + blockIdx.x + 1) - __ldg(D.cta_off + blockIdx.x) : 0;
  for (int i = threadIdx.x; i < QPK_TILE_GROUPS * nu; i += blockDim.x)
    cacc[(i / nu) * QPK_TILE_UMAX + (i % nu)] = 0.0;
  __syncthreads();
  double pacc = 0.0, rzb = 0.0;
  double fs[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};     // folded bottom sums (E.fold)
  if (warp == CW) {
    // ---------------------------------------------------------- producer ----
    // In a PCG iteration (fuse) it streams only data written two or more
    // kernels back (the matrix, d, and the bottom windows of p, r, x[cur]), so
    // under programmatic launch the ring fills while the top kernel is still
    // running; in CHECK / FINAL the top kernel materialises the x it reads.
    if (!fuse) pdl_wait();
    // Tile descriptors are prefetched a warp-batch ahead: lane l holds the
    // descriptor of tile (batch + l) and lane 0 takes them by shuffle, so no
    // dependent descriptor load sits between a stage's release and its refill.
    const double* wsrc = v;
    const double* xsrc = E.x[c.cur];
    // The dense blocks are streamed once per pass (1.4 GB on cfg4, far beyond
    // L2): an L2 evict-first policy on their copies keeps the vectors the
    // slot's kernels re-read (p, r, x, y, d: ~14 MB each) resident instead of
    // being flushed by the stream (A/B: cfg4 tile pass 318 -> 297 us, cfg3 42.9 -> 39.5 us)
#ifndef QPK_TILE_NO_EVICT_FIRST
    const unsigned long long pol = l2_evict_first_policy();
#define TILE_A_COPY(dst, src, bytes, bar) bulk_g2s_stream(dst, src, bytes, bar, pol)
#else
#define TILE_A_COPY(dst, src, bytes, bar) bulk_g2s(dst, src, bytes, bar)
#endif
#define TILE_C_COPY(dst, src, bytes, bar) bulk_g2s(dst, src, bytes, bar)
    auto ld_desc = [&](int base) {
      int4 lo = make_int4(0, 0, 0, 0), hi = lo;
      const int k = base + lane;
      if (k < my) {
        const int4* q = reinterpret_cast<const int4*>(D.tiles + tb + (long long)k * tstep);
        lo = __ldg(q);
        hi = __ldg(q + 1);
      }
      return TileDescD{lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    };
    TileDescD cur_b = ld_desc(0), nxt_b = ld_desc(32);
    for (int it = 0; it < my; ++it) {
      const int l = it & 31;
      if (l == 0 && it > 0) { cur_b = nxt_b; nxt_b = ld_desc(it + 32); }
      TileDescD td;
      td.ra = __shfl_sync(0xffffffffu, cur_b.ra, l);
      td.rb = __shfl_sync(0xffffffffu, cur_b.rb, l);
      td.d0 = __shfl_sync(0xffffffffu, cur_b.d0, l);
      td.ndp = __shfl_sync(0xffffffffu, cur_b.ndp, l);
      td.v0 = __shfl_sync(0xffffffffu, cur_b.v0, l);
      td.pad0 = __shfl_sync(0xffffffffu, cur_b.pad0, l);
      td.pad1 = __shfl_sync(0xffffffffu, cur_b.pad1, l);
      td.pad2 = __shfl_sync(0xffffffffu, cur_b.pad2, l);
      if (D.l2pf) {
        // L2 prefetch of the dense block D.l2pf tiles ahead (beyond the ring),
        // so the stage's bulk copy is served from L2 when the stage frees
        const int lp = l + D.l2pf;
        const int pf_v0 = __shfl_sync(0xffffffffu, lp < 32 ? cur_b.v0 : nxt_b.v0, lp & 31);
        const int pf_ra = __shfl_sync(0xffffffffu, lp < 32 ? cur_b.ra : nxt_b.ra, lp & 31);
        const int pf_rb = __shfl_sync(0xffffffffu, lp < 32 ? cur_b.rb : nxt_b.rb, lp & 31);
        const int pf_p = __shfl_sync(0xffffffffu, lp < 32 ? cur_b.pad0 : nxt_b.pad0, lp & 31);
        if (lane == 0 && it + D.l2pf < my)
          bulk_prefetch_l2(D.tval + pf_v0, round_up16((uint32_t)((pf_rb - pf_ra) * pf_p) * 8u));
      }
      if (lane == 0) {
        const int s = it % QPK_TILE_STAGES;
        mbar_wait(&S.empty[s], ((it / QPK_TILE_STAGES) & 1) ^ 1);
        DTileStage& st = S.st[s];
        st.t = td;
        const int v0 = td.ra & ~1, w0 = (op.n + td.ra) & ~1;
        st.v0 = v0;
        st.w0 = w0;
        const uint32_t b_a = round_up16((uint32_t)((td.rb - td.ra) * td.pad0) * 8u);
        const uint32_t b_c = round_up16((uint32_t)td.ndp * 4u);
        if (td.pad1) {                                  // Hessian tile: no per-row vectors
          // (its row ids hperm[ra .. rb) land in st.d, from a 16-byte aligned start)
          const uint32_t b_j = D.hperm ? round_up16((uint32_t)(td.rb - (td.ra & ~3)) * 4u) : 0u;
          mbar_expect_tx(&S.full[s], b_a + b_c + b_j);
          TILE_A_COPY(st.a, D.tval + td.v0, b_a, &S.full[s]);
          TILE_C_COPY(st.cols, D.cols + td.d0, b_c, &S.full[s]);
          if (b_j) bulk_g2s(st.d, D.hperm + (td.ra & ~3), b_j, &S.full[s]);
        } else {
          const uint32_t b_d = round_up16((uint32_t)(((td.rb + 1) & ~1) - v0) * 8u);
          const uint32_t b_w = round_up16((uint32_t)(((op.n + td.rb + 1) & ~1) - w0) * 8u);
          mbar_expect_tx(&S.full[s], b_a + b_c + b_d + b_w + (fuse ? 2 * b_w : 0u));
          TILE_A_COPY(st.a, D.tval + td.v0, b_a, &S.full[s]);
          TILE_C_COPY(st.cols, D.cols + td.d0, b_c, &S.full[s]);
          bulk_g2s(st.d, op.d + v0, b_d, &S.full[s]);
          bulk_g2s(st.w, wsrc + w0, b_w, &S.full[s]);
          if (fuse) {
            bulk_g2s(st.r, E.r + w0, b_w, &S.full[s]);
            bulk_g2s(st.x, xsrc + w0, b_w, &S.full[s]);
          }
        }
      }
      __syncwarp();
    }
  } else if (warp > CW) {
    // ----------------------------------------------------- gather warps ----
    pdl_wait();                                        // u = p_top comes from the top kernel
    pdl_trigger();
    // u[cols] for each landed tile (warp CW+1+k takes tiles it = k mod NGW),
    // 8 independent gathers in flight per lane, then "u ready"
    constexpr int NGW = QPK_TILE_GATHER_WARPS;
    const double* u = v;
    for (int it = warp - CW - 1; it < my; it += NGW) {
      const int s = it % QPK_TILE_STAGES;
      mbar_wait(&S.full[s], (it / QPK_TILE_STAGES) & 1);
      DTileStage& st = S.st[s];
      const int nd = st.t.ndp;
      // (CTA accumulation: the tile's column list is no longer needed once
      // gathered, so its slots in the CTA accumulator replace it in place)
      const bool slots = D.cacc && !st.t.pad1;
      const int d0 = st.t.d0;
      // Hessian tile: its rows are top indices j (hperm window in st.d); stage
      // u_j and the current y_j (this tile is y_j's only writer in the pass)
      // in the row arrays the TMA leaves unused for such tiles, so the
      // consumers' row finish has no dependent global loads
      const bool hrows = st.t.pad1;
      const int hra = st.t.ra, hR = st.t.rb - st.t.ra;
      const int* jrow = reinterpret_cast<const int*>(st.d) + (hra & 3);
      double hu[2] = {0.0, 0.0}, hy[2] = {0.0, 0.0};
      if (hrows) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int rr = lane + 32 * q;
          if (rr < hR) {
            const int j = D.hperm ? jrow[rr] : hra + rr;
            hu[q] = u[j];
            hy[q] = E.y[j];
          }
        }
      }
      for (int cb = lane; cb < nd; cb += 32 * 8) {
        double g8[8];
        int s8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int cc = cb + 32 * q;
          const int col = cc < nd ? st.cols[cc] : -1;
          g8[q] = col >= 0 ? u[col] : 0.0;
          s8[q] = (slots && cc < nd) ? __ldg(D.tslot + d0 + cc) : -1;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int cc = cb + 32 * q;
          if (cc < nd) {
            st.ud[cc] = g8[q];
            if (slots) st.cols[cc] = s8[q];
          }
        }
      }
      // Hessian tile: its rows are top indices j = hperm[ra + rr]; stage j,
      // u_j and the current y_j (this tile is y_j's only writer in the pass)
      // in the row arrays the TMA leaves unused for such tiles, so the
      // consumers' row finish has no dependent global loads
      if (hrows) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int rr = lane + 32 * q;
          if (rr < hR) { st.w[rr] = hu[q]; st.x[rr] = hy[q]; }
        }
      }
      // generic-proxy writes into a stage the TMA (async proxy) refills later
      if (slots || hrows) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.uready[s]);
    }
  } else {
    // ---------------------------------------------------------- consumers ---
    pdl_wait();                                        // y_top is initialised by the top kernel
    pdl_trigger();
    constexpr int T = QPK_TILE_GWARPS * 32;          // threads per group
    const int g = warp / QPK_TILE_GWARPS, gw = warp % QPK_TILE_GWARPS;
    const int tid = threadIdx.x - g * T;
    double* wv = v + op.n;
    for (int it = g; it < my; it += QPK_TILE_GROUPS) {
      const int s = it % QPK_TILE_STAGES;
      mbar_wait(&S.uready[s], (it / QPK_TILE_STAGES) & 1);
      const DTileStage& st = S.st[s];
      const TileDescD td = st.t;
      const int nd = td.ndp, pitch = td.pad0, R = td.rb - td.ra;
      const double* ud = st.ud;
      {
        const int cs = (nd + QPK_TILE_GWARPS - 1) / QPK_TILE_GWARPS;
        const int c0 = gw * cs, c1 = min(nd, c0 + cs);
        for (int rr = lane; rr < R; rr += 32) {
          const double* arow = st.a + rr * pitch;
          double s0 = 0.0, s1 = 0.0;
          int cc = c0;
          for (; cc + 1 < c1; cc += 2) {
            s0 = fma(arow[cc], ud[cc], s0);
            s1 = fma(arow[cc + 1], ud[cc + 1], s1);
          }
          if (cc < c1) s0 = fma(arow[cc], ud[cc], s0);
          S.rpart[g][gw][rr] = s0 + s1;
        }
      }
      tile_group_bar(g);
      if (td.pad1) {
        // Hessian tile: rows are top indices j; y_j += (H u)_j, p'Hp partial
        for (int rr = tid; rr < R; rr += T) {
          double tt = 0.0;
#pragma unroll
          for (int ww = 0; ww < QPK_TILE_GWARPS; ++ww) tt += S.rpart[g][ww][rr];
          const int j = D.hperm ? reinterpret_cast<const int*>(st.d)[(td.ra & 3) + rr] : td.ra + rr;
          E.y[j] = st.x[rr] + tt;                         // y_j and u_j staged by the gather warps
          pacc += st.w[rr] * tt;
        }
        tile_group_bar(g);                              // rpart is rewritten by the next tile
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
        continue;
      }
      for (int rr = tid; rr < R; rr += T) {
        double tt = 0.0;
#pragma unroll
        for (int ww = 0; ww < QPK_TILE_GWARPS; ++ww) tt += S.rpart[g][ww][rr];
        const int r = td.ra + rr;
        const double dr = st.d[r - st.v0];
        double wr = st.w[op.n + r - st.w0];
        if (fuse) {
          const double rres = st.r[op.n + r - st.w0];
          const double zr = __dmul_rn(1.0 / dr, rres);
          if (c.xupd) E.x[c.xn][op.n + r] = __dadd_rn(st.x[op.n + r - st.w0], __dmul_rn(c.alpha_prev, wr));
          const double pn = (c.mode == MODE_RESTART) ? zr : __dadd_rn(zr, __dmul_rn(c.beta, wr));
          wv[r] = pn;
          rzb += rres * zr;
          wr = pn;
        }
        const double z = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, tt), dr), wr);
        const double yb = __dadd_rn(tt, __dmul_rn(dr, wr));
        E.y[op.n + r] = yb;
        pacc += tt * z + wr * yb;
        S.zs[g][rr] = z;
        if (E.fold) {
          if (fuse) {
            const double rres = st.r[op.n + r - st.w0], mi = 1.0 / dr;
            fs[0] += rres * rres; fs[1] += rres * yb; fs[2] += yb * yb;
            fs[3] += rres * __dmul_rn(mi, rres); fs[4] += rres * __dmul_rn(mi, yb); fs[5] += yb * __dmul_rn(mi, yb);
          } else {
            const double e = __dsub_rn(__ldg(E.rhs + op.n + r), yb);   // explicit residual (the update kernel stores it)
            fs[0] += e * e;
          }
        }
      }
      tile_group_bar(g);
      for (int cc = tid; cc < nd; cc += T) {
        double s0 = 0.0, s1 = 0.0;
        int rr = 0;
#ifndef QPK_TILE_NO_COLUNROLL
        {
          const double* ac = st.a + cc;
          const double* zz = S.zs[g];
          for (; rr + 7 < R; rr += 8) {
            double av[8], zv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) { av[q] = ac[(rr + q) * pitch]; zv[q] = zz[rr + q]; }
#pragma unroll
            for (int q = 0; q < 8; q += 2) { s0 = fma(av[q], zv[q], s0); s1 = fma(av[q + 1], zv[q + 1], s1); }
          }
        }
#endif
        for (; rr + 1 < R; rr += 2) {
          s0 = fma(st.a[rr * pitch + cc], S.zs[g][rr], s0);
          s1 = fma(st.a[(rr + 1) * pitch + cc], S.zs[g][rr + 1], s1);
        }
        if (rr < R) s0 = fma(st.a[rr * pitch + cc], S.zs[g][rr], s0);
        const double colsum = s0 + s1;
        if (D.cacc) {
          const int sl = st.cols[cc];                     // slot (gather warps), distinct per tile column
          if (sl >= 0) cacc[g * QPK_TILE_UMAX + sl] += colsum;
        } else {
          D.bpart[td.d0 + cc] = colsum;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[s]);
    }
  }
  __syncthreads();
  if (D.cacc) {                                       // CTA partials, groups added in order
    const int off = __ldg(D.cta_off + blockIdx.x);
    for (int u = threadIdx.x; u < nu; u += blockDim.x) {
      double sum = 0.0;
#pragma unroll
      for (int g = 0; g < QPK_TILE_GROUPS; ++g) sum += cacc[g * QPK_TILE_UMAX + u];
      D.cpart[off + u] = sum;
    }
  }
  // (the non-diagonal Hessian part runs in k_slot_hess: more blocks than this grid)
  double t = block_sum(pacc, S.red);
  if (threadIdx.x == 0) E.part[SLOT_ROWS * E.G + blockIdx.x] = t;
  t = block_sum(rzb, S.red);
  if (threadIdx.x == 0) E.part[SLOT_AUX2 * E.G + blockIdx.x] = t;
  if (E.fold) {
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      t = block_sum(fs[q], S.red);
      if (threadIdx.x == 0) E.part[(SLOT_F + q) * E.G + blockIdx.x] = t;
    }
  }
}

// y_top += H' u for CSR / dense / low-rank H, its u'H'u added to the slot's
// PREP partial (same grid as the top kernel).  CSR H: LH lanes per row with
// four independent gathers in flight per lane; y_j is final after the tile
// combine, so the row owner adds without atomics.
__global__ void __launch_bounds__(QPK_BLOCK) k_slot_hess(Engine E, int par) {
  __shared__ double red[32];
  __shared__ double s_lr[QPK_KMAX];
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  const bool fuse = c.mode == MODE_NORMAL || c.mode == MODE_RESTART;
  const double* v = fuse ? E.p : E.x[c.mode == MODE_CHECK ? c.xn : c.best];
  const Op& op = E.op;
  double acc = 0.0;
  if (op.H.kind == HESS_CSR) {
    // the H rows this rank applies (sharded: its row list; single GPU: all rows)
    const int LH = op.H.lanes, lh = threadIdx.x & (LH - 1);
    const int per = 32 / LH, sw = (threadIdx.x & 31) / LH;
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
    const int nr = op.H.rows ? op.H.nrows : op.n;
    for (long long jb = (long long)gwarp * per; jb < nr; jb += (long long)nwarp * per) {
      const int q = (int)jb + sw;
      const int j = q < nr ? (op.H.rows ? __ldg(op.H.rows + q) : q) : 0;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (q < nr) {
        const int b = __ldg(op.H.rp + j), e = __ldg(op.H.rp + j + 1);
        int k = b + lh;
        for (; k + 3 * LH < e; k += 4 * LH) {
          const int c0 = __ldg(op.H.ci + k), c1 = __ldg(op.H.ci + k + LH);
          const int c2 = __ldg(op.H.ci + k + 2 * LH), c3 = __ldg(op.H.ci + k + 3 * LH);
          s0 = fma(__ldg(op.H.v + k), v[c0], s0);
          s1 = fma(__ldg(op.H.v + k + LH), v[c1], s1);
          s2 = fma(__ldg(op.H.v + k + 2 * LH), v[c2], s2);
          s3 = fma(__ldg(op.H.v + k + 3 * LH), v[c3], s3);
        }
        for (; k < e; k += LH) s0 = fma(__ldg(op.H.v + k), v[__ldg(op.H.ci + k)], s0);
      }
      double sum = (s0 + s1) + (s2 + s3);
      for (int o = LH / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (q < nr && lh == 0) { E.y[j] += sum; acc += v[j] * sum; }
    }
  } else if (op.H.kind == HESS_DENSE && op.H.sym) {
    acc = hess_sym(op, v, E.y);                     // packed symmetric tiles (large dense H)
  } else {
    acc = hess_rows(op, v, E.y, E.part, E.G, red, s_lr);
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) E.part[SLOT_PREP * E.G + blockIdx.x] += t;
}

// y_top += H u for a large dense symmetric H from its packed upper tiles
// (hess_sym_t; its u'Hu partial is added into the slot's PREP partials)
#ifndef QPK_SYM_MINB
#define QPK_SYM_MINB 1            // blocks per SM (RG 32: ~250 registers; measured best of RG 16/32 x 1/2)
#endif
__global__ void __launch_bounds__(QPK_BLOCK, QPK_SYM_MINB) k_slot_hess_sym(Engine E, int par) {
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  const bool fuse = c.mode == MODE_NORMAL || c.mode == MODE_RESTART;
  const double* v = fuse ? E.p : E.x[c.mode == MODE_CHECK ? c.xn : c.best];
  hess_sym_t<QPK_SYM_RG>(E.op, v, E.y);              // partials only; k_slot_sym_combine adds them into y
}

// the packed symmetric H's partials summed into y_top in a fixed order, u'H u
// into the slot's PREP partials (grid <= E.G, one partial slot per block)
#define QPK_SYMC_BLOCK 1024       // 16 parts per output: ~300 partials per output are summed in ~5 round trips
__global__ void __launch_bounds__(QPK_SYMC_BLOCK) k_slot_sym_combine(Engine E, int par) {
  __shared__ double red[32];
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  const bool fuse = c.mode == MODE_NORMAL || c.mode == MODE_RESTART;
  const double* v = fuse ? E.p : E.x[c.mode == MODE_CHECK ? c.xn : c.best];
  __shared__ double sh[QPK_SYMC_BLOCK];
  const double t = block_sum(sym_combine(E.op, v, E.y, sh), red);
  if (threadIdx.x == 0) E.part[SLOT_PREP * E.G + blockIdx.x] += t;
}

// Column sums of the B-tile partials in two deterministic levels, balanced for
// columns present in thousands of tiles (cfg2's dense X block):
//   k_comb_seg:  seg_sum[q] = sum of <= QPK_COMB_CHUNK partials of one column
//                (LC lanes per segment, lane-strided then a butterfly)
//   k_comb_col:  out[j] (+)= sum of column j's segment sums, in order
#define QPK_COMB_CHUNK 128
__global__ void __launch_bounds__(QPK_BLOCK) k_comb_seg(Engine E, int par) {
  pdl_wait();
  pdl_trigger();
  if (par >= 0 && E.ctrl[par].mode == MODE_DONE) return;
  if (par >= 0 && blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_mid = globaltimer_ns();
  const int LC = E.dict.comb_lanes, lc = threadIdx.x & (LC - 1);
  const int per = 32 / LC, sw = (threadIdx.x & 31) / LC;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
  for (long long qb = (long long)gwarp * per; qb < E.dict.nseg; qb += (long long)nwarp * per) {
    const int q = (int)qb + sw;
    double s0 = 0.0, s1 = 0.0;
    if (q < E.dict.nseg) {
      const int b = __ldg(E.dict.seg_beg + q), e = __ldg(E.dict.seg_beg + q + 1);
      int k = b + lc;
      const double* src = E.dict.cacc ? E.dict.cpart : E.dict.bpart;
      for (; k + LC < e; k += 2 * LC) {
        s0 += src[__ldg(E.dict.col_pos + k)];
        s1 += src[__ldg(E.dict.col_pos + k + LC)];
      }
      if (k < e) s0 += src[__ldg(E.dict.col_pos + k)];
    }
    double sum = s0 + s1;
    for (int o = LC / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (q < E.dict.nseg && lc == 0) E.dict.seg_sum[q] = sum;
  }
}

__global__ void __launch_bounds__(QPK_BLOCK) k_comb_col(Engine E, double* out, int add, int par) {
  pdl_wait();
  pdl_trigger();
  if (par >= 0 && E.ctrl[par].mode == MODE_DONE) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < E.op.n; j += gridDim.x * blockDim.x) {
    const int qb = __ldg(E.dict.col_seg + j), qe = __ldg(E.dict.col_seg + j + 1);
    double sum = 0.0;
    for (int q = qb; q < qe; ++q) sum += E.dict.seg_sum[q];
    out[j] = add ? out[j] + sum : sum;
  }
}

// Single-level combine for the CTA-accumulation mode, where a column has only
// a few CTA partials (banded B: the CTAs whose tile range meets the column's
// band): out[j] (+)= sum of column j's partials in CTA order, thread per column.
__global__ void __launch_bounds__(QPK_BLOCK) k_comb_direct(Engine E, double* out, int add, int par) {
  pdl_wait();
  pdl_trigger();
  if (par >= 0 && E.ctrl[par].mode == MODE_DONE) return;
  if (par >= 0 && blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_mid = globaltimer_ns();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < E.op.n; j += gridDim.x * blockDim.x) {
    const int b = __ldg(E.dict.col_ptr + j), e = __ldg(E.dict.col_ptr + j + 1);
    double sum = 0.0;
    for (int q = b; q < e; ++q) sum += E.dict.cpart[__ldg(E.dict.col_pos + q)];
    out[j] = add ? out[j] + sum : sum;
  }
}

// Jacobi through the tiles: bpart[c] = sum_r A[r][c]^2 / d_r (once per IPM iteration)
__global__ void __launch_bounds__(QPK_BLOCK) k_jac_tile(Engine E) {
  const Dict& D = E.dict;
  for (int t = blockIdx.x; t < D.nblk; t += gridDim.x) {
    const TileDescD td = D.tiles[t];
    if (td.pad1) continue;                              // Hessian tiles: diag(H) is precomputed
    const int R = td.rb - td.ra;
    for (int cc = threadIdx.x; cc < td.ndp; cc += blockDim.x) {
      double s0 = 0.0;
      for (int rr = 0; rr < R; ++rr) {
        const double a = __ldg(D.tval + td.v0 + (size_t)rr * td.pad0 + cc);
        s0 += __dmul_rn(a, a) * (1.0 / __ldg(E.op.d + td.ra + rr));
      }
      D.bpart[td.d0 + cc] = s0;
    }
  }
}

}  // namespace qpk
