// qpk_panel.cuh -- the dense-column-panel apply (QPK_SCATTER_PANEL).
//
// For B whose nonzeros sit mostly in a block of columns present in (nearly)
// every row -- the SVM primal of BASELINE config 2, B = [diag(y)X, y | I] --
// the operator apply of kkt.py:211-221 is two dense GEMVs sharing one pass
// over the panel:
//     t_r  = P_r . u_P + sum_k E_rk u[c_rk]                 (A u, kkt.py:177-178)
//     z_r  = 2 t_r / d_r + w_r ;  y_B,r = t_r + d_r w_r      (kkt.py:217-220)
//     y_P += sum_r z_r P_r                                   (B'z, kkt.py:180-184)
// One warp per row: lane l holds the row's elements 2l + 64q (+1) as double2
// streamed from HBM (ld.global.nc.L1::no_allocate, one row ahead in flight),
// u_P sits in shared memory, the B'z partial of the panel stays in registers
// for the whole pass (2Q doubles per lane), then warps -> CTA partial
// (ppart[cta][j]) -> k_panel_comb sums the CTA partials of each column in a
// fixed order.  No atomics anywhere: bitwise reproducible.  The remainder of
// each row (the identity block of the SVM, <= 32 entries) is a fixed-width
// ELL strip; when every remainder column has at most one entry its B'z term is
// written directly (single writer), otherwise z_B is stored for the CSC pass.
#pragma once
#include "qpk_engine.cuh"
#include "qpk_tma.cuh"

namespace qpk {

// per-row scalars of the fused bottom update (see RowFuse in qpk_device.cuh)
struct PanelRow {
  double d, w, r, x;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

#ifndef QPK_PANEL_STAGES
#define QPK_PANEL_STAGES 3        // ring stages (chunks in flight: up to S)
#endif
#define QPK_PANEL_CW 8            // warps per CTA, one CTA per SM (lane 0 of warp 0 also produces)
#ifndef QPK_PANEL_CHUNK
#define QPK_PANEL_CHUNK 65536     // target panel bytes per chunk (one bulk copy)
#endif
#ifndef QPK_PANEL_RPW
#define QPK_PANEL_RPW 2           // rows per warp step (interleaved reduction chains), kp <= 512
#endif

template <int Q> struct PanelRpw { static constexpr int value = Q <= 8 ? QPK_PANEL_RPW : 1; };
__host__ __device__ __forceinline__ int panel_rpw(int kp) { return kp <= 512 ? QPK_PANEL_RPW : 1; }

// Shared-memory layout of one ring stage (a chunk of rc consecutive rows):
// panel rows, the 4 bottom vectors' slices (d, w, r, x; 16-byte aligned
// windows), the remainder's values, its staged u values (direct) or columns.
// Offsets in doubles.
struct PanelStage {
  int rc;                  // rows per chunk (multiple of CW * rpw)
  int o_d, o_w, o_r, o_x, o_ev, o_ue, o_ec, size;
};
__host__ __device__ __forceinline__ PanelStage panel_stage(int kp, int ew) {
  PanelStage L;
  const int step = QPK_PANEL_CW * panel_rpw(kp);
  int g = QPK_PANEL_CHUNK / (step * kp * 8);
  g = g < 1 ? 1 : g;
  L.rc = step * g;
  const int vec = L.rc + 4;                      // (rc + 2 rounded) doubles per vector window
  const int ent = (L.rc * ew + 4 + 1) & ~1;
  L.o_d = L.rc * kp;
  L.o_w = L.o_d + vec;
  L.o_r = L.o_w + vec;
  L.o_x = L.o_r + vec;
  L.o_ev = L.o_x + vec;
  L.o_ue = L.o_ev + ent;
  L.o_ec = L.o_ue + ent;
  L.size = (L.o_ec + (L.rc * ew + 8) / 2 + 2 + 1) & ~1;
  return L;
}
__host__ __device__ __forceinline__ size_t panel_smem_bytes(int kp, int ew) {
  const PanelStage L = panel_stage(kp, ew);
  return (size_t)(kp + 32 + (size_t)QPK_PANEL_STAGES * L.size) * sizeof(double) +
         2 * QPK_PANEL_STAGES * sizeof(unsigned long long);
}

// One pass over the panel + remainder (a PCG iteration's apply, or the
// CHECK / FINAL apply of an iterate).  CTA b owns rows [m b / G, m (b+1) / G),
// cut into chunks of rc consecutive rows.  A producer lane (lane 0 of warp 0,
// S - 1 chunks ahead of its own consumption) streams each chunk
// -- its panel rows (one bulk copy), the slices of d, w, r, x the fused update
// needs, its remainder entries and (direct mode) their u values staged by the
// top kernel -- with cp.async.bulk into an S-stage ring (mbarrier
// complete_tx).  Consumer warp k takes rows k*RPW .. k*RPW+RPW-1 (+ CW*RPW
// steps) of every chunk, RPW rows interleaved so their reduction chains
// overlap; fixed order -> deterministic.  No random access in direct mode (the
// remainder's B'z terms go to yrem in entry order).
template <int Q>
__global__ void __launch_bounds__(QPK_PANEL_CW * 32, 1) k_slot_panel(Engine E, int par) {
  extern __shared__ __align__(128) double psm[];
  constexpr int S = QPK_PANEL_STAGES, CW = QPK_PANEL_CW, RPW = PanelRpw<Q>::value;
  pdl_wait();                                    // the top kernel stages u (p_top, remainder u values)
  pdl_trigger();
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_rows = globaltimer_ns();
  const bool fuse = c.mode == MODE_NORMAL || c.mode == MODE_RESTART;
  double* v = fuse ? E.p : E.x[c.mode == MODE_CHECK ? c.xn : c.best];
  const Op& op = E.op;
  const Panel& P = E.panel;
  const int kp = P.kp, ew = P.ew, n = op.n;
  const bool direct = P.direct;
  const PanelStage L = panel_stage(kp, ew);
  double* red = psm + kp;                        // [32]
  double* ring = psm + kp + 32;                  // [S][L.size]; reused as warp partials [CW][kp]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + (size_t)S * L.size);
  unsigned long long* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int k = 0; k < S; ++k) { mbar_init(&full[k], 1); mbar_init(&empty[k], CW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();                               // barriers initialised
  const int ra = (int)((long long)op.m * blockIdx.x / gridDim.x);
  const int rb = (int)((long long)op.m * (blockIdx.x + 1) / gridDim.x);
  const int nch = (rb - ra + L.rc - 1) / L.rc;
  const double* xsrc = E.x[c.cur];
  double pacc = 0.0, rzb = 0.0;
  double2 acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = make_double2(0.0, 0.0);
  // producer: lane 0 of warp 0 issues chunk `it` into stage it % S once the
  // stage's previous chunk has been consumed by every warp
  const bool ldx = fuse && c.xupd;
  const unsigned long long pol = l2_evict_first_policy();
  auto produce = [&](int it) {
    if (it >= nch) return;
    const int s = it % S;
    mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
    double* st = ring + (size_t)s * L.size;
    const int r0 = ra + it * L.rc, r1 = min(rb, r0 + L.rc);
    const uint32_t b_p = (uint32_t)(r1 - r0) * kp * 8u;
    const int v0 = r0 & ~1, w0 = (n + r0) & ~1;
    const uint32_t b_d = round_up16((uint32_t)(((r1 + 1) & ~1) - v0) * 8u);
    const uint32_t b_w = round_up16((uint32_t)(((n + r1 + 1) & ~1) - w0) * 8u);
    uint32_t b_e = 0, b_ec = 0;
    long long e0 = 0, c0 = 0;
    if (ew > 0) {
      e0 = ((long long)r0 * ew) & ~1LL;
      b_e = round_up16((uint32_t)((((long long)r1 * ew + 1) & ~1LL) - e0) * 8u);
      if (!direct) {
        c0 = ((long long)r0 * ew) & ~3LL;
        b_ec = round_up16((uint32_t)((((long long)r1 * ew + 3) & ~3LL) - c0) * 4u);
      }
    }
    mbar_expect_tx(&full[s], b_p + b_d + b_w + (fuse ? b_w : 0u) + (ldx ? b_w : 0u) + (direct ? 2u : 1u) * b_e + b_ec);
#ifndef QPK_NO_STREAM_HINT
    bulk_g2s_stream(st, P.P + (size_t)r0 * kp, b_p, &full[s], pol);   // the panel is streamed once per pass
#else
    bulk_g2s(st, P.P + (size_t)r0 * kp, b_p, &full[s]);
#endif
    bulk_g2s(st + L.o_d, op.d + v0, b_d, &full[s]);
    bulk_g2s(st + L.o_w, v + w0, b_w, &full[s]);
    if (fuse) bulk_g2s(st + L.o_r, E.r + w0, b_w, &full[s]);
    if (ldx) bulk_g2s(st + L.o_x, xsrc + w0, b_w, &full[s]);
    if (ew > 0) {
      bulk_g2s(st + L.o_ev, P.ev + e0, b_e, &full[s]);
      if (direct) bulk_g2s(st + L.o_ue, P.ue + e0, b_e, &full[s]);
      else bulk_g2s(st + L.o_ec, P.eci + c0, b_ec, &full[s]);
    }
  };
  const bool producer = warp == 0 && lane == 0;
  if (producer)
    for (int k = 0; k < S - 1; ++k) produce(k);
  {
    // ----------------------------------------------------------- consumers --
    double* xdst = E.x[c.xn];
    double* wv = v + n;
    const double* u = v;
    // u_P in registers: lane holds elements 2 lane + 64 q (+1), as the rows
    double2 ur[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = 64 * q + 2 * lane;
      const int c0 = __ldg(P.pcols + j), c1 = __ldg(P.pcols + j + 1);
      ur[q] = make_double2(c0 >= 0 ? u[c0] : 0.0, c1 >= 0 ? u[c1] : 0.0);
    }
    for (int it = 0; it < nch; ++it) {
      const int s = it % S;
      if (producer) produce(it + S - 1);
      mbar_wait(&full[s], (it / S) & 1);
      const double* st = ring + (size_t)s * L.size;
      const int r0 = ra + it * L.rc, r1 = min(rb, r0 + L.rc);
      const int v0 = r0 & ~1, w0 = (n + r0) & ~1;
      const long long e0 = ((long long)r0 * ew) & ~1LL, c0 = ((long long)r0 * ew) & ~3LL;
      for (int g0 = warp * RPW; r0 + g0 < r1; g0 += CW * RPW) {
        double sum[RPW], ea[RPW];
        double2 av[RPW][Q];                        // the rows, read from shared memory once
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          const bool ok = r0 + g0 + i < r1;
          const double* a = st + (size_t)(ok ? g0 + i : g0) * kp + 2 * lane;
#pragma unroll
          for (int q = 0; q < Q; ++q) av[i][q] = *reinterpret_cast<const double2*>(a + 64 * q);
        }
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          const bool ok = r0 + g0 + i < r1;
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            s0 = fma(av[i][q].x, ur[q].x, s0);
            s1 = fma(av[i][q].y, ur[q].y, s1);
          }
          sum[i] = s0 + s1;
          ea[i] = 0.0;
          if (ok && lane < ew) {
            const long long p = (long long)(r0 + g0 + i) * ew + lane;
            ea[i] = st[L.o_ev + p - e0];
            double ug;
            if (direct) {
              ug = st[L.o_ue + p - e0];
            } else {
              const int ec = reinterpret_cast<const int*>(st + L.o_ec)[p - c0];
              ug = ec >= 0 ? u[ec] : 0.0;
            }
            sum[i] = fma(ea[i], ug, sum[i]);
          }
        }
        // transposed reduction: with RPW = 2 the first butterfly level splits
        // the warp into two half-warps, one per row, so both rows' scalar
        // work (division included) runs side by side
        double tr;
        int mine;
        if (RPW == 2) {
          const bool hi = lane & 16;
          tr = (hi ? sum[RPW - 1] : sum[0]) + __shfl_xor_sync(0xffffffffu, hi ? sum[0] : sum[RPW - 1], 16);
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
          mine = hi ? 1 : 0;
        } else {
          tr = sum[0];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
          mine = 0;
        }
        constexpr int GS = 32 / RPW;             // lanes per row group
        const bool leader = (lane & (GS - 1)) == 0;
        double zm = 0.0;
        {
          const int r = r0 + g0 + mine;
          if (r < r1) {
            const double t = tr;
            const double dr = st[L.o_d + r - v0];
            double wr = st[L.o_w + n + r - w0];
            if (fuse) {
              const double rres = st[L.o_r + n + r - w0];
              const double zr = __dmul_rn(1.0 / dr, rres);
              const double pn = (c.mode == MODE_RESTART) ? zr : __dadd_rn(zr, __dmul_rn(c.beta, wr));
              if (leader) {
                if (c.xupd) xdst[n + r] = __dadd_rn(st[L.o_x + n + r - w0], __dmul_rn(c.alpha_prev, wr));
                wv[r] = pn;
                rzb += rres * zr;
              }
              wr = pn;
            }
            zm = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, t), dr), wr);
            const double yb = __dadd_rn(t, __dmul_rn(dr, wr));
            if (leader) {
              E.y[n + r] = yb;
              pacc += t * zm + wr * yb;
              if (!direct) E.zb[r] = zm;
            }
          }
        }
        double z[RPW];
#pragma unroll
        for (int i = 0; i < RPW; ++i) z[i] = __shfl_sync(0xffffffffu, zm, i * GS);
        if (direct && lane < ew) {
#pragma unroll
          for (int i = 0; i < RPW; ++i)
            if (r0 + g0 + i < r1) P.yrem[(long long)(r0 + g0 + i) * ew + lane] = z[i] * ea[i];
        }
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            acc[q].x = fma(z[i], av[i][q].x, acc[q].x);
            acc[q].y = fma(z[i], av[i][q].y, acc[q].y);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncwarp();
  __syncthreads();                               // every stage consumed: the ring is free
#pragma unroll
  for (int q = 0; q < Q; ++q) *reinterpret_cast<double2*>(ring + (size_t)warp * kp + 64 * q + 2 * lane) = acc[q];
  __syncthreads();
  for (int j = threadIdx.x; j < kp; j += blockDim.x) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < CW; ++w) sum += ring[(size_t)w * kp + j];
    P.ppart[(size_t)blockIdx.x * kp + j] = sum;
  }
  double tt = block_sum(pacc, red);
  if (threadIdx.x == 0) E.part[SLOT_ROWS * E.G + blockIdx.x] = tt;
  tt = block_sum(rzb, red);
  if (threadIdx.x == 0) E.part[SLOT_AUX2 * E.G + blockIdx.x] = tt;
}

// out[pcols[j]] (+)= sum over CTAs of ppart[cta][j], in CTA order.  Block b
// covers panel columns 32 b .. 32 b + 31; warp w sums CTAs w, w + 8, ...;
// the 8 warp sums are then added in warp order.
__global__ void __launch_bounds__(1024) k_panel_comb(Engine E, double* out, int add, int par) {
  __shared__ double ws[32][33];
  pdl_wait();
  pdl_trigger();
  if (par >= 0 && E.ctrl[par].mode == MODE_DONE) return;
  if (par >= 0 && blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_mid = globaltimer_ns();
  const Panel& P = E.panel;
  const int nb = P.kp / 32;
  if ((int)blockIdx.x >= nb) {
    // direct remainder: y[col] += yrem[p] (one entry per column: single writer)
    const long long ne = (long long)E.op.m * P.ew;
    for (long long p = (long long)(blockIdx.x - nb) * blockDim.x + threadIdx.x; p < ne;
         p += (long long)(gridDim.x - nb) * blockDim.x) {
      const int col = __ldg(P.eci + p);
      if (col >= 0) out[col] += P.yrem[p];
    }
    return;
  }
  // block b: panel columns 32 b .. 32 b + 31; warp w sums CTAs w, w + 32, ...
  // (independent loads), then the 32 warp sums in warp order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 32 + lane;
  double s0 = 0.0, s1 = 0.0;
  int g = warp;
  for (; g + 32 < P.G; g += 64) {
    s0 += P.ppart[(size_t)g * P.kp + j];
    s1 += P.ppart[(size_t)(g + 32) * P.kp + j];
  }
  if (g < P.G) s0 += P.ppart[(size_t)g * P.kp + j];
  ws[warp][lane] = s0 + s1;
  __syncthreads();
  if (warp == 0) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < 32; ++w) sum += ws[w][lane];
    const int col = __ldg(P.pcols + j);
    if (col >= 0) out[col] = add ? out[col] + sum : sum;
  }
}

// Jacobi partials of the panel: ppart[cta][j] = sum_r P_rj^2 / d_r over the
// CTA's rows (same row partition and order as k_slot_panel)
template <int Q>
__global__ void __launch_bounds__(QPK_PANEL_CW * 32, 1) k_jac_panel(Engine E) {
  extern __shared__ __align__(128) double psm[];
  const int W = blockDim.x >> 5;
  const Op& op = E.op;
  const Panel& P = E.panel;
  const int kp = P.kp;
  double* wacc = psm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ra = (int)((long long)op.m * blockIdx.x / gridDim.x);
  const int rb = (int)((long long)op.m * (blockIdx.x + 1) / gridDim.x);
  double2 acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int r = ra + warp; r < rb; r += W) {
    const double dinv = 1.0 / __ldg(op.d + r);
    const double* row = P.P + (size_t)r * kp + 2 * lane;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const double2 a = ld_stream_d2(row + 64 * q);
      acc[q].x += __dmul_rn(a.x, a.x) * dinv;
      acc[q].y += __dmul_rn(a.y, a.y) * dinv;
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) *reinterpret_cast<double2*>(wacc + warp * kp + 64 * q + 2 * lane) = acc[q];
  __syncthreads();
  for (int j = threadIdx.x; j < kp; j += blockDim.x) {
    double sum = 0.0;
    for (int w = 0; w < W; ++w) sum += wacc[w * kp + j];
    P.ppart[(size_t)blockIdx.x * kp + j] = sum;
  }
}

}  // namespace qpk
