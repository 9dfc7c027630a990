// qpk_engine.cuh -- the "slot engine": Jacobi-PCG (linalg.py:66-133) as a
// sequence of lean kernels instead of one cooperative kernel.
//
// One slot = three launches  top -> rows -> update.  A slot is either a PCG
// iteration (NORMAL / RESTART), the explicit-residual check the reference
// makes when the recurrence says "converged" (CHECK, linalg.py:112-125), the
// final true residual of the best iterate at the iteration cap (FINAL,
// linalg.py:132-133), or empty (DONE).  Which one is decided on the device:
// the control state lives in HBM, double-buffered by slot parity (slot s
// reads ctrl[s&1], the last block of its update kernel writes ctrl[(s+1)&1]),
// so the host only enqueues identical slots (replayed as a CUDA graph) and
// polls for DONE every few slots.  Each kernel has its own launch bounds, and
// the multi-GPU path inserts its collectives between the kernels of a slot.
#pragma once
#include "qpk_device.cuh"

#ifndef QPK_ROWS_PIPE
#define QPK_ROWS_PIPE false
#endif
#ifndef QPK_ROWS_MINB
#define QPK_ROWS_MINB 4
#endif

namespace qpk {

enum { MODE_NORMAL = 0, MODE_RESTART = 1, MODE_CHECK = 2, MODE_FINAL = 3, MODE_DONE = 4 };

struct Ctrl {
  int mode, k, cur, best, xn, xupd, status, converged, restarts, applies, result, pad;
  double rz, rnorm, best_rnorm, thr, rhs_norm, alpha_prev, beta, final_norm;
  unsigned long long t_top, t_rows, t_upd, t_mid, ph[4];   // t_mid: start of the B'z combine (tile / panel)
};

struct EngineCfg {
  double tol;
  long long max_iters;
  int rel;
  int pad;
  double* hist;       // nullable, max_iters + 1
};

#ifndef QPK_TILE_DOUBLES
#define QPK_TILE_DOUBLES 3072     // a dense tile holds <= 3072 values (24 KB)
#endif
#define QPK_TILE_ROWS 64
#ifndef QPK_TILE_DMAX
#define QPK_TILE_DMAX 512         // distinct columns per tile
#endif

// Dense row tiles (the "dictionary" mode): tile t covers rows [ra, rb) of B
// and its ndp (multiple of 4) distinct columns cols[d0 .. d0+ndp) (-1 pads);
// its entries are stored as a dense row-major (rb-ra) x ndp block at
// tval[v0 ..] -- banded / clustered B is 85-100 % dense inside such a tile,
// so no per-entry index is needed (~8-9 B per nonzero instead of 12).
// bpart[d0 + c] is the tile's partial of (B'z) for its column c;
// col_pos[col_ptr[j] .. col_ptr[j+1]) lists column j's bpart positions in
// tile order (deterministic combination).
struct TileDescD {
  int ra, rb, d0, ndp, v0, pad0, pad1, pad2;
};

struct Dict {
  int nblk;                 // number of tiles
  const TileDescD* tiles;
  const int* cols;
  const double* tval;
  double* bpart;
  const int* col_ptr;
  const int* col_pos;
  int comb_lanes;            // lanes per combine segment
  int nseg;                  // combine segments (<= QPK_COMB_CHUNK partials each)
  const int* seg_beg;        // segment q: col_pos[seg_beg[q] .. seg_beg[q+1])
  const int* col_seg;        // column j: segments [col_seg[j], col_seg[j+1])
  double* seg_sum;
  // CTA-level accumulation (cacc = 1): CTA b runs the consecutive tiles
  // [tile_beg[b], tile_beg[b+1]) and sums their B'z partials in shared memory
  // per column of its union cta_cols (tile column c -> slot tslot[d0 + c]),
  // written once to cpart[cta_off[b] ..]; the combine then reads these few
  // CTA partials (through the same segment structures) instead of one
  // partial per tile and column.
  const int* hperm;          // Hessian tiles: tile row q is H row hperm[q] (null: identity)
  int cacc;
  int l2pf;                  // producer L2 prefetch distance in tiles (0 = off, < 32)
  const int* tile_beg;
  const int* cta_off;
  const int* tslot;
  double* cpart;
};

// Dense column panel (the "panel" mode, for B with a block of dense columns --
// the SVM primal's [diag(y)X, y | I]): the columns present in most rows are
// stored as a dense row-major m x kp panel (no indices, 8 B per entry), the
// rest of each row ("remainder", <= 32 entries) as a fixed-width ELL strip.
// B'z of the panel accumulates in registers per warp, then per CTA
// (ppart[cta][j]), combined over CTAs in a fixed order (k_panel_comb).
struct Panel {
  int kp;                     // padded panel width (multiple of 64)
  int ew;                     // remainder ELL width (0..32)
  int direct;                 // every remainder column has <= 1 entry: y[col] += z a written directly
  int G;                      // CTAs of the panel kernel (partials)
  const double* P;            // m x kp row-major
  const int* pcols;           // kp panel columns (-1 pads)
  const int* eci;             // m x ew remainder columns (-1 pads)
  const double* ev;           // m x ew remainder values
  double* ppart;              // G x kp per-CTA partials of B'z (or of sum B^2/d)
  // direct mode: the remainder's u values are staged by the top kernel into
  // ue[] (entry order), and its B'z terms leave the panel kernel in yrem[]
  // (entry order), added to y by k_panel_comb -- no random access in the pass
  const int* cpos;            // n: entry position of column j's remainder entry, or -1 (direct mode)
  double* ue;                 // m x ew
  double* yrem;               // m x ew
};

struct Engine {
  Op op;
  Dict dict;
  Panel panel;
  int scatter;                // 1 atomic, 2 CSC segments, 3 row-block dictionary, 4 dense panel
  int sharded;                // row-sharded over ranks: collectives between the slot kernels
  int fold;                   // sharded tile format: [r'r, r'z] folded into the slot's one all-reduce
  double* gscal;              // [4] rank-summed ROWS, PREP, AUX, AUX2 totals (sharded)
  double* lscal2;             // [2] r'r, r'z (rank-local, then rank-summed)
  double* abuf;               // [2] alpha and the r'z it used (identical on every rank)
  const int* seg_ptr;         // CSC segments: column j owns segments [seg_ptr[j], seg_ptr[j+1])
  const int* seg_beg;         // segment q covers padded CSC entries [seg_beg[q], seg_beg[q+1])
  double* seg_sum;            // per-segment partial of (B'z)
  int n_seg;
  int seg_lanes;              // lanes per segment (segment <= 8 * seg_lanes entries)
  const double* rhs;
  double* x[3];
  double* r; double* p; double* y; double* zb;
  const double* minv;
  double* part; int G;
  int G_rows;                 // blocks of the rows kernel (its partials; <= G)
  Ctrl* ctrl;                 // [2]
  unsigned int* counter;      // last-block ticket
  const EngineCfg* cfg;
};

__device__ __forceinline__ int spare_of(int cur, int best) {
  return (cur != best) ? 3 - cur - best : (cur + 1) % 3;
}

// Last-block-done: every block has written its partials; the block that takes
// the final ticket sees all of them.  Returns true in exactly one block.
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
  }
  return am_last;
}

// initial control state from ||rhs||^2 (linalg.py:83, 93-94)
__device__ __forceinline__ void engine_init_state(const Engine& E, double rr0) {
  const double rn = sqrt(rr0);
  {
    const EngineCfg cfg = *E.cfg;
    Ctrl c;
    memset(&c, 0, sizeof c);
    c.rhs_norm = rn;
    c.thr = cfg.rel ? cfg.tol * rn : cfg.tol;
    c.rnorm = rn;
    c.best_rnorm = rn;
    c.mode = (rn <= c.thr) ? MODE_DONE : MODE_RESTART;
    c.converged = rn <= c.thr;
    c.final_norm = rn;
    c.t_top = globaltimer_ns();
    if (cfg.hist) cfg.hist[0] = rn;
    E.ctrl[0] = c;
  }
}

// ----------------------------------------------------------------- init ----
// x0 = 0, r = rhs (linalg.py:85-87); last block: ||rhs||, threshold
// (linalg.py:83), early return when rnorm <= threshold (linalg.py:93-94).
__global__ void __launch_bounds__(QPK_BLOCK) k_engine_init(Engine E) {
  __shared__ double red[32];
  const int N = E.op.n + E.op.m;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const double b = __ldg(E.rhs + i);
    E.x[0][i] = 0.0;
    E.r[i] = b;
    if (owns(E.op, i)) acc += b * b;
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) E.part[SLOT_AUX * E.G + blockIdx.x] = t;
  if (!last_block(E.counter)) return;
  const double rr0 = grid_total(E.part + SLOT_AUX * E.G, E.G, red);
  if (threadIdx.x == 0) {
    E.ctrl[1].mode = MODE_NORMAL;        // never a stale DONE from a previous solve
    if (E.sharded) { E.lscal2[0] = rr0; return; }   // summed over ranks, then k_engine_init2
    engine_init_state(E, rr0);
  }
}

// after the rank-sum of ||rhs||^2 (sharded)
__global__ void k_engine_init2(Engine E) {
  if (threadIdx.x == 0 && blockIdx.x == 0) engine_init_state(E, E.lscal2[0]);
}

// ------------------------------------------------------------------ top ----
__global__ void __launch_bounds__(QPK_BLOCK) k_slot_top(Engine E, int par) {
  __shared__ double red[32];
  pdl_wait();
  pdl_trigger();
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_top = globaltimer_ns();
  const Op& op = E.op;
  const int N = op.n + op.m, G = E.G;
  double rz = 0.0, acc = 0.0;
  double sacc[QPK_KMAX];
  double dacc[QPK_DENSE_ROWS_MAX] = {0.0, 0.0, 0.0, 0.0};   // dense B rows: partial c_r . v
  const int nd = op.ndense;
  const bool lr = op.H.kind == HESS_LOWRANK;
  if (lr) for (int kk = 0; kk < op.H.k; ++kk) sacc[kk] = 0.0;
  if ((c.mode == MODE_NORMAL || c.mode == MODE_RESTART) && nd && blockIdx.x == 0 && threadIdx.x == 0) {
    // the fused bottom update of the dense rows (phase_rows skips them)
    const double* xs = E.x[c.cur];
    double* xd = E.x[c.xn];
    for (int r = 0; r < nd; ++r) {
      const int i = op.n + r;
      const double dr = __ldg(op.d + r), rr = E.r[i], wr = E.p[i];
      const double zr = __dmul_rn(1.0 / dr, rr);
      if (c.xupd) xd[i] = __dadd_rn(xs[i], __dmul_rn(c.alpha_prev, wr));
      E.p[i] = (c.mode == MODE_RESTART) ? zr : __dadd_rn(zr, __dmul_rn(c.beta, wr));
      rz += rr * zr;
    }
  }
  if (c.mode == MODE_NORMAL || c.mode == MODE_RESTART) {
    // x_t += alpha_prev p_t (lazy), z = M^-1 r, p_t = z (+ beta p_t), y_t = diag(Q) p_t
    const bool restart = c.mode == MODE_RESTART;
    const double* xs = E.x[c.cur];
    double* xd = E.x[c.xn];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < op.n; j += gridDim.x * blockDim.x) {
      const double pold = E.p[j];
      if (c.xupd) xd[j] = __dadd_rn(xs[j], __dmul_rn(c.alpha_prev, pold));
      const double rj = E.r[j];
      const double zj = __dmul_rn(__ldg(E.minv + j), rj);
      if (j >= op.t_lo && j < op.t_hi) rz += rj * zj;
      const double pn = restart ? zj : __dadd_rn(zj, __dmul_rn(c.beta, pold));
      E.p[j] = pn;
      if (E.panel.cpos) { const int pp = __ldg(E.panel.cpos + j); if (pp >= 0) E.panel.ue[pp] = pn; }
      acc += prep_elem(op, j, pn, E.y);
      if (lr) lowrank_accum(op, j, pn, sacc);
      for (int q = 0; q < nd; ++q) dacc[q] = fma(__ldg(op.cdense + (size_t)q * op.n + j), pn, dacc[q]);
    }
  } else {
    // CHECK: materialise the pending x_k into x[xn] and prep(x_k).
    // FINAL: materialise the pending x (if any) and prep(x_best).
    const int target = (c.mode == MODE_CHECK) ? c.xn : c.best;
    const double* xs = E.x[c.cur];
    double* xd = E.x[c.xn];
    const double* xt = E.x[target];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
      double xv = 0.0;
      if (c.xupd) { xv = __dadd_rn(xs[i], __dmul_rn(c.alpha_prev, E.p[i])); xd[i] = xv; }
      if (i < op.n) {
        const double v = (c.xupd && target == c.xn) ? xv : xt[i];
        if (E.panel.cpos) { const int pp = __ldg(E.panel.cpos + i); if (pp >= 0) E.panel.ue[pp] = v; }
        acc += prep_elem(op, i, v, E.y);
        if (lr) lowrank_accum(op, i, v, sacc);
        for (int q = 0; q < nd; ++q) dacc[q] = fma(__ldg(op.cdense + (size_t)q * op.n + i), v, dacc[q]);
      }
    }
  }
  double t = block_sum(rz, red);
  if (threadIdx.x == 0) E.part[SLOT_AUX * G + blockIdx.x] = t;
  t = block_sum(acc, red);
  if (threadIdx.x == 0) E.part[SLOT_PREP * G + blockIdx.x] = t;
  if (lr) lowrank_flush(op, sacc, E.part, G, red);
  for (int q = 0; q < nd; ++q) {
    t = block_sum(dacc[q], red);
    if (threadIdx.x == 0) E.part[(SLOT_DR + q) * G + blockIdx.x] = t;
  }
}

// The dense rows of B after the row pass (same grid as the top kernel):
// t_r = c_r . v from the top kernel's partials (fixed order, every block gets
// the same value), z_r = 2 t_r / d_r + w_r, y_b = t_r + d_r w_r (block 0), and
// y_top += z_r c_r spread over the grid (atomic scatter mode; in CSC mode the
// column gather reads z_r).  v'Kv gets t z + w y_b.
template <bool CSC>
__global__ void __launch_bounds__(QPK_BLOCK) k_slot_dense(Engine E, int par) {
  __shared__ double red[32];
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  const Op& op = E.op;
  const int G = E.G;
  const double* v = (c.mode == MODE_NORMAL || c.mode == MODE_RESTART) ? E.p : E.x[c.mode == MODE_CHECK ? c.xn : c.best];
  double acc = 0.0;
  for (int q = 0; q < op.ndense; ++q) {
    const double t = grid_total(E.part + (SLOT_DR + q) * G, G, red);
    const double dr = __ldg(op.d + q), wr = v[op.n + q];
    const double z = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, t), dr), wr);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const double yb = __dadd_rn(t, __dmul_rn(dr, wr));
      E.y[op.n + q] = yb;
      E.zb[q] = z;
      acc += t * z + wr * yb;
    }
    if (!CSC) {
      const double* cr = op.cdense + (size_t)q * op.n;
      for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < op.n; j += gridDim.x * blockDim.x) {
        const double a = __ldg(cr + j);
        if (a != 0.0) atomicAdd(E.y + j, z * a);
      }
    }
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) E.part[SLOT_PREP * G + blockIdx.x] += t;
}

// ----------------------------------------------------------------- rows ----
template <int L, bool CSC>
__global__ void __launch_bounds__(QPK_BLOCK, QPK_ROWS_MINB) k_slot_rows(Engine E, int par) {
  __shared__ double red[32];
  __shared__ double s_lr[QPK_KMAX];
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par].t_rows = globaltimer_ns();
  if (c.mode == MODE_NORMAL || c.mode == MODE_RESTART) {
    RowFuse f;
    f.r = E.r;
    f.xsrc = E.x[c.cur];
    f.xdst = E.x[c.xn];
    f.alpha_prev = c.alpha_prev;
    f.beta = c.beta;
    f.restart = c.mode == MODE_RESTART;
    f.xupd = c.xupd;
    phase_rows<L, CSC, true, QPK_ROWS_PIPE>(E.op, E.p, E.y, E.zb, E.part, E.G, red, s_lr, f);
  } else {
    RowFuse none{};
    double* v = E.x[c.mode == MODE_CHECK ? c.xn : c.best];
    phase_rows<L, CSC, false, QPK_ROWS_PIPE>(E.op, v, E.y, E.zb, E.part, E.G, red, s_lr, none);
  }
}

// ------------------------------------------------------------------ csc ----
// B'z by column segments (deterministic, no atomics): each group of LS lanes
// owns one segment of <= 8 LS entries, so every lane issues its two chunks of
// row indices / values and all 8 z gathers at once.  Long columns (the dense
// X block of cfg2, RT bands) are split over many groups; short ones fill one.
__global__ void __launch_bounds__(QPK_BLOCK) k_slot_csc(Engine E, int par) {
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  const Op& op = E.op;
  const int LS = E.seg_lanes;
  const int ls = threadIdx.x & (LS - 1);
  const int per = 32 / LS, sw = (threadIdx.x & 31) / LS;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  const double* zb = E.zb;
  for (long long qb = (long long)gwarp * per; qb < E.n_seg; qb += (long long)nwarp * per) {
    const int q = (int)qb + sw;
    double s0 = 0.0, s1 = 0.0;
    if (q < E.n_seg) {
      const int b = __ldg(E.seg_beg + q), e = __ldg(E.seg_beg + q + 1);
      const int k = b + 4 * ls, k2 = k + 4 * LS;
      int4 c0 = make_int4(-1, -1, -1, -1), c1 = c0;
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, b0 = a0, b1 = a0;
      if (k < e) { c0 = ld_stream_i4(op.ri + k); a0 = ld_stream_d2(op.cv + k); a1 = ld_stream_d2(op.cv + k + 2); }
      if (k2 < e) { c1 = ld_stream_i4(op.ri + k2); b0 = ld_stream_d2(op.cv + k2); b1 = ld_stream_d2(op.cv + k2 + 2); }
      if (c0.x >= 0) s0 = fma(a0.x, zb[c0.x], s0);
      if (c0.y >= 0) s0 = fma(a0.y, zb[c0.y], s0);
      if (c0.z >= 0) s0 = fma(a1.x, zb[c0.z], s0);
      if (c0.w >= 0) s0 = fma(a1.y, zb[c0.w], s0);
      if (c1.x >= 0) s1 = fma(b0.x, zb[c1.x], s1);
      if (c1.y >= 0) s1 = fma(b0.y, zb[c1.y], s1);
      if (c1.z >= 0) s1 = fma(b1.x, zb[c1.z], s1);
      if (c1.w >= 0) s1 = fma(b1.y, zb[c1.w], s1);
    }
    double s = s0 + s1;
    for (int o = LS / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (q < E.n_seg && ls == 0) E.seg_sum[q] = s;
  }
}

// y_j (final) of a top entry: y_j plus its column's deterministic partials
// (CSC segments, or dictionary block partials), summed in a fixed order
template <int SC>
__device__ __forceinline__ double top_value(const Engine& E, int j) {
  double s = 0.0;
  if (SC == 2) {
    const int qb = __ldg(E.seg_ptr + j), qe = __ldg(E.seg_ptr + j + 1);
    for (int q = qb; q < qe; ++q) s += E.seg_sum[q];
  } else if (SC == 3) {
    // 8 partial positions, then 8 partials in flight per round trip; the sum
    // keeps the partial order (bitwise the same as one at a time)
    const int qb = __ldg(E.dict.col_ptr + j), qe = __ldg(E.dict.col_ptr + j + 1);
    const double* src = E.dict.cacc ? E.dict.cpart : E.dict.bpart;
    for (int q = qb; q < qe; q += 8) {
      int pos[8];
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pos[k] = (q + k < qe) ? __ldg(E.dict.col_pos + q + k) : -1;
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (pos[k] >= 0) ? src[pos[k]] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (q + k < qe) s += v[k];
    }
  }
  return E.y[j] + s;
}


// Sharded slot: finish this rank's top block (y_top + its local B'z
// partials) and the rank-local totals of the slot's scalar partials, both
// then summed over ranks by one grouped all-reduce.
template <int SC>
__global__ void __launch_bounds__(QPK_BLOCK) k_shard_reduce(Engine E, int par) {
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) return;
  if (SC != 1)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < E.op.n; j += gridDim.x * blockDim.x)
      E.y[j] = top_value<SC>(E, j);
  if (!last_block(E.counter)) return;
  // the last block: one warp per scalar, all of them side by side (lane-strided
  // partial sums, then a butterfly: a fixed order)
  const int G = E.G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nq = E.fold ? 10 : 4;
  for (int q = warp; q < nq; q += nw) {
    const int slot = q == 0 ? SLOT_ROWS : q == 1 ? SLOT_PREP : q == 2 ? SLOT_AUX : q == 3 ? SLOT_AUX2 : SLOT_F + (q - 4);
    const int cnt = (q == 1 || q == 2) ? G : E.G_rows;
    const double* src = E.part + slot * G;
    double t = 0.0;
    for (int i = lane; i < cnt; i += 32) t += src[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) E.gscal[q] = t;
  }
}


// The PCG control decision after a slot (one thread): next mode, iteration
// count, best iterate, beta -- linalg.py:104-133 for the scalars.
__device__ __forceinline__ void decide(const Engine& E, const Ctrl& c, int par, double rr_tot, double rz_tot,
                                       double alpha, double rz, unsigned long long t_upd) {
  const EngineCfg cfg = *E.cfg;
  const unsigned long long now = globaltimer_ns();
  Ctrl o = c;
  o.applies += 1;
  o.ph[0] += c.t_rows - c.t_top;
  if (c.t_mid > c.t_rows && c.t_mid < t_upd) {
    o.ph[1] += c.t_mid - c.t_rows;
    o.ph[3] += t_upd - c.t_mid;
  } else {
    o.ph[1] += t_upd - c.t_rows;
  }
  o.ph[2] += now - t_upd;
  o.t_mid = 0;
  const double nrm = sqrt(rr_tot);
  if (c.mode == MODE_NORMAL || c.mode == MODE_RESTART) {
    const int cur = c.xupd ? c.xn : c.cur;               // x_{k-1} was materialised this slot
    o.k = c.k + 1;
    if (cfg.hist) cfg.hist[o.k] = nrm;
    o.rnorm = nrm;
    o.cur = cur;
    o.xn = spare_of(cur, c.best);                        // x_k = x_{k-1} + alpha p lands here
    o.xupd = 1;
    o.alpha_prev = alpha;
    if (nrm < c.best_rnorm) { o.best = o.xn; o.best_rnorm = nrm; }   // linalg.py:110-111
    if (nrm <= c.thr) {
      o.mode = MODE_CHECK;                                // linalg.py:112
    } else if (o.k >= cfg.max_iters) {
      o.mode = MODE_FINAL;
    } else {
      o.mode = MODE_NORMAL;                               // linalg.py:126-130
      o.beta = rz_tot / rz;
      o.rz = rz_tot;
    }
  } else if (c.mode == MODE_CHECK) {
    o.cur = c.xn;
    o.xupd = 0;
    if (nrm <= c.thr) {                                   // linalg.py:115-116
      o.mode = MODE_DONE;
      o.converged = 1;
      o.final_norm = nrm;
      o.result = c.xn;
    } else {                                              // linalg.py:117-125
      o.restarts += 1;
      o.rnorm = nrm;
      if (nrm < c.best_rnorm) { o.best = c.xn; o.best_rnorm = nrm; }
      o.xn = spare_of(o.cur, o.best);
      o.mode = (c.k >= cfg.max_iters) ? MODE_FINAL : MODE_RESTART;
    }
  } else {                                                // FINAL (linalg.py:132-133)
    o.mode = MODE_DONE;
    o.k = (int)cfg.max_iters;
    o.converged = nrm <= c.thr;
    o.final_norm = nrm;
    o.result = c.best;
    o.cur = c.xupd ? c.xn : c.cur;
    o.xupd = 0;
  }
  E.ctrl[par ^ 1] = o;
}

// --------------------------------------------------------------- update ----
#define QPK_FOLD_BLOCKS 128       // blocks that walk the replicated top block in the folded sharded slot
#ifndef QPK_UPD_U
#define QPK_UPD_U 4               // independent double2 pairs in flight per thread
#endif
template <int SC>
__global__ void __launch_bounds__(QPK_BLOCK) k_slot_update(Engine E, int par) {
  constexpr bool CSC = SC != 1;
  __shared__ double red[32];
  pdl_wait();
  pdl_trigger();
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE) {
    if (blockIdx.x == 0 && threadIdx.x == 0) E.ctrl[par ^ 1] = c;
    return;
  }
  const unsigned long long t_upd = globaltimer_ns();
  const Op& op = E.op;
  const int G = E.G;
  const int N = op.n + op.m;
  double rr = 0.0, rzn = 0.0;
  double alpha = 0.0, rz = c.rz;
  if (c.mode == MODE_NORMAL || c.mode == MODE_RESTART) {
    double pap;
    if (E.sharded) {
      pap = E.gscal[0] + E.gscal[1];
      if (c.mode == MODE_RESTART) rz = E.gscal[2] + E.gscal[3];
    } else {
      double t_rows, t_prep;
      grid_total2(E.part + SLOT_ROWS * G, E.G_rows, E.part + SLOT_PREP * G, G, red, t_rows, t_prep);
      pap = t_rows + t_prep;
      if (c.mode == MODE_RESTART) {
        double t_aux, t_aux2;
        grid_total2(E.part + SLOT_AUX * G, G, E.part + SLOT_AUX2 * G, E.G_rows, red, t_aux, t_aux2);
        rz = t_aux + t_aux2;
      }
    }
    if (pap <= 0.0) {                                                   // linalg.py:102-103
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        Ctrl o = c;
        o.mode = MODE_DONE;
        o.status = QPK_PCG_BREAKDOWN;
        o.converged = 0;
        o.applies += 1;
        o.final_norm = c.best_rnorm;
        o.result = c.best;
        E.ctrl[par ^ 1] = o;
      }
      return;
    }
    alpha = rz / pap;
    if (E.fold) {
      // Folded sharded slot: every rank sums the WHOLE replicated top block
      // itself and takes the control decision from it, so the sum must come out
      // bit-identical on all ranks whatever their grids are: the top entries
      // are walked by a FIXED geometry (QPK_FOLD_BLOCKS blocks), the bottom
      // entries (whose sums arrive through the all-reduce) by the whole grid.
      if ((int)blockIdx.x < QPK_FOLD_BLOCKS) {
        // pairs (16-byte accesses; r, y, minv are 16-byte aligned), the odd last entry by one thread
        const int ntp = op.n >> 1, stride = QPK_FOLD_BLOCKS * blockDim.x;
        double2* r2 = reinterpret_cast<double2*>(E.r);
        const double2* y2 = reinterpret_cast<const double2*>(E.y);
        const double2* m2 = reinterpret_cast<const double2*>(E.minv);
        for (int base = blockIdx.x * blockDim.x + threadIdx.x; base < ntp; base += 2 * stride) {
          const int i1 = base + stride;
          double2 ra = r2[base], ya = y2[base], ma = __ldg(m2 + base), rb, yb, mb;
          if (i1 < ntp) { rb = r2[i1]; yb = y2[i1]; mb = __ldg(m2 + i1); }
          ra.x = __dsub_rn(ra.x, __dmul_rn(alpha, ya.x));
          ra.y = __dsub_rn(ra.y, __dmul_rn(alpha, ya.y));
          r2[base] = ra;
          rr += ra.x * ra.x; rzn += ra.x * __dmul_rn(ma.x, ra.x);
          rr += ra.y * ra.y; rzn += ra.y * __dmul_rn(ma.y, ra.y);
          if (i1 < ntp) {
            rb.x = __dsub_rn(rb.x, __dmul_rn(alpha, yb.x));
            rb.y = __dsub_rn(rb.y, __dmul_rn(alpha, yb.y));
            r2[i1] = rb;
            rr += rb.x * rb.x; rzn += rb.x * __dmul_rn(mb.x, rb.x);
            rr += rb.y * rb.y; rzn += rb.y * __dmul_rn(mb.y, rb.y);
          }
        }
        if ((op.n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
          const int i = op.n - 1;
          const double ri = __dsub_rn(E.r[i], __dmul_rn(alpha, E.y[i]));
          E.r[i] = ri;
          rr += ri * ri;
          rzn += ri * __dmul_rn(__ldg(E.minv + i), ri);
        }
      }
      {
        constexpr int U = 4;
        const int stride = gridDim.x * blockDim.x;
        for (int base = op.n + blockIdx.x * blockDim.x + threadIdx.x; base < N; base += U * stride) {
          double rv[U], yv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = base + u * stride;
            if (i < N) { rv[u] = E.r[i]; yv[u] = E.y[i]; }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = base + u * stride;
            if (i < N) E.r[i] = __dsub_rn(rv[u], __dmul_rn(alpha, yv[u]));
          }
        }
      }
    } else {
    // scalar head: top entries whose y needs its column partials (CSC / tile
    // modes), rounded up to an even index so the rest runs on double2 pairs
    const int nb = CSC ? min(N, (op.n + 1) & ~1) : 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
      const double yi = (i < op.n) ? top_value<SC>(E, i) : E.y[i];
      const double ri = __dsub_rn(E.r[i], __dmul_rn(alpha, yi));
      E.r[i] = ri;
      if (owns(op, i)) {
        rr += ri * ri;
        rzn += ri * __dmul_rn(__ldg(E.minv + i), ri);
      }
    }
    // pairs: QPK_UPD_U independent pairs per thread with every load issued
    // before the first store (r is read and written, so the compiler cannot
    // hoist the next iteration's loads on its own)
    {
      constexpr int U = QPK_UPD_U;
      const int p0 = nb >> 1, np = N >> 1;
      const int stride = gridDim.x * blockDim.x;
      double2* r2 = reinterpret_cast<double2*>(E.r);
      const double2* y2 = reinterpret_cast<const double2*>(E.y);
      const double2* m2 = reinterpret_cast<const double2*>(E.minv);
      for (int base = p0 + blockIdx.x * blockDim.x + threadIdx.x; base < np; base += U * stride) {
        double2 rv[U], yv[U], mv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = base + u * stride;
          if (i < np) { rv[u] = r2[i]; yv[u] = __ldg(y2 + i); mv[u] = __ldg(m2 + i); }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = base + u * stride;
          if (i < np) {
            double2 ri = rv[u];
            ri.x = __dsub_rn(ri.x, __dmul_rn(alpha, yv[u].x));
            ri.y = __dsub_rn(ri.y, __dmul_rn(alpha, yv[u].y));
            r2[i] = ri;
            // replicated top entries count once over the ranks (rank 0)
            const bool cx = owns(op, 2 * i), cy = owns(op, 2 * i + 1);
            if (cx) { rr += ri.x * ri.x; rzn += ri.x * __dmul_rn(mv[u].x, ri.x); }
            if (cy) { rr += ri.y * ri.y; rzn += ri.y * __dmul_rn(mv[u].y, ri.y); }
          }
        }
      }
      if ((N & 1) && N - 1 >= nb && blockIdx.x == 0 && threadIdx.x == 0) {
        const double ri = __dsub_rn(E.r[N - 1], __dmul_rn(alpha, E.y[N - 1]));
        E.r[N - 1] = ri;
        if (owns(op, N - 1)) {
          rr += ri * ri;
          rzn += ri * __dmul_rn(__ldg(E.minv + N - 1), ri);
        }
      }
    }
    }
  } else if (E.fold) {
    // explicit residual, folded slot: top block by the fixed geometry (see above)
    const bool store = c.mode == MODE_CHECK;
    if ((int)blockIdx.x < QPK_FOLD_BLOCKS)
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < op.n; i += QPK_FOLD_BLOCKS * blockDim.x) {
        const double ri = __dsub_rn(__ldg(E.rhs + i), E.y[i]);
        if (store) E.r[i] = ri;
        rr += ri * ri;
      }
    if (store)
      for (int i = op.n + blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
        E.r[i] = __dsub_rn(__ldg(E.rhs + i), E.y[i]);
  } else {
    // explicit residual rhs - K x (CHECK stores it as the new r; FINAL only needs its norm)
    const bool store = c.mode == MODE_CHECK;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
      const double yi = (CSC && i < op.n) ? top_value<SC>(E, i) : E.y[i];
      const double ri = __dsub_rn(__ldg(E.rhs + i), yi);
      if (store) E.r[i] = ri;
      if (owns(op, i)) rr += ri * ri;
    }
  }
  double t = block_sum(rr, red);
  if (threadIdx.x == 0) E.part[SLOT_RR * G + blockIdx.x] = t;
  t = block_sum(rzn, red);
  if (threadIdx.x == 0) E.part[SLOT_RZ * G + blockIdx.x] = t;
  if (!last_block(E.counter)) return;

  // ---- decision (one block) ----
  double rr_tot, rz_tot;
  grid_total2(E.part + SLOT_RR * G, G, E.part + SLOT_RZ * G, G, red, rr_tot, rz_tot);
  if (threadIdx.x != 0) return;
  if (E.fold) {
    // One all-reduce per iteration: every rank summed the WHOLE replicated top
    // block above (identical on all ranks); the bottom block's share comes
    // from the sums the tile pass formed before alpha was known and the slot's
    // all-reduce added over the ranks:
    //   |r - a y|^2 = r'r - 2 a r'y + a^2 y'y      (and the same weighted by M^-1)
    // (explicit-residual slots: gscal[4] = sum (rhs - y)^2 over the bottom block)
    const double* F = E.gscal + 4;
    if (c.mode == MODE_NORMAL || c.mode == MODE_RESTART) {
      rr_tot += fma(alpha, fma(alpha, F[2], -2.0 * F[1]), F[0]);
      rz_tot += fma(alpha, fma(alpha, F[5], -2.0 * F[4]), F[3]);
    } else {
      rr_tot += F[0];
    }
    decide(E, c, par, rr_tot, rz_tot, alpha, rz, t_upd);
    return;
  }
  if (E.sharded) {
    // rank-local totals; summed over ranks by the collective, then k_slot_decide
    E.lscal2[0] = rr_tot;
    E.lscal2[1] = rz_tot;
    E.abuf[0] = alpha;
    E.abuf[1] = rz;
    E.ctrl[par].t_upd = t_upd;
    return;
  }
  decide(E, c, par, rr_tot, rz_tot, alpha, rz, t_upd);
}

// out = K v after the operator part of a MODE_CHECK slot (qpk_apply in the
// tile / panel modes): y plus, in CSC mode, the top entries' segment sums
template <int SC>
__global__ void __launch_bounds__(QPK_BLOCK) k_apply_finish(Engine E, double* out) {
  const int N = E.op.n + E.op.m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
    out[i] = (SC != 1 && i < E.op.n) ? top_value<SC>(E, i) : E.y[i];
}

// decision after a sharded slot: the collective has summed rr / rz over ranks
__global__ void k_slot_decide(Engine E, int par) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const Ctrl c = E.ctrl[par];
  if (c.mode == MODE_DONE || E.ctrl[par ^ 1].mode == MODE_DONE) return;   // done, or breakdown already decided
  decide(E, c, par, E.lscal2[0], E.lscal2[1], E.abuf[0], E.abuf[1], c.t_upd);
}

}  // namespace qpk
