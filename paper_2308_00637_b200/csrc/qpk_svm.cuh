// qpk_svm.cuh -- SVM dual frontend on the device.
//
// The reference builds the dual of the kernel SVM (qpipm/svm.py:179-195) with
// a dense RBF Gram matrix (svm.py:146-176):
//     sq = rowwise |x_i|^2 ; g = X X' ; d2 = max(sq_i + sq_j - 2 g_ij, 0)
//     K = exp(-d2 / (2 sigma)) ; H = (y y') * K        (exactly symmetric)
// k_rbf_hessian computes H in one pass over the upper triangle of 64 x 64
// output tiles: X panels staged in shared memory, a 4 x 4 register block of
// dot products per thread, the RBF epilogue fused, and each off-diagonal tile
// written twice (directly and, through shared memory, transposed) so H is
// symmetric bit for bit: g_ij and g_ji come from the same fma sequence.
// fp64 throughout; X is n x d row-major, H n x n row-major.
#pragma once

#define QPK_GRAM_T 64     // output tile edge
#define QPK_GRAM_K 16     // features per shared-memory stage

__global__ void __launch_bounds__(256) k_rowsq(const double* __restrict__ X, long long n, long long d,
                                              double* __restrict__ sq) {
  // one thread per row, the same fma chain over k as the tile's dot products,
  // so that d2_ii = sq_i + sq_i - 2 g_ii is exactly 0 (K_ii = 1)
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* row = X + i * d;
  double s = 0.0;
  for (long long k = 0; k < d; ++k) s = fma(row[k], row[k], s);
  sq[i] = s;
}

__global__ void __launch_bounds__(256) k_rbf_hessian(const double* __restrict__ X, long long n, long long d,
                                                    const double* __restrict__ y, const double* __restrict__ sq,
                                                    double inv2s, double* __restrict__ H) {
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bi > bj) return;                                   // upper triangle of tiles only
  // the X stages and the output tile share one buffer (the tile is formed
  // after the last stage is consumed)
  __shared__ double buf[QPK_GRAM_T * (QPK_GRAM_T + 1)];
  double (*As)[QPK_GRAM_T + 1] = reinterpret_cast<double (*)[QPK_GRAM_T + 1]>(buf);
  double (*Bs)[QPK_GRAM_T + 1] = reinterpret_cast<double (*)[QPK_GRAM_T + 1]>(buf + QPK_GRAM_K * (QPK_GRAM_T + 1));
  double (*Ct)[QPK_GRAM_T + 1] = reinterpret_cast<double (*)[QPK_GRAM_T + 1]>(buf);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // 16 x 16 threads, 4 x 4 outputs each
  const long long i0 = (long long)bi * QPK_GRAM_T, j0 = (long long)bj * QPK_GRAM_T;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (long long k0 = 0; k0 < d; k0 += QPK_GRAM_K) {
    // stage X[i0:i0+64, k0:k0+16] and X[j0:j0+64, k0:k0+16] transposed (feature-major)
    for (int e = threadIdx.x; e < QPK_GRAM_T * QPK_GRAM_K; e += 256) {
      const int r = e / QPK_GRAM_K, kk = e % QPK_GRAM_K;
      const long long k = k0 + kk;
      const long long ia = i0 + r, jb = j0 + r;
      As[kk][r] = (ia < n && k < d) ? X[ia * d + k] : 0.0;
      Bs[kk][r] = (jb < n && k < d) ? X[jb * d + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < QPK_GRAM_K; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = As[kk][ty * 4 + q]; b[q] = Bs[kk][tx * 4 + q]; }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
  // epilogue: RBF of the squared distance, label product (svm.py:171-176, 185)
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const long long i = i0 + ty * 4 + p;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long j = j0 + tx * 4 + q;
      double h = 0.0;
      if (i < n && j < n) {
        const double d2 = fmax(__dsub_rn(__dadd_rn(sq[i], sq[j]), __dmul_rn(2.0, acc[p][q])), 0.0);
        h = __dmul_rn(__dmul_rn(y[i], y[j]), exp(-__dmul_rn(d2, inv2s)));
        H[i * n + j] = h;
      }
      Ct[ty * 4 + p][tx * 4 + q] = h;
    }
  }
  if (bi == bj) return;                                  // diagonal tile: both halves written above
  __syncthreads();
  // transposed copy: H[j][i] = H[i][j], coalesced along i
  for (int e = threadIdx.x; e < QPK_GRAM_T * QPK_GRAM_T; e += 256) {
    const int jl = e / QPK_GRAM_T, il = e % QPK_GRAM_T;
    const long long i = i0 + il, j = j0 + jl;
    if (i < n && j < n) H[j * n + i] = Ct[il][jl];
  }
}

// out = H v for a dense row-major n x n matrix: one warp per row, 16-byte
// loads with four independent accumulators (fixed order: deterministic)
__global__ void __launch_bounds__(256) k_dense_gemv(const double* __restrict__ Hm, long long n,
                                                   const double* __restrict__ v, double* __restrict__ out) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int ln = threadIdx.x & 31;
  for (long long j = w; j < n; j += nw) {
    const double* row = Hm + j * n;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if ((n & 1) == 0 && (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
      const double2* r2 = reinterpret_cast<const double2*>(row);
      const double2* v2 = reinterpret_cast<const double2*>(v);
      const long long h = n >> 1;
      long long c = ln;
      for (; c + 32 < h; c += 64) {
        const double2 a = __ldg(r2 + c), b = __ldg(r2 + c + 32);
        const double2 x = v2[c], z = v2[c + 32];
        s0 = fma(a.x, x.x, s0); s1 = fma(a.y, x.y, s1);
        s2 = fma(b.x, z.x, s2); s3 = fma(b.y, z.y, s3);
      }
      for (; c < h; c += 32) {
        const double2 a = __ldg(r2 + c), x = v2[c];
        s0 = fma(a.x, x.x, s0); s1 = fma(a.y, x.y, s1);
      }
    } else {
      for (long long c = ln; c < n; c += 32) s0 = fma(__ldg(row + c), v[c], s0);
    }
    double s = (s0 + s1) + (s2 + s3);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (ln == 0) out[j] = s;
  }
}
