// Throwaway-style microbenchmark kept for evidence: how fast can B200 stream a
// cfg5-shaped CSR (4M x 1M, 16 nnz/row, fp64) with random-column gathers, and
// what does the one-pass fused apply (gather + fp64 atomic scatter) cost versus
// a two-pass CSR + CSC (gather-only) apply.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o probes/spmv_probe probes/spmv_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ int4 ldg_nc_i4(const int* p) {
  int4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r;
}
__device__ __forceinline__ double2 ldg_nc_d2(const double* p) {
  double2 r; asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                          : "=d"(r.x), "=d"(r.y) : "l"(p)); return r;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// 4 lanes per row, 4 nnz per lane (exactly 16 nnz per row)
template <bool FUSED>
__global__ void __launch_bounds__(256) apply16(int m, const int* __restrict__ cols, const double* __restrict__ vals,
                                               const double* __restrict__ u, const double* __restrict__ w,
                                               const double* __restrict__ d, double* __restrict__ bottom,
                                               double* __restrict__ top) {
  int lane4 = threadIdx.x & 3;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < 4LL * m; g += (long long)gridDim.x * blockDim.x) {
    int row = (int)(g >> 2);
    long long base = (long long)row * 16 + lane4 * 4;
    int4 c = ldg_nc_i4(cols + base);
    double2 v0 = ldg_nc_d2(vals + base);
    double2 v1 = ldg_nc_d2(vals + base + 2);
    double s = v0.x * __ldg(u + c.x) + v0.y * __ldg(u + c.y) + v1.x * __ldg(u + c.z) + v1.y * __ldg(u + c.w);
    s += __shfl_xor_sync(0xffffffff, s, 1);
    s += __shfl_xor_sync(0xffffffff, s, 2);
    if (FUSED) {
      double dd = __ldg(d + row), ww = __ldg(w + row);
      double coef = 2.0 * s / dd + ww;
      if (lane4 == 0) bottom[row] = s + dd * ww;
      atomicAdd(top + c.x, coef * v0.x);
      atomicAdd(top + c.y, coef * v0.y);
      atomicAdd(top + c.z, coef * v1.x);
      atomicAdd(top + c.w, coef * v1.y);
    } else {
      if (lane4 == 0) bottom[row] = s;
    }
  }
}

// generic CSR vector kernel, L lanes per row (gather only)
template <int L>
__global__ void __launch_bounds__(256) csr_vec(int m, const int* __restrict__ rp, const int* __restrict__ ci,
                                               const double* __restrict__ v, const double* __restrict__ x,
                                               double* __restrict__ y) {
  int lane = threadIdx.x & (L - 1);
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < (long long)L * m; g += (long long)gridDim.x * blockDim.x) {
    int row = (int)(g / L);
    int b = rp[row], e = rp[row + 1];
    double s = 0;
    for (int k = b + lane; k < e; k += L) s += __ldg(v + k) * __ldg(x + __ldg(ci + k));
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
    if (lane == 0) y[row] = s;
  }
}

__global__ void scatter_only(int m, const int* __restrict__ cols, double* __restrict__ top) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < 4LL * m; g += (long long)gridDim.x * blockDim.x) {
    int4 c = ldg_nc_i4(cols + g * 4);
    atomicAdd(top + c.x, 1.0); atomicAdd(top + c.y, 1.0); atomicAdd(top + c.z, 1.0); atomicAdd(top + c.w, 1.0);
  }
}

__global__ void gather_only(int m, const int* __restrict__ cols, const double* __restrict__ u, double* __restrict__ out) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < 4LL * m; g += (long long)gridDim.x * blockDim.x) {
    int4 c = ldg_nc_i4(cols + g * 4);
    double s = __ldg(u + c.x) + __ldg(u + c.y) + __ldg(u + c.z) + __ldg(u + c.w);
    if (s == 12345.678) out[0] = s;
  }
}

template <typename F>
float time_it(F f, int reps = 20) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; i++) f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; i++) f();
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGetLastError());
  return ms / reps;
}

int main(int argc, char** argv) {
  const int m = 4000000, n = 1000000, K = 16;
  const long long nnz = (long long)m * K;
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d L2 %d MB smem/SM %zu\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20,
         prop.sharedMemPerMultiprocessor);
  int sms = prop.multiProcessorCount;
  std::mt19937_64 rng(5);
  std::vector<int> cols(nnz);
  std::vector<double> vals(nnz);
  std::normal_distribution<double> nd;
  for (long long r = 0; r < m; r++) {
    int* c = &cols[r * K];
    for (int k = 0; k < K; k++) c[k] = (int)(rng() % n);
    std::sort(c, c + K);
    for (int k = 0; k < K; k++) vals[r * K + k] = nd(rng);
  }
  // CSC via counting sort
  std::vector<int> cp(n + 1, 0), ri(nnz);
  std::vector<double> cv(nnz);
  for (long long k = 0; k < nnz; k++) cp[cols[k] + 1]++;
  for (int j = 0; j < n; j++) cp[j + 1] += cp[j];
  {
    std::vector<int> pos(cp.begin(), cp.end() - 1);
    for (long long r = 0; r < m; r++)
      for (int k = 0; k < K; k++) { long long q = r * K + k; int p = pos[cols[q]]++; ri[p] = (int)r; cv[p] = vals[q]; }
  }
  std::vector<int> rp(m + 1);
  for (int r = 0; r <= m; r++) rp[r] = r * K;

  int *d_cols, *d_rp, *d_cp, *d_ri; double *d_vals, *d_cv, *d_u, *d_w, *d_d, *d_bot, *d_top;
  CK(cudaMalloc(&d_cols, nnz * 4)); CK(cudaMalloc(&d_vals, nnz * 8));
  CK(cudaMalloc(&d_rp, (m + 1) * 4)); CK(cudaMalloc(&d_cp, (n + 1) * 4));
  CK(cudaMalloc(&d_ri, nnz * 4)); CK(cudaMalloc(&d_cv, nnz * 8));
  CK(cudaMalloc(&d_u, n * 8)); CK(cudaMalloc(&d_top, n * 8));
  CK(cudaMalloc(&d_w, m * 8)); CK(cudaMalloc(&d_d, m * 8)); CK(cudaMalloc(&d_bot, m * 8));
  CK(cudaMemcpy(d_cols, cols.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_vals, vals.data(), nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rp, rp.data(), (m + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cp, cp.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ri, ri.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cv, cv.data(), nnz * 8, cudaMemcpyHostToDevice));
  std::vector<double> h(m, 1.0);
  CK(cudaMemcpy(d_u, h.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_w, h.data(), m * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_d, h.data(), m * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(d_top, 0, n * 8));

  // copy bandwidth
  size_t cn = (size_t)1 << 26;  // 64M double2 = 1 GiB
  double2 *ca, *cb; CK(cudaMalloc(&ca, cn * 16)); CK(cudaMalloc(&cb, cn * 16));
  CK(cudaMemset(ca, 0, cn * 16));
  float t = time_it([&] { copy_kernel<<<sms * 8, 256>>>(ca, cb, cn); });
  printf("copy: %.3f ms  %.1f GB/s\n", t, 2.0 * cn * 16 / t / 1e6);
  CK(cudaFree(ca)); CK(cudaFree(cb));

  double bytes_csr = nnz * 12.0 + m * 4.0;
  for (int occ : {4, 8, 16}) {
    int grid = sms * occ;
    t = time_it([&] { apply16<false><<<grid, 256>>>(m, d_cols, d_vals, d_u, d_w, d_d, d_bot, d_top); });
    printf("csr16 gather-only SpMV grid=%d: %.3f ms  algorithmic(CSR+x+y) %.1f GB/s\n", grid, t,
           (nnz * 12.0 + m * 8.0 + n * 8.0) / t / 1e6);
    t = time_it([&] { apply16<true><<<grid, 256>>>(m, d_cols, d_vals, d_u, d_w, d_d, d_bot, d_top); });
    printf("fused one-pass apply (atomics) grid=%d: %.3f ms  algorithmic %.1f GB/s\n", grid, t,
           (bytes_csr + 8.0 * n * 2 + 8.0 * m * 3) / t / 1e6);
  }
  t = time_it([&] { scatter_only<<<sms * 8, 256>>>(m, d_cols, d_top); });
  printf("scatter-only (64M f64 atomics + col stream): %.3f ms  %.2f Gatomic/s\n", t, nnz / t / 1e6);
  t = time_it([&] { gather_only<<<sms * 8, 256>>>(m, d_cols, d_u, d_bot); });
  printf("gather-only (64M random f64 loads + col stream): %.3f ms  %.2f Gload/s\n", t, nnz / t / 1e6);
  t = time_it([&] { csr_vec<4><<<sms * 8, 256>>>(m, d_rp, d_cols, d_vals, d_u, d_bot); });
  printf("csr_vec<4> B*u: %.3f ms  %.1f GB/s\n", t, (bytes_csr + 8.0 * (n + m)) / t / 1e6);
  for (int L : {8, 16, 32}) {
    if (L == 8) t = time_it([&] { csr_vec<8><<<sms * 8, 256>>>(n, d_cp, d_ri, d_cv, d_bot, d_top); });
    if (L == 16) t = time_it([&] { csr_vec<16><<<sms * 8, 256>>>(n, d_cp, d_ri, d_cv, d_bot, d_top); });
    if (L == 32) t = time_it([&] { csr_vec<32><<<sms * 8, 256>>>(n, d_cp, d_ri, d_cv, d_bot, d_top); });
    printf("csc csr_vec<%d> B^T*z: %.3f ms  %.1f GB/s\n", L, t, (nnz * 12.0 + n * 4.0 + 8.0 * (n + m)) / t / 1e6);
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
