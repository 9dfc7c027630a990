// Random-access throughput probe (B200): where is the limit for the random
// fp64 gathers / atomics that dominate the cfg5 operator apply?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probes/random_probe probes/random_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if (MODE == 0) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if (MODE == 1) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if (MODE == 2) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// each thread does `per` random gathers (indices from a hash, no index stream)
template <int MODE>
__global__ void gather(const double* __restrict__ u, int n, long long total, double* out) {
  double s = 0;
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < total; i += nth) {
    uint32_t h = hash((uint32_t)i);
    s += ld<MODE>(u + (h % n));
  }
  if (s == 1.2345) out[0] = s;
}

__global__ void gather2(const double2* __restrict__ u, int n2, long long total, double* out) {
  double s = 0;
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < total; i += nth) {
    uint32_t h = hash((uint32_t)i);
    double2 v = u[h % n2];
    s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}

template <typename T>
__global__ void scatter(T* y, int n, long long total) {
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < total; i += nth) {
    uint32_t h = hash((uint32_t)i);
    atomicAdd(y + (h % n), (T)1);
  }
}

// random fp64 gathers from shared memory (smem-resident slice)
__global__ void smem_gather(long long total_per_block, double* out) {
  extern __shared__ double sm[];
  const int ns = 24 * 1024;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double s = 0;
  for (long long i = threadIdx.x; i < total_per_block; i += blockDim.x) {
    uint32_t h = hash((uint32_t)(i + blockIdx.x * 7919));
    s += sm[h % ns];
  }
  if (s == 1.2345) out[0] = s;
}

__global__ void smem_atomic(long long total_per_block, double* out) {
  extern __shared__ double sm[];
  const int ns = 24 * 1024;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  for (long long i = threadIdx.x; i < total_per_block; i += blockDim.x) {
    uint32_t h = hash((uint32_t)(i + blockIdx.x * 7919));
    atomicAdd(sm + (h % ns), 1.0);
  }
  __syncthreads();
  if (sm[threadIdx.x] == 1.2345) out[0] = 1;
}

// hash-only baseline
__global__ void hash_only(long long total, double* out) {
  uint32_t s = 0;
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < total; i += nth) s += hash((uint32_t)i) % 1000000;
  if (s == 12345) out[0] = s;
}

template <typename F>
float time_it(F f, int reps = 10) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int i = 0; i < 2; i++) f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; i++) f();
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGetLastError());
  return ms / reps;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("SMs %d clock %d MHz\n", sms, clk / 1000);
  const int n = 1 << 20;  // 1M doubles = 8 MB
  const long long total = 64LL << 20;
  double *u, *out; float* uf;
  CK(cudaMalloc(&u, (size_t)n * 32 * 8)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&uf, n * 4));
  CK(cudaMemset(u, 0, (size_t)n * 32 * 8)); CK(cudaMemset(uf, 0, n * 4));
  float t;
  t = time_it([&] { hash_only<<<sms * 8, 256>>>(total, out); });
  printf("hash only: %.3f ms\n", t);
  for (int occ : {4, 8}) {
    t = time_it([&] { gather<0><<<sms * occ, 256>>>(u, n, total, out); });
    printf("gather ld.global (occ %d): %.3f ms  %.1f G/s\n", occ, t, total / t / 1e6);
  }
  t = time_it([&] { gather<1><<<sms * 8, 256>>>(u, n, total, out); });
  printf("gather ld.global.cg: %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  t = time_it([&] { gather<2><<<sms * 8, 256>>>(u, n, total, out); });
  printf("gather ld.global.nc: %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  t = time_it([&] { gather<3><<<sms * 8, 256>>>(u, n, total, out); });
  printf("gather ld.nc.L1::no_allocate: %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  t = time_it([&] { gather<0><<<sms / 2 * 8, 256>>>(u, n, total, out); });
  printf("gather ld.global, half the SMs' worth of blocks (%d): %.3f ms  %.1f G/s\n", sms / 2 * 8, t, total / t / 1e6);
  t = time_it([&] { gather<0><<<sms * 8, 256>>>(u, 1 << 14, total, out); });
  printf("gather ld.global, 128 KB table (L1-resident-ish): %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  t = time_it([&] { gather<0><<<sms * 8, 256>>>(u, n * 32, total, out); });
  printf("gather ld.global, 256 MB table (HBM): %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  t = time_it([&] { gather2<<<sms * 8, 256>>>((const double2*)u, n / 2, total, out); });
  printf("gather double2 (16B), 8 MB: %.3f ms  %.1f G req/s\n", t, total / t / 1e6);
  t = time_it([&] { scatter<double><<<sms * 8, 256>>>(u, n, total); });
  printf("atomic f64 8 MB: %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  t = time_it([&] { scatter<float><<<sms * 8, 256>>>(uf, n, total); });
  printf("atomic f32 4 MB: %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  t = time_it([&] { scatter<double><<<sms * 8, 256>>>(u, n * 32, total); });
  printf("atomic f64 256 MB: %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  CK(cudaFuncSetAttribute(smem_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024 * 8));
  CK(cudaFuncSetAttribute(smem_atomic, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024 * 8));
  long long per_block = total / sms;
  t = time_it([&] { smem_gather<<<sms, 1024, 24 * 1024 * 8>>>(per_block, out); });
  printf("smem random gather (1 block/SM, 1024 thr): %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  t = time_it([&] { smem_atomic<<<sms, 1024, 24 * 1024 * 8>>>(per_block, out); });
  printf("smem random f64 atomicAdd: %.3f ms  %.1f G/s\n", t, total / t / 1e6);
  printf("done\n");
  return 0;
}
