// How fast do the SMs read / atomically update an L2-resident vector with
// COALESCED accesses?  (cfg5: would sweeping u through shared memory in blocks,
// or flushing per-block y slices with coalesced atomics, beat one random
// sector request per nonzero?)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probes/l2_stream_probe probes/l2_stream_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

// every block sweeps the whole table `reps` times, 16-byte loads
__global__ void sweep(const double2* __restrict__ u, int n2, int reps, double* out) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x + ((blockIdx.x * 37 + r * 11) % 64) * blockDim.x; i < n2; i += blockDim.x * 64) {
      // each block reads 1/64 of the table per rep, a different part each time
      const double2 v = u[i];
      s += v.x + v.y;
    }
  if (s == 1.2345) out[0] = s;
}
// full sweep into shared memory with cp.async-like plain loads + st.shared
__global__ void sweep_full(const double2* __restrict__ u, int n2, int reps, double* out) {
  extern __shared__ double2 sm[];
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (int base = 0; base < n2; base += 4096) {
      for (int i = threadIdx.x; i < 4096 && base + i < n2; i += blockDim.x) sm[i] = u[base + i];
      __syncthreads();
      s += sm[(threadIdx.x * 7) & 4095].x;
      __syncthreads();
    }
  if (s == 1.2345) out[0] = s;
}
// coalesced atomics: every block adds a vector into the table, consecutive lanes -> consecutive doubles
__global__ void atomic_sweep(double* y, int n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x + ((blockIdx.x * 37 + r * 11) % 64) * blockDim.x; i < n; i += blockDim.x * 64)
      atomicAdd(y + i, 1.0);
}
template <typename F> float time_it(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a)); for (int i = 0; i < reps; i++) f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); CK(cudaGetLastError()); return ms / reps;
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  const int n = 1 << 20;                       // 1M doubles = 8 MB (cfg5's u / y_top)
  double *u, *out; CK(cudaMalloc(&u, n * 8)); CK(cudaMalloc(&out, 8)); CK(cudaMemset(u, 0, n * 8));
  const int reps = 64;
  for (int bps : {1, 2, 4}) {
    float t = time_it([&] { sweep<<<sms * bps, 512>>>((const double2*)u, n / 2, reps, out); });
    double bytes = (double)sms * bps * reps * (n * 8.0 / 64);
    printf("coalesced L2 read, %d blocks/SM x 512 thr: %.3f ms  %.1f GB/s  (%.2f sectors/clk/SM at 1.9 GHz)\n", bps, t,
           bytes / t / 1e6, bytes / 32 / (t * 1e-3) / sms / 1.9e9);
  }
  CK(cudaFuncSetAttribute(sweep_full, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  {
    float t = time_it([&] { sweep_full<<<sms, 1024, 65536>>>((const double2*)u, n / 2, 4, out); });
    double bytes = (double)sms * 4 * n * 8.0;
    printf("full sweeps of the 8 MB table into smem, 1 block/SM: %.3f ms  %.1f GB/s -> one sweep per SM = %.1f us\n", t,
           bytes / t / 1e6, t * 1e3 / 4);
  }
  for (int bps : {1, 4}) {
    float t = time_it([&] { atomic_sweep<<<sms * bps, 512>>>(u, n, reps); });
    double ops = (double)sms * bps * reps * (n / 64.0);
    printf("coalesced fp64 atomics, %d blocks/SM: %.3f ms  %.1f G atomics/s  (%.1f G sectors/s)\n", bps, t, ops / t / 1e6,
           ops / 4 / t / 1e6);
  }
  return 0;
}
