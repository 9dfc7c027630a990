// TMA 1-D bulk-copy streaming probe (B200): global -> shared through a ring of
// mbarrier-tracked stages, one producer lane per CTA, consumers only touch one
// word per stage.  How does throughput depend on stage size and on splitting
// a stage into several copies?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probes/tma_probe probes/tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

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
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int STAGES>
__global__ void stream(const char* __restrict__ src, long long total, int stage_bytes, int pieces, double* out) {
  extern __shared__ __align__(128) char sm[];
  unsigned long long* full = (unsigned long long*)(sm + STAGES * stage_bytes);
  unsigned long long* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw - 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long ntiles = total / stage_bytes;
  double acc = 0;
  if (warp == nw - 1) {
    if ((threadIdx.x & 31) == 0) {
      int it = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % STAGES;
        mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[s], stage_bytes);
        const int piece = stage_bytes / pieces;
        for (int p = 0; p < pieces; ++p)
          bulk_g2s(sm + s * stage_bytes + p * piece, src + t * stage_bytes + p * piece, piece, &full[s]);
      }
    }
  } else {
    int it = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      acc += ((const double*)(sm + s * stage_bytes))[threadIdx.x];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long total = 2LL << 30;
  char* src; double* out;
  CK(cudaMalloc(&src, total)); CK(cudaMalloc(&out, 8)); CK(cudaMemset(src, 0, total));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  const int sizes[] = {4096, 8192, 16384, 32768};
  for (int stages : {2, 4, 6}) {
    for (int sz : sizes) {
      for (int pieces : {1, 4, 16}) {
        const int smem = stages * sz + 2 * stages * 8;
        if (smem > 220 * 1024) continue;
        auto k = stages == 2 ? stream<2> : stages == 4 ? stream<4> : stream<6>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int ctas_per_sm : {1, 2}) {
          if (ctas_per_sm * smem > 220 * 1024) continue;
          k<<<sms * ctas_per_sm, 288, smem>>>(src, total, sz, pieces, out);
          CK(cudaDeviceSynchronize());
          CK(cudaEventRecord(a));
          for (int r = 0; r < 5; ++r) k<<<sms * ctas_per_sm, 288, smem>>>(src, total, sz, pieces, out);
          CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
          float ms; CK(cudaEventElapsedTime(&ms, a, b));
          printf("stages %d stage %6d B pieces %2d ctas/SM %d: %7.1f GB/s\n", stages, sz, pieces, ctas_per_sm,
                 5.0 * total / (ms * 1e6));
        }
      }
    }
  }
  return 0;
}
