// DSMEM random-access throughput probe (B200): can a thread-block cluster hold
// a slab of the cfg5 gather/scatter vector in distributed shared memory and
// serve random fp64 gathers / atomics faster than L2 (~287 G/s gathers,
// ~190 G/s fp64 atomics; profiles/r01_probe_random_access2.txt)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probes/dsmem_probe probes/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double ld_dsmem(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void red_dsmem(uint32_t a, double v) {
  asm volatile("red.shared::cluster.add.f64 [%0], %1;" :: "r"(a), "d"(v) : "memory");
}

// MODE 0: gathers, random rank; 1: fp64 red, random rank; 2: gathers, own rank
template <int MODE>
__global__ void probe(int ns, long long per_block, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t cs = cl.num_blocks();
  for (int i = threadIdx.x; i < ns; i += blockDim.x) sm[i] = i;
  cl.sync();
  const uint32_t base = smem_u32(sm);
  double s = 0;
  const uint32_t me = cl.block_rank();
  for (long long i = threadIdx.x; i < per_block; i += blockDim.x) {
    uint32_t h = hash((uint32_t)(i + (long long)blockIdx.x * 1000003));
    uint32_t rank = (MODE == 2) ? me : (h % cs);
    uint32_t off = (h >> 4) % ns;
    uint32_t a = mapa(base + 8 * off, rank);
    if (MODE == 1) red_dsmem(a, 1.0);
    else s += ld_dsmem(a);
  }
  cl.sync();
  if (s == 1.2345) out[0] = s;
}

template <int MODE>
float run(int cs, int blocks, int threads, int ns, long long per_block) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = ns * 8;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  CK(cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * 8));
  CK(cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, (void*)probe<MODE>, &cfg) != cudaSuccess) { cudaGetLastError(); ncl = -1; }
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaLaunchKernelEx(&cfg, probe<MODE>, ns, per_block, out));
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int it = 0; it < 3; ++it) CK(cudaLaunchKernelEx(&cfg, probe<MODE>, ns, per_block, out));
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  double total = (double)per_block * blocks;
  printf("mode %d cluster %2d blocks %3d (max active clusters %d) threads %4d smem %6d B: %.3f ms  %.1f G/s\n",
         MODE, cs, blocks, ncl, threads, ns * 8, ms, total / ms / 1e6);
  cudaFree(out);
  return ms;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("%s SMs %d\n", p.name, p.multiProcessorCount);
  const long long per_block = 1 << 21;
  const int ns = 24 * 1024;                 // 192 KB per CTA
  int css[] = {1, 2, 4, 8, 16};
  for (int cs : css) {
    int blocks = (p.multiProcessorCount / cs) * cs;
    if (cs == 16) blocks = 128;
    if (cs == 8) blocks = 144;
    run<0>(cs, blocks, 1024, ns, per_block);
    run<2>(cs, blocks, 1024, ns, per_block);
    run<1>(cs, blocks, 1024, ns, per_block);
  }
  run<0>(8, 144, 512, ns, per_block);
  run<0>(16, 128, 512, ns, per_block);
  return 0;
}
