// Microbenchmark: L1/LSU data-pipe cost of staging a tile through TMA + LDS
// versus loading it straight into registers with coalesced LDG.  Each block
// reads TILE u32 keys per iteration from an L2-resident buffer and folds
// them into a checksum.  Compare l1tex__data_pipe_lsu_wavefronts per 128 B.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int THREADS = 256, ITEMS = 40, TILE = THREADS * ITEMS, ITERS = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(THREADS, 4) k_tma(const uint32_t* __restrict__ src, size_t words, uint32_t* out) {
  extern __shared__ __align__(128) uint32_t tile[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t acc = 0, phase = 0;
  for (int it = 0; it < ITERS; ++it) {
    const size_t off = (size_t(blockIdx.x) * ITERS + it) * TILE % (words - TILE);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(TILE * 4));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(tile)), "l"(src + off), "r"(TILE * 4), "r"(smem_u32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
    phase ^= 1;
#pragma unroll 8
    for (int i = 0; i < ITEMS; ++i) acc += tile[i * THREADS + threadIdx.x] * (i + 1);
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (acc == 0x12345u) out[0] = acc;
}

__global__ void __launch_bounds__(THREADS, 4) k_ldg(const uint32_t* __restrict__ src, size_t words, uint32_t* out) {
  uint32_t acc = 0;
  for (int it = 0; it < ITERS; ++it) {
    const size_t off = (size_t(blockIdx.x) * ITERS + it) * TILE % (words - TILE);
#pragma unroll 8
    for (int i = 0; i < ITEMS; ++i) {
      uint32_t v;
      asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(src + off + i * THREADS + threadIdx.x));
      acc += v * (i + 1);
    }
  }
  if (acc == 0x12345u) out[0] = acc;
}

int main() {
  const size_t words = size_t(16) << 20;  // 64 MiB: L2-resident-ish working set
  uint32_t *src, *out;
  cudaMalloc(&src, words * 4);
  cudaMalloc(&out, 4);
  cudaMemset(src, 1, words * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int r = 0; r < 2; ++r) {
    float t1, t2;
    cudaEventRecord(a);
    k_tma<<<sms * 4, THREADS, TILE * 4>>>(src, words, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&t1, a, b);
    cudaEventRecord(a);
    k_ldg<<<sms * 4, THREADS>>>(src, words, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&t2, a, b);
    const double bytes = double(sms) * 4 * ITERS * TILE * 4;
    printf("TMA+LDS %.3f ms (%.0f GB/s)   LDG %.3f ms (%.0f GB/s)\n", t1, bytes / t1 / 1e6, t2, bytes / t2 / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
