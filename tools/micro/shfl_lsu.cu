// Microbenchmark: does SHFL compete with shared-memory loads for the L1/LSU
// data pipe?  Kernels: LDS only, SHFL only, both interleaved (same counts).
// If time(both) ~ time(LDS) + time(SHFL), they share the pipe.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_lds(unsigned* out, int salt) {
  __shared__ unsigned s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 2654435761u;
  __syncthreads();
  unsigned x = threadIdx.x * 33u + salt, acc = 0;
  #pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(&s[(x + i * 32) & 4095])));
    acc += v;
  }
  if (acc == 0x12345) out[0] = acc;
}
__global__ void k_shfl(unsigned* out, int salt) {
  unsigned x = threadIdx.x * 33u + salt, acc = 0;
  #pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    unsigned v = __shfl_sync(0xffffffffu, x + i, (x + i) & 31);
    acc += v;
  }
  if (acc == 0x12345) out[0] = acc;
}
__global__ void k_both(unsigned* out, int salt) {
  __shared__ unsigned s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 2654435761u;
  __syncthreads();
  unsigned x = threadIdx.x * 33u + salt, acc = 0;
  #pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    unsigned v, w;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(&s[(x + i * 32) & 4095])));
    w = __shfl_sync(0xffffffffu, x + i, (x + i) & 31);
    acc += v ^ w;
  }
  if (acc == 0x12345) out[0] = acc;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}

int main() {
  unsigned* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  dim3 g(sms * 4), b(256);
  float t1 = timeit([&] { k_lds<<<g, b>>>(out, 1); });
  float t2 = timeit([&] { k_shfl<<<g, b>>>(out, 1); });
  float t3 = timeit([&] { k_both<<<g, b>>>(out, 1); });
  double warp_ops = double(g.x) * (b.x / 32) * ITERS;
  double clk = 1.965e9 * sms;
  printf("LDS only : %.3f ms  %.2f warp-instr/clk/SM\n", t1, warp_ops / (t1 * 1e-3) / clk);
  printf("SHFL only: %.3f ms  %.2f warp-instr/clk/SM\n", t2, warp_ops / (t2 * 1e-3) / clk);
  printf("both     : %.3f ms  (sum of the two: %.3f, max: %.3f)\n", t3, t1 + t2, t1 > t2 ? t1 : t2);
  return 0;
}
