/*
 * sort_keys.c -- the C ABI used from plain C, without Python or torch.
 *
 * Generates keys on the device with os_keygen (keygen.py:46-76), sorts them
 * with os_sort (binning.py:278-337) carrying each key's input index as its
 * value, times the sort with CUDA events, and checks the result on the host:
 * keys ascend in the reference's encoded order (keycodec.py:157-181), the
 * values are a permutation of 0..n-1, every value points at an input key with
 * the same bits, and equal keys keep their input order (stability).
 *
 *   make -C examples            (or see the Makefile next to this file)
 *   examples/sort_keys [log2_n] [u32|u64|i32|i64|f32|f64] [values: 0|1]
 *
 * Prints "OK ..." and exits 0, or prints what failed and exits 1.
 */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "onesweep_b200.h"

#define CK(call)                                                                 \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #call,               \
              cudaGetErrorString(e_));                                           \
      return 1;                                                                  \
    }                                                                            \
  } while (0)
#define OS(call)                                                                 \
  do {                                                                           \
    int s_ = (call);                                                             \
    if (s_ != OS_OK) {                                                           \
      fprintf(stderr, "%s:%d %s: status %d: %s\n", __FILE__, __LINE__, #call, s_, \
              os_last_error());                                                  \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

/* encoded (order-preserving unsigned) form of a key's bits */
static uint64_t encode(uint64_t x, int type) {
  switch (type) {
    case OS_KEY_I32: return (x ^ 0x80000000u) & 0xffffffffu;
    case OS_KEY_I64: return x ^ 0x8000000000000000ull;
    case OS_KEY_F32: return ((x >> 31) ? ~x : (x | 0x80000000u)) & 0xffffffffu;
    case OS_KEY_F64: return (x >> 63) ? ~x : (x | 0x8000000000000000ull);
    default: return x;
  }
}

int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 24;
  const char* tname = argc > 2 ? argv[2] : "u32";
  const int with_values = argc > 3 ? atoi(argv[3]) : 1;
  static const char* names[] = {"u32", "u64", "i32", "i64", "f32", "f64"};
  int type = -1;
  for (int t = 0; t < 6; ++t)
    if (strcmp(tname, names[t]) == 0) type = t;
  if (type < 0 || lg < 0 || lg > 30) {
    fprintf(stderr, "usage: %s [log2_n <= 30] [u32|u64|i32|i64|f32|f64] [0|1]\n", argv[0]);
    return 2;
  }
  const size_t n = (size_t)1 << lg;
  const int kb = (type == OS_KEY_U64 || type == OS_KEY_I64 || type == OS_KEY_F64) ? 8 : 4;
  const int vb = with_values ? 4 : 0;

  void *keys, *keys_out, *vals = NULL, *vals_out = NULL, *ws;
  CK(cudaMalloc(&keys, n * kb));
  CK(cudaMalloc(&keys_out, n * kb));
  OS(os_keygen(keys, n, kb * 8, 1, 2026ull, 0ull, NULL));
  uint32_t* idx = (uint32_t*)malloc(n * 4);
  if (with_values) {
    for (size_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
    CK(cudaMalloc(&vals, n * 4));
    CK(cudaMalloc(&vals_out, n * 4));
    CK(cudaMemcpy(vals, idx, n * 4, cudaMemcpyHostToDevice));
  }
  const size_t wsb = os_sort_workspace_bytes(n, type, vb, 8, 0, kb * 8, 0, 0);
  if (wsb == 0) {
    fprintf(stderr, "os_sort_workspace_bytes: %s\n", os_last_error());
    return 1;
  }
  CK(cudaMalloc(&ws, wsb));

  cudaStream_t st;
  cudaEvent_t e0, e1;
  CK(cudaStreamCreate(&st));
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  OS(os_sort(keys, keys_out, vals, vals_out, n, type, vb, 8, 0, kb * 8, 0, 0, ws, wsb, NULL, st));
  const int reps = 10;
  CK(cudaEventRecord(e0, st));
  for (int r = 0; r < reps; ++r)
    OS(os_sort(keys, keys_out, vals, vals_out, n, type, vb, 8, 0, kb * 8, 0, 0, ws, wsb, NULL, st));
  CK(cudaEventRecord(e1, st));
  OS(os_stream_check(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;

  unsigned char* hin = (unsigned char*)malloc(n * kb);
  unsigned char* hout = (unsigned char*)malloc(n * kb);
  uint32_t* hv = (uint32_t*)malloc(n * 4);
  unsigned char* seen = (unsigned char*)calloc(n, 1);
  CK(cudaMemcpy(hin, keys, n * kb, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hout, keys_out, n * kb, cudaMemcpyDeviceToHost));
  if (with_values) CK(cudaMemcpy(hv, vals_out, n * 4, cudaMemcpyDeviceToHost));

  uint64_t prev = 0;
  for (size_t i = 0; i < n; ++i) {
    uint64_t raw = 0, src = 0;
    memcpy(&raw, hout + i * kb, kb);
    const uint64_t enc = encode(raw, type);
    if (i && enc < prev) {
      fprintf(stderr, "FAIL: not ascending at %zu\n", i);
      return 1;
    }
    if (with_values) {
      const uint32_t v = hv[i];
      if (v >= n || seen[v]) {
        fprintf(stderr, "FAIL: values not a permutation at %zu\n", i);
        return 1;
      }
      seen[v] = 1;
      memcpy(&src, hin + (size_t)v * kb, kb);
      if (src != raw) {
        fprintf(stderr, "FAIL: value %u does not point at its key (output %zu)\n", v, i);
        return 1;
      }
      if (i && enc == prev && hv[i - 1] > v) {
        fprintf(stderr, "FAIL: unstable at %zu\n", i);
        return 1;
      }
    }
    prev = enc;
  }
  printf("OK n=%zu type=%s values=%d ms=%.3f GKey/s=%.2f\n", n, tname, with_values, ms,
         (double)n / (ms * 1e6));
  cudaFree(keys); cudaFree(keys_out); cudaFree(vals); cudaFree(vals_out); cudaFree(ws);
  free(idx); free(hin); free(hout); free(hv); free(seen);
  return 0;
}
