// lat_probe.cu -- latency of ONE thread's sequential SHA-256 compressions on
// B200 (the critical path of small batches: msg_prep, T_len, T_k, Merkle
// levels).  For each arithmetic path and code shape it times, with clock64 in
// one warp: the first compression (cold instruction cache) and the steady
// state over 64 dependent compressions.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//        -o tools/lat_probe tools/lat_probe.cu && tools/lat_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2512_23969_b200/csrc/sha256.cuh"

using namespace hs;

template <class V, int SHAPE>
__device__ __forceinline__ void one(uint32_t st[8], uint32_t W[16]) {
  if (SHAPE == 0) {
    compress<V>(st, W);
  } else {
    compress_compact<V>(st, W);
  }
}

template <class V, int SHAPE>
__global__ void lat_kernel(uint32_t* out, long long* cyc, int n) {
  uint32_t st[8], W[16];
  for (int i = 0; i < 8; i++) st[i] = IVc(i) ^ threadIdx.x;
  for (int j = 0; j < 16; j++) W[j] = 0x01010101u * j;
  long long t0 = clock64();
  one<V, SHAPE>(st, W);
  for (int j = 0; j < 16; j++) W[j] = st[j & 7] + j;  // next block depends on this one
  long long t1 = clock64();
#pragma unroll 1
  for (int r = 0; r < n; r++) {
    one<V, SHAPE>(st, W);
    for (int j = 0; j < 16; j++) W[j] = st[j & 7] + j;
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
  out[threadIdx.x] = st[0];
}

template <class V, int SHAPE>
void run(const char* name, uint32_t* d_out, long long* d_cyc) {
  const int n = 64;
  long long h[2];
  for (int rep = 0; rep < 3; rep++) {
    lat_kernel<V, SHAPE><<<1, 32>>>(d_out, d_cyc, n);
    cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-10s %-8s rep %d: first %6lld cycles, steady %6.0f cycles/compression\n", name,
           SHAPE == 0 ? "unrolled" : "compact", rep, h[0], (double)h[1] / n);
  }
}

int main() {
  uint32_t* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 32 * sizeof(uint32_t));
  cudaMalloc(&d_cyc, 2 * sizeof(long long));
  run<Native, 0>("native", d_out, d_cyc);
  run<Native, 1>("native", d_out, d_cyc);
  run<Mx<248>, 0>("mx248", d_out, d_cyc);
  run<Mx<248>, 1>("mx248", d_out, d_cyc);
  run<Fast, 0>("fast", d_out, d_cyc);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
