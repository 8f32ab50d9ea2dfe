// ilp_probe.cu -- chain step with ILP chains per thread interleaved step by step (Mx paths);
// result (profiles/r01f_ilp_probe.txt): two chains per thread are 5-20 % slower than one.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2512_23969_b200/csrc/sha256.cuh"
using namespace hs;
// chain step x15 per chain; ILP chains per thread interleaved step by step
template <class V, int NW, int ILP>
__global__ void __launch_bounds__(128) k(uint32_t* out, int reps) {
  uint32_t mid[8];
  for (int i = 0; i < 8; i++) mid[i] = 0x6a09e667u * (i + 1);
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t x[ILP][NW];
  for (int c = 0; c < ILP; c++) for (int j = 0; j < NW; j++) x[c][j] = (tid * ILP + c) * 2654435761u + 17u * j;
  for (int r = 0; r < reps; r++) {
    Adrs a[ILP]; uint32_t pre[ILP][8];
    for (int c = 0; c < ILP; c++) {
      a[c] = make_adrs(3, (tid * ILP + c) + r, 0u, 1, r & 63, 0);
      const uint32_t W04[5] = {a[c].w0, a[c].w1, a[c].w2, a[c].w3, a[c].w4};
      for (int i = 0; i < 8; i++) pre[c][i] = mid[i];
      rounds_prefix<V, 5>(pre[c], W04);
    }
#pragma unroll 1
    for (uint32_t s = 0; s < 15; s++) {
#pragma unroll
      for (int c = 0; c < ILP; c++) {
        uint32_t W[16];
        W[0] = a[c].w0; W[1] = a[c].w1; W[2] = a[c].w2; W[3] = a[c].w3; W[4] = a[c].w4;
        W[5] = join16(s, x[c][0]);
        for (int j = 1; j < NW; j++) W[5 + j] = join16(x[c][j - 1], x[c][j]);
        W[5 + NW] = (x[c][NW - 1] << 16) | 0x8000u;
        for (int j = 6 + NW; j < 15; j++) W[j] = 0;
        W[15] = (64 + 22 + 4 * NW) * 8;
        uint32_t st[8];
        for (int i = 0; i < 8; i++) st[i] = mid[i];
        compress_resume<V, 5>(st, pre[c], W);
        for (int j = 0; j < NW; j++) x[c][j] = st[j];
      }
    }
  }
  for (int c = 0; c < ILP; c++) for (int j = 0; j < NW; j++) out[((size_t)tid * ILP + c) * NW + j] = x[c][j];
}
template <class V, int NW, int ILP>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 64 / ILP, reps = 8; const size_t threads = (size_t)blocks * 128;
  uint32_t* out; cudaMalloc(&out, threads * ILP * NW * 4);
  k<V, NW, ILP><<<blocks, 128>>>(out, 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int t = 0; t < 3; t++) { cudaEventRecord(a); k<V, NW, ILP><<<blocks, 128>>>(out, reps); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k<V, NW, ILP>);
  printf("%s NW=%d ILP=%d regs=%d %.3f Gstep/s\n", name, NW, ILP, fa.numRegs, (double)threads * ILP * reps * 15 / best / 1e6);
  cudaFree(out);
}
int main() {
  run<Mx<248>, 4, 1>("mx248"); run<Mx<248>, 4, 2>("mx248");
  run<Mx<248>, 6, 1>("mx248"); run<Mx<248>, 6, 2>("mx248");
  run<Mx<248>, 8, 1>("mx248"); run<Mx<248>, 8, 2>("mx248");
  run<Mx<232>, 4, 2>("mx232"); run<Mx<104>, 4, 2>("mx104"); run<Native, 4, 2>("native");
  return 0;
}
