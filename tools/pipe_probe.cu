// pipe_probe.cu -- integer pipe throughput microbenchmark for sm_100a.
// Measures warp-instructions per clock per SM for the instruction forms the
// SHA-256 paths use (IADD3, LOP3, SHF, IMAD with constant-bank operand,
// IMAD.HI, IMAD.WIDE, PRMT) and for ALU/FMA mixes.  Each thread runs 8
// independent dependency chains so latency is hidden.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__constant__ uint32_t c_one = 1u, c_m = 0x20000000u;

#define CH 8
template <int OP>
__global__ void probe(uint32_t* out, int iters, long long* clk) {
  uint32_t x[CH];
  for (int i = 0; i < CH; i++) x[i] = threadIdx.x * 7 + i;
  uint32_t one = c_one, m = c_m;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int i = 0; i < CH; i++) {
        if (OP == 0) x[i] = x[i] + x[(i + 1) % CH] + 0x1234567u;                     // IADD3
        if (OP == 1) x[i] = x[i] ^ (x[(i + 1) % CH] & x[(i + 2) % CH]);               // LOP3
        if (OP == 2) x[i] = __funnelshift_r(x[i], x[i], 7) ^ 0;                        // SHF
        if (OP == 3) x[i] = x[i] * one + x[(i + 1) % CH];                              // IMAD (cbank)
        if (OP == 4) x[i] = __umulhi(x[i], m) + x[(i + 1) % CH] * one;                 // IMAD.HI + IMAD
        if (OP == 5) { uint64_t w = (uint64_t)x[i] * m; x[i] = (uint32_t)w ^ (uint32_t)(w >> 32); }  // IMAD.WIDE + LOP
        if (OP == 6) x[i] = __byte_perm(x[i], x[(i + 1) % CH], 0x5432);                 // PRMT
        if (OP == 7) { x[i] = x[i] * one + x[(i + 1) % CH]; x[i] = __funnelshift_r(x[i], x[i], 7); }  // IMAD+SHF 1:1
        if (OP == 8) { x[i] = x[i] + x[(i + 1) % CH] + 3u; x[i] = __funnelshift_r(x[i], x[i], 7); }   // IADD3+SHF
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < CH; i++) acc ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int OP>
void run(const char* name, int ops_per_unit) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* clk;
  cudaMalloc(&out, sizeof(uint32_t) * sms * 8 * 1024);
  cudaMalloc(&clk, sizeof(long long));
  const int iters = 2000, threads = 1024, blocks = sms;
  probe<OP><<<blocks, threads>>>(out, 10, clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<OP><<<blocks, threads>>>(out, iters, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  long long c;
  cudaMemcpy(&c, clk, sizeof c, cudaMemcpyDeviceToHost);
  double warp_inst = (double)iters * 16 * CH * ops_per_unit * (threads / 32);
  printf("%-26s %6.3f warp-inst/clk/SM  (%.2f lanes/clk/SM)\n", name, warp_inst / c, 32 * warp_inst / c);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  run<0>("IADD3", 1);
  run<1>("LOP3", 1);
  run<2>("SHF.R.W", 1);
  run<3>("IMAD (cbank one)", 1);
  run<4>("IMAD.HI + IMAD", 2);
  run<5>("IMAD.WIDE + LOP3", 2);
  run<6>("PRMT", 1);
  run<7>("IMAD + SHF (1:1)", 2);
  run<8>("IADD3 + SHF (1:1)", 2);
  return 0;
}
