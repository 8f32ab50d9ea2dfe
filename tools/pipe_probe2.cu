// pipe_probe2.cu -- second integer pipe microbenchmark for sm_100a: the forms
// the first probe (pipe_probe.cu) did not cover -- VIADD, IMAD with an
// immediate or a third register, mad.hi with addend, and ALU:FMA mixes in the
// ratios the SHA-256 paths produce.  8 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__constant__ uint32_t c_one = 1u, c_m = 0x20000000u;
__device__ uint32_t g_r[2] = {3u, 0x20000000u};

__device__ __forceinline__ uint32_t madhi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

#define CH 8
template <int OP>
__global__ void probe(uint32_t* out, int iters, long long* clk) {
  uint32_t x[CH];
  for (int i = 0; i < CH; i++) x[i] = threadIdx.x * 7 + i;
  uint32_t one = c_one, m = c_m, r = g_r[0], mr = g_r[1];
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int i = 0; i < CH; i++) {
        const uint32_t y = x[(i + 1) % CH], z = x[(i + 2) % CH];
        if (OP == 0) x[i] = __funnelshift_r(x[i] + 0x1234567u, x[i] + 0x1234567u, 7);  // VIADD + SHF 1:1
        if (OP == 1) x[i] = x[i] * 0x9E3779B1u + y;                               // IMAD imm
        if (OP == 2) x[i] = x[i] * r + y;                                         // IMAD 3-reg
        if (OP == 3) x[i] = madhi(x[i], m, y);                                    // IMAD.HI (+addend)
        if (OP == 4) { x[i] = x[i] ^ (y & z); x[i] = x[i] * one + y; }             // LOP3 + IMAD
        if (OP == 5) { x[i] = __funnelshift_r(x[i], x[i], 7) ^ y; x[i] = x[i] * one + z; }  // SHF LOP3 IMAD (2:1)
        if (OP == 6) { x[i] = __funnelshift_r(x[i], x[i], 7); x[i] = madhi(x[i], m, y); }   // SHF + IMAD.HI
        if (OP == 7) { x[i] = __funnelshift_r(x[i], x[i], 7) ^ y; x[i] = __umulhi(x[i], m) + z; }  // SHF LOP3 + IMAD.HI
        if (OP == 8) x[i] = x[i] + y + z;                                          // IADD3 3-reg
        if (OP == 9) x[i] = madhi(x[i], mr, y);                                    // IMAD.HI reg mult
        if (OP == 10) x[i] = one * 0x9E3779B1u + x[i];                             // IMAD Rone, imm, Rx
        if (OP == 11) { x[i] = x[i] ^ (y & z); x[i] = x[i] * 0x9E3779B1u + y; }      // LOP3 + IMAD imm
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
  printf("%-30s %6.3f warp-inst/clk/SM  (%.2f lanes/clk/SM)\n", name, warp_inst / c, 32 * warp_inst / c);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  run<0>("VIADD + SHF 1:1", 2);
  run<1>("IMAD x*imm+y", 1);
  run<2>("IMAD x*r+y (3 reg)", 1);
  run<3>("IMAD.HI x*c+y", 1);
  run<4>("LOP3 + IMAD(cbank) 1:1", 2);
  run<5>("SHF LOP3 + IMAD 2:1", 3);
  run<6>("SHF + IMAD.HI 1:1", 2);
  run<7>("SHF LOP3 + IMAD.HI 2:1", 3);
  run<8>("IADD3 3-reg", 1);
  run<9>("IMAD.HI x*r+y (reg mult)", 1);
  run<10>("IMAD one*imm+x", 1);
  run<11>("LOP3 + IMAD imm 1:1", 2);
  return 0;
}
