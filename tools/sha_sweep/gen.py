"""SHA-256 path sweep (sha256.cuh Mx<B>, every mask B in 0..255).  Generates the sweep sources: part_<k>.cu instantiate Mx<B> chain kernels for
B in their slice and NW in {4, 6, 8}; main.cu times every (B, NW) and checks
it against Native (B = -1)."""
import sys
from pathlib import Path
D = Path(__file__).parent
NPART = int(sys.argv[1]) if len(sys.argv) > 1 else 16
NB = 256
KERNEL = r'''
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_23969_b200/csrc/sha256.cuh"
using namespace hs;
template <class V, int NW>
__global__ void __launch_bounds__(128) chain_kernel(uint32_t* out, int reps) {
  uint32_t mid[8];
  for (int i = 0; i < 8; i++) mid[i] = 0x6a09e667u * (i + 1);
  uint32_t x[NW];
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int j = 0; j < NW; j++) x[j] = tid * 2654435761u + 17u * j;
  for (int r = 0; r < reps; r++) {
    Adrs a = make_adrs(3, tid + r, 0u, 1, r & 63, 0);
    chain_F<V, NW>(x, mid, a, 0u, 15u);
  }
  for (int j = 0; j < NW; j++) out[(size_t)tid * NW + j] = x[j];
}
typedef void (*launch_fn)(uint32_t*, int, int, int);
template <class V, int NW>
void launch(uint32_t* out, int reps, int blocks, int regs_query) {
  if (regs_query) { cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, chain_kernel<V, NW>); *(int*)out = fa.numRegs; return; }
  chain_kernel<V, NW><<<blocks, 128>>>(out, reps);
}
'''
for k in range(NPART):
    lo, hi = k * NB // NPART, (k + 1) * NB // NPART
    s = KERNEL + f"void part_{k}(launch_fn* tab) {{\n"
    for b in range(lo, hi):
        for j, nw in enumerate((4, 6, 8)):
            s += f"  tab[{b * 3 + j}] = launch<Mx<{b}>, {nw}>;\n"
    if k == 0:
        for j, nw in enumerate((4, 6, 8)):
            s += f"  tab[{NB * 3 + j}] = launch<Native, {nw}>;\n"
    s += "}\n"
    (D / f"part_{k}.cu").write_text(s)
main = r'''
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
typedef void (*launch_fn)(uint32_t*, int, int, int);
''' + "".join(f"void part_{k}(launch_fn*);\n" for k in range(NPART)) + r'''
int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  static launch_fn tab[%d * 3 + 3];
''' % NB + "".join(f"  part_{k}(tab);\n" for k in range(NPART)) + r'''
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 64, reps = 8;
  const size_t threads = (size_t)blocks * 128;
  uint32_t* out; cudaMalloc(&out, threads * 8 * 4);
  uint32_t* ref[3]; uint32_t* h = (uint32_t*)malloc(threads * 8 * 4);
  int* regbuf; cudaMallocManaged(&regbuf, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int NWs[3] = {4, 6, 8};
  for (int j = 0; j < 3; j++) {
    tab[%d * 3 + j](out, 1, blocks, 0);
    ref[j] = (uint32_t*)malloc(threads * NWs[j] * 4);
    cudaMemcpy(ref[j], out, threads * NWs[j] * 4, cudaMemcpyDeviceToHost);
  }
  for (int v = -1; v < %d; v++) {
    for (int j = 0; j < 3; j++) {
      launch_fn f = tab[(v < 0 ? %d : v) * 3 + j];
      f(out, 1, blocks, 0);
      cudaMemcpy(h, out, threads * NWs[j] * 4, cudaMemcpyDeviceToHost);
      int bad = memcmp(h, ref[j], threads * NWs[j] * 4) != 0;
      float best = 1e30f;
      for (int t = 0; t < 3; t++) {
        cudaEventRecord(a); f(out, reps, blocks, 0); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      f((uint32_t*)regbuf, 0, 0, 1); cudaDeviceSynchronize();
      printf("B=%%d NW=%%d regs=%%d %%.3f Gstep/s%%s\n", v, NWs[j], *regbuf, (double)threads * reps * 15 / best / 1e6, bad ? " MISMATCH" : "");
    }
  }
  return 0;
}
''' % (NB, NB, NB)
(D / "main.cu").write_text(main)
(D / "Makefile").write_text(
    "NV = nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a\n"
    f"OBJS = main.o {' '.join(f'part_{k}.o' for k in range(NPART))}\n"
    "sweep: $(OBJS)\n\t$(NV) -o $@ $(OBJS)\n"
    "%.o: %.cu ../../paper_2512_23969_b200/csrc/sha256.cuh\n\t$(NV) -c $< -o $@\n"
    "clean:\n\trm -f *.o sweep\n")
