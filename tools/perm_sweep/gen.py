"""Operand-order sweep of the chain step: sha256.cuh Mx<B> with the adds and
Sigma rotations re-associated / re-ordered (16 orders, bits of P below), for a
few masks B and node widths 4/6/8.  Same arithmetic, different instruction
order for ptxas (register assignment and bank conflicts change with it).
    P bit0: T1 = IMAD(IMAD(hk, S1), IMAD(w, Ch)) instead of IMAD(IMAD(w, hk), IMAD(S1, Ch))
    P bit1: a' = IMAD(IMAD(T1, S0), Maj) instead of IMAD(T1, IMAD(S0, Maj))
    P bit2: W  = IMAD(IMAD(IMAD(s1, w16), w7), s0) instead of IMAD(IMAD(s1, w7), IMAD(s0, w16))
    P bit3: Sigma rotations in reverse order
"""
import sys
from pathlib import Path
D = Path(__file__).parent
MASKS = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "248,232,184,104,216").split(",")]
NPART = 8
HDR = r'''
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_23969_b200/csrc/sha256.cuh"
using namespace hs;
template <int B, int P>
struct MxP : Mx<B> {
  static __device__ __forceinline__ uint32_t S0(uint32_t a) {
    if (P & 8) return rotr(a, 22) ^ rotr(a, 13) ^ ((B & 2) ? fma_rotr(a, 2) : rotr(a, 2));
    return Mx<B>::S0(a);
  }
  static __device__ __forceinline__ uint32_t S1(uint32_t e) {
    if (P & 8) return rotr(e, 25) ^ rotr(e, 11) ^ ((B & 1) ? fma_rotr(e, 6) : rotr(e, 6));
    return Mx<B>::S1(e);
  }
  static __device__ __forceinline__ uint32_t t1(uint32_t h, uint32_t k, uint32_t w, uint32_t s1v, uint32_t chv) {
    if ((P & 1) && Mx<B>::T1F == 3) return fma_add(fma_add(fma_addk(h, k), s1v), fma_add(w, chv));
    return Mx<B>::t1(h, k, w, s1v, chv);
  }
  static __device__ __forceinline__ uint32_t anew(uint32_t t, uint32_t s0v, uint32_t mj) {
    if ((P & 2) && (B & 32)) return fma_add(fma_add(t, s0v), mj);
    return Mx<B>::anew(t, s0v, mj);
  }
  static __device__ __forceinline__ uint32_t wnew(uint32_t s1v, uint32_t w7, uint32_t s0v, uint32_t w16) {
    if ((P & 4) && (B & 64)) return fma_add(fma_add(fma_add(s1v, w16), w7), s0v);
    return Mx<B>::wnew(s1v, w7, s0v, w16);
  }
};
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
typedef void (*launch_fn)(uint32_t*, int, int);
template <class V, int NW>
void launch(uint32_t* out, int reps, int blocks) { chain_kernel<V, NW><<<blocks, 128>>>(out, reps); }
'''
combos = [(b, p) for b in MASKS for p in range(16)]
for k in range(NPART):
    part = combos[k::NPART]
    s = HDR + f"void part_{k}(launch_fn* tab) {{\n"
    for b, p in part:
        i = combos.index((b, p))
        for j, nw in enumerate((4, 6, 8)):
            s += f"  tab[{i * 3 + j}] = launch<MxP<{b}, {p}>, {nw}>;\n"
    s += "}\n"
    (D / f"part_{k}.cu").write_text(s)
names = ",".join(f'"{b}/{p}"' for b, p in combos)
main = r'''
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
typedef void (*launch_fn)(uint32_t*, int, int);
''' + "".join(f"void part_{k}(launch_fn*);\n" for k in range(NPART)) + r'''
static const char* NAMES[] = {''' + names + r'''};
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int N = ''' + str(len(combos)) + r''';
  static launch_fn tab[''' + str(3 * len(combos)) + r'''];
''' + "".join(f"  part_{k}(tab);\n" for k in range(NPART)) + r'''
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 64, reps = 8;
  const size_t threads = (size_t)blocks * 128;
  uint32_t* out; cudaMalloc(&out, threads * 8 * 4);
  uint32_t* ref[3] = {0, 0, 0}; uint32_t* h = (uint32_t*)malloc(threads * 8 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int NWs[3] = {4, 6, 8};
  for (int v = 0; v < N; v++) for (int j = 0; j < 3; j++) {
    launch_fn f = tab[v * 3 + j];
    f(out, 1, blocks);
    cudaMemcpy(h, out, threads * NWs[j] * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    if (!ref[j]) { ref[j] = (uint32_t*)malloc(threads * NWs[j] * 4); memcpy(ref[j], h, threads * NWs[j] * 4); }
    else bad = memcmp(h, ref[j], threads * NWs[j] * 4) != 0;
    float best = 1e30f;
    for (int t = 0; t < 3; t++) {
      cudaEventRecord(a); f(out, reps, blocks); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("BP=%s NW=%d %.3f Gstep/s%s\n", NAMES[v], NWs[j], (double)threads * reps * 15 / best / 1e6, bad ? " MISMATCH" : "");
  }
  return 0;
}
'''
(D / "main.cu").write_text(main)
(D / "Makefile").write_text(
    "NV = nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a\n"
    f"OBJS = main.o {' '.join(f'part_{k}.o' for k in range(NPART))}\n"
    "sweep: $(OBJS)\n\t$(NV) -o $@ $(OBJS)\n"
    "%.o: %.cu ../../paper_2512_23969_b200/csrc/sha256.cuh\n\t$(NV) -c $< -o $@\n")
