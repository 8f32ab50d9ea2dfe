// sha256.cuh -- register-resident SHA-256 device library for sm_100a.
//
// Replaces the reference's two bit-identical compression backends
// (backends.py:51-123, selected per (kernel,set) by BackendSelection
// backends.py:201-257) with compile-time arithmetic paths:
//
//   Native : plain C; ptxas picks IADD3/LOP3/SHF (ALU pipe) for almost all.
//   Fast   : Mix<0,0,0,SHR,1,ANF,-> -- the schedule shifts as IMAD.HI (inline
//            PTX mad.hi) and the 3-input adds of T1 and `a` as IMAD chains with
//            an opaque constant-bank multiplier, moving work from the
//            saturated ALU pipe to the idle FMA pipe (the sm_100a analog of
//            the paper's `mad.lo.u32` PTX path).  Chosen by
//            tools/sha_probe.cu on B200: 17.2 vs 15.5 G chain-steps/s.
//   Imad / other Mix<...>: kept for the probe.
//
// Tweakable hashes follow hashes.py:124-150: thash = SHA-256(PKseed-midstate,
// ADRS(22B) || M)[:n]; PRF = SHA-256(SKseed || ADRS)[:n] from the IV.  Nodes
// are kept as big-endian 32-bit words (exactly the digest's state words), so
// no byte swapping happens inside the hypertree; the 22-byte ADRS puts every
// node at a 2-byte offset, handled with one PRMT/funnel-shift per word.
#pragma once
#include <cstdint>

#include "hs_variants.h"

namespace hs {

static __constant__ uint32_t c_one = 1u;  // opaque multiplicative identity (Imad path)

__device__ __forceinline__ constexpr uint32_t Kc(int i) {
  constexpr uint32_t K[64] = {
      0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
      0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
      0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
      0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
      0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
      0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
      0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
      0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2,
  };
  return K[i];
}

__device__ __forceinline__ constexpr uint32_t IVc(int i) {
  constexpr uint32_t IV[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                              0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  return IV[i];
}

// ---------------------------------------------------------------------------
// arithmetic paths
//
// SHA-256 on sm_100a is bound by the ALU pipe (SHF/LOP3/IADD3/PRMT; 16
// lanes/clk/SMSP) while the FMA pipe (IMAD family, also 16 lanes/clk/SMSP)
// idles.  A path decides, per operation site, which pipe does the work:
//   fma_add(a,b)   a*one+b            IMAD      (one from the constant bank)
//   fma_shr(x,r)   hi(x * 2^(32-r))   IMAD.HI
//   fma_rotr(x,r)  hi(x*m) + lo(x*m), m = 2^(32-r)   IMAD + IMAD.HI
// Multipliers live in constant memory so ptxas cannot fold them back into
// shifts.  Native leaves every choice to ptxas; Imad moves all adds; Mix<>
// moves a chosen subset of rotates / shifts / two-input adds.
// ---------------------------------------------------------------------------
static __constant__ uint32_t c_pow2[33] = {
    1u << 0,  1u << 1,  1u << 2,  1u << 3,  1u << 4,  1u << 5,  1u << 6,  1u << 7,  1u << 8,
    1u << 9,  1u << 10, 1u << 11, 1u << 12, 1u << 13, 1u << 14, 1u << 15, 1u << 16, 1u << 17,
    1u << 18, 1u << 19, 1u << 20, 1u << 21, 1u << 22, 1u << 23, 1u << 24, 1u << 25, 1u << 26,
    1u << 27, 1u << 28, 1u << 29, 1u << 30, 1u << 31, 0u};

// Rotations as plain shifts: LLVM turns them into a funnel-shift intrinsic
// (SHF.R.W, one ALU instruction, the same as __funnelshift_r) that it can
// constant-fold and hoist out of loops.  __funnelshift_r is inline PTX, which
// NVVM treats as opaque: in the WOTS chain loop the rotations of the
// chain-invariant schedule words (ADRS words, constant padding) were then
// recomputed at every step.  HS_ROTR_ASM=1 restores the inline-PTX form.
#ifndef HS_ROTR_ASM
#define HS_ROTR_ASM 0
#endif
__device__ __forceinline__ uint32_t rotr(uint32_t x, int r) {
#if HS_ROTR_ASM
  return __funnelshift_r(x, x, r);
#else
  return (x >> r) | (x << ((32 - r) & 31));
#endif
}
__device__ __forceinline__ uint32_t fma_add(uint32_t a, uint32_t b) { return a * c_one + b; }
__device__ __forceinline__ uint32_t fma_shr(uint32_t x, int r) { return __umulhi(x, c_pow2[32 - r]); }
__device__ __forceinline__ uint32_t fma_rotr(uint32_t x, int r) {
  const uint32_t m = c_pow2[32 - r];
  const uint32_t lo = x * m;
  uint32_t out;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(out) : "r"(x), "r"(m), "r"(lo));
  return out;
}
// x + K for a compile-time K: one * K + x with `one` opaque, so ptxas keeps
// it on the FMA pipe as IMAD Rd, Rone, K, Rx.
__device__ __forceinline__ uint32_t fma_addk(uint32_t x, uint32_t k) { return c_one * k + x; }
__device__ __forceinline__ uint32_t ch(uint32_t e, uint32_t f, uint32_t g) { return g ^ (e & (f ^ g)); }
__device__ __forceinline__ uint32_t maj(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

// rotation helper: the first NF rotations of a sigma run on the FMA pipe
template <int NF, int IDX>
__device__ __forceinline__ uint32_t rot_sel(uint32_t x, int r) { return IDX < NF ? fma_rotr(x, r) : rotr(x, r); }

struct Native {
  static constexpr int id = 0;
  static __device__ __forceinline__ uint32_t S0(uint32_t a) { return rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22); }
  static __device__ __forceinline__ uint32_t S1(uint32_t e) { return rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25); }
  static __device__ __forceinline__ uint32_t s0(uint32_t x) { return rotr(x, 7) ^ rotr(x, 18) ^ (x >> 3); }
  static __device__ __forceinline__ uint32_t s1(uint32_t x) { return rotr(x, 17) ^ rotr(x, 19) ^ (x >> 10); }
  static __device__ __forceinline__ uint32_t t1(uint32_t h, uint32_t k, uint32_t w, uint32_t s1v, uint32_t chv) {
    return h + k + w + s1v + chv;
  }
  static __device__ __forceinline__ uint32_t enew(uint32_t d, uint32_t t) { return d + t; }
  static __device__ __forceinline__ uint32_t anew(uint32_t t, uint32_t s0v, uint32_t mj) { return t + s0v + mj; }
  static __device__ __forceinline__ uint32_t wnew(uint32_t s1v, uint32_t w7, uint32_t s0v, uint32_t w16) {
    return s1v + w7 + s0v + w16;
  }
  static __device__ __forceinline__ uint32_t ff(uint32_t x, uint32_t y) { return x + y; }
};

struct Imad : Native {
  static constexpr int id = 1;
  static __device__ __forceinline__ uint32_t t1(uint32_t h, uint32_t k, uint32_t w, uint32_t s1v, uint32_t chv) {
    return fma_add(fma_add(fma_add(h, k), w), fma_add(s1v, chv));
  }
  static __device__ __forceinline__ uint32_t enew(uint32_t d, uint32_t t) { return fma_add(d, t); }
  static __device__ __forceinline__ uint32_t anew(uint32_t t, uint32_t s0v, uint32_t mj) {
    return fma_add(t, fma_add(s0v, mj));
  }
  static __device__ __forceinline__ uint32_t wnew(uint32_t s1v, uint32_t w7, uint32_t s0v, uint32_t w16) {
    return fma_add(fma_add(s1v, w7), fma_add(s0v, w16));
  }
  static __device__ __forceinline__ uint32_t ff(uint32_t x, uint32_t y) { return fma_add(x, y); }
};

// Mix<NS1, NS0, NSS, SHR, T1F, ANF, WF>: NS1/NS0 rotations of Sigma1/Sigma0
// and NSS of each schedule sigma on the FMA pipe (IMAD + IMAD.HI); SHR: the
// schedule's plain shifts via IMAD.HI; T1F (0..2) of the two 3-input adds of
// T1, ANF the 3-input add of the new `a`, WF the schedule sum split into
// IMADs.  Two-input adds (e = d + T1, feed-forward) always use IMAD.
// Measured on B200 (tools/sha_probe.cu): IMAD issues at the ALU rate on the
// FMA pipe, IMAD.HI at half rate; ALU and FMA pipes dual-issue.
template <int NS1, int NS0, int NSS, bool SHR, int T1F, bool ANF, bool WF>
struct Mix : Native {
  static constexpr int id = 2;
  static __device__ __forceinline__ uint32_t S0(uint32_t a) {
    return rot_sel<NS0, 0>(a, 2) ^ rot_sel<NS0, 1>(a, 13) ^ rot_sel<NS0, 2>(a, 22);
  }
  static __device__ __forceinline__ uint32_t S1(uint32_t e) {
    return rot_sel<NS1, 0>(e, 6) ^ rot_sel<NS1, 1>(e, 11) ^ rot_sel<NS1, 2>(e, 25);
  }
  static __device__ __forceinline__ uint32_t s0(uint32_t x) {
    return rot_sel<NSS, 0>(x, 7) ^ rot_sel<NSS, 1>(x, 18) ^ (SHR ? fma_shr(x, 3) : (x >> 3));
  }
  static __device__ __forceinline__ uint32_t s1(uint32_t x) {
    return rot_sel<NSS, 0>(x, 17) ^ rot_sel<NSS, 1>(x, 19) ^ (SHR ? fma_shr(x, 10) : (x >> 10));
  }
  static __device__ __forceinline__ uint32_t t1(uint32_t h, uint32_t k, uint32_t w, uint32_t s1v, uint32_t chv) {
    if (T1F == 0) return h + k + w + s1v + chv;
    if (T1F == 1) return fma_add(h + k + w, fma_add(s1v, chv));
    if (T1F == 2) return fma_add(fma_add(fma_add(w, h), k), fma_add(s1v, chv));
    return fma_add(fma_add(w, fma_addk(h, k)), fma_add(s1v, chv));
  }
  static __device__ __forceinline__ uint32_t enew(uint32_t d, uint32_t t) { return fma_add(d, t); }
  static __device__ __forceinline__ uint32_t anew(uint32_t t, uint32_t s0v, uint32_t mj) {
    return ANF ? fma_add(t, fma_add(s0v, mj)) : t + s0v + mj;
  }
  static __device__ __forceinline__ uint32_t wnew(uint32_t s1v, uint32_t w7, uint32_t s0v, uint32_t w16) {
    return WF ? fma_add(fma_add(s1v, w7), fma_add(s0v, w16)) : fma_add(s1v + w7 + s0v, w16);
  }
  static __device__ __forceinline__ uint32_t ff(uint32_t x, uint32_t y) { return fma_add(x, y); }
};

using Fast = Mix<0, 0, 0, true, 1, true, false>;

// Mx<B>: the arithmetic path as a bitmask, the family swept on B200 by
// tools/sha_sweep (all 256 masks x node widths 4/6/8, profiles/r01_sha_sweep.txt):
//   bit0  Sigma1's first rotation on the FMA pipe (IMAD + IMAD.HI)
//   bit1  Sigma0's first rotation on the FMA pipe
//   bit2  schedule plain shifts as IMAD.HI
//   bit3-4 T1: 0 native sum, 1 IMAD(h+k+w, IMAD(S1,Ch)), 2 all IMAD, 3 IMAD with
//         the round constant folded into an IMAD immediate
//   bit5  new a as an IMAD chain       bit6  schedule sum as three IMADs
//   bit7  new e = d + T1 as an IMAD
// SHA-256 on sm_100a is co-limited by the ALU pipe (2 cycles per warp
// instruction per SMSP) and by register-file bank reads (profiles/
// r01_pipe_probe2.txt: a 3-register LOP3 + 2-register IMAD pair issues at 0.8
// instead of 1 per cycle); which split wins depends on ptxas's register
// assignment for the surrounding kernel, so the engine compiles a few masks
// and the on-device tuner times them per (kernel, set).
// P (operand order, tools/perm_sweep): bit0 T1 = IMAD(IMAD(hk, S1), IMAD(w, Ch))
// (with T1 form 3), bit1 a' = IMAD(IMAD(T1, S0), Maj), bit2 W = IMAD(IMAD(IMAD(
// s1, w16), w7), s0) (with bit6), bit3 Sigma rotations in reverse order.  Same
// arithmetic; ptxas's schedule and register assignment change with the order.
template <int B, int P = 0>
struct Mx : Native {
  static constexpr int id = 100 + B + 256 * P;
  static constexpr int T1F = (B >> 3) & 3;
  static __device__ __forceinline__ uint32_t S0(uint32_t a) {
    const uint32_t r2 = (B & 2) ? fma_rotr(a, 2) : rotr(a, 2);
    if (P & 8) return rotr(a, 22) ^ rotr(a, 13) ^ r2;
    return r2 ^ rotr(a, 13) ^ rotr(a, 22);
  }
  static __device__ __forceinline__ uint32_t S1(uint32_t e) {
    const uint32_t r6 = (B & 1) ? fma_rotr(e, 6) : rotr(e, 6);
    if (P & 8) return rotr(e, 25) ^ rotr(e, 11) ^ r6;
    return r6 ^ rotr(e, 11) ^ rotr(e, 25);
  }
  static __device__ __forceinline__ uint32_t s0(uint32_t x) {
    return rotr(x, 7) ^ rotr(x, 18) ^ ((B & 4) ? fma_shr(x, 3) : (x >> 3));
  }
  static __device__ __forceinline__ uint32_t s1(uint32_t x) {
    return rotr(x, 17) ^ rotr(x, 19) ^ ((B & 4) ? fma_shr(x, 10) : (x >> 10));
  }
  static __device__ __forceinline__ uint32_t t1(uint32_t h, uint32_t k, uint32_t w, uint32_t s1v, uint32_t chv) {
    if (T1F == 0) return h + k + w + s1v + chv;
    if (T1F == 1) return fma_add(h + k + w, fma_add(s1v, chv));
    if (T1F == 2) return fma_add(fma_add(fma_add(w, h), k), fma_add(s1v, chv));
    if (P & 1) return fma_add(fma_add(fma_addk(h, k), s1v), fma_add(w, chv));
    return fma_add(fma_add(w, fma_addk(h, k)), fma_add(s1v, chv));
  }
  static __device__ __forceinline__ uint32_t enew(uint32_t d, uint32_t t) { return (B & 128) ? fma_add(d, t) : d + t; }
  static __device__ __forceinline__ uint32_t anew(uint32_t t, uint32_t s0v, uint32_t mj) {
    if (!(B & 32)) return t + s0v + mj;
    return (P & 2) ? fma_add(fma_add(t, s0v), mj) : fma_add(t, fma_add(s0v, mj));
  }
  static __device__ __forceinline__ uint32_t wnew(uint32_t s1v, uint32_t w7, uint32_t s0v, uint32_t w16) {
    if (!(B & 64)) return fma_add(s1v + w7 + s0v, w16);
    return (P & 4) ? fma_add(fma_add(fma_add(s1v, w16), w7), s0v) : fma_add(fma_add(s1v, w7), fma_add(s0v, w16));
  }
  static __device__ __forceinline__ uint32_t ff(uint32_t x, uint32_t y) { return x + y; }
};

// Engine variant ids (hs_set_config.variant): 0 Native, 1 Fast, then one Mx
// per code of HS_MX_MASKS (hs_variants.h; set at build time); code = mask B +
// 256 * operand order P.
constexpr int kMxMasks[] = {HS_MX_MASKS};
constexpr int kNumVariants = 2 + (int)(sizeof(kMxMasks) / sizeof(kMxMasks[0]));
template <int ID> struct VariantOf { using T = Mx<(kMxMasks[ID - 2] & 255), (kMxMasks[ID - 2] >> 8)>; };
template <> struct VariantOf<0> { using T = Native; };
template <> struct VariantOf<1> { using T = Fast; };

// Rounds [R0, R1) of SHA-256 on working state s, expanding the schedule in
// place for rounds >= 16.  Fully unrolled so constant message words
// (padding, lengths, zeros, chain-invariant ADRS words) fold.
template <class V, int R0, int R1>
__device__ __forceinline__ void sha_rounds(uint32_t s[8], uint32_t* W) {
  const V v{};  // paths may carry per-call state (e.g. an opaque register)
  uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
  for (int i = R0; i < R1; i++) {
    if (i >= 16) {
      W[i & 15] = v.wnew(v.s1(W[(i - 2) & 15]), W[(i - 7) & 15], v.s0(W[(i - 15) & 15]), W[i & 15]);
    }
    const uint32_t t = v.t1(h, Kc(i), W[i & 15], v.S1(e), ch(e, f, g));
    const uint32_t an = v.anew(t, v.S0(a), maj(a, b, c));
    h = g; g = f; f = e; e = v.enew(d, t);
    d = c; c = b; b = a; a = an;
  }
  s[0] = a; s[1] = b; s[2] = c; s[3] = d; s[4] = e; s[5] = f; s[6] = g; s[7] = h;
}

// One SHA-256 compression; W is consumed (used as the rolling schedule).
template <class V>
__device__ __forceinline__ void compress(uint32_t st[8], uint32_t W[16]) {
  uint32_t s[8];
#pragma unroll
  for (int i = 0; i < 8; i++) s[i] = st[i];
  sha_rounds<V, 0, 64>(s, W);
  const V v{};
#pragma unroll
  for (int i = 0; i < 8; i++) st[i] = v.ff(st[i], s[i]);
}

// Compact compression for latency-bound single-thread code (message
// preparation, verification prologue): the 64 rounds as a 4-trip loop over a
// 16-round unrolled body with K from constant memory, so the code is ~4x
// smaller than the fully unrolled compress (whose instruction fetch, not its
// arithmetic, dominates a lone warp's hash chain).  Same result as compress.
static __constant__ uint32_t c_K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2,
};
template <class V>
__device__ __noinline__ void compress_compact(uint32_t st[8], const uint32_t Win[16]) {
  uint32_t W[16];
#pragma unroll
  for (int j = 0; j < 16; j++) W[j] = Win[j];
  const V v{};
  uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll 1
  for (int r = 0; r < 64; r += 16) {
#pragma unroll
    for (int j = 0; j < 16; j++) {
      if (r > 0) W[j] = v.wnew(v.s1(W[(j + 14) & 15]), W[(j + 9) & 15], v.s0(W[(j + 1) & 15]), W[j]);
      const uint32_t t = v.t1(h, c_K[r + j], W[j], v.S1(e), ch(e, f, g));
      const uint32_t an = v.anew(t, v.S0(a), maj(a, b, c));
      h = g; g = f; f = e; e = v.enew(d, t);
      d = c; c = b; b = a; a = an;
    }
  }
  st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
}

// The same compression fully unrolled but out of line: one copy of the code
// for every call site of a latency-bound single-thread hash chain.  A lone
// warp runs it in ~3000 cycles against ~4400 for compress_compact, whose
// round loop and constant-memory K reads sit on the critical path
// (tools/lat_probe.cu, profiles/r02t_lat_probe.txt).
// State and block travel by value (registers under the device ABI), so the
// call does not stage them through local memory.
struct ShaState {
  uint32_t w[8];
};
struct ShaBlock {
  uint32_t w[16];
};
template <class V>
__device__ __noinline__ ShaState compress_ool_v(ShaState st, ShaBlock W) {
  compress<V>(st.w, W.w);
  return st;
}
template <class V>
__device__ __forceinline__ void compress_ool(uint32_t st[8], const uint32_t Win[16]) {
  ShaState s;
  ShaBlock b;
#pragma unroll
  for (int j = 0; j < 8; j++) s.w[j] = st[j];
#pragma unroll
  for (int j = 0; j < 16; j++) b.w[j] = Win[j];
  s = compress_ool_v<V>(s, b);
#pragma unroll
  for (int j = 0; j < 8; j++) st[j] = s.w[j];
}
// message preparation / verify prologue compression: HS_PREP_UNROLLED=0
// restores the compact form
#ifndef HS_PREP_UNROLLED
#define HS_PREP_UNROLLED 1
#endif
template <class V>
__device__ __forceinline__ void compress_prep(uint32_t st[8], const uint32_t W[16]) {
#if HS_PREP_UNROLLED
  compress_ool<V>(st, W);
#else
  compress_compact<V>(st, W);
#endif
}
// the many-thread verify prologue keeps the compact loop (its warps share the
// SM, the short loop body stays in the instruction cache: 0.5-2 % faster
// verification than the unrolled form, profiles/r02ae_verify_ab.txt)
template <class V, bool Prep>
__device__ __forceinline__ void compress_sel(uint32_t st[8], const uint32_t W[16]) {
  if (Prep) compress_prep<V>(st, W);
  else compress_compact<V>(st, W);
}

// Rounds [0, R) only (no schedule expansion needed while R <= 16).
template <class V, int R>
__device__ __forceinline__ void rounds_prefix(uint32_t s[8], const uint32_t* W) {
  static_assert(R <= 16, "prefix rounds read W directly");
  uint32_t Wc[16];
#pragma unroll
  for (int i = 0; i < R; i++) Wc[i] = W[i];
  sha_rounds<V, 0, R>(s, Wc);
}

// Compression resumed after R0 rounds: `sR` is the working state after rounds
// [0, R0) (computed once by rounds_prefix while W[0..R0) stay fixed), `st`
// the chaining value for the feed-forward.  W must still hold all 16 words.
template <class V, int R0>
__device__ __forceinline__ void compress_resume(uint32_t st[8], const uint32_t sR[8], uint32_t W[16]) {
  uint32_t s[8];
#pragma unroll
  for (int i = 0; i < 8; i++) s[i] = sR[i];
  sha_rounds<V, R0, 64>(s, W);
  const V v{};
#pragma unroll
  for (int i = 0; i < 8; i++) st[i] = v.ff(st[i], s[i]);
}

// ---------------------------------------------------------------------------
// addresses (address.py:3-10): 22 bytes big-endian packed into 5.5 words
// ---------------------------------------------------------------------------
struct Adrs {
  uint32_t w0, w1, w2, w3, w4, h5;  // h5 = bytes 20..21 in the low 16 bits
};

__device__ __forceinline__ Adrs make_adrs(uint32_t layer, uint64_t tree, uint32_t type, uint32_t keypair,
                                          uint32_t chain, uint32_t hash) {
  Adrs a;
  a.w0 = (layer << 24) | ((uint32_t)(tree >> 40) & 0xFFFFFFu);
  a.w1 = (uint32_t)(tree >> 8);
  a.w2 = ((uint32_t)tree << 24) | (type << 16) | (keypair >> 16);
  a.w3 = (keypair << 16) | (chain >> 16);
  a.w4 = (chain << 16) | (hash >> 16);
  a.h5 = hash & 0xFFFFu;
  return a;
}
__device__ __forceinline__ void adrs_set_chain_hash(Adrs& a, uint32_t chain, uint32_t hash) {
  a.w3 = (a.w3 & 0xFFFF0000u) | (chain >> 16);
  a.w4 = (chain << 16) | (hash >> 16);
  a.h5 = hash & 0xFFFFu;
}

// (hi << 16) | (lo >> 16): joins two big-endian words across a 2-byte offset
__device__ __forceinline__ uint32_t join16(uint32_t hi, uint32_t lo) { return __byte_perm(lo, hi, 0x5432); }
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// ---------------------------------------------------------------------------
// tweakable hash with a register-resident message of MW words (F: MW = n/4,
// H: MW = n/2).  hashes.py:124-137.
// ---------------------------------------------------------------------------
template <class V, int MW>
__device__ __forceinline__ void thash_reg(uint32_t st[8], const uint32_t mid[8], const Adrs& a, const uint32_t* m) {
  constexpr int total = 22 + 4 * MW;                 // bytes after the midstate block
  constexpr int nblk = (total + 9 + 63) / 64;
  constexpr int SW = 16 * nblk;
  uint32_t s[SW];
  s[0] = a.w0; s[1] = a.w1; s[2] = a.w2; s[3] = a.w3; s[4] = a.w4;
  s[5] = join16(a.h5, m[0]);
#pragma unroll
  for (int j = 1; j < MW; j++) s[5 + j] = join16(m[j - 1], m[j]);
  s[5 + MW] = (m[MW - 1] << 16) | 0x8000u;
#pragma unroll
  for (int j = 6 + MW; j < SW - 1; j++) s[j] = 0;
  s[SW - 1] = (uint32_t)((64 + total) * 8);
#pragma unroll
  for (int i = 0; i < 8; i++) st[i] = mid[i];
#pragma unroll
  for (int blk = 0; blk < nblk; blk++) {
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 16; j++) W[j] = s[16 * blk + j];
    compress<V>(st, W);
  }
}

// thash_reg with the first block resumed after round 5: `pre5` is the state
// after rounds 0..4 from `mid` over ADRS words 0..4, computed once for every
// hash that shares them (e.g. one FORS level of one message).
template <class V, int MW>
__device__ __forceinline__ void thash_reg_pre(uint32_t st[8], const uint32_t mid[8], const uint32_t pre5[8],
                                              const Adrs& a, const uint32_t* m) {
  constexpr int total = 22 + 4 * MW;
  constexpr int nblk = (total + 9 + 63) / 64;
  constexpr int SW = 16 * nblk;
  uint32_t s[SW];
  s[0] = a.w0; s[1] = a.w1; s[2] = a.w2; s[3] = a.w3; s[4] = a.w4;
  s[5] = join16(a.h5, m[0]);
#pragma unroll
  for (int j = 1; j < MW; j++) s[5 + j] = join16(m[j - 1], m[j]);
  s[5 + MW] = (m[MW - 1] << 16) | 0x8000u;
#pragma unroll
  for (int j = 6 + MW; j < SW - 1; j++) s[j] = 0;
  s[SW - 1] = (uint32_t)((64 + total) * 8);
  uint32_t sR[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { st[i] = mid[i]; sR[i] = pre5[i]; }
#pragma unroll
  for (int blk = 0; blk < nblk; blk++) {
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 16; j++) W[j] = s[16 * blk + j];
    if (blk == 0) compress_resume<V, 5>(st, sR, W);
    else compress<V>(st, W);
  }
}

// WOTS+ chain (wots.py:42-60): `steps` applications of F starting at hash
// index `start`, x updated in place.  Along a chain only ADRS bytes 20..21
// (the hash index, < 2^16) and the node change, so message words W0..W4 are
// fixed and SHA-256 rounds 0-4 are computed once per chain, not per step.
// When `rec` is non-null, the node after step s is also stored at
// rec[(s + 1) * NW ...] (TREE_Sign keeps the signing leaf's chain so that
// WOTS_Sign becomes a gather).
template <class V, int NW>
__device__ __forceinline__ void chain_F(uint32_t* x, const uint32_t mid[8], const Adrs& a, uint32_t start,
                                        uint32_t steps, uint32_t* rec = nullptr) {
  constexpr int total = 22 + 4 * NW;
  static_assert(total + 9 <= 64, "F is a single block after the midstate");
  uint32_t pre[8];
  const uint32_t W04[5] = {a.w0, a.w1, a.w2, a.w3, a.w4};
#pragma unroll
  for (int i = 0; i < 8; i++) pre[i] = mid[i];
  rounds_prefix<V, 5>(pre, W04);
#pragma unroll 1
  for (uint32_t s = start; s < start + steps; s++) {
    uint32_t W[16];
    W[0] = a.w0; W[1] = a.w1; W[2] = a.w2; W[3] = a.w3; W[4] = a.w4;
    W[5] = join16(s, x[0]);
#pragma unroll
    for (int j = 1; j < NW; j++) W[5 + j] = join16(x[j - 1], x[j]);
    W[5 + NW] = (x[NW - 1] << 16) | 0x8000u;
#pragma unroll
    for (int j = 6 + NW; j < 15; j++) W[j] = 0;
    W[15] = (uint32_t)((64 + total) * 8);
    uint32_t st[8];
#pragma unroll
    for (int i = 0; i < 8; i++) st[i] = mid[i];
    compress_resume<V, 5>(st, pre, W);
#pragma unroll
    for (int j = 0; j < NW; j++) x[j] = st[j];
    if (rec) {
#pragma unroll
      for (int j = 0; j < NW; j++) rec[(s + 1) * NW + j] = x[j];
    }
  }
}

// Out-of-line form of chain_F for the leaf kernels.  Inlined into a large
// kernel, the chain loop's register assignment (and with it the register-bank
// conflicts that co-limit SHA-256 on sm_100a) depends on everything live
// around it; compiled as its own function, the loop is allocated like the
// standalone chain-step kernel the B200 sweep measured.  Arguments and result
// travel by value so nothing spills to local memory.
template <int NW>
struct NodeW {
  uint32_t w[NW];
};
struct State8 {
  uint32_t w[8];
};
#ifndef HS_CHAIN_NOINLINE
#define HS_CHAIN_NOINLINE 0
#endif
template <class V, int NW>
__device__ __noinline__ NodeW<NW> chain_F_ool(NodeW<NW> x, State8 mid, Adrs a, uint32_t start, uint32_t steps,
                                              uint32_t* rec) {
  chain_F<V, NW>(x.w, mid.w, a, start, steps, rec);
  return x;
}
// Measured on B200 (tools/variant_sweep.py): out of line was 3% faster for
// 8-word nodes at 4 blocks/SM but 2-7% slower for 4/6-word nodes, and inline
// wins again at the 3 blocks/SM the fused 256f kernel now uses; kept as a
// build option (HS_CHAIN_NOINLINE=1) for the next sweep.
template <class V, int NW>
__device__ __forceinline__ void chain_F_leaf(uint32_t* x, const uint32_t mid[8], const Adrs& a, uint32_t start,
                                             uint32_t steps, uint32_t* rec = nullptr) {
  if constexpr (HS_CHAIN_NOINLINE && NW == 8) {
    NodeW<NW> xv;
    State8 m;
#pragma unroll
    for (int j = 0; j < NW; j++) xv.w[j] = x[j];
#pragma unroll
    for (int j = 0; j < 8; j++) m.w[j] = mid[j];
    xv = chain_F_ool<V, NW>(xv, m, a, start, steps, rec);
#pragma unroll
    for (int j = 0; j < NW; j++) x[j] = xv.w[j];
  } else {
    chain_F<V, NW>(x, mid, a, start, steps, rec);
  }
}

// PRF(SK.seed, ADRS) = SHA-256(SK.seed || ADRS)[:n] from the IV (hashes.py:139-150).
template <class V, int NW>
__device__ __forceinline__ void prf_reg(uint32_t st[8], const uint32_t* sk_seed, const Adrs& a) {
  uint32_t W[16];
#pragma unroll
  for (int j = 0; j < NW; j++) W[j] = sk_seed[j];
  W[NW + 0] = a.w0; W[NW + 1] = a.w1; W[NW + 2] = a.w2; W[NW + 3] = a.w3; W[NW + 4] = a.w4;
  W[NW + 5] = (a.h5 << 16) | 0x8000u;
#pragma unroll
  for (int j = NW + 6; j < 15; j++) W[j] = 0;
  W[15] = (uint32_t)((4 * NW + 22) * 8);
#pragma unroll
  for (int i = 0; i < 8; i++) st[i] = IVc(i);
  compress<V>(st, W);
}

// PRF resumed from the key's state after rounds 0..NW-1 (those rounds read
// only SK.seed, identical for every PRF of the key; KeyDev::prf_mid).
template <class V, int NW>
__device__ __forceinline__ void prf_keyed(uint32_t st[8], const uint32_t prf_mid[8], const uint32_t* sk_seed,
                                          const Adrs& a) {
  uint32_t W[16], sR[8];
#pragma unroll
  for (int j = 0; j < NW; j++) W[j] = sk_seed[j];
  W[NW + 0] = a.w0; W[NW + 1] = a.w1; W[NW + 2] = a.w2; W[NW + 3] = a.w3; W[NW + 4] = a.w4;
  W[NW + 5] = (a.h5 << 16) | 0x8000u;
#pragma unroll
  for (int j = NW + 6; j < 15; j++) W[j] = 0;
  W[15] = (uint32_t)((4 * NW + 22) * 8);
#pragma unroll
  for (int i = 0; i < 8; i++) { st[i] = IVc(i); sR[i] = prf_mid[i]; }
  compress_resume<V, NW>(st, sR, W);
}

// ---------------------------------------------------------------------------
// Streaming tweakable hash over many nodes (T_len, T_k).  Message words go
// into a 32-word ring (two SHA blocks) in a caller-provided column of shared
// memory (one word every `stride` words, so a warp's columns are bank-
// conflict free); a block is compressed as soon as it is complete.  Write
// positions are warp-uniform in every caller, and there are exactly two
// compression sites (push_node, finish) to keep the kernels' code small.
// ---------------------------------------------------------------------------
template <class V>
struct TStream {
  uint32_t st[8];
  uint32_t carry;
  uint32_t pos;   // absolute word index of the next write
  uint32_t done;  // absolute word index of the next block not yet compressed
  uint32_t* buf;
  int stride;

  __device__ __forceinline__ void begin(const uint32_t mid[8], const Adrs& a, uint32_t* column, int col_stride) {
#pragma unroll
    for (int i = 0; i < 8; i++) st[i] = mid[i];
    buf = column;
    stride = col_stride;
    buf[0] = a.w0; buf[stride] = a.w1; buf[2 * stride] = a.w2; buf[3 * stride] = a.w3; buf[4 * stride] = a.w4;
    carry = a.h5;
    pos = 5;
    done = 0;
  }
  __device__ __forceinline__ void put(uint32_t at, uint32_t w) { buf[(at & 31u) * stride] = w; }
  __device__ __forceinline__ void compress_block() {
    uint32_t W[16];
    const uint32_t base = done & 31u;
#pragma unroll
    for (int j = 0; j < 16; j++) W[j] = buf[(base + j) * stride];
    compress<V>(st, W);
    done += 16;
  }
  template <int NW>
  __device__ __forceinline__ void push_node(const uint32_t* x) {
#pragma unroll
    for (int j = 0; j < NW; j++) {
      put(pos + j, (carry << 16) | (x[j] >> 16));
      carry = x[j] & 0xFFFFu;
    }
    pos += NW;
    if (pos >= done + 16) compress_block();
  }
  // total_bytes: bytes after the midstate block (22 + message length)
  __device__ __forceinline__ void finish(uint32_t total_bytes) {
    put(pos++, (carry << 16) | 0x8000u);
    const uint32_t end = ((pos & 15u) <= 14u ? (pos | 15u) + 1u : (pos | 15u) + 17u);
    while (pos < end - 1) put(pos++, 0u);
    put(pos++, (64u + total_bytes) * 8u);
#pragma unroll 1
    while (done < end) compress_block();
  }
};

// ---------------------------------------------------------------------------
// Word-level SHA-256 over  prefix (P big-endian words, compile-time count) ||
// M (mlen bytes, arbitrary length and alignment) || padding, starting from
// state `st` after `absorbed` bytes (a midstate: 64, or 0 from the IV).  Every
// message-preparation hash has this shape with M word-aligned after the prefix
// (HMAC inner: opt_rand || M; H_msg: R || PK.seed || PK.root || M), so M is
// read as whole words and no block buffer is indexed dynamically (a byte
// streamer would keep its block in local memory).  hashes.py:152-191.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t msg_word(const uint8_t* m, uint64_t mlen, uint64_t w) {
  const uint64_t b = 4 * w;
  if (b + 4 <= mlen) return ((uint32_t)m[b] << 24) | ((uint32_t)m[b + 1] << 16) | ((uint32_t)m[b + 2] << 8) | m[b + 3];
  if (b > mlen) return 0u;
  uint32_t v = 0;
  const int r = (int)(mlen - b);  // 0..3 bytes left, then the 0x80 padding byte
  for (int i = 0; i < r; i++) v |= (uint32_t)m[b + i] << (24 - 8 * i);
  return v | (0x80u << (24 - 8 * r));
}

template <class V, int P, bool Prep = true>
__device__ __forceinline__ void sha_prefix_msg(uint32_t st[8], uint64_t absorbed, const uint32_t (&pre)[P > 0 ? P : 1],
                                               const uint8_t* m, uint64_t mlen) {
  const uint64_t data = 4ull * P + mlen;                 // bytes hashed here
  const uint64_t nblk = (data + 9 + 63) / 64;
  const uint64_t bits = (absorbed + data) * 8;
  constexpr int PB = (P + 15) / 16;                      // blocks holding prefix words
#pragma unroll
  for (int b = 0; b < PB; b++) {
    if ((uint64_t)b >= nblk) break;
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const int k = 16 * b + j;
      W[j] = k < P ? pre[k < P ? k : 0] : msg_word(m, mlen, (uint64_t)(k - P));
    }
    if ((uint64_t)b == nblk - 1) { W[14] = (uint32_t)(bits >> 32); W[15] = (uint32_t)bits; }
    compress_sel<V, Prep>(st, W);
  }
#pragma unroll 1
  for (uint64_t b = PB; b < nblk; b++) {
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 16; j++) W[j] = msg_word(m, mlen, 16 * b + j - P);
    if (b == nblk - 1) { W[14] = (uint32_t)(bits >> 32); W[15] = (uint32_t)bits; }
    compress_sel<V, Prep>(st, W);
  }
}

// Short messages (mlen <= 64): M is loaded once as 17 padded words (all loads
// issued up front, predicated on mlen) and every hash over prefix || M reads
// it from registers -- the message-preparation chain is latency bound (one
// thread per message), so the loads must not sit between compressions.
constexpr int kShortMsgBytes = 64;
__device__ __forceinline__ void load_short_msg(const uint8_t* m, uint64_t mlen, uint32_t (&mw)[17]) {
#pragma unroll
  for (int j = 0; j < 17; j++) mw[j] = msg_word(m, mlen, (uint64_t)j);
}

template <class V, int P, bool Prep = true>
__device__ __forceinline__ void sha_prefix_words(uint32_t st[8], uint64_t absorbed, const uint32_t (&pre)[P],
                                                 const uint32_t (&mw)[17], uint64_t mlen) {
  const uint64_t data = 4ull * P + mlen;
  const uint32_t nblk = (uint32_t)((data + 9 + 63) / 64);
  const uint64_t bits = (absorbed + data) * 8;
  constexpr int NBMAX = (4 * P + kShortMsgBytes + 9 + 63) / 64;
#pragma unroll
  for (int b = 0; b < NBMAX; b++) {
    if ((uint32_t)b >= nblk) break;
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const int k = 16 * b + j;
      W[j] = k < P ? pre[k < P ? k : 0] : (k - P < 17 ? mw[k - P < 17 ? k - P : 0] : 0u);
    }
    if ((uint32_t)b == nblk - 1) { W[14] = (uint32_t)(bits >> 32); W[15] = (uint32_t)bits; }
    compress_sel<V, Prep>(st, W);
  }
}

}  // namespace hs
