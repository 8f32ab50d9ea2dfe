// sha256.cuh -- register-resident SHA-256 device library for sm_100a.
//
// Replaces the reference's two bit-identical compression backends
// (backends.py:51-123, selected per (kernel,set) by BackendSelection
// backends.py:201-257) with two compile-time arithmetic paths:
//
//   Native : plain C; ptxas picks IADD3/LOP3/SHF (ALU pipe) for almost all.
//   Imad   : every 32-bit add is written as a*one+b with `one` read from the
//            constant bank, so ptxas must emit IMAD (FMA pipe).  SHA-256 is
//            ALU-pipe bound on Blackwell (SHF+LOP3 have nowhere else to go);
//            moving the ~360 adds per compression to the otherwise idle FMA
//            pipe is the sm_100a analog of the paper's `mad.lo.u32` PTX path
//            (PAPER.md:341-382).
//
// Tweakable hashes follow hashes.py:124-150: thash = SHA-256(PKseed-midstate,
// ADRS(22B) || M)[:n]; PRF = SHA-256(SKseed || ADRS)[:n] from the IV.  Nodes
// are kept as big-endian 32-bit words (exactly the digest's state words), so
// no byte swapping happens inside the hypertree; the 22-byte ADRS puts every
// node at a 2-byte offset, handled with one PRMT/funnel-shift per word.
#pragma once
#include <cstdint>

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
// ---------------------------------------------------------------------------
struct Native {
  static constexpr int id = 0;
  static __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) { return a + b; }
};

struct Imad {
  static constexpr int id = 1;
  static __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) { return a * c_one + b; }
};

__device__ __forceinline__ uint32_t rotr(uint32_t x, int r) { return __funnelshift_r(x, x, r); }
__device__ __forceinline__ uint32_t bsig0(uint32_t a) { return rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22); }
__device__ __forceinline__ uint32_t bsig1(uint32_t e) { return rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25); }
__device__ __forceinline__ uint32_t ssig0(uint32_t x) { return rotr(x, 7) ^ rotr(x, 18) ^ (x >> 3); }
__device__ __forceinline__ uint32_t ssig1(uint32_t x) { return rotr(x, 17) ^ rotr(x, 19) ^ (x >> 10); }
__device__ __forceinline__ uint32_t ch(uint32_t e, uint32_t f, uint32_t g) { return g ^ (e & (f ^ g)); }
__device__ __forceinline__ uint32_t maj(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

// One SHA-256 compression; W is consumed (used as the rolling schedule).
// Fully unrolled so that constant message words (padding, lengths, zeros)
// fold into the schedule.
template <class V>
__device__ __forceinline__ void compress(uint32_t st[8], uint32_t W[16]) {
  uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
  for (int i = 0; i < 64; i++) {
    if (i >= 16) {
      W[i & 15] = V::add(V::add(ssig1(W[(i - 2) & 15]), W[(i - 7) & 15]),
                         V::add(ssig0(W[(i - 15) & 15]), W[i & 15]));
    }
    uint32_t t1 = V::add(V::add(V::add(h, Kc(i)), W[i & 15]), V::add(bsig1(e), ch(e, f, g)));
    uint32_t t2 = V::add(bsig0(a), maj(a, b, c));
    h = g; g = f; f = e; e = V::add(d, t1);
    d = c; c = b; b = a; a = V::add(t1, t2);
  }
  st[0] = V::add(st[0], a); st[1] = V::add(st[1], b); st[2] = V::add(st[2], c); st[3] = V::add(st[3], d);
  st[4] = V::add(st[4], e); st[5] = V::add(st[5], f); st[6] = V::add(st[6], g); st[7] = V::add(st[7], h);
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

// ---------------------------------------------------------------------------
// Streaming tweakable hash over many nodes (T_len, T_k).  The 16-word block
// under construction lives in a caller-provided column (shared memory, one
// word every `stride` words so a warp's columns are bank-conflict free).
// The write position is warp-uniform in every caller.
// ---------------------------------------------------------------------------
template <class V>
struct TStream {
  uint32_t st[8];
  uint32_t carry;
  int pos;
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
  }
  __device__ __forceinline__ void flush() {
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 16; j++) W[j] = buf[j * stride];
    compress<V>(st, W);
    pos = 0;
  }
  __device__ __forceinline__ void push(uint32_t w) {
    buf[pos * stride] = w;
    if (++pos == 16) flush();
  }
  template <int NW>
  __device__ __forceinline__ void push_node(const uint32_t* x) {
#pragma unroll
    for (int j = 0; j < NW; j++) {
      push((carry << 16) | (x[j] >> 16));
      carry = x[j] & 0xFFFFu;
    }
  }
  // total_bytes: bytes after the midstate block (22 + message length)
  __device__ __forceinline__ void finish(uint32_t total_bytes) {
    push((carry << 16) | 0x8000u);
    while (pos != 14) push(0u);
    push(0u);
    push((64u + total_bytes) * 8u);
  }
};

// ---------------------------------------------------------------------------
// Generic byte-stream SHA-256 (message preparation only: HMAC, H_msg, MGF1).
// One thread per message; the block buffer is thread-local.
// ---------------------------------------------------------------------------
template <class V>
struct ByteSha {
  uint32_t st[8];
  uint32_t blk[16];
  uint32_t fill;    // bytes in blk
  uint64_t total;   // bytes absorbed, including any midstate blocks

  __device__ void init_iv() {
    for (int i = 0; i < 8; i++) st[i] = IVc(i);
    fill = 0; total = 0;
  }
  __device__ void init_mid(const uint32_t mid[8], uint64_t absorbed) {
    for (int i = 0; i < 8; i++) st[i] = mid[i];
    fill = 0; total = absorbed;
  }
  __device__ void byte(uint32_t b) {
    int wi = fill >> 2, sh = 24 - 8 * (fill & 3);
    if ((fill & 3) == 0) blk[wi] = 0;
    blk[wi] |= (b & 0xFFu) << sh;
    fill++;
    total++;
    if (fill == 64) {
      uint32_t W[16];
      for (int j = 0; j < 16; j++) W[j] = blk[j];
      compress<V>(st, W);
      fill = 0;
    }
  }
  __device__ void bytes(const uint8_t* p, uint64_t len) {
    for (uint64_t i = 0; i < len; i++) byte(p[i]);
  }
  __device__ void word(uint32_t w) {  // 4 big-endian bytes
    byte(w >> 24); byte(w >> 16); byte(w >> 8); byte(w);
  }
  __device__ void words(const uint32_t* w, int nbytes) {  // first nbytes of BE words
    for (int i = 0; i < nbytes; i++) byte(w[i >> 2] >> (24 - 8 * (i & 3)));
  }
  __device__ void final(uint32_t out[8]) {
    uint64_t bits = total * 8;
    byte(0x80);
    while (fill != 56) byte(0);
    word((uint32_t)(bits >> 32));
    word((uint32_t)bits);
    for (int i = 0; i < 8; i++) out[i] = st[i];
  }
};

}  // namespace hs
