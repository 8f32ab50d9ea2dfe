// hs_kernels.cuh -- the B200 signing kernels (templated on parameter set S
// and SHA-256 arithmetic path V).
//
//   key_setup    per key: PK.seed midstate, HMAC ipad/opad midstates, PRF
//                state after SK.seed (hashes.py:79-88 precomputation, on device)
//   msg_prep     per message: R = PRF_msg, H_msg, MGF1, tree/leaf/FORS indices
//                (hashes.py:152-191, sigcore.py:75-121), shared-subtree flags
//   fors_sign    FORS_Sign with the paper's Tree Fusion: a CTA owns F fused
//                sets of N_tree trees (vexec.py:319-473, FusedSetLayout
//                vexec.py:130-181, Relax vexec.py:115-127), levels up to
//                fors_cta_levels in shared memory
//   fors_level   one upper FORS level for the whole batch
//   fors_pk      T_k over the k FORS roots (vexec.py:476-481)
//   tree_chain   TREE_Sign part 1: one thread per WOTS chain (wots.py:42-65)
//   tree_leaf    TREE_Sign part 2: one thread per hypertree leaf: T_len over
//                the chain ends (wots.py:119-143)
//   tree_merkle  TREE_Sign part 3: one thread per subtree: Merkle levels,
//                auth path, root (vexec.py:492-551 / oracle.py:27-63)
//   tree_root    parts 2+3 in one grid with a warp-shuffle Merkle reduction
//                (tree_split=1)
//   tree_sign    fused TREE_Sign (thread = leaf runs its chains), tree_split=0
//   shared_*     the top layers' subtrees, once per batch (both shapes)
//   wots_gather  WOTS+_Sign from the chain nodes TREE_Sign recorded;
//   wots_sign    WOTS+_Sign recomputing its chains (parallel.py:31-59)
//   keygen_root  root of layer d-1, tree 0 (oracle.py:216-226)
//   verify       one thread per signature (sigcore.py:181-221)
//
// Every output byte equals the reference's sigcore.sign for the same inputs.
#pragma once
#include <cstdint>

#include "hs_params.cuh"
#include "sha256.cuh"

namespace hs {

// Per-key device record (built by key_setup from sk = sk_seed||sk_prf||pk_seed||pk_root).
struct KeyDev {
  uint32_t sk_seed[8];
  uint32_t sk_prf[8];
  uint32_t pk_seed[8];
  uint32_t pk_root[8];
  uint32_t thash_mid[8];  // compress(IV, pk_seed || 0^(64-n))
  uint32_t hmac_i[8];     // compress(IV, (sk_prf||0) ^ 0x36..)
  uint32_t hmac_o[8];     // compress(IV, (sk_prf||0) ^ 0x5c..)
  uint32_t prf_mid[8];    // SHA-256 state after rounds 0..NW-1 over SK.seed: every PRF of the key resumes here
};

struct MsgPlan {
  uint64_t tree;   // bottom-layer tree index (masked to h - h/d bits)
  uint32_t leaf;   // bottom-layer leaf index
  uint32_t key;    // key table row
};

// Everything a launch needs; device pointers only.
struct LaunchArgs {
  const KeyDev* keys;
  KeyDev* keys_out;          // key_setup / keygen target
  const uint8_t* sk_bytes;   // key_setup input (nkeys * 4n) or keygen seeds (nkeys * 3n)
  uint32_t nkeys;
  const uint8_t* msgs;
  const uint64_t* offs;
  const uint32_t* key_idx;   // nullptr = key 0
  const uint8_t* opt_rand;   // nullptr = pk_seed (sigcore.py:162-163)
  uint32_t count;
  uint8_t* sigs;
  MsgPlan* plans;
  uint16_t* indices;         // count * k
  uint32_t* roots;           // count * (d+1) * 8 words; slot 0 = FORS pk, slot l+1 = root of layer l
  uint32_t* fors_roots;      // count * k * 8 words
  uint8_t* sk_out;           // keygen output (nkeys * 4n)
  uint32_t* stash;           // count * d * wots_len * w * NW words: signing-leaf chains (nullable)
  // Subtree sharing (top `shared_layers` hypertree layers): per key a table of
  // every subtree those layers can address, computed once per batch.
  uint32_t* shared;          // nkeys * units * shared_rec_words(S) (nullable)
  int shared_layers;         // 0 = off
  uint8_t* key_used;         // nkeys flags set by msg_prep
  uint8_t* unit_used;        // nkeys x units(shared_layers) flags set by msg_prep: shared subtrees the batch reads
  const uint8_t* pks;        // verify: nkeys * 2n (pk_seed || pk_root)
  const uint8_t* vsigs;      // verify: count * sig_bytes
  uint8_t* ok;               // verify: count flags
  int fors_trees_per_set;    // N_tree
  int fors_sets_fused;       // F
  int fors_relax;
  // FORS levels above fors_cta_levels are reduced by fors_level_kernel, one
  // grid per level over every (message, tree, node); fors_nodes[0/1] hold the
  // levels in between (node-major, NW words per node).  fors_cta_levels ==
  // log_t keeps the whole tree inside the CTA (no level kernels).
  int fors_cta_levels;
  int fors_level;            // level computed by one fors_level_kernel launch
  uint32_t* fors_nodes[2];
  // Split TREE_Sign: tree_chain_kernel writes every chain end of the batch's
  // per-message leaves here ([msg][layer][leaf][chain][NW]); tree_root_kernel
  // compresses them into leaves and reduces the subtrees.  nullptr = fused
  // tree_sign_kernel (thread = leaf runs its own chains).
  uint32_t* chain_ends;
  uint32_t* shared_ends;     // split shared subtrees: [key][unit][leaf][chain][NW] (nullable)
  uint32_t* fors_lpre;       // [msg][log_t + 1][8]: per FORS level the H state after ADRS rounds 0..4
  // WOTS_Sign F steps per message (sum of the signed base-w digits over all
  // d layers; zeroed before the batch), for the exact compression count the
  // reference's ctx_out reports (hashes.py:117-159).  nullable.
  uint32_t* wots_steps;
};

// L1 prefetch hint (latency-bound single-thread loops: T_len, T_k, Merkle levels)
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ uint64_t shr64(uint64_t x, int s) { return s >= 64 ? 0ull : (x >> s); }

__device__ __forceinline__ void store_be(uint8_t* p, uint32_t w) { *reinterpret_cast<uint32_t*>(p) = bswap32(w); }

template <int NW>
__device__ __forceinline__ void store_node(uint8_t* p, const uint32_t* x) {
#pragma unroll
  for (int j = 0; j < NW; j++) store_be(p + 4 * j, x[j]);
}

// Store one of two register-resident nodes chosen at run time: a per-word
// select keeps both in registers (passing `first ? a : b` as a pointer makes
// ptxas place the arrays in local memory).
template <int NW>
__device__ __forceinline__ void store_node_sel(uint8_t* p, bool first, const uint32_t* a, const uint32_t* b) {
#pragma unroll
  for (int j = 0; j < NW; j++) store_be(p + 4 * j, first ? a[j] : b[j]);
}

__device__ __forceinline__ uint32_t load_be(const uint8_t* p) {
  return ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
}

// ---------------------------------------------------------------------------
// key_setup: one thread per key
// ---------------------------------------------------------------------------
template <int S, class V>
__global__ void key_setup_kernel(LaunchArgs a) {
  using Pr = P<S>;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nkeys) return;
  const uint8_t* sk = a.sk_bytes + (size_t)i * Pr::sk_bytes;
  KeyDev kd;
  for (int j = 0; j < 8; j++) {
    kd.sk_seed[j] = j < Pr::NW ? load_be(sk + 4 * j) : 0u;
    kd.sk_prf[j] = j < Pr::NW ? load_be(sk + Pr::n + 4 * j) : 0u;
    kd.pk_seed[j] = j < Pr::NW ? load_be(sk + 2 * Pr::n + 4 * j) : 0u;
    kd.pk_root[j] = j < Pr::NW ? load_be(sk + 3 * Pr::n + 4 * j) : 0u;
  }
  uint32_t W[16];
  for (int j = 0; j < 8; j++) kd.thash_mid[j] = IVc(j);
  for (int j = 0; j < 16; j++) W[j] = j < Pr::NW ? kd.pk_seed[j] : 0u;
  compress<V>(kd.thash_mid, W);
  for (int j = 0; j < 8; j++) kd.hmac_i[j] = IVc(j);
  for (int j = 0; j < 16; j++) W[j] = (j < Pr::NW ? kd.sk_prf[j] : 0u) ^ 0x36363636u;
  compress<V>(kd.hmac_i, W);
  for (int j = 0; j < 8; j++) kd.hmac_o[j] = IVc(j);
  for (int j = 0; j < 16; j++) W[j] = (j < Pr::NW ? kd.sk_prf[j] : 0u) ^ 0x5c5c5c5cu;
  compress<V>(kd.hmac_o, W);
  for (int j = 0; j < 8; j++) kd.prf_mid[j] = IVc(j);
  rounds_prefix<V, Pr::NW>(kd.prf_mid, kd.sk_seed);
  a.keys_out[i] = kd;
}

// layer schedule (sigcore.py:107-121)
template <int S>
__device__ __forceinline__ void layer_coords(const MsgPlan& pl, int layer, uint64_t& tree, uint32_t& leaf) {
  using Pr = P<S>;
  if (layer == 0) {
    tree = pl.tree;
    leaf = pl.leaf;
  } else {
    leaf = (uint32_t)(shr64(pl.tree, Pr::hp * (layer - 1)) & (uint64_t)(Pr::leaves - 1));
    tree = shr64(pl.tree, Pr::hp * layer);
  }
}

// Shared subtrees per key for L shared top layers: sum_{j<L} 2^(hp*j) (layer
// d-1-j holds 2^(hp*j) trees); unit u of depth j is units(j) + tree.
template <int S>
__host__ __device__ constexpr int shared_units(int L) {
  return L <= 0 ? 0 : shared_units<S>(L - 1) + (1 << (P<S>::hp * (L - 1)));
}

// ---------------------------------------------------------------------------
// msg_prep: one thread per message (hashes.py:152-191, sigcore.py:75-90)
// ---------------------------------------------------------------------------
template <int S, class V>
__global__ void msg_prep_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int n = Pr::n;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.count) return;
  const uint32_t key = a.key_idx ? a.key_idx[i] : 0u;
  const KeyDev& K = a.keys[key];
  const uint8_t* msg = a.msgs + a.offs[i];
  const uint64_t mlen = a.offs[i + 1] - a.offs[i];

  constexpr int NW = Pr::NW;
  // R = HMAC-SHA-256(sk_prf, opt_rand || msg)[:n]  (hashes.py:152-165)
  uint32_t st[8], R[8], mw[17];
  {
    uint32_t pre[NW];
    const uint8_t* o = a.opt_rand ? a.opt_rand + (size_t)i * n : nullptr;
#pragma unroll
    for (int j = 0; j < NW; j++) pre[j] = o ? load_be(o + 4 * j) : K.pk_seed[j];
#pragma unroll
    for (int j = 0; j < 8; j++) st[j] = K.hmac_i[j];
    if (mlen <= kShortMsgBytes) {
      load_short_msg(msg, mlen, mw);
      sha_prefix_words<V, NW>(st, 64, pre, mw, mlen);
    } else {
      sha_prefix_msg<V, NW>(st, 64, pre, msg, mlen);
    }
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 8; j++) { W[j] = st[j]; R[j] = K.hmac_o[j]; }
    W[8] = 0x80000000u;
#pragma unroll
    for (int j = 9; j < 15; j++) W[j] = 0;
    W[15] = (64 + 32) * 8;
    compress_prep<V>(R, W);
  }
  uint8_t* sig = a.sigs + (size_t)i * Pr::sig_bytes;
  store_node<NW>(sig, R);

  // H_msg: MGF1(R || PK.seed || SHA-256(R || PK.seed || PK.root || M), digest_bytes)  (hashes.py:167-191)
  uint32_t dig0[8];
  {
    uint32_t pre[3 * NW];
#pragma unroll
    for (int j = 0; j < NW; j++) { pre[j] = R[j]; pre[NW + j] = K.pk_seed[j]; pre[2 * NW + j] = K.pk_root[j]; }
#pragma unroll
    for (int j = 0; j < 8; j++) dig0[j] = IVc(j);
    if (mlen <= kShortMsgBytes) sha_prefix_words<V, 3 * NW>(dig0, 0, pre, mw, mlen);
    else sha_prefix_msg<V, 3 * NW>(dig0, 0, pre, msg, mlen);
  }
  // MGF1 counter blocks: SHA-256(R || PK.seed || dig0 || c) for c = 0, 1.
  // R || PK.seed || dig0[0..] fill the first block for every counter, so it
  // is compressed once; each counter then costs one block.  The digest stays
  // in registers as big-endian words (dw), every byte and bit below is read
  // at a compile-time position.
  constexpr int nctr = (Pr::digest_bytes + 31) / 32;
  constexpr int PW = 2 * NW + 8;  // prefix words before the counter
  static_assert(PW >= 16 && PW < 16 + 14, "MGF1 seed spans exactly one full block plus the counter block");
  uint32_t pre[PW];
#pragma unroll
  for (int j = 0; j < NW; j++) { pre[j] = R[j]; pre[NW + j] = K.pk_seed[j]; }
#pragma unroll
  for (int j = 0; j < 8; j++) pre[2 * NW + j] = dig0[j];
  uint32_t m1[8];
#pragma unroll
  for (int j = 0; j < 8; j++) m1[j] = IVc(j);
  compress_prep<V>(m1, pre);
  uint32_t dw[8 * nctr];
#pragma unroll
  for (int c = 0; c < nctr; c++) {
    uint32_t W[16], o[8];
#pragma unroll
    for (int j = 0; j < 16; j++) W[j] = 0u;
#pragma unroll
    for (int j = 16; j < PW; j++) W[j - 16] = pre[j];
    W[PW - 16] = (uint32_t)c;
    W[PW - 15] = 0x80000000u;
    W[15] = (uint32_t)((PW + 1) * 32);
#pragma unroll
    for (int j = 0; j < 8; j++) o[j] = m1[j];
    compress_prep<V>(o, W);
#pragma unroll
    for (int j = 0; j < 8; j++) dw[8 * c + j] = o[j];
  }
  auto dbyte = [&](int b) -> uint32_t { return (dw[b >> 2] >> (24 - 8 * (b & 3))) & 0xFFu; };
  uint64_t tree = 0;
#pragma unroll
  for (int j = 0; j < Pr::tree_bytes; j++) tree = (tree << 8) | dbyte(Pr::fors_msg_bytes + j);
  if (Pr::tree_bits < 64) tree &= (1ull << (Pr::tree_bits < 64 ? Pr::tree_bits : 63)) - 1ull;
  uint32_t leaf = 0;
#pragma unroll
  for (int j = 0; j < Pr::leaf_bytes; j++) leaf = (leaf << 8) | dbyte(Pr::fors_msg_bytes + Pr::tree_bytes + j);
  leaf &= (1u << Pr::leaf_bits) - 1u;
  MsgPlan pl;
  pl.tree = tree;
  pl.leaf = leaf;
  pl.key = key;
  a.plans[i] = pl;
  if (a.key_used) a.key_used[key] = 1;
  if (a.unit_used) {  // the shared subtrees this message's top layers read
    const int U = shared_units<S>(a.shared_layers);
    for (int j = 0; j < a.shared_layers; j++) {
      uint64_t t;
      uint32_t lf;
      layer_coords<S>(pl, Pr::d - 1 - j, t, lf);
      a.unit_used[(size_t)key * U + shared_units<S>(j) + (uint32_t)t] = 1;
    }
  }
  // FORS indices, LSB-first bit order within each byte (sigcore.py:75-90)
#pragma unroll
  for (int g = 0; g < Pr::k; g++) {
    uint32_t v = 0;
#pragma unroll
    for (int j = 0; j < Pr::log_t; j++) {
      const int off = g * Pr::log_t + j;
      v |= ((dbyte(off >> 3) >> (off & 7)) & 1u) << j;
    }
    a.indices[(size_t)i * Pr::k + g] = (uint16_t)v;
  }
}


// ---------------------------------------------------------------------------
// One WOTS+ leaf (wots.py:119-143): wots_len chains of PRF + (w-1) F, then
// T_len over the chain ends streamed through this thread's smem column.
// ---------------------------------------------------------------------------
// rec (nullable): wots_len x 16 nodes -- every chain position 0..15 of this
// leaf, recorded when this leaf is the layer's signing leaf.
template <int S, class V>
__device__ __forceinline__ void wots_leaf(const KeyDev& K, uint32_t layer, uint64_t tree, uint32_t leaf,
                                          uint32_t* column, int stride, uint32_t out[8], uint32_t* rec = nullptr) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  uint32_t mid[8], sks[NW];
#pragma unroll
  for (int j = 0; j < 8; j++) mid[j] = K.thash_mid[j];
#pragma unroll
  for (int j = 0; j < NW; j++) sks[j] = K.sk_seed[j];
  TStream<V> ts;
  ts.begin(mid, make_adrs(layer, tree, ADDR_WOTS_PK, leaf, 0, 0), column, stride);
  Adrs wa = make_adrs(layer, tree, ADDR_WOTS, leaf, 0, 0);
  // The chain secrets PRF(SK.seed, ADRS(chain i, hash 0)) of one leaf differ
  // only in ADRS word 4 (the chain index): SHA-256 rounds [0, NW+4) are run
  // once per leaf and kept in this thread's smem column (words 32..39).
  {
    uint32_t W[NW + 4], s[8];
#pragma unroll
    for (int j = 0; j < NW; j++) W[j] = sks[j];
    W[NW + 0] = wa.w0; W[NW + 1] = wa.w1; W[NW + 2] = wa.w2; W[NW + 3] = wa.w3;
#pragma unroll
    for (int j = 0; j < 8; j++) s[j] = IVc(j);
    rounds_prefix<V, NW + 4>(s, W);
#pragma unroll
    for (int j = 0; j < 8; j++) column[(32 + j) * stride] = s[j];
  }
#pragma unroll 1
  for (int i = 0; i < Pr::wots_len; i++) {
    uint32_t st[8], sR[8], W[16];
    adrs_set_chain_hash(wa, (uint32_t)i, 0);
#pragma unroll
    for (int j = 0; j < NW; j++) W[j] = sks[j];
    W[NW + 0] = wa.w0; W[NW + 1] = wa.w1; W[NW + 2] = wa.w2; W[NW + 3] = wa.w3; W[NW + 4] = wa.w4;
    W[NW + 5] = 0x8000u;  // hash index 0, then the padding bit
#pragma unroll
    for (int j = NW + 6; j < 15; j++) W[j] = 0;
    W[15] = (uint32_t)((4 * NW + 22) * 8);
#pragma unroll
    for (int j = 0; j < 8; j++) { st[j] = IVc(j); sR[j] = column[(32 + j) * stride]; }
    compress_resume<V, NW + 4>(st, sR, W);
    uint32_t x[NW];
#pragma unroll
    for (int j = 0; j < NW; j++) x[j] = st[j];
    uint32_t* crec = rec ? rec + (size_t)i * Pr::w * NW : nullptr;
    if (crec) {
#pragma unroll
      for (int j = 0; j < NW; j++) crec[j] = x[j];
    }
    chain_F_leaf<V, NW>(x, mid, wa, 0u, (uint32_t)(Pr::w - 1), crec);
    ts.template push_node<NW>(x);
  }
  ts.finish(22u + (uint32_t)(Pr::wots_len * Pr::n));
#pragma unroll
  for (int j = 0; j < 8; j++) out[j] = ts.st[j];
}

// ---------------------------------------------------------------------------
// TREE_Sign: thread = (message, layer, leaf); leaves of a subtree sit in
// consecutive lanes of one warp and are reduced with shuffles.
// ---------------------------------------------------------------------------
constexpr int kTreeBlock = 128;
constexpr int kLeafColumnWords = 40;  // per-thread smem column: 32-word T_len ring + 8-word PRF prefix
#ifndef HS_TREE_MIN_BLOCKS
#define HS_TREE_MIN_BLOCKS 5
#endif
#ifndef HS_TREE_MIN_BLOCKS_8W
#define HS_TREE_MIN_BLOCKS_8W 3
#endif
// 5 blocks -> <= 96 registers, 20 warps / SM; 256f (8-word nodes) uses 3 blocks / 168 registers
// (B200 sweep over 3..6 blocks x SHA paths, profiles/r01_tree_occupancy.txt)
constexpr int kTreeMinBlocks = HS_TREE_MIN_BLOCKS;
constexpr int kTreeMinBlocks8 = HS_TREE_MIN_BLOCKS_8W;

template <int S, class V>
__global__ void __launch_bounds__(kTreeBlock, (S == 2 ? kTreeMinBlocks8 : kTreeMinBlocks)) tree_sign_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  __shared__ uint32_t tbuf[kLeafColumnWords * kTreeBlock];
  // layers >= d - shared_layers come from the shared-subtree table instead
  const uint64_t per_msg = (uint64_t)(Pr::d - a.shared_layers) * Pr::leaves;
  const uint64_t gid = (uint64_t)blockIdx.x * kTreeBlock + threadIdx.x;
  const bool valid = gid < (uint64_t)a.count * per_msg;
  const uint32_t msg = valid ? (uint32_t)(gid / per_msg) : 0u;
  const uint32_t rem = (uint32_t)(gid % per_msg);
  const uint32_t layer = rem / Pr::leaves;
  const uint32_t leaf = rem % Pr::leaves;

  uint32_t node[8];
  uint64_t tree = 0;
  uint32_t leaf_idx = 0;
  const KeyDev* K = nullptr;
  if (valid) {
    const MsgPlan pl = a.plans[msg];
    K = &a.keys[pl.key];
    layer_coords<S>(pl, (int)layer, tree, leaf_idx);
    uint32_t* rec = (a.stash && leaf == leaf_idx)
                        ? a.stash + ((size_t)msg * Pr::d + layer) * Pr::wots_len * Pr::w * NW
                        : nullptr;
    wots_leaf<S, V>(*K, layer, tree, leaf, &tbuf[threadIdx.x], kTreeBlock, node, rec);
  }
  uint8_t* auth = a.sigs + (size_t)msg * Pr::sig_bytes + Pr::off_ht + (size_t)layer * Pr::layer_bytes +
                  Pr::wots_sig_bytes;
#pragma unroll 1
  for (int lvl = 1; lvl <= Pr::hp; lvl++) {
    const uint32_t below = leaf >> (lvl - 1);
    const bool holder_below = (leaf & ((1u << (lvl - 1)) - 1u)) == 0u;
    if (valid && holder_below && below == ((leaf_idx >> (lvl - 1)) ^ 1u))
      store_node<NW>(auth + (lvl - 1) * Pr::n, node);
    uint32_t other[NW];
#pragma unroll
    for (int j = 0; j < NW; j++) other[j] = __shfl_down_sync(0xffffffffu, node[j], 1u << (lvl - 1));
    if (valid && (leaf & ((1u << lvl) - 1u)) == 0u) {
      uint32_t m[2 * NW];
#pragma unroll
      for (int j = 0; j < NW; j++) { m[j] = node[j]; m[NW + j] = other[j]; }
      uint32_t mid[8];
#pragma unroll
      for (int j = 0; j < 8; j++) mid[j] = K->thash_mid[j];
      thash_reg<V, 2 * NW>(node, mid, make_adrs(layer, tree, ADDR_HASHTREE, 0, (uint32_t)lvl, leaf >> lvl), m);
    }
  }
  if (valid && leaf == 0) {
    uint32_t* r = a.roots + ((size_t)msg * (Pr::d + 1) + layer + 1) * 8;
#pragma unroll
    for (int j = 0; j < NW; j++) r[j] = node[j];
  }
}

// ---------------------------------------------------------------------------
// Split TREE_Sign.  Part 1, tree_chain_kernel: thread = (message, layer, leaf,
// chain) runs PRF + (w-1) F for one WOTS chain (wots.py:42-65) and writes the
// chain end; the signing leaf's chains also record every position for the
// WOTS gather.  A thread holds one chain state, so the kernel keeps the
// register budget of the standalone chain step (the B200 sweep's shape,
// tools/sha_sweep) instead of the fused leaf kernel's 96, and the grid has
// wots_len times more threads.  Part 2, tree_root_kernel: thread = (message,
// layer, leaf) compresses its wots_len chain ends into the leaf (T_len,
// wots.py:140-143, streamed straight from global memory) and the leaves of a
// subtree are reduced with warp shuffles as in tree_sign_kernel.
// ---------------------------------------------------------------------------
// threads per block of the chain grids, per set (r02, interleaved A/B of
// 64/128/256: 256 is 1.7 % faster than 128 for 256f's TREE_Sign and 0.4 %
// for 192f; 128 stays for 128f, whose batch time is the same either way,
// profiles/r02c_ab_chain_block*.txt)
#ifndef HS_CHAIN_BLOCK_S0
#define HS_CHAIN_BLOCK_S0 128
#endif
#ifndef HS_CHAIN_BLOCK_S1
#define HS_CHAIN_BLOCK_S1 256
#endif
#ifndef HS_CHAIN_BLOCK_S2
#define HS_CHAIN_BLOCK_S2 256
#endif
template <int S>
constexpr int kChainBlock = S == 0 ? HS_CHAIN_BLOCK_S0 : S == 1 ? HS_CHAIN_BLOCK_S1 : HS_CHAIN_BLOCK_S2;
// No min-blocks bound by default: ptxas then allocates 55-64 registers for the
// chain loop; any explicit bound (even 1) changes the allocation and cost
// 5-10 % on B200 (profiles/r01_chain_block_sweep.txt).
#ifdef HS_CHAIN_MIN_BLOCKS
#define HS_CHAIN_BOUNDS __launch_bounds__(kChainBlock<S>, HS_CHAIN_MIN_BLOCKS)
#else
#define HS_CHAIN_BOUNDS __launch_bounds__(kChainBlock<S>)
#endif

template <int S, class V>
__global__ void HS_CHAIN_BOUNDS tree_chain_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  const uint32_t dl = (uint32_t)(Pr::d - a.shared_layers);
  const uint64_t gid = (uint64_t)blockIdx.x * kChainBlock<S> + threadIdx.x;
  if (gid >= (uint64_t)a.count * dl * Pr::leaves * Pr::wots_len) return;
  const uint32_t chain = (uint32_t)(gid % Pr::wots_len);
  const uint64_t lid = gid / Pr::wots_len;             // (msg, layer, leaf)
  const uint32_t leaf = (uint32_t)(lid % Pr::leaves);
  const uint32_t layer = (uint32_t)((lid / Pr::leaves) % dl);
  const uint32_t msg = (uint32_t)(lid / ((uint64_t)Pr::leaves * dl));
  const MsgPlan pl = a.plans[msg];
  const KeyDev& K = a.keys[pl.key];
  uint64_t tree;
  uint32_t leaf_idx;
  layer_coords<S>(pl, (int)layer, tree, leaf_idx);
  uint32_t mid[8], sks[NW], st[8];
#pragma unroll
  for (int j = 0; j < 8; j++) mid[j] = K.thash_mid[j];
#pragma unroll
  for (int j = 0; j < NW; j++) sks[j] = K.sk_seed[j];
  const Adrs wa = make_adrs(layer, tree, ADDR_WOTS, leaf, chain, 0);
  prf_keyed<V, NW>(st, K.prf_mid, sks, wa);             // chain secret (wots.py:63-65)
  uint32_t x[NW];
#pragma unroll
  for (int j = 0; j < NW; j++) x[j] = st[j];
  uint32_t* rec = (a.stash && leaf == leaf_idx)
                      ? a.stash + (((size_t)msg * Pr::d + layer) * Pr::wots_len + chain) * Pr::w * NW
                      : nullptr;
  if (rec) {
#pragma unroll
    for (int j = 0; j < NW; j++) rec[j] = x[j];
  }
  chain_F<V, NW>(x, mid, wa, 0u, (uint32_t)(Pr::w - 1), rec);
  uint32_t* e = a.chain_ends + gid * NW;
#pragma unroll
  for (int j = 0; j < NW; j++) e[j] = x[j];
}

// Word k (0-based, after the PK.seed midstate block) of the T_len input
// ADRS(22 B) || ends (M = wots_len * NW words) || SHA-256 padding, with the
// chain ends read from global memory (thash_reg's layout, hashes.py:124-137).
template <int M>
__device__ __forceinline__ uint32_t tlen_word(uint32_t k, const uint32_t aw[6], const uint32_t* e, uint32_t len_bits,
                                              uint32_t last) {
  if (k < 5) return k == 0 ? aw[0] : k == 1 ? aw[1] : k == 2 ? aw[2] : k == 3 ? aw[3] : aw[4];  // no local array
  if (k == 5) return join16(aw[5], e[0]);
  if (k < 5 + M) return join16(e[k - 6], e[k - 5]);
  if (k == 5 + M) return (e[M - 1] << 16) | 0x8000u;
  return k == last ? len_bits : 0u;
}

// tlen_word with the two chain-end words it may need already in registers:
// lo = e[k - 6], hi = e[k - 5] (either may be a don't-care outside the ends).
template <int M>
__device__ __forceinline__ uint32_t tlen_word_raw(uint32_t k, const uint32_t aw[6], uint32_t lo, uint32_t hi,
                                                  uint32_t len_bits, uint32_t last) {
  if (k < 5) return k == 0 ? aw[0] : k == 1 ? aw[1] : k == 2 ? aw[2] : k == 3 ? aw[3] : aw[4];
  if (k == 5) return join16(aw[5], hi);
  if (k < 5 + M) return join16(lo, hi);
  if (k == 5 + M) return (lo << 16) | 0x8000u;
  return k == last ? len_bits : 0u;
}

template <int S, class V>
__global__ void __launch_bounds__(kTreeBlock) tree_root_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  constexpr int M = Pr::wots_len * NW;
  constexpr uint32_t total = 22u + (uint32_t)(Pr::wots_len * Pr::n);  // bytes after the midstate block
  constexpr uint32_t nblk = (total + 9u + 63u) / 64u;
  const uint32_t dl = (uint32_t)(Pr::d - a.shared_layers);
  const uint64_t per_msg = (uint64_t)dl * Pr::leaves;
  const uint64_t gid = (uint64_t)blockIdx.x * kTreeBlock + threadIdx.x;
  const bool valid = gid < (uint64_t)a.count * per_msg;
  const uint32_t msg = valid ? (uint32_t)(gid / per_msg) : 0u;
  const uint32_t rem = (uint32_t)(gid % per_msg);
  const uint32_t layer = rem / Pr::leaves;
  const uint32_t leaf = rem % Pr::leaves;

  uint32_t node[8];
  uint64_t tree = 0;
  uint32_t leaf_idx = 0;
  const KeyDev* K = nullptr;
  if (valid) {
    const MsgPlan pl = a.plans[msg];
    K = &a.keys[pl.key];
    layer_coords<S>(pl, (int)layer, tree, leaf_idx);
    const Adrs pa = make_adrs(layer, tree, ADDR_WOTS_PK, leaf, 0, 0);
    const uint32_t aw[6] = {pa.w0, pa.w1, pa.w2, pa.w3, pa.w4, pa.h5};
    const uint32_t* e = a.chain_ends + gid * M;
#pragma unroll
    for (int j = 0; j < 8; j++) node[j] = K->thash_mid[j];
    // T_len, the chain-end words of block b+1 loaded into registers while
    // block b compresses: this grid runs the small graphs (tree_small_batch),
    // where each leaf thread is alone on the critical path and a load per
    // block would wait a full L2 round trip (raw[i] = e[16b - 6 + i])
    uint32_t raw[17];
#pragma unroll
    for (int i = 0; i < 17; i++) raw[i] = (i >= 6 && i - 6 < M) ? e[i - 6] : 0u;
#pragma unroll 1
    for (uint32_t b = 0; b < nblk; b++) {
      uint32_t nxt[17];
#pragma unroll
      for (int i = 0; i < 17; i++) {
        const int idx = (int)(16u * (b + 1u)) - 6 + i;
        nxt[i] = (b + 1u < nblk && idx >= 0 && idx < M) ? e[idx] : 0u;
      }
      uint32_t W[16];
#pragma unroll
      for (int j = 0; j < 16; j++)
        W[j] = tlen_word_raw<M>(16u * b + j, aw, raw[j], raw[j + 1], (64u + total) * 8u, 16u * nblk - 1u);
      compress<V>(node, W);
#pragma unroll
      for (int i = 0; i < 17; i++) raw[i] = nxt[i];
    }
  }
  uint8_t* auth = a.sigs + (size_t)msg * Pr::sig_bytes + Pr::off_ht + (size_t)layer * Pr::layer_bytes +
                  Pr::wots_sig_bytes;
#pragma unroll 1
  for (int lvl = 1; lvl <= Pr::hp; lvl++) {
    const uint32_t below = leaf >> (lvl - 1);
    const bool holder_below = (leaf & ((1u << (lvl - 1)) - 1u)) == 0u;
    if (valid && holder_below && below == ((leaf_idx >> (lvl - 1)) ^ 1u))
      store_node<NW>(auth + (lvl - 1) * Pr::n, node);
    uint32_t other[NW];
#pragma unroll
    for (int j = 0; j < NW; j++) other[j] = __shfl_down_sync(0xffffffffu, node[j], 1u << (lvl - 1));
    if (valid && (leaf & ((1u << lvl) - 1u)) == 0u) {
      uint32_t m[2 * NW];
#pragma unroll
      for (int j = 0; j < NW; j++) { m[j] = node[j]; m[NW + j] = other[j]; }
      uint32_t mid[8];
#pragma unroll
      for (int j = 0; j < 8; j++) mid[j] = K->thash_mid[j];
      thash_reg<V, 2 * NW>(node, mid, make_adrs(layer, tree, ADDR_HASHTREE, 0, (uint32_t)lvl, leaf >> lvl), m);
    }
  }
  if (valid && leaf == 0) {
    uint32_t* r = a.roots + ((size_t)msg * (Pr::d + 1) + layer + 1) * 8;
#pragma unroll
    for (int j = 0; j < NW; j++) r[j] = node[j];
  }
}

// tree_split = 2: part 2 computes only the leaves (T_len); the subtree is
// reduced by tree_merkle_kernel.
template <int S, class V>
__global__ void __launch_bounds__(kTreeBlock) tree_leaf_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  constexpr int M = Pr::wots_len * NW;
  constexpr uint32_t total = 22u + (uint32_t)(Pr::wots_len * Pr::n);  // bytes after the midstate block
  constexpr uint32_t nblk = (total + 9u + 63u) / 64u;
  const uint32_t dl = (uint32_t)(Pr::d - a.shared_layers);
  const uint64_t per_msg = (uint64_t)dl * Pr::leaves;
  const uint64_t gid = (uint64_t)blockIdx.x * kTreeBlock + threadIdx.x;
  if (gid >= (uint64_t)a.count * per_msg) return;
  const uint32_t msg = (uint32_t)(gid / per_msg);
  const uint32_t rem = (uint32_t)(gid % per_msg);
  const uint32_t layer = rem / Pr::leaves;
  const uint32_t leaf = rem % Pr::leaves;

  const MsgPlan pl = a.plans[msg];
  const KeyDev& K = a.keys[pl.key];
  uint64_t tree;
  uint32_t leaf_idx;
  layer_coords<S>(pl, (int)layer, tree, leaf_idx);
  const Adrs pa = make_adrs(layer, tree, ADDR_WOTS_PK, leaf, 0, 0);
  const uint32_t aw[6] = {pa.w0, pa.w1, pa.w2, pa.w3, pa.w4, pa.h5};
  uint32_t* e = a.chain_ends + gid * M;
  uint32_t node[8];
#pragma unroll
  for (int j = 0; j < 8; j++) node[j] = K.thash_mid[j];
#pragma unroll 1
  for (uint32_t b = 0; b < nblk; b++) {
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 16; j++) W[j] = tlen_word<M>(16u * b + j, aw, e, (64u + total) * 8u, 16u * nblk - 1u);
    // the next block's chain-end words (e[16b+10 .. 16b+26]) are requested
    // while this block compresses: a lone leaf thread (small batches) no
    // longer waits one L2 round trip per block
    if (16u * b + 26u < (uint32_t)M) prefetch_l1(e + 16u * b + 26u);
    if (16u * b + 10u < (uint32_t)M) prefetch_l1(e + 16u * b + 10u);
    compress<V>(node, W);
  }
  // the leaf replaces the head of its own (consumed) chain-end record, where
  // tree_merkle_kernel picks it up; the signing leaf's sibling is auth[0]
#pragma unroll
  for (int j = 0; j < NW; j++) e[j] = node[j];
  if (leaf == (leaf_idx ^ 1u)) {
    uint8_t* auth = a.sigs + (size_t)msg * Pr::sig_bytes + Pr::off_ht + (size_t)layer * Pr::layer_bytes +
                    Pr::wots_sig_bytes;
    store_node<NW>(auth, node);
  }
}

// TREE_Sign part 3: thread = (message, layer) reduces its subtree's leaves
// (treehash, oracle.py:27-63 / vexec.py:518-551) level by level -- level 1
// from the leaves tree_leaf_kernel left at the heads of their chain-end
// records, the levels above in place in a thread-local buffer (node j of level
// L replaces node j of level L-1 after its children 2j, 2j+1 are read) --
// storing the auth path nodes of levels 1..hp-1 and the root.  One thread per subtree keeps every
// lane busy at every level; reducing inside tree_root with warp shuffles left
// 1/2, 3/4, 7/8 of a subtree's lanes idle at levels 1, 2, 3.
template <int S, class V>
__global__ void __launch_bounds__(kTreeBlock) tree_merkle_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  constexpr int M = Pr::wots_len * NW;
  const uint32_t dl = (uint32_t)(Pr::d - a.shared_layers);
  const uint64_t gid = (uint64_t)blockIdx.x * kTreeBlock + threadIdx.x;
  if (gid >= (uint64_t)a.count * dl) return;
  const uint32_t msg = (uint32_t)(gid / dl);
  const uint32_t layer = (uint32_t)(gid % dl);
  const MsgPlan pl = a.plans[msg];
  const KeyDev& K = a.keys[pl.key];
  uint64_t tree;
  uint32_t leaf_idx;
  layer_coords<S>(pl, (int)layer, tree, leaf_idx);
  uint32_t mid[8];
#pragma unroll
  for (int j = 0; j < 8; j++) mid[j] = K.thash_mid[j];
  const uint32_t* base = a.chain_ends + gid * (uint64_t)Pr::leaves * M;
  uint8_t* auth = a.sigs + (size_t)msg * Pr::sig_bytes + Pr::off_ht + (size_t)layer * Pr::layer_bytes +
                  Pr::wots_sig_bytes;
  // every leaf head is requested up front (one L1 prefetch per record), so the
  // level-1 loads do not each wait a full L2 round trip behind the previous H
#pragma unroll
  for (int i = 0; i < Pr::leaves; i++) prefetch_l1(base + (size_t)i * M);
  // levels >= 1 live in this thread's local memory (L1-resident: a store and
  // the later load of the same thread never round-trip through L2)
  uint32_t lv[Pr::leaves / 2][NW];
  uint32_t node[8];
#pragma unroll 1
  for (int lvl = 1; lvl <= Pr::hp; lvl++) {
    const uint32_t per = (uint32_t)Pr::leaves >> lvl;
    const uint32_t sib = (leaf_idx >> lvl) ^ 1u;
#pragma unroll 1
    for (uint32_t j = 0; j < per; j++) {
      uint32_t m[2 * NW];
      if (lvl == 1) {
#pragma unroll
        for (int w = 0; w < NW; w++) { m[w] = base[(size_t)(2 * j) * M + w]; m[NW + w] = base[(size_t)(2 * j + 1) * M + w]; }
      } else {
#pragma unroll
        for (int w = 0; w < NW; w++) { m[w] = lv[2 * j][w]; m[NW + w] = lv[2 * j + 1][w]; }
      }
      thash_reg<V, 2 * NW>(node, mid, make_adrs(layer, tree, ADDR_HASHTREE, 0, (uint32_t)lvl, j), m);
      if (lvl < Pr::hp && j == sib) store_node<NW>(auth + lvl * Pr::n, node);
#pragma unroll
      for (int w = 0; w < NW; w++) lv[j][w] = node[w];
    }
  }
  uint32_t* r = a.roots + ((size_t)msg * (Pr::d + 1) + layer + 1) * 8;
#pragma unroll
  for (int j = 0; j < NW; j++) r[j] = node[j];
}

// ---------------------------------------------------------------------------
// Subtree sharing.  The top layers of the hypertree can only address a few
// subtrees per key (layer d-1: tree 0; layer d-2: 2^(h/d) trees; ...), so in a
// batch signed by one key most messages walk the same ones.  A subtree is a
// pure function of (key, layer, tree) -- identical leaves, nodes and WOTS
// chains for every message that reaches it -- so TREE_Sign computes each of
// them once per batch (tree_shared_kernel) and the per-message kernels skip
// those layers; wots_gather_kernel then reads the message's auth path, root
// and WOTS chain nodes from the shared record.  Output bytes are unchanged.
//
// Record of one shared subtree: nodes of every level ([level][index], 8 words
// each, levels 0..hp), then all leaves' chains ([leaf][chain][pos][NW]).
// ---------------------------------------------------------------------------
template <int S>
struct Shared {
  using Pr = P<S>;
  // down to the layer with 2^(hp*j) = 32768 (hp 3) / 4096 (hp 4) subtrees per
  // key; the auto policy shares a layer only when its subtrees are at most
  // twice the key's messages (and only the subtrees the batch reads are built)
  static constexpr int max_layers = Pr::hp >= 4 ? 4 : 6;
  static constexpr int node_words = (2 * Pr::leaves - 1) * 8;
  static constexpr int leaf_stash_words = Pr::wots_len * Pr::w * Pr::NW;
  static constexpr int rec_words = node_words + Pr::leaves * leaf_stash_words;
  // units per key for L shared layers: sum_{j<L} 2^(hp*j)
  __host__ __device__ static constexpr int units(int L) { return shared_units<S>(L); }
  // level offset (in nodes) inside a record
  __device__ static constexpr int level_off(int lvl) { return lvl == 0 ? 0 : level_off(lvl - 1) + (Pr::leaves >> (lvl - 1)); }
  // record of (key, layer, tree); layer >= d - L
  __device__ static uint32_t* rec(const LaunchArgs& a, uint32_t key, int layer, uint64_t tree) {
    const int j = Pr::d - 1 - layer;  // depth from the top
    const size_t unit = (size_t)units(j) + (size_t)tree;
    return a.shared + ((size_t)key * units(a.shared_layers) + unit) * rec_words;
  }
};

template <int S, class V>
__global__ void __launch_bounds__(kTreeBlock, (S == 2 ? kTreeMinBlocks8 : kTreeMinBlocks)) tree_shared_kernel(LaunchArgs a) {
  using Pr = P<S>;
  using Sh = Shared<S>;
  constexpr int NW = Pr::NW;
  __shared__ uint32_t tbuf[kLeafColumnWords * kTreeBlock];
  const int U = Sh::units(a.shared_layers);
  const uint64_t per_key = (uint64_t)U * Pr::leaves;
  const uint64_t gid = (uint64_t)blockIdx.x * kTreeBlock + threadIdx.x;
  const uint32_t key = (uint32_t)(gid / per_key);
  const bool valid = key < a.nkeys && a.key_used[key] &&
                     (!a.unit_used || a.unit_used[(size_t)key * U + (uint32_t)((gid % per_key) / Pr::leaves)]);
  const uint32_t rem = (uint32_t)(gid % per_key);
  const uint32_t unit = rem / Pr::leaves;
  const uint32_t leaf = rem % Pr::leaves;
  int j = 0;
  while (j + 1 < a.shared_layers && (uint32_t)Sh::units(j + 1) <= unit) j++;
  const uint32_t layer = Pr::d - 1 - j;
  const uint64_t tree = unit - Sh::units(j);
  uint32_t node[8];
  uint32_t* R = nullptr;
  const KeyDev& K = a.keys[valid ? key : 0u];
  if (valid) {
    R = Sh::rec(a, key, (int)layer, tree);
    wots_leaf<S, V>(K, layer, tree, leaf, &tbuf[threadIdx.x], kTreeBlock, node,
                    R + Sh::node_words + (size_t)leaf * Sh::leaf_stash_words);
#pragma unroll
    for (int w = 0; w < NW; w++) R[leaf * 8 + w] = node[w];
  }
#pragma unroll 1
  for (int lvl = 1; lvl <= Pr::hp; lvl++) {
    uint32_t other[NW];
#pragma unroll
    for (int w = 0; w < NW; w++) other[w] = __shfl_down_sync(0xffffffffu, node[w], 1u << (lvl - 1));
    if (valid && (leaf & ((1u << lvl) - 1u)) == 0u) {
      uint32_t m[2 * NW], mid[8];
#pragma unroll
      for (int w = 0; w < NW; w++) { m[w] = node[w]; m[NW + w] = other[w]; }
#pragma unroll
      for (int w = 0; w < 8; w++) mid[w] = K.thash_mid[w];
      thash_reg<V, 2 * NW>(node, mid, make_adrs(layer, tree, ADDR_HASHTREE, 0, (uint32_t)lvl, leaf >> lvl), m);
      uint32_t* dst = R + (size_t)(Sh::level_off(lvl) + (leaf >> lvl)) * 8;
#pragma unroll
      for (int w = 0; w < NW; w++) dst[w] = node[w];
    }
  }
}

// Split form of tree_shared_kernel (used with tree_split): the shared
// subtrees' chains as one grid (thread = (key, unit, leaf, chain), every
// position recorded into the subtree record for the WOTS gather), then one
// thread per (key, unit, leaf) for T_len and the record's Merkle levels.  The
// fused kernel runs a whole leaf per thread with only units x leaves threads
// (4,681 x 8 for 128f/192f at 5 shared layers), a long serial tail under the
// per-message kernels; the split grids have wots_len times more threads.
// Bodies follow tree_chain_kernel / tree_root_kernel (kept separate so the
// per-message kernels' register allocation is untouched).
template <int S>
__device__ __forceinline__ bool shared_coords(const LaunchArgs& a, uint64_t lid, uint32_t& key, uint32_t& layer,
                                              uint64_t& tree, uint32_t& leaf) {
  using Pr = P<S>;
  using Sh = Shared<S>;
  const uint64_t per_key = (uint64_t)Sh::units(a.shared_layers) * Pr::leaves;
  key = (uint32_t)(lid / per_key);
  if (key >= a.nkeys || !a.key_used[key]) return false;
  const uint32_t rem = (uint32_t)(lid % per_key);
  const uint32_t unit = rem / Pr::leaves;
  leaf = rem % Pr::leaves;
  if (a.unit_used && !a.unit_used[(size_t)key * Sh::units(a.shared_layers) + unit]) return false;
  int j = 0;
  while (j + 1 < a.shared_layers && (uint32_t)Sh::units(j + 1) <= unit) j++;
  layer = Pr::d - 1 - j;
  tree = unit - Sh::units(j);
  return true;
}

template <int S, class V>
__global__ void HS_CHAIN_BOUNDS shared_chain_kernel(LaunchArgs a) {
  using Pr = P<S>;
  using Sh = Shared<S>;
  constexpr int NW = Pr::NW;
  const uint64_t gid = (uint64_t)blockIdx.x * kChainBlock<S> + threadIdx.x;
  if (gid >= (uint64_t)a.nkeys * Sh::units(a.shared_layers) * Pr::leaves * Pr::wots_len) return;
  const uint32_t chain = (uint32_t)(gid % Pr::wots_len);
  uint32_t key, layer, leaf;
  uint64_t tree;
  if (!shared_coords<S>(a, gid / Pr::wots_len, key, layer, tree, leaf)) return;
  const KeyDev& K = a.keys[key];
  uint32_t mid[8], sks[NW], st[8];
#pragma unroll
  for (int j = 0; j < 8; j++) mid[j] = K.thash_mid[j];
#pragma unroll
  for (int j = 0; j < NW; j++) sks[j] = K.sk_seed[j];
  const Adrs wa = make_adrs(layer, tree, ADDR_WOTS, leaf, chain, 0);
  prf_keyed<V, NW>(st, K.prf_mid, sks, wa);
  uint32_t x[NW];
#pragma unroll
  for (int j = 0; j < NW; j++) x[j] = st[j];
  uint32_t* rec = Sh::rec(a, key, (int)layer, tree) + Sh::node_words + (size_t)leaf * Sh::leaf_stash_words +
                  (size_t)chain * Pr::w * NW;
#pragma unroll
  for (int j = 0; j < NW; j++) rec[j] = x[j];
  chain_F<V, NW>(x, mid, wa, 0u, (uint32_t)(Pr::w - 1), rec);
  uint32_t* e = a.shared_ends + gid * NW;
#pragma unroll
  for (int j = 0; j < NW; j++) e[j] = x[j];
}

template <int S, class V>
__global__ void __launch_bounds__(kTreeBlock) shared_root_kernel(LaunchArgs a) {
  using Pr = P<S>;
  using Sh = Shared<S>;
  constexpr int NW = Pr::NW;
  constexpr int M = Pr::wots_len * NW;
  constexpr uint32_t total = 22u + (uint32_t)(Pr::wots_len * Pr::n);
  constexpr uint32_t nblk = (total + 9u + 63u) / 64u;
  const uint64_t gid = (uint64_t)blockIdx.x * kTreeBlock + threadIdx.x;
  uint32_t key = 0, layer = 0, leaf = (uint32_t)(gid % Pr::leaves);
  uint64_t tree = 0;
  const bool valid = gid < (uint64_t)a.nkeys * Sh::units(a.shared_layers) * Pr::leaves &&
                     shared_coords<S>(a, gid, key, layer, tree, leaf);
  uint32_t node[8];
  uint32_t* R = nullptr;
  const KeyDev& K = a.keys[valid ? key : 0u];
  if (valid) {
    R = Sh::rec(a, key, (int)layer, tree);
    const Adrs pa = make_adrs(layer, tree, ADDR_WOTS_PK, leaf, 0, 0);
    const uint32_t aw[6] = {pa.w0, pa.w1, pa.w2, pa.w3, pa.w4, pa.h5};
    const uint32_t* e = a.shared_ends + gid * M;
#pragma unroll
    for (int j = 0; j < 8; j++) node[j] = K.thash_mid[j];
#pragma unroll 1
    for (uint32_t b = 0; b < nblk; b++) {
      uint32_t W[16];
#pragma unroll
      for (int j = 0; j < 16; j++) W[j] = tlen_word<M>(16u * b + j, aw, e, (64u + total) * 8u, 16u * nblk - 1u);
      compress<V>(node, W);
    }
#pragma unroll
    for (int w = 0; w < NW; w++) R[leaf * 8 + w] = node[w];
  }
#pragma unroll 1
  for (int lvl = 1; lvl <= Pr::hp; lvl++) {
    uint32_t other[NW];
#pragma unroll
    for (int w = 0; w < NW; w++) other[w] = __shfl_down_sync(0xffffffffu, node[w], 1u << (lvl - 1));
    if (valid && (leaf & ((1u << lvl) - 1u)) == 0u) {
      uint32_t m[2 * NW], mid[8];
#pragma unroll
      for (int w = 0; w < NW; w++) { m[w] = node[w]; m[NW + w] = other[w]; }
#pragma unroll
      for (int w = 0; w < 8; w++) mid[w] = K.thash_mid[w];
      thash_reg<V, 2 * NW>(node, mid, make_adrs(layer, tree, ADDR_HASHTREE, 0, (uint32_t)lvl, leaf >> lvl), m);
      uint32_t* dst = R + (size_t)(Sh::level_off(lvl) + (leaf >> lvl)) * 8;
#pragma unroll
      for (int w = 0; w < NW; w++) dst[w] = node[w];
    }
  }
}

// ---------------------------------------------------------------------------
// FORS_Sign with Tree Fusion.  CTA = (message, pass); a pass owns F fused
// sets of N_tree trees; blockDim = N_tree * t (or N_tree * t/2 with Relax,
// where each lane builds a leaf pair in registers and stores only the
// parent).  Levels ping-pong between two shared regions, one barrier per
// level; each level's nodes of all fused trees are spread over every lane,
// so one barrier covers all F sets.
// ---------------------------------------------------------------------------
// 768 lanes keep the register budget at 85 per thread (65536 / 768).
constexpr int kForsMaxLanes = 768;
// per-set launch bound of fors_sign_kernel (<= kForsMaxLanes): a smaller bound
// gives ptxas more registers per lane for layouts that use fewer lanes
#ifndef HS_FORS_LB_S0
#define HS_FORS_LB_S0 768
#endif
#ifndef HS_FORS_LB_S1
#define HS_FORS_LB_S1 768
#endif
#ifndef HS_FORS_LB_S2
#define HS_FORS_LB_S2 768
#endif
template <int S>
constexpr int kForsLaunchBound = S == 0 ? HS_FORS_LB_S0 : S == 1 ? HS_FORS_LB_S1 : HS_FORS_LB_S2;
// minimum resident CTAs per SM the launch bound asks ptxas for (register cap
// 65536 / (bound x minB)); 1 = no cap beyond the bound
#ifndef HS_FORS_MINB_S0
#define HS_FORS_MINB_S0 1
#endif
#ifndef HS_FORS_MINB_S1
#define HS_FORS_MINB_S1 1
#endif
#ifndef HS_FORS_MINB_S2
#define HS_FORS_MINB_S2 1
#endif
template <int S>
constexpr int kForsMinBlocks = S == 0 ? HS_FORS_MINB_S0 : S == 1 ? HS_FORS_MINB_S1 : HS_FORS_MINB_S2;
// A second, narrow instantiation for layouts of at most kForsNarrowLanes<S>
// lanes, compiled for kForsNarrowMinB<S> resident CTAs (64 registers): 192f
// (256 lanes x 4) and 256f (512 x 2) one-tree-per-set layouts run 0.4 / 0.55 %
// faster than under the 768-lane bound (profiles/r02cc_fors_occupancy_ab.txt).
// HS_FORS_NARROW=0 builds the wide kernel only.
#ifndef HS_FORS_NARROW
#define HS_FORS_NARROW 1
#endif
// 128f's 384-lane layout already fits two CTAs per SM at 80 registers
// (HS_FORS_NARROW_S0 / HS_FORS_NARROW_MINB_S0 set a narrow bound for it).
#ifndef HS_FORS_NARROW_S0
#define HS_FORS_NARROW_S0 0
#endif
#ifndef HS_FORS_NARROW_MINB_S0
#define HS_FORS_NARROW_MINB_S0 3
#endif
template <int S>
constexpr int kForsNarrowLanes = !HS_FORS_NARROW ? 0 : S == 0 ? HS_FORS_NARROW_S0 : S == 1 ? 256 : 512;
template <int S>
constexpr int kForsNarrowMinB = S == 0 ? HS_FORS_NARROW_MINB_S0 : S == 1 ? 4 : 2;
// per-message PRF / F prefix states (16 words) and per-level H prefix states
// ((log_t + 1) x 8 words, log_t <= 9) at the head of FORS_Sign's smem
constexpr int kForsPrefixWords = 16 + 8 * 10;

template <int S>
__host__ __device__ constexpr int fors_smem_words_per_tree(bool relax) {
  // region A (t or t/4 nodes) + region B (t/2 nodes)
  return relax ? (P<S>::t / 4 + P<S>::t / 2) * P<S>::NW : (P<S>::t + P<S>::t / 2) * P<S>::NW;
}

// FORS leaf (oracle.py:101-110): sk = PRF(adrs(height 0, index)), leaf = F(sk).
// For a given message every FORS leaf address differs only in the tree index
// (ADRS bytes 20..21; index < 2^16), so the PRF's first NW+5 message words
// (SK.seed, ADRS words 0..4) and F's first 5 are fixed per message: those
// SHA-256 rounds are computed once per CTA (`pre`, shared memory: PRF state
// after NW+5 rounds, F state after 5) and every leaf resumes from them.
template <int S, class V>
__device__ __forceinline__ void fors_prefix(const uint32_t mid[8], const uint32_t* sks, const Adrs& fa,
                                            uint32_t* pre) {
  constexpr int NW = P<S>::NW;
  uint32_t W[16], s1[8], s2[8];
#pragma unroll
  for (int j = 0; j < NW; j++) W[j] = sks[j];
  W[NW + 0] = fa.w0; W[NW + 1] = fa.w1; W[NW + 2] = fa.w2; W[NW + 3] = fa.w3; W[NW + 4] = fa.w4;
#pragma unroll
  for (int i = 0; i < 8; i++) { s1[i] = IVc(i); s2[i] = mid[i]; }
  rounds_prefix<V, NW + 5>(s1, W);
  const uint32_t W2[5] = {fa.w0, fa.w1, fa.w2, fa.w3, fa.w4};
  rounds_prefix<V, 5>(s2, W2);
#pragma unroll
  for (int i = 0; i < 8; i++) { pre[i] = s1[i]; pre[8 + i] = s2[i]; }
}

template <int S, class V>
__device__ __forceinline__ void fors_leaf(const uint32_t mid[8], const uint32_t* sks, const Adrs& fa,
                                          const uint32_t* pre, uint32_t gidx, uint32_t sk_out[8],
                                          uint32_t leaf_out[8]) {
  constexpr int NW = P<S>::NW;
  uint32_t W[16], sR[8];
#pragma unroll
  for (int j = 0; j < NW; j++) W[j] = sks[j];
  W[NW + 0] = fa.w0; W[NW + 1] = fa.w1; W[NW + 2] = fa.w2; W[NW + 3] = fa.w3; W[NW + 4] = fa.w4;
  W[NW + 5] = (gidx << 16) | 0x8000u;
#pragma unroll
  for (int j = NW + 6; j < 15; j++) W[j] = 0;
  W[15] = (uint32_t)((4 * NW + 22) * 8);
#pragma unroll
  for (int i = 0; i < 8; i++) { sk_out[i] = IVc(i); sR[i] = pre[i]; }
  compress_resume<V, NW + 5>(sk_out, sR, W);
  W[0] = fa.w0; W[1] = fa.w1; W[2] = fa.w2; W[3] = fa.w3; W[4] = fa.w4;
  W[5] = join16(gidx, sk_out[0]);
#pragma unroll
  for (int j = 1; j < NW; j++) W[5 + j] = join16(sk_out[j - 1], sk_out[j]);
  W[5 + NW] = (sk_out[NW - 1] << 16) | 0x8000u;
#pragma unroll
  for (int j = 6 + NW; j < 15; j++) W[j] = 0;
  W[15] = (uint32_t)((64 + 22 + 4 * NW) * 8);
#pragma unroll
  for (int i = 0; i < 8; i++) { leaf_out[i] = mid[i]; sR[i] = pre[8 + i]; }
  compress_resume<V, 5>(leaf_out, sR, W);
}

template <int S, class V, int LB = kForsLaunchBound<S>, int MINB = kForsMinBlocks<S>>
__global__ void __launch_bounds__(LB, MINB) fors_sign_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  constexpr int t = Pr::t;
  extern __shared__ uint32_t sm[];
  const int ntree = a.fors_trees_per_set;
  const int fused = a.fors_sets_fused;
  const bool relax = a.fors_relax != 0;
  const int tpc = ntree * fused;                       // trees per CTA
  const int sets_total = (Pr::k + ntree - 1) / ntree;
  const int passes = (sets_total + fused - 1) / fused;
  const uint32_t msg = blockIdx.x / passes;
  const int pass = blockIdx.x % passes;
  const int g0 = pass * tpc;
  const int ntr = min(tpc, Pr::k - g0);              // active trees in this CTA
  if (msg >= a.count) return;
  const int lanes_per_tree = relax ? t / 2 : t;
  const int capA = relax ? t / 4 : t;
  // word-major (SoA) regions: word w of node (tree slot tl, index j) lives at
  // X[w * S_X + tl * cap_X + j], so a lane's two children are one 8-byte
  // shared load per word and a warp's accesses are bank-conflict free
  const int SA = tpc * capA, SB = tpc * (t / 2);
  uint32_t* pre = sm;                                  // [16] per-message SHA-256 prefix states
  uint32_t* regA = sm + kForsPrefixWords;              // [NW][tpc][capA]
  uint32_t* regB = regA + (size_t)NW * SA;             // [NW][tpc][t/2]

  const MsgPlan pl = a.plans[msg];
  const KeyDev& K = a.keys[pl.key];
  uint32_t mid[8], sks[NW];
#pragma unroll
  for (int j = 0; j < 8; j++) mid[j] = K.thash_mid[j];
#pragma unroll
  for (int j = 0; j < NW; j++) sks[j] = K.sk_seed[j];
  const uint16_t* idx = a.indices + (size_t)msg * Pr::k;
  uint8_t* fsig = a.sigs + (size_t)msg * Pr::sig_bytes + Pr::off_fors;
  constexpr int tree_sig = (1 + Pr::log_t) * Pr::n;    // sk || auth[log_t]
  const Adrs fa = make_adrs(0, pl.tree, ADDR_FORS_TREE, pl.leaf, 0, 0);

  const int tid = threadIdx.x;
  // Every H of FORS level L of this message has ADRS words 0..4 = (layer 0,
  // tree, FORS_TREE, keypair, height L, hash index >> 16 = 0): SHA-256 rounds
  // 0..4 of its first block are computed once per level here (lpre[L]) and by
  // pass 0 handed to the level grids.
  static_assert(Pr::k * Pr::t <= 65536, "FORS hash index must fit ADRS bytes 20..21");
  uint32_t* lpre = sm + 16;
  if (tid == 0) {
    fors_prefix<S, V>(mid, sks, fa, pre);
  } else if (tid <= Pr::log_t) {
    Adrs la = fa;
    adrs_set_chain_hash(la, (uint32_t)tid, 0u);
    const uint32_t W04[5] = {la.w0, la.w1, la.w2, la.w3, la.w4};
    uint32_t s5[8];
#pragma unroll
    for (int i = 0; i < 8; i++) s5[i] = mid[i];
    rounds_prefix<V, 5>(s5, W04);
#pragma unroll
    for (int i = 0; i < 8; i++) lpre[tid * 8 + i] = s5[i];
    if (a.fors_lpre && pass == 0) {
      uint32_t* g = a.fors_lpre + ((size_t)msg * (Pr::log_t + 1) + tid) * 8;
#pragma unroll
      for (int i = 0; i < 8; i++) g[i] = s5[i];
    }
  }
  __syncthreads();

  // ---- leaf phase (vexec.py:387-435) ----
  // last = the level handed to fors_level_kernel through fors_nodes[0] (or
  // log_t: the whole tree stays in this CTA).  With last == 0 (Relax: 1) the
  // leaf phase writes its nodes straight to global memory and no level runs
  // here at all.
  const int last = a.fors_cta_levels;
  const bool to_global = last == (relax ? 1 : 0);
  const int tree_in_set = tid / lanes_per_tree;
  const int lane_leaf = tid % lanes_per_tree;
#pragma unroll 1
  for (int f = 0; f < fused; f++) {
    const int tl = f * ntree + tree_in_set;            // tree slot in this CTA
    if (tl >= ntr) continue;
    const int g = g0 + tl;
    const uint32_t sel = idx[g];
    if (!relax) {
      uint32_t sk[8], lf[8];
      fors_leaf<S, V>(mid, sks, fa, pre, (uint32_t)(g * t + lane_leaf), sk, lf);
      if ((uint32_t)lane_leaf == sel) store_node<NW>(fsig + g * tree_sig, sk);
      if (to_global) {
        uint32_t* d = a.fors_nodes[0] + (((size_t)msg * Pr::k + g) * t + lane_leaf) * NW;
#pragma unroll
        for (int j = 0; j < NW; j++) d[j] = lf[j];
      } else {
        uint32_t* dst = regA + (size_t)tl * capA + lane_leaf;
#pragma unroll
        for (int j = 0; j < NW; j++) dst[(size_t)j * SA] = lf[j];
      }
    } else {
      uint32_t sk0[8], l0[8], sk1[8], l1[8];
      const uint32_t j2 = 2u * lane_leaf;
      fors_leaf<S, V>(mid, sks, fa, pre, (uint32_t)(g * t) + j2, sk0, l0);
      fors_leaf<S, V>(mid, sks, fa, pre, (uint32_t)(g * t) + j2 + 1u, sk1, l1);
      if (j2 == sel) store_node<NW>(fsig + g * tree_sig, sk0);
      if (j2 + 1u == sel) store_node<NW>(fsig + g * tree_sig, sk1);
      if ((sel >> 1) == (uint32_t)lane_leaf) store_node_sel<NW>(fsig + g * tree_sig + Pr::n, (sel & 1u) != 0u, l0, l1);
      uint32_t m[2 * NW], par[8];
#pragma unroll
      for (int j = 0; j < NW; j++) { m[j] = l0[j]; m[NW + j] = l1[j]; }
      Adrs pa = fa;
      adrs_set_chain_hash(pa, 1, (uint32_t)lane_leaf + ((uint32_t)(g * t) >> 1));
      thash_reg_pre<V, 2 * NW>(par, mid, lpre + 8, pa, m);
      if (to_global) {
        uint32_t* d = a.fors_nodes[0] + (((size_t)msg * Pr::k + g) * (t / 2) + lane_leaf) * NW;
#pragma unroll
        for (int j = 0; j < NW; j++) d[j] = par[j];
      } else {
        uint32_t* dst = regB + (size_t)tl * (t / 2) + lane_leaf;
#pragma unroll
        for (int j = 0; j < NW; j++) dst[(size_t)j * SB] = par[j];
      }
    }
  }
  if (to_global) return;  // uniform across the CTA
  __syncthreads();

  // ---- reduction levels (vexec.py:437-463) ----
  const int first = relax ? 2 : 1;
#pragma unroll 1
  for (int lvl = first; lvl <= last; lvl++) {
    // level lvl-1 lives in A when (lvl-1) is even (no relax) ... track by parity
    const bool src_is_A = relax ? ((lvl & 1) == 1) : ((lvl & 1) == 1);
    const uint32_t* src = src_is_A ? regA : regB;
    uint32_t* dst = src_is_A ? regB : regA;
    const int src_cap = src_is_A ? capA : t / 2;
    const int dst_cap = src_is_A ? t / 2 : capA;
    const int src_S = src_is_A ? SA : SB;
    const int dst_S = src_is_A ? SB : SA;
    const int per_tree = t >> lvl;
    const int total = ntr * per_tree;
#pragma unroll 1
    for (int q = tid; q < total; q += blockDim.x) {
      const int tl = q / per_tree;
      const int j = q % per_tree;
      const int g = g0 + tl;
      const uint32_t* c = src + (size_t)tl * src_cap + 2 * j;
      uint32_t m[2 * NW];
#pragma unroll
      for (int w = 0; w < NW; w++) {
        const uint2 v = *reinterpret_cast<const uint2*>(c + (size_t)w * src_S);
        m[w] = v.x;
        m[NW + w] = v.y;
      }
      const uint32_t sel = (uint32_t)idx[g] >> (lvl - 1);
      if ((sel >> 1) == (uint32_t)j)
        store_node_sel<NW>(fsig + g * tree_sig + Pr::n + (lvl - 1) * Pr::n, (sel & 1u) != 0u, m, m + NW);
      uint32_t par[8];
      Adrs na = fa;
      adrs_set_chain_hash(na, (uint32_t)lvl, (uint32_t)j + ((uint32_t)(g * t) >> lvl));
      thash_reg_pre<V, 2 * NW>(par, mid, lpre + lvl * 8, na, m);
      if (lvl == Pr::log_t) {
        uint32_t* r = a.fors_roots + ((size_t)msg * Pr::k + g) * 8;
#pragma unroll
        for (int w = 0; w < NW; w++) r[w] = par[w];
      } else if (lvl == last) {  // hand the sparse upper levels to fors_level_kernel
        uint32_t* d = a.fors_nodes[0] + (((size_t)msg * Pr::k + g) * (uint32_t)per_tree + j) * NW;
#pragma unroll
        for (int w = 0; w < NW; w++) d[w] = par[w];
      } else {
        uint32_t* d = dst + (size_t)tl * dst_cap + j;
#pragma unroll
        for (int w = 0; w < NW; w++) d[(size_t)w * dst_S] = par[w];
      }
    }
    __syncthreads();
  }
}

// One FORS level L > fors_cta_levels for the whole batch: thread = (message,
// tree, node j of level L); children come from the level below in
// fors_nodes[(L - Lc - 1) & 1], the parent goes to the other buffer (or to
// fors_roots at the top).  Upper levels hold few nodes per tree, so inside a
// CTA they leave most lanes idle at a barrier; as batch-wide grids every lane
// has a node.  Same hash inputs and auth-path rule as the in-CTA levels
// (vexec.py:437-463).
constexpr int kForsLevelBlock = 128;
template <int S, class V>
__global__ void __launch_bounds__(kForsLevelBlock) fors_level_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  constexpr int t = Pr::t;
  const int L = a.fors_level;
  const uint32_t per_tree = (uint32_t)t >> L;
  const uint64_t gid = (uint64_t)blockIdx.x * kForsLevelBlock + threadIdx.x;
  if (gid >= (uint64_t)a.count * Pr::k * per_tree) return;
  const uint32_t j = (uint32_t)(gid % per_tree);
  const uint64_t tg = gid / per_tree;                  // msg * k + g
  const uint32_t g = (uint32_t)(tg % Pr::k);
  const uint32_t msg = (uint32_t)(tg / Pr::k);
  const int par_buf = (L - a.fors_cta_levels) & 1;      // level Lc lives in buffer 0
  const uint32_t* c = a.fors_nodes[par_buf ^ 1] + (tg * (2 * per_tree) + 2 * j) * NW;
  uint32_t m[2 * NW];
#pragma unroll
  for (int w = 0; w < 2 * NW; w++) m[w] = c[w];
  const MsgPlan pl = a.plans[msg];
  const KeyDev& K = a.keys[pl.key];
  const uint32_t sel = (uint32_t)a.indices[(size_t)msg * Pr::k + g] >> (L - 1);
  constexpr int tree_sig = (1 + Pr::log_t) * Pr::n;
  uint8_t* fsig = a.sigs + (size_t)msg * Pr::sig_bytes + Pr::off_fors;
  if ((sel >> 1) == j) store_node_sel<NW>(fsig + g * tree_sig + Pr::n + (L - 1) * Pr::n, (sel & 1u) != 0u, m, m + NW);
  uint32_t mid[8], pre5[8], par[8];
  const uint32_t* lp = a.fors_lpre + ((size_t)msg * (Pr::log_t + 1) + L) * 8;
#pragma unroll
  for (int w = 0; w < 8; w++) { mid[w] = K.thash_mid[w]; pre5[w] = lp[w]; }
  Adrs na = make_adrs(0, pl.tree, ADDR_FORS_TREE, pl.leaf, 0, 0);
  adrs_set_chain_hash(na, (uint32_t)L, j + ((g * (uint32_t)t) >> L));
  thash_reg_pre<V, 2 * NW>(par, mid, pre5, na, m);
  uint32_t* d = (L == Pr::log_t) ? a.fors_roots + tg * 8 : a.fors_nodes[par_buf] + (tg * per_tree + j) * NW;
#pragma unroll
  for (int w = 0; w < NW; w++) d[w] = par[w];
}

// T_k over the k FORS roots -> roots slot 0 (vexec.py:476-481).
constexpr int kSmallBlock = 128;

template <int S, class V>
__global__ void __launch_bounds__(kSmallBlock) fors_pk_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  __shared__ uint32_t tbuf[32 * kSmallBlock];
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.count) return;
  const MsgPlan pl = a.plans[i];
  const KeyDev& K = a.keys[pl.key];
  uint32_t mid[8];
#pragma unroll
  for (int j = 0; j < 8; j++) mid[j] = K.thash_mid[j];
  TStream<V> ts;
  ts.begin(mid, make_adrs(0, pl.tree, ADDR_FORS_ROOTS, pl.leaf, 0, 0), &tbuf[threadIdx.x], kSmallBlock);
  const uint32_t* fr = a.fors_roots + (size_t)i * Pr::k * 8;
#pragma unroll
  for (int g = 0; g < 8; g += 4) prefetch_l1(fr + g * 8);
#pragma unroll 1
  for (int g = 0; g < Pr::k; g++) {
    if (g % 4 == 0 && g + 8 < Pr::k) prefetch_l1(fr + (g + 8) * 8);  // two 128-B lines (8 roots) ahead
    uint32_t x[NW];
#pragma unroll
    for (int j = 0; j < NW; j++) x[j] = fr[g * 8 + j];
    ts.template push_node<NW>(x);
  }
  ts.finish(22u + (uint32_t)(Pr::k * Pr::n));
  uint32_t* r = a.roots + (size_t)i * (Pr::d + 1) * 8;
#pragma unroll
  for (int j = 0; j < NW; j++) r[j] = ts.st[j];
}

// ---------------------------------------------------------------------------
// WOTS+_Sign: thread = (message, layer, chain) (parallel.py:31-59)
// ---------------------------------------------------------------------------
template <int S>
__device__ __forceinline__ uint32_t wots_digit(const uint32_t* msg_w, int chain) {
  using Pr = P<S>;
  // base_w / checksum (wots.py:16-39); lg_w = 4, len2 = 3 for every set
  static_assert(Pr::lg_w == 4 && Pr::len2 == 3, "digit extraction assumes w = 16");
  if (chain < Pr::len1) return (msg_w[chain >> 3] >> (28 - 4 * (chain & 7))) & 15u;
  uint32_t csum = 0;
#pragma unroll
  for (int i = 0; i < Pr::len1; i++) csum += 15u - ((msg_w[i >> 3] >> (28 - 4 * (i & 7))) & 15u);
  csum <<= (8 - ((Pr::len2 * Pr::lg_w) % 8)) % 8;  // now a 16-bit big-endian value
  const int c = chain - Pr::len1;                  // 0..2
  return (csum >> (12 - 4 * c)) & 15u;
}

// ctr[msg] += v over the calling threads, one atomic per distinct msg in the
// warp (threads of a message are contiguous in the WOTS grids).
__device__ __forceinline__ void add_per_message(uint32_t* ctr, uint32_t msg, uint32_t v) {
  const unsigned active = __activemask();
  const unsigned peers = __match_any_sync(active, msg);
  const uint32_t sum = __reduce_add_sync(peers, v);
  if ((int)(threadIdx.x & 31u) == __ffs(peers) - 1) atomicAdd(ctr + msg, sum);
}

template <int S, class V>
__global__ void __launch_bounds__(kSmallBlock) wots_sign_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  const uint64_t per_msg = (uint64_t)Pr::d * Pr::wots_len;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (uint64_t)a.count * per_msg) return;
  const uint32_t msg = (uint32_t)(gid / per_msg);
  const uint32_t rem = (uint32_t)(gid % per_msg);
  const int layer = (int)(rem / Pr::wots_len);
  const int chain = (int)(rem % Pr::wots_len);
  const MsgPlan pl = a.plans[msg];
  const KeyDev& K = a.keys[pl.key];
  uint64_t tree;
  uint32_t leaf;
  layer_coords<S>(pl, layer, tree, leaf);
  uint32_t mw[8];
  const uint32_t* r = a.roots + ((size_t)msg * (Pr::d + 1) + layer) * 8;
#pragma unroll
  for (int j = 0; j < NW; j++) mw[j] = r[j];
  const uint32_t digit = wots_digit<S>(mw, chain);
  uint32_t mid[8], sks[NW];
#pragma unroll
  for (int j = 0; j < 8; j++) mid[j] = K.thash_mid[j];
#pragma unroll
  for (int j = 0; j < NW; j++) sks[j] = K.sk_seed[j];
  Adrs wa = make_adrs((uint32_t)layer, tree, ADDR_WOTS, leaf, (uint32_t)chain, 0);
  uint32_t st[8];
  prf_keyed<V, NW>(st, K.prf_mid, sks, wa);
  uint32_t x[NW];
#pragma unroll
  for (int j = 0; j < NW; j++) x[j] = st[j];
  chain_F<V, NW>(x, mid, wa, 0u, digit);
  store_node<NW>(a.sigs + (size_t)msg * Pr::sig_bytes + Pr::off_ht + (size_t)layer * Pr::layer_bytes + chain * Pr::n,
                 x);
  if (a.wots_steps) add_per_message(a.wots_steps, msg, digit);
}

// WOTS+_Sign as a gather: TREE_Sign already walked every chain of each
// layer's signing leaf (wots_gen_leaf computes the same values wots_sign
// needs, wots.py:85-95 vs :119-143), so the signature chain i of layer l is
// the recorded node at position digit_i.  Thread = (message, layer, chain).
template <int S>
__global__ void __launch_bounds__(kSmallBlock) wots_gather_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  const uint64_t per_msg = (uint64_t)Pr::d * Pr::wots_len;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (uint64_t)a.count * per_msg) return;
  const uint32_t msg = (uint32_t)(gid / per_msg);
  const uint32_t rem = (uint32_t)(gid % per_msg);
  const int layer = (int)(rem / Pr::wots_len);
  const int chain = (int)(rem % Pr::wots_len);
  using Sh = Shared<S>;
  const int first_shared = Pr::d - a.shared_layers;
  const MsgPlan pl = a.plans[msg];
  uint64_t tree;
  uint32_t leaf;
  layer_coords<S>(pl, layer, tree, leaf);
  // the value this layer signs: the FORS pk, or the root of the layer below
  const uint32_t* r;
  if (layer > first_shared) {
    uint64_t tb;
    uint32_t lb;
    layer_coords<S>(pl, layer - 1, tb, lb);
    r = Sh::rec(a, pl.key, layer - 1, tb) + (size_t)Sh::level_off(Pr::hp) * 8;
  } else {
    r = a.roots + ((size_t)msg * (Pr::d + 1) + layer) * 8;
  }
  uint32_t mw[8];
#pragma unroll
  for (int j = 0; j < NW; j++) mw[j] = r[j];
  const uint32_t digit = wots_digit<S>(mw, chain);
  uint8_t* lsig = a.sigs + (size_t)msg * Pr::sig_bytes + Pr::off_ht + (size_t)layer * Pr::layer_bytes;
  const uint32_t* src;
  if (layer >= first_shared) {
    const uint32_t* R = Sh::rec(a, pl.key, layer, tree);
    src = R + Sh::node_words + (size_t)leaf * Sh::leaf_stash_words + ((size_t)chain * Pr::w + digit) * NW;
    if (chain < Pr::hp) {  // auth node of level `chain` (vexec.py:529-532)
      const uint32_t* sib = R + (size_t)(Sh::level_off(chain) + ((leaf >> chain) ^ 1u)) * 8;
      uint32_t y[NW];
#pragma unroll
      for (int j = 0; j < NW; j++) y[j] = sib[j];
      store_node<NW>(lsig + Pr::wots_sig_bytes + chain * Pr::n, y);
    }
  } else {
    src = a.stash + ((((size_t)msg * Pr::d + layer) * Pr::wots_len + chain) * Pr::w + digit) * NW;
  }
  uint32_t x[NW];
#pragma unroll
  for (int j = 0; j < NW; j++) x[j] = src[j];
  store_node<NW>(lsig + chain * Pr::n, x);
  if (a.wots_steps) add_per_message(a.wots_steps, msg, digit);
}

// ---------------------------------------------------------------------------
// keygen: root of the top subtree (layer d-1, tree 0) per key.  Thread =
// (key, leaf); same leaf routine and shuffle reduction as TREE_Sign.
// a.sk_bytes holds seed || 0^n per key (4n stride); a.keys the setup records.
// ---------------------------------------------------------------------------
template <int S, class V>
__global__ void __launch_bounds__(kTreeBlock) keygen_root_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  __shared__ uint32_t tbuf[kLeafColumnWords * kTreeBlock];
  const uint64_t gid = (uint64_t)blockIdx.x * kTreeBlock + threadIdx.x;
  const bool valid = gid < (uint64_t)a.nkeys * Pr::leaves;
  const uint32_t key = valid ? (uint32_t)(gid / Pr::leaves) : 0u;
  const uint32_t leaf = (uint32_t)(gid % Pr::leaves);
  const uint32_t layer = Pr::d - 1;
  uint32_t node[8];
  const KeyDev& K = a.keys[key];
  if (valid) wots_leaf<S, V>(K, layer, 0ull, leaf, &tbuf[threadIdx.x], kTreeBlock, node);
#pragma unroll 1
  for (int lvl = 1; lvl <= Pr::hp; lvl++) {
    uint32_t other[NW];
#pragma unroll
    for (int j = 0; j < NW; j++) other[j] = __shfl_down_sync(0xffffffffu, node[j], 1u << (lvl - 1));
    if (valid && (leaf & ((1u << lvl) - 1u)) == 0u) {
      uint32_t m[2 * NW], mid[8];
#pragma unroll
      for (int j = 0; j < NW; j++) { m[j] = node[j]; m[NW + j] = other[j]; }
#pragma unroll
      for (int j = 0; j < 8; j++) mid[j] = K.thash_mid[j];
      thash_reg<V, 2 * NW>(node, mid, make_adrs(layer, 0ull, ADDR_HASHTREE, 0, (uint32_t)lvl, leaf >> lvl), m);
    }
  }
  if (valid && leaf == 0) {
    uint8_t* sk = a.sk_out + (size_t)key * Pr::sk_bytes;
    for (int j = 0; j < 3 * Pr::n; j++) sk[j] = a.sk_bytes[(size_t)key * Pr::sk_bytes + j];
    store_node<NW>(sk + 3 * Pr::n, node);
  }
}

// ---------------------------------------------------------------------------
// Batched verification: one warp per message (sigcore.py:181-221,
// fors_pk_from_sig oracle.py:149-178, wots_pk_from_sig wots.py:98-116,
// compute_root oracle.py:66-95).  FORS trees and WOTS chains spread over the
// lanes; the serial T_k / T_len / auth-path walks run on lane 0.
// ---------------------------------------------------------------------------

template <int S>
__device__ __forceinline__ void load_node(const uint8_t* p, uint32_t* x) {
#pragma unroll
  for (int j = 0; j < P<S>::NW; j++) x[j] = bswap32(*reinterpret_cast<const uint32_t*>(p + 4 * j));
}

// compute_root (oracle.py:66-95) for a node at leaf_idx within a forest offset
template <int S, class V>
__device__ __forceinline__ void walk_auth(uint32_t node[8], const uint32_t mid[8], Adrs a, uint32_t li, uint32_t off,
                                          const uint8_t* auth, int height) {
  constexpr int NW = P<S>::NW;
#pragma unroll 1
  for (int i = 0; i < height; i++) {
    uint32_t sib[NW], m[2 * NW];
    load_node<S>(auth + i * P<S>::n, sib);
    const bool odd = li & 1u;
#pragma unroll
    for (int j = 0; j < NW; j++) {
      m[j] = odd ? sib[j] : node[j];
      m[NW + j] = odd ? node[j] : sib[j];
    }
    li >>= 1;
    off >>= 1;
    adrs_set_chain_hash(a, (uint32_t)(i + 1), li + off);
    thash_reg<V, 2 * NW>(node, mid, a, m);
  }
}

// ---------------------------------------------------------------------------
// verify_thread_kernel: one thread per signature (sigcore.py:181-221).  A
// warp-per-message kernel (round-1 first version) left 31 lanes idle through
// every T_len and auth walk and ran 35-67 chains of unequal length on 32
// lanes (1.8-2.4x slower, profiles/r01f_stress_verify_thread.txt); here each
// thread walks its own signature and the wots_len chains of a layer as ONE
// flattened loop of F steps (sum of 15 - digit over the chains, nearly the
// same count for every thread), so lanes stay busy.  Each chain end goes to
// a thread-local array and T_len runs after the loop, every lane compressing
// block b at the same time: streaming the ends into T_len as chains completed
// ran each T_len block inside the divergent chain-completion branch, where
// the warp executed it ~17x per useful lane-block (ncu: a full compression
// executed 7.8M times next to the F step's 14.8M, profiles/r02ak_*).
// ---------------------------------------------------------------------------
#ifndef HS_VERIFY_THREADS
#define HS_VERIFY_THREADS 128
#endif
constexpr int kVerifyThreads = HS_VERIFY_THREADS;

template <int S, class V>
__global__ void __launch_bounds__(kVerifyThreads) verify_thread_kernel(LaunchArgs a) {
  using Pr = P<S>;
  constexpr int NW = Pr::NW;
  __shared__ uint32_t col[32 * kVerifyThreads];  // per-thread T stream ring (word-interleaved)
  const uint32_t i = blockIdx.x * kVerifyThreads + threadIdx.x;
  if (i >= a.count) return;
  uint32_t* mycol = col + threadIdx.x;
  const uint8_t* pk = a.pks;
  if (a.key_idx) pk += (size_t)a.key_idx[i] * 2 * Pr::n;
  const uint8_t* sig = a.vsigs + (size_t)i * Pr::sig_bytes;
  uint32_t pk_seed[8], pk_root[8], mid[8];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    pk_seed[j] = j < NW ? load_be(pk + 4 * j) : 0u;
    pk_root[j] = j < NW ? load_be(pk + Pr::n + 4 * j) : 0u;
  }
  {
    uint32_t W[16];
#pragma unroll
    for (int j = 0; j < 8; j++) mid[j] = IVc(j);
#pragma unroll
    for (int j = 0; j < 16; j++) W[j] = j < NW ? pk_seed[j] : 0u;
    compress<V>(mid, W);
  }
  // H_msg with R = sig[0:n] (hashes.py:175-191), word-level as msg_prep
  uint32_t R[8], dig0[8];
#pragma unroll
  for (int j = 0; j < 8; j++) R[j] = j < NW ? load_be(sig + 4 * j) : 0u;
  const uint8_t* msg = a.msgs + a.offs[i];
  const uint64_t mlen = a.offs[i + 1] - a.offs[i];
  {
    uint32_t pre[3 * NW];
#pragma unroll
    for (int j = 0; j < NW; j++) { pre[j] = R[j]; pre[NW + j] = pk_seed[j]; pre[2 * NW + j] = pk_root[j]; }
#pragma unroll
    for (int j = 0; j < 8; j++) dig0[j] = IVc(j);
    sha_prefix_msg<V, 3 * NW, false>(dig0, 0, pre, msg, mlen);
  }
  uint8_t dg[64];
  constexpr int nctr = (Pr::digest_bytes + 31) / 32;
#pragma unroll 1
  for (int c = 0; c < nctr; c++) {
    uint32_t pre[2 * NW + 9], o[8];
#pragma unroll
    for (int j = 0; j < NW; j++) { pre[j] = R[j]; pre[NW + j] = pk_seed[j]; }
#pragma unroll
    for (int j = 0; j < 8; j++) { pre[2 * NW + j] = dig0[j]; o[j] = IVc(j); }
    pre[2 * NW + 8] = (uint32_t)c;
    sha_prefix_msg<V, 2 * NW + 9, false>(o, 0, pre, msg, 0);
    for (int j = 0; j < 32; j++) dg[32 * c + j] = (uint8_t)(o[j >> 2] >> (24 - 8 * (j & 3)));
  }
  uint64_t tree = 0;
  for (int j = 0; j < Pr::tree_bytes; j++) tree = (tree << 8) | dg[Pr::fors_msg_bytes + j];
  if (Pr::tree_bits < 64) tree &= (1ull << (Pr::tree_bits < 64 ? Pr::tree_bits : 63)) - 1ull;
  uint32_t leaf_idx = 0;
  for (int j = 0; j < Pr::leaf_bytes; j++) leaf_idx = (leaf_idx << 8) | dg[Pr::fors_msg_bytes + Pr::tree_bytes + j];
  leaf_idx &= (1u << Pr::leaf_bits) - 1u;

  // FORS public key (oracle.py:113-146 in reverse): k roots streamed into T_k
  uint32_t root[8];
  {
    const uint8_t* fsig = sig + Pr::off_fors;
    constexpr int tree_sig = (1 + Pr::log_t) * Pr::n;
    TStream<V> ts;
    ts.begin(mid, make_adrs(0, tree, ADDR_FORS_ROOTS, leaf_idx, 0, 0), mycol, kVerifyThreads);
    int off = 0;
#pragma unroll 1
    for (int g = 0; g < Pr::k; g++) {
      uint32_t sel = 0;
      for (int j = 0; j < Pr::log_t; j++, off++) sel |= (uint32_t)((dg[off >> 3] >> (off & 7)) & 1) << j;
      const Adrs fa = make_adrs(0, tree, ADDR_FORS_TREE, leaf_idx, 0, (uint32_t)(g * Pr::t) + sel);
      uint32_t sk[NW], node[8];
      load_node<S>(fsig + g * tree_sig, sk);
      thash_reg<V, NW>(node, mid, fa, sk);
      walk_auth<S, V>(node, mid, fa, sel, (uint32_t)(g * Pr::t), fsig + g * tree_sig + Pr::n, Pr::log_t);
      ts.template push_node<NW>(node);
    }
    ts.finish(22u + (uint32_t)(Pr::k * Pr::n));
#pragma unroll
    for (int j = 0; j < 8; j++) root[j] = ts.st[j];
  }

  // hypertree: per layer, the wots_len chains as one flattened loop of F steps
  const uint8_t* ht = sig + Pr::off_ht;
  constexpr int M = Pr::wots_len * NW;
  uint32_t ends[M];  // this layer's chain ends (thread-local; T_len reads them after the loop)
#pragma unroll 1
  for (int layer = 0; layer < Pr::d; layer++) {
    const uint8_t* wsig = ht + (size_t)layer * Pr::layer_bytes;
    Adrs wa = make_adrs((uint32_t)layer, tree, ADDR_WOTS, leaf_idx, 0, 0);
    uint32_t x[NW], pre5[8];
    int c = -1;
    uint32_t s = Pr::w - 1;  // current hash index; == w-1 means "chain done"
#pragma unroll 1
    while (true) {
      // finish completed chains (a digit of 15 gives a zero-length chain)
      while (s == (uint32_t)(Pr::w - 1)) {
        if (c >= 0) {
#pragma unroll
          for (int j = 0; j < NW; j++) ends[c * NW + j] = x[j];
        }
        if (++c >= Pr::wots_len) break;
        load_node<S>(wsig + c * Pr::n, x);
        s = wots_digit<S>(root, c);
        adrs_set_chain_hash(wa, (uint32_t)c, 0);
        const uint32_t W04[5] = {wa.w0, wa.w1, wa.w2, wa.w3, wa.w4};
#pragma unroll
        for (int j = 0; j < 8; j++) pre5[j] = mid[j];
        rounds_prefix<V, 5>(pre5, W04);  // chain-invariant rounds 0-4 (as chain_F)
      }
      if (c >= Pr::wots_len) break;
      uint32_t W[16];
      W[0] = wa.w0; W[1] = wa.w1; W[2] = wa.w2; W[3] = wa.w3; W[4] = wa.w4;
      W[5] = join16(s, x[0]);
#pragma unroll
      for (int j = 1; j < NW; j++) W[5 + j] = join16(x[j - 1], x[j]);
      W[5 + NW] = (x[NW - 1] << 16) | 0x8000u;
#pragma unroll
      for (int j = 6 + NW; j < 15; j++) W[j] = 0;
      W[15] = (uint32_t)((64 + 22 + 4 * NW) * 8);
      uint32_t st[8];
#pragma unroll
      for (int j = 0; j < 8; j++) st[j] = mid[j];
      compress_resume<V, 5>(st, pre5, W);
#pragma unroll
      for (int j = 0; j < NW; j++) x[j] = st[j];
      s++;
    }
    // T_len over the chain ends, every lane on block b together (wots.py:140-143)
    uint32_t node[8];
    {
      constexpr uint32_t total = 22u + (uint32_t)(Pr::wots_len * Pr::n);
      constexpr uint32_t nblk = (total + 9u + 63u) / 64u;
      const Adrs pa = make_adrs((uint32_t)layer, tree, ADDR_WOTS_PK, leaf_idx, 0, 0);
      const uint32_t aw[6] = {pa.w0, pa.w1, pa.w2, pa.w3, pa.w4, pa.h5};
#pragma unroll
      for (int j = 0; j < 8; j++) node[j] = mid[j];
#pragma unroll 1
      for (uint32_t b = 0; b < nblk; b++) {
        uint32_t W[16];
#pragma unroll
        for (int j = 0; j < 16; j++) W[j] = tlen_word<M>(16u * b + j, aw, ends, (64u + total) * 8u, 16u * nblk - 1u);
        compress<V>(node, W);
      }
    }
    walk_auth<S, V>(node, mid, make_adrs((uint32_t)layer, tree, ADDR_HASHTREE, 0, 0, 0), leaf_idx, 0,
                    wsig + Pr::wots_sig_bytes, Pr::hp);
#pragma unroll
    for (int j = 0; j < 8; j++) root[j] = node[j];
    leaf_idx = (uint32_t)(tree & (uint64_t)(Pr::leaves - 1));
    tree = shr64(tree, Pr::hp);
  }
  bool eq = true;
#pragma unroll
  for (int j = 0; j < NW; j++) eq = eq && (root[j] == pk_root[j]);
  a.ok[i] = eq ? 1 : 0;
}

}  // namespace hs
