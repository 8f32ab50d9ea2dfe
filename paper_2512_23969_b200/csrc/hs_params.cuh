// hs_params.cuh -- compile-time SPHINCS+-{128f,192f,256f} constants.
//
// Restates params.py:31-35 (the table) and params.py:97-149 (derive) of the
// reference as constexpr so every size, loop bound and signature offset folds
// into the kernels.  Set ids: 0 = 128f, 1 = 192f, 2 = 256f.
#pragma once
#include <cstdint>

namespace hs {

constexpr int kMaxN = 32;

template <int S> struct SetBase;
template <> struct SetBase<0> { static constexpr int n = 16, h = 66, d = 22, log_t = 6, k = 33, w = 16; };
template <> struct SetBase<1> { static constexpr int n = 24, h = 66, d = 22, log_t = 8, k = 33, w = 16; };
template <> struct SetBase<2> { static constexpr int n = 32, h = 68, d = 17, log_t = 9, k = 35, w = 16; };

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }
constexpr int len2_of(int len1, int w) {  // params.py:77-83
  long cap = (long)len1 * (w - 1), pw = w;
  int e = 0;
  while (pw <= cap) { e++; pw *= w; }
  return e + 1;
}
constexpr int blocks_of(int total_len) { return (total_len + 72) / 64; }  // hashes.py:39-41

template <int S> struct P : SetBase<S> {
  using B = SetBase<S>;
  static constexpr int set = S;
  static constexpr int n = B::n, h = B::h, d = B::d, log_t = B::log_t, k = B::k, w = B::w;
  static constexpr int NW = n / 4;                       // node words
  static constexpr int lg_w = ilog2(w);
  static constexpr int len1 = (8 * n + lg_w - 1) / lg_w;
  static constexpr int len2 = len2_of(len1, w);
  static constexpr int wots_len = len1 + len2;
  static constexpr int hp = h / d;                       // subtree height
  static constexpr int leaves = 1 << hp;                 // leaves per subtree
  static constexpr int t = 1 << log_t;                   // FORS leaves per tree
  static constexpr int fors_msg_bytes = (k * log_t + 7) / 8;
  static constexpr int tree_bits = hp * (d - 1);
  static constexpr int tree_bytes = (tree_bits + 7) / 8;
  static constexpr int leaf_bits = hp;
  static constexpr int leaf_bytes = (leaf_bits + 7) / 8;
  static constexpr int digest_bytes = fors_msg_bytes + tree_bytes + leaf_bytes;
  static constexpr int wots_sig_bytes = wots_len * n;
  static constexpr int fors_sig_bytes = k * (1 + log_t) * n;
  static constexpr int layer_bytes = wots_sig_bytes + hp * n;
  static constexpr int ht_sig_bytes = d * layer_bytes;
  static constexpr int sig_bytes = n + fors_sig_bytes + ht_sig_bytes;
  static constexpr int sk_bytes = 4 * n;
  // signature regions (sigcore.py:124-136)
  static constexpr int off_fors = n;
  static constexpr int off_ht = n + fors_sig_bytes;
  // tweakable-hash block counts after the PK.seed midstate (Appendix A)
  static constexpr int f_blocks = blocks_of(64 + 22 + n) - 1;
  static constexpr int h_blocks = blocks_of(64 + 22 + 2 * n) - 1;
  static constexpr int tlen_blocks = blocks_of(64 + 22 + wots_len * n) - 1;
  static constexpr int tk_blocks = blocks_of(64 + 22 + k * n) - 1;
};

// address types (address.py:21-25)
enum : uint32_t { ADDR_WOTS = 0, ADDR_WOTS_PK = 1, ADDR_HASHTREE = 2, ADDR_FORS_TREE = 3, ADDR_FORS_ROOTS = 4 };

}  // namespace hs
