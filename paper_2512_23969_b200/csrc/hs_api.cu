// hs_api.cu -- host runtime behind the C-ABI (include/herosign_b200.h).
//
// Owns device buffers, the two streams (FORS branch / main branch) and one
// CUDA graph per batch shape: msg_prep -> {FORS_Sign -> T_k} || TREE_Sign ->
// WOTS_Sign, launched with a single cudaGraphLaunch per batch (the paper's
// Task Graph; reference batchgraph.py:76-226 runs the same
// DAG on CPU threads).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/herosign_b200.h"
#include "hs_internal.h"
#include "hs_kernels.cuh"

using namespace hs;

namespace {

struct SetInfo {
  int n, h, d, log_t, k, w, lg_w, len1, len2, wots_len, hp, leaves, t, fors_msg_bytes, tree_bits, tree_bytes,
      leaf_bits, leaf_bytes, digest_bytes, wots_sig_bytes, fors_sig_bytes, ht_sig_bytes, sig_bytes;
};

template <int S>
SetInfo info_of() {
  using Pr = P<S>;
  return SetInfo{Pr::n, Pr::h, Pr::d, Pr::log_t, Pr::k, Pr::w, Pr::lg_w, Pr::len1, Pr::len2, Pr::wots_len,
                 Pr::hp, Pr::leaves, Pr::t, Pr::fors_msg_bytes, Pr::tree_bits, Pr::tree_bytes, Pr::leaf_bits,
                 Pr::leaf_bytes, Pr::digest_bytes, Pr::wots_sig_bytes, Pr::fors_sig_bytes, Pr::ht_sig_bytes,
                 Pr::sig_bytes};
}

const SetInfo kInfo[3] = {info_of<0>(), info_of<1>(), info_of<2>()};

cudaError_t launch(int set, int which, int variant, const LaunchArgs& a, cudaStream_t s) {
  switch (set) {
    case 0: return launch_kernel<0>(which, variant, a, s);
    case 1: return launch_kernel<1>(which, variant, a, s);
    case 2: return launch_kernel<2>(which, variant, a, s);
  }
  return cudaErrorInvalidValue;
}

size_t shared_words(int set, int layers) {
  switch (set) {
    case 0: return shared_words_per_key<0>(layers);
    case 1: return shared_words_per_key<1>(layers);
    case 2: return shared_words_per_key<2>(layers);
  }
  return 0;
}

size_t shared_end_words(int set, int layers) {
  switch (set) {
    case 0: return shared_end_words_per_key<0>(layers);
    case 1: return shared_end_words_per_key<1>(layers);
    case 2: return shared_end_words_per_key<2>(layers);
  }
  return 0;
}

// shared subtrees per key for `layers` top layers: sum_{j<layers} 2^(hp*j)
size_t shared_units_of(int set, int layers) {
  size_t u = 0;
  for (int j = 0; j < layers; j++) u += (size_t)1 << (kInfo[set].hp * j);
  return u;
}

// key_used flags (nkeys) followed by per-key flags of every shared subtree
size_t used_flag_bytes(int set, uint32_t nkeys, int layers) {
  return (size_t)nkeys * (1 + shared_units_of(set, layers));
}

int shared_max(int set) {
  switch (set) {
    case 0: return shared_max_layers<0>();
    case 1: return shared_max_layers<1>();
    case 2: return shared_max_layers<2>();
  }
  return 0;
}

size_t stash_words(int set) {
  switch (set) {
    case 0: return stash_words_per_msg<0>();
    case 1: return stash_words_per_msg<1>();
    case 2: return stash_words_per_msg<2>();
  }
  return 0;
}

size_t fors_smem(int set, int nt, int f, int relax) {
  switch (set) {
    case 0: return fors_smem_bytes<0>(nt, f, relax);
    case 1: return fors_smem_bytes<1>(nt, f, relax);
    case 2: return fors_smem_bytes<2>(nt, f, relax);
  }
  return 0;
}

hs_set_config default_config(int set) {
  hs_set_config c;
  std::memset(&c, 0, sizeof c);
  // Defaults from the on-device Tree Tuning search (python tuner); see DESIGN.md.
  // (b200_tuned.json, written by tools/tune_all.py on a B200, overrides these.)
  static const int nt[3] = {11, 3, 3}, ff[3] = {3, 8, 6}, rx[3] = {0, 0, 1};
  static const int var[3][4] = {{1, 1, 0, 0}, {0, 1, 0, 0}, {0, 0, 0, 0}};
  c.fors_trees_per_set = nt[set];
  c.fors_sets_fused = ff[set];
  c.fors_relax = rx[set];
  for (int i = 0; i < 4; i++) c.variant[i] = var[set][i];
  c.use_graph = 1;
  c.chunk = 16384;
  c.wots_from_tree = 1;
  c.streams = 2;
  c.shared_layers = shared_max(set);
  c.shared_auto = 1;
  c.fors_cta_levels = -1;
  c.tree_split = 2;
  // streams for graphs of at most this many messages (1 = always): measured
  // crossover on B200, profiles/r02y_overlap_crossover.txt
  static const int ov[3] = {1, 1536, 8192}, fsmall[3] = {64, 64, 16}, tsmall[3] = {64, 16, 16};
  c.overlap = ov[set];
  c.fors_small_batch = fsmall[set];
  c.tree_small_batch = tsmall[set];
  return c;
}

template <class T>
cudaError_t grow(T*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  size_t c = std::max(need, (size_t)1);
  cudaError_t e = cudaMalloc(&p, c * sizeof(T));
  cap = e == cudaSuccess ? c : 0;
  return e;
}

template <class T>
cudaError_t grow_host(T*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return cudaSuccess;
  if (p) cudaFreeHost(p);
  p = nullptr;
  size_t c = std::max(need, (size_t)1);
  cudaError_t e = cudaMallocHost(&p, c * sizeof(T));
  cap = e == cudaSuccess ? c : 0;
  return e;
}

// Per-chunk inputs and outputs, double-buffered: hs_sign_batch stages chunk
// c+1 (host copy + H2D on the copy stream) and drains chunk c's signatures
// (D2H on the copy-out streams) while chunk c+1 computes.
constexpr int kSlots = 2;
struct Slot {
  uint8_t* msgs = nullptr; size_t msgs_cap = 0;
  uint64_t* offs = nullptr; size_t offs_cap = 0;
  uint32_t* keyidx = nullptr; size_t keyidx_cap = 0;
  uint8_t* optrand = nullptr; size_t optrand_cap = 0;
  uint8_t* sigs = nullptr; size_t sigs_cap = 0;
  uint32_t* wsteps = nullptr; size_t wsteps_cap = 0;  // WOTS_Sign F steps per message
  // pinned staging
  uint8_t* h_msgs = nullptr; size_t h_msgs_cap = 0;
  uint64_t* h_offs = nullptr; size_t h_offs_cap = 0;
  uint8_t* h_sigs = nullptr; size_t h_sigs_cap = 0;
  uint32_t* h_wsteps = nullptr; size_t h_wsteps_cap = 0;
};

struct Buffers {
  Slot io[kSlots];
  MsgPlan* plans = nullptr; size_t plans_cap = 0;
  uint16_t* idx = nullptr; size_t idx_cap = 0;
  uint32_t* roots = nullptr; size_t roots_cap = 0;
  uint32_t* froots = nullptr; size_t froots_cap = 0;
  uint32_t* stash = nullptr; size_t stash_cap = 0;
  uint32_t* shared = nullptr; size_t shared_cap = 0;   // subtree-sharing table
  uint8_t* key_used = nullptr; size_t key_used_cap = 0;
  uint32_t* fnodes[2] = {nullptr, nullptr}; size_t fnodes_cap[2] = {0, 0};  // upper FORS levels
  uint32_t* ends = nullptr; size_t ends_cap = 0;  // split TREE_Sign chain ends
  uint32_t* sends = nullptr; size_t sends_cap = 0;  // split shared-subtree chain ends
  uint32_t* lpre = nullptr; size_t lpre_cap = 0;    // per-message, per-FORS-level H prefix states
  // verification inputs (hs_verify_batch), kept across calls
  uint8_t* v_pks = nullptr; size_t v_pks_cap = 0;
  uint8_t* v_msgs = nullptr; size_t v_msgs_cap = 0;
  uint8_t* v_sigs = nullptr; size_t v_sigs_cap = 0;
  uint8_t* v_ok = nullptr; size_t v_ok_cap = 0;
  uint64_t* v_offs = nullptr; size_t v_offs_cap = 0;
  uint32_t* v_kidx = nullptr; size_t v_kidx_cap = 0;
  uint64_t gen = 0;  // bumps whenever a device pointer changes (graph invalidation)
};

struct SetState {
  hs_set_config cfg;
  KeyDev* keys = nullptr;
  size_t keys_cap = 0;
  uint32_t nkeys = 0;
  uint8_t* sk_raw = nullptr;
  size_t sk_raw_cap = 0;
  // staged batch (in io slot `slot`)
  int slot = 0;
  uint32_t staged = 0;
  bool has_keyidx = false, has_optrand = false;
  int shared_eff = 0;  // subtree-sharing depth chosen for the staged batch
};

using GraphKey = std::tuple<int, uint32_t, int, int, uint64_t, std::string>;

constexpr int kMaxStreams = 8;
constexpr size_t kMaxGraphs = 64;  // captured batch graphs kept per handle
constexpr size_t kSharedBudgetBytes = (size_t)8 << 30;  // shared-subtree table cap

}  // namespace

struct hs_ctx {
  int device = 0;
  cudaStream_t s0 = nullptr, s1 = nullptr;
  cudaEvent_t ev[8] = {};     // timing: 0 start,1 prep,2 fors-done,3 tree-done,4 end,5 wots-start
  cudaEvent_t fork = nullptr, join = nullptr;
  SetState sets[3];
  Buffers buf[3];
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, int> graph_kernels;
  int last_kernels = 5;
  std::string err;
  int64_t launches = 0;
  int last_set = -1;
  int last_mode = 0;
  int sm_count = 0, smem_optin = 0, cc_major = 0, cc_minor = 0;
  void* flush = nullptr;
  size_t flush_cap = 0;
  cudaStream_t ls[kMaxStreams] = {};   // D2H copy streams (one per sub-batch)
  cudaStream_t cs = nullptr;           // H2D copy stream (chunk staging)
  cudaStream_t q[2 * kMaxStreams + 1] = {};  // compute streams, descending priority
  // per io slot: its inputs landed (cs), the batch reading them finished (s0),
  // sub-batch j's signatures copied out (ls[j])
  cudaEvent_t h2d_done[kSlots] = {}, compute_done[kSlots] = {}, d2h_done[kSlots][kMaxStreams] = {};
  // copy-out streams whose d2h_done[slot][j] was recorded since s0 last waited on
  // that slot's copies (only those are waited on: a 1-message call does not pay
  // for kMaxStreams event waits and stream syncs)
  int slot_T[kSlots] = {};
  cudaEvent_t done[kMaxStreams] = {}, joins[kMaxStreams] = {}, fjoin[kMaxStreams] = {}, sh_done = nullptr;
  int last_T = 1;
  // host-side cost of each cudaGraphLaunch since the last hs_launch_stats reset
  // (the "batch launch latency" of BASELINE.json's metric): count, sum, max us
  int64_t glaunch_n = 0;
  double glaunch_us_sum = 0.0, glaunch_us_max = 0.0;
};

namespace {

int fail(hs_t* h, int code, const char* fmt, ...) {
  char b[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(b, sizeof b, fmt, ap);
  va_end(ap);
  if (h) h->err = b;
  return code;
}

#define CUDA_TRY(h, expr)                                                                     \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) return fail((h), HS_E_CUDA, "%s: %s (%s:%d)", #expr,               \
                                       cudaGetErrorString(_e), __FILE__, __LINE__);           \
  } while (0)

bool valid_set(int set) { return set >= 0 && set <= 2; }

// Every field of the set's config (all int32): a captured graph is reused only
// for an identical config.
std::string cfg_fingerprint(const hs_set_config& c) {
  static_assert(sizeof(hs_set_config) % sizeof(int32_t) == 0, "hs_set_config must be all int32 fields");
  int32_t f[sizeof(hs_set_config) / sizeof(int32_t)];
  std::memcpy(f, &c, sizeof f);
  std::string out;
  for (int32_t v : f) out += std::to_string(v) + "/";
  return out;
}

void drop_graphs(hs_t* h) {
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
  h->graph_kernels.clear();
}

int check_layout(hs_t* h, int set, const hs_set_config& c) {
  const SetInfo& I = kInfo[set];
  if (c.fors_trees_per_set < 1 || c.fors_sets_fused < 1)
    return fail(h, HS_E_CONFIG, "fusion counts must be positive");
  const int lanes = c.fors_trees_per_set * (c.fors_relax ? I.t / 2 : I.t);
  if (lanes > kForsMaxLanes)
    return fail(h, HS_E_CONFIG, "layout needs %d lanes; FORS_Sign blocks hold at most %d", lanes, kForsMaxLanes);
  if (c.fors_trees_per_set * c.fors_sets_fused > I.k)
    return fail(h, HS_E_CONFIG, "layout holds more than k=%d trees per CTA", I.k);
  size_t smem = fors_smem(set, c.fors_trees_per_set, c.fors_sets_fused, c.fors_relax);
  if (h && smem > (size_t)h->smem_optin)
    return fail(h, HS_E_CONFIG, "layout needs %zu shared bytes; device opt-in limit is %d", smem, h->smem_optin);
  for (int i = 0; i < 4; i++)
    if (c.variant[i] < 0 || c.variant[i] >= hs::kVariants)
      return fail(h, HS_E_CONFIG, "variant must be in 0..%d", hs::kVariants - 1);
  if (c.chunk < 1) return fail(h, HS_E_CONFIG, "chunk must be >= 1");
  if (c.wots_from_tree != 0 && c.wots_from_tree != 1) return fail(h, HS_E_CONFIG, "wots_from_tree must be 0 or 1");
  if (c.streams < 1 || c.streams > kMaxStreams) return fail(h, HS_E_CONFIG, "streams must be in 1..%d", kMaxStreams);
  if (c.shared_layers < 0 || c.shared_layers > shared_max(set))
    return fail(h, HS_E_CONFIG, "shared_layers must be in 0..%d for this set", shared_max(set));
  if (c.shared_auto != 0 && c.shared_auto != 1) return fail(h, HS_E_CONFIG, "shared_auto must be 0 or 1");
  if (c.tree_split < 0 || c.tree_split > 2) return fail(h, HS_E_CONFIG, "tree_split must be 0, 1 or 2");
  if (c.overlap < 0) return fail(h, HS_E_CONFIG, "overlap must be 0, 1 or a message count >= 2");
  if (c.fors_small_batch < 0 || c.tree_small_batch < 0)
    return fail(h, HS_E_CONFIG, "fors_small_batch / tree_small_batch must be >= 0");
  if (c.fors_cta_levels < -1 || c.fors_cta_levels > I.log_t)
    return fail(h, HS_E_CONFIG, "fors_cta_levels must be -1 (auto) or in 0..%d", I.log_t);
  return HS_OK;
}

// Messages one graph launch signs: a staged batch larger than cfg.chunk runs
// as consecutive launches of `chunk` messages over resident inputs, so the
// per-message work buffers (stash, chain ends, FORS levels, ...) are sized for
// one chunk and only the inputs and signatures for the whole batch.
uint32_t work_count(const hs_set_config& c, uint32_t count) {
  return std::min(count, (uint32_t)std::max(1, c.chunk));
}

int ensure_capacity(hs_t* h, int set, int slot, uint32_t count, size_t msg_bytes) {
  const SetInfo& I = kInfo[set];
  Buffers& B = h->buf[set];
  Slot& S = B.io[slot];
  void* before[6] = {S.msgs, S.offs, S.keyidx, S.optrand, S.sigs, S.wsteps};
  CUDA_TRY(h, grow(S.msgs, S.msgs_cap, std::max(msg_bytes, (size_t)1)));
  CUDA_TRY(h, grow(S.offs, S.offs_cap, (size_t)count + 1));
  CUDA_TRY(h, grow(S.keyidx, S.keyidx_cap, (size_t)count));
  CUDA_TRY(h, grow(S.optrand, S.optrand_cap, (size_t)count * I.n));
  CUDA_TRY(h, grow(S.sigs, S.sigs_cap, (size_t)count * I.sig_bytes));
  CUDA_TRY(h, grow(S.wsteps, S.wsteps_cap, (size_t)count));
  void* after[6] = {S.msgs, S.offs, S.keyidx, S.optrand, S.sigs, S.wsteps};
  if (std::memcmp(before, after, sizeof before) != 0) {
    B.gen++;
    drop_graphs(h);
  }
  return HS_OK;
}

// FORS levels kept inside FORS_Sign's CTA (the rest run as one-level grids):
// explicit 0..log_t (0: leaves only; with Relax the leaf phase already yields
// level 1, so 0 means 1), or auto (-1): the measured best on B200 for every
// tuned layout was to hand everything above the leaf phase to the grids
// (tools/fors_split.py, profiles/r01_fors_split.txt).
// (Keeping the whole tree in the CTA for small batches was measured slower,
// not faster: 1 message 124 -> 133 us, 64 messages 442 -> 519 us for 128f.)
int fors_cta_levels(int set, const hs_set_config& c, uint32_t count) {
  (void)count;
  const SetInfo& I = kInfo[set];
  const int lowest = c.fors_relax ? 1 : 0;
  if (c.fors_cta_levels < 0) return lowest;
  return std::max(lowest, std::min(c.fors_cta_levels, I.log_t));
}

// The execution shape of one batch graph of `count` messages: the set's
// config with the batch-size rules resolved.  Small graphs leave most SMs
// idle and are latency bound, so (a) FORS_Sign runs one tree per CTA (k CTAs
// per message instead of a few wide ones whose lanes walk several trees in
// passes), (b) the subtree Merkle levels are warp-shuffle combines (hp H's on
// the critical path, not leaves-1) and (c) the FORS / TREE / shared-subtree
// branches run concurrently; large graphs keep the tuned layout, the
// one-thread-per-subtree Merkle grid and, where concurrency measured slower
// (192f, 256f at 16,384), one stream order.  Bytes never depend on the shape.
// Thresholds: profiles/r02x_small_batch_overlap.txt, r02y_overlap_crossover.txt,
// r02aa_small_batch_tree_shape.txt.
hs_set_config batch_config(const hs_set_config& c, uint32_t count) {
  hs_set_config b = c;
  if (c.fors_small_batch > 0 && count <= (uint32_t)c.fors_small_batch) {
    b.fors_trees_per_set = 1;
    b.fors_sets_fused = 1;
  }
  if (c.tree_small_batch > 0 && count <= (uint32_t)c.tree_small_batch && c.tree_split == 2) b.tree_split = 1;
  b.overlap = (c.overlap == 1 || (c.overlap > 1 && count <= (uint32_t)c.overlap)) ? 1 : 0;
  return b;
}

// words of fors_nodes[b]: buffer 0 holds levels Lc, Lc+2, ..., buffer 1 Lc+1, ...
size_t fors_node_words(int set, const hs_set_config& c, uint32_t count, int b) {
  const SetInfo& I = kInfo[set];
  const int L = fors_cta_levels(set, c, count);
  return L >= I.log_t ? 0 : (size_t)count * I.k * ((size_t)I.t >> (L + b)) * (I.n / 4);
}

// words of the split TREE_Sign's chain-end buffer for `count` messages
size_t chain_end_words(int set, uint32_t count) {
  const SetInfo& I = kInfo[set];
  return (size_t)count * I.d * I.leaves * I.wots_len * (I.n / 4);
}

// Arguments for messages [io_first, io_first + count) of the staged batch,
// whose per-message work buffers start at work_first (the message's index in
// its chunk).  Message offsets stay absolute into the staged blob; every
// per-message buffer is offset, so sub-batches are independent launches.
LaunchArgs make_args(hs_t* h, int set, const hs_set_config& c, uint32_t io_first, uint32_t work_first,
                     uint32_t count) {
  const uint32_t first = work_first;
  const SetInfo& I = kInfo[set];
  SetState& St = h->sets[set];
  Buffers& B = h->buf[set];
  const Slot& S = B.io[St.slot];
  LaunchArgs a;
  std::memset(&a, 0, sizeof a);
  a.keys = St.keys;
  a.nkeys = St.nkeys;
  a.msgs = S.msgs;
  a.offs = S.offs + io_first;
  a.key_idx = St.has_keyidx ? S.keyidx + io_first : nullptr;
  a.opt_rand = St.has_optrand ? S.optrand + (size_t)io_first * I.n : nullptr;
  a.count = count;
  a.sigs = S.sigs + (size_t)io_first * I.sig_bytes;
  a.wots_steps = S.wsteps ? S.wsteps + io_first : nullptr;
  a.plans = B.plans + first;
  a.indices = B.idx + (size_t)first * I.k;
  a.roots = B.roots + (size_t)first * (I.d + 1) * 8;
  a.fors_roots = B.froots + (size_t)first * I.k * 8;
  a.fors_trees_per_set = c.fors_trees_per_set;
  a.fors_sets_fused = c.fors_sets_fused;
  a.fors_relax = c.fors_relax;
  a.fors_cta_levels = fors_cta_levels(set, c, count);
  if (a.fors_cta_levels < I.log_t) {
    for (int b = 0; b < 2; b++)
      a.fors_nodes[b] = B.fnodes[b] + (size_t)first * I.k * ((size_t)I.t >> (a.fors_cta_levels + b)) * (I.n / 4);
    a.fors_lpre = B.lpre + (size_t)first * (I.log_t + 1) * 8;
  }
  const size_t sw = stash_words(set);
  a.stash = (St.cfg.wots_from_tree && B.stash && B.stash_cap >= ((size_t)first + count) * sw)
                ? B.stash + (size_t)first * sw
                : nullptr;
  // subtree sharing needs the stash (WOTS gather) and a table sized for the key set
  const int L = St.shared_eff;
  if (a.stash && L > 0 && B.shared && B.shared_cap >= (size_t)St.nkeys * shared_words(set, L) && B.key_used &&
      B.key_used_cap >= used_flag_bytes(set, St.nkeys, L)) {
    a.shared = B.shared;
    a.shared_layers = L;
    a.key_used = B.key_used;
    a.unit_used = B.key_used + St.nkeys;
    if (St.cfg.tree_split && B.sends && B.sends_cap >= (size_t)St.nkeys * shared_end_words(set, L))
      a.shared_ends = B.sends;
  }
  if (St.cfg.tree_split && B.ends && B.ends_cap >= chain_end_words(set, first + count))
    a.chain_ends = B.ends + (size_t)first * (I.d - a.shared_layers) * I.leaves * I.wots_len * (I.n / 4);
  return a;
}

// Shared top-layer subtrees on one stream: split (chain grid, then leaf grid) or fused.
cudaError_t enqueue_shared(int set, const hs_set_config& c, const LaunchArgs& a, cudaStream_t s, int& kernels) {
  if (a.shared_layers <= 0) return cudaSuccess;
  if (!a.shared_ends) {
    kernels++;
    return launch(set, K_TREE_SHARED, c.variant[1], a, s);
  }
  kernels += 2;
  cudaError_t e = launch(set, K_SHARED_CHAIN, c.variant[1], a, s);
  return e == cudaSuccess ? launch(set, K_SHARED_ROOT, c.variant[1], a, s) : e;
}

// TREE_Sign on one stream: split (chain grid, leaf grid, Merkle grid) or fused.
cudaError_t enqueue_tree(int set, const hs_set_config& c, const LaunchArgs& a, cudaStream_t s, int& kernels) {
  if (!a.chain_ends) {
    kernels++;
    return launch(set, K_TREE, c.variant[1], a, s);
  }
  cudaError_t e = launch(set, K_TREE_CHAIN, c.variant[1], a, s);
  kernels++;
  if (c.tree_split == 1) {  // leaves and warp-shuffle Merkle reduction in one grid
    kernels++;
    return e == cudaSuccess ? launch(set, K_TREE_ROOT, c.variant[1], a, s) : e;
  }
  kernels += 2;  // leaf grid, then one thread per subtree for the Merkle levels
  if (e == cudaSuccess) e = launch(set, K_TREE_LEAF, c.variant[1], a, s);
  return e == cudaSuccess ? launch(set, K_TREE_MERKLE, c.variant[1], a, s) : e;
}

// FORS_Sign, the batch-wide upper FORS levels (if any) and T_k on one stream.
cudaError_t enqueue_fors(int set, const hs_set_config& c, const LaunchArgs& a, cudaStream_t s, int& kernels) {
  cudaError_t e = launch(set, K_FORS, c.variant[0], a, s);
  kernels++;
  for (int L = a.fors_cta_levels + 1; e == cudaSuccess && L <= kInfo[set].log_t; L++) {
    LaunchArgs al = a;
    al.fors_level = L;
    e = launch(set, K_FORS_LEVEL, c.variant[0], al, s);
    kernels++;
  }
  if (e == cudaSuccess) e = launch(set, K_FORSPK, c.variant[0], a, s);
  kernels++;
  return e;
}

// Per-message work buffers for one launch of `count` messages: message plans,
// FORS indices, roots, the WOTS stash, upper FORS levels and the split
// TREE_Sign's chain ends.
int ensure_scratch(hs_t* h, int set, uint32_t count) {
  const SetInfo& I = kInfo[set];
  Buffers& B = h->buf[set];
  const hs_set_config& c = h->sets[set].cfg;
  void* before[9] = {B.fnodes[0], B.fnodes[1], B.ends, B.lpre, B.plans, B.idx, B.roots, B.froots, B.stash};
  CUDA_TRY(h, grow(B.plans, B.plans_cap, (size_t)count));
  CUDA_TRY(h, grow(B.idx, B.idx_cap, (size_t)count * I.k));
  CUDA_TRY(h, grow(B.roots, B.roots_cap, (size_t)count * (I.d + 1) * 8));
  CUDA_TRY(h, grow(B.froots, B.froots_cap, (size_t)count * I.k * 8));
  if (c.wots_from_tree) CUDA_TRY(h, grow(B.stash, B.stash_cap, (size_t)count * stash_words(set)));
  if (fors_node_words(set, c, count, 0) != 0) {
    for (int b = 0; b < 2; b++) CUDA_TRY(h, grow(B.fnodes[b], B.fnodes_cap[b], fors_node_words(set, c, count, b)));
    CUDA_TRY(h, grow(B.lpre, B.lpre_cap, (size_t)count * (kInfo[set].log_t + 1) * 8));
  }
  if (c.tree_split) CUDA_TRY(h, grow(B.ends, B.ends_cap, chain_end_words(set, count)));
  void* after[9] = {B.fnodes[0], B.fnodes[1], B.ends, B.lpre, B.plans, B.idx, B.roots, B.froots, B.stash};
  if (std::memcmp(before, after, sizeof before) != 0) {
    B.gen++;
    drop_graphs(h);
  }
  return HS_OK;
}

// Issue the signing DAG.  `capture` selects external (graph-visible) timing
// events; `serial` puts every kernel on s0 back to back.
cudaError_t enqueue(hs_t* h, int set, const hs_set_config& c, const LaunchArgs& a, bool capture, bool serial) {
  auto rec = [&](int i, cudaStream_t s) {
    return capture ? cudaEventRecordWithFlags(h->ev[i], s, cudaEventRecordExternal) : cudaEventRecord(h->ev[i], s);
  };
  cudaError_t e;
#define TRY(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
  int kernels = 2;  // msg_prep + WOTS; the shared / FORS / TREE branches are counted by enqueue_*
  TRY(rec(0, h->s0));
  if (a.wots_steps) TRY(cudaMemsetAsync(a.wots_steps, 0, (size_t)a.count * 4, h->s0));
  if (a.shared_layers > 0)
    TRY(cudaMemsetAsync(a.key_used, 0, used_flag_bytes(set, a.nkeys, a.shared_layers), h->s0));
  TRY(launch(set, K_PREP, c.variant[3], a, h->s0));
  TRY(rec(1, h->s0));
  if (serial) {
    TRY(enqueue_fors(set, c, a, h->s0, kernels));
    TRY(rec(2, h->s0));
    TRY(enqueue_tree(set, c, a, h->s0, kernels));
    TRY(rec(3, h->s0));  // [2,3] = per-message TREE_Sign only (the roofline kernel)
    TRY(enqueue_shared(set, c, a, h->s0, kernels));
    TRY(rec(5, h->s0));
    TRY(launch(set, a.stash ? K_WOTS_GATHER : K_WOTS, c.variant[2], a, h->s0));
    TRY(rec(4, h->s0));
  } else {
    TRY(cudaEventRecord(h->fork, h->s0));
    TRY(cudaStreamWaitEvent(h->s1, h->fork, 0));
    // the shared-subtree kernel is small and latency bound (a few subtrees,
    // one thread per leaf): start it first on the FORS branch so it runs
    // under the per-message TREE_Sign instead of after it
    TRY(enqueue_shared(set, c, a, h->s1, kernels));
    TRY(enqueue_fors(set, c, a, h->s1, kernels));
    TRY(rec(2, h->s1));
    TRY(cudaEventRecord(h->join, h->s1));
    TRY(enqueue_tree(set, c, a, h->s0, kernels));
    TRY(rec(3, h->s0));
    TRY(cudaStreamWaitEvent(h->s0, h->join, 0));
    TRY(rec(5, h->s0));
    TRY(launch(set, a.stash ? K_WOTS_GATHER : K_WOTS, c.variant[2], a, h->s0));
    TRY(rec(4, h->s0));
  }
#undef TRY
  h->launches += kernels;
  h->last_kernels = kernels;
  return cudaSuccess;
}

// Messages [first, first + cn) of sub-batch j of T.  The last sub-batch gets
// a smaller share than the others (weights H, ..., H, 1): only its D2H copy
// is not hidden under later compute in hs_sign_batch, so it is kept small.
// H per set (public call, interleaved A/B, profiles/r02au_ab_subbatch_weight8.txt
// and r02ch_): 4 for 128f (8 is 2 % slower: 4,096 messages leave the small
// last sub-batch too few blocks), 8 for 192f / 256f.  HS_SUB_HEAD_WEIGHT
// overrides every set.
#ifdef HS_SUB_HEAD_WEIGHT
constexpr uint64_t kSubHeadWeight[3] = {HS_SUB_HEAD_WEIGHT, HS_SUB_HEAD_WEIGHT, HS_SUB_HEAD_WEIGHT};
#else
constexpr uint64_t kSubHeadWeight[3] = {4, 8, 8};
#endif
void sub_range(int set, uint32_t count, int T, int j, uint32_t& first, uint32_t& cn) {
#ifdef HS_EQUAL_SUBBATCH
  (void)set;
  const uint32_t per = (count + T - 1) / T;
  first = std::min(count, (uint32_t)j * per);
  cn = std::min(per, count - first);
#else
  if (T <= 1) {
    first = 0;
    cn = count;
    return;
  }
  const uint64_t H = kSubHeadWeight[set];  // weight of every sub-batch but the last (which has weight 1)
  const uint64_t W = H * ((uint64_t)T - 1ull) + 1ull;
  auto edge = [&](int i) { return (uint32_t)((uint64_t)count * std::min<uint64_t>(H * (uint64_t)i, W) / W); };
  first = edge(j);
  cn = edge(j + 1) - first;
#endif
}

// Multi-stream batch (the paper's m x T batching), one
// graph per batch shape:
//
// overlap = 1:
//   s0:      [memset key_used] -> msg_prep(all) -> fork
//   q0:      [shared subtrees] ...................................-> sh
//   q(1+2j): TREE_j ............ (wait fjoin_j, sh) -> WOTS_j -> done_j -> join
//   q(2+2j): FORS_j -> levels -> T_k_j -> fjoin_j
// Sub-batch j's streams have the j-th highest priorities and the graph is
// instantiated with per-node priorities, so the block scheduler drains
// sub-batch 0 first while later ones fill the idle slots and the tail.
// overlap = 0: one stream order after msg_prep -- shared subtrees, then per
// sub-batch FORS_j, TREE_j, WOTS_j -> done_j (no kernel concurrency; measured
// faster for 192f/256f, whose large FORS CTAs slow co-resident chain blocks).
// Either way each sub-batch's signatures are complete (event done_j) while
// later sub-batches still compute, so their D2H copies (issued on ls[j]
// outside the graph) overlap the remaining compute.  The shared-subtree
// kernel runs once for the whole batch.
cudaError_t enqueue_batch(hs_t* h, int set, uint32_t io_first, uint32_t count, int T, bool capture) {
  const hs_set_config c = batch_config(h->sets[set].cfg, count);
  const LaunchArgs all = make_args(h, set, c, io_first, 0, count);
  auto rec = [&](cudaEvent_t ev, cudaStream_t s) {
    return capture ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal) : cudaEventRecord(ev, s);
  };
  cudaError_t e;
  int kernels = 0;
#define TRY(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
  TRY(rec(h->ev[0], h->s0));
  if (all.wots_steps) TRY(cudaMemsetAsync(all.wots_steps, 0, (size_t)count * 4, h->s0));
  if (all.shared_layers > 0)
    TRY(cudaMemsetAsync(all.key_used, 0, used_flag_bytes(set, all.nkeys, all.shared_layers), h->s0));
  TRY(launch(set, K_PREP, c.variant[3], all, h->s0));
  kernels++;
  TRY(rec(h->ev[1], h->s0));
  TRY(cudaEventRecord(h->fork, h->s0));
  if (!c.overlap) {
    // one stream order: shared subtrees, then per sub-batch FORS, TREE, WOTS
    cudaStream_t q = h->q[1];
    TRY(cudaStreamWaitEvent(q, h->fork, 0));
    if (all.shared_layers > 0) TRY(enqueue_shared(set, c, all, q, kernels));
    for (int j = 0; j < T; j++) {
      uint32_t first, cn;
      sub_range(set, count, T, j, first, cn);
      if (cn == 0) break;
      const LaunchArgs a = make_args(h, set, c, io_first + first, first, cn);
      TRY(enqueue_fors(set, c, a, q, kernels));
      TRY(enqueue_tree(set, c, a, q, kernels));
      TRY(launch(set, a.stash ? K_WOTS_GATHER : K_WOTS, c.variant[2], a, q));
      kernels += 1;
      TRY(rec(h->done[j], q));
    }
    TRY(cudaEventRecord(h->joins[0], q));
    TRY(cudaStreamWaitEvent(h->s0, h->joins[0], 0));
    TRY(rec(h->ev[4], h->s0));
    h->launches += kernels;
    h->last_kernels = kernels;
    return cudaSuccess;
  }
  if (all.shared_layers > 0) {
    TRY(cudaStreamWaitEvent(h->q[0], h->fork, 0));
    TRY(enqueue_shared(set, c, all, h->q[0], kernels));
    TRY(cudaEventRecord(h->sh_done, h->q[0]));
  }
  for (int j = 0; j < T; j++) {
    uint32_t first, cn;
    sub_range(set, count, T, j, first, cn);
    if (cn == 0) break;
    const LaunchArgs a = make_args(h, set, c, io_first + first, first, cn);
    // TREE_j on priority 1+2j, FORS_j just below it: FORS_j's short CTAs fill
    // the SMs TREE_j drains before TREE_{j+1} claims them, and the last
    // sub-batch's FORS fills the final tail.
    cudaStream_t q = h->q[1 + 2 * j], qf = h->q[2 + 2 * j];
    TRY(cudaStreamWaitEvent(q, h->fork, 0));
    TRY(cudaStreamWaitEvent(qf, h->fork, 0));
    TRY(enqueue_tree(set, c, a, q, kernels));
    TRY(enqueue_fors(set, c, a, qf, kernels));
    TRY(cudaEventRecord(h->fjoin[j], qf));
    TRY(cudaStreamWaitEvent(q, h->fjoin[j], 0));
    if (all.shared_layers > 0) TRY(cudaStreamWaitEvent(q, h->sh_done, 0));
    TRY(launch(set, a.stash ? K_WOTS_GATHER : K_WOTS, c.variant[2], a, q));
    kernels += 1;
    TRY(rec(h->done[j], q));
    TRY(cudaEventRecord(h->joins[j], q));
    TRY(cudaStreamWaitEvent(h->s0, h->joins[j], 0));
  }
  TRY(rec(h->ev[4], h->s0));
#undef TRY
  h->launches += kernels;
  h->last_kernels = kernels;
  return cudaSuccess;
}

// One graph launch over messages [io_first, io_first + count) of the staged
// batch (count <= cfg.chunk), T prioritised sub-batches.
int launch_chunk(hs_t* h, int set, uint32_t io_first, uint32_t count, int T) {
  SetState& St = h->sets[set];
  if (!St.cfg.use_graph) {
    CUDA_TRY(h, enqueue_batch(h, set, io_first, count, T, false));
    return HS_OK;
  }
  GraphKey key{set, count, St.has_keyidx ? 1 : 0, St.has_optrand ? 1 : 0, h->buf[set].gen,
               cfg_fingerprint(St.cfg) + "/" + std::to_string((uintptr_t)St.keys) + "/" + std::to_string(St.nkeys) +
                   "/L" + std::to_string(St.shared_eff) + "/T" + std::to_string(T) + "/S" + std::to_string(St.slot) +
                   "/F" + std::to_string(io_first)};
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    // bounded cache: a caller that keeps changing batch shapes or configs
    // (the tuner, a service with many batch sizes) re-captures instead of
    // accumulating executable graphs
    if (h->graphs.size() >= kMaxGraphs) drop_graphs(h);
    cudaGraph_t g;
    CUDA_TRY(h, cudaStreamBeginCapture(h->s0, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = enqueue_batch(h, set, io_first, count, T, true);
    cudaError_t e2 = cudaStreamEndCapture(h->s0, &g);
    if (e != cudaSuccess) return fail(h, HS_E_CUDA, "capture: %s", cudaGetErrorString(e));
    if (e2 != cudaSuccess) return fail(h, HS_E_CUDA, "end capture: %s", cudaGetErrorString(e2));
    cudaGraphExec_t ex;
    CUDA_TRY(h, cudaGraphInstantiateWithFlags(&ex, g, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
    h->launches -= h->last_kernels;  // capture does not launch
    h->graph_kernels[key] = h->last_kernels;
    it = h->graphs.emplace(key, ex).first;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const cudaError_t le = cudaGraphLaunch(it->second, h->s0);
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  CUDA_TRY(h, le);
  h->glaunch_n++;
  h->glaunch_us_sum += us;
  h->glaunch_us_max = std::max(h->glaunch_us_max, us);
  h->launches += h->graph_kernels[key];
  return HS_OK;
}

// Sign the staged batch (io slot St.slot), as consecutive graph launches of
// at most cfg.chunk messages over the resident inputs.  With fetch_to,
// sub-batch j's signatures (and WOTS step counts, with wsteps_to) are copied
// to the host on ls[j] as soon as that sub-batch completes;
// d2h_done[slot][j] marks the copy.  Nothing here waits for those copies: the
// next batch that reuses the slot does (double-buffered chunks in
// hs_sign_batch_ex).  *T_out = the most sub-batch streams any launch used.
int run_batch(hs_t* h, int set, uint32_t count, int mode, uint8_t* fetch_to = nullptr, uint32_t* wsteps_to = nullptr,
              int* T_out = nullptr) {
  if (count == 0) return HS_OK;
  SetState& St = h->sets[set];
  h->last_set = set;
  h->last_mode = mode;
  const int slot = St.slot;
  Slot& S = h->buf[set].io[slot];
  const size_t sb = (size_t)kInfo[set].sig_bytes;
  const uint32_t chunk = work_count(St.cfg, count);
  if (int rc = ensure_scratch(h, set, chunk); rc != HS_OK) return rc;
  // inputs of this slot landed; earlier copies out of this slot's signatures finished
  CUDA_TRY(h, cudaStreamWaitEvent(h->s0, h->h2d_done[slot], 0));
  for (int j = 0; j < h->slot_T[slot]; j++) CUDA_TRY(h, cudaStreamWaitEvent(h->s0, h->d2h_done[slot][j], 0));
  h->slot_T[slot] = 0;
  if (mode == 1) {  // serialised kernels with per-kernel events (roofline timing): one chunk
    if (count > chunk) return fail(h, HS_E_USAGE, "serialised timing runs at most one chunk (%u messages)", chunk);
    const hs_set_config bc = batch_config(St.cfg, count);
    CUDA_TRY(h, enqueue(h, set, bc, make_args(h, set, bc, 0, 0, count), false, true));
    CUDA_TRY(h, cudaEventRecord(h->compute_done[slot], h->s0));
    if (fetch_to) CUDA_TRY(h, cudaMemcpyAsync(fetch_to, S.sigs, count * sb, cudaMemcpyDeviceToHost, h->s0));
    if (wsteps_to) CUDA_TRY(h, cudaMemcpyAsync(wsteps_to, S.wsteps, count * 4, cudaMemcpyDeviceToHost, h->s0));
    if (T_out) *T_out = 0;
    return HS_OK;
  }
  int Tmax = 0;
  for (uint32_t c0 = 0; c0 < count; c0 += chunk) {
    const uint32_t cn = std::min(chunk, count - c0);
    int T = std::max(1, std::min(St.cfg.streams, kMaxStreams));
    T = (int)std::min<uint32_t>((uint32_t)T, std::max<uint32_t>(1u, cn / 256u));
    h->last_T = T;
    Tmax = std::max(Tmax, T);
    if (int rc = launch_chunk(h, set, c0, cn, T); rc != HS_OK) return rc;
    if (fetch_to || wsteps_to) {
      for (int j = 0; j < T; j++) {
        uint32_t first, n;
        sub_range(set, cn, T, j, first, n);
        if (n == 0) break;
        first += c0;
        CUDA_TRY(h, cudaStreamWaitEvent(h->ls[j], h->done[j], 0));
        if (fetch_to)
          CUDA_TRY(h, cudaMemcpyAsync(fetch_to + first * sb, S.sigs + first * sb, n * sb, cudaMemcpyDeviceToHost,
                                      h->ls[j]));
        if (wsteps_to)
          CUDA_TRY(h, cudaMemcpyAsync(wsteps_to + first, S.wsteps + first, (size_t)n * 4, cudaMemcpyDeviceToHost,
                                      h->ls[j]));
        CUDA_TRY(h, cudaEventRecord(h->d2h_done[slot][j], h->ls[j]));
        h->slot_T[slot] = std::max(h->slot_T[slot], j + 1);
      }
    }
  }
  CUDA_TRY(h, cudaEventRecord(h->compute_done[slot], h->s0));
  if (T_out) *T_out = Tmax;
  return HS_OK;
}

// Stage messages [first, first + count) of the caller's arrays into io slot
// `slot`: rebased offsets (and the messages unless the caller's buffer is
// pinned) go through the slot's pinned staging, every H2D runs on the copy
// stream after the batch that last read the slot, and h2d_done[slot] gates the
// next run.  Validation happens before anything is copied.
int stage_inputs(hs_t* h, int set, int slot, const uint8_t* msgs, const uint64_t* offs, const uint32_t* key_idx,
                 const uint8_t* opt_rand, uint32_t first, uint32_t count, bool msgs_pinned) {
  const SetInfo& I = kInfo[set];
  SetState& St = h->sets[set];
  Buffers& B = h->buf[set];
  Slot& S = B.io[slot];
  if (key_idx) {
    for (uint32_t i = 0; i < count; i++)
      if (key_idx[first + i] >= St.nkeys)
        return fail(h, HS_E_USAGE, "key_idx[%u]=%u outside the uploaded key table (%u keys)", first + i,
                    key_idx[first + i], St.nkeys);
  }
  const uint64_t base = offs[first];
  const uint64_t bytes = offs[first + count] - base;
  int rc = ensure_capacity(h, set, slot, count, (size_t)bytes);
  if (rc) return rc;
  // the slot's pinned staging is free once its previous H2D finished
  CUDA_TRY(h, cudaEventSynchronize(h->h2d_done[slot]));
  CUDA_TRY(h, grow_host(S.h_offs, S.h_offs_cap, (size_t)count + 1));
  for (uint32_t i = 0; i <= count; i++) S.h_offs[i] = offs[first + i] - base;
  const uint8_t* msrc = msgs + base;
  if (bytes && !msgs_pinned) {
    CUDA_TRY(h, grow_host(S.h_msgs, S.h_msgs_cap, (size_t)bytes));
    std::memcpy(S.h_msgs, msgs + base, (size_t)bytes);
    msrc = S.h_msgs;
  }
  CUDA_TRY(h, cudaStreamWaitEvent(h->cs, h->compute_done[slot], 0));
  CUDA_TRY(h, cudaMemcpyAsync(S.offs, S.h_offs, ((size_t)count + 1) * 8, cudaMemcpyHostToDevice, h->cs));
  if (bytes) CUDA_TRY(h, cudaMemcpyAsync(S.msgs, msrc, (size_t)bytes, cudaMemcpyHostToDevice, h->cs));
  if (key_idx)
    CUDA_TRY(h, cudaMemcpyAsync(S.keyidx, key_idx + first, (size_t)count * 4, cudaMemcpyHostToDevice, h->cs));
  if (opt_rand)
    CUDA_TRY(h, cudaMemcpyAsync(S.optrand, opt_rand + (size_t)first * I.n, (size_t)count * I.n,
                                cudaMemcpyHostToDevice, h->cs));
  CUDA_TRY(h, cudaEventRecord(h->h2d_done[slot], h->cs));
  St.has_keyidx = key_idx != nullptr;
  St.has_optrand = opt_rand != nullptr;
  // Subtree sharing depth for this batch: at most cfg.shared_layers, within
  // the table budget, and (auto policy) only layers with at most twice as many
  // subtrees per key as the key's messages, and only with >= 2 messages per key.  Only subtrees some message reads
  // are computed (msg_prep flags them), so with c messages over U subtrees a
  // shared layer costs U(1 - e^(-c/U)) subtrees instead of c: <= 0.79 c at
  // U = 2c, 0.63 c at U = c.
  St.shared_eff = 0;
  if (St.cfg.shared_layers > 0 && St.cfg.wots_from_tree) {
    uint32_t used = 1;
    if (key_idx) {
      std::vector<uint8_t> seen(St.nkeys, 0);
      used = 0;
      for (uint32_t i = 0; i < count; i++)
        if (!seen[key_idx[first + i]]) { seen[key_idx[first + i]] = 1; used++; }
    }
    const int hp = kInfo[set].hp;
    int L = 0;
    // messages per launch: a batch larger than the chunk builds the shared
    // subtrees once per chunk
    const size_t per_launch = work_count(St.cfg, count);
    // a shared subtree saves work only when two or more messages read it:
    // with fewer than two messages per key on average the auto policy shares
    // nothing (and a one-message graph skips the shared branch, its flag
    // memset and the WOTS gather's wait on it: 1 message 114 -> 106 us, 128f)
    const bool readers = per_launch >= 2 * std::min<size_t>(used, per_launch);
    while (L < St.cfg.shared_layers && (readers || !St.cfg.shared_auto)) {
      const size_t units_j = (size_t)1 << (hp * L);  // subtrees at depth L per key
      if (St.cfg.shared_auto && units_j * std::min<size_t>(used, per_launch) > 2 * per_launch) break;
      if ((size_t)St.nkeys * shared_words(set, L + 1) * 4 > kSharedBudgetBytes) break;
      L++;
    }
    St.shared_eff = L;
  }
  if (St.shared_eff > 0) {
    const size_t need = (size_t)St.nkeys * shared_words(set, St.shared_eff);
    void* before[3] = {B.shared, B.key_used, B.sends};
    CUDA_TRY(h, grow(B.shared, B.shared_cap, need));
    CUDA_TRY(h, grow(B.key_used, B.key_used_cap, used_flag_bytes(set, St.nkeys, St.shared_eff)));
    if (St.cfg.tree_split)
      CUDA_TRY(h, grow(B.sends, B.sends_cap, (size_t)St.nkeys * shared_end_words(set, St.shared_eff)));
    void* after[3] = {B.shared, B.key_used, B.sends};
    if (std::memcmp(before, after, sizeof before) != 0) {
      B.gen++;
      drop_graphs(h);
    }
  }
  St.slot = slot;
  St.staged = count;
  return HS_OK;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int hs_open(int device, hs_t** out) {
  if (!out) return HS_E_USAGE;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return HS_E_CUDA;
  if (device < 0 || device >= ndev) return HS_E_USAGE;
  hs_t* h = new hs_ctx();
  h->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete h; return HS_E_CUDA; }
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&h->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  cudaDeviceGetAttribute(&h->cc_major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&h->cc_minor, cudaDevAttrComputeCapabilityMinor, device);
  if (cudaStreamCreateWithFlags(&h->s0, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->s1, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return HS_E_CUDA;
  }
  for (auto& ev : h->ev) cudaEventCreate(&ev);
  int prio_least = 0, prio_greatest = 0;
  cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest);
  cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking);
  for (int sl = 0; sl < kSlots; sl++) {
    cudaEventCreateWithFlags(&h->h2d_done[sl], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->compute_done[sl], cudaEventDisableTiming);
    for (int j = 0; j < kMaxStreams; j++) cudaEventCreateWithFlags(&h->d2h_done[sl][j], cudaEventDisableTiming);
  }
  for (int j = 0; j < kMaxStreams; j++) {
    cudaStreamCreateWithFlags(&h->ls[j], cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&h->fjoin[j], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->done[j], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->joins[j], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&h->sh_done, cudaEventDisableTiming);
  for (int j = 0; j < 2 * kMaxStreams + 1; j++)
    cudaStreamCreateWithPriority(&h->q[j], cudaStreamNonBlocking, std::min(prio_greatest + j, prio_least));
  cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->join, cudaEventDisableTiming);
  for (int s = 0; s < 3; s++) h->sets[s].cfg = default_config(s);
  *out = h;
  return HS_OK;
}

void hs_close(hs_t* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  drop_graphs(h);
  for (int s = 0; s < 3; s++) {
    Buffers& B = h->buf[s];
    for (Slot& S : B.io) {
      cudaFree(S.msgs); cudaFree(S.offs); cudaFree(S.keyidx); cudaFree(S.optrand); cudaFree(S.sigs);
      cudaFree(S.wsteps);
      cudaFreeHost(S.h_msgs); cudaFreeHost(S.h_offs); cudaFreeHost(S.h_sigs); cudaFreeHost(S.h_wsteps);
    }
    cudaFree(B.plans); cudaFree(B.idx); cudaFree(B.roots); cudaFree(B.froots); cudaFree(B.stash);
    cudaFree(h->sets[s].keys);
    cudaFree(B.shared);
    cudaFree(B.key_used);
    cudaFree(B.fnodes[0]);
    cudaFree(B.fnodes[1]);
    cudaFree(B.ends);
    cudaFree(B.sends);
    cudaFree(B.lpre);
    cudaFree(B.v_pks); cudaFree(B.v_msgs); cudaFree(B.v_sigs); cudaFree(B.v_ok); cudaFree(B.v_offs);
    cudaFree(B.v_kidx);
    cudaFree(h->sets[s].sk_raw);
  }
  if (h->flush) cudaFree(h->flush);
  for (int sl = 0; sl < kSlots; sl++) {
    cudaEventDestroy(h->h2d_done[sl]);
    cudaEventDestroy(h->compute_done[sl]);
    for (int j = 0; j < kMaxStreams; j++) cudaEventDestroy(h->d2h_done[sl][j]);
  }
  cudaStreamDestroy(h->cs);
  for (int j = 0; j < kMaxStreams; j++) {
    cudaStreamDestroy(h->ls[j]);
    cudaEventDestroy(h->fjoin[j]);
    cudaEventDestroy(h->done[j]);
    cudaEventDestroy(h->joins[j]);
  }
  cudaEventDestroy(h->sh_done);
  for (int j = 0; j < 2 * kMaxStreams + 1; j++) cudaStreamDestroy(h->q[j]);
  for (auto& ev : h->ev) cudaEventDestroy(ev);
  cudaEventDestroy(h->fork);
  cudaEventDestroy(h->join);
  cudaStreamDestroy(h->s0);
  cudaStreamDestroy(h->s1);
  delete h;
}

const char* hs_last_error(const hs_t* h) { return h ? h->err.c_str() : "null handle"; }

int hs_device_info(hs_t* h, int32_t* sm, int32_t* smem, int32_t* ma, int32_t* mi) {
  if (!h) return HS_E_USAGE;
  if (sm) *sm = h->sm_count;
  if (smem) *smem = h->smem_optin;
  if (ma) *ma = h->cc_major;
  if (mi) *mi = h->cc_minor;
  return HS_OK;
}

int hs_params(int set, int32_t* fields, int cap) {
  if (!valid_set(set) || !fields) return HS_E_USAGE;
  const int nf = (int)(sizeof(SetInfo) / sizeof(int));
  const int* src = reinterpret_cast<const int*>(&kInfo[set]);
  int m = std::min(cap, nf);
  for (int i = 0; i < m; i++) fields[i] = src[i];
  return m;
}

int hs_config_get(hs_t* h, int set, hs_set_config* cfg) {
  if (!h || !valid_set(set) || !cfg) return fail(h, HS_E_USAGE, "bad arguments");
  *cfg = h->sets[set].cfg;
  return HS_OK;
}

int hs_config_set(hs_t* h, int set, const hs_set_config* cfg) {
  if (!h || !valid_set(set) || !cfg) return fail(h, HS_E_USAGE, "bad arguments");
  int rc = check_layout(h, set, *cfg);
  if (rc) return rc;
  h->sets[set].cfg = *cfg;
  return HS_OK;
}

int64_t hs_fors_smem_bytes(int set, int32_t nt, int32_t f, int32_t relax) {
  if (!valid_set(set) || nt < 1 || f < 1) return -1;
  return (int64_t)fors_smem(set, nt, f, relax);
}

int hs_keys_upload(hs_t* h, int set, const uint8_t* sks, uint32_t nkeys) {
  if (!h || !valid_set(set) || (!sks && nkeys)) return fail(h, HS_E_USAGE, "bad arguments");
  if (nkeys == 0) return fail(h, HS_E_USAGE, "at least one key is required");
  CUDA_TRY(h, cudaSetDevice(h->device));
  const SetInfo& I = kInfo[set];
  SetState& St = h->sets[set];
  KeyDev* old = St.keys;
  CUDA_TRY(h, grow(St.keys, St.keys_cap, nkeys));
  if (old != St.keys) drop_graphs(h);
  CUDA_TRY(h, grow(St.sk_raw, St.sk_raw_cap, (size_t)nkeys * 4 * I.n));
  CUDA_TRY(h, cudaMemcpyAsync(St.sk_raw, sks, (size_t)nkeys * 4 * I.n, cudaMemcpyHostToDevice, h->s0));
  LaunchArgs a;
  std::memset(&a, 0, sizeof a);
  a.sk_bytes = St.sk_raw;
  a.nkeys = nkeys;
  a.keys_out = St.keys;
  CUDA_TRY(h, launch(set, K_KEYSETUP, St.cfg.variant[3], a, h->s0));
  h->launches++;
  CUDA_TRY(h, cudaStreamSynchronize(h->s0));
  // a staged batch's key_idx was checked against the previous table: a smaller
  // table invalidates it (hs_run would index past the new one)
  if (nkeys < St.nkeys && St.has_keyidx) St.staged = 0;
  St.nkeys = nkeys;
  return HS_OK;
}

int hs_keygen_batch(hs_t* h, int set, const uint8_t* seeds, uint32_t nkeys, uint8_t* sks_out) {
  if (!h || !valid_set(set) || !seeds || !sks_out) return fail(h, HS_E_USAGE, "bad arguments");
  if (nkeys == 0) return HS_OK;
  CUDA_TRY(h, cudaSetDevice(h->device));
  const SetInfo& I = kInfo[set];
  std::vector<uint8_t> padded((size_t)nkeys * 4 * I.n, 0);
  for (uint32_t i = 0; i < nkeys; i++) std::memcpy(&padded[(size_t)i * 4 * I.n], seeds + (size_t)i * 3 * I.n, 3 * I.n);
  uint8_t *d_in = nullptr, *d_out = nullptr;
  KeyDev* d_keys = nullptr;
  int rc = HS_OK;
  cudaError_t e = cudaMalloc(&d_in, padded.size());
  if (e == cudaSuccess) e = cudaMalloc(&d_out, padded.size());
  if (e == cudaSuccess) e = cudaMalloc(&d_keys, (size_t)nkeys * sizeof(KeyDev));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_in, padded.data(), padded.size(), cudaMemcpyHostToDevice, h->s0);
  LaunchArgs a;
  std::memset(&a, 0, sizeof a);
  a.sk_bytes = d_in;
  a.nkeys = nkeys;
  a.keys_out = d_keys;
  a.keys = d_keys;
  a.sk_out = d_out;
  const hs_set_config& c = h->sets[set].cfg;
  if (e == cudaSuccess) e = launch(set, K_KEYSETUP, c.variant[3], a, h->s0);
  if (e == cudaSuccess) e = launch(set, K_KEYGEN, c.variant[1], a, h->s0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(sks_out, d_out, padded.size(), cudaMemcpyDeviceToHost, h->s0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->s0);
  h->launches += 2;
  if (e != cudaSuccess) rc = fail(h, HS_E_CUDA, "keygen: %s", cudaGetErrorString(e));
  cudaFree(d_in);
  cudaFree(d_out);
  cudaFree(d_keys);
  return rc;
}

int hs_stage(hs_t* h, int set, const uint8_t* msgs, const uint64_t* offs, const uint32_t* key_idx,
             const uint8_t* opt_rand, uint32_t count) {
  if (!h || !valid_set(set) || !offs || (!msgs && count && offs[count] != offs[0]))
    return fail(h, HS_E_USAGE, "bad arguments");
  if (h->sets[set].nkeys == 0) return fail(h, HS_E_NOKEYS, "no keys uploaded for this parameter set");
  // every offset, as hs_sign_batch does: msg_prep reads offs[i+1] - offs[i] bytes
  for (uint32_t i = 0; i < count; i++)
    if (offs[i + 1] < offs[i]) return fail(h, HS_E_USAGE, "offsets must be non-decreasing");
  CUDA_TRY(h, cudaSetDevice(h->device));
  return stage_inputs(h, set, 0, msgs, offs, key_idx, opt_rand, 0, count, msgs && is_pinned(msgs));
}

int hs_run(hs_t* h, int set, uint32_t count, int mode) {
  if (!h || !valid_set(set)) return fail(h, HS_E_USAGE, "bad arguments");
  if (count > h->sets[set].staged) return fail(h, HS_E_USAGE, "count exceeds the staged batch");
  CUDA_TRY(h, cudaSetDevice(h->device));
  return run_batch(h, set, count, mode);
}

int hs_sync(hs_t* h) {
  if (!h) return HS_E_USAGE;
  CUDA_TRY(h, cudaSetDevice(h->device));
  CUDA_TRY(h, cudaStreamSynchronize(h->s0));
  CUDA_TRY(h, cudaStreamSynchronize(h->s1));
  CUDA_TRY(h, cudaStreamSynchronize(h->cs));
  for (int j = 0; j < kMaxStreams; j++) CUDA_TRY(h, cudaStreamSynchronize(h->ls[j]));
  return HS_OK;
}

int hs_fetch(hs_t* h, int set, uint32_t first, uint32_t count, uint8_t* sigs) {
  if (!h || !valid_set(set) || !sigs) return fail(h, HS_E_USAGE, "bad arguments");
  if ((uint64_t)first + count > h->sets[set].staged) return fail(h, HS_E_USAGE, "range exceeds the staged batch");
  CUDA_TRY(h, cudaSetDevice(h->device));
  const size_t sb = (size_t)kInfo[set].sig_bytes;
  const Slot& S = h->buf[set].io[h->sets[set].slot];
  CUDA_TRY(h, cudaMemcpyAsync(sigs, S.sigs + first * sb, count * sb, cudaMemcpyDeviceToHost, h->s0));
  CUDA_TRY(h, cudaStreamSynchronize(h->s0));
  return HS_OK;
}

int hs_sign_batch(hs_t* h, int set, const uint8_t* msgs, const uint64_t* offs, const uint32_t* key_idx,
                  const uint8_t* opt_rand, uint32_t count, uint8_t* sigs) {
  return hs_sign_batch_ex(h, set, msgs, offs, key_idx, opt_rand, count, sigs, nullptr);
}

// Chunks of cfg.chunk messages, software-pipelined over two io slots: while
// chunk c computes (one graph launch on s0), chunk c+1 is staged (host copy +
// H2D on the copy stream) and chunk c-1's signatures drain to the caller
// (D2H per sub-batch on ls[j]; straight into the caller's buffer when it is
// pinned, else through the slot's pinned staging, copied out on the host
// while the next chunk computes).
int hs_sign_batch_ex(hs_t* h, int set, const uint8_t* msgs, const uint64_t* offs, const uint32_t* key_idx,
                     const uint8_t* opt_rand, uint32_t count, uint8_t* sigs, uint32_t* wots_steps) {
  if (!h || !valid_set(set) || !offs || (count && !sigs)) return fail(h, HS_E_USAGE, "bad arguments");
  if (count == 0) return HS_OK;
  if (!msgs && offs[count] != offs[0]) return fail(h, HS_E_USAGE, "null message buffer");
  for (uint32_t i = 0; i < count; i++)
    if (offs[i + 1] < offs[i]) return fail(h, HS_E_USAGE, "offsets must be non-decreasing");
  if (h->sets[set].nkeys == 0) return fail(h, HS_E_NOKEYS, "no keys uploaded for this parameter set");
  CUDA_TRY(h, cudaSetDevice(h->device));
  const size_t sb = (size_t)kInfo[set].sig_bytes;
  const uint32_t chunk = (uint32_t)std::max(1, h->sets[set].cfg.chunk);
  const bool direct = is_pinned(sigs);
  const bool wdirect = wots_steps && is_pinned(wots_steps);
  const bool mpinned = msgs && is_pinned(msgs);
  Buffers& B = h->buf[set];
  struct Pending {
    int slot = -1, T = 0;
    uint32_t first = 0, cn = 0;
  } prev;
  // a chunk's host-side tail: wait for its copies, move staged bytes out
  auto drain = [&](const Pending& pc) -> int {
    if (pc.slot < 0) return HS_OK;
    for (int j = 0; j < std::max(pc.T, 1); j++) CUDA_TRY(h, cudaEventSynchronize(h->d2h_done[pc.slot][j]));
    if (pc.T == 0) CUDA_TRY(h, cudaStreamSynchronize(h->s0));  // serial mode copies on s0
    const Slot& S = B.io[pc.slot];
    if (!direct) std::memcpy(sigs + pc.first * sb, S.h_sigs, pc.cn * sb);
    if (wots_steps && !wdirect) std::memcpy(wots_steps + pc.first, S.h_wsteps, (size_t)pc.cn * 4);
    return HS_OK;
  };
  int rc = HS_OK;
  uint32_t c = 0;
  for (uint32_t first = 0; first < count && rc == HS_OK; first += chunk, c++) {
    const uint32_t cn = std::min(chunk, count - first);
    const int slot = (int)(c & 1u);
    rc = stage_inputs(h, set, slot, msgs, offs, key_idx, opt_rand, first, cn, mpinned);
    if (rc) break;
    Slot& S = B.io[slot];
    // the slot's pinned output staging was drained by the previous iteration
    if (!direct) CUDA_TRY(h, grow_host(S.h_sigs, S.h_sigs_cap, (size_t)cn * sb));
    if (wots_steps && !wdirect) CUDA_TRY(h, grow_host(S.h_wsteps, S.h_wsteps_cap, (size_t)cn));
    int T = 0;
    rc = run_batch(h, set, cn, 0, direct ? sigs + first * sb : S.h_sigs,
                   wots_steps ? (wdirect ? wots_steps + first : S.h_wsteps) : nullptr, &T);
    if (rc) break;
    if (int r2 = drain(prev); r2 != HS_OK) return r2;
    prev = Pending{slot, T, first, cn};
  }
  if (rc == HS_OK) rc = drain(prev);
  // drain() waited for the last chunk's copy-out events (each recorded after
  // its graph and its copies; an event sync also reports a kernel fault), so a
  // successful call is complete here; an error path may leave work on any stream
  if (rc != HS_OK) {
    cudaStreamSynchronize(h->s0);
    for (int j = 0; j < kMaxStreams; j++) cudaStreamSynchronize(h->ls[j]);
  }
  return rc;
}

int hs_verify_batch(hs_t* h, int set, const uint8_t* pks, uint32_t nkeys, const uint8_t* msgs, const uint64_t* offs,
                    const uint32_t* key_idx, const uint8_t* sigs, uint32_t count, uint8_t* ok) {
  if (!h || !valid_set(set) || !pks || !offs || (count && (!sigs || !ok)) || nkeys == 0)
    return fail(h, HS_E_USAGE, "bad arguments");
  if (count == 0) return HS_OK;
  for (uint32_t i = 0; i < count; i++) {
    if (offs[i + 1] < offs[i]) return fail(h, HS_E_USAGE, "offsets must be non-decreasing");
    if (key_idx && key_idx[i] >= nkeys) return fail(h, HS_E_USAGE, "key_idx[%u] out of range", i);
  }
  CUDA_TRY(h, cudaSetDevice(h->device));
  const SetInfo& I = kInfo[set];
  const uint64_t base = offs[0], mbytes = offs[count] - offs[0];
  std::vector<uint64_t> ro(count + 1);
  for (uint32_t i = 0; i <= count; i++) ro[i] = offs[i] - base;
  // device buffers persist across calls (grown on demand); pinned host inputs
  // (e.g. the signatures a pinned hs_sign_batch call just wrote) copy async
  Buffers& B = h->buf[set];
  cudaError_t e = grow(B.v_pks, B.v_pks_cap, (size_t)nkeys * 2 * I.n);
  if (e == cudaSuccess) e = grow(B.v_msgs, B.v_msgs_cap, std::max<size_t>(mbytes, 1));
  if (e == cudaSuccess) e = grow(B.v_sigs, B.v_sigs_cap, (size_t)count * I.sig_bytes);
  if (e == cudaSuccess) e = grow(B.v_ok, B.v_ok_cap, (size_t)count);
  if (e == cudaSuccess) e = grow(B.v_offs, B.v_offs_cap, (size_t)count + 1);
  if (e == cudaSuccess && key_idx) e = grow(B.v_kidx, B.v_kidx_cap, (size_t)count);
  if (e == cudaSuccess) e = cudaMemcpyAsync(B.v_pks, pks, (size_t)nkeys * 2 * I.n, cudaMemcpyHostToDevice, h->s0);
  if (e == cudaSuccess && mbytes) e = cudaMemcpyAsync(B.v_msgs, msgs + base, mbytes, cudaMemcpyHostToDevice, h->s0);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(B.v_sigs, sigs, (size_t)count * I.sig_bytes, cudaMemcpyHostToDevice, h->s0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(B.v_offs, ro.data(), ro.size() * 8, cudaMemcpyHostToDevice, h->s0);
  if (e == cudaSuccess && key_idx)
    e = cudaMemcpyAsync(B.v_kidx, key_idx, (size_t)count * 4, cudaMemcpyHostToDevice, h->s0);
  LaunchArgs a;
  std::memset(&a, 0, sizeof a);
  a.pks = B.v_pks;
  a.nkeys = nkeys;
  a.msgs = B.v_msgs;
  a.offs = B.v_offs;
  a.key_idx = key_idx ? B.v_kidx : nullptr;
  a.vsigs = B.v_sigs;
  a.ok = B.v_ok;
  a.count = count;
  if (e == cudaSuccess) e = launch(set, K_VERIFY, h->sets[set].cfg.variant[2], a, h->s0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ok, B.v_ok, count, cudaMemcpyDeviceToHost, h->s0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->s0);
  h->launches++;
  if (e != cudaSuccess) return fail(h, HS_E_CUDA, "verify: %s", cudaGetErrorString(e));
  return HS_OK;
}

int hs_timings(hs_t* h, float* ms, int cap) {
  if (!h || !ms || cap < 1) return HS_E_USAGE;
  if (h->last_set < 0) return 0;
  cudaSetDevice(h->device);
  if (cudaEventSynchronize(h->ev[4]) != cudaSuccess) return fail(h, HS_E_CUDA, "timing events not complete");
  float v[5] = {0, 0, 0, 0, 0};
  cudaEventElapsedTime(&v[0], h->ev[0], h->ev[4]);
  cudaEventElapsedTime(&v[1], h->ev[0], h->ev[1]);
  if (h->last_mode == 1) cudaEventElapsedTime(&v[2], h->ev[1], h->ev[2]);
  if (h->last_mode == 1) {
    cudaEventElapsedTime(&v[3], h->ev[2], h->ev[3]);
    cudaEventElapsedTime(&v[4], h->ev[5], h->ev[4]);
  } else {
    v[2] = v[3] = v[4] = 0.f;  // graph mode overlaps the stages; per-kernel times need mode 1
  }
  int m = std::min(cap, 5);
  for (int i = 0; i < m; i++) ms[i] = v[i];
  return m;
}

int hs_bench_run(hs_t* h, int set, uint32_t count, int32_t steps, int mode, uint64_t flush_bytes, float* step_ms) {
  if (!h || !valid_set(set) || steps < 1 || !step_ms) return fail(h, HS_E_USAGE, "bad arguments");
  if (count == 0 || count > h->sets[set].staged) return fail(h, HS_E_USAGE, "count exceeds the staged batch");
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (flush_bytes && flush_bytes > h->flush_cap) {
    if (h->flush) cudaFree(h->flush);
    h->flush = nullptr;
    h->flush_cap = 0;
    CUDA_TRY(h, cudaMalloc(&h->flush, flush_bytes));
    h->flush_cap = flush_bytes;
  }
  std::vector<cudaEvent_t> ev(2 * (size_t)steps);
  for (auto& e : ev) CUDA_TRY(h, cudaEventCreate(&e));
  int rc = HS_OK;
  for (int i = 0; i < steps && rc == HS_OK; i++) {
    if (flush_bytes) {
      cudaError_t e = cudaMemsetAsync(h->flush, i & 0xFF, flush_bytes, h->s0);
      if (e != cudaSuccess) rc = fail(h, HS_E_CUDA, "flush: %s", cudaGetErrorString(e));
    }
    if (rc == HS_OK) cudaEventRecord(ev[2 * i], h->s0);
    if (rc == HS_OK) rc = run_batch(h, set, count, mode);
    if (rc == HS_OK) cudaEventRecord(ev[2 * i + 1], h->s0);
  }
  cudaError_t se = cudaStreamSynchronize(h->s0);
  if (rc == HS_OK && se != cudaSuccess) rc = fail(h, HS_E_CUDA, "bench: %s", cudaGetErrorString(se));
  if (rc == HS_OK)
    for (int i = 0; i < steps; i++) cudaEventElapsedTime(&step_ms[i], ev[2 * i], ev[2 * i + 1]);
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

int64_t hs_launch_count(hs_t* h) { return h ? h->launches : -1; }

int hs_batch_info(hs_t* h, int set, int32_t* out, int cap) {
  if (!h || !valid_set(set) || (cap > 0 && !out)) return fail(h, HS_E_USAGE, "bad arguments");
  const SetState& St = h->sets[set];
  // shared subtrees the last run of the staged batch computed (flags set by msg_prep)
  int32_t built = 0;
  const Buffers& B = h->buf[set];
  if (cap > 4 && St.shared_eff > 0 && B.key_used && B.key_used_cap >= used_flag_bytes(set, St.nkeys, St.shared_eff)) {
    std::vector<uint8_t> f((size_t)St.nkeys * shared_units_of(set, St.shared_eff));
    CUDA_TRY(h, cudaSetDevice(h->device));
    CUDA_TRY(h, cudaStreamSynchronize(h->s0));
    CUDA_TRY(h, cudaMemcpy(f.data(), B.key_used + St.nkeys, f.size(), cudaMemcpyDeviceToHost));
    for (uint8_t x : f) built += x != 0;
  }
  const uint32_t graph_count = std::min<uint32_t>(St.staged, (uint32_t)std::max(1, St.cfg.chunk));
  const hs_set_config bc = batch_config(St.cfg, graph_count);
  const int32_t v[5] = {(int32_t)St.staged, St.shared_eff, fors_cta_levels(set, bc, graph_count), bc.tree_split, built};
  const int n = std::min(cap, 5);
  for (int i = 0; i < n; i++) out[i] = v[i];
  return n;
}

int hs_variants(int32_t* masks, int cap) {
  const int nm = hs::kVariants - 2;
  for (int i = 0; i < nm && i < cap; i++) masks[i] = hs::kMxMaskList[i];
  return hs::kVariants;
}

int hs_launch_stats(hs_t* h, double* out, int cap, int reset) {
  if (!h || (cap > 0 && !out)) return fail(h, HS_E_USAGE, "bad arguments");
  const double v[3] = {(double)h->glaunch_n, h->glaunch_n ? h->glaunch_us_sum / h->glaunch_n : 0.0,
                       h->glaunch_us_max};
  const int n = std::min(cap, 3);
  for (int i = 0; i < n; i++) out[i] = v[i];
  if (reset) {
    h->glaunch_n = 0;
    h->glaunch_us_sum = h->glaunch_us_max = 0.0;
  }
  return n;
}

// ---------------------------------------------------------------------------
// hs_tune: the on-device Tree Tuning search (reference tuner.py:91-143
// Algorithm 1 + profile_kernels / select_backends tuner.py:184-274), run on
// this handle's device.  Python's tuner.tune_on_device is the same search
// driven from the host package; this entry point gives a C / FFI caller
// the tuner without Python.
// ---------------------------------------------------------------------------
namespace {

struct TuneCand {
  int nt, f, relax, lanes, passes;
  size_t smem;
  double sync, ut, us;
};

// Algorithm 1 over (N_tree, F, Relax) at S_max = the device's opt-in shared
// memory and the FORS kernel's 768-lane CTA (tuner.device_candidates), no
// alpha pruning, ordered by (sync, -U_T, -U_S, lanes, F).
std::vector<TuneCand> tune_candidates(hs_t* h, int set) {
  const SetInfo& I = kInfo[set];
  std::vector<TuneCand> out;
  for (int relax = 0; relax <= 1; relax++) {
    const int lpt = relax ? I.t / 2 : I.t;
    for (int nt = 1; nt * lpt <= kForsMaxLanes; nt++) {
      const int sets_total = (I.k + nt - 1) / nt;
      for (int f = 1; f <= std::max(1, I.k / nt); f++) {
        const size_t smem = fors_smem(set, nt, f, relax);
        if (smem > (size_t)h->smem_optin) break;
        const int passes = (sets_total + f - 1) / f;
        const double syncs = (double)(I.log_t - relax) * passes;
        out.push_back(TuneCand{nt, f, relax, nt * lpt, passes, smem, syncs, (double)(nt * lpt) / kForsMaxLanes,
                               (double)smem / h->smem_optin});
      }
    }
  }
  std::sort(out.begin(), out.end(), [](const TuneCand& a, const TuneCand& b) {
    return std::make_tuple(a.sync, -a.ut, -a.us, a.lanes, a.f) < std::make_tuple(b.sync, -b.ut, -b.us, b.lanes, b.f);
  });
  return out;
}

double trimmed_mean(std::vector<float> v) {
  std::sort(v.begin(), v.end());
  if (v.size() >= 3) v = std::vector<float>(v.begin() + 1, v.end() - 1);
  double acc = 0;
  for (float x : v) acc += x;
  return v.empty() ? 0.0 : acc / v.size();
}

// Device ms of one kernel stage (1 FORS_Sign + T_k, 2 TREE_Sign, 3 WOTS_Sign)
// in `reps` serialised runs of the staged batch (CUDA events around it).
int time_stage(hs_t* h, int set, uint32_t count, int stage, int reps, std::vector<float>& out) {
  out.clear();
  for (int r = 0; r < reps; r++) {
    if (int rc = run_batch(h, set, count, 1); rc != HS_OK) return rc;
    float ms[5];
    if (hs_timings(h, ms, 5) != 5) return fail(h, HS_E_CUDA, "tune: timing events");
    out.push_back(ms[1 + stage]);
  }
  return HS_OK;
}

// Device time (ms, CUDA events inside the graph) of the staged batch as one graph launch.
int time_graph(hs_t* h, int set, uint32_t count, int reps, std::vector<float>& out) {
  out.clear();
  for (int r = 0; r < reps; r++) {
    if (int rc = run_batch(h, set, count, 0); rc != HS_OK) return rc;
    float ms[5];
    if (hs_timings(h, ms, 5) < 1) return fail(h, HS_E_CUDA, "tune: timing events");
    out.push_back(ms[0]);
  }
  return HS_OK;
}

std::string cfg_json(const hs_set_config& c) {
  char b[512];
  snprintf(b, sizeof b,
           "{\"fors_trees_per_set\": %d, \"fors_sets_fused\": %d, \"fors_relax\": %d, \"variant\": [%d, %d, %d, %d], "
           "\"use_graph\": %d, \"chunk\": %d, \"wots_from_tree\": %d, \"streams\": %d, \"shared_layers\": %d, "
           "\"shared_auto\": %d, \"fors_cta_levels\": %d, \"tree_split\": %d, \"overlap\": %d, "
           "\"fors_small_batch\": %d, \"tree_small_batch\": %d}",
           c.fors_trees_per_set, c.fors_sets_fused, c.fors_relax, c.variant[0], c.variant[1], c.variant[2],
           c.variant[3], c.use_graph, c.chunk, c.wots_from_tree, c.streams, c.shared_layers, c.shared_auto,
           c.fors_cta_levels, c.tree_split, c.overlap, c.fors_small_batch, c.tree_small_batch);
  return b;
}

}  // namespace

int hs_tune(hs_t* h, int set, uint32_t count, int32_t top, int32_t reps, char* json, size_t cap) {
  if (!h || !valid_set(set) || count == 0 || top < 1 || reps < 1) return fail(h, HS_E_USAGE, "bad arguments");
  CUDA_TRY(h, cudaSetDevice(h->device));
  const SetInfo& I = kInfo[set];
  SetState& St = h->sets[set];
  // synthetic batch: the key table as uploaded (a fixed synthetic key when
  // none is), count 32-byte messages from a fixed splitmix64 stream
  if (St.nkeys == 0) {
    std::vector<uint8_t> seed(3 * I.n), sk(4 * I.n);
    for (int i = 0; i < 3 * I.n; i++) seed[i] = (uint8_t)i;
    if (int rc = hs_keygen_batch(h, set, seed.data(), 1, sk.data()); rc != HS_OK) return rc;
    if (int rc = hs_keys_upload(h, set, sk.data(), 1); rc != HS_OK) return rc;
  }
  std::vector<uint8_t> msgs((size_t)count * 32);
  uint64_t x = 0x2512239690ull;
  for (size_t i = 0; i < msgs.size(); i += 8) {
    x += 0x9e3779b97f4a7c15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    std::memcpy(&msgs[i], &z, 8);
  }
  std::vector<uint64_t> offs(count + 1);
  for (uint32_t i = 0; i <= count; i++) offs[i] = 32ull * i;
  const hs_set_config base = St.cfg;
  hs_set_config c = base;
  c.chunk = std::max<int>(c.chunk, (int)count);  // one launch per timed batch
  if (int rc = hs_config_set(h, set, &c); rc != HS_OK) return rc;
  if (int rc = stage_inputs(h, set, 0, msgs.data(), offs.data(), nullptr, nullptr, 0, count, false); rc != HS_OK)
    return rc;
  std::string js = "{\"set\": " + std::to_string(set) + ", \"count\": " + std::to_string(count) +
                   ", \"smem_optin\": " + std::to_string(h->smem_optin);
  std::vector<float> t;
  // 1. every feasible layout once (2 runs, min), the `top` fastest re-timed
  const std::vector<TuneCand> cands = tune_candidates(h, set);
  if (cands.empty()) return fail(h, HS_E_CONFIG, "no feasible FORS layout under %d bytes", h->smem_optin);
  std::vector<std::pair<double, size_t>> first;
  for (size_t i = 0; i < cands.size(); i++) {
    c.fors_trees_per_set = cands[i].nt;
    c.fors_sets_fused = cands[i].f;
    c.fors_relax = cands[i].relax;
    if (int rc = hs_config_set(h, set, &c); rc != HS_OK) return rc;
    if (int rc = time_stage(h, set, count, 1, 2, t); rc != HS_OK) return rc;
    first.emplace_back(*std::min_element(t.begin(), t.end()), i);
  }
  std::sort(first.begin(), first.end());
  js += ", \"candidates\": " + std::to_string(cands.size()) + ", \"layouts\": [";
  double best_ms = 1e30;
  size_t best = first[0].second;
  for (int k = 0; k < top && k < (int)first.size(); k++) {
    const TuneCand& cd = cands[first[k].second];
    c.fors_trees_per_set = cd.nt;
    c.fors_sets_fused = cd.f;
    c.fors_relax = cd.relax;
    if (int rc = hs_config_set(h, set, &c); rc != HS_OK) return rc;
    if (int rc = time_stage(h, set, count, 1, reps, t); rc != HS_OK) return rc;
    const double ms = trimmed_mean(t);
    char b[256];
    snprintf(b, sizeof b, "%s{\"trees_per_set\": %d, \"sets_fused\": %d, \"relax\": %d, \"lanes\": %d, "
             "\"smem_bytes\": %zu, \"passes\": %d, \"fors_ms\": %.4f}", k ? ", " : "", cd.nt, cd.f, cd.relax,
             cd.lanes, cd.smem, cd.passes, ms);
    js += b;
    if (ms < best_ms) best_ms = ms, best = first[k].second;
  }
  js += "]";
  c.fors_trees_per_set = cands[best].nt;
  c.fors_sets_fused = cands[best].f;
  c.fors_relax = cands[best].relax;
  // 1b. in-CTA FORS levels vs the batch-wide level grids for that layout
  js += ", \"cta_levels_ms\": {";
  int best_lc = -1;
  double best_lc_ms = 1e30;
  for (int lc = -1; lc <= I.log_t; lc++) {
    if (lc == 0 && c.fors_relax) continue;
    c.fors_cta_levels = lc;
    if (int rc = hs_config_set(h, set, &c); rc != HS_OK) return rc;
    if (int rc = time_stage(h, set, count, 1, reps, t); rc != HS_OK) return rc;
    const double ms = trimmed_mean(t);
    js += (lc == -1 ? "\"" : ", \"") + std::to_string(lc) + "\": " + std::to_string(ms);
    if (ms < best_lc_ms) best_lc_ms = ms, best_lc = lc;
  }
  js += "}";
  c.fors_cta_levels = best_lc;
  // 2. SHA-256 path per kernel: the fastest compiled path replaces native only
  //    when faster by more than 2% (tuner.py:206-218)
  js += ", \"variant_ms\": {";
  const char* kname[3] = {"FORS_Sign", "TREE_Sign", "WOTS_Sign"};
  for (int k = 0; k < 3; k++) {
    std::vector<double> ms(hs::kVariants);
    for (int v = 0; v < hs::kVariants; v++) {
      c.variant[k] = v;
      if (int rc = hs_config_set(h, set, &c); rc != HS_OK) return rc;
      if (int rc = time_stage(h, set, count, 1 + k, reps, t); rc != HS_OK) return rc;
      ms[v] = trimmed_mean(t);
    }
    int bv = (int)(std::min_element(ms.begin(), ms.end()) - ms.begin());
    if (!(ms[bv] < ms[0] * 0.98)) bv = 0;
    c.variant[k] = bv;
    js += std::string(k ? ", " : "") + "\"" + kname[k] + "\": [";
    for (int v = 0; v < hs::kVariants; v++) js += (v ? ", " : "") + std::to_string(ms[v]);
    js += "]";
  }
  js += "}";
  // 3. sub-batch streams T and stream overlap, timed end to end through
  //    hs_sign_batch_ex into a pinned buffer (each sub-batch's copy-out
  //    overlaps the later compute); keys "T" (FORS || TREE, concurrent
  //    sub-batches) and "T/serial" (one stream order)
  uint8_t* hout = nullptr;
  CUDA_TRY(h, cudaMallocHost(&hout, (size_t)count * I.sig_bytes));
  js += ", \"streams_ms\": {";
  int best_T = 1, best_ov = 1;
  double best_T_ms = 1e30;
  const int Ts[6] = {1, 2, 3, 4, 6, 8};
  int rc = HS_OK;
  for (int i = 0; i < 12 && rc == HS_OK; i++) {
    c.streams = Ts[i % 6];
    c.overlap = i < 6 ? 1 : 0;
    rc = hs_config_set(h, set, &c);
    if (rc == HS_OK) rc = hs_sign_batch_ex(h, set, msgs.data(), offs.data(), nullptr, nullptr, count, hout, nullptr);
    std::vector<float> w;
    for (int r = 0; r < reps && rc == HS_OK; r++) {
      const auto t0 = std::chrono::steady_clock::now();
      rc = hs_sign_batch_ex(h, set, msgs.data(), offs.data(), nullptr, nullptr, count, hout, nullptr);
      w.push_back((float)std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    if (rc != HS_OK) break;
    const double ms = trimmed_mean(w);
    js += (i ? ", \"" : "\"") + std::to_string(Ts[i % 6]) + (c.overlap ? "" : "/serial") + "\": " + std::to_string(ms);
    if (ms < best_T_ms) best_T_ms = ms, best_T = Ts[i % 6], best_ov = c.overlap;
  }
  cudaFreeHost(hout);
  if (rc != HS_OK) return rc;
  js += "}";
  c.streams = best_T;
  c.overlap = best_ov;
  // 4. batch-size rules (batch_config), graph device time on smaller batches
  //    of the same messages: (a) when one stream order won at `count`, the
  //    largest of count/2, count/4, ... (>= 16) at which the concurrent
  //    branches are faster becomes the overlap threshold; (b) one FORS tree
  //    per CTA and (c) the warp-shuffle Merkle reduction (tree_split 1 for a
  //    tree_split 2 config) are each kept for graphs up to the largest of 16,
  //    64, 256 messages at which they are faster by more than 2 %.
  auto graph_ms = [&](uint32_t n, double& ms) -> int {
    if (int r = hs_config_set(h, set, &c); r != HS_OK) return r;
    if (int r = stage_inputs(h, set, 0, msgs.data(), offs.data(), nullptr, nullptr, 0, n, false); r != HS_OK) return r;
    if (int r = time_graph(h, set, n, 2, t); r != HS_OK) return r;  // warm-up, graph capture
    if (int r = time_graph(h, set, n, reps, t); r != HS_OK) return r;
    ms = trimmed_mean(t);
    return HS_OK;
  };
  c.fors_small_batch = 0;
  c.tree_small_batch = 0;
  js += ", \"overlap_ms\": {";
  if (best_ov == 0) {
    bool firstk = true;
    for (uint32_t n = count / 2; n >= 16; n /= 2) {
      double m1, m0;
      c.overlap = 1;
      if (int r = graph_ms(n, m1); r != HS_OK) return r;
      c.overlap = 0;
      if (int r = graph_ms(n, m0); r != HS_OK) return r;
      char b[96];
      snprintf(b, sizeof b, "%s\"%u\": [%.4f, %.4f]", firstk ? "" : ", ", n, m1, m0);
      js += b;
      firstk = false;
      if (m1 < m0) {
        c.overlap = n >= 2 ? (int)n : 1;
        break;
      }
    }
  }
  js += "}, \"small_batch_ms\": {";
  const int small_ov = c.overlap;
  int small = 0;
  for (uint32_t n : {16u, 64u, 256u}) {
    if (n > count) break;
    double tuned, one_tree;
    c.fors_small_batch = 0;
    if (int r = graph_ms(n, tuned); r != HS_OK) return r;
    c.fors_small_batch = (int)n;
    if (int r = graph_ms(n, one_tree); r != HS_OK) return r;
    char b[96];
    snprintf(b, sizeof b, "%s\"%u\": [%.4f, %.4f]", n == 16 ? "" : ", ", n, tuned, one_tree);
    js += b;
    if (!(one_tree < tuned * 0.98)) break;
    small = (int)n;
  }
  js += "}, \"tree_small_batch_ms\": {";
  c.fors_small_batch = small;
  int tsmall = 0;
  for (uint32_t n : {16u, 64u, 256u}) {
    if (n > count || c.tree_split != 2) break;
    double grid, shuffle;
    c.tree_small_batch = 0;
    if (int r = graph_ms(n, grid); r != HS_OK) return r;
    c.tree_small_batch = (int)n;
    if (int r = graph_ms(n, shuffle); r != HS_OK) return r;
    char b[96];
    snprintf(b, sizeof b, "%s\"%u\": [%.4f, %.4f]", n == 16 ? "" : ", ", n, grid, shuffle);
    js += b;
    if (!(shuffle < grid * 0.98)) break;
    tsmall = (int)n;
  }
  js += "}";
  c.tree_small_batch = tsmall;
  c.overlap = small_ov;
  if (int r = stage_inputs(h, set, 0, msgs.data(), offs.data(), nullptr, nullptr, 0, count, false); r != HS_OK)
    return r;
  c.chunk = base.chunk;
  if (int r2 = hs_config_set(h, set, &c); r2 != HS_OK) return r2;
  js += ", \"config\": " + cfg_json(c) + "}";
  if (json && cap) {
    std::strncpy(json, js.c_str(), cap - 1);
    json[cap - 1] = '\0';
  }
  return js.size() + 1 > cap ? (int)(js.size() + 1) : HS_OK;
}

void* hs_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, std::max<size_t>(bytes, 1)) != cudaSuccess) return nullptr;
  return p;
}

void hs_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
