// hs_set.cu -- per-parameter-set kernel instantiation and launch table.
// Compiled three times with -DHS_SET=0/1/2; the SHA-256-heavy kernels are
// instantiated per arithmetic path in hs_var.cu so the objects build in parallel.
#include <cuda_runtime.h>

#include "hs_internal.h"
#include "hs_kernels.cuh"

#ifndef HS_SET
#error "compile with -DHS_SET=<0|1|2>"
#endif

namespace hs {

namespace {

inline unsigned blocks_for(uint64_t threads, int b) { return (unsigned)((threads + b - 1) / b); }

template <int V>
cudaError_t launch_var(int which, int variant, const LaunchArgs& a, cudaStream_t s) {
  if constexpr (V >= kVariants) {
    return cudaErrorInvalidValue;
  } else {
    return variant == V ? launch_variant<HS_SET, V>(which, a, s) : launch_var<V + 1>(which, variant, a, s);
  }
}

}  // namespace

// Message preparation, key setup, T_k and the WOTS gather are a vanishing
// share of the work and use the native SHA-256 path (verification: Mx<248>); the
// compression-heavy kernels come from hs_var.cu, one object per (set, path).
template <>
cudaError_t launch_kernel<HS_SET>(int which, int variant, const LaunchArgs& a, cudaStream_t s) {
  constexpr int S = HS_SET;
  using Pr = P<S>;
  switch (which) {
    case K_KEYSETUP:
      if (a.nkeys == 0) return cudaSuccess;
      key_setup_kernel<S, Native><<<blocks_for(a.nkeys, 64), 64, 0, s>>>(a);
      return cudaGetLastError();
    case K_PREP:
      msg_prep_kernel<S, Native><<<blocks_for(a.count, 64), 64, 0, s>>>(a);
      return cudaGetLastError();
    case K_FORSPK:
      fors_pk_kernel<S, Native><<<blocks_for(a.count, kSmallBlock), kSmallBlock, 0, s>>>(a);
      return cudaGetLastError();
    case K_WOTS_GATHER:
      wots_gather_kernel<S><<<blocks_for((uint64_t)a.count * Pr::d * Pr::wots_len, kSmallBlock), kSmallBlock, 0,
                              s>>>(a);
      return cudaGetLastError();
    case K_VERIFY:
      // verification is ~86 % WOTS chain steps: the FMA-offload path of the
      // chain grids (+4..9 % at 65,536 signatures, profiles/r02aw_verify_ab_mx248.txt)
      verify_thread_kernel<S, Mx<248>><<<blocks_for(a.count, kVerifyThreads), kVerifyThreads, 0, s>>>(a);
      return cudaGetLastError();
    default:
      break;
  }
  return launch_var<0>(which, variant, a, s);
}

template <>
size_t shared_words_per_key<HS_SET>(int layers) {
  return (size_t)Shared<HS_SET>::units(layers) * Shared<HS_SET>::rec_words;
}

template <>
size_t shared_end_words_per_key<HS_SET>(int layers) {
  using Pr = P<HS_SET>;
  return (size_t)Shared<HS_SET>::units(layers) * Pr::leaves * Pr::wots_len * Pr::NW;
}

template <>
int shared_max_layers<HS_SET>() {
  return Shared<HS_SET>::max_layers;
}

template <>
size_t stash_words_per_msg<HS_SET>() {
  return (size_t)P<HS_SET>::d * P<HS_SET>::wots_len * P<HS_SET>::w * P<HS_SET>::NW;
}

template <>
size_t fors_smem_bytes<HS_SET>(int trees_per_set, int sets_fused, int relax) {
  return ((size_t)trees_per_set * sets_fused * fors_smem_words_per_tree<HS_SET>(relax != 0) + kForsPrefixWords) * 4;
}

}  // namespace hs
