// hs_set.cu -- per-parameter-set kernel instantiation and launch table.
// Compiled three times with -DHS_SET=0/1/2 so the heavy template
// instantiations build in parallel.
#include <cuda_runtime.h>

#include "hs_internal.h"
#include "hs_kernels.cuh"

#ifndef HS_SET
#error "compile with -DHS_SET=<0|1|2>"
#endif

namespace hs {

namespace {

template <int S, class V>
cudaError_t launch_v(int which, const LaunchArgs& a, cudaStream_t s) {
  using Pr = P<S>;
  auto blocks = [](uint64_t threads, int b) { return (unsigned)((threads + b - 1) / b); };
  switch (which) {
    case K_KEYSETUP:
      if (a.nkeys == 0) return cudaSuccess;
      key_setup_kernel<S, Native><<<blocks(a.nkeys, 64), 64, 0, s>>>(a);
      break;
    case K_PREP:
      msg_prep_kernel<S, Native><<<blocks(a.count, 64), 64, 0, s>>>(a);
      break;
    case K_FORS: {
      const bool relax = a.fors_relax != 0;
      const int lanes = a.fors_trees_per_set * (relax ? Pr::t / 2 : Pr::t);
      const int tpc = a.fors_trees_per_set * a.fors_sets_fused;
      const int sets_total = (Pr::k + a.fors_trees_per_set - 1) / a.fors_trees_per_set;
      const int passes = (sets_total + a.fors_sets_fused - 1) / a.fors_sets_fused;
      const size_t smem = ((size_t)tpc * fors_smem_words_per_tree<S>(relax) + kForsPrefixWords) * 4;
      cudaError_t e = cudaFuncSetAttribute(fors_sign_kernel<S, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      fors_sign_kernel<S, V><<<(unsigned)((uint64_t)a.count * passes), lanes, smem, s>>>(a);
      break;
    }
    case K_FORSPK:
      fors_pk_kernel<S, Native><<<blocks(a.count, kSmallBlock), kSmallBlock, 0, s>>>(a);
      break;
    case K_TREE:
      tree_sign_kernel<S, V><<<blocks((uint64_t)a.count * (Pr::d - a.shared_layers) * Pr::leaves, kTreeBlock),
                               kTreeBlock, 0, s>>>(a);
      break;
    case K_TREE_SHARED:
      if (a.shared_layers <= 0 || a.nkeys == 0) return cudaSuccess;
      tree_shared_kernel<S, V><<<blocks((uint64_t)a.nkeys * Shared<S>::units(a.shared_layers) * Pr::leaves,
                                        kTreeBlock),
                                 kTreeBlock, 0, s>>>(a);
      break;
    case K_WOTS:
      wots_sign_kernel<S, V><<<blocks((uint64_t)a.count * Pr::d * Pr::wots_len, kSmallBlock), kSmallBlock, 0, s>>>(a);
      break;
    case K_KEYGEN:
      keygen_root_kernel<S, V><<<blocks((uint64_t)a.nkeys * Pr::leaves, kTreeBlock), kTreeBlock, 0, s>>>(a);
      break;
    case K_WOTS_GATHER:
      wots_gather_kernel<S><<<blocks((uint64_t)a.count * Pr::d * Pr::wots_len, kSmallBlock), kSmallBlock, 0, s>>>(a);
      break;
    case K_VERIFY:
      verify_kernel<S, Native><<<blocks(a.count, kVerifyWarps), 32 * kVerifyWarps, 0, s>>>(a);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

template <>
cudaError_t launch_kernel<HS_SET>(int which, int variant, const LaunchArgs& a, cudaStream_t s) {
  // message preparation, key setup, T_k and verification are a vanishing
  // share of the work: launch_v instantiates them with the native path only
  return variant ? launch_v<HS_SET, Fast>(which, a, s) : launch_v<HS_SET, Native>(which, a, s);
}

template <>
size_t shared_words_per_key<HS_SET>(int layers) {
  return (size_t)Shared<HS_SET>::units(layers) * Shared<HS_SET>::rec_words;
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
