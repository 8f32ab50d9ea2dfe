// hs_var.cu -- the compression-heavy kernels (FORS_Sign, TREE_Sign, shared
// subtrees, the WOTS chain kernel, keygen root) of one parameter set
// instantiated for one SHA-256 arithmetic path (sha256.cuh VariantOf<ID>).
// (+ the batch-wide upper FORS levels).  Compiled once per (HS_SET, HS_VAR) so the 18 objects build in parallel.
#include <cuda_runtime.h>

#include "hs_internal.h"
#include "hs_kernels.cuh"

#if !defined(HS_SET) || !defined(HS_VAR)
#error "compile with -DHS_SET=<0|1|2> -DHS_VAR=<0..kNumVariants-1>"
#endif

namespace hs {

static_assert(HS_VAR >= 0 && HS_VAR < kNumVariants, "unknown SHA-256 path");
static_assert(kVariants == kNumVariants, "hs_internal.h kVariants out of date");

template <>
cudaError_t launch_variant<HS_SET, HS_VAR>(int which, const LaunchArgs& a, cudaStream_t s) {
  constexpr int S = HS_SET;
  using V = typename VariantOf<HS_VAR>::T;
  using Pr = P<S>;
  auto blocks = [](uint64_t threads, int b) { return (unsigned)((threads + b - 1) / b); };
  switch (which) {
    case K_FORS: {
      const bool relax = a.fors_relax != 0;
      const int lanes = a.fors_trees_per_set * (relax ? Pr::t / 2 : Pr::t);
      const int tpc = a.fors_trees_per_set * a.fors_sets_fused;
      const int sets_total = (Pr::k + a.fors_trees_per_set - 1) / a.fors_trees_per_set;
      const int passes = (sets_total + a.fors_sets_fused - 1) / a.fors_sets_fused;
      // leaves-only CTAs (fors_cta_levels at its lowest) keep no tree levels in shared memory
      const bool leaves_only = a.fors_cta_levels == (relax ? 1 : 0);
      const size_t smem =
          ((leaves_only ? 0 : (size_t)tpc * fors_smem_words_per_tree<S>(relax)) + kForsPrefixWords) * 4;
      const unsigned grid = (unsigned)((uint64_t)a.count * passes);
      if constexpr (kForsNarrowLanes<S> > 0) {
        if (lanes <= kForsNarrowLanes<S>) {
          auto* k = fors_sign_kernel<S, V, kForsNarrowLanes<S>, kForsNarrowMinB<S>>;
          cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          if (e != cudaSuccess) return e;
          k<<<grid, lanes, smem, s>>>(a);
          break;
        }
      }
      cudaError_t e = cudaFuncSetAttribute(fors_sign_kernel<S, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      fors_sign_kernel<S, V><<<grid, lanes, smem, s>>>(a);
      break;
    }
    case K_FORS_LEVEL:
      fors_level_kernel<S, V><<<blocks((uint64_t)a.count * Pr::k * ((uint32_t)Pr::t >> a.fors_level), kForsLevelBlock),
                                kForsLevelBlock, 0, s>>>(a);
      break;
    case K_TREE:
      tree_sign_kernel<S, V><<<blocks((uint64_t)a.count * (Pr::d - a.shared_layers) * Pr::leaves, kTreeBlock),
                               kTreeBlock, 0, s>>>(a);
      break;
    case K_TREE_CHAIN:
      tree_chain_kernel<S, V><<<blocks((uint64_t)a.count * (Pr::d - a.shared_layers) * Pr::leaves * Pr::wots_len,
                                       kChainBlock<S>),
                                kChainBlock<S>, 0, s>>>(a);
      break;
    case K_TREE_ROOT:
      tree_root_kernel<S, V><<<blocks((uint64_t)a.count * (Pr::d - a.shared_layers) * Pr::leaves, kTreeBlock),
                               kTreeBlock, 0, s>>>(a);
      break;
    case K_TREE_LEAF:
      tree_leaf_kernel<S, V><<<blocks((uint64_t)a.count * (Pr::d - a.shared_layers) * Pr::leaves, kTreeBlock),
                               kTreeBlock, 0, s>>>(a);
      break;
    case K_TREE_MERKLE:
      tree_merkle_kernel<S, V><<<blocks((uint64_t)a.count * (Pr::d - a.shared_layers), kTreeBlock), kTreeBlock, 0,
                                 s>>>(a);
      break;
    case K_SHARED_CHAIN:
      if (a.shared_layers <= 0 || a.nkeys == 0) return cudaSuccess;
      shared_chain_kernel<S, V><<<blocks((uint64_t)a.nkeys * Shared<S>::units(a.shared_layers) * Pr::leaves *
                                             Pr::wots_len,
                                         kChainBlock<S>),
                                  kChainBlock<S>, 0, s>>>(a);
      break;
    case K_SHARED_ROOT:
      if (a.shared_layers <= 0 || a.nkeys == 0) return cudaSuccess;
      shared_root_kernel<S, V><<<blocks((uint64_t)a.nkeys * Shared<S>::units(a.shared_layers) * Pr::leaves,
                                        kTreeBlock),
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
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace hs
