// hs_internal.h -- glue between the host runtime (hs_api.cu) and the
// per-set kernel objects (hs_set.cu compiled with -DHS_SET=0/1/2).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "hs_variants.h"

namespace hs {

struct LaunchArgs;


enum KernelId : int {
  K_KEYSETUP = 0,
  K_PREP = 1,
  K_FORS = 2,
  K_FORSPK = 3,
  K_TREE = 4,
  K_WOTS = 5,
  K_KEYGEN = 6,
  K_VERIFY = 7,
  K_WOTS_GATHER = 8,
  K_TREE_SHARED = 9,
  K_FORS_LEVEL = 10,
  K_TREE_CHAIN = 11,
  K_TREE_ROOT = 12,
  K_SHARED_CHAIN = 13,
  K_SHARED_ROOT = 14,
  K_TREE_MERKLE = 15,
  K_TREE_LEAF = 16,
};

// variant: SHA-256 arithmetic path id, 0..kNumVariants-1 (sha256.cuh VariantOf)
template <int S>
cudaError_t launch_kernel(int which, int variant, const LaunchArgs& a, cudaStream_t s);

// compression-heavy kernels of set S on path V (hs_var.cu)
template <int S, int V>
cudaError_t launch_variant(int which, const LaunchArgs& a, cudaStream_t s);

template <int S>
size_t fors_smem_bytes(int trees_per_set, int sets_fused, int relax);

template <int S>
size_t stash_words_per_msg();

template <int S>
size_t shared_words_per_key(int layers);

template <int S>
int shared_max_layers();

// words of the split shared-subtree chain-end buffer per key for `layers`
template <int S>
size_t shared_end_words_per_key(int layers);

}  // namespace hs
