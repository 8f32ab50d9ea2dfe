// hs_variants.h -- which SHA-256 arithmetic paths the library is built with.
// Variant id 0 = Native, 1 = Fast, 2.. = sha256.cuh Mx<mask, order> for each
// code below (code = mask + 256 * operand order) (override with make MASKS=...; tools/sha_sweep and
// tools/variant_sweep.py choose them from B200 timings of the real kernels).
#pragma once
#ifndef HS_MX_MASKS
#define HS_MX_MASKS 248, 232, 104, 1272
#endif
namespace hs {
constexpr int kMxMaskList[] = {HS_MX_MASKS};
constexpr int kVariants = 2 + (int)(sizeof(kMxMaskList) / sizeof(kMxMaskList[0]));
}  // namespace hs
