/*
 * herosign_b200.h -- C-ABI of the B200 batched SPHINCS+-{128f,192f,256f}
 * signing engine (libherosign_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types.  The caller owns
 * every host buffer; the library owns device buffers, streams and CUDA
 * graphs.  One handle drives one device and is not reentrant; ctypes releases
 * the GIL around every call, so one host thread per handle drives 8 GPUs.
 *
 * Which reference interface each entry point replaces (paths relative to the
 * reference's pkg/src/herosign/):
 *
 *   hs_keygen_batch   sigcore.keygen            sigcore.py:62-72
 *   hs_keys_upload    HashContext.__init__      hashes.py:57-88 (per-key midstates)
 *   hs_sign_batch     sigcore.sign              sigcore.py:139-178, and the batch
 *                     driver cli bench / execute_graphs  batchgraph.py:110-226
 *   hs_sign_batch_ex  sigcore.sign + its ctx_out work counter  sigcore.py:166-168
 *   hs_verify_batch   sigcore.verify            sigcore.py:181-221
 *   hs_config_get/set TuningConfig per-set row  config.py:33-60 (fusion, relax,
 *                     backends row backends.py:201-257)
 *   hs_params         params.derive             params.py:97-149
 *   hs_tune           tuner.tree_tune + profile_kernels / select_backends
 *                     tuner.py:91-143, 184-274 (cli.py:119-148 `tune`)
 *   hs_stage/hs_run/hs_fetch
 *                     GraphSigner.prepare / run_fors|run_tree|run_wots
 *                     (batchgraph.py:288-353): the stage plugin, split so the
 *                     device part can be timed with inputs resident in HBM
 *
 * Parameter-set ids: 0 = "128f", 1 = "192f", 2 = "256f".
 * Return codes: 0 on success, negative on error (see HS_E_*); the message is
 * available from hs_last_error().  Usage-shaped errors map to the reference's
 * UsageError/FormatError/ConfigError (errors.py:8-37), CUDA failures to
 * HeroSignError.
 */
#ifndef HEROSIGN_B200_H
#define HEROSIGN_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HS_API __attribute__((visibility("default")))
#else
#define HS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HS_OK 0
#define HS_E_USAGE (-1)   /* bad argument / size          -> UsageError  */
#define HS_E_FORMAT (-2)  /* malformed key or signature   -> FormatError */
#define HS_E_CONFIG (-3)  /* infeasible layout / config   -> ConfigError */
#define HS_E_NOKEYS (-4)  /* sign before hs_keys_upload   -> UsageError  */
#define HS_E_CUDA (-10)   /* device / runtime failure     -> HeroSignError */

typedef struct hs_ctx hs_t;

/* Per-set tuning row (config.py:33-38 SetConfig, extended for B200). */
typedef struct {
  int32_t fors_trees_per_set; /* N_tree: trees sharing one set of lanes      */
  int32_t fors_sets_fused;    /* F: sets resident in one CTA's shared memory */
  int32_t fors_relax;         /* Relax_FORS: lanes build leaf pairs          */
  int32_t variant[4];         /* SHA-256 path per kernel: 0 native, 1 fast,
                                 2..5 the Mx<mask> paths (csrc/sha256.cuh
                                 VariantOf; backends.py:201-257 analog);
                                 [0] FORS_Sign, [1] TREE_Sign, [2] WOTS_Sign,
                                 [3] message preparation                     */
  int32_t use_graph;          /* 1: one CUDA graph launch per batch          */
  int32_t chunk;              /* messages per device pass in hs_sign_batch   */
  int32_t wots_from_tree;     /* 1: TREE_Sign records the signing leaf's
                                 chains and WOTS_Sign gathers them; 0: WOTS_Sign
                                 recomputes its chains (reference shape)     */
  int32_t streams;            /* T: concurrent sub-batch graphs per batch
                                 (paper's multi-stream batching), 1..8       */
  int32_t shared_layers;      /* top hypertree layers whose subtrees are
                                 computed once per (key, tree) per batch
                                 instead of once per message (0 = off; max
                                 6 for 128f/192f, 4 for 256f; only the
                                 subtrees the batch reads are computed)      */
  int32_t shared_auto;        /* 1: per batch, share a layer only when its
                                 subtrees per key are at most twice the key's
                                 messages (and within the table budget);
                                 0: share exactly shared_layers              */
  int32_t fors_cta_levels;    /* FORS tree levels reduced inside FORS_Sign's
                                 CTA; the levels above run as batch-wide
                                 one-level grids (fors_level_kernel).
                                 0 = leaves only (1 with Relax), log_t =
                                 whole tree in the CTA (reference shape,
                                 vexec.py:437-463), -1 = auto (leaves only:
                                 the measured best on B200)                  */
  int32_t tree_split;         /* TREE_Sign shape.  0: fused, one thread per
                                 leaf runs its chains, T_len and the warp-
                                 shuffle Merkle reduction; 1: one thread per
                                 WOTS chain, then one per leaf (T_len +
                                 warp-shuffle Merkle); 2: chain grid, leaf
                                 grid (T_len), then one thread per subtree
                                 for the Merkle levels                       */
  int32_t overlap;            /* 1: inside a batch graph, sub-batch j's
                                 FORS_Sign and TREE_Sign run on two streams
                                 and sub-batches run concurrently (priority
                                 ordered); 0: every kernel of the batch in one
                                 stream order -- sub-batches then only
                                 pipeline the signatures' D2H copies; N >= 2:
                                 streams for graphs of at most N messages,
                                 one stream order above (small batches leave
                                 the GPU idle without the concurrency)       */
  int32_t fors_small_batch;   /* graphs of at most this many messages run
                                 FORS_Sign with one tree per CTA (N_tree = F
                                 = 1; Relax and fors_cta_levels as set):
                                 k CTAs per message spread over the SMs
                                 instead of a few wide CTAs; 0 = off.  Bytes
                                 are unchanged (layouts never change them)   */
  int32_t tree_small_batch;   /* graphs of at most this many messages run a
                                 tree_split 2 config as tree_split 1: the
                                 subtree's Merkle levels as warp-shuffle
                                 combines (hp H's deep) instead of one thread
                                 walking all leaves-1 H's; 0 = off           */
} hs_set_config;

HS_API int hs_open(int device, hs_t **out);
HS_API void hs_close(hs_t *h);
HS_API const char *hs_last_error(const hs_t *h);

/* SM count, opt-in shared memory per block (bytes), compute capability. */
HS_API int hs_device_info(hs_t *h, int32_t *sm_count, int32_t *smem_optin, int32_t *cc_major, int32_t *cc_minor);

/* Derived constants of a set, same order as the reference DerivedParams
 * minus the id (n h d log_t k w lg_w len1 len2 wots_len subtree_height
 * subtree_leaves fors_t fors_msg_bytes tree_bits tree_bytes leaf_bits
 * leaf_bytes digest_bytes wots_sig_bytes fors_sig_bytes ht_sig_bytes
 * sig_bytes); returns the count written. */
HS_API int hs_params(int set, int32_t *fields, int cap);

HS_API int hs_config_get(hs_t *h, int set, hs_set_config *cfg);
HS_API int hs_config_set(hs_t *h, int set, const hs_set_config *cfg);
/* Shared-memory bytes one FORS CTA needs under a layout (feasibility check
 * for the tuner's S_max = opt-in smem). */
HS_API int64_t hs_fors_smem_bytes(int set, int32_t trees_per_set, int32_t sets_fused, int32_t relax);

/* Key table for a set: nkeys records of sk = sk_seed||sk_prf||pk_seed||pk_root. */
HS_API int hs_keys_upload(hs_t *h, int set, const uint8_t *sks, uint32_t nkeys);

/* Batched keygen: seeds (nkeys x 3n: sk_seed||sk_prf||pk_seed) -> sks (nkeys x 4n). */
HS_API int hs_keygen_batch(hs_t *h, int set, const uint8_t *seeds, uint32_t nkeys, uint8_t *sks_out);

/* Batched signing.  msgs is the concatenation of `count` messages with
 * offs[count+1] byte offsets; key_idx[count] selects a row of the uploaded
 * key table (NULL = row 0); opt_rand is count x n bytes (NULL = pk_seed,
 * the reference's deterministic default); sigs receives count x sig_bytes. */
HS_API int hs_sign_batch(hs_t *h, int set, const uint8_t *msgs, const uint64_t *offs, const uint32_t *key_idx,
                  const uint8_t *opt_rand, uint32_t count, uint8_t *sigs);

/* hs_sign_batch plus the exact work count: wots_steps[count] (nullable)
 * receives, per message, the WOTS_Sign F steps of its signature -- the sum of
 * the signed base-w digits over all d layers -- which is the only
 * data-dependent term of the reference's HashContext.compressions
 * (hashes.py:117-159, sigcore.py:166-168 ctx_out); the host adds the fixed
 * terms (params.compressions_per_signature).  Chunks of cfg.chunk messages
 * are pipelined: one chunk's staging and copy-out overlap the next one's
 * signing. */
HS_API int hs_sign_batch_ex(hs_t *h, int set, const uint8_t *msgs, const uint64_t *offs, const uint32_t *key_idx,
                            const uint8_t *opt_rand, uint32_t count, uint8_t *sigs, uint32_t *wots_steps);

/* Batched verification; ok[i] = 1 iff sig i verifies under pk row key_idx[i]
 * (pks: nkeys x 2n = pk_seed||pk_root).  sigs is count x sig_bytes. */
HS_API int hs_verify_batch(hs_t *h, int set, const uint8_t *pks, uint32_t nkeys, const uint8_t *msgs,
                    const uint64_t *offs, const uint32_t *key_idx, const uint8_t *sigs, uint32_t count,
                    uint8_t *ok);

/* Device-resident stages: hs_stage copies inputs into the library's device
 * buffers; hs_run signs the staged batch (mode 0: as one CUDA graph with the
 * FORS and TREE branches on two streams; mode 1: kernels serialised with a
 * CUDA event between each, for per-kernel timing); hs_fetch copies
 * signatures [first, first+count) back. */
HS_API int hs_stage(hs_t *h, int set, const uint8_t *msgs, const uint64_t *offs, const uint32_t *key_idx,
             const uint8_t *opt_rand, uint32_t count);
HS_API int hs_run(hs_t *h, int set, uint32_t count, int mode);
HS_API int hs_sync(hs_t *h);
HS_API int hs_fetch(hs_t *h, int set, uint32_t first, uint32_t count, uint8_t *sigs);

/* Device time (ms, CUDA events) of the last hs_run / hs_sign_batch pass:
 * [0] whole batch, [1] msg_prep, [2] FORS_Sign (+T_k), [3] TREE_Sign,
 * [4] WOTS_Sign.  Returns the number of values written. */
HS_API int hs_timings(hs_t *h, float *ms, int cap);

/* Benchmark loop over the staged batch: `steps` runs (mode as hs_run), each
 * bracketed by CUDA events on the launching stream; when flush_bytes > 0 a
 * device buffer of that size is rewritten between steps (outside the events)
 * to evict L2.  step_ms[steps] receives the per-step device times. */
HS_API int hs_bench_run(hs_t *h, int set, uint32_t count, int32_t steps, int mode, uint64_t flush_bytes,
                        float *step_ms);

/* Kernel launches issued by this handle since open (for bench accounting). */
HS_API int64_t hs_launch_count(hs_t *h);

/* Shape of the staged batch as the engine will run it: out[0] staged
 * messages, out[1] subtree-sharing depth chosen for it (shared_auto policy),
 * out[2] FORS levels kept in the CTA (fors_cta_levels resolved), out[3]
 * tree_split, out[4] shared subtrees its last run computed (synchronises the
 * handle's stream).  Returns the number of values written. */
HS_API int hs_batch_info(hs_t *h, int set, int32_t *out, int cap);

/* SHA-256 arithmetic paths compiled into this library (hs_set_config.variant
 * ids): returns their number n; id 0 is the native path, id 1 the fast path,
 * ids 2..n-1 are csrc/sha256.cuh Mx<mask> with masks[id-2] written to
 * masks[0..min(cap, n-2)).  The paper's per-kernel PTX/native choice
 * (reference backends.py:131-141 _COMPRESS registry) generalised. */
HS_API int hs_variants(int32_t *masks, int cap);

/* Batch launch latency (BASELINE.json metric): host time spent inside
 * cudaGraphLaunch, one call per signed batch (or per `chunk` of a larger
 * hs_sign_batch).  out[0] = graph launches, out[1] = mean us, out[2] = max us,
 * accumulated since the last reset; reset != 0 clears them after reading.
 * Returns the number of values written.  (No reference counterpart: the
 * reference's batchgraph.py:245-353 runs its DAG on host threads.) */
HS_API int hs_launch_stats(hs_t *h, double *out, int cap, int reset);

/* On-device Tree Tuning (reference tuner.py:91-143 Algorithm 1 and the
 * profiling / backend selection of tuner.py:184-274, driven from cli.py:119-148
 * `tune`), run on this handle's device over `count` synthetic 32-byte messages
 * signed with key row 0 (a fixed synthetic key when none is uploaded):
 *   1. every FORS layout (N_tree, F, Relax) Algorithm 1 admits at S_max = the
 *      device's opt-in shared memory is timed (FORS_Sign, CUDA events), the
 *      `top` fastest re-timed `reps` times, the best trimmed mean kept; then
 *      every split between in-CTA levels and level grids (fors_cta_levels);
 *   2. per kernel, every compiled SHA-256 path; a non-native path replaces
 *      native only when > 2% faster (the reference's tie rule);
 *   3. the sub-batch stream count T and stream overlap, timed end to end
 *      (hs_sign_batch_ex);
 *   4. the batch-size rules from graph device times on smaller batches: the
 *      overlap threshold (when one stream order won at `count`) and the
 *      largest of 16 / 64 / 256 messages at which one FORS tree per CTA
 *      (fors_small_batch) and the warp-shuffle Merkle reduction
 *      (tree_small_batch) win by more than 2%.
 * The handle is left configured with the result; json receives a report
 * (layouts, timings, final hs_set_config).  Returns 0, or the report's size
 * + 1 when cap is too small (truncated; the configuration is applied either
 * way), or a negative HS_E_* code. */
HS_API int hs_tune(hs_t *h, int set, uint32_t count, int32_t top, int32_t reps, char *json, size_t cap);

/* Page-locked host memory for zero-copy-staging callers (cudaMallocHost). */
HS_API void *hs_host_alloc(size_t bytes);
HS_API void hs_host_free(void *p);

#ifdef __cplusplus
}
#endif

#endif /* HEROSIGN_B200_H */
