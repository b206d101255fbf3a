/*
 * b2l.h -- C ABI of the B200-native hash + trace-analysis engine
 * (libb2l.so, built from paper_2601_12713_b200/csrc/).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as void* = cudaStream_t, NULL = legacy default stream).
 * Every entry point returns B2L_OK (0) or a negative B2L_E_* code; the
 * message of the last failure on the calling thread is b2l_last_error().
 *
 * Reference interfaces replaced (paths relative to the reference checkout):
 *   b2l_hash_batch / b2l_hash_host / b2l_hash_bytes
 *       -> dmlens.hashing._fold64 + make_hasher + hash_bytes
 *          pkg/src/dmlens/hashing.py:34-67 (HashFn = Callable[[bytes], int], :26)
 *   b2l_analyze -> dmlens.detectors.analyze  pkg/src/dmlens/detectors.py:274-326
 *          (validate model.py:125-200, get_alloc_delete_pairs prep.py:45-96,
 *           the five detectors detectors.py:85-271)
 *   b2l_savings -> integer parts of dmlens.estimator.estimate estimator.py:61-130
 *          and dmlens.report.attribute report.py:44-95
 * See INTEGRATION.md for the ctypes binding the reference would add.
 */
#ifndef B2L_H
#define B2L_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2L_ABI_VERSION 1

enum {
    B2L_OK = 0,
    B2L_E_INVALID_ARG = -1,
    B2L_E_EMPTY_PAYLOAD = -2,   /* dmlens.hashing.EmptyPayload (hashing.py:29-31) */
    B2L_E_INVALID_TRACE = -3,   /* dmlens.detectors.InvalidTrace (detectors.py:79-82) */
    B2L_E_DEVICE_RANGE = -4,    /* dmlens.prep.DeviceOutOfRange (prep.py:35-39) */
    B2L_E_CUDA = -5,
    B2L_E_OOM = -6,
    B2L_E_MISMATCH = -7,        /* dmlens.estimator.FindingsTraceMismatch (estimator.py:35-38) */
    B2L_E_NO_DEVICE = -8
};

int b2l_abi_version(void);
const char *b2l_last_error(void);
int b2l_device_count(int *count);

/* ---------------------------------------------------------------- hashing
 * Digest of buffer i = the reference _fold64 (FNV-1a-64 over little-endian
 * u64 words, zero-extended tail word, ^len, murmur3 fmix64, 0 -> 1).
 * Buffers may have any alignment.  A zero-length buffer gets digest 0 (the
 * reserved "no hash" value; the reference raises EmptyPayload instead, which
 * the host wrapper does when it sees a zero length).
 *
 * b2l_hash_batch: d_ptrs / d_lens / d_digests / d_order are DEVICE arrays of
 * n entries.  d_order (nullable) is a permutation giving the processing
 * order (the host wrapper passes a longest-first order for ragged batches);
 * digests are always written at the buffer's own index.  Asynchronous on
 * `stream`.
 */
int b2l_hash_batch(const uint64_t *d_ptrs, const uint64_t *d_lens, uint64_t n,
                   uint64_t *d_digests, const uint32_t *d_order, void *stream);

/* Host buffers (pinned for full speed; pageable works) -> host digests.
 * Copies run on a side stream through a double-buffered device ring and
 * overlap with hashing.  Synchronous.  Returns B2L_E_EMPTY_PAYLOAD if any
 * length is zero (digests of the others are still written). */
int b2l_hash_host(const void *const *h_bufs, const uint64_t *h_lens, uint64_t n,
                  uint64_t *h_digests);

/* One host payload (the HashFn drop-in). */
int b2l_hash_bytes(const void *h_buf, uint64_t len, uint64_t *digest);

/* Synthetic payload generator (bench / tests): buffer b occupies
 * d_base + h-supplied offsets[b], length lens[b], content = counter-based
 * splitmix64 stream of (seed, content_ids[b]); equal content ids give
 * byte-identical payloads.  Device arrays.  Asynchronous. */
int b2l_fill_payloads(uint8_t *d_base, const uint64_t *d_offsets, const uint64_t *d_lens,
                      const uint64_t *d_content_ids, uint64_t n, uint64_t seed, void *stream);

/* Kernel variant selection (tuning / tests): variant -1 only reports the
 * number of variants in *count, -2 restores the default (the tuned variant,
 * DESIGN.md K1).  Process-wide. */
int b2l_hash_select_variant(int variant, int *count);

/* Device-side occupancy/launch info of the hash kernel (diagnostics). */
int b2l_hash_launch_info(uint64_t n, int *grid, int *block, int *smem_bytes);

#ifdef __cplusplus
}
#endif
#endif /* B2L_H */
