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
 * overlap with hashing; small calls (<= 64 buffers, <= 64 KiB) are packed into
 * one pinned block and moved by a single copy each way.  Synchronous.  Returns B2L_E_EMPTY_PAYLOAD if any
 * length is zero (digests of the others are still written). */
int b2l_hash_host(const void *const *h_bufs, const uint64_t *h_lens, uint64_t n,
                  uint64_t *h_digests);

/* One DEVICE buffer hashed by the whole GPU (K2: exact 4-bit-group decomposition of the
 * serial fold, cooperative launch).  For buffers whose serial chain would dominate a batch
 * (b2l_hash_host routes buffers >= 32 MiB here automatically, and a call holding a single
 * buffer from 96 KiB).  Asynchronous. */
int b2l_hash_large(const void *d_buf, uint64_t len, uint64_t *d_digest, void *stream);

/* n huge DEVICE buffers (host array of device addresses + host lengths) -> d_digests[0..n)
 * (device).  K2 over several buffers per cooperative launch (up to 16, longest first), each
 * with its own share of the CTAs, so one buffer's cross-CTA waits overlap the others'
 * arithmetic.  Same digests as n b2l_hash_large calls (hashing.py:34-52 per buffer).
 * Asynchronous on `stream`; B2L_E_EMPTY_PAYLOAD if any length is zero. */
int b2l_hash_large_many(const void *const *d_bufs, const uint64_t *lens, uint64_t n,
                        uint64_t *d_digests, void *stream);

/* One host payload (the HashFn drop-in). */
int b2l_hash_bytes(const void *h_buf, uint64_t len, uint64_t *digest);

/* Synthetic payload generator (bench / tests): buffer b occupies
 * d_base + h-supplied offsets[b], length lens[b], content = counter-based
 * splitmix64 stream of (seed, content_ids[b]); equal content ids give
 * byte-identical payloads.  Device arrays.  Asynchronous. */
int b2l_fill_payloads(uint8_t *d_base, const uint64_t *d_offsets, const uint64_t *d_lens,
                      const uint64_t *d_content_ids, uint64_t n, uint64_t seed, void *stream);

/* Collision audit (hashing.py:70-92 CollisionAuditStore.observe over n observations in
 * order, used by `dmlens audit`, cli.py:206-236): observation i = (d_hashes[i], payload at
 * d_ptrs[i] of d_lens[i] bytes), device arrays.  *collisions = observations whose payload
 * differs from the first payload seen with the same hash; *distinct = distinct hashes
 * (len(store)).  Synchronous. */
int b2l_audit_batch(const uint64_t *d_hashes, const uint64_t *d_ptrs, const uint64_t *d_lens, uint64_t n,
                    uint64_t *collisions, uint64_t *distinct);

/* Native NDJSON ingest (traceio.py:153-191 wire format).  Parses the header and every
 * event record into columns (input order, not yet sorted or validated) over `threads`
 * host threads.  If any line is not a record the parser can vouch the reference accepts
 * without error, no columns are returned: err_line names the first such line (1-based) and
 * err_lines[0..n_err_lines) lists them (ascending; a header it cannot vouch for is listed
 * alone, body lines up to 64k per thread chunk).  The caller checks those lines the
 * reference's way (traceio.py:153-181): the first bad one raises the reference's exception,
 * unusual-but-valid ones are rewritten canonically and the input is parsed again.
 * Free with b2l_ingest_free. */
typedef struct b2l_ingest {
    uint64_t err_line;            /* 0 = every line accepted */
    uint64_t header_line;         /* 0 = no header line found */
    uint64_t version, num_devices, host_device, wall_time_ns;
    int32_t has_wall;
    uint64_t n_events;
    const uint64_t *seq, *start_ns, *end_ns, *src_device, *dst_device, *src_addr, *dst_addr, *bytes, *hash;
    const uint8_t *kind;
    const uint32_t *loc;
    uint32_t n_locs;
    const uint64_t *loc_codeptr;
    const int64_t *loc_line;      /* -1 = None */
    const uint64_t *loc_file_off; /* into strings; UINT64_MAX = None */
    const uint32_t *loc_file_len;
    const char *strings;          /* UTF-8 file names (lone surrogates in their 3-byte form) */
    uint64_t n_err_lines;
    const uint64_t *err_lines;
} b2l_ingest;
int b2l_ingest_ndjson(const char *data, uint64_t len, int threads, b2l_ingest **out);
void b2l_ingest_free(b2l_ingest *p);

/* serialize_trace (traceio.py:193-237) over HOST columns: `header` is the caller's rendered
 * header line (with its '\n'); every event then becomes
 *   {"seq":..,"kind":"..","t0":..,"t1":..,"src_dev":..,"dst_dev":..,"src_addr":..,"dst_addr":..,
 *    "bytes":..,"hash":..<suffix of its location>\n
 * where suffix_data[suffix_off[l] .. suffix_off[l+1]) is location l's pre-rendered tail
 * ',"codeptr":N[,"file":"<json-escaped>","line":L]}' (the only string data; escaped once per
 * location by the caller).  Events are written in column order over `threads` host threads.
 * The caller validates first (the reference refuses invalid traces).  *text is malloc'ed:
 * free with b2l_serialize_free. */
int b2l_serialize_ndjson(const struct b2l_trace_cols *cols, const char *header, uint64_t header_len,
                         const char *suffix_data, const uint64_t *suffix_off, int threads, char **text,
                         uint64_t *len);
void b2l_serialize_free(char *text);

/* Stable sort of n (k0, k1) u64 key pairs (host arrays): out_perm = sorting permutation
 * (parse_trace's events.sort(key=(start_ns, seq)), traceio.py:183). */
int b2l_sort_u64_pairs(const uint64_t *k0, const uint64_t *k1, uint64_t n, uint32_t *out_perm);
/* The same with DEVICE arrays (synchronous): the group orders of the multi-GPU merge on rank 0. */
int b2l_sort_u64_pairs_device(const uint64_t *d_k0, const uint64_t *d_k1, uint64_t n, uint32_t *d_perm);

/* Kernel variant selection (tuning / tests): variant -1 only reports the
 * number of variants in *count, -2 restores the default (the tuned variant,
 * DESIGN.md K1).  Process-wide. */
int b2l_hash_select_variant(int variant, int *count);

/* Device-side occupancy/launch info of the hash kernel (diagnostics). */
int b2l_hash_launch_info(uint64_t n, int *grid, int *block, int *smem_bytes);

/* ------------------------------------------------------------ trace analysis
 * Event i is trace.events[i].  Kinds: */
enum { B2L_KIND_TRANSFER = 0, B2L_KIND_ALLOC = 1, B2L_KIND_DELETE = 2, B2L_KIND_KERNEL = 3 };
/* Per-location validation flags (model.py:186-190). */
enum { B2L_LOC_FILE_NO_LINE = 1, B2L_LOC_LINE_NONPOS = 2 };
/* Violated-rule bits per event, in the order model.py:125-200 reports them. */
enum {
    B2L_RULE_INTERVAL = 1 << 0,      /* "interval": start_ns > end_ns */
    B2L_RULE_SRC_DEVICE = 1 << 1,    /* "device": src_device out of range */
    B2L_RULE_DST_DEVICE = 1 << 2,    /* "device": dst_device out of range */
    B2L_RULE_TRANSFER_HASH = 1 << 3, /* "transfer": non-empty transfer has no content hash */
    B2L_RULE_ALLOC_BYTES = 1 << 4,   /* "alloc": allocation of zero bytes */
    B2L_RULE_ALLOC_ADDR = 1 << 5,    /* "alloc": allocation with null device address */
    B2L_RULE_DELETE_ADDR = 1 << 6,   /* "delete": deletion with null device address */
    B2L_RULE_KERNEL_DEVICE = 1 << 7, /* "kernel": kernel src_device must equal dst_device */
    B2L_RULE_LOC_FILE = 1 << 8,      /* "location": file present but line missing */
    B2L_RULE_LOC_LINE = 1 << 9,      /* "location": line must be positive */
    B2L_RULE_ORDER_SORT = 1 << 10,   /* "order": events not sorted by (start_ns, seq) */
    B2L_RULE_ORDER_SEQ = 1 << 11     /* "order": seq values not strictly increasing */
};
enum {
    B2L_ANALYZE_STRICT_RT = 1,      /* analyze(strict_pseudocode=True), detectors.py:145-160 */
    B2L_ANALYZE_VALIDATE_ONLY = 2,  /* stop after validation (sharded analysis validates shards) */
    B2L_ANALYZE_SYNTH_END = 4,      /* b2l_analyze_ex: use the given synthetic-delete time (prep.py:61-62
                                       max end over ALL data ops -- a trace-wide value for a shard) */
    B2L_ANALYZE_SKIP_DDRT = 8,      /* shard holds no hash-keyed work: skip DD / RT */
    B2L_ANALYZE_SKIP_ALLOC = 16,    /* shard holds no device-keyed work: skip pairs / RA / UA / UT */
    B2L_ANALYZE_NO_VALIDATE = 32,   /* standalone detectors (find_*) take event lists as given */
    B2L_ANALYZE_RAW_HASHED = 64,    /* DD/RT over every transfer row (find_duplicate_transfers /
                                       find_round_trips group whatever they are given) */
    B2L_ANALYZE_WITH_SAVINGS = 128  /* also compute b2l_savings_compute's results (estimate + attribute
                                       aggregates), category by category as the detector chains finish;
                                       the next b2l_savings_compute of the same columns returns them */
};
#define B2L_SYNTHETIC 0xFFFFFFFFu   /* pair_delete of a synthetic trace-end delete (prep.py:78-93) */

/* Trace columns (structure of arrays, one entry per event). */
typedef struct b2l_trace_cols {
    uint64_t n_events;
    int32_t num_devices_total;
    int32_t host_device;
    const uint64_t *seq, *start_ns, *end_ns, *src_addr, *dst_addr, *bytes, *hash;
    const int32_t *src_device, *dst_device;
    const uint8_t *kind;       /* B2L_KIND_* */
    const uint32_t *loc;       /* per event: location id < n_locs */
    uint32_t n_locs;
    const uint8_t *loc_flags;  /* per location: B2L_LOC_* */
    const uint32_t *loc_bucket;/* per location: attribution bucket id < n_buckets (report.py:67-70) */
    uint32_t n_buckets;
    int32_t device_resident;   /* 1: every array above is a device pointer, 0: host pointers */
} b2l_trace_cols;

/* Findings in columnar form.  Engine-owned HOST arrays (b2l_findings_free);
 * event indices are positions in the trace, pair indices positions in pair_*.
 * Orders are the reference's: groups as sorted by detectors.py:102/166/180,
 * members in trace order, pairs by allocation (prep.py:95), lists by (start, seq). */
typedef struct b2l_findings {
    uint64_t n_events;
    /* validation: events violating >= 1 rule, ascending, with their B2L_RULE_* bits */
    uint64_t n_bad;
    uint32_t *bad_index, *bad_rules;
    /* DD (detectors.py:85-103): dd_offsets[g]..dd_offsets[g+1] index dd_members */
    uint64_t dd_groups;
    uint64_t *dd_offsets;
    uint32_t *dd_members;
    /* RT (detectors.py:106-167): trips rt_tx[t] -> rt_rx[t] */
    uint64_t rt_groups;
    uint64_t *rt_offsets;
    uint32_t *rt_tx, *rt_rx;
    /* alloc/delete pairs (prep.py:45-96), one per allocation, in allocation order */
    uint64_t n_pairs;
    uint32_t *pair_alloc, *pair_delete;  /* B2L_SYNTHETIC = synthetic trace-end delete */
    uint64_t synthetic_end_ns;           /* start/end of the synthetic deletes (max data-op end) */
    uint64_t n_warnings;                 /* unmatched deletes, trace order (prep.py:73-76) */
    uint32_t *warn_index;
    /* RA (detectors.py:170-191): groups of pair indices */
    uint64_t ra_groups;
    uint64_t *ra_offsets;
    uint32_t *ra_pairs;
    /* UA (detectors.py:194-229): pair indices; UT (detectors.py:232-271): event indices */
    uint64_t n_ua;
    uint32_t *ua_pairs;
    uint64_t n_ut;
    uint32_t *ut_events;
    void *internal;  /* engine state (device copies for b2l_savings) */
} b2l_findings;

/* analyze(trace, warn, strict_pseudocode).  Returns B2L_E_INVALID_TRACE when any
 * event violates a rule (only n_bad / bad_* are filled) -- header rules
 * (num_devices_total, host_device) are the caller's.  *out must be freed with
 * b2l_findings_free (also on B2L_E_INVALID_TRACE). */
int b2l_analyze(const b2l_trace_cols *cols, uint32_t flags, b2l_findings **out);
/* Shard form used by the multi-GPU analysis (paper_2601_12713_b200/sharded.py). */
int b2l_analyze_ex(const b2l_trace_cols *cols, uint32_t flags, uint64_t synthetic_end_ns, b2l_findings **out);
void b2l_findings_free(b2l_findings *f);

typedef struct b2l_u128 { uint64_t lo, hi; } b2l_u128;

/* Integer parts of estimate() (estimator.py:61-130) and attribute() (report.py:44-95)
 * for findings given as a b2l_findings (from b2l_analyze, or filled by the caller
 * with host arrays -- then `internal` must be NULL).  Sums are exact 128-bit. */
typedef struct b2l_savings {
    b2l_u128 per_category_ns[5];  /* DD, RT, RA, UA, UT */
    b2l_u128 union_ns;
    uint64_t n_union;
    uint32_t *union_index;        /* eliminable events, ascending (engine-owned host array) */
    int32_t has_overlaps;         /* estimator.py:51-58 */
    uint64_t min_start_ns, max_end_ns;
    uint32_t n_buckets;
    /* per category c (0..4) and bucket b, at [c * n_buckets + b]: */
    uint64_t *attr_count;
    b2l_u128 *attr_ns, *attr_bytes;
    uint64_t *attr_first;         /* (multiset position << 32) | event index of the first member;
                                     UINT64_MAX when the bucket has no member */
    void *internal;               /* engine-owned pinned memory behind the arrays above */
} b2l_savings;
int b2l_savings_compute(const b2l_trace_cols *cols, const b2l_findings *f, b2l_savings **out);
void b2l_savings_free(b2l_savings *s);

/* Stable sort of n u32 keys (host arrays): out_perm[i] = index of the i-th smallest key
 * (equal keys keep their order) -- sort_by_device (prep.py:99-115). */
int b2l_stable_sort_u32(const uint32_t *keys, uint64_t n, uint32_t *out_perm);

/* Stable sort of n u64 keys (host arrays) with one of the engine's strategies -- the grouping
 * sorts behind detectors.py:85-191 (content hashes, group orders); exposed so the tests can
 * drive each strategy with adversarial keys.  strategy: 0 = LSD over the live bytes,
 * 1 = wide (LSD over the top live bytes + segmented fix-up of equal-prefix runs),
 * 16 + b = LSD over live bytes >= b, then the fix-up. */
int b2l_stable_sort_u64(const uint64_t *keys, uint64_t n, uint32_t strategy, uint32_t *out_perm);

/* Positions of `n` seq values in the trace's seq column (ascending seq, as in a
 * validated trace); UINT32_MAX when absent.  Host arrays. */
int b2l_lookup_seqs(const b2l_trace_cols *cols, const uint64_t *seqs, uint64_t n, uint32_t *out_index);

/* Key-range sharding (the reference has no multi-process analysis -- these route
 * the events detectors.py:85-271 relate so that each rank's sub-traces are exact):
 * b2l_shard_kernel_summary: per target device (num_devices_total entries) of a device-resident
 * shard: has_kernels (0/1) and the max end of its target kernels.  All-gathered, these give
 * every rank the carry of the shards before it.
 * b2l_shard_route: for a device-resident seq-range shard whose first event has global index
 * `base`, writes one 12 x i64 row per record into d_rows, grouped by destination rank in event
 * order: space 0 -- hashed transfers to the owner of their hash range ((hash * n_ranks) >> 64);
 * space 1 -- allocs and deletes to the pairing owner of (dst_device, dst_addr) ((dst_device +
 * owner(mix(dst_addr))) % n_ranks), target transfers to the owner of (dst_device, src_addr),
 * and the target kernels those ranks need for exact UA/UT cursors: each target transfer's /
 * target alloc's cursor kernel (to that query's rank), the shard's first kernel of every device
 * (to every rank), and at the head of every rank's block one carry kernel per device whose
 * carry_max_end (the max kernel end on earlier shards; carry_has[d] = any) reaches the shard's
 * first start (owner(key) = top 32 bits of a splitmix64 mix of the key, times n_ranks, >> 32).
 * Row: [global index | space << 63, seq, start_ns, end_ns, src_addr, dst_addr, bytes, hash,
 * src_device, dst_device, kind, loc].  d_rows NULL: sizing call (*n_rows = an upper bound, and
 * data_end_ns); else capacity >= that bound, *n_rows is not updated and counts[r] = rows for
 * rank r.  data_end_ns = max end over non-kernel events (prep.py:61-62's synthetic delete time).
 * b2l_shard_route_pairs: the second exchange.  For a device sub-trace (global indices d_gid) and
 * its alloc/delete pairs (indices, delete 0xFFFFFFFF = synthetic), every pair's alloc and real
 * delete go to the owner of the RA key (alloc src_addr, dst_device, bytes; detectors.py:170-176)
 * as space-1 rows, sub-trace order per destination.  d_rows NULL: sizing call.
 * b2l_shard_unpack: received rows of one space -> device columns d_cols[0..11] (global index,
 * seq, start, end, src_addr, dst_addr, bytes, hash as i64; src, dst as i32; kind u8; loc u32),
 * capacity n_rows each; *n_out = rows of that space. */
int b2l_shard_kernel_summary(const b2l_trace_cols *cols, uint64_t *has_kernels, uint64_t *max_kernel_end);
int b2l_shard_route(const b2l_trace_cols *cols, uint32_t n_ranks, uint64_t base, uint32_t flags,
                    const uint8_t *carry_has, const uint64_t *carry_max_end, int64_t *d_rows, uint64_t *counts,
                    uint64_t *n_rows, uint64_t *data_end_ns);
int b2l_shard_route_pairs(const b2l_trace_cols *cols, const int64_t *d_gid, const uint32_t *d_pair_alloc,
                          const uint32_t *d_pair_delete, uint64_t n_pairs, uint32_t n_ranks, int64_t *d_rows,
                          uint64_t *counts, uint64_t *n_rows);
int b2l_shard_unpack(const int64_t *d_rows, uint64_t n_rows, uint32_t space, int64_t *const *d_cols,
                     uint64_t *n_out);

/* ---------------------------------------------------------------- multi-GPU (one process)
 * SURVEY 8(b)/8(e).  b2l_init(ngpus, devs): the devices this process drives (devs NULL:
 * 0..ngpus-1; a device may repeat, e.g. for tests on one GPU); b2l_shutdown drains them.  The
 * single-device entry points keep using the calling thread's current device. */
int b2l_init(int ngpus, const int *devs);
int b2l_shutdown(void);
/* number of initialised devices (*n) and up to `cap` of their ordinals */
int b2l_ngpus(int *n, int *devs, int cap);
/* Placement of n buffers on `parts` devices by LPT (longest first, each to the least-loaded
 * part; ties to the lowest part, equal lengths in index order): owner[i] in [0, parts),
 * load[p] = bytes placed on part p (optional).  Host arrays. */
int b2l_lpt_partition(const uint64_t *lens, uint64_t n, uint32_t parts, uint32_t *owner, uint64_t *load);
/* b2l_hash_host over every initialised device: contiguous byte-balanced ranges of the batch, one
 * host thread per device (its own pipeline and PCIe link), digests written in place into
 * h_digests.  Same contract as b2l_hash_host (hashing.py:34-67 per buffer). */
int b2l_hash_host_multi(const void *const *h_bufs, const uint64_t *h_lens, uint64_t n, uint64_t *h_digests);

/* ---------------------------------------------------------------- capture agent
 * Native model of the reference's OMPT capture shim (SPEC.md "ompt-shim",
 * pkg/shim/src/capture.ts:93-327): paired begin/end callbacks -> trace events, per-thread
 * buffers merged by (t0, arrival), runtime device ids -> dense slots (host at slot 0).
 * Transfer payloads are hashed on the GPU where they live: `device_buffer` (the landed
 * destination of a host-to-device copy at end, the source of a device-to-host copy) with K1/K2
 * synchronously in the callback; `host_buffer` only when the runtime offers nothing else
 * (host-to-device at begin, device-to-host at end, capture.ts:210,262).  time_ns = UINT64_MAX:
 * the agent's monotonic clock (origin at create).  Data-op types are OMPT's
 * ompt_target_data_op_t values.  A device buffer is hashed on its own GPU (found with
 * cudaPointerGetAttributes; one agent stream per device; the caller's current device is kept).
 * A payload that cannot be hashed never drops the event: it is emitted opaque (bytes 0, hash 0,
 * counted in hash_skipped), exactly as capture.ts:212-217 records an unreadable one. */
typedef struct b2l_capture b2l_capture;
enum { B2L_CAPTURE_BEGIN = 1, B2L_CAPTURE_END = 2 };  /* ompt_scope_begin / ompt_scope_end */
enum { B2L_OP_ALLOC = 1, B2L_OP_TO_DEVICE = 2, B2L_OP_FROM_DEVICE = 3, B2L_OP_DELETE = 4 };
b2l_capture *b2l_capture_create(int32_t host_runtime_id);
void b2l_capture_destroy(b2l_capture *c);
/* audit mode (payload sidecars "<seq>.bin"); the default comes from $DMLENS_AUDIT_DIR */
int b2l_capture_set_audit_dir(b2l_capture *c, const char *dir);
/* CaptureShim.deviceSlot (capture.ts:126-134) */
int32_t b2l_capture_device_slot(b2l_capture *c, int32_t runtime_id);
/* onTargetBegin / onTargetEnd (capture.ts:164-189) */
int b2l_capture_target(b2l_capture *c, int endpoint, uint64_t target_id, int32_t device_id, uint64_t codeptr,
                       uint64_t thread_id, uint64_t time_ns);
/* onDataOpBegin / onDataOpEnd (capture.ts:193-275) */
int b2l_capture_data_op(b2l_capture *c, int endpoint, uint64_t host_op_id, int optype, int32_t src_device,
                        int32_t dst_device, uint64_t src_addr, uint64_t dst_addr, uint64_t bytes, uint64_t codeptr,
                        uint64_t thread_id, uint64_t time_ns, const void *device_buffer, const void *host_buffer);
/* finalize (capture.ts:279-303): NDJSON text (free with b2l_capture_free_text); wall_time_ns =
 * UINT64_MAX derives it from the last event end.  Capture state is left untouched. */
int b2l_capture_finalize(b2l_capture *c, uint64_t wall_time_ns, char **text, uint64_t *len);
void b2l_capture_free_text(char *text);
/* writeTrace (capture.ts:305-321): out_path NULL -> $DMLENS_OUT (error if unset) */
int b2l_capture_write(b2l_capture *c, const char *out_path, uint64_t wall_time_ns);
/* ShimWarnings: [unmatched_ends, unfinished_at_exit, hash_skipped, dropped_malformed] */
int b2l_capture_warnings(b2l_capture *c, uint64_t *out4);

#ifdef __cplusplus
}
#endif
#endif /* B2L_H */
