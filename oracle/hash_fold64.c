/*
 * oracle/hash_fold64.c -- TEST INFRASTRUCTURE ONLY (CPU checker, never shipped).
 *
 * Plain-C restatement of the reference content hash:
 *   _fold64      /root/reference/pkg/src/dmlens/hashing.py:34-52
 *   make_hasher  /root/reference/pkg/src/dmlens/hashing.py:55-64   (n==0 rejected, 0 -> 1)
 *   TS port      /root/reference/pkg/shim/src/hash64.ts:13-41
 *
 * Pinned against the reference's frozen cross-language vectors
 * (pkg/shim/test/hash64.test.ts:8-24) and against digests produced by the
 * reference's own Python hash_bytes (tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker / the timed CPU baseline.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <pthread.h>

#define ORC_FNV_OFFSET 0xCBF29CE484222325ull
#define ORC_FNV_PRIME  0x100000001B3ull

static uint64_t orc_fmix64(uint64_t h) {
    h ^= h >> 33;
    h *= 0xFF51AFD7ED558CCDull;
    h ^= h >> 33;
    h *= 0xC4CEB9FE1A85EC53ull;
    h ^= h >> 33;
    return h;
}

/* Returns 0 only for n == 0 (the reference raises EmptyPayload there). */
uint64_t orc_hash_bytes(const uint8_t *p, uint64_t n) {
    if (n == 0) return 0;
    uint64_t h = ORC_FNV_OFFSET;
    uint64_t full = n >> 3, i;
    for (i = 0; i < full; i++) {
        uint64_t w = 0;
        for (int b = 7; b >= 0; b--) w = (w << 8) | p[i * 8 + b];  /* little-endian word */
        h = (h ^ w) * ORC_FNV_PRIME;
    }
    uint64_t tail = n & 7;
    if (tail) {
        uint64_t w = 0;
        for (int b = (int)tail - 1; b >= 0; b--) w = (w << 8) | p[full * 8 + b];
        h = (h ^ w) * ORC_FNV_PRIME;
    }
    h ^= n;
    h = orc_fmix64(h);
    return h ? h : 1;
}

void orc_hash_batch(const uint8_t *const *bufs, const uint64_t *lens, uint64_t n, uint64_t *out) {
    for (uint64_t i = 0; i < n; i++) out[i] = orc_hash_bytes(bufs[i], lens[i]);
}

/* Multi-threaded batch over host cores (CPU-baseline leg of bench.py). */
typedef struct { const uint8_t *const *bufs; const uint64_t *lens; uint64_t *out; uint64_t lo, hi; } orc_job;
static void *orc_worker(void *arg) {
    orc_job *j = (orc_job *)arg;
    for (uint64_t i = j->lo; i < j->hi; i++) j->out[i] = orc_hash_bytes(j->bufs[i], j->lens[i]);
    return NULL;
}
int orc_hash_batch_mt(const uint8_t *const *bufs, const uint64_t *lens, uint64_t n, uint64_t *out, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    orc_job jobs[256];
    for (int t = 0; t < threads; t++) {
        jobs[t].bufs = bufs; jobs[t].lens = lens; jobs[t].out = out;
        jobs[t].lo = n * (uint64_t)t / threads; jobs[t].hi = n * (uint64_t)(t + 1) / threads;
        if (pthread_create(&tid[t], NULL, orc_worker, &jobs[t]) != 0) return -1;
    }
    for (int t = 0; t < threads; t++) pthread_join(tid[t], NULL);
    return 0;
}

/* Counter-based payload generator shared by bench/tests:
 * word j of buffer b = splitmix64(seed ^ (b * GOLDEN) + j * C2) written little-endian. */
static uint64_t orc_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
uint64_t orc_payload_word(uint64_t seed, uint64_t content_id, uint64_t j) {
    return orc_splitmix64(seed ^ orc_splitmix64(content_id * 0xD1B54A32D192ED03ull + j));
}
void orc_fill_payload(uint8_t *dst, uint64_t nbytes, uint64_t seed, uint64_t content_id) {
    uint64_t nw = nbytes >> 3, j;
    for (j = 0; j < nw; j++) {
        uint64_t w = orc_payload_word(seed, content_id, j);
        memcpy(dst + j * 8, &w, 8);   /* x86/aarch64 hosts are little-endian */
    }
    if (nbytes & 7) {
        uint64_t w = orc_payload_word(seed, content_id, nw);
        memcpy(dst + nw * 8, &w, nbytes & 7);
    }
}
