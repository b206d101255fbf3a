// Capture agent (SPEC.md "ompt-shim"): turns paired begin/end OMPT-EMI
// callbacks into dmlens trace events, B200-side.  Behaviour follows the reference's model of
// the agent (pkg/shim/src/capture.ts:93-327): begin/end pairs become one event with both
// timestamps; per-thread append buffers merged at finalize by (t0, arrival) and renumbered;
// runtime device ids normalised to dense slots with the host at slot 0; malformed ops dropped
// and counted; unreadable transfers recorded opaque (bytes 0, hash 0); audit mode keeps a
// snapshot of every hashed payload for "<seq>.bin" sidecars.
//
// What is B200-native: payload hashing.  The reference hashes the host-side bytes on the CPU
// (capture.ts:210,262).  Here a transfer's DEVICE copy is hashed where it lives -- the
// destination of a host-to-device copy once it has landed (end callback), the source of a
// device-to-host copy -- with the K1 kernel on the agent's own stream, synchronously inside
// the callback (a later kernel of the program may overwrite the buffer, so the digest must be
// taken before the callback returns); buffers of 96 KiB and more go to K2 (whole GPU).  Host
// buffers, when that is all the runtime offers, are hashed on the GPU through b2l_hash_host.
// Digests equal hashing.hash_bytes (the shared contract, capture.ts:21 / hash64.ts).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <sys/stat.h>
#include <thread>
#include <unordered_map>
#include <vector>

#include "b2l_common.cuh"

namespace b2l {
int hash_batch_launch(const uint64_t *d_ptrs, const uint64_t *d_lens, uint64_t n, uint64_t *d_digests,
                      const uint32_t *d_order, cudaStream_t stream);
int hash_planes_launch(const void *d_buf, uint64_t nbytes, uint64_t *d_digest, cudaStream_t stream);
int hash_host_impl(const void *const *h_bufs, const uint64_t *h_lens, uint64_t n, uint64_t *h_digests);

namespace cap {

enum Kind : uint8_t { TRANSFER = 0, ALLOC = 1, DELETE = 2, KERNEL = 3 };
const char *kind_name(uint8_t k) {
    static const char *n[] = {"transfer", "alloc", "delete", "kernel"};
    return n[k & 3];
}

struct Ev {
    uint64_t provisional, t0, t1, src_addr, dst_addr, bytes, hash, codeptr;
    int32_t src_dev, dst_dev;
    uint8_t kind;
    uint64_t thread;
    std::vector<uint8_t> payload;  // audit snapshot
    bool has_payload = false;
};

struct Capture {
    int32_t host_runtime_id;
    std::chrono::steady_clock::time_point origin = std::chrono::steady_clock::now();
    std::atomic<uint64_t> provisional{0};
    std::mutex mu;  // device slots, pending maps and the buffer registry (never held while hashing)
    std::unordered_map<int32_t, int32_t> slots;
    std::unordered_map<uint64_t, Ev> pending_targets, pending_ops;
    // per-thread append buffers: each has its own (uncontended) lock, deques keep element
    // addresses stable, so a snapshot can read events while their threads keep appending
    struct Buf {
        std::mutex m;
        std::deque<Ev> v;
    };
    std::unordered_map<uint64_t, Buf *> buffers;
    std::vector<Buf *> owned;
    uint64_t unmatched_ends = 0, unfinished_at_exit = 0, hash_skipped = 0, dropped_malformed = 0;
    std::string audit_dir;  // empty: no payload snapshots
    // device hashing scratch: one stream + pinned argument block per device the agent has seen
    // (offload programs may map buffers on several GPUs; each buffer is hashed on its own GPU)
    struct DevScratch {
        cudaStream_t stream = nullptr;
        uint64_t *h_args = nullptr;  // pinned [ptr, len, digest], addressed by the kernels in place
    };
    std::unordered_map<int, DevScratch> dev_scratch;
    std::mutex hash_mu;

    explicit Capture(int32_t host_id) : host_runtime_id(host_id) {
        slots[host_id] = 0;
        if (const char *a = getenv("DMLENS_AUDIT_DIR")) audit_dir = a;
    }
    ~Capture() {
        for (auto *b : owned) delete b;
        for (auto &d : dev_scratch) {
            if (d.second.h_args) cudaFreeHost(d.second.h_args);
            if (d.second.stream) cudaStreamDestroy(d.second.stream);
        }
    }
    uint64_t now() const {
        return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() -
                                                                              origin)
            .count();
    }
    int32_t slot_locked(int32_t rid) {
        auto it = slots.find(rid);
        if (it != slots.end()) return it->second;
        const int32_t s = (int32_t)slots.size();
        slots[rid] = s;
        return s;
    }
    int32_t slot(int32_t rid) {
        std::lock_guard<std::mutex> l(mu);
        return slot_locked(rid);
    }
    Buf &buffer(uint64_t thread) {
        std::lock_guard<std::mutex> l(mu);
        auto it = buffers.find(thread);
        if (it != buffers.end()) return *it->second;
        auto *b = new Buf();
        owned.push_back(b);
        buffers[thread] = b;
        return *b;
    }
    void append(Ev &&e) {
        Buf &b = buffer(e.thread);
        std::lock_guard<std::mutex> l(b.m);
        b.v.push_back(std::move(e));
    }

    // One device buffer -> digest, on the agent's stream of the buffer's own GPU, before returning.
    // The calling thread's current device is restored on every path.
    int hash_device(const void *d_buf, uint64_t n, uint64_t &digest, std::vector<uint8_t> *snap) {
        std::lock_guard<std::mutex> l(hash_mu);
        cudaPointerAttributes pa{};
        B2L_CUDA(cudaPointerGetAttributes(&pa, d_buf));
        if (pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged)
            return fail(B2L_E_INVALID_ARG, "capture: device_buffer is not device memory");
        int prev = 0;
        B2L_CUDA(cudaGetDevice(&prev));
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{prev};
        B2L_CUDA(cudaSetDevice(pa.device));
        DevScratch &D = dev_scratch[pa.device];
        if (!D.stream) B2L_CUDA(cudaStreamCreateWithFlags(&D.stream, cudaStreamNonBlocking));
        if (!D.h_args) B2L_CUDA(cudaMallocHost(&D.h_args, 3 * sizeof(uint64_t)));
        // (ptr, len) and the digest live in pinned host memory the kernels address directly
        // (unified addressing): no copy launches around the hash
        if (n >= (96ull << 10)) {  // one buffer at a time: K2's floor beats the serial chain here
            const int rc = hash_planes_launch(d_buf, n, D.h_args + 2, D.stream);
            if (rc) return rc;
        } else {
            D.h_args[0] = (uint64_t)d_buf, D.h_args[1] = n;
            const int rc = hash_batch_launch(D.h_args, D.h_args + 1, 1, D.h_args + 2, nullptr, D.stream);
            if (rc) return rc;
        }
        if (snap) {
            snap->resize(n);
            B2L_CUDA(cudaMemcpyAsync(snap->data(), d_buf, n, cudaMemcpyDeviceToHost, D.stream));
        }
        B2L_CUDA(cudaStreamSynchronize(D.stream));
        digest = D.h_args[2];
        return B2L_OK;
    }
    int hash_host(const void *h_buf, uint64_t n, uint64_t &digest, std::vector<uint8_t> *snap) {
        if (snap) snap->assign((const uint8_t *)h_buf, (const uint8_t *)h_buf + n);
        const void *bufs[1] = {h_buf};
        return hash_host_impl(bufs, &n, 1, &digest);
    }
    // Digest of a transfer payload from whichever view the runtime offers (device preferred).
    int hash_payload(Ev &e, const void *device_buf, const void *host_buf) {
        std::vector<uint8_t> *snap = audit_dir.empty() ? nullptr : &e.payload;
        int rc = B2L_OK;
        if (device_buf) rc = hash_device(device_buf, e.bytes, e.hash, snap);
        else if (host_buf) rc = hash_host(host_buf, e.bytes, e.hash, snap);
        else return B2L_OK;
        if (rc == B2L_OK) {
            e.has_payload = snap != nullptr;
        } else {  // no digest: the event is still emitted, opaque (capture.ts:212-217)
            e.hash = 0;
            e.payload.clear();
            e.has_payload = false;
        }
        return rc;
    }
};

std::string ndjson(Capture &C, uint64_t wall, bool have_wall, std::vector<std::pair<uint64_t, const Ev *>> *sidecars) {
    std::vector<const Ev *> merged;
    {
        std::lock_guard<std::mutex> l(C.mu);
        for (auto *b : C.owned) {
            std::lock_guard<std::mutex> lb(b->m);
            for (const Ev &e : b->v) merged.push_back(&e);
        }
        C.unfinished_at_exit = C.pending_targets.size() + C.pending_ops.size();
    }
    std::stable_sort(merged.begin(), merged.end(), [](const Ev *a, const Ev *b) {
        return a->t0 != b->t0 ? a->t0 < b->t0 : a->provisional < b->provisional;
    });
    uint64_t w = 0;
    for (const Ev *e : merged) w = std::max(w, e->t1);
    if (have_wall) w = wall;
    std::string out;
    out.reserve(64 + merged.size() * 160);
    char line[512];
    int32_t ndev;
    {
        std::lock_guard<std::mutex> l(C.mu);
        ndev = (int32_t)C.slots.size();
    }
    snprintf(line, sizeof(line), "{\"dmlens\":1,\"num_devices\":%d,\"host_device\":0,\"wall_time_ns\":%llu}\n", ndev,
             (unsigned long long)w);
    out += line;
    uint64_t seq = 0;
    for (const Ev *e : merged) {
        // field order and bare-integer hash exactly as model.ts:38-48 serializeEvent
        snprintf(line, sizeof(line),
                 "{\"seq\":%llu,\"kind\":\"%s\",\"t0\":%llu,\"t1\":%llu,\"src_dev\":%d,\"dst_dev\":%d,"
                 "\"src_addr\":%llu,\"dst_addr\":%llu,\"bytes\":%llu,\"hash\":%llu,\"codeptr\":%llu}\n",
                 (unsigned long long)seq, kind_name(e->kind), (unsigned long long)e->t0, (unsigned long long)e->t1,
                 e->src_dev, e->dst_dev, (unsigned long long)e->src_addr, (unsigned long long)e->dst_addr,
                 (unsigned long long)e->bytes, (unsigned long long)e->hash, (unsigned long long)e->codeptr);
        out += line;
        if (sidecars && e->has_payload) sidecars->emplace_back(seq, e);
        ++seq;
    }
    return out;
}

}  // namespace cap
}  // namespace b2l

using b2l::cap::Capture;
using b2l::cap::Ev;

extern "C" {

b2l_capture *b2l_capture_create(int32_t host_runtime_id) {
    try {
        return reinterpret_cast<b2l_capture *>(new Capture(host_runtime_id));
    } catch (...) {
        b2l::set_error("b2l_capture_create: allocation failed");
        return nullptr;
    }
}

void b2l_capture_destroy(b2l_capture *c) { delete reinterpret_cast<Capture *>(c); }

int b2l_capture_set_audit_dir(b2l_capture *c, const char *dir) {
    if (!c) return b2l::fail(B2L_E_INVALID_ARG, "null capture");
    reinterpret_cast<Capture *>(c)->audit_dir = dir ? dir : "";
    return B2L_OK;
}

int32_t b2l_capture_device_slot(b2l_capture *c, int32_t runtime_id) {
    if (!c) return b2l::fail(B2L_E_INVALID_ARG, "null capture");
    return reinterpret_cast<Capture *>(c)->slot(runtime_id);
}

int b2l_capture_target(b2l_capture *cp, int endpoint, uint64_t target_id, int32_t device_id, uint64_t codeptr,
                       uint64_t thread_id, uint64_t time_ns) {
    if (!cp) return b2l::fail(B2L_E_INVALID_ARG, "null capture");
    Capture &C = *reinterpret_cast<Capture *>(cp);
    const uint64_t t = time_ns == UINT64_MAX ? C.now() : time_ns;
    if (endpoint == B2L_CAPTURE_BEGIN) {  // capture.ts:164-179
        Ev e{};
        e.t0 = t, e.provisional = C.provisional++, e.kind = b2l::cap::KERNEL, e.codeptr = codeptr;
        e.thread = thread_id;
        std::lock_guard<std::mutex> l(C.mu);
        e.src_dev = e.dst_dev = C.slot_locked(device_id);
        C.pending_targets[target_id] = std::move(e);
        return B2L_OK;
    }
    if (endpoint != B2L_CAPTURE_END) return b2l::fail(B2L_E_INVALID_ARG, "endpoint must be begin or end");
    Ev e;
    {  // capture.ts:181-189
        std::lock_guard<std::mutex> l(C.mu);
        auto it = C.pending_targets.find(target_id);
        if (it == C.pending_targets.end()) {
            ++C.unmatched_ends;
            return B2L_OK;
        }
        e = std::move(it->second);
        C.pending_targets.erase(it);
    }
    e.t1 = t;
    C.append(std::move(e));
    return B2L_OK;
}

int b2l_capture_data_op(b2l_capture *cp, int endpoint, uint64_t host_op_id, int optype, int32_t src_device,
                        int32_t dst_device, uint64_t src_addr, uint64_t dst_addr, uint64_t bytes, uint64_t codeptr,
                        uint64_t thread_id, uint64_t time_ns, const void *device_buffer, const void *host_buffer) {
    if (!cp) return b2l::fail(B2L_E_INVALID_ARG, "null capture");
    Capture &C = *reinterpret_cast<Capture *>(cp);
    const uint64_t t = time_ns == UINT64_MAX ? C.now() : time_ns;
    if (endpoint == B2L_CAPTURE_BEGIN) {  // makeDataOp, capture.ts:226-275
        Ev e{};
        e.t0 = t, e.provisional = C.provisional++, e.codeptr = codeptr, e.thread = thread_id;
        if (optype == B2L_OP_ALLOC) {
            if (bytes == 0 || dst_addr == 0) {
                std::lock_guard<std::mutex> l(C.mu);
                ++C.dropped_malformed;
                return B2L_OK;
            }
            e.kind = b2l::cap::ALLOC, e.src_addr = src_addr, e.dst_addr = dst_addr, e.bytes = bytes;
        } else if (optype == B2L_OP_DELETE) {
            if (dst_addr == 0) {
                std::lock_guard<std::mutex> l(C.mu);
                ++C.dropped_malformed;
                return B2L_OK;
            }
            e.kind = b2l::cap::DELETE, e.dst_addr = dst_addr;
        } else if (optype == B2L_OP_TO_DEVICE || optype == B2L_OP_FROM_DEVICE) {
            e.kind = b2l::cap::TRANSFER, e.src_addr = src_addr, e.dst_addr = dst_addr, e.bytes = bytes;
            // host-to-device bytes are complete at begin in host memory; the device copy only at end
            if (bytes > 0 && host_buffer && optype == B2L_OP_TO_DEVICE && !device_buffer)
                C.hash_payload(e, nullptr, host_buffer);  // on failure: opaque at end, never dropped
        } else {
            return b2l::fail(B2L_E_INVALID_ARG, "unknown data-op type");
        }
        std::lock_guard<std::mutex> l(C.mu);
        e.src_dev = C.slot_locked(src_device), e.dst_dev = C.slot_locked(dst_device);
        C.pending_ops[host_op_id] = std::move(e);
        return B2L_OK;
    }
    if (endpoint != B2L_CAPTURE_END) return b2l::fail(B2L_E_INVALID_ARG, "endpoint must be begin or end");
    Ev e;
    {
        std::lock_guard<std::mutex> l(C.mu);
        auto it = C.pending_ops.find(host_op_id);
        if (it == C.pending_ops.end()) {
            ++C.unmatched_ends;
            return B2L_OK;
        }
        e = std::move(it->second);
        C.pending_ops.erase(it);
    }
    if (e.kind == b2l::cap::TRANSFER) {  // capture.ts:198-219
        if (e.bytes > 0 && (device_buffer || host_buffer))
            C.hash_payload(e, device_buffer, host_buffer);  // on failure: opaque below, never dropped
        if (e.bytes > 0 && e.hash == 0) {  // no content identity: recorded as opaque
            std::lock_guard<std::mutex> l(C.mu);
            ++C.hash_skipped;
            e.bytes = 0;
        }
    }
    e.t1 = t;
    C.append(std::move(e));
    return B2L_OK;
}

int b2l_capture_finalize(b2l_capture *cp, uint64_t wall_time_ns, char **text, uint64_t *len) {
    if (!cp || !text || !len) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    Capture &C = *reinterpret_cast<Capture *>(cp);
    const std::string s = b2l::cap::ndjson(C, wall_time_ns, wall_time_ns != UINT64_MAX, nullptr);
    char *out = (char *)malloc(s.size() + 1);
    if (!out) return b2l::fail(B2L_E_OOM, "host allocation failed");
    memcpy(out, s.c_str(), s.size() + 1);
    *text = out;
    *len = s.size();
    return B2L_OK;
}

void b2l_capture_free_text(char *text) { free(text); }

int b2l_capture_write(b2l_capture *cp, const char *out_path, uint64_t wall_time_ns) {
    if (!cp) return b2l::fail(B2L_E_INVALID_ARG, "null capture");
    Capture &C = *reinterpret_cast<Capture *>(cp);
    const char *path = out_path ? out_path : getenv("DMLENS_OUT");
    if (!path || !*path)  // capture.ts:307-310
        return b2l::fail(B2L_E_INVALID_ARG, "no output path: pass out_path or set DMLENS_OUT");
    std::vector<std::pair<uint64_t, const Ev *>> side;
    const std::string s = b2l::cap::ndjson(C, wall_time_ns, wall_time_ns != UINT64_MAX, &side);
    FILE *f = fopen(path, "wb");
    if (!f) return b2l::fail(B2L_E_INVALID_ARG, std::string("cannot open ") + path);
    const bool ok = fwrite(s.data(), 1, s.size(), f) == s.size();
    fclose(f);
    if (!ok) return b2l::fail(B2L_E_INVALID_ARG, std::string("short write to ") + path);
    if (!C.audit_dir.empty()) {  // "<seq>.bin" sidecars, capture.ts:314-320
        mkdir(C.audit_dir.c_str(), 0755);
        for (auto &p : side) {
            const std::string name = C.audit_dir + "/" + std::to_string(p.first) + ".bin";
            FILE *g = fopen(name.c_str(), "wb");
            if (!g) return b2l::fail(B2L_E_INVALID_ARG, "cannot write " + name);
            fwrite(p.second->payload.data(), 1, p.second->payload.size(), g);
            fclose(g);
        }
    }
    return B2L_OK;
}

int b2l_capture_warnings(b2l_capture *cp, uint64_t *out4) {
    if (!cp || !out4) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    Capture &C = *reinterpret_cast<Capture *>(cp);
    std::lock_guard<std::mutex> l(C.mu);
    out4[0] = C.unmatched_ends, out4[1] = C.unfinished_at_exit, out4[2] = C.hash_skipped;
    out4[3] = C.dropped_malformed;
    return B2L_OK;
}

}  // extern "C"
