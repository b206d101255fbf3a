// OMPT tool glue for the capture agent (SPEC.md "ompt-shim": "requires the OpenMP runtime to
// support two OMPT callbacks: ompt_callback_target_emi and ompt_callback_target_data_op_emi").
// Built as libb2l_ompt.so; an OMPT-capable runtime loads it through OMP_TOOL_LIBRARIES and calls
// ompt_start_tool.  Every callback forwards to the b2l_capture C ABI (b2l_capture.cu); at
// finalize the trace goes to $DMLENS_OUT (sidecars to $DMLENS_AUDIT_DIR).
//
// The few OMPT declarations needed are restated from the OpenMP 5.1 tools interface
// (omp-tools.h is not part of this toolchain): the EMI callback signatures, the callback and
// data-op enumerations, ompt_data_t and the start-tool handshake.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <thread>

#include "b2l.h"

extern "C" {
typedef union ompt_data_t {
    uint64_t value;
    void *ptr;
} ompt_data_t;
typedef uint64_t ompt_id_t;
typedef void (*ompt_interface_fn_t)(void);
typedef ompt_interface_fn_t (*ompt_function_lookup_t)(const char *interface_function_name);
typedef void (*ompt_callback_t)(void);
typedef int (*ompt_set_callback_t)(int event, ompt_callback_t callback);
typedef int (*ompt_initialize_t)(ompt_function_lookup_t lookup, int initial_device_num, ompt_data_t *tool_data);
typedef void (*ompt_finalize_t)(ompt_data_t *tool_data);
typedef struct ompt_start_tool_result_t {
    ompt_initialize_t initialize;
    ompt_finalize_t finalize;
    ompt_data_t tool_data;
} ompt_start_tool_result_t;
}

namespace {
// OpenMP 5.1 enumerations (ompt_callbacks_t, ompt_scope_endpoint_t, ompt_target_data_op_t)
constexpr int ompt_callback_target_emi = 33, ompt_callback_target_data_op_emi = 34;
constexpr int ompt_scope_begin = 1, ompt_scope_end = 2, ompt_scope_beginend = 3;
constexpr int ompt_set_always = 5;
constexpr int op_alloc = 1, op_to_device = 2, op_from_device = 3, op_delete = 4;
constexpr int op_async_base = 16;  // ompt_target_data_*_async = the synchronous value + 16

b2l_capture *g_cap = nullptr;
std::atomic<uint64_t> g_ids{1};

uint64_t thread_id() { return (uint64_t)std::hash<std::thread::id>{}(std::this_thread::get_id()); }

// A device pointer of the CUDA runtime's address space (hashed where it lives), else null.
const void *device_view(const void *p) {
    if (!p) return nullptr;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged ? p : nullptr;
}

void on_target_emi(int kind, int endpoint, int device_num, ompt_data_t *task_data, ompt_data_t *target_task_data,
                   ompt_data_t *target_data, const void *codeptr_ra) {
    (void)kind, (void)task_data, (void)target_task_data;
    if (!g_cap || !target_data) return;
    if (endpoint == ompt_scope_begin) target_data->value = g_ids++;
    const int ep = endpoint == ompt_scope_begin ? B2L_CAPTURE_BEGIN : B2L_CAPTURE_END;
    b2l_capture_target(g_cap, ep, target_data->value, device_num, (uint64_t)codeptr_ra, thread_id(), UINT64_MAX);
}

void on_target_data_op_emi(int endpoint, ompt_data_t *target_task_data, ompt_data_t *target_data,
                           ompt_id_t *host_op_id, int optype, void *src_addr, int src_device_num, void *dest_addr,
                           int dest_device_num, size_t bytes, const void *codeptr_ra) {
    (void)target_task_data, (void)target_data;
    if (!g_cap || !host_op_id) return;
    if (optype > op_async_base) optype -= op_async_base;
    if (optype < op_alloc || optype > op_delete) return;  // associate / disassociate / memset ...
    if (endpoint == ompt_scope_begin) *host_op_id = g_ids++;
    const void *dev = nullptr, *host = nullptr;
    if (optype == op_to_device) {  // the landed device copy at end; the host source at begin
        if (endpoint == ompt_scope_end) dev = device_view(dest_addr);
        else host = device_view(dest_addr) ? nullptr : src_addr;
    } else if (optype == op_from_device && endpoint == ompt_scope_end) {
        dev = device_view(src_addr);
        host = dev ? nullptr : dest_addr;
    }
    const int ep = endpoint == ompt_scope_begin ? B2L_CAPTURE_BEGIN : B2L_CAPTURE_END;
    b2l_capture_data_op(g_cap, ep, *host_op_id, optype, src_device_num, dest_device_num, (uint64_t)src_addr,
                        (uint64_t)dest_addr, bytes, (uint64_t)codeptr_ra, thread_id(), UINT64_MAX, dev, host);
}

int tool_initialize(ompt_function_lookup_t lookup, int initial_device_num, ompt_data_t *tool_data) {
    (void)tool_data;
    // the host is the initial device; runtimes number it after the targets
    g_cap = b2l_capture_create(initial_device_num);
    auto set_cb = (ompt_set_callback_t)lookup("ompt_set_callback");
    if (!g_cap || !set_cb) return 0;
    const int a = set_cb(ompt_callback_target_emi, (ompt_callback_t)on_target_emi);
    const int b = set_cb(ompt_callback_target_data_op_emi, (ompt_callback_t)on_target_data_op_emi);
    return a == ompt_set_always && b == ompt_set_always ? 1 : 0;
}

void tool_finalize(ompt_data_t *tool_data) {
    (void)tool_data;
    if (!g_cap) return;
    if (b2l_capture_write(g_cap, nullptr, UINT64_MAX) != 0) fprintf(stderr, "b2l_ompt: %s\n", b2l_last_error());
    uint64_t w[4] = {0, 0, 0, 0};
    b2l_capture_warnings(g_cap, w);
    if (w[0] || w[1] || w[2] || w[3])
        fprintf(stderr, "b2l_ompt: unmatched_ends=%llu unfinished_at_exit=%llu hash_skipped=%llu dropped=%llu\n",
                (unsigned long long)w[0], (unsigned long long)w[1], (unsigned long long)w[2],
                (unsigned long long)w[3]);
    b2l_capture_destroy(g_cap);
    g_cap = nullptr;
}

ompt_start_tool_result_t g_result = {tool_initialize, tool_finalize, {0}};
}  // namespace

extern "C" ompt_start_tool_result_t *ompt_start_tool(unsigned int omp_version, const char *runtime_version) {
    (void)omp_version, (void)runtime_version;
    return &g_result;
}
