// host_common.h — host-side helpers shared by the translation units of libmapi.so: the thread-local
// error message, launch counter, optional kernel timing (mapi_set_profiling / mapi_last_kernel_ms) and
// the cached device query.  Inline variables (C++17) give each one definition across the TUs.
#pragma once
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/mapi.h"

namespace mapi_host {

inline thread_local char g_err[512] = "";
inline std::atomic<uint64_t> g_launches{0};
inline std::atomic<int> g_profiling{0};
inline thread_local float g_last_kernel_ms = 0.0f;

inline mapi_status fail(mapi_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

#define MAPI_CUDA(call)                                                                          \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return ::mapi_host::fail(MAPI_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                     __FILE__, __LINE__);                                        \
    } while (0)

#define MAPI_LAUNCHED()                                                                         \
    do {                                                                                        \
        ::mapi_host::g_launches.fetch_add(1, std::memory_order_relaxed);                        \
        cudaError_t e_ = cudaGetLastError();                                                    \
        if (e_ != cudaSuccess)                                                                  \
            return ::mapi_host::fail(MAPI_ERR_CUDA, "launch failed: %s (%s:%d)",                \
                                     cudaGetErrorString(e_), __FILE__, __LINE__);               \
    } while (0)

struct Device {
    int id = -1;
    int sms = 0;
    int smem_optin = 0;
    int cc_major = 0;
    size_t l2_bytes = 0;
};

inline mapi_status device_info(Device& d) {
    int id = 0;
    MAPI_CUDA(cudaGetDevice(&id));
    static thread_local Device cache;
    if (cache.id != id) {
        Device x;
        x.id = id;
        MAPI_CUDA(cudaDeviceGetAttribute(&x.sms, cudaDevAttrMultiProcessorCount, id));
        MAPI_CUDA(cudaDeviceGetAttribute(&x.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, id));
        MAPI_CUDA(cudaDeviceGetAttribute(&x.cc_major, cudaDevAttrComputeCapabilityMajor, id));
        int l2 = 0;
        MAPI_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, id));
        x.l2_bytes = (size_t)l2;
        if (x.cc_major != 10)
            return fail(MAPI_ERR_CUDA, "libmapi is built for sm_100a; device %d has compute capability %d.x",
                        id, x.cc_major);
        cache = x;
    }
    d = cache;
    return MAPI_OK;
}


// CUDA events for the optional kernel timing come from a per-thread pool (creating / destroying two
// events per call cost several microseconds of host time inside small problems' steps)
inline std::vector<cudaEvent_t>& event_pool() {
    static thread_local std::vector<cudaEvent_t> pool;
    return pool;
}
inline cudaEvent_t event_take() {
    auto& pool = event_pool();
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s = nullptr;
    bool on = false;
    explicit Timer(cudaStream_t st) : s(st) {
        on = g_profiling.load() != 0;
        if (on) {
            a = event_take();
            b = event_take();
        }
    }
    void start() {
        if (on) cudaEventRecord(a, s);
    }
    void stop() {
        if (on) cudaEventRecord(b, s);
    }
    void harvest() {  // after a stream sync
        if (on) {
            float ms = 0.0f;
            if (cudaEventElapsedTime(&ms, a, b) == cudaSuccess) g_last_kernel_ms = ms;
        }
    }
    ~Timer() {
        if (a) event_pool().push_back(a);
        if (b) event_pool().push_back(b);
    }
};

}  // namespace mapi_host
