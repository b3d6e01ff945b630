// Shared device/host helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../host/status.hpp"

namespace carma_b200 {

#define CARMA_CUDA(call)                                                                  \
    do {                                                                                  \
        cudaError_t err__ = (call);                                                       \
        if (err__ != cudaSuccess)                                                         \
            throw ::carma_b200::CudaFailure(std::string(#call) + ": " +                  \
                                            cudaGetErrorString(err__));                   \
    } while (0)

// Throws unless `device` is a usable sm_100 device. No CPU fallback exists:
// every compute entry point calls this first.
void require_device(int device);

// Caching device allocator: cudaFree returns memory to the driver and the
// next cudaMalloc maps it again (~0.5 ms per pair on B200), which dominated
// short calls (one replay plan: ~7 ms of create + destroy for a 0.9 ms run).
// Blocks go back to a per-device free list instead; the cache is capped.
// Contract: a block is released only when no queued work still uses it
// (owners synchronise their streams first; DeviceBuffer::ensure synchronises
// the device before recycling a block it outgrew).
void* pool_alloc(size_t bytes, size_t* capacity);
void pool_free(void* p, size_t capacity);

// RAII device buffer (grow-only), backed by the caching allocator.
struct DeviceBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    void ensure(size_t want) {
        if (want <= bytes) return;
        if (ptr) CARMA_CUDA(cudaDeviceSynchronize());  // queued work may still use the old block
        release();
        if (want == 0) return;
        ptr = pool_alloc(want, &bytes);
    }
    void release() {
        if (ptr) pool_free(ptr, bytes);
        ptr = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
    ~DeviceBuffer() { release(); }
};

// RAII pinned host buffer (grow-only).
struct PinnedBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    void ensure(size_t want) {
        if (want <= bytes) return;
        release();
        if (want == 0) return;
        CARMA_CUDA(cudaMallocHost(&ptr, want));
        bytes = want;
    }
    void release() {
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
    ~PinnedBuffer() { release(); }
};

// Orders the reuse of a handle's shared device buffers (scratch, counters)
// across streams: a call that enqueues work touching them on stream s first
// makes s wait for the last user's work (acquire), then marks its own work
// as the last user (release). Host-side reuse (pinned staging, host-stream
// pipelines) waits on the host instead (host_wait).
struct StreamFence {
    cudaEvent_t ev = nullptr;
    bool live = false;
    void acquire(cudaStream_t s) {
        if (live) CARMA_CUDA(cudaStreamWaitEvent(s, ev, 0));
    }
    void release(cudaStream_t s) {
        if (!ev) CARMA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CARMA_CUDA(cudaEventRecord(ev, s));
        live = true;
    }
    void host_wait() {
        if (live) CARMA_CUDA(cudaEventSynchronize(ev));
    }
    void destroy() {
        if (ev) cudaEventDestroy(ev);
        ev = nullptr;
        live = false;
    }
};

// Makes `caller` (when given) wait for everything queued so far on `own`:
// device calls that run on a handle's stream stay ordered before the
// caller's later work (and inside its CUDA-event timings).
inline void join_stream(cudaStream_t caller, cudaStream_t own) {
    if (!caller || caller == own) return;
    cudaEvent_t ev;
    CARMA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CARMA_CUDA(cudaEventRecord(ev, own));
    CARMA_CUDA(cudaStreamWaitEvent(caller, ev, 0));
    CARMA_CUDA(cudaEventDestroy(ev));
}

// Scoped device switch.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CARMA_CUDA(cudaGetDevice(&prev));
        if (prev != dev) CARMA_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

bool is_pinned(const void* p);

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 1u << 20) {
    uint64_t g = (n + block - 1) / block;
    if (g == 0) g = 1;
    return static_cast<unsigned>(g < cap ? g : cap);
}

}  // namespace carma_b200
