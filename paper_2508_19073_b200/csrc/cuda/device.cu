// Device discovery, error reporting and small runtime helpers.

#include <atomic>
#include <map>
#include <mutex>
#include <cstdint>
#include <string>

#include "../../../include/carma_gpu.h"
#include "common.cuh"

namespace carma_b200 {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

// Checked once per device and cached: cudaGetDeviceProperties costs
// milliseconds, and every compute entry point calls this.
void require_device(int device) {
    static std::atomic<uint64_t> ok_mask{0};
    if (device >= 0 && device < 64 && ((ok_mask.load(std::memory_order_relaxed) >> device) & 1ull)) return;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw CudaFailure(std::string("no CUDA device available (") +
                          (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                          "); the CARMA GPU path has no CPU fallback");
    if (device < 0 || device >= n) throw InvalidArg("device index out of range");
    int major = 0, minor = 0;
    CARMA_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CARMA_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10)
        throw CudaFailure("device " + std::to_string(device) + " is sm_" + std::to_string(major) +
                          std::to_string(minor) + "; this build targets sm_100a only");
    if (device < 64) ok_mask.fetch_or(1ull << device, std::memory_order_relaxed);
}

namespace {
struct DevicePool {
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks[64];
    size_t cached[64] = {};
    std::map<void*, int> owner;  // block -> device
};
DevicePool& pool() {
    static DevicePool* p = new DevicePool();  // never destroyed: blocks outlive static teardown
    return *p;
}
constexpr size_t kPoolCap = size_t{8} << 30;  // cached bytes per device

size_t size_class(size_t b) {
    if (b <= (size_t{256} << 20)) {
        size_t c = 512;
        while (c < b) c <<= 1;
        return c;
    }
    const size_t g = size_t{2} << 20;
    return (b + g - 1) / g * g;
}
}  // namespace

void* pool_alloc(size_t bytes, size_t* capacity) {
    int dev = 0;
    CARMA_CUDA(cudaGetDevice(&dev));
    const size_t c = size_class(bytes);
    DevicePool& P = pool();
    {
        std::lock_guard<std::mutex> lock(P.mu);
        auto& fl = P.free_blocks[dev & 63];
        auto it = fl.find(c);
        if (it != fl.end()) {
            void* p = it->second;
            fl.erase(it);
            P.cached[dev & 63] -= c;
            *capacity = c;
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, c);
    if (e != cudaSuccess) {  // drop this device's cache and retry once
        cudaGetLastError();
        std::lock_guard<std::mutex> lock(P.mu);
        for (auto& kv : P.free_blocks[dev & 63]) {
            cudaFree(kv.second);
            P.owner.erase(kv.second);
        }
        P.free_blocks[dev & 63].clear();
        P.cached[dev & 63] = 0;
        CARMA_CUDA(cudaMalloc(&p, c));
    }
    {
        std::lock_guard<std::mutex> lock(P.mu);
        P.owner[p] = dev;
    }
    *capacity = c;
    return p;
}

void pool_free(void* p, size_t capacity) {
    if (!p) return;
    DevicePool& P = pool();
    std::lock_guard<std::mutex> lock(P.mu);
    auto o = P.owner.find(p);
    const int dev = o == P.owner.end() ? 0 : o->second;
    if (P.cached[dev & 63] + capacity > kPoolCap) {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        cudaFree(p);
        if (cur != dev) cudaSetDevice(cur);
        if (o != P.owner.end()) P.owner.erase(o);
        return;
    }
    P.free_blocks[dev & 63].emplace(capacity, p);
    P.cached[dev & 63] += capacity;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace carma_b200

extern "C" {

const char* carma_last_error(void) { return carma_b200::g_last_error.c_str(); }

int carma_version(void) { return 100; }

int carma_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int usable = 0;
    for (int d = 0; d < n; ++d) {
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) == cudaSuccess && major == 10)
            ++usable;
    }
    return usable;
}

}  // extern "C"
