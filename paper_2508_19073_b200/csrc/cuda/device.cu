// Device discovery, error reporting and small runtime helpers.

#include <atomic>
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
