// Device discovery, error reporting and small runtime helpers.

#include <string>

#include "../../../include/carma_gpu.h"
#include "common.cuh"

namespace carma_b200 {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void require_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw CudaFailure(std::string("no CUDA device available (") +
                          (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                          "); the CARMA GPU path has no CPU fallback");
    if (device < 0 || device >= n) throw InvalidArg("device index out of range");
    cudaDeviceProp prop;
    CARMA_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        throw CudaFailure("device " + std::to_string(device) + " is sm_" + std::to_string(prop.major) +
                          std::to_string(prop.minor) + "; this build targets sm_100a only");
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
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10) ++usable;
    }
    return usable;
}

}  // extern "C"
