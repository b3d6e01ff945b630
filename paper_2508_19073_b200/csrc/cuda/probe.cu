// fp64 pipe probe: the measured roofline denominator for the k-NN distance
// kernel (separately rounded DADD/DMUL, no FMA — the kernel's instruction mix).

#include "../../../include/carma_gpu.h"
#include "common.cuh"

namespace carma_b200 {
namespace {

constexpr int kChains = 8;
constexpr int kIters = 2048;

__global__ void fp64_probe(double seed, double* sink) {
    double a[kChains], m[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        a[c] = seed + threadIdx.x + c;
        m[c] = 1.0 + 1e-9 * c;
    }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            a[c] = __dadd_rn(a[c], 1.0e-7);
            m[c] = __dmul_rn(m[c], 0.9999999);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s = __dadd_rn(s, __dadd_rn(a[c], m[c]));
    if (s == 12345.678) sink[0] = s;  // keep the work alive
}

}  // namespace
}  // namespace carma_b200

using namespace carma_b200;

extern "C" carma_status carma_probe_fp64(int device, double* flops_per_s) {
    return guarded([&] {
        if (!flops_per_s) throw InvalidArg("null output");
        require_device(device);
        DeviceGuard g(device);
        int sms = 148;
        CARMA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        DeviceBuffer sink;
        sink.ensure(8);
        const unsigned grid = static_cast<unsigned>(sms) * 8, block = 256;
        cudaEvent_t e0, e1;
        CARMA_CUDA(cudaEventCreate(&e0));
        CARMA_CUDA(cudaEventCreate(&e1));
        double best = 0.0;
        for (int rep = 0; rep < 4; ++rep) {
            CARMA_CUDA(cudaEventRecord(e0));
            fp64_probe<<<grid, block>>>(1.0 + rep, sink.as<double>());
            CARMA_CUDA(cudaEventRecord(e1));
            CARMA_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            CARMA_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            const double ops = static_cast<double>(grid) * block * kIters * kChains * 2.0;
            if (rep > 0 && ops / (ms * 1e-3) > best) best = ops / (ms * 1e-3);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        CARMA_CUDA(cudaGetLastError());
        *flops_per_s = best;
    });
}

namespace carma_b200 {
namespace {
__global__ void fp32x2_probe(float seed, float* sink) {
    unsigned long long a[kChains];
    const unsigned long long m = 0x3f7fffff3f7fffffull;  // (0.99999994, 0.99999994)
    const unsigned long long c = 0x33d6bf9533d6bf95ull;  // (1e-7, 1e-7)
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
        const float v = seed + threadIdx.x + i;
        asm("mov.b64 %0, {%1, %1};" : "=l"(a[i]) : "f"(v));
    }
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(m), "l"(c));
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
        float x, y;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i]));
        s += x + y;
    }
    if (s == 12345.678f) sink[0] = s;
}
}  // namespace
}  // namespace carma_b200

extern "C" carma_status carma_probe_fp32(int device, double* flops_per_s) {
    return guarded([&] {
        if (!flops_per_s) throw InvalidArg("null output");
        require_device(device);
        DeviceGuard g(device);
        int sms = 148;
        CARMA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        DeviceBuffer sink;
        sink.ensure(8);
        const unsigned grid = static_cast<unsigned>(sms) * 8, block = 256;
        cudaEvent_t e0, e1;
        CARMA_CUDA(cudaEventCreate(&e0));
        CARMA_CUDA(cudaEventCreate(&e1));
        double best = 0.0;
        for (int rep = 0; rep < 4; ++rep) {
            CARMA_CUDA(cudaEventRecord(e0));
            fp32x2_probe<<<grid, block>>>(1.0f + rep, sink.as<float>());
            CARMA_CUDA(cudaEventRecord(e1));
            CARMA_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            CARMA_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            // kChains packed FMAs per iteration, 2 lanes x 2 flops each
            const double flops = static_cast<double>(grid) * block * kIters * kChains * 4.0;
            if (rep > 0 && flops / (ms * 1e-3) > best) best = flops / (ms * 1e-3);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        CARMA_CUDA(cudaGetLastError());
        *flops_per_s = best;
    });
}
