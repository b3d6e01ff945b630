// Row formats of the estimator inputs and their featurisers, shared by the
// k-NN (knn.cu) and the neural GPUMemNet (gpumemnet.cu) kernels.
// scalar_features (proj/src/estimators.cpp:317-342) of one query row, in
// fp64 with separately rounded operations (the reference's FMA-free build).
// P is any parameter struct carrying the row source: act[16] (packed rows),
// bbase/boff/bw/bwpr (bit-packed rows), rows, family, default_family.
#pragma once

#include <cstdint>

#include "../../../include/carma_gpu.h"

namespace carma_b200 {

constexpr int kFeatureDims = 19;

__device__ __forceinline__ double u2d(uint64_t v) { return __ull2double_rn(v); }

// scalar_features dim d of a feature row (estimators.cpp:317-342).
__device__ __forceinline__ void featurize(const carma_feature_row& r, double* raw) {
    raw[0] = u2d(r.n_linear);
    raw[1] = u2d(r.n_batchnorm);
    raw[2] = u2d(r.n_dropout);
    raw[3] = u2d(r.n_conv);
    raw[4] = u2d(r.batch_size);
    raw[5] = u2d(r.total_params);
    raw[6] = u2d(r.total_activations);
    raw[7] = r.act_cos;
    raw[8] = r.act_sin;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const bool h = r.has_layers != 0;
        raw[9 + 3 * k] = h ? static_cast<double>(r.kind[k]) : 0.0;
        raw[10 + 3 * k] = h ? u2d(r.tuple_acts[k]) : 0.0;
        raw[11 + 3 * k] = h ? u2d(r.tuple_params[k]) : 0.0;
    }
    raw[18] = __dadd_rn(__dmul_rn(16.0, raw[5]), __dmul_rn(__dmul_rn(4.0, raw[4]), raw[6]));
}

constexpr uint64_t kLow48 = (1ull << 48) - 1ull;

// Unpacks a carma_feature_packed row (layout in carma_gpu.h).
template <class P>
__device__ __forceinline__ void featurize_packed(const P& p, const carma_feature_packed& r, double* raw) {
    const uint64_t w0 = r.w[0], w1 = r.w[1], w2 = r.w[2], w3 = r.w[3], w5 = r.w[5];
    raw[0] = u2d((w0 >> 48) & 0xff);
    raw[1] = u2d(w0 >> 56);
    raw[2] = u2d((w1 >> 48) & 0xff);
    raw[3] = u2d(w1 >> 56);
    raw[4] = u2d((w2 >> 48) | ((w5 >> 48) << 16));
    raw[5] = u2d(w0 & kLow48);
    raw[6] = u2d(w1 & kLow48);
    const int code = static_cast<int>(w3 >> 61);
    raw[7] = p.act[2 * code];
    raw[8] = p.act[2 * code + 1];
    const bool h = (w3 >> 60) & 1ull;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        raw[9 + 3 * k] = h ? static_cast<double>((w3 >> (48 + 4 * k)) & 0xf) : 0.0;
        raw[10 + 3 * k] = h ? u2d(r.w[2 + 2 * k] & kLow48) : 0.0;
        raw[11 + 3 * k] = h ? u2d(r.w[3 + 2 * k] & kLow48) : 0.0;
    }
    raw[18] = __dadd_rn(__dmul_rn(16.0, raw[5]), __dmul_rn(__dmul_rn(4.0, raw[4]), raw[6]));
}

// Field f of a bit-packed row: base + the width-bit value at its offset.
template <class P>
__device__ __forceinline__ uint64_t bit_field(const P& p, const uint32_t* row, int f) {
    const uint32_t w = p.bw[f];
    if (w == 0) return p.bbase[f];
    const uint32_t off = p.boff[f];
    const uint32_t* q = row + (off >> 5);
    const uint32_t sh = off & 31;
    uint64_t v = (static_cast<uint64_t>(__ldg(q + 1)) << 32) | __ldg(q);
    v >>= sh;
    if (sh + w > 64) v |= static_cast<uint64_t>(__ldg(q + 2)) << (64 - sh);
    return p.bbase[f] + (v & ((1ull << w) - 1ull));
}

template <class P>
__device__ __forceinline__ const uint32_t* bit_row(const P& p, uint64_t i) {
    return static_cast<const uint32_t*>(p.rows) + i * p.bwpr;
}

template <class P>
__device__ __forceinline__ void featurize_bits(const P& p, const uint32_t* r, double* raw) {
#pragma unroll
    for (int f = 0; f < 7; ++f) raw[f] = u2d(bit_field(p, r, f));
    const int code = static_cast<int>(bit_field(p, r, 7)) & 7;
    raw[7] = p.act[2 * code];
    raw[8] = p.act[2 * code + 1];
    const bool h = bit_field(p, r, 11) != 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        raw[9 + 3 * k] = h ? static_cast<double>(static_cast<int32_t>(bit_field(p, r, 8 + k))) : 0.0;
        raw[10 + 3 * k] = h ? u2d(bit_field(p, r, 12 + 2 * k)) : 0.0;
        raw[11 + 3 * k] = h ? u2d(bit_field(p, r, 13 + 2 * k)) : 0.0;
    }
    raw[18] = __dadd_rn(__dmul_rn(16.0, raw[5]), __dmul_rn(__dmul_rn(4.0, raw[4]), raw[6]));
}


template <int FMT, class P>
__device__ __forceinline__ void load_raw(const P& p, uint64_t row, double* raw) {
    if constexpr (FMT == CARMA_ROWS_SCALAR) {
        const double* r = static_cast<const double*>(p.rows) + row * kFeatureDims;
#pragma unroll
        for (int d = 0; d < kFeatureDims; ++d) raw[d] = r[d];
    } else if constexpr (FMT == CARMA_ROWS_PACKED) {
        featurize_packed(p, static_cast<const carma_feature_packed*>(p.rows)[row], raw);
    } else if constexpr (FMT == CARMA_ROWS_BITPACKED) {
        featurize_bits(p, bit_row(p, row), raw);
    } else {
        featurize(static_cast<const carma_feature_row*>(p.rows)[row], raw);
    }
}

// Family code carried by the row (packed / bit-packed formats), else the
// per-row family array or the default. Range checks are the caller's.
template <int FMT, class P>
__device__ __forceinline__ int row_family(const P& p, uint64_t i) {
    if constexpr (FMT == CARMA_ROWS_PACKED)
        return static_cast<int>((static_cast<const carma_feature_packed*>(p.rows)[i].w[4] >> 48) & 0xff);
    else if constexpr (FMT == CARMA_ROWS_BITPACKED)
        return static_cast<int>(bit_field(p, bit_row(p, i), 18));
    else
        return p.family ? static_cast<int>(p.family[i]) : p.default_family;
}

}  // namespace carma_b200
