// Stage 1 — GPUMemNet (the reference's k-NN memory-bin classifier) on sm_100a.
//
// Semantics: LearnedEstimator::predict_scalar + estimate_learned
// (proj/src/estimators.cpp:438-475, :540-551), bit-exact:
//   q[d]  = hi>lo ? (raw-lo)/(hi-lo) : 0                    (:439-441)
//   d2    = sum_{d=0..18} diff_d^2 in dim order, diff_18 *= 64 (:445-457)
//   top-k = k smallest (d2, training index) pairs              (:460-462)
//   vote  = most votes, ties to the larger bucket             (:463-474)
//   bytes = (bucket + 1) * bucket_range                        (:540-551)
// Built with --fmad=false: every sub/mul/add is rounded separately, as in
// the reference's FMA-free x86-64 build.
//
// Algorithm (exact, not approximate). Because every term is >= 0 and
// rounding is monotone, a point's computed d2 is >= its own last term
// t18 = fl(fl(64*fl(p18-q18))^2). Training points are stored sorted by p18,
// so t18 grows monotonically walking outward from q18's position; a side can
// be abandoned as soon as its next t18 exceeds the current k-th best d2 —
// every point beyond it provably cannot enter the top-k, ties included.
// Queries are bucketed by (family, position of q18 in the sorted model) so a
// warp holds 32 queries with nearly identical search windows; the warp walks
// one common frontier and every lane evaluates the same point, so model
// reads are warp-uniform broadcasts from L1. Per query the work drops from
// N = 2800 to the window size (~150-300 points).
//
// Pipeline per batch (all on one stream):
//   knn_keys     featurise dim 18, normalise, binary-search -> (bin, pos); CTA histograms
//   bin_totals / scan_bins / bin_offsets  exclusive scan of the [bin][cta] histogram
//   knn_scatter  counting-sort scatter of row ids into bin order
//   knn_search   warp-per-32-queries frontier search + fused vote/bucket/bytes epilogue

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <type_traits>
#include <vector>

#include "../../../include/carma_gpu.h"
#include "../../../include/carma_host.h"
#include "common.cuh"
#include "../host/stage.hpp"
#include "../host/stage.hpp"
#include "rows.cuh"

namespace carma_b200 {
namespace {

constexpr int kDims = 19;
constexpr int kStride = 20;  // doubles per stored point (160 B, 16-B aligned)
constexpr int kMaxK = 16;
constexpr uint32_t kInvalidBin = 0xffffffffu;
constexpr int kScatterCtas = 296;  // 2 per SM on a 148-SM B200
constexpr int kMaxBins = 4096;
constexpr int kBlock = 8;  // points per frontier step
constexpr int kF32Dims = 16;  // fp32 pre-filter: active dims per point
#ifndef KNN_CAND_CAP
#define KNN_CAND_CAP 24
#endif
constexpr int kCandCap = KNN_CAND_CAP;  // fp32 pre-filter: candidate buffer per lane

struct ModelDev {
    const double* pts;    // N x 20, sorted by (p18, original index)
    const double* key18;  // N, pts[i][18]
    const int32_t* orig;  // N, original training index
    const int32_t* label_by_orig;
    uint64_t n;
    uint64_t bucket_range;
    uint32_t k;
    uint32_t bin_base;
    uint32_t bin_shift;
    int32_t present;
    uint32_t active;  // dims whose term can be non-zero (see carma_knn_set_model)
    int32_t f32_ok;   // fp32 pre-filter usable: <= 16 active dims, |points| <= 1e15
    const float* ptsf;  // (N + 2 kBlock) x 16: fl32(w * p[a_j]) for the active dims a_j
    double pmax[kF32Dims];  // max |p[a_j]| over the model
    uint8_t adim[kF32Dims]; // active dim a_j (0xff: padding)
    double lo[kDims];
    double hi[kDims];
};

struct KnnParams {
    ModelDev m[CARMA_FAMILIES];
    double act[16];  // packed rows: (cos, sin) per activation code
    // bit-packed rows (CARMA_ROWS_BITPACKED)
    uint64_t bbase[CARMA_BIT_FIELDS];
    uint16_t boff[CARMA_BIT_FIELDS];
    uint8_t bw[CARMA_BIT_FIELDS];
    uint32_t bwpr;
    const void* rows;
    int32_t format;
    const int8_t* family;
    int32_t default_family;
    uint64_t q;
    double* qrec;  // fp32 path: per row the normalised query (19) + eta, written by knn_prep
    // sorted layout: qrec indexed by the bucketed slot (written by
    // knn_prep_sorted), and bucket / bytes written by slot, un-permuted after
    int32_t qrec_by_slot;
    int32_t out_by_slot;
};

// Query record (fp32 path): normalised query (19), eta, t_in (the smallest
// t18 around the start position), the start position (bits). 176 B.
constexpr int kQrec = 22;

__device__ __forceinline__ double raw18_of(const KnnParams& p, uint64_t i) {
    if (p.format == CARMA_ROWS_BITPACKED) {
        const uint32_t* r = bit_row(p, i);
        return __dadd_rn(__dmul_rn(16.0, u2d(bit_field(p, r, 5))),
                         __dmul_rn(__dmul_rn(4.0, u2d(bit_field(p, r, 4))), u2d(bit_field(p, r, 6))));
    }
    if (p.format == CARMA_ROWS_SCALAR) return static_cast<const double*>(p.rows)[i * kDims + 18];
    if (p.format == CARMA_ROWS_PACKED) {
        const carma_feature_packed* r = static_cast<const carma_feature_packed*>(p.rows) + i;
        const uint64_t w0 = r->w[0], w1 = r->w[1], w2 = r->w[2], w5 = r->w[5];
        const double batch = u2d((w2 >> 48) | ((w5 >> 48) << 16));
        return __dadd_rn(__dmul_rn(16.0, u2d(w0 & kLow48)), __dmul_rn(__dmul_rn(4.0, batch), u2d(w1 & kLow48)));
    }
    const carma_feature_row& r = static_cast<const carma_feature_row*>(p.rows)[i];
    return __dadd_rn(__dmul_rn(16.0, u2d(r.total_params)),
                     __dmul_rn(__dmul_rn(4.0, u2d(r.batch_size)), u2d(r.total_activations)));
}

// t18 = fl(fl(64 * fl(key - q18))^2): the last term of a point's d2 and a lower
// bound of the whole d2 (every term is >= 0, rounding is monotone).
__device__ __forceinline__ double t18_of(double key, double q18) {
    const double diff = __dmul_rn(__dsub_rn(key, q18), 64.0);
    return __dmul_rn(diff, diff);
}

__device__ __forceinline__ double normalize(double raw, double lo, double hi) {
    return hi > lo ? __ddiv_rn(__dsub_rn(raw, lo), __dsub_rn(hi, lo)) : 0.0;
}

__device__ __forceinline__ int family_of(const KnnParams& p, uint64_t i) {
    const int f = p.format == CARMA_ROWS_PACKED
                      ? static_cast<int>((static_cast<const carma_feature_packed*>(p.rows)[i].w[4] >> 48) & 0xff)
                      : p.format == CARMA_ROWS_BITPACKED
                            ? static_cast<int>(bit_field(p, bit_row(p, i), 18))
                            : (p.family ? static_cast<int>(p.family[i]) : p.default_family);
    return (f >= 0 && f < CARMA_FAMILIES && p.m[f].present) ? f : -1;
}

// Compile-time row format versions for the search kernel: each instance
// carries one featuriser only (smaller code, no per-row format branches).
template <int FMT>
__device__ __forceinline__ int family_of_t(const KnnParams& p, uint64_t i) {
    int f;
    if constexpr (FMT == CARMA_ROWS_PACKED)
        f = static_cast<int>((static_cast<const carma_feature_packed*>(p.rows)[i].w[4] >> 48) & 0xff);
    else if constexpr (FMT == CARMA_ROWS_BITPACKED)
        f = static_cast<int>(bit_field(p, bit_row(p, i), 18));
    else
        f = p.family ? static_cast<int>(p.family[i]) : p.default_family;
    return (f >= 0 && f < CARMA_FAMILIES && p.m[f].present) ? f : -1;
}

// first index with key18[i] >= x
__device__ __forceinline__ uint32_t lower_bound(const double* key, uint64_t n, double x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (__ldg(key + mid) < x) lo = mid + 1;
        else hi = mid;
    }
    return static_cast<uint32_t>(lo);
}

// Same over keys in shared or global memory (generic loads).
__device__ __forceinline__ uint32_t lower_bound_any(const double* key, uint32_t n, double x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (key[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Pass 1: bin and start position per row; per-CTA histogram -> hist[bin][cta].
__global__ void knn_keys(KnnParams p, uint32_t n_bins, uint32_t* __restrict__ qbin,
                         uint32_t* __restrict__ qpos, uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t sh[];
    for (uint32_t b = threadIdx.x; b < n_bins; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    const uint64_t per = (p.q + gridDim.x - 1) / gridDim.x;
    const uint64_t beg = per * blockIdx.x;
    const uint64_t end = min(p.q, beg + per);
    for (uint64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
        const int f = family_of(p, i);
        uint32_t bin = kInvalidBin, pos = 0;
        if (f >= 0) {
            const ModelDev& m = p.m[f];
            const double q18 = normalize(raw18_of(p, i), m.lo[18], m.hi[18]);
            pos = lower_bound(m.key18, m.n, q18);
            bin = m.bin_base + (pos >> m.bin_shift);
        }
        const uint32_t b = bin == kInvalidBin ? n_bins - 1 : bin;
        qbin[i] = b;
        qpos[i] = pos;
        atomicAdd(&sh[b], 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < n_bins; b += blockDim.x)
        hist[static_cast<uint64_t>(b) * gridDim.x + blockIdx.x] = sh[b];
}

// The fp32 path's query record of row i (family f >= 0, start position pos
// over the keys): featurise, the 19 correctly rounded normalisations
// (estimators.cpp:439-441), the fp32 error radius eta, t_in.
template <int FMT>
__device__ __forceinline__ void write_qrec(const KnnParams& p, uint64_t i, int f, uint32_t pos,
                                           const double* __restrict__ keys, double2* rec) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const ModelDev& m = p.m[f];
    double raw[kDims];
    load_raw<FMT>(p, static_cast<uint32_t>(i), raw);
    double qn[kDims];
    double qmax = 0.0;
#pragma unroll
    for (int d = 0; d < kDims; ++d) {
        qn[d] = normalize(raw[d], m.lo[d], m.hi[d]);
        const double av = fabs(qn[d]);
        qmax = (av > qmax || av != av) ? av : qmax;
    }
    // active dims in ascending order are adim[0..]: walk d with a running j
    double e2 = 0.0;
    int j = 0;
#pragma unroll
    for (int d = 0; d < kDims; ++d) {
        if ((m.active >> d) & 1u) {
            const double w = d == 18 ? 64.0 : 1.0;
            const double ej = 2.0 * 0x1.0p-24 * (1.0 + 0x1.0p-24) * w * (m.pmax[j] + fabs(qn[d])) + 0x1.0p-140;
            e2 += ej * ej;
            ++j;
        }
    }
    double eta = sqrt(e2) * (1.0 + 0x1.0p-40);
    if (!(qmax <= 1e15)) eta = inf;  // huge or NaN query: exact on every point
#pragma unroll
    for (int h = 0; h < 9; ++h) rec[h] = make_double2(qn[2 * h], qn[2 * h + 1]);
    rec[9] = make_double2(qn[18], eta);
    const double t_in = fmin(pos > 0 ? t18_of(keys[pos - 1], qn[18]) : inf,
                             pos < m.n ? t18_of(keys[pos], qn[18]) : inf);
    rec[10] = make_double2(t_in, __longlong_as_double(static_cast<long long>(pos)));
}

// Sorted layout, pass 2 (after the bucketing): the record of the row in each
// bucketed slot, written at the slot, so the search reads its warp's 32
// records as one contiguous 5.6 KB span instead of 32 random ones.
template <int FMT>
__global__ void __launch_bounds__(256) knn_prep_sorted(KnnParams p, const uint32_t* __restrict__ perm,
                                                       const uint32_t* __restrict__ qpos) {
    const uint64_t slot = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (slot >= p.q) return;
    const uint32_t row = perm[slot];
    const int f = family_of_t<FMT>(p, row);
    if (f < 0) return;
    write_qrec<FMT>(p, row, f, qpos[row], p.m[f].key18, reinterpret_cast<double2*>(p.qrec + slot * kQrec));
}

// bucket / bytes from slot order back to row order.
__global__ void __launch_bounds__(256) knn_unpermute(uint64_t q, const uint32_t* __restrict__ perm,
                                                     const int32_t* __restrict__ sb, const uint64_t* __restrict__ sby,
                                                     int32_t* __restrict__ bucket, uint64_t* __restrict__ bytes) {
    const uint64_t slot = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (slot >= q) return;
    const uint32_t row = perm[slot];
    if (bucket) bucket[row] = sb[slot];
    if (bytes) bytes[row] = sby[slot];
}

// Pass 1 of the fp32 path: knn_keys plus the whole per-query setup of the
// search (featurise, the 19 correctly rounded normalisations of
// estimators.cpp:439-441, the fp32 error radius eta), written as a 160-B
// record per row. This high-occupancy streaming kernel hides the division
// latency that the search kernel (4 warps per scheduler) cannot.
// When every model's keys fit (kPrepKeysMax doubles), the binary search runs
// on a shared-memory copy of key18 (12 dependent probes per row).
constexpr uint32_t kPrepKeysMax = 8192;

template <int FMT>
#ifndef KNN_PREP_MINB
#define KNN_PREP_MINB 2
#endif
__global__ void __launch_bounds__(512, KNN_PREP_MINB) knn_prep(KnnParams p, uint32_t n_bins, uint32_t* __restrict__ qbin, uint32_t* __restrict__ qpos,
                         uint32_t* __restrict__ hist, int keys_in_smem) {
    extern __shared__ __align__(16) uint32_t sh[];
    double* skeys = reinterpret_cast<double*>(sh + ((n_bins + 3) & ~3u));
    const double* keys[CARMA_FAMILIES];
    {
        uint32_t off = 0;
        for (int f = 0; f < CARMA_FAMILIES; ++f) {
            keys[f] = p.m[f].key18;
            if (keys_in_smem && p.m[f].present) {
                for (uint32_t i = threadIdx.x; i < p.m[f].n; i += blockDim.x) skeys[off + i] = p.m[f].key18[i];
                keys[f] = skeys + off;
                off += static_cast<uint32_t>(p.m[f].n);
            }
        }
    }
    for (uint32_t b = threadIdx.x; b < n_bins; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const uint64_t per = (p.q + gridDim.x - 1) / gridDim.x;
    const uint64_t beg = per * blockIdx.x;
    const uint64_t end = min(p.q, beg + per);
    for (uint64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
        const int f = family_of_t<FMT>(p, i);
        uint32_t bin = kInvalidBin, pos = 0;
        if (f >= 0) {
            const ModelDev& m = p.m[f];
            pos = lower_bound_any(keys[f], static_cast<uint32_t>(m.n), normalize(raw18_of(p, i), m.lo[18], m.hi[18]));
            write_qrec<FMT>(p, i, f, pos, keys[f], reinterpret_cast<double2*>(p.qrec + i * kQrec));
            bin = m.bin_base + (pos >> m.bin_shift);
        }
        const uint32_t b = bin == kInvalidBin ? n_bins - 1 : bin;
        qbin[i] = b;
        qpos[i] = pos;
        atomicAdd(&sh[b], 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < n_bins; b += blockDim.x)
        hist[static_cast<uint64_t>(b) * gridDim.x + blockIdx.x] = sh[b];
}

// Exclusive scan of the [bin][cta] histogram matrix in three small steps:
// per-bin totals (warp per bin), a one-CTA scan of the bin totals, then a
// warp-level scan over each bin's CTAs.
__global__ void bin_totals(const uint32_t* __restrict__ hist, uint32_t n_bins, uint32_t n_ctas,
                           uint32_t* __restrict__ tot) {
    const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (b >= n_bins) return;
    uint32_t s = 0;
    for (uint32_t c = lane; c < n_ctas; c += 32) s += hist[static_cast<uint64_t>(b) * n_ctas + c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) tot[b] = s;
}

__global__ void scan_bins(uint32_t* __restrict__ v, uint32_t n) {
    __shared__ uint32_t part[1024];
    const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t beg = per * threadIdx.x, end = min(n, beg + per);
    uint32_t s = 0;
    for (uint32_t i = beg; i < end; ++i) s += v[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (unsigned off = 1; off < blockDim.x; off <<= 1) {
        const uint32_t add = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - s;
    for (uint32_t i = beg; i < end; ++i) {
        const uint32_t x = v[i];
        v[i] = run;
        run += x;
    }
}

__global__ void bin_offsets(uint32_t* __restrict__ hist, uint32_t n_bins, uint32_t n_ctas,
                            const uint32_t* __restrict__ base) {
    const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (b >= n_bins) return;
    uint32_t run = base[b];
    uint32_t* row = hist + static_cast<uint64_t>(b) * n_ctas;
    for (uint32_t c0 = 0; c0 < n_ctas; c0 += 32) {
        const uint32_t c = c0 + lane;
        const uint32_t x = c < n_ctas ? row[c] : 0;
        uint32_t incl = x;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<unsigned>(o)) incl += y;
        }
        if (c < n_ctas) row[c] = run + incl - x;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// Pass 2: scatter row ids into bin order (same CTA tiling as knn_keys).
__global__ void knn_scatter(uint64_t q, uint32_t n_bins, const uint32_t* __restrict__ qbin,
                            const uint32_t* __restrict__ base, uint32_t* __restrict__ perm) {
    extern __shared__ uint32_t sh[];
    for (uint32_t b = threadIdx.x; b < n_bins; b += blockDim.x)
        sh[b] = base[static_cast<uint64_t>(b) * gridDim.x + blockIdx.x];
    __syncthreads();
    const uint64_t per = (q + gridDim.x - 1) / gridDim.x;
    const uint64_t beg = per * blockIdx.x;
    const uint64_t end = min(q, beg + per);
    for (uint64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
        const uint32_t slot = atomicAdd(&sh[qbin[i]], 1u);
        perm[slot] = static_cast<uint32_t>(i);
    }
}

// k best (d2, training index) pairs, ascending, register resident. For a
// runtime k < K the first K-k slots hold (-inf, INT_MIN) sentinels that never
// move, so the k-th best is always slot K-1 (static register indexing).
template <int K>
struct TopK {
    double d[K];
    int32_t id[K];
    __device__ __forceinline__ void init(int k) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const bool sentinel = j < K - k;
            d[j] = __longlong_as_double(sentinel ? 0xfff0000000000000ll : 0x7ff0000000000000ll);
            id[j] = sentinel ? static_cast<int32_t>(0x80000000u) : 0x7fffffff;
        }
    }
    __device__ __forceinline__ double kth() const { return d[K - 1]; }
    __device__ __forceinline__ void insert(double d2, int32_t oi) {
        if (!(d2 < d[K - 1] || (d2 == d[K - 1] && oi < id[K - 1]))) return;
        bool placed = false;
#pragma unroll
        for (int j = K - 1; j >= 0; --j) {
            if (placed) continue;
            const bool prev_greater =
                j > 0 && (d[j - 1] > d2 || (d[j - 1] == d2 && id[j - 1] > oi));
            if (prev_greater) {
                d[j] = d[j - 1];
                id[j] = id[j - 1];
            } else {
                d[j] = d2;
                id[j] = oi;
                placed = true;
            }
        }
    }
};

template <int K>
__device__ __forceinline__ void insert_block(TopK<K>& top, const double (&d2)[kBlock], unsigned cand,
                                          const int32_t* orig) {
    while (cand) {
        const int c = __ffs(cand) - 1;
        cand &= cand - 1;
        double v = d2[0];
#pragma unroll
        for (int j = 1; j < kBlock; ++j)
            if (j == c) v = d2[j];
        top.insert(v, __ldg(orig + c));
    }
}


template <int K>
__global__ void __launch_bounds__(128, 4)
    knn_search(KnnParams p, const uint32_t* __restrict__ perm, const uint32_t* __restrict__ qpos,
               int32_t* __restrict__ bucket_out, uint64_t* __restrict__ bytes_out,
               double* __restrict__ topk_d2, int64_t* __restrict__ topk_idx,
               unsigned long long* __restrict__ evals) {
    const unsigned lane = threadIdx.x & 31;
    // Each CTA walks one contiguous range of the bin-sorted queries (its
    // warps interleaved), so an SM's warps search neighbouring regions of the
    // model and the points stay L1-resident.
    const uint64_t total_w = (p.q + 31) / 32;
    const uint64_t per_cta = (total_w + gridDim.x - 1) / gridDim.x;
    const uint64_t w_beg = per_cta * blockIdx.x;
    const uint64_t w_end = min(total_w, w_beg + per_cta);
    const unsigned wpc = blockDim.x >> 5;
    unsigned long long my_evals = 0;

    for (uint64_t w = w_beg + (threadIdx.x >> 5); w < w_end; w += wpc) {
        const uint64_t slot = w * 32 + lane;
        const bool live = slot < p.q;
        const uint32_t row = live ? perm[slot] : 0;
        const int fam = live ? family_of(p, row) : -1;
        if (live && fam < 0) {  // FamilyMismatch -> no estimate
            if (bucket_out) bucket_out[row] = -1;
            if (bytes_out) bytes_out[row] = ~0ull;
        }
        unsigned pending = __ballot_sync(0xffffffffu, fam >= 0);
        while (pending) {
            const int f = __shfl_sync(0xffffffffu, fam, __ffs(pending) - 1);
            const bool mine = fam == f && ((pending >> lane) & 1u);
            const unsigned members = __ballot_sync(0xffffffffu, mine);
            pending &= ~members;
            const ModelDev& m = p.m[f];
            const int k = static_cast<int>(m.k < K ? m.k : K);

            // Query in registers (normalised), same arithmetic as estimators.cpp:439-441.
            double q[kDims];
            if (mine) {
                double raw[kDims];
                if (p.format == CARMA_ROWS_SCALAR) {
                    const double* r = static_cast<const double*>(p.rows) + static_cast<uint64_t>(row) * kDims;
#pragma unroll
                    for (int d = 0; d < kDims; ++d) raw[d] = r[d];
                } else if (p.format == CARMA_ROWS_PACKED) {
                    featurize_packed(p, static_cast<const carma_feature_packed*>(p.rows)[row], raw);
                } else if (p.format == CARMA_ROWS_BITPACKED) {
                    featurize_bits(p, bit_row(p, row), raw);
                } else {
                    featurize(static_cast<const carma_feature_row*>(p.rows)[row], raw);
                }
#pragma unroll
                for (int d = 0; d < kDims; ++d) q[d] = normalize(raw[d], m.lo[d], m.hi[d]);
            } else {
#pragma unroll
                for (int d = 0; d < kDims; ++d) q[d] = 0.0;
            }
            TopK<K> top;
            top.init(k);

            // Common frontier: evaluated range [L, R), started at the middle
            // member's position. A lane's own position pos may differ from the
            // start, so its per-side lower bound is t18 of the next point only
            // when that side moves away from pos; otherwise it is t_in, the
            // minimum t18 around pos (t18 decreases toward pos, then grows).
            unsigned mm = members;
            for (int j = (__popc(members) - 1) / 2; j > 0; --j) mm &= mm - 1;
            const int mid_lane = __ffs(mm) - 1;
            const int64_t n = static_cast<int64_t>(m.n);
            const int64_t pos = live ? static_cast<int64_t>(qpos[row]) : 0;
            const int64_t start = __shfl_sync(0xffffffffu, pos, mid_lane);
            int64_t L = start, R = start;
            const double inf = __longlong_as_double(0x7ff0000000000000ll);
            const double t_in = fmin(pos > 0 ? t18_of(__ldg(m.key18 + pos - 1), q[18]) : inf,
                                     pos < n ? t18_of(__ldg(m.key18 + pos), q[18]) : inf);
            double tl = L > 0 ? (L <= pos ? t18_of(__ldg(m.key18 + L - 1), q[18]) : t_in) : inf;
            double tr = R < n ? (R >= pos ? t18_of(__ldg(m.key18 + R), q[18]) : t_in) : inf;
            const uint32_t act = m.active;
            uint64_t steps = 0;
            for (;;) {
                const double kth = top.kth();
                const bool need_l = mine && L > 0 && tl <= kth;
                const bool need_r = mine && R < n && tr <= kth;
                const unsigned bl = __ballot_sync(0xffffffffu, need_l);
                const unsigned br = __ballot_sync(0xffffffffu, need_r);
                if ((bl | br) == 0) break;
                // Best-first for the representative lane, else whichever side is wanted.
                const double rl = __shfl_sync(0xffffffffu, need_l ? tl : inf, mid_lane);
                const double rr = __shfl_sync(0xffffffffu, need_r ? tr : inf, mid_lane);
                const bool go_left = bl != 0 && (br == 0 || rl <= rr);
                // Next block of kBlock contiguous points on that side. The
                // stored model is padded by kBlock points at both ends, so a
                // block never leaves the allocation; slots outside [0, n) are
                // evaluated but never inserted.
                int64_t s0;
                unsigned valid;
                if (go_left) {
                    s0 = L - kBlock;
                    valid = L >= kBlock ? 0xffu : (0xffu << (kBlock - L)) & 0xffu;
                    L = L > kBlock ? L - kBlock : 0;
                } else {
                    s0 = R;
                    valid = n - R >= kBlock ? 0xffu : (1u << (n - R)) - 1u;
                    R = n - R > kBlock ? R + kBlock : n;
                }
                const int64_t cnt = __popc(valid);
                // kBlock independent accumulation chains; each d2 keeps the
                // reference's dim order. Dims outside `act` contribute exactly
                // +0.0 and are skipped (warp-uniform branch).
                double d2[kBlock];
                const double* blk = m.pts + s0 * kStride;
#pragma unroll
                for (int c = 0; c < kBlock; ++c) d2[c] = 0.0;
#pragma unroll
                for (int h = 0; h < 9; ++h) {
                    if (!(act & (3u << (2 * h)))) continue;
                    double2 v[kBlock];
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) v[c] = __ldg(reinterpret_cast<const double2*>(blk + c * kStride) + h);
                    if (act & (1u << (2 * h))) {
#pragma unroll
                        for (int c = 0; c < kBlock; ++c) {
                            const double a = __dsub_rn(v[c].x, q[2 * h]);
                            d2[c] = __dadd_rn(d2[c], __dmul_rn(a, a));
                        }
                    }
                    if (act & (2u << (2 * h))) {
#pragma unroll
                        for (int c = 0; c < kBlock; ++c) {
                            const double b = __dsub_rn(v[c].y, q[2 * h + 1]);
                            d2[c] = __dadd_rn(d2[c], __dmul_rn(b, b));
                        }
                    }
                }
                if (act & (1u << 18)) {
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) {
                        const double a = __dmul_rn(__dsub_rn(__ldg(blk + c * kStride + 18), q[18]), 64.0);
                        d2[c] = __dadd_rn(d2[c], __dmul_rn(a, a));
                    }
                }
                // Candidates: d2 <= k-th best (ties resolved by index inside).
                // The insertion is rare after the first blocks; keep it off
                // the straight-line path so it is not if-converted.
                const double kb = top.kth();
                unsigned cand = 0;
#pragma unroll
                for (int c = 0; c < kBlock; ++c) cand |= (d2[c] <= kb) ? (1u << c) : 0u;
                cand &= valid;
                if (!mine) cand = 0;
                if (cand) insert_block<K>(top, d2, cand, m.orig + s0);
                if (go_left) tl = L > 0 ? (L <= pos ? t18_of(__ldg(m.key18 + L - 1), q[18]) : t_in) : inf;
                else tr = R < n ? (R >= pos ? t18_of(__ldg(m.key18 + R), q[18]) : t_in) : inf;
                steps += static_cast<uint64_t>(cnt);
            }
            my_evals += steps * static_cast<unsigned long long>(__popc(members));

            if (mine) {
                // Vote over the kk = min(k, n) neighbours (estimators.cpp:463-474):
                // real entries are slots [K-k, K) whose id is a training index.
                int best = 0, best_votes = 0;
                // labels of the k nearest, loaded once (vm: filled slots)
                int lab[K];
                unsigned vm = 0;
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    const bool ok = a >= K - k && top.id[a] != 0x7fffffff;
                    lab[a] = ok ? __ldg(m.label_by_orig + top.id[a]) : 0;
                    vm |= ok ? (1u << a) : 0u;
                }
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    if (!((vm >> a) & 1u)) continue;
                    const int la = lab[a];
                    int votes = 0;
#pragma unroll
                    for (int b = 0; b < K; ++b) votes += (((vm >> b) & 1u) && lab[b] == la) ? 1 : 0;
                    if (votes > best_votes || (votes == best_votes && la > best)) {
                        best = la;
                        best_votes = votes;
                    }
                }
                if (bucket_out) bucket_out[row] = best;
                if (bytes_out) bytes_out[row] = (static_cast<uint64_t>(best) + 1ull) * m.bucket_range;
                if (topk_d2 || topk_idx) {
#pragma unroll
                    for (int a = 0; a < K; ++a) {
                        if (a < K - k) continue;
                        const uint64_t o = static_cast<uint64_t>(row) * m.k + (a - (K - k));
                        const bool real = top.id[a] != 0x7fffffff;
                        if (topk_d2) topk_d2[o] = real ? top.d[a] : inf;
                        if (topk_idx) topk_idx[o] = real ? top.id[a] : -1;
                    }
                }
            }
        }
    }
    if (evals && lane == 0 && my_evals) atomicAdd(evals, my_evals);
}

// ------------------------------------------------------------------------
// knn_search_f32: the same exact search with an fp32 pre-filter.
//
// Phase A walks the frontier in blocks of 8 points exactly like knn_search,
// but evaluates each point in fp32 (one FADD + FFMA per active dim, from a
// compact fp32 copy of the model). With a = the fp32 difference vector and
// b = the real weighted difference vector, every component satisfies
// |a_j - b_j| <= eps_j = 2u(1+u) w_j (pmax_j + |q_j|)  (u = 2^-24: two input
// conversions + one rounded subtraction), so ||a - b|| <= eta and
//   LB = (sqrt(sf/(1+g)) - eta)^2 (1-g64)  <=  d2_fp64  <=
//   UB = (sqrt(sf/(1-g)) + eta)^2 (1+g64)
// where sf is the FFMA-accumulated sum (relative error g = 17u) and g64
// bounds the reference's own fp64 rounding. A point can enter the exact
// top-k only if LB <= kth, tested without a sqrt as sf <= T_lb(kth). kth is
// an upper bound of the exact k-th best: the k-th smallest UB seen so far
// (UB is monotone in sf, so that is UB of the k-th smallest sf, kept in a
// branch-free sorted register array), or the exact k-th best after a flush.
// Surviving candidates are buffered per lane and evaluated exactly in fp64
// (reference arithmetic) in phase B, which also runs before any lane's
// buffer could overflow. Queries whose magnitudes
// could overflow fp32 (|q| > 1e15 or NaN) never filter (eta = inf) and so
// are evaluated exactly on every visited point.
// ------------------------------------------------------------------------

// Bound arithmetic in fp32 with directed rounding (every step rounds toward
// the safe side). Constants: g = 17 u (FFMA accumulation of 16 terms),
// g64 = 64 * 2^-53 (the reference's own fp64 rounding of d2), each folded
// into a factor that dominates it.
struct F32Bounds {
    static constexpr float up_g = 1.0f + 0x1.0p-19f;     // >= (1 + g), g = 17u covers 2 x 8-term chains + fold
    static constexpr float dn_g = 1.0f - 0x1.0p-19f;     // <= (1 - g)
    static constexpr float up_g64 = 1.0f + 0x1.0p-22f;   // >= 1/(1 - g64), (1 + g64)
    static constexpr float dn_g64 = 1.0f - 0x1.0p-22f;   // <= 1/(1 + g64)
};

// Largest sf that may still hold a candidate: sf <= (1+g)(sqrt(kth/(1-g64)) + eta)^2.
__device__ __forceinline__ float t_lb(float kth, float eta) {
    const float r = __fadd_ru(__fsqrt_ru(__fmul_ru(kth, F32Bounds::up_g64)), eta);
    return __fmul_ru(__fmul_ru(r, r), F32Bounds::up_g);  // inf stays inf
}

// UB = (sqrt(sf/(1-g)) + eta)^2 (1+g64), rounded up.
__device__ __forceinline__ float ub_of(float sf, float eta) {
    const float r = __fadd_ru(__fsqrt_ru(__fmul_ru(sf, F32Bounds::up_g)), eta);
    return __fmul_ru(__fmul_ru(r, r), F32Bounds::up_g64);
}

// Packed fp32x2 arithmetic (sm_100: FADD2 / FFMA2, two lanes per instruction).
__device__ __forceinline__ unsigned long long f2pack(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 f2unpack(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ unsigned long long f2sub(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Sorted insert into the ascending k-smallest array a, branch-free: slot j of
// the result is min(a[j], max(a[j-1], v)); v = +inf leaves a unchanged and
// the -1 sentinels (slots j < K-k) never move.
template <int K>
__device__ __forceinline__ void sorted_insert(float (&a)[K], float v) {
#pragma unroll
    for (int j = K - 1; j > 0; --j) a[j] = fminf(a[j], fmaxf(a[j - 1], v));
    a[0] = fminf(a[0], v);
}

#ifndef KNN_LAYOUT
#define KNN_LAYOUT 0
#endif
#ifndef KNN_SPLIT
#define KNN_SPLIT 4
#endif
#ifndef KNN_F32_CTAS
#define KNN_F32_CTAS 4
#endif
// Host-buffer calls pipeline H2D / search / D2H over chunks of this many rows
// on two streams.
#ifndef KNN_E2E_SMALL_LOG2
#define KNN_E2E_SMALL_LOG2 18
#endif
#ifndef KNN_E2E_CHUNK_LOG2
#define KNN_E2E_CHUNK_LOG2 21
#endif
constexpr size_t kF32Smem = kDims * 128 * 8 + kCandCap * 128 * 8 + 4 * 2 * kBlock * kF32Dims * 4;
template <int K, int FMT>
__global__ void __launch_bounds__(128, KNN_F32_CTAS)
    knn_search_f32(KnnParams p, const uint32_t* __restrict__ perm, const uint32_t* __restrict__ qpos,
                   int32_t* __restrict__ bucket_out, uint64_t* __restrict__ bytes_out,
                   double* __restrict__ topk_d2, int64_t* __restrict__ topk_idx,
                   unsigned long long* __restrict__ evals) {
    // Per-thread rows are stored column-major ([item][thread]) so that lanes
    // touching their own rows never share a bank. Dynamic shared memory
    // (kF32Smem bytes): qsh[19][128] f64, cbuf_i/cbuf_s[kCandCap][128],
    // per warp the next fp32 block on the left [0] and right [1] of the frontier.
    extern __shared__ __align__(16) char f32_smem[];
    auto qsh = reinterpret_cast<double (*)[128]>(f32_smem);
    auto cbuf_i = reinterpret_cast<uint32_t (*)[128]>(f32_smem + kDims * 128 * 8);
    auto cbuf_s = reinterpret_cast<float (*)[128]>(f32_smem + kDims * 128 * 8 + kCandCap * 128 * 4);
    auto stage = reinterpret_cast<float4 (*)[2][kBlock * kF32Dims / 4]>(f32_smem + kDims * 128 * 8 +
                                                                          kCandCap * 128 * 8);
    const unsigned lane = threadIdx.x & 31;
    const unsigned tid = threadIdx.x;
    float4 (*stg)[kBlock * kF32Dims / 4] = stage[threadIdx.x >> 5];
    const uint64_t total_w = (p.q + 31) / 32;
    const uint64_t per_cta = (total_w + gridDim.x - 1) / gridDim.x;
    const uint64_t w_beg = per_cta * blockIdx.x;
    const uint64_t w_end = min(total_w, w_beg + per_cta);
    const unsigned wpc = blockDim.x >> 5;
    unsigned long long my_visits = 0, my_exact = 0;
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const float finf = __int_as_float(0x7f800000);

    for (uint64_t w = w_beg + (threadIdx.x >> 5); w < w_end; w += wpc) {
        const uint64_t slot = w * 32 + lane;
        const bool live = slot < p.q;
        const uint32_t row = live ? perm[slot] : 0;
        const int fam = live ? family_of_t<FMT>(p, row) : -1;
        const uint64_t orow = p.out_by_slot ? slot : row;  // output index
        if (live && fam < 0) {  // FamilyMismatch -> no estimate
            if (bucket_out) bucket_out[orow] = -1;
            if (bytes_out) bytes_out[orow] = ~0ull;
        }
        unsigned pending = __ballot_sync(0xffffffffu, fam >= 0);
        while (pending) {
            const int f = __shfl_sync(0xffffffffu, fam, __ffs(pending) - 1);
            const bool mine = fam == f && ((pending >> lane) & 1u);
            const unsigned members = __ballot_sync(0xffffffffu, mine);
            pending &= ~members;
            const ModelDev& m = p.m[f];
            const int k = static_cast<int>(m.k < K ? m.k : K);

            // Query: exact fp64 normalisation (estimators.cpp:439-441) into
            // The query record written by knn_prep: normalised query into
            // shared memory, eta, and the fp32 copy of the active dims.
            float qf[kF32Dims];
            double eta = 0.0;
            double q18 = 0.0;
            double t_in = inf;  // precomputed by knn_prep
            int32_t pos = 0;
            {
                if (mine) {
                    const double2* rec =
                        reinterpret_cast<const double2*>(p.qrec + (p.qrec_by_slot ? slot : static_cast<uint64_t>(row)) * kQrec);
#pragma unroll
                    for (int h = 0; h < 9; ++h) {
                        const double2 v = __ldg(rec + h);
                        qsh[2 * h][tid] = v.x;
                        qsh[2 * h + 1][tid] = v.y;
                    }
                    const double2 v = __ldg(rec + 9);
                    qsh[18][tid] = v.x;
                    q18 = v.x;
                    eta = v.y;
                    const double2 w = __ldg(rec + 10);
                    t_in = w.x;
                    pos = static_cast<int32_t>(__double_as_longlong(w.y));
                } else {
#pragma unroll
                    for (int d = 0; d < kDims; ++d) qsh[d][tid] = 0.0;
                }
#pragma unroll
                for (int j = 0; j < kF32Dims; ++j) {
                    const int a = m.adim[j];
                    qf[j] = a < kDims ? __double2float_rn((a == 18 ? 64.0 : 1.0) * qsh[a][tid]) : 0.0f;
                }
            }

            unsigned long long qf2[kF32Dims / 2];
#pragma unroll
            for (int j = 0; j < kF32Dims / 2; ++j) qf2[j] = f2pack(qf[2 * j], qf[2 * j + 1]);
            TopK<K> top;
            top.init(k);
            // k smallest fp32 sums seen (same sentinel layout as TopK). UB is
            // monotone in sf, so ub_of(sfk[K-1]) is the k-th smallest UB.
            float sfk[K];
#pragma unroll
            for (int j = 0; j < K; ++j) sfk[j] = j < K - k ? -1.0f : finf;
            double kth = inf;  // filter bound: >= the exact k-th best
            const float etaf = __double2float_ru(eta);
            float T_lb = t_lb(finf, etaf);
            int cnt = 0;

            unsigned mm = members;
            for (int j = (__popc(members) - 1) / 2; j > 0; --j) mm &= mm - 1;
            const int mid_lane = __ffs(mm) - 1;
            // model indices fit int32 (carma_knn_set_model rejects n > 2^31 - 1)
            const int32_t n = static_cast<int32_t>(m.n);
            const int32_t start = __shfl_sync(0xffffffffu, pos, mid_lane);
            int32_t L = start, R = start;
            double tl = L > 0 ? (L <= pos ? t18_of(__ldg(m.key18 + L - 1), q18) : t_in) : inf;
            double tr = R < n ? (R >= pos ? t18_of(__ldg(m.key18 + R), q18) : t_in) : inf;
            uint64_t visits = 0, exact = 0;
            // Stage both neighbouring blocks (one coalesced 16-B load per lane
            // each); every step then prefetches the next block on its side.
            const float4* pf4 = reinterpret_cast<const float4*>(m.ptsf);
            __syncwarp();
            stg[0][lane] = __ldg(pf4 + static_cast<int64_t>(L - kBlock) * (kF32Dims / 4) + lane);
            stg[1][lane] = __ldg(pf4 + static_cast<int64_t>(R) * (kF32Dims / 4) + lane);
            __syncwarp();

            // Phase B: exact fp64 evaluation (reference arithmetic) of the
            // buffered candidates that still pass the (possibly tightened)
            // bound, then tighten kth.
            auto flush = [&]() {
                // Two candidates per lane per round: their fp64 chains (19
                // dependent adds each, reference order) interleave, which
                // halves this latency-bound phase. The top-k is independent
                // of insertion order.
                for (;;) {
                    if (!__any_sync(0xffffffffu, cnt > 0)) break;
                    uint32_t ia = 0xffffffffu, ib = 0xffffffffu;
                    if (cnt > 0) {
                        --cnt;
                        if (!(cbuf_s[cnt][tid] > T_lb)) ia = cbuf_i[cnt][tid];
                    }
                    if (cnt > 0) {
                        --cnt;
                        if (!(cbuf_s[cnt][tid] > T_lb)) ib = cbuf_i[cnt][tid];
                    }
                    if (ia == 0xffffffffu) {
                        ia = ib;
                        ib = 0xffffffffu;
                    }
                    if (ia != 0xffffffffu) {
                        const bool two = ib != 0xffffffffu;
                        const double* pa = m.pts + static_cast<int64_t>(ia) * kStride;
                        const double* pb = m.pts + static_cast<int64_t>(two ? ib : ia) * kStride;
                        double da = 0.0, db = 0.0;
#pragma unroll
                        for (int h = 0; h < 9; ++h) {
                            const double2 va = __ldg(reinterpret_cast<const double2*>(pa) + h);
                            const double2 vb = __ldg(reinterpret_cast<const double2*>(pb) + h);
                            const double q0 = qsh[2 * h][tid], q1 = qsh[2 * h + 1][tid];
                            const double a0 = __dsub_rn(va.x, q0), b0 = __dsub_rn(vb.x, q0);
                            da = __dadd_rn(da, __dmul_rn(a0, a0));
                            db = __dadd_rn(db, __dmul_rn(b0, b0));
                            const double a1 = __dsub_rn(va.y, q1), b1 = __dsub_rn(vb.y, q1);
                            da = __dadd_rn(da, __dmul_rn(a1, a1));
                            db = __dadd_rn(db, __dmul_rn(b1, b1));
                        }
                        const double a = __dmul_rn(__dsub_rn(__ldg(pa + 18), q18), 64.0);
                        const double b = __dmul_rn(__dsub_rn(__ldg(pb + 18), q18), 64.0);
                        da = __dadd_rn(da, __dmul_rn(a, a));
                        db = __dadd_rn(db, __dmul_rn(b, b));
                        top.insert(da, __ldg(m.orig + ia));
                        ++exact;
                        if (two) {
                            top.insert(db, __ldg(m.orig + ib));
                            ++exact;
                        }
                    }
                }
                const double kx = top.kth();
                if (kx < kth) {
                    kth = kx;
                    T_lb = t_lb(__double2float_ru(kth), etaf);
                }
            };

            for (;;) {
                const bool need_l = mine && L > 0 && tl <= kth;
                const bool need_r = mine && R < n && tr <= kth;
                const unsigned bl = __ballot_sync(0xffffffffu, need_l);
                const unsigned br = __ballot_sync(0xffffffffu, need_r);
                const bool done = (bl | br) == 0;
                // Phase B at one code site: at the end, and whenever a lane
                // could not buffer a whole block.
                if (done || __any_sync(0xffffffffu, cnt > kCandCap - kBlock)) {
                    flush();
                    if (done) break;
                }
                const double rl = __shfl_sync(0xffffffffu, need_l ? tl : inf, mid_lane);
                const double rr = __shfl_sync(0xffffffffu, need_r ? tr : inf, mid_lane);
                const bool go_left = bl != 0 && (br == 0 || rl <= rr);
                int32_t s0;
                unsigned valid;
                if (go_left) {
                    s0 = L - kBlock;
                    valid = L >= kBlock ? 0xffu : (0xffu << (kBlock - L)) & 0xffu;
                    L = L > kBlock ? L - kBlock : 0;
                } else {
                    s0 = R;
                    valid = n - R >= kBlock ? 0xffu : (1u << (n - R)) - 1u;
                    R = n - R > kBlock ? R + kBlock : n;
                }
                // Phase A: fp32 sums for the block's 8 points, read from the
                // staged copy; the side's next block loads meanwhile.
                const int side = go_left ? 0 : 1;
                const int32_t nxt = go_left ? L - kBlock : R;
                const float4 pre = __ldg(pf4 + static_cast<int64_t>(nxt) * (kF32Dims / 4) + lane);
                // The side's next bound key, loaded before the block's math so
                // its latency hides behind it (consumed by the next ballot).
                const int32_t kidx = go_left ? (L > 0 ? L - 1 : 0) : (R < n ? R : n - 1);
                const double knext = __ldg(m.key18 + kidx);
                // Two packed partial sums per point (even / odd active dims),
                // folded at the end: any order of the 16 non-negative terms
                // stays within the 17u accumulation bound.
                float sf[kBlock];
                const float4* blk = stg[side];
                unsigned long long acc[kBlock];
#pragma unroll
                for (int c = 0; c < kBlock; ++c) acc[c] = 0ull;
#pragma unroll
                for (int h = 0; h < kF32Dims / 4; ++h) {
                    float4 v[kBlock];
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) v[c] = blk[c * (kF32Dims / 4) + h];
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) {
                        const unsigned long long d0 = f2sub(f2pack(v[c].x, v[c].y), qf2[2 * h]);
                        acc[c] = f2fma(d0, d0, acc[c]);
                        const unsigned long long d1 = f2sub(f2pack(v[c].z, v[c].w), qf2[2 * h + 1]);
                        acc[c] = f2fma(d1, d1, acc[c]);
                    }
                }
#pragma unroll
                for (int c = 0; c < kBlock; ++c) {
                    const float2 a = f2unpack(acc[c]);
                    sf[c] = a.x + a.y;
                }
                __syncwarp();
                stg[side][lane] = pre;
                __syncwarp();
                visits += static_cast<uint64_t>(__popc(valid));
                // Fast path: after the first blocks almost no point improves
                // the k smallest sums or passes the bound; one min decides.
                float mn = sf[0];
#pragma unroll
                for (int c = 1; c < kBlock; ++c) mn = fminf(mn, sf[c]);
                unsigned cand = 0;
                if (mine && (mn < sfk[K - 1] || !(mn > T_lb))) {
                    unsigned upd = 0;
                    const float sk = sfk[K - 1];
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) upd |= (sf[c] < sk) ? (1u << c) : 0u;
                    upd &= valid;
                    if (upd) {  // the k smallest sums moved: tighten the bound
                        // every point of the block through the branch-free
                        // insert (+inf, or any value >= the k-th, leaves the
                        // array unchanged); cheaper than extracting the set
                        // bits one by one (11.69 -> 11.60 ms on c2)
#pragma unroll
                        for (int c = 0; c < kBlock; ++c) sorted_insert<K>(sfk, ((upd >> c) & 1u) ? sf[c] : finf);
                        const float kub = ub_of(sfk[K - 1], etaf);
                        if (static_cast<double>(kub) < kth) {
                            kth = static_cast<double>(kub);
                            T_lb = t_lb(kub, etaf);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) cand |= !(sf[c] > T_lb) ? (1u << c) : 0u;
                    cand &= valid;
                }
                if (cand) {
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) {
                        if ((cand >> c) & 1u) {
                            cbuf_i[cnt][tid] = static_cast<uint32_t>(s0 + c);
                            cbuf_s[cnt][tid] = sf[c];
                            ++cnt;
                        }
                    }
                }
                if (go_left) tl = L > 0 ? (L <= pos ? t18_of(knext, q18) : t_in) : inf;
                else tr = R < n ? (R >= pos ? t18_of(knext, q18) : t_in) : inf;
            }
            my_visits += visits;
            my_exact += exact;

            if (mine) {
                int best = 0, best_votes = 0;
                // labels of the k nearest, loaded once (vm: filled slots)
                int lab[K];
                unsigned vm = 0;
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    const bool ok = a >= K - k && top.id[a] != 0x7fffffff;
                    lab[a] = ok ? __ldg(m.label_by_orig + top.id[a]) : 0;
                    vm |= ok ? (1u << a) : 0u;
                }
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    if (!((vm >> a) & 1u)) continue;
                    const int la = lab[a];
                    int votes = 0;
#pragma unroll
                    for (int b = 0; b < K; ++b) votes += (((vm >> b) & 1u) && lab[b] == la) ? 1 : 0;
                    if (votes > best_votes || (votes == best_votes && la > best)) {
                        best = la;
                        best_votes = votes;
                    }
                }
                if (bucket_out) bucket_out[orow] = best;
                if (bytes_out) bytes_out[orow] = (static_cast<uint64_t>(best) + 1ull) * m.bucket_range;
                if (topk_d2 || topk_idx) {
#pragma unroll
                    for (int a = 0; a < K; ++a) {
                        if (a < K - k) continue;
                        const uint64_t o = static_cast<uint64_t>(row) * m.k + (a - (K - k));
                        const bool real = top.id[a] != 0x7fffffff;
                        if (topk_d2) topk_d2[o] = real ? top.d[a] : inf;
                        if (topk_idx) topk_idx[o] = real ? top.id[a] : -1;
                    }
                }
            }
        }
    }
    if (evals) {
        for (int o = 16; o > 0; o >>= 1) {
            my_visits += __shfl_xor_sync(0xffffffffu, my_visits, o);
            my_exact += __shfl_xor_sync(0xffffffffu, my_exact, o);
        }
        if (lane == 0) {
            atomicAdd(evals, my_exact);
            atomicAdd(evals + 1, my_visits);
        }
    }
}

// ------------------------------------------------------------------------
// k > kMaxK: exact brute force, one thread per query. The reference's whole
// predict_scalar (estimators.cpp:438-475) without pruning: every point's d2 in
// the reference's dim order, the k smallest (d2, training index) pairs kept
// sorted in a per-thread list in global scratch ([slot][thread], coalesced),
// the vote over their labels. Used only for models with k > 16 (no register
// top-k); correctness over speed.
template <int FMT>
__global__ void __launch_bounds__(128) knn_brute(KnnParams p, uint64_t q0, uint64_t nq, double* __restrict__ sd2,
                                                 int32_t* __restrict__ sid, int32_t* __restrict__ bucket_out,
                                                 uint64_t* __restrict__ bytes_out, double* __restrict__ topk_d2,
                                                 int64_t* __restrict__ topk_idx) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (t >= nq) return;
    const uint64_t row = q0 + t;
    const int f = family_of_t<FMT>(p, row);
    if (f < 0) {
        if (bucket_out) bucket_out[row] = -1;
        if (bytes_out) bytes_out[row] = ~0ull;
        return;
    }
    const ModelDev& m = p.m[f];
    double raw[kDims], q[kDims];
    load_raw<FMT>(p, row, raw);
#pragma unroll
    for (int d = 0; d < kDims; ++d) q[d] = normalize(raw[d], m.lo[d], m.hi[d]);
    const uint32_t k = static_cast<uint32_t>(m.k < m.n ? m.k : m.n);
    uint32_t cnt = 0;
    for (uint64_t s = 0; s < m.n; ++s) {
        const double* pt = m.pts + s * kStride;
        double d2 = 0.0;
#pragma unroll
        for (int d = 0; d < kDims; ++d) {
            double diff = __dsub_rn(__ldg(pt + d), q[d]);
            if (d == kDims - 1) diff = __dmul_rn(diff, 64.0);
            d2 = __dadd_rn(d2, __dmul_rn(diff, diff));
        }
        const int32_t oi = __ldg(m.orig + s);
        if (cnt == k) {
            const double ld = sd2[(k - 1) * nq + t];
            const int32_t li = sid[(k - 1) * nq + t];
            if (!(d2 < ld || (d2 == ld && oi < li))) continue;
        } else {
            ++cnt;
        }
        uint32_t j = cnt - 1;  // shift larger entries up by one
        while (j > 0) {
            const double pd = sd2[(j - 1) * nq + t];
            const int32_t pi = sid[(j - 1) * nq + t];
            if (!(pd > d2 || (pd == d2 && pi > oi))) break;
            sd2[j * nq + t] = pd;
            sid[j * nq + t] = pi;
            --j;
        }
        sd2[j * nq + t] = d2;
        sid[j * nq + t] = oi;
    }
    // votes; ties go to the larger label (estimators.cpp:463-474)
    int best = 0, best_votes = 0;
    for (uint32_t a = 0; a < cnt; ++a) {
        const int la = __ldg(m.label_by_orig + sid[a * nq + t]);
        int votes = 0;
        for (uint32_t b = 0; b < cnt; ++b) votes += __ldg(m.label_by_orig + sid[b * nq + t]) == la ? 1 : 0;
        if (votes > best_votes || (votes == best_votes && la > best)) {
            best = la;
            best_votes = votes;
        }
    }
    if (bucket_out) bucket_out[row] = best;
    if (bytes_out) bytes_out[row] = (static_cast<uint64_t>(best) + 1ull) * m.bucket_range;
    if (topk_d2 || topk_idx) {
        const double inf = __longlong_as_double(0x7ff0000000000000ll);
        for (uint32_t a = 0; a < m.k; ++a) {
            const uint64_t o = row * m.k + a;
            if (topk_d2) topk_d2[o] = a < cnt ? sd2[a * nq + t] : inf;
            if (topk_idx) topk_idx[o] = a < cnt ? sid[a * nq + t] : -1;
        }
    }
}

// ------------------------------------------------------------------------
// train_learned_estimator on the device (estimators.cpp:344-436).

// Order-preserving 64-bit key of a double (+0 and -0 collapse) and back.
__device__ __forceinline__ unsigned long long fkey(double x) {
    if (x == 0.0) x = 0.0;
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

struct Bounds {
    double lo[kDims], hi[kDims];
};

// lo/hi = min/max of scalar_features over the training rows (:363-374):
// min and max are order-independent, so a reduction gives the sequential
// result (up to the sign of a zero, which the features never carry).
__global__ void fit_bounds(const carma_feature_row* __restrict__ rows, const uint64_t* __restrict__ order,
                           uint64_t train_n, unsigned long long* __restrict__ keys /* [2][19] */) {
    unsigned long long mn[kDims], mx[kDims];
#pragma unroll
    for (int d = 0; d < kDims; ++d) {
        mn[d] = ~0ull;
        mx[d] = 0ull;
    }
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < train_n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double raw[kDims];
        featurize(rows[order[i]], raw);
#pragma unroll
        for (int d = 0; d < kDims; ++d) {
            const unsigned long long k = fkey(raw[d]);
            mn[d] = k < mn[d] ? k : mn[d];
            mx[d] = k > mx[d] ? k : mx[d];
        }
    }
#pragma unroll
    for (int d = 0; d < kDims; ++d) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn[d], o);
            const unsigned long long b = __shfl_xor_sync(0xffffffffu, mx[d], o);
            mn[d] = a < mn[d] ? a : mn[d];
            mx[d] = b > mx[d] ? b : mx[d];
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(keys + d, mn[d]);
            atomicMax(keys + kDims + d, mx[d]);
        }
    }
}

// The normalised training points in training order (:380-393).
__global__ void fit_points(const carma_feature_row* __restrict__ rows, const uint64_t* __restrict__ order,
                           uint64_t train_n, Bounds b, double* __restrict__ points) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < train_n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double raw[kDims];
        featurize(rows[order[i]], raw);
#pragma unroll
        for (int d = 0; d < kDims; ++d) points[i * kDims + d] = normalize(raw[d], b.lo[d], b.hi[d]);
    }
}

__global__ void gather_rows(const carma_feature_row* __restrict__ rows, const uint64_t* __restrict__ idx, uint64_t n,
                            carma_feature_row* __restrict__ out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = rows[idx[i]];
}

constexpr int kMaxLabel = 256;
// Holdout counts (:396-419): per label tp / fp / fn, correct, underestimates.
__global__ void holdout_counts(const int32_t* __restrict__ pred, const uint64_t* __restrict__ pred_bytes,
                               const int32_t* __restrict__ bucket, const uint64_t* __restrict__ mem,
                               const uint64_t* __restrict__ idx, uint64_t n, unsigned long long* __restrict__ cnt) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int p = pred[i], g = bucket[idx[i]];
        if (p == g) {
            atomicAdd(cnt + 3 * kMaxLabel, 1ull);
            atomicAdd(cnt + 3 * p, 1ull);
        } else {
            atomicAdd(cnt + 3 * p + 1, 1ull);
            atomicAdd(cnt + 3 * g + 2, 1ull);
        }
        if (pred_bytes[i] < mem[idx[i]]) atomicAdd(cnt + 3 * kMaxLabel + 1, 1ull);
    }
}

struct HostModel {
    DeviceBuffer pts, ptsf, key18, orig, label_by_orig;
    bool f32_ok = false;
    double pmax[kF32Dims] = {0};
    uint8_t adim[kF32Dims] = {0};
    uint64_t n = 0;
    uint64_t bucket_range = 0;
    uint32_t k = 0;
    double lo[kDims], hi[kDims];
    uint32_t active = 0;
    bool present = false;
};

}  // namespace

struct KnnHandle {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t pipe[2] = {nullptr, nullptr};
    HostModel model[CARMA_FAMILIES];
    struct Scratch {
        DeviceBuffer rows, family, qbin, qpos, perm, hist, tot, bucket, bytes, qrec, brute_d2, brute_id, sbucket, sbytes;
        PinnedBuffer stage_rows, stage_family, stage_packed;
        cudaEvent_t staged = nullptr;  // the H2D copy out of stage_packed is done
    } scratch[2];
    DeviceBuffer evals;
    StreamFence fence;        // last device-stream user of scratch[0] + evals
    DeviceBuffer train_rows;  // carma_knn_train: the uploaded dataset
    double act[16] = {0};
    carma_bit_schema schema{};
    int path = 0;  // 0 auto (fp32 pre-filter when every model allows it), 1 exact fp64 blocks, 2 fp32 pre-filter
    uint64_t last_visits = 0;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // pipeline start, (unused), (unused), pipeline end
    static constexpr int kTimedChunks = 8;
    cudaEvent_t sev[kTimedChunks][2] = {};  // search start / end per chunk of the last device call
    int timed_chunks = 0;
    bool timed = false;
    uint64_t last_launches = 0, last_evals = 0;
    uint64_t last_h2d = 0;  // bytes copied host -> device by the last host-buffer call
    std::mutex mu;
};

namespace {

KnnParams make_params(const KnnHandle& h, uint32_t* n_bins) {
    KnnParams p{};
    std::memcpy(p.act, h.act, sizeof(p.act));
    for (int f = 0; f < CARMA_BIT_FIELDS; ++f) {
        p.bbase[f] = h.schema.base[f];
        p.boff[f] = h.schema.offset[f];
        p.bw[f] = h.schema.width[f];
    }
    p.bwpr = h.schema.words_per_row;
    uint32_t base = 0;
    for (int f = 0; f < CARMA_FAMILIES; ++f) {
        const HostModel& hm = h.model[f];
        ModelDev& m = p.m[f];
        m.present = hm.present ? 1 : 0;
        if (!hm.present) continue;
        m.pts = hm.pts.as<double>() + kBlock * kStride;
        m.key18 = hm.key18.as<double>();
        m.orig = hm.orig.as<int32_t>();
        m.label_by_orig = hm.label_by_orig.as<int32_t>();
        m.n = hm.n;
        m.bucket_range = hm.bucket_range;
        m.k = hm.k;
        m.active = hm.active;
        m.f32_ok = hm.f32_ok ? 1 : 0;
        m.ptsf = hm.f32_ok ? hm.ptsf.as<float>() + kBlock * kF32Dims : nullptr;
        std::memcpy(m.pmax, hm.pmax, sizeof(m.pmax));
        std::memcpy(m.adim, hm.adim, sizeof(m.adim));
        std::memcpy(m.lo, hm.lo, sizeof(m.lo));
        std::memcpy(m.hi, hm.hi, sizeof(m.hi));
        uint32_t shift = 0;
        while (((hm.n + (1ull << shift) - 1) >> shift) > (kMaxBins / CARMA_FAMILIES) - 1) ++shift;
        m.bin_shift = shift;
        m.bin_base = base;
        base += static_cast<uint32_t>((hm.n >> shift) + 1);
    }
    *n_bins = base + 1;  // + invalid-family bin
    return p;
}

int max_k(const KnnHandle& h) {
    uint32_t k = 1;
    for (const auto& m : h.model)
        if (m.present) k = std::max(k, m.k);
    return static_cast<int>(k);
}

void launch_search(const KnnParams& p, int kmax, bool f32, const uint32_t* perm, const uint32_t* qpos,
                   int32_t* bucket, uint64_t* bytes, double* d2, int64_t* idx, unsigned long long* evals,
                   cudaStream_t s) {
    const uint64_t warps = (p.q + 31) / 32;
    const unsigned block = 128;
    // ~16 CTAs per SM over the run (4 resident): small contiguous chunks keep
    // the tail short while each CTA stays in one region of the model.
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, 148u * 16u)));
    if (f32) {
        auto go = [&](auto kc) {
            constexpr int KK = decltype(kc)::value;
            if (kF32Smem > 48 * 1024) {
                static const cudaError_t attr = [] {
                    cudaError_t e = cudaSuccess;
                    const int b = static_cast<int>(kF32Smem);
                    for (auto fn : {knn_search_f32<KK, CARMA_ROWS_SCALAR>, knn_search_f32<KK, CARMA_ROWS_PACKED>,
                                    knn_search_f32<KK, CARMA_ROWS_BITPACKED>, knn_search_f32<KK, CARMA_ROWS_FEATURES>})
                        if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
                    return e;
                }();
                CARMA_CUDA(attr);
            }
            switch (p.format) {
                case CARMA_ROWS_SCALAR:
                    knn_search_f32<KK, CARMA_ROWS_SCALAR><<<grid, block, kF32Smem, s>>>(p, perm, qpos, bucket, bytes, d2, idx, evals);
                    break;
                case CARMA_ROWS_PACKED:
                    knn_search_f32<KK, CARMA_ROWS_PACKED><<<grid, block, kF32Smem, s>>>(p, perm, qpos, bucket, bytes, d2, idx, evals);
                    break;
                case CARMA_ROWS_BITPACKED:
                    knn_search_f32<KK, CARMA_ROWS_BITPACKED><<<grid, block, kF32Smem, s>>>(p, perm, qpos, bucket, bytes, d2, idx,
                                                                                     evals);
                    break;
                default:
                    knn_search_f32<KK, CARMA_ROWS_FEATURES><<<grid, block, kF32Smem, s>>>(p, perm, qpos, bucket, bytes, d2, idx,
                                                                                   evals);
            }
        };
        if (kmax <= 5) go(std::integral_constant<int, 5>{});
        else if (kmax <= 8) go(std::integral_constant<int, 8>{});
        else go(std::integral_constant<int, kMaxK>{});
    } else {
        if (kmax <= 5)
            knn_search<5><<<grid, block, 0, s>>>(p, perm, qpos, bucket, bytes, d2, idx, evals);
        else if (kmax <= 8)
            knn_search<8><<<grid, block, 0, s>>>(p, perm, qpos, bucket, bytes, d2, idx, evals);
        else
            knn_search<kMaxK><<<grid, block, 0, s>>>(p, perm, qpos, bucket, bytes, d2, idx, evals);
    }
}

bool use_f32(const KnnHandle& h) {
    if (h.path == 1) return false;
    bool ok = true;
    for (const auto& m : h.model)
        if (m.present) ok = ok && m.f32_ok;
    if (h.path == 2 && !ok) throw Unsupported("fp32 pre-filter requested but a model has > 16 active dims");
    return ok;
}

// Runs the 4-kernel pipeline on device-resident rows.
uint64_t run_pipeline(KnnHandle& h, KnnHandle::Scratch& sc, const void* rows, int32_t format,
                      const int8_t* family, int32_t default_family, uint64_t q,
                      int32_t* bucket, uint64_t* bytes, double* d2, int64_t* idx,
                      unsigned long long* evals, cudaStream_t s, int chunk = 0,
                      bool outer = true, const carma_bit_schema* bits = nullptr) {
    uint32_t n_bins = 0;
    KnnParams p = make_params(h, &n_bins);
    if (bits) {  // this call's bit-packed schema instead of the handle's
        for (int f = 0; f < CARMA_BIT_FIELDS; ++f) {
            p.bbase[f] = bits->base[f];
            p.boff[f] = bits->offset[f];
            p.bw[f] = bits->width[f];
        }
        p.bwpr = bits->words_per_row;
    }
    p.rows = rows;
    p.format = format;
    p.family = family;
    p.default_family = default_family;
    p.q = q;
    const unsigned ctas = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(kScatterCtas, (q + 4095) / 4096)));
    sc.qbin.ensure(q * 4);
    sc.qpos.ensure(q * 4);
    sc.perm.ensure(q * 4);
    sc.hist.ensure(static_cast<size_t>(n_bins) * ctas * 4);
    const size_t shmem = n_bins * 4;
    const bool timed = h.timed && h.ev[0] && chunk < KnnHandle::kTimedChunks;
    if (timed) h.timed_chunks = std::max(h.timed_chunks, chunk + 1);
    cudaEvent_t* se = timed ? h.sev[chunk] : nullptr;
    if (max_k(h) > kMaxK) {  // exact brute force, query chunks bounded by the scratch
        if (timed && outer) CARMA_CUDA(cudaEventRecord(h.ev[0], s));
        if (timed) CARMA_CUDA(cudaEventRecord(se[0], s));
        const uint64_t kc = static_cast<uint64_t>(max_k(h));
        const uint64_t chunk = std::max<uint64_t>(1024, (256ull << 20) / (kc * 12));
        uint64_t launches = 0;
        for (uint64_t q0 = 0; q0 < q; q0 += chunk) {
            const uint64_t nq = std::min(chunk, q - q0);
            sc.brute_d2.ensure(nq * kc * 8);
            sc.brute_id.ensure(nq * kc * 4);
            const unsigned grid = static_cast<unsigned>((nq + 127) / 128);
            double* bd = sc.brute_d2.as<double>();
            int32_t* bi = sc.brute_id.as<int32_t>();
            switch (format) {
                case CARMA_ROWS_SCALAR:
                    knn_brute<CARMA_ROWS_SCALAR><<<grid, 128, 0, s>>>(p, q0, nq, bd, bi, bucket, bytes, d2, idx);
                    break;
                case CARMA_ROWS_PACKED:
                    knn_brute<CARMA_ROWS_PACKED><<<grid, 128, 0, s>>>(p, q0, nq, bd, bi, bucket, bytes, d2, idx);
                    break;
                case CARMA_ROWS_BITPACKED:
                    knn_brute<CARMA_ROWS_BITPACKED><<<grid, 128, 0, s>>>(p, q0, nq, bd, bi, bucket, bytes, d2, idx);
                    break;
                default:
                    knn_brute<CARMA_ROWS_FEATURES><<<grid, 128, 0, s>>>(p, q0, nq, bd, bi, bucket, bytes, d2, idx);
            }
            CARMA_CUDA(cudaGetLastError());
            ++launches;
        }
        if (timed) CARMA_CUDA(cudaEventRecord(se[1], s));
        if (timed && outer) CARMA_CUDA(cudaEventRecord(h.ev[3], s));
        return launches;
    }
    const bool f32 = use_f32(h);
    // Layout of the fp32 path (KNN_LAYOUT; CARMA_KNN_LAYOUT overrides for
    // A/B runs): 0 query records by row, written by knn_prep; 1 records by
    // bucketed slot (knn_keys, bucketing, knn_prep_sorted), so each warp
    // reads one contiguous span; 2 = 1 + bucket / bytes written by slot and
    // un-permuted by knn_unpermute (the search's scattered 4-B / 8-B stores
    // move to a streaming kernel). Measured on c2 (136-B rows): the search
    // 11.87 / 11.73 / 11.67 ms, its DRAM 7.1 / ~5 / 3.3 GB, the whole
    // pipeline 14.02 / 14.33 / 14.83 ms (knn_prep_sorted reads its rows at
    // random), so 0 is the default. Writing the records at random slots from
    // an in-order pass instead (fused into the scatter) took 4.7 ms.
    static const int layout = [] {
        const char* e = std::getenv("CARMA_KNN_LAYOUT");
        return e ? std::atoi(e) : KNN_LAYOUT;
    }();
    const bool sorted = f32 && layout >= 1;
    const bool sorted_out = sorted && layout == 2 && (bucket || bytes);
    if (timed && outer) CARMA_CUDA(cudaEventRecord(h.ev[0], s));
    if (f32 && !sorted) {
        uint64_t nkeys = 0;
        for (const auto& m : h.model)
            if (m.present) nkeys += m.n;
        const int keys_in_smem = nkeys <= kPrepKeysMax ? 1 : 0;
        const size_t pshmem = ((n_bins + 3) & ~3u) * 4 + (keys_in_smem ? nkeys * 8 : 0);
        if (pshmem > 48 * 1024) {
            static const cudaError_t attr_ok = [] {
                cudaError_t e = cudaSuccess;
                const int lim = 100 * 1024;
                e = cudaFuncSetAttribute(knn_prep<CARMA_ROWS_SCALAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
                if (e == cudaSuccess)
                    e = cudaFuncSetAttribute(knn_prep<CARMA_ROWS_PACKED>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
                if (e == cudaSuccess)
                    e = cudaFuncSetAttribute(knn_prep<CARMA_ROWS_BITPACKED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             lim);
                if (e == cudaSuccess)
                    e = cudaFuncSetAttribute(knn_prep<CARMA_ROWS_FEATURES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             lim);
                return e;
            }();
            CARMA_CUDA(attr_ok);
        }
        sc.qrec.ensure(q * kQrec * sizeof(double));
        p.qrec = sc.qrec.as<double>();
        uint32_t* qb = sc.qbin.as<uint32_t>();
        uint32_t* qp = sc.qpos.as<uint32_t>();
        uint32_t* hs = sc.hist.as<uint32_t>();
        switch (format) {
            case CARMA_ROWS_SCALAR: knn_prep<CARMA_ROWS_SCALAR><<<ctas, 512, pshmem, s>>>(p, n_bins, qb, qp, hs, keys_in_smem); break;
            case CARMA_ROWS_PACKED: knn_prep<CARMA_ROWS_PACKED><<<ctas, 512, pshmem, s>>>(p, n_bins, qb, qp, hs, keys_in_smem); break;
            case CARMA_ROWS_BITPACKED:
                knn_prep<CARMA_ROWS_BITPACKED><<<ctas, 512, pshmem, s>>>(p, n_bins, qb, qp, hs, keys_in_smem);
                break;
            default: knn_prep<CARMA_ROWS_FEATURES><<<ctas, 512, pshmem, s>>>(p, n_bins, qb, qp, hs, keys_in_smem);
        }
    } else {
        knn_keys<<<ctas, 512, shmem, s>>>(p, n_bins, sc.qbin.as<uint32_t>(), sc.qpos.as<uint32_t>(),
                                          sc.hist.as<uint32_t>());
    }
    uint64_t extra = 0;
    sc.tot.ensure(n_bins * 4);
    bin_totals<<<(n_bins + 7) / 8, 256, 0, s>>>(sc.hist.as<uint32_t>(), n_bins, ctas, sc.tot.as<uint32_t>());
    scan_bins<<<1, 1024, 0, s>>>(sc.tot.as<uint32_t>(), n_bins);
    bin_offsets<<<(n_bins + 7) / 8, 256, 0, s>>>(sc.hist.as<uint32_t>(), n_bins, ctas, sc.tot.as<uint32_t>());
    int32_t* sb = bucket;
    uint64_t* sby = bytes;
    knn_scatter<<<ctas, 512, shmem, s>>>(q, n_bins, sc.qbin.as<uint32_t>(), sc.hist.as<uint32_t>(),
                                         sc.perm.as<uint32_t>());
    if (sorted) {
        sc.qrec.ensure(q * kQrec * sizeof(double));
        p.qrec = sc.qrec.as<double>();
        p.qrec_by_slot = 1;
        const unsigned g = static_cast<unsigned>((q + 255) / 256);
        const uint32_t* pm = sc.perm.as<uint32_t>();
        const uint32_t* qp = sc.qpos.as<uint32_t>();
        switch (format) {
            case CARMA_ROWS_SCALAR: knn_prep_sorted<CARMA_ROWS_SCALAR><<<g, 256, 0, s>>>(p, pm, qp); break;
            case CARMA_ROWS_PACKED: knn_prep_sorted<CARMA_ROWS_PACKED><<<g, 256, 0, s>>>(p, pm, qp); break;
            case CARMA_ROWS_BITPACKED: knn_prep_sorted<CARMA_ROWS_BITPACKED><<<g, 256, 0, s>>>(p, pm, qp); break;
            default: knn_prep_sorted<CARMA_ROWS_FEATURES><<<g, 256, 0, s>>>(p, pm, qp);
        }
        ++extra;
        if (sorted_out) {
            p.out_by_slot = 1;
            sc.sbucket.ensure(q * 4);
            sc.sbytes.ensure(q * 8);
            sb = sc.sbucket.as<int32_t>();
            sby = sc.sbytes.as<uint64_t>();
        }
    }
    if (timed) CARMA_CUDA(cudaEventRecord(se[0], s));
    launch_search(p, max_k(h), f32, sc.perm.as<uint32_t>(), sc.qpos.as<uint32_t>(), sb, sby, d2,
                  idx, evals, s);
    if (timed) CARMA_CUDA(cudaEventRecord(se[1], s));
    if (sorted_out) {
        knn_unpermute<<<static_cast<unsigned>((q + 255) / 256), 256, 0, s>>>(q, sc.perm.as<uint32_t>(), sb, sby,
                                                                          bucket, bytes);
        ++extra;
    }
    if (timed && outer) CARMA_CUDA(cudaEventRecord(h.ev[3], s));
    CARMA_CUDA(cudaGetLastError());
    return 6 + extra;
}

void check_ready(const KnnHandle* h) {
    if (!h) throw InvalidArg("null handle");
    bool any = false;
    for (const auto& m : h->model) any |= m.present;
    if (!any) throw CarmaFailure(CARMA_ERR_FAMILY, "no model installed");
}

carma_status predict_host(carma_knn* hh, const void* rows, size_t row_bytes, int32_t format,
                          const int8_t* family, int32_t default_family, uint64_t q,
                          int32_t* bucket_out, uint64_t* bytes_out, size_t tail_bytes = 0,
                          const double* act_table = nullptr) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        check_ready(h);
        if (q == 0) return;
        if (!rows) throw InvalidArg("rows is null");
        std::lock_guard<std::mutex> lock(h->mu);
        if (act_table) std::memcpy(h->act, act_table, sizeof(h->act));  // under the lock
        DeviceGuard g(h->device);
        // Chunks grow geometrically from 2^18 rows to the steady size and
        // shrink again over the last rows (at most half of what remains), so
        // the first H2D copy (pipeline fill) and the last search + D2H
        // (drain) are short; scratch is sized for the steady chunk.
        const uint64_t chunk = uint64_t{1} << KNN_E2E_CHUNK_LOG2;
        const uint64_t small = uint64_t{1} << KNN_E2E_SMALL_LOG2;
        auto chunk_rows = [&](uint64_t c, uint64_t remaining) -> uint64_t {
            const uint64_t grow = std::min<uint64_t>(chunk, small << std::min<uint64_t>(c, 20));
            return std::min<uint64_t>(grow, std::max<uint64_t>(small, remaining / 2));
        };
        const bool rows_pinned = is_pinned(rows);
        const bool fam_pinned = !family || is_pinned(family);
        const bool out_pinned = (!bucket_out || is_pinned(bucket_out)) && (!bytes_out || is_pinned(bytes_out));
        h->timed = false;
        h->fence.host_wait();  // a device call may still use scratch[0] / evals
        h->evals.ensure(16);
        CARMA_CUDA(cudaMemsetAsync(h->evals.ptr, 0, 16, h->pipe[0]));
        CARMA_CUDA(cudaStreamSynchronize(h->pipe[0]));
        auto copy_out = [&](KnnHandle::Scratch& sc, cudaStream_t s, uint64_t beg, uint64_t cnt) {
            if (out_pinned) {
                if (bucket_out)
                    CARMA_CUDA(cudaMemcpyAsync(bucket_out + beg, sc.bucket.ptr, cnt * 4, cudaMemcpyDeviceToHost, s));
                if (bytes_out)
                    CARMA_CUDA(cudaMemcpyAsync(bytes_out + beg, sc.bytes.ptr, cnt * 8, cudaMemcpyDeviceToHost, s));
            } else {
                CARMA_CUDA(cudaStreamSynchronize(s));
                if (bucket_out)
                    CARMA_CUDA(cudaMemcpy(bucket_out + beg, sc.bucket.ptr, cnt * 4, cudaMemcpyDeviceToHost));
                if (bytes_out)
                    CARMA_CUDA(cudaMemcpy(bytes_out + beg, sc.bytes.ptr, cnt * 8, cudaMemcpyDeviceToHost));
            }
        };
        uint64_t launches = 0, h2d = 0;
        uint64_t beg = 0, cnt = 0;
        // Feature rows travel re-encoded as 64-byte packed rows (family inside;
        // stage.hpp), packed by the host pool while the previous chunk copies
        // and searches. CARMA_E2E_RAW=1 sends the 136-byte rows as they are.
        static const bool raw_env = std::getenv("CARMA_E2E_RAW") && std::atoi(std::getenv("CARMA_E2E_RAW")) != 0;
        const bool pack = format == CARMA_ROWS_FEATURES && !raw_env;
        if (pack) std::memcpy(h->act, canonical_act_table(), sizeof(h->act));
        for (uint64_t c = 0; beg < q; ++c, beg += cnt) {
            KnnHandle::Scratch& sc = h->scratch[c & 1];
            cudaStream_t s = h->pipe[c & 1];
            cnt = std::min<uint64_t>(chunk_rows(c, q - beg), q - beg);
            const uint64_t cap_rows = std::min<uint64_t>(chunk, q);
            if (pack && !raw_chunk(c, rows_pinned && fam_pinned)) {
                sc.stage_packed.ensure(cap_rows * sizeof(carma_feature_packed));
                sc.rows.ensure(cap_rows * row_bytes);
                sc.bucket.ensure(cap_rows * 4);
                sc.bytes.ensure(cap_rows * 8);
                if (!sc.staged) CARMA_CUDA(cudaEventCreateWithFlags(&sc.staged, cudaEventDisableTiming));
                CARMA_CUDA(cudaEventSynchronize(sc.staged));  // the previous copy out of this stage buffer
                auto* pk = sc.stage_packed.as<carma_feature_packed>();
                // 40-byte compact rows first (bit-packed, fixed schema), then
                // the 64-byte packed format, else the raw rows
                if (compact_rows() &&
                    pack_rows_compact(static_cast<const carma_feature_row*>(rows) + beg, family ? family + beg : nullptr,
                                      default_family, cnt, reinterpret_cast<uint64_t*>(pk))) {
                    const uint64_t nb = cnt * 4ull * kCompactWords;
                    CARMA_CUDA(cudaMemcpyAsync(sc.rows.ptr, pk, nb, cudaMemcpyHostToDevice, s));
                    h2d += nb;
                    CARMA_CUDA(cudaEventRecord(sc.staged, s));
                    launches += run_pipeline(*h, sc, sc.rows.ptr, CARMA_ROWS_BITPACKED, nullptr, default_family, cnt,
                                             sc.bucket.as<int32_t>(), sc.bytes.as<uint64_t>(), nullptr, nullptr,
                                             h->evals.as<unsigned long long>(), s, 0, true, &compact_schema());
                    copy_out(sc, s, beg, cnt);
                    continue;
                }
                if (pack_rows_canonical(static_cast<const carma_feature_row*>(rows) + beg, family ? family + beg : nullptr,
                                        default_family, cnt, pk)) {
                    CARMA_CUDA(cudaMemcpyAsync(sc.rows.ptr, pk, cnt * sizeof(carma_feature_packed),
                                               cudaMemcpyHostToDevice, s));
                    h2d += cnt * sizeof(carma_feature_packed);
                    CARMA_CUDA(cudaEventRecord(sc.staged, s));
                    launches += run_pipeline(*h, sc, sc.rows.ptr, CARMA_ROWS_PACKED, nullptr, default_family, cnt,
                                             sc.bucket.as<int32_t>(), sc.bytes.as<uint64_t>(), nullptr, nullptr,
                                             h->evals.as<unsigned long long>(), s);
                    copy_out(sc, s, beg, cnt);
                    continue;
                }
            }
            const char* src = static_cast<const char*>(rows) + beg * row_bytes;
            // buffers for the largest chunk this call uses (not the steady
            // size: pinned staging for 2^21 rows costs ~0.1 s to allocate)
            sc.rows.ensure(cap_rows * row_bytes + tail_bytes);
            sc.bucket.ensure(cap_rows * 4);
            sc.bytes.ensure(cap_rows * 8);
            if (family) sc.family.ensure(cap_rows);
            if (!rows_pinned || !fam_pinned) {
                // Stage through pinned memory; wait until this buffer's previous
                // chunk has been consumed.
                CARMA_CUDA(cudaStreamSynchronize(s));
                sc.stage_rows.ensure(cap_rows * row_bytes + tail_bytes);
                std::memcpy(sc.stage_rows.ptr, src, cnt * row_bytes + tail_bytes);
                src = sc.stage_rows.as<char>();
                if (family) {
                    sc.stage_family.ensure(cap_rows);
                    std::memcpy(sc.stage_family.ptr, family + beg, cnt);
                }
            }
            CARMA_CUDA(cudaMemcpyAsync(sc.rows.ptr, src, cnt * row_bytes + tail_bytes, cudaMemcpyHostToDevice, s));
            h2d += cnt * row_bytes + tail_bytes + (family ? cnt : 0);
            if (family)
                CARMA_CUDA(cudaMemcpyAsync(sc.family.ptr,
                                           (!rows_pinned || !fam_pinned) ? sc.stage_family.as<int8_t>() : family + beg,
                                           cnt, cudaMemcpyHostToDevice, s));
            launches += run_pipeline(*h, sc, sc.rows.ptr, format, family ? sc.family.as<int8_t>() : nullptr,
                                     default_family, cnt, sc.bucket.as<int32_t>(), sc.bytes.as<uint64_t>(),
                                     nullptr, nullptr, h->evals.as<unsigned long long>(), s);
            copy_out(sc, s, beg, cnt);
        }
        CARMA_CUDA(cudaStreamSynchronize(h->pipe[0]));
        CARMA_CUDA(cudaStreamSynchronize(h->pipe[1]));
        unsigned long long ev[2] = {0, 0};
        CARMA_CUDA(cudaMemcpy(ev, h->evals.ptr, 16, cudaMemcpyDeviceToHost));
        h->last_launches = launches;
        h->last_h2d = h2d;
        h->last_evals = ev[0];
        h->last_visits = ev[1];
    });
}

}  // namespace
}  // namespace carma_b200

using namespace carma_b200;

extern "C" {

carma_status carma_knn_create(int device, carma_knn** out) {
    return guarded([&] {
        if (!out) throw InvalidArg("out is null");
        require_device(device);
        DeviceGuard g(device);
        auto* h = new KnnHandle();
        h->device = device;
        CARMA_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        CARMA_CUDA(cudaStreamCreateWithFlags(&h->pipe[0], cudaStreamNonBlocking));
        CARMA_CUDA(cudaStreamCreateWithFlags(&h->pipe[1], cudaStreamNonBlocking));
        for (auto& e : h->ev) CARMA_CUDA(cudaEventCreate(&e));
        for (auto& pr : h->sev)
            for (auto& e : pr) CARMA_CUDA(cudaEventCreate(&e));
        *out = reinterpret_cast<carma_knn*>(h);
    });
}

carma_status carma_knn_destroy(carma_knn* hh) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h) return;
        {
            DeviceGuard g(h->device);
            cudaDeviceSynchronize();  // device calls may have queued work on caller streams
            for (auto& m : h->model) {
                m.pts.release();
                m.ptsf.release();
                m.key18.release();
                m.orig.release();
                m.label_by_orig.release();
            }
            for (auto& sc : h->scratch) {
                sc.rows.release(); sc.family.release(); sc.qbin.release(); sc.qpos.release();
                sc.perm.release(); sc.hist.release(); sc.tot.release(); sc.bucket.release(); sc.bytes.release();
                sc.brute_d2.release(); sc.brute_id.release(); sc.sbucket.release(); sc.sbytes.release();
                sc.stage_rows.release(); sc.stage_family.release(); sc.stage_packed.release();
                if (sc.staged) cudaEventDestroy(sc.staged);
            }
            h->evals.release();
            h->fence.destroy();
            for (auto& e : h->ev)
                if (e) cudaEventDestroy(e);
            for (auto& pr : h->sev)
                for (auto& e : pr)
                    if (e) cudaEventDestroy(e);
            cudaStreamDestroy(h->stream);
            cudaStreamDestroy(h->pipe[0]);
            cudaStreamDestroy(h->pipe[1]);
        }
        delete h;
    });
}

carma_status carma_knn_set_model(carma_knn* hh, int32_t family, const double* lo, const double* hi,
                                 const double* points, const int32_t* labels, uint64_t n,
                                 uint32_t k, uint64_t bucket_range) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h) throw InvalidArg("null handle");
        if (family < 0 || family >= CARMA_FAMILIES) throw InvalidArg("unknown family");
        if (n == 0) throw InvalidArg("EmptyDataset: model has no points");
        if (n > 0x7fffffffull) throw InvalidArg("model too large");
        if (k < 1) throw InvalidArg("k must be >= 1");
        if (k > 65536) throw Unsupported("k > 65536 is not supported by the GPU kernel");
        if (bucket_range == 0) throw InvalidArg("NonPositiveRange: bucket range must be > 0");
        if (!lo || !hi || !points || !labels) throw InvalidArg("null model array");
        std::lock_guard<std::mutex> lock(h->mu);
        DeviceGuard g(h->device);
        // Sort by (p18, original index): the search order (see file header).
        std::vector<int32_t> order(n);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
            return points[static_cast<uint64_t>(a) * kDims + 18] < points[static_cast<uint64_t>(b) * kDims + 18];
        });
        // kBlock padding points on both sides (never inserted; see knn_search)
        std::vector<double> pts((n + 2 * kBlock) * kStride, 0.0), key(n);
        for (uint64_t i = 0; i < n; ++i) {
            const double* src = points + static_cast<uint64_t>(order[i]) * kDims;
            std::memcpy(&pts[(i + kBlock) * kStride], src, sizeof(double) * kDims);
            key[i] = src[18];
        }
        HostModel& m = h->model[family];
        // fp32 pre-filter copy: fl32(w * p) of the active dims (w = 64 for dim 18)
        {
            int ad = 0;
            uint32_t act = 0;
            bool small = true;
            for (int d = 0; d < kDims; ++d) {
                bool zero = !(hi[d] > lo[d]);
                for (uint64_t i = 0; zero && i < n; ++i) zero = points[i * kDims + d] == 0.0;
                if (!zero) act |= 1u << d;
            }
            for (int j = 0; j < kF32Dims; ++j) {
                m.adim[j] = 0xff;
                m.pmax[j] = 0.0;
            }
            for (int d = 0; d < kDims; ++d)
                if (act & (1u << d)) {
                    if (ad < kF32Dims) {
                        m.adim[ad] = static_cast<uint8_t>(d);
                        double pm = 0.0;
                        for (uint64_t i = 0; i < n; ++i) pm = std::max(pm, std::fabs(points[i * kDims + d]));
                        small = small && pm <= 1e15 && pm == pm;
                        m.pmax[ad] = pm;
                    }
                    ++ad;
                }
            m.f32_ok = ad <= kF32Dims && small;
            if (m.f32_ok) {
                std::vector<float> pf((n + 2 * kBlock) * kF32Dims, 0.0f);
                for (uint64_t i = 0; i < n; ++i) {
                    const double* src = points + static_cast<uint64_t>(order[i]) * kDims;
                    for (int j = 0; j < ad; ++j) {
                        const int d = m.adim[j];
                        pf[(i + kBlock) * kF32Dims + j] = static_cast<float>(d == 18 ? 64.0 * src[d] : src[d]);
                    }
                }
                m.ptsf.ensure(pf.size() * 4);
                CARMA_CUDA(cudaMemcpy(m.ptsf.ptr, pf.data(), pf.size() * 4, cudaMemcpyHostToDevice));
            }
        }
        m.pts.ensure((n + 2 * kBlock) * kStride * 8);
        m.key18.ensure(n * 8);
        m.orig.ensure(n * 4);
        m.label_by_orig.ensure(n * 4);
        CARMA_CUDA(cudaMemcpy(m.pts.ptr, pts.data(), (n + 2 * kBlock) * kStride * 8, cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(m.key18.ptr, key.data(), n * 8, cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(m.orig.ptr, order.data(), n * 4, cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(m.label_by_orig.ptr, labels, n * 4, cudaMemcpyHostToDevice));
        m.n = n;
        m.k = k;
        m.bucket_range = bucket_range;
        // A dim contributes exactly +0.0 to every d2 when the query side is
        // always 0 (hi <= lo, or NaN bounds: normalise yields 0) and every
        // stored point is +-0 there: diff = +-0, diff^2 = +0, d2 + 0 = d2.
        m.active = 0;
        for (int d = 0; d < kDims; ++d) {
            bool zero = !(hi[d] > lo[d]);
            for (uint64_t i = 0; zero && i < n; ++i) zero = points[i * kDims + d] == 0.0;
            if (!zero) m.active |= 1u << d;
        }
        std::memcpy(m.lo, lo, sizeof(m.lo));
        std::memcpy(m.hi, hi, sizeof(m.hi));
        m.present = true;
    });
}

carma_status carma_knn_predict(carma_knn* h, const carma_feature_row* rows, const int8_t* family,
                               int32_t default_family, uint64_t q, int32_t* bucket_out,
                               uint64_t* bytes_out) {
    return predict_host(h, rows, sizeof(carma_feature_row), CARMA_ROWS_FEATURES, family, default_family,
                        q, bucket_out, bytes_out);
}

carma_status carma_knn_set_act_table(carma_knn* hh, const double* act_table) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h || !act_table) throw InvalidArg("null argument");
        std::lock_guard<std::mutex> lock(h->mu);
        std::memcpy(h->act, act_table, sizeof(h->act));
    });
}

carma_status carma_knn_predict_packed(carma_knn* hh, const carma_feature_packed* rows, const double* act_table,
                                      uint64_t q, int32_t* bucket_out, uint64_t* bytes_out) {
    return predict_host(hh, rows, sizeof(carma_feature_packed), CARMA_ROWS_PACKED, nullptr, 0, q, bucket_out,
                        bytes_out, 0, act_table);
}

carma_status carma_knn_set_bit_schema(carma_knn* hh, const carma_bit_schema* schema) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h || !schema) throw InvalidArg("null argument");
        if (schema->words_per_row == 0) throw InvalidArg("schema has no words per row");
        for (int f = 0; f < CARMA_BIT_FIELDS; ++f)
            if (schema->width[f] > 48) throw InvalidArg("schema field wider than 48 bits");
        std::lock_guard<std::mutex> lock(h->mu);
        h->schema = *schema;
        std::memcpy(h->act, schema->act_table, sizeof(h->act));
    });
}

carma_status carma_knn_predict_bitpacked(carma_knn* hh, const uint32_t* words, const carma_bit_schema* schema,
                                         uint64_t q, int32_t* bucket_out, uint64_t* bytes_out) {
    const carma_status st = carma_knn_set_bit_schema(hh, schema);
    if (st != CARMA_OK) return st;
    return predict_host(hh, words, 4ull * schema->words_per_row, CARMA_ROWS_BITPACKED, nullptr, 0, q, bucket_out,
                        bytes_out, 8);
}

carma_status carma_knn_predict_scalar(carma_knn* h, const double* raw, const int8_t* family,
                                      int32_t default_family, uint64_t q, int32_t* bucket_out,
                                      uint64_t* bytes_out) {
    return predict_host(h, raw, sizeof(double) * kDims, CARMA_ROWS_SCALAR, family, default_family, q,
                        bucket_out, bytes_out);
}

carma_status carma_knn_predict_device(carma_knn* hh, const void* rows, int32_t format,
                                      const int8_t* family, int32_t default_family, uint64_t q,
                                      int32_t* bucket_out, uint64_t* bytes_out, double* topk_d2,
                                      int64_t* topk_idx, void* stream) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        check_ready(h);
        if (format < CARMA_ROWS_FEATURES || format > CARMA_ROWS_BITPACKED) throw InvalidArg("unknown row format");
        if (q == 0) return;
        if (!rows) throw InvalidArg("rows is null");
        std::lock_guard<std::mutex> lock(h->mu);
        DeviceGuard g(h->device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->stream;
        h->evals.ensure(16);
        h->fence.acquire(s);  // scratch[0] / evals may be in use on another stream
        CARMA_CUDA(cudaMemsetAsync(h->evals.ptr, 0, 16, s));
        h->timed = true;
        h->timed_chunks = 0;
        // KNN_SPLIT chunks on the two pipeline streams: a chunk's bucketing
        // pre-pass overlaps the previous chunk's search (CARMA_KNN_SPLIT)
        static const int split = [] {
            const char* e = std::getenv("CARMA_KNN_SPLIT");
            return e ? std::atoi(e) : KNN_SPLIT;
        }();
        const size_t rb = format == CARMA_ROWS_FEATURES ? sizeof(carma_feature_row)
                          : format == CARMA_ROWS_PACKED ? sizeof(carma_feature_packed)
                          : format == CARMA_ROWS_SCALAR ? sizeof(double) * kDims
                                                        : 0;
        if (split > 1 && rb && q >= (uint64_t{1} << 22) && !topk_d2 && !topk_idx) {
            cudaEvent_t ev_in, ev_out[2];
            CARMA_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
            for (auto& e : ev_out) CARMA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CARMA_CUDA(cudaEventRecord(h->ev[0], s));
            CARMA_CUDA(cudaEventRecord(ev_in, s));
            for (auto ps : h->pipe) CARMA_CUDA(cudaStreamWaitEvent(ps, ev_in, 0));
            uint64_t launches = 0;
            for (int c = 0; c < split; ++c) {
                const uint64_t b = q * c / split, e = q * (c + 1) / split;
                launches += run_pipeline(*h, h->scratch[c & 1], static_cast<const char*>(rows) + b * rb, format,
                                         family ? family + b : nullptr, default_family, e - b,
                                         bucket_out ? bucket_out + b : nullptr, bytes_out ? bytes_out + b : nullptr,
                                         nullptr, nullptr, h->evals.as<unsigned long long>(), h->pipe[c & 1], c,
                                         false);
            }
            for (int k = 0; k < 2; ++k) {
                CARMA_CUDA(cudaEventRecord(ev_out[k], h->pipe[k]));
                CARMA_CUDA(cudaStreamWaitEvent(s, ev_out[k], 0));
            }
            CARMA_CUDA(cudaEventRecord(h->ev[3], s));
            cudaEventDestroy(ev_in);
            for (auto e : ev_out) cudaEventDestroy(e);
            h->last_launches = launches;
        } else {
            h->last_launches = run_pipeline(*h, h->scratch[0], rows, format, family, default_family, q,
                                            bucket_out, bytes_out, topk_d2, topk_idx,
                                            h->evals.as<unsigned long long>(), s);
        }
        h->fence.release(s);
    });
}

carma_status carma_knn_train(carma_knn* hh, int32_t family, const carma_feature_row* rows, const int32_t* bucket,
                             const uint64_t* mem, uint64_t n, uint64_t seed, uint32_t k, uint64_t bucket_range,
                             carma_holdout_report* report, double* lo_out, double* hi_out, double* points_out,
                             int32_t* labels_out) {
    // The model install reuses carma_knn_set_model (it takes the handle's lock).
    std::vector<double> lo(kDims), hi(kDims), points;
    std::vector<int32_t> labels;
    std::vector<uint64_t> order(n);
    uint64_t train_n = 0;
    carma_status st = guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h) throw InvalidArg("null handle");
        if (family < 0 || family >= CARMA_FAMILIES) throw InvalidArg("unknown family");
        if (n == 0) throw InvalidArg("EmptyDataset: dataset has no rows");
        if (k < 1) throw InvalidArg("ConfigError: k must be >= 1");
        if (!rows || !bucket || !mem) throw InvalidArg("null dataset array");
        const carma_status so = carma_host_split_order(n, seed, order.data(), &train_n);
        if (so != CARMA_OK) throw CarmaFailure(so, carma_last_error());
        require_device(h->device);
        DeviceGuard g(h->device);
        DeviceBuffer d_rows, d_order, d_keys, d_points;
        d_rows.ensure(n * sizeof(carma_feature_row));
        d_order.ensure(n * 8);
        d_keys.ensure(2 * kDims * 8);
        d_points.ensure(train_n * kDims * 8);
        CARMA_CUDA(cudaMemcpy(d_rows.ptr, rows, n * sizeof(carma_feature_row), cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(d_order.ptr, order.data(), n * 8, cudaMemcpyHostToDevice));
        std::vector<unsigned long long> keys(2 * kDims);
        for (int d = 0; d < kDims; ++d) {
            keys[d] = ~0ull;
            keys[kDims + d] = 0ull;
        }
        CARMA_CUDA(cudaMemcpy(d_keys.ptr, keys.data(), keys.size() * 8, cudaMemcpyHostToDevice));
        const unsigned grid = grid_for(train_n, 256, 148u * 8u);
        fit_bounds<<<grid, 256>>>(d_rows.as<carma_feature_row>(), d_order.as<uint64_t>(), train_n,
                                  d_keys.as<unsigned long long>());
        CARMA_CUDA(cudaGetLastError());
        CARMA_CUDA(cudaMemcpy(keys.data(), d_keys.ptr, keys.size() * 8, cudaMemcpyDeviceToHost));
        auto unkey = [](unsigned long long k2) {
            const unsigned long long u = (k2 >> 63) ? (k2 & 0x7fffffffffffffffull) : ~k2;
            double x;
            std::memcpy(&x, &u, 8);
            return x;
        };
        Bounds b;
        bool varying = false;
        for (int d = 0; d < kDims; ++d) {
            b.lo[d] = lo[d] = unkey(keys[d]);
            b.hi[d] = hi[d] = unkey(keys[kDims + d]);
            varying |= hi[d] > lo[d];
        }
        if (!varying) throw InvalidArg("DegenerateFeature: all features have zero variance");
        fit_points<<<grid, 256>>>(d_rows.as<carma_feature_row>(), d_order.as<uint64_t>(), train_n, b,
                                  d_points.as<double>());
        CARMA_CUDA(cudaGetLastError());
        points.resize(train_n * kDims);
        CARMA_CUDA(cudaMemcpy(points.data(), d_points.ptr, points.size() * 8, cudaMemcpyDeviceToHost));
        labels.resize(train_n);
        for (uint64_t i = 0; i < train_n; ++i) labels[i] = bucket[order[i]];
        // keep the uploaded rows for the holdout below
        h->train_rows.ensure(n * sizeof(carma_feature_row));
        CARMA_CUDA(cudaMemcpy(h->train_rows.ptr, d_rows.ptr, n * sizeof(carma_feature_row),
                              cudaMemcpyDeviceToDevice));
    });
    if (st != CARMA_OK) return st;
    st = carma_knn_set_model(hh, family, lo.data(), hi.data(), points.data(), labels.data(), train_n, k,
                             bucket_range);
    if (st != CARMA_OK) return st;
    if (lo_out) std::copy(lo.begin(), lo.end(), lo_out);
    if (hi_out) std::copy(hi.begin(), hi.end(), hi_out);
    if (points_out) std::copy(points.begin(), points.end(), points_out);
    if (labels_out) std::copy(labels.begin(), labels.end(), labels_out);
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        const uint64_t nh = n - train_n;
        carma_holdout_report rep{};
        rep.train_size = train_n;
        rep.holdout_size = nh;
        if (nh > 0) {
            std::lock_guard<std::mutex> lock(h->mu);
            DeviceGuard g(h->device);
            DeviceBuffer d_idx, d_hrows, d_pred, d_bytes, d_bucket, d_mem, d_cnt;
            d_idx.ensure(nh * 8);
            d_hrows.ensure(nh * sizeof(carma_feature_row));
            d_pred.ensure(nh * 4);
            d_bytes.ensure(nh * 8);
            d_bucket.ensure(n * 4);
            d_mem.ensure(n * 8);
            d_cnt.ensure((3 * kMaxLabel + 2) * 8);
            for (uint64_t i = 0; i < n; ++i)
                if (bucket[i] < 0 || bucket[i] >= kMaxLabel) throw Unsupported("bucket labels must be in [0, 256)");
            CARMA_CUDA(cudaMemcpy(d_idx.ptr, order.data() + train_n, nh * 8, cudaMemcpyHostToDevice));
            CARMA_CUDA(cudaMemcpy(d_bucket.ptr, bucket, n * 4, cudaMemcpyHostToDevice));
            CARMA_CUDA(cudaMemcpy(d_mem.ptr, mem, n * 8, cudaMemcpyHostToDevice));
            CARMA_CUDA(cudaMemset(d_cnt.ptr, 0, (3 * kMaxLabel + 2) * 8));
            const unsigned grid = grid_for(nh, 256, 148u * 8u);
            gather_rows<<<grid, 256, 0, h->stream>>>(h->train_rows.as<carma_feature_row>(), d_idx.as<uint64_t>(), nh,
                                                     d_hrows.as<carma_feature_row>());
            // estimate_learned on the holdout rows (every row is of `family`)
            h->timed = false;
            h->evals.ensure(16);
            CARMA_CUDA(cudaMemsetAsync(h->evals.ptr, 0, 16, h->stream));
            run_pipeline(*h, h->scratch[0], d_hrows.ptr, CARMA_ROWS_FEATURES, nullptr, family, nh,
                         d_pred.as<int32_t>(), d_bytes.as<uint64_t>(), nullptr, nullptr,
                         h->evals.as<unsigned long long>(), h->stream);
            holdout_counts<<<grid, 256, 0, h->stream>>>(d_pred.as<int32_t>(), d_bytes.as<uint64_t>(),
                                                        d_bucket.as<int32_t>(), d_mem.as<uint64_t>(),
                                                        d_idx.as<uint64_t>(), nh, d_cnt.as<unsigned long long>());
            CARMA_CUDA(cudaGetLastError());
            std::vector<unsigned long long> c(3 * kMaxLabel + 2);
            CARMA_CUDA(cudaStreamSynchronize(h->stream));
            CARMA_CUDA(cudaMemcpy(c.data(), d_cnt.ptr, c.size() * 8, cudaMemcpyDeviceToHost));
            const double hn = static_cast<double>(nh);
            rep.accuracy = static_cast<double>(c[3 * kMaxLabel]) / hn;
            rep.underestimate_rate = static_cast<double>(c[3 * kMaxLabel + 1]) / hn;
            // macro F1 over the labels of the confusion map in ascending order (:420-433)
            double f1_sum = 0.0;
            uint64_t classes = 0;
            for (int l = 0; l < kMaxLabel; ++l) {
                const double tp = static_cast<double>(c[3 * l]), fp = static_cast<double>(c[3 * l + 1]),
                             fn = static_cast<double>(c[3 * l + 2]);
                if (tp + fp + fn == 0) continue;  // not in the map
                if (tp + fn == 0) continue;       // class never appears in gold labels
                const double prec = tp + fp > 0 ? tp / (tp + fp) : 0.0;
                const double rec = tp / (tp + fn);
                f1_sum += prec + rec > 0 ? 2 * prec * rec / (prec + rec) : 0.0;
                ++classes;
            }
            rep.macro_f1 = classes ? f1_sum / static_cast<double>(classes) : 0.0;
        }
        if (report) *report = rep;
    });
}

carma_status carma_knn_last_timing(carma_knn* hh, double* search_ms, double* pipeline_ms) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h) throw InvalidArg("null handle");
        DeviceGuard g(h->device);
        CARMA_CUDA(cudaEventSynchronize(h->ev[3]));
        float a = 0.f, b = 0.f;
        for (int c = 0; c < h->timed_chunks; ++c) {  // the search kernels of every chunk
            float x = 0.f;
            CARMA_CUDA(cudaEventElapsedTime(&x, h->sev[c][0], h->sev[c][1]));
            a += x;
        }
        CARMA_CUDA(cudaEventElapsedTime(&b, h->ev[0], h->ev[3]));
        if (search_ms) *search_ms = a;
        if (pipeline_ms) *pipeline_ms = b;
    });
}

// Diagnostic: per chunk of the last timed device call, the search kernel's
// start and end in ms from the pipeline start (out[2c], out[2c+1]); *n gets
// the chunk count (at most cap / 2 written).
extern "C" carma_status carma_debug_knn_chunk_times(carma_knn* hh, float* out, int32_t cap, int32_t* n) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h || !out || !n) throw InvalidArg("null argument");
        DeviceGuard g(h->device);
        CARMA_CUDA(cudaEventSynchronize(h->ev[3]));
        *n = h->timed_chunks;
        for (int c = 0; c < h->timed_chunks && 2 * c + 1 < cap; ++c) {
            CARMA_CUDA(cudaEventElapsedTime(out + 2 * c, h->ev[0], h->sev[c][0]));
            CARMA_CUDA(cudaEventElapsedTime(out + 2 * c + 1, h->ev[0], h->sev[c][1]));
        }
    });
}

carma_status carma_knn_last_stats(carma_knn* hh, uint64_t* launches, uint64_t* evaluations) {
    uint64_t visits = 0;
    return carma_knn_last_work(hh, launches, evaluations, &visits);
}

carma_status carma_knn_last_work(carma_knn* hh, uint64_t* launches, uint64_t* fp64_evals, uint64_t* fp32_evals) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h) throw InvalidArg("null handle");
        DeviceGuard g(h->device);
        unsigned long long ev[2] = {0, 0};
        if (h->evals.ptr) {
            CARMA_CUDA(cudaDeviceSynchronize());
            CARMA_CUDA(cudaMemcpy(ev, h->evals.ptr, 16, cudaMemcpyDeviceToHost));
        }
        const bool f32 = use_f32(*h);
        if (launches) *launches = h->last_launches;
        // the exact kernel counts every (query, point) evaluation in ev[0]
        if (fp64_evals) *fp64_evals = ev[0];
        if (fp32_evals) *fp32_evals = f32 ? ev[1] : 0;
    });
}

carma_status carma_knn_set_path(carma_knn* hh, int32_t path) {
    return guarded([&] {
        KnnHandle* h = reinterpret_cast<KnnHandle*>(hh);
        if (!h) throw InvalidArg("null handle");
        if (path < 0 || path > 2) throw InvalidArg("path must be 0 (auto), 1 (exact fp64) or 2 (fp32 pre-filter)");
        h->path = path;
    });
}

}  // extern "C"

extern "C" carma_status carma_knn_last_h2d_bytes(carma_knn* hh, uint64_t* bytes) {
    return guarded([&] {
        const KnnHandle* h = reinterpret_cast<const KnnHandle*>(hh);
        if (!h || !bytes) throw InvalidArg("null argument");
        *bytes = h->last_h2d;
    });
}
