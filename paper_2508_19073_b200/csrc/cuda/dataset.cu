// Estimator datasets on the device: generate_synthetic_dataset
// (proj/src/estimators.cpp:221-264; samplers :108-217; ground_truth_memory
// memory_model.cpp:5-13; extract_features task.cpp:301-323), bit-identical
// to the reference's sequential generator.
//
// The reference draws every row from ONE std::mt19937_64 stream, and a row
// consumes a data-dependent number of draws, so the rows cannot be handed to
// threads by index. The number of draws of a row depends only on its third
// draw (the layer count): MLP 5 + 2n, CNN 8 + n, Transformer 7 + n words
// (uniform() is a multiply-shift, no rejection loop; every coin of a layer is
// drawn whether it lands or not; the batch is drawn after the layers; an
// infeasible row is redrawn from the next word on). So a generation round is:
//
//  1. ds_mt_gen: the engine's state recurrence x[j] = x[j-156] ^ f(x[j-312],
//     x[j-311]) is 156-wide parallel — one CTA of 156 threads emits 156
//     tempered words per step, the stream itself, into HBM.
//  2. ds_maps: the parsed region is cut into 512-word chunks. A row boundary
//     enters a chunk at one of 64 offsets; for each offset a lane walks the
//     row starts (one word lookup per row) to the offset at which the walk
//     leaves the chunk. Each chunk is a map [0, 64) -> [0, 64).
//  3. ds_compose / ds_entries: the maps compose associatively, so a 32-ary
//     tree (up: compose 32 maps; down: push entries through them) gives every
//     chunk its true entry offset — the row boundaries of the whole stream —
//     in log32(chunks) levels.
//  4. ds_count / scan / ds_starts: row starts per chunk, their prefix, the
//     start of every row.
//  5. ds_flags / scan / ds_emit: one thread per row evaluates the sampled
//     architecture (layers, ground-truth bytes, feasibility); the feasible
//     rows are compacted in stream order and the first n written as
//     carma_feature_row + bucket + bytes.
//
// Rows whose words run past the round's stream are left for the next round
// (their words are carried over). The host synchronises once per round to
// read the accepted count; rounds are sized from the observed words per
// accepted row.
//
// fp64 arithmetic (shaped_width's scale) is compiled with --fmad=false, so
// every product and sum rounds exactly as the host build's; (act_cos,
// act_sin) come from the host's glibc cos/sin of the 8 registry angles.

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../../include/carma_gpu.h"
#include "../host/model.hpp"
#include "common.cuh"

namespace carma_b200 {
namespace {

constexpr int kMt = 312;
constexpr int kHalf = 156;
constexpr int kMaxWords = 64;      // words per row (family bounds: MLP 25, CNN 48, Transformer 31)
constexpr uint32_t kChunk = 512;   // words per chunk of the boundary maps
constexpr uint32_t kFan = 32;      // composition tree arity

struct DsConst {
    int32_t family;
    uint32_t pad;
    uint64_t min_layers, max_layers, min_width, max_width, min_batch, max_batch;
    uint64_t min_input, max_input, min_output, max_output;
    uint64_t bytes_per_value, param_copies, alloc_block, framework_base, feasible, bucket_range;
    double act_cos[8], act_sin[8];
};

// Per-round results read back by the host (one pinned copy per round).
struct DsRound {
    unsigned long long rows;      // row starts parsed this round
    unsigned long long accepted;  // feasible rows among them
    unsigned long long tail;      // first row start not parsed (carried to the next round)
};

// rng.hpp:24-34: uniform(n) = (u128(w) * n) >> 64; uniform_int(lo, hi) = lo + uniform(hi - lo + 1).
__device__ __forceinline__ uint64_t draw(uint64_t w, uint64_t lo, uint64_t hi) {
    return lo + __umul64hi(w, hi - lo + 1);
}
// rng.hpp:20-22: next_double() = (w >> 11) * 2^-53 (exact), compared with p.
__device__ __forceinline__ bool coin(uint64_t w, double p) {
    return __dmul_rn(static_cast<double>(w >> 11), 0x1.0p-53) < p;
}

__device__ __forceinline__ uint32_t row_words(const DsConst& c, uint64_t w2) {
    const uint64_t n = draw(w2, c.min_layers, c.max_layers);
    if (c.family == 0) return static_cast<uint32_t>(5 + 2 * n);  // 6 + 2(n-1) coins + batch
    if (c.family == 1) return static_cast<uint32_t>(8 + n);      // 6 + n + dropout coin + batch
    return static_cast<uint32_t>(7 + n);                         // 6 + n + batch
}

// estimators.cpp:110-123
__device__ __forceinline__ uint64_t shaped_width(uint32_t shape, uint64_t base, uint64_t i, uint64_t n,
                                                 uint64_t floor_width) {
    if (n <= 1) return base;
    const double pos = __ddiv_rn(static_cast<double>(i), static_cast<double>(n - 1));
    double scale = 1.0;
    if (shape == 1) scale = __dsub_rn(1.0, __dmul_rn(0.75, pos));
    if (shape == 2) scale = __dsub_rn(1.0, __dmul_rn(0.75, __dsub_rn(1.0, fabs(__dsub_rn(__dmul_rn(2.0, pos), 1.0)))));
    const uint64_t v = static_cast<uint64_t>(__dmul_rn(scale, static_cast<double>(base)));
    return v > floor_width ? v : floor_width;
}

// Layer kind codes (task.hpp:14-22).
constexpr int kLinear = 0, kConv2d = 2, kBatchnorm = 3, kDropout = 4, kAttention = 5, kEmbedding = 6;

// The sampled architecture of the row whose words start at w: calls
// visit(kind, params, acts) per layer in the reference's order; returns the
// batch and writes the activation registry index.
template <class V>
__device__ __forceinline__ uint64_t architecture(const DsConst& c, const uint64_t* __restrict__ w, uint32_t& act,
                                                 V&& visit) {
    const uint64_t a0 = draw(w[0], c.min_input, c.max_input);
    const uint64_t out = draw(w[1], c.min_output, c.max_output);
    const uint64_t n = draw(w[2], c.min_layers, c.max_layers);
    const uint64_t base = draw(w[3], c.min_width, c.max_width);
    const uint32_t shape = static_cast<uint32_t>(__umul64hi(w[4], 3));
    act = static_cast<uint32_t>(__umul64hi(w[5], 8));
    uint32_t k = 6;
    if (c.family == 0) {  // sample_mlp, estimators.cpp:125-153
        uint64_t prev = a0;
        for (uint64_t i = 0; i < n; ++i) {
            const bool head = i + 1 == n;
            const uint64_t wd = head ? out : shaped_width(shape, base, i, n, c.min_width);
            visit(kLinear, prev * wd + wd, wd);
            if (!head) {
                if (coin(w[k++], 0.5)) visit(kBatchnorm, 2 * wd, wd);
                if (coin(w[k++], 0.3)) visit(kDropout, 0ull, wd);
            }
            prev = wd;
        }
    } else if (c.family == 1) {  // sample_cnn, estimators.cpp:155-186
        uint64_t c_prev = 3, spatial = a0 * a0;
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t ch = shaped_width(shape, base, n - 1 - i, n, c.min_width);
            visit(kConv2d, 9 * c_prev * ch + ch, ch * spatial);
            if (coin(w[k++], 0.7)) visit(kBatchnorm, 2 * ch, ch * spatial);
            if (i % 2 == 1 && spatial > 64) spatial /= 4;
            c_prev = ch;
        }
        if (coin(w[k++], 0.3)) visit(kDropout, 0ull, c_prev);
        visit(kLinear, c_prev * out + out, out);
    } else {  // sample_transformer, estimators.cpp:188-217
        const uint64_t d0 = (base / 64) * 64;
        visit(kEmbedding, out * d0, a0 * d0);
        for (uint64_t i = 0; i < n; ++i) {
            uint64_t d = shaped_width(shape, base, i, n, c.min_width);
            d = (d / 64) * 64;
            if (d < 64) d = 64;
            visit(kAttention, 4 * d * d, 2 * a0 * d);
            visit(kLinear, 8 * d * d, 5 * a0 * d);
            if (coin(w[k++], 0.4)) visit(kDropout, 0ull, a0 * d);
        }
    }
    return draw(w[k], c.min_batch, c.max_batch);
}

// One row: features (extract_features), ground-truth bytes and feasibility.
template <bool FULL>
__device__ __forceinline__ bool eval_row(const DsConst& c, const uint64_t* __restrict__ w, carma_feature_row& f,
                                         uint64_t& mem) {
    uint32_t act = 0;
    uint32_t size = 0;
    if (FULL) architecture(c, w, act, [&](int, uint64_t, uint64_t) { ++size; });
    const uint32_t pick1 = size / 2, pick2 = size - 1;
    uint64_t nl = 0, nb = 0, nd = 0, nc = 0, params = 0, acts = 0;
    uint32_t idx = 0;
    const uint64_t batch = architecture(c, w, act, [&](int kind, uint64_t prm, uint64_t ac) {
        nl += kind == kLinear;
        nb += kind == kBatchnorm;
        nd += kind == kDropout;
        nc += kind == 1 || kind == kConv2d;
        params += prm;
        acts += ac;
        if (FULL) {
            if (idx == 0) { f.kind[0] = kind; f.tuple_acts[0] = ac; f.tuple_params[0] = prm; }
            if (idx == pick1) { f.kind[1] = kind; f.tuple_acts[1] = ac; f.tuple_params[1] = prm; }
            if (idx == pick2) { f.kind[2] = kind; f.tuple_acts[2] = ac; f.tuple_params[2] = prm; }
        }
        ++idx;
    });
    // memory_model.cpp:5-13
    const uint64_t raw = c.bytes_per_value * c.param_copies * params + c.bytes_per_value * batch * acts;
    const uint64_t blocks = (raw + c.alloc_block - 1) / c.alloc_block;
    mem = c.framework_base + blocks * c.alloc_block;
    if (FULL) {
        f.n_linear = nl;
        f.n_batchnorm = nb;
        f.n_dropout = nd;
        f.n_conv = nc;
        f.batch_size = batch;
        f.total_params = params;
        f.total_activations = acts;
        f.act_cos = c.act_cos[act];
        f.act_sin = c.act_sin[act];
        f.has_layers = 1;
    }
    return mem <= c.feasible;
}

// ---------------------------------------------------------------- the stream
// Thread t owns state words x[312 + 156 s + t], s = 0, 1, ...: its own
// previous word is x[j-156] and the one before x[j-312]; x[j-311] is the
// neighbour's word of two steps back (thread 155: thread 0's of one step
// back). st[0..311] holds the 312 state words preceding the call and is
// updated to the 312 words following it. out[k] = temper(x[312 + k]).
// Multi-segment form: CTA c starts from the window starts[c] (the state
// jumped c * seg_steps * 156 words ahead, ds_mt_jump) and emits its segment
// out[c * seg_steps * 156 ...]; the last CTA's final window goes to st.
__global__ void __launch_bounds__(kHalf) ds_mt_gen(uint64_t* __restrict__ st, const uint64_t* __restrict__ starts,
                                                   uint64_t* __restrict__ out, uint32_t seg_steps, uint32_t last_steps) {
    constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull, kA = 0xB5026F5AA96619E9ull;
    __shared__ uint64_t ring[3][kHalf];
    const int t = threadIdx.x;
    const bool last = blockIdx.x + 1 == gridDim.x;
    const uint32_t steps = last ? last_steps : seg_steps;
    const uint64_t* w0 = starts ? starts + static_cast<uint64_t>(blockIdx.x) * kMt : st;
    out += static_cast<uint64_t>(blockIdx.x) * seg_steps * kHalf;
    uint64_t p2 = w0[t], p1 = w0[kHalf + t];  // own words of steps s-2, s-1
    ring[1][t] = p2;                          // slot (s mod 3) holds step s; s = -2 -> 1, -1 -> 2
    ring[2][t] = p1;
    __syncthreads();
    for (uint32_t s = 0; s < steps; ++s) {
        const uint32_t s2 = (s + 1) % 3, s1 = (s + 2) % 3, s0 = s % 3;
        const uint64_t nb = t + 1 < kHalf ? ring[s2][t + 1] : ring[s1][0];
        const uint64_t y = (p2 & kUpper) | (nb & kLower);
        const uint64_t v = p1 ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
        ring[s0][t] = v;
        uint64_t z = v;
        z ^= (z >> 29) & 0x5555555555555555ull;
        z ^= (z << 17) & 0x71D67FFFEDA60000ull;
        z ^= (z << 37) & 0xFFF7EEE000000000ull;
        z ^= z >> 43;
        out[static_cast<uint64_t>(s) * kHalf + t] = z;
        p2 = p1;
        p1 = v;
        __syncthreads();
    }
    if (last) {
        st[t] = p2;
        st[kHalf + t] = p1;
    }
}

// Jump-ahead (the engine is F2-linear: the window after k words is g(A)
// applied to the window, g = x^k mod the characteristic polynomial). CTA c
// composes the jumps of the set bits of c (polys[b] = x^(J 2^b) mod P) with
// Horner's rule on a 312-word circular window in shared memory: per bit of
// g, advance the accumulator one word (one thread: x[j+312] = x[j+156] ^
// f(x[j], x[j+1])), then add the input window if the bit is set (all
// threads). One warp: __syncwarp is the only barrier.
constexpr int kPolyWords = 312;  // 19968 bits >= deg P + 1 = 19938
__global__ void __launch_bounds__(32) ds_mt_jump(const uint64_t* __restrict__ st, const uint64_t* __restrict__ polys,
                                                 const int32_t* __restrict__ degs, int n_polys,
                                                 uint64_t* __restrict__ starts) {
    constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull, kA = 0xB5026F5AA96619E9ull;
    __shared__ uint64_t R[kMt], T[kMt];
    const unsigned lane = threadIdx.x;
    const uint32_t c = blockIdx.x;
    for (int k = lane; k < kMt; k += 32) R[k] = st[k];
    __syncwarp();
    for (int b = 0; b < n_polys; ++b) {
        if (!((c >> b) & 1u)) continue;
        const uint64_t* g = polys + static_cast<uint64_t>(b) * kPolyWords;
        for (int k = lane; k < kMt; k += 32) T[k] = 0;
        uint32_t h = 0;  // T's first word
        __syncwarp();
        for (int i = degs[b]; i >= 0; --i) {
            if (lane == 0) {  // T = A T
                const uint32_t h1 = h + 1 == kMt ? 0 : h + 1, hm = h + 156 >= kMt ? h + 156 - kMt : h + 156;
                const uint64_t y = (T[h] & kUpper) | (T[h1] & kLower);
                T[h] = T[hm] ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
            }
            h = h + 1 == kMt ? 0 : h + 1;
            __syncwarp();
            if ((g[i >> 6] >> (i & 63)) & 1ull) {  // T += R
                for (int k = lane; k < kMt; k += 32) {
                    const uint32_t x = h + k >= kMt ? h + k - kMt : h + k;
                    T[x] ^= R[k];
                }
                __syncwarp();
            }
        }
        for (int k = lane; k < kMt; k += 32) {
            const uint32_t x = h + k >= kMt ? h + k - kMt : h + k;
            R[k] = T[x];
        }
        __syncwarp();
    }
    for (int k = lane; k < kMt; k += 32) starts[static_cast<uint64_t>(c) * kMt + k] = R[k];
}

// ---------------------------------------------------------------- row boundaries
// Chunk t covers row starts in [t*C, min((t+1)*C, P)). Lane l of the chunk's
// warp walks from entry offsets l and l + 32.
__global__ void __launch_bounds__(256) ds_maps(const DsConst c, const uint64_t* __restrict__ w, uint64_t P,
                                               uint32_t nc, uint8_t* __restrict__ maps) {
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (warp >= nc) return;
    const uint64_t begin = warp * kChunk, end = min(begin + kChunk, P);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t e = lane + 32 * h;
        uint64_t pos = begin + e;
        while (pos < end) pos += row_words(c, __ldg(w + pos + 2));
        maps[warp * kMaxWords + e] = static_cast<uint8_t>(pos - end);
    }
}

// out[g] = in[g*32 + 31] o ... o in[g*32] (applied in stream order).
__global__ void __launch_bounds__(256) ds_compose(const uint8_t* __restrict__ in, uint32_t m,
                                                  uint8_t* __restrict__ out, uint32_t groups) {
    const uint64_t g = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (g >= groups) return;
    const uint32_t j_end = min(static_cast<uint32_t>(g * kFan + kFan), m);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t v = lane + 32 * h;
        for (uint32_t j = static_cast<uint32_t>(g * kFan); j < j_end; ++j) v = in[static_cast<uint64_t>(j) * kMaxWords + v];
        out[g * kMaxWords + lane + 32 * h] = static_cast<uint8_t>(v);
    }
}

// entry[j] for the members of group g, from the group's entry (parent, or 0
// at the root); at the root also the tail offset past the last chunk.
__global__ void __launch_bounds__(128) ds_entries(const uint8_t* __restrict__ in, uint32_t m,
                                                  const uint8_t* __restrict__ parent, uint32_t groups,
                                                  uint8_t* __restrict__ entry, uint64_t P, DsRound* res) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= groups) return;
    uint32_t v = parent ? parent[g] : 0u;
    const uint32_t j_end = min(g * kFan + kFan, m);
    for (uint32_t j = g * kFan; j < j_end; ++j) {
        entry[j] = static_cast<uint8_t>(v);
        v = in[static_cast<uint64_t>(j) * kMaxWords + v];
    }
    if (res && j_end == m) res->tail = P + v;  // the group holding the last chunk
}

__global__ void __launch_bounds__(256) ds_count(const DsConst c, const uint64_t* __restrict__ w, uint64_t P,
                                                uint32_t nc, const uint8_t* __restrict__ entry,
                                                uint32_t* __restrict__ counts) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nc) return;
    const uint64_t begin = static_cast<uint64_t>(t) * kChunk, end = min(begin + kChunk, P);
    uint64_t pos = begin + entry[t];
    uint32_t n = 0;
    while (pos < end) {
        ++n;
        pos += row_words(c, __ldg(w + pos + 2));
    }
    counts[t] = n;
}

__global__ void __launch_bounds__(256) ds_starts(const DsConst c, const uint64_t* __restrict__ w, uint64_t P,
                                                 uint32_t nc, const uint8_t* __restrict__ entry,
                                                 const uint32_t* __restrict__ counts,
                                                 const uint32_t* __restrict__ roff, uint32_t* __restrict__ starts,
                                                 DsRound* res) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nc) return;
    const uint64_t begin = static_cast<uint64_t>(t) * kChunk, end = min(begin + kChunk, P);
    uint64_t pos = begin + entry[t];
    uint32_t o = roff[t];
    while (pos < end) {
        starts[o++] = static_cast<uint32_t>(pos);
        pos += row_words(c, __ldg(w + pos + 2));
    }
    if (t == nc - 1) res->rows = o;
}

__global__ void __launch_bounds__(256) ds_flags(const DsConst c, const uint64_t* __restrict__ w,
                                                const uint32_t* __restrict__ starts, const DsRound* res,
                                                uint32_t* __restrict__ flags) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= res->rows) return;
    carma_feature_row f;
    uint64_t mem;
    flags[r] = eval_row<false>(c, w + starts[r], f, mem) ? 1u : 0u;
}

__global__ void __launch_bounds__(256) ds_emit(const DsConst c, const uint64_t* __restrict__ w,
                                               const uint32_t* __restrict__ starts, const uint32_t* __restrict__ flags,
                                               const uint32_t* __restrict__ aidx, DsRound* res, uint64_t done,
                                               uint64_t n, carma_feature_row* __restrict__ rows,
                                               int32_t* __restrict__ bucket, uint64_t* __restrict__ mem_out) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nr = res->rows;
    if (r >= nr) return;
    if (r == nr - 1) res->accepted = aidx[r] + flags[r];
    if (!flags[r]) return;
    const uint64_t o = done + aidx[r];
    if (o >= n) return;
    carma_feature_row f{};
    uint64_t mem;
    eval_row<true>(c, w + starts[r], f, mem);
    if (rows) rows[o] = f;
    if (bucket) bucket[o] = static_cast<int32_t>(mem / c.bucket_range);
    if (mem_out) mem_out[o] = mem;
}

// Carries the unparsed words [tail, V) to the front of the buffer (< 64
// words, so source and destination never overlap: tail >= V - 63 >= 64).
__global__ void ds_carry(uint64_t* w, const DsRound* res, uint64_t V) {
    const uint64_t tail = res->tail;
    for (uint64_t i = threadIdx.x; tail + i < V; i += blockDim.x) w[i] = w[tail + i];
}

// ------------------------------------------------ jump-ahead (host side)
// The characteristic polynomial of the mt19937_64 transition (degree 19937)
// by Berlekamp-Massey over one bit of the raw state sequence, and the jump
// polynomials x^(J 2^b) mod P (J = 156 * 2^kSegLog2 words), by squaring.
using Poly = std::vector<uint64_t>;  // bit i = coefficient of x^i

int poly_deg(const Poly& p) {
    for (size_t w = p.size(); w-- > 0;)
        if (p[w]) return static_cast<int>(w * 64 + 63 - __builtin_clzll(p[w]));
    return -1;
}

// The raw window sequence from a seed (the host twin of the device recurrence).
void mt_raw_words(uint64_t seed, std::vector<uint64_t>& x, size_t n) {
    constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull, kA = 0xB5026F5AA96619E9ull;
    x.assign(n, 0);
    x[0] = seed;
    for (size_t i = 1; i < kMt; ++i) x[i] = 6364136223846793005ull * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    for (size_t j = kMt; j < n; ++j) {
        const uint64_t y = (x[j - kMt] & kUpper) | (x[j - kMt + 1] & kLower);
        x[j] = x[j - kHalf] ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
    }
}

// Berlekamp-Massey over GF(2): the connection polynomial C of the bit
// sequence s (C(x) = 1 + c1 x + ... ; the characteristic polynomial is its
// reciprocal).
Poly berlekamp_massey(const std::vector<uint8_t>& s) {
    const size_t n = s.size(), W = (n + 64) / 64 + 1;
    Poly C(W, 0), B(W, 0);
    C[0] = B[0] = 1;
    int L = 0;
    long m = -1;
    for (size_t N = 0; N < n; ++N) {
        uint8_t d = s[N];
        for (int i = 1; i <= L; ++i) d ^= static_cast<uint8_t>((C[i >> 6] >> (i & 63)) & 1ull) & s[N - i];
        if (!d) continue;
        const Poly T = C;
        const size_t sh = N - static_cast<size_t>(m);  // C ^= B << sh
        const size_t ws = sh / 64, bs = sh % 64;
        for (size_t w = W; w-- > ws;) {
            uint64_t v = B[w - ws] << bs;
            if (bs && w - ws > 0) v |= B[w - ws - 1] >> (64 - bs);
            C[w] ^= v;
        }
        if (2 * L <= static_cast<int>(N)) {
            L = static_cast<int>(N) + 1 - L;
            m = static_cast<long>(N);
            B = T;
        }
    }
    // characteristic polynomial = x^L C(1/x): reverse the first L + 1 coefficients
    Poly P(kPolyWords, 0);
    for (int i = 0; i <= L; ++i)
        if ((C[i >> 6] >> (i & 63)) & 1ull) {
            const int j = L - i;
            P[j >> 6] |= 1ull << (j & 63);
        }
    return P;
}

// a * a mod P (deg a < deg P).
Poly poly_sqr_mod(const Poly& a, const Poly& P, int dp) {
    Poly r(2 * kPolyWords + 1, 0);
    for (int i = 0; i <= poly_deg(a); ++i)
        if ((a[i >> 6] >> (i & 63)) & 1ull) {
            const int j = 2 * i;
            r[j >> 6] |= 1ull << (j & 63);
        }
    for (int i = poly_deg(r); i >= dp; --i) {
        if (!((r[i >> 6] >> (i & 63)) & 1ull)) continue;
        const int sh = i - dp;  // r ^= P << sh
        const int ws = sh / 64, bs = sh % 64;
        for (int w = kPolyWords - 1; w >= 0; --w) {
            if (!P[w]) continue;
            r[w + ws] ^= P[w] << bs;
            if (bs && w + ws + 1 < static_cast<int>(r.size())) r[w + ws + 1] ^= P[w] >> (64 - bs);
        }
    }
    r.resize(kPolyWords);
    return r;
}

constexpr int kSegLog2 = 13;    // segment = 156 * 2^13 = 1,277,952 words
constexpr int kJumpPolys = 9;   // up to 512 segments per round

struct JumpTables {
    Poly P;
    int deg = 0;
    std::vector<uint64_t> polys;  // kJumpPolys x kPolyWords: x^(156 * 2^(kSegLog2 + b)) mod P
    std::vector<int32_t> degs;
};

const JumpTables& jump_tables() {
    static const JumpTables t = [] {
        JumpTables j;
        std::vector<uint64_t> x;
        const size_t nb = 2 * 19937 + 64;
        mt_raw_words(5489, x, kMt + nb);
        std::vector<uint8_t> bits(nb);
        for (size_t i = 0; i < nb; ++i) bits[i] = static_cast<uint8_t>(x[kMt + i] & 1ull);
        j.P = berlekamp_massey(bits);
        j.deg = poly_deg(j.P);
        if (j.deg != 19937) throw CudaFailure("mt19937_64 characteristic polynomial: unexpected degree");
        Poly g(kPolyWords, 0);
        g[156 >> 6] |= 1ull << (156 & 63);  // x^156
        for (int k = 0; k < kSegLog2; ++k) g = poly_sqr_mod(g, j.P, j.deg);
        for (int b = 0; b < kJumpPolys; ++b) {
            if (b > 0) g = poly_sqr_mod(g, j.P, j.deg);
            j.polys.insert(j.polys.end(), g.begin(), g.end());
            j.degs.push_back(poly_deg(g));
        }
        return j;
    }();
    return t;
}

// Host Horner: the window w advanced by the jump g (for the self-check).
std::vector<uint64_t> host_jump(const std::vector<uint64_t>& w, const uint64_t* g, int deg) {
    constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull, kA = 0xB5026F5AA96619E9ull;
    std::vector<uint64_t> T(kMt, 0);
    uint32_t h = 0;
    for (int i = deg; i >= 0; --i) {
        const uint32_t h1 = h + 1 == kMt ? 0 : h + 1, hm = h + 156 >= kMt ? h + 156 - kMt : h + 156;
        const uint64_t y = (T[h] & kUpper) | (T[h1] & kLower);
        T[h] = T[hm] ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
        h = h1;
        if ((g[i >> 6] >> (i & 63)) & 1ull)
            for (uint32_t k = 0; k < kMt; ++k) T[(h + k) % kMt] ^= w[k];
    }
    std::vector<uint64_t> r(kMt);
    for (uint32_t k = 0; k < kMt; ++k) r[k] = T[(h + k) % kMt];
    return r;
}

DsConst make_const(int32_t family) {
    if (family < 0 || family > 2) throw InvalidArg("unknown model family");
    const Bounds b = Bounds::for_family(static_cast<Family>(family));
    const SimConstants sc;
    DsConst c{};
    c.family = family;
    c.min_layers = b.min_layers;
    c.max_layers = b.max_layers;
    c.min_width = b.min_width;
    c.max_width = b.max_width;
    c.min_batch = b.min_batch;
    c.max_batch = b.max_batch;
    c.min_input = b.min_input;
    c.max_input = b.max_input;
    c.min_output = b.min_output;
    c.max_output = b.max_output;
    c.bytes_per_value = sc.bytes_per_value;
    c.param_copies = sc.param_copies;
    c.alloc_block = sc.alloc_block;
    c.framework_base = sc.framework_base;
    c.feasible = sc.gpu_capacity;
    c.bucket_range = default_bucket_range(static_cast<Family>(family));
    for (int i = 0; i < 8; ++i) {  // extract_features' glibc cos / sin of the registry angle
        c.act_cos[i] = std::cos(activation_angle(i));
        c.act_sin[i] = std::sin(activation_angle(i));
    }
    const uint64_t lmax = family == 0 ? 5 + 2 * b.max_layers : family == 1 ? 8 + b.max_layers : 7 + b.max_layers;
    if (lmax > static_cast<uint64_t>(kMaxWords)) throw Unsupported("rows longer than 64 draws");
    return c;
}

unsigned blocks_for(uint64_t threads, unsigned per_block) {
    return static_cast<unsigned>((threads + per_block - 1) / per_block);
}

}  // namespace

// generate_synthetic_dataset(family, n, seed) into device buffers on stream s.
void generate_dataset_device(int32_t family, uint64_t n, uint64_t seed, carma_feature_row* rows, int32_t* bucket,
                             uint64_t* mem, cudaStream_t s, carma_dataset_stats* stats) {
    const DsConst c = make_const(family);
    // Words per feasible row: the bounds' mean layer count over the measured
    // feasible fraction of the family (MLP 100%, CNN ~84.6%, Transformer
    // ~97.5%, default bounds); later rounds use the observed rate.
    const double mean_n = 0.5 * static_cast<double>(c.min_layers + c.max_layers);
    const double mean_words = family == 0 ? 5 + 2 * mean_n : family == 1 ? 8 + mean_n : 7 + mean_n;
    const double feasible_frac = family == 0 ? 1.0 : family == 1 ? 0.84 : 0.97;
    uint64_t max_round = 1ull << 29;  // words per round (4 GiB)
    if (const char* e = std::getenv("CARMA_DATASET_ROUND_WORDS"))  // test knob: force many rounds
        max_round = std::max<uint64_t>(std::strtoull(e, nullptr, 10), 4 * kChunk);

    // engine state after seeding (std::mt19937_64: x0 = seed, x_i = f * (x_{i-1} ^ x_{i-1} >> 62) + i)
    std::vector<uint64_t> init(kMt);
    init[0] = seed;
    for (int i = 1; i < kMt; ++i) init[i] = 6364136223846793005ull * (init[i - 1] ^ (init[i - 1] >> 62)) + i;

    DeviceBuffer d_state, d_w, d_maps, d_entry, d_counts, d_roff, d_starts, d_flags, d_aidx, d_res, d_tmp;
    DeviceBuffer d_polys, d_degs, d_seg;  // jump-ahead tables, segment start windows
    PinnedBuffer h_res;
    h_res.ensure(sizeof(DsRound));
    d_state.ensure(kMt * 8);
    d_res.ensure(sizeof(DsRound));
    CARMA_CUDA(cudaMemcpyAsync(d_state.ptr, init.data(), kMt * 8, cudaMemcpyHostToDevice, s));

    uint64_t done = 0, carried = 0, words = 0, parsed = 0, accepted = 0;
    uint32_t rounds = 0;
    double words_per_row = mean_words / feasible_frac;
    uint64_t cap_words = 0;  // the word buffer holds carried + fresh words; allocated once
    while (done < n) {
        const uint64_t want = static_cast<uint64_t>(static_cast<double>(n - done) * words_per_row * 1.02) + 8192;
        uint64_t steps = std::min<uint64_t>((want + kHalf - 1) / kHalf, max_round / kHalf);
        if (cap_words == 0) {
            cap_words = steps * kHalf + kMaxWords;
            d_w.ensure(cap_words * 8);
        }
        steps = std::min<uint64_t>(steps, (cap_words - carried) / kHalf);  // the carried words stay in place
        const uint64_t fresh = steps * kHalf;
        const uint64_t V = carried + fresh;
        // scratch (grow-only; DeviceBuffer::ensure synchronises before recycling)
        const uint64_t P = V - kMaxWords + 1;  // parse row starts < P: their words end <= V
        const uint32_t nc = static_cast<uint32_t>((P + kChunk - 1) / kChunk);
        std::vector<uint32_t> level_n{nc};
        while (level_n.back() > 1) level_n.push_back((level_n.back() + kFan - 1) / kFan);
        uint64_t map_bytes = 0, entry_bytes = 0;
        for (uint32_t m : level_n) {
            map_bytes += static_cast<uint64_t>(m) * kMaxWords;
            entry_bytes += m;
        }
        d_maps.ensure(map_bytes);
        d_entry.ensure(entry_bytes);
        d_counts.ensure(static_cast<uint64_t>(nc) * 4);
        d_roff.ensure(static_cast<uint64_t>(nc) * 4);
        const uint64_t max_rows = P / 7 + 1;  // every family's row has >= 7 words
        d_starts.ensure(max_rows * 4);
        d_flags.ensure(max_rows * 4);
        d_aidx.ensure(max_rows * 4);
        size_t tmp1 = 0, tmp2 = 0;
        CARMA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp1, d_counts.as<uint32_t>(), d_roff.as<uint32_t>(), nc, s));
        CARMA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, d_flags.as<uint32_t>(), d_aidx.as<uint32_t>(),
                                                 static_cast<int64_t>(max_rows), s));
        d_tmp.ensure(std::max(tmp1, tmp2));

        uint64_t* w = d_w.as<uint64_t>();
        // the stream: segments of 156 * 2^kSegLog2 words, one CTA each, from
        // windows jumped ahead on the device
        constexpr uint64_t seg_steps = 1ull << kSegLog2;
        const uint64_t n_seg = (steps + seg_steps - 1) / seg_steps;
        const uint32_t last_steps = static_cast<uint32_t>(steps - (n_seg - 1) * seg_steps);
        if (n_seg > 1) {
            if (n_seg > (1ull << kJumpPolys)) throw CudaFailure("dataset generator: too many stream segments");
            const JumpTables& jt = jump_tables();
            if (!d_polys.ptr) {
                d_polys.ensure(jt.polys.size() * 8);
                d_degs.ensure(jt.degs.size() * 4);
                CARMA_CUDA(cudaMemcpyAsync(d_polys.ptr, jt.polys.data(), jt.polys.size() * 8, cudaMemcpyHostToDevice, s));
                CARMA_CUDA(cudaMemcpyAsync(d_degs.ptr, jt.degs.data(), jt.degs.size() * 4, cudaMemcpyHostToDevice, s));
            }
            d_seg.ensure(n_seg * kMt * 8);
            ds_mt_jump<<<static_cast<unsigned>(n_seg), 32, 0, s>>>(d_state.as<uint64_t>(), d_polys.as<uint64_t>(),
                                                                   d_degs.as<int32_t>(), kJumpPolys, d_seg.as<uint64_t>());
            ds_mt_gen<<<static_cast<unsigned>(n_seg), kHalf, 0, s>>>(d_state.as<uint64_t>(), d_seg.as<uint64_t>(),
                                                                     w + carried, static_cast<uint32_t>(seg_steps),
                                                                     last_steps);
        } else {
            ds_mt_gen<<<1, kHalf, 0, s>>>(d_state.as<uint64_t>(), nullptr, w + carried, last_steps, last_steps);
        }
        CARMA_CUDA(cudaGetLastError());
        // boundary maps and the composition tree
        std::vector<uint8_t*> lmap(level_n.size()), lent(level_n.size());
        {
            uint8_t* pm = d_maps.as<uint8_t>();
            uint8_t* pe = d_entry.as<uint8_t>();
            for (size_t l = 0; l < level_n.size(); ++l) {
                lmap[l] = pm;
                lent[l] = pe;
                pm += static_cast<uint64_t>(level_n[l]) * kMaxWords;
                pe += level_n[l];
            }
        }
        ds_maps<<<blocks_for(static_cast<uint64_t>(nc) * 32, 256), 256, 0, s>>>(c, w, P, nc, lmap[0]);
        for (size_t l = 1; l < level_n.size(); ++l)
            ds_compose<<<blocks_for(static_cast<uint64_t>(level_n[l]) * 32, 256), 256, 0, s>>>(
                lmap[l - 1], level_n[l - 1], lmap[l], level_n[l]);
        // top-down: level L-1 has one map (or nc == 1: level 0 is the root)
        for (size_t l = level_n.size(); l-- > 0;) {
            const uint32_t groups = l + 1 < level_n.size() ? level_n[l + 1] : 1;
            ds_entries<<<blocks_for(groups, 128), 128, 0, s>>>(lmap[l], level_n[l],
                                                               l + 1 < level_n.size() ? lent[l + 1] : nullptr, groups,
                                                               lent[l], P, l == 0 ? d_res.as<DsRound>() : nullptr);
        }
        CARMA_CUDA(cudaGetLastError());
        ds_count<<<blocks_for(nc, 256), 256, 0, s>>>(c, w, P, nc, lent[0], d_counts.as<uint32_t>());
        size_t t1 = d_tmp.bytes;
        CARMA_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp.ptr, t1, d_counts.as<uint32_t>(), d_roff.as<uint32_t>(), nc, s));
        ds_starts<<<blocks_for(nc, 256), 256, 0, s>>>(c, w, P, nc, lent[0], d_counts.as<uint32_t>(),
                                                      d_roff.as<uint32_t>(), d_starts.as<uint32_t>(),
                                                      d_res.as<DsRound>());
        ds_flags<<<blocks_for(max_rows, 256), 256, 0, s>>>(c, w, d_starts.as<uint32_t>(), d_res.as<DsRound>(),
                                                           d_flags.as<uint32_t>());
        size_t t2 = d_tmp.bytes;
        CARMA_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp.ptr, t2, d_flags.as<uint32_t>(), d_aidx.as<uint32_t>(),
                                                 static_cast<int64_t>(max_rows), s));
        ds_emit<<<blocks_for(max_rows, 256), 256, 0, s>>>(c, w, d_starts.as<uint32_t>(), d_flags.as<uint32_t>(),
                                                          d_aidx.as<uint32_t>(), d_res.as<DsRound>(), done, n, rows,
                                                          bucket, mem);
        CARMA_CUDA(cudaGetLastError());
        CARMA_CUDA(cudaMemcpyAsync(h_res.ptr, d_res.ptr, sizeof(DsRound), cudaMemcpyDeviceToHost, s));
        CARMA_CUDA(cudaStreamSynchronize(s));
        const DsRound r = *h_res.as<DsRound>();
        if (r.tail < P || r.tail > V) throw CudaFailure("dataset generator: inconsistent row boundary");
        ++rounds;
        words += fresh;
        if (r.accepted == 0 && r.rows > 10000)  // estimators.cpp:249-250
            throw InvalidArg("InvalidBounds: bounds generate almost no feasible configs");
        parsed += r.rows;
        accepted += r.accepted;
        done += std::min<uint64_t>(r.accepted, n - done);
        if (r.accepted > 0) words_per_row = static_cast<double>(P) / static_cast<double>(r.accepted);
        if (done < n) {
            ds_carry<<<1, 64, 0, s>>>(w, d_res.as<DsRound>(), V);
            CARMA_CUDA(cudaGetLastError());
            carried = V > r.tail ? V - r.tail : 0;
        }
    }
    if (stats) {
        stats->words_generated = words;
        stats->rows_parsed = parsed;
        stats->rows_accepted = accepted;
        stats->rounds = rounds;
    }
}

}  // namespace carma_b200

using namespace carma_b200;

extern "C" {

carma_status carma_dataset_generate_device(int32_t device, int32_t family, uint64_t n, uint64_t seed,
                                           carma_feature_row* rows, int32_t* bucket, uint64_t* mem, void* stream,
                                           carma_dataset_stats* stats) {
    return guarded([&] {
        if (n == 0) throw InvalidArg("InvalidBounds: n_samples must be > 0");
        require_device(device);
        DeviceGuard guard(device);
        generate_dataset_device(family, n, seed, rows, bucket, mem, static_cast<cudaStream_t>(stream), stats);
    });
}

carma_status carma_dataset_generate(int32_t device, int32_t family, uint64_t n, uint64_t seed,
                                    carma_feature_row* rows, int32_t* bucket, uint64_t* mem,
                                    carma_dataset_stats* stats) {
    return guarded([&] {
        if (n == 0) throw InvalidArg("InvalidBounds: n_samples must be > 0");
        require_device(device);
        DeviceGuard guard(device);
        cudaStream_t s;
        CARMA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{s};
        DeviceBuffer d_rows, d_bucket, d_mem;
        if (rows) d_rows.ensure(n * sizeof(carma_feature_row));
        if (bucket) d_bucket.ensure(n * 4);
        if (mem) d_mem.ensure(n * 8);
        generate_dataset_device(family, n, seed, d_rows.as<carma_feature_row>(), d_bucket.as<int32_t>(),
                                d_mem.as<uint64_t>(), s, stats);
        if (rows) CARMA_CUDA(cudaMemcpyAsync(rows, d_rows.ptr, n * sizeof(carma_feature_row), cudaMemcpyDeviceToHost, s));
        if (bucket) CARMA_CUDA(cudaMemcpyAsync(bucket, d_bucket.ptr, n * 4, cudaMemcpyDeviceToHost, s));
        if (mem) CARMA_CUDA(cudaMemcpyAsync(mem, d_mem.ptr, n * 8, cudaMemcpyDeviceToHost, s));
        CARMA_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

// Self-check of the jump-ahead math on the host (tests): the window jumped by
// polynomial b of the device tables equals the window reached by stepping
// 156 * 2^(kSegLog2 + b) words (the first word's low 31 bits, which no later
// word depends on, excluded). *mismatches = differing words.
extern "C" carma_status carma_host_check_mt_jump(uint64_t seed, int32_t b, uint64_t* mismatches) {
    return carma_b200::guarded([&] {
        using namespace carma_b200;
        if (!mismatches || b < 0 || b > 2) throw InvalidArg("bad argument");
        const JumpTables& jt = jump_tables();
        const uint64_t k = 156ull << (kSegLog2 + b);
        std::vector<uint64_t> x;
        mt_raw_words(seed, x, kMt + k + 1);
        const std::vector<uint64_t> w0(x.begin(), x.begin() + kMt);
        const std::vector<uint64_t> wj = host_jump(w0, jt.polys.data() + static_cast<size_t>(b) * kPolyWords, jt.degs[b]);
        uint64_t bad = 0;
        for (int i = 0; i < kMt; ++i) {
            const uint64_t mask = i == 0 ? 0xFFFFFFFF80000000ull : ~0ull;
            bad += ((wj[i] ^ x[k + i]) & mask) != 0;
        }
        *mismatches = bad;
    });
}
