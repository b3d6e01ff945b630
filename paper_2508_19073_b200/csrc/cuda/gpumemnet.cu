// Stage 1, neural estimator — the paper's GPUMemNet MLP ensemble on sm_100a
// tensor cores (tcgen05 + TMEM), fused end to end.
//
// Semantics (carma_gpu.h "neural GPUMemNet"): E members,
// each a stack of 1..8 ReLU layers of <= 8 neurons (batch norm folded) and a
// linear head over C memory bins; softmax per member, probabilities averaged
// over members, argmax (ties to the larger bin), bytes = (bin + 1) * range
// (estimate_learned, proj/src/estimators.cpp:540-551). Inputs are the 19
// scalar_features (estimators.cpp:317-342) of any estimator row format.
//
// Layout on the tensor cores. The E members run side by side, sorted by
// depth (descending): layer l of the members still running (a prefix of
// alive_l members) is one block-diagonal GEMM
//     H_l[128 rows x 8 alive_l] = relu(H_{l-1} . W_l^T + b_l)
// (member m owns columns 8m..8m+7; N and K padded to 16 with zero weights).
// A member that has finished keeps its last activations in its A-tile
// columns, untouched, until the head reads every member with one K = 64 GEMM
// per pass of up to 128 columns (members side by side, CP = C rounded up to 8
// columns each). Layer 0 reads the 19 transformed features (K padded to 32).
// Each MMA is tcgen05.mma.cta_group::1.kind::f16, M = 128, bf16 operands from
// shared memory (K-major, canonical no-swizzle layout), fp32 accumulators in
// TMEM.
//
// Precision: weights are bf16 values. Activations are split into three
// bf16 parts, h = a0 + a1 + a2 exactly (a0 = trunc_bf16(h), a1 =
// trunc_bf16(h - a0), a2 = h - a0 - a1), and every layer accumulates
// A0.W + A1.W + A2.W in fp32: the products are exact and the activations
// keep all 24 bits of their fp32 value, as in an fp32 evaluation. (Two parts keep ~17 bits: measured 6.5e-4 relative
// logit error on the 8-layer MLP-family ensemble, against 1e-5 for fp32 —
// re-rounding the activations at every layer dominates. The north star's bar
// is 1e-3.)
//
// Work split. A CTA per SM holds the model (~42 KB for the 6-bin families,
// ~90 KB for the 41-bin MLP family) in shared memory and runs G groups of
// 256 threads (3, or 2 for the MLP family: 48 KB of A tiles per group). A
// group owns a 128-row tile at a time, its A tiles (3 x 16 KB), 128 TMEM
// columns and an mbarrier; its two warp halves share the TMEM lanes and split
// the columns (see nn_ensemble). Per layer: the group stores its activations,
// fences them into the async proxy, one thread issues the MMAs and commits
// them to the mbarrier, one warp polls it while the others sleep in the group
// barrier, then everyone reads the accumulators back with tcgen05.ld for the
// fused bias + ReLU + split epilogue. The G groups interleave, so one's MMAs
// overlap another's epilogue.
//
// Mixed-family batches are partitioned first (nn_count / nn_scatter: a
// warp-aggregated counting partition of row ids per family), then one
// ensemble launch per installed family reads its range of the permutation.

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../../include/carma_gpu.h"
#include "common.cuh"
#include "../host/stage.hpp"
#include "rows.cuh"

namespace carma_b200 {
namespace {

constexpr int kTileRows = 128;
constexpr int kHidden = 64;           // 8 members x 8 neurons
constexpr int kK0 = 32;               // 19 features padded to two K=16 steps
constexpr uint32_t kATile = kTileRows * kHidden * 2; // 16 KB per activation part
constexpr int kSplit = 3;                             // bf16 parts per activation
constexpr int kMaxPasses = 8;
constexpr int kTmemCols = 512;
constexpr uint32_t kSmemLimit = 227 * 1024;

struct NnModelDev {
    const uint8_t* blob;  // shared-memory image: weights (canonical bf16), biases (fp32)
    uint32_t blob_bytes;  // multiple of 16
    uint32_t smem_blob;   // blob_bytes rounded up to 1024
    uint32_t depth;       // L: hidden layers (max over members)
    uint32_t members;     // E
    uint32_t classes;     // C
    uint32_t cp;          // C rounded up to 8: TMEM / head-row stride per member
    uint32_t mpp;         // members per head pass
    uint32_t passes;
    uint32_t pass_n[kMaxPasses];     // N of each head pass (multiple of 16)
    uint32_t pass_row0[kMaxPasses];  // first head row of each pass
    uint32_t alive[CARMA_NN_MAX_DEPTH];      // members with depth > l (members sorted by depth, descending)
    uint32_t layer_n[CARMA_NN_MAX_DEPTH];    // MMA N of layer l (alive columns, padded to 16)
    uint32_t layer_k[CARMA_NN_MAX_DEPTH];    // K steps (16) of layer l
    uint32_t layer_off[CARMA_NN_MAX_DEPTH];  // byte offset of W_l in the blob (SBO = 16 * K_l)
    uint8_t orig[CARMA_NN_MAX_MEMBERS];      // spec member index of sorted member m
    uint32_t arch;                           // CARMA_NN_ARCH_*
    uint32_t tf_off[CARMA_NN_MAX_MEMBERS];   // transformer: float offset of member e's parameters
    uint8_t tf_d[CARMA_NN_MAX_MEMBERS];      // transformer: model width d
    uint8_t tf_layers[CARMA_NN_MAX_MEMBERS]; // transformer: encoder layers
    const float* fblob;   // MLP, CUDA-core path: fp32 padded image (see mlp_ffma)
    uint32_t fblob_bytes;
    uint32_t ff_off[CARMA_NN_MAX_MEMBERS];   // float offset of member e (spec order) in fblob
    uint8_t ff_depth[CARMA_NN_MAX_MEMBERS];  // hidden layers of member e
    uint32_t off_head;    // byte offset of the head weights in the blob
    uint32_t off_bias;    // byte offset of the fp32 biases (L x 64, then head rows)
    uint32_t log_mask;
    uint64_t bucket_range;
    float shift[kFeatureDims];
    float scale[kFeatureDims];
};

struct NnParams {
    // row source (rows.cuh)
    double act[16];
    uint64_t bbase[CARMA_BIT_FIELDS];
    uint16_t boff[CARMA_BIT_FIELDS];
    uint8_t bw[CARMA_BIT_FIELDS];
    uint32_t bwpr;
    const void* rows;
    const int8_t* family;
    int32_t default_family;
    // this launch
    NnModelDev m;
    int32_t fam;              // family of this launch
    const uint32_t* perm;     // row ids grouped by family (null: rows [0, n))
    const uint32_t* counts;   // per-family row counts (null: n rows)
    uint64_t n;
    int32_t* bucket;
    uint64_t* bytes;
    float* probs;   // q x CARMA_NN_MAX_CLASSES (nullable)
    float* logits;  // q x CARMA_NN_MAX_MEMBERS x CARMA_NN_MAX_CLASSES (nullable)
};

// ---------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, K-major, no swizzle (cute::UMMA::SmemDescriptor):
// start >> 4 at [0,14), leading (K core-matrix) byte offset >> 4 at [16,30),
// stride (8-row group) byte offset >> 4 at [32,46), version 1 at [46,48).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

// Instruction descriptor, kind::f16: fp32 accumulator, bf16 A and B, both
// K-major, N >> 3 at [17,23), M >> 4 at [24,29) (cute::UMMA::InstrDescriptor).
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((kTileRows >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(a), "r"(phase)
            : "memory");
    }
}

__device__ __forceinline__ void group_bar(int g);
__device__ __forceinline__ void fence_after();

// Completion of a group's MMAs: one warp polls the mbarrier, the others sleep
// in the group's hardware barrier (a polling warp per thread would take issue
// slots from the other groups' epilogues).
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t phase, bool waiter, int g) {
    if (waiter) mbar_wait(bar, phase);
    group_bar(g);
    fence_after();
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void group_bar(int g) { asm volatile("bar.sync %0, 256;" ::"r"(g + 1) : "memory"); }

// 32 lanes x 32 bit, 8 consecutive columns per thread, and the wait for
// them in the same asm statement: tcgen05.ld writes its registers
// asynchronously, so nothing (a register spill included) may read them
// before tcgen05.wait::ld — with the wait in a separate statement the
// compiler could spill a destination in between and reload a stale value.
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&r)[8]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(addr)
        : "memory");
}

// Upper 16 bits of a (low half) and of b (high half): the bf16 truncations
// of two fp32 values, packed, in one PRMT.
__device__ __forceinline__ uint32_t pack_hi16(float a, float b) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
    return r;
}

// Splits 8 consecutive activations into kSplit bf16 parts and stores part j
// at byte offset `off` of A tile j (tiles kATile bytes apart from `a`). Each
// part is the truncation of what is left (top 8 significant bits); the
// remainder x - trunc(x) is exact in fp32, so three parts hold all 24 bits of
// the fp32 value exactly. Integer moves only (PRMT, LOP, FADD), no
// conversion-pipe instructions.
__device__ __forceinline__ void store_split8(uint8_t* a, uint32_t off, const float (&h)[8]) {
    float rem[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) rem[i] = h[i];
#pragma unroll
    for (int j = 0; j < kSplit; ++j) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            w[i] = pack_hi16(rem[2 * i], rem[2 * i + 1]);
            if (j + 1 < kSplit) {
                rem[2 * i] = __fsub_rn(rem[2 * i], __uint_as_float(__float_as_uint(rem[2 * i]) & 0xffff0000u));
                rem[2 * i + 1] =
                    __fsub_rn(rem[2 * i + 1], __uint_as_float(__float_as_uint(rem[2 * i + 1]) & 0xffff0000u));
            }
        }
        *reinterpret_cast<uint4*>(a + j * kATile + off) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// Canonical K-major no-swizzle placement of (row r, K chunk kc) in a tile
// whose 8-row groups are `sbo` bytes apart: core matrices of 8 rows x 16 B.
__device__ __forceinline__ uint32_t a_off(int r, int kc, uint32_t sbo) {
    return static_cast<uint32_t>(r >> 3) * sbo + static_cast<uint32_t>(kc) * 128u + static_cast<uint32_t>(r & 7) * 16u;
}

// Issues the MMAs of one layer: D = sum_j A_j.B over `ksteps` K=16 steps.
__device__ __forceinline__ void issue_layer(uint32_t tmem_d, uint32_t a, uint32_t b, uint32_t b_sbo, int ksteps,
                                            uint32_t idesc) {
    for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t bd = sdesc(b + ks * 256u, 128u, b_sbo);
#pragma unroll
        for (int j = 0; j < kSplit; ++j)
            mma_bf16(tmem_d, sdesc(a + j * kATile + ks * 256u, 128u, 1024u), bd, idesc, (ks | j) ? 1u : 0u);
    }
}

// ------------------------------------------------------------- the ensemble

// z for the 8 features of K chunk kc (zeros past feature 18).
template <int KC, class P>
__device__ __forceinline__ void transform_chunk(const P& p, const double (&raw)[kFeatureDims], float (&z)[8]) {
    const NnModelDev& m = p.m;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        constexpr int d0 = KC * 8;
        const int d = d0 + j;
        if (d < kFeatureDims) {
            const float x = __double2float_rn(raw[d]);
            const float t = ((m.log_mask >> d) & 1u) ? log1pf(fmaxf(x, 0.f)) : x;
            z[j] = __fmul_rn(__fsub_rn(t, m.shift[d]), m.scale[d]);
        } else {
            z[j] = 0.f;
        }
    }
}

// tcgen05.st reads its source registers asynchronously: the wait::st sits in
// the same asm statement so the registers cannot be reused before it.
__device__ __forceinline__ void tmem_st8(uint32_t addr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n\t"
                 "tcgen05.wait::st.sync.aligned;" ::"r"(addr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}

// One warpgroup pair per 128-row tile: 256 threads, thread (half h, row r).
// Both halves' warps w and w + 4 reach the same TMEM lanes (32 (w % 4) ..),
// so they split the columns: half h owns hidden columns 32h..32h+31 (members
// 4h..4h+3), every other member of the head, and K chunks {0, 3} / {1, 2} of
// the input features. Twice the warps per tile of a one-thread-per-row split,
// with the same shared memory and TMEM.
template <int FMT, int G, int CP, bool DIAG>
__global__ void __launch_bounds__(G * 256, 1) nn_ensemble(const __grid_constant__ NnParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const NnModelDev& m = p.m;
    const int tid = threadIdx.x;
    const int g = tid >> 8;
    const int h = (tid >> 7) & 1;
    const int r = tid & 127;
    const int warp = tid >> 5;
    uint8_t* a_t = smem + m.smem_blob + g * (kSplit * kATile);  // this group's A tiles
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + m.smem_blob + G * (kSplit * kATile));
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + G);

    // The model image: weights in their canonical layouts, biases.
    {
        const uint4* src = reinterpret_cast<const uint4*>(m.blob);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (uint32_t i = tid; i < m.blob_bytes / 16; i += G * 256) dst[i] = __ldg(src + i);
        // A tiles start at zero: columns of absent members are read (times
        // zero weights) by the head and by K padding, and must be finite.
        uint4* at = reinterpret_cast<uint4*>(smem + m.smem_blob);
        for (uint32_t i = tid; i < G * (kSplit * kATile) / 16; i += G * 256) at[i] = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) {
        for (int i = 0; i < G; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + i)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot + static_cast<uint32_t>(g * 128);                // this group's columns
    const uint32_t tmem_row = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);  // this warp's lanes

    const float* bias = reinterpret_cast<const float*>(smem + m.off_bias);
    const float* head_bias = bias + m.depth * kHidden;
    const uint32_t s_a = smem_u32(a_t), s_blob = smem_u32(smem);

    uint64_t n = p.n, base = 0;
    if (p.counts) {
        n = p.counts[p.fam];
        for (int f = 0; f < p.fam; ++f) base += p.counts[f];
    }
    // rows already grouped by family (nn_count's flag): read them in place
    const bool grouped = !p.perm || p.counts[2 * (CARMA_FAMILIES + 1)] == 0;
    const uint64_t tiles = (n + kTileRows - 1) / kTileRows;
    uint32_t phase = 0;
    const bool issuer = tid == g * 256;
    const bool waiter = (tid >> 5) == g * 8;  // the issuer's warp

    for (uint64_t tile = static_cast<uint64_t>(blockIdx.x) * G + g; tile < tiles;
         tile += static_cast<uint64_t>(gridDim.x) * G) {
        const uint64_t i = tile * kTileRows + r;
        const bool valid = i < n;
        const uint64_t row = valid ? (grouped ? base + i : static_cast<uint64_t>(p.perm[base + i])) : 0;

        // ---- features -> z (fp32) -> layer-0 A tile (K 0..31): half 0 writes
        // chunks 0 and 3, half 1 chunks 1 and 2 (7 log1p features each)
        {
            double raw[kFeatureDims];
            if (valid) load_raw<FMT>(p, row, raw);
            else
#pragma unroll
                for (int d = 0; d < kFeatureDims; ++d) raw[d] = 0.0;
            float z[8];
            if (h == 0) {
                transform_chunk<0>(p, raw, z);
                if (!valid)
#pragma unroll
                    for (int j = 0; j < 8; ++j) z[j] = 0.f;
                store_split8(a_t, a_off(r, 0, 1024u), z);
#pragma unroll
                for (int j = 0; j < 8; ++j) z[j] = 0.f;
                store_split8(a_t, a_off(r, 3, 1024u), z);
            } else {
                transform_chunk<1>(p, raw, z);
                if (!valid)
#pragma unroll
                    for (int j = 0; j < 8; ++j) z[j] = 0.f;
                store_split8(a_t, a_off(r, 1, 1024u), z);
                transform_chunk<2>(p, raw, z);
                if (!valid)
#pragma unroll
                    for (int j = 0; j < 8; ++j) z[j] = 0.f;
                store_split8(a_t, a_off(r, 2, 1024u), z);
            }
        }
        fence_async_smem();
        fence_before();
        group_bar(g);
        if (issuer) {
            fence_after();
            issue_layer(tmem, s_a, s_blob + m.layer_off[0], 256u * m.layer_k[0], m.layer_k[0],
                        idesc_bf16(m.layer_n[0]));
            mma_commit(mbar + g);
        }
        mma_wait(mbar + g, phase, waiter, g);
        phase ^= 1u;

        // ---- hidden layers: epilogue of layer l-1 feeds the MMAs of layer l.
        // Half h owns members h, h + 2, h + 4, h + 6; only the members still
        // running (a prefix) are computed and stored — a finished member's
        // columns keep its last activations for the head.
        for (uint32_t l = 1; l <= m.depth; ++l) {
            const uint32_t alive = m.alive[l - 1];
            const float* b = bias + (l - 1) * kHidden;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                const int mem = 2 * c + h;
                if (mem >= static_cast<int>(alive)) break;
                uint32_t v[1][8];
                tmem_ld8(tmem_row + mem * 8, v[0]);
                const float4 b0 = reinterpret_cast<const float4*>(b + mem * 8)[0];
                const float4 b1 = reinterpret_cast<const float4*>(b + mem * 8)[1];
                const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                float x[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = fmaxf(__fadd_rn(__uint_as_float(v[0][j]), bb[j]), 0.f);
                store_split8(a_t, a_off(r, mem, 1024u), x);
            }
            fence_async_smem();
            fence_before();
            group_bar(g);
            if (l == m.depth) break;  // the head passes issue from the final activations
            if (issuer) {
                fence_after();
                issue_layer(tmem, s_a, s_blob + m.layer_off[l], 256u * m.layer_k[l], m.layer_k[l],
                            idesc_bf16(m.layer_n[l]));
                mma_commit(mbar + g);
            }
            mma_wait(mbar + g, phase, waiter, g);
            phase ^= 1u;
        }

        // ---- head passes: logits, softmax per member, partial means per half
        float pm[CP];
#pragma unroll
        for (int c = 0; c < CP; ++c) pm[c] = 0.f;
        for (uint32_t ps = 0; ps < m.passes; ++ps) {
            if (ps > 0) {  // every lane's reads of the previous pass precede its overwrite
                fence_before();
                group_bar(g);
            }
            if (issuer) {
                fence_after();
                issue_layer(tmem, s_a, s_blob + m.off_head + m.pass_row0[ps] * 128u, 1024u, kHidden / 16,
                            idesc_bf16(m.pass_n[ps]));
                mma_commit(mbar + g);
            }
            mma_wait(mbar + g, phase, waiter, g);
            phase ^= 1u;
            const uint32_t m0 = ps * m.mpp;
            const uint32_t m1 = min(m.members, m0 + m.mpp);
            for (uint32_t mem = m0 + h; mem < m1; mem += 2) {
                const uint32_t col = (mem - m0) * m.cp;
                uint32_t v[CP / 8][8];
#pragma unroll
                for (int c = 0; c < CP / 8; ++c) tmem_ld8(tmem_row + col + c * 8, v[c]);
                float lg[CP];
#pragma unroll
                for (int c = 0; c < CP; ++c) lg[c] = __uint_as_float(v[c / 8][c % 8]);
                const float* hb = head_bias + m.pass_row0[ps] + col;
                float mx = -INFINITY;
#pragma unroll
                for (int c = 0; c < CP; ++c) {
                    if (c < static_cast<int>(m.classes)) {
                        lg[c] = __fadd_rn(lg[c], hb[c]);
                        mx = fmaxf(mx, lg[c]);
                    }
                }
                if (DIAG && valid && p.logits) {
                    float* out = p.logits + (row * CARMA_NN_MAX_MEMBERS + m.orig[mem]) * CARMA_NN_MAX_CLASSES;
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        if (c < static_cast<int>(m.classes)) out[c] = lg[c];
                }
                float s = 0.f;
#pragma unroll
                for (int c = 0; c < CP; ++c) {
                    if (c < static_cast<int>(m.classes)) {
                        lg[c] = __expf(__fsub_rn(lg[c], mx));
                        s = __fadd_rn(s, lg[c]);
                    }
                }
                const float inv_s = __frcp_rn(s);
#pragma unroll
                for (int c = 0; c < CP; ++c)
                    if (c < static_cast<int>(m.classes)) pm[c] = __fadd_rn(pm[c], __fmul_rn(lg[c], inv_s));
            }
        }
        // ---- combine the halves through TMEM: half 1 parks its partial sums
        // in the group's first columns once every read of the head is done;
        // half 0 adds them (members in ascending order within each half).
        fence_before();
        group_bar(g);
        if (h == 1) {
#pragma unroll
            for (int c = 0; c < CP / 8; ++c) {
                float w[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) w[j] = pm[c * 8 + j];
                tmem_st8(tmem_row + c * 8, w);
            }
        }
        fence_before();
        group_bar(g);
        fence_after();
        if (h == 0) {
            uint32_t v[CP / 8][8];
#pragma unroll
            for (int c = 0; c < CP / 8; ++c) tmem_ld8(tmem_row + c * 8, v[c]);
            // The next tile's first MMA overwrites TMEM and the A tiles: its
            // fence_before + group barrier orders it after these reads.
            if (valid) {
                const float inv_e = 1.0f / static_cast<float>(m.members);
                int best = 0;
                float bv = -1.f;
#pragma unroll
                for (int c = 0; c < CP; ++c) {
                    if (c < static_cast<int>(m.classes)) {
                        pm[c] = __fmul_rn(__fadd_rn(pm[c], __uint_as_float(v[c / 8][c % 8])), inv_e);
                        if (pm[c] >= bv) {  // ties to the larger bin
                            bv = pm[c];
                            best = c;
                        }
                    }
                }
                p.bucket[row] = best;
                p.bytes[row] = static_cast<uint64_t>(best + 1) * m.bucket_range;
                if (DIAG && p.probs) {
                    float* out = p.probs + row * CARMA_NN_MAX_CLASSES;
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        if (c < static_cast<int>(m.classes)) out[c] = pm[c];
                }
            }
        }
    }

    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "n"(kTmemCols)
                     : "memory");
    }
}

// ------------------------------------------------- the Transformer ensemble

// LayerNorm over D values (biased variance, eps 1e-5), in place.
template <int D>
__device__ __forceinline__ void layer_norm(float (&x)[D], const float* g, const float* b) {
    float mu = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) mu += x[i];
    mu *= 1.0f / D;
    float var = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) var = __fmaf_rn(x[i] - mu, x[i] - mu, var);
    const float inv = rsqrtf(__fmaf_rn(var, 1.0f / D, 1e-5f));
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = __fmaf_rn((x[i] - mu) * inv, g[i], b[i]);
}

// One member's logits for one row: the tokens are z[9..17], the auxiliary
// features z[0..8], z[18]; w points at the member's parameters in shared
// memory (layout in carma_gpu.h). The keys and values of all three tokens
// are formed first; then each token's query, attention, residual, LayerNorm
// and feed-forward update its own row of e in place. lg: this thread's
// logits, strided by the block size in shared memory.
template <int D>
__device__ __noinline__ void tf_member(const float* w, int layers, int classes, const float (&z)[kFeatureDims],
                                       float* lg, int lstride) {
    float e[3][D];
    const float* W = w;
    const float* pos = w + 4 * D;
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int i = 0; i < D; ++i) {
            float a = W[3 * D + i];
#pragma unroll
            for (int j = 0; j < 3; ++j) a = __fmaf_rn(W[i * 3 + j], z[9 + 3 * t + j], a);
            e[t][i] = fmaxf(a, 0.f) + pos[t * D + i];
        }
    const float* p = w + 7 * D;
    const float rs = rsqrtf(static_cast<float>(D));
#pragma unroll 1
    for (int l = 0; l < layers; ++l) {
        const float *Wq = p, *bq = p + D * D, *Wk = bq + D, *bk = Wk + D * D, *Wv = bk + D, *bv = Wv + D * D;
        const float *Wo = bv + D, *bo = Wo + D * D, *g1 = bo + D, *c1 = g1 + D, *W1 = c1 + D, *b1 = W1 + 4 * D;
        const float *W2 = b1 + 4, *b2 = W2 + 4 * D, *g2 = b2 + D, *c2 = g2 + D;
        p = c2 + D;
        float k[3][D], v[3][D];
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int i = 0; i < D; ++i) {
                float ak = bk[i], av = bv[i];
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    ak = __fmaf_rn(Wk[i * D + j], e[t][j], ak);
                    av = __fmaf_rn(Wv[i * D + j], e[t][j], av);
                }
                k[t][i] = ak;
                v[t][i] = av;
            }
#pragma unroll 1
        for (int t = 0; t < 3; ++t) {
            float et[D];  // e[t] by selects: no dynamically indexed (local-memory) arrays
#pragma unroll
            for (int i = 0; i < D; ++i) et[i] = t == 0 ? e[0][i] : (t == 1 ? e[1][i] : e[2][i]);
            float q[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                float a = bq[i];
#pragma unroll
                for (int j = 0; j < D; ++j) a = __fmaf_rn(Wq[i * D + j], et[j], a);
                q[i] = a;
            }
            float sc[3];
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                float a = 0.f;
#pragma unroll
                for (int j = 0; j < D; ++j) a = __fmaf_rn(q[j], k[u][j], a);
                sc[u] = a * rs;
            }
            const float mx = fmaxf(sc[0], fmaxf(sc[1], sc[2]));
            float ssum = 0.f;
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                sc[u] = __expf(sc[u] - mx);
                ssum += sc[u];
            }
            const float inv = __frcp_rn(ssum);
            float o[D];
#pragma unroll
            for (int j = 0; j < D; ++j) o[j] = (sc[0] * v[0][j] + sc[1] * v[1][j] + sc[2] * v[2][j]) * inv;
            float x[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                float a = bo[i];
#pragma unroll
                for (int j = 0; j < D; ++j) a = __fmaf_rn(Wo[i * D + j], o[j], a);
                x[i] = et[i] + a;
            }
            layer_norm<D>(x, g1, c1);
            float f[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                float a = b1[r];
#pragma unroll
                for (int j = 0; j < D; ++j) a = __fmaf_rn(W1[r * D + j], x[j], a);
                f[r] = fmaxf(a, 0.f);
            }
#pragma unroll
            for (int i = 0; i < D; ++i) {
                float a = b2[i];
#pragma unroll
                for (int r = 0; r < 4; ++r) a = __fmaf_rn(W2[i * 4 + r], f[r], a);
                x[i] += a;
            }
            layer_norm<D>(x, g2, c2);
#pragma unroll
            for (int i = 0; i < D; ++i) {  // other tokens need only k, v
                if (t == 0) e[0][i] = x[i];
                else if (t == 1) e[1][i] = x[i];
                else e[2][i] = x[i];
            }
        }
    }
    // head: relu(H1 [mean(e); aux] + b) -> H2 . + b
    float in[D + 10];
#pragma unroll
    for (int i = 0; i < D; ++i) in[i] = (e[0][i] + e[1][i] + e[2][i]) * (1.0f / 3.0f);
#pragma unroll
    for (int j = 0; j < 9; ++j) in[D + j] = z[j];
    in[D + 9] = z[18];
    const float *H1 = p, *h1 = H1 + 8 * (D + 10), *H2 = h1 + 8, *h2 = H2 + 8 * classes;
    float hh[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        float a = h1[r];
#pragma unroll
        for (int j = 0; j < D + 10; ++j) a = __fmaf_rn(H1[r * (D + 10) + j], in[j], a);
        hh[r] = fmaxf(a, 0.f);
    }
#pragma unroll 1
    for (int c = 0; c < classes; ++c) {
        float a = h2[c];
#pragma unroll
        for (int r = 0; r < 8; ++r) a = __fmaf_rn(H2[c * 8 + r], hh[r], a);
        lg[c * lstride] = a;
    }
}

// Thread per row: the attention is over three tokens of width d <= 8 (a
// 3 x 3 score matrix per row), far below any tensor-core tile, so the
// Transformer ensemble runs on the FMA pipes from registers, its parameters
// (~10 KB per family) broadcast from shared memory.
template <int FMT, int CP, bool DIAG>
__global__ void __launch_bounds__(128, 2) tf_ensemble(const __grid_constant__ NnParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const NnModelDev& m = p.m;
    {
        const uint4* src = reinterpret_cast<const uint4*>(m.blob);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (uint32_t i = threadIdx.x; i < m.blob_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const float* wts = reinterpret_cast<const float*>(smem);
    float* lg = reinterpret_cast<float*>(smem + m.blob_bytes) + threadIdx.x;  // [class][thread]
    const int ls = blockDim.x;
    uint64_t n = p.n, base = 0;
    if (p.counts) {
        n = p.counts[p.fam];
        for (int f = 0; f < p.fam; ++f) base += p.counts[f];
    }
    // rows already grouped by family (nn_count's flag): read them in place
    const bool grouped = !p.perm || p.counts[2 * (CARMA_FAMILIES + 1)] == 0;
    const int C = static_cast<int>(m.classes);
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t row = grouped ? base + i : static_cast<uint64_t>(p.perm[base + i]);
        double raw[kFeatureDims];
        load_raw<FMT>(p, row, raw);
        float z[kFeatureDims];
#pragma unroll
        for (int d = 0; d < kFeatureDims; ++d) {
            const float x = __double2float_rn(raw[d]);
            const float t = ((m.log_mask >> d) & 1u) ? log1pf(fmaxf(x, 0.f)) : x;
            z[d] = __fmul_rn(__fsub_rn(t, m.shift[d]), m.scale[d]);
        }
        float pm[CP];
#pragma unroll
        for (int c = 0; c < CP; ++c) pm[c] = 0.f;
#pragma unroll 1
        for (uint32_t mem = 0; mem < m.members; ++mem) {
            const float* w = wts + m.tf_off[mem];
            const int d = m.tf_d[mem];
            if (d == 4) tf_member<4>(w, m.tf_layers[mem], C, z, lg, ls);
            else tf_member<6>(w, m.tf_layers[mem], C, z, lg, ls);
            if (DIAG && p.logits) {
                float* out = p.logits + (row * CARMA_NN_MAX_MEMBERS + mem) * CARMA_NN_MAX_CLASSES;
                for (int c = 0; c < C; ++c) out[c] = lg[c * ls];
            }
            float mx = -INFINITY;
            for (int c = 0; c < C; ++c) mx = fmaxf(mx, lg[c * ls]);
            float s = 0.f;
            for (int c = 0; c < C; ++c) {
                const float ex = __expf(lg[c * ls] - mx);
                lg[c * ls] = ex;
                s += ex;
            }
            const float inv = __frcp_rn(s);
#pragma unroll
            for (int c = 0; c < CP; ++c)
                if (c < C) pm[c] = __fmaf_rn(lg[c * ls], inv, pm[c]);
        }
        const float inv_e = 1.0f / static_cast<float>(m.members);
        int best = 0;
        float bv = -1.f;
#pragma unroll
        for (int c = 0; c < CP; ++c)
            if (c < C) {
                pm[c] *= inv_e;
                if (pm[c] >= bv) {  // ties to the larger bin
                    bv = pm[c];
                    best = c;
                }
            }
        p.bucket[row] = best;
        p.bytes[row] = static_cast<uint64_t>(best + 1) * m.bucket_range;
        if (DIAG && p.probs) {
            float* out = p.probs + row * CARMA_NN_MAX_CLASSES;
#pragma unroll
            for (int c = 0; c < CP; ++c)
                if (c < C) out[c] = pm[c];
        }
    }
}

// ------------------------------------------------ MLP ensemble, CUDA cores
//
// The same ensemble as nn_ensemble on the FMA pipes, thread per row (R rows
// per thread share every weight load). Each member's layers are tiny (<= 8
// neurons, K <= 19): as GEMMs they fill an M = 128 tensor-core tile only
// through block-diagonal padding and three bf16 activation parts (26.7x
// the useful flops, bench "neural" roofline), while here every useful FMA
// is one FFMA and the weights are warp-uniform broadcasts from shared memory
// (LDS.128: 4 weights per load, reused by the R rows). Arithmetic is fp32
// throughout (the bf16-valued weights of the model, fp32 activations), so
// logits are at least as close to the oracle as the tensor path's.
//
// fblob, per member (spec order), floats: W0 [8][20] (19 features + pad,
// rows past the layer width zero) and b0 [8]; layers l = 1..depth-1: W [8][8],
// b [8]; head W [C][8], b [C]. Zero rows give relu(0) = 0 activations,
// which zero columns of the next layer ignore.
constexpr int kFfIn = 20;
#ifndef NN_FFMA_ROWS
#define NN_FFMA_ROWS 2
#endif

// NN_FFMA_MINB > 0 caps the registers (A/B knob; uncapped measured fastest)
#ifndef NN_FFMA_MINB
#define NN_FFMA_MINB 0
#endif
#if NN_FFMA_MINB > 0
#define NN_FFMA_BOUNDS __launch_bounds__(128, NN_FFMA_MINB)
#else
#define NN_FFMA_BOUNDS __launch_bounds__(128)
#endif
template <int FMT, int R, int CP, bool DIAG>
__global__ void NN_FFMA_BOUNDS mlp_ffma(const __grid_constant__ NnParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const NnModelDev& m = p.m;
    {
        const uint4* src = reinterpret_cast<const uint4*>(m.fblob);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (uint32_t i = threadIdx.x; i < m.fblob_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const float* wts = reinterpret_cast<const float*>(smem);
    // CP > 8: logits spill to shared memory, [class][thread][r]
    float* lgs = reinterpret_cast<float*>(smem + m.fblob_bytes) + threadIdx.x * R;
    const int ls = blockDim.x * R;
    uint64_t n = p.n, base = 0;
    if (p.counts) {
        n = p.counts[p.fam];
        for (int f = 0; f < p.fam; ++f) base += p.counts[f];
    }
    const bool grouped = !p.perm || p.counts[2 * (CARMA_FAMILIES + 1)] == 0;
    const int C = static_cast<int>(m.classes);
    const uint64_t n_items = (n + R - 1) / R;
    for (uint64_t it = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; it < n_items;
         it += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t row[R];
        bool live[R];
        float z[R][kFeatureDims];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint64_t i = it * R + r;
            live[r] = i < n;
            const uint64_t ii = live[r] ? i : it * R;
            row[r] = grouped ? base + ii : static_cast<uint64_t>(p.perm[base + ii]);
            double raw[kFeatureDims];
            load_raw<FMT>(p, row[r], raw);
#pragma unroll
            for (int d = 0; d < kFeatureDims; ++d) {
                const float x = __double2float_rn(raw[d]);
                const float t = ((m.log_mask >> d) & 1u) ? log1pf(fmaxf(x, 0.f)) : x;
                z[r][d] = __fmul_rn(__fsub_rn(t, m.shift[d]), m.scale[d]);
            }
        }
        float pm[R][CP];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < CP; ++c) pm[r][c] = 0.f;
#pragma unroll 1
        for (uint32_t mem = 0; mem < m.members; ++mem) {
            const float* w = wts + m.ff_off[mem];
            float h[R][8];
#pragma unroll
            for (int o = 0; o < 8; ++o) {
                const float* wr = w + o * kFfIn;
                float a[R];
#pragma unroll
                for (int r = 0; r < R; ++r) a[r] = w[8 * kFfIn + o];
#pragma unroll
                for (int k4 = 0; k4 < kFfIn / 4; ++k4) {
                    const float4 v = *reinterpret_cast<const float4*>(wr + 4 * k4);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        a[r] = __fmaf_rn(v.x, z[r][4 * k4], a[r]);
                        a[r] = __fmaf_rn(v.y, z[r][4 * k4 + 1], a[r]);
                        a[r] = __fmaf_rn(v.z, z[r][4 * k4 + 2], a[r]);
                        if (4 * k4 + 3 < kFeatureDims) a[r] = __fmaf_rn(v.w, z[r][4 * k4 + 3], a[r]);
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) h[r][o] = fmaxf(a[r], 0.f);
            }
            w += 8 * kFfIn + 8;
            const int depth = m.ff_depth[mem];
#pragma unroll 1
            for (int l = 1; l < depth; ++l) {
                float g[R][8];
#pragma unroll
                for (int o = 0; o < 8; ++o) {
                    const float4 v0 = *reinterpret_cast<const float4*>(w + o * 8);
                    const float4 v1 = *reinterpret_cast<const float4*>(w + o * 8 + 4);
                    const float bo = w[64 + o];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        float a = __fmaf_rn(v0.x, h[r][0], bo);
                        a = __fmaf_rn(v0.y, h[r][1], a);
                        a = __fmaf_rn(v0.z, h[r][2], a);
                        a = __fmaf_rn(v0.w, h[r][3], a);
                        a = __fmaf_rn(v1.x, h[r][4], a);
                        a = __fmaf_rn(v1.y, h[r][5], a);
                        a = __fmaf_rn(v1.z, h[r][6], a);
                        a = __fmaf_rn(v1.w, h[r][7], a);
                        g[r][o] = fmaxf(a, 0.f);
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int o = 0; o < 8; ++o) h[r][o] = g[r][o];
                w += 72;
            }
            // head logits, softmax, running mean of the probabilities
            float lg[R][CP <= 8 ? CP : 1];
            float mx[R];
#pragma unroll
            for (int r = 0; r < R; ++r) mx[r] = -INFINITY;
            const float* hb = w + 8 * C;
#pragma unroll(CP <= 8 ? CP : 1)
            for (int c = 0; c < (CP <= 8 ? CP : C); ++c) {
                if (CP <= 8 && c >= C) break;
                const float4 v0 = *reinterpret_cast<const float4*>(w + c * 8);
                const float4 v1 = *reinterpret_cast<const float4*>(w + c * 8 + 4);
                const float bc = hb[c];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float a = __fmaf_rn(v0.x, h[r][0], bc);
                    a = __fmaf_rn(v0.y, h[r][1], a);
                    a = __fmaf_rn(v0.z, h[r][2], a);
                    a = __fmaf_rn(v0.w, h[r][3], a);
                    a = __fmaf_rn(v1.x, h[r][4], a);
                    a = __fmaf_rn(v1.y, h[r][5], a);
                    a = __fmaf_rn(v1.z, h[r][6], a);
                    a = __fmaf_rn(v1.w, h[r][7], a);
                    if constexpr (CP <= 8) lg[r][CP <= 8 ? c : 0] = a;
                    else lgs[c * ls + r] = a;
                    mx[r] = fmaxf(mx[r], a);
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (DIAG && p.logits && live[r]) {
                    float* out = p.logits + (row[r] * CARMA_NN_MAX_MEMBERS + mem) * CARMA_NN_MAX_CLASSES;
                    for (int c = 0; c < C; ++c) out[c] = CP <= 8 ? lg[r][CP <= 8 ? (c < CP ? c : 0) : 0] : lgs[c * ls + r];
                }
                float sum = 0.f;
                if constexpr (CP <= 8) {
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        if (c < C) {
                            lg[r][c] = __expf(lg[r][c] - mx[r]);
                            sum += lg[r][c];
                        }
                    const float inv = __frcp_rn(sum);
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        if (c < C) pm[r][c] = __fmaf_rn(lg[r][c], inv, pm[r][c]);
                } else {
                    for (int c = 0; c < C; ++c) {
                        const float ex = __expf(lgs[c * ls + r] - mx[r]);
                        lgs[c * ls + r] = ex;
                        sum += ex;
                    }
                    const float inv = __frcp_rn(sum);
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        if (c < C) pm[r][c] = __fmaf_rn(lgs[c * ls + r], inv, pm[r][c]);
                }
            }
        }
        const float inv_e = 1.0f / static_cast<float>(m.members);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!live[r]) continue;
            int best = 0;
            float bv = -1.f;
#pragma unroll
            for (int c = 0; c < CP; ++c)
                if (c < C) {
                    pm[r][c] *= inv_e;
                    if (pm[r][c] >= bv) {  // ties to the larger bin
                        bv = pm[r][c];
                        best = c;
                    }
                }
            p.bucket[row[r]] = best;
            p.bytes[row[r]] = static_cast<uint64_t>(best + 1) * m.bucket_range;
            if (DIAG && p.probs) {
                float* out = p.probs + row[r] * CARMA_NN_MAX_CLASSES;
#pragma unroll
                for (int c = 0; c < CP; ++c)
                    if (c < C) out[c] = pm[r][c];
            }
        }
    }
}

// ------------------------------------------------------ family partition

constexpr int kBins = CARMA_FAMILIES + 1;  // + rows without a model
constexpr int kUnsorted = 2 * kBins;        // counts[]: bins, cursors, then the "not grouped" flag

template <int FMT>
__device__ __forceinline__ int nn_bin(const NnParams& p, uint64_t i, uint32_t present) {
    const int f = row_family<FMT>(p, i);
    return (f >= 0 && f < CARMA_FAMILIES && ((present >> f) & 1u)) ? f : CARMA_FAMILIES;
}

template <int FMT>
__global__ void nn_count(const __grid_constant__ NnParams p, uint64_t q, uint32_t present, uint32_t* counts) {
    const unsigned lane = threadIdx.x & 31;
    uint32_t local[kBins] = {0, 0, 0, 0};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); i0 < q; i0 += stride) {
        const uint64_t i = i0 + lane;
        const int b = i < q ? nn_bin<FMT>(p, i, present) : -1;
#pragma unroll
        for (int k = 0; k < kBins; ++k) local[k] += __popc(__ballot_sync(0xffffffffu, b == k));
        // rows already grouped by family (non-decreasing bins)? else flag it
        const bool down = i < q && i > 0 && b < nn_bin<FMT>(p, i - 1, present);
        if (__any_sync(0xffffffffu, down) && lane == 0) atomicOr(counts + kUnsorted, 1u);
    }
    if (lane == 0)
        for (int k = 0; k < kBins; ++k)
            if (local[k]) atomicAdd(counts + k, local[k]);
}

// Row ids grouped by family. Positions are claimed per block (shared-memory
// counters, then one global atomic per family per block step): per-warp
// global atomics on two counters serialised at ~1M operations per 16.7M rows.
template <int FMT>
__global__ void __launch_bounds__(256) nn_scatter(const __grid_constant__ NnParams p, uint64_t q, uint32_t present,
                                                  const uint32_t* __restrict__ counts, uint32_t* __restrict__ cursor,
                                                  uint32_t* __restrict__ perm) {
    __shared__ uint32_t s_cnt[CARMA_FAMILIES], s_base[CARMA_FAMILIES];
    const unsigned lane = threadIdx.x & 31;
    if (counts[kUnsorted] == 0) {  // already grouped: row ids are positions, only mark rows without a model
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < q;
             i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
            if (nn_bin<FMT>(p, i, present) == CARMA_FAMILIES) {
                p.bucket[i] = -1;
                p.bytes[i] = UINT64_MAX;
            }
        return;
    }
    uint32_t off[kBins];
    off[0] = 0;
#pragma unroll
    for (int k = 1; k < kBins; ++k) off[k] = off[k - 1] + counts[k - 1];
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x; b0 < q; b0 += stride) {
        const uint64_t i = b0 + threadIdx.x;
        const int b = i < q ? nn_bin<FMT>(p, i, present) : -1;
        if (b == CARMA_FAMILIES) {  // FamilyMismatch -> no estimate (manager.cpp:99-105)
            p.bucket[i] = -1;
            p.bytes[i] = UINT64_MAX;
        }
        if (threadIdx.x < CARMA_FAMILIES) s_cnt[threadIdx.x] = 0;
        __syncthreads();
        uint32_t local = 0;
#pragma unroll
        for (int k = 0; k < CARMA_FAMILIES; ++k) {
            const unsigned mask = __ballot_sync(0xffffffffu, b == k);
            if (!mask) continue;
            uint32_t at = 0;
            if (lane == 0) at = atomicAdd(s_cnt + k, static_cast<uint32_t>(__popc(mask)));
            at = __shfl_sync(0xffffffffu, at, 0);
            if (b == k) local = at + __popc(mask & ((1u << lane) - 1u));
        }
        __syncthreads();
        if (threadIdx.x < CARMA_FAMILIES && s_cnt[threadIdx.x])
            s_base[threadIdx.x] = atomicAdd(cursor + threadIdx.x, s_cnt[threadIdx.x]);
        __syncthreads();
        if (b >= 0 && b < CARMA_FAMILIES) perm[off[b] + s_base[b] + local] = static_cast<uint32_t>(i);
        __syncthreads();  // s_cnt / s_base are reused by the next step
    }
}

__global__ void nn_mark_missing(uint64_t q, int32_t* bucket, uint64_t* bytes) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < q;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        bucket[i] = -1;
        bytes[i] = UINT64_MAX;
    }
}

// ----------------------------------------------------------------- host side

struct HostNn {
    bool present = false;
    carma_nn_spec spec{};
    NnModelDev dev{};
    DeviceBuffer blob;
    DeviceBuffer fblob;  // MLP: fp32 image of the CUDA-core path (mlp_ffma)
};

uint16_t bf16_bits(float x) {  // round to nearest even (finite inputs)
    uint32_t u;
    std::memcpy(&u, &x, 4);
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return static_cast<uint16_t>(u >> 16);
}

uint64_t tf_member_params(uint32_t d, uint32_t layers, uint32_t classes) {
    return 3ull * d + d + 3ull * d + layers * (4ull * d * d + 17ull * d + 4) + 8ull * (d + 10) + 8 + 8ull * classes +
           classes;
}

uint64_t param_count(const carma_nn_spec& s) {
    if (s.arch == CARMA_NN_ARCH_TRANSFORMER) {
        uint64_t n = 0;
        for (uint32_t e = 0; e < s.members && e < CARMA_NN_MAX_MEMBERS; ++e)
            n += tf_member_params(s.width[e][0], s.depth[e], s.classes);
        return n;
    }
    uint64_t n = 0;
    for (uint32_t e = 0; e < s.members; ++e) {
        uint32_t in = kFeatureDims;
        for (uint32_t l = 0; l < s.depth[e]; ++l) {
            n += static_cast<uint64_t>(s.width[e][l]) * in + s.width[e][l];
            in = s.width[e][l];
        }
        n += static_cast<uint64_t>(s.classes) * in + s.classes;
    }
    return n;
}

void validate(const carma_nn_spec& s) {
    if (s.members < 1 || s.members > CARMA_NN_MAX_MEMBERS) throw InvalidArg("members must be 1..8");
    if (s.classes < 2 || s.classes > CARMA_NN_MAX_CLASSES) throw InvalidArg("classes must be 2..48");
    if (s.bucket_range == 0) throw InvalidArg("bucket range must be > 0");
    if (s.arch > CARMA_NN_ARCH_TRANSFORMER) throw InvalidArg("unknown estimator architecture");
    if (s.arch == CARMA_NN_ARCH_TRANSFORMER) {
        for (uint32_t e = 0; e < s.members; ++e) {
            if (s.depth[e] < 1 || s.depth[e] > 4) throw InvalidArg("encoder layers must be 1..4");
            const uint32_t d = s.width[e][0];
            if (d != 4 && d != 6) throw InvalidArg("transformer width must be 4 or 6 (PAPER.md:440)");
        }
        if (s.log_mask >> kFeatureDims) throw InvalidArg("log_mask has bits past feature 18");
        return;
    }
    for (uint32_t e = 0; e < s.members; ++e) {
        if (s.depth[e] < 1 || s.depth[e] > CARMA_NN_MAX_DEPTH) throw InvalidArg("member depth must be 1..8");
        for (uint32_t l = 0; l < s.depth[e]; ++l)
            if (s.width[e][l] < 1 || s.width[e][l] > CARMA_NN_MAX_WIDTH) throw InvalidArg("layer width must be 1..8");
    }
    if (s.log_mask >> kFeatureDims) throw InvalidArg("log_mask has bits past feature 18");
}

// Position of element (row, k) of a [rows x K] bf16 operand in the canonical
// K-major no-swizzle layout with 8-row groups `sbo` bytes apart.
size_t canon(uint32_t row, uint32_t k, uint32_t sbo) {
    return static_cast<size_t>(row >> 3) * sbo + (k >> 3) * 128u + (row & 7u) * 16u + (k & 7u) * 2u;
}

// Builds the shared-memory image of a model. Members are sorted by depth
// (descending, stable), so the members still running at layer l are a prefix
// [0, alive_l): layer l is a block-diagonal GEMM over that prefix only
// (N = 8 alive_l, K = 8 alive_{l-1}, both padded to 16 with zero weights),
// and a member that has finished keeps its last activations in its A-tile
// columns, untouched, until the head reads all of them. Then the head passes
// and the fp32 biases.
void build_model_tf(HostNn& hm, int device, const carma_nn_spec& s, const float* params) {
    NnModelDev d{};
    d.arch = CARMA_NN_ARCH_TRANSFORMER;
    d.members = s.members;
    d.classes = s.classes;
    d.cp = (s.classes + 7u) & ~7u;
    d.log_mask = s.log_mask;
    d.bucket_range = s.bucket_range;
    std::memcpy(d.shift, s.shift, sizeof(d.shift));
    std::memcpy(d.scale, s.scale, sizeof(d.scale));
    uint64_t off = 0;
    for (uint32_t e = 0; e < s.members; ++e) {
        d.orig[e] = static_cast<uint8_t>(e);
        d.tf_off[e] = static_cast<uint32_t>(off);
        d.tf_d[e] = static_cast<uint8_t>(s.width[e][0]);
        d.tf_layers[e] = static_cast<uint8_t>(s.depth[e]);
        off += tf_member_params(s.width[e][0], s.depth[e], s.classes);
    }
    d.blob_bytes = static_cast<uint32_t>((off * 4 + 15) & ~15ull);
    d.smem_blob = d.blob_bytes;
    std::vector<uint8_t> blob(d.blob_bytes, 0);
    std::memcpy(blob.data(), params, off * 4);
    DeviceGuard gd(device);
    hm.blob.ensure(blob.size());
    CARMA_CUDA(cudaMemcpy(hm.blob.ptr, blob.data(), blob.size(), cudaMemcpyHostToDevice));
    d.blob = hm.blob.as<uint8_t>();
    hm.dev = d;
    hm.spec = s;
    hm.present = true;
}

void build_model(HostNn& hm, int device, const carma_nn_spec& s, const float* params) {
    if (s.arch == CARMA_NN_ARCH_TRANSFORMER) return build_model_tf(hm, device, s, params);
    const uint32_t E = s.members;
    uint32_t L = 0;
    for (uint32_t e = 0; e < E; ++e) L = std::max(L, s.depth[e]);
    // spec offsets of each member's parameters
    std::vector<const float*> mp(E);
    {
        const float* pp = params;
        for (uint32_t e = 0; e < E; ++e) {
            mp[e] = pp;
            uint32_t in = kFeatureDims;
            for (uint32_t l = 0; l < s.depth[e]; ++l) {
                pp += static_cast<size_t>(s.width[e][l]) * in + s.width[e][l];
                in = s.width[e][l];
            }
            pp += static_cast<size_t>(s.classes) * in + s.classes;
        }
    }
    std::vector<uint32_t> ord(E);
    for (uint32_t e = 0; e < E; ++e) ord[e] = e;
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return s.depth[a] > s.depth[b]; });

    const uint32_t cp = (s.classes + 7u) & ~7u;
    const uint32_t mpp = std::min<uint32_t>(E, 128u / cp);
    const uint32_t passes = (E + mpp - 1) / mpp;
    if (passes > static_cast<uint32_t>(kMaxPasses)) throw Unsupported("too many head passes");
    auto pad16 = [](uint32_t x) { return (x + 15u) & ~15u; };
    NnModelDev d{};
    d.depth = L;
    d.members = E;
    d.classes = s.classes;
    d.cp = cp;
    d.mpp = mpp;
    d.passes = passes;
    for (uint32_t i = 0; i < E; ++i) d.orig[i] = static_cast<uint8_t>(ord[i]);
    uint32_t off = 0;
    for (uint32_t l = 0; l < L; ++l) {
        uint32_t a = 0;
        for (uint32_t e = 0; e < E; ++e) a += s.depth[e] > l ? 1u : 0u;
        d.alive[l] = a;
        d.layer_n[l] = pad16(8 * a);
        const uint32_t k = l == 0 ? kK0 : pad16(8 * d.alive[l - 1]);
        d.layer_k[l] = k / 16;
        d.layer_off[l] = off;
        off += d.layer_n[l] * k * 2;
    }
    uint32_t head_rows = 0;
    for (uint32_t ps = 0; ps < passes; ++ps) {
        const uint32_t mems = std::min(mpp, E - ps * mpp);
        d.pass_row0[ps] = head_rows;
        d.pass_n[ps] = pad16(mems * cp);
        head_rows += d.pass_n[ps];
    }
    d.off_head = off;
    d.off_bias = d.off_head + head_rows * 128u;
    d.blob_bytes = (d.off_bias + 4u * (L * kHidden + head_rows) + 15u) & ~15u;
    d.smem_blob = (d.blob_bytes + 1023u) & ~1023u;
    d.log_mask = s.log_mask;
    d.bucket_range = s.bucket_range;
    std::memcpy(d.shift, s.shift, sizeof(d.shift));
    std::memcpy(d.scale, s.scale, sizeof(d.scale));

    std::vector<uint8_t> blob(d.blob_bytes, 0);
    auto put = [&](size_t o, float w) {
        const uint16_t b = bf16_bits(w);
        std::memcpy(blob.data() + o, &b, 2);
    };
    float* bias = reinterpret_cast<float*>(blob.data() + d.off_bias);
    for (uint32_t m = 0; m < E; ++m) {
        const uint32_t e = ord[m];
        const float* pp = mp[e];
        uint32_t in = kFeatureDims;
        for (uint32_t l = 0; l < s.depth[e]; ++l) {
            const uint32_t w = s.width[e][l];
            const uint32_t sbo = 16u * 16u * d.layer_k[l];  // 8 rows x (K_l * 2 B)
            for (uint32_t o = 0; o < w; ++o)
                for (uint32_t k = 0; k < in; ++k)
                    put(d.layer_off[l] + canon(8 * m + o, l == 0 ? k : 8 * m + k, sbo), pp[o * in + k]);
            pp += static_cast<size_t>(w) * in;
            for (uint32_t o = 0; o < w; ++o) bias[l * kHidden + 8 * m + o] = pp[o];
            pp += w;
            in = w;
        }
        const uint32_t ps = m / mpp, slot = m % mpp;
        const uint32_t row0 = d.pass_row0[ps] + slot * cp;
        for (uint32_t c = 0; c < s.classes; ++c)
            for (uint32_t k = 0; k < in; ++k) put(d.off_head + canon(row0 + c, 8 * m + k, 1024u), pp[c * in + k]);
        pp += static_cast<size_t>(s.classes) * in;
        for (uint32_t c = 0; c < s.classes; ++c) bias[L * kHidden + row0 + c] = pp[c];
    }
    // the CUDA-core path's image (mlp_ffma): per member in spec order, the
    // same bf16-valued weights as fp32, padded to 8 neurons
    std::vector<float> fb;
    for (uint32_t e = 0; e < E; ++e) {
        d.ff_off[e] = static_cast<uint32_t>(fb.size());
        d.ff_depth[e] = static_cast<uint8_t>(s.depth[e]);
        const float* pp = mp[e];
        uint32_t in = kFeatureDims;
        auto bfv = [](float x) {
            const uint32_t u = static_cast<uint32_t>(bf16_bits(x)) << 16;
            float f;
            std::memcpy(&f, &u, 4);
            return f;
        };
        for (uint32_t l = 0; l < s.depth[e]; ++l) {
            const uint32_t w = s.width[e][l], cols = l == 0 ? kFfIn : 8;
            const size_t o0 = fb.size();
            fb.resize(o0 + 8 * cols + 8, 0.f);
            for (uint32_t o = 0; o < w; ++o)
                for (uint32_t k = 0; k < in; ++k) fb[o0 + o * cols + k] = bfv(pp[o * in + k]);
            pp += static_cast<size_t>(w) * in;
            for (uint32_t o = 0; o < w; ++o) fb[o0 + 8 * cols + o] = pp[o];
            pp += w;
            in = w;
        }
        const size_t h0 = fb.size();
        fb.resize(h0 + 9ull * s.classes, 0.f);
        for (uint32_t c = 0; c < s.classes; ++c)
            for (uint32_t k = 0; k < in; ++k) fb[h0 + c * 8 + k] = bfv(pp[c * in + k]);
        pp += static_cast<size_t>(s.classes) * in;
        for (uint32_t c = 0; c < s.classes; ++c) fb[h0 + 8ull * s.classes + c] = pp[c];
        fb.resize((fb.size() + 3) & ~size_t{3}, 0.f);  // members 16-B aligned
    }
    d.fblob_bytes = static_cast<uint32_t>(fb.size() * 4);
    DeviceGuard gd(device);
    hm.blob.ensure(blob.size());
    CARMA_CUDA(cudaMemcpy(hm.blob.ptr, blob.data(), blob.size(), cudaMemcpyHostToDevice));
    hm.fblob.ensure(fb.size() * 4);
    CARMA_CUDA(cudaMemcpy(hm.fblob.ptr, fb.data(), fb.size() * 4, cudaMemcpyHostToDevice));
    d.blob = hm.blob.as<uint8_t>();
    d.fblob = hm.fblob.as<float>();
    hm.dev = d;
    hm.spec = s;
    hm.present = true;
}

}  // namespace

struct NnHandle {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t pipe[2] = {nullptr, nullptr};
    HostNn model[CARMA_FAMILIES];
    struct Scratch {
        DeviceBuffer rows, family, perm, counts, bucket, bytes;
        PinnedBuffer stage_rows, stage_family, stage_packed;
        cudaEvent_t staged = nullptr;  // the H2D copy out of stage_packed is done
    } scratch[2];
    double act[16] = {0};
    carma_bit_schema schema{};
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};  // call start, ensemble start, ensemble end
    bool timed = false;
    uint64_t last_launches = 0, last_mmas = 0;
    uint64_t last_h2d = 0;  // bytes copied host -> device by the last host-buffer call
    StreamFence fence;                 // last device-stream user of scratch[0]
    PinnedBuffer counts_host;          // family counts of the last device call
    cudaStream_t counts_stream = nullptr;
    bool counts_pending = false;
    int32_t path = 0;  // MLP ensembles: 0 auto (CUDA cores), 1 tcgen05, 2 CUDA cores
    std::mutex mu;
};

namespace {

int sm_count(int device) {
    static int cached[64] = {0};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    int n = 0;
    CARMA_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    if (device >= 0 && device < 64) cached[device] = n;
    return n;
}

NnParams base_params(const NnHandle& h) {
    NnParams p{};
    std::memcpy(p.act, h.act, sizeof(p.act));
    for (int f = 0; f < CARMA_BIT_FIELDS; ++f) {
        p.bbase[f] = h.schema.base[f];
        p.boff[f] = h.schema.offset[f];
        p.bw[f] = h.schema.width[f];
    }
    p.bwpr = h.schema.words_per_row;
    return p;
}

template <int FMT, int G, int CP, bool DIAG>
void launch_ensemble_t(const NnParams& p, int device, cudaStream_t s) {
    const size_t smem = p.m.smem_blob + G * (kSplit * kATile) + G * 8 + 16;
    if (smem > kSmemLimit) throw Unsupported("model too large for shared memory");
    static cudaError_t attr = cudaFuncSetAttribute(nn_ensemble<FMT, G, CP, DIAG>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(kSmemLimit));
    CARMA_CUDA(attr);
    nn_ensemble<FMT, G, CP, DIAG><<<sm_count(device), G * 256, smem, s>>>(p);
    CARMA_CUDA(cudaGetLastError());
}

// Warpgroups per CTA: as many 48-KB A-tile triples as fit beside the model
// (<= 4: TMEM holds 4 x 128 columns), and CP = 8 or 48 columns per member.
template <int FMT, int CP, bool DIAG>
void launch_tf_t(const NnParams& p, int device, cudaStream_t s) {
    const size_t smem = p.m.blob_bytes + 128u * CARMA_NN_MAX_CLASSES * 4u;  // + per-thread logits
    if (smem > kSmemLimit) throw Unsupported("model too large for shared memory");
    static cudaError_t attr = cudaFuncSetAttribute(tf_ensemble<FMT, CP, DIAG>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(kSmemLimit));
    CARMA_CUDA(attr);
    const uint64_t want = (p.counts ? 0 : (p.n + 127) / 128);
    const unsigned grid = static_cast<unsigned>(
        want ? std::min<uint64_t>(want, 8ull * sm_count(device)) : 8ull * sm_count(device));
    tf_ensemble<FMT, CP, DIAG><<<grid, 128, smem, s>>>(p);
    CARMA_CUDA(cudaGetLastError());
}

template <int FMT, int R, int CP, bool DIAG>
void launch_ffma_t(const NnParams& p, int device, cudaStream_t s) {
    const size_t smem = p.m.fblob_bytes + (CP > 8 ? 128u * R * CP * 4u : 0u);
    if (smem > kSmemLimit) throw Unsupported("model too large for shared memory");
    static cudaError_t attr = cudaFuncSetAttribute(mlp_ffma<FMT, R, CP, DIAG>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(kSmemLimit));
    CARMA_CUDA(attr);
    int per_sm = 1;
    CARMA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mlp_ffma<FMT, R, CP, DIAG>, 128, smem));
    const uint64_t cap = static_cast<uint64_t>(std::max(per_sm, 1)) * sm_count(device);
    const uint64_t want = p.counts ? cap : (p.n + 128ull * R - 1) / (128ull * R);
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
    mlp_ffma<FMT, R, CP, DIAG><<<grid, 128, smem, s>>>(p);
    CARMA_CUDA(cudaGetLastError());
}

template <int FMT, bool DIAG>
void launch_ensemble(const NnParams& p, int device, cudaStream_t s, int32_t path) {
    if (p.m.arch == CARMA_NN_ARCH_MLP && path != 1) {
        if (p.m.cp <= 8) launch_ffma_t<FMT, NN_FFMA_ROWS, 8, DIAG>(p, device, s);
        else launch_ffma_t<FMT, 1, 48, DIAG>(p, device, s);
        return;
    }
    if (p.m.arch == CARMA_NN_ARCH_TRANSFORMER) {
        if (p.m.cp <= 8) launch_tf_t<FMT, 8, DIAG>(p, device, s);
        else launch_tf_t<FMT, 48, DIAG>(p, device, s);
        return;
    }
    const uint32_t room = kSmemLimit - p.m.smem_blob - 64;
    const int g = static_cast<int>(std::min<uint32_t>(3, room / (kSplit * kATile)));
    if (g < 1) throw Unsupported("model too large for shared memory");
    if constexpr (DIAG) {
        // The diagnostic variants (probabilities / per-member logits out, for
        // the parity tests) run one group per CTA: full register budget, no
        // spills.
        if (p.m.cp <= 8) launch_ensemble_t<FMT, 1, 8, DIAG>(p, device, s);
        else launch_ensemble_t<FMT, 1, 48, DIAG>(p, device, s);
    } else if (p.m.cp <= 8) {
        if (g >= 3) launch_ensemble_t<FMT, 3, 8, DIAG>(p, device, s);
        else if (g == 2) launch_ensemble_t<FMT, 2, 8, DIAG>(p, device, s);
        else launch_ensemble_t<FMT, 1, 8, DIAG>(p, device, s);
    } else {
        // at most two groups: three 48-bin groups (85 registers per thread) spill
        if (g >= 2) launch_ensemble_t<FMT, 2, 48, DIAG>(p, device, s);
        else launch_ensemble_t<FMT, 1, 48, DIAG>(p, device, s);
    }
}

template <int FMT>
void dispatch_diag(bool diag, const NnParams& p, int device, cudaStream_t s, int32_t path) {
    if (diag) launch_ensemble<FMT, true>(p, device, s, path);
    else launch_ensemble<FMT, false>(p, device, s, path);
}

template <int FMT>
void launch_partition(const NnParams& p, uint64_t q, uint32_t present, uint32_t* counts, uint32_t* perm, int device,
                      cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((q + 255) / 256, 4ull * sm_count(device)));
    nn_count<FMT><<<grid, 256, 0, s>>>(p, q, present, counts);
    nn_scatter<FMT><<<grid, 256, 0, s>>>(p, q, present, counts, counts + kBins, perm);
    CARMA_CUDA(cudaGetLastError());
}

// One predict on device-resident rows. Returns the number of launches.
uint64_t run_predict(NnHandle& h, NnHandle::Scratch& sc, const void* rows, int32_t format, const int8_t* family,
                     int32_t default_family, uint64_t q, int32_t* bucket, uint64_t* bytes, float* probs,
                     float* logits, cudaStream_t s, const carma_bit_schema* bits = nullptr) {
    NnParams p = base_params(h);
    if (bits) {  // this call's bit-packed schema instead of the handle's
        for (int f = 0; f < CARMA_BIT_FIELDS; ++f) {
            p.bbase[f] = bits->base[f];
            p.boff[f] = bits->offset[f];
            p.bw[f] = bits->width[f];
        }
        p.bwpr = bits->words_per_row;
    }
    p.rows = rows;
    p.family = family;
    p.default_family = default_family;
    p.bucket = bucket;
    p.bytes = bytes;
    p.probs = probs;
    p.logits = logits;
    const bool diag = probs || logits;
    uint32_t present = 0;
    for (int f = 0; f < CARMA_FAMILIES; ++f)
        if (h.model[f].present) present |= 1u << f;
    const bool timed = h.timed && h.ev[0];
    if (timed) CARMA_CUDA(cudaEventRecord(h.ev[0], s));
    uint64_t launches = 0;
    const bool per_row = format == CARMA_ROWS_PACKED || format == CARMA_ROWS_BITPACKED || family;
    std::vector<int> fams;
    if (!per_row) {
        const bool ok = default_family >= 0 && default_family < CARMA_FAMILIES && ((present >> default_family) & 1u);
        if (!ok) {
            nn_mark_missing<<<grid_for(q, 256, 4u * sm_count(h.device)), 256, 0, s>>>(q, bucket, bytes);
            CARMA_CUDA(cudaGetLastError());
            if (timed) {
                CARMA_CUDA(cudaEventRecord(h.ev[1], s));
                CARMA_CUDA(cudaEventRecord(h.ev[2], s));
            }
            return 1;
        }
        p.n = q;
        fams.push_back(default_family);
    } else {
        if (q > 0xffffffffull) throw Unsupported("more than 2^32 rows in one device call");
        sc.counts.ensure((2 * kBins + 1) * sizeof(uint32_t));
        sc.perm.ensure(q * sizeof(uint32_t));
        CARMA_CUDA(cudaMemsetAsync(sc.counts.ptr, 0, (2 * kBins + 1) * sizeof(uint32_t), s));
        switch (format) {
            case CARMA_ROWS_PACKED:
                launch_partition<CARMA_ROWS_PACKED>(p, q, present, sc.counts.as<uint32_t>(), sc.perm.as<uint32_t>(), h.device, s);
                break;
            case CARMA_ROWS_BITPACKED:
                launch_partition<CARMA_ROWS_BITPACKED>(p, q, present, sc.counts.as<uint32_t>(), sc.perm.as<uint32_t>(), h.device, s);
                break;
            case CARMA_ROWS_SCALAR:
                launch_partition<CARMA_ROWS_SCALAR>(p, q, present, sc.counts.as<uint32_t>(), sc.perm.as<uint32_t>(), h.device, s);
                break;
            default:
                launch_partition<CARMA_ROWS_FEATURES>(p, q, present, sc.counts.as<uint32_t>(), sc.perm.as<uint32_t>(), h.device, s);
        }
        launches += 3;  // memset + count + scatter
        p.perm = sc.perm.as<uint32_t>();
        p.counts = sc.counts.as<uint32_t>();
        for (int f = 0; f < CARMA_FAMILIES; ++f)
            if ((present >> f) & 1u) fams.push_back(f);
    }
    if (timed) CARMA_CUDA(cudaEventRecord(h.ev[1], s));
    for (int f : fams) {
        p.fam = f;
        p.m = h.model[f].dev;
        switch (format) {
            case CARMA_ROWS_PACKED: dispatch_diag<CARMA_ROWS_PACKED>(diag, p, h.device, s, h.path); break;
            case CARMA_ROWS_BITPACKED: dispatch_diag<CARMA_ROWS_BITPACKED>(diag, p, h.device, s, h.path); break;
            case CARMA_ROWS_SCALAR: dispatch_diag<CARMA_ROWS_SCALAR>(diag, p, h.device, s, h.path); break;
            default: dispatch_diag<CARMA_ROWS_FEATURES>(diag, p, h.device, s, h.path);
        }
        ++launches;
    }
    if (timed) CARMA_CUDA(cudaEventRecord(h.ev[2], s));
    return launches;
}

// MMAs per 128-row tile of a model: the K steps of every layer and of the
// head passes (K = 64: 4 steps each), kSplit MMAs per step.
uint64_t mmas_per_tile(const NnModelDev& d, int32_t path) {
    if (d.arch == CARMA_NN_ARCH_MLP && path != 1) return 0;  // CUDA-core path
    if (d.arch == CARMA_NN_ARCH_TRANSFORMER) return 0;
    uint64_t steps = 4ull * d.passes;
    for (uint32_t l = 0; l < d.depth; ++l) steps += d.layer_k[l];
    return kSplit * steps;
}

void check_ready(NnHandle* h) {
    if (!h) throw InvalidArg("null handle");
    bool any = false;
    for (const auto& m : h->model) any = any || m.present;
    if (!any) throw InvalidArg("no model installed");
}

carma_status predict_host(carma_nn* hh, const void* rows, size_t row_bytes, int32_t format, const int8_t* family,
                          int32_t default_family, uint64_t q, int32_t* bucket_out, uint64_t* bytes_out,
                          size_t tail_bytes = 0) {
    return guarded([&] {
        NnHandle* h = reinterpret_cast<NnHandle*>(hh);
        check_ready(h);
        if (q == 0) return;
        if (!rows) throw InvalidArg("rows is null");
        std::lock_guard<std::mutex> lock(h->mu);
        DeviceGuard g(h->device);
        const uint64_t chunk = uint64_t{1} << 21;
        const uint64_t small = uint64_t{1} << 18;
        auto chunk_rows = [&](uint64_t c, uint64_t remaining) -> uint64_t {
            const uint64_t grow = std::min<uint64_t>(chunk, small << std::min<uint64_t>(c, 20));
            return std::min<uint64_t>(grow, std::max<uint64_t>(small, remaining / 2));
        };
        const bool rows_pinned = is_pinned(rows);
        const bool fam_pinned = !family || is_pinned(family);
        const bool out_pinned = (!bucket_out || is_pinned(bucket_out)) && (!bytes_out || is_pinned(bytes_out));
        h->timed = false;
        h->fence.host_wait();  // a device call may still use scratch[0]
        auto copy_out = [&](NnHandle::Scratch& sc, cudaStream_t s, uint64_t beg, uint64_t cnt) {
            if (bucket_out)
                CARMA_CUDA(cudaMemcpyAsync(bucket_out + beg, sc.bucket.ptr, cnt * 4, cudaMemcpyDeviceToHost, s));
            if (bytes_out)
                CARMA_CUDA(cudaMemcpyAsync(bytes_out + beg, sc.bytes.ptr, cnt * 8, cudaMemcpyDeviceToHost, s));
            if (!out_pinned) CARMA_CUDA(cudaStreamSynchronize(s));
        };
        // Feature rows travel re-encoded as 64-byte packed rows (stage.hpp);
        // CARMA_E2E_RAW=1 sends the 136-byte rows as they are.
        static const bool raw_env = std::getenv("CARMA_E2E_RAW") && std::atoi(std::getenv("CARMA_E2E_RAW")) != 0;
        const bool pack = format == CARMA_ROWS_FEATURES && !raw_env;
        if (pack) std::memcpy(h->act, canonical_act_table(), sizeof(h->act));
        uint64_t launches = 0, beg = 0, cnt = 0, h2d = 0;
        for (uint64_t c = 0; beg < q; ++c, beg += cnt) {
            NnHandle::Scratch& sc = h->scratch[c & 1];
            cudaStream_t s = h->pipe[c & 1];
            cnt = std::min<uint64_t>(chunk_rows(c, q - beg), q - beg);
            const uint64_t cap_rows = std::min<uint64_t>(chunk, q);
            if (pack && !raw_chunk(c, rows_pinned && fam_pinned)) {
                sc.stage_packed.ensure(cap_rows * sizeof(carma_feature_packed));
                sc.rows.ensure(cap_rows * row_bytes);
                sc.bucket.ensure(cap_rows * 4);
                sc.bytes.ensure(cap_rows * 8);
                if (!sc.staged) CARMA_CUDA(cudaEventCreateWithFlags(&sc.staged, cudaEventDisableTiming));
                CARMA_CUDA(cudaEventSynchronize(sc.staged));
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
                    launches += run_predict(*h, sc, sc.rows.ptr, CARMA_ROWS_BITPACKED, nullptr, default_family, cnt,
                                            sc.bucket.as<int32_t>(), sc.bytes.as<uint64_t>(), nullptr, nullptr, s,
                                            &compact_schema());
                    copy_out(sc, s, beg, cnt);
                    continue;
                }
                if (pack_rows_canonical(static_cast<const carma_feature_row*>(rows) + beg, family ? family + beg : nullptr,
                                        default_family, cnt, pk)) {
                    CARMA_CUDA(cudaMemcpyAsync(sc.rows.ptr, pk, cnt * sizeof(carma_feature_packed),
                                               cudaMemcpyHostToDevice, s));
                    h2d += cnt * sizeof(carma_feature_packed);
                    CARMA_CUDA(cudaEventRecord(sc.staged, s));
                    launches += run_predict(*h, sc, sc.rows.ptr, CARMA_ROWS_PACKED, nullptr, default_family, cnt,
                                            sc.bucket.as<int32_t>(), sc.bytes.as<uint64_t>(), nullptr, nullptr, s);
                    copy_out(sc, s, beg, cnt);
                    continue;
                }
            }
            const char* src = static_cast<const char*>(rows) + beg * row_bytes;
            sc.rows.ensure(cap_rows * row_bytes + tail_bytes);
            sc.bucket.ensure(cap_rows * 4);
            sc.bytes.ensure(cap_rows * 8);
            if (family) sc.family.ensure(cap_rows);
            if (!rows_pinned || !fam_pinned) {
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
            launches += run_predict(*h, sc, sc.rows.ptr, format, family ? sc.family.as<int8_t>() : nullptr,
                                    default_family, cnt, sc.bucket.as<int32_t>(), sc.bytes.as<uint64_t>(), nullptr,
                                    nullptr, s);
            copy_out(sc, s, beg, cnt);
        }
        CARMA_CUDA(cudaStreamSynchronize(h->pipe[0]));
        CARMA_CUDA(cudaStreamSynchronize(h->pipe[1]));
        h->last_launches = launches;
        h->last_h2d = h2d;
        h->last_mmas = 0;
        h->counts_pending = false;
    });
}

}  // namespace
}  // namespace carma_b200

using namespace carma_b200;

extern "C" {

uint64_t carma_nn_param_count(const carma_nn_spec* spec) { return spec ? param_count(*spec) : 0; }

carma_status carma_nn_create(int device, carma_nn** out) {
    return guarded([&] {
        if (!out) throw InvalidArg("out is null");
        require_device(device);
        DeviceGuard g(device);
        auto* h = new NnHandle();
        h->device = device;
        CARMA_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        CARMA_CUDA(cudaStreamCreateWithFlags(&h->pipe[0], cudaStreamNonBlocking));
        CARMA_CUDA(cudaStreamCreateWithFlags(&h->pipe[1], cudaStreamNonBlocking));
        for (auto& e : h->ev) CARMA_CUDA(cudaEventCreate(&e));
        *out = reinterpret_cast<carma_nn*>(h);
    });
}

carma_status carma_nn_destroy(carma_nn* hh) {
    return guarded([&] {
        NnHandle* h = reinterpret_cast<NnHandle*>(hh);
        if (!h) return;
        {
            DeviceGuard g(h->device);
            cudaDeviceSynchronize();
            for (auto& m : h->model) {
                m.blob.release();
                m.fblob.release();
            }
            h->counts_host.release();
            h->fence.destroy();
            for (auto& sc : h->scratch) {
                for (DeviceBuffer* b : {&sc.rows, &sc.family, &sc.perm, &sc.counts, &sc.bucket, &sc.bytes}) b->release();
                sc.stage_rows.release();
                sc.stage_family.release();
                sc.stage_packed.release();
                if (sc.staged) cudaEventDestroy(sc.staged);
            }
            for (auto e : h->ev)
                if (e) cudaEventDestroy(e);
            if (h->stream) cudaStreamDestroy(h->stream);
            for (auto s : h->pipe)
                if (s) cudaStreamDestroy(s);
        }
        delete h;
    });
}

carma_status carma_nn_set_model(carma_nn* hh, int32_t family, const carma_nn_spec* spec, const float* params,
                                uint64_t n_params) {
    return guarded([&] {
        NnHandle* h = reinterpret_cast<NnHandle*>(hh);
        if (!h || !spec || !params) throw InvalidArg("null argument");
        if (family < 0 || family >= CARMA_FAMILIES) throw InvalidArg("family out of range");
        validate(*spec);
        if (n_params != param_count(*spec)) throw InvalidArg("parameter count does not match the spec");
        for (uint64_t i = 0; i < n_params; ++i)
            if (!std::isfinite(params[i])) throw InvalidArg("non-finite parameter");
        std::lock_guard<std::mutex> lock(h->mu);
        DeviceGuard g(h->device);
        CARMA_CUDA(cudaDeviceSynchronize());  // a queued call may still read the old blob
        build_model(h->model[family], h->device, *spec, params);
    });
}

carma_status carma_nn_set_act_table(carma_nn* hh, const double* act_table) {
    return guarded([&] {
        NnHandle* h = reinterpret_cast<NnHandle*>(hh);
        if (!h || !act_table) throw InvalidArg("null argument");
        std::lock_guard<std::mutex> lock(h->mu);
        std::memcpy(h->act, act_table, sizeof(h->act));
    });
}

carma_status carma_nn_set_path(carma_nn* hh, int32_t path) {
    return guarded([&] {
        NnHandle* h = reinterpret_cast<NnHandle*>(hh);
        if (!h) throw InvalidArg("null handle");
        if (path < 0 || path > 2) throw InvalidArg("path must be 0 (auto), 1 (tcgen05) or 2 (CUDA cores)");
        std::lock_guard<std::mutex> lock(h->mu);
        h->path = path;
    });
}

carma_status carma_nn_set_bit_schema(carma_nn* hh, const carma_bit_schema* schema) {
    return guarded([&] {
        NnHandle* h = reinterpret_cast<NnHandle*>(hh);
        if (!h || !schema) throw InvalidArg("null argument");
        if (schema->words_per_row == 0) throw InvalidArg("schema has no words per row");
        for (int f = 0; f < CARMA_BIT_FIELDS; ++f)
            if (schema->width[f] > 48) throw InvalidArg("schema field wider than 48 bits");
        std::lock_guard<std::mutex> lock(h->mu);
        h->schema = *schema;
        std::memcpy(h->act, schema->act_table, sizeof(h->act));
    });
}

carma_status carma_nn_predict_device(carma_nn* hh, const void* rows, int32_t format, const int8_t* family,
                                     int32_t default_family, uint64_t q, int32_t* bucket_out, uint64_t* bytes_out,
                                     float* probs, float* logits, void* stream) {
    return guarded([&] {
        NnHandle* h = reinterpret_cast<NnHandle*>(hh);
        check_ready(h);
        if (q == 0) return;
        if (!rows || !bucket_out || !bytes_out) throw InvalidArg("null device buffer");
        if (format < CARMA_ROWS_FEATURES || format > CARMA_ROWS_BITPACKED) throw InvalidArg("unknown row format");
        std::lock_guard<std::mutex> lock(h->mu);
        DeviceGuard g(h->device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->stream;
        h->timed = true;
        NnHandle::Scratch& sc = h->scratch[0];
        h->fence.acquire(s);  // scratch[0] may be in use on another stream
        h->last_launches = run_predict(*h, sc, rows, format, family, default_family, q, bucket_out, bytes_out, probs,
                                       logits, s);
        h->fence.release(s);
        // MMA count of this call: from the family counts, read back (async,
        // into pinned memory) and summed by carma_nn_last_timing
        h->last_mmas = 0;
        h->counts_pending = false;
        const bool per_row = format == CARMA_ROWS_PACKED || format == CARMA_ROWS_BITPACKED || family;
        if (per_row) {
            h->counts_host.ensure(sizeof(uint32_t) * kBins);
            CARMA_CUDA(cudaMemcpyAsync(h->counts_host.ptr, sc.counts.ptr, sizeof(uint32_t) * kBins,
                                       cudaMemcpyDeviceToHost, s));
            h->counts_stream = s;
            h->counts_pending = true;
        } else if (default_family >= 0 && default_family < CARMA_FAMILIES && h->model[default_family].present) {
            h->last_mmas = (q + 127) / 128 * mmas_per_tile(h->model[default_family].dev, h->path);
        }
    });
}

carma_status carma_nn_predict(carma_nn* h, const carma_feature_row* rows, const int8_t* family,
                              int32_t default_family, uint64_t q, int32_t* bucket_out, uint64_t* bytes_out) {
    return predict_host(h, rows, sizeof(carma_feature_row), CARMA_ROWS_FEATURES, family, default_family, q,
                        bucket_out, bytes_out);
}

carma_status carma_nn_predict_bitpacked(carma_nn* hh, const uint32_t* words, const carma_bit_schema* schema,
                                        uint64_t q, int32_t* bucket_out, uint64_t* bytes_out) {
    const carma_status st = carma_nn_set_bit_schema(hh, schema);
    if (st != CARMA_OK) return st;
    return predict_host(hh, words, 4ull * schema->words_per_row, CARMA_ROWS_BITPACKED, nullptr, 0, q, bucket_out,
                        bytes_out, 8);
}

carma_status carma_nn_last_timing(carma_nn* hh, double* kernel_ms, double* call_ms, uint64_t* launches,
                                  uint64_t* mmas) {
    return guarded([&] {
        NnHandle* h = reinterpret_cast<NnHandle*>(hh);
        if (!h) throw InvalidArg("null handle");
        DeviceGuard g(h->device);
        float a = 0.f, b = 0.f;
        if (h->timed) {
            CARMA_CUDA(cudaEventSynchronize(h->ev[2]));
            CARMA_CUDA(cudaEventElapsedTime(&a, h->ev[1], h->ev[2]));
            CARMA_CUDA(cudaEventElapsedTime(&b, h->ev[0], h->ev[2]));
        }
        if (kernel_ms) *kernel_ms = a;
        if (call_ms) *call_ms = b;
        if (h->counts_pending) {
            CARMA_CUDA(cudaStreamSynchronize(h->counts_stream));
            const uint32_t* c = h->counts_host.as<uint32_t>();
            uint64_t n = 0;
            for (int f = 0; f < CARMA_FAMILIES; ++f)
                if (h->model[f].present) n += (c[f] + 127ull) / 128ull * mmas_per_tile(h->model[f].dev, h->path);
            h->last_mmas = n;
            h->counts_pending = false;
        }
        if (launches) *launches = h->last_launches;
        if (mmas) *mmas = h->last_mmas;
    });
}

}  // extern "C"

extern "C" carma_status carma_nn_last_h2d_bytes(carma_nn* hh, uint64_t* bytes) {
    return guarded([&] {
        const NnHandle* h = reinterpret_cast<const NnHandle*>(hh);
        if (!h || !bytes) throw InvalidArg("null argument");
        *bytes = h->last_h2d;
    });
}
