// Placement scoring shared by carma_pick_batch and the replay kernel:
// Manager::eligible_gpus + map_task (proj/src/manager.cpp:109-245); MIG
// instance choice (pick_instance) is made by the caller and enters as inst_ok.
//
// A group of `width` lanes (a whole warp in the replay, 2..32 lanes per
// decision in the batched kernel) scores one decision; lane l of the group
// owns GPUs l, l+width, ... (GPL per lane). Feasibility is a ballot, MAGM /
// LUG / MUG are (key, id) arg-reductions over butterfly shuffles, RR and
// exclusive are bit scans of the eligibility mask. The result is uniform
// across the group.
#pragma once

#include <cstdint>

#include "../../../include/carma_gpu.h"

namespace carma_b200 {

struct PickInput {
    uint64_t free_bytes;  // GpuDevice::total_free()
    double smact;         // windowed_smact(now, monitor_window)
    bool idle;            // no residents
    bool valid;           // g < gpu_count
    bool inst_ok;         // MIG: pick_instance found an instance (manager.cpp:176-187); else true
};

// Lane-local helpers over a `width`-lane group inside a warp.
__device__ __forceinline__ unsigned group_bits(unsigned ballot, unsigned base, unsigned width) {
    return width == 32 ? ballot : (ballot >> base) & ((1u << width) - 1u);
}

// Orderable 64-bit key of a double: same order as <, +0 == -0.
__device__ __forceinline__ uint64_t dkey(double x) {
    if (x == 0.0) x = 0.0;
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// The policy's sort key as "larger is better" (manager.cpp:217-224):
// MAGM total_free descending, LUG windowed SMACT ascending, MUG descending.
__device__ __forceinline__ uint64_t policy_key(int policy, const PickInput& in) {
    if (policy == CARMA_POLICY_MAGM) return in.free_bytes;
    const uint64_t k = dkey(in.smact);
    return policy == CARMA_POLICY_LUG ? ~k : k;
}

// (ka, ia) better than (kb, ib): key descending, id ascending — the borrow of
// the 96-bit subtraction (kb : ~ib) - (ka : ~ia), one carry chain.
__device__ __forceinline__ bool key_better(uint64_t ka, int ia, uint64_t kb, int ib) {
    uint32_t r;
    asm("{\n\t.reg .u32 t;\n\t"
        "sub.cc.u32 t, %2, %1;\n\t"
        "subc.cc.u32 t, %4, %3;\n\t"
        "subc.cc.u32 t, %6, %5;\n\t"
        "subc.u32 %0, 0, 0;\n\t}"
        : "=r"(r)
        : "r"(~static_cast<uint32_t>(ia)), "r"(~static_cast<uint32_t>(ib)), "r"(static_cast<uint32_t>(ka)),
          "r"(static_cast<uint32_t>(kb)), "r"(static_cast<uint32_t>(ka >> 32)), "r"(static_cast<uint32_t>(kb >> 32)));
    return r != 0;
}

// Arg-best of (key desc, id asc) over the lane's candidates, then across the
// group (stable_sort by key with ties to the lowest id). -1 when none.
template <int GPL>
__device__ __forceinline__ int arg_best(int policy, const PickInput (&in)[GPL], const bool (&cand)[GPL],
                                        unsigned lane_in_group, unsigned width) {
    uint64_t bk = 0;
    int bid = 0x7fffffff;  // sentinel: loses to every real candidate
#pragma unroll
    for (int j = 0; j < GPL; ++j) {
        const uint64_t k = policy_key(policy, in[j]);
        const int id = static_cast<int>(lane_in_group + j * width);
        if (cand[j] && key_better(k, id, bk, bid)) {
            bk = k;
            bid = id;
        }
    }
    if (GPL >= 2 && width == 32) {
        // whole-warp group over > 32 GPUs (the replay's large tiers; on the
        // throughput-bound small tiers the shuffles measured faster): three
        // 32-bit max reductions — key
        // high word, key low word among the leaders, then the smallest id
        // (as its complement) among those
        const bool has = bid != 0x7fffffff;
        if (!__any_sync(0xffffffffu, has)) return -1;
        const unsigned hi = static_cast<unsigned>(bk >> 32), lo = static_cast<unsigned>(bk);
        const unsigned m1 = __reduce_max_sync(0xffffffffu, has ? hi : 0u);
        const bool h1 = has && hi == m1;
        const unsigned m2 = __reduce_max_sync(0xffffffffu, h1 ? lo : 0u);
        const bool h2 = h1 && lo == m2;
        const unsigned m3 = __reduce_max_sync(0xffffffffu, h2 ? ~static_cast<unsigned>(bid) : 0u);
        return static_cast<int>(~m3);
    }
#pragma unroll 1
    for (unsigned off = 1; off < width; off <<= 1) {
        const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, off, width);
        const int oid = __shfl_xor_sync(0xffffffffu, bid, off, width);
        if (key_better(ok, oid, bk, bid)) {
            bk = ok;
            bid = oid;
        }
    }
    return bid == 0x7fffffff ? -1 : bid;
}

// One decision. policy is the effective policy (exclusive for recovery tasks).
// need_floor = max(min_free, min(estimate, capacity)) or min_free when no estimate.
// Returns the number of GPUs chosen (0 = defer) in out[0..1]; updates rr_cursor.
// Every shuffle/ballot is reached by all 32 lanes (groups of one warp may hold
// different decisions), so data-dependent work is gated by warp votes.
template <int GPL>
__device__ __forceinline__ int pick_gpus(const carma_replay_config& c, int policy, uint32_t want,
                                         uint64_t need_floor, const PickInput (&in)[GPL],
                                         unsigned lane_in_group, unsigned group_base, unsigned width,
                                         int& rr_cursor, int* out) {
    const int n = c.gpu_count;
    const bool rr_all = policy == CARMA_POLICY_RR && !c.rr_apply_preconditions;
    if constexpr (GPL > 2) {
        // > 64 GPUs (the replay's many-GPU tier: one decision per warp, GPU
        // g = lane + 32 j): the eligibility set as one ballot word per j.
        bool el[GPL];
        unsigned mw[GPL];
        uint32_t total = 0;
#pragma unroll
        for (int j = 0; j < GPL; ++j) {
            bool e;
            if (!in[j].valid) e = false;
            else if (policy == CARMA_POLICY_EXCLUSIVE) e = in[j].idle;
            else if (rr_all) e = in[j].inst_ok;
            else e = in[j].inst_ok && !(in[j].smact > c.max_smact) && !(in[j].free_bytes < need_floor);
            el[j] = e;
            mw[j] = __ballot_sync(0xffffffffu, e);
            total += static_cast<uint32_t>(__popc(mw[j]));
        }
        // first eligible id >= from (-1 when none)
        auto next_from = [&](int from) {
            int res = -1;
#pragma unroll
            for (int j = GPL - 1; j >= 0; --j) {
                unsigned m = mw[j];
                if (j < (from >> 5)) m = 0u;
                else if (j == (from >> 5)) m &= ~0u << (from & 31);
                if (m) res = j * 32 + __ffs(m) - 1;
            }
            return res;
        };
        out[0] = out[1] = -1;
        const bool ok = total >= want;
        const bool sorted = policy == CARMA_POLICY_MAGM || policy == CARMA_POLICY_LUG || policy == CARMA_POLICY_MUG;
        if (!ok) return 0;
        // want <= CARMA_MAX_TASK_GPUS devices (the many-GPU tier's multi-GPU tasks)
        if (sorted) {  // stable sort by key then id == repeated arg-best
            bool cand[GPL];
#pragma unroll
            for (int j = 0; j < GPL; ++j) cand[j] = el[j];
            for (uint32_t r = 0; r < want; ++r) {
                const int g = arg_best<GPL>(policy, in, cand, lane_in_group, width);
                out[r] = g;
#pragma unroll
                for (int j = 0; j < GPL; ++j)
                    if (static_cast<int>(lane_in_group + j * width) == g) cand[j] = false;
            }
            return static_cast<int>(want);
        }
        if (policy == CARMA_POLICY_EXCLUSIVE) {  // the first idle devices in id order
            int bgn = 0;
            for (uint32_t r = 0; r < want; ++r) {
                out[r] = next_from(bgn);
                bgn = out[r] + 1;
            }
            return static_cast<int>(want);
        }
        // RR: cyclic scan from the cursor (manager.cpp:196-209)
        int from = rr_cursor;
        for (uint32_t r = 0; r < want; ++r) {
            int g = next_from(from);
            if (g < 0) g = next_from(0);
            out[r] = g;
            from = g + 1;
        }
        const int last = out[want - 1];
        rr_cursor = last + 1 == n ? 0 : last + 1;
        return static_cast<int>(want);
    }
    bool el[GPL];
    uint64_t mask = 0;
#pragma unroll
    for (int j = 0; j < GPL; ++j) {
        bool e;
        if (!in[j].valid) e = false;
        else if (policy == CARMA_POLICY_EXCLUSIVE) e = in[j].idle;
        else if (rr_all) e = in[j].inst_ok;
        else e = in[j].inst_ok && !(in[j].smact > c.max_smact) && !(in[j].free_bytes < need_floor);
        el[j] = e;
        const unsigned b = group_bits(__ballot_sync(0xffffffffu, e), group_base, width);
        mask |= static_cast<uint64_t>(b) << (j * width);
    }
    out[0] = out[1] = -1;
    const bool ok = static_cast<uint32_t>(__popcll(static_cast<long long>(mask))) >= want;
    const bool sorted = policy == CARMA_POLICY_MAGM || policy == CARMA_POLICY_LUG || policy == CARMA_POLICY_MUG;
    // MAGM / LUG / MUG: stable sort by key then id == repeated arg-best.
    int best0 = -1, best1 = -1;  // scalars: a dynamically indexed array would live in local memory
    const int rounds = __any_sync(0xffffffffu, ok && sorted && want > 1) ? 2
                       : (__any_sync(0xffffffffu, ok && sorted) ? 1 : 0);
    bool cand[GPL];
#pragma unroll
    for (int j = 0; j < GPL; ++j) cand[j] = el[j];
#pragma unroll 1
    for (int r = 0; r < rounds; ++r) {
        const int g = arg_best<GPL>(policy, in, cand, lane_in_group, width);
        if (r == 0) best0 = g;
        else best1 = g;
#pragma unroll
        for (int j = 0; j < GPL; ++j)
            if (static_cast<int>(lane_in_group + j * width) == g) cand[j] = false;
    }
    if (!ok) return 0;
    if (sorted) {
        out[0] = best0;
        if (want > 1) out[1] = best1;
        return static_cast<int>(want);
    }
    // want <= 2: out[] is written with constant indices (a dynamic index
    // would put the caller's array in local memory)
    if (policy == CARMA_POLICY_EXCLUSIVE) {
        uint64_t m = mask;
        out[0] = __ffsll(static_cast<long long>(m)) - 1;
        m &= m - 1;
        if (want > 1) out[1] = __ffsll(static_cast<long long>(m)) - 1;
        return static_cast<int>(want);
    }
    // RR: cyclic scan from the cursor (manager.cpp:196-209): rotate the mask
    // so the scan order becomes ascending bit order.
    const int cur = rr_cursor;
    const uint64_t nmask = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    uint64_t rot = cur == 0 ? mask : (((mask >> cur) | (mask << (n - cur))) & nmask);
    // b, cur < n: the wrap-around is one conditional subtraction
    const int b0 = __ffsll(static_cast<long long>(rot)) - 1 + cur;
    out[0] = b0 >= n ? b0 - n : b0;
    rot &= rot - 1;
    int last = out[0];
    if (want > 1) {
        const int b1 = __ffsll(static_cast<long long>(rot)) - 1 + cur;
        out[1] = b1 >= n ? b1 - n : b1;
        last = out[1];
    }
    rr_cursor = last + 1 == n ? 0 : last + 1;
    return static_cast<int>(want);
}

// One decision by one thread over its n (<= 16) GPU views (the batched
// scoring kernel for small servers: no shuffles, the views are staged in
// shared memory by the warp with coalesced loads). Same rules and tie
// breaks as pick_gpus: exclusive = first `want` idle GPUs; RR = cyclic scan
// from the cursor; MAGM/LUG/MUG = the `want` best keys, ties to the lower id.
__device__ __forceinline__ int pick_serial(const carma_replay_config& c, int policy, uint32_t want,
                                           uint64_t need_floor, const carma_gpu_view* v, int n, int& rr_cursor,
                                           int* out) {
    out[0] = out[1] = -1;
    const bool rr_all = policy == CARMA_POLICY_RR && !c.rr_apply_preconditions;
    uint32_t mask = 0;
#pragma unroll 1
    for (int g = 0; g < n; ++g) {
        bool e;
        if (policy == CARMA_POLICY_EXCLUSIVE) e = v[g].idle != 0;
        else if (rr_all) e = true;
        else e = !(v[g].windowed_smact > c.max_smact) && !(v[g].total_free < need_floor);
        mask |= (e ? 1u : 0u) << g;
    }
    if (static_cast<uint32_t>(__popc(mask)) < want) return 0;
    if (policy == CARMA_POLICY_EXCLUSIVE) {
        out[0] = __ffs(mask) - 1;
        if (want > 1) out[1] = __ffs(mask & (mask - 1)) - 1;
        return static_cast<int>(want);
    }
    if (policy == CARMA_POLICY_RR) {
        const int cur = rr_cursor;
        const uint32_t rot = cur == 0 ? mask : ((mask >> cur) | (mask << (n - cur))) & ((n >= 32 ? 0u : (1u << n)) - 1u);
        const int b0 = __ffs(rot) - 1 + cur;
        out[0] = b0 >= n ? b0 - n : b0;
        int last = out[0];
        if (want > 1) {
            const int b1 = __ffs(rot & (rot - 1)) - 1 + cur;
            out[1] = b1 >= n ? b1 - n : b1;
            last = out[1];
        }
        rr_cursor = last + 1 == n ? 0 : last + 1;
        return static_cast<int>(want);
    }
    // MAGM / LUG / MUG: stable sort by key, ties to the lower id == arg-best
    // (strictly better key wins; the scan is in id order).
    int best0 = -1, best1 = -1;
    uint64_t k0 = 0, k1 = 0;
#pragma unroll 1
    for (int g = 0; g < n; ++g) {
        if (!((mask >> g) & 1u)) continue;
        PickInput in;
        in.free_bytes = v[g].total_free;
        in.smact = v[g].windowed_smact;
        const uint64_t k = policy_key(policy, in);
        if (best0 < 0 || k > k0) {
            best1 = best0;
            k1 = k0;
            best0 = g;
            k0 = k;
        } else if (best1 < 0 || k > k1) {
            best1 = g;
            k1 = k;
        }
    }
    out[0] = best0;
    if (want > 1) out[1] = best1;
    return static_cast<int>(want);
}

}  // namespace carma_b200
