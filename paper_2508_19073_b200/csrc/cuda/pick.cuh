// Placement scoring shared by carma_pick_batch and the replay kernel:
// Manager::eligible_gpus + map_task (proj/src/manager.cpp:109-245), non-MIG.
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
};

// Lane-local helpers over a `width`-lane group inside a warp.
__device__ __forceinline__ unsigned group_bits(unsigned ballot, unsigned base, unsigned width) {
    return width == 32 ? ballot : (ballot >> base) & ((1u << width) - 1u);
}

// Argmax of (free desc, id asc) / argmin|argmax of (smact, id asc) over the
// lane's candidates, then across the group.
template <int GPL>
__device__ __forceinline__ int arg_best(int policy, const PickInput (&in)[GPL], const bool (&cand)[GPL],
                                        unsigned lane_in_group, unsigned width) {
    // best key per lane: (valid, value, id)
    bool have = false;
    uint64_t bf = 0;
    double bs = 0.0;
    int bid = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < GPL; ++j) {
        if (!cand[j]) continue;
        const int id = static_cast<int>(lane_in_group + j * width);
        bool better;
        if (!have) better = true;
        else if (policy == CARMA_POLICY_MAGM)
            better = in[j].free_bytes > bf || (in[j].free_bytes == bf && id < bid);
        else if (policy == CARMA_POLICY_LUG)
            better = in[j].smact < bs || (in[j].smact == bs && id < bid);
        else
            better = in[j].smact > bs || (in[j].smact == bs && id < bid);
        if (better) {
            have = true;
            bf = in[j].free_bytes;
            bs = in[j].smact;
            bid = id;
        }
    }
    for (unsigned off = 1; off < width; off <<= 1) {
        const bool oh = __shfl_xor_sync(0xffffffffu, have, off, width);
        const uint64_t of = __shfl_xor_sync(0xffffffffu, bf, off, width);
        const double os = __shfl_xor_sync(0xffffffffu, bs, off, width);
        const int oid = __shfl_xor_sync(0xffffffffu, bid, off, width);
        bool take;
        if (!oh) take = false;
        else if (!have) take = true;
        else if (policy == CARMA_POLICY_MAGM)
            take = of > bf || (of == bf && oid < bid);
        else if (policy == CARMA_POLICY_LUG)
            take = os < bs || (os == bs && oid < bid);
        else
            take = os > bs || (os == bs && oid < bid);
        if (take) {
            have = true;
            bf = of;
            bs = os;
            bid = oid;
        }
    }
    return have ? bid : -1;
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
    bool el[GPL];
    uint64_t mask = 0;
#pragma unroll
    for (int j = 0; j < GPL; ++j) {
        bool e;
        if (!in[j].valid) e = false;
        else if (policy == CARMA_POLICY_EXCLUSIVE) e = in[j].idle;
        else if (rr_all) e = true;
        else e = !(in[j].smact > c.max_smact) && !(in[j].free_bytes < need_floor);
        el[j] = e;
        const unsigned b = group_bits(__ballot_sync(0xffffffffu, e), group_base, width);
        mask |= static_cast<uint64_t>(b) << (j * width);
    }
    out[0] = out[1] = -1;
    const bool ok = static_cast<uint32_t>(__popcll(static_cast<long long>(mask))) >= want;
    const bool sorted = policy == CARMA_POLICY_MAGM || policy == CARMA_POLICY_LUG || policy == CARMA_POLICY_MUG;
    // MAGM / LUG / MUG: stable sort by key then id == repeated arg-best.
    int best[2] = {-1, -1};
    if (__any_sync(0xffffffffu, ok && sorted)) {
        bool cand[GPL];
#pragma unroll
        for (int j = 0; j < GPL; ++j) cand[j] = el[j];
        best[0] = arg_best<GPL>(policy, in, cand, lane_in_group, width);
        if (__any_sync(0xffffffffu, ok && sorted && want > 1)) {
#pragma unroll
            for (int j = 0; j < GPL; ++j)
                if (static_cast<int>(lane_in_group + j * width) == best[0]) cand[j] = false;
            best[1] = arg_best<GPL>(policy, in, cand, lane_in_group, width);
        }
    }
    if (!ok) return 0;
    if (sorted) {
        out[0] = best[0];
        if (want > 1) out[1] = best[1];
        return static_cast<int>(want);
    }
    if (policy == CARMA_POLICY_EXCLUSIVE) {
        uint64_t m = mask;
        for (uint32_t k = 0; k < want; ++k) {
            out[k] = __ffsll(static_cast<long long>(m)) - 1;
            m &= m - 1;
        }
        return static_cast<int>(want);
    }
    // RR: cyclic scan from the cursor (manager.cpp:196-209): rotate the mask
    // so the scan order becomes ascending bit order.
    const int cur = rr_cursor;
    const uint64_t nmask = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    uint64_t rot = cur == 0 ? mask : (((mask >> cur) | (mask << (n - cur))) & nmask);
    for (uint32_t k = 0; k < want; ++k) {
        const int b = __ffsll(static_cast<long long>(rot)) - 1;
        out[k] = (b + cur) % n;
        rot &= rot - 1;
    }
    rr_cursor = (out[want - 1] + 1) % n;
    return static_cast<int>(want);
}

}  // namespace carma_b200
