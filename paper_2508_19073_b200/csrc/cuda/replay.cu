// Stage 2 host side: replay plans (upload once, run many times), tier
// dispatch and the batched placement-scoring kernel. The replay kernel itself
// is in replay_kernel.cuh; the scoring device code in pick.cuh.

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../../include/carma_gpu.h"
#include "common.cuh"
#include "pick.cuh"
#include "replay_kernel.cuh"
#include "tracegen.cuh"

#ifndef REPLAY_SMALL_PLAN
#define REPLAY_SMALL_PLAN 64  // plans with at most this many jobs in a class use the large tier
#endif

namespace carma_b200 {
namespace {

// Batched carma_pick_batch: `width` lanes per decision.
template <int GPL>
__global__ void pick_kernel(carma_replay_config cf, const carma_gpu_view* __restrict__ views, uint32_t n_gpus,
                            const carma_pick_request* __restrict__ reqs, uint64_t n, int32_t* __restrict__ cursor,
                            int32_t* __restrict__ out, unsigned width) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned gib = lane / width, lig = lane % width;
    const unsigned groups_per_warp = 32 / width;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t w = warp; w * groups_per_warp < n; w += n_warps) {
        const uint64_t d = w * groups_per_warp + gib;
        const bool live = d < n;
        PickInput in[GPL];
#pragma unroll
        for (int j = 0; j < GPL; ++j) {
            const uint32_t g = lig + j * width;
            const bool valid = live && g < n_gpus;
            carma_gpu_view v{};
            if (valid) v = views[d * n_gpus + g];
            in[j].valid = valid;
            in[j].inst_ok = true;
            in[j].idle = v.idle != 0;
            in[j].free_bytes = v.total_free;
            in[j].smact = v.windowed_smact;
        }
        carma_pick_request rq{};
        int cur = 0;
        if (live) {
            rq = reqs[d];
            cur = cursor[d];
        }
        const int policy = rq.from_recovery ? CARMA_POLICY_EXCLUSIVE : cf.policy;
        uint64_t floor = cf.min_free;
        if (!rq.from_recovery && cf.policy != CARMA_POLICY_EXCLUSIVE && rq.estimate != CARMA_NO_ESTIMATE) {
            const uint64_t need = rq.estimate < cf.gpu_capacity ? rq.estimate : cf.gpu_capacity;
            if (need > floor) floor = need;
        }
        int ids[2];
        const uint32_t want = live ? rq.want : 1u;
        pick_gpus<GPL>(cf, policy, want, floor, in, lig, gib * width, width, cur, ids);
        if (live && lig == 0) {
            out[d * 2] = ids[0];
            out[d * 2 + 1] = ids[1];
            cursor[d] = cur;
        }
    }
}

// carma_pick_batch_wide: one decision per warp over up to 256 GPUs (8 per
// lane) and up to 8 GPUs per decision; out is n x 8.
__global__ void __launch_bounds__(128) pick_kernel_wide(carma_replay_config cf, const carma_gpu_view* __restrict__ views,
                                                        uint32_t n_gpus, const carma_pick_request* __restrict__ reqs,
                                                        uint64_t n, int32_t* __restrict__ cursor,
                                                        int32_t* __restrict__ out) {
    constexpr int GPL = CARMA_MAX_REPLAY_GPUS / 32;
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t d = warp; d < n; d += n_warps) {
        PickInput in[GPL];
#pragma unroll
        for (int j = 0; j < GPL; ++j) {
            const uint32_t g = lane + 32 * j;
            const bool valid = g < n_gpus;
            carma_gpu_view v{};
            if (valid) v = views[d * n_gpus + g];
            in[j].valid = valid;
            in[j].inst_ok = true;
            in[j].idle = v.idle != 0;
            in[j].free_bytes = v.total_free;
            in[j].smact = v.windowed_smact;
        }
        const carma_pick_request rq = reqs[d];
        int cur = cursor[d];
        const int policy = rq.from_recovery ? CARMA_POLICY_EXCLUSIVE : cf.policy;
        uint64_t floor = cf.min_free;
        if (!rq.from_recovery && cf.policy != CARMA_POLICY_EXCLUSIVE && rq.estimate != CARMA_NO_ESTIMATE) {
            const uint64_t need = rq.estimate < cf.gpu_capacity ? rq.estimate : cf.gpu_capacity;
            if (need > floor) floor = need;
        }
        int ids[CARMA_MAX_TASK_GPUS];
#pragma unroll
        for (int k = 0; k < CARMA_MAX_TASK_GPUS; ++k) ids[k] = -1;
        const int got = pick_gpus<GPL>(cf, policy, rq.want, floor, in, lane, 0, 32, cur, ids);
        if (lane < CARMA_MAX_TASK_GPUS) {
            int v = -1;
#pragma unroll
            for (int k = 0; k < CARMA_MAX_TASK_GPUS; ++k)
                if (static_cast<int>(lane) == k && k < got) v = ids[k];
            out[d * CARMA_MAX_TASK_GPUS + lane] = v;
        }
        if (lane == 0) cursor[d] = cur;
    }
}

// Batched carma_pick_batch for n_gpus <= 16: one thread per decision. Each
// warp streams its chunks of 32 decisions' views (32 * n_gpus * 24
// contiguous bytes) into shared memory with asynchronous 16-byte copies
// (LDGSTS), then every lane scores its own decision serially — no shuffles,
// so the kernel streams at HBM speed (a double-buffered variant was slower:
// the doubled shared memory cost more occupancy than the overlap gained).
constexpr int kPickWarps = 4;
constexpr int kPickMaxSerialGpus = 16;

__device__ __forceinline__ void pick_stage(carma_gpu_view* sv, const carma_gpu_view* src_views, uint32_t bytes,
                                           unsigned lane) {
    const char* src = reinterpret_cast<const char*>(src_views);
    if ((bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(sv));
        for (uint32_t i = lane * 16; i < bytes; i += 32 * 16)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + i), "l"(src + i) : "memory");
    } else {  // unaligned tail chunk: plain 8-byte loads
        const uint64_t* s8 = reinterpret_cast<const uint64_t*>(src);
        uint64_t* dst = reinterpret_cast<uint64_t*>(sv);
        for (uint32_t i = lane; i < bytes / 8; i += 32) dst[i] = __ldg(s8 + i);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(32 * kPickWarps) pick_kernel_thread(
    carma_replay_config cf, const carma_gpu_view* __restrict__ views, uint32_t n_gpus,
    const carma_pick_request* __restrict__ reqs, uint64_t n, int32_t* __restrict__ cursor,
    int32_t* __restrict__ out) {
    extern __shared__ __align__(16) char pick_smem[];
    const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    carma_gpu_view* sv = reinterpret_cast<carma_gpu_view*>(pick_smem) + static_cast<size_t>(wib) * 32 * n_gpus;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t base = warp * 32; base < n; base += n_warps * 32) {
        const uint32_t cnt = static_cast<uint32_t>(n - base < 32 ? n - base : 32);
        pick_stage(sv, views + base * n_gpus, cnt * n_gpus * static_cast<uint32_t>(sizeof(carma_gpu_view)), lane);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        if (lane < cnt) {
            const uint64_t d = base + lane;
            const carma_pick_request rq = reqs[d];
            int cur = cursor[d];
            const int policy = rq.from_recovery ? CARMA_POLICY_EXCLUSIVE : cf.policy;
            uint64_t floor = cf.min_free;
            if (!rq.from_recovery && cf.policy != CARMA_POLICY_EXCLUSIVE && rq.estimate != CARMA_NO_ESTIMATE) {
                const uint64_t need = rq.estimate < cf.gpu_capacity ? rq.estimate : cf.gpu_capacity;
                if (need > floor) floor = need;
            }
            int ids[2];
            pick_serial(cf, policy, rq.want, floor, sv + lane * n_gpus, static_cast<int>(n_gpus), cur, ids);
            reinterpret_cast<int2*>(out)[d] = make_int2(ids[0], ids[1]);
            cursor[d] = cur;
        }
        __syncwarp();
    }
}

__global__ void compact_outcomes(const carma_task_result* __restrict__ in, uint64_t n,
                                 carma_task_outcome* __restrict__ out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const carma_task_result r = in[i];
        carma_task_outcome o;
        o.final_dispatch = r.final_dispatch;
        o.complete = r.complete;
        o.ooms = r.ooms;
        o.attempts = r.attempts;
        out[i] = o;
    }
}

}  // namespace

// --------------------------------------------------------------- host side
struct ReplayPlan {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::vector<carma_replay_config> cfgs;
    std::vector<carma_replay_job> jobs;
    uint32_t n_traces = 0;
    uint64_t n_tasks = 0, n_task_out = 0, n_gpu_out = 0;
    int max_g = 1;
    int max_blocks = 1;
    // classes 3F + {light, heavy, global-only} for feature bits F (1 = MIG, 2 = timeline,
    // 4 = tasks requesting more than 2 GPUs)
    static constexpr int kClasses = 24;
    uint32_t class_count[kClasses] = {};
    int class_max_g[kClasses] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
    std::vector<uint32_t> trace_max_gpus;  // max gpus_requested per trace (host-built plans)
    std::vector<uint32_t> class_list;  // jobs ordered by class
    DeviceBuffer d_cfgs, d_tasks, d_trace_off, d_jobs, d_task_off, d_gpu_off, d_list, d_task_out,
        d_trace_out, d_gpu_out, d_inv, d_begin, d_counters, d_gstate, d_outcomes, d_tl, d_tl_count, d_log,
        d_log_count, d_entries;
    uint64_t tl_cap = 0, log_cap = 0;
    const uint64_t* est_override = nullptr;
    carma_task_outcome* outcome_sink = nullptr;  // device view of a pinned host buffer
    uint64_t launches = 0, retried = 0;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};  // run start, shared-memory tiers end, run end
    std::mutex mu;
};

namespace {

using replay::Layout;
// State capacities per tier, sized from the oracle's peak-state statistics
// over t90 seeds 1..3000 (oracle_replay_stats): MAGM / LUG / exclusive peak
// at <= 34 pending events and 8 residents; RR without preconditions stacks
// up to 34 residents (11 per GPU) and ~200 pending events (stale completion
// events stay queued: they are energy-integration breakpoints).
// F = feature bits (1 = MIG collocation, 2 = timeline ticks): those jobs run in
// their own kernel instantiations (classes 3F..3F+2); timeline jobs use the
// large and global tiers only.
template <int G, int F> using LightL = Layout<G, 64, 32, 16, 16, 16, 2, F>;
template <int G, int F> using HeavyL = Layout<G, 320, 64, 32, 16, 16, 2, F>;
// Large shared-memory tier for long traces on many GPUs (c5: 10^6 tasks on
// 64 GPUs peaks at 128 residents and ~215 pending events): one warp per CTA.
template <int F> using LargeL = Layout<64, 1024, 256, 32, 16, 128, 2, F>;
template <int F> using GlobalL = Layout<64, 8192, 2048, 256, 256, 4096, 4, F>;
// The same with 64 bitmap words per GPU (<= 4096 allocation blocks: e.g. a
// 192 GiB device at 512 MiB blocks, or 40 GiB at 16 MiB) for plans that
// hold such a config.
template <int F> using GlobalWideL = Layout<64, 8192, 2048, 256, 256, 4096, replay::kMaxWords, F>;
// Plans with more than 64 simulated GPUs: up to 256 GPUs (8 per lane) and
// up to 4096 blocks per GPU, global memory.
template <int F> using GlobalManyL = Layout<CARMA_MAX_REPLAY_GPUS, 8192, 2048, 256, 256, 4096, replay::kMaxWords, F>;
constexpr int kGlobalBlocks = 64 * 4;

// Configs the block bitmap cannot represent (GpuDevice is byte-granular).
bool needs_segments(const carma_replay_config& c) {
    return c.alloc_block == 0 || c.gpu_capacity % c.alloc_block != 0 ||
           c.gpu_capacity / c.alloc_block > 64ull * replay::kMaxWords;
}

// Configs whose policy can stack tasks without utilisation preconditions.
bool heavy_config(const carma_replay_config& c) {
    return (c.policy == CARMA_POLICY_RR && !c.rr_apply_preconditions) || c.max_smact >= 1.0 ||
           c.mode == CARMA_MODE_STREAMS;
}

void validate_config(const carma_replay_config& c) {
    if (c.mode != CARMA_MODE_MPS && c.mode != CARMA_MODE_STREAMS && c.mode != CARMA_MODE_MIG)
        throw InvalidArg("unknown collocation mode");
    if (c.policy < CARMA_POLICY_EXCLUSIVE || c.policy > CARMA_POLICY_MUG) throw InvalidArg("unknown policy");
    if (c.gpu_count < 1 || c.gpu_count > CARMA_MAX_REPLAY_GPUS) throw Unsupported("gpu_count must be in [1, 256]");
    if (!(c.monitor_window > 0.0)) throw InvalidArg("ConfigError: window must be > 0");
    // alloc_block = 0, capacities that are not a block multiple and more than
    // 4096 blocks run on the byte-granular segment allocator of the generic
    // instantiations (needs_segments); MIG instance tables stay block-based.
    // (MIG on a byte-granular device uses the byte instance table)
    if (!(c.sample_interval >= 0.0)) throw InvalidArg("ConfigError: sample_interval must be >= 0");
    if (c.log_flags & ~(CARMA_LOG_EVENTS | CARMA_LOG_DECISIONS)) throw InvalidArg("unknown log_flags bits");
    if (c.mode == CARMA_MODE_MIG) {
        // the table carma_mig_layout builds (gpu.cpp:29-51)
        if (c.mig_count < 1 || c.mig_count > CARMA_MAX_MIG)
            throw InvalidArg("ConfigError: MIG mode needs 1..8 instances (carma_mig_layout)");
        uint64_t end = 0, end_b = 0;
        const bool seg = needs_segments(c);
        for (int i = 0; i < c.mig_count; ++i) {
            if (!(c.mig_fraction[i] > 0.0) || c.mig_fraction[i] > 1.0)
                throw InvalidArg("ConfigError: mig instance fraction out of (0, 1]");
            if (c.mig_base_bytes[i] != end_b || (!seg && c.mig_base[i] != end))
                throw InvalidArg("ConfigError: MIG instances must tile the device in order (carma_mig_layout)");
            end += c.mig_blocks[i];
            end_b += c.mig_cap_bytes[i];
        }
        if (end_b > c.gpu_capacity || (!seg && end > c.gpu_capacity / c.alloc_block))
            throw InvalidArg("ConfigError: mig instances exceed capacity");
    }
}

template <class L, bool SMEM>
void launch(ReplayPlan& pl, replay::Params p, int sms, int warps_per_cta = 4) {
    auto kern = replay::replay_kernel<L, SMEM>;
    if (SMEM) {
        const size_t shmem = L::bytes * warps_per_cta;
        CARMA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(shmem)));
        int per_sm = 0;
        CARMA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps_per_cta, shmem));
        if (per_sm < 1) throw Unsupported("replay state does not fit in shared memory");
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(
            static_cast<uint64_t>(per_sm) * sms, (p.n_list + warps_per_cta - 1) / warps_per_cta));
        kern<<<grid, 32 * warps_per_cta, shmem, pl.stream>>>(p);
    } else {
        const unsigned warps = static_cast<unsigned>(std::min<uint64_t>(p.n_list, static_cast<uint64_t>(sms) * 2));
        const unsigned grid = (warps + 3) / 4;
        pl.d_gstate.ensure(static_cast<size_t>(grid) * 4 * L::bytes);
        p.gstate = pl.d_gstate.as<char>();
        kern<<<grid, 128, 0, pl.stream>>>(p);
    }
    CARMA_CUDA(cudaGetLastError());
    pl.launches++;
}

template <template <int, int> class LL, int F>
void launch_shared(ReplayPlan& pl, const replay::Params& p, int max_g, int sms) {
    if (max_g <= 4) launch<LL<4, F>, true>(pl, p, sms);
    else if (max_g <= 8) launch<LL<8, F>, true>(pl, p, sms);
    else if (max_g <= 16) launch<LL<16, F>, true>(pl, p, sms);
    else if (max_g <= 32) launch<LL<32, F>, true>(pl, p, sms);
    else launch<LL<64, F>, true>(pl, p, sms);
}

// tier 0 = light shared-memory layout, 1 = heavy shared-memory, 2 = global
// memory, 3 = large shared-memory (one warp per CTA)
template <int F>
void launch_tier(ReplayPlan& pl, const replay::Params& base, const uint32_t* list_dev, uint32_t n_list, int tier,
                 int max_g, uint32_t* counters, uint32_t* retry_base) {
    replay::Params p = base;
    p.job_list = list_dev;
    p.n_list = n_list;
    p.next_job = counters;         // [0]
    p.retry_count = counters + 1;  // [1]
    p.retry_list = retry_base;
    CARMA_CUDA(cudaMemsetAsync(counters, 0, 8, pl.stream));
    int sms = 148;
    CARMA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pl.device));
    if constexpr ((F & 4) != 0) {
        // multi-GPU tasks: the many-GPU global tier only (up to 8 GPUs per task)
        (void)tier;
        (void)max_g;
        launch<GlobalManyL<F>, false>(pl, p, sms);
    } else {
        if constexpr ((F & 2) == 0) {
            if (tier == 0) return launch_shared<LightL, F>(pl, p, max_g, sms);
            if (tier == 1) return launch_shared<HeavyL, F>(pl, p, max_g, sms);
        }
        if (tier == 3) launch<LargeL<F>, true>(pl, p, sms, 1);
        else if (pl.max_g > 64) launch<GlobalManyL<F>, false>(pl, p, sms);
        else if (pl.max_blocks > kGlobalBlocks) launch<GlobalWideL<F>, false>(pl, p, sms);
        else launch<GlobalL<F>, false>(pl, p, sms);
    }
}

// One collocation group (classes cb..cb+2, jobs list[off0, ...)): the two
// shared-memory classes, then overflowed and global-only jobs through the
// large shared-memory tier and the global-memory tier.
template <int F>
bool run_group(ReplayPlan& pl, const replay::Params& p, uint32_t off0) {
    constexpr int cb = 3 * F;
    uint32_t* list = pl.d_list.as<uint32_t>() + off0;
    uint32_t* retry = pl.d_list.as<uint32_t>() + pl.jobs.size() + off0;
    uint32_t* counters = pl.d_counters.as<uint32_t>() + 2 * cb;  // class c: {next, retries}
    uint32_t off = 0;
    for (int cls = 0; cls < 2; ++cls) {
        const uint32_t cnt = pl.class_count[cb + cls];
        // A handful of jobs cannot fill the GPU: the one-warp-per-CTA large
        // tier (no register cap) finishes each of them sooner.
        const int tier = (REPLAY_SMALL_PLAN > 0 && cnt <= REPLAY_SMALL_PLAN && pl.max_blocks <= 128) ? 3 : cls;
        if (cnt) launch_tier<F>(pl, p, list + off, cnt, tier, pl.class_max_g[cb + cls], counters + 2 * cls, retry + off);
        off += cnt;
    }
    if (F == 0) CARMA_CUDA(cudaEventRecord(pl.ev[1], pl.stream));
    uint32_t n_retry[4] = {0, 0, 0, 0};
    CARMA_CUDA(cudaMemcpyAsync(n_retry, counters, 16, cudaMemcpyDeviceToHost, pl.stream));
    CARMA_CUDA(cudaStreamSynchronize(pl.stream));
    const uint32_t c0 = pl.class_count[cb], c1 = pl.class_count[cb + 1];
    uint32_t total = (c0 ? n_retry[1] : 0) + (c1 ? n_retry[3] : 0);
    std::vector<uint32_t> ids(total);
    const uint32_t r0 = c0 ? n_retry[1] : 0;
    if (r0) CARMA_CUDA(cudaMemcpy(ids.data(), retry, r0 * 4, cudaMemcpyDeviceToHost));
    if (total > r0) CARMA_CUDA(cudaMemcpy(ids.data() + r0, retry + c0, (total - r0) * 4, cudaMemcpyDeviceToHost));
    // jobs that only fit the global tier
    const auto gb = pl.class_list.begin() + off0 + c0 + c1;
    ids.insert(ids.end(), gb, gb + pl.class_count[cb + 2]);
    pl.retried += total;  // jobs that overflowed a shared-memory tier
    total = static_cast<uint32_t>(ids.size());
    const bool list_dirty = total > 0;
    // Overflowed, global-only or begin-corrected jobs: the large shared-memory
    // tier first, then the global-memory tier (a begin correction can follow
    // an overflow, so up to three rounds).
    for (int round = 0; round < 3 && total > 0; ++round) {
        if (round > 0) pl.retried += total;
        CARMA_CUDA(cudaMemcpy(list, ids.data(), total * 4, cudaMemcpyHostToDevice));
        const bool large_ok = round == 0 && pl.max_blocks <= 128 && pl.max_g <= 64 && (F & 4) == 0;
        launch_tier<F>(pl, p, list, total, large_ok ? 3 : 2, pl.max_g, counters, retry);
        uint32_t nr = 0;
        CARMA_CUDA(cudaMemcpyAsync(&nr, counters + 1, 4, cudaMemcpyDeviceToHost, pl.stream));
        CARMA_CUDA(cudaStreamSynchronize(pl.stream));
        total = nr;
        ids.resize(total);
        if (total) CARMA_CUDA(cudaMemcpy(ids.data(), retry, total * 4, cudaMemcpyDeviceToHost));
    }
    return list_dirty;
}

void run_plan(ReplayPlan& pl) {
    replay::Params p{};
    p.cfgs = pl.d_cfgs.as<carma_replay_config>();
    p.tasks = pl.d_tasks.as<carma_task>();
    p.trace_off = pl.d_trace_off.as<uint64_t>();
    p.jobs = pl.d_jobs.as<carma_replay_job>();
    p.task_out_off = pl.d_task_off.as<uint64_t>();
    p.gpu_out_off = pl.d_gpu_off.as<uint64_t>();
    p.est_override = pl.est_override;
    p.task_out = pl.d_task_out.as<carma_task_result>();
    p.trace_out = pl.d_trace_out.as<carma_trace_result>();
    p.gpu_out = pl.d_gpu_out.as<carma_gpu_result>();
    p.inv_scratch = pl.d_inv.as<uint32_t>();
    p.smact_begin = pl.d_begin.as<double>();
    p.tl_out = pl.d_tl.as<carma_timeline_row>();
    p.tl_cap = pl.tl_cap;
    p.tl_count = pl.d_tl_count.as<uint64_t>();
    p.log_out = pl.d_log.as<carma_log_record>();
    p.log_cap = pl.log_cap;
    p.log_count = pl.d_log_count.as<uint64_t>();
    p.outcome_sink = pl.outcome_sink;
    const uint32_t n = static_cast<uint32_t>(pl.jobs.size());
    pl.launches = 0;
    pl.retried = 0;
    CARMA_CUDA(cudaMemsetAsync(pl.d_begin.ptr, 0xff, n * sizeof(double), pl.stream));  // NaN: derive
    CARMA_CUDA(cudaMemsetAsync(pl.d_counters.ptr, 0, 512, pl.stream));
    CARMA_CUDA(cudaEventRecord(pl.ev[0], pl.stream));
    uint32_t off[8];
    for (int f = 0, o = 0; f < 8; ++f) {
        off[f] = static_cast<uint32_t>(o);
        o += pl.class_count[3 * f] + pl.class_count[3 * f + 1] + pl.class_count[3 * f + 2];
    }
    auto count = [&](int f) { return pl.class_count[3 * f] + pl.class_count[3 * f + 1] + pl.class_count[3 * f + 2]; };
    bool dirty = false;
    if (count(0)) dirty |= run_group<0>(pl, p, off[0]);
    else CARMA_CUDA(cudaEventRecord(pl.ev[1], pl.stream));
    if (count(1)) dirty |= run_group<1>(pl, p, off[1]);
    if (count(2) || count(3) || count(6) || count(7)) {
        for (const auto& jb : pl.jobs) {
            const carma_replay_config& c = pl.cfgs[jb.config];
            if (c.sample_interval > 0.0 && pl.tl_cap == 0)
                throw InvalidArg("timeline jobs need carma_replay_plan_set_timeline_capacity first");
            if (c.log_flags != 0 && pl.log_cap == 0)
                throw InvalidArg("logging jobs need carma_replay_plan_set_log_capacity first");
        }
        if (count(2)) dirty |= run_group<2>(pl, p, off[2]);
        if (count(3)) dirty |= run_group<3>(pl, p, off[3]);
        if (count(6)) dirty |= run_group<6>(pl, p, off[6]);
        if (count(7)) dirty |= run_group<7>(pl, p, off[7]);
    }
    if (count(4)) dirty |= run_group<4>(pl, p, off[4]);
    if (count(5)) dirty |= run_group<5>(pl, p, off[5]);
    CARMA_CUDA(cudaEventRecord(pl.ev[2], pl.stream));
    if (dirty) CARMA_CUDA(cudaMemcpy(pl.d_list.ptr, pl.class_list.data(), n * 4, cudaMemcpyHostToDevice));
}

}  // namespace
}  // namespace carma_b200

namespace carma_b200 {
// Plan construction shared by carma_replay_plan_create (host tasks, validated
// and uploaded) and carma_replay_plan_create_generated (tasks == nullptr: the
// caller fills d_tasks on the device).
void build_plan(int device, const carma_replay_config* configs, uint32_t n_configs, const carma_task* tasks,
                const uint64_t* trace_offsets, uint32_t n_traces, const carma_replay_job* jobs, uint32_t n_jobs,
                carma_replay_plan** out) {
    {
        if (!out || !configs || !trace_offsets || !jobs) throw InvalidArg("null argument");
        if (n_configs == 0 || n_traces == 0 || n_jobs == 0) throw InvalidArg("empty plan");
        require_device(device);
        DeviceGuard guard(device);
        auto* pl = new ReplayPlan();
        try {
            pl->device = device;
            pl->cfgs.assign(configs, configs + n_configs);
            pl->jobs.assign(jobs, jobs + n_jobs);
            pl->n_traces = n_traces;
            pl->n_tasks = trace_offsets[n_traces];
            for (const auto& c : pl->cfgs) {
                validate_config(c);
                pl->max_g = std::max(pl->max_g, c.gpu_count);
                if (!needs_segments(c))
                    pl->max_blocks = std::max(pl->max_blocks, static_cast<int>(c.gpu_capacity / c.alloc_block));
            }
            for (uint32_t t = 0; t < n_traces; ++t) {
                if (trace_offsets[t + 1] <= trace_offsets[t]) throw InvalidArg("ConfigError: trace contains no tasks");
                if (trace_offsets[t + 1] - trace_offsets[t] > (1u << 30)) throw Unsupported("trace too long");
            }
            pl->trace_max_gpus.assign(n_traces, 1);
            for (uint32_t t = 0; tasks && t < n_traces; ++t)
                for (uint64_t i = trace_offsets[t]; i < trace_offsets[t + 1]; ++i)
                    pl->trace_max_gpus[t] = std::max(pl->trace_max_gpus[t], tasks[i].gpus);
            for (uint64_t i = 0; tasks && i < pl->n_tasks; ++i) {
                if (tasks[i].gpus < 1 || tasks[i].gpus > CARMA_MAX_TASK_GPUS)
                    throw Unsupported("gpus_requested must be in [1, 8]");
                if (i > 0 && tasks[i].submit < tasks[i - 1].submit) {
                    // arrivals must be non-decreasing within a trace (load_trace_file)
                    bool boundary = false;
                    for (uint32_t t = 0; t <= n_traces; ++t) boundary |= trace_offsets[t] == i;
                    if (!boundary) throw InvalidArg("MalformedTrace: submit times must be non-decreasing");
                }
            }
            std::vector<uint64_t> task_off(n_jobs), gpu_off(n_jobs);
            uint64_t to = 0, go = 0;
            for (uint32_t j = 0; j < n_jobs; ++j) {
                if (jobs[j].trace >= n_traces || jobs[j].config >= n_configs) throw InvalidArg("job index out of range");
                task_off[j] = to;
                gpu_off[j] = go;
                to += trace_offsets[jobs[j].trace + 1] - trace_offsets[jobs[j].trace];
                go += static_cast<uint64_t>(configs[jobs[j].config].gpu_count);
            }
            pl->n_task_out = to;
            pl->n_gpu_out = go;
            CARMA_CUDA(cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking));
            for (auto& e : pl->ev) CARMA_CUDA(cudaEventCreate(&e));
            auto up = [&](DeviceBuffer& b, const void* src, size_t bytes) {
                b.ensure(bytes);
                CARMA_CUDA(cudaMemcpy(b.ptr, src, bytes, cudaMemcpyHostToDevice));
            };
            up(pl->d_cfgs, configs, n_configs * sizeof(carma_replay_config));
            if (tasks) up(pl->d_tasks, tasks, pl->n_tasks * sizeof(carma_task));
            else pl->d_tasks.ensure(pl->n_tasks * sizeof(carma_task));
            up(pl->d_trace_off, trace_offsets, (n_traces + 1) * sizeof(uint64_t));
            up(pl->d_jobs, jobs, n_jobs * sizeof(carma_replay_job));
            up(pl->d_task_off, task_off.data(), n_jobs * sizeof(uint64_t));
            up(pl->d_gpu_off, gpu_off.data(), n_jobs * sizeof(uint64_t));
            std::vector<uint32_t> list(2 * static_cast<size_t>(n_jobs));
            for (int cls = 0; cls < ReplayPlan::kClasses; ++cls)
                for (uint32_t i = 0; i < n_jobs; ++i) {
                    const carma_replay_config& c = configs[jobs[i].config];
                    // > 128 allocation blocks: the shared-memory layouts hold 2 bitmap words;
                    // MIG / timeline jobs form classes 3F.. (their own kernels); timeline
                    // jobs are global-only (large and global tiers)
                    const int feat = (c.mode == CARMA_MODE_MIG ? 1 : 0) |
                                     ((c.sample_interval > 0.0 || c.log_flags != 0) ? 2 : 0) |
                                     ((pl->trace_max_gpus[jobs[i].trace] > 2 || needs_segments(c)) ? 4 : 0);
                    const int tier = ((feat & 6) || c.gpu_count > 64 || c.gpu_capacity / c.alloc_block > 128) ? 2
                                                                                           : static_cast<int>(heavy_config(c));
                    const int jc = tier + 3 * feat;
                    if (jc != cls) continue;
                    pl->class_list.push_back(i);
                    pl->class_count[cls]++;
                    pl->class_max_g[cls] = std::max(pl->class_max_g[cls], c.gpu_count);
                }
            std::copy(pl->class_list.begin(), pl->class_list.end(), list.begin());
            up(pl->d_list, list.data(), list.size() * 4);
            pl->d_task_out.ensure(to * sizeof(carma_task_result));
            pl->d_trace_out.ensure(n_jobs * sizeof(carma_trace_result));
            pl->d_gpu_out.ensure(go * sizeof(carma_gpu_result));
            pl->d_inv.ensure(to * 4);
            pl->d_begin.ensure(n_jobs * sizeof(double));
            pl->d_counters.ensure(512);
            pl->d_tl_count.ensure(n_jobs * sizeof(uint64_t));
            pl->d_log_count.ensure(n_jobs * sizeof(uint64_t));
        } catch (...) {
            if (pl->stream) cudaStreamDestroy(pl->stream);
            delete pl;
            throw;
        }
        *out = reinterpret_cast<carma_replay_plan*>(pl);
    }
}

}  // namespace carma_b200

using namespace carma_b200;

extern "C" {

carma_status carma_replay_plan_create(int device, const carma_replay_config* configs, uint32_t n_configs,
                                      const carma_task* tasks, const uint64_t* trace_offsets, uint32_t n_traces,
                                      const carma_replay_job* jobs, uint32_t n_jobs, int32_t want_task_results,
                                      carma_replay_plan** out) {
    (void)want_task_results;
    return guarded([&] {
        if (!tasks) throw InvalidArg("null argument");
        build_plan(device, configs, n_configs, tasks, trace_offsets, n_traces, jobs, n_jobs, out);
    });
}

carma_status carma_replay_plan_create_generated(int device, const carma_replay_config* configs, uint32_t n_configs,
                                                int32_t mix, const uint64_t* seeds, uint32_t n_seeds,
                                                const uint64_t* entry_estimates, uint32_t n_tables,
                                                const carma_replay_job* jobs, uint32_t n_jobs,
                                                carma_replay_plan** out) {
    return guarded([&] {
        if (!seeds || n_seeds == 0) throw InvalidArg("ConfigError: sweep has no seeds");
        if (n_tables == 0) n_tables = 1;
        if (!entry_estimates && n_tables != 1) throw InvalidArg("estimate tables missing");
        const uint32_t T = trace_rows(mix);
        const uint64_t n_traces64 = static_cast<uint64_t>(n_seeds) * n_tables;
        if (n_traces64 > 0xffffffffull) throw Unsupported("too many traces");
        const uint32_t n_traces = static_cast<uint32_t>(n_traces64);
        std::vector<uint64_t> offs(n_traces + 1);
        for (uint32_t t = 0; t <= n_traces; ++t) offs[t] = static_cast<uint64_t>(t) * T;
        build_plan(device, configs, n_configs, nullptr, offs.data(), n_traces, jobs, n_jobs, out);
        auto* pl = reinterpret_cast<ReplayPlan*>(*out);
        try {
            DeviceGuard guard(device);
            DeviceBuffer d_seeds, d_tables;
            d_seeds.ensure(n_seeds * sizeof(uint64_t));
            CARMA_CUDA(cudaMemcpyAsync(d_seeds.ptr, seeds, n_seeds * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                       pl->stream));
            if (entry_estimates) {
                const size_t tb = static_cast<size_t>(n_tables) * catalog_size() * sizeof(uint64_t);
                d_tables.ensure(tb);
                CARMA_CUDA(cudaMemcpyAsync(d_tables.ptr, entry_estimates, tb, cudaMemcpyHostToDevice, pl->stream));
            }
            pl->d_entries.ensure(pl->n_tasks * sizeof(int32_t));
            launch_generate_traces(mix, d_seeds.as<uint64_t>(), n_seeds,
                                   entry_estimates ? d_tables.as<uint64_t>() : nullptr, n_tables,
                                   pl->d_tasks.as<carma_task>(), pl->d_entries.as<int32_t>(), pl->stream);
            CARMA_CUDA(cudaStreamSynchronize(pl->stream));  // the staging buffers go out of scope
        } catch (...) {
            carma_replay_plan_destroy(*out);
            *out = nullptr;
            throw;
        }
    });
}

carma_status carma_replay_plan_entries(carma_replay_plan* hp, int32_t* entries) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl || !entries) throw InvalidArg("null argument");
        if (!pl->d_entries.ptr) throw InvalidArg("plan was not generated on the device");
        std::lock_guard<std::mutex> lock(pl->mu);
        DeviceGuard guard(pl->device);
        CARMA_CUDA(cudaMemcpyAsync(entries, pl->d_entries.ptr, pl->n_tasks * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                   pl->stream));
        CARMA_CUDA(cudaStreamSynchronize(pl->stream));
    });
}

carma_status carma_replay_plan_tasks(carma_replay_plan* hp, carma_task* tasks) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl || !tasks) throw InvalidArg("null argument");
        std::lock_guard<std::mutex> lock(pl->mu);
        DeviceGuard guard(pl->device);
        CARMA_CUDA(cudaMemcpyAsync(tasks, pl->d_tasks.ptr, pl->n_tasks * sizeof(carma_task), cudaMemcpyDeviceToHost,
                                   pl->stream));
        CARMA_CUDA(cudaStreamSynchronize(pl->stream));
    });
}

carma_status carma_replay_plan_set_estimates_device(carma_replay_plan* hp, const uint64_t* est) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        pl->est_override = est;
    });
}

carma_status carma_replay_plan_run(carma_replay_plan* hp, void* stream) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        std::lock_guard<std::mutex> lock(pl->mu);
        DeviceGuard guard(pl->device);
        if (stream) {
            // order after work already queued on the caller's stream
            cudaEvent_t ev;
            CARMA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CARMA_CUDA(cudaEventRecord(ev, static_cast<cudaStream_t>(stream)));
            CARMA_CUDA(cudaStreamWaitEvent(pl->stream, ev, 0));
            CARMA_CUDA(cudaEventDestroy(ev));
        }
        run_plan(*pl);
        // ... and the caller's later work (and its event timings) after the replay
        join_stream(static_cast<cudaStream_t>(stream), pl->stream);
    });
}

carma_status carma_replay_plan_upload_tasks(carma_replay_plan* hp, const carma_task* tasks) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl || !tasks) throw InvalidArg("null argument");
        std::lock_guard<std::mutex> lock(pl->mu);
        DeviceGuard guard(pl->device);
        CARMA_CUDA(cudaMemcpyAsync(pl->d_tasks.ptr, tasks, pl->n_tasks * sizeof(carma_task), cudaMemcpyHostToDevice,
                                   pl->stream));
        if (!is_pinned(tasks)) CARMA_CUDA(cudaStreamSynchronize(pl->stream));
    });
}

carma_status carma_replay_plan_set_outcome_sink(carma_replay_plan* hp, carma_task_outcome* host_outcomes) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        std::lock_guard<std::mutex> lock(pl->mu);
        if (!host_outcomes) {
            pl->outcome_sink = nullptr;
            return;
        }
        if (!is_pinned(host_outcomes)) throw InvalidArg("the outcome sink must be pinned (page-locked) host memory");
        DeviceGuard guard(pl->device);
        void* dp = nullptr;
        CARMA_CUDA(cudaHostGetDevicePointer(&dp, host_outcomes, 0));
        pl->outcome_sink = static_cast<carma_task_outcome*>(dp);
    });
}

carma_status carma_replay_plan_outcomes(carma_replay_plan* hp, carma_task_outcome* tasks,
                                        carma_trace_result* traces, carma_gpu_result* gpus) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        std::lock_guard<std::mutex> lock(pl->mu);
        DeviceGuard guard(pl->device);
        if (tasks) {
            pl->d_outcomes.ensure(pl->n_task_out * sizeof(carma_task_outcome));
            compact_outcomes<<<grid_for(pl->n_task_out, 256, 148u * 16u), 256, 0, pl->stream>>>(
                pl->d_task_out.as<carma_task_result>(), pl->n_task_out, pl->d_outcomes.as<carma_task_outcome>());
            CARMA_CUDA(cudaGetLastError());
            CARMA_CUDA(cudaMemcpyAsync(tasks, pl->d_outcomes.ptr, pl->n_task_out * sizeof(carma_task_outcome),
                                       cudaMemcpyDeviceToHost, pl->stream));
        }
        if (traces)
            CARMA_CUDA(cudaMemcpyAsync(traces, pl->d_trace_out.ptr, pl->jobs.size() * sizeof(carma_trace_result),
                                       cudaMemcpyDeviceToHost, pl->stream));
        if (gpus)
            CARMA_CUDA(cudaMemcpyAsync(gpus, pl->d_gpu_out.ptr, pl->n_gpu_out * sizeof(carma_gpu_result),
                                       cudaMemcpyDeviceToHost, pl->stream));
        CARMA_CUDA(cudaStreamSynchronize(pl->stream));
    });
}

carma_status carma_replay_plan_results(carma_replay_plan* hp, carma_task_result* tasks,
                                       carma_trace_result* traces, carma_gpu_result* gpus) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        std::lock_guard<std::mutex> lock(pl->mu);
        DeviceGuard guard(pl->device);
        if (tasks)
            CARMA_CUDA(cudaMemcpyAsync(tasks, pl->d_task_out.ptr, pl->n_task_out * sizeof(carma_task_result),
                                       cudaMemcpyDeviceToHost, pl->stream));
        if (traces)
            CARMA_CUDA(cudaMemcpyAsync(traces, pl->d_trace_out.ptr, pl->jobs.size() * sizeof(carma_trace_result),
                                       cudaMemcpyDeviceToHost, pl->stream));
        if (gpus)
            CARMA_CUDA(cudaMemcpyAsync(gpus, pl->d_gpu_out.ptr, pl->n_gpu_out * sizeof(carma_gpu_result),
                                       cudaMemcpyDeviceToHost, pl->stream));
        CARMA_CUDA(cudaStreamSynchronize(pl->stream));
    });
}

carma_status carma_replay_plan_stats(carma_replay_plan* hp, uint64_t* launches, uint64_t* retried_jobs) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        if (launches) *launches = pl->launches;
        if (retried_jobs) *retried_jobs = pl->retried;
    });
}

carma_status carma_replay_plan_timing(carma_replay_plan* hp, double* kernel_ms, double* run_ms) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        DeviceGuard guard(pl->device);
        CARMA_CUDA(cudaEventSynchronize(pl->ev[2]));
        float a = 0.f, b = 0.f;
        CARMA_CUDA(cudaEventElapsedTime(&a, pl->ev[0], pl->ev[1]));
        CARMA_CUDA(cudaEventElapsedTime(&b, pl->ev[0], pl->ev[2]));
        if (kernel_ms) *kernel_ms = a;
        if (run_ms) *run_ms = b;
    });
}

carma_status carma_replay_plan_set_timeline_capacity(carma_replay_plan* hp, uint64_t rows_per_job) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        std::lock_guard<std::mutex> lock(pl->mu);
        DeviceGuard guard(pl->device);
        pl->d_tl.ensure(rows_per_job * pl->jobs.size() * sizeof(carma_timeline_row));
        pl->tl_cap = rows_per_job;
    });
}

carma_status carma_replay_plan_set_log_capacity(carma_replay_plan* hp, uint64_t records_per_job) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        std::lock_guard<std::mutex> lock(pl->mu);
        DeviceGuard guard(pl->device);
        pl->d_log.ensure(records_per_job * pl->jobs.size() * sizeof(carma_log_record));
        pl->log_cap = records_per_job;
    });
}

carma_status carma_replay_plan_log(carma_replay_plan* hp, uint32_t job, carma_log_record* recs, uint64_t cap,
                                   uint64_t* n_out) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        if (job >= pl->jobs.size()) throw InvalidArg("job index out of range");
        if (pl->cfgs[pl->jobs[job].config].log_flags == 0) throw InvalidArg("job has no log");
        DeviceGuard guard(pl->device);
        CARMA_CUDA(cudaStreamSynchronize(pl->stream));
        uint64_t n = 0;
        CARMA_CUDA(cudaMemcpy(&n, pl->d_log_count.as<uint64_t>() + job, sizeof(n), cudaMemcpyDeviceToHost));
        if (n_out) *n_out = n;
        const uint64_t k = std::min(std::min(n, pl->log_cap), cap);
        if (recs && k)
            CARMA_CUDA(cudaMemcpy(recs, pl->d_log.as<carma_log_record>() + static_cast<uint64_t>(job) * pl->log_cap,
                                  k * sizeof(carma_log_record), cudaMemcpyDeviceToHost));
    });
}

carma_status carma_replay_plan_timeline(carma_replay_plan* hp, uint32_t job, carma_timeline_row* rows, uint64_t cap,
                                        uint64_t* n_rows) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) throw InvalidArg("null plan");
        if (job >= pl->jobs.size()) throw InvalidArg("job index out of range");
        if (!(pl->cfgs[pl->jobs[job].config].sample_interval > 0.0)) throw InvalidArg("job has no timeline");
        DeviceGuard guard(pl->device);
        CARMA_CUDA(cudaStreamSynchronize(pl->stream));
        uint64_t n = 0;
        CARMA_CUDA(cudaMemcpy(&n, pl->d_tl_count.as<uint64_t>() + job, sizeof(n), cudaMemcpyDeviceToHost));
        if (n_rows) *n_rows = n;
        const uint64_t k = std::min(std::min(n, pl->tl_cap), cap);
        if (rows && k)
            CARMA_CUDA(cudaMemcpy(rows, pl->d_tl.as<carma_timeline_row>() + static_cast<uint64_t>(job) * pl->tl_cap,
                                  k * sizeof(carma_timeline_row), cudaMemcpyDeviceToHost));
    });
}

carma_status carma_replay_plan_destroy(carma_replay_plan* hp) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) return;
        {
            DeviceGuard guard(pl->device);
            cudaStreamSynchronize(pl->stream);
            DeviceBuffer* bufs[] = {&pl->d_cfgs, &pl->d_tasks, &pl->d_trace_off, &pl->d_jobs, &pl->d_task_off,
                                    &pl->d_gpu_off, &pl->d_list, &pl->d_task_out, &pl->d_trace_out, &pl->d_gpu_out,
                                    &pl->d_inv, &pl->d_begin, &pl->d_counters, &pl->d_gstate, &pl->d_outcomes,
                                    &pl->d_tl, &pl->d_tl_count, &pl->d_log, &pl->d_log_count};
            for (auto* b : bufs) b->release();
            for (auto& e : pl->ev)
                if (e) cudaEventDestroy(e);
            cudaStreamDestroy(pl->stream);
        }
        delete pl;
    });
}

carma_status carma_replay_batch(int device, const carma_replay_config* configs, uint32_t n_configs,
                                const carma_task* tasks, const uint64_t* trace_offsets, uint32_t n_traces,
                                const carma_replay_job* jobs, uint32_t n_jobs, carma_task_result* task_results,
                                carma_trace_result* trace_results, carma_gpu_result* gpu_results) {
    carma_replay_plan* pl = nullptr;
    carma_status st = carma_replay_plan_create(device, configs, n_configs, tasks, trace_offsets, n_traces, jobs,
                                               n_jobs, task_results != nullptr, &pl);
    if (st != CARMA_OK) return st;
    st = carma_replay_plan_run(pl, nullptr);
    if (st == CARMA_OK) st = carma_replay_plan_results(pl, task_results, trace_results, gpu_results);
    const std::string err = st == CARMA_OK ? std::string() : std::string(carma_last_error());
    carma_replay_plan_destroy(pl);
    if (st != CARMA_OK) set_last_error(err);
    return st;
}

}  // extern "C"

namespace carma_b200 {
namespace {

void validate_pick(const carma_replay_config* cfg, uint32_t n_gpus) {
    if (!cfg) throw InvalidArg("null config");
    if (n_gpus < 1 || n_gpus > CARMA_MAX_GPUS) throw Unsupported("n_gpus must be in [1, 64]");
    if (cfg->mode == CARMA_MODE_MIG) throw Unsupported("carma_pick_batch: MIG needs per-instance views; use the replay");
}

// One launch over device-resident views / requests / cursors / outputs.
void launch_pick(const carma_replay_config& cfg, const carma_gpu_view* views, uint32_t n_gpus,
                 const carma_pick_request* reqs, uint64_t n, int32_t* cursor, int32_t* out, cudaStream_t s) {
    carma_replay_config c = cfg;
    c.gpu_count = static_cast<int32_t>(n_gpus);
    if (n_gpus <= static_cast<uint32_t>(kPickMaxSerialGpus)) {
        const size_t shmem = static_cast<size_t>(kPickWarps) * 32 * n_gpus * sizeof(carma_gpu_view);
        if (shmem > 48 * 1024)
            CARMA_CUDA(cudaFuncSetAttribute(pick_kernel_thread, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(shmem)));
        const uint64_t warps = (n + 31) / 32;
        const unsigned grid = grid_for(warps * 32, 32 * kPickWarps, 148u * 32u);
        pick_kernel_thread<<<grid, 32 * kPickWarps, shmem, s>>>(c, views, n_gpus, reqs, n, cursor, out);
        CARMA_CUDA(cudaGetLastError());
        return;
    }
    unsigned width = 1;
    while (width < n_gpus && width < 32) width <<= 1;
    const unsigned groups_per_warp = 32 / width;
    const uint64_t warps = (n + groups_per_warp - 1) / groups_per_warp;
    const unsigned grid = grid_for(warps * 32, 256, 148u * 16u);
    if (n_gpus > 32)
        pick_kernel<2><<<grid, 256, 0, s>>>(c, views, n_gpus, reqs, n, cursor, out, width);
    else
        pick_kernel<1><<<grid, 256, 0, s>>>(c, views, n_gpus, reqs, n, cursor, out, width);
    CARMA_CUDA(cudaGetLastError());
}

}  // namespace
}  // namespace carma_b200

extern "C" {

carma_status carma_pick_batch(int device, const carma_replay_config* cfg, const carma_gpu_view* views,
                              uint32_t n_gpus, const carma_pick_request* reqs, uint64_t n, int32_t* rr_cursor,
                              int32_t* out_gpus) {
    return guarded([&] {
        validate_pick(cfg, n_gpus);
        if (!views || !reqs || !rr_cursor || !out_gpus) throw InvalidArg("null argument");
        if (n == 0) return;
        for (uint64_t i = 0; i < n; ++i)
            if (reqs[i].want < 1 || reqs[i].want > 2) throw Unsupported("want must be 1 or 2");
        require_device(device);
        DeviceGuard guard(device);
        DeviceBuffer dv, dr, dc, dout;
        dv.ensure(n * n_gpus * sizeof(carma_gpu_view));
        dr.ensure(n * sizeof(carma_pick_request));
        dc.ensure(n * 4);
        dout.ensure(n * 8);
        CARMA_CUDA(cudaMemcpy(dv.ptr, views, n * n_gpus * sizeof(carma_gpu_view), cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(dr.ptr, reqs, n * sizeof(carma_pick_request), cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(dc.ptr, rr_cursor, n * 4, cudaMemcpyHostToDevice));
        launch_pick(*cfg, dv.as<carma_gpu_view>(), n_gpus, dr.as<carma_pick_request>(), n, dc.as<int32_t>(),
                    dout.as<int32_t>(), nullptr);
        CARMA_CUDA(cudaMemcpy(out_gpus, dout.ptr, n * 8, cudaMemcpyDeviceToHost));
        CARMA_CUDA(cudaMemcpy(rr_cursor, dc.ptr, n * 4, cudaMemcpyDeviceToHost));
    });
}

carma_status carma_pick_batch_wide(int device, const carma_replay_config* cfg, const carma_gpu_view* views,
                                   uint32_t n_gpus, const carma_pick_request* reqs, uint64_t n, int32_t* rr_cursor,
                                   int32_t* out_gpus) {
    return guarded([&] {
        if (!cfg) throw InvalidArg("null config");
        if (n_gpus < 1 || n_gpus > CARMA_MAX_REPLAY_GPUS) throw Unsupported("n_gpus must be in [1, 256]");
        if (cfg->mode == CARMA_MODE_MIG) throw Unsupported("carma_pick_batch: MIG needs per-instance views; use the replay");
        if (!views || !reqs || !rr_cursor || !out_gpus) throw InvalidArg("null argument");
        if (n == 0) return;
        for (uint64_t i = 0; i < n; ++i)
            if (reqs[i].want < 1 || reqs[i].want > CARMA_MAX_TASK_GPUS) throw Unsupported("want must be in [1, 8]");
        require_device(device);
        DeviceGuard guard(device);
        DeviceBuffer dv, dr, dc, dout;
        dv.ensure(n * n_gpus * sizeof(carma_gpu_view));
        dr.ensure(n * sizeof(carma_pick_request));
        dc.ensure(n * 4);
        dout.ensure(n * 4 * CARMA_MAX_TASK_GPUS);
        CARMA_CUDA(cudaMemcpy(dv.ptr, views, n * n_gpus * sizeof(carma_gpu_view), cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(dr.ptr, reqs, n * sizeof(carma_pick_request), cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(dc.ptr, rr_cursor, n * 4, cudaMemcpyHostToDevice));
        carma_replay_config c = *cfg;
        c.gpu_count = static_cast<int32_t>(n_gpus);
        const unsigned grid = grid_for(n * 32, 128, 148u * 16u);
        pick_kernel_wide<<<grid, 128>>>(c, dv.as<carma_gpu_view>(), n_gpus, dr.as<carma_pick_request>(), n,
                                        dc.as<int32_t>(), dout.as<int32_t>());
        CARMA_CUDA(cudaGetLastError());
        CARMA_CUDA(cudaMemcpy(out_gpus, dout.ptr, n * 4 * CARMA_MAX_TASK_GPUS, cudaMemcpyDeviceToHost));
        CARMA_CUDA(cudaMemcpy(rr_cursor, dc.ptr, n * 4, cudaMemcpyDeviceToHost));
    });
}

carma_status carma_pick_batch_device(int device, const carma_replay_config* cfg, const carma_gpu_view* views,
                                     uint32_t n_gpus, const carma_pick_request* reqs, uint64_t n,
                                     int32_t* rr_cursor, int32_t* out_gpus, void* stream) {
    return guarded([&] {
        validate_pick(cfg, n_gpus);
        if (!views || !reqs || !rr_cursor || !out_gpus) throw InvalidArg("null argument");
        if (n == 0) return;
        require_device(device);
        DeviceGuard guard(device);
        launch_pick(*cfg, views, n_gpus, reqs, n, rr_cursor, out_gpus, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"

#if REPLAY_PROF
// Diagnostic builds only: reads and clears the per-region cycle counters.
extern "C" int carma_debug_replay_prof(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, carma_b200::replay::g_replay_prof, 16 * sizeof(unsigned long long)) != cudaSuccess)
        return 1;
    const unsigned long long z[16] = {};
    return cudaMemcpyToSymbol(carma_b200::replay::g_replay_prof, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
extern "C" int carma_debug_replay_sub(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, carma_b200::replay::g_replay_sub, 8 * sizeof(unsigned long long)) != cudaSuccess)
        return 1;
    const unsigned long long z[8] = {};
    return cudaMemcpyToSymbol(carma_b200::replay::g_replay_sub, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
#endif
