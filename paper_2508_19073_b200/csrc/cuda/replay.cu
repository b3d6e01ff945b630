// Stage 2 — collocation-aware placement and trace replay on sm_100a.
//
// One warp replays one (trace, config) job end to end: the deterministic
// discrete-event loop of World (proj/src/world.cpp:31-186) driving the CARMA
// Manager pipeline (proj/src/manager.cpp:58-357) over simulated GpuDevices
// in MPS / streams mode (proj/src/gpu.cpp:58-274), then the runner tail
// (runner.cpp:97-141) and compute_report's scalars (metrics.cpp:16-70).
// Results are bit-identical to the reference (built with --fmad=false; every
// floating-point expression keeps the reference's operation order).
//
// Warp organisation. Sequential event logic (queue heads, the event heap,
// dispatch decisions, rate refresh) runs warp-uniformly — every lane
// computes the same values — while per-GPU work is lane-parallel: lane l
// owns simulated GPUs l and l+32. Energy integration, windowed-SMACT,
// feasibility and the MAGM/LUG/MUG arg-reductions (pick.cuh) are one step
// across the lanes; the first-fit allocator runs on the owner lane's bitmap.
//
// State layout (per warp, shared memory for the common tier, global memory
// for the large tier; see Layout):
//   * per GPU (SoA): allocation bitmap (block = SimConstants::alloc_block),
//     cached per-resident rate / instantaneous SMACT / power, energy, peak,
//     the resident list in insertion order, a ring of recent SMACT steps for
//     windowed_smact, and a running integrator reproducing the full-history
//     windowed_smact(last_complete, span) of runner.cpp:135-137 term by term;
//   * resident-task slots (remaining work, rate, last update, live event);
//   * a binary min-heap of dynamic events ordered by (t, seq); arrivals are a
//     pre-sorted stream with seq = trace index (runner.cpp:72-78), merged at pop;
//   * the main queue is the index range [mq_head, arrived) (FIFO, manager.cpp:58-78);
//     the recovery queue a ring.
// A completion event is live iff its seq equals its slot's live seq — the
// same test as TaskRun::gen (world.cpp:52-57), since every reschedule draws
// a fresh seq.
// Capacity overflow of any structure aborts the job in the shared-memory
// tier and re-runs it in the global-memory tier with large capacities.

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../../include/carma_gpu.h"
#include "common.cuh"
#include "pick.cuh"

namespace carma_b200 {
namespace {

constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kKindWindow = 1u, kKindCompletion = 2u, kKindCrash = 3u;
constexpr int32_t kStatusRetry = -1;      // overflowed this tier
constexpr int32_t kStatusRedoSmact = -2;  // full-history SMACT needs a known window begin

struct Caps {
    uint32_t G;   // simulated GPUs (max over the launch's jobs)
    uint32_t W;   // bitmap words per GPU
    uint32_t H;   // event heap entries
    uint32_t S;   // resident-task slots
    uint32_t RC;  // residents per GPU
    uint32_t RG;  // SMACT ring entries per GPU
    uint32_t RQ;  // recovery queue entries
};

// Per-warp state view; pointers into shared or global memory.
struct St {
    uint64_t* used;  // [W][G]
    double *energy, *rate, *inst, *power, *lvl, *cur, *integ, *last_t, *last_v;
    uint32_t *nres, *nsteps, *rhead, *rcnt, *peak, *has_step;
    double *ring_t, *ring_v;  // [G][RG]
    double* ht;               // [H]
    uint32_t *hs, *hinfo;     // [H]
    double *s_rem, *s_rate, *s_last, *s_exec, *s_dem;  // [S]
    uint32_t *s_task, *s_rank, *s_seq, *s_gp, *s_off, *s_nb;  // [S]
    uint32_t* free_stack;  // [S]
    uint32_t* rq;          // [RQ]
    uint64_t *aff, *aff2;  // [2*RC]
    uint16_t* res;         // [G][RC]
};

__host__ __device__ inline size_t layout_bytes(const Caps& c, St* st, char* base) {
    // Order: 8-byte fields, then 4-byte, then 2-byte.
    size_t b = 0;
    auto take = [&](size_t n, size_t align) {
        b = (b + align - 1) / align * align;
        const size_t o = b;
        b += n;
        return o;
    };
    const size_t G = c.G, S = c.S, H = c.H;
    size_t o_used = take(8 * c.W * G, 16);
    size_t o_d[9];
    for (int i = 0; i < 9; ++i) o_d[i] = take(8 * G, 8);
    size_t o_rt = take(8 * G * c.RG, 8), o_rv = take(8 * G * c.RG, 8);
    size_t o_ht = take(8 * H, 8);
    size_t o_sd[5];
    for (int i = 0; i < 5; ++i) o_sd[i] = take(8 * S, 8);
    size_t o_aff = take(8 * 2 * c.RC, 8), o_aff2 = take(8 * 2 * c.RC, 8);
    size_t o_u[6];
    for (int i = 0; i < 6; ++i) o_u[i] = take(4 * G, 4);
    size_t o_hs = take(4 * H, 4), o_hi = take(4 * H, 4);
    size_t o_su[6];
    for (int i = 0; i < 6; ++i) o_su[i] = take(4 * S, 4);
    size_t o_fs = take(4 * S, 4), o_rq = take(4 * c.RQ, 4);
    size_t o_res = take(2 * G * c.RC, 2);
    b = (b + 15) / 16 * 16;
    if (st) {
        st->used = reinterpret_cast<uint64_t*>(base + o_used);
        double** dp[9] = {&st->energy, &st->rate, &st->inst, &st->power, &st->lvl,
                          &st->cur, &st->integ, &st->last_t, &st->last_v};
        for (int i = 0; i < 9; ++i) *dp[i] = reinterpret_cast<double*>(base + o_d[i]);
        st->ring_t = reinterpret_cast<double*>(base + o_rt);
        st->ring_v = reinterpret_cast<double*>(base + o_rv);
        st->ht = reinterpret_cast<double*>(base + o_ht);
        double** sp[5] = {&st->s_rem, &st->s_rate, &st->s_last, &st->s_exec, &st->s_dem};
        for (int i = 0; i < 5; ++i) *sp[i] = reinterpret_cast<double*>(base + o_sd[i]);
        st->aff = reinterpret_cast<uint64_t*>(base + o_aff);
        st->aff2 = reinterpret_cast<uint64_t*>(base + o_aff2);
        uint32_t** up[6] = {&st->nres, &st->nsteps, &st->rhead, &st->rcnt, &st->peak, &st->has_step};
        for (int i = 0; i < 6; ++i) *up[i] = reinterpret_cast<uint32_t*>(base + o_u[i]);
        st->hs = reinterpret_cast<uint32_t*>(base + o_hs);
        st->hinfo = reinterpret_cast<uint32_t*>(base + o_hi);
        uint32_t** su[6] = {&st->s_task, &st->s_rank, &st->s_seq, &st->s_gp, &st->s_off, &st->s_nb};
        for (int i = 0; i < 6; ++i) *su[i] = reinterpret_cast<uint32_t*>(base + o_su[i]);
        st->free_stack = reinterpret_cast<uint32_t*>(base + o_fs);
        st->rq = reinterpret_cast<uint32_t*>(base + o_rq);
        st->res = reinterpret_cast<uint16_t*>(base + o_res);
    }
    return b;
}

struct ReplayParams {
    const carma_replay_config* cfgs;
    const carma_task* tasks;
    const uint64_t* trace_off;
    const carma_replay_job* jobs;
    const uint64_t* task_out_off;
    const uint64_t* gpu_out_off;
    const uint64_t* est_override;  // nullable, indexed like tasks
    const uint32_t* job_list;      // jobs to run in this launch
    uint32_t n_list;
    carma_task_result* task_out;
    carma_trace_result* trace_out;
    carma_gpu_result* gpu_out;
    uint32_t* inv_scratch;          // rank -> index, indexed like task_out
    double* smact_begin;            // per job; NaN = derive from first_submit
    uint32_t* retry_list;           // jobs that overflowed this tier
    uint32_t* retry_count;
    unsigned int* next_job;         // dynamic scheduler counter
    char* gstate;                   // global-tier state, per warp
    size_t state_bytes;
    Caps caps;
};

// Warp-uniform scalar state (replicated in every lane).
struct Sc {
    double now, deadline;
    uint32_t seq_next, arrived, mq_head, rq_head, rq_cnt, hsize, nfree;
    int rr_cursor;
    int32_t oom;
    uint64_t events;
    int32_t status;
};

__device__ __forceinline__ double dmax0(double x) { return 0.0 < x ? x : 0.0; }  // std::max(0.0, x)
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min(a, b)
__device__ __forceinline__ bool later(double ta, uint32_t sa, double tb, uint32_t sb) {
    return ta != tb ? ta > tb : sa > sb;
}

// ---------------------------------------------------------------- heap
__device__ __forceinline__ uint32_t heap_push(St& s, Sc& c, const Caps& cap, double t, uint32_t info) {
    if (c.hsize >= cap.H) {
        c.status = kStatusRetry;
        return kNone;
    }
    const uint32_t seq = c.seq_next++;
    uint32_t i = c.hsize++;
    while (i > 0) {
        const uint32_t p = (i - 1) >> 1;
        const double pt = s.ht[p];
        const uint32_t ps = s.hs[p];
        if (!later(pt, ps, t, seq)) break;
        s.ht[i] = pt;
        s.hs[i] = ps;
        s.hinfo[i] = s.hinfo[p];
        i = p;
    }
    s.ht[i] = t;
    s.hs[i] = seq;
    s.hinfo[i] = info;
    return seq;
}

__device__ __forceinline__ void heap_pop(St& s, Sc& c) {
    const uint32_t n = --c.hsize;
    if (n == 0) return;
    const double t = s.ht[n];
    const uint32_t sq = s.hs[n], inf = s.hinfo[n];
    uint32_t i = 0;
    for (;;) {
        uint32_t l = 2 * i + 1;
        if (l >= n) break;
        const uint32_t r = l + 1;
        if (r < n && later(s.ht[l], s.hs[l], s.ht[r], s.hs[r])) l = r;
        if (!later(t, sq, s.ht[l], s.hs[l])) break;
        s.ht[i] = s.ht[l];
        s.hs[i] = s.hs[l];
        s.hinfo[i] = s.hinfo[l];
        i = l;
    }
    s.ht[i] = t;
    s.hs[i] = sq;
    s.hinfo[i] = inf;
}

// ------------------------------------------------------------ allocator
// Bit = 1: block used (bits past the device's block count are set).
__device__ __forceinline__ int next_bit(const St& s, const Caps& cap, int g, int from, int nblk, bool one) {
    for (int w = from >> 6; w < static_cast<int>(cap.W); ++w) {
        uint64_t bits = s.used[w * cap.G + g];
        if (!one) bits = ~bits;
        if (w == (from >> 6)) bits &= ~0ull << (from & 63);
        if (bits) {
            const int b = w * 64 + __ffsll(static_cast<long long>(bits)) - 1;
            return b < nblk ? b : nblk;
        }
    }
    return nblk;
}

__device__ __forceinline__ void set_bits(St& s, const Caps& cap, int g, int off, int nb, bool on) {
    for (int b = off; b < off + nb;) {
        const int w = b >> 6, lo = b & 63;
        const int cnt = min(64 - lo, off + nb - b);
        const uint64_t m = (cnt == 64 ? ~0ull : ((1ull << cnt) - 1ull)) << lo;
        uint64_t& word = s.used[w * cap.G + g];
        word = on ? (word | m) : (word & ~m);
        b += cnt;
    }
}

__device__ __forceinline__ uint32_t free_blocks(const St& s, const Caps& cap, int g) {
    uint32_t f = 0;
    for (uint32_t w = 0; w < cap.W; ++w) f += __popcll(static_cast<long long>(~s.used[w * cap.G + g]));
    return f;
}

// GpuDevice::allocate_range in whole-device mode (gpu.cpp:72-114): first fit
// over maximal free runs; carve from the tail iff the left neighbour is used
// and the run reaches the end of the device.
__device__ __forceinline__ int first_fit(St& s, const Caps& cap, int g, int nblk, int want) {
    int pos = 0;
    while (pos < nblk) {
        const int start = next_bit(s, cap, g, pos, nblk, false);
        if (start >= nblk) break;
        const int end = next_bit(s, cap, g, start, nblk, true);
        if (end - start >= want) {
            const bool tail = start > 0 && end == nblk;
            const int place = tail ? end - want : start;
            set_bits(s, cap, g, place, want, true);
            const uint32_t used = static_cast<uint32_t>(nblk) - free_blocks(s, cap, g);
            if (used > s.peak[g]) s.peak[g] = used;
            return place;
        }
        pos = end;
    }
    return -1;
}

// ----------------------------------------------------------------- SMACT
// windowed_smact (gpu.cpp:244-267) over the ring of recent steps.
__device__ __forceinline__ double windowed(const St& s, const Caps& cap, int g, double now, double window) {
    const double begin = dmax0(now - window);
    const double span = now - begin;
    if (span <= 0.0) return s.inst[g];
    double integral = 0.0, level = 0.0, cursor = begin;
    const uint32_t h = s.rhead[g], n = s.rcnt[g];
    for (uint32_t k = 0; k < n; ++k) {
        uint32_t idx = h + k;
        if (idx >= cap.RG) idx -= cap.RG;
        const double t = s.ring_t[g * cap.RG + idx];
        const double v = s.ring_v[g * cap.RG + idx];
        if (t <= begin) {
            level = v;
            continue;
        }
        if (t >= now) break;
        integral = __dadd_rn(integral, __dmul_rn(level, __dsub_rn(t, cursor)));
        cursor = t;
        level = v;
    }
    integral = __dadd_rn(integral, __dmul_rn(level, __dsub_rn(now, cursor)));
    return __ddiv_rn(integral, span);
}

// record_smact (gpu.cpp:231-242) + ring + running full-history integrator.
__device__ __forceinline__ void record_smact(St& s, Sc& c, const Caps& cap, int g, double v,
                                             double window, double begin0) {
    const double now = c.now;
    if (s.has_step[g]) {
        if (s.last_v[g] == v) return;
        if (s.last_t[g] == now) {
            s.last_v[g] = v;
            uint32_t li = s.rhead[g] + s.rcnt[g] - 1;
            if (li >= cap.RG) li -= cap.RG;
            s.ring_v[g * cap.RG + li] = v;
            s.lvl[g] = v;
            return;
        }
    }
    // Drop ring entries no future window can need: begin only grows, so an
    // entry whose successor is already at or before begin is dead.
    const double begin_now = dmax0(now - window);
    while (s.rcnt[g] >= 2) {
        uint32_t second = s.rhead[g] + 1;
        if (second >= cap.RG) second -= cap.RG;
        if (!(s.ring_t[g * cap.RG + second] <= begin_now)) break;
        s.rhead[g] = second;
        s.rcnt[g] -= 1;
    }
    if (s.rcnt[g] >= cap.RG) {
        c.status = kStatusRetry;  // lane-local; merged by the caller
        return;
    }
    uint32_t slot = s.rhead[g] + s.rcnt[g];
    if (slot >= cap.RG) slot -= cap.RG;
    s.ring_t[g * cap.RG + slot] = now;
    s.ring_v[g * cap.RG + slot] = v;
    s.rcnt[g] += 1;
    // Full-history integral from begin0 (= windowed_smact(last_complete, span)).
    if (now <= begin0) {
        s.lvl[g] = v;
    } else {
        s.integ[g] = __dadd_rn(s.integ[g], __dmul_rn(s.lvl[g], __dsub_rn(now, s.cur[g])));
        s.cur[g] = now;
        s.lvl[g] = v;
    }
    s.has_step[g] = 1;
    s.last_t[g] = now;
    s.last_v[g] = v;
    s.nsteps[g] += 1;
}

// effective_rates / instantaneous_smact / power_draw (gpu.cpp:183-229, 269-274)
// for GPU g, cached after its resident list changes.
__device__ __forceinline__ void refresh_gpu(St& s, const Caps& cap, const carma_replay_config& cf, int g) {
    const uint32_t n = s.nres[g];
    double rate = 0.0, inst = 0.0;
    if (n > 0) {
        if (cf.mode == CARMA_MODE_MPS) {
            double total = 0.0;
            for (uint32_t r = 0; r < n; ++r) total = __dadd_rn(total, s.s_dem[s.res[g * cap.RC + r]]);
            rate = dmin(1.0, __ddiv_rn(1.0, total));
        } else {
            rate = __ddiv_rn(1.0, static_cast<double>(n));
        }
        double sum = 0.0;
        for (uint32_t r = 0; r < n; ++r) sum = __dadd_rn(sum, __dmul_rn(s.s_dem[s.res[g * cap.RC + r]], rate));
        inst = dmin(1.0, sum);
    }
    s.rate[g] = rate;
    s.inst[g] = inst;
    double p = __dadd_rn(cf.p_idle_w, __dmul_rn(__dsub_rn(cf.p_max_w, cf.p_idle_w), inst));
    if (inst > cf.boost_threshold) p = __dadd_rn(p, cf.p_boost_w);
    s.power[g] = p;
}

struct Job {
    const carma_replay_config* cf;
    const carma_task* tasks;
    uint32_t T;
    int nblk;
    double window, begin0;
    carma_task_result* out;
};

// World::refresh_rates (world.cpp:157-186) for the touched GPUs.
__device__ void refresh_rates(St& s, Sc& c, const Caps& cap, const Job& jb, const int* touched, int nt,
                              unsigned lane) {
    for (int k = 0; k < nt; ++k) {
        const int g = touched[k];
        if ((g & 31) == static_cast<int>(lane)) {
            refresh_gpu(s, cap, *jb.cf, g);
            Sc lc = c;
            record_smact(s, lc, cap, g, s.inst[g], jb.window, jb.begin0);
            if (lc.status) c.status = lc.status;
        }
        __syncwarp();
    }
    if (__any_sync(0xffffffffu, c.status != 0)) {
        c.status = kStatusRetry;
        return;
    }
    // Affected tasks: residents of the touched GPUs, deduplicated, ordered by
    // id (std::set<std::string>) == by rank.
    uint32_t na = 0;
    for (int k = 0; k < nt; ++k) {
        const int g = touched[k];
        const uint32_t n = s.nres[g];
        for (uint32_t r = 0; r < n; ++r) {
            const uint32_t slot = s.res[g * cap.RC + r];
            if (k == 1) {
                const uint32_t gp = s.s_gp[slot];
                const int ng = static_cast<int>(gp >> 16);
                bool dup = static_cast<int>(gp & 0xff) == touched[0] ||
                           (ng > 1 && static_cast<int>((gp >> 8) & 0xff) == touched[0]);
                if (dup) continue;
            }
            s.aff[na++] = (static_cast<uint64_t>(s.s_rank[slot]) << 32) | slot;
        }
    }
    __syncwarp();
    for (uint32_t e = lane; e < na; e += 32) {
        const uint64_t key = s.aff[e];
        uint32_t pos = 0;
        for (uint32_t j = 0; j < na; ++j) pos += s.aff[j] < key;
        s.aff2[pos] = key;
    }
    __syncwarp();
    for (uint32_t e = 0; e < na; ++e) {
        const uint32_t slot = static_cast<uint32_t>(s.aff2[e] & 0xffffffffu);
        const uint32_t gp = s.s_gp[slot];
        const int ng = static_cast<int>(gp >> 16);
        double rate = 1.0;
        rate = dmin(rate, s.rate[gp & 0xff]);
        if (ng > 1) rate = dmin(rate, s.rate[(gp >> 8) & 0xff]);
        const double old = s.s_rate[slot];
        if (rate == old && s.s_seq[slot] != kNone) continue;
        const double dt = __dsub_rn(c.now, s.s_last[slot]);
        s.s_exec[slot] = __dadd_rn(s.s_exec[slot], __dmul_rn(old, dt));
        const double rem = dmax0(__dsub_rn(s.s_rem[slot], __dmul_rn(old, dt)));
        s.s_rem[slot] = rem;
        s.s_last[slot] = c.now;
        s.s_rate[slot] = rate;
        const uint32_t seq = heap_push(s, c, cap, __dadd_rn(c.now, __ddiv_rn(rem, rate)),
                                       (kKindCompletion << 30) | slot);
        if (c.status) return;
        s.s_seq[slot] = seq;
    }
    __syncwarp();
}

// World::place (world.cpp:73-130). Returns true when the task became resident.
__device__ bool place(St& s, Sc& c, const Caps& cap, const Job& jb, uint32_t task, const int* gids, int want,
                      unsigned lane) {
    const carma_task& tk = jb.tasks[task];
    const uint64_t block = jb.cf->alloc_block;
    const uint64_t bytes = tk.true_mem > 0 ? tk.true_mem : 1;
    const uint64_t nb64 = (bytes + block - 1) / block;
    const int nb = nb64 > static_cast<uint64_t>(jb.nblk) ? jb.nblk + 1 : static_cast<int>(nb64);
    int offs[2] = {-1, -1};
    for (int k = 0; k < want; ++k) {
        const int g = gids[k];
        int off = -1;
        if ((g & 31) == static_cast<int>(lane) && nb <= jb.nblk) off = first_fit(s, cap, g, jb.nblk, nb);
        off = __shfl_sync(0xffffffffu, off, g & 31);
        if (off < 0) {
            for (int j = 0; j < k; ++j)
                if ((gids[j] & 31) == static_cast<int>(lane)) set_bits(s, cap, gids[j], offs[j], nb, false);
            __syncwarp();
            return false;
        }
        offs[k] = off;
    }
    if (c.nfree == 0) {
        c.status = kStatusRetry;
        return false;
    }
    const uint32_t slot = s.free_stack[--c.nfree];
    s.s_task[slot] = task;
    s.s_rank[slot] = tk.rank;
    s.s_rem[slot] = tk.work;
    s.s_rate[slot] = 0.0;
    s.s_last[slot] = c.now;
    s.s_exec[slot] = 0.0;
    s.s_dem[slot] = tk.demand;
    s.s_seq[slot] = kNone;
    s.s_gp[slot] = static_cast<uint32_t>(gids[0]) | (static_cast<uint32_t>(want > 1 ? gids[1] : 0) << 8) |
                   (static_cast<uint32_t>(want) << 16);
    s.s_off[slot] = static_cast<uint32_t>(offs[0]) | (static_cast<uint32_t>(want > 1 ? offs[1] : 0) << 16);
    s.s_nb[slot] = static_cast<uint32_t>(nb);
    for (int k = 0; k < want; ++k) {
        const int g = gids[k];
        const uint32_t n = s.nres[g];
        if (n >= cap.RC) {
            c.status = kStatusRetry;
            return false;
        }
        s.res[g * cap.RC + n] = static_cast<uint16_t>(slot);
        s.nres[g] = n + 1;
    }
    __syncwarp();
    refresh_rates(s, c, cap, jb, gids, want, lane);
    return true;
}

// World::finish (world.cpp:132-155) for a live completion of `slot`.
__device__ void finish(St& s, Sc& c, const Caps& cap, const Job& jb, uint32_t slot, unsigned lane) {
    const double dt = __dsub_rn(c.now, s.s_last[slot]);
    const double rate = s.s_rate[slot];
    const double exec = __dadd_rn(s.s_exec[slot], __dmul_rn(rate, dt));
    s.s_rem[slot] = dmax0(__dsub_rn(s.s_rem[slot], __dmul_rn(rate, dt)));
    s.s_last[slot] = c.now;
    s.s_exec[slot] = exec;
    const uint32_t gp = s.s_gp[slot], of = s.s_off[slot];
    const int want = static_cast<int>(gp >> 16);
    int gids[2] = {static_cast<int>(gp & 0xff), static_cast<int>((gp >> 8) & 0xff)};
    const int offs[2] = {static_cast<int>(of & 0xffff), static_cast<int>(of >> 16)};
    const int nb = static_cast<int>(s.s_nb[slot]);
    for (int k = 0; k < want; ++k) {
        const int g = gids[k];
        if ((g & 31) == static_cast<int>(lane)) {
            set_bits(s, cap, g, offs[k], nb, false);
            // remove_resident preserving insertion order (gpu.cpp:175-181)
            const uint32_t n = s.nres[g];
            uint32_t r = 0;
            while (r < n && s.res[g * cap.RC + r] != slot) ++r;
            for (; r + 1 < n; ++r) s.res[g * cap.RC + r] = s.res[g * cap.RC + r + 1];
            s.nres[g] = n - 1;
        }
        __syncwarp();
    }
    const uint32_t task = s.s_task[slot];
    if (lane == 0) {
        jb.out[task].executed = exec;
        jb.out[task].complete = c.now;
    }
    s.s_seq[slot] = kNone;
    s.free_stack[c.nfree++] = slot;
    __syncwarp();
    refresh_rates(s, c, cap, jb, gids, want, lane);
}

template <int GPL>
__device__ void try_schedule(St& s, Sc& c, const Caps& cap, const Job& jb, const uint64_t* est_override,
                             uint32_t task_base, unsigned lane) {
    const carma_replay_config& cf = *jb.cf;
    // gate_open (manager.cpp:269-273)
    bool idle_all = true;
#pragma unroll
    for (int j = 0; j < GPL; ++j) {
        const int g = static_cast<int>(lane) + 32 * j;
        if (g < cf.gpu_count && s.nres[g] != 0) idle_all = false;
    }
    idle_all = __all_sync(0xffffffffu, idle_all);
    if (!(c.now >= c.deadline) && !idle_all) return;
    const bool from_recovery = c.rq_cnt > 0;
    uint32_t head;
    if (from_recovery) head = s.rq[c.rq_head];
    else if (c.mq_head < c.arrived) head = c.mq_head;
    else return;
    const carma_task& tk = jb.tasks[head];
    const int policy = from_recovery ? CARMA_POLICY_EXCLUSIVE : cf.policy;
    uint64_t floor = cf.min_free;
    if (!from_recovery && cf.policy != CARMA_POLICY_EXCLUSIVE) {
        const uint64_t est = est_override ? est_override[task_base + head] : tk.estimate;
        if (est != CARMA_NO_ESTIMATE) {
            const uint64_t need = est < cf.gpu_capacity ? est : cf.gpu_capacity;
            if (need > floor) floor = need;
        }
    }
    PickInput in[GPL];
    const bool need_smact = policy != CARMA_POLICY_EXCLUSIVE &&
                            !(policy == CARMA_POLICY_RR && !cf.rr_apply_preconditions);
#pragma unroll
    for (int j = 0; j < GPL; ++j) {
        const int g = static_cast<int>(lane) + 32 * j;
        const bool valid = g < cf.gpu_count;
        in[j].valid = valid;
        in[j].idle = valid && s.nres[g] == 0;
        in[j].free_bytes = valid ? static_cast<uint64_t>(free_blocks(s, cap, g)) * cf.alloc_block : 0;
        in[j].smact = (valid && need_smact) ? windowed(s, cap, g, c.now, cf.monitor_window) : 0.0;
    }
    int gids[2];
    const int got = pick_gpus<GPL>(cf, policy, tk.gpus, floor, in, lane, 0, 32, c.rr_cursor, gids);
    if (got == 0) return;  // defer; retried on the next completion / expiry
    if (from_recovery) {
        c.rq_head = c.rq_head + 1 == cap.RQ ? 0 : c.rq_head + 1;
        c.rq_cnt--;
    } else {
        c.mq_head++;
    }
    // dispatch (manager.cpp:247-260)
    carma_task_result& o = jb.out[head];
    if (lane == 0 && !from_recovery) o.first_attempt = c.now;
    const bool ok = place(s, c, cap, jb, head, gids, got, lane);
    if (c.status) return;
    if (!ok) {
        heap_push(s, c, cap, __dadd_rn(c.now, cf.oom_startup_delay), (kKindCrash << 30) | head);
    } else if (lane == 0) {
        o.final_dispatch = c.now;
        o.gpu[0] = static_cast<int16_t>(gids[0]);
        o.gpu[1] = static_cast<int16_t>(got > 1 ? gids[1] : -1);
    }
    if (c.status) return;
    // arm_window (manager.cpp:275-278)
    c.deadline = __dadd_rn(c.now, cf.monitor_window);
    heap_push(s, c, cap, c.deadline, kKindWindow << 30);
}

template <int GPL>
__device__ void run_job(St& s, const Caps& cap, const ReplayParams& p, uint32_t j, unsigned lane) {
    const carma_replay_job job = p.jobs[j];
    const carma_replay_config& cf = p.cfgs[job.config];
    const uint64_t tb = p.trace_off[job.trace];
    const uint32_t T = static_cast<uint32_t>(p.trace_off[job.trace + 1] - tb);
    const int G = cf.gpu_count;
    Job jb;
    jb.cf = &cf;
    jb.tasks = p.tasks + tb;
    jb.T = T;
    jb.nblk = static_cast<int>(cf.gpu_capacity / cf.alloc_block);
    jb.window = cf.monitor_window;
    jb.out = p.task_out + p.task_out_off[j];
    carma_gpu_result* gout = p.gpu_out + p.gpu_out_off[j];
    uint32_t* inv = p.inv_scratch + p.task_out_off[j];

    // first_submit (runner.cpp:108-109) and the full-history window begin.
    double fs = jb.tasks[0].submit;
    for (uint32_t i = lane; i < T; i += 32) fs = dmin(fs, jb.tasks[i].submit);
    for (int o = 16; o > 0; o >>= 1) fs = dmin(fs, __shfl_xor_sync(0xffffffffu, fs, o));
    const double forced = p.smact_begin[j];
    jb.begin0 = forced == forced ? forced : dmax0(fs);

    // Init outputs and state.
    for (uint32_t i = lane; i < T; i += 32) {
        carma_task_result r;
        r.first_attempt = r.final_dispatch = r.complete = r.first_crash = r.last_crash = -1.0;
        r.executed = 0.0;
        r.attempts = r.ooms = 0;
        r.gpu[0] = r.gpu[1] = -1;
        r.reserved = 0;
        jb.out[i] = r;
    }
    for (uint32_t g = lane; g < cap.G; g += 32) {
        for (uint32_t w = 0; w < cap.W; ++w) {
            const int lo = static_cast<int>(w) * 64;
            uint64_t m = ~0ull;
            if (jb.nblk > lo) m = jb.nblk - lo >= 64 ? 0ull : (~0ull << (jb.nblk - lo));
            s.used[w * cap.G + g] = m;
        }
        s.energy[g] = 0.0;
        s.rate[g] = 0.0;
        s.inst[g] = 0.0;
        s.lvl[g] = 0.0;
        s.cur[g] = jb.begin0;
        s.integ[g] = 0.0;
        s.last_t[g] = 0.0;
        s.last_v[g] = 0.0;
        s.nres[g] = 0;
        s.nsteps[g] = 0;
        s.rhead[g] = 0;
        s.rcnt[g] = 0;
        s.peak[g] = 0;
        s.has_step[g] = 0;
        double pw = __dadd_rn(cf.p_idle_w, __dmul_rn(__dsub_rn(cf.p_max_w, cf.p_idle_w), 0.0));
        if (0.0 > cf.boost_threshold) pw = __dadd_rn(pw, cf.p_boost_w);
        s.power[g] = pw;
    }
    for (uint32_t k = lane; k < cap.S; k += 32) s.free_stack[k] = cap.S - 1 - k;
    __syncwarp();

    Sc c;
    c.now = 0.0;
    c.deadline = 0.0;
    c.seq_next = T;
    c.arrived = 0;
    c.mq_head = 0;
    c.rq_head = 0;
    c.rq_cnt = 0;
    c.hsize = 0;
    c.nfree = cap.S;
    c.rr_cursor = 0;
    c.oom = 0;
    c.events = 0;
    c.status = 0;
    const uint64_t max_events = 1000ull * T + 1000000ull;

    for (;;) {
        // Next event: arrival stream (seq = index) vs heap top.
        const bool have_arr = c.arrived < T;
        const bool have_heap = c.hsize > 0;
        if (!have_arr && !have_heap) break;
        if (c.events >= max_events) {
            c.status = CARMA_ERR_INCOMPLETE;
            break;
        }
        double t;
        uint32_t kind, payload, seq = 0;
        const double at = have_arr ? jb.tasks[c.arrived].submit : 0.0;
        if (have_arr && (!have_heap || !later(at, c.arrived, s.ht[0], s.hs[0]))) {
            t = at;
            kind = 0;
            payload = c.arrived;
        } else {
            t = s.ht[0];
            seq = s.hs[0];
            const uint32_t info = s.hinfo[0];
            kind = info >> 30;
            payload = info & 0x3fffffffu;
            heap_pop(s, c);
        }
        __syncwarp();
        c.events++;
        // integrate_to (world.cpp:37-44)
        const double dt = __dsub_rn(t, c.now);
        if (dt > 0.0) {
#pragma unroll
            for (int jj = 0; jj < GPL; ++jj) {
                const int g = static_cast<int>(lane) + 32 * jj;
                if (g < G) s.energy[g] = __dadd_rn(s.energy[g], __dmul_rn(s.power[g], dt));
            }
        }
        c.now = t;
        if (kind == 0) {
            c.arrived++;  // Manager::submit: joins the main queue
            try_schedule<GPL>(s, c, cap, jb, p.est_override, static_cast<uint32_t>(tb), lane);
        } else if (kind == kKindWindow) {
            if (t == c.deadline) try_schedule<GPL>(s, c, cap, jb, p.est_override, static_cast<uint32_t>(tb), lane);
        } else if (kind == kKindCompletion) {
            if (s.s_seq[payload] != seq) continue;  // superseded by a rate change
            finish(s, c, cap, jb, payload, lane);
            if (!c.status) try_schedule<GPL>(s, c, cap, jb, p.est_override, static_cast<uint32_t>(tb), lane);
        } else {
            // oom_crash -> handle_oom (manager.cpp:262-267)
            c.oom++;
            if (lane == 0) {
                carma_task_result& o = jb.out[payload];
                o.ooms += 1;
                if (o.first_crash < 0.0) o.first_crash = c.now;
                o.last_crash = c.now;
            }
            if (c.rq_cnt >= cap.RQ) {
                c.status = kStatusRetry;
            } else {
                uint32_t tail = c.rq_head + c.rq_cnt;
                if (tail >= cap.RQ) tail -= cap.RQ;
                s.rq[tail] = payload;
                c.rq_cnt++;
                __syncwarp();
                try_schedule<GPL>(s, c, cap, jb, p.est_override, static_cast<uint32_t>(tb), lane);
            }
        }
        if (c.status) break;
        __syncwarp();
    }
    __syncwarp();
    carma_trace_result& tr = p.trace_out[j];
    if (c.status == kStatusRetry) {
        if (lane == 0) {
            tr.status = kStatusRetry;
            const uint32_t k = atomicAdd(p.retry_count, 1u);
            p.retry_list[k] = j;
        }
        return;
    }

    // ---- runner tail (runner.cpp:97-141) and compute_report (metrics.cpp:16-70)
    double lc = 0.0;
    bool complete = true;
    for (uint32_t i = lane; i < T; i += 32) {
        carma_task_result& o = jb.out[i];
        const double cpl = o.complete;
        lc = lc < cpl ? cpl : lc;  // std::max(last_complete, t.complete)
        complete = complete && cpl >= 0.0;
        o.attempts = o.ooms + (o.final_dispatch >= 0.0 ? 1u : 0u);
        inv[jb.tasks[i].rank] = i;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, lc, o);
        lc = lc < x ? x : lc;
    }
    complete = __all_sync(0xffffffffu, complete);
    if (c.status == 0 && !complete) c.status = CARMA_ERR_INCOMPLETE;
    const double span = __dsub_rn(lc, fs);
    const double begin_actual = dmax0(__dsub_rn(lc, span));
    if (c.status == 0 && span > 0.0 && !(forced == forced) && begin_actual != jb.begin0) {
        // Re-run with the true window begin (see file header).
        if (lane == 0) {
            p.smact_begin[j] = begin_actual;
            tr.status = kStatusRedoSmact;
            const uint32_t k = atomicAdd(p.retry_count, 1u);
            p.retry_list[k] = j;
        }
        return;
    }
    const double overshoot = __dsub_rn(c.now, lc);
    double energy = 0.0;
    for (int g = 0; g < G; ++g) {
        double e = s.energy[g];
        if (overshoot > 0.0) e = __dsub_rn(e, __dmul_rn(s.power[g], overshoot));
        energy = __dadd_rn(energy, e);
        if ((g & 31) == static_cast<int>(lane)) {
            carma_gpu_result r;
            r.energy_j = e;
            double mean = 0.0;
            if (span > 0.0) {
                const double integral = __dadd_rn(s.integ[g], __dmul_rn(s.lvl[g], __dsub_rn(lc, s.cur[g])));
                mean = __ddiv_rn(integral, span);
            }
            r.mean_smact = mean;
            r.peak_used = static_cast<uint64_t>(s.peak[g]) * cf.alloc_block;
            r.smact_steps = s.nsteps[g];
            gout[g] = r;
        }
    }
    __syncwarp();
    // Sums in id (rank) order: each lane stages 32 values, lane order is rank order.
    double ws = 0.0, es = 0.0, js = 0.0;
    for (uint32_t base = 0; base < T; base += 32) {
        const uint32_t r = base + lane;
        double w = 0.0, e = 0.0, jc = 0.0;
        if (r < T) {
            const uint32_t i = inv[r];
            const double sub = jb.tasks[i].submit;
            const double fd = jb.out[i].final_dispatch, cp = jb.out[i].complete;
            w = __dsub_rn(fd, sub);
            e = __dsub_rn(cp, fd);
            jc = __dsub_rn(cp, sub);
        }
        const uint32_t cnt = min(32u, T - base);
        for (uint32_t l = 0; l < cnt; ++l) {
            ws = __dadd_rn(ws, __shfl_sync(0xffffffffu, w, l));
            es = __dadd_rn(es, __shfl_sync(0xffffffffu, e, l));
            js = __dadd_rn(js, __shfl_sync(0xffffffffu, jc, l));
        }
    }
    if (lane == 0) {
        const double nd = static_cast<double>(T);
        carma_trace_result r;
        r.trace_total_time = span;
        r.avg_wait = __ddiv_rn(ws, nd);
        r.avg_exec = __ddiv_rn(es, nd);
        r.avg_jct = __ddiv_rn(js, nd);
        r.energy_mj = __ddiv_rn(energy, 1e6);
        r.first_submit = fs;
        r.last_complete = lc;
        r.end_time = c.now;
        r.oom_count = c.oom;
        r.status = c.status;
        r.events = c.events;
        tr = r;
    }
}

template <int GPL, bool SMEM>
__global__ void __launch_bounds__(128) replay_kernel(ReplayParams p) {
    extern __shared__ __align__(16) char smem[];
    const unsigned lane = threadIdx.x & 31;
    const unsigned wib = threadIdx.x >> 5;
    const unsigned gw = blockIdx.x * (blockDim.x >> 5) + wib;
    char* base = SMEM ? smem + static_cast<size_t>(wib) * p.state_bytes
                      : p.gstate + static_cast<size_t>(gw) * p.state_bytes;
    St s;
    layout_bytes(p.caps, &s, base);
    for (;;) {
        unsigned k = 0;
        if (lane == 0) k = atomicAdd(p.next_job, 1u);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= p.n_list) break;
        run_job<GPL>(s, p.caps, p, p.job_list[k], lane);
        __syncwarp();
    }
}

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
    DeviceBuffer d_cfgs, d_tasks, d_trace_off, d_jobs, d_task_off, d_gpu_off, d_list, d_task_out,
        d_trace_out, d_gpu_out, d_inv, d_begin, d_retry, d_counters, d_gstate;
    const uint64_t* est_override = nullptr;
    uint64_t launches = 0, retried = 0;
    std::mutex mu;
};

namespace {

Caps caps_for(int max_g, int max_blocks, bool big) {
    Caps c;
    c.G = static_cast<uint32_t>(max_g);
    c.W = static_cast<uint32_t>((max_blocks + 63) / 64);
    if (!big) {
        c.H = 64;
        c.S = 32;
        c.RC = 24;
        c.RG = 16;
        c.RQ = 16;
    } else {
        c.H = 8192;
        c.S = 2048;
        c.RC = 256;
        c.RG = 256;
        c.RQ = 4096;
    }
    return c;
}

void validate_config(const carma_replay_config& c) {
    if (c.mode == CARMA_MODE_MIG) throw Unsupported("MIG collocation is not supported by the replay kernel");
    if (c.mode != CARMA_MODE_MPS && c.mode != CARMA_MODE_STREAMS) throw InvalidArg("unknown collocation mode");
    if (c.policy < CARMA_POLICY_EXCLUSIVE || c.policy > CARMA_POLICY_MUG) throw InvalidArg("unknown policy");
    if (c.gpu_count < 1 || c.gpu_count > CARMA_MAX_GPUS) throw Unsupported("gpu_count must be in [1, 64]");
    if (!(c.monitor_window > 0.0)) throw InvalidArg("ConfigError: window must be > 0");
    if (c.alloc_block == 0) throw Unsupported("alloc_block = 0 is not supported");
    if (c.gpu_capacity % c.alloc_block != 0)
        throw Unsupported("gpu_capacity must be a multiple of alloc_block");
    if (c.gpu_capacity / c.alloc_block > 256) throw Unsupported("more than 256 allocation blocks per GPU");
    if (c.gpu_capacity / c.alloc_block > 65535) throw Unsupported("too many blocks");
}

void launch_tier(ReplayPlan& pl, const ReplayParams& base, const uint32_t* list_dev, uint32_t n_list,
                 bool big) {
    int max_blocks = 1;
    for (const auto& c : pl.cfgs) max_blocks = std::max<int>(max_blocks, static_cast<int>(c.gpu_capacity / c.alloc_block));
    ReplayParams p = base;
    p.caps = caps_for(pl.max_g, max_blocks, big);
    p.job_list = list_dev;
    p.n_list = n_list;
    p.state_bytes = layout_bytes(p.caps, nullptr, nullptr);
    uint32_t* counters = pl.d_counters.as<uint32_t>();
    p.next_job = counters;          // [0]
    p.retry_count = counters + 1;   // [1]
    CARMA_CUDA(cudaMemsetAsync(counters, 0, 8, pl.stream));
    const bool gpl2 = pl.max_g > 32;
    int sms = 148;
    CARMA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pl.device));
    if (!big) {
        const int warps_per_cta = 4;
        const size_t shmem = p.state_bytes * warps_per_cta;
        auto kern = gpl2 ? replay_kernel<2, true> : replay_kernel<1, true>;
        CARMA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(shmem)));
        int per_sm = 0;
        CARMA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, shmem));
        if (per_sm < 1) throw Unsupported("replay state does not fit in shared memory");
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(
            static_cast<uint64_t>(per_sm) * sms, (n_list + warps_per_cta - 1) / warps_per_cta));
        kern<<<grid, 128, shmem, pl.stream>>>(p);
    } else {
        const unsigned warps = static_cast<unsigned>(std::min<uint64_t>(n_list, static_cast<uint64_t>(sms) * 8));
        const unsigned grid = (warps + 3) / 4;
        pl.d_gstate.ensure(static_cast<size_t>(grid) * 4 * p.state_bytes);
        p.gstate = pl.d_gstate.as<char>();
        auto kern = gpl2 ? replay_kernel<2, false> : replay_kernel<1, false>;
        kern<<<grid, 128, 0, pl.stream>>>(p);
    }
    CARMA_CUDA(cudaGetLastError());
    pl.launches++;
}

void run_plan(ReplayPlan& pl) {
    ReplayParams p{};
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
    const uint32_t n = static_cast<uint32_t>(pl.jobs.size());
    uint32_t* list = pl.d_list.as<uint32_t>();      // [0, n): all jobs
    uint32_t* retry = list + n;                     // [n, 2n): retry list
    p.retry_list = retry;
    pl.launches = 0;
    pl.retried = 0;
    // NaN begin = derive from first_submit.
    CARMA_CUDA(cudaMemsetAsync(pl.d_begin.ptr, 0xff, n * sizeof(double), pl.stream));
    launch_tier(pl, p, list, n, false);
    uint32_t n_retry = 0;
    CARMA_CUDA(cudaMemcpyAsync(&n_retry, pl.d_counters.as<uint32_t>() + 1, 4, cudaMemcpyDeviceToHost, pl.stream));
    CARMA_CUDA(cudaStreamSynchronize(pl.stream));
    // Overflowed or begin-corrected jobs: re-run in the large global-memory
    // tier (at most twice: a begin correction can follow an overflow).
    for (int round = 0; round < 2 && n_retry > 0; ++round) {
        pl.retried += n_retry;
        std::vector<uint32_t> ids(n_retry);
        CARMA_CUDA(cudaMemcpy(ids.data(), retry, n_retry * 4, cudaMemcpyDeviceToHost));
        CARMA_CUDA(cudaMemcpy(list, ids.data(), n_retry * 4, cudaMemcpyHostToDevice));
        launch_tier(pl, p, list, n_retry, true);
        CARMA_CUDA(cudaMemcpyAsync(&n_retry, pl.d_counters.as<uint32_t>() + 1, 4, cudaMemcpyDeviceToHost, pl.stream));
        CARMA_CUDA(cudaStreamSynchronize(pl.stream));
    }
    // restore the full job list for the next run
    if (pl.retried) {
        std::vector<uint32_t> all(n);
        for (uint32_t i = 0; i < n; ++i) all[i] = i;
        CARMA_CUDA(cudaMemcpy(list, all.data(), n * 4, cudaMemcpyHostToDevice));
    }
}

}  // namespace
}  // namespace carma_b200

using namespace carma_b200;

extern "C" {

carma_status carma_replay_plan_create(int device, const carma_replay_config* configs, uint32_t n_configs,
                                      const carma_task* tasks, const uint64_t* trace_offsets, uint32_t n_traces,
                                      const carma_replay_job* jobs, uint32_t n_jobs, int32_t want_task_results,
                                      carma_replay_plan** out) {
    (void)want_task_results;
    return guarded([&] {
        if (!out || !configs || !tasks || !trace_offsets || !jobs) throw InvalidArg("null argument");
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
            }
            for (uint32_t t = 0; t < n_traces; ++t) {
                if (trace_offsets[t + 1] <= trace_offsets[t]) throw InvalidArg("ConfigError: trace contains no tasks");
                if (trace_offsets[t + 1] - trace_offsets[t] > (1u << 30)) throw Unsupported("trace too long");
            }
            for (uint64_t i = 0; i < pl->n_tasks; ++i) {
                if (tasks[i].gpus < 1 || tasks[i].gpus > 2) throw Unsupported("gpus_requested must be 1 or 2");
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
            auto up = [&](DeviceBuffer& b, const void* src, size_t bytes) {
                b.ensure(bytes);
                CARMA_CUDA(cudaMemcpy(b.ptr, src, bytes, cudaMemcpyHostToDevice));
            };
            up(pl->d_cfgs, configs, n_configs * sizeof(carma_replay_config));
            up(pl->d_tasks, tasks, pl->n_tasks * sizeof(carma_task));
            up(pl->d_trace_off, trace_offsets, (n_traces + 1) * sizeof(uint64_t));
            up(pl->d_jobs, jobs, n_jobs * sizeof(carma_replay_job));
            up(pl->d_task_off, task_off.data(), n_jobs * sizeof(uint64_t));
            up(pl->d_gpu_off, gpu_off.data(), n_jobs * sizeof(uint64_t));
            std::vector<uint32_t> list(2 * static_cast<size_t>(n_jobs));
            for (uint32_t i = 0; i < n_jobs; ++i) list[i] = i;
            up(pl->d_list, list.data(), list.size() * 4);
            pl->d_task_out.ensure(to * sizeof(carma_task_result));
            pl->d_trace_out.ensure(n_jobs * sizeof(carma_trace_result));
            pl->d_gpu_out.ensure(go * sizeof(carma_gpu_result));
            pl->d_inv.ensure(to * 4);
            pl->d_begin.ensure(n_jobs * sizeof(double));
            pl->d_counters.ensure(16);
        } catch (...) {
            if (pl->stream) cudaStreamDestroy(pl->stream);
            delete pl;
            throw;
        }
        *out = reinterpret_cast<carma_replay_plan*>(pl);
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

carma_status carma_replay_plan_destroy(carma_replay_plan* hp) {
    return guarded([&] {
        auto* pl = reinterpret_cast<ReplayPlan*>(hp);
        if (!pl) return;
        {
            DeviceGuard guard(pl->device);
            cudaStreamSynchronize(pl->stream);
            DeviceBuffer* bufs[] = {&pl->d_cfgs, &pl->d_tasks, &pl->d_trace_off, &pl->d_jobs, &pl->d_task_off,
                                    &pl->d_gpu_off, &pl->d_list, &pl->d_task_out, &pl->d_trace_out, &pl->d_gpu_out,
                                    &pl->d_inv, &pl->d_begin, &pl->d_retry, &pl->d_counters, &pl->d_gstate};
            for (auto* b : bufs) b->release();
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

carma_status carma_pick_batch(int device, const carma_replay_config* cfg, const carma_gpu_view* views,
                              uint32_t n_gpus, const carma_pick_request* reqs, uint64_t n, int32_t* rr_cursor,
                              int32_t* out_gpus) {
    return guarded([&] {
        if (!cfg || !views || !reqs || !rr_cursor || !out_gpus) throw InvalidArg("null argument");
        if (n_gpus < 1 || n_gpus > CARMA_MAX_GPUS) throw Unsupported("n_gpus must be in [1, 64]");
        if (n == 0) return;
        for (uint64_t i = 0; i < n; ++i)
            if (reqs[i].want < 1 || reqs[i].want > 2) throw Unsupported("want must be 1 or 2");
        require_device(device);
        DeviceGuard guard(device);
        carma_replay_config c = *cfg;
        c.gpu_count = static_cast<int32_t>(n_gpus);
        DeviceBuffer dv, dr, dc, dout;
        dv.ensure(n * n_gpus * sizeof(carma_gpu_view));
        dr.ensure(n * sizeof(carma_pick_request));
        dc.ensure(n * 4);
        dout.ensure(n * 8);
        CARMA_CUDA(cudaMemcpy(dv.ptr, views, n * n_gpus * sizeof(carma_gpu_view), cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(dr.ptr, reqs, n * sizeof(carma_pick_request), cudaMemcpyHostToDevice));
        CARMA_CUDA(cudaMemcpy(dc.ptr, rr_cursor, n * 4, cudaMemcpyHostToDevice));
        unsigned width = 1;
        while (width < n_gpus && width < 32) width <<= 1;
        const unsigned groups_per_warp = 32 / width;
        const uint64_t warps = (n + groups_per_warp - 1) / groups_per_warp;
        const unsigned grid = grid_for(warps * 32, 256, 148u * 16u);
        if (n_gpus > 32)
            pick_kernel<2><<<grid, 256>>>(c, dv.as<carma_gpu_view>(), n_gpus, dr.as<carma_pick_request>(), n,
                                          dc.as<int32_t>(), dout.as<int32_t>(), width);
        else
            pick_kernel<1><<<grid, 256>>>(c, dv.as<carma_gpu_view>(), n_gpus, dr.as<carma_pick_request>(), n,
                                          dc.as<int32_t>(), dout.as<int32_t>(), width);
        CARMA_CUDA(cudaGetLastError());
        CARMA_CUDA(cudaMemcpy(out_gpus, dout.ptr, n * 8, cudaMemcpyDeviceToHost));
        CARMA_CUDA(cudaMemcpy(rr_cursor, dc.ptr, n * 4, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
