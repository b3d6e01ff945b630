// Stage 2 device code: the warp-per-job replay kernel.
//
// One warp replays one (trace, config) job end to end: the deterministic
// discrete-event loop of World (proj/src/world.cpp:31-186) driving the CARMA
// Manager pipeline (proj/src/manager.cpp:58-357) over simulated GpuDevices in
// MPS / streams mode (proj/src/gpu.cpp:58-274), then the runner tail
// (runner.cpp:97-141) and compute_report's scalars (metrics.cpp:16-70).
// Bit-identical to the reference: built with --fmad=false, every
// floating-point expression keeps the reference's operation order.
//
// Warp organisation. Sequential event logic (queue heads, the event heap,
// dispatch decisions, rate refresh) runs warp-uniformly — every lane computes
// the same values — while per-GPU work is lane-parallel: lane l owns
// simulated GPUs l and l+32. Energy integration, windowed SMACT, feasibility
// and the MAGM/LUG/MUG arg-reductions (pick.cuh) take one step across the
// lanes; the first-fit allocator runs on the owner lane's bitmap.
//
// Code shape. The event loop is flat: the handlers for the four event kinds
// only set flags, and try_schedule / place / finish / refresh_rates each
// occur once in the instruction stream (a fully inlined version thrashed the
// instruction cache: 84% of stall samples were no_instructions). The state
// layout is a compile-time struct of offsets from one per-warp base pointer,
// so no register holds a layout pointer.
//
// State (per warp; shared memory for the two common tiers, global memory for
// the large tier):
//   * per GPU (SoA): allocation bitmap (block = SimConstants::alloc_block),
//     cached per-resident rate / instantaneous SMACT / power, energy, peak,
//     the resident list in insertion order, a ring of recent SMACT steps for
//     windowed_smact, and a running integrator that reproduces the
//     full-history windowed_smact(last_complete, span) of runner.cpp:135-137
//     term by term;
//   * resident-task slots (remaining work, rate, last update, live event seq);
//   * a binary min-heap of dynamic events ordered by (t, seq); arrivals are a
//     pre-sorted stream with seq = trace index (runner.cpp:72-78), merged at pop;
//   * the main queue is the index range [mq_head, arrived) (FIFO,
//     manager.cpp:58-78); the recovery queue is a ring.
// A completion event is live iff its seq equals its slot's live seq — the
// same test as TaskRun::gen (world.cpp:52-57), since every reschedule draws a
// fresh seq. Any capacity overflow aborts the job in its tier and the host
// re-runs it in the global-memory tier.
#pragma once

#include <cstdint>

#include "../../../include/carma_gpu.h"
#include "pick.cuh"

namespace carma_b200 {
namespace replay {

// Shared-memory tiers: 72 registers, 7 CTAs x 4 warps resident (throughput
// of many jobs; c4 on B200: 8 CTAs / 64 registers 139.1 ms, 7 / 72 125.5,
// 6 / 74 125.9, 5 / 81 134.4, 4 / 91 133.5, 9 / 56 (spills) 153.3). The large
// tier (one long trace per warp, latency bound) and the global tier take all
// the registers they want.
#ifndef REPLAY_KLATER_CHAIN
#define REPLAY_KLATER_CHAIN 1
#endif
#ifndef REPLAY_MIN_CTAS
#define REPLAY_MIN_CTAS 7
#endif

#ifndef REPLAY_PROF
#define REPLAY_PROF 0
#endif
#if REPLAY_PROF
// Diagnostic builds only (-DREPLAY_PROF=1): clock64 cycles per event-loop
// region, summed over jobs: 0 next event, 1 integrate, 2 handle, 3 refresh,
// 4 decide, 5 place, 6 push, 7 events.
__device__ unsigned long long g_replay_prof[16];
// sub-regions: 0 refresh_gpu, 1 affected list + sort, 2 re-push loop,
// 3 decide gate / head, 4 decide inputs (free, SMACT), 5 decide pick
__device__ unsigned long long g_replay_sub[8];
#define RSUB_T(v) const long long v = clock64()
#define RSUB_ADD(r, a, b) if ((threadIdx.x & 31) == 0) atomicAdd(&g_replay_sub[r], static_cast<unsigned long long>((b) - (a)))
#define RPROF_T(v) const long long v = clock64()
#define RPROF_ADD(r, t0) prof[r] += static_cast<unsigned long long>(clock64() - (t0))
#else
#define RPROF_T(v)
#define RPROF_ADD(r, t0)
#define RSUB_T(v)
#define RSUB_ADD(r, a, b)
#endif

constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kWindow = 1u, kCompletion = 2u, kCrash = 3u, kTick = 4u;
constexpr int32_t kStatusRetry = -1;      // overflowed this tier
constexpr int32_t kStatusRedoSmact = -2;  // full-history SMACT needs the true window begin
constexpr int kMaxWords = 64;             // bitmap words per GPU: <= 4096 blocks (wide global tier)

struct Params {
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
    uint32_t* inv_scratch;   // rank -> index, indexed like task_out
    double* smact_begin;     // per job; NaN = derive from first_submit
    uint32_t* retry_list;    // jobs that overflowed this tier
    uint32_t* retry_count;
    unsigned int* next_job;  // dynamic scheduler counter
    char* gstate;            // global-tier state, per warp
    carma_timeline_row* tl_out;  // timeline rows, tl_cap per job (TL kernels only)
    uint64_t tl_cap;
    uint64_t* tl_count;          // rows produced, per job
    carma_log_record* log_out;   // event / decision log records, log_cap per job (TL kernels only)
    uint64_t log_cap;
    uint64_t* log_count;         // records produced, per job
    carma_task_outcome* outcome_sink;  // nullable: per-task outcomes written straight to pinned host memory
};

// alloc_oom details of a failed placement (OomFailure, gpu.hpp:26-35), in
// blocks (bitmap allocator) or bytes (segment allocator: *_b).
struct OomInfo {
    int gpu;
    uint32_t free_blk, largest_blk;
    uint64_t free_b, largest_b;
};

// Compile-time state layout: G GPUs, H heap entries, S slots, RC residents
// per GPU, RG SMACT ring entries per GPU, RQ recovery-queue entries.
// F = feature bits compiled into the kernel: 1 = MIG collocation, 2 = timeline
// sample ticks. Jobs that need them run in their own kernel instantiations.
template <int G_, int H_, int S_, int RC_, int RG_, int RQ_, int W_, int F_ = 0>
struct Layout {
    static constexpr int G = G_, H = H_, S = S_, RC = RC_, RG = RG_, RQ = RQ_, W = W_;
    static constexpr bool MIG = (F_ & 1) != 0;
    static constexpr bool TL = (F_ & 2) != 0;  // diagnostics: timeline ticks and/or event/decision logs
    // Event queue: a sorted ring (O(1) pop, warp-parallel insert) for the
    // long-trace tiers, a 4-ary heap for the short-trace tiers.
    static constexpr bool SQ = H_ >= 1024;
    // F bit 4: tasks may request up to 8 GPUs (multi-GPU jobs run in their
    // own global-tier instantiations); the slot keeps its full GPU list.
    // The generic instantiations (F bit 4) also carry the reference's
    // byte-granular segment allocator (gpu.cpp:58-130), chosen per config at
    // run time for alloc_block = 0, capacities that are not a block multiple
    // and more than 4096 blocks.
    static constexpr bool MG = (F_ & 4) != 0;
    static constexpr int WM = MG ? CARMA_MAX_TASK_GPUS : 2;
    static constexpr size_t MGI = MG ? 1 : 0;
    static constexpr int NSEG = 2 * RC_ + 2;  // segments per GPU: <= 2 x live allocations + 1
    static constexpr size_t MI = MIG ? 1 : 0;
    static constexpr int GPL = (G + 31) / 32;
    static constexpr size_t al8(size_t x) { return (x + 15) / 16 * 16; }
    static constexpr size_t cfg = 0;                                   // carma_replay_config
    static constexpr size_t used = al8(cfg + sizeof(carma_replay_config));  // u64 [W][G]
    static constexpr size_t energy = al8(used + 8ull * W * G);    // f64 [G] x 9
    static constexpr size_t rate = energy + 8ull * G;
    static constexpr size_t inst = rate + 8ull * G;
    static constexpr size_t power = inst + 8ull * G;
    static constexpr size_t lvl = power + 8ull * G;
    static constexpr size_t cur = lvl + 8ull * G;
    static constexpr size_t integ = cur + 8ull * G;
    static constexpr size_t last_t = integ + 8ull * G;
    static constexpr size_t last_v = last_t + 8ull * G;
    static constexpr size_t ring_t = al8(last_v + 8ull * G);           // f64 [G][RG]
    static constexpr size_t ring_v = ring_t + 8ull * G * RG;
    static constexpr size_t ht = al8(ring_v + 8ull * G * RG);          // HeapEnt [H] (16 B each)
    static constexpr size_t s_rem = ht + 16ull * H;                    // f64 [S] x 5
    static constexpr size_t s_rate = s_rem + 8ull * S;
    static constexpr size_t s_last = s_rate + 8ull * S;
    static constexpr size_t s_exec = s_last + 8ull * S;
    static constexpr size_t s_dem = s_exec + 8ull * S;
    static constexpr size_t aff = s_dem + 8ull * S;                    // u64 [WM RC] x 2
    static constexpr size_t aff2 = aff + 8ull * WM * RC;
    static constexpr size_t nres = aff2 + 8ull * WM * RC;              // u32 [G] x 7
    static constexpr size_t nsteps = nres + 4ull * G;
    static constexpr size_t rhead = nsteps + 4ull * G;
    static constexpr size_t rcnt = rhead + 4ull * G;
    static constexpr size_t peak = rcnt + 4ull * G;
    static constexpr size_t has_step = peak + 4ull * G;
    static constexpr size_t imask = has_step + 4ull * G;               // MIG: occupied instances
    static constexpr size_t s_task = imask + 4ull * G * MI;            // u32 [S] x 7
    static constexpr size_t s_rank = s_task + 4ull * S;
    static constexpr size_t s_seq = s_rank + 4ull * S;
    static constexpr size_t s_gp = s_seq + 4ull * S;
    static constexpr size_t s_off = s_gp + 4ull * S;
    static constexpr size_t s_nb = s_off + 4ull * S;
    static constexpr size_t s_inst = s_nb + 4ull * S;                  // MIG: inst0 | inst1 << 8
    static constexpr size_t s_gl = s_inst + 4ull * S * MI;             // MG: u8 [S][WM] GPU ids
    static constexpr size_t s_il = s_gl + 1ull * S * WM * MGI;         // MG + MIG: u8 [S][WM] instances
    static constexpr size_t s_ol = al8(s_il + 1ull * S * WM * MGI * MI);  // MG: u16 [S][WM] block offsets
    static constexpr size_t s_ob = al8(s_ol + 2ull * S * WM * MGI);   // MG: u64 [S][WM] byte offsets (segments)
    static constexpr size_t s_wb = s_ob + 8ull * S * WM * MGI;        // MG: u64 [S] bytes per device (segments)
    static constexpr size_t seg_off = s_wb + 8ull * S * MGI;          // MG: u64 [G][NSEG] segment offsets
    static constexpr size_t seg_len = seg_off + 8ull * G * NSEG * MGI;  // u64 [G][NSEG] size | used << 63
    static constexpr size_t seg_n = seg_len + 8ull * G * NSEG * MGI;    // u32 [G]
    static constexpr size_t seg_free = al8(seg_n + 4ull * G * MGI);   // u64 [G] total free bytes
    static constexpr size_t seg_peak = seg_free + 8ull * G * MGI;     // u64 [G] peak used bytes
    static constexpr size_t free_stack = al8(seg_peak + 8ull * G * MGI);  // u32 [S]
    static constexpr size_t rq = free_stack + 4ull * S;                // u32 [RQ]
    static constexpr size_t res = rq + 4ull * RQ;                      // u16 [G][RC]
    static constexpr size_t ptrs = al8(res + 2ull * G * RC);          // tasks, out, est, nblk (warp-uniform)
    static constexpr size_t bytes = ptrs + 32;
};

#define RP_F64(f) reinterpret_cast<double*>(b + L::f)
#define RP_U32(f) reinterpret_cast<uint32_t*>(b + L::f)
#define RP_U64(f) reinterpret_cast<uint64_t*>(b + L::f)
#define RP_U16(f) reinterpret_cast<uint16_t*>(b + L::f)
#define RP_CFG (*reinterpret_cast<const carma_replay_config*>(b + L::cfg))

__device__ __forceinline__ double dmax0(double x) { return 0.0 < x ? x : 0.0; }      // std::max(0.0, x)
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min(a, b)
__device__ __forceinline__ bool later(double ta, uint32_t sa, double tb, uint32_t sb) {
    return ta != tb ? ta > tb : sa > sb;
}

// Warp-uniform scalar state (replicated in every lane).
struct Sc {
    double now, deadline, window, begin0;
    uint32_t seq_next, arrived, mq_head, rq_head, rq_cnt, hsize, hhead, nfree, T;
    int rr_cursor;
    int32_t oom, status;
    uint32_t events_lo, events_hi;
};

// ---------------------------------------------------------------- heap
// 4-ary min-heap on (time, seq). Times are stored as order-preserving u64
// keys (same order as the doubles; +0 and -0 collapse), so sifting uses
// integer compares instead of long-latency fp64 compares.
__device__ __forceinline__ uint64_t tkey(double t) {
    if (t == 0.0) t = 0.0;
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(t));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double tval(uint64_t k) {
    const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(u));
}
// (ka, sa) > (kb, sb) lexicographically, as the borrow of the 96-bit
// subtraction (kb:sb) - (ka:sa): one carry chain instead of compare-and-select.
__device__ __forceinline__ bool klater(uint64_t ka, uint32_t sa, uint64_t kb, uint32_t sb) {
#if REPLAY_KLATER_CHAIN
    uint32_t r;
    asm("{\n\t.reg .u32 t;\n\t"
        "sub.cc.u32 t, %2, %1;\n\t"
        "subc.cc.u32 t, %4, %3;\n\t"
        "subc.cc.u32 t, %6, %5;\n\t"
        "subc.u32 %0, 0, 0;\n\t}"
        : "=r"(r)
        : "r"(sa), "r"(sb), "r"(static_cast<uint32_t>(ka)), "r"(static_cast<uint32_t>(kb)),
          "r"(static_cast<uint32_t>(ka >> 32)), "r"(static_cast<uint32_t>(kb >> 32)));
    return r != 0;
#else
    return ka != kb ? ka > kb : sa > sb;
#endif
}

// One heap entry: order key, seq and payload in 16 bytes, so a child or
// parent moves with one 16-byte shared-memory load / store.
struct __align__(16) HeapEnt {
    uint64_t key;
    uint32_t seq;
    uint32_t info;
};

// The earliest pending event (the queue is non-empty).
template <class L>
__device__ __forceinline__ const HeapEnt& heap_top(const char* b, const Sc& c) {
    return reinterpret_cast<const HeapEnt*>(b + L::ht)[L::SQ ? c.hhead : 0];
}

template <class L>
__device__ __forceinline__ uint32_t heap_push(char* b, Sc& c, double t, uint32_t info) {
    if (c.hsize >= static_cast<uint32_t>(L::H)) {
        c.status = kStatusRetry;
        return kNone;
    }
    HeapEnt* h = reinterpret_cast<HeapEnt*>(b + L::ht);
    HeapEnt e;
    e.key = tkey(t);
    e.seq = c.seq_next++;
    e.info = info;
    if constexpr (L::SQ) {
        // Sorted ring [hhead, hhead + hsize): the new event has the largest
        // seq so far, so it goes after every entry whose key is <= its key.
        // The lanes find that position in parallel, then shift the shorter
        // side by one slot, 32 entries at a time.
        const unsigned lane = threadIdx.x & 31;
        const uint32_t n = c.hsize, hd = c.hhead;
        auto at = [&](uint32_t i) {
            const uint32_t x = hd + i;
            return x >= static_cast<uint32_t>(L::H) ? x - static_cast<uint32_t>(L::H) : x;
        };
        // two parallel probes: 32 evenly spaced samples pick the segment,
        // then the segment's entries (<= 32 at a time) give the position
        const uint32_t stride = (n + 31) >> 5;
        const uint32_t si = lane * stride;
        const unsigned below = __ballot_sync(0xffffffffu, si < n && h[at(si)].key <= e.key);
        uint32_t pos = 0;
        if (below) {
            const uint32_t m = static_cast<uint32_t>(__popc(below));
            const uint32_t seg_end = min(m * stride, n);
#pragma unroll 1
            for (uint32_t base = (m - 1) * stride; base < seg_end; base += 32) {
                const uint32_t i = base + lane;
                const unsigned le = __ballot_sync(0xffffffffu, i < seg_end && h[at(i)].key <= e.key);
                pos = base + static_cast<uint32_t>(__popc(le));
                if (le != 0xffffffffu) break;
            }
        }
        constexpr uint32_t H = static_cast<uint32_t>(L::H);
        if (pos < n - pos) {
            // nearer the head: move [0, pos) down one slot (the head moves
            // back), bottom chunk first
#pragma unroll 1
            for (uint32_t lo = 0; lo < pos; lo += 32) {
                const uint32_t i = lo + lane;
                HeapEnt v;
                if (i < pos) v = h[at(i)];
                __syncwarp();
                if (i < pos) {
                    const uint32_t x = at(i);
                    h[x == 0 ? H - 1 : x - 1] = v;
                }
                __syncwarp();
            }
            const uint32_t x = at(pos);
            if (lane == 0) h[x == 0 ? H - 1 : x - 1] = e;
            c.hhead = hd == 0 ? H - 1 : hd - 1;
        } else {
            // nearer the tail: move [pos, n) up one slot, top chunk first
#pragma unroll 1
            for (uint32_t hi = n; hi > pos;) {
                const uint32_t lo = hi - pos > 32 ? hi - 32 : pos;
                const uint32_t i = lo + lane;
                HeapEnt v;
                if (i < hi) v = h[at(i)];
                __syncwarp();
                if (i < hi) h[at(i + 1)] = v;
                __syncwarp();
                hi = lo;
            }
            if (lane == 0) h[at(pos)] = e;
        }
        __syncwarp();
        c.hsize = n + 1;
        return e.seq;
    }
    uint32_t i = c.hsize++;
    while (i > 0) {
        const uint32_t p = (i - 1) >> 2;
        const HeapEnt pe = h[p];
        if (!klater(pe.key, pe.seq, e.key, e.seq)) break;
        h[i] = pe;
        i = p;
    }
    h[i] = e;
    return e.seq;
}

template <class L>
__device__ __forceinline__ void heap_pop(char* b, Sc& c) {
    if constexpr (L::SQ) {
        c.hhead = c.hhead + 1 == static_cast<uint32_t>(L::H) ? 0 : c.hhead + 1;
        --c.hsize;
        return;
    }
    HeapEnt* h = reinterpret_cast<HeapEnt*>(b + L::ht);
    const uint32_t n = --c.hsize;
    if (n == 0) return;
    const HeapEnt last = h[n];
    uint32_t i = 0;
    for (;;) {
        const uint32_t c0 = 4 * i + 1;
        if (c0 >= n) break;
        uint32_t m = c0;
        HeapEnt me = h[c0];
#pragma unroll
        for (uint32_t d = 1; d < 4; ++d) {
            const uint32_t cc = c0 + d;
            if (cc < n) {
                const HeapEnt ce = h[cc];
                if (klater(me.key, me.seq, ce.key, ce.seq)) {
                    m = cc;
                    me = ce;
                }
            }
        }
        if (!klater(last.key, last.seq, me.key, me.seq)) break;
        h[i] = me;
        i = m;
    }
    h[i] = last;
}

// ------------------------------------------------------------ allocator
// Bit = 1: block used (bits past the device's block count are set).
template <class L>
__device__ __forceinline__ int next_bit(const uint64_t* used, int g, int from, int nblk, bool one) {
    for (int w = from >> 6; w < L::W; ++w) {
        uint64_t bits = used[w * L::G + g];
        if (!one) bits = ~bits;
        if (w == (from >> 6)) bits &= ~0ull << (from & 63);
        if (bits) {
            const int bit = w * 64 + __ffsll(static_cast<long long>(bits)) - 1;
            return bit < nblk ? bit : nblk;
        }
    }
    return nblk;
}

template <class L>
__device__ __forceinline__ void set_bits(uint64_t* used, int g, int off, int nb, bool on) {
#pragma unroll 1
    for (int x = off; x < off + nb;) {
        const int w = x >> 6, lo = x & 63;
        const int cnt = min(64 - lo, off + nb - x);
        const uint64_t m = (cnt == 64 ? ~0ull : ((1ull << cnt) - 1ull)) << lo;
        uint64_t& word = used[w * L::G + g];
        word = on ? (word | m) : (word & ~m);
        x += cnt;
    }
}

template <class L>
__device__ __forceinline__ uint32_t free_blocks(const uint64_t* used, int g) {
    uint32_t f = 0;
#pragma unroll
    for (int w = 0; w < L::W; ++w) f += __popcll(static_cast<long long>(~used[w * L::G + g]));
    return f;
}

// GpuDevice::allocate_range (gpu.cpp:72-114) over blocks [r0, r1): first
// fit over the device's maximal free runs clipped to the range; carve from
// the tail iff the run starts inside the range after a used block (left
// neighbour used) and does not end at a used block inside the range (right
// neighbour free or absent). The whole device is r0 = 0, r1 = nblk.
template <class L>
__device__ __forceinline__ int first_fit(char* b, int g, int nblk, int want, int r0, int r1) {
    uint64_t* used = RP_U64(used);
    int pos = 0;
    while (pos < nblk) {
        const int start = next_bit<L>(used, g, pos, nblk, false);
        if (start >= nblk || start >= r1) break;
        const int end = next_bit<L>(used, g, start, nblk, true);
        const int lo = start > r0 ? start : r0, hi = end < r1 ? end : r1;
        if (lo < hi && hi - lo >= want) {
            const bool left_used = start > 0 && start == lo;
            const bool right_used = end < nblk && end == hi;
            const int place = (left_used && !right_used) ? hi - want : lo;
            set_bits<L>(used, g, place, want, true);
            const uint32_t u = static_cast<uint32_t>(nblk) - free_blocks<L>(used, g);
            uint32_t* peak = RP_U32(peak);
            if (u > peak[g]) peak[g] = u;
            return place;
        }
        pos = end;
    }
    return -1;
}

// ------------------------------------------------ segment allocator (bytes)
// GpuDevice's segment list (gpu.cpp:58-130) for the generic instantiations:
// segments in address order, size | used << 63. Owner lane only.
constexpr uint64_t kSegUsed = 1ull << 63;

template <class L>
__device__ __forceinline__ void seg_init(char* b, int g, uint64_t capacity) {
    RP_U64(seg_off)[g * L::NSEG] = 0;
    RP_U64(seg_len)[g * L::NSEG] = capacity;
    RP_U32(seg_n)[g] = 1;
    RP_U64(seg_free)[g] = capacity;
    RP_U64(seg_peak)[g] = 0;
}

// allocate_range(r0, r1, want) with want already rounded (gpu.cpp:72-114):
// first fit over the free segments clipped to the range, carved from the end
// facing away from a live neighbour. Returns false (with the range's free
// and largest free bytes) on failure, or when the list would overflow (*ovf).
template <class L>
__device__ __forceinline__ bool seg_alloc(char* b, int g, uint64_t capacity, uint64_t r0, uint64_t r1, uint64_t want,
                                          uint64_t& off, uint64_t& tot_free, uint64_t& largest, bool& ovf) {
    uint64_t* so = RP_U64(seg_off) + g * L::NSEG;
    uint64_t* sl = RP_U64(seg_len) + g * L::NSEG;
    const uint32_t n = RP_U32(seg_n)[g];
    tot_free = largest = 0;
    ovf = false;
#pragma unroll 1
    for (uint32_t i = 0; i < n; ++i) {
        const uint64_t len = sl[i];
        if (len & kSegUsed) continue;
        const uint64_t lo = so[i] > r0 ? so[i] : r0;
        const uint64_t end = so[i] + len;
        const uint64_t hi = end < r1 ? end : r1;
        if (lo >= hi) continue;
        const uint64_t avail = hi - lo;
        tot_free += avail;
        if (avail > largest) largest = avail;
        if (avail < want) continue;
        const bool left_used = i > 0 && (sl[i - 1] & kSegUsed) && so[i] == lo;
        const bool right_used = i + 1 < n && (sl[i + 1] & kSegUsed) && end == hi;
        const uint64_t place = (left_used && !right_used) ? hi - want : lo;
        const uint32_t k = (place > so[i] ? 1u : 0u) + 1u + (place + want < end ? 1u : 0u);
        if (n + k - 1 > static_cast<uint32_t>(L::NSEG)) {
            ovf = true;
            return false;
        }
        // shift [i + 1, n) up by k - 1, then write the replacement at i
#pragma unroll 1
        for (uint32_t x = n; x-- > i + 1;) {
            so[x + k - 1] = so[x];
            sl[x + k - 1] = sl[x];
        }
        const uint64_t base = so[i];
        uint32_t w = i;
        if (place > base) {
            so[w] = base;
            sl[w++] = place - base;
        }
        so[w] = place;
        sl[w++] = want | kSegUsed;
        if (place + want < end) {
            so[w] = place + want;
            sl[w] = end - place - want;
        }
        RP_U32(seg_n)[g] = n + k - 1;
        const uint64_t fr = RP_U64(seg_free)[g] - want;
        RP_U64(seg_free)[g] = fr;
        if (capacity - fr > RP_U64(seg_peak)[g]) RP_U64(seg_peak)[g] = capacity - fr;
        off = place;
        return true;
    }
    return false;
}

// Free bytes of the segments clipped to [r0, r1) (instance_free, gpu.cpp:151-160).
template <class L>
__device__ __forceinline__ uint64_t seg_free_in_range(const char* b, int g, uint64_t r0, uint64_t r1) {
    const uint64_t* so = reinterpret_cast<const uint64_t*>(b + L::seg_off) + g * L::NSEG;
    const uint64_t* sl = reinterpret_cast<const uint64_t*>(b + L::seg_len) + g * L::NSEG;
    const uint32_t n = reinterpret_cast<const uint32_t*>(b + L::seg_n)[g];
    uint64_t f = 0;
#pragma unroll 1
    for (uint32_t i = 0; i < n; ++i) {
        if (sl[i] & kSegUsed) continue;
        const uint64_t lo = so[i] > r0 ? so[i] : r0, end = so[i] + sl[i], hi = end < r1 ? end : r1;
        if (lo < hi) f += hi - lo;
    }
    return f;
}

// free_region (gpu.cpp:116-130): mark free, coalesce right then left.
template <class L>
__device__ __forceinline__ void seg_release(char* b, int g, uint64_t off, uint64_t size) {
    uint64_t* so = RP_U64(seg_off) + g * L::NSEG;
    uint64_t* sl = RP_U64(seg_len) + g * L::NSEG;
    uint32_t n = RP_U32(seg_n)[g];
    uint32_t i = 0;
    while (i < n && !(so[i] == off && sl[i] == (size | kSegUsed))) ++i;
    if (i == n) return;
    sl[i] = size;
    RP_U64(seg_free)[g] += size;
    if (i + 1 < n && !(sl[i + 1] & kSegUsed)) {
        sl[i] += sl[i + 1];
#pragma unroll 1
        for (uint32_t x = i + 1; x + 1 < n; ++x) {
            so[x] = so[x + 1];
            sl[x] = sl[x + 1];
        }
        --n;
    }
    if (i > 0 && !(sl[i - 1] & kSegUsed)) {
        sl[i - 1] += sl[i];
#pragma unroll 1
        for (uint32_t x = i; x + 1 < n; ++x) {
            so[x] = so[x + 1];
            sl[x] = sl[x + 1];
        }
        --n;
    }
    RP_U32(seg_n)[g] = n;
}

// Free blocks in [r0, r1) (GpuDevice::instance_free, gpu.cpp:151-160).
template <class L>
__device__ __forceinline__ uint32_t free_in_range(const uint64_t* used, int g, int r0, int r1) {
    uint32_t f = 0;
#pragma unroll
    for (int w = 0; w < L::W; ++w) {
        const int lo = w * 64;
        uint64_t m = ~0ull;
        if (r0 > lo) m = r0 - lo >= 64 ? 0ull : (m & (~0ull << (r0 - lo)));
        if (r1 < lo + 64) m = r1 <= lo ? 0ull : (m & (~0ull >> (lo + 64 - r1)));
        f += __popcll(static_cast<long long>(~used[w * L::G + g] & m));
    }
    return f;
}

// Free blocks and the largest free run inside [r0, r1) (allocate_range's
// total_free_in_range / largest_free_in_range, gpu.cpp:77-86).
template <class L>
__device__ __forceinline__ void range_stats(char* b, int g, int nblk, int r0, int r1, uint32_t& free_blk,
                                            uint32_t& largest) {
    const uint64_t* used = RP_U64(used);
    free_blk = 0;
    largest = 0;
    int pos = 0;
#pragma unroll 1
    while (pos < nblk) {
        const int start = next_bit<L>(used, g, pos, nblk, false);
        if (start >= nblk || start >= r1) break;
        const int end = next_bit<L>(used, g, start, nblk, true);
        const int lo = start > r0 ? start : r0, hi = end < r1 ? end : r1;
        if (lo < hi) {
            free_blk += static_cast<uint32_t>(hi - lo);
            if (static_cast<uint32_t>(hi - lo) > largest) largest = static_cast<uint32_t>(hi - lo);
        }
        pos = end;
    }
}

// MIG instance of slot on GPU g (the slot's first or second device).
template <class L>
__device__ __forceinline__ int inst_of(const char* b, uint32_t slot, int g) {
    if constexpr (L::MG) {
        const uint8_t* gl = reinterpret_cast<const uint8_t*>(b + L::s_gl) + slot * L::WM;
        const uint8_t* il = reinterpret_cast<const uint8_t*>(b + L::s_il) + slot * L::WM;
        const int want = static_cast<int>(reinterpret_cast<const uint32_t*>(b + L::s_gp)[slot] >> 16);
        int r = 0;
        for (int k = 0; k < want; ++k)
            if (gl[k] == g) r = il[k];
        return r;
    }
    const uint32_t gp = reinterpret_cast<const uint32_t*>(b + L::s_gp)[slot];
    const uint32_t in = reinterpret_cast<const uint32_t*>(b + L::s_inst)[slot];
    return static_cast<int>(((gp & 0xff) == static_cast<uint32_t>(g) ? in : (in >> 8)) & 0xff);
}

// ----------------------------------------------------------------- SMACT
// Drops ring entries no window from `begin` on can need (an entry whose
// successor is at or before begin only sets a level the successor
// overrides): the rule record_smact applies, applied here too so a GPU that
// is not touched for a while is not rescanned over its stale steps at every
// decision. begin never decreases, so the result is unchanged. Owner lane.
template <class L>
__device__ __forceinline__ void prune_ring(char* b, int g, double begin) {
    uint32_t* rh = RP_U32(rhead);
    uint32_t* rc = RP_U32(rcnt);
    const double* rt = RP_F64(ring_t) + g * L::RG;
    uint32_t h = rh[g], n = rc[g];
    const uint32_t n_in = n;
#pragma unroll 1
    while (n >= 2) {
        const uint32_t second = h + 1 == static_cast<uint32_t>(L::RG) ? 0 : h + 1;
        if (!(rt[second] <= begin)) break;
        h = second;
        --n;
    }
    if (n != n_in) {
        rh[g] = h;
        rc[g] = n;
    }
}

// windowed_smact (gpu.cpp:244-267) over the ring of recent steps.
template <class L>
__device__ __forceinline__ double windowed(char* b, int g, double now, double window) {
    const double begin = dmax0(now - window);
    const double span = now - begin;
    if (span <= 0.0) return RP_F64(inst)[g];
    if constexpr (L::SQ) prune_ring<L>(b, g, begin);  // long-trace tiers (measured slower on c4's)
    const double* rt = RP_F64(ring_t) + g * L::RG;
    const double* rv = RP_F64(ring_v) + g * L::RG;
    double integral = 0.0, level = 0.0, cursor = begin;
    const uint32_t h = RP_U32(rhead)[g], n = RP_U32(rcnt)[g];
#pragma unroll 1
    for (uint32_t k = 0; k < n; ++k) {
        uint32_t idx = h + k;
        if (idx >= static_cast<uint32_t>(L::RG)) idx -= L::RG;
        const double t = rt[idx];
        const double v = rv[idx];
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

// windowed for a lane's two GPUs (G > 32) in lockstep: the same sums in the
// same order per GPU, but two independent dependency chains per step.
template <class L>
__device__ __forceinline__ void windowed2(char* b, int g0, int g1, bool v1, double now, double window, double& o0,
                                          double& o1) {
    const double begin = dmax0(now - window);
    const double span = now - begin;
    if (span <= 0.0) {
        o0 = RP_F64(inst)[g0];
        o1 = v1 ? RP_F64(inst)[g1] : 0.0;
        return;
    }
    if constexpr (L::SQ) {  // long-trace tiers (measured slower on c4's)
        prune_ring<L>(b, g0, begin);
        if (v1) prune_ring<L>(b, g1, begin);
    }
    const double* rt0 = RP_F64(ring_t) + g0 * L::RG;
    const double* rv0 = RP_F64(ring_v) + g0 * L::RG;
    const double* rt1 = RP_F64(ring_t) + g1 * L::RG;
    const double* rv1 = RP_F64(ring_v) + g1 * L::RG;
    double i0 = 0.0, l0 = 0.0, c0 = begin, i1 = 0.0, l1 = 0.0, c1 = begin;
    uint32_t k0 = RP_U32(rhead)[g0], n0 = RP_U32(rcnt)[g0];
    uint32_t k1 = RP_U32(rhead)[g1], n1 = v1 ? RP_U32(rcnt)[g1] : 0;
#pragma unroll 1
    while (n0 | n1) {
        if (n0) {
            const double t = rt0[k0], v = rv0[k0];
            k0 = k0 + 1 == static_cast<uint32_t>(L::RG) ? 0 : k0 + 1;
            --n0;
            if (t >= now && !(t <= begin)) {
                n0 = 0;
            } else {
                if (!(t <= begin)) i0 = __dadd_rn(i0, __dmul_rn(l0, __dsub_rn(t, c0)));
                if (!(t <= begin)) c0 = t;
                l0 = v;
            }
        }
        if (n1) {
            const double t = rt1[k1], v = rv1[k1];
            k1 = k1 + 1 == static_cast<uint32_t>(L::RG) ? 0 : k1 + 1;
            --n1;
            if (t >= now && !(t <= begin)) {
                n1 = 0;
            } else {
                if (!(t <= begin)) i1 = __dadd_rn(i1, __dmul_rn(l1, __dsub_rn(t, c1)));
                if (!(t <= begin)) c1 = t;
                l1 = v;
            }
        }
    }
    i0 = __dadd_rn(i0, __dmul_rn(l0, __dsub_rn(now, c0)));
    i1 = __dadd_rn(i1, __dmul_rn(l1, __dsub_rn(now, c1)));
    o0 = __ddiv_rn(i0, span);
    o1 = v1 ? __ddiv_rn(i1, span) : 0.0;
}

// effective_rates / instantaneous_smact / power_draw (gpu.cpp:183-229,
// 269-274) for GPU g after its resident list changed, then record_smact
// (gpu.cpp:231-242) into the ring and the full-history integrator.
// Owner lane only. Returns false on ring overflow.
template <class L>
__device__ __forceinline__ bool refresh_gpu(char* b, int g, double now, double window, double begin0) {
    const carma_replay_config& cf = RP_CFG;
    const uint32_t n = RP_U32(nres)[g];
    const uint16_t* res = RP_U16(res) + g * L::RC;
    const double* dem = RP_F64(s_dem);
    double rate = 0.0, inst = 0.0;
    if (L::MIG && n > 0) {
        // per resident min(1, f_instance / demand) (gpu.cpp:187-195); the
        // per-GPU rate cache is unused in MIG mode
        double sum = 0.0;
#pragma unroll 1
        for (uint32_t r = 0; r < n; ++r) {
            const uint32_t slot = res[r];
            const double rr = dmin(1.0, __ddiv_rn(cf.mig_fraction[inst_of<L>(b, slot, g)], dem[slot]));
            sum = __dadd_rn(sum, __dmul_rn(dem[slot], rr));
        }
        inst = dmin(1.0, sum);
    } else if (n > 0) {
        if (cf.mode == CARMA_MODE_MPS) {
            double total = 0.0;
#pragma unroll 1
            for (uint32_t r = 0; r < n; ++r) total = __dadd_rn(total, dem[res[r]]);
            rate = dmin(1.0, __ddiv_rn(1.0, total));
        } else {
            rate = __ddiv_rn(1.0, static_cast<double>(n));
        }
        double sum = 0.0;
#pragma unroll 1
        for (uint32_t r = 0; r < n; ++r) sum = __dadd_rn(sum, __dmul_rn(dem[res[r]], rate));
        inst = dmin(1.0, sum);
    }
    RP_F64(rate)[g] = rate;
    RP_F64(inst)[g] = inst;
    double p = __dadd_rn(cf.p_idle_w, __dmul_rn(__dsub_rn(cf.p_max_w, cf.p_idle_w), inst));
    if (inst > cf.boost_threshold) p = __dadd_rn(p, cf.p_boost_w);
    RP_F64(power)[g] = p;

    // record_smact
    const double v = inst;
    uint32_t* has = RP_U32(has_step);
    double* lt = RP_F64(last_t);
    double* lv = RP_F64(last_v);
    uint32_t* rh = RP_U32(rhead);
    uint32_t* rc = RP_U32(rcnt);
    double* rt = RP_F64(ring_t) + g * L::RG;
    double* rv = RP_F64(ring_v) + g * L::RG;
    if (has[g]) {
        if (lv[g] == v) return true;
        if (lt[g] == now) {
            lv[g] = v;
            uint32_t li = rh[g] + rc[g] - 1;
            if (li >= static_cast<uint32_t>(L::RG)) li -= L::RG;
            rv[li] = v;
            RP_F64(lvl)[g] = v;
            return true;
        }
    }
    // Drop ring entries no future window can need: begin only grows, so an
    // entry whose successor is already at or before begin is dead.
    const double begin_now = dmax0(now - window);
    while (rc[g] >= 2) {
        uint32_t second = rh[g] + 1;
        if (second >= static_cast<uint32_t>(L::RG)) second -= L::RG;
        if (!(rt[second] <= begin_now)) break;
        rh[g] = second;
        rc[g] -= 1;
    }
    if (rc[g] >= static_cast<uint32_t>(L::RG)) return false;
    uint32_t slot = rh[g] + rc[g];
    if (slot >= static_cast<uint32_t>(L::RG)) slot -= L::RG;
    rt[slot] = now;
    rv[slot] = v;
    rc[g] += 1;
    double* lvl = RP_F64(lvl);
    if (now <= begin0) {
        lvl[g] = v;
    } else {
        double* integ = RP_F64(integ);
        double* cur = RP_F64(cur);
        integ[g] = __dadd_rn(integ[g], __dmul_rn(lvl[g], __dsub_rn(now, cur[g])));
        cur[g] = now;
        lvl[g] = v;
    }
    has[g] = 1;
    lt[g] = now;
    lv[g] = v;
    RP_U32(nsteps)[g] += 1;
    return true;
}

// World::refresh_rates (world.cpp:157-186) for the touched GPUs tg[0, nt).
template <class L>
__device__ __forceinline__ void refresh_rates(char* b, Sc& c, const int (&tg)[L::WM], int nt, unsigned lane) {
    RSUB_T(ra);
    const int t0 = tg[0], t1 = tg[1];
    bool ok = true;
    if constexpr (L::MG) {
#pragma unroll
        for (int k = 0; k < L::WM; ++k) {
            if (k >= nt) break;
            const int g = tg[k];
            if ((g & 31) == static_cast<int>(lane)) ok = refresh_gpu<L>(b, g, c.now, c.window, c.begin0) && ok;
        }
    } else {
#pragma unroll 1
        for (int k = 0; k < nt; ++k) {
            const int g = k == 0 ? t0 : t1;
            if ((g & 31) == static_cast<int>(lane)) ok = refresh_gpu<L>(b, g, c.now, c.window, c.begin0) && ok;
        }
    }
    if (!__all_sync(0xffffffffu, ok)) {
        c.status = kStatusRetry;
        return;
    }
    RSUB_T(rb);
    RSUB_ADD(0, ra, rb);
    // Affected tasks: residents of the touched GPUs, deduplicated, ordered by
    // id (std::set<std::string>) == by rank.
    const uint32_t* nres = RP_U32(nres);
    const uint16_t* res = RP_U16(res);
    const uint32_t* gp = RP_U32(s_gp);
    const uint32_t* rank = RP_U32(s_rank);
    uint64_t* aff = RP_U64(aff);
    uint64_t* aff2 = RP_U64(aff2);
    uint32_t na = 0;
    if constexpr (L::MG) {
        // residents of tg[k] not already collected from tg[0..k)
        const uint8_t* gls = reinterpret_cast<const uint8_t*>(b + L::s_gl);
#pragma unroll
        for (int k = 0; k < L::WM; ++k) {
            if (k >= nt) break;
            const uint32_t nk = nres[tg[k]];
#pragma unroll 1
            for (uint32_t base = 0; base < nk; base += 32) {
                const uint32_t r = base + lane;
                bool keep = false;
                uint32_t slot = 0;
                if (r < nk) {
                    slot = res[tg[k] * L::RC + r];
                    keep = true;
                    const uint32_t w = gp[slot] >> 16;
                    for (uint32_t m = 0; m < w; ++m)
                        for (int j = 0; j < k; ++j)
                            if (gls[slot * L::WM + m] == tg[j]) keep = false;
                }
                const unsigned bm = __ballot_sync(0xffffffffu, keep);
                if (keep) aff[na + __popc(bm & ((1u << lane) - 1u))] = (static_cast<uint64_t>(rank[slot]) << 32) | slot;
                na += __popc(bm);
            }
        }
    } else {
        const uint32_t n0 = nres[t0];
#pragma unroll 1
        for (uint32_t r = lane; r < n0; r += 32) {
            const uint32_t slot = res[t0 * L::RC + r];
            aff[r] = (static_cast<uint64_t>(rank[slot]) << 32) | slot;
        }
        na = n0;
        if (nt > 1) {
            const uint32_t n1 = nres[t1];
#pragma unroll 1
            for (uint32_t base = 0; base < n1; base += 32) {
                const uint32_t r = base + lane;
                bool keep = false;
                uint32_t slot = 0;
                if (r < n1) {
                    slot = res[t1 * L::RC + r];
                    const uint32_t g = gp[slot];
                    keep = !(static_cast<int>(g & 0xff) == t0 || ((g >> 16) > 1 && static_cast<int>((g >> 8) & 0xff) == t0));
                }
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (keep) aff[na + __popc(m & ((1u << lane) - 1u))] = (static_cast<uint64_t>(rank[slot]) << 32) | slot;
                na += __popc(m);
            }
        }
    }
    __syncwarp();
#pragma unroll 1
    for (uint32_t e = lane; e < na; e += 32) {
        const uint64_t key = aff[e];
        uint32_t pos = 0;
#pragma unroll 1
        for (uint32_t k = 0; k < na; ++k) pos += aff[k] < key;
        aff2[pos] = key;
    }
    __syncwarp();
    RSUB_T(rc);
    RSUB_ADD(1, rb, rc);
    const double* grate = RP_F64(rate);
    double* s_rate = RP_F64(s_rate);
    double* s_last = RP_F64(s_last);
    double* s_exec = RP_F64(s_exec);
    double* s_rem = RP_F64(s_rem);
    uint32_t* s_seq = RP_U32(s_seq);
#pragma unroll 1
    for (uint32_t e = 0; e < na; ++e) {
        const uint32_t slot = static_cast<uint32_t>(aff2[e] & 0xffffffffu);
        const uint32_t g = gp[slot];
        double r0, r1 = 0.0;
        if constexpr (L::MG) {  // min over every device of the task (world.cpp:165-175)
            const uint8_t* gls = reinterpret_cast<const uint8_t*>(b + L::s_gl) + slot * L::WM;
            const uint8_t* ils = reinterpret_cast<const uint8_t*>(b + L::s_il) + slot * L::WM;
            const double d = RP_F64(s_dem)[slot];
            double rate = 1.0;
            for (uint32_t m = 0; m < (g >> 16); ++m) {
                double rm;
                if constexpr (L::MIG) rm = dmin(1.0, __ddiv_rn(RP_CFG.mig_fraction[ils[m]], d));
                else rm = grate[gls[m]];
                rate = dmin(rate, rm);
            }
            r0 = rate;
        } else if constexpr (L::MIG) {  // effective_rates (gpu.cpp:187-195)
            const uint32_t in = RP_U32(s_inst)[slot];
            const double d = RP_F64(s_dem)[slot];
            r0 = dmin(1.0, __ddiv_rn(RP_CFG.mig_fraction[in & 0xff], d));
            if ((g >> 16) > 1) r1 = dmin(1.0, __ddiv_rn(RP_CFG.mig_fraction[(in >> 8) & 0xff], d));
        } else {
            r0 = grate[g & 0xff];
            if ((g >> 16) > 1) r1 = grate[(g >> 8) & 0xff];
        }
        double rate = dmin(1.0, r0);
        if (!L::MG && (g >> 16) > 1) rate = dmin(rate, r1);
        const double old = s_rate[slot];
        if (rate == old && s_seq[slot] != kNone) continue;
        const double dt = __dsub_rn(c.now, s_last[slot]);
        s_exec[slot] = __dadd_rn(s_exec[slot], __dmul_rn(old, dt));
        const double rem = dmax0(__dsub_rn(s_rem[slot], __dmul_rn(old, dt)));
        s_rem[slot] = rem;
        s_last[slot] = c.now;
        s_rate[slot] = rate;
        const uint32_t seq = heap_push<L>(b, c, __dadd_rn(c.now, __ddiv_rn(rem, rate)), (kCompletion << 30) | slot);
        if (c.status) return;
        s_seq[slot] = seq;
    }
    __syncwarp();
    RSUB_T(rd);
    RSUB_ADD(2, rc, rd);
}

// World::place (world.cpp:73-130) without the trailing refresh_rates:
// allocate on every GPU in order (rolling back on failure), then take a
// slot and append the task to the resident lists.
template <class L>
__device__ __forceinline__ bool place(char* b, Sc& c, const carma_task& tk, uint32_t task, const int (&gl)[L::WM],
                                      const int (&il)[L::WM], int want, int nblk, unsigned lane, OomInfo& oi) {
    const int g0 = gl[0], g1 = gl[1], i0 = il[0], i1 = il[1];
    const carma_replay_config& cf = RP_CFG;
    const uint64_t block = cf.alloc_block;
    const uint64_t bytes = tk.true_mem > 0 ? tk.true_mem : 1;
    const bool seg = L::MG && nblk < 0;  // byte-granular segment allocator (nblk = -1)
    const uint64_t nb64 = seg ? 0 : (bytes + block - 1) / block;
    const int nb = seg ? 0 : (nb64 > static_cast<uint64_t>(nblk) ? nblk + 1 : static_cast<int>(nb64));
    // MIG: allocate_on_instance (gpu.cpp:67-70) inside the instance's blocks
    constexpr bool mig = L::MIG;
    const int a0 = mig ? cf.mig_base[i0] : 0, e0 = mig ? a0 + cf.mig_blocks[i0] : nblk;
    // failure details on the failing device (diagnostic kernels only)
    auto oom = [&](int g, int r0, int r1) {
        if constexpr (L::TL) {
            uint32_t f = 0, lg = 0;
            if ((g & 31) == static_cast<int>(lane)) range_stats<L>(b, g, nblk, r0, r1, f, lg);
            oi.gpu = g;
            oi.free_blk = __shfl_sync(0xffffffffu, f, g & 31);
            oi.largest_blk = __shfl_sync(0xffffffffu, lg, g & 31);
        }
    };
    if constexpr (L::MG) {
        // allocate on every device in order, rolling back on the first failure (world.cpp:84-110)
        int offs[L::WM];
        uint64_t offs_b[L::WM];
        // round_up(max(bytes, 1)) (gpu.cpp:58-61, 74)
        const uint64_t want_b = seg ? (block == 0 ? bytes : (bytes + block - 1) / block * block) : 0;
#pragma unroll
        for (int k = 0; k < L::WM; ++k) {
            if (k >= want) break;
            const int g = gl[k];
            if (seg) {
                uint64_t o = 0, f = 0, lg = 0;
                bool okk = false, ovf = false;
                const uint64_t r0 = mig ? cf.mig_base_bytes[il[k]] : 0;
                const uint64_t r1 = mig ? r0 + cf.mig_cap_bytes[il[k]] : cf.gpu_capacity;
                if ((g & 31) == static_cast<int>(lane)) okk = seg_alloc<L>(b, g, cf.gpu_capacity, r0, r1, want_b, o, f, lg, ovf);
                okk = __shfl_sync(0xffffffffu, okk, g & 31);
                ovf = __shfl_sync(0xffffffffu, ovf, g & 31);
                o = __shfl_sync(0xffffffffu, o, g & 31);
                if (ovf) {
                    c.status = kStatusRetry;
                    return false;
                }
                if (!okk) {
                    oi.gpu = g;
                    oi.free_b = __shfl_sync(0xffffffffu, f, g & 31);
                    oi.largest_b = __shfl_sync(0xffffffffu, lg, g & 31);
#pragma unroll
                    for (int j = 0; j < L::WM; ++j) {
                        if (j >= k) break;
                        if ((gl[j] & 31) == static_cast<int>(lane)) seg_release<L>(b, gl[j], offs_b[j], want_b);
                    }
                    __syncwarp();
                    return false;
                }
                offs_b[k] = o;
                offs[k] = 0;
                continue;
            }
            const int a = mig ? cf.mig_base[il[k]] : 0, e = mig ? a + cf.mig_blocks[il[k]] : nblk;
            int o = -1;
            if ((g & 31) == static_cast<int>(lane) && nb <= nblk) o = first_fit<L>(b, g, nblk, nb, a, e);
            o = __shfl_sync(0xffffffffu, o, g & 31);
            if (o < 0) {
                oom(g, a, e);
#pragma unroll
                for (int j = 0; j < L::WM; ++j) {
                    if (j >= k) break;
                    if ((gl[j] & 31) == static_cast<int>(lane)) set_bits<L>(RP_U64(used), gl[j], offs[j], nb, false);
                }
                __syncwarp();
                return false;
            }
            offs[k] = o;
        }
        if (c.nfree == 0) {
            c.status = kStatusRetry;
            return false;
        }
        const uint32_t slot = RP_U32(free_stack)[--c.nfree];
        RP_U32(s_task)[slot] = task;
        RP_U32(s_rank)[slot] = tk.rank;
        RP_F64(s_rem)[slot] = tk.work;
        RP_F64(s_rate)[slot] = 0.0;
        RP_F64(s_last)[slot] = c.now;
        RP_F64(s_exec)[slot] = 0.0;
        RP_F64(s_dem)[slot] = tk.demand;
        RP_U32(s_seq)[slot] = kNone;
        RP_U32(s_gp)[slot] = static_cast<uint32_t>(g0) | (static_cast<uint32_t>(want > 1 ? g1 : 0) << 8) |
                             (static_cast<uint32_t>(want) << 16);
        RP_U32(s_nb)[slot] = static_cast<uint32_t>(nb);
        if (seg && lane == 0) RP_U64(s_wb)[slot] = want_b;
        uint8_t* gls = reinterpret_cast<uint8_t*>(b + L::s_gl) + slot * L::WM;
        uint8_t* ils = reinterpret_cast<uint8_t*>(b + L::s_il) + slot * L::WM;
        uint16_t* ols = reinterpret_cast<uint16_t*>(b + L::s_ol) + slot * L::WM;
        uint32_t* nres = RP_U32(nres);
        uint16_t* res = RP_U16(res);
#pragma unroll
        for (int k = 0; k < L::WM; ++k) {
            if (k >= want) break;
            const int g = gl[k];
            if (lane == 0) {
                gls[k] = static_cast<uint8_t>(g);
                ols[k] = static_cast<uint16_t>(offs[k]);
                if (seg) RP_U64(s_ob)[slot * L::WM + k] = offs_b[k];
                if (mig) ils[k] = static_cast<uint8_t>(il[k]);
            }
            const uint32_t n = nres[g];
            if (n >= static_cast<uint32_t>(L::RC)) {
                c.status = kStatusRetry;
                return false;
            }
            res[g * L::RC + n] = static_cast<uint16_t>(slot);
            nres[g] = n + 1;
            if (mig && (g & 31) == static_cast<int>(lane)) RP_U32(imask)[g] |= 1u << il[k];
            __syncwarp();
        }
        __syncwarp();
        return true;
    }
    int off0 = -1, off1 = 0;
    if ((g0 & 31) == static_cast<int>(lane) && nb <= nblk) off0 = first_fit<L>(b, g0, nblk, nb, a0, e0);
    off0 = __shfl_sync(0xffffffffu, off0, g0 & 31);
    if (off0 < 0) {
        oom(g0, a0, e0);
        return false;
    }
    if (want > 1) {
        const int a1 = mig ? cf.mig_base[i1] : 0, e1 = mig ? a1 + cf.mig_blocks[i1] : nblk;
        int o = -1;
        if ((g1 & 31) == static_cast<int>(lane) && nb <= nblk) o = first_fit<L>(b, g1, nblk, nb, a1, e1);
        o = __shfl_sync(0xffffffffu, o, g1 & 31);
        if (o < 0) {
            oom(g1, a1, e1);
            if ((g0 & 31) == static_cast<int>(lane)) set_bits<L>(RP_U64(used), g0, off0, nb, false);
            __syncwarp();
            return false;
        }
        off1 = o;
    }
    if (c.nfree == 0) {
        c.status = kStatusRetry;
        return false;
    }
    const uint32_t slot = RP_U32(free_stack)[--c.nfree];
    RP_U32(s_task)[slot] = task;
    RP_U32(s_rank)[slot] = tk.rank;
    RP_F64(s_rem)[slot] = tk.work;
    RP_F64(s_rate)[slot] = 0.0;
    RP_F64(s_last)[slot] = c.now;
    RP_F64(s_exec)[slot] = 0.0;
    RP_F64(s_dem)[slot] = tk.demand;
    RP_U32(s_seq)[slot] = kNone;
    RP_U32(s_gp)[slot] = static_cast<uint32_t>(g0) | (static_cast<uint32_t>(want > 1 ? g1 : 0) << 8) |
                         (static_cast<uint32_t>(want) << 16);
    RP_U32(s_off)[slot] = static_cast<uint32_t>(off0) | (static_cast<uint32_t>(off1) << 16);
    RP_U32(s_nb)[slot] = static_cast<uint32_t>(nb);
    if (mig) RP_U32(s_inst)[slot] = static_cast<uint32_t>(i0) | (static_cast<uint32_t>(want > 1 ? i1 : 0) << 8);
    uint32_t* nres = RP_U32(nres);
    uint16_t* res = RP_U16(res);
    for (int k = 0; k < want; ++k) {
        const int g = k == 0 ? g0 : g1;
        const uint32_t n = nres[g];
        if (n >= static_cast<uint32_t>(L::RC)) {
            c.status = kStatusRetry;
            return false;
        }
        res[g * L::RC + n] = static_cast<uint16_t>(slot);
        nres[g] = n + 1;
        if (mig && (g & 31) == static_cast<int>(lane)) RP_U32(imask)[g] |= 1u << (k == 0 ? i0 : i1);
    }
    __syncwarp();
    return true;
}

// World::finish (world.cpp:132-155) without the trailing refresh_rates.
template <class L>
__device__ __forceinline__ void finish(char* b, Sc& c, uint32_t slot, carma_task_result* out, int (&tg)[L::WM],
                                       int& want, unsigned lane, bool nblk_seg = false) {
    double* s_last = RP_F64(s_last);
    double* s_rem = RP_F64(s_rem);
    const double dt = __dsub_rn(c.now, s_last[slot]);
    const double rate = RP_F64(s_rate)[slot];
    const double exec = __dadd_rn(RP_F64(s_exec)[slot], __dmul_rn(rate, dt));
    s_rem[slot] = dmax0(__dsub_rn(s_rem[slot], __dmul_rn(rate, dt)));
    s_last[slot] = c.now;
    const uint32_t gp = RP_U32(s_gp)[slot], of = RP_U32(s_off)[slot];
    want = static_cast<int>(gp >> 16);
    const int g0 = static_cast<int>(gp & 0xff), g1 = static_cast<int>((gp >> 8) & 0xff);
    tg[0] = g0;
    tg[1] = g1;
    const uint8_t* gls = reinterpret_cast<const uint8_t*>(b + L::s_gl) + slot * L::WM;
    const uint16_t* ols = reinterpret_cast<const uint16_t*>(b + L::s_ol) + slot * L::WM;
    if constexpr (L::MG) {
#pragma unroll
        for (int k = 0; k < L::WM; ++k)
            if (k < want) tg[k] = gls[k];
    }
    const int nb = static_cast<int>(RP_U32(s_nb)[slot]);
    uint32_t* nres = RP_U32(nres);
    uint16_t* res = RP_U16(res);
    for (int k = 0; k < want; ++k) {
        const int g = L::MG ? tg[k < L::WM ? k : 0] : (k == 0 ? g0 : g1);
        if ((g & 31) == static_cast<int>(lane)) {
            if (L::MG && nblk_seg) seg_release<L>(b, g, RP_U64(s_ob)[slot * L::WM + k], RP_U64(s_wb)[slot]);
            else
                set_bits<L>(RP_U64(used), g,
                            L::MG ? static_cast<int>(ols[k])
                                  : (k == 0 ? static_cast<int>(of & 0xffff) : static_cast<int>(of >> 16)),
                            nb, false);
            // remove_resident preserving insertion order (gpu.cpp:175-181)
            const uint32_t n = nres[g];
            uint16_t* rl = res + g * L::RC;
            uint32_t r = 0;
            while (r < n && rl[r] != slot) ++r;
#pragma unroll 1
            for (; r + 1 < n; ++r) rl[r] = rl[r + 1];
            nres[g] = n - 1;
            if constexpr (L::MIG) RP_U32(imask)[g] &= ~(1u << inst_of<L>(b, slot, g));
        }
    }
    const uint32_t task = RP_U32(s_task)[slot];
    if (lane == 0) {
        out[task].executed = exec;
        out[task].complete = c.now;
    }
    RP_U32(s_seq)[slot] = kNone;
    RP_U32(free_stack)[c.nfree++] = slot;
    __syncwarp();
}

// Manager::try_schedule's decision half (manager.cpp:280-316): gate, head,
// estimate, map_task. Returns the number of GPUs chosen (0 = no dispatch).
template <class L>
__device__ __forceinline__ int decide(char* b, Sc& c, const carma_task* tasks, const uint64_t* est,
                                      uint32_t& head, bool& from_recovery, int (&gl)[L::WM], int (&il)[L::WM],
                                      uint64_t& est_bytes, unsigned lane, bool seg_mode = false) {
    RSUB_T(da);
    const carma_replay_config& cf = RP_CFG;
    const int G = cf.gpu_count;
    const uint32_t* nres = RP_U32(nres);
    bool idle_all = true;
#pragma unroll
    for (int j = 0; j < L::GPL; ++j) {
        const int g = static_cast<int>(lane) + 32 * j;
        if (g < G && nres[g] != 0) idle_all = false;
    }
    idle_all = __all_sync(0xffffffffu, idle_all);
    if (!(c.now >= c.deadline) && !idle_all) return 0;  // gate_open (manager.cpp:269-273)
    from_recovery = c.rq_cnt > 0;
    if (from_recovery) head = RP_U32(rq)[c.rq_head];
    else if (c.mq_head < c.arrived) head = c.mq_head;
    else return 0;
    const int policy = from_recovery ? CARMA_POLICY_EXCLUSIVE : cf.policy;
    uint64_t floor = cf.min_free, need = 0;
    est_bytes = 0;  // the decision log's est_bytes (manager.cpp:292-294, 301-315)
    if (!from_recovery && cf.policy != CARMA_POLICY_EXCLUSIVE) {
        const uint64_t e = est ? est[head] : tasks[head].estimate;
        if (e != CARMA_NO_ESTIMATE) {
            est_bytes = e;
            need = e < cf.gpu_capacity ? e : cf.gpu_capacity;
            if (need > floor) floor = need;
        }
    }
    RSUB_T(db);
    RSUB_ADD(3, da, db);
    constexpr bool mig = L::MIG;
    // pick_instance's bar (manager.cpp:125-134): max(need, 1) bytes; 1 for exclusive
    const uint64_t inst_need = need > 1 ? need : 1;
    const bool need_smact = policy != CARMA_POLICY_EXCLUSIVE &&
                            !(policy == CARMA_POLICY_RR && !cf.rr_apply_preconditions);
    const uint64_t* used = RP_U64(used);
    PickInput in[L::GPL];
    int inst[L::GPL];
#pragma unroll
    for (int j = 0; j < L::GPL; ++j) {
        const int g = static_cast<int>(lane) + 32 * j;
        const bool valid = g < G;
        in[j].valid = valid;
        in[j].idle = valid && nres[g] == 0;
        if (L::MG && seg_mode) in[j].free_bytes = valid ? RP_U64(seg_free)[g] : 0;
        else in[j].free_bytes = valid ? static_cast<uint64_t>(free_blocks<L>(used, g)) * cf.alloc_block : 0;
        if (L::GPL == 1) in[j].smact = (valid && need_smact) ? windowed<L>(b, g, c.now, c.window) : 0.0;
        in[j].inst_ok = true;
        inst[j] = -1;
        if (mig && valid) {
            // first idle instance with enough free memory (pick_instance)
            const uint32_t busy = RP_U32(imask)[g];
            for (int i = 0; i < cf.mig_count; ++i) {
                if ((busy >> i) & 1u) continue;
                const int r0 = cf.mig_base[i];
                uint64_t fb;
                if (L::MG && seg_mode)
                    fb = seg_free_in_range<L>(b, g, cf.mig_base_bytes[i], cf.mig_base_bytes[i] + cf.mig_cap_bytes[i]);
                else
                    fb = static_cast<uint64_t>(free_in_range<L>(used, g, r0, r0 + cf.mig_blocks[i])) * cf.alloc_block;
                if (fb < inst_need) continue;
                inst[j] = i;
                break;
            }
            in[j].inst_ok = inst[j] >= 0;
        }
    }
    if constexpr (L::GPL >= 2) {  // the lane's GPUs in pairs: two independent chains per step
#pragma unroll
        for (int j = 0; j < L::GPL; j += 2) {
            double s0 = 0.0, s1 = 0.0;
            const bool v1 = j + 1 < L::GPL && in[j + 1 < L::GPL ? j + 1 : j].valid;
            if (need_smact && in[j].valid)
                windowed2<L>(b, static_cast<int>(lane) + 32 * j, static_cast<int>(lane) + 32 * (j + 1), v1, c.now,
                             c.window, s0, s1);
            in[j].smact = s0;
            if (j + 1 < L::GPL) in[j + 1].smact = s1;
        }
    }
    RSUB_T(dc);
    RSUB_ADD(4, db, dc);
    const int got = pick_gpus<L::GPL>(cf, policy, tasks[head].gpus, floor, in, lane, 0, 32, c.rr_cursor, gl);
    RSUB_T(dd);
    RSUB_ADD(5, dc, dd);
    const int g0 = gl[0], g1 = gl[1];
#pragma unroll
    for (int k = 0; k < L::WM; ++k) il[k] = 0;
    if constexpr (L::MG) {
        if (mig && got > 0) {
#pragma unroll
            for (int k = 0; k < L::WM; ++k) {
                if (k >= got) break;
                int mine = 0;
#pragma unroll
                for (int j = 0; j < L::GPL; ++j)
                    if (static_cast<int>(lane) + 32 * j == gl[k]) mine = inst[j] < 0 ? 0 : inst[j];
                il[k] = __shfl_sync(0xffffffffu, mine, gl[k] & 31);
            }
        }
        return got;
    }
    if (mig && got > 0) {  // the chosen devices' instances (exclusive: value_or(0))
        int mine0 = 0, mine1 = 0;
#pragma unroll
        for (int j = 0; j < L::GPL; ++j) {
            const int g = static_cast<int>(lane) + 32 * j;
            if (g == g0) mine0 = inst[j] < 0 ? 0 : inst[j];
            if (g == g1) mine1 = inst[j] < 0 ? 0 : inst[j];
        }
        il[0] = __shfl_sync(0xffffffffu, mine0, g0 & 31);
        if (got > 1) il[1] = __shfl_sync(0xffffffffu, mine1, g1 & 31);
    }
    return got;
}

// Per-job setup. Cold (once per job): kept out of line.
template <class L>
__device__ __noinline__ void init_job(char* b, const Params& p, uint32_t j, unsigned lane, Sc& c,
                                      const carma_task*& tasks, carma_task_result*& out, int& nblk) {
    const carma_replay_job job = p.jobs[j];
    const carma_replay_config* src = p.cfgs + job.config;
    for (uint32_t k = lane; k < sizeof(carma_replay_config) / 8; k += 32)  // 43 words
        reinterpret_cast<uint64_t*>(b + L::cfg)[k] = reinterpret_cast<const uint64_t*>(src)[k];
    __syncwarp();
    const carma_replay_config& cf = RP_CFG;
    const uint64_t tb = p.trace_off[job.trace];
    const uint32_t T = static_cast<uint32_t>(p.trace_off[job.trace + 1] - tb);
    tasks = p.tasks + tb;
    out = p.task_out + p.task_out_off[j];
    // byte-granular segments (generic instantiations): nblk = -1
    const bool seg = L::MG && (cf.alloc_block == 0 || cf.gpu_capacity % cf.alloc_block != 0 ||
                               cf.gpu_capacity / cf.alloc_block > 64ull * L::W);
    nblk = seg ? -1 : static_cast<int>(cf.gpu_capacity / cf.alloc_block);
    // first_submit (runner.cpp:108-109) and the full-history window begin.
    double fs = tasks[0].submit;
    bool bad = false;  // gpus_requested outside what this instantiation places (1..WM)
#pragma unroll 1
    for (uint32_t i = lane; i < T; i += 32) {
        fs = dmin(fs, tasks[i].submit);
        bad |= tasks[i].gpus < 1 || tasks[i].gpus > static_cast<uint32_t>(L::WM);
    }
    bad = __any_sync(0xffffffffu, bad);
#pragma unroll 1
    for (int o = 16; o > 0; o >>= 1) fs = dmin(fs, __shfl_xor_sync(0xffffffffu, fs, o));
    const double forced = p.smact_begin[j];
    c.begin0 = forced == forced ? forced : dmax0(fs);
#pragma unroll 1
    for (uint32_t i = lane; i < T; i += 32) {
        carma_task_result r;
        r.first_attempt = r.final_dispatch = r.complete = r.first_crash = r.last_crash = -1.0;
        r.executed = 0.0;
        r.attempts = r.ooms = 0;
        r.gpu[0] = r.gpu[1] = -1;
        r.reserved = 0;
        out[i] = r;
    }
    uint64_t* used = RP_U64(used);
    double p0 = __dadd_rn(cf.p_idle_w, __dmul_rn(__dsub_rn(cf.p_max_w, cf.p_idle_w), 0.0));
    if (0.0 > cf.boost_threshold) p0 = __dadd_rn(p0, cf.p_boost_w);
    for (int g = static_cast<int>(lane); g < L::G; g += 32) {
#pragma unroll
        for (int w = 0; w < L::W; ++w) {
            const int lo = w * 64;
            uint64_t m = ~0ull;
            if (nblk > lo) m = nblk - lo >= 64 ? 0ull : (~0ull << (nblk - lo));
            used[w * L::G + g] = m;
        }
        RP_F64(energy)[g] = 0.0;
        RP_F64(rate)[g] = 0.0;
        RP_F64(inst)[g] = 0.0;
        RP_F64(power)[g] = p0;
        RP_F64(lvl)[g] = 0.0;
        RP_F64(cur)[g] = c.begin0;
        RP_F64(integ)[g] = 0.0;
        RP_F64(last_t)[g] = 0.0;
        RP_F64(last_v)[g] = 0.0;
        RP_U32(nres)[g] = 0;
        RP_U32(nsteps)[g] = 0;
        RP_U32(rhead)[g] = 0;
        RP_U32(rcnt)[g] = 0;
        RP_U32(peak)[g] = 0;
        if constexpr (L::MG) {
            if (seg) seg_init<L>(b, g, cf.gpu_capacity);
        }
        RP_U32(has_step)[g] = 0;
        if constexpr (L::MIG) RP_U32(imask)[g] = 0;
    }
    for (int k = static_cast<int>(lane); k < L::S; k += 32) RP_U32(free_stack)[k] = L::S - 1 - k;
    c.now = 0.0;
    c.deadline = 0.0;
    c.window = cf.monitor_window;
    c.seq_next = T;
    c.arrived = 0;
    c.mq_head = 0;
    c.rq_head = 0;
    c.rq_cnt = 0;
    c.hsize = 0;
    c.hhead = 0;
    c.nfree = L::S;
    c.T = T;
    c.rr_cursor = 0;
    c.oom = 0;
    c.status = 0;
    c.events_lo = c.events_hi = 0;
    if (bad) {  // tasks re-uploaded after the plan was classified: no event runs
        c.status = CARMA_ERR_UNSUPPORTED;
        c.arrived = T;
    }
    __syncwarp();
}

// Runner tail + report. Cold: out of line.
template <class L>
__device__ __noinline__ void finish_job(char* b, const Params& p, uint32_t j, unsigned lane, const Sc& c,
                                        const carma_task* tasks, carma_task_result* out) {
    const carma_replay_config& cf = RP_CFG;
    const bool seg_job = L::MG && static_cast<int>(reinterpret_cast<const uint64_t*>(b + L::ptrs)[3]) < 0;
    carma_trace_result& tr = p.trace_out[j];
    if (c.status == kStatusRetry) {
        if (lane == 0) {
            tr.status = kStatusRetry;
            p.retry_list[atomicAdd(p.retry_count, 1u)] = j;
        }
        return;
    }
    const uint32_t T = c.T;
    uint32_t* inv = p.inv_scratch + p.task_out_off[j];
    double lc = 0.0, fs = tasks[0].submit;
    bool complete = true;
#pragma unroll 1
    for (uint32_t i = lane; i < T; i += 32) {
        carma_task_result& o = out[i];
        const double cpl = o.complete;
        lc = lc < cpl ? cpl : lc;  // std::max(last_complete, t.complete)
        fs = dmin(fs, tasks[i].submit);
        complete = complete && cpl >= 0.0;
        o.attempts = o.ooms + (o.final_dispatch >= 0.0 ? 1u : 0u);
        inv[tasks[i].rank] = i;
        if (p.outcome_sink) {  // the D2H of the outcomes streams out while later jobs still run
            carma_task_outcome oc;
            oc.final_dispatch = o.final_dispatch;
            oc.complete = cpl;
            oc.ooms = o.ooms;
            oc.attempts = o.attempts;
            p.outcome_sink[p.task_out_off[j] + i] = oc;
        }
    }
#pragma unroll 1
    for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, lc, o);
        lc = lc < x ? x : lc;
        fs = dmin(fs, __shfl_xor_sync(0xffffffffu, fs, o));
    }
    complete = __all_sync(0xffffffffu, complete);
    int32_t status = c.status;
    if (status == 0 && !complete) status = CARMA_ERR_INCOMPLETE;
    const double span = __dsub_rn(lc, fs);
    const double begin_actual = dmax0(__dsub_rn(lc, span));
    const double forced = p.smact_begin[j];
    if (status == 0 && span > 0.0 && !(forced == forced) && begin_actual != c.begin0) {
        // Re-run with the true window begin (see file header).
        if (lane == 0) {
            p.smact_begin[j] = begin_actual;
            tr.status = kStatusRedoSmact;
            p.retry_list[atomicAdd(p.retry_count, 1u)] = j;
        }
        return;
    }
    const int G = cf.gpu_count;
    carma_gpu_result* gout = p.gpu_out + p.gpu_out_off[j];
    const double overshoot = __dsub_rn(c.now, lc);
    double energy = 0.0;
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
        double e = RP_F64(energy)[g];
        if (overshoot > 0.0) e = __dsub_rn(e, __dmul_rn(RP_F64(power)[g], overshoot));
        energy = __dadd_rn(energy, e);
        if ((g & 31) == static_cast<int>(lane)) {
            carma_gpu_result r;
            r.energy_j = e;
            double mean = 0.0;
            if (span > 0.0)
                mean = __ddiv_rn(__dadd_rn(RP_F64(integ)[g], __dmul_rn(RP_F64(lvl)[g], __dsub_rn(lc, RP_F64(cur)[g]))),
                                 span);
            r.mean_smact = mean;
            if (L::MG && seg_job) r.peak_used = RP_U64(seg_peak)[g];
            else r.peak_used = static_cast<uint64_t>(RP_U32(peak)[g]) * cf.alloc_block;
            r.smact_steps = RP_U32(nsteps)[g];
            gout[g] = r;
        }
    }
    __syncwarp();
    // Sums in id (rank) order (metrics.cpp:25-45): each lane stages 32
    // values; lane order is rank order.
    double ws = 0.0, es = 0.0, js = 0.0;
#pragma unroll 1
    for (uint32_t base = 0; base < T; base += 32) {
        const uint32_t r = base + lane;
        double w = 0.0, e = 0.0, jc = 0.0;
        if (r < T) {
            const uint32_t i = inv[r];
            const double sub = tasks[i].submit;
            const double fd = out[i].final_dispatch, cp = out[i].complete;
            w = __dsub_rn(fd, sub);
            e = __dsub_rn(cp, fd);
            jc = __dsub_rn(cp, sub);
        }
        const uint32_t cnt = min(32u, T - base);
#pragma unroll 1
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
        r.status = status;
        r.events = (static_cast<uint64_t>(c.events_hi) << 32) | c.events_lo;
        tr = r;
    }
}

template <class L>
__device__ __forceinline__ void run_job(char* b, const Params& p, uint32_t j, unsigned lane) {
    // init_job / finish_job are out of line and take their state by
    // reference; the loop works on a copy whose address never escapes, so
    // it stays in registers instead of local memory.
    Sc c;
    {
        Sc c0;
        const carma_task* tasks0;
        carma_task_result* out0;
        int nblk0;
        init_job<L>(b, p, j, lane, c0, tasks0, out0, nblk0);
        c = c0;
        // The warp-uniform base pointers live in shared memory, not in
        // registers: under the 64-register cap they were spilled to local
        // memory, which thrashed L1 (every reload a 256-B per-lane access).
        if (lane == 0) {
            uint64_t* q = RP_U64(ptrs);
            q[0] = reinterpret_cast<uint64_t>(tasks0);
            q[1] = reinterpret_cast<uint64_t>(out0);
            q[2] = p.est_override ? reinterpret_cast<uint64_t>(p.est_override + p.trace_off[p.jobs[j].trace]) : 0ull;
            q[3] = static_cast<uint64_t>(nblk0);
        }
        __syncwarp();
    }
#define tasks (reinterpret_cast<const carma_task* const*>(b + L::ptrs)[0])
#define out (reinterpret_cast<carma_task_result* const*>(b + L::ptrs)[1])
#define est (reinterpret_cast<const uint64_t* const*>(b + L::ptrs)[2])
#define nblk (static_cast<int>(reinterpret_cast<const uint64_t*>(b + L::ptrs)[3]))
    const uint64_t max_events = 1000ull * c.T + 1000000ull;
    uint64_t events = 0;
    // timeline (L::TL only; dead code otherwise): the pending sample tick —
    // the first at the first row's submit time, scheduled after every arrival
    // (seq = T, runner.cpp:80-83) — completions so far and rows written
    double tick_t = 0.0;
    uint32_t tick_seq = 0, n_done = 0;
    bool tick_live = false;
    uint64_t tl_rows = 0;
    // event / decision log (L::TL kernels): records in run order, lane 0 writes
    const int32_t log_flags = L::TL ? RP_CFG.log_flags : 0;
    uint64_t n_log = 0;
    auto log = [&](uint8_t kind, uint32_t task, int gpu, uint64_t a, uint64_t b2, uint64_t c2, uint8_t pol) {
        if constexpr (L::TL) {
            if (lane == 0 && n_log < p.log_cap) {
                carma_log_record r;
                r.t = c.now;
                r.a = a;
                r.b = b2;
                r.c = c2;
                r.task = task;
                r.gpu = static_cast<int16_t>(gpu);
                r.kind = kind;
                r.policy = pol;
                p.log_out[static_cast<uint64_t>(j) * p.log_cap + n_log] = r;
            }
            ++n_log;
        }
    };
    if constexpr (L::TL) {
        tick_live = RP_CFG.sample_interval > 0.0;
        tick_t = tasks[0].submit;
        tick_seq = c.T;
        if (tick_live) c.seq_next = c.T + 1;
    }
    const double delay = RP_CFG.oom_startup_delay;
#if REPLAY_PROF
    unsigned long long prof[16] = {};
#endif
    for (;;) {
        RPROF_T(tp0);
        // ---- next event: arrival stream (seq = index) vs heap top
        const bool have_arr = c.arrived < c.T;
        const bool have_heap = c.hsize > 0;
        if (!have_arr && !have_heap && !(L::TL && tick_live)) break;
        if (events >= max_events) {
            c.status = CARMA_ERR_INCOMPLETE;
            break;
        }
        double t;
        uint32_t kind, payload, seq = 0;
        const double at = have_arr ? tasks[c.arrived].submit : 0.0;
        bool tick = false;
        if constexpr (L::TL) {  // the pending sample tick against both heads
            if (tick_live) {
                const uint64_t tk = tkey(tick_t);
                tick = !(have_arr && klater(tk, tick_seq, tkey(at), c.arrived)) &&
                       !(have_heap && klater(tk, tick_seq, heap_top<L>(b, c).key, heap_top<L>(b, c).seq));
            }
        }
        if (tick) {
            t = tick_t;
            kind = kTick;
            payload = 0;
        } else if (have_arr && (!have_heap || !klater(tkey(at), c.arrived, heap_top<L>(b, c).key,
                                                      heap_top<L>(b, c).seq))) {
            t = at;
            kind = 0;
            payload = c.arrived;
        } else {
            const HeapEnt top = heap_top<L>(b, c);
            t = tval(top.key);
            seq = top.seq;
            const uint32_t info = top.info;
            kind = info >> 30;
            payload = info & 0x3fffffffu;
#if REPLAY_PROF
            prof[8] += c.hsize;
            prof[9] += 1;
#endif
            heap_pop<L>(b, c);
        }
        ++events;
        RPROF_ADD(0, tp0);
        RPROF_T(tp1);
        // ---- integrate_to (world.cpp:37-44)
        const double dt = __dsub_rn(t, c.now);
        if (dt > 0.0) {
            double* energy = RP_F64(energy);
            const double* power = RP_F64(power);
            const int G = RP_CFG.gpu_count;
#pragma unroll
            for (int jj = 0; jj < L::GPL; ++jj) {
                const int g = static_cast<int>(lane) + 32 * jj;
                if (g < G) energy[g] = __dadd_rn(energy[g], __dmul_rn(power[g], dt));
            }
        }
        c.now = t;
        RPROF_ADD(1, tp1);
        RPROF_T(tp2);
        if constexpr (L::TL) {
            if (kind == kTick) {
                // emit_timeline_row (world.cpp:210-219), then reschedule while
                // Manager::all_done() is false (runner.cpp:85-92)
                const carma_replay_config& cf = RP_CFG;
                const int G = cf.gpu_count;
                const uint64_t* used = RP_U64(used);
                const bool seg_tl = L::MG && nblk < 0;
                const int nblk_g = seg_tl ? 0 : static_cast<int>(cf.gpu_capacity / cf.alloc_block);
#pragma unroll
                for (int jj = 0; jj < L::GPL; ++jj) {
                    const int g = static_cast<int>(lane) + 32 * jj;
                    const uint64_t r = tl_rows + static_cast<uint64_t>(g);
                    if (g < G && r < p.tl_cap) {
                        carma_timeline_row row;
                        row.t = t;
                        row.smact = RP_F64(inst)[g];
                        row.power_w = RP_F64(power)[g];
                        if (seg_tl) row.used = cf.gpu_capacity - RP_U64(seg_free)[g];
                        else row.used = static_cast<uint64_t>(nblk_g - static_cast<int>(free_blocks<L>(used, g))) *
                                        cf.alloc_block;
                        row.gpu = g;
                        row.reserved = 0;
                        p.tl_out[static_cast<uint64_t>(j) * p.tl_cap + r] = row;
                    }
                }
                tl_rows += static_cast<uint64_t>(G);
                if (!(c.arrived > 0 && n_done == c.arrived)) {
                    tick_t = __dadd_rn(c.now, cf.sample_interval);
                    tick_seq = c.seq_next++;
                } else {
                    tick_live = false;
                }
                __syncwarp();
                continue;
            }
        }
        // ---- handle (World::step + Manager::on_event, manager.cpp:333-357)
        bool sched = true;
        int tg[L::WM];
#pragma unroll
        for (int k = 0; k < L::WM; ++k) tg[k] = 0;
        int nt = 0;
        if (kind == 0) {
            c.arrived++;  // Manager::submit: joins the main queue
        } else if (kind == kWindow) {
            sched = t == c.deadline;
        } else if (kind == kCompletion) {
            if (RP_U32(s_seq)[payload] != seq) continue;  // superseded by a rate change
            finish<L>(b, c, payload, out, tg, nt, lane, nblk < 0);
            if constexpr (L::TL) {
                ++n_done;
                if (log_flags & CARMA_LOG_EVENTS)
                    log(CARMA_REC_COMPLETE, RP_U32(s_task)[payload], 0, 0, 0, 0, 0);  // world.cpp:151-153
            }
        } else {  // oom_crash -> handle_oom (manager.cpp:262-267)
            c.oom++;
            if (lane == 0) {
                carma_task_result& o = out[payload];
                o.ooms += 1;
                if (o.first_crash < 0.0) o.first_crash = c.now;
                o.last_crash = c.now;
            }
            if (c.rq_cnt >= static_cast<uint32_t>(L::RQ)) {
                c.status = kStatusRetry;
                break;
            }
            uint32_t tail = c.rq_head + c.rq_cnt;
            if (tail >= static_cast<uint32_t>(L::RQ)) tail -= L::RQ;
            RP_U32(rq)[tail] = payload;
            c.rq_cnt++;
            __syncwarp();
        }
        RPROF_ADD(2, tp2);
        // ---- refresh_rates after finish / place, then try_schedule
        for (;;) {
            if (nt) {
                RPROF_T(tp3);
                refresh_rates<L>(b, c, tg, nt, lane);
                RPROF_ADD(3, tp3);
#if REPLAY_PROF
                prof[12] += RP_U32(nres)[tg[0]] + (nt > 1 ? RP_U32(nres)[tg[1]] : 0);
                prof[13] += 1;
                prof[14] += RP_U32(rcnt)[tg[0]];
#endif
                nt = 0;
                if (c.status) break;
            }
            if (!sched) break;
            sched = false;
            uint32_t head = kNone;
            bool from_recovery = false;
            int gl[L::WM], il[L::WM];
#pragma unroll
            for (int k = 0; k < L::WM; ++k) gl[k] = il[k] = 0;
            uint64_t est_bytes = 0;
            RPROF_T(tp4);
            const int got = decide<L>(b, c, tasks, est, head, from_recovery, gl, il, est_bytes, lane, nblk < 0);
            const int g0 = gl[0], g1 = gl[1];
            RPROF_ADD(4, tp4);
#if REPLAY_PROF
            prof[10] += head != kNone;
            prof[11] += 1;
#endif
            if constexpr (L::TL) {
                // the decision log of try_schedule (manager.cpp:298-318): logged whenever
                // map_task ran; a deferral prints the configured policy
                if ((log_flags & CARMA_LOG_DECISIONS) && head != kNone) {
                    const int pol = got == 0 ? RP_CFG.policy : (from_recovery ? CARMA_POLICY_EXCLUSIVE : RP_CFG.policy);
                    log(CARMA_REC_DECIDE, head, got == 0 ? -1 : g0, est_bytes, 0, 0, static_cast<uint8_t>(pol));
                }
            }
            if (got == 0) break;  // defer; retried on the next completion / expiry
            if (from_recovery) {
                c.rq_head = c.rq_head + 1 == static_cast<uint32_t>(L::RQ) ? 0 : c.rq_head + 1;
                c.rq_cnt--;
            } else {
                c.mq_head++;
            }
            // dispatch (manager.cpp:247-260)
            if (lane == 0 && !from_recovery) out[head].first_attempt = c.now;
            OomInfo oi{};
            RPROF_T(tp5);
            const bool ok = place<L>(b, c, tasks[head], head, gl, il, got, nblk, lane, oi);
            RPROF_ADD(5, tp5);
            if (c.status) break;
            if constexpr (L::TL) {
                if (log_flags & CARMA_LOG_EVENTS) {
                    const uint64_t blk = RP_CFG.alloc_block;
                    if (ok) {
                        log(CARMA_REC_PLACE, head, got, 0, 0, 0, 0);  // world.cpp:126-128
                    } else {  // world.cpp:94-104: want = round_up(max(bytes, 1))
                        const uint64_t bytes = tasks[head].true_mem > 0 ? tasks[head].true_mem : 1;
                        if (L::MG && nblk < 0)
                            log(CARMA_REC_OOM, head, oi.gpu, blk == 0 ? bytes : (bytes + blk - 1) / blk * blk,
                                oi.free_b, oi.largest_b, 0);
                        else
                            log(CARMA_REC_OOM, head, oi.gpu, (bytes + blk - 1) / blk * blk, oi.free_blk * blk,
                                oi.largest_blk * blk, 0);
                    }
                }
            }
            if (ok) {
                if (lane == 0) {
                    carma_task_result& o = out[head];
                    o.final_dispatch = c.now;
                    o.gpu[0] = static_cast<int16_t>(g0);
                    o.gpu[1] = static_cast<int16_t>(got > 1 ? g1 : -1);
                }
#pragma unroll
                for (int k = 0; k < L::WM; ++k) tg[k] = gl[k];
                nt = got;
            }
            // crash (on failure, manager.cpp:251-256) then arm_window
            // (manager.cpp:275-278): one push site for both.
            c.deadline = __dadd_rn(c.now, c.window);
            RPROF_T(tp6);
#pragma unroll 1
            for (int e = ok ? 1 : 0; e < 2; ++e) {
                if (e == 0) heap_push<L>(b, c, __dadd_rn(c.now, delay), (kCrash << 30) | head);
                else heap_push<L>(b, c, c.deadline, kWindow << 30);
            }
            RPROF_ADD(6, tp6);
            if (c.status) break;
        }
        if (c.status) break;
        __syncwarp();
    }
    if constexpr (L::TL) {
        if (lane == 0) {
            p.tl_count[j] = tl_rows;
            p.log_count[j] = n_log;
        }
    }
#if REPLAY_PROF
    prof[7] = events;
    prof[15] = c.seq_next;
    if (lane == 0)
        for (int r = 0; r < 16; ++r) atomicAdd(&g_replay_prof[r], prof[r]);
#endif
    c.events_lo = static_cast<uint32_t>(events);
    c.events_hi = static_cast<uint32_t>(events >> 32);
    __syncwarp();
    const Sc c1 = c;
    finish_job<L>(b, p, j, lane, c1, tasks, out);
#undef tasks
#undef out
#undef est
#undef nblk
}

template <class L, bool SMEM>
__global__ void __launch_bounds__(128, (SMEM && L::H < 1024) ? REPLAY_MIN_CTAS : 1) replay_kernel(Params p) {
    extern __shared__ __align__(16) char smem[];
    const unsigned lane = threadIdx.x & 31;
    const unsigned wib = threadIdx.x >> 5;
    char* b = SMEM ? smem + static_cast<size_t>(wib) * L::bytes
                   : p.gstate + (static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + wib) * L::bytes;
    for (;;) {
        unsigned k = 0;
        if (lane == 0) k = atomicAdd(p.next_job, 1u);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= p.n_list) break;
        run_job<L>(b, p, p.job_list[k], lane);
        __syncwarp();
    }
}

#undef RP_F64
#undef RP_U32
#undef RP_U64
#undef RP_U16
#undef RP_CFG

}  // namespace replay
}  // namespace carma_b200
