// Sweep inputs on the device: generate_trace + materialisation
// (proj/src/traces.cpp:266-306 and task_from_catalog :238-254), one thread
// per (seed, estimate table), written straight into a replay plan's task
// array — run_sweep's per-seed host loop (runner.cpp:213-249) without the
// host: 100,000 t90 traces take ~11 s to generate and materialise on the
// host, far longer than their replay.
//
// Bit-identical to the host generator: the engine is std::mt19937_64 (the
// reference's Rng, rng.hpp:13-53: seeding, twist and tempering of the
// standard), uniform(n) is the 128-bit multiply-shift, next_double the top
// 53 bits, the exponential gap -mean * log1p(-u), the millisecond grid
// round(t * 1000) / 1000 (no FMA contraction: --fmad=false). log1p is
// glibc's own algorithm and operation order (glibc_log1p.cuh), so every seed
// gives the host generator's bits by construction, not by sampling.

#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../../include/carma_gpu.h"
#include "../../../include/carma_host.h"
#include "../host/model.hpp"
#include "common.cuh"
#include "glibc_log1p.cuh"
#include "tracegen.cuh"

namespace carma_b200 {
namespace {

constexpr int kMaxCatalog = 64;
constexpr int kMt = 312;

struct GenEntry {
    uint64_t true_mem;   // llround(mem_gib * 2^30)
    double epoch_work;   // epoch_minutes * 60.0
    double demand;
    uint64_t opts[2];    // epoch choices
    uint32_t n_opts;
    uint32_t gpus;
};

struct GenCatalog {
    GenEntry e[kMaxCatalog];
    uint8_t pool[3][kMaxCatalog];  // entries per weight class, catalog order
    uint32_t pool_n[3];
    uint32_t n;
};

__constant__ GenCatalog c_cat;

struct Mt64 {
    uint64_t s[kMt];
    int i;
    __device__ __forceinline__ void seed(uint64_t v) {
        s[0] = v;
        for (int k = 1; k < kMt; ++k) s[k] = 6364136223846793005ull * (s[k - 1] ^ (s[k - 1] >> 62)) + static_cast<uint64_t>(k);
        i = kMt;
    }
    __device__ __forceinline__ void twist() {
        constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull, kA = 0xB5026F5AA96619E9ull;
#pragma unroll 1
        for (int k = 0; k < kMt; ++k) {
            const uint64_t x = (s[k] & kUpper) | (s[k + 1 < kMt ? k + 1 : 0] & kLower);
            uint64_t xa = x >> 1;
            if (x & 1ull) xa ^= kA;
            s[k] = s[k + 156 < kMt ? k + 156 : k + 156 - kMt] ^ xa;
        }
        i = 0;
    }
    __device__ __forceinline__ uint64_t next() {
        if (i >= kMt) twist();
        uint64_t y = s[i++];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        y ^= y >> 43;
        return y;
    }
    __device__ __forceinline__ uint64_t uniform(uint64_t n) { return __umul64hi(next(), n); }
    __device__ __forceinline__ double next_double() {
        return __dmul_rn(static_cast<double>(next() >> 11), 0x1.0p-53);
    }
};

template <int T>
__global__ void __launch_bounds__(128) gen_traces(int32_t mix, const uint64_t* __restrict__ seeds, uint32_t n_seeds,
                                                  const uint64_t* __restrict__ tables, uint32_t n_tables,
                                                  carma_task* __restrict__ tasks, int32_t* __restrict__ entries) {
    const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= static_cast<uint64_t>(n_seeds) * n_tables) return;
    const uint32_t si = static_cast<uint32_t>(gid % n_seeds);
    const uint32_t tb = static_cast<uint32_t>(gid / n_seeds);
    Mt64 rng;
    rng.seed(seeds[si]);
    // class quotas (traces.cpp:268-276): t90 = 59 light, 24 medium, 7 heavy; t60 = 50 medium, 10 heavy
    uint8_t picks[T];
    int n = 0;
    const int wc0 = mix == CARMA_MIX_T90 ? 0 : 1;
    for (int wc = wc0; wc < 3; ++wc) {
        const int count = mix == CARMA_MIX_T90 ? (wc == 0 ? 59 : wc == 1 ? 24 : 7) : (wc == 1 ? 50 : 10);
        const uint32_t pn = c_cat.pool_n[wc];
        for (int k = 0; k < count; ++k) picks[n++] = c_cat.pool[wc][rng.uniform(pn)];
    }
    for (int k = T; k > 1; --k) {  // Rng::shuffle (rng.hpp:46-52)
        const int j = static_cast<int>(rng.uniform(static_cast<uint64_t>(k)));
        const uint8_t t = picks[k - 1];
        picks[k - 1] = picks[j];
        picks[j] = t;
    }
    const uint64_t trace = static_cast<uint64_t>(tb) * n_seeds + si;
    carma_task* out = tasks + trace * T;
    const uint64_t* table = tables ? tables + static_cast<uint64_t>(tb) * c_cat.n : nullptr;
    double clock = 0.0;
    for (int k = 0; k < T; ++k) {
        const GenEntry& e = c_cat.e[picks[k]];
        if (k > 0) clock = __dadd_rn(clock, __dmul_rn(-120.0, glibc_log1p(-rng.next_double())));
        carma_task t;
        t.submit = __ddiv_rn(round(__dmul_rn(clock, 1000.0)), 1000.0);
        const uint64_t epochs = e.n_opts == 1 ? e.opts[0] : e.opts[rng.uniform(e.n_opts)];
        t.work = __dmul_rn(static_cast<double>(epochs), e.epoch_work);
        t.demand = e.demand;
        t.true_mem = e.true_mem;
        t.estimate = table ? table[picks[k]] : CARMA_NO_ESTIMATE;
        t.gpus = e.gpus;
        t.rank = static_cast<uint32_t>(k);  // ids t000-.. t0NN-: string order = row order below 1000 rows
        out[k] = t;
        if (entries) entries[trace * T + k] = picks[k];
    }
}

void upload_catalog() {
    static std::mutex mu;
    static int done_mask = 0;  // per device bit (devices < 31)
    int dev = 0;
    CARMA_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 31 && ((done_mask >> dev) & 1)) return;
    const auto& cat = catalog();
    if (cat.size() > static_cast<size_t>(kMaxCatalog)) throw Unsupported("catalog too large");
    GenCatalog g{};
    g.n = static_cast<uint32_t>(cat.size());
    for (size_t i = 0; i < cat.size(); ++i) {
        const CatalogEntry& e = cat[i];
        GenEntry& d = g.e[i];
        d.true_mem = static_cast<uint64_t>(std::llround(e.mem_gib * static_cast<double>(kGiB)));  // materialize
        d.epoch_work = e.epoch_minutes * 60.0;
        d.demand = e.demand;
        if (e.epoch_options.empty() || e.epoch_options.size() > 2) throw Unsupported("epoch options");
        d.n_opts = static_cast<uint32_t>(e.epoch_options.size());
        for (size_t k = 0; k < e.epoch_options.size(); ++k) d.opts[k] = e.epoch_options[k];
        d.gpus = static_cast<uint32_t>(e.gpus);
        const int wc = static_cast<int>(e.wclass);
        g.pool[wc][g.pool_n[wc]++] = static_cast<uint8_t>(i);
    }
    CARMA_CUDA(cudaMemcpyToSymbol(c_cat, &g, sizeof(g)));
    if (dev < 31) done_mask |= 1 << dev;
}

}  // namespace

uint32_t trace_rows(int32_t mix) {
    if (mix == CARMA_MIX_T90) return 90;
    if (mix == CARMA_MIX_T60) return 60;
    throw InvalidArg("ConfigError: unknown trace mix");
}

uint32_t catalog_size() { return static_cast<uint32_t>(catalog().size()); }

void launch_generate_traces(int32_t mix, const uint64_t* d_seeds, uint32_t n_seeds, const uint64_t* d_tables,
                            uint32_t n_tables, carma_task* d_tasks, int32_t* d_entries, cudaStream_t s) {
    upload_catalog();
    const uint64_t n = static_cast<uint64_t>(n_seeds) * n_tables;
    if (n == 0) return;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    if (trace_rows(mix) == 90)
        gen_traces<90><<<grid, 128, 0, s>>>(mix, d_seeds, n_seeds, d_tables, n_tables, d_tasks, d_entries);
    else
        gen_traces<60><<<grid, 128, 0, s>>>(mix, d_seeds, n_seeds, d_tables, n_tables, d_tasks, d_entries);
    CARMA_CUDA(cudaGetLastError());
}

}  // namespace carma_b200

// Pins glibc_log1p (the code the device runs, built for the host) to the C
// library's log1p: n inputs from a xorshift stream over the ranges the trace
// generator and the branch boundaries exercise. Returns the mismatch count.
extern "C" carma_status carma_host_check_log1p(uint64_t n, uint64_t seed, uint64_t* mismatches) {
    return carma_b200::guarded([&] {
        if (!mismatches) throw carma_b200::InvalidArg("null argument");
        uint64_t s = seed ? seed : 88172645463325252ull, bad = 0;
        for (uint64_t i = 0; i < n; ++i) {
            s ^= s << 13;
            s ^= s >> 7;
            s ^= s << 17;
            const double u = static_cast<double>(s >> 11) * 0x1.0p-53;
            double x = -u;  // the generator's domain: log1p(-u), u in [0, 1)
            switch (i % 6) {
                case 1: x = -static_cast<double>(s >> 40) * 0x1.0p-24; break;
                case 2: x = -u * 1e-6; break;
                case 3: x = u * 0.5 - 0.25; break;
                case 4: {  // hi words around the k = 0 boundary 0xbfd2bec3
                    const uint64_t b = (static_cast<uint64_t>(0xbfd2bec2u + (s & 3)) << 32) | (s >> 32);
                    std::memcpy(&x, &b, 8);
                    break;
                }
                case 5: x = (u - 0.5) * 0x1.0p-27; break;  // the |x| < 2^-29 branch
                default: break;
            }
            const double a = std::log1p(x), b = carma_b200::glibc_log1p(x);
            if (std::memcmp(&a, &b, 8) != 0) ++bad;
        }
        *mismatches = bad;
    });
}
