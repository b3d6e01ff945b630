// Host staging for the host-buffer predict calls (see stage.hpp).

#include "stage.hpp"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numbers>
#include <thread>
#include <vector>

namespace carma_b200 {

const double* canonical_act_table() {
    static const struct T {
        double v[16];
        T() {
            for (int i = 0; i < 8; ++i) {
                const double a = 2.0 * std::numbers::pi * static_cast<double>(i) / 8.0;  // task.cpp:181-189
                v[2 * i] = std::cos(a);
                v[2 * i + 1] = std::sin(a);
            }
        }
    } t;
    return t.v;
}

namespace {

// A fixed pool of workers; one bulk job at a time (callers serialise on mu_).
class Pool {
  public:
    Pool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        n_ = std::min(hw, 32u);
        for (uint32_t i = 1; i < n_; ++i) threads_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> l(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    uint32_t size() const { return n_; }
    void run(uint32_t parts, const std::function<void(uint32_t, uint32_t)>& fn) {
        std::lock_guard<std::mutex> job(mu_);
        parts = std::max(1u, std::min(parts, n_));
        {
            std::lock_guard<std::mutex> l(m_);
            fn_ = &fn;
            parts_ = parts;
            pending_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0, parts);
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

  private:
    void loop(uint32_t id) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(uint32_t, uint32_t)>* fn;
            uint32_t parts;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                fn = fn_;
                parts = parts_;
            }
            if (id < parts) {
                (*fn)(id, parts);
                std::lock_guard<std::mutex> l(m_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    uint32_t n_ = 1;
    std::vector<std::thread> threads_;
    std::mutex mu_, m_;
    std::condition_variable cv_, done_;
    const std::function<void(uint32_t, uint32_t)>* fn_ = nullptr;
    uint32_t parts_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

inline bool pack_one(const carma_feature_row& r, uint64_t f, const uint64_t* canon, long long* o) {
    constexpr uint64_t k48 = 1ull << 48;
    const uint64_t big = r.total_params | r.total_activations | r.tuple_acts[0] | r.tuple_params[0] |
                         r.tuple_acts[1] | r.tuple_params[1] | r.tuple_acts[2] | r.tuple_params[2];
    const uint64_t tally = r.n_linear | r.n_batchnorm | r.n_dropout | r.n_conv;
    const uint32_t kinds = static_cast<uint32_t>(r.kind[0]) | static_cast<uint32_t>(r.kind[1]) |
                           static_cast<uint32_t>(r.kind[2]);
    uint64_t cb, sb;
    std::memcpy(&cb, &r.act_cos, 8);
    std::memcpy(&sb, &r.act_sin, 8);
    uint64_t code = 8;
    for (uint64_t k = 0; k < 8; ++k)
        if (cb == canon[2 * k] && sb == canon[2 * k + 1]) code = k;
    if (big >= k48 || tally > 255 || r.batch_size >= (1ull << 32) || kinds > 15 || code == 8) return false;
    const uint64_t w[8] = {
        r.total_params | (r.n_linear << 48) | (r.n_batchnorm << 56),
        r.total_activations | (r.n_dropout << 48) | (r.n_conv << 56),
        r.tuple_acts[0] | ((r.batch_size & 0xffffull) << 48),
        r.tuple_params[0] | (static_cast<uint64_t>(r.kind[0]) << 48) | (static_cast<uint64_t>(r.kind[1]) << 52) |
            (static_cast<uint64_t>(r.kind[2]) << 56) | (static_cast<uint64_t>(r.has_layers ? 1 : 0) << 60) |
            (code << 61),
        r.tuple_acts[1] | (f << 48),
        r.tuple_params[1] | ((r.batch_size >> 16) << 48),
        r.tuple_acts[2],
        r.tuple_params[2]};
    for (int k = 0; k < 8; ++k) _mm_stream_si64(o + k, static_cast<long long>(w[k]));
    return true;
}

// One row in the compact encoding (stage.hpp): five u64 words.
inline bool pack_one_compact(const carma_feature_row& r, uint64_t f, const uint64_t* canon, long long* o) {
    constexpr uint64_t k32 = 1ull << 32;
    const uint64_t big = r.total_params | r.total_activations | r.tuple_acts[0] | r.tuple_params[0] |
                         r.tuple_acts[1] | r.tuple_params[1] | r.tuple_acts[2] | r.tuple_params[2];
    const uint64_t tally = r.n_linear | r.n_batchnorm | r.n_dropout | r.n_conv;
    const uint32_t kinds = static_cast<uint32_t>(r.kind[0]) | static_cast<uint32_t>(r.kind[1]) |
                           static_cast<uint32_t>(r.kind[2]);
    uint64_t cb, sb;
    std::memcpy(&cb, &r.act_cos, 8);
    std::memcpy(&sb, &r.act_sin, 8);
    uint64_t code = 8;
    for (uint64_t k = 0; k < 8; ++k)
        if (cb == canon[2 * k] && sb == canon[2 * k + 1]) code = k;
    if (big >= k32 || tally > 255 || r.batch_size >= 4096 || kinds > 15 || code == 8) return false;
    const uint64_t w[5] = {
        r.total_params | (r.total_activations << 32),
        r.tuple_acts[0] | (r.tuple_params[0] << 32),
        r.tuple_acts[1] | (r.tuple_params[1] << 32),
        r.tuple_acts[2] | (r.tuple_params[2] << 32),
        r.n_linear | (r.n_batchnorm << 8) | (r.n_dropout << 16) | (r.n_conv << 24) | (r.batch_size << 32) |
            (code << 44) | (static_cast<uint64_t>(r.kind[0]) << 47) | (static_cast<uint64_t>(r.kind[1]) << 51) |
            (static_cast<uint64_t>(r.kind[2]) << 55) | (static_cast<uint64_t>(r.has_layers ? 1 : 0) << 59) |
            (f << 60)};
    for (int k = 0; k < 5; ++k) _mm_stream_si64(o + k, static_cast<long long>(w[k]));
    return true;
}

}  // namespace

const carma_bit_schema& compact_schema() {
    static const carma_bit_schema s = [] {
        carma_bit_schema c{};
        c.words_per_row = kCompactWords;
        // field order of featurize_bits: 0-6 tallies / batch / totals, 7 act
        // code, 8-10 kinds, 11 has_layers, 12-17 (acts, params) per tuple, 18 family
        const struct { int f, off, w; } lay[] = {
            {5, 0, 32},   {6, 32, 32},  {12, 64, 32},  {13, 96, 32},  {14, 128, 32}, {15, 160, 32}, {16, 192, 32},
            {17, 224, 32}, {0, 256, 8}, {1, 264, 8},   {2, 272, 8},   {3, 280, 8},   {4, 288, 12},  {7, 300, 3},
            {8, 303, 4},  {9, 307, 4},  {10, 311, 4},  {11, 315, 1},  {18, 316, 4}};
        for (const auto& l : lay) {
            c.offset[l.f] = static_cast<uint16_t>(l.off);
            c.width[l.f] = static_cast<uint8_t>(l.w);
        }
        std::memcpy(c.act_table, canonical_act_table(), sizeof(c.act_table));
        return c;
    }();
    return s;
}

bool pack_rows_compact(const carma_feature_row* rows, const int8_t* family, int32_t default_family, uint64_t n,
                       uint64_t* out) {
    uint64_t canon[16];
    std::memcpy(canon, canonical_act_table(), sizeof(canon));
    std::atomic<bool> ok{true};
    const uint32_t parts = static_cast<uint32_t>(std::min<uint64_t>(host_workers(), (n + 16383) / 16384));
    host_parallel(parts, [&](uint32_t p, uint32_t np) {
        const uint64_t b = n * p / np, e = n * (p + 1) / np;
        bool good = true;
        for (uint64_t i = b; i < e && good; ++i) {
            // a negative, absent or unknown family decodes to "no model" (15)
            const int fi = family ? family[i] : default_family;
            const uint64_t f = fi >= 0 && fi < 15 ? static_cast<uint64_t>(fi) : 15u;
            good = pack_one_compact(rows[i], f, canon, reinterpret_cast<long long*>(out + 5 * i));
        }
        _mm_sfence();
        if (!good) ok.store(false, std::memory_order_relaxed);
    });
    return ok.load();
}

void host_parallel(uint32_t parts, const std::function<void(uint32_t, uint32_t)>& fn) { pool().run(parts, fn); }

uint32_t host_workers() { return pool().size(); }

bool compact_rows() {
    static const bool on = [] {
        const char* e = std::getenv("CARMA_E2E_COMPACT");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

bool raw_chunk(uint64_t c, bool inputs_pinned) {
    static const uint64_t every = [] {
        const char* e = std::getenv("CARMA_E2E_RAW_EVERY");
        return e ? std::strtoull(e, nullptr, 10) : 2ull;
    }();
    // CARMA_E2E_RAW_FIRST=1: the raw chunks are 0, k, 2k, ... (the copy
    // engine starts at once while the pool packs chunk 1)
    static const uint64_t phase = [] {
        const char* e = std::getenv("CARMA_E2E_RAW_FIRST");
        return e && std::atoi(e) != 0 ? 0ull : 1ull;
    }();
    return inputs_pinned && every > 0 && (c + phase) % every == 0;
}

bool pack_rows_canonical(const carma_feature_row* rows, const int8_t* family, int32_t default_family, uint64_t n,
                         carma_feature_packed* out) {
    uint64_t canon[16];
    std::memcpy(canon, canonical_act_table(), sizeof(canon));
    std::atomic<bool> ok{true};
    const uint32_t parts = static_cast<uint32_t>(std::min<uint64_t>(host_workers(), (n + 16383) / 16384));
    const int8_t dflt = default_family >= 0 && default_family < CARMA_FAMILIES ? static_cast<int8_t>(default_family)
                                                                                 : static_cast<int8_t>(-1);
    host_parallel(parts, [&](uint32_t p, uint32_t np) {
        const uint64_t b = n * p / np, e = n * (p + 1) / np;
        bool good = true;
        for (uint64_t i = b; i < e && good; ++i) {
            // the family byte as the packed format stores it (w4 >> 48 & 0xff):
            // a negative or absent family decodes to "no model", as for raw rows
            const uint64_t f = static_cast<uint8_t>(family ? family[i] : dflt);
            good = pack_one(rows[i], f, canon, reinterpret_cast<long long*>(out + i));
        }
        _mm_sfence();
        if (!good) ok.store(false, std::memory_order_relaxed);
    });
    return ok.load();
}

}  // namespace carma_b200
