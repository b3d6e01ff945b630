// extern "C" provisioning entry points (include/carma_host.h) over model.cpp.

#include <algorithm>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/carma_host.h"
#include "model.hpp"
#include "status.hpp"

using namespace carma_b200;

namespace {

carma_feature_row to_abi(const FeatureRow& f) {
    carma_feature_row r{};
    r.n_linear = f.n_linear;
    r.n_batchnorm = f.n_batchnorm;
    r.n_dropout = f.n_dropout;
    r.n_conv = f.n_conv;
    r.batch_size = f.batch;
    r.total_params = f.params;
    r.total_activations = f.acts;
    r.act_cos = f.act_cos;
    r.act_sin = f.act_sin;
    r.has_layers = f.has_layers ? 1 : 0;
    for (int k = 0; k < 3; ++k) {
        r.kind[k] = f.kind[k];
        r.tuple_acts[k] = f.tuple_acts[k];
        r.tuple_params[k] = f.tuple_params[k];
    }
    return r;
}

FeatureRow from_abi(const carma_feature_row& r) {
    FeatureRow f;
    f.n_linear = r.n_linear;
    f.n_batchnorm = r.n_batchnorm;
    f.n_dropout = r.n_dropout;
    f.n_conv = r.n_conv;
    f.batch = r.batch_size;
    f.params = r.total_params;
    f.acts = r.total_activations;
    f.act_cos = r.act_cos;
    f.act_sin = r.act_sin;
    f.has_layers = r.has_layers != 0;
    for (int k = 0; k < 3; ++k) {
        f.kind[k] = r.kind[k];
        f.tuple_acts[k] = r.tuple_acts[k];
        f.tuple_params[k] = r.tuple_params[k];
    }
    return f;
}

Trace rows_to_trace(const double* submit, const int32_t* entry, const uint64_t* epochs,
                    uint64_t n) {
    Trace t;
    t.rows.resize(n);
    const int cat = static_cast<int>(catalog().size());
    for (uint64_t i = 0; i < n; ++i) {
        if (entry[i] < 0 || entry[i] >= cat) throw InvalidArg("unknown catalog index");
        t.rows[i] = {submit[i], entry[i], epochs[i]};
    }
    return t;
}

void trace_to_rows(const Trace& t, double* submit, int32_t* entry, uint64_t* epochs) {
    for (std::size_t i = 0; i < t.rows.size(); ++i) {
        submit[i] = t.rows[i].submit;
        entry[i] = t.rows[i].entry;
        epochs[i] = t.rows[i].epochs;
    }
}

}  // namespace

extern "C" {

int carma_host_catalog_size(void) { return static_cast<int>(catalog().size()); }

carma_status carma_host_catalog_entry(int i, char* key, int cap, int32_t* family,
                                      uint64_t* gpus, uint64_t* batch, double* mem_gib) {
    return guarded([&] {
        if (i < 0 || i >= static_cast<int>(catalog().size())) throw InvalidArg("catalog index");
        const CatalogEntry& e = catalog()[static_cast<std::size_t>(i)];
        if (key && cap > 0) {
            std::strncpy(key, e.key.c_str(), static_cast<std::size_t>(cap - 1));
            key[cap - 1] = 0;
        }
        if (family) *family = static_cast<int32_t>(e.family);
        if (gpus) *gpus = e.gpus;
        if (batch) *batch = e.batch;
        if (mem_gib) *mem_gib = e.mem_gib;
    });
}

carma_status carma_host_generate_trace(int32_t mix, uint64_t seed, double* submit,
                                       int32_t* entry, uint64_t* epochs, uint64_t cap,
                                       uint64_t* n_out) {
    return guarded([&] {
        if (mix != CARMA_MIX_T90 && mix != CARMA_MIX_T60) throw InvalidArg("unknown trace mix");
        Trace t = generate_trace(static_cast<Mix>(mix), seed);
        if (t.rows.size() > cap) throw InvalidArg("capacity too small");
        trace_to_rows(t, submit, entry, epochs);
        *n_out = t.rows.size();
    });
}

carma_status carma_host_generate_uniform_trace(uint64_t n, double mean_gap, uint64_t seed,
                                               double* submit, int32_t* entry,
                                               uint64_t* epochs) {
    return guarded([&] {
        if (n == 0 || !(mean_gap > 0.0)) throw InvalidArg("n and mean_gap must be > 0");
        trace_to_rows(generate_uniform_trace(n, mean_gap, seed), submit, entry, epochs);
    });
}

carma_status carma_host_save_trace(const char* path, uint64_t seed, const char* mix,
                                   const double* submit, const int32_t* entry,
                                   const uint64_t* epochs, uint64_t n) {
    return guarded([&] {
        Trace t = rows_to_trace(submit, entry, epochs, n);
        t.seed = seed;
        t.mix = mix ? mix : "";
        save_trace(t, path);
    });
}

carma_status carma_host_load_trace(const char* path, double* submit, int32_t* entry,
                                   uint64_t* epochs, uint64_t cap, uint64_t* n_out) {
    return guarded([&] {
        Trace t = load_trace(path);
        *n_out = t.rows.size();
        if (!submit) return;
        if (t.rows.size() > cap) throw InvalidArg("capacity too small");
        trace_to_rows(t, submit, entry, epochs);
    });
}

carma_status carma_host_materialize(const double* submit, const int32_t* entry,
                                    const uint64_t* epochs, uint64_t n, carma_task* tasks,
                                    carma_feature_row* features, int8_t* family) {
    return guarded([&] {
        if (n == 0) throw InvalidArg("trace contains no tasks");
        std::vector<Task> ts = materialize(rows_to_trace(submit, entry, epochs, n));
        // std::map<std::string, ...> iteration order of the ids
        // (world.cpp:160 std::set, metrics.cpp:26 std::map).
        std::vector<uint32_t> order(n);
        std::iota(order.begin(), order.end(), 0u);
        std::sort(order.begin(), order.end(),
                  [&](uint32_t a, uint32_t b) { return ts[a].id < ts[b].id; });
        for (uint64_t r = 0; r < n; ++r) tasks[order[r]].rank = static_cast<uint32_t>(r);
        for (uint64_t i = 0; i < n; ++i) {
            carma_task& k = tasks[i];
            k.submit = ts[i].submit;
            k.work = ts[i].work;
            k.demand = ts[i].demand;
            k.true_mem = ts[i].true_mem;
            k.estimate = CARMA_NO_ESTIMATE;
            k.gpus = ts[i].gpus;
            if (family) family[i] = static_cast<int8_t>(ts[i].family);
        }
        if (features) {
            // Feature rows depend only on the catalog entry: featurise each
            // entry once (catalog_descriptor is the expensive part).
            std::vector<carma_feature_row> per_entry(catalog().size());
            std::vector<bool> done(catalog().size(), false);
            for (uint64_t i = 0; i < n; ++i) {
                const auto e = static_cast<std::size_t>(entry[i]);
                if (!done[e]) {
                    const CatalogEntry& ce = catalog()[e];
                    per_entry[e] = to_abi(extract_features(catalog_architecture(ce), ce.batch));
                    done[e] = true;
                }
                features[i] = per_entry[e];
            }
        }
    });
}

carma_status carma_host_estimates(int32_t kind, uint64_t safety_margin, const int32_t* entry,
                                  uint64_t n, carma_task* tasks) {
    return guarded([&] {
        if (kind == CARMA_EST_LEARNED) throw InvalidArg("learned estimates come from carma_knn_predict");
        if (kind < CARMA_EST_NONE || kind > CARMA_EST_LEARNED) throw InvalidArg("unknown estimator kind");
        std::vector<FeatureRow> fr(catalog().size());
        std::vector<bool> done(catalog().size(), false);
        for (uint64_t i = 0; i < n; ++i) {
            carma_task& t = tasks[i];
            const auto e = static_cast<std::size_t>(entry[i]);
            const CatalogEntry& ce = catalog().at(e);
            if (!done[e]) {
                fr[e] = extract_features(catalog_architecture(ce), ce.batch);
                done[e] = true;
            }
            const FeatureRow& f = fr[e];
            switch (kind) {
                case CARMA_EST_NONE:
                    t.estimate = CARMA_NO_ESTIMATE;
                    break;
                case CARMA_EST_ORACLE:  // estimators.cpp:34-39
                    t.estimate = t.true_mem + safety_margin;
                    break;
                case CARMA_EST_ANALYTICAL:  // estimators.cpp:41-51
                    t.estimate = 4ull * (4ull * f.params + f.batch * f.acts) + kGiB;
                    break;
                case CARMA_EST_STATIC_GRAPH:  // estimators.cpp:53-61; TF -> no estimate
                    t.estimate = ce.family == Family::Transformer
                                     ? CARMA_NO_ESTIMATE
                                     : 4ull * 4ull * f.params + 64 * kMiB;
                    break;
            }
        }
    });
}

carma_status carma_host_dataset(int32_t family, uint64_t n, uint64_t seed,
                                carma_feature_row* rows, int32_t* bucket, uint64_t* mem) {
    return guarded([&] {
        if (family < 0 || family > 2) throw InvalidArg("unknown family");
        Dataset ds = generate_dataset(static_cast<Family>(family), n, seed);
        for (uint64_t i = 0; i < n; ++i) {
            if (rows) rows[i] = to_abi(ds.rows[i]);
            if (bucket) bucket[i] = ds.bucket[i];
            if (mem) mem[i] = ds.mem[i];
        }
    });
}

carma_status carma_host_fit(int32_t family, uint64_t samples, uint64_t seed, uint32_t k,
                            double* lo, double* hi, double* points, int32_t* labels,
                            uint64_t cap, uint64_t* n_out, uint64_t* bucket_range,
                            uint64_t* holdout_rows, uint64_t* n_holdout) {
    return guarded([&] {
        if (family < 0 || family > 2) throw InvalidArg("unknown family");
        KnnModel m = fit_knn(generate_dataset(static_cast<Family>(family), samples, seed), k);
        if (m.size() > cap || m.holdout_rows.size() > cap) throw InvalidArg("capacity too small");
        std::copy(m.lo.begin(), m.lo.end(), lo);
        std::copy(m.hi.begin(), m.hi.end(), hi);
        std::copy(m.points.begin(), m.points.end(), points);
        std::copy(m.labels.begin(), m.labels.end(), labels);
        *n_out = m.size();
        *bucket_range = m.bucket_range;
        if (holdout_rows) std::copy(m.holdout_rows.begin(), m.holdout_rows.end(), holdout_rows);
        if (n_holdout) *n_holdout = m.holdout_rows.size();
    });
}

// train_learned_estimator's seeded 70/30 split (estimators.cpp:355-361): the
// shuffled row order (a sequential mt19937_64 stream, so it stays on the
// host) and the training-set size.
carma_status carma_host_split_order(uint64_t n, uint64_t seed, uint64_t* order, uint64_t* train_n) {
    return guarded([&] {
        if (n == 0) throw InvalidArg("EmptyDataset: dataset has no rows");
        std::vector<std::size_t> o(n);
        for (std::size_t i = 0; i < o.size(); ++i) o[i] = i;
        Rng rng(seed ^ 0x9e3779b97f4a7c15ull);
        rng.shuffle(o);
        std::copy(o.begin(), o.end(), order);
        *train_n = std::max<uint64_t>(1, n * 7 / 10);
    });
}

// GpuDevice::GpuDevice's MIG branch (gpu.cpp:29-51): instance capacities are
// round_up(fraction * capacity) clipped to what is left, the last instance
// absorbing the remainder when the fractions sum to 1.
carma_status carma_mig_layout(const double* fractions, uint32_t n, carma_replay_config* cfg) {
    return guarded([&] {
        if (!cfg) throw InvalidArg("null config");
        if (n && !fractions) throw InvalidArg("null fractions");
        static const double kDefault[2] = {0.5, 0.5};  // gpu.cpp:31
        const double* src = n ? fractions : kDefault;
        const std::vector<double> f(src, src + (n ? n : 2));
        if (f.size() > CARMA_MAX_MIG) throw Unsupported("more than 8 MIG instances per GPU");
        double sum = 0.0;
        for (double x : f) {
            if (!(x > 0.0) || x > 1.0) throw InvalidArg("ConfigError: mig instance fraction out of (0, 1]");
            sum += x;
        }
        if (sum > 1.0 + 1e-9) throw InvalidArg("ConfigError: mig instance fractions exceed the device");
        const uint64_t capacity = cfg->gpu_capacity, block = cfg->alloc_block;
        // gpu.cpp:58-61: round_up is the identity for alloc_block = 0
        auto round_up = [&](uint64_t b) { return block == 0 ? b : (b + block - 1) / block * block; };
        // block tables (mig_base / mig_blocks) only where the bitmap applies
        const bool blocks = block != 0 && capacity % block == 0 && capacity / block <= 4096;
        uint64_t base = 0;
        carma_replay_config c = *cfg;
        std::memset(c.mig_fraction, 0, sizeof(c.mig_fraction));
        std::memset(c.mig_base, 0, sizeof(c.mig_base));
        std::memset(c.mig_blocks, 0, sizeof(c.mig_blocks));
        std::memset(c.mig_base_bytes, 0, sizeof(c.mig_base_bytes));
        std::memset(c.mig_cap_bytes, 0, sizeof(c.mig_cap_bytes));
        for (std::size_t i = 0; i < f.size(); ++i) {
            uint64_t cap = round_up(static_cast<uint64_t>(f[i] * static_cast<double>(capacity)));
            cap = std::min(cap, capacity - base);
            if (i + 1 == f.size() && sum > 1.0 - 1e-9) cap = capacity - base;
            c.mig_fraction[i] = f[i];
            if (blocks) {
                c.mig_base[i] = static_cast<uint16_t>(base / block);
                c.mig_blocks[i] = static_cast<uint16_t>(cap / block);
            }
            c.mig_base_bytes[i] = base;
            c.mig_cap_bytes[i] = cap;
            base += cap;
        }
        if (base > capacity) throw InvalidArg("ConfigError: mig instances exceed capacity");
        c.mig_count = static_cast<int32_t>(f.size());
        *cfg = c;
    });
}

carma_status carma_host_scalar_features(const carma_feature_row* rows, uint64_t n, double* out) {
    return guarded([&] {
        for (uint64_t i = 0; i < n; ++i) {
            const ScalarRow s = scalar_features(from_abi(rows[i]));
            std::copy(s.begin(), s.end(), out + i * kFeatureDims);
        }
    });
}

}  // extern "C"
