// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (CARMA artifact,
// compiled from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libcarma_ref.so). It exists so pytest (ctypes) and bench.py's
// cpu_baseline / `--impl reference` legs can drive the reference's own
// public API and read its outputs as flat arrays:
//   * generate_synthetic_dataset / train_learned_estimator / estimate_learned
//     (proj/src/estimators.cpp:221-264, :344-436, :540-551)
//   * generate_trace / materialize_trace / save_trace (proj/src/traces.cpp)
//   * run_simulation (proj/src/runner.cpp:40-147) and compute_report
//     (proj/src/metrics.cpp:16-70)
// Nothing here re-implements reference behaviour; it only marshals.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nlohmann/json.hpp>

#include "carma/errors.hpp"
#include "carma/estimators.hpp"
#include "carma/runner.hpp"
#include "carma/traces.hpp"

using namespace carma;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return 1;
}

ModelFamily fam(int f) { return static_cast<ModelFamily>(f); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_catalog_size() { return static_cast<int>(builtin_catalog().size()); }

// Catalog row i: family, gpus, batch, weight class, mem_gib, epoch minutes,
// demand, n epoch options (<=2) and the options.
int ref_catalog_entry(int i, char* key, int key_cap, int* family, uint64_t* gpus,
                      uint64_t* batch, int* wclass, double* mem_gib, double* et_min,
                      double* demand, int* n_epochs, uint64_t* epochs2) {
    const auto& e = builtin_catalog().at(static_cast<std::size_t>(i));
    std::snprintf(key, static_cast<std::size_t>(key_cap), "%s", e.key.c_str());
    *family = static_cast<int>(e.family);
    *gpus = e.gpus;
    *batch = e.batch_size;
    *wclass = static_cast<int>(e.weight_class);
    *mem_gib = e.mem_gib;
    *et_min = e.epoch_time_minutes;
    *demand = e.smact_demand;
    *n_epochs = static_cast<int>(e.epoch_options.size());
    for (std::size_t k = 0; k < e.epoch_options.size() && k < 2; ++k)
        epochs2[k] = e.epoch_options[k];
    return 0;
}

// Dataset rows as the 19 scalar features (scalar_features, estimators.cpp:317),
// plus labels and true bytes.
int ref_dataset(int family, uint64_t n, uint64_t seed, double* feats,
                int32_t* bucket, uint64_t* mem) {
    try {
        EstimatorDataset ds = generate_synthetic_dataset(fam(family), n, seed);
        for (std::size_t i = 0; i < ds.rows.size(); ++i) {
            ScalarFeatures s = scalar_features(ds.rows[i].features);
            std::memcpy(feats + i * kScalarFeatureCount, s.data(), sizeof(double) * kScalarFeatureCount);
            bucket[i] = ds.rows[i].bucket;
            mem[i] = ds.rows[i].mem_bytes;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Compact FeatureVector view of dataset rows: 7 tallies, cos, sin, and the
// first/middle/last layer tuples (kind, acts, params) — the inputs
// scalar_features consumes.
int ref_dataset_fv(int family, uint64_t n, uint64_t seed, uint64_t* tallies /*n*7*/,
                   double* cossin /*n*2*/, int32_t* kinds /*n*3*/,
                   uint64_t* tup /*n*6: acts,params x3*/, uint64_t* n_layers) {
    try {
        EstimatorDataset ds = generate_synthetic_dataset(fam(family), n, seed);
        for (std::size_t i = 0; i < ds.rows.size(); ++i) {
            const FeatureVector& f = ds.rows[i].features;
            uint64_t* t = tallies + i * 7;
            t[0] = f.n_linear; t[1] = f.n_batchnorm; t[2] = f.n_dropout; t[3] = f.n_conv;
            t[4] = f.batch_size; t[5] = f.total_params; t[6] = f.total_activations;
            cossin[i * 2] = f.act_cos;
            cossin[i * 2 + 1] = f.act_sin;
            const auto& L = f.layer_tuples;
            n_layers[i] = L.size();
            const LayerTuple* pick[3] = {&L.front(), &L[L.size() / 2], &L.back()};
            for (int k = 0; k < 3; ++k) {
                kinds[i * 3 + k] = pick[k]->kind_code;
                tup[i * 6 + 2 * k] = pick[k]->activation_count;
                tup[i * 6 + 2 * k + 1] = pick[k]->param_count;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Trains exactly like provision_estimators (runner.cpp:17-38) and exports the
// snapshot (LearnedEstimator::save, estimators.cpp:481) as arrays.
int ref_train(int family, uint64_t samples, uint64_t seed, uint64_t k,
              const char* tmp_json, double* lo, double* hi, double* points,
              int32_t* labels, uint64_t cap, uint64_t* n_out, uint64_t* bucket_range,
              double* holdout3) {
    try {
        EstimatorDataset ds = generate_synthetic_dataset(fam(family), samples, seed);
        LearnedEstimator est = train_learned_estimator(ds, k);
        est.save(tmp_json);
        std::ifstream in(tmp_json);
        nlohmann::ordered_json j = nlohmann::ordered_json::parse(in);
        auto vlo = j.at("lo").get<std::vector<double>>();
        auto vhi = j.at("hi").get<std::vector<double>>();
        std::copy(vlo.begin(), vlo.end(), lo);
        std::copy(vhi.begin(), vhi.end(), hi);
        auto lab = j.at("labels").get<std::vector<int>>();
        if (lab.size() > cap) throw CarmaError("cap too small");
        *n_out = lab.size();
        std::size_t i = 0;
        for (const auto& p : j.at("points")) {
            auto v = p.get<std::vector<double>>();
            std::copy(v.begin(), v.end(), points + i * kScalarFeatureCount);
            labels[i] = lab[i];
            ++i;
        }
        *bucket_range = est.bucket_range();
        holdout3[0] = est.holdout().accuracy;
        holdout3[1] = est.holdout().macro_f1;
        holdout3[2] = est.holdout().underestimate_rate;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

namespace {
std::map<std::pair<int, std::uint64_t>, LearnedEstimator> g_models;
std::mutex g_models_mu;

const LearnedEstimator& model_for(int family, uint64_t samples, uint64_t seed, uint64_t k) {
    std::lock_guard<std::mutex> lock(g_models_mu);
    auto key = std::make_pair(family, seed * 1000003ull + samples * 31ull + k);
    auto it = g_models.find(key);
    if (it == g_models.end()) {
        EstimatorDataset ds = generate_synthetic_dataset(fam(family), samples, seed);
        it = g_models.emplace(key, train_learned_estimator(ds, k)).first;
    }
    return it->second;
}
}  // namespace

// estimate_learned over the FeatureVectors of generate_synthetic_dataset(qfamily, n, qseed).
int ref_predict_dataset(int family, uint64_t samples, uint64_t seed, uint64_t k,
                        uint64_t n, uint64_t qseed, int32_t* out_bucket,
                        uint64_t* out_bytes) {
    try {
        const LearnedEstimator& est = model_for(family, samples, seed, k);
        EstimatorDataset q = generate_synthetic_dataset(fam(family), n, qseed);
        for (std::size_t i = 0; i < q.rows.size(); ++i) {
            MemoryEstimate m = estimate_learned(est, q.rows[i].features, fam(family));
            out_bucket[i] = *m.bucket;
            out_bytes[i] = m.bytes;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// CPU throughput of the reference predict (estimate_learned) on n_threads
// host threads over `reps` passes of the rows of dataset (family, n, qseed).
// Returns elapsed seconds of the timed region (dataset generation excluded).
double ref_bench_predict(int family, uint64_t samples, uint64_t seed, uint64_t k,
                         uint64_t n, uint64_t qseed, int n_threads, int reps,
                         uint64_t* checksum) {
    try {
        const LearnedEstimator& est = model_for(family, samples, seed, k);
        EstimatorDataset q = generate_synthetic_dataset(fam(family), n, qseed);
        std::atomic<std::uint64_t> sum{0};
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < n_threads; ++t) {
            pool.emplace_back([&, t]() {
                std::uint64_t local = 0;
                for (int r = 0; r < reps; ++r)
                    for (std::size_t i = static_cast<std::size_t>(t); i < q.rows.size();
                         i += static_cast<std::size_t>(n_threads))
                        local += estimate_learned(est, q.rows[i].features, fam(family)).bytes >> 20;
                sum += local;
            });
        }
        for (auto& th : pool) th.join();
        double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *checksum = sum.load();
        return s;
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

// The FeatureVector summary the product's batch API consumes (the
// carma_feature_row layout of include/carma_gpu.h, restated here so the
// reference side needs no product header).
struct FeatRow {
    uint64_t n_linear, n_batchnorm, n_dropout, n_conv;
    uint64_t batch_size, total_params, total_activations;
    double act_cos, act_sin;
    int32_t kind[3];
    int32_t has_layers;
    uint64_t tuple_acts[3];
    uint64_t tuple_params[3];
};
static_assert(sizeof(FeatRow) == 136, "FeatRow must match carma_feature_row");

// estimate_learned (estimators.cpp:540-551) over n feature rows on `threads`
// host threads, each row routed to the model of its family trained exactly as
// provision_estimators does (seed est_seed + 101 * family, runner.cpp:31-32).
// The FeatureVector carries the first / middle / last layer tuples, which is
// all scalar_features reads (estimators.cpp:317-342): with three tuples
// [first, middle, last], L[size/2] is the middle one.
int ref_estimate_rows(const FeatRow* rows, const int8_t* family, uint64_t n, uint64_t samples,
                      uint64_t est_seed, uint64_t k, int threads, int32_t* out_bucket, uint64_t* out_bytes) {
    try {
        for (int f = 0; f < 3; ++f) model_for(f, samples, est_seed + 101ull * static_cast<uint64_t>(f), k);
        std::vector<std::thread> pool;
        std::atomic<int> bad{0};
        std::string err;
        std::mutex err_mu;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t]() {
                try {
                    const uint64_t b = n * static_cast<uint64_t>(t) / static_cast<uint64_t>(threads);
                    const uint64_t e = n * static_cast<uint64_t>(t + 1) / static_cast<uint64_t>(threads);
                    FeatureVector fv;
                    fv.layer_tuples.resize(3);
                    for (uint64_t i = b; i < e; ++i) {
                        const FeatRow& r = rows[i];
                        const int f = family[i];
                        fv.n_linear = r.n_linear; fv.n_batchnorm = r.n_batchnorm; fv.n_dropout = r.n_dropout;
                        fv.n_conv = r.n_conv; fv.batch_size = r.batch_size; fv.total_params = r.total_params;
                        fv.total_activations = r.total_activations; fv.act_cos = r.act_cos; fv.act_sin = r.act_sin;
                        fv.layer_tuples.resize(r.has_layers ? 3 : 0);
                        for (int j = 0; r.has_layers && j < 3; ++j)
                            fv.layer_tuples[static_cast<std::size_t>(j)] = {r.kind[j], r.tuple_acts[j], r.tuple_params[j]};
                        const LearnedEstimator& est =
                            model_for(f, samples, est_seed + 101ull * static_cast<uint64_t>(f), k);
                        MemoryEstimate m = estimate_learned(est, fv, fam(f));
                        out_bucket[i] = *m.bucket;
                        out_bytes[i] = m.bytes;
                    }
                } catch (const std::exception& ex) {
                    std::lock_guard<std::mutex> lock(err_mu);
                    err = ex.what();
                    bad = 1;
                }
            });
        }
        for (auto& th : pool) th.join();
        if (bad) throw CarmaError(err);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Trace generation (traces.cpp:266-306): rows as (submit, catalog index, epochs).
int ref_gen_trace(int mix, uint64_t seed, double* submit, int32_t* cat_idx,
                  uint64_t* epochs, uint64_t cap, uint64_t* n_out) {
    try {
        TraceFile tf = generate_trace(static_cast<TraceMix>(mix), seed);
        if (tf.rows.size() > cap) throw CarmaError("cap too small");
        const auto& cat = builtin_catalog();
        for (std::size_t i = 0; i < tf.rows.size(); ++i) {
            submit[i] = tf.rows[i].submit_s;
            epochs[i] = tf.rows[i].epochs;
            for (std::size_t c = 0; c < cat.size(); ++c)
                if (cat[c].key == tf.rows[i].catalog_key) cat_idx[i] = static_cast<int32_t>(c);
        }
        *n_out = tf.rows.size();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Writes a `#carma-trace v1` file from rows (save_trace, traces.cpp:308).
int ref_save_trace(const char* path, uint64_t seed, const char* mix, const double* submit,
                   const int32_t* cat_idx, const uint64_t* epochs, uint64_t n) {
    try {
        TraceFile tf;
        tf.seed = seed;
        tf.mix = mix;
        const auto& cat = builtin_catalog();
        for (uint64_t i = 0; i < n; ++i)
            tf.rows.push_back({submit[i], cat.at(static_cast<std::size_t>(cat_idx[i])).key, epochs[i]});
        save_trace(tf, path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// materialize_trace(load_trace_file(path)) (traces.cpp:368-385): per task the
// replay inputs and the 19 scalar features of the task's FeatureVector.
int ref_materialize(const char* path, uint64_t cap, double* submit, uint64_t* true_mem,
                    double* work, double* demand, uint64_t* gpus, int32_t* family,
                    uint64_t* batch, double* feats, char* ids, int id_stride,
                    uint64_t* n_out) {
    try {
        std::vector<TaskSpec> tasks = load_trace(path);
        if (tasks.size() > cap) throw CarmaError("cap too small");
        for (std::size_t i = 0; i < tasks.size(); ++i) {
            const TaskSpec& t = tasks[i];
            submit[i] = t.submit_time;
            true_mem[i] = t.true_mem_bytes;
            work[i] = t.total_work();
            demand[i] = t.smact_demand;
            gpus[i] = t.gpus_requested;
            family[i] = static_cast<int32_t>(t.model.family);
            batch[i] = t.batch_size;
            ScalarFeatures s = scalar_features(extract_features(t.model, t.batch_size));
            std::memcpy(feats + i * kScalarFeatureCount, s.data(), sizeof(double) * kScalarFeatureCount);
            if (ids) std::snprintf(ids + i * id_stride, static_cast<std::size_t>(id_stride), "%s", t.id.c_str());
        }
        *n_out = tasks.size();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

struct RefConfig {
    int policy;        // Policy enum (manager.hpp:15)
    int estimator;     // EstimatorKind (manager.hpp:19)
    int mode;          // CollocationMode (gpu.hpp:14)
    int rr_apply_preconditions;
    double max_smact;
    int has_min_free;
    uint64_t min_free;
    uint64_t safety_margin;
    double monitor_window;
    int gpu_count;
    uint64_t gpu_capacity;
    uint64_t alloc_block;
    uint64_t estimator_seed;
    uint64_t estimator_k;
    uint64_t estimator_samples;
    int32_t mig_count;         // RunConfig::mig_instances (runner.hpp:23)
    int32_t mig_reserved;
    double mig_fractions[8];
    double sample_interval;    // > 0: RunConfig::enable_timeline with this interval
    int32_t log_flags;         // 1: enable_event_log, 2: verbose_decisions
    int32_t log_reserved;
};

struct RefTaskOut {
    double submit;
    double first_attempt;
    double final_dispatch;
    double complete;
    double first_crash;
    double last_crash;
    double executed;
    uint32_t n_attempts;
    uint32_t ooms;
    int32_t gpu0;
    int32_t gpu1;
};

struct RefTraceOut {
    double trace_total_time;
    double avg_wait;
    double avg_exec;
    double avg_jct;
    double energy_mj;
    double last_complete;
    double first_submit;
    int32_t oom_count;
    int32_t n_tasks;
};

namespace {
RunConfig make_rc(const RefConfig& c) {
    RunConfig rc;
    rc.policy.policy = static_cast<Policy>(c.policy);
    rc.policy.estimator = static_cast<EstimatorKind>(c.estimator);
    rc.policy.collocation_mode = static_cast<CollocationMode>(c.mode);
    rc.policy.rr_apply_preconditions = c.rr_apply_preconditions != 0;
    rc.policy.preconditions.max_smact = c.max_smact;
    if (c.has_min_free) rc.policy.preconditions.min_free_mem = c.min_free;
    rc.policy.preconditions.safety_margin = c.safety_margin;
    rc.policy.monitor_window = c.monitor_window;
    rc.constants.gpu_count = c.gpu_count;
    rc.constants.gpu_capacity = c.gpu_capacity;
    rc.constants.alloc_block = c.alloc_block;
    rc.estimator_seed = c.estimator_seed;
    rc.estimator_k = c.estimator_k;
    rc.estimator_samples = c.estimator_samples;
    for (int i = 0; i < c.mig_count && i < 8; ++i) rc.mig_instances.push_back(c.mig_fractions[i]);
    if (c.sample_interval > 0.0) {
        rc.enable_timeline = true;
        rc.sample_interval = c.sample_interval;
    }
    rc.enable_event_log = (c.log_flags & 1) != 0;
    rc.verbose_decisions = (c.log_flags & 2) != 0;
    return rc;
}

void export_run(const RunArtifacts& art, const std::vector<std::string>& order,
                RefTaskOut* tout, RefTraceOut* rout, double* gpu_energy,
                double* gpu_smact, uint64_t* gpu_peak) {
    const auto& timing = art.record.timing;
    for (std::size_t i = 0; i < order.size(); ++i) {
        const TaskTiming& t = timing.at(order[i]);
        RefTaskOut& o = tout[i];
        o.submit = t.submit;
        o.first_attempt = t.dispatch_attempts.empty() ? -1.0 : t.dispatch_attempts.front();
        o.final_dispatch = t.final_dispatch;
        o.complete = t.complete;
        o.first_crash = t.crash_times.empty() ? -1.0 : t.crash_times.front();
        o.last_crash = t.crash_times.empty() ? -1.0 : t.crash_times.back();
        o.n_attempts = static_cast<uint32_t>(t.dispatch_attempts.size());
        o.ooms = static_cast<uint32_t>(t.oom_count);
        const TaskRun& run = art.runs.at(order[i]);
        o.executed = run.executed_integral;
        o.gpu0 = run.gpu_ids.size() > 0 ? run.gpu_ids[0] : -1;
        o.gpu1 = run.gpu_ids.size() > 1 ? run.gpu_ids[1] : -1;
    }
    rout->trace_total_time = art.report.trace_total_time;
    rout->avg_wait = art.report.avg_wait;
    rout->avg_exec = art.report.avg_exec;
    rout->avg_jct = art.report.avg_jct;
    rout->energy_mj = art.report.energy_mj;
    rout->last_complete = art.record.last_complete;
    rout->first_submit = art.record.first_submit;
    rout->oom_count = art.report.oom_count;
    rout->n_tasks = static_cast<int32_t>(order.size());
    for (std::size_t g = 0; g < art.record.gpu_energy_j.size(); ++g) {
        gpu_energy[g] = art.record.gpu_energy_j[g];
        gpu_smact[g] = art.record.gpu_mean_smact[g];
        gpu_peak[g] = art.record.gpu_peak_mem[g];
    }
}
}  // namespace

// One run_simulation over a generated trace (mix >= 0) or a trace file.
// Per-task outputs are in materialized (trace row) order.
int ref_run(const RefConfig* cfg, int mix, uint64_t seed, const char* trace_path,
            RefTaskOut* tout, uint64_t task_cap, RefTraceOut* rout,
            double* gpu_energy, double* gpu_smact, uint64_t* gpu_peak) {
    try {
        RunConfig rc = make_rc(*cfg);
        std::vector<TaskSpec> tasks;
        if (mix >= 0) {
            rc.mix = static_cast<TraceMix>(mix);
            rc.trace_seed = seed;
            tasks = materialize_trace(generate_trace(*rc.mix, seed));
        } else {
            rc.trace_path = trace_path;
            tasks = load_trace(trace_path);
        }
        if (tasks.size() > task_cap) throw CarmaError("task cap too small");
        std::vector<std::string> order;
        for (const auto& t : tasks) order.push_back(t.id);
        RunArtifacts art = run_simulation(rc);
        export_run(art, order, tout, rout, gpu_energy, gpu_smact, gpu_peak);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Reference CPU sweep throughput (run_sweep's pool shape, runner.cpp:209-249):
// seeds [seed0, seed0+n_seeds) x policies, n_threads workers. Returns elapsed
// seconds; *placed = total tasks placed (sum of n_tasks over runs).
double ref_bench_sweep(const RefConfig* base, int mix, uint64_t seed0, uint64_t n_seeds,
                       const int32_t* policies, int n_policies, int n_threads,
                       uint64_t* placed, double* energy_checksum) {
    try {
        struct Job { int policy; uint64_t seed; };
        std::vector<Job> jobs;
        for (int p = 0; p < n_policies; ++p)
            for (uint64_t s = 0; s < n_seeds; ++s) jobs.push_back({policies[p], seed0 + s});
        std::atomic<std::size_t> next{0};
        std::atomic<std::uint64_t> tasks{0};
        std::vector<double> esum(static_cast<std::size_t>(n_threads), 0.0);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < n_threads; ++t) {
            pool.emplace_back([&, t]() {
                for (;;) {
                    std::size_t i = next.fetch_add(1);
                    if (i >= jobs.size()) return;
                    RefConfig c = *base;
                    c.policy = jobs[i].policy;
                    RunConfig rc = make_rc(c);
                    rc.mix = static_cast<TraceMix>(mix);
                    rc.trace_seed = jobs[i].seed;
                    RunArtifacts art = run_simulation(rc);
                    tasks += art.report.tasks.size();
                    esum[static_cast<std::size_t>(t)] += art.report.energy_mj;
                }
            });
        }
        for (auto& th : pool) th.join();
        double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *placed = tasks.load();
        double e = 0.0;
        for (double v : esum) e += v;
        *energy_checksum = e;
        return s;
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

// run_simulation for every (config, seed) job of a generated-trace sweep on
// `threads` host threads (run_sweep's pool, runner.cpp:209-249): job
// j = c * n_seeds + s runs cfgs[c] on generate_trace(mix, seed0 + s). Outputs
// per job (rout[j]; GPU results at j * G) and per task (tout at j *
// tasks_per_trace, materialized order); every trace must have
// tasks_per_trace tasks.
int ref_run_jobs(const RefConfig* cfgs, int n_cfg, int mix, uint64_t seed0, uint64_t n_seeds, int threads,
                 uint64_t tasks_per_trace, RefTaskOut* tout, RefTraceOut* rout, double* gpu_energy,
                 double* gpu_smact, uint64_t* gpu_peak) {
    try {
        const uint64_t n_jobs = static_cast<uint64_t>(n_cfg) * n_seeds;
        std::atomic<uint64_t> next{0};
        std::atomic<int> bad{0};
        std::string err;
        std::mutex err_mu;
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&]() {
                for (;;) {
                    const uint64_t j = next.fetch_add(1);
                    if (j >= n_jobs || bad) return;
                    try {
                        const RefConfig& c = cfgs[j / n_seeds];
                        const uint64_t g = static_cast<uint64_t>(c.gpu_count);
                        RunConfig rc = make_rc(c);
                        rc.mix = static_cast<TraceMix>(mix);
                        rc.trace_seed = seed0 + j % n_seeds;
                        std::vector<TaskSpec> tasks = materialize_trace(generate_trace(*rc.mix, rc.trace_seed));
                        if (tasks.size() != tasks_per_trace) throw CarmaError("unexpected trace length");
                        std::vector<std::string> order;
                        for (const auto& tk : tasks) order.push_back(tk.id);
                        RunArtifacts art = run_simulation(rc);
                        export_run(art, order, tout + j * tasks_per_trace, rout + j, gpu_energy + j * g,
                                   gpu_smact + j * g, gpu_peak + j * g);
                    } catch (const std::exception& ex) {
                        std::lock_guard<std::mutex> lock(err_mu);
                        err = ex.what();
                        bad = 1;
                    }
                }
            });
        }
        for (auto& th : pool) th.join();
        if (bad) throw CarmaError(err);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The timeline of one run (RunArtifacts::timeline, header included),
// newline-joined into buf[cap].
int ref_timeline(const RefConfig* cfg, int mix, uint64_t seed, char* buf, uint64_t cap) {
    try {
        RunConfig rc = make_rc(*cfg);
        rc.mix = static_cast<TraceMix>(mix);
        rc.trace_seed = seed;
        RunArtifacts art = run_simulation(rc);
        std::string out;
        for (const auto& l : art.timeline) out += l + "\n";
        if (out.size() + 1 > cap) throw CarmaError("timeline buffer too small");
        std::memcpy(buf, out.c_str(), out.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The event log and decision log of one run, newline-joined.
int ref_logs(const RefConfig* cfg, int mix, uint64_t seed, char* events, uint64_t ecap, char* decisions,
             uint64_t dcap) {
    try {
        RunConfig rc = make_rc(*cfg);
        rc.mix = static_cast<TraceMix>(mix);
        rc.trace_seed = seed;
        RunArtifacts art = run_simulation(rc);
        std::string e, d;
        for (const auto& l : art.event_log) e += l + "\n";
        for (const auto& l : art.decision_log) d += l + "\n";
        if (e.size() + 1 > ecap || d.size() + 1 > dcap) throw CarmaError("log buffer too small");
        std::memcpy(events, e.c_str(), e.size() + 1);
        std::memcpy(decisions, d.c_str(), d.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The reference's own run_sweep (runner.cpp:192-283): cells from RefConfig
// rows (policy part), base constants/estimator provisioning from cells[0],
// trace mix `mix`, the given seeds, one worker per hardware thread. Writes the
// sweep CSV (per-seed rows + median rows) into csv[cap].
int ref_run_sweep(const RefConfig* cells, int n_cells, int mix, const uint64_t* seeds, int n_seeds,
                  char* csv, uint64_t cap) {
    try {
        SweepConfig sc;
        sc.base = make_rc(cells[0]);
        sc.base.mix = static_cast<TraceMix>(mix);
        for (int c = 0; c < n_cells; ++c) sc.cells.push_back({make_rc(cells[c]).policy, std::string()});
        sc.seeds.assign(seeds, seeds + n_seeds);
        SweepResult r = run_sweep(sc);
        if (r.csv.size() + 1 > cap) throw CarmaError("csv buffer too small");
        std::memcpy(csv, r.csv.c_str(), r.csv.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
