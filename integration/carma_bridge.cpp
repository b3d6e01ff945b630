// Reference-side bridge (see carma_bridge.hpp). Compiled against the
// reference's headers and linked with the unmodified reference library and
// libcarma_b200.so (integration/Makefile).

#include "carma_bridge.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numeric>
#include <set>
#include <sstream>

#include <unistd.h>

#include "carma/errors.hpp"
#include "carma/world.hpp"

namespace carma::b200 {

void gpu_check(carma_status s) {
    switch (s) {
        case CARMA_OK: return;
        case CARMA_ERR_FAMILY: throw FamilyMismatch(carma_last_error());
        case CARMA_ERR_INCOMPLETE: throw IncompleteRun(carma_last_error());
        case CARMA_ERR_INVALID: throw ConfigError(carma_last_error());
        default: throw CarmaError(carma_last_error());  // CUDA / OVERFLOW / UNSUPPORTED
    }
}

carma_feature_row to_row(const FeatureVector& fv) {
    carma_feature_row r{};
    r.n_linear = fv.n_linear;
    r.n_batchnorm = fv.n_batchnorm;
    r.n_dropout = fv.n_dropout;
    r.n_conv = fv.n_conv;
    r.batch_size = fv.batch_size;
    r.total_params = fv.total_params;
    r.total_activations = fv.total_activations;
    r.act_cos = fv.act_cos;
    r.act_sin = fv.act_sin;
    r.has_layers = fv.layer_tuples.empty() ? 0 : 1;
    if (r.has_layers) {
        const LayerTuple* pick[3] = {&fv.layer_tuples.front(), &fv.layer_tuples[fv.layer_tuples.size() / 2],
                                     &fv.layer_tuples.back()};
        for (int k = 0; k < 3; ++k) {
            r.kind[k] = pick[k]->kind_code;
            r.tuple_acts[k] = pick[k]->activation_count;
            r.tuple_params[k] = pick[k]->param_count;
        }
    }
    return r;
}

carma_replay_config to_config(const PolicyConfig& policy, const SimConstants& consts,
                              const std::vector<double>& mig_instances) {
    carma_replay_config c{};
    c.policy = static_cast<int32_t>(policy.policy);
    c.mode = static_cast<int32_t>(policy.collocation_mode);
    c.gpu_count = consts.gpu_count;
    c.rr_apply_preconditions = policy.rr_apply_preconditions ? 1 : 0;
    c.max_smact = policy.preconditions.max_smact;
    c.min_free = policy.preconditions.min_free_mem.value_or(0);
    c.monitor_window = policy.monitor_window;
    c.gpu_capacity = consts.gpu_capacity;
    c.alloc_block = consts.alloc_block;
    c.p_idle_w = consts.p_idle_w;
    c.p_max_w = consts.p_max_w;
    c.p_boost_w = consts.p_boost_w;
    c.boost_threshold = consts.boost_threshold;
    c.oom_startup_delay = consts.oom_startup_delay;
    if (policy.collocation_mode == CollocationMode::mig)
        gpu_check(carma_mig_layout(mig_instances.empty() ? nullptr : mig_instances.data(),
                                   static_cast<uint32_t>(mig_instances.size()), &c));
    return c;
}

// ------------------------------------------------------------ estimator bank

GpuEstimatorBank::GpuEstimatorBank(int device) { gpu_check(carma_knn_create(device, &h_)); }

GpuEstimatorBank::~GpuEstimatorBank() {
    if (h_) carma_knn_destroy(h_);
}

void GpuEstimatorBank::add(const LearnedEstimator& est) {
    // The reference keeps the fitted state private; its own snapshot is the
    // public way out (no edit of LearnedEstimator needed).
    char tmpl[] = "/tmp/carma_bridge_snapshot_XXXXXX";
    const int fd = mkstemp(tmpl);
    if (fd < 0) throw CarmaError("cannot create a snapshot file");
    close(fd);
    const std::string path = tmpl;
    try {
        est.save(path);
        load(path);
    } catch (...) {
        std::remove(path.c_str());
        throw;
    }
    std::remove(path.c_str());
}

void GpuEstimatorBank::load(const std::string& snapshot_path) {
    int32_t fam = -1;
    gpu_check(carma_knn_load_snapshot_file(h_, snapshot_path.c_str(), &fam, nullptr));
    const LearnedEstimator est = LearnedEstimator::load(snapshot_path);  // bucket range for estimate()
    families_[static_cast<ModelFamily>(fam)] = est.bucket_range();
}

HoldoutReport GpuEstimatorBank::train(const EstimatorDataset& ds, std::size_t k) {
    if (ds.rows.empty()) throw EmptyDataset("dataset has no rows");
    if (k < 1) throw ConfigError("k must be >= 1");
    std::vector<carma_feature_row> rows(ds.rows.size());
    std::vector<int32_t> bucket(ds.rows.size());
    std::vector<uint64_t> mem(ds.rows.size());
    for (std::size_t i = 0; i < rows.size(); ++i) {
        rows[i] = to_row(ds.rows[i].features);
        bucket[i] = ds.rows[i].bucket;
        mem[i] = ds.rows[i].mem_bytes;
    }
    carma_holdout_report rep{};
    gpu_check(carma_knn_train(h_, static_cast<int32_t>(ds.family), rows.data(), bucket.data(), mem.data(),
                              rows.size(), ds.seed, static_cast<uint32_t>(k), ds.bucket_range, &rep, nullptr,
                              nullptr, nullptr, nullptr));
    families_[ds.family] = ds.bucket_range;
    HoldoutReport out;
    out.accuracy = rep.accuracy;
    out.macro_f1 = rep.macro_f1;
    out.underestimate_rate = rep.underestimate_rate;
    out.train_size = rep.train_size;
    out.holdout_size = rep.holdout_size;
    return out;
}

std::vector<std::optional<MemoryEstimate>> GpuEstimatorBank::estimate(const std::vector<FeatureVector>& features,
                                                                      ModelFamily family) const {
    std::vector<carma_feature_row> rows(features.size());
    for (std::size_t i = 0; i < features.size(); ++i) rows[i] = to_row(features[i]);
    std::vector<int32_t> bucket(features.size());
    std::vector<uint64_t> bytes(features.size());
    std::vector<std::optional<MemoryEstimate>> out(features.size());
    if (features.empty()) return out;
    gpu_check(carma_knn_predict(h_, rows.data(), nullptr, static_cast<int32_t>(family), rows.size(), bucket.data(),
                                bytes.data()));
    for (std::size_t i = 0; i < features.size(); ++i) {
        if (bucket[i] < 0) continue;
        MemoryEstimate m;
        m.bucket = bucket[i];
        m.bucket_range = families_.at(family);
        m.bytes = bytes[i];
        m.source = EstimateSource::learned;
        out[i] = m;
    }
    return out;
}

std::optional<MemoryEstimate> GpuEstimatorBank::estimate(const TaskSpec& task) const {
    return estimate(std::vector<TaskSpec>{task}).front();
}

std::vector<std::optional<MemoryEstimate>> GpuEstimatorBank::estimate(const std::vector<TaskSpec>& tasks) const {
    std::vector<std::optional<MemoryEstimate>> out(tasks.size());
    if (tasks.empty()) return out;
    std::vector<carma_feature_row> rows(tasks.size());
    std::vector<int8_t> fam(tasks.size());
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        rows[i] = to_row(extract_features(tasks[i].model, tasks[i].batch_size));
        fam[i] = static_cast<int8_t>(tasks[i].model.family);
    }
    std::vector<int32_t> bucket(tasks.size());
    std::vector<uint64_t> bytes(tasks.size());
    gpu_check(carma_knn_predict(h_, rows.data(), fam.data(), 0, rows.size(), bucket.data(), bytes.data()));
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        if (bucket[i] < 0) continue;  // FamilyMismatch -> no estimate (manager.cpp:99-105)
        MemoryEstimate m;
        m.bucket = bucket[i];
        m.bucket_range = families_.at(tasks[i].model.family);
        m.bytes = bytes[i];
        m.source = EstimateSource::learned;
        out[i] = m;
    }
    return out;
}

void provision_bank(GpuEstimatorBank& bank, const RunConfig& config, const std::vector<TaskSpec>& tasks) {
    std::set<ModelFamily> families;
    for (const auto& t : tasks) families.insert(t.model.family);
    for (ModelFamily family : families) {
        if (bank.has(family)) continue;
        auto snap = config.estimator_snapshots.find(family);
        if (snap != config.estimator_snapshots.end()) {
            bank.load(snap->second);
            continue;
        }
        const std::uint64_t seed = config.estimator_seed + static_cast<std::uint64_t>(family) * 101;
        bank.train(generate_synthetic_dataset(family, config.estimator_samples, seed), config.estimator_k);
    }
}

// ------------------------------------------------------------------ runner

namespace {

struct Trace {
    std::vector<TaskSpec> tasks;
    std::string name;
    std::vector<uint32_t> rank;  // rank of each task id in std::string order
};

Trace load_run_trace(const RunConfig& config) {
    Trace tr;
    if (config.mix) {
        tr.tasks = materialize_trace(generate_trace(*config.mix, config.trace_seed));
        tr.name = std::string(mix_name(*config.mix)) + "-seed" + std::to_string(config.trace_seed);
    } else {
        if (config.trace_path.empty()) throw ConfigError("run needs either a trace path or a mix+seed");
        tr.tasks = load_trace(config.trace_path);
        tr.name = config.trace_path;
    }
    if (tr.tasks.empty()) throw ConfigError("trace contains no tasks");
    std::vector<uint32_t> order(tr.tasks.size());
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return tr.tasks[a].id < tr.tasks[b].id; });
    tr.rank.assign(tr.tasks.size(), 0);
    for (uint32_t r = 0; r < order.size(); ++r) {
        if (r > 0 && tr.tasks[order[r]].id == tr.tasks[order[r - 1]].id)
            throw DuplicateTaskId("trace repeats task id '" + tr.tasks[order[r]].id + "'");
        tr.rank[order[r]] = r;
    }
    return tr;
}

// Manager::make_estimate for every task of `tr` under `config` (learned from
// the bank, the personas from the reference's own formulas).
std::vector<uint64_t> estimates_for(const RunConfig& config, const Trace& tr, GpuEstimatorBank* bank) {
    std::vector<uint64_t> est(tr.tasks.size(), CARMA_NO_ESTIMATE);
    if (config.policy.estimator == EstimatorKind::learned) {
        const auto e = bank->estimate(tr.tasks);
        for (std::size_t i = 0; i < e.size(); ++i)
            if (e[i]) est[i] = e[i]->bytes;
        return est;
    }
    World world(config.constants, config.policy.collocation_mode, config.mig_instances);
    Manager manager(world, config.policy);
    for (std::size_t i = 0; i < tr.tasks.size(); ++i) {
        const auto e = manager.make_estimate(tr.tasks[i]);
        if (e) est[i] = e->bytes;
    }
    return est;
}

void append_tasks(const Trace& tr, const std::vector<uint64_t>& est, std::vector<carma_task>& out) {
    for (std::size_t i = 0; i < tr.tasks.size(); ++i) {
        const TaskSpec& t = tr.tasks[i];
        carma_task g{};
        g.submit = t.submit_time;
        g.work = t.total_work();
        g.demand = t.smact_demand;
        g.true_mem = t.true_mem_bytes;
        g.estimate = est[i];
        g.gpus = static_cast<uint32_t>(t.gpus_requested);
        g.rank = tr.rank[i];
        out.push_back(g);
    }
}

// compute_report (metrics.cpp:16-70) from one job's device results: the
// scalars are the kernel's (summed in the reference's id order), the per-task
// outcomes and per-GPU summaries are assembled the way compute_report does.
RunReport report_of(const RunConfig& config, const Trace& tr, const carma_task_result* tres,
                    const carma_trace_result& rep, const carma_gpu_result* gres) {
    if (rep.status == CARMA_ERR_INCOMPLETE) {
        int pending = 0;
        for (std::size_t i = 0; i < tr.tasks.size(); ++i)
            if (tres[i].complete < 0.0) ++pending;
        throw IncompleteRun(std::to_string(pending) +
                            " task(s) never completed; the platform cannot host them under this config");
    }
    gpu_check(static_cast<carma_status>(rep.status));
    RunReport r;
    r.config = config.policy;
    r.seed = config.trace_seed;
    r.trace_name = tr.name;
    r.oom_count = rep.oom_count;
    for (std::size_t i = 0; i < tr.tasks.size(); ++i) {
        TaskOutcome o;
        o.id = tr.tasks[i].id;
        o.submit = tr.tasks[i].submit_time;
        o.final_dispatch = tres[i].final_dispatch;
        o.complete = tres[i].complete;
        o.wait = o.final_dispatch - o.submit;
        o.exec = o.complete - o.final_dispatch;
        o.jct = o.complete - o.submit;
        o.ooms = static_cast<int>(tres[i].ooms);
        r.tasks.push_back(std::move(o));
    }
    std::sort(r.tasks.begin(), r.tasks.end(), [](const TaskOutcome& a, const TaskOutcome& b) {
        if (a.submit != b.submit) return a.submit < b.submit;
        return a.id < b.id;
    });
    r.avg_wait = rep.avg_wait;
    r.avg_exec = rep.avg_exec;
    r.avg_jct = rep.avg_jct;
    r.trace_total_time = rep.trace_total_time;
    r.energy_mj = rep.energy_mj;
    for (int g = 0; g < config.constants.gpu_count; ++g) {
        GpuSummary s;
        s.id = g;
        s.energy_j = gres[g].energy_j;
        s.mean_smact = gres[g].mean_smact;
        s.peak_mem = gres[g].peak_used;
        r.per_gpu.push_back(s);
    }
    return r;
}

// runner.cpp's csv_row (anonymous there): the sweep table's line format.
std::string csv_row(const RunReport& rep, const std::string& seed_field) {
    char buf[512];
    const auto& c = rep.config;
    char min_free[32];
    if (c.preconditions.min_free_mem)
        std::snprintf(min_free, sizeof(min_free), "%.2f", as_gib(*c.preconditions.min_free_mem));
    else
        std::snprintf(min_free, sizeof(min_free), "none");
    std::snprintf(buf, sizeof(buf), "%s,%s,%s,%.2f,%s,%.0f,%s,%s,%.3f,%.3f,%.3f,%.3f,%d,%.2f",
                  std::string(policy_name(c.policy)).c_str(), std::string(estimator_kind_name(c.estimator)).c_str(),
                  std::string(mode_name(c.collocation_mode)).c_str(), c.preconditions.max_smact, min_free,
                  c.monitor_window, seed_field.c_str(), rep.trace_name.c_str(), rep.trace_total_time, rep.avg_wait,
                  rep.avg_exec, rep.avg_jct, rep.oom_count, rep.energy_mj);
    return buf;
}

}  // namespace

RunReport gpu_run_simulation(const RunConfig& config, int device, GpuEstimatorBank* bank) {
    const Trace tr = load_run_trace(config);
    std::optional<GpuEstimatorBank> own;
    if (config.policy.estimator == EstimatorKind::learned) {
        if (!bank) bank = &own.emplace(device);
        provision_bank(*bank, config, tr.tasks);
    }
    std::vector<carma_task> tasks;
    append_tasks(tr, estimates_for(config, tr, bank), tasks);
    const carma_replay_config cfg = to_config(config.policy, config.constants, config.mig_instances);
    const uint64_t offs[2] = {0, tasks.size()};
    const carma_replay_job job{0, 0};
    std::vector<carma_task_result> tres(tasks.size());
    carma_trace_result rep{};
    std::vector<carma_gpu_result> gres(static_cast<std::size_t>(config.constants.gpu_count));
    gpu_check(carma_replay_batch(device, &cfg, 1, tasks.data(), offs, 1, &job, 1, tres.data(), &rep, gres.data()));
    return report_of(config, tr, tres.data(), rep, gres.data());
}

SweepResult gpu_run_sweep(const SweepConfig& config, int device) {
    if (config.cells.empty()) throw ConfigError("sweep has no cells");
    if (config.seeds.empty()) throw ConfigError("sweep has no seeds");
    const std::size_t nc = config.cells.size(), ns = config.seeds.size();

    // One materialised trace per seed; the learned bank is the same for every
    // run (provision_estimators depends on the config's estimator settings
    // and the trace's families only), so it is provisioned once.
    std::vector<Trace> traces;
    traces.reserve(ns);
    for (std::size_t s = 0; s < ns; ++s) {
        RunConfig rc = config.base;
        rc.trace_seed = config.seeds[s];
        traces.push_back(load_run_trace(rc));
    }
    std::optional<GpuEstimatorBank> bank;
    for (const auto& cell : config.cells)
        if (cell.policy.estimator == EstimatorKind::learned && !bank) {
            bank.emplace(device);
            std::vector<TaskSpec> all;
            for (const auto& t : traces) all.insert(all.end(), t.tasks.begin(), t.tasks.end());
            provision_bank(*bank, config.base, all);
        }

    // Job (cell c, seed s) = trace c * ns + s: the cell's estimates over seed s.
    std::vector<carma_replay_config> cfgs;
    std::vector<carma_task> tasks;
    std::vector<uint64_t> offs{0};
    std::vector<carma_replay_job> jobs;
    std::vector<std::size_t> task_base, gpu_base;
    std::size_t n_gpu_rows = 0;
    for (std::size_t c = 0; c < nc; ++c) {
        RunConfig rc = config.base;
        rc.policy = config.cells[c].policy;
        cfgs.push_back(to_config(rc.policy, rc.constants, rc.mig_instances));
        for (std::size_t s = 0; s < ns; ++s) {
            rc.trace_seed = config.seeds[s];
            task_base.push_back(tasks.size());
            append_tasks(traces[s], estimates_for(rc, traces[s], bank ? &*bank : nullptr), tasks);
            offs.push_back(tasks.size());
            jobs.push_back({static_cast<uint32_t>(c * ns + s), static_cast<uint32_t>(c)});
            gpu_base.push_back(n_gpu_rows);
            n_gpu_rows += static_cast<std::size_t>(rc.constants.gpu_count);
        }
    }
    std::vector<carma_task_result> tres(tasks.size());
    std::vector<carma_trace_result> reps(jobs.size());
    std::vector<carma_gpu_result> gres(n_gpu_rows);
    gpu_check(carma_replay_batch(device, cfgs.data(), static_cast<uint32_t>(cfgs.size()), tasks.data(), offs.data(),
                                 static_cast<uint32_t>(offs.size() - 1), jobs.data(),
                                 static_cast<uint32_t>(jobs.size()), tres.data(), reps.data(), gres.data()));

    SweepResult result;
    result.reports.assign(nc, std::vector<RunReport>(ns));
    for (std::size_t c = 0; c < nc; ++c)
        for (std::size_t s = 0; s < ns; ++s) {
            const std::size_t j = c * ns + s;
            RunConfig rc = config.base;
            rc.policy = config.cells[c].policy;
            rc.trace_seed = config.seeds[s];
            try {
                result.reports[c][s] = report_of(rc, traces[s], tres.data() + task_base[j], reps[j],
                                                 gres.data() + gpu_base[j]);
            } catch (const std::exception& e) {
                const std::string label = config.cells[c].label.empty()
                                              ? std::string(policy_name(config.cells[c].policy.policy))
                                              : config.cells[c].label;
                throw CarmaError("sweep cell '" + label + "' seed " + std::to_string(config.seeds[s]) +
                                 " failed: " + e.what());
            }
        }

    std::ostringstream csv;
    csv << report_csv_header() << "\n";
    for (std::size_t c = 0; c < nc; ++c) {
        for (std::size_t s = 0; s < ns; ++s) csv << csv_row(result.reports[c][s], std::to_string(config.seeds[s])) << "\n";
        if (ns > 1) {
            RunReport med = result.reports[c][0];
            std::vector<double> total, wait, exec, jct, oom, energy;
            for (const auto& r : result.reports[c]) {
                total.push_back(r.trace_total_time);
                wait.push_back(r.avg_wait);
                exec.push_back(r.avg_exec);
                jct.push_back(r.avg_jct);
                oom.push_back(r.oom_count);
                energy.push_back(r.energy_mj);
            }
            med.trace_total_time = median(total);
            med.avg_wait = median(wait);
            med.avg_exec = median(exec);
            med.avg_jct = median(jct);
            med.oom_count = static_cast<int>(std::llround(median(oom)));
            med.energy_mj = median(energy);
            csv << csv_row(med, "median") << "\n";
        }
    }
    result.csv = csv.str();
    return result;
}

}  // namespace carma::b200
