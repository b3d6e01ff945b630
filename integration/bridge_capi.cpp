// Test entry points of the bridge (ctypes, tests/test_gpu_bridge.py): each
// runs the UNMODIFIED reference and the bridge on the same inputs and hands
// both results back as text (emit_report JSON, sweep CSV) or arrays, so the
// test compares them byte for byte. Failures come back as
// "ERR:<message>" in the same buffers (the error behaviour is compared too).

#include <cstring>
#include <string>
#include <vector>

#include "carma/errors.hpp"
#include "carma_bridge.hpp"

using namespace carma;
using namespace carma::b200;

namespace {

struct BridgeCase {
    int32_t mix;  // 0 t90, 1 t60, -1 trace_path
    int32_t policy;
    int32_t estimator;
    int32_t mode;
    uint64_t seed;
    int32_t gpu_count;
    int32_t rr_pre;
    int32_t has_min_free;
    int32_t n_mig;
    double max_smact;
    double window;
    uint64_t min_free;
    uint64_t capacity;
    uint64_t block;
    double mig[8];
};

RunConfig run_config(const BridgeCase& c, const char* trace_path) {
    RunConfig rc;
    if (c.mix >= 0)
        rc.mix = c.mix == 0 ? TraceMix::t90 : TraceMix::t60;
    else
        rc.trace_path = trace_path ? trace_path : "";
    rc.trace_seed = c.seed;
    rc.policy.policy = static_cast<Policy>(c.policy);
    rc.policy.estimator = static_cast<EstimatorKind>(c.estimator);
    rc.policy.collocation_mode = static_cast<CollocationMode>(c.mode);
    rc.policy.preconditions.max_smact = c.max_smact;
    if (c.has_min_free) rc.policy.preconditions.min_free_mem = c.min_free;
    rc.policy.monitor_window = c.window;
    rc.policy.rr_apply_preconditions = c.rr_pre != 0;
    rc.constants.gpu_count = c.gpu_count;
    rc.constants.gpu_capacity = c.capacity;
    rc.constants.alloc_block = c.block;
    for (int i = 0; i < c.n_mig; ++i) rc.mig_instances.push_back(c.mig[i]);
    return rc;
}

void put(const std::string& s, char* buf, uint64_t cap) {
    if (!buf || cap == 0) return;
    const uint64_t n = std::min<uint64_t>(s.size(), cap - 1);
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
}

template <typename F>
std::string capture(F&& f) {
    try {
        return "OK:" + f();
    } catch (const std::exception& e) {
        return std::string("ERR:") + e.what();
    }
}

}  // namespace

extern "C" {

// run_simulation(rc).report vs gpu_run_simulation(rc), both as emit_report JSON.
int bridge_run_pair(const BridgeCase* c, const char* trace_path, int device, char* ref_out, uint64_t ref_cap,
                    char* gpu_out, uint64_t gpu_cap) {
    const RunConfig rc = run_config(*c, trace_path);
    const std::string r = capture([&] { return emit_report(run_simulation(rc).report, ReportFormat::json); });
    const std::string g = capture([&] { return emit_report(gpu_run_simulation(rc, device), ReportFormat::json); });
    put(r, ref_out, ref_cap);
    put(g, gpu_out, gpu_cap);
    return static_cast<int>(std::max(r.size(), g.size()) + 1);
}

// run_sweep vs gpu_run_sweep over cells (policy part of each case; the base
// run config is cells[0]'s) x seeds: the CSV text plus every report's JSON.
int bridge_sweep_pair(const BridgeCase* cells, int n_cells, const uint64_t* seeds, int n_seeds, int device,
                      char* ref_out, uint64_t ref_cap, char* gpu_out, uint64_t gpu_cap) {
    SweepConfig sc;
    sc.base = run_config(cells[0], nullptr);
    for (int i = 0; i < n_cells; ++i) sc.cells.push_back({run_config(cells[i], nullptr).policy, ""});
    sc.seeds.assign(seeds, seeds + n_seeds);
    auto text = [&](const SweepResult& res) {
        std::string s = res.csv;
        for (const auto& row : res.reports)
            for (const auto& rep : row) s += emit_report(rep, ReportFormat::json) + "\n";
        return s;
    };
    const std::string r = capture([&] { return text(run_sweep(sc)); });
    const std::string g = capture([&] { return text(gpu_run_sweep(sc, device)); });
    put(r, ref_out, ref_cap);
    put(g, gpu_out, gpu_cap);
    return static_cast<int>(std::max(r.size(), g.size()) + 1);
}

// estimate_learned over generate_synthetic_dataset(family, n, qseed) with the
// model train_learned_estimator fits on (family, samples, est_seed, k),
// served three ways: how = 0 GpuEstimatorBank::add(LearnedEstimator),
// 1 GpuEstimatorBank::train on the device, 2 GpuEstimatorBank::load(snapshot).
int bridge_estimate_pair(int family, uint64_t n, uint64_t qseed, uint64_t samples, uint64_t est_seed, uint64_t k,
                         int how, int device, int32_t* ref_bucket, uint64_t* ref_bytes, int32_t* gpu_bucket,
                         uint64_t* gpu_bytes, char* err, uint64_t err_cap) {
    try {
        const auto fam = static_cast<ModelFamily>(family);
        const EstimatorDataset train = generate_synthetic_dataset(fam, samples, est_seed);
        const LearnedEstimator est = train_learned_estimator(train, k);
        const EstimatorDataset q = generate_synthetic_dataset(fam, n, qseed);
        std::vector<FeatureVector> fv;
        for (std::size_t i = 0; i < q.rows.size(); ++i) {
            const MemoryEstimate m = estimate_learned(est, q.rows[i].features, fam);
            ref_bucket[i] = *m.bucket;
            ref_bytes[i] = m.bytes;
            fv.push_back(q.rows[i].features);
        }
        GpuEstimatorBank bank(device);
        if (how == 0) {
            bank.add(est);
        } else if (how == 1) {
            const HoldoutReport h = bank.train(train, k);
            if (h.accuracy != est.holdout().accuracy || h.macro_f1 != est.holdout().macro_f1 ||
                h.underestimate_rate != est.holdout().underestimate_rate ||
                h.train_size != est.holdout().train_size || h.holdout_size != est.holdout().holdout_size)
                throw CarmaError("device holdout report differs from the reference's");
        } else {
            const std::string path = "/tmp/carma_bridge_test_snapshot.json";
            est.save(path);
            bank.load(path);
        }
        const auto g = bank.estimate(fv, fam);
        for (std::size_t i = 0; i < g.size(); ++i) {
            if (!g[i] || g[i]->bucket_range != est.bucket_range() || g[i]->source != EstimateSource::learned)
                throw CarmaError("missing / malformed estimate");
            gpu_bucket[i] = *g[i]->bucket;
            gpu_bytes[i] = g[i]->bytes;
        }
        return 0;
    } catch (const std::exception& e) {
        put(e.what(), err, err_cap);
        return 1;
    }
}

// LearnedEstimator::load of a snapshot written by this repository (the
// Python LearnedEstimator.save), then estimate_learned over
// generate_synthetic_dataset(family, n, qseed): the reference's own buckets.
int bridge_snapshot_predict(const char* path, int family, uint64_t n, uint64_t qseed, int32_t* bucket,
                            char* err, uint64_t err_cap) {
    try {
        const auto fam = static_cast<ModelFamily>(family);
        const LearnedEstimator est = LearnedEstimator::load(path);
        const EstimatorDataset q = generate_synthetic_dataset(fam, n, qseed);
        for (std::size_t i = 0; i < q.rows.size(); ++i) bucket[i] = *estimate_learned(est, q.rows[i].features, fam).bucket;
        return 0;
    } catch (const std::exception& e) {
        put(e.what(), err, err_cap);
        return 1;
    }
}

// Manager::make_estimate (bank of provision_estimators) vs the GPU bank over
// the materialised tasks of generate_trace(mix, seed): -1 / UINT64_MAX for
// "no estimate".
int bridge_manager_estimates(int mix, uint64_t seed, int device, uint64_t* ref_bytes, uint64_t* gpu_bytes,
                             uint64_t cap, uint64_t* n_out, char* err, uint64_t err_cap) {
    try {
        RunConfig rc;
        rc.mix = mix == 0 ? TraceMix::t90 : TraceMix::t60;
        rc.trace_seed = seed;
        rc.policy.estimator = EstimatorKind::learned;
        const std::vector<TaskSpec> tasks = materialize_trace(generate_trace(*rc.mix, seed));
        if (tasks.size() > cap) throw CarmaError("cap too small");
        World world(rc.constants, rc.policy.collocation_mode);
        Manager manager(world, rc.policy);
        manager.set_learned_estimators(provision_estimators(rc, tasks));
        GpuEstimatorBank bank(device);
        provision_bank(bank, rc, tasks);
        const auto g = bank.estimate(tasks);
        for (std::size_t i = 0; i < tasks.size(); ++i) {
            const auto r = manager.make_estimate(tasks[i]);
            ref_bytes[i] = r ? r->bytes : UINT64_MAX;
            gpu_bytes[i] = g[i] ? g[i]->bytes : UINT64_MAX;
        }
        *n_out = tasks.size();
        return 0;
    } catch (const std::exception& e) {
        put(e.what(), err, err_cap);
        return 1;
    }
}

}  // extern "C"
