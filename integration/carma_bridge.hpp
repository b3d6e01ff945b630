// Reference-side bridge: the code a maintainer of the reference adds to
// serve its estimator / simulator API from libcarma_b200.so. It is written
// against the reference's own public headers (proj/include/carma/*.hpp) and
// links the unmodified reference library; nothing here is product code of
// this repository (the product is the C ABI in include/carma_gpu.h).
//
//   GpuEstimatorBank   Manager::set_learned_estimators + estimate_learned
//                      (manager.hpp:77, manager.cpp:80-107,
//                      estimators.cpp:540-551) over a device-resident bank
//   gpu_run_simulation run_simulation(...).report (runner.hpp:49,
//                      runner.cpp:40-147): same RunReport, every field
//   gpu_run_sweep      run_sweep (runner.hpp:72, runner.cpp:192-283): same
//                      reports and the same CSV text
//
// Errors map onto the reference's exception types (errors.hpp:12-57).
#pragma once

#include <map>
#include <optional>
#include <string>
#include <vector>

#include "carma/estimators.hpp"
#include "carma/manager.hpp"
#include "carma/metrics.hpp"
#include "carma/runner.hpp"
#include "carma/traces.hpp"
#include "carma_gpu.h"
#include "carma_host.h"

namespace carma::b200 {

// carma_status -> the reference's exceptions.
void gpu_check(carma_status s);

// FeatureVector -> the C ABI's 136-B row (the fields scalar_features reads,
// estimators.cpp:317-342: the tallies and the front / middle / back tuples).
carma_feature_row to_row(const FeatureVector& fv);

// PolicyConfig + SimConstants (+ RunConfig::mig_instances) -> carma_replay_config.
carma_replay_config to_config(const PolicyConfig& policy, const SimConstants& consts,
                              const std::vector<double>& mig_instances);

class GpuEstimatorBank {
  public:
    explicit GpuEstimatorBank(int device = 0);
    ~GpuEstimatorBank();
    GpuEstimatorBank(const GpuEstimatorBank&) = delete;
    GpuEstimatorBank& operator=(const GpuEstimatorBank&) = delete;

    // An already fitted estimator, read through its own snapshot
    // (LearnedEstimator::save, estimators.cpp:481-501).
    void add(const LearnedEstimator& est);
    // LearnedEstimator::load of a snapshot file straight into the bank.
    void load(const std::string& snapshot_path);
    // train_learned_estimator(dataset, k) on the device (carma_knn_train).
    HoldoutReport train(const EstimatorDataset& dataset, std::size_t k);
    bool has(ModelFamily family) const { return families_.count(family) != 0; }
    carma_knn* handle() const { return h_; }

    // Manager::make_estimate for EstimatorKind::learned: std::nullopt where
    // the bank has no model for the task's family (FamilyMismatch,
    // manager.cpp:99-105).
    std::optional<MemoryEstimate> estimate(const TaskSpec& task) const;
    // The same for many tasks in one batched device call.
    std::vector<std::optional<MemoryEstimate>> estimate(const std::vector<TaskSpec>& tasks) const;
    // estimate_learned(est_of(family), fv, family) for many feature vectors.
    std::vector<std::optional<MemoryEstimate>> estimate(const std::vector<FeatureVector>& features,
                                                        ModelFamily family) const;

  private:
    carma_knn* h_ = nullptr;
    std::map<ModelFamily, Bytes> families_;  // family -> bucket range
};

// provision_estimators (runner.cpp:17-38) into a GPU bank: snapshots when
// given, otherwise seeded synthetic datasets trained on the device.
void provision_bank(GpuEstimatorBank& bank, const RunConfig& config, const std::vector<TaskSpec>& tasks);

// run_simulation(config).report with the estimator and the replay on the GPU.
// `bank` (optional) serves EstimatorKind::learned; without one a bank is
// provisioned for the call.
RunReport gpu_run_simulation(const RunConfig& config, int device = 0, GpuEstimatorBank* bank = nullptr);

// run_sweep on the GPU: every (cell, seed) run is one job of one replay call.
SweepResult gpu_run_sweep(const SweepConfig& config, int device = 0);

}  // namespace carma::b200
