// Host-side domain model of the CARMA hot path (B200 build).
//
// Value types and the input-provisioning side of the path: seeded RNG,
// the Table-5 catalog, trace generation / file I/O / materialisation,
// synthetic architecture datasets, featurisation and k-NN fitting. These are
// the callers and data formats on either side of the GPU kernels; the
// kernels themselves sit behind include/carma_gpu.h.
//
// Behavioural contract (reference file:line):
//   Rng                 proj/include/carma/rng.hpp:13-56
//   SimConstants        proj/include/carma/memory_model.hpp:11-29
//   catalog / traces    proj/src/traces.cpp:37-379
//   datasets            proj/src/estimators.cpp:67-264
//   features            proj/src/task.cpp:301-323, estimators.cpp:317-342
//   k-NN fit            proj/src/estimators.cpp:344-436
#pragma once

#include <array>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

namespace carma_b200 {

using Bytes = std::uint64_t;
inline constexpr Bytes kMiB = 1ull << 20;
inline constexpr Bytes kGiB = 1ull << 30;

// units.hpp:15-17 — round-half-up conversion of a GiB count to bytes.
inline constexpr Bytes gib(double v) {
    return static_cast<Bytes>(v * static_cast<double>(kGiB) + 0.5);
}

enum class Family : int { MLP = 0, CNN = 1, Transformer = 2 };
enum class WeightClass : int { light = 0, medium = 1, heavy = 2 };
// Layer kind codes are the enum ordinals of task.hpp:14-22.
enum class LayerKind : int { linear = 0, conv1d, conv2d, batchnorm, dropout, attention, embedding };

const char* family_name(Family f);
Bytes default_bucket_range(Family f);  // 1 GiB for MLP, 8 GiB otherwise

// mt19937_64 with the toolchain-stable samplers of rng.hpp.
class Rng {
  public:
    explicit Rng(std::uint64_t seed) : mt_(seed) {}
    std::uint64_t next_u64() { return mt_(); }
    double next_double() { return static_cast<double>(mt_() >> 11) * 0x1.0p-53; }
    std::uint64_t uniform(std::uint64_t n) {
        return static_cast<std::uint64_t>((static_cast<unsigned __int128>(mt_()) * n) >> 64);
    }
    std::int64_t uniform_int(std::int64_t lo, std::int64_t hi) {
        return lo + static_cast<std::int64_t>(uniform(static_cast<std::uint64_t>(hi - lo + 1)));
    }
    double exponential(double mean);
    template <typename T>
    void shuffle(std::vector<T>& v) {
        for (std::size_t i = v.size(); i > 1; --i) {
            std::size_t j = static_cast<std::size_t>(uniform(i));
            std::swap(v[i - 1], v[j]);
        }
    }

  private:
    std::mt19937_64 mt_;
};

struct SimConstants {
    Bytes gpu_capacity = 40 * kGiB;
    int gpu_count = 4;
    Bytes alloc_block = 512 * kMiB;
    Bytes framework_base = gib(0.75);
    std::uint64_t bytes_per_value = 4;
    std::uint64_t param_copies = 4;
    double p_idle_w = 55.0;
    double p_max_w = 400.0;
    double p_boost_w = 30.0;
    double boost_threshold = 0.9;
    double oom_startup_delay = 5.0;
};

struct Layer {
    LayerKind kind;
    std::uint64_t params;
    std::uint64_t acts;
};

struct Architecture {
    Family family = Family::MLP;
    std::vector<Layer> layers;
    double activation_angle = 0.0;
    std::uint64_t total_params() const;
    std::uint64_t total_activations() const;
};

// Activation registry angle (task.cpp:181-189): 2*pi*i/8.
double activation_angle(int registry_index);
int activation_index(const char* name);  // -1 when unknown

// The FeatureVector summary a k-NN query consumes: seven tallies, the
// activation (cos, sin) and the first / middle / last layer tuples.
struct FeatureRow {
    std::uint64_t n_linear = 0, n_batchnorm = 0, n_dropout = 0, n_conv = 0;
    std::uint64_t batch = 0, params = 0, acts = 0;
    double act_cos = 1.0, act_sin = 0.0;
    std::int32_t kind[3] = {0, 0, 0};
    std::uint64_t tuple_acts[3] = {0, 0, 0};
    std::uint64_t tuple_params[3] = {0, 0, 0};
    bool has_layers = false;
};

FeatureRow extract_features(const Architecture& a, std::uint64_t batch);
constexpr int kFeatureDims = 19;
using ScalarRow = std::array<double, kFeatureDims>;
ScalarRow scalar_features(const FeatureRow& f);

// ground_truth_memory (memory_model.cpp:5-13).
Bytes ground_truth_memory(const Architecture& a, std::uint64_t batch,
                          const SimConstants& c = SimConstants{});

// ---------------------------------------------------------------- catalog
struct CatalogEntry {
    std::string key;
    std::string model;
    std::string dataset;
    Family family;
    std::uint64_t batch;
    std::uint64_t gpus;
    double epoch_minutes;
    std::vector<std::uint64_t> epoch_options;
    double mem_gib;
    WeightClass wclass;
    double demand;
};

const std::vector<CatalogEntry>& catalog();
int catalog_index(const std::string& key);  // -1 when unknown
Architecture catalog_architecture(const CatalogEntry& e);

// ----------------------------------------------------------------- traces
enum class Mix : int { t90 = 0, t60 = 1 };

struct TraceRow {
    double submit;
    std::int32_t entry;  // catalog index
    std::uint64_t epochs;
};

struct Trace {
    std::uint64_t seed = 0;
    std::string mix;
    std::vector<TraceRow> rows;
};

Trace generate_trace(Mix mix, std::uint64_t seed);
// Like generate_trace, but with every catalog row eligible and a chosen mean
// gap: the large single-trace workload.
Trace generate_uniform_trace(std::size_t n, double mean_gap, std::uint64_t seed);
void save_trace(const Trace& t, const std::string& path);
Trace load_trace(const std::string& path);  // throws std::runtime_error

// A materialised task (task_from_catalog, traces.cpp:238-254) in the form the
// replay consumes, plus its id and family for estimator routing.
struct Task {
    std::string id;
    double submit;
    Bytes true_mem;
    double work;
    double demand;
    std::uint32_t gpus;
    Family family;
    std::uint64_t batch;
    std::int32_t entry;
};

std::vector<Task> materialize(const Trace& t);

// --------------------------------------------------------------- datasets
struct Bounds {
    std::uint64_t min_layers = 1, max_layers = 10;
    std::uint64_t min_width = 64, max_width = 6144;
    std::uint64_t min_batch = 8, max_batch = 512;
    std::uint64_t min_input = 64, max_input = 4096;
    std::uint64_t min_output = 10, max_output = 1024;
    static Bounds for_family(Family f);
};

struct Dataset {
    Family family = Family::MLP;
    Bytes bucket_range = kGiB;
    std::uint64_t seed = 0;
    std::vector<FeatureRow> rows;
    std::vector<std::int32_t> bucket;
    std::vector<Bytes> mem;
};

Dataset generate_dataset(Family f, std::size_t n, std::uint64_t seed);

// k-NN model as fitted by train_learned_estimator (estimators.cpp:344-395):
// min-max bounds and the normalised training rows, in training order.
struct KnnModel {
    Family family = Family::MLP;
    Bytes bucket_range = kGiB;
    std::uint32_t k = 5;
    std::uint64_t seed = 0;
    ScalarRow lo{}, hi{};
    std::vector<double> points;  // n x 19, row-major, normalised
    std::vector<std::int32_t> labels;
    std::vector<std::size_t> holdout_rows;  // dataset rows held out, in order
    std::size_t size() const { return labels.size(); }
};

KnnModel fit_knn(const Dataset& ds, std::uint32_t k);

}  // namespace carma_b200
