// Host provisioning for the CARMA hot path. See model.hpp for the contract.
//
// Every floating-point expression below is written in the operation order of
// the reference and this file is compiled with -ffp-contract=off, so the
// produced inputs (traces, datasets, features, k-NN models) are bit-identical
// to the reference's. tests/test_host_parity.py pins that against
// oracle/_ref.

#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <map>
#include <numbers>
#include <sstream>
#include <stdexcept>

namespace carma_b200 {

const char* family_name(Family f) {
    switch (f) {
        case Family::MLP: return "mlp";
        case Family::CNN: return "cnn";
        case Family::Transformer: return "transformer";
    }
    return "unknown";
}

Bytes default_bucket_range(Family f) { return f == Family::MLP ? kGiB : 8 * kGiB; }

// rng.hpp:41-44 (glibc log1p; host only).
double Rng::exponential(double mean) {
    const double u = next_double();
    return -mean * std::log1p(-u);
}

std::uint64_t Architecture::total_params() const {
    std::uint64_t s = 0;
    for (const auto& l : layers) s += l.params;
    return s;
}

std::uint64_t Architecture::total_activations() const {
    std::uint64_t s = 0;
    for (const auto& l : layers) s += l.acts;
    return s;
}

namespace {
constexpr const char* kActivations[8] = {"relu", "gelu",       "tanh", "sigmoid",
                                         "silu", "leaky_relu", "elu",  "none"};
}

double activation_angle(int i) {
    return 2.0 * std::numbers::pi * static_cast<double>(i) / 8.0;
}

int activation_index(const char* name) {
    for (int i = 0; i < 8; ++i)
        if (std::string(kActivations[i]) == name) return i;
    return -1;
}

// task.cpp:301-323
FeatureRow extract_features(const Architecture& a, std::uint64_t batch) {
    FeatureRow f;
    f.batch = batch;
    f.act_cos = std::cos(a.activation_angle);
    f.act_sin = std::sin(a.activation_angle);
    for (const auto& l : a.layers) {
        switch (l.kind) {
            case LayerKind::linear: ++f.n_linear; break;
            case LayerKind::batchnorm: ++f.n_batchnorm; break;
            case LayerKind::dropout: ++f.n_dropout; break;
            case LayerKind::conv1d:
            case LayerKind::conv2d: ++f.n_conv; break;
            default: break;
        }
        f.params += l.params;
        f.acts += l.acts;
    }
    if (!a.layers.empty()) {
        f.has_layers = true;
        const std::size_t pick[3] = {0, a.layers.size() / 2, a.layers.size() - 1};
        for (int k = 0; k < 3; ++k) {
            const Layer& l = a.layers[pick[k]];
            f.kind[k] = static_cast<std::int32_t>(l.kind);
            f.tuple_acts[k] = l.acts;
            f.tuple_params[k] = l.params;
        }
    }
    return f;
}

// estimators.cpp:317-342
ScalarRow scalar_features(const FeatureRow& f) {
    ScalarRow s{};
    s[0] = static_cast<double>(f.n_linear);
    s[1] = static_cast<double>(f.n_batchnorm);
    s[2] = static_cast<double>(f.n_dropout);
    s[3] = static_cast<double>(f.n_conv);
    s[4] = static_cast<double>(f.batch);
    s[5] = static_cast<double>(f.params);
    s[6] = static_cast<double>(f.acts);
    s[7] = f.act_cos;
    s[8] = f.act_sin;
    if (f.has_layers) {
        for (int k = 0; k < 3; ++k) {
            s[9 + 3 * k] = static_cast<double>(f.kind[k]);
            s[10 + 3 * k] = static_cast<double>(f.tuple_acts[k]);
            s[11 + 3 * k] = static_cast<double>(f.tuple_params[k]);
        }
    }
    const double t1 = 16.0 * static_cast<double>(f.params);
    const double t2 = 4.0 * static_cast<double>(f.batch) * static_cast<double>(f.acts);
    s[18] = t1 + t2;
    return s;
}

Bytes ground_truth_memory(const Architecture& a, std::uint64_t batch, const SimConstants& c) {
    const Bytes raw = c.bytes_per_value * c.param_copies * a.total_params() +
                      c.bytes_per_value * batch * a.total_activations();
    const Bytes blocks = (raw + c.alloc_block - 1) / c.alloc_block;
    return c.framework_base + blocks * c.alloc_block;
}

// ---------------------------------------------------------------- catalog
namespace {

struct Row {
    const char* model;
    Family family;
    const char* dataset;
    std::uint64_t batch, gpus;
    double epoch_minutes;
    int epochs;  // 0: the light {20, 50} choice
    double mem_gib;
    double demand;
};

// Table 5 of the paper as encoded by the reference catalog
// (traces.cpp:37-100), in catalog order: WikiText-2 transformers, ImageNet
// CNNs, CIFAR-100 CNNs.
constexpr Row kTable[] = {
    {"xlnet_base", Family::Transformer, "wikitext2", 8, 2, 8.95, 8, 9.72, 0.43},
    {"bert_base", Family::Transformer, "wikitext2", 32, 1, 14.87, 1, 20.77, 0.45},
    {"xlnet_large", Family::Transformer, "wikitext2", 4, 2, 25.31, 3, 14.55, 0.44},
    {"bert_large", Family::Transformer, "wikitext2", 8, 1, 44.93, 1, 13.57, 0.45},
    {"gpt2_large", Family::Transformer, "wikitext2", 8, 2, 64.96, 1, 27.90, 0.46},
    {"efficientnet_b0", Family::CNN, "imagenet", 32, 1, 36.21, 1, 4.96, 0.41},
    {"efficientnet_b0", Family::CNN, "imagenet", 64, 1, 35.41, 1, 7.84, 0.43},
    {"efficientnet_b0", Family::CNN, "imagenet", 128, 1, 35.21, 1, 13.83, 0.45},
    {"resnet50", Family::CNN, "imagenet", 32, 1, 36.32, 1, 5.26, 0.42},
    {"resnet50", Family::CNN, "imagenet", 64, 1, 35.50, 1, 8.54, 0.44},
    {"resnet50", Family::CNN, "imagenet", 128, 1, 35.01, 1, 15.12, 0.45},
    {"mobilenet_v2", Family::CNN, "imagenet", 32, 1, 36.09, 1, 4.54, 0.41},
    {"mobilenet_v2", Family::CNN, "imagenet", 64, 1, 35.43, 1, 7.22, 0.42},
    {"mobilenet_v2", Family::CNN, "imagenet", 128, 1, 34.91, 1, 12.58, 0.44},
    {"vgg16", Family::CNN, "imagenet", 32, 1, 48.45, 1, 8.22, 0.42},
    {"vgg16", Family::CNN, "imagenet", 64, 1, 44.38, 1, 13.64, 0.44},
    {"vgg16", Family::CNN, "imagenet", 128, 1, 42.42, 1, 24.41, 0.45},
    {"xception", Family::CNN, "imagenet", 32, 1, 46.86, 1, 7.20, 0.42},
    {"xception", Family::CNN, "imagenet", 64, 1, 45.78, 1, 11.52, 0.43},
    {"xception", Family::CNN, "imagenet", 128, 1, 44.44, 1, 22.98, 0.44},
    {"inception", Family::CNN, "imagenet", 32, 1, 50.10, 1, 6.35, 0.41},
    {"inception", Family::CNN, "imagenet", 64, 1, 46.29, 1, 10.56, 0.43},
    {"inception", Family::CNN, "imagenet", 128, 1, 44.85, 1, 19.02, 0.44},
    {"efficientnet_b0", Family::CNN, "cifar100", 32, 1, 0.77, 0, 1.86, 0.66},
    {"efficientnet_b0", Family::CNN, "cifar100", 64, 1, 0.48, 0, 1.91, 0.70},
    {"efficientnet_b0", Family::CNN, "cifar100", 128, 1, 0.27, 0, 2.05, 0.74},
    {"resnet18", Family::CNN, "cifar100", 32, 1, 0.33, 0, 1.96, 0.64},
    {"resnet18", Family::CNN, "cifar100", 64, 1, 0.22, 0, 1.97, 0.68},
    {"resnet18", Family::CNN, "cifar100", 128, 1, 0.16, 0, 2.01, 0.72},
    {"resnet34", Family::CNN, "cifar100", 32, 1, 0.49, 0, 2.15, 0.65},
    {"resnet34", Family::CNN, "cifar100", 64, 1, 0.30, 0, 2.17, 0.69},
    {"resnet34", Family::CNN, "cifar100", 128, 1, 0.20, 0, 2.19, 0.73},
    {"mobilenetv3_small", Family::CNN, "cifar100", 32, 1, 0.54, 0, 1.78, 0.62},
    {"mobilenetv3_small", Family::CNN, "cifar100", 64, 1, 0.32, 0, 1.79, 0.66},
    {"mobilenetv3_small", Family::CNN, "cifar100", 128, 1, 0.22, 0, 1.82, 0.70},
};

std::vector<CatalogEntry> build() {
    std::vector<CatalogEntry> out;
    for (const Row& r : kTable) {
        CatalogEntry e;
        e.model = r.model;
        e.dataset = r.dataset;
        e.key = e.model + "_" + e.dataset + "_bs" + std::to_string(r.batch);
        e.family = r.family;
        e.batch = r.batch;
        e.gpus = r.gpus;
        e.epoch_minutes = r.epoch_minutes;
        if (r.epochs == 0)
            e.epoch_options = {20, 50};
        else
            e.epoch_options = {static_cast<std::uint64_t>(r.epochs)};
        e.mem_gib = r.mem_gib;
        e.demand = r.demand;
        // Transformers are heavy; ImageNet CNNs are heavy from 19 GiB up;
        // CIFAR rows are light (traces.cpp:44, :76, :97).
        if (r.family == Family::Transformer)
            e.wclass = WeightClass::heavy;
        else if (e.dataset == "cifar100")
            e.wclass = WeightClass::light;
        else
            e.wclass = r.mem_gib >= 19.0 ? WeightClass::heavy : WeightClass::medium;
        out.push_back(std::move(e));
    }
    return out;
}

int model_depth(const std::string& name) {
    static const std::map<std::string, int> kDepth = {
        {"resnet18", 18},     {"resnet34", 34},      {"resnet50", 50},
        {"vgg16", 16},        {"efficientnet_b0", 25}, {"mobilenet_v2", 19},
        {"mobilenetv3_small", 13}, {"xception", 36}, {"inception", 22},
        {"xlnet_base", 12},   {"xlnet_large", 24},   {"bert_base", 12},
        {"bert_large", 24},   {"gpt2_large", 36},
    };
    auto it = kDepth.find(name);
    return it == kDepth.end() ? 16 : it->second;
}

// Integer rescale so the column sums hit the targets; the remainder lands on
// the (first) largest rescaled layer (traces.cpp:135-170).
void rescale(std::vector<Layer>& layers, std::uint64_t p_target, std::uint64_t a_target) {
    std::uint64_t p_sum = 0, a_sum = 0;
    for (const auto& l : layers) {
        p_sum += l.params;
        a_sum += l.acts;
    }
    std::size_t p_big = 0, a_big = 0;
    std::uint64_t p_new = 0, a_new = 0;
    for (std::size_t i = 0; i < layers.size(); ++i) {
        Layer& l = layers[i];
        l.params = p_sum ? static_cast<std::uint64_t>(static_cast<double>(l.params) *
                                                      static_cast<double>(p_target) /
                                                      static_cast<double>(p_sum))
                         : 0;
        l.acts = a_sum ? static_cast<std::uint64_t>(static_cast<double>(l.acts) *
                                                    static_cast<double>(a_target) /
                                                    static_cast<double>(a_sum))
                       : 0;
        if (l.params > layers[p_big].params) p_big = i;
        if (l.acts > layers[a_big].acts) a_big = i;
        p_new += l.params;
        a_new += l.acts;
    }
    layers[p_big].params += p_target - p_new;
    layers[a_big].acts += a_target - a_new;
}

}  // namespace

const std::vector<CatalogEntry>& catalog() {
    static const std::vector<CatalogEntry> kCat = build();
    return kCat;
}

int catalog_index(const std::string& key) {
    const auto& c = catalog();
    for (std::size_t i = 0; i < c.size(); ++i)
        if (c[i].key == key) return static_cast<int>(i);
    return -1;
}

// catalog_descriptor (traces.cpp:175-236): a layer stack whose footprint lands
// on the catalog's measured memory.
Architecture catalog_architecture(const CatalogEntry& e) {
    const SimConstants c;
    const Bytes mem = static_cast<Bytes>(std::llround(e.mem_gib * static_cast<double>(kGiB)));
    const Bytes raw = mem > c.framework_base ? mem - c.framework_base : 0;
    const bool tf = e.family == Family::Transformer;
    const double act_share = tf ? 0.45 : 0.72;
    const std::uint64_t A = static_cast<std::uint64_t>(
        act_share * static_cast<double>(raw) /
        static_cast<double>(c.bytes_per_value * e.batch));
    const std::uint64_t P = static_cast<std::uint64_t>(
        (1.0 - act_share) * static_cast<double>(raw) /
        static_cast<double>(c.bytes_per_value * c.param_copies));

    Architecture a;
    a.family = e.family;
    const std::uint64_t depth = static_cast<std::uint64_t>(model_depth(e.model));
    if (tf) {
        a.activation_angle = activation_angle(1);  // gelu
        std::uint64_t d = static_cast<std::uint64_t>(
            std::sqrt(0.8 * static_cast<double>(P) / (12.0 * static_cast<double>(depth))));
        d = std::max<std::uint64_t>(64, d / 64 * 64);
        const std::uint64_t seq = std::max<std::uint64_t>(16, A / (d * (7 * depth + 1)));
        a.layers.push_back({LayerKind::embedding, 30000 * d, seq * d});
        for (std::uint64_t i = 0; i < depth; ++i) {
            a.layers.push_back({LayerKind::attention, 4 * d * d, 2 * seq * d});
            a.layers.push_back({LayerKind::linear, 8 * d * d, 5 * seq * d});
        }
    } else {
        a.activation_angle = activation_angle(0);  // relu
        const bool cifar = e.dataset == "cifar100";
        const std::uint64_t side = cifar ? 32 : 224;
        const std::uint64_t out = cifar ? 100 : 1000;
        std::uint64_t c_prev = 3, spatial = side * side;
        for (std::uint64_t i = 0; i < depth; ++i) {
            const std::uint64_t stage = std::min<std::uint64_t>(3, i * 4 / depth);
            const std::uint64_t ch = 64ull << stage;
            a.layers.push_back({LayerKind::conv2d, 9 * c_prev * ch + ch, ch * spatial});
            if (i % 2 == 0) a.layers.push_back({LayerKind::batchnorm, 2 * ch, ch * spatial});
            if (i % 2 == 1 && spatial > 64) spatial /= 4;
            c_prev = ch;
        }
        a.layers.push_back({LayerKind::linear, c_prev * out + out, out});
    }
    rescale(a.layers, P, A);
    return a;
}

// ----------------------------------------------------------------- traces
namespace {
Trace draw_rows(Rng& rng, std::vector<std::int32_t> picks, double mean_gap) {
    rng.shuffle(picks);
    Trace t;
    const auto& cat = catalog();
    double clock = 0.0;
    for (std::size_t i = 0; i < picks.size(); ++i) {
        const CatalogEntry& e = cat[static_cast<std::size_t>(picks[i])];
        if (i > 0) clock += rng.exponential(mean_gap);
        TraceRow r;
        r.submit = std::round(clock * 1000.0) / 1000.0;
        r.entry = picks[i];
        r.epochs = e.epoch_options.size() == 1
                       ? e.epoch_options[0]
                       : e.epoch_options[rng.uniform(e.epoch_options.size())];
        t.rows.push_back(r);
    }
    return t;
}
}  // namespace

// traces.cpp:266-306: class quotas, uniform draws within class, shuffle,
// exponential gaps on a millisecond grid, light-row epoch choice.
Trace generate_trace(Mix mix, std::uint64_t seed) {
    std::vector<std::pair<WeightClass, std::size_t>> plan;
    if (mix == Mix::t90)
        plan = {{WeightClass::light, 59}, {WeightClass::medium, 24}, {WeightClass::heavy, 7}};
    else
        plan = {{WeightClass::medium, 50}, {WeightClass::heavy, 10}};
    std::map<WeightClass, std::vector<std::int32_t>> pools;
    const auto& cat = catalog();
    for (std::size_t i = 0; i < cat.size(); ++i)
        pools[cat[i].wclass].push_back(static_cast<std::int32_t>(i));
    Rng rng(seed);
    std::vector<std::int32_t> picks;
    for (const auto& [wc, count] : plan) {
        const auto& pool = pools.at(wc);
        for (std::size_t i = 0; i < count; ++i) picks.push_back(pool[rng.uniform(pool.size())]);
    }
    Trace t = draw_rows(rng, std::move(picks), 120.0);
    t.seed = seed;
    t.mix = mix == Mix::t90 ? "t90" : "t60";
    return t;
}

Trace generate_uniform_trace(std::size_t n, double mean_gap, std::uint64_t seed) {
    Rng rng(seed);
    std::vector<std::int32_t> picks(n);
    const std::uint64_t m = catalog().size();
    for (auto& p : picks) p = static_cast<std::int32_t>(rng.uniform(m));
    Trace t = draw_rows(rng, std::move(picks), mean_gap);
    t.seed = seed;
    t.mix = "uniform";
    return t;
}

// `#carma-trace v1` (traces.cpp:308-366).
void save_trace(const Trace& t, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
    out << "#carma-trace v1 seed=" << t.seed << " mix=" << t.mix << "\n";
    const auto& cat = catalog();
    char buf[64];
    for (const auto& r : t.rows) {
        std::snprintf(buf, sizeof(buf), "%.3f", r.submit);
        out << buf << ',' << cat[static_cast<std::size_t>(r.entry)].key << ',' << r.epochs << '\n';
    }
}

Trace load_trace(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open '" + path + "'");
    std::string header;
    if (!std::getline(in, header)) throw std::runtime_error("empty trace file");
    Trace t;
    {
        std::istringstream hs(header);
        std::string magic, field;
        hs >> magic >> field;
        if (magic != "#carma-trace" || field != "v1") throw std::runtime_error("bad trace header");
        while (hs >> field) {
            const auto eq = field.find('=');
            if (eq == std::string::npos) throw std::runtime_error("bad header field");
            if (field.substr(0, eq) == "seed") t.seed = std::stoull(field.substr(eq + 1));
            if (field.substr(0, eq) == "mix") t.mix = field.substr(eq + 1);
        }
    }
    std::string line;
    double prev = -1.0;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        const auto c1 = line.find(',');
        const auto c2 = c1 == std::string::npos ? c1 : line.find(',', c1 + 1);
        if (c2 == std::string::npos) throw std::runtime_error("bad trace row: " + line);
        TraceRow r;
        try {
            r.submit = std::stod(line.substr(0, c1));
            r.epochs = std::stoull(line.substr(c2 + 1));
        } catch (const std::exception&) {
            throw std::runtime_error("non-numeric trace row: " + line);
        }
        r.entry = catalog_index(line.substr(c1 + 1, c2 - c1 - 1));
        if (r.entry < 0) throw std::runtime_error("unknown catalog key in: " + line);
        if (r.submit < prev) throw std::runtime_error("submit times must be non-decreasing");
        prev = r.submit;
        t.rows.push_back(r);
    }
    return t;
}

// materialize_trace + task_from_catalog (traces.cpp:238-254, :368-379).
std::vector<Task> materialize(const Trace& t) {
    std::vector<Task> out;
    out.reserve(t.rows.size());
    const auto& cat = catalog();
    char id[96];
    for (std::size_t i = 0; i < t.rows.size(); ++i) {
        const TraceRow& r = t.rows[i];
        const CatalogEntry& e = cat[static_cast<std::size_t>(r.entry)];
        std::snprintf(id, sizeof(id), "t%03zu-%s", i, e.key.c_str());
        Task k;
        k.id = id;
        k.submit = r.submit;
        k.true_mem = static_cast<Bytes>(std::llround(e.mem_gib * static_cast<double>(kGiB)));
        k.work = static_cast<double>(r.epochs) * (e.epoch_minutes * 60.0);
        k.demand = e.demand;
        k.gpus = static_cast<std::uint32_t>(e.gpus);
        k.family = e.family;
        k.batch = e.batch;
        k.entry = r.entry;
        out.push_back(std::move(k));
    }
    return out;
}

// --------------------------------------------------------------- datasets
Bounds Bounds::for_family(Family f) {
    Bounds b;
    if (f == Family::CNN) {
        b = {4, 40, 16, 1152, 16, 256, 32, 224, 10, 1000};
    } else if (f == Family::Transformer) {
        b = {2, 24, 256, 2048, 1, 64, 64, 1280, 8000, 50000};
    }
    return b;
}

namespace {

enum class Shape { uniform, pyramid, hourglass };

std::uint64_t shaped_width(Shape shape, std::uint64_t base, std::size_t i, std::size_t n,
                           std::uint64_t floor_width) {
    if (n <= 1) return base;
    const double pos = static_cast<double>(i) / static_cast<double>(n - 1);
    double scale = 1.0;
    if (shape == Shape::pyramid) scale = 1.0 - 0.75 * pos;
    if (shape == Shape::hourglass) scale = 1.0 - 0.75 * (1.0 - std::abs(2.0 * pos - 1.0));
    return std::max<std::uint64_t>(floor_width,
                                   static_cast<std::uint64_t>(scale * static_cast<double>(base)));
}

std::uint64_t draw(Rng& rng, std::uint64_t lo, std::uint64_t hi) {
    return static_cast<std::uint64_t>(
        rng.uniform_int(static_cast<std::int64_t>(lo), static_cast<std::int64_t>(hi)));
}

double draw_activation(Rng& rng) { return activation_angle(static_cast<int>(rng.uniform(8))); }

// estimators.cpp:125-153
Architecture sample_mlp(Rng& rng, const Bounds& b) {
    Architecture m;
    m.family = Family::MLP;
    const std::uint64_t input = draw(rng, b.min_input, b.max_input);
    const std::uint64_t output = draw(rng, b.min_output, b.max_output);
    const std::size_t n = draw(rng, b.min_layers, b.max_layers);
    const std::uint64_t base = draw(rng, b.min_width, b.max_width);
    const Shape shape = static_cast<Shape>(rng.uniform(3));
    m.activation_angle = draw_activation(rng);
    std::uint64_t prev = input;
    for (std::size_t i = 0; i < n; ++i) {
        const bool head = i + 1 == n;
        const std::uint64_t w = head ? output : shaped_width(shape, base, i, n, b.min_width);
        m.layers.push_back({LayerKind::linear, prev * w + w, w});
        if (!head && rng.next_double() < 0.5) m.layers.push_back({LayerKind::batchnorm, 2 * w, w});
        if (!head && rng.next_double() < 0.3) m.layers.push_back({LayerKind::dropout, 0, w});
        prev = w;
    }
    return m;
}

// estimators.cpp:155-186
Architecture sample_cnn(Rng& rng, const Bounds& b) {
    Architecture m;
    m.family = Family::CNN;
    const std::uint64_t side = draw(rng, b.min_input, b.max_input);
    const std::uint64_t output = draw(rng, b.min_output, b.max_output);
    const std::size_t n = draw(rng, b.min_layers, b.max_layers);
    const std::uint64_t base = draw(rng, b.min_width, b.max_width);
    const Shape shape = static_cast<Shape>(rng.uniform(3));
    m.activation_angle = draw_activation(rng);
    std::uint64_t c_prev = 3, spatial = side * side;
    for (std::size_t i = 0; i < n; ++i) {
        const std::uint64_t c = shaped_width(shape, base, n - 1 - i, n, b.min_width);
        m.layers.push_back({LayerKind::conv2d, 9 * c_prev * c + c, c * spatial});
        if (rng.next_double() < 0.7) m.layers.push_back({LayerKind::batchnorm, 2 * c, c * spatial});
        if (i % 2 == 1 && spatial > 64) spatial /= 4;
        c_prev = c;
    }
    if (rng.next_double() < 0.3) m.layers.push_back({LayerKind::dropout, 0, c_prev});
    m.layers.push_back({LayerKind::linear, c_prev * output + output, output});
    return m;
}

// estimators.cpp:188-217
Architecture sample_transformer(Rng& rng, const Bounds& b) {
    Architecture m;
    m.family = Family::Transformer;
    const std::uint64_t seq = draw(rng, b.min_input, b.max_input);
    const std::uint64_t vocab = draw(rng, b.min_output, b.max_output);
    const std::size_t n = draw(rng, b.min_layers, b.max_layers);
    const std::uint64_t base = draw(rng, b.min_width, b.max_width);
    const Shape shape = static_cast<Shape>(rng.uniform(3));
    m.activation_angle = draw_activation(rng);
    const std::uint64_t d0 = (base / 64) * 64;
    m.layers.push_back({LayerKind::embedding, vocab * d0, seq * d0});
    for (std::size_t i = 0; i < n; ++i) {
        std::uint64_t d = shaped_width(shape, base, i, n, b.min_width);
        d = std::max<std::uint64_t>(64, (d / 64) * 64);
        m.layers.push_back({LayerKind::attention, 4 * d * d, 2 * seq * d});
        m.layers.push_back({LayerKind::linear, 8 * d * d, 5 * seq * d});
        if (rng.next_double() < 0.4) m.layers.push_back({LayerKind::dropout, 0, seq * d});
    }
    return m;
}

}  // namespace

// estimators.cpp:221-264, with infeasible (> device capacity) draws resampled.
Dataset generate_dataset(Family f, std::size_t n, std::uint64_t seed) {
    if (n == 0) throw std::invalid_argument("n_samples must be > 0");
    const Bounds b = Bounds::for_family(f);
    Dataset ds;
    ds.family = f;
    ds.bucket_range = default_bucket_range(f);
    ds.seed = seed;
    ds.rows.reserve(n);
    ds.bucket.reserve(n);
    ds.mem.reserve(n);
    const Bytes feasible = SimConstants{}.gpu_capacity;
    Rng rng(seed);
    int rejects = 0;
    while (ds.rows.size() < n) {
        Architecture a = f == Family::MLP ? sample_mlp(rng, b)
                         : f == Family::CNN ? sample_cnn(rng, b)
                                            : sample_transformer(rng, b);
        const std::uint64_t batch = draw(rng, b.min_batch, b.max_batch);
        const Bytes mem = ground_truth_memory(a, batch);
        if (mem > feasible) {
            if (++rejects > 10000) throw std::runtime_error("bounds generate almost no feasible configs");
            continue;
        }
        rejects = 0;
        ds.rows.push_back(extract_features(a, batch));
        ds.mem.push_back(mem);
        ds.bucket.push_back(static_cast<std::int32_t>(mem / ds.bucket_range));
    }
    return ds;
}

// estimators.cpp:344-395: seeded 70/30 split, min-max bounds over the
// training rows, normalised training points. The holdout evaluation
// (:396-434) runs the GPU predict (see knn.cpp).
KnnModel fit_knn(const Dataset& ds, std::uint32_t k) {
    if (ds.rows.empty()) throw std::invalid_argument("dataset has no rows");
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    KnnModel m;
    m.family = ds.family;
    m.bucket_range = ds.bucket_range;
    m.k = k;
    m.seed = ds.seed;
    std::vector<std::size_t> order(ds.rows.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
    Rng rng(ds.seed ^ 0x9e3779b97f4a7c15ull);
    rng.shuffle(order);
    const std::size_t train_n = std::max<std::size_t>(1, order.size() * 7 / 10);
    ScalarRow lo, hi;
    lo.fill(std::numeric_limits<double>::infinity());
    hi.fill(-std::numeric_limits<double>::infinity());
    std::vector<ScalarRow> raw(train_n);
    for (std::size_t i = 0; i < train_n; ++i) {
        raw[i] = scalar_features(ds.rows[order[i]]);
        for (int d = 0; d < kFeatureDims; ++d) {
            lo[d] = std::min(lo[d], raw[i][d]);
            hi[d] = std::max(hi[d], raw[i][d]);
        }
    }
    bool varying = false;
    for (int d = 0; d < kFeatureDims; ++d) varying |= hi[d] > lo[d];
    if (!varying) throw std::invalid_argument("all features have zero variance");
    m.lo = lo;
    m.hi = hi;
    m.points.resize(train_n * kFeatureDims);
    m.labels.resize(train_n);
    for (std::size_t i = 0; i < train_n; ++i) {
        for (int d = 0; d < kFeatureDims; ++d)
            m.points[i * kFeatureDims + d] =
                hi[d] > lo[d] ? (raw[i][d] - lo[d]) / (hi[d] - lo[d]) : 0.0;
        m.labels[i] = ds.bucket[order[i]];
    }
    m.holdout_rows.assign(order.begin() + static_cast<std::ptrdiff_t>(train_n), order.end());
    return m;
}

}  // namespace carma_b200
