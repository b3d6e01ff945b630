// LearnedEstimator snapshots (the reference's "carma-knn-estimator/v1" JSON,
// LearnedEstimator::save / ::load, proj/src/estimators.cpp:481-538) read
// straight into a k-NN bank: carma_host_parse_snapshot returns the fitted
// state, carma_knn_load_snapshot installs it (carma_knn_set_model).
//
// The parser is a small strict JSON reader: objects, arrays, strings,
// numbers, true/false/null. Integers are parsed as integers (bucket_range,
// k, seed, labels and sizes stay exact beyond 2^53); every other number goes
// through strtod, which rounds correctly, so the shortest round-trip digits
// the reference writes come back as the same doubles.

#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../../include/carma_gpu.h"
#include "../../../include/carma_host.h"
#include "status.hpp"

using namespace carma_b200;

namespace {

struct JValue {
    enum Kind { Null, Bool, Int, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    int64_t i = 0;
    uint64_t u = 0;  // Int: the unsigned value when non-negative
    bool neg = false;
    double d = 0.0;
    std::string s;
    std::vector<JValue> a;
    std::vector<std::pair<std::string, JValue>> o;

    const JValue& at(const std::string& key) const {
        for (const auto& kv : o)
            if (kv.first == key) return kv.second;
        throw InvalidArg("estimator snapshot: missing key '" + key + "'");
    }
    const JValue* find(const std::string& key) const {
        for (const auto& kv : o)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
    double num() const {
        if (kind == Num) return d;
        if (kind == Int) return neg ? static_cast<double>(i) : static_cast<double>(u);
        throw InvalidArg("estimator snapshot: number expected");
    }
    uint64_t uint() const {
        if (kind != Int || neg) throw InvalidArg("estimator snapshot: non-negative integer expected");
        return u;
    }
    int64_t sint() const {
        if (kind != Int) throw InvalidArg("estimator snapshot: integer expected");
        return neg ? i : static_cast<int64_t>(u);
    }
};

struct Parser {
    const char* p;
    const char* e;

    [[noreturn]] void fail(const char* what) const {
        throw InvalidArg(std::string("estimator snapshot: malformed JSON (") + what + ")");
    }
    void ws() {
        while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (static_cast<size_t>(e - p) >= n && std::memcmp(p, w, n) == 0) {
            p += n;
            return true;
        }
        return false;
    }
    std::string str() {
        if (p >= e || *p != '"') fail("string expected");
        ++p;
        std::string out;
        while (p < e && *p != '"') {
            if (*p == '\\') {
                if (++p >= e) fail("escape");
                switch (*p) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    default: fail("unsupported escape");
                }
                ++p;
            } else {
                out += *p++;
            }
        }
        if (p >= e) fail("unterminated string");
        ++p;
        return out;
    }
    JValue number() {
        const char* s = p;
        if (p < e && *p == '-') ++p;
        bool integral = true;
        while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '+' ||
                         *p == '-')) {
            if (*p == '.' || *p == 'e' || *p == 'E') integral = false;
            ++p;
        }
        const std::string tok(s, p);
        if (tok.empty() || tok == "-") fail("number expected");
        JValue v;
        errno = 0;
        if (integral) {
            v.kind = JValue::Int;
            v.neg = tok[0] == '-';
            char* end = nullptr;
            if (v.neg) {
                v.i = std::strtoll(tok.c_str(), &end, 10);
            } else {
                v.u = std::strtoull(tok.c_str(), &end, 10);
            }
            if (errno || *end) fail("integer out of range");
        } else {
            v.kind = JValue::Num;
            char* end = nullptr;
            v.d = std::strtod(tok.c_str(), &end);
            if (*end) fail("number");
        }
        return v;
    }
    JValue value(int depth = 0) {
        if (depth > 16) fail("nesting");
        ws();
        if (p >= e) fail("value expected");
        JValue v;
        if (*p == '{') {
            ++p;
            v.kind = JValue::Obj;
            ws();
            if (p < e && *p == '}') {
                ++p;
                return v;
            }
            for (;;) {
                ws();
                std::string k = str();
                ws();
                if (p >= e || *p != ':') fail("':' expected");
                ++p;
                v.o.emplace_back(std::move(k), value(depth + 1));
                ws();
                if (p < e && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < e && *p == '}') {
                    ++p;
                    return v;
                }
                fail("',' or '}' expected");
            }
        }
        if (*p == '[') {
            ++p;
            v.kind = JValue::Arr;
            ws();
            if (p < e && *p == ']') {
                ++p;
                return v;
            }
            for (;;) {
                v.a.push_back(value(depth + 1));
                ws();
                if (p < e && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < e && *p == ']') {
                    ++p;
                    return v;
                }
                fail("',' or ']' expected");
            }
        }
        if (*p == '"') {
            v.kind = JValue::Str;
            v.s = str();
            return v;
        }
        if (lit("true")) {
            v.kind = JValue::Bool;
            v.b = true;
            return v;
        }
        if (lit("false")) {
            v.kind = JValue::Bool;
            return v;
        }
        if (lit("null")) return v;
        return number();
    }
};

int32_t family_code(const std::string& name) {
    std::string l = name;
    for (auto& c : l) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    if (l == "mlp") return CARMA_FAMILY_MLP;
    if (l == "cnn") return CARMA_FAMILY_CNN;
    if (l == "transformer") return CARMA_FAMILY_TRANSFORMER;
    throw InvalidArg("estimator snapshot: unsupported model family '" + name + "'");
}

struct Snapshot {
    int32_t family = 0;
    uint64_t bucket_range = 0, k = 0, seed = 0;
    double lo[19] = {0}, hi[19] = {0};
    std::vector<double> points;  // n x 19
    std::vector<int32_t> labels;
    carma_holdout_report holdout{};
};

// LearnedEstimator::load's checks (estimators.cpp:503-538), same messages.
Snapshot parse(const char* text, uint64_t len) {
    if (!text) throw InvalidArg("estimator snapshot: null text");
    Parser ps{text, text + len};
    const JValue j = ps.value();
    ps.ws();
    if (ps.p != ps.e) throw InvalidArg("estimator snapshot: trailing characters");
    if (j.kind != JValue::Obj) throw InvalidArg("estimator snapshot: object expected");
    const JValue* schema = j.find("schema");
    if (!schema || schema->kind != JValue::Str || schema->s != "carma-knn-estimator/v1")
        throw InvalidArg("unrecognized estimator snapshot schema");
    Snapshot s;
    s.family = family_code(j.at("family").s);
    s.bucket_range = j.at("bucket_range").uint();
    s.k = j.at("k").uint();
    s.seed = j.at("seed").uint();
    const JValue& lo = j.at("lo");
    const JValue& hi = j.at("hi");
    if (lo.a.size() != 19 || hi.a.size() != 19) throw InvalidArg("estimator snapshot has wrong feature width");
    for (int d = 0; d < 19; ++d) {
        s.lo[d] = lo.a[d].num();
        s.hi[d] = hi.a[d].num();
    }
    for (const JValue& l : j.at("labels").a) s.labels.push_back(static_cast<int32_t>(l.sint()));
    const JValue& pts = j.at("points");
    s.points.reserve(pts.a.size() * 19);
    for (const JValue& row : pts.a) {
        if (row.a.size() != 19) throw InvalidArg("estimator snapshot has wrong feature width");
        for (const JValue& x : row.a) s.points.push_back(x.num());
    }
    if (s.labels.size() != pts.a.size()) throw InvalidArg("estimator snapshot labels/points mismatch");
    const JValue& h = j.at("holdout");
    s.holdout.accuracy = h.at("accuracy").num();
    s.holdout.macro_f1 = h.at("macro_f1").num();
    s.holdout.train_size = h.at("train_size").uint();
    s.holdout.holdout_size = h.at("holdout_size").uint();
    s.holdout.underestimate_rate = h.at("underestimate_rate").num();
    return s;
}

}  // namespace

extern "C" {

carma_status carma_host_parse_snapshot(const char* json, uint64_t len, int32_t* family, uint64_t* k,
                                       uint64_t* bucket_range, uint64_t* seed, double* lo, double* hi,
                                       double* points, int32_t* labels, uint64_t capacity, uint64_t* n,
                                       carma_holdout_report* holdout) {
    return guarded([&] {
        const Snapshot s = parse(json, len);
        const uint64_t rows = s.labels.size();
        if (n) *n = rows;
        if (family) *family = s.family;
        if (k) *k = s.k;
        if (bucket_range) *bucket_range = s.bucket_range;
        if (seed) *seed = s.seed;
        if (lo) std::memcpy(lo, s.lo, sizeof s.lo);
        if (hi) std::memcpy(hi, s.hi, sizeof s.hi);
        if (holdout) *holdout = s.holdout;
        if (points || labels) {
            if (capacity < rows) throw InvalidArg("estimator snapshot: capacity below the point count");
            if (points) std::memcpy(points, s.points.data(), s.points.size() * sizeof(double));
            if (labels) std::memcpy(labels, s.labels.data(), rows * sizeof(int32_t));
        }
    });
}

carma_status carma_knn_load_snapshot(carma_knn* h, const char* json, uint64_t len, int32_t* family_out,
                                     carma_holdout_report* holdout_out) {
    carma_status st = guarded([&] {
        const Snapshot s = parse(json, len);
        if (s.k == 0 || s.k > 0xffffffffull) throw InvalidArg("k must be >= 1");
        if (family_out) *family_out = s.family;
        if (holdout_out) *holdout_out = s.holdout;
        const carma_status r = carma_knn_set_model(h, s.family, s.lo, s.hi, s.points.data(), s.labels.data(),
                                                   s.labels.size(), static_cast<uint32_t>(s.k), s.bucket_range);
        if (r != CARMA_OK) throw CarmaFailure(r, carma_last_error());
    });
    return st;
}

carma_status carma_knn_load_snapshot_file(carma_knn* h, const char* path, int32_t* family_out,
                                          carma_holdout_report* holdout_out) {
    std::string text;
    carma_status st = guarded([&] {
        if (!path) throw InvalidArg("null path");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw InvalidArg(std::string("cannot open '") + path + "'");
        std::ostringstream ss;
        ss << in.rdbuf();
        text = ss.str();
    });
    if (st != CARMA_OK) return st;
    return carma_knn_load_snapshot(h, text.data(), text.size(), family_out, holdout_out);
}

}  // extern "C"
