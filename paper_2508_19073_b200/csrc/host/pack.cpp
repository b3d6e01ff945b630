// carma_pack_features: the 64-byte lossless packing of feature rows (layout
// in include/carma_gpu.h). Host-side data formatting for bulk callers.

#include <cstring>

#include "../../../include/carma_gpu.h"
#include "status.hpp"

using namespace carma_b200;

extern "C" carma_status carma_pack_features(const carma_feature_row* rows, const int8_t* family,
                                            int32_t default_family, uint64_t n, double* act_table,
                                            carma_feature_packed* out) {
    return guarded([&] {
        if (!rows || !act_table || !out) throw InvalidArg("null argument");
        constexpr uint64_t k48 = 1ull << 48;
        int n_act = 0;
        for (int i = 0; i < 16; ++i) act_table[i] = 0.0;
        auto code_of = [&](double c, double s) -> uint64_t {
            for (int k = 0; k < n_act; ++k)
                if (std::memcmp(&act_table[2 * k], &c, 8) == 0 && std::memcmp(&act_table[2 * k + 1], &s, 8) == 0)
                    return static_cast<uint64_t>(k);
            if (n_act == 8) throw Unsupported("more than 8 distinct activations in one packed batch");
            act_table[2 * n_act] = c;
            act_table[2 * n_act + 1] = s;
            return static_cast<uint64_t>(n_act++);
        };
        for (uint64_t i = 0; i < n; ++i) {
            const carma_feature_row& r = rows[i];
            const int f = family ? family[i] : default_family;
            if (f < 0 || f > 255) throw InvalidArg("family out of range");
            const uint64_t big[8] = {r.total_params, r.total_activations, r.tuple_acts[0], r.tuple_params[0],
                                     r.tuple_acts[1], r.tuple_params[1], r.tuple_acts[2], r.tuple_params[2]};
            for (uint64_t v : big)
                if (v >= k48) throw Unsupported("count >= 2^48 does not fit the packed format");
            if (r.n_linear > 255 || r.n_batchnorm > 255 || r.n_dropout > 255 || r.n_conv > 255)
                throw Unsupported("layer tally > 255 does not fit the packed format");
            if (r.batch_size >= (1ull << 32)) throw Unsupported("batch >= 2^32 does not fit the packed format");
            for (int k = 0; k < 3; ++k)
                if (r.kind[k] < 0 || r.kind[k] > 15) throw Unsupported("layer kind code out of range");
            const uint64_t code = code_of(r.act_cos, r.act_sin);
            carma_feature_packed& o = out[i];
            o.w[0] = r.total_params | (r.n_linear << 48) | (r.n_batchnorm << 56);
            o.w[1] = r.total_activations | (r.n_dropout << 48) | (r.n_conv << 56);
            o.w[2] = r.tuple_acts[0] | ((r.batch_size & 0xffffull) << 48);
            o.w[3] = r.tuple_params[0] | (static_cast<uint64_t>(r.kind[0]) << 48) |
                     (static_cast<uint64_t>(r.kind[1]) << 52) | (static_cast<uint64_t>(r.kind[2]) << 56) |
                     (static_cast<uint64_t>(r.has_layers ? 1 : 0) << 60) | (code << 61);
            o.w[4] = r.tuple_acts[1] | (static_cast<uint64_t>(f) << 48);
            o.w[5] = r.tuple_params[1] | ((r.batch_size >> 16) << 48);
            o.w[6] = r.tuple_acts[2];
            o.w[7] = r.tuple_params[2];
        }
    });
}
