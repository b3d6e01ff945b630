// carma_pack_features: the 64-byte lossless packing of feature rows (layout
// in include/carma_gpu.h). Host-side data formatting for bulk callers.

#include <algorithm>
#include <cstring>

#include "../../../include/carma_gpu.h"
#include "stage.hpp"
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

// Frame-of-reference bit packing (layout in include/carma_gpu.h).
extern "C" carma_status carma_pack_features_bits(const carma_feature_row* rows, const int8_t* family,
                                                 int32_t default_family, uint64_t n, carma_bit_schema* schema,
                                                 uint32_t* words, uint64_t* n_words) {
    return guarded([&] {
        if (!rows || !schema || !n_words) throw InvalidArg("null argument");
        constexpr int F = CARMA_BIT_FIELDS;
        // activation codes via the 8-entry table
        double table[16];
        int n_act = 0;
        for (double& t : table) t = 0.0;
        auto code_of = [&](double c, double s) -> uint64_t {
            for (int k = 0; k < n_act; ++k)
                if (std::memcmp(&table[2 * k], &c, 8) == 0 && std::memcmp(&table[2 * k + 1], &s, 8) == 0)
                    return static_cast<uint64_t>(k);
            if (n_act == 8) throw Unsupported("more than 8 distinct activations in one packed batch");
            table[2 * n_act] = c;
            table[2 * n_act + 1] = s;
            return static_cast<uint64_t>(n_act++);
        };
        auto fields = [&](uint64_t i, uint64_t* v) {
            const carma_feature_row& r = rows[i];
            const int f = family ? family[i] : default_family;
            if (f < 0 || f > 255) throw InvalidArg("family out of range");
            v[0] = r.n_linear; v[1] = r.n_batchnorm; v[2] = r.n_dropout; v[3] = r.n_conv;
            v[4] = r.batch_size; v[5] = r.total_params; v[6] = r.total_activations;
            v[7] = code_of(r.act_cos, r.act_sin);
            for (int k = 0; k < 3; ++k) {
                if (r.kind[k] < 0) throw Unsupported("negative layer kind code");
                v[8 + k] = static_cast<uint64_t>(r.kind[k]);
                v[12 + 2 * k] = r.tuple_acts[k];
                v[13 + 2 * k] = r.tuple_params[k];
            }
            v[11] = r.has_layers ? 1 : 0;
            v[18] = static_cast<uint64_t>(f);
        };
        uint64_t lo[F], hi[F], v[F];
        for (int f = 0; f < F; ++f) {
            lo[f] = ~0ull;
            hi[f] = 0;
        }
        for (uint64_t i = 0; i < n; ++i) {
            fields(i, v);
            for (int f = 0; f < F; ++f) {
                lo[f] = std::min(lo[f], v[f]);
                hi[f] = std::max(hi[f], v[f]);
            }
        }
        std::memset(schema, 0, sizeof(*schema));
        uint32_t off = 0;
        for (int f = 0; f < F; ++f) {
            if (n == 0) lo[f] = hi[f] = 0;
            const uint64_t span = hi[f] - lo[f];
            int w = 0;
            while (w < 64 && (span >> w) != 0) ++w;
            if (w > 48) throw Unsupported("a field spans more than 48 bits in this batch");
            schema->width[f] = static_cast<uint8_t>(w);
            schema->offset[f] = static_cast<uint16_t>(off);
            schema->base[f] = lo[f];
            off += static_cast<uint32_t>(w);
        }
        schema->words_per_row = (off + 31) / 32;
        if (schema->words_per_row == 0) schema->words_per_row = 1;
        std::memcpy(schema->act_table, table, sizeof(table));
        *n_words = n * schema->words_per_row + 2;
        if (!words) return;
        const uint32_t wpr = schema->words_per_row;
        std::memset(words, 0, (n * wpr + 2) * 4);
        for (uint64_t i = 0; i < n; ++i) {
            fields(i, v);
            uint32_t* row = words + i * wpr;
            for (int f = 0; f < F; ++f) {
                const int w = schema->width[f];
                if (!w) continue;
                const uint64_t x = v[f] - lo[f];
                const uint32_t o = schema->offset[f];
                for (int b = 0; b < w;) {  // write up to 32 bits at a time
                    const uint32_t pos = o + static_cast<uint32_t>(b);
                    const int take = std::min(w - b, 32 - static_cast<int>(pos & 31));
                    const uint32_t bits = static_cast<uint32_t>((x >> b) & ((1ull << take) - 1ull));
                    row[pos >> 5] |= bits << (pos & 31);
                    b += take;
                }
            }
        }
    });
}

// The compact 40-byte encoding the host-buffer predicts ship (stage.hpp):
// bit-packed rows with one fixed schema, so no pass over the batch is needed
// to size the fields. Rows that do not fit report UNSUPPORTED.
extern "C" carma_status carma_pack_features_compact(const carma_feature_row* rows, const int8_t* family,
                                                    int32_t default_family, uint64_t n, carma_bit_schema* schema,
                                                    uint32_t* words) {
    return guarded([&] {
        if (!schema) throw InvalidArg("null argument");
        *schema = compact_schema();
        if (n == 0) return;
        if (!rows || !words) throw InvalidArg("null argument");
        words[n * kCompactWords] = 0;
        words[n * kCompactWords + 1] = 0;
        if (!pack_rows_compact(rows, family, default_family, n, reinterpret_cast<uint64_t*>(words)))
            throw Unsupported("a row does not fit the compact format");
    });
}
