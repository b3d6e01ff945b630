// Host-side staging for the host-buffer predict calls (carma_knn_predict,
// carma_nn_predict): the 136-byte carma_feature_row batch is re-encoded, by a
// pool of host threads and chunk by chunk, into the 40-byte compact rows
// (fixed-schema bit packing) or the 64-byte lossless packed format
// (include/carma_gpu.h) in pinned staging memory, overlapped with the
// previous chunk's H2D copy and search — the PCIe bytes per row fall from 137
// (row + family) to 40. The activation code indexes the canonical table of
// the 8 registry activations (extract_features' glibc cos / sin of
// 2*pi*i/8, task.cpp:181-189, 301-323); a chunk holding any row the packed
// format cannot carry is sent as raw rows instead.
#pragma once

#include <cstdint>
#include <functional>

#include "../../../include/carma_gpu.h"

namespace carma_b200 {

// The 16-double (cos, sin) table of the 8 registry activations.
const double* canonical_act_table();

// Runs fn(part, parts) on `parts` persistent worker threads (the caller's
// thread takes part 0) and returns when all parts are done.
void host_parallel(uint32_t parts, const std::function<void(uint32_t, uint32_t)>& fn);
uint32_t host_workers();  // parts host_parallel uses for a bulk pass

// Packs rows[0, n) (+ family, nullable -> default_family) into out with
// non-temporal stores; false if some row does not fit the packed format
// (out is then unspecified).
bool pack_rows_canonical(const carma_feature_row* rows, const int8_t* family, int32_t default_family, uint64_t n,
                         carma_feature_packed* out);

// The compact 40-byte encoding of the same rows: ten 32-bit words read as
// CARMA_ROWS_BITPACKED with the fixed schema compact_schema() (every base 0):
//   bits   0- 63  total_params (32) | total_activations (32)
//   bits  64-255  (tuple_acts[k] (32) | tuple_params[k] (32)) for k = 0..2
//   bits 256-319  n_linear, n_batchnorm, n_dropout, n_conv (8 each),
//                 batch_size (12), act code (3), kind[0..2] (4 each),
//                 has_layers (1), family (4; 15 = none)
// false if some row does not fit (callers then try the 64-byte format).
// out holds n * 5 words.
constexpr uint32_t kCompactWords = 10;  // 32-bit words per row
const carma_bit_schema& compact_schema();
bool pack_rows_compact(const carma_feature_row* rows, const int8_t* family, int32_t default_family, uint64_t n,
                       uint64_t* out);

// Whether host-buffer calls try the compact encoding first
// (CARMA_E2E_COMPACT=0 turns it off).
bool compact_rows();

// Whether chunk c of a host-buffer call ships raw rows although it could be
// packed: with pinned inputs the copy engine reads raw rows straight from
// host memory while the pool packs the other chunks, so PCIe and host memory
// bandwidth are both busy (CARMA_E2E_RAW_EVERY = k: every k-th chunk raw;
// 0 = pack every chunk).
bool raw_chunk(uint64_t c, bool inputs_pinned);

}  // namespace carma_b200
