// Device-side sweep inputs (tracegen.cu): generate_trace + materialisation.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/carma_gpu.h"

namespace carma_b200 {

uint32_t trace_rows(int32_t mix);  // tasks per generated trace (t90: 90, t60: 60)
uint32_t catalog_size();
// Trace (table k, seed i) = generate_trace(mix, seeds[i]) materialised into
// tasks[(k * n_seeds + i) * T ..], estimates from tables[k * catalog_size() + entry]
// (d_tables nullable: no estimate); d_entries (nullable) gets the catalog entries.
void launch_generate_traces(int32_t mix, const uint64_t* d_seeds, uint32_t n_seeds, const uint64_t* d_tables,
                            uint32_t n_tables, carma_task* d_tasks, int32_t* d_entries, cudaStream_t s);

}  // namespace carma_b200
