/* TEST INFRASTRUCTURE ONLY — the CPU restatement of the CARMA hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker. It restates, in plain C++ with
 * simple containers, the reference algorithm for:
 *   oracle_knn_predict   LearnedEstimator::predict_scalar + estimate_learned
 *                        (proj/src/estimators.cpp:438-475, :540-551)
 *   oracle_replay        run_simulation's event loop: World (world.cpp:31-186),
 *                        Manager (manager.cpp:58-357), GpuDevice MPS/streams
 *                        (gpu.cpp:58-274), the runner tail (runner.cpp:97-141)
 *                        and compute_report (metrics.cpp:16-70)
 *   oracle_pick          eligible_gpus + map_task on a given GPU snapshot
 *                        (manager.cpp:109-245)
 * Inputs and outputs use the same flat layouts as include/carma_gpu.h so the
 * GPU path and the oracle run on identical bytes.
 * Parity: pinned against the compiled reference (oracle/_ref) by
 * tests/test_oracle_vs_ref.py and tests/golden/.
 */
#pragma once
#include <stdint.h>

#include "../include/carma_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

int oracle_knn_predict(const double* lo, const double* hi, const double* points,
                       const int32_t* labels, uint64_t n, uint32_t k, uint64_t bucket_range,
                       const double* raw, uint64_t q, int32_t* bucket, uint64_t* bytes,
                       double* topk_d2, int64_t* topk_idx);

/* One trace. tasks: n entries in trace (arrival) order. Returns 0 on success,
 * nonzero when the run cannot complete (IncompleteRun). */
int oracle_replay(const carma_replay_config* cfg, const carma_task* tasks, uint32_t n,
                  carma_task_result* out_tasks, carma_trace_result* out_trace,
                  carma_gpu_result* out_gpus);

/* One placement decision on a GPU snapshot (see carma_pick in carma_gpu.h). */
int oracle_pick(const carma_replay_config* cfg, const carma_gpu_view* gpus, uint32_t n_gpus,
                const carma_pick_request* req, int32_t* rr_cursor, int32_t* out_gpus);

#ifdef __cplusplus
}
#endif
