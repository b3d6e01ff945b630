/* carma_host.h — host-side provisioning around the GPU hot path.
 *
 * The callers and data formats on either side of include/carma_gpu.h:
 * trace generation / `#carma-trace v1` I/O / materialisation
 * (proj/src/traces.cpp:238-379), synthetic architecture datasets and k-NN
 * fitting (proj/src/estimators.cpp:221-436), featurisation
 * (proj/src/task.cpp:301-323, estimators.cpp:317-342) and the analytic
 * estimator personas (estimators.cpp:34-61). Pure host code (C++ in
 * paper_2508_19073_b200/csrc/host/), bit-identical to the reference's
 * outputs; none of it is on the GPU hot path.
 */
#ifndef CARMA_HOST_H
#define CARMA_HOST_H

#include "carma_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

#define CARMA_MIX_T90 0
#define CARMA_MIX_T60 1

#define CARMA_EST_NONE 0 /* EstimatorKind, manager.hpp:19 */
#define CARMA_EST_ORACLE 1
#define CARMA_EST_ANALYTICAL 2
#define CARMA_EST_STATIC_GRAPH 3
#define CARMA_EST_LEARNED 4

int carma_host_catalog_size(void);
/* Catalog row i: key (NUL-terminated into key[cap]), family, gpus, batch. */
carma_status carma_host_catalog_entry(int i, char* key, int cap, int32_t* family,
                                      uint64_t* gpus, uint64_t* batch, double* mem_gib);

/* Trace rows: submit time, catalog index, epochs. cap = capacity of arrays. */
carma_status carma_host_generate_trace(int32_t mix, uint64_t seed, double* submit,
                                       int32_t* entry, uint64_t* epochs, uint64_t cap,
                                       uint64_t* n_out);
/* n rows drawn uniformly over the whole catalog with exponential gaps of the
 * given mean (the single large-trace workload). */
carma_status carma_host_generate_uniform_trace(uint64_t n, double mean_gap, uint64_t seed,
                                               double* submit, int32_t* entry,
                                               uint64_t* epochs);
carma_status carma_host_save_trace(const char* path, uint64_t seed, const char* mix,
                                   const double* submit, const int32_t* entry,
                                   const uint64_t* epochs, uint64_t n);
/* Two-phase: call with submit == NULL to get the row count in *n_out. */
carma_status carma_host_load_trace(const char* path, double* submit, int32_t* entry,
                                   uint64_t* epochs, uint64_t cap, uint64_t* n_out);

/* materialize_trace: per row the replay task (estimate = CARMA_NO_ESTIMATE,
 * rank = lexicographic rank of the "t%03zu-<key>" id), optional feature rows
 * of the catalog architecture and family codes. */
carma_status carma_host_materialize(const double* submit, const int32_t* entry,
                                    const uint64_t* epochs, uint64_t n, carma_task* tasks,
                                    carma_feature_row* features, int8_t* family);
/* Estimator personas oracle / analytical / static_graph / none
 * (estimators.cpp:34-61, manager.cpp:80-107) written into tasks[i].estimate.
 * CARMA_EST_LEARNED is not handled here: use carma_knn_predict. */
carma_status carma_host_estimates(int32_t kind, uint64_t safety_margin, const int32_t* entry,
                                  uint64_t n, carma_task* tasks);

/* generate_synthetic_dataset rows as feature rows + labels + true bytes. */
carma_status carma_host_dataset(int32_t family, uint64_t n, uint64_t seed,
                                carma_feature_row* rows, int32_t* bucket, uint64_t* mem);
/* train_learned_estimator's fit on generate_synthetic_dataset(family, samples,
 * seed): bounds, normalised points (cap rows), labels, and the dataset row
 * indices of the 30% holdout (cap rows, *n_holdout). */
carma_status carma_host_fit(int32_t family, uint64_t samples, uint64_t seed, uint32_t k,
                            double* lo, double* hi, double* points, int32_t* labels,
                            uint64_t cap, uint64_t* n_out, uint64_t* bucket_range,
                            uint64_t* holdout_rows, uint64_t* n_holdout);
/* The MIG instance table of GpuDevice's constructor (gpu.cpp:26-54) for
 * cfg->gpu_capacity / cfg->alloc_block, written into cfg->mig_*. n = 0 uses
 * the reference default {0.5, 0.5}. ConfigError cases return INVALID; more
 * than CARMA_MAX_MIG instances or a table that is not block aligned return
 * UNSUPPORTED. */
carma_status carma_mig_layout(const double* fractions, uint32_t n, carma_replay_config* cfg);
/* The seeded 70/30 split of train_learned_estimator (estimators.cpp:355-361):
 * order[n] = shuffled row indices, *train_n = max(1, 7n/10). */
carma_status carma_host_split_order(uint64_t n, uint64_t seed, uint64_t* order, uint64_t* train_n);
/* The fitted state of a LearnedEstimator snapshot (estimators.cpp:481-538):
 * family, k, bucket_range, seed, lo[19], hi[19], holdout; points[n x 19] and
 * labels[n] when non-NULL (capacity >= n). *n = the stored point count. Every
 * output pointer is nullable. */
carma_status carma_host_parse_snapshot(const char* json, uint64_t len, int32_t* family, uint64_t* k,
                                       uint64_t* bucket_range, uint64_t* seed, double* lo, double* hi,
                                       double* points, int32_t* labels, uint64_t capacity, uint64_t* n,
                                       carma_holdout_report* holdout);
/* Test hook: compares the device trace generator's log1p (glibc's own
 * algorithm, csrc/cuda/glibc_log1p.cuh, built for the host) with the C
 * library's log1p on n pseudo-random inputs; *mismatches = differing results. */
carma_status carma_host_check_log1p(uint64_t n, uint64_t seed, uint64_t* mismatches);
/* scalar_features for n feature rows -> n x 19 doubles. */
carma_status carma_host_scalar_features(const carma_feature_row* rows, uint64_t n, double* out);

/* Self-check of the device dataset generator's mt19937_64 jump-ahead tables
 * (characteristic polynomial by Berlekamp-Massey, x^(156 2^(13+b)) mod P): the
 * jumped window vs stepping the recurrence; *mismatches = differing words. */
carma_status carma_host_check_mt_jump(uint64_t seed, int32_t b, uint64_t* mismatches);

#ifdef __cplusplus
}
#endif
#endif /* CARMA_HOST_H */
