/* carma_gpu.h — C ABI of the B200-native CARMA hot path.
 *
 * Drop-in boundary for the two stages of the reference's data-parallel path
 * (see DESIGN.md §2 and INTEGRATION.md). Plain pointers and sizes only; no
 * C++ or torch types cross this boundary. Every call returns a
 * carma_status; carma_last_error() gives the thread-local message. No
 * exception crosses the boundary and there is no CPU fallback: without a
 * usable sm_100 device every compute entry point fails with
 * CARMA_ERR_CUDA.
 *
 * Stage 1 — GPUMemNet (the reference's k-NN memory-bin classifier):
 *   carma_knn_*    replaces LearnedEstimator::predict / predict_scalar
 *                  (proj/include/carma/estimators.hpp:115, src/estimators.cpp:438-475)
 *                  and estimate_learned (estimators.hpp:140-142,
 *                  src/estimators.cpp:540-551), batched; a handle holds one
 *                  model per ModelFamily like Manager::set_learned_estimators
 *                  (manager.hpp:77) so rows route by family (manager.cpp:91-97).
 * Stage 2 — placement scoring and trace replay:
 *   carma_pick_batch   replaces Manager::eligible_gpus + map_task
 *                      (manager.hpp:82-86, src/manager.cpp:109-245) for a batch of
 *                      independent decisions on GPU snapshots.
 *   carma_replay_*     replaces run_simulation's event loop for many
 *                      independent traces (runner.hpp:49, src/runner.cpp:40-147;
 *                      World::run/step/place/finish world.hpp:73-90; the Manager
 *                      pipeline manager.cpp:247-357) and the per-trace part of
 *                      compute_report (metrics.cpp:16-70) — the engine under
 *                      run_sweep (runner.hpp:72).
 */
#ifndef CARMA_GPU_H
#define CARMA_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum carma_status {
    CARMA_OK = 0,
    CARMA_ERR_INVALID = 1,     /* bad argument / ConfigError, NonPositiveRange, EmptyDataset */
    CARMA_ERR_CUDA = 2,        /* no device, launch or copy failure */
    CARMA_ERR_OVERFLOW = 3,    /* a trace exceeded every state capacity tier */
    CARMA_ERR_FAMILY = 4,      /* FamilyMismatch: no model for a requested family */
    CARMA_ERR_UNSUPPORTED = 5, /* a config outside the kernel's domain (e.g. > 256 simulated GPUs) */
    CARMA_ERR_INCOMPLETE = 6   /* IncompleteRun: a trace could not finish */
} carma_status;

const char* carma_last_error(void);
int carma_version(void);
/* Number of usable sm_100 devices (0 when none). */
int carma_device_count(void);

/* ------------------------------------------------------------ stage 1 */

#define CARMA_FEATURE_DIMS 19
#define CARMA_MAX_K 32
#define CARMA_FAMILIES 3 /* ModelFamily: 0 MLP, 1 CNN, 2 Transformer (task.hpp:30) */
#define CARMA_FAMILY_MLP 0
#define CARMA_FAMILY_CNN 1
#define CARMA_FAMILY_TRANSFORMER 2

/* The FeatureVector summary a prediction consumes (task.hpp:89-100):
 * tallies, activation (cos, sin) and the first / middle / last layer tuples
 * (kind code, activations, params) that scalar_features reads
 * (estimators.cpp:317-342). has_layers = 0 leaves dims 9..17 at zero. */
typedef struct carma_feature_row {
    uint64_t n_linear, n_batchnorm, n_dropout, n_conv;
    uint64_t batch_size, total_params, total_activations;
    double act_cos, act_sin;
    int32_t kind[3];
    int32_t has_layers;
    uint64_t tuple_acts[3];
    uint64_t tuple_params[3];
} carma_feature_row; /* 136 bytes */

typedef struct carma_knn carma_knn;

/* Row formats accepted by carma_knn_predict_device. */
#define CARMA_ROWS_FEATURES 0 /* carma_feature_row[q] */
#define CARMA_ROWS_SCALAR 1   /* double[q][19] raw scalar features */
#define CARMA_ROWS_PACKED 2   /* carma_feature_packed[q] (+ activation table) */

/* Lossless 64-byte packing of a carma_feature_row plus its family, for bulk
 * callers (half the PCIe bytes of the 136-byte row). Eight u64 words:
 *   w0 = total_params      | n_linear   << 48 | n_batchnorm << 56
 *   w1 = total_activations | n_dropout  << 48 | n_conv      << 56
 *   w2 = tuple_acts[0]     | (batch & 0xffff) << 48
 *   w3 = tuple_params[0]   | kind0 << 48 | kind1 << 52 | kind2 << 56
 *                          | has_layers << 60 | act_code << 61
 *   w4 = tuple_acts[1]     | family << 48
 *   w5 = tuple_params[1]   | (batch >> 16) << 48
 *   w6 = tuple_acts[2]
 *   w7 = tuple_params[2]
 * 48-bit counts, 8-bit tallies, 4-bit kinds, 32-bit batch; (act_cos,
 * act_sin) is entry act_code of an 8-entry table passed with the batch.
 * carma_pack_features reports CARMA_ERR_UNSUPPORTED for rows that do not
 * fit; callers then use the 136-byte format. */
typedef struct carma_feature_packed {
    uint64_t w[8];
} carma_feature_packed;

/* Packs n rows (family per row, nullable -> default_family) and builds the
 * activation table act_table[16] = {cos0, sin0, cos1, sin1, ...}. */
carma_status carma_pack_features(const carma_feature_row* rows, const int8_t* family,
                                 int32_t default_family, uint64_t n, double* act_table,
                                 carma_feature_packed* out);

/* Frame-of-reference bit packing for bulk transfers: per batch, each field is
 * stored as (value - base) in `width` bits at bit `offset` of a row of
 * words_per_row little-endian u32 words; constant fields cost 0 bits. Field
 * order: 0 n_linear, 1 n_batchnorm, 2 n_dropout, 3 n_conv, 4 batch_size,
 * 5 total_params, 6 total_activations, 7 activation code, 8-10 kind[0..2],
 * 11 has_layers, 12 tuple_acts[0], 13 tuple_params[0], 14 tuple_acts[1],
 * 15 tuple_params[1], 16 tuple_acts[2], 17 tuple_params[2], 18 family.
 * Every field must fit in 48 bits after the base is removed. */
#define CARMA_ROWS_BITPACKED 3
#define CARMA_BIT_FIELDS 19
typedef struct carma_bit_schema {
    uint32_t words_per_row;
    uint32_t reserved;
    uint8_t width[CARMA_BIT_FIELDS + 1];
    uint16_t offset[CARMA_BIT_FIELDS + 1];
    uint64_t base[CARMA_BIT_FIELDS + 1];
    double act_table[16];
} carma_bit_schema;

/* Builds the schema for n rows (pass words == NULL to size: *n_words gets
 * n * words_per_row + 2 padding words), then encodes the rows. */
carma_status carma_pack_features_bits(const carma_feature_row* rows, const int8_t* family,
                                      int32_t default_family, uint64_t n, carma_bit_schema* schema,
                                      uint32_t* words, uint64_t* n_words);
/* The fixed 40-byte bit-packed encoding (ten words per row, every base 0;
 * field widths: 32 for the six tuple counts and the two totals, 8 per layer
 * tally, 12 batch, 3 activation code, 4 per kind, 1 has_layers, 4 family with
 * 15 = none) that carma_knn_predict / carma_nn_predict ship for chunks whose
 * rows all fit. Fills *schema; words holds n * 10 + 2 (padding) words.
 * CARMA_ERR_UNSUPPORTED if a row does not fit. */
carma_status carma_pack_features_compact(const carma_feature_row* rows, const int8_t* family,
                                         int32_t default_family, uint64_t n, carma_bit_schema* schema,
                                         uint32_t* words);

carma_status carma_knn_create(int device, carma_knn** out);
carma_status carma_knn_destroy(carma_knn* h);
/* Installs the model of one family: min/max bounds, the n normalised training
 * points (row-major n x 19, training order) and their labels, as produced by
 * train_learned_estimator (estimators.cpp:344-395). */
carma_status carma_knn_set_model(carma_knn* h, int32_t family, const double* lo,
                                 const double* hi, const double* points,
                                 const int32_t* labels, uint64_t n, uint32_t k,
                                 uint64_t bucket_range);

/* generate_synthetic_dataset(family, n, seed) (estimators.cpp:221-264, with
 * the family's default GenerationBounds, bucket range and SimConstants) on the
 * device, bit-identical to the reference's sequential mt19937_64 generator:
 * rows[i] = extract_features of the i-th feasible sampled architecture,
 * bucket[i] = bucketize(mem), mem[i] = ground_truth_memory (outputs nullable).
 * The _device form takes device buffers and a stream (synchronised once per
 * generation round); the plain form takes host buffers. stats (nullable):
 * the engine words drawn, rows parsed / feasible (rounds may parse past the
 * n-th feasible row), rounds. n = 0 returns INVALID (InvalidBounds). */
typedef struct carma_dataset_stats {
    uint64_t words_generated;
    uint64_t rows_parsed;
    uint64_t rows_accepted;
    uint32_t rounds;
    uint32_t reserved;
} carma_dataset_stats;
carma_status carma_dataset_generate_device(int32_t device, int32_t family, uint64_t n, uint64_t seed,
                                           carma_feature_row* rows, int32_t* bucket, uint64_t* mem, void* stream,
                                           carma_dataset_stats* stats);
carma_status carma_dataset_generate(int32_t device, int32_t family, uint64_t n, uint64_t seed,
                                    carma_feature_row* rows, int32_t* bucket, uint64_t* mem,
                                    carma_dataset_stats* stats);

/* HoldoutReport (estimators.hpp:96-103). */
typedef struct carma_holdout_report {
    double accuracy;
    double macro_f1;
    double underestimate_rate;
    uint64_t train_size;
    uint64_t holdout_size;
} carma_holdout_report;

/* train_learned_estimator (estimators.cpp:344-436) on the device, installing
 * the model for `family`: the dataset (host rows, bucket labels, true bytes as
 * generate_synthetic_dataset returns them) is uploaded once; the seeded split
 * is the host's sequential shuffle (carma_host_split_order); the min/max
 * bounds, the normalised training points, the holdout predictions and the
 * confusion / underestimate counts are computed on the GPU; macro-F1 is summed
 * on the host in the reference's label order. Bit-identical to the CPU fit. */
carma_status carma_knn_train(carma_knn* h, int32_t family, const carma_feature_row* rows,
                             const int32_t* bucket, const uint64_t* mem, uint64_t n, uint64_t seed,
                             uint32_t k, uint64_t bucket_range, carma_holdout_report* report,
                             double* lo_out, double* hi_out, double* points_out, int32_t* labels_out);
/* The optional *_out buffers (nullable) receive the fitted LearnedEstimator
 * state (estimators.hpp:108-133): lo[19], hi[19], points[train_size x 19] and
 * labels[train_size] in training order (train_size = max(1, 7n/10)). */

/* LearnedEstimator::load (estimators.cpp:503-538) into the bank: installs a
 * "carma-knn-estimator/v1" snapshot (the JSON text LearnedEstimator::save
 * writes, estimators.cpp:481-501) as the model of its family. The family and
 * the stored holdout report are returned (both nullable). Snapshot errors
 * return INVALID with the reference's message. */
carma_status carma_knn_load_snapshot(carma_knn* h, const char* json, uint64_t len, int32_t* family_out,
                                     carma_holdout_report* holdout_out);
carma_status carma_knn_load_snapshot_file(carma_knn* h, const char* path, int32_t* family_out,
                                          carma_holdout_report* holdout_out);

/* Host-buffer batch predict (the drop-in for estimate_learned over q rows).
 * family: per-row family (nullable: every row is default_family).
 * bucket_out[i] = LearnedEstimator::predict; bytes_out[i] = (bucket+1)*range.
 * Rows whose family has no model get bucket -1 and bytes UINT64_MAX
 * (FamilyMismatch -> no estimate, manager.cpp:99-105). Either output may be
 * NULL. H2D, compute and D2H are pipelined in chunks on the handle's
 * streams. */
carma_status carma_knn_predict(carma_knn* h, const carma_feature_row* rows,
                               const int8_t* family, int32_t default_family, uint64_t q,
                               int32_t* bucket_out, uint64_t* bytes_out);
/* Same over packed rows; the family of each row is in the packing. */
carma_status carma_knn_predict_packed(carma_knn* h, const carma_feature_packed* rows,
                                      const double* act_table, uint64_t q,
                                      int32_t* bucket_out, uint64_t* bytes_out);
/* Same over bit-packed rows (the family of each row is in the packing). */
carma_status carma_knn_predict_bitpacked(carma_knn* h, const uint32_t* words,
                                         const carma_bit_schema* schema, uint64_t q,
                                         int32_t* bucket_out, uint64_t* bytes_out);
/* Schema used by CARMA_ROWS_BITPACKED device calls. */
carma_status carma_knn_set_bit_schema(carma_knn* h, const carma_bit_schema* schema);
/* Same over raw 19-feature rows (predict_scalar). */
carma_status carma_knn_predict_scalar(carma_knn* h, const double* raw, const int8_t* family,
                                      int32_t default_family, uint64_t q,
                                      int32_t* bucket_out, uint64_t* bytes_out);
/* Device-resident predict: all pointers are device pointers on the handle's
 * device; runs on `stream` (a cudaStream_t, NULL = the handle's stream).
 * topk_d2 / topk_idx (nullable, q x k) receive the k nearest (d2, training
 * index) pairs in ascending (d2, index) order for parity checks. */
carma_status carma_knn_predict_device(carma_knn* h, const void* rows, int32_t format,
                                      const int8_t* family, int32_t default_family,
                                      uint64_t q, int32_t* bucket_out, uint64_t* bytes_out,
                                      double* topk_d2, int64_t* topk_idx, void* stream);
/* Activation table (host, 16 doubles) used by CARMA_ROWS_PACKED device calls. */
carma_status carma_knn_set_act_table(carma_knn* h, const double* act_table);
/* Kernel statistics of the last predict: launches and the number of exact
 * fp64 (query, point) distance evaluations performed. */
carma_status carma_knn_last_stats(carma_knn* h, uint64_t* launches, uint64_t* evaluations);
/* Same, plus the fp32 pre-filter evaluations (0 on the exact-only path). */
/* Bytes the last host-buffer predict copied host -> device (rows travel as
 * 64-byte packed rows or as they are, chunk by chunk; see stage.hpp). */
carma_status carma_knn_last_h2d_bytes(carma_knn* h, uint64_t* bytes);
carma_status carma_knn_last_work(carma_knn* h, uint64_t* launches, uint64_t* fp64_evals,
                                 uint64_t* fp32_evals);
/* Search path: 0 auto (fp32 pre-filter whenever every installed model has
 * <= 16 active dims), 1 exact fp64 blocks only, 2 fp32 pre-filter. Both
 * paths return identical, exact results. */
carma_status carma_knn_set_path(carma_knn* h, int32_t path);
/* CUDA-event timing of the last carma_knn_predict_device on its stream:
 * the knn_search kernel alone and the whole 4-kernel pipeline (ms). */
carma_status carma_knn_last_timing(carma_knn* h, double* search_ms, double* pipeline_ms);

/* ------------------------------------------ stage 1, neural GPUMemNet */
/* The paper's GPUMemNet MLP ensemble (fig. "MLP
 * Ensemble"): E members, each 1..8 hidden ReLU layers of <= 8 neurons
 * (batch norm folded into the linear layers), a linear head over C memory
 * bins, a softmax per member, the probabilities averaged over the members;
 * the predicted bin is the argmax (ties to the larger bin, as the k-NN vote,
 * estimators.cpp:463-474) and bytes = (bin + 1) * bucket_range
 * (estimate_learned, estimators.cpp:540-551). The reference artifact ships
 * the k-NN instead: this estimator is the north
 * star's neural one, an extra EstimatorKind next to carma_knn_*. It plugs
 * into Manager::make_estimate (manager.cpp:80-107) through the same
 * per-family bank and the same FamilyMismatch convention.
 *
 * Input transform per feature d of scalar_features (estimators.cpp:317-342),
 * in fp32 on x_d = fp32(raw_d):  t_d = log1p(max(x_d, 0)) if bit d of
 * log_mask is set, else x_d;  z_d = (t_d - shift_d) * scale_d.
 * Weights are bf16 values (rounded to nearest-even on install); biases,
 * activations, logits and probabilities are fp32. */
#define CARMA_NN_MAX_MEMBERS 8
#define CARMA_NN_MAX_DEPTH 8
#define CARMA_NN_MAX_WIDTH 8
#define CARMA_NN_MAX_CLASSES 48
typedef struct carma_nn_spec {
    uint32_t members;      /* E, 1..8 */
    uint32_t classes;      /* C, 2..48 */
    uint64_t bucket_range; /* bytes per bin */
    uint32_t depth[CARMA_NN_MAX_MEMBERS];                      /* hidden layers, 1..8 */
    uint32_t width[CARMA_NN_MAX_MEMBERS][CARMA_NN_MAX_DEPTH]; /* hidden widths, 1..8 */
    uint32_t log_mask;
    uint32_t arch; /* CARMA_NN_ARCH_MLP or CARMA_NN_ARCH_TRANSFORMER */
    float shift[CARMA_FEATURE_DIMS];
    float scale[CARMA_FEATURE_DIMS];
} carma_nn_spec;
#define CARMA_NN_ARCH_MLP 0
#define CARMA_NN_ARCH_TRANSFORMER 1
/* MLP parameters (fp32, n_params values): member by member, layer by layer,
 * W_l [width_l x in_l] row-major then b_l [width_l], with in_0 = 19 and
 * in_l = width_{l-1}; then the head W [C x width_last] and b [C].
 *
 * Transformer ensemble (arch = 1; depth[e] = encoder layers
 * 1..4, width[e][0] = d in {4, 6}): tokens are the three layer tuples
 * z[9..11], z[12..14], z[15..17]; per member: embedding W [d x 3], b [d]
 * (ReLU), positional encodings [3 x d]; per encoder layer (post-LN, one
 * head, scores / sqrt(d), LayerNorm eps 1e-5): Wq [d x d], bq, Wk, bk, Wv,
 * bv, Wo, bo, ln1 gain [d], bias [d], W1 [4 x d], b1 [4] (ReLU), W2 [d x 4],
 * b2 [d], ln2 gain, bias; then mean pooling over the tokens, concatenated
 * with the auxiliary features z[0..8], z[18]: H1 [8 x (d + 10)], b [8]
 * (ReLU), H2 [C x 8], b [C]. Transformer weights stay fp32 (CUDA cores). */
uint64_t carma_nn_param_count(const carma_nn_spec* spec);

typedef struct carma_nn carma_nn;
/* Bytes the last host-buffer carma_nn_predict copied host -> device. */
carma_status carma_nn_last_h2d_bytes(carma_nn* h, uint64_t* bytes);
carma_status carma_nn_create(int device, carma_nn** out);
carma_status carma_nn_destroy(carma_nn* h);
carma_status carma_nn_set_model(carma_nn* h, int32_t family, const carma_nn_spec* spec,
                                const float* params, uint64_t n_params);
carma_status carma_nn_set_act_table(carma_nn* h, const double* act_table);
/* MLP ensembles: 0 = auto (the CUDA-core kernel, mlp_ffma: fp32 FFMA, thread
 * per row), 1 = the tcgen05 kernel (nn_ensemble: block-diagonal bf16 GEMMs),
 * 2 = CUDA cores. Results agree within the 1e-3 logit bar; both are tested.
 * Transformer ensembles always run on the CUDA cores. */
carma_status carma_nn_set_path(carma_nn* h, int32_t path);
carma_status carma_nn_set_bit_schema(carma_nn* h, const carma_bit_schema* schema);
/* Device-resident predict (formats as carma_knn_predict_device). probs
 * (nullable, q x CARMA_NN_MAX_CLASSES fp32) receives the ensemble's mean
 * probabilities, logits (nullable, q x CARMA_NN_MAX_MEMBERS x
 * CARMA_NN_MAX_CLASSES fp32) each member's logits; entries past the row's
 * model E / C are left untouched. Rows whose family has no model get bin -1
 * and bytes UINT64_MAX. */
carma_status carma_nn_predict_device(carma_nn* h, const void* rows, int32_t format,
                                     const int8_t* family, int32_t default_family, uint64_t q,
                                     int32_t* bucket_out, uint64_t* bytes_out, float* probs,
                                     float* logits, void* stream);
/* Host-buffer predicts, chunked H2D / compute / D2H on the handle's streams. */
carma_status carma_nn_predict(carma_nn* h, const carma_feature_row* rows, const int8_t* family,
                              int32_t default_family, uint64_t q, int32_t* bucket_out,
                              uint64_t* bytes_out);
carma_status carma_nn_predict_bitpacked(carma_nn* h, const uint32_t* words,
                                        const carma_bit_schema* schema, uint64_t q,
                                        int32_t* bucket_out, uint64_t* bytes_out);
/* CUDA-event time of the last carma_nn_predict_device (ms): the ensemble
 * kernels alone and the whole call (family partition included), plus the
 * number of kernel launches and of tcgen05 MMA instructions issued. */
carma_status carma_nn_last_timing(carma_nn* h, double* kernel_ms, double* call_ms,
                                  uint64_t* launches, uint64_t* mmas);

/* ------------------------------------------------------------ stage 2 */

#define CARMA_POLICY_EXCLUSIVE 0 /* manager.hpp:15 */
#define CARMA_POLICY_RR 1
#define CARMA_POLICY_MAGM 2
#define CARMA_POLICY_LUG 3
#define CARMA_POLICY_MUG 4
#define CARMA_MODE_STREAMS 0 /* gpu.hpp:14 */
#define CARMA_MODE_MPS 1
#define CARMA_MODE_MIG 2 /* replay: yes; carma_pick_batch: UNSUPPORTED (views carry no instances) */
#define CARMA_NO_ESTIMATE UINT64_MAX
#define CARMA_MAX_GPUS 64 /* carma_pick_batch views per decision */
/* Simulated GPUs per replay config: <= 64 run in the shared-memory tiers,
 * 65..256 in a global-memory tier (GPU ids fit the packed 8-bit fields). */
#define CARMA_MAX_REPLAY_GPUS 256
/* GPUs one task may request (TaskSpec::gpus_requested) in the replay. */
#define CARMA_MAX_TASK_GPUS 8

#define CARMA_MAX_MIG 8

/* PolicyConfig (manager.hpp:29-37) + SimConstants (memory_model.hpp:11-29). */
typedef struct carma_replay_config {
    int32_t policy;
    int32_t mode;
    int32_t gpu_count;
    int32_t rr_apply_preconditions;
    double max_smact;
    uint64_t min_free; /* PreconditionSet::min_free_mem; 0 == unset */
    double monitor_window;
    uint64_t gpu_capacity;
    uint64_t alloc_block;
    double p_idle_w, p_max_w, p_boost_w, boost_threshold;
    double oom_startup_delay;
    /* CARMA_MODE_MIG only: every GPU's static instance table (GpuDevice ctor,
     * gpu.cpp:26-54; RunConfig::mig_instances, runner.hpp:23), filled by
     * carma_mig_layout (carma_host.h). Instance i owns allocation blocks
     * [mig_base[i], mig_base[i] + mig_blocks[i]) and compute share
     * mig_fraction[i]. */
    int32_t mig_count; /* instances per GPU; 0 outside MIG mode */
    int32_t mig_reserved;
    double mig_fraction[CARMA_MAX_MIG];
    uint16_t mig_base[CARMA_MAX_MIG];
    uint16_t mig_blocks[CARMA_MAX_MIG];
    /* RunConfig::enable_timeline / sample_interval (runner.hpp:32-33): > 0
     * schedules sample ticks from the first trace row's submit time every
     * sample_interval seconds while any submitted task is unfinished
     * (runner.cpp:80-93). Ticks are events (energy-integration breakpoints),
     * so they change the run exactly as in the reference. 0 = off. */
    double sample_interval;
    /* RunConfig::enable_event_log (bit 0, World::log_event, world.cpp:94-153)
     * and verbose_decisions (bit 1, the decision log, manager.cpp:298-318):
     * records are written per job (carma_replay_plan_log) and formatted by
     * the host. They do not change the run. */
    int32_t log_flags;
    int32_t log_reserved;
    /* CARMA_MODE_MIG: the same instance table in bytes (carma_mig_layout
     * fills both); the replay uses it on byte-granular devices (alloc_block
     * = 0 or a capacity that is not a block multiple, where instance
     * boundaries need not fall on blocks). */
    uint64_t mig_base_bytes[CARMA_MAX_MIG];
    uint64_t mig_cap_bytes[CARMA_MAX_MIG];
} carma_replay_config; /* 344 bytes */

/* One materialised task (TaskSpec, task.hpp:63-80) as the replay sees it. */
typedef struct carma_task {
    double submit;     /* submit_time */
    double work;       /* total_work() = epochs * nominal_epoch_time */
    double demand;     /* smact_demand */
    uint64_t true_mem; /* true_mem_bytes */
    uint64_t estimate; /* make_estimate(task).bytes, CARMA_NO_ESTIMATE for none */
    uint32_t gpus;     /* gpus_requested */
    uint32_t rank;     /* rank of the task id in std::string order within its trace */
} carma_task;          /* 48 bytes */

/* TaskTiming (manager.hpp:39-46) + TaskRun placement (world.hpp:32-44). */
typedef struct carma_task_result {
    double first_attempt;  /* dispatch_attempts.front(), -1 when none */
    double final_dispatch; /* -1 when never placed */
    double complete;       /* -1 when never completed */
    double first_crash;    /* crash_times.front(), -1 when none */
    double last_crash;     /* crash_times.back(), -1 when none */
    double executed;       /* TaskRun::executed_integral */
    uint32_t attempts;     /* dispatch_attempts.size() */
    uint32_t ooms;         /* TaskTiming::oom_count */
    int16_t gpu[2];        /* TaskRun::gpu_ids, -1 padded */
    uint32_t reserved;
} carma_task_result; /* 64 bytes */

/* RunReport scalars (metrics.hpp:44-57) + replay counters. */
typedef struct carma_trace_result {
    double trace_total_time;
    double avg_wait, avg_exec, avg_jct;
    double energy_mj;
    double first_submit, last_complete;
    double end_time; /* World::now() when the queue ran dry */
    int32_t oom_count;
    int32_t status;  /* carma_status of this trace */
    uint64_t events; /* World::step pops */
} carma_trace_result; /* 80 bytes */

typedef struct carma_gpu_result {
    double energy_j;   /* after the overshoot correction (runner.cpp:117-120) */
    double mean_smact; /* windowed_smact(last_complete, span) (runner.cpp:135-137) */
    uint64_t peak_used;
    uint64_t smact_steps; /* size of the SMACT step history */
} carma_gpu_result;      /* 32 bytes */

/* A replay job: one trace under one config. Task results of job j are laid
 * out at sum_{i<j} n_tasks(job_i); GPU results at sum_{i<j} gpu_count(job_i). */
typedef struct carma_replay_job {
    uint32_t trace;
    uint32_t config;
} carma_replay_job;

typedef struct carma_replay_plan carma_replay_plan;

/* Uploads configs, tasks (trace t = tasks[trace_offsets[t] .. trace_offsets[t+1]))
 * and jobs to `device`. want_task_results is ignored (kept for ABI shape):
 * per-task results are always produced on the device; what crosses PCIe is
 * chosen per call in carma_replay_plan_results / carma_replay_batch_mode. */
carma_status carma_replay_plan_create(int device, const carma_replay_config* configs,
                                      uint32_t n_configs, const carma_task* tasks,
                                      const uint64_t* trace_offsets, uint32_t n_traces,
                                      const carma_replay_job* jobs, uint32_t n_jobs,
                                      int32_t want_task_results, carma_replay_plan** out);
/* Overrides every task's estimate with a device array (one u64 per task, same
 * indexing as `tasks`), e.g. the bytes_out of carma_knn_predict_device. */
carma_status carma_replay_plan_set_estimates_device(carma_replay_plan* p, const uint64_t* est);
/* Re-uploads the task array (same shape as at creation) from host memory,
 * e.g. the next sweep's traces; pinned host memory copies asynchronously. */
carma_status carma_replay_plan_upload_tasks(carma_replay_plan* p, const carma_task* tasks);
/* run_sweep's inputs generated on the device (runner.cpp:213-249 without the
 * host loop): trace k * n_seeds + i = generate_trace(mix, seeds[i])
 * (traces.cpp:266-306) materialised (task_from_catalog, traces.cpp:238-254;
 * ids t000-.. so rank = row) with estimates from table k (n_tables tables of
 * one u64 per catalog entry, host memory; NULL = no estimate, n_tables = 1):
 * every estimator persona, learned included, is a function of the catalog
 * entry. mix: CARMA_MIX_T90 (90 tasks) or CARMA_MIX_T60 (60). jobs index those
 * traces as in carma_replay_plan_create. Bit-identical to the host generator. */
carma_status carma_replay_plan_create_generated(int device, const carma_replay_config* configs,
                                                uint32_t n_configs, int32_t mix, const uint64_t* seeds,
                                                uint32_t n_seeds, const uint64_t* entry_estimates,
                                                uint32_t n_tables, const carma_replay_job* jobs,
                                                uint32_t n_jobs, carma_replay_plan** out);
/* The catalog entry of every generated task (int32 per task, host buffer). */
carma_status carma_replay_plan_entries(carma_replay_plan* p, int32_t* entries);
/* The plan's task array as the replay sees it (host buffer, n_tasks). */
carma_status carma_replay_plan_tasks(carma_replay_plan* p, carma_task* tasks);
/* Runs all jobs on the device (inputs resident). stream: cudaStream_t or NULL. */
carma_status carma_replay_plan_run(carma_replay_plan* p, void* stream);
/* One timeline row per GPU per sample tick: World::emit_timeline_row
 * (world.cpp:210-219) before formatting ("%.3f,%d,%.4f,%llu,%.2f"). */
typedef struct carma_timeline_row {
    double t;        /* World::now() */
    double smact;    /* instantaneous_smact() */
    double power_w;  /* power_draw() */
    uint64_t used;   /* used_bytes() */
    int32_t gpu;
    int32_t reserved;
} carma_timeline_row; /* 40 bytes */

#define CARMA_LOG_EVENTS 1
#define CARMA_LOG_DECISIONS 2
#define CARMA_REC_PLACE 0     /* "t=%.3f ev=place task=%s gpus=%zu": gpu = #gpus */
#define CARMA_REC_COMPLETE 1  /* "t=%.3f ev=complete task=%s" */
#define CARMA_REC_OOM 2       /* "t=%.3f ev=alloc_oom gpu=%d task=%s req=%llu free=%llu largest=%llu" */
#define CARMA_REC_DECIDE 3    /* "t=%.3f decide task=%s policy=%s gpu=%d|defer est_bytes=%llu" */

/* One event-log or decision-log line before formatting. */
typedef struct carma_log_record {
    double t;
    uint64_t a;     /* OOM: requested bytes; DECIDE: est_bytes */
    uint64_t b;     /* OOM: free bytes in the allocation range */
    uint64_t c;     /* OOM: largest free run in the range */
    uint32_t task;  /* trace row */
    int16_t gpu;    /* PLACE: GPUs used; OOM: device; DECIDE: first GPU or -1 (defer) */
    uint8_t kind;   /* CARMA_REC_* */
    uint8_t policy; /* DECIDE: policy printed */
} carma_log_record; /* 40 bytes */

/* Device capacity for log records of every job whose config has log_flags
 * set (call before carma_replay_plan_run); extra records are counted. */
carma_status carma_replay_plan_set_log_capacity(carma_replay_plan* p, uint64_t records_per_job);
/* Records of job j in run order (host buffer of cap); *n = produced. */
carma_status carma_replay_plan_log(carma_replay_plan* p, uint32_t job, carma_log_record* recs, uint64_t cap,
                                   uint64_t* n);

/* Device capacity for timeline rows of every job whose config has
 * sample_interval > 0 (call before carma_replay_plan_run). A job that
 * produces more rows keeps running; its extra rows are counted, not stored. */
carma_status carma_replay_plan_set_timeline_capacity(carma_replay_plan* p, uint64_t rows_per_job);
/* Rows of job j (host buffer of cap rows); *n_rows = rows produced (may
 * exceed cap: then only cap were kept). */
carma_status carma_replay_plan_timeline(carma_replay_plan* p, uint32_t job, carma_timeline_row* rows,
                                        uint64_t cap, uint64_t* n_rows);
carma_status carma_replay_plan_results(carma_replay_plan* p, carma_task_result* tasks,
                                       carma_trace_result* traces, carma_gpu_result* gpus);
/* Kernel launches of the last run and the state tier each job finished in. */
carma_status carma_replay_plan_stats(carma_replay_plan* p, uint64_t* launches,
                                     uint64_t* retried_jobs);
/* CUDA-event timing of the last run on the plan's stream: the first-tier
 * replay kernel and the whole run including retries (ms). */
carma_status carma_replay_plan_timing(carma_replay_plan* p, double* kernel_ms, double* run_ms);
carma_status carma_replay_plan_destroy(carma_replay_plan* p);

/* Per-task outcome in compact form (TaskOutcome, metrics.hpp:29-38 inputs). */
typedef struct carma_task_outcome {
    double final_dispatch;
    double complete;
    uint32_t ooms;
    uint32_t attempts;
} carma_task_outcome; /* 24 bytes */

/* Outcome sink: every later run writes each job's per-task outcomes (the
 * layout of carma_replay_plan_outcomes) straight into this pinned host
 * buffer as the job finishes, so the D2H overlaps the jobs still running;
 * NULL detaches it. The buffer must stay valid and pinned while attached. */
carma_status carma_replay_plan_set_outcome_sink(carma_replay_plan* p, carma_task_outcome* host_outcomes);

/* Compact results: per-task outcomes (nullable) + traces + GPUs. */
carma_status carma_replay_plan_outcomes(carma_replay_plan* p, carma_task_outcome* tasks,
                                        carma_trace_result* traces, carma_gpu_result* gpus);

/* One-shot host API: create + run + results + destroy (the run_sweep engine). */
carma_status carma_replay_batch(int device, const carma_replay_config* configs,
                                uint32_t n_configs, const carma_task* tasks,
                                const uint64_t* trace_offsets, uint32_t n_traces,
                                const carma_replay_job* jobs, uint32_t n_jobs,
                                carma_task_result* task_results,
                                carma_trace_result* trace_results,
                                carma_gpu_result* gpu_results);

/* --- batched placement scoring (eligible_gpus + map_task) --- */
typedef struct carma_gpu_view {
    uint64_t total_free;   /* GpuDevice::total_free() */
    double windowed_smact; /* windowed_smact(now, monitor_window) */
    int32_t idle;          /* no residents */
    int32_t reserved;
} carma_gpu_view;

typedef struct carma_pick_request {
    uint64_t estimate; /* CARMA_NO_ESTIMATE for none */
    uint32_t want;     /* gpus_requested (1 or 2; up to 8 in carma_pick_batch_wide) */
    int32_t from_recovery;
} carma_pick_request;

/* n decisions over n x n_gpus views (row-major), each with its own RR cursor
 * (in/out). out_gpus is n x 2 (-1 padded; {-1,-1} = defer). Host buffers. */
carma_status carma_pick_batch(int device, const carma_replay_config* cfg,
                              const carma_gpu_view* views, uint32_t n_gpus,
                              const carma_pick_request* reqs, uint64_t n,
                              int32_t* rr_cursor, int32_t* out_gpus);
/* carma_pick_batch beyond its fast paths: up to 256 GPUs per snapshot and
 * up to 8 GPUs per decision (want in [1, 8]); out_gpus is n x 8 (-1 padded;
 * all -1 = defer). One decision per warp. Host buffers. */
carma_status carma_pick_batch_wide(int device, const carma_replay_config* cfg,
                                   const carma_gpu_view* views, uint32_t n_gpus,
                                   const carma_pick_request* reqs, uint64_t n,
                                   int32_t* rr_cursor, int32_t* out_gpus);
/* Same on device-resident arrays (views, reqs, rr_cursor, out_gpus are device
 * pointers; cfg is host memory), launched on `stream` (cudaStream_t or NULL).
 * want must be 1 or 2 (not checked on the device path). */
carma_status carma_pick_batch_device(int device, const carma_replay_config* cfg,
                                     const carma_gpu_view* views, uint32_t n_gpus,
                                     const carma_pick_request* reqs, uint64_t n,
                                     int32_t* rr_cursor, int32_t* out_gpus, void* stream);

/* ------------------------------------------- one-process multi-device */
/* The run_sweep worker pool (runner.cpp:209-249) over the GPUs of one box:
 * units (rows, replay jobs) are split into contiguous shards balanced by
 * weight, one host thread per device drives its own handle / plan and
 * stream, and each writes its shard's results straight into the caller's
 * output buffers at the shard's offsets (pin them for asynchronous DMA). No
 * collective: nothing is reduced across GPUs. Results are identical to the
 * single-device calls. The first failing shard's status is returned. */

/* bounds[p] .. bounds[p+1] (p < parts): contiguous shards of n units whose
 * weights (NULL: 1 each) are balanced; shard p starts at the first unit whose
 * prefix weight reaches total * p / parts. */
carma_status carma_shard_ranges(const uint64_t* weights, uint64_t n, uint32_t parts, uint64_t* bounds);
/* carma_knn_predict over n_handles handles (one per device; models installed
 * on each), rows sharded evenly. */
carma_status carma_knn_predict_multi(carma_knn* const* handles, uint32_t n_handles,
                                     const carma_feature_row* rows, const int8_t* family,
                                     int32_t default_family, uint64_t q, int32_t* bucket_out,
                                     uint64_t* bytes_out);
/* carma_nn_predict likewise. */
carma_status carma_nn_predict_multi(carma_nn* const* handles, uint32_t n_handles, const carma_feature_row* rows,
                                    const int8_t* family, int32_t default_family, uint64_t q,
                                    int32_t* bucket_out, uint64_t* bytes_out);
/* carma_replay_batch over n_devices devices: jobs sharded by task count, each
 * device replays its shard's traces; outputs laid out as carma_replay_batch's. */
carma_status carma_replay_batch_multi(const int32_t* devices, uint32_t n_devices,
                                      const carma_replay_config* configs, uint32_t n_configs,
                                      const carma_task* tasks, const uint64_t* trace_offsets, uint32_t n_traces,
                                      const carma_replay_job* jobs, uint32_t n_jobs,
                                      carma_task_result* task_results, carma_trace_result* trace_results,
                                      carma_gpu_result* gpu_results);

/* ------------------------------------------------------------ probes */
/* Measured fp64 add/mul issue throughput of `device` (separately rounded
 * ops per second, 1 op = 1 flop): the roofline denominator of the k-NN
 * distance kernel, which is FP64-pipe bound and FMA-free by contract. */
carma_status carma_probe_fp64(int device, double* flops_per_s);
/* Measured packed fp32 FMA throughput (FFMA2, 1 FMA = 2 flops): the roofline
 * denominator of the k-NN fp32 pre-filter pass. */
carma_status carma_probe_fp32(int device, double* flops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* CARMA_GPU_H */
