// One-process multi-device driver: the B200 equivalent of run_sweep's worker
// pool (proj/src/runner.cpp:209-249), spread over the GPUs of one box instead
// of host threads (SURVEY §2.1 "Sweep driver", §8(e)).
//
// Estimator rows and replay jobs are independent units, so every call shards
// them into contiguous ranges balanced by weight (rows: 1 each; jobs: their
// task counts), runs one host thread per device — each drives its own
// handle / plan and stream — and each thread writes its shard's results
// straight into the caller's output buffers at the shard's offsets (pinned
// buffers make those device-to-host copies asynchronous DMA). There is no
// cross-device collective: nothing is reduced across GPUs.

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/carma_gpu.h"
#include "status.hpp"

using namespace carma_b200;

namespace {

// bounds[p] .. bounds[p + 1] for p < parts: cut p starts at the first unit
// whose prefix weight reaches total * p / parts (the shard rule of
// paper_2508_19073_b200/dist.py).
void shard_ranges(const uint64_t* weights, uint64_t n, uint32_t parts, uint64_t* bounds) {
    std::vector<double> cum(n + 1, 0.0);
    for (uint64_t i = 0; i < n; ++i) cum[i + 1] = cum[i] + static_cast<double>(weights ? weights[i] : 1);
    const double total = cum[n];
    bounds[0] = 0;
    for (uint32_t p = 1; p < parts; ++p) {
        const double target = total * static_cast<double>(p) / static_cast<double>(parts);
        uint64_t c = static_cast<uint64_t>(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        c = std::min(c, n);
        bounds[p] = std::max(c, bounds[p - 1]);
    }
    bounds[parts] = n;
}

// Runs work(p) on one thread per part; the first failing part's status and
// message are returned on the calling thread.
template <typename F>
void run_parts(uint32_t parts, F&& work) {
    std::vector<carma_status> st(parts, CARMA_OK);
    std::vector<std::string> msg(parts);
    std::vector<std::thread> pool;
    pool.reserve(parts);
    for (uint32_t p = 0; p < parts; ++p)
        pool.emplace_back([&, p] {
            st[p] = work(p);
            if (st[p] != CARMA_OK) msg[p] = carma_last_error();
        });
    for (auto& t : pool) t.join();
    for (uint32_t p = 0; p < parts; ++p)
        if (st[p] != CARMA_OK) throw CarmaFailure(st[p], "shard " + std::to_string(p) + ": " + msg[p]);
}

}  // namespace

extern "C" {

carma_status carma_shard_ranges(const uint64_t* weights, uint64_t n, uint32_t parts, uint64_t* bounds) {
    return guarded([&] {
        if (!bounds || parts == 0) throw InvalidArg("need parts >= 1 and a bounds array");
        shard_ranges(weights, n, parts, bounds);
    });
}

carma_status carma_knn_predict_multi(carma_knn* const* handles, uint32_t n_handles,
                                     const carma_feature_row* rows, const int8_t* family,
                                     int32_t default_family, uint64_t q, int32_t* bucket_out,
                                     uint64_t* bytes_out) {
    return guarded([&] {
        if (!handles || n_handles == 0) throw InvalidArg("no handles");
        if (q && !rows) throw InvalidArg("rows is null");
        std::vector<uint64_t> b(n_handles + 1);
        shard_ranges(nullptr, q, n_handles, b.data());
        run_parts(n_handles, [&](uint32_t p) -> carma_status {
            const uint64_t n = b[p + 1] - b[p];
            if (n == 0) return CARMA_OK;
            return carma_knn_predict(handles[p], rows + b[p], family ? family + b[p] : nullptr, default_family, n,
                                     bucket_out ? bucket_out + b[p] : nullptr, bytes_out ? bytes_out + b[p] : nullptr);
        });
    });
}

carma_status carma_nn_predict_multi(carma_nn* const* handles, uint32_t n_handles, const carma_feature_row* rows,
                                    const int8_t* family, int32_t default_family, uint64_t q,
                                    int32_t* bucket_out, uint64_t* bytes_out) {
    return guarded([&] {
        if (!handles || n_handles == 0) throw InvalidArg("no handles");
        if (q && !rows) throw InvalidArg("rows is null");
        std::vector<uint64_t> b(n_handles + 1);
        shard_ranges(nullptr, q, n_handles, b.data());
        run_parts(n_handles, [&](uint32_t p) -> carma_status {
            const uint64_t n = b[p + 1] - b[p];
            if (n == 0) return CARMA_OK;
            return carma_nn_predict(handles[p], rows + b[p], family ? family + b[p] : nullptr, default_family, n,
                                    bucket_out ? bucket_out + b[p] : nullptr, bytes_out ? bytes_out + b[p] : nullptr);
        });
    });
}

carma_status carma_replay_batch_multi(const int32_t* devices, uint32_t n_devices,
                                      const carma_replay_config* configs, uint32_t n_configs,
                                      const carma_task* tasks, const uint64_t* trace_offsets, uint32_t n_traces,
                                      const carma_replay_job* jobs, uint32_t n_jobs,
                                      carma_task_result* task_results, carma_trace_result* trace_results,
                                      carma_gpu_result* gpu_results) {
    return guarded([&] {
        if (!devices || n_devices == 0) throw InvalidArg("no devices");
        if (!configs || !tasks || !trace_offsets || !jobs) throw InvalidArg("null argument");
        if (n_configs == 0 || n_traces == 0 || n_jobs == 0) throw InvalidArg("empty plan");
        // job weights = task counts; output offsets in global job order
        std::vector<uint64_t> w(n_jobs), task_off(n_jobs + 1, 0), gpu_off(n_jobs + 1, 0);
        for (uint32_t j = 0; j < n_jobs; ++j) {
            if (jobs[j].trace >= n_traces || jobs[j].config >= n_configs) throw InvalidArg("job index out of range");
            w[j] = trace_offsets[jobs[j].trace + 1] - trace_offsets[jobs[j].trace];
            task_off[j + 1] = task_off[j] + w[j];
            gpu_off[j + 1] = gpu_off[j] + static_cast<uint64_t>(std::max(0, configs[jobs[j].config].gpu_count));
        }
        std::vector<uint64_t> b(n_devices + 1);
        shard_ranges(w.data(), n_jobs, n_devices, b.data());
        run_parts(n_devices, [&](uint32_t p) -> carma_status {
            const uint64_t j0 = b[p], j1 = b[p + 1];
            if (j1 == j0) return CARMA_OK;
            // the shard's traces, in first-use order, copied into a compact plan
            std::vector<int64_t> local_of(n_traces, -1);
            std::vector<uint32_t> used;
            std::vector<carma_replay_job> lj(j1 - j0);
            for (uint64_t j = j0; j < j1; ++j) {
                const uint32_t t = jobs[j].trace;
                if (local_of[t] < 0) {
                    local_of[t] = static_cast<int64_t>(used.size());
                    used.push_back(t);
                }
                lj[j - j0] = {static_cast<uint32_t>(local_of[t]), jobs[j].config};
            }
            std::vector<uint64_t> loff(used.size() + 1, 0);
            for (size_t i = 0; i < used.size(); ++i)
                loff[i + 1] = loff[i] + trace_offsets[used[i] + 1] - trace_offsets[used[i]];
            std::vector<carma_task> lt(loff.back());
            for (size_t i = 0; i < used.size(); ++i)
                std::memcpy(lt.data() + loff[i], tasks + trace_offsets[used[i]],
                            (loff[i + 1] - loff[i]) * sizeof(carma_task));
            return carma_replay_batch(devices[p], configs, n_configs, lt.data(), loff.data(),
                                      static_cast<uint32_t>(used.size()), lj.data(), static_cast<uint32_t>(lj.size()),
                                      task_results ? task_results + task_off[j0] : nullptr,
                                      trace_results ? trace_results + j0 : nullptr,
                                      gpu_results ? gpu_results + gpu_off[j0] : nullptr);
        });
    });
}

}  // extern "C"
