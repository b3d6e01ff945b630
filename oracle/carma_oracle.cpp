// TEST INFRASTRUCTURE ONLY — CPU restatement of the CARMA hot path.
// See carma_oracle.h for scope and rules. Each block cites the reference
// lines it restates. Deliberately written with the reference's own data
// shapes (segment lists, full SMACT step history, ordered sets, a binary
// heap of events) rather than the GPU kernel's (bitmaps, rings, running
// integrals), so the parity tests compare two independent implementations.
// Compiled with -ffp-contract=off: every product/sum is rounded separately,
// as in the reference build.

#include "carma_oracle.h"

#include <algorithm>
#include <cmath>
#include <deque>
#include <limits>
#include <map>
#include <queue>
#include <set>
#include <vector>

namespace {

// ----------------------------------------------------------- stage 1
// estimators.cpp:438-475
int predict_one(const double* lo, const double* hi, const double* points, const int32_t* labels,
                uint64_t n, uint32_t k, const double* raw, double* topk_d2, int64_t* topk_idx) {
    double q[19];
    for (int d = 0; d < 19; ++d) q[d] = hi[d] > lo[d] ? (raw[d] - lo[d]) / (hi[d] - lo[d]) : 0.0;
    std::vector<std::pair<double, uint64_t>> dist(n);
    for (uint64_t i = 0; i < n; ++i) {
        double d2 = 0.0;
        for (int d = 0; d < 19; ++d) {
            double diff = points[i * 19 + d] - q[d];
            if (d == 18) diff *= 64.0;
            d2 += diff * diff;
        }
        dist[i] = {d2, i};
    }
    const uint64_t kk = std::min<uint64_t>(k, n);
    std::partial_sort(dist.begin(), dist.begin() + static_cast<std::ptrdiff_t>(kk), dist.end());
    std::map<int, uint64_t> votes;
    for (uint64_t i = 0; i < kk; ++i) {
        votes[labels[dist[i].second]]++;
        if (topk_d2) topk_d2[i] = dist[i].first;
        if (topk_idx) topk_idx[i] = static_cast<int64_t>(dist[i].second);
    }
    int best = 0;
    uint64_t best_votes = 0;
    for (const auto& [label, count] : votes)
        if (count > best_votes || (count == best_votes && label > best)) {
            best = label;
            best_votes = count;
        }
    return best;
}

// ----------------------------------------------------------- stage 2
enum Kind { ARRIVAL = 0, WINDOW = 1, COMPLETION = 2, CRASH = 3 };

struct Event {
    double t;
    uint64_t seq;
    int kind;
    int task;
    uint64_t gen;
};
struct Later {
    bool operator()(const Event& a, const Event& b) const {
        if (a.t != b.t) return a.t > b.t;
        return a.seq > b.seq;
    }
};

struct Seg {
    uint64_t off, size;
    bool used;
};

struct Resident {
    int id;
    double demand;
    int inst;  // MIG instance; 0 outside MIG mode (gpu.hpp:43-47)
};

struct Gpu {
    std::vector<Seg> segs;
    std::vector<Resident> residents;  // insertion order
    std::vector<std::pair<double, double>> steps;
    double energy = 0.0;
    uint64_t peak = 0;
    uint64_t capacity = 0;
};

struct Run {
    std::vector<int> gpus;
    std::vector<int> insts;  // MIG instance per entry of gpus
    std::vector<uint64_t> region_off, region_size;
    double remaining = 0.0, rate = 0.0, last_update = 0.0, executed = 0.0;
    uint64_t gen = 0;
    bool resident = false, completed = false, exists = false;
};

struct Sim {
    const carma_replay_config& c;
    const carma_task* tasks;
    uint32_t n;
    std::vector<Gpu> gpu;
    std::vector<Run> run;
    std::priority_queue<Event, std::vector<Event>, Later> pq;
    uint64_t next_seq = 0;
    double now = 0.0;
    uint64_t events = 0;
    uint64_t max_events = 0;
    bool collect = false;
    uint32_t arrivals_seen = 0;
    // manager
    std::deque<int> main_q, recovery_q;
    int rr_cursor = 0, oom_count = 0;
    double deadline = 0.0;
    carma_task_result* out;
    // capacity statistics (oracle_replay_stats)
    uint64_t st_heap = 0, st_resident = 0, st_res_gpu = 0, st_window = 0, st_rq = 0;
    void sample_stats() {
        { const int64_t dyn = static_cast<int64_t>(pq.size()) - (static_cast<int64_t>(n) - arrivals_seen); st_heap = std::max<uint64_t>(st_heap, dyn > 0 ? static_cast<uint64_t>(dyn) : 0); }
        uint64_t tot = 0;
        for (const auto& g : gpu) {
            tot += g.residents.size();
            st_res_gpu = std::max<uint64_t>(st_res_gpu, g.residents.size());
            const double begin = std::max(0.0, now - c.monitor_window);
            uint64_t in_window = 0;
            for (const auto& stp : g.steps) in_window += stp.first > begin ? 1 : 0;
            st_window = std::max<uint64_t>(st_window, in_window + 1);
        }
        st_resident = std::max(st_resident, tot);
        st_rq = std::max<uint64_t>(st_rq, recovery_q.size());
    }

    Sim(const carma_replay_config& cfg, const carma_task* t, uint32_t nt, carma_task_result* o)
        : c(cfg), tasks(t), n(nt), gpu(static_cast<size_t>(cfg.gpu_count)), run(nt), out(o) {
        for (auto& g : gpu) {
            g.capacity = c.gpu_capacity;
            g.segs.push_back({0, c.gpu_capacity, false});
        }
    }

    // gpu.cpp:58-65
    uint64_t round_up(uint64_t b) const {
        if (c.alloc_block == 0) return b;
        return (b + c.alloc_block - 1) / c.alloc_block * c.alloc_block;
    }
    uint64_t total_free(const Gpu& g) const {
        uint64_t s = 0;
        for (const auto& x : g.segs)
            if (!x.used) s += x.size;
        return s;
    }
    bool mig() const { return c.mode == CARMA_MODE_MIG; }
    uint64_t inst_base(int i) const { return c.mig_base_bytes[i]; }
    uint64_t inst_cap(int i) const { return c.mig_cap_bytes[i]; }
    // gpu.cpp:72-114
    bool allocate_range(Gpu& g, uint64_t range_begin, uint64_t range_end, uint64_t bytes, uint64_t* off,
                        uint64_t* size) {
        const uint64_t want = round_up(std::max<uint64_t>(bytes, 1));
        for (size_t i = 0; i < g.segs.size(); ++i) {
            Seg s = g.segs[i];
            if (s.used) continue;
            const uint64_t lo = std::max(s.off, range_begin);
            const uint64_t hi = std::min(s.off + s.size, range_end);
            if (lo >= hi) continue;
            if (hi - lo < want) continue;
            // first fit picks the segment; carve from the end facing away
            // from a live neighbour (gpu.cpp:88-97)
            const bool left_used = i > 0 && g.segs[i - 1].used && s.off == lo;
            const bool right_used = i + 1 < g.segs.size() && g.segs[i + 1].used && s.off + s.size == hi;
            const bool tail = left_used && !right_used;
            const uint64_t place = tail ? hi - want : lo;
            std::vector<Seg> rep;
            if (place > s.off) rep.push_back({s.off, place - s.off, false});
            rep.push_back({place, want, true});
            if (place + want < s.off + s.size) rep.push_back({place + want, s.off + s.size - place - want, false});
            g.segs.erase(g.segs.begin() + static_cast<std::ptrdiff_t>(i));
            g.segs.insert(g.segs.begin() + static_cast<std::ptrdiff_t>(i), rep.begin(), rep.end());
            g.peak = std::max(g.peak, g.capacity - total_free(g));
            *off = place;
            *size = want;
            return true;
        }
        return false;
    }
    // gpu.cpp:151-167
    uint64_t instance_free(const Gpu& g, int i) const {
        uint64_t sum = 0;
        for (const auto& x : g.segs) {
            if (x.used) continue;
            const uint64_t lo = std::max(x.off, inst_base(i));
            const uint64_t hi = std::min(x.off + x.size, inst_base(i) + inst_cap(i));
            if (lo < hi) sum += hi - lo;
        }
        return sum;
    }
    bool instance_idle(const Gpu& g, int i) const {
        for (const auto& r : g.residents)
            if (r.inst == i) return false;
        return true;
    }
    // manager.cpp:125-134
    int pick_instance(const Gpu& g, uint64_t need) const {
        for (int i = 0; i < c.mig_count; ++i) {
            if (!instance_idle(g, i)) continue;
            if (instance_free(g, i) < std::max<uint64_t>(need, 1)) continue;
            return i;
        }
        return -1;
    }
    // gpu.cpp:116-135
    void free_region(Gpu& g, uint64_t off, uint64_t size) {
        for (size_t i = 0; i < g.segs.size(); ++i) {
            if (!(g.segs[i].used && g.segs[i].off == off && g.segs[i].size == size)) continue;
            g.segs[i].used = false;
            if (i + 1 < g.segs.size() && !g.segs[i + 1].used) {
                g.segs[i].size += g.segs[i + 1].size;
                g.segs.erase(g.segs.begin() + static_cast<std::ptrdiff_t>(i) + 1);
            }
            if (i > 0 && !g.segs[i - 1].used) {
                g.segs[i - 1].size += g.segs[i].size;
                g.segs.erase(g.segs.begin() + static_cast<std::ptrdiff_t>(i));
            }
            return;
        }
    }
    // gpu.cpp:183-216: effective rate of resident r (MIG: its instance's
    // share; MPS: min(1, 1/sum demand); streams: 1/n).
    double rate_of(const Gpu& g, const Resident& r) const {
        if (mig()) return std::min(1.0, c.mig_fraction[r.inst] / r.demand);
        if (c.mode == CARMA_MODE_MPS) {
            double total = 0.0;
            for (const auto& x : g.residents) total += x.demand;
            return std::min(1.0, 1.0 / total);
        }
        return 1.0 / static_cast<double>(g.residents.size());
    }
    double task_rate(const Gpu& g, int id) const {
        for (const auto& r : g.residents)
            if (r.id == id) return rate_of(g, r);
        return 0.0;
    }
    // gpu.cpp:218-229
    double inst_smact(const Gpu& g) const {
        if (g.residents.empty()) return 0.0;
        double s = 0.0;
        for (const auto& x : g.residents) s += x.demand * rate_of(g, x);
        return std::min(1.0, s);
    }
    // gpu.cpp:231-242
    void record_smact(Gpu& g) {
        const double v = inst_smact(g);
        if (!g.steps.empty()) {
            auto& [t, last] = g.steps.back();
            if (last == v) return;
            if (t == now) {
                last = v;
                return;
            }
        }
        g.steps.push_back({now, v});
    }
    // gpu.cpp:244-267
    double windowed(const Gpu& g, double at, double window) const {
        const double begin = std::max(0.0, at - window);
        const double span = at - begin;
        if (span <= 0.0) return inst_smact(g);
        double integral = 0.0, level = 0.0, cursor = begin;
        for (const auto& [t, v] : g.steps) {
            if (t <= begin) {
                level = v;
                continue;
            }
            if (t >= at) break;
            integral += level * (t - cursor);
            cursor = t;
            level = v;
        }
        integral += level * (at - cursor);
        return integral / span;
    }
    // gpu.cpp:269-274
    double power(const Gpu& g) const {
        const double s = inst_smact(g);
        double p = c.p_idle_w + (c.p_max_w - c.p_idle_w) * s;
        if (s > c.boost_threshold) p += c.p_boost_w;
        return p;
    }
    // world.cpp:31-35
    void schedule(double t, int kind, int task, uint64_t gen) {
        pq.push(Event{t, next_seq++, kind, task, gen});
    }
    // world.cpp:37-44
    void integrate_to(double t) {
        const double dt = t - now;
        if (dt > 0.0)
            for (auto& g : gpu) g.energy += power(g) * dt;
        now = t;
    }
    // world.cpp:157-186: affected tasks in lexicographic id order (rank).
    void refresh_rates(const std::vector<int>& touched) {
        std::set<std::pair<uint32_t, int>> affected;
        for (int g : touched) {
            record_smact(gpu[static_cast<size_t>(g)]);
            for (const auto& r : gpu[static_cast<size_t>(g)].residents)
                affected.insert({tasks[r.id].rank, r.id});
        }
        for (const auto& [rank, id] : affected) {
            Run& r = run[static_cast<size_t>(id)];
            double rate = 1.0;
            for (int g : r.gpus) rate = std::min(rate, task_rate(gpu[static_cast<size_t>(g)], id));
            if (rate == r.rate && r.gen != 0) continue;
            const double dt = now - r.last_update;
            r.executed += r.rate * dt;
            r.remaining = std::max(0.0, r.remaining - r.rate * dt);
            r.last_update = now;
            r.rate = rate;
            r.gen++;
            schedule(now + r.remaining / rate, COMPLETION, id, r.gen);
        }
    }
    // world.cpp:73-130
    bool place(int id, const std::vector<int>& ids, const std::vector<int>& insts) {
        Run& r = run[static_cast<size_t>(id)];
        r.exists = true;
        std::vector<std::pair<uint64_t, uint64_t>> placed;
        for (size_t k = 0; k < ids.size(); ++k) {
            uint64_t off = 0, size = 0;
            const uint64_t lo = mig() ? inst_base(insts[k]) : 0;
            const uint64_t hi = mig() ? lo + inst_cap(insts[k]) : c.gpu_capacity;
            if (!allocate_range(gpu[static_cast<size_t>(ids[k])], lo, hi, tasks[id].true_mem, &off, &size)) {
                for (size_t j = 0; j < placed.size(); ++j)
                    free_region(gpu[static_cast<size_t>(ids[j])], placed[j].first, placed[j].second);
                return false;
            }
            placed.push_back({off, size});
        }
        r.gpus = ids;
        r.insts = insts;
        r.region_off.clear();
        r.region_size.clear();
        for (auto& p : placed) {
            r.region_off.push_back(p.first);
            r.region_size.push_back(p.second);
        }
        r.remaining = tasks[id].work;
        r.last_update = now;
        r.resident = true;
        for (size_t k = 0; k < ids.size(); ++k)
            gpu[static_cast<size_t>(ids[k])].residents.push_back({id, tasks[id].demand, insts[k]});
        refresh_rates(ids);
        return true;
    }
    // world.cpp:132-155
    void finish(int id) {
        Run& r = run[static_cast<size_t>(id)];
        const double dt = now - r.last_update;
        r.executed += r.rate * dt;
        r.remaining = std::max(0.0, r.remaining - r.rate * dt);
        r.last_update = now;
        r.resident = false;
        r.completed = true;
        for (size_t k = 0; k < r.gpus.size(); ++k) {
            Gpu& g = gpu[static_cast<size_t>(r.gpus[k])];
            free_region(g, r.region_off[k], r.region_size[k]);
            for (size_t j = 0; j < g.residents.size(); ++j)
                if (g.residents[j].id == id) {
                    g.residents.erase(g.residents.begin() + static_cast<std::ptrdiff_t>(j));
                    break;
                }
        }
        refresh_rates(r.gpus);
    }
    bool all_idle() const {
        for (const auto& g : gpu)
            if (!g.residents.empty()) return false;
        return true;
    }
    // manager.cpp:109-123
    std::vector<int> eligible(uint64_t need) const {
        std::vector<int> e;
        const uint64_t floor = std::max<uint64_t>(c.min_free, need);
        for (int g = 0; g < c.gpu_count; ++g) {
            if (windowed(gpu[static_cast<size_t>(g)], now, c.monitor_window) > c.max_smact) continue;
            if (total_free(gpu[static_cast<size_t>(g)]) < floor) continue;
            e.push_back(g);
        }
        return e;
    }
    // manager.cpp:136-245; inst receives the MIG instance of each chosen GPU.
    std::vector<int> map_task(int id, bool from_recovery, std::vector<int>& inst) {
        std::vector<int> ids;
        inst.clear();
        const size_t want = tasks[id].gpus;
        const int policy = from_recovery ? CARMA_POLICY_EXCLUSIVE : c.policy;
        if (policy == CARMA_POLICY_EXCLUSIVE) {
            for (int g = 0; g < c.gpu_count; ++g) {
                if (!gpu[static_cast<size_t>(g)].residents.empty()) continue;
                ids.push_back(g);
                if (mig()) {
                    const int i = pick_instance(gpu[static_cast<size_t>(g)], 1);
                    inst.push_back(i < 0 ? 0 : i);
                }
                if (ids.size() == want) break;
            }
            if (ids.size() != want) ids.clear();
            if (!mig()) inst.assign(ids.size(), 0);
            return ids;
        }
        const uint64_t est = tasks[id].estimate;
        const uint64_t need = est == CARMA_NO_ESTIMATE ? 0 : std::min(est, c.gpu_capacity);
        std::vector<int> el;
        if (policy == CARMA_POLICY_RR && !c.rr_apply_preconditions) {
            for (int g = 0; g < c.gpu_count; ++g) el.push_back(g);
        } else {
            el = eligible(need);
        }
        std::map<int, int> inst_of;
        if (mig()) {
            std::vector<int> kept;
            for (int g : el) {
                const int i = pick_instance(gpu[static_cast<size_t>(g)], std::max<uint64_t>(need, 1));
                if (i >= 0) {
                    kept.push_back(g);
                    inst_of[g] = i;
                }
            }
            el.swap(kept);
        }
        auto fill_inst = [&]() {
            for (int g : ids) inst.push_back(mig() ? inst_of[g] : 0);
        };
        if (el.size() < want) return {};
        if (policy == CARMA_POLICY_RR) {
            for (int step = 0; step < c.gpu_count && ids.size() < want; ++step) {
                int g = (rr_cursor + step) % c.gpu_count;
                if (std::find(el.begin(), el.end(), g) != el.end()) ids.push_back(g);
            }
            if (ids.size() == want) rr_cursor = (ids.back() + 1) % c.gpu_count;
            else ids.clear();
            fill_inst();
            return ids;
        }
        std::vector<int> sorted = el;
        std::stable_sort(sorted.begin(), sorted.end(), [&](int a, int b) {
            const Gpu& ga = gpu[static_cast<size_t>(a)];
            const Gpu& gb = gpu[static_cast<size_t>(b)];
            if (policy == CARMA_POLICY_MAGM) {
                if (total_free(ga) != total_free(gb)) return total_free(ga) > total_free(gb);
            } else {
                const double sa = windowed(ga, now, c.monitor_window);
                const double sb = windowed(gb, now, c.monitor_window);
                if (sa != sb) return policy == CARMA_POLICY_LUG ? sa < sb : sa > sb;
            }
            return a < b;
        });
        ids.assign(sorted.begin(), sorted.begin() + static_cast<std::ptrdiff_t>(want));
        fill_inst();
        return ids;
    }
    // manager.cpp:269-331
    void try_schedule() {
        const bool gate = now >= deadline || all_idle();
        if (!gate) return;
        const bool from_recovery = !recovery_q.empty();
        int head;
        if (from_recovery) head = recovery_q.front();
        else if (!main_q.empty()) head = main_q.front();
        else return;
        std::vector<int> insts;
        std::vector<int> ids = map_task(head, from_recovery, insts);
        if (ids.empty()) return;
        if (from_recovery) recovery_q.pop_front();
        else main_q.pop_front();
        // dispatch, manager.cpp:247-260
        carma_task_result& o = out[head];
        if (o.attempts == 0) o.first_attempt = now;
        o.attempts++;
        if (!place(head, ids, insts)) {
            schedule(now + c.oom_startup_delay, CRASH, head, 0);
        } else {
            o.final_dispatch = now;
            o.gpu[0] = static_cast<int16_t>(ids[0]);
            o.gpu[1] = static_cast<int16_t>(ids.size() > 1 ? ids[1] : -1);
        }
        // arm_window, manager.cpp:275-278
        deadline = now + c.monitor_window;
        schedule(deadline, WINDOW, -1, 0);
    }
    // world.cpp:46-60 + runner.cpp:85-95 + manager.cpp:333-357
    bool step() {
        if (pq.empty()) return false;
        if (events >= max_events) return false;
        Event ev = pq.top();
        pq.pop();
        ++events;
        if (collect) sample_stats();
        integrate_to(ev.t);
        if (ev.kind == COMPLETION) {
            Run& r = run[static_cast<size_t>(ev.task)];
            if (!r.exists || !r.resident || r.gen != ev.gen) return true;
            finish(ev.task);
        }
        switch (ev.kind) {
            case ARRIVAL:
                ++arrivals_seen;
                main_q.push_back(ev.task);
                try_schedule();
                break;
            case WINDOW:
                if (ev.t == deadline) try_schedule();
                break;
            case COMPLETION:
                out[ev.task].complete = now;
                try_schedule();
                break;
            case CRASH: {
                oom_count++;
                carma_task_result& o = out[ev.task];
                o.ooms++;
                if (o.first_crash < 0.0) o.first_crash = now;
                o.last_crash = now;
                recovery_q.push_back(ev.task);
                try_schedule();
                break;
            }
        }
        return true;
    }
};

}  // namespace

extern "C" int oracle_knn_predict(const double* lo, const double* hi, const double* points,
                                  const int32_t* labels, uint64_t n, uint32_t k,
                                  uint64_t bucket_range, const double* raw, uint64_t q,
                                  int32_t* bucket, uint64_t* bytes, double* topk_d2,
                                  int64_t* topk_idx) {
    if (n == 0 || k == 0) return 1;
    for (uint64_t i = 0; i < q; ++i) {
        const int b = predict_one(lo, hi, points, labels, n, k, raw + i * 19,
                                  topk_d2 ? topk_d2 + i * k : nullptr,
                                  topk_idx ? topk_idx + i * k : nullptr);
        if (bucket) bucket[i] = b;
        if (bytes) bytes[i] = (static_cast<uint64_t>(b) + 1) * bucket_range;
    }
    return 0;
}

extern "C" int oracle_replay(const carma_replay_config* cfg, const carma_task* tasks, uint32_t n,
                             carma_task_result* out_tasks, carma_trace_result* out_trace,
                             carma_gpu_result* out_gpus) {
    if (n == 0 || cfg->gpu_count < 1) return 1;
    for (uint32_t i = 0; i < n; ++i) {
        carma_task_result& o = out_tasks[i];
        o.first_attempt = o.final_dispatch = o.complete = o.first_crash = o.last_crash = -1.0;
        o.executed = 0.0;
        o.attempts = o.ooms = 0;
        o.gpu[0] = o.gpu[1] = -1;
        o.reserved = 0;
    }
    Sim s(*cfg, tasks, n, out_tasks);
    s.max_events = 1000ull * n + 1000000ull;  // guard against non-terminating configs
    // runner.cpp:72-78: arrivals first, seq = trace index.
    for (uint32_t i = 0; i < n; ++i) s.schedule(tasks[i].submit, ARRIVAL, static_cast<int>(i), 0);
    while (s.step()) {
    }
    for (uint32_t i = 0; i < n; ++i) out_tasks[i].executed = s.run[i].executed;
    // runner.cpp:97-141
    carma_trace_result& tr = *out_trace;
    tr.events = s.events;
    tr.end_time = s.now;
    tr.oom_count = s.oom_count;
    tr.status = 0;
    for (uint32_t i = 0; i < n; ++i)
        if (out_tasks[i].complete < 0.0) tr.status = CARMA_ERR_INCOMPLETE;
    double first_submit = tasks[0].submit;
    for (uint32_t i = 0; i < n; ++i) first_submit = std::min(first_submit, tasks[i].submit);
    double last_complete = 0.0;
    for (uint32_t i = 0; i < n; ++i) last_complete = std::max(last_complete, out_tasks[i].complete);
    tr.first_submit = first_submit;
    tr.last_complete = last_complete;
    const double overshoot = s.now - last_complete;
    if (overshoot > 0.0)
        for (auto& g : s.gpu) g.energy -= s.power(g) * overshoot;
    double energy = 0.0;
    for (int g = 0; g < cfg->gpu_count; ++g) {
        Gpu& d = s.gpu[static_cast<size_t>(g)];
        carma_gpu_result& og = out_gpus[g];
        og.energy_j = d.energy;
        const double span = last_complete - first_submit;
        og.mean_smact = span > 0.0 ? s.windowed(d, last_complete, span) : 0.0;
        og.peak_used = d.peak;
        og.smact_steps = d.steps.size();
        energy += d.energy;
    }
    // metrics.cpp:16-70: sums in std::map<std::string> order == rank order.
    std::vector<uint32_t> by_rank(n);
    for (uint32_t i = 0; i < n; ++i) by_rank[tasks[i].rank] = i;
    double ws = 0.0, es = 0.0, js = 0.0;
    for (uint32_t r = 0; r < n; ++r) {
        const carma_task_result& o = out_tasks[by_rank[r]];
        const double submit = tasks[by_rank[r]].submit;
        ws += o.final_dispatch - submit;
        es += o.complete - o.final_dispatch;
        js += o.complete - submit;
    }
    const double nd = static_cast<double>(n);
    tr.avg_wait = ws / nd;
    tr.avg_exec = es / nd;
    tr.avg_jct = js / nd;
    tr.trace_total_time = last_complete - first_submit;
    tr.energy_mj = energy / 1e6;
    return tr.status;
}

// map_task over one snapshot; out[0, out_n) gets the chosen ids, -1 padded.
static int oracle_pick_n(const carma_replay_config* cfg, const carma_gpu_view* gpus, uint32_t n_gpus,
                         const carma_pick_request* req, int32_t* rr_cursor, int32_t* out, uint32_t out_n) {
    for (uint32_t i = 0; i < out_n; ++i) out[i] = -1;
    const uint32_t want = req->want;
    const int policy = req->from_recovery ? CARMA_POLICY_EXCLUSIVE : cfg->policy;
    std::vector<int> ids;
    if (policy == CARMA_POLICY_EXCLUSIVE) {
        for (uint32_t g = 0; g < n_gpus && ids.size() < want; ++g)
            if (gpus[g].idle) ids.push_back(static_cast<int>(g));
        if (ids.size() != want) ids.clear();
    } else {
        const uint64_t need = req->estimate == CARMA_NO_ESTIMATE ? 0 : std::min(req->estimate, cfg->gpu_capacity);
        const uint64_t floor = std::max<uint64_t>(cfg->min_free, need);
        std::vector<int> el;
        for (uint32_t g = 0; g < n_gpus; ++g) {
            if (policy == CARMA_POLICY_RR && !cfg->rr_apply_preconditions) {
                el.push_back(static_cast<int>(g));
                continue;
            }
            if (gpus[g].windowed_smact > cfg->max_smact) continue;
            if (gpus[g].total_free < floor) continue;
            el.push_back(static_cast<int>(g));
        }
        if (el.size() >= want) {
            if (policy == CARMA_POLICY_RR) {
                for (uint32_t step = 0; step < n_gpus && ids.size() < want; ++step) {
                    int g = static_cast<int>((static_cast<uint32_t>(*rr_cursor) + step) % n_gpus);
                    if (std::find(el.begin(), el.end(), g) != el.end()) ids.push_back(g);
                }
                if (ids.size() == want) *rr_cursor = static_cast<int32_t>((ids.back() + 1) % static_cast<int>(n_gpus));
                else ids.clear();
            } else {
                std::stable_sort(el.begin(), el.end(), [&](int a, int b) {
                    if (policy == CARMA_POLICY_MAGM) {
                        if (gpus[a].total_free != gpus[b].total_free) return gpus[a].total_free > gpus[b].total_free;
                    } else {
                        const double sa = gpus[a].windowed_smact, sb = gpus[b].windowed_smact;
                        if (sa != sb) return policy == CARMA_POLICY_LUG ? sa < sb : sa > sb;
                    }
                    return a < b;
                });
                ids.assign(el.begin(), el.begin() + want);
            }
        }
    }
    for (size_t i = 0; i < ids.size() && i < out_n; ++i) out[i] = ids[i];
    return 0;
}

extern "C" int oracle_pick(const carma_replay_config* cfg, const carma_gpu_view* gpus,
                           uint32_t n_gpus, const carma_pick_request* req, int32_t* rr_cursor,
                           int32_t* out) {
    return oracle_pick_n(cfg, gpus, n_gpus, req, rr_cursor, out, 2);
}

// The same for up to 8 GPUs per decision (out: 8 ids).
extern "C" int oracle_pick_wide(const carma_replay_config* cfg, const carma_gpu_view* gpus,
                                uint32_t n_gpus, const carma_pick_request* req, int32_t* rr_cursor,
                                int32_t* out) {
    return oracle_pick_n(cfg, gpus, n_gpus, req, rr_cursor, out, 8);
}

// Test-only: peak sizes of the replay state over one run (heap of pending
// events, resident tasks, residents per GPU, SMACT steps inside the window
// + 1, recovery queue). Used to size the GPU kernel's state tiers.
extern "C" int oracle_replay_stats(const carma_replay_config* cfg, const carma_task* tasks, uint32_t n,
                                   uint64_t* stats5) {
    std::vector<carma_task_result> out(n);
    for (auto& o : out) {
        o.first_attempt = o.final_dispatch = o.complete = o.first_crash = o.last_crash = -1.0;
        o.attempts = o.ooms = 0;
    }
    Sim s(*cfg, tasks, n, out.data());
    s.max_events = 1000ull * n + 1000000ull;
    s.collect = true;
    for (uint32_t i = 0; i < n; ++i) s.schedule(tasks[i].submit, ARRIVAL, static_cast<int>(i), 0);
    while (s.step()) {
    }
    // arrivals sit in the oracle's heap; the kernel streams them separately
    stats5[0] = s.st_heap;
    stats5[1] = s.st_resident;
    stats5[2] = s.st_res_gpu;
    stats5[3] = s.st_window;
    stats5[4] = s.st_rq;
    return 0;
}
