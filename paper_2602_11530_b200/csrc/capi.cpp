// capi.cpp — the C ABI of libpascal.so (include/pascal.h + include/pascal_b200.h).
//
// Contract of the reference's capi (proj/src/capi.cpp:13-254): guarded calls
// map std::invalid_argument -> 1, std::runtime_error -> 2, other
// std::exception -> 3; success clears the thread-local message; NULL handles
// -> 1 "null argument"; *_free, pascal_trace_size and pascal_run_config_init
// are unguarded. pascal_run drives the sm_100a engine (engine_host.cpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <filesystem>
#include <memory>
#include <numeric>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pascal.h"
#include "../../include/pascal_b200.h"
#include "host/common.hpp"

using namespace pbh;

namespace pbh {  // host/probe.cpp
void probe_maybe_start(const pascal_probe_state& st, const pb::Profile& prof,
                       pascal_probe_plan& out);
void probe_select(int mode, long count, int n, const unsigned char* t, const long* k1,
                  const long* k2, int* out);
}  // namespace pbh

namespace {

thread_local std::string g_err;

template <class F>
pascal_status guarded(F&& body) {
    try {
        body();
        g_err.clear();
        return PASCAL_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return PASCAL_ERR_INVALID_ARGUMENT;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return PASCAL_ERR_IO;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PASCAL_ERR_INTERNAL;
    }
}

void need(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

RunCfg to_cfg(const pascal_run_config* c) {
    need(c->policy != nullptr, "policy is null");
    RunCfg r;
    r.instances = c->instance_count;
    r.gpu_capacity = c->gpu_capacity;
    r.capacity_fraction = c->capacity_fraction;
    r.quantum = c->token_quantum;
    r.demotion = c->demotion_threshold;
    r.policy = parse_policy(c->policy);
    r.no_migration = c->no_migration != 0;
    r.non_adaptive = c->non_adaptive != 0;
    r.tpot = c->target_tpot;
    r.ttfat_target = c->ttfat_target;
    r.qoe_threshold = c->qoe_threshold;
    r.slack = c->pacer_slack_tokens;
    return r;
}

// Predicted device work of a replica: its request-iterations (policy- and
// rate-independent) times a per-policy factor (the Pascal /
// RR planners scan, partition and preempt; FCFS and the oracle admit in
// order), plus one oracle pass when the capacity is derived.
double replica_cost(const Job& j) {
    const double t = (double)request_iterations(*j.trace) + (double)j.trace->size();
    double f = j.cfg.policy == pb::kPascal ? 4.0 : j.cfg.policy == pb::kRr ? 3.0 : 1.0;
    if (j.cfg.gpu_capacity <= 0 && j.cfg.policy != pb::kOracle) f += 1.0;
    return t * f;
}

// Longest-processing-time-first: replicas in descending predicted cost (ties
// by index) each go to the currently least-loaded part (ties to the lowest
// part index). Deterministic.
std::vector<int> partition_lpt(const std::vector<Job>& jobs, int parts) {
    std::vector<int> part(jobs.size(), 0);
    if (parts <= 1) return part;
    std::vector<double> cost(jobs.size());
    for (size_t k = 0; k < jobs.size(); ++k) cost[k] = replica_cost(jobs[k]);
    std::vector<size_t> ord(jobs.size());
    std::iota(ord.begin(), ord.end(), size_t{0});
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return cost[a] > cost[b]; });
    std::vector<double> load(parts, 0.0);
    for (size_t k : ord) {
        int best = 0;
        for (int p = 1; p < parts; ++p)
            if (load[p] < load[best]) best = p;
        part[k] = best;
        load[best] += cost[k];
    }
    return part;
}

// Simulates `jobs` over `devices` (one host thread per device, each running
// one device batch of its part), results in input order.
void run_jobs_devices(const std::vector<Job>& jobs, const std::vector<int>& devices,
                      std::vector<DeviceSummary>& sum, std::vector<std::vector<Row>>* rows) {
    if (!device_available()) throw std::logic_error("no CUDA device available for the B200 engine");
    const int nd = (int)devices.size();
    const std::vector<int> part = partition_lpt(jobs, nd);
    sum.assign(jobs.size(), DeviceSummary{});
    if (rows) rows->assign(jobs.size(), {});
    std::vector<std::exception_ptr> err(nd);
    auto work = [&](int d) {
        try {
            std::vector<size_t> idx;
            std::vector<Job> sub;
            for (size_t k = 0; k < jobs.size(); ++k)
                if (part[k] == d) idx.push_back(k), sub.push_back(jobs[k]);
            if (sub.empty()) return;
            set_device(devices[d]);
            std::unique_ptr<Batch, void (*)(Batch*)> b(batch_create(sub), batch_free);
            batch_execute(b.get());
            std::vector<DeviceSummary> s;
            batch_summaries(b.get(), s);
            std::vector<std::vector<Row>> r;
            if (rows) batch_rows(b.get(), r);
            for (size_t q = 0; q < idx.size(); ++q) {
                sum[idx[q]] = s[q];
                if (rows) (*rows)[idx[q]] = std::move(r[q]);
            }
        } catch (...) {
            err[d] = std::current_exception();
        }
    };
    if (nd == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int d = 0; d < nd; ++d) th.emplace_back(work, d);
        for (auto& x : th) x.join();
    }
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

std::vector<int> device_list(const int* devices, int n_devices) {
    std::vector<int> d;
    if (devices == nullptr || n_devices <= 0) {
        int cur = 0;
        if (cudaGetDevice(&cur) != cudaSuccess) cur = 0;
        d.push_back(cur);
        return d;
    }
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    for (int k = 0; k < n_devices; ++k) {
        need(devices[k] >= 0 && devices[k] < count, "device index out of range");
        for (int x : d) need(x != devices[k], "device listed twice");
        d.push_back(devices[k]);
    }
    return d;
}

const char* kKindName[] = {"arrival",       "demote",           "evict",        "swap_in",
                           "block",         "prefill_start",    "decode_start", "prefill_complete",
                           "token",         "transition",       "migrate",      "finish",
                           "swap_complete", "transfer_complete"};

// pascal-events-v1 text (proj/src/engine.cpp:91-97,391)
void write_event_log(FILE* f, const Trace& t, const std::vector<pb::LogEnt>& log) {
    std::fputs("pascal-events-v1\n", f);
    char det[48];
    for (const pb::LogEnt& e : log) {
        det[0] = 0;
        if (e.kind == pb::kLMigrate) std::snprintf(det, sizeof det, "to=%d", e.detail);
        else if (e.kind == pb::kLDecodeStart) std::snprintf(det, sizeof det, "batch=%d", e.detail);
        std::fprintf(f, "%.9f,%s,%d,%ld,%s\n", e.t, kKindName[e.kind], e.inst,
                     e.req >= 0 ? t[(size_t)e.req].id : -1L, det);
    }
}

std::vector<size_t> id_order(const Trace& t) {
    std::vector<size_t> ord(t.size());
    std::iota(ord.begin(), ord.end(), size_t{0});
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return t[a].id < t[b].id; });
    return ord;
}

// metrics::build_report + the config echo of pascal_run (proj/src/capi.cpp:
// 191-203): rows in id order, device-computed aggregates, tail bins.
Report make_report(const Trace& t, const pascal_run_config& cfg, const RunCfg& rc,
                   const std::vector<Row>& rows, const DeviceSummary& s, long long capacity) {
    Report rep;
    std::vector<std::pair<long, double>> pts;
    for (size_t k : id_order(t)) {
        rep.rows.push_back(rows[k]);
        pts.emplace_back(rows[k].reasoning, rows[k].ttft);
    }
    if (!t.empty()) {
        rep.ttft_mean = s.ttft_mean;
        rep.ttft_p50 = s.ttft_p50;
        rep.ttft_p90 = s.ttft_p90;
        rep.ttft_p95 = s.ttft_p95;
        rep.ttft_p99 = s.ttft_p99;
        rep.slo_rate = s.slo_rate;
        rep.ttfat_attain = s.ttfat_attain;
        rep.throughput = s.throughput;
        rep.bins = tail_bins(pts);
    }
    rep.echo = {
        {"policy", cfg.policy},
        {"instance_count", std::to_string(rc.instances)},
        {"gpu_capacity", std::to_string(capacity)},
        {"token_quantum", std::to_string(rc.quantum)},
        {"demotion_threshold", std::to_string(rc.demotion)},
        {"no_migration", std::to_string(cfg.no_migration != 0)},
        {"non_adaptive", std::to_string(cfg.non_adaptive != 0)},
        {"requests", std::to_string(t.size())},
    };
    return rep;
}

}  // namespace

struct pascal_trace {
    Trace t;
};
struct pascal_profile {
    pb::Profile p;
};
struct pascal_report {
    Report r;
};
struct pascal_batch {
    Batch* b = nullptr;
};

extern "C" {

const char* pascal_last_error(void) { return g_err.c_str(); }

pascal_status pascal_trace_load(const char* path, pascal_trace** out) {
    return guarded([&] {
        need(path && out, "null argument");
        *out = new pascal_trace{read_trace(path)};
    });
}

pascal_status pascal_trace_save(const pascal_trace* t, const char* path) {
    return guarded([&] {
        need(t && path, "null argument");
        write_trace(t->t, path);
    });
}

pascal_status pascal_trace_generate(long count, double arrival_rate, const char* prompt_dist,
                                    const char* reasoning_dist, const char* answering_dist,
                                    uint64_t seed, int kv_preloaded, pascal_trace** out) {
    return guarded([&] {
        need(prompt_dist && reasoning_dist && answering_dist && out, "null argument");
        *out = new pascal_trace{generate(count, arrival_rate, LengthDist::parse(prompt_dist),
                                         LengthDist::parse(reasoning_dist),
                                         LengthDist::parse(answering_dist), seed,
                                         kv_preloaded != 0)};
    });
}

pascal_status pascal_trace_mix(const pascal_trace* base, const pascal_trace* replacement,
                               double fraction, uint64_t seed, pascal_trace** out) {
    return guarded([&] {
        need(base && replacement && out, "null argument");
        *out = new pascal_trace{mix(base->t, replacement->t, fraction, seed)};
    });
}

long pascal_trace_size(const pascal_trace* t) { return t ? (long)t->t.size() : 0; }

void pascal_trace_free(pascal_trace* t) { delete t; }

pascal_status pascal_profile_default(pascal_profile** out) {
    return guarded([&] {
        need(out, "null argument");
        *out = new pascal_profile{default_profile()};
    });
}

pascal_status pascal_profile_load(const char* path, pascal_profile** out) {
    return guarded([&] {
        need(path && out, "null argument");
        *out = new pascal_profile{read_profile(path)};
    });
}

pascal_status pascal_profile_save(const pascal_profile* p, const char* path) {
    return guarded([&] {
        need(p && path, "null argument");
        write_profile(p->p, path);
    });
}

pascal_status pascal_profile_set(pascal_profile* p, const char* key, double value) {
    return guarded([&] {
        need(p && key, "null argument");
        set_profile_field(p->p, key, value);
    });
}

pascal_status pascal_profile_calibrate(const char* samples_path, pascal_profile* p,
                                       double* rmse_out) {
    return guarded([&] {
        need(samples_path && p, "null argument");
        Fit f = calibrate_file(samples_path);
        p->p.decode_base = f.base;
        p->p.decode_per_request = f.per_req;
        p->p.decode_per_kv_token = f.per_kv;
        if (rmse_out) *rmse_out = f.rmse;
    });
}

void pascal_profile_free(pascal_profile* p) { delete p; }

void pascal_run_config_init(pascal_run_config* cfg) {
    if (!cfg) return;
    RunCfg d;
    cfg->instance_count = d.instances;
    cfg->gpu_capacity = d.gpu_capacity;
    cfg->capacity_fraction = d.capacity_fraction;
    cfg->token_quantum = d.quantum;
    cfg->demotion_threshold = d.demotion;
    cfg->policy = "pascal";
    cfg->no_migration = 0;
    cfg->non_adaptive = 0;
    cfg->target_tpot = d.tpot;
    cfg->ttfat_target = d.ttfat_target;
    cfg->qoe_threshold = d.qoe_threshold;
    cfg->pacer_slack_tokens = d.slack;
}

pascal_status pascal_run(const pascal_trace* t, const pascal_profile* p,
                         const pascal_run_config* cfg, const char* report_prefix,
                         const char* event_log_path) {
    return guarded([&] {
        need(t && p && cfg && report_prefix, "null argument");
        RunCfg rc = to_cfg(cfg);
        FILE* logf = nullptr;
        if (event_log_path) {
            logf = std::fopen(event_log_path, "w");
            if (!logf)
                throw std::runtime_error(std::string("cannot open event log: ") + event_log_path);
        }
        struct Closer {
            FILE* f;
            ~Closer() {
                if (f) std::fclose(f);
            }
        } closer{logf};
        check_trace(t->t);
        check_profile(p->p);
        Job job{&t->t, rc, p->p};
        RunOutputs o = run_single(job, false, logf != nullptr);
        if (logf) write_event_log(logf, t->t, o.log);

        write_report(make_report(t->t, *cfg, rc, o.rows, o.summary, o.capacity), report_prefix);
    });
}

pascal_status pascal_report_load(const char* prefix, pascal_report** out) {
    return guarded([&] {
        need(prefix && out, "null argument");
        *out = new pascal_report{read_report(prefix)};
    });
}

pascal_status pascal_report_summary_value(const pascal_report* r, const char* key, double* out) {
    return guarded([&] {
        need(r && key && out, "null argument");
        const Report& p = r->r;
        const std::string k = key;
        if (k == "ttft_mean") *out = p.ttft_mean;
        else if (k == "ttft_p50") *out = p.ttft_p50;
        else if (k == "ttft_p90") *out = p.ttft_p90;
        else if (k == "ttft_p95") *out = p.ttft_p95;
        else if (k == "ttft_p99") *out = p.ttft_p99;
        else if (k == "slo_violation_rate") *out = p.slo_rate;
        else if (k == "ttfat_attainment") *out = p.ttfat_attain;
        else if (k == "throughput") *out = p.throughput;
        else throw std::invalid_argument("unknown summary key: " + k);
    });
}

void pascal_report_free(pascal_report* r) { delete r; }

pascal_status pascal_compare(const char* const* prefixes, const char* const* names,
                             size_t count, const char* out_path) {
    return guarded([&] {
        need(prefixes && names && out_path, "null argument");
        need(count >= 2, "compare needs at least 2 reports");
        std::vector<Report> reps;
        std::vector<std::string> labels;
        for (size_t i = 0; i < count; ++i) {
            need(prefixes[i] && names[i], "null argument");
            reps.push_back(read_report(prefixes[i]));
            labels.emplace_back(names[i]);
        }
        std::string text = compare_text(reps, labels);
        FILE* f = std::fopen(out_path, "w");
        if (!f) throw std::runtime_error(std::string("cannot open: ") + out_path);
        std::fwrite(text.data(), 1, text.size(), f);
        std::fclose(f);
    });
}

// ------------------------------------------------------------ extensions
pascal_status pascal_batch_create(const pascal_trace* const* traces,
                                  const pascal_profile* const* profiles,
                                  const pascal_run_config* cfgs, size_t count,
                                  pascal_batch** out) {
    return guarded([&] {
        need(traces && profiles && cfgs && out, "null argument");
        if (!device_available()) throw std::logic_error("no CUDA device available for the B200 engine");
        std::vector<Job> jobs(count);
        for (size_t k = 0; k < count; ++k) {
            need(traces[k] && profiles[k], "null argument");
            jobs[k] = Job{&traces[k]->t, to_cfg(&cfgs[k]), profiles[k]->p};
        }
        auto* h = new pascal_batch;
        try {
            h->b = batch_create(jobs);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

pascal_status pascal_batch_execute(pascal_batch* b) {
    return guarded([&] {
        need(b && b->b, "null argument");
        batch_execute(b->b);
    });
}

pascal_status pascal_batch_summaries(pascal_batch* b, pascal_summary* out) {
    return guarded([&] {
        need(b && b->b && out, "null argument");
        static_assert(sizeof(pascal_summary) == sizeof(DeviceSummary), "summary layout");
        std::vector<DeviceSummary> s;
        batch_summaries(b->b, s);
        std::copy(s.begin(), s.end(), reinterpret_cast<DeviceSummary*>(out));
    });
}

pascal_status pascal_batch_rows(pascal_batch* b, size_t replica, pascal_request_row* out) {
    return guarded([&] {
        need(b && b->b && out, "null argument");
        std::vector<std::vector<Row>> rows;
        batch_rows(b->b, rows);
        need(replica < rows.size(), "replica out of range");
        for (size_t k = 0; k < rows[replica].size(); ++k) {
            const Row& w = rows[replica][k];
            out[k] = pascal_request_row{w.id, w.ttft, w.ttfat, w.qoe, w.blocking, w.tpot,
                                        w.slo ? 1 : 0, 0};
        }
    });
}

void pascal_batch_free(pascal_batch* b) {
    if (!b) return;
    batch_free(b->b);
    delete b;
}

pascal_status pascal_batch_set_groups(pascal_batch* b, const int* group_of_replica,
                                      int n_groups) {
    return guarded([&] {
        need(b && b->b && group_of_replica, "null argument");
        batch_set_groups(b->b, group_of_replica, n_groups);
    });
}

pascal_status pascal_batch_histograms(pascal_batch* b, unsigned long long* hist,
                                      unsigned long long* slo) {
    return guarded([&] {
        need(b && b->b && hist && slo, "null argument");
        batch_histograms(b->b, hist, slo);
    });
}

pascal_status pascal_run_batch(const pascal_trace* const* traces,
                               const pascal_profile* const* profiles,
                               const pascal_run_config* cfgs, size_t count,
                               pascal_summary* out) {
    pascal_batch* b = nullptr;
    pascal_status st = pascal_batch_create(traces, profiles, cfgs, count, &b);
    if (st != PASCAL_OK) return st;
    st = pascal_batch_execute(b);
    if (st == PASCAL_OK) st = pascal_batch_summaries(b, out);
    std::string keep = g_err;
    pascal_batch_free(b);
    g_err = keep;
    return st;
}

pascal_status pascal_partition_replicas(const pascal_trace* const* traces,
                                        const pascal_run_config* cfgs, size_t count, int n_parts,
                                        int* part_of_replica) {
    return guarded([&] {
        need(traces && cfgs && part_of_replica, "null argument");
        need(n_parts >= 1, "n_parts must be >= 1");
        std::vector<Job> jobs(count);
        for (size_t k = 0; k < count; ++k) {
            need(traces[k] != nullptr, "null argument");
            jobs[k] = Job{&traces[k]->t, to_cfg(&cfgs[k]), pb::Profile{}};
        }
        const std::vector<int> part = partition_lpt(jobs, n_parts);
        std::copy(part.begin(), part.end(), part_of_replica);
    });
}

pascal_status pascal_run_batch_devices(const pascal_trace* const* traces,
                                       const pascal_profile* const* profiles,
                                       const pascal_run_config* cfgs, size_t count,
                                       const int* devices, int n_devices, pascal_summary* out) {
    return guarded([&] {
        need(traces && profiles && cfgs && out, "null argument");
        std::vector<Job> jobs(count);
        for (size_t k = 0; k < count; ++k) {
            need(traces[k] && profiles[k], "null argument");
            check_trace(traces[k]->t);
            check_profile(profiles[k]->p);
            jobs[k] = Job{&traces[k]->t, to_cfg(&cfgs[k]), profiles[k]->p};
        }
        std::vector<DeviceSummary> sum;
        run_jobs_devices(jobs, device_list(devices, n_devices), sum, nullptr);
        static_assert(sizeof(pascal_summary) == sizeof(DeviceSummary), "summary layout");
        std::copy(sum.begin(), sum.end(), reinterpret_cast<DeviceSummary*>(out));
    });
}

pascal_status pascal_sweep(const pascal_trace* t, const pascal_profile* p,
                           const pascal_run_config* base, const char* const* policies,
                           size_t n_policies, const double* fractions, size_t n_fractions,
                           const char* out_dir) {
    return pascal_sweep_devices(t, p, base, policies, n_policies, fractions, n_fractions, out_dir,
                                nullptr, 0);
}

pascal_status pascal_sweep_devices(const pascal_trace* t, const pascal_profile* p,
                                   const pascal_run_config* base, const char* const* policies,
                                   size_t n_policies, const double* fractions, size_t n_fractions,
                                   const char* out_dir, const int* devices, int n_devices) {
    return guarded([&] {
        need(t && p && base && policies && fractions && out_dir, "null argument");
        need(n_policies >= 1 && n_fractions >= 1, "sweep needs at least one point");
        check_trace(t->t);
        check_profile(p->p);
        // grid points in the reference CLI's order (policy-major,
        // proj/tools/pascalsim_cli.cpp:312-336), all simulated in one batch
        std::vector<pascal_run_config> cfgs;
        std::vector<Job> jobs;
        for (size_t a = 0; a < n_policies; ++a) {
            need(policies[a] != nullptr, "null argument");
            for (size_t b = 0; b < n_fractions; ++b) {
                pascal_run_config c = *base;
                c.policy = policies[a];
                c.capacity_fraction = fractions[b];
                cfgs.push_back(c);
            }
        }
        for (const pascal_run_config& c : cfgs) jobs.push_back(Job{&t->t, to_cfg(&c), p->p});
        if (!device_available()) throw std::logic_error("no CUDA device available for the B200 engine");
        std::vector<DeviceSummary> sum;
        std::vector<std::vector<Row>> rows;
        run_jobs_devices(jobs, device_list(devices, n_devices), sum, &rows);
        std::error_code ignored;
        std::filesystem::create_directories(out_dir, ignored);
        std::string index =
            "policy,capacity_fraction,slo_violation_rate,ttft_p50,ttft_p99,"
            "ttfat_attainment,throughput\n";
        for (size_t k = 0; k < cfgs.size(); ++k) {
            if (sum[k].status != 0) throw std::logic_error(status_message(sum[k].status));
            char tag[64];
            std::snprintf(tag, sizeof tag, "%s_f%.2f", cfgs[k].policy, cfgs[k].capacity_fraction);
            const std::string prefix = std::string(out_dir) + "/" + tag;
            write_report(make_report(t->t, cfgs[k], jobs[k].cfg, rows[k], sum[k], sum[k].capacity),
                         prefix);
            // the CLI reads the values back from the written report
            const Report rep = read_report(prefix);
            char row[256];
            std::snprintf(row, sizeof row, "%s,%.2f,%.6f,%.6f,%.6f,%.6f,%.6f\n", cfgs[k].policy,
                          cfgs[k].capacity_fraction, rep.slo_rate, rep.ttft_p50, rep.ttft_p99,
                          rep.ttfat_attain, rep.throughput);
            index += row;
        }
        const std::string idx = std::string(out_dir) + "/sweep.csv";
        FILE* f = std::fopen(idx.c_str(), "w");
        if (!f) throw std::runtime_error("cannot open: " + idx);
        std::fwrite(index.data(), 1, index.size(), f);
        std::fclose(f);
    });
}

pascal_status pascal_last_timing(pascal_timing* out) {
    return guarded([&] {
        need(out, "null argument");
        const Timing& t = last_timing();
        out->derive_ms = t.derive_ms;
        out->engine_ms = t.engine_ms;
        out->metrics_ms = t.metrics_ms;
        out->total_ms = t.total_ms;
        out->h2d_ms = t.h2d_ms;
        out->d2h_ms = t.d2h_ms;
        out->h2d_bytes = t.h2d_bytes;
        out->d2h_bytes = t.d2h_bytes;
        out->kernel_launches = t.launches;
        out->instance_parallel = t.instance_parallel;
    });
}

pascal_status pascal_run_dump(const pascal_trace* t, const pascal_profile* p,
                              const pascal_run_config* cfg, const char* records_path,
                              const char* event_log_path) {
    return guarded([&] {
        need(t && p && cfg && records_path, "null argument");
        RunCfg rc = to_cfg(cfg);
        check_trace(t->t);
        check_profile(p->p);
        Job job{&t->t, rc, p->p};
        RunOutputs o = run_single(job, true, event_log_path != nullptr);
        if (event_log_path) {
            FILE* f = std::fopen(event_log_path, "w");
            if (!f) throw std::runtime_error(std::string("cannot open event log: ") + event_log_path);
            write_event_log(f, t->t, o.log);
            std::fclose(f);
        }
        FILE* f = std::fopen(records_path, "w");
        if (!f) throw std::runtime_error(std::string("cannot open: ") + records_path);
        for (size_t k : id_order(t->t)) {
            const pb::RecOut& r = o.rec[k];
            const int nd = r.pad;
            std::fprintf(f, "R %ld %a %a %a %a %a %a %a %d", t->t[k].id, r.arrival,
                         r.prefill_complete, r.reasoning_end, r.first_answer_delivery,
                         r.first_answer_iter_start, r.blocked, r.completion, r.nmig);
            if (r.nmig) std::fprintf(f, " %a %a", r.mig_start, r.mig_end);
            const double* del = o.del.data() + o.aoff[k];
            const double* dig = o.dig.data() + o.aoff[k];
            std::fprintf(f, " %d", nd);
            for (int i = 0; i < nd; ++i) std::fprintf(f, " %a", del[i]);
            std::fprintf(f, " %d", nd);
            for (int i = 0; i < nd; ++i) std::fprintf(f, " %a", dig[i]);
            std::fputc('\n', f);
        }
        std::fclose(f);
    });
}

pascal_status pascal_derive_capacity(const pascal_trace* t, const pascal_profile* p,
                                     const pascal_run_config* cfg, long* out) {
    return guarded([&] {
        need(t && p && cfg && out, "null argument");
        RunCfg rc = to_cfg(cfg);
        check_trace(t->t);
        check_profile(p->p);
        *out = (long)derive_capacity_dev(Job{&t->t, rc, p->p});
    });
}

pascal_status pascal_trace_load_hex(const char* path, pascal_trace** out) {
    return guarded([&] {
        need(path && out, "null argument");
        *out = new pascal_trace{read_trace_hex(path)};
    });
}

pascal_status pascal_trace_save_hex(const pascal_trace* t, const char* path) {
    return guarded([&] {
        need(t && path, "null argument");
        write_trace_hex(t->t, path);
    });
}

pascal_status pascal_trace_from_arrays(long n, const long* ids, const double* arrivals,
                                       const long* prompt, const long* reasoning,
                                       const long* answering, const int* preloaded,
                                       pascal_trace** out) {
    return guarded([&] {
        need(out && n >= 0, "null argument");
        need(n == 0 || (ids && arrivals && prompt && reasoning && answering), "null argument");
        Trace t((size_t)n);
        for (long k = 0; k < n; ++k) {
            t[k].id = ids[k];
            t[k].arrival = arrivals[k];
            t[k].prompt = prompt[k];
            t[k].reasoning = reasoning[k];
            t[k].answering = answering[k];
            t[k].preloaded = preloaded ? preloaded[k] != 0 : false;
        }
        *out = new pascal_trace{std::move(t)};
    });
}

pascal_status pascal_trace_get(const pascal_trace* t, long i, long* id, double* arrival,
                               long* prompt, long* reasoning, long* answering, int* preloaded) {
    return guarded([&] {
        need(t, "null argument");
        need(i >= 0 && (size_t)i < t->t.size(), "index out of range");
        const Spec& s = t->t[(size_t)i];
        if (id) *id = s.id;
        if (arrival) *arrival = s.arrival;
        if (prompt) *prompt = s.prompt;
        if (reasoning) *reasoning = s.reasoning;
        if (answering) *answering = s.answering;
        if (preloaded) *preloaded = s.preloaded ? 1 : 0;
    });
}

long long pascal_trace_request_iterations(const pascal_trace* t) {
    return t ? request_iterations(t->t) : 0;
}

pascal_status pascal_probe_maybe_start(const pascal_probe_state* st, const pascal_profile* p,
                                       pascal_probe_plan* out) {
    return guarded([&] {
        need(st && p && out, "null argument");
        check_profile(p->p);
        probe_maybe_start(*st, p->p, *out);
    });
}

pascal_status pascal_probe_select(int mode, long count, int n, const unsigned char* on_track,
                                  const long* key1, const long* key2, int* out) {
    return guarded([&] { probe_select(mode, count, n, on_track, key1, key2, out); });
}

pascal_status pascal_set_device(int device) {
    return guarded([&] { set_device(device); });
}

int pascal_device_available(void) { return device_available() ? 1 : 0; }

pascal_status pascal_release_cached_memory(void) {
    return guarded([&] { release_cached_memory(); });
}

}  // extern "C"
