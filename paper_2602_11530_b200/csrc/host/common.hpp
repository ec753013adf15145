// common.hpp — host-side types of libpascal.so (B200 build).
//
// Host code here is the C-ABI layer and the host-only formats around the hot
// path: trace generation and IO (proj/src/workload.cpp), profile IO and
// calibration (proj/src/costmodel.cpp), report IO / tail bins / compare
// (proj/src/metrics.cpp:85-113,155-323). The scheduling loop itself only runs
// on the GPU (engine.cu); this layer packs inputs and formats outputs.
//
// Error taxonomy mirrors the reference's exception-to-status mapping
// (proj/src/capi.cpp:21-37): std::invalid_argument -> 1, std::runtime_error
// -> 2, any other std::exception -> 3.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../engine.h"

namespace pbh {

// proj/include/pascalsim/workload.hpp:14-28
struct Spec {
    long id = 0;
    double arrival = 0.0;
    long prompt = 1;
    long reasoning = 0;
    long answering = 1;
    bool preloaded = false;
    long max_kv() const { return prompt + reasoning + answering; }
};
using Trace = std::vector<Spec>;

// ---- text helpers (behaviour of proj/include/pascalsim/textio.hpp) -------
std::string_view strip(std::string_view s);
std::vector<std::string_view> cut(std::string_view s, char sep);
long to_long(std::string_view s, const std::string& what);
double to_double(std::string_view s, const std::string& what);

// ---- workload ------------------------------------------------------------
class LengthDist {
public:
    enum class Kind { Constant, Uniform, Hist };
    static LengthDist parse(const std::string& spec);
    long draw(std::mt19937_64& rng) const;
    long lowest() const;

private:
    Kind kind_ = Kind::Constant;
    long value_ = 0, lo_ = 0, hi_ = 0;
    std::vector<std::pair<long, double>> bins_;
    std::vector<double> cdf_;
};

Trace generate(long count, double rate, const LengthDist& p, const LengthDist& r,
               const LengthDist& a, std::uint64_t seed, bool preloaded);
Trace mix(const Trace& base, const Trace& repl, double fraction, std::uint64_t seed);
void check_trace(const Trace& t);
Trace read_trace(const std::string& path);
void write_trace(const Trace& t, const std::string& path);
Trace read_trace_hex(const std::string& path);
void write_trace_hex(const Trace& t, const std::string& path);

// ---- latency profile -----------------------------------------------------
pb::Profile default_profile();
void check_profile(const pb::Profile& p);
void set_profile_field(pb::Profile& p, const std::string& key, double v);
pb::Profile read_profile(const std::string& path);
void write_profile(const pb::Profile& p, const std::string& path);
struct Fit {
    double base = 0, per_req = 0, per_kv = 0, rmse = 0;
};
Fit calibrate_file(const std::string& samples_path);

// ---- run configuration ---------------------------------------------------
struct RunCfg {  // proj/include/pascalsim/engine.hpp:18-33
    int instances = 8;
    long gpu_capacity = 0;
    double capacity_fraction = 0.0;
    long quantum = 500;
    long demotion = 5000;
    int policy = pb::kPascal;
    bool no_migration = false;
    bool non_adaptive = false;
    double tpot = 0.1;
    double ttfat_target = 0.25;
    double qoe_threshold = 0.95;
    long slack = 0;
};
int parse_policy(const std::string& name);  // engine.cpp:22-28

// ---- reports -------------------------------------------------------------
struct Row {  // proj/include/pascalsim/metrics.hpp:58-67
    long id = 0, reasoning = 0, answering = 0;
    double ttft = 0, ttfat = 0, qoe = 0;
    bool slo = false;
    double blocking = 0;
    double tpot = 0;  // device-only output (not written to requests.csv)
};
struct Bin {
    long lo = 0, hi = 0, count = 0;
    std::string stat;
    double value = 0;
};
struct Report {
    std::vector<Row> rows;
    double ttft_mean = 0, ttft_p50 = 0, ttft_p90 = 0, ttft_p95 = 0, ttft_p99 = 0;
    double slo_rate = 0, ttfat_attain = 0, throughput = 0;
    std::vector<Bin> bins;
    std::vector<std::pair<std::string, std::string>> echo;
};
std::vector<Bin> tail_bins(const std::vector<std::pair<long, double>>& rows);
void write_report(const Report& r, const std::string& prefix);
Report read_report(const std::string& prefix);
std::string compare_text(const std::vector<Report>& reps, const std::vector<std::string>& names);

// ---- device engine driver (engine_host.cpp) ------------------------------
struct DeviceSummary {  // mirrors pascal_summary
    double ttft_mean, ttft_p50, ttft_p90, ttft_p95, ttft_p99;
    double slo_rate, ttfat_attain, throughput;
    long long capacity, requests, req_iters, answer_tokens, events, plans, visits, health;
    long long slo_violations;
    long long adm_rounds, adm_slow;
    int status, pad;
    double tpot_mean;
    long long tpot_requests;
};

struct Job {
    const Trace* trace = nullptr;
    RunCfg cfg;
    pb::Profile prof{};
};

struct RunOutputs {  // full per-replica outputs for pascal_run / pascal_run_dump
    int status = 0;
    long long capacity = 0;
    DeviceSummary summary{};
    std::vector<Row> rows;          // trace order
    std::vector<pb::RecOut> rec;    // trace order
    std::vector<double> dig, del;   // answer arenas (per aoff)
    std::vector<long long> aoff;
    std::vector<pb::LogEnt> log;
};

const char* status_message(int status);
long long request_iterations(const Trace& t);
// Runs one replica with full outputs (records, rows, optional log).
RunOutputs run_single(const Job& job, bool want_records, bool want_log);
// Capacity only (engine::derive_capacity).
long long derive_capacity_dev(const Job& job);

class Batch;  // device-resident replica batch (engine_host.cpp)
Batch* batch_create(const std::vector<Job>& jobs);
void batch_execute(Batch* b);
void batch_summaries(Batch* b, std::vector<DeviceSummary>& out);
void batch_free(Batch* b);
void batch_rows(Batch* b, std::vector<std::vector<Row>>& rows);
void batch_set_groups(Batch* b, const int* group_of_replica, int n_groups);
void batch_histograms(Batch* b, unsigned long long* hist, unsigned long long* slo);

struct Timing {
    double derive_ms = 0, engine_ms = 0, metrics_ms = 0, total_ms = 0, h2d_ms = 0, d2h_ms = 0;
    long long h2d_bytes = 0, d2h_bytes = 0;
    int launches = 0;
    int instance_parallel = 0;  // policy-run replicas completed by the instance-parallel engine
};
Timing& last_timing();
void release_cached_memory();
void set_device(int dev);
bool device_available();

}  // namespace pbh
