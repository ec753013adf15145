// ref_dump — TEST INFRASTRUCTURE. Drives the real reference core (compiled
// from /root/reference/proj/src by oracle/Makefile, never copied) and writes
// its outputs in the exact-text formats the parity tests diff against:
//
//   ref_dump gen  COUNT RATE PDIST RDIST ADIST SEED PRELOADED OUT.hex
//   ref_dump mix  BASE.hex REPL.hex FRACTION SEED OUT.hex
//   ref_dump run  TRACE.hex CFG RECORDS_OUT EVENTS_OUT|-
//   ref_dump capacity TRACE.hex CFG
//   ref_dump time TRACE.hex CFG REPEATS            (CPU baseline timing)
//   ref_dump report TRACE.hex CFG PREFIX           (build_report + write_report)
//   ref_dump sim  TRACE.hex CFG                    (engine::run only, no output files;
//                                                   the bench.py reference arm)
//   ref_dump all  TRACE.hex CFG RECORDS|-|'|cmd' EVENTS|-|'|cmd' PREFIX
//        one derive_capacity + one engine::run with that capacity made explicit
//        (identical by engine.cpp:370-377,456: derive_capacity(explicit c) =
//        max(c, biggest) = c), records / event log (a leading '|' pipes into a
//        shell command, e.g. '|sha256sum > x'), and the three pascal-report-v1
//        files with the config echo pascal_run writes (proj/src/capi.cpp:
//        189-203). Prints {"capacity", "derive_s", "run_s"}. For the large
//        goldens, where the C-ABI path would simulate twice more.
//
// Trace files use the lossless hex-float format "pascal-trace-hex-v1"
// (one line per request: id arrival(%a) prompt reasoning answering preloaded).
// CFG is key=value lines for RunConfig (proj/include/pascalsim/engine.hpp:18-33)
// and LatencyProfile (proj/include/pascalsim/costmodel.hpp:12-21) fields;
// numbers go through strtod so "%a" hex floats and "inf" are accepted.
//
// Record dump line (one per request, id order), all doubles as %a:
//   R id arrival prefill_complete reasoning_end first_answer_delivery
//     first_answer_iter_start blocked_interval_total completion
//     NMIG (start end)* NDEL delivery* NDIG digest*
// (fields of metrics::RequestRecord, proj/include/pascalsim/metrics.hpp:15-28)

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pascalsim/cluster.hpp"
#include "pascalsim/engine.hpp"
#include "pascalsim/instance.hpp"
#include "pascalsim/metrics.hpp"
#include "pascalsim/workload.hpp"

using namespace pascalsim;

namespace {

workload::Trace read_hex_trace(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::string line;
    std::getline(in, line);
    if (line != "pascal-trace-hex-v1") throw std::runtime_error("bad hex trace header");
    workload::Trace t;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::istringstream ls(line);
        std::string arr;
        workload::RequestSpec r;
        int pre = 0;
        ls >> r.id >> arr >> r.prompt_tokens >> r.reasoning_tokens >> r.answering_tokens >> pre;
        r.arrival_time = std::strtod(arr.c_str(), nullptr);
        r.kv_preloaded = pre != 0;
        t.push_back(r);
    }
    return t;
}

void write_hex_trace(const workload::Trace& t, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("cannot write " + path);
    std::fprintf(f, "pascal-trace-hex-v1\n");
    for (const auto& r : t)
        std::fprintf(f, "%ld %a %ld %ld %ld %d\n", r.id, r.arrival_time, r.prompt_tokens,
                     r.reasoning_tokens, r.answering_tokens, r.kv_preloaded ? 1 : 0);
    std::fclose(f);
}

struct Cfg {
    engine::RunConfig rc;
    costmodel::LatencyProfile prof;
    std::string policy = "pascal";
};

Cfg read_cfg(const std::string& path) {
    Cfg c;
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::string line;
    while (std::getline(in, line)) {
        auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        std::string k = line.substr(0, eq), v = line.substr(eq + 1);
        double d = std::strtod(v.c_str(), nullptr);
        long l = std::strtol(v.c_str(), nullptr, 10);
        if (k == "instance_count") c.rc.instance_count = static_cast<int>(l);
        else if (k == "gpu_capacity") c.rc.gpu_capacity = l;
        else if (k == "capacity_fraction") c.rc.capacity_fraction = d;
        else if (k == "token_quantum") c.rc.token_quantum = l;
        else if (k == "demotion_threshold") c.rc.demotion_threshold = l;
        else if (k == "policy") c.rc.policy = engine::parse_policy(v), c.policy = v;
        else if (k == "no_migration") c.rc.ablations.no_migration = l != 0;
        else if (k == "non_adaptive") c.rc.ablations.non_adaptive = l != 0;
        else if (k == "target_tpot") c.rc.target_tpot = d;
        else if (k == "ttfat_target") c.rc.ttfat_target = d;
        else if (k == "qoe_threshold") c.rc.qoe_threshold = d;
        else if (k == "pacer_slack_tokens") c.rc.pacer_slack_tokens = l;
        else costmodel::profile_set_field(c.prof, k, d);
    }
    return c;
}

void dump_records(const std::vector<metrics::RequestRecord>& recs, FILE* f) {
    for (const auto& r : recs) {
        std::fprintf(f, "R %ld %a %a %a %a %a %a %a %zu", r.spec.id, r.arrival,
                     r.prefill_complete, r.reasoning_end, r.first_answer_delivery,
                     r.first_answer_iter_start, r.blocked_interval_total, r.completion,
                     r.migration_intervals.size());
        for (auto& [s, e] : r.migration_intervals) std::fprintf(f, " %a %a", s, e);
        std::fprintf(f, " %zu", r.answer_delivery_times.size());
        for (double d : r.answer_delivery_times) std::fprintf(f, " %a", d);
        std::fprintf(f, " %zu", r.answer_digest_times.size());
        for (double d : r.answer_digest_times) std::fprintf(f, " %a", d);
        std::fprintf(f, "\n");
    }
}

// Output sink: a file, or a shell pipeline when the spec starts with '|'.
struct Sink {
    FILE* f = nullptr;
    bool pipe = false;
    explicit Sink(const std::string& spec) {
        if (spec == "-") return;
        pipe = !spec.empty() && spec[0] == '|';
        f = pipe ? popen(spec.c_str() + 1, "w") : std::fopen(spec.c_str(), "w");
        if (!f) throw std::runtime_error("cannot open " + spec);
    }
    ~Sink() {
        if (f) pipe ? pclose(f) : std::fclose(f);
    }
};

// std::ostream over a FILE* (the event log writer takes an ostream).
struct FileBuf : std::streambuf {
    FILE* f;
    explicit FileBuf(FILE* fp) : f(fp) {}
    int overflow(int c) override { return c == EOF ? 0 : std::fputc(c, f); }
    std::streamsize xsputn(const char* s, std::streamsize n) override {
        return (std::streamsize)std::fwrite(s, 1, (size_t)n, f);
    }
};

// ---- unit parity: one maybe_start step on a hand-built state -------------
// STATE lines:  policy P | capacity C | gpu_used G | cpu_used U | counter K |
//   demotion D | now T(%a) | prof KEY VALUE | req ARRIVAL(%a) PROMPT REASONING
//   ANSWERING PHASE LOC SWIN SWOUT TOKENS KV QUSED QUANTA SEQ | high IDX... |
//   low IDX...   (request k has id k)
int plan_state(const std::string& path) {
    using namespace instance;
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    InstanceState st;
    std::vector<RequestState> reqs;
    costmodel::LatencyProfile prof;
    Policy policy = Policy::Pascal;
    std::uint64_t counter = 0;
    double now = 0.0;
    std::string line;
    while (std::getline(in, line)) {
        std::istringstream ls(line);
        std::string k;
        ls >> k;
        if (k == "policy") {
            std::string v;
            ls >> v;
            policy = engine::parse_policy(v);
        } else if (k == "capacity") ls >> st.gpu_capacity;
        else if (k == "gpu_used") ls >> st.gpu_used;
        else if (k == "cpu_used") ls >> st.cpu_used;
        else if (k == "counter") ls >> counter;
        else if (k == "demotion") ls >> st.demotion_threshold;
        else if (k == "now") {
            std::string v;
            ls >> v;
            now = std::strtod(v.c_str(), nullptr);
        } else if (k == "prof") {
            std::string f, v;
            ls >> f >> v;
            costmodel::profile_set_field(prof, f, std::strtod(v.c_str(), nullptr));
        } else if (k == "req") {
            RequestState r;
            std::string arr;
            int phase = 0, loc = 0, sin = 0, sout = 0;
            ls >> arr >> r.spec.prompt_tokens >> r.spec.reasoning_tokens >>
                r.spec.answering_tokens >> phase >> loc >> sin >> sout >> r.tokens_generated >>
                r.kv_tokens >> r.quantum_used_in_round >> r.quanta_exhausted >> r.enqueue_seq;
            r.spec.id = static_cast<long>(reqs.size());
            r.spec.arrival_time = std::strtod(arr.c_str(), nullptr);
            r.phase = static_cast<Phase>(phase);
            r.kv_location = static_cast<KvLocation>(loc);
            r.swapping_in = sin != 0;
            r.swapping_out = sout != 0;
            r.owner = 0;
            reqs.push_back(r);
        } else if (k == "high" || k == "low") {
            long idx;
            while (ls >> idx) (k == "high" ? st.high_queue : st.low_queue).push_back(idx);
        }
    }
    auto list = [](const char* tag, const std::vector<long>& v) {
        std::printf("%s", tag);
        for (long x : v) std::printf(" %ld", x);
        std::printf("\n");
    };
    // Simulator::maybe_start (proj/src/engine.cpp:192-258) minus emit/push:
    // pushes are printed as (request, time) in push order.
    std::vector<long> demoted;
    if (policy == Policy::Pascal) demoted = apply_demotion(st, reqs, counter);
    IterationPlan plan = plan_iteration(st, reqs, prof, policy, now);
    std::vector<std::pair<long, double>> swap_events;
    for (long v : plan.evictions) {
        RequestState& r = reqs[static_cast<std::size_t>(v)];
        st.gpu_used -= r.kv_tokens;
        st.cpu_used += r.kv_tokens;
        r.kv_location = KvLocation::Cpu;
        double dur = costmodel::swap_latency(prof, r.kv_tokens);
        if (dur > 0.0) {
            r.swapping_out = true;
            swap_events.emplace_back(v, now + dur);
        }
    }
    for (long s : plan.swap_ins) {
        RequestState& r = reqs[static_cast<std::size_t>(s)];
        st.cpu_used -= r.kv_tokens;
        st.gpu_used += r.kv_tokens;
        r.swapping_in = true;
        swap_events.emplace_back(s, now + costmodel::swap_latency(prof, r.kv_tokens));
    }
    for (long s : plan.immediate_swap_ins) {
        RequestState& r = reqs[static_cast<std::size_t>(s)];
        st.cpu_used -= r.kv_tokens;
        st.gpu_used += r.kv_tokens;
        r.kv_location = KvLocation::Gpu;
    }
    double completion = 0.0;
    int kind = 0;
    if (plan.kind == IterationPlan::Kind::Prefill) {
        RequestState& r = reqs[static_cast<std::size_t>(plan.prefill_request)];
        long extra = r.spec.reasoning_tokens == 0 ? 1 : 0;
        st.gpu_used += r.spec.prompt_tokens + extra;
        completion = now + plan.duration;
        kind = 1;
    } else if (plan.kind == IterationPlan::Kind::Decode) {
        st.gpu_used += static_cast<long>(plan.batch.size());
        completion = now + plan.duration;
        kind = 2;
    }
    list("demoted", demoted);
    list("evict", plan.evictions);
    list("swapin", plan.swap_ins);
    list("immediate", plan.immediate_swap_ins);
    list("denied", plan.denied);
    std::printf("kind %d prefill %ld\n", kind, kind == 1 ? plan.prefill_request : -1L);
    list("batch", kind == 2 ? plan.batch : std::vector<long>{});
    std::printf("used %ld %ld\n", st.gpu_used, st.cpu_used);
    std::printf("completion %a\n", completion);
    std::printf("swapev");
    for (auto& [id, t] : swap_events) std::printf(" %ld %a", id, t);
    std::printf("\n");
    // rec(d).blocked_interval_total += plan.duration, from 0
    std::printf("blocked %a\n", plan.denied.empty() ? 0.0 : 0.0 + plan.duration);
    std::printf("over %d\n", st.gpu_used > st.gpu_capacity ? 1 : 0);
    return 0;
}

// acceptance.cpp criterion 2's vectors (proj/tests/acceptance.cpp:168-216).
int select_vectors(const std::string& out) {
    std::vector<unsigned char> bytes;
    using instance::MonitorSnapshot;
    for (int pass = 0; pass < 2; ++pass) {  // 0: Alg. 1, 1: baseline argmin m
        for (int n = 1; n <= 4; ++n) {
            long combos = 1;
            for (int i = 0; i < n; ++i) combos *= 8;
            for (long code = 0; code < combos; ++code) {
                long c = code;
                std::vector<MonitorSnapshot> snaps(static_cast<std::size_t>(n));
                for (int i = 0; i < n; ++i) {
                    snaps[i].instance_id = i;
                    snaps[i].all_answering_on_track = (c % 2) != 0;
                    c /= 2;
                    snaps[i].total_kv = c % 4;
                    c /= 4;
                }
                int id = pass == 0 ? cluster::select_instance_reasoning(snaps)
                                   : cluster::route_arrival(snaps, instance::Policy::Fcfs);
                bytes.push_back(static_cast<unsigned char>(id));
            }
        }
    }
    for (int n = 1; n <= 4; ++n) {
        long combos = 1;
        for (int i = 0; i < n; ++i) combos *= 32;
        for (long code = 0; code < combos; ++code) {
            long c = code;
            std::vector<MonitorSnapshot> snaps(static_cast<std::size_t>(n));
            for (int i = 0; i < n; ++i) {
                snaps[i].instance_id = i;
                snaps[i].all_answering_on_track = (c % 2) != 0;
                c /= 2;
                snaps[i].reasoning_count = c % 4;
                c /= 4;
                snaps[i].fresh_answering_count = c % 4;
                c /= 4;
            }
            bytes.push_back(static_cast<unsigned char>(cluster::select_instance_answering(snaps)));
        }
    }
    FILE* f = std::fopen(out.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + out);
    std::fwrite(bytes.data(), 1, bytes.size(), f);
    std::fclose(f);
    return 0;
}

int usage() {
    std::fprintf(stderr, "usage: see header of oracle/ref_dump.cpp\n");
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    std::string mode = argv[1];
    try {
        if (mode == "gen" && argc == 10) {
            using workload::LengthDistribution;
            auto t = workload::generate_trace(
                std::strtol(argv[2], nullptr, 10), std::strtod(argv[3], nullptr),
                LengthDistribution::parse(argv[4]), LengthDistribution::parse(argv[5]),
                LengthDistribution::parse(argv[6]), std::strtoull(argv[7], nullptr, 10),
                std::atoi(argv[8]) != 0);
            write_hex_trace(t, argv[9]);
        } else if (mode == "mix" && argc == 7) {
            auto t = workload::mix_traces(read_hex_trace(argv[2]), read_hex_trace(argv[3]),
                                          std::strtod(argv[4], nullptr),
                                          std::strtoull(argv[5], nullptr, 10));
            write_hex_trace(t, argv[6]);
        } else if (mode == "run" && argc == 6) {
            auto t = read_hex_trace(argv[2]);
            Cfg c = read_cfg(argv[3]);
            std::ofstream log;
            std::ostream* logp = nullptr;
            if (std::strcmp(argv[5], "-") != 0) {
                log.open(argv[5]);
                logp = &log;
            }
            auto recs = engine::run(t, c.rc, c.prof, logp);
            FILE* f = std::fopen(argv[4], "w");
            if (!f) throw std::runtime_error("cannot write records");
            dump_records(recs, f);
            std::fclose(f);
        } else if (mode == "capacity" && argc == 4) {
            auto t = read_hex_trace(argv[2]);
            Cfg c = read_cfg(argv[3]);
            std::printf("%ld\n", engine::derive_capacity(t, c.rc, c.prof));
        } else if (mode == "time" && argc == 5) {
            auto t = read_hex_trace(argv[2]);
            Cfg c = read_cfg(argv[3]);
            int reps = std::atoi(argv[4]);
            using clk = std::chrono::steady_clock;
            auto t0 = clk::now();
            long cap = engine::derive_capacity(t, c.rc, c.prof);
            auto t1 = clk::now();
            engine::RunConfig rc = c.rc;
            rc.gpu_capacity = cap;  // run-only: capacity pre-derived
            double run_s = 0.0;
            for (int i = 0; i < reps; ++i) {
                auto a = clk::now();
                auto recs = engine::run(t, rc, c.prof);
                auto b = clk::now();
                run_s += std::chrono::duration<double>(b - a).count();
                if (recs.size() != t.size()) throw std::runtime_error("lost records");
            }
            std::printf("{\"capacity\": %ld, \"derive_s\": %.6f, \"run_s\": %.6f, \"reps\": %d}\n",
                        cap, std::chrono::duration<double>(t1 - t0).count(), run_s / reps, reps);
        } else if (mode == "sim" && argc == 4) {
            auto t = read_hex_trace(argv[2]);
            Cfg c = read_cfg(argv[3]);
            auto recs = engine::run(t, c.rc, c.prof);
            auto rep = metrics::build_report(recs, c.rc.target_tpot, c.rc.qoe_threshold,
                                             c.rc.ttfat_target);
            std::printf("%zu %a %a %a\n", recs.size(), rep.ttft_p99, rep.slo_violation_rate,
                        rep.ttft_mean);
        } else if (mode == "all" && argc == 7) {
            using clk = std::chrono::steady_clock;
            auto t = read_hex_trace(argv[2]);
            Cfg c = read_cfg(argv[3]);
            auto t0 = clk::now();
            const long cap = engine::derive_capacity(t, c.rc, c.prof);
            auto t1 = clk::now();
            engine::RunConfig rc = c.rc;
            rc.gpu_capacity = cap;
            Sink ev(argv[5]);
            FileBuf eb(ev.f);
            std::ostream evs(&eb);
            auto recs = engine::run(t, rc, c.prof, ev.f ? &evs : nullptr);
            evs.flush();
            auto t2 = clk::now();
            {
                Sink rs(argv[4]);
                if (rs.f) dump_records(recs, rs.f);
            }
            auto rep = metrics::build_report(recs, c.rc.target_tpot, c.rc.qoe_threshold,
                                             c.rc.ttfat_target);
            rep.config_echo = {
                {"policy", c.policy},
                {"instance_count", std::to_string(c.rc.instance_count)},
                {"gpu_capacity", std::to_string(cap)},
                {"token_quantum", std::to_string(c.rc.token_quantum)},
                {"demotion_threshold", std::to_string(c.rc.demotion_threshold)},
                {"no_migration", std::to_string(c.rc.ablations.no_migration)},
                {"non_adaptive", std::to_string(c.rc.ablations.non_adaptive)},
                {"requests", std::to_string(t.size())},
            };
            metrics::write_report(rep, argv[6]);
            std::printf("{\"capacity\": %ld, \"derive_s\": %.3f, \"run_s\": %.3f}\n", cap,
                        std::chrono::duration<double>(t1 - t0).count(),
                        std::chrono::duration<double>(t2 - t1).count());
        } else if (mode == "plan" && argc == 3) {
            return plan_state(argv[2]);
        } else if (mode == "select" && argc == 3) {
            return select_vectors(argv[2]);
        } else if (mode == "report" && argc == 5) {
            auto t = read_hex_trace(argv[2]);
            Cfg c = read_cfg(argv[3]);
            auto recs = engine::run(t, c.rc, c.prof);
            auto rep = metrics::build_report(recs, c.rc.target_tpot, c.rc.qoe_threshold,
                                             c.rc.ttfat_target);
            metrics::write_report(rep, argv[4]);
        } else {
            return usage();
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_dump: %s\n", e.what());
        return 1;
    }
    return 0;
}
