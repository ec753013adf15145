// report.cpp — pascal-report-v1 files, tail-TTFT bins and report comparison.
// Host post-processing of the per-request rows the GPU produced (SURVEY.md
// §8f row 2). Byte formats follow proj/src/metrics.cpp:155-205 (writer),
// :207-263 (loader), :85-113 (bins), :265-323 (compare).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>

#include "common.hpp"

namespace pbh {

namespace {
constexpr long kBinWidth = 256;

double nearest_rank_sorted(const std::vector<double>& v, double pct) {
    size_t rank = static_cast<size_t>(std::ceil(pct * static_cast<double>(v.size())));
    rank = std::max<size_t>(rank, 1);
    rank = std::min(rank, v.size());
    return v[rank - 1];
}

void put_atomic(const std::string& path, const std::string& text) {
    const std::string tmp = path + ".tmp";
    {
        std::ofstream out(tmp);
        if (!out) throw std::runtime_error("cannot open for writing: " + tmp);
        out << text;
        if (!out) throw std::runtime_error("write failed: " + tmp);
    }
    std::filesystem::rename(tmp, path);
}

std::string fmt(const char* f, ...) __attribute__((format(printf, 1, 2)));
std::string fmt(const char* f, ...) {
    char buf[320];
    va_list ap;
    va_start(ap, f);
    std::vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}
}  // namespace

std::vector<Bin> tail_bins(const std::vector<std::pair<long, double>>& rows) {
    std::map<long, std::vector<double>> groups;
    for (const auto& [reasoning, ttft] : rows) groups[reasoning / kBinWidth].push_back(ttft);
    std::vector<Bin> out;
    for (auto& [key, vals] : groups) {
        if (vals.size() < 5) continue;
        std::sort(vals.begin(), vals.end());
        Bin b;
        b.lo = key * kBinWidth;
        b.hi = b.lo + kBinWidth - 1;
        b.count = static_cast<long>(vals.size());
        const size_t n = vals.size();
        if (n < 10) {
            b.stat = "max";
            b.value = vals.back();
        } else {
            const double pct = n < 20 ? 0.90 : n < 100 ? 0.95 : 0.99;
            b.stat = n < 20 ? "p90" : n < 100 ? "p95" : "p99";
            b.value = nearest_rank_sorted(vals, pct);
        }
        out.push_back(b);
    }
    return out;
}

void write_report(const Report& r, const std::string& prefix) {
    std::string req = "pascal-report-v1\n";
    req += "id,reasoning_tokens,answering_tokens,ttft,ttfat,qoe,slo_violated,blocking_latency\n";
    for (const Row& w : r.rows)
        req += fmt("%ld,%ld,%ld,%.9f,%.9f,%.9f,%d,%.9f\n", w.id, w.reasoning, w.answering, w.ttft,
                   w.ttfat, w.qoe, w.slo ? 1 : 0, w.blocking);
    put_atomic(prefix + ".requests.csv", req);

    std::string sum = "pascal-report-v1\n";
    for (const auto& [k, v] : r.echo) sum += k + "=" + v + "\n";
    const std::pair<const char*, double> keys[] = {
        {"ttft_mean", r.ttft_mean}, {"ttft_p50", r.ttft_p50},
        {"ttft_p90", r.ttft_p90},   {"ttft_p95", r.ttft_p95},
        {"ttft_p99", r.ttft_p99},   {"slo_violation_rate", r.slo_rate},
        {"ttfat_attainment", r.ttfat_attain}, {"throughput", r.throughput},
    };
    for (const auto& [k, v] : keys) sum += fmt("%s=%.9f\n", k, v);
    put_atomic(prefix + ".summary.txt", sum);

    std::string bins = "pascal-report-v1\nbin_lo,bin_hi,n,stat_kind,value\n";
    for (const Bin& b : r.bins)
        bins += fmt("%ld,%ld,%ld,%s,%.9f\n", b.lo, b.hi, b.count, b.stat.c_str(), b.value);
    put_atomic(prefix + ".bins.csv", bins);
}

Report read_report(const std::string& prefix) {
    Report rep;
    {
        const std::string path = prefix + ".requests.csv";
        std::ifstream in(path);
        if (!in) throw std::runtime_error("cannot open report file: " + path);
        std::string line;
        if (!std::getline(in, line) || std::string(strip(line)) != "pascal-report-v1")
            throw std::runtime_error(path + ": bad or missing version header");
        std::getline(in, line);
        long no = 2;
        while (std::getline(in, line)) {
            ++no;
            std::string_view body = strip(line);
            if (body.empty()) continue;
            auto f = cut(body, ',');
            if (f.size() != 8)
                throw std::runtime_error(path + ":" + std::to_string(no) + ": expected 8 fields");
            Row w;
            w.id = to_long(f[0], "id");
            w.reasoning = to_long(f[1], "reasoning_tokens");
            w.answering = to_long(f[2], "answering_tokens");
            w.ttft = to_double(f[3], "ttft");
            w.ttfat = to_double(f[4], "ttfat");
            w.qoe = to_double(f[5], "qoe");
            w.slo = to_long(f[6], "slo_violated") != 0;
            w.blocking = to_double(f[7], "blocking_latency");
            rep.rows.push_back(w);
        }
    }
    {
        const std::string path = prefix + ".summary.txt";
        std::ifstream in(path);
        if (!in) throw std::runtime_error("cannot open report file: " + path);
        std::string line;
        std::getline(in, line);
        std::map<std::string, double*> dst = {
            {"ttft_mean", &rep.ttft_mean}, {"ttft_p50", &rep.ttft_p50},
            {"ttft_p90", &rep.ttft_p90},   {"ttft_p95", &rep.ttft_p95},
            {"ttft_p99", &rep.ttft_p99},   {"slo_violation_rate", &rep.slo_rate},
            {"ttfat_attainment", &rep.ttfat_attain}, {"throughput", &rep.throughput},
        };
        while (std::getline(in, line)) {
            auto kv = cut(strip(line), '=');
            if (kv.size() != 2) continue;
            std::string key(strip(kv[0])), val(strip(kv[1]));
            auto it = dst.find(key);
            if (it != dst.end()) *it->second = to_double(val, key);
            else rep.echo.emplace_back(key, val);
        }
    }
    std::vector<std::pair<long, double>> pts;
    for (const Row& w : rep.rows) pts.emplace_back(w.reasoning, w.ttft);
    rep.bins = tail_bins(pts);
    return rep;
}

std::string compare_text(const std::vector<Report>& reps, const std::vector<std::string>& names) {
    if (reps.size() < 2) throw std::invalid_argument("compare: need at least 2 reports");
    const Report& base = reps.front();
    for (size_t i = 1; i < reps.size(); ++i) {
        const Report& o = reps[i];
        bool same = o.rows.size() == base.rows.size();
        for (size_t j = 0; same && j < base.rows.size(); ++j)
            same = base.rows[j].id == o.rows[j].id &&
                   base.rows[j].reasoning == o.rows[j].reasoning &&
                   base.rows[j].answering == o.rows[j].answering;
        if (!same) throw std::invalid_argument("compare: reports cover different traces");
    }
    std::string out = "comparison vs " + names.front() + "\n\n";
    out += "tail TTFT per reasoning-length bin (value, delta%)\nbin_lo,bin_hi,stat";
    for (const auto& n : names) out += "," + n;
    out += "\n";
    for (const Bin& b : base.bins) {
        out += fmt("%ld,%ld,%s,%.4f", b.lo, b.hi, b.stat.c_str(), b.value);
        for (size_t i = 1; i < reps.size(); ++i) {
            const Bin* hit = nullptr;
            for (const Bin& ob : reps[i].bins)
                if (ob.lo == b.lo) hit = &ob;
            if (hit && b.value > 0.0)
                out += fmt(",%.4f (%+.1f%%)", hit->value, 100.0 * (hit->value - b.value) / b.value);
            else
                out += ",-";
        }
        out += "\n";
    }
    out += "\naggregates\nmetric";
    for (const auto& n : names) out += "," + n;
    out += "\n";
    const std::pair<const char*, double Report::*> aggs[] = {
        {"slo_violation_rate", &Report::slo_rate},
        {"throughput", &Report::throughput},
        {"ttft_p50", &Report::ttft_p50},
        {"ttft_p99", &Report::ttft_p99},
    };
    for (const auto& [label, field] : aggs) {
        out += label;
        for (const Report& r : reps) out += fmt(",%.6f", r.*field);
        out += "\n";
    }
    return out;
}

}  // namespace pbh
