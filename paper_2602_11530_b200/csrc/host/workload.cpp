// workload.cpp — synthetic traces and trace files (host side, feeds the GPU).
//
// Must reproduce the reference generator bit for bit so parity runs see the
// same inputs: std::mt19937_64, 53-bit uniforms,
// `rng() % span` integers, glibc log1p for Poisson gaps
// (proj/src/workload.cpp:24-32,140-162), partial Fisher-Yates mixing
// (:164-198), validation (:200-219) and the pascal-trace-v1 text format
// (:221-274).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <numeric>
#include <sstream>
#include <unordered_set>

#include "common.hpp"

namespace pbh {

// ------------------------------------------------------------ text helpers
std::string_view strip(std::string_view s) {
    auto ws = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
    size_t a = 0, b = s.size();
    while (a < b && ws(s[a])) ++a;
    while (b > a && ws(s[b - 1])) --b;
    return s.substr(a, b - a);
}

std::vector<std::string_view> cut(std::string_view s, char sep) {
    std::vector<std::string_view> parts;
    size_t from = 0;
    while (true) {
        size_t at = s.find(sep, from);
        if (at == std::string_view::npos) {
            parts.push_back(s.substr(from));
            return parts;
        }
        parts.push_back(s.substr(from, at - from));
        from = at + 1;
    }
}

long to_long(std::string_view s, const std::string& what) {
    s = strip(s);
    long v = 0;
    const char* end = s.data() + s.size();
    auto res = std::from_chars(s.data(), end, v);
    if (res.ec != std::errc() || res.ptr != end)
        throw std::invalid_argument("invalid integer for " + what + ": '" + std::string(s) + "'");
    return v;
}

double to_double(std::string_view s, const std::string& what) {
    s = strip(s);
    if (s == "inf") return std::numeric_limits<double>::infinity();
    double v = 0;
    const char* end = s.data() + s.size();
    auto res = std::from_chars(s.data(), end, v);
    if (res.ec != std::errc() || res.ptr != end)
        throw std::invalid_argument("invalid number for " + what + ": '" + std::string(s) + "'");
    return v;
}

// ------------------------------------------------------------ distributions
namespace {
double unit53(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
}  // namespace

LengthDist LengthDist::parse(const std::string& spec) {
    auto parts = cut(spec, ':');
    const std::string kind(strip(parts[0]));
    LengthDist d;
    if (kind == "constant") {
        if (parts.size() != 2) throw std::invalid_argument("constant distribution needs one value");
        d.kind_ = Kind::Constant;
        d.value_ = to_long(parts[1], "constant value");
        return d;
    }
    if (kind == "uniform") {
        if (parts.size() != 3) throw std::invalid_argument("uniform distribution needs low:high");
        d.kind_ = Kind::Uniform;
        d.lo_ = to_long(parts[1], "uniform low");
        d.hi_ = to_long(parts[2], "uniform high");
        if (d.lo_ > d.hi_) throw std::invalid_argument("uniform distribution: low > high");
        return d;
    }
    if (kind == "hist") {
        if (parts.size() != 2)
            throw std::invalid_argument("hist distribution needs value=weight pairs");
        d.kind_ = Kind::Hist;
        for (auto item : cut(parts[1], ',')) {
            auto vw = cut(item, '=');
            if (vw.size() != 2) throw std::invalid_argument("hist entry must be value=weight");
            d.bins_.emplace_back(to_long(vw[0], "hist value"), to_double(vw[1], "hist weight"));
        }
        if (d.bins_.empty()) throw std::invalid_argument("histogram distribution: no bins");
        double sum = 0.0;
        for (const auto& b : d.bins_) {
            if (b.second < 0.0) throw std::invalid_argument("histogram distribution: negative weight");
            sum += b.second;
        }
        if (sum <= 0.0) throw std::invalid_argument("histogram distribution: all weights zero");
        double run = 0.0;
        for (const auto& b : d.bins_) {
            run += b.second / sum;
            d.cdf_.push_back(run);
        }
        d.cdf_.back() = 1.0;
        return d;
    }
    throw std::invalid_argument("unknown distribution kind: '" + kind + "'");
}

long LengthDist::draw(std::mt19937_64& g) const {
    if (kind_ == Kind::Constant) return value_;
    if (kind_ == Kind::Uniform) {
        unsigned long long span = static_cast<unsigned long long>(hi_ - lo_) + 1ull;
        return lo_ + static_cast<long>(g() % span);
    }
    double u = unit53(g);
    size_t k = static_cast<size_t>(std::lower_bound(cdf_.begin(), cdf_.end(), u) - cdf_.begin());
    return bins_[std::min(k, bins_.size() - 1)].first;
}

long LengthDist::lowest() const {
    if (kind_ == Kind::Constant) return value_;
    if (kind_ == Kind::Uniform) return lo_;
    long m = std::numeric_limits<long>::max();
    for (const auto& b : bins_)
        if (b.second > 0.0) m = std::min(m, b.first);
    return m;
}

// ------------------------------------------------------------ generation
Trace generate(long count, double rate, const LengthDist& p, const LengthDist& r,
               const LengthDist& a, std::uint64_t seed, bool preloaded) {
    if (count < 0) throw std::invalid_argument("count must be >= 0");
    if (rate <= 0.0) throw std::invalid_argument("arrival_rate must be > 0");
    if (p.lowest() < 1)
        throw std::invalid_argument("prompt_tokens distribution can produce values < 1");
    if (r.lowest() < 0)
        throw std::invalid_argument("reasoning_tokens distribution can produce values < 0");
    if (a.lowest() < 1)
        throw std::invalid_argument("answering_tokens distribution can produce values < 1");
    std::mt19937_64 g(seed);
    Trace t(static_cast<size_t>(count));
    double clock = 0.0;
    for (long i = 0; i < count; ++i) {
        Spec& s = t[static_cast<size_t>(i)];
        clock += -std::log1p(-unit53(g)) / rate;  // exponential gap; first arrival after one gap
        s.id = i;
        s.arrival = clock;
        s.prompt = p.draw(g);
        s.reasoning = r.draw(g);
        s.answering = a.draw(g);
        s.preloaded = preloaded;
    }
    check_trace(t);
    return t;
}

Trace mix(const Trace& base, const Trace& repl, double fraction, std::uint64_t seed) {
    if (fraction < 0.0 || fraction > 1.0) throw std::invalid_argument("fraction must be in [0,1]");
    if (fraction > 0.0 && fraction < 1.0 && (base.empty() || repl.empty()))
        throw std::invalid_argument("mix_traces: both traces must be non-empty");
    if (fraction > 0.0 && repl.empty())
        throw std::invalid_argument("mix_traces: replacement trace is empty");
    Trace out = base;
    const size_t k = static_cast<size_t>(std::floor(fraction * static_cast<double>(base.size())));
    if (k == 0) return out;
    std::mt19937_64 g(seed);
    std::vector<size_t> pick(base.size());
    std::iota(pick.begin(), pick.end(), size_t{0});
    for (size_t i = 0; i < k; ++i) std::swap(pick[i], pick[i + g() % (pick.size() - i)]);
    for (size_t i = 0; i < k; ++i) {
        const Spec& from = repl[g() % repl.size()];
        Spec& to = out[pick[i]];
        to.prompt = from.prompt;
        to.reasoning = from.reasoning;
        to.answering = from.answering;
        to.preloaded = from.preloaded;
    }
    std::sort(out.begin(), out.end(), [](const Spec& x, const Spec& y) {
        return x.arrival < y.arrival || (x.arrival == y.arrival && x.id < y.id);
    });
    return out;
}

void check_trace(const Trace& t) {
    // duplicate-id check: a bitmap when ids are small (generated traces use
    // 0..n-1), a hash set otherwise
    long max_id = -1;
    for (const Spec& s : t) max_id = std::max(max_id, s.id);
    const bool dense = max_id < 4 * (long)t.size() + 64;
    std::vector<unsigned char> seen_bits(dense ? (size_t)(max_id + 1) : 0, 0);
    std::unordered_set<long> seen;
    if (!dense) seen.reserve(t.size() * 2);
    double last_arrival = -1.0;
    long last_id = -1;
    for (const Spec& s : t) {
        auto bad = [&](const char* msg) {
            throw std::invalid_argument(std::string(msg) + " (request " + std::to_string(s.id) + ")");
        };
        if (s.id < 0) bad("id must be non-negative");
        if (s.arrival < 0.0) bad("arrival_time must be >= 0");
        if (s.prompt < 1) bad("prompt_tokens must be >= 1");
        if (s.reasoning < 0) bad("reasoning_tokens must be >= 0");
        if (s.answering < 1) bad("answering_tokens must be >= 1");
        if (dense ? seen_bits[(size_t)s.id]++ != 0 : !seen.insert(s.id).second) bad("duplicate id");
        if (s.arrival < last_arrival || (s.arrival == last_arrival && s.id < last_id))
            bad("trace not sorted by (arrival_time, id)");
        last_arrival = s.arrival;
        last_id = s.id;
    }
}

// ------------------------------------------------------------ trace files
void write_trace(const Trace& t, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("cannot open trace file for writing: " + path);
    bool ok = std::fputs("pascal-trace-v1\n", f) >= 0;
    for (const Spec& s : t)
        ok = ok && std::fprintf(f, "%ld,%.9f,%ld,%ld,%ld,%d\n", s.id, s.arrival, s.prompt,
                                s.reasoning, s.answering, s.preloaded ? 1 : 0) > 0;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("write failed: " + path);
}

Trace read_trace(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open trace file: " + path);
    std::string line;
    if (!std::getline(in, line)) return {};
    if (std::string(strip(line)) != "pascal-trace-v1")
        throw std::runtime_error(path + ":1: expected header 'pascal-trace-v1'");
    Trace t;
    long no = 1;
    while (std::getline(in, line)) {
        ++no;
        std::string_view body = strip(line);
        if (body.empty()) continue;
        try {
            auto f = cut(body, ',');
            if (f.size() != 5 && f.size() != 6) throw std::invalid_argument("expected 5 or 6 fields");
            Spec s;
            s.id = to_long(f[0], "id");
            s.arrival = to_double(f[1], "arrival_time");
            s.prompt = to_long(f[2], "prompt_tokens");
            s.reasoning = to_long(f[3], "reasoning_tokens");
            s.answering = to_long(f[4], "answering_tokens");
            if (f.size() == 6) s.preloaded = to_long(f[5], "kv_preloaded") != 0;
            t.push_back(s);
        } catch (const std::exception& e) {
            throw std::runtime_error(path + ":" + std::to_string(no) + ": " + e.what());
        }
    }
    try {
        check_trace(t);
    } catch (const std::exception& e) {
        throw std::runtime_error(path + ": " + e.what());
    }
    return t;
}

void write_trace_hex(const Trace& t, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("cannot open trace file for writing: " + path);
    std::fputs("pascal-trace-hex-v1\n", f);
    for (const Spec& s : t)
        std::fprintf(f, "%ld %a %ld %ld %ld %d\n", s.id, s.arrival, s.prompt, s.reasoning,
                     s.answering, s.preloaded ? 1 : 0);
    if (std::fclose(f) != 0) throw std::runtime_error("write failed: " + path);
}

Trace read_trace_hex(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open trace file: " + path);
    std::string line;
    if (!std::getline(in, line) || std::string(strip(line)) != "pascal-trace-hex-v1")
        throw std::runtime_error(path + ":1: expected header 'pascal-trace-hex-v1'");
    Trace t;
    while (std::getline(in, line)) {
        if (strip(line).empty()) continue;
        std::istringstream ls(line);
        std::string arr;
        Spec s;
        int pre = 0;
        if (!(ls >> s.id >> arr >> s.prompt >> s.reasoning >> s.answering >> pre))
            throw std::runtime_error(path + ": malformed line");
        s.arrival = std::strtod(arr.c_str(), nullptr);
        s.preloaded = pre != 0;
        t.push_back(s);
    }
    try {
        check_trace(t);
    } catch (const std::exception& e) {
        throw std::runtime_error(path + ": " + e.what());
    }
    return t;
}

long long request_iterations(const Trace& t) {
    long long n = 0;
    for (const Spec& s : t)
        n += s.reasoning + s.answering - ((s.reasoning == 0 && !s.preloaded) ? 1 : 0) +
             (s.preloaded ? 0 : 1);
    return n;
}

}  // namespace pbh
