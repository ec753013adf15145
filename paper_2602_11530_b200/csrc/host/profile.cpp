// profile.cpp — latency profiles (pascal-profile-v1) and decode-step
// calibration. Off the hot path; kept so the 19-symbol ABI is complete
// (SURVEY.md §8f row 4). Behaviour follows proj/src/costmodel.cpp:21-33
// (validation), :53-98 (least squares), :100-182 (file formats).
#include <array>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>

#include "common.hpp"

namespace pbh {

pb::Profile default_profile() {  // proj/include/pascalsim/costmodel.hpp:12-21
    pb::Profile p;
    p.prefill_base = 0.0;
    p.prefill_per_token = 0.00025;
    p.decode_base = 0.03;
    p.decode_per_request = 0.0;
    p.decode_per_kv_token = 0.0;
    p.swap_bandwidth = 51200.0;
    p.fabric_bandwidth = 51200.0;
    p.fabric_latency = 0.0;
    return p;
}

void check_profile(const pb::Profile& p) {
    const std::pair<double, const char*> nonneg[] = {
        {p.prefill_base, "prefill_base"},
        {p.prefill_per_token, "prefill_per_token"},
        {p.decode_base, "decode_base"},
        {p.decode_per_request, "decode_per_request"},
        {p.decode_per_kv_token, "decode_per_kv_token"},
        {p.fabric_latency, "fabric_latency"},
    };
    for (const auto& [v, name] : nonneg)
        if (!(v >= 0.0)) throw std::invalid_argument(std::string(name) + " must be >= 0");
    if (!(p.swap_bandwidth > 0.0)) throw std::invalid_argument("swap_bandwidth must be > 0");
    if (!(p.fabric_bandwidth > 0.0)) throw std::invalid_argument("fabric_bandwidth must be > 0");
}

namespace {
struct Field {
    const char* key;
    double pb::Profile::*ptr;
};
constexpr Field kFields[] = {
    {"prefill_base", &pb::Profile::prefill_base},
    {"prefill_per_token", &pb::Profile::prefill_per_token},
    {"decode_base", &pb::Profile::decode_base},
    {"decode_per_request", &pb::Profile::decode_per_request},
    {"decode_per_kv_token", &pb::Profile::decode_per_kv_token},
    {"swap_bandwidth", &pb::Profile::swap_bandwidth},
    {"fabric_bandwidth", &pb::Profile::fabric_bandwidth},
    {"fabric_latency", &pb::Profile::fabric_latency},
};
}  // namespace

void set_profile_field(pb::Profile& p, const std::string& key, double v) {
    for (const Field& f : kFields)
        if (key == f.key) {
            p.*(f.ptr) = v;
            return;
        }
    throw std::invalid_argument("unknown profile field: " + key);
}

pb::Profile read_profile(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open profile file: " + path);
    std::string line;
    if (!std::getline(in, line) || std::string(strip(line)) != "pascal-profile-v1")
        throw std::runtime_error(path + ":1: expected header 'pascal-profile-v1'");
    pb::Profile p = default_profile();
    long no = 1;
    while (std::getline(in, line)) {
        ++no;
        std::string_view body = strip(line);
        if (body.empty() || body.front() == '#') continue;
        auto kv = cut(body, '=');
        if (kv.size() != 2)
            throw std::runtime_error(path + ":" + std::to_string(no) + ": expected key=value");
        try {
            std::string key(strip(kv[0]));
            set_profile_field(p, key, to_double(kv[1], key));
        } catch (const std::exception& e) {
            throw std::runtime_error(path + ":" + std::to_string(no) + ": " + e.what());
        }
    }
    check_profile(p);
    return p;
}

void write_profile(const pb::Profile& p, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("cannot open profile file for writing: " + path);
    std::fputs("pascal-profile-v1\n", f);
    for (const Field& fd : kFields) {
        double v = p.*(fd.ptr);
        if (std::isinf(v)) std::fprintf(f, "%s=inf\n", fd.key);
        else std::fprintf(f, "%s=%.12g\n", fd.key, v);
    }
    if (std::fclose(f) != 0) throw std::runtime_error("write failed: " + path);
}

// Least-squares plane step = c0 + c1*batch + c2*kv through the 3x3 normal
// equations, Gauss-Jordan with partial pivoting (costmodel.cpp:53-98).
Fit calibrate_file(const std::string& samples_path) {
    std::ifstream in(samples_path);
    if (!in) throw std::runtime_error("cannot open calibration file: " + samples_path);
    struct S {
        long b, kv;
        double y;
    };
    std::vector<S> xs;
    std::string line;
    long no = 0;
    while (std::getline(in, line)) {
        ++no;
        std::string_view body = strip(line);
        if (body.empty() || body.front() == '#') continue;
        auto f = cut(body, ',');
        if (f.size() != 3)
            throw std::runtime_error(samples_path + ":" + std::to_string(no) +
                                     ": expected batch,kv,seconds");
        xs.push_back({to_long(f[0], "batch"), to_long(f[1], "kv"), to_double(f[2], "seconds")});
    }
    if (xs.size() < 3) throw std::invalid_argument("calibrate: need at least 3 samples");
    std::array<std::array<double, 4>, 3> m{};
    for (const S& s : xs) {
        const double x[3] = {1.0, static_cast<double>(s.b), static_cast<double>(s.kv)};
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) m[r][c] += x[r] * x[c];
            m[r][3] += x[r] * s.y;
        }
    }
    for (int col = 0; col < 3; ++col) {
        int piv = col;
        for (int r = col + 1; r < 3; ++r)
            if (std::abs(m[r][col]) > std::abs(m[piv][col])) piv = r;
        std::swap(m[col], m[piv]);
        if (std::abs(m[col][col]) < 1e-12)
            throw std::invalid_argument(
                "calibrate: rank-deficient sample set; vary batch size and KV totals");
        for (int r = 0; r < 3; ++r) {
            if (r == col) continue;
            const double k = m[r][col] / m[col][col];
            for (int c = col; c < 4; ++c) m[r][c] -= k * m[col][c];
        }
    }
    Fit fit;
    fit.base = m[0][3] / m[0][0];
    fit.per_req = m[1][3] / m[1][1];
    fit.per_kv = m[2][3] / m[2][2];
    double sq = 0.0;
    for (const S& s : xs) {
        const double e = fit.base + fit.per_req * static_cast<double>(s.b) +
                         fit.per_kv * static_cast<double>(s.kv) - s.y;
        sq += e * e;
    }
    fit.rmse = std::sqrt(sq / static_cast<double>(xs.size()));
    return fit;
}

int parse_policy(const std::string& name) {
    if (name == "fcfs") return pb::kFcfs;
    if (name == "rr") return pb::kRr;
    if (name == "oracle") return pb::kOracle;
    if (name == "pascal") return pb::kPascal;
    throw std::invalid_argument("unknown policy: '" + name + "'");
}

}  // namespace pbh
