// engine_host.cpp — host driver of the device scheduling engine.
//
// Packs traces into the struct-of-arrays layout of engine.h, owns the device
// arenas, launches (1) the oracle pre-run for capacity derivation
// (proj/src/engine.cpp:449-471), (2) the capacity kernel, (3) the policy run,
// (4) the metric kernels — all on one stream with no host round trip in
// between — and fetches summaries, per-request rows, records and the decision
// log. There is no CPU execution path: without a CUDA device every run fails
// with PASCAL_ERR_INTERNAL.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <climits>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <exception>
#include <thread>
#include <unordered_map>

#include "common.hpp"

namespace pbh {

namespace {

thread_local Timing g_timing;

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::logic_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// Switches the calling thread to `dev` for a scope and restores the
// previous device after it.
struct ScopedDevice {
    int prev = -1;
    explicit ScopedDevice(int dev) {
        if (dev < 0) return;
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~ScopedDevice() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Device allocations are cached per device for the life of the process: a
// batch of thousands of replicas allocates ~20 arenas of up to GBs, and
// cudaMalloc / cudaFree of those cost 0.3-1 s per end-to-end call against a
// ~5.7 s simulation. Freed blocks are reused for requests of up to 2x smaller
// size; on an out-of-memory the cache is released and the allocation retried.
// Every block remembers the device it was allocated on and returns to that
// device's free list whatever device is current when it is released. The
// cache is bounded (PB_POOL_CACHE_MB, default 16 GiB per device of idle
// blocks; the largest idle blocks are released first) and can be released
// explicitly (pascal_release_cached_memory).
class DevicePool {
public:
    void* get(size_t bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        bytes = round(bytes);
        {
            std::lock_guard<std::mutex> g(m_);
            auto& fl = free_[dev];
            auto it = fl.lower_bound(bytes);
            if (it != fl.end() && it->first <= 2 * bytes) {
                void* p = it->second;
                live_[p] = Block{it->first, dev};
                idle_bytes_[dev] -= it->first;
                fl.erase(it);
                return p;
            }
        }
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            trim(dev);
            ck(cudaMalloc(&p, bytes), "cudaMalloc");
        }
        std::lock_guard<std::mutex> g(m_);
        live_[p] = Block{bytes, dev};
        return p;
    }
    void put(void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> g(m_);
        auto it = live_.find(p);
        if (it == live_.end()) return;
        const Block b = it->second;
        live_.erase(it);
        free_[b.dev].emplace(b.bytes, p);
        idle_bytes_[b.dev] += b.bytes;
        // bound the idle cache: release the largest idle blocks first
        auto& fl = free_[b.dev];
        while (idle_bytes_[b.dev] > cap_bytes() && !fl.empty()) {
            auto last = std::prev(fl.end());
            ScopedDevice sd(b.dev);
            cudaFree(last->second);
            idle_bytes_[b.dev] -= last->first;
            fl.erase(last);
        }
    }
    void trim(int dev) {
        std::lock_guard<std::mutex> g(m_);
        trim_locked(dev);
    }
    void trim_all() {
        std::lock_guard<std::mutex> g(m_);
        for (auto& kv : free_) trim_locked(kv.first);
    }

private:
    struct Block {
        size_t bytes;
        int dev;
    };
    void trim_locked(int dev) {
        ScopedDevice sd(dev);
        for (auto& kv : free_[dev]) cudaFree(kv.second);
        free_[dev].clear();
        idle_bytes_[dev] = 0;
    }
    static size_t cap_bytes() {
        static const size_t cap = [] {
            const char* e = std::getenv("PB_POOL_CACHE_MB");
            const long long mb = e ? std::atoll(e) : 16384;
            return (size_t)std::max<long long>(0, mb) << 20;
        }();
        return cap;
    }
    static size_t round(size_t b) {
        static const int mode = std::getenv("PB_POOL_ROUND") ? std::atoi(std::getenv("PB_POOL_ROUND")) : 1;
        if (mode == 0) return std::max<size_t>(b, 1);
        const size_t q = b >= (64u << 20) ? (2u << 20) : (b >= (1u << 20) ? (64u << 10) : 512);
        return (std::max<size_t>(b, 1) + q - 1) / q * q;
    }
    static void ck(cudaError_t e, const char* what) {
        if (e != cudaSuccess)
            throw std::logic_error(std::string("CUDA error in ") + what + ": " +
                                   cudaGetErrorString(e));
    }
    std::mutex m_;
    std::map<int, std::multimap<size_t, void*>> free_;
    std::map<int, size_t> idle_bytes_;
    std::unordered_map<void*, Block> live_;
};

DevicePool& pool() {
    static DevicePool* p = new DevicePool;  // never destroyed: outlives every batch
    return *p;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { pool().put(p); }
    void ensure(size_t count) {
        if (count <= n && p) return;
        pool().put(p);
        p = nullptr;
        n = 0;
        size_t c = std::max<size_t>(count, 1);
        p = static_cast<T*>(pool().get(c * sizeof(T)));
        n = c;
    }
};

// Launch shape. One warp per replica. The replica's hot request state and
// the planner's candidate scratch go to shared memory when they fit (60 B per
// request + 37 B per candidate slot); otherwise they stay in HBM. Few
// replicas -> one warp per CTA so they spread over all SMs; many -> up to four
// per CTA, as many as the shared-memory budget allows.
struct Shape {
    int n_smem, c_smem, wpb, blocks, h_slots, b_smem;
};

Shape pick_shape(int reps, int max_ni, int max_n) {
    int dev = 0, sms = 148, optin = 0, per_sm_smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const int budget = std::max(48 * 1024, optin) - 1024;  // per CTA
    const int sm_budget = std::max(budget, per_sm_smem - 2048);
    // Measured on C2 replicas (HBM/L2-resident request state): 8 warps per SM
    // (unconstrained registers) beats 12 and 16 (register-capped variants
    // spill around the out-of-line calls, and more concurrent replicas
    // overflow L2); more replicas than warps are work-stolen.
    const char* menv = std::getenv("PB_MAX_WARPS_PER_SM");
    const int kMaxWarpsPerSm = menv ? std::max(1, std::min(16, std::atoi(menv))) : 8;
    const char* env = std::getenv("PB_SMEM");
    const int mode = env ? std::atoi(env) : -1;  // 0: HBM request state, 1: shared, -1: auto
    const char* henv = std::getenv("PB_SMEM_HEAP");  // test hook: tiny heap forces HBM spills
    const int h_slots = henv ? std::max(2, std::atoi(henv)) : pb::kSmemHeapSlots;
    const int need_w = std::max(1, std::min(kMaxWarpsPerSm, (reps + sms - 1) / std::max(1, sms)));
    auto warps_fit = [&](int per_warp) {
        return std::max(0, std::min(kMaxWarpsPerSm, sm_budget / std::max(1, per_warp)));
    };
    // A: request state + heap + candidate scratch in shared memory
    Shape a{max_n, std::min(max_n, 1024), 0, 0, h_slots, 0};
    int pa = pb::smem_per_warp(max_ni, a.n_smem, a.c_smem, h_slots);
    bool a_ok = pa <= budget && mode != 0;
    // B: request state in HBM (L2-resident), small shared candidate scratch
    const char* cenv = std::getenv("PB_CAND_SMEM");  // experiment hook: scratch slots
    Shape b{0, std::min(max_n, cenv ? std::max(32, std::atoi(cenv)) : 512), 0, 0, h_slots, 0};
    // blocked-time totals in shared memory when they fit beside a candidate
    // scratch of >= 256 slots at 8 warps per SM (C2: 2,000 requests = 16 KB)
    const char* benv = std::getenv("PB_BLOCKED_SMEM");  // experiment hook: 0 disables
    if (!benv || std::atoi(benv) != 0) {
        Shape t = b;
        t.b_smem = max_n;
        while (t.c_smem > 256 &&
               pb::smem_per_warp(max_ni, 0, t.c_smem, h_slots, t.b_smem) * 8 > sm_budget)
            t.c_smem /= 2;
        if (pb::smem_per_warp(max_ni, 0, t.c_smem, h_slots, t.b_smem) * 8 <= sm_budget) b = t;
    }
    while (b.c_smem > 32 &&
           pb::smem_per_warp(max_ni, 0, b.c_smem, h_slots, b.b_smem) * 8 > sm_budget)
        b.c_smem /= 2;
    int pbw = pb::smem_per_warp(max_ni, 0, b.c_smem, h_slots, b.b_smem);
    const bool use_a = a_ok && (mode == 1 || warps_fit(pa) >= std::min(need_w, 4));
    Shape sh = use_a ? a : b;
    const int per_warp = use_a ? pa : pbw;
    int w = std::max(1, std::min(need_w, warps_fit(per_warp)));
    if (const char* wenv = std::getenv("PB_WARPS_PER_SM"))  // experiment hook
        w = std::max(1, std::min(w, std::atoi(wenv)));
    // warps per CTA: the divisor of the per-SM warp count that keeps all w
    // warps resident (6 warps/SM = 2 CTAs of 3, not 1 CTA of 4)
    const int wpb_max = std::max(1, std::min({4, w, budget / per_warp}));
    sh.wpb = wpb_max;
    for (int c = wpb_max - 1; c >= 1; --c)
        if (c * (w / c) > sh.wpb * (w / sh.wpb)) sh.wpb = c;
    const int blocks_per_sm = std::max(1, w / sh.wpb);
    sh.blocks = std::max(1, std::min((reps + sh.wpb - 1) / sh.wpb, sms * blocks_per_sm));
    return sh;
}

constexpr long long kMaxReq = (1ll << 26) - 1;  // heap id field
constexpr int kMaxInst = 512;


void check_limits(const Job& j) {
    const RunCfg& c = j.cfg;
    if (c.instances < 1) throw std::invalid_argument("instance_count must be >= 1");
    if (c.instances > kMaxInst)
        throw std::invalid_argument("instance_count exceeds the device engine limit (512)");
    if ((long long)j.trace->size() > kMaxReq)
        throw std::invalid_argument("trace exceeds the device engine limit (2^26-1 requests)");
    if (!(c.tpot > 0.0)) throw std::invalid_argument("target_tpot must be > 0");
    for (const Spec& s : *j.trace)
        if (s.max_kv() >= (1l << 26) - 1)
            throw std::invalid_argument(
                "request KV footprint exceeds the device engine limit (2^26 - 2 tokens)");
}

}  // namespace

Timing& last_timing() { return g_timing; }

void release_cached_memory() { pool().trim_all(); }

bool device_available() {
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

void set_device(int dev) { ck(cudaSetDevice(dev), "cudaSetDevice"); }

const char* status_message(int st) {
    switch (st) {
        case pb::kErrPast: return "event scheduled in the past";
        case pb::kErrClock: return "clock moved backwards";
        case pb::kErrCapacity: return "instance over GPU capacity";
        case pb::kErrStall: return "simulation stalled with unfinished requests";
        case pb::kErrHeap: return "device event heap overflow";
        default: return "ok";
    }
}

// ------------------------------------------------------------------ Batch
class Batch {
public:
    explicit Batch(const std::vector<Job>& jobs);
    ~Batch();
    void execute();
    void fetch_summaries(std::vector<DeviceSummary>& out);
    void fetch_single(RunOutputs& o, bool records, bool log);
    void fetch_rows(std::vector<std::vector<Row>>& rows);
    void enable_log(long long cap) { log_cap_ = cap; }
    void enable_records() { records_ = true; }
    void build();

    std::vector<Job> jobs_;
    bool records_ = false;
    long long log_cap_ = 0;
    bool built_ = false;
    int dev_ = -1;  // the device the batch's arenas and stream live on

    int n_rep_ = 0, max_ni_ = 1, max_n_ = 0, max_on_ = 0;
    int pdes_w_ = 0;             // warps per replica of the instance-parallel engine (0: off)
    long long pheap_total_ = 0;  // per-instance heaps of the instance-parallel engine
    std::vector<int> declined_;  // replicas the instance-parallel engine handed back
    long long total_req_ = 0, total_ans_ = 0, total_q_ = 0, total_batch_ = 0, total_heap_ = 0,
              total_log_ = 0;
    std::vector<pb::ReplicaDesc> desc_;
    std::vector<pb::ReplicaDesc> odesc_;  // oracle pre-run descriptors
    std::vector<int> omap_, oref_, orep_, order_, oorder_;  // omap_/oref_: replica -> its pre-run
    std::vector<long long> echo_static_;

    cudaStream_t st_ = nullptr;
    cudaEvent_t ev_[5] = {};
    DevBuf<pb::ReplicaDesc> d_desc_, d_odesc_, d_desc_init_;
    DevBuf<pb::ReplicaOut> d_out_, d_oout_;
    DevBuf<int> d_work_, d_omap_, d_oref_, d_rid_, d_order_, d_oorder_, d_sub_;
    DevBuf<pb::PdesRec> d_prec_;  // instance-parallel engine: per-CTA event records
    DevBuf<int> d_pord_;          // and their merged order
    DevBuf<double> d_arrival_, d_frac_;
    DevBuf<int4> d_spec_, d_cand_, d_tmp_;
    DevBuf<pb::ReqState> d_rs_;
    DevBuf<long long> d_aoff_, d_biggest_, d_echo_, d_seg_;
    DevBuf<unsigned> d_batch_, d_tmpq_, d_elist_, d_stack_;
    DevBuf<int> d_aoff32_;
    DevBuf<double> d_blocked_, d_plog_;
    DevBuf<int> d_pfrom_;
    DevBuf<pb::RecOut> d_rec_;
    DevBuf<double> d_dig_, d_del_, d_bpv_;
    DevBuf<int> d_bpk_;
    DevBuf<pb::PacerHot> d_ph_;
    DevBuf<uint2> d_qent_;
    DevBuf<pb::HeapEnt> d_heap_;
    DevBuf<unsigned char> d_cstat_, d_slo_;
    DevBuf<pb::LogEnt> d_log_;
    DevBuf<pb::MetricParams> d_params_;
    DevBuf<double> d_ttft_, d_ttfat_, d_qoe_, d_block_, d_sorted_, d_tpot_;
    DevBuf<pb::DevSummary> d_sum_;
    DevBuf<char> d_sort_tmp_;
    size_t sort_bytes_ = 0;
    // sweep histograms
    int n_groups_ = 0;
    DevBuf<int> d_group_;
    DevBuf<unsigned long long> d_hist_, d_slo_hist_;

    pb::Arena arena(bool oracle) const;
};

// Host staging of a batch touches every request a few times (lookahead,
// footprint bounds, costs, the upload arrays): one pass per replica, run over
// the host cores (replicas are independent; results land in per-replica
// slots or disjoint ranges).
template <class F>
void parallel_replicas(int n, F fn) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int nt = (int)std::min<long long>(hw, std::max(1, n / 64));
    if (nt <= 1) {
        for (int r = 0; r < n; ++r) fn(r);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int r = t; r < n; r += nt) fn(r);
        });
    for (auto& x : th) x.join();
}

Batch::Batch(const std::vector<Job>& jobs) : jobs_(jobs) {
    // validation in parallel; the first failing replica's error is thrown,
    // as the sequential loop would
    std::vector<std::exception_ptr> err(jobs_.size());
    parallel_replicas((int)jobs_.size(), [&](int r) {
        try {
            const Job& j = jobs_[r];
            check_trace(*j.trace);
            check_profile(j.prof);
            check_limits(j);
        } catch (...) {
            err[r] = std::current_exception();
        }
    });
    for (const auto& e : err)
        if (e) std::rethrow_exception(e);
}

Batch::~Batch() {
    ScopedDevice sd(dev_);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    if (st_) cudaStreamDestroy(st_);
}

void Batch::build() {
    if (built_) return;
    built_ = true;
    ck(cudaGetDevice(&dev_), "cudaGetDevice");
    n_rep_ = (int)jobs_.size();
    ck(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
    for (auto& e : ev_) ck(cudaEventCreate(&e), "event");
    Timing& tm = g_timing;
    tm = Timing{};

    // ---- layout
    desc_.resize(n_rep_);
    std::vector<pb::MetricParams> params(n_rep_);
    std::vector<double> frac(n_rep_);
    std::vector<long long> biggest(n_rep_), seg(n_rep_ + 1);
    echo_static_.assign(n_rep_, 0);
    odesc_.clear();
    omap_.clear();
    oref_.clear();
    orep_.clear();
    std::map<std::string, int> oracle_of;
    long long rq = 0, ans = 0, q = 0, bt = 0, hp = 0, lg = 0, pl = 0;
    // per-replica scans of the trace (parallel): the shortest prompt of an
    // R = 0, not preloaded, A > 1 request (lookahead), the largest footprint,
    // the answer tokens and the request-iterations (hand-out cost)
    std::vector<long long> r_pmin(n_rep_), r_big(n_rep_), r_ans(n_rep_), r_iters(n_rep_);
    parallel_replicas(n_rep_, [&](int r) {
        long long pmin = -1, big = 0, a = 0;
        for (const Spec& s : *jobs_[r].trace) {
            if (s.reasoning == 0 && !s.preloaded && s.answering > 1)
                pmin = pmin < 0 ? s.prompt : std::min<long long>(pmin, s.prompt);
            big = std::max(big, (long long)s.max_kv());
            a += s.answering;
        }
        r_pmin[r] = pmin;
        r_big[r] = big;
        r_ans[r] = a;
        r_iters[r] = (long long)request_iterations(*jobs_[r].trace);
    });
    for (int r = 0; r < n_rep_; ++r) {
        const Job& j = jobs_[r];
        const long long n = (long long)j.trace->size();
        const int ni = j.cfg.instances;
        pb::ReplicaDesc d{};
        d.n = (int)n;
        d.ni = ni;
        d.policy = j.cfg.policy;
        d.flags = (j.cfg.no_migration ? pb::kNoMigration : 0) |
                  (j.cfg.non_adaptive ? pb::kNonAdaptive : 0) |
                  (records_ ? pb::kRecordDeliv : 0) | (log_cap_ > 0 ? pb::kLogEvents : 0);
        d.quantum = j.cfg.quantum;
        d.demotion = j.cfg.demotion;
        d.slack = j.cfg.slack;
        d.tpot = j.cfg.tpot;
        d.prof = j.prof;
        d.req_base = rq;
        d.ans_base = ans;
        d.qcap = n + 1;
        d.queue_base = q;
        d.batch_base = bt;
        d.heap_base = hp;
        d.pheap_base = 0;  // set below when the instance-parallel engine is used
        d.log_base = lg;
        // parked-tail duration logs: read only by the lean Pascal build
        d.plog_base = pl;
        if (j.cfg.policy == pb::kPascal) pl += (long long)ni * pb::kParkLog;
        {
            // lookahead of the instance-parallel engine (engine_pdes.cuh): a
            // lower bound on the duration of any decode iteration
            // ((base + per_request * B) + per_kv * K >= base + per_request for
            // B >= 1, K >= 0; rounding is monotone) and of any prefill that
            // ends in a phase boundary (R = 0, not preloaded, A > 1).
            double la = j.prof.decode_base + j.prof.decode_per_request * 1.0;
            const long long pmin = r_pmin[r];
            if (pmin >= 0)
                la = std::min(la, j.prof.prefill_base + j.prof.prefill_per_token * (double)pmin);
            d.lookahead = la;
        }
        d.log_cap = log_cap_;
        const long long big = r_big[r];
        biggest[r] = big;
        frac[r] = j.cfg.capacity_fraction;
        const long long kOracleCap = LONG_MAX / 4;
        if (j.cfg.gpu_capacity > 0) {
            echo_static_[r] = std::max<long long>(j.cfg.gpu_capacity, big);
            d.capacity = j.cfg.policy == pb::kOracle ? kOracleCap : echo_static_[r];
        } else {
            d.capacity = kOracleCap;  // overwritten by the capacity kernel unless oracle
            // One oracle pre-run per distinct (trace, instances, profile, ...):
            // the oracle never evicts, demotes, paces or counts quanta, so the
            // peak it measures does not depend on the policy, the ablations
            // or the capacity fraction (a sweep over those shares one).
            std::string key(reinterpret_cast<const char*>(&j.trace), sizeof(j.trace));
            auto add = [&key](const void* p, size_t b) {
                key.append(reinterpret_cast<const char*>(p), b);
            };
            add(&ni, sizeof ni);
            add(&j.prof, sizeof j.prof);
            add(&d.quantum, sizeof d.quantum);
            add(&d.demotion, sizeof d.demotion);
            add(&d.slack, sizeof d.slack);
            add(&d.tpot, sizeof d.tpot);
            auto it = oracle_of.find(key);
            int k;
            if (it != oracle_of.end()) {
                k = it->second;
            } else {
                pb::ReplicaDesc od = d;
                od.policy = pb::kOracle;
                od.flags = 0;
                od.capacity = kOracleCap;
                od.log_cap = 0;
                k = (int)odesc_.size();
                odesc_.push_back(od);
                orep_.push_back(r);
                oracle_of.emplace(std::move(key), k);
            }
            omap_.push_back(r);
            oref_.push_back(k);
        }
        desc_[r] = d;
        params[r] = pb::MetricParams{j.cfg.tpot, j.cfg.qoe_threshold, j.cfg.ttfat_target, rq,
                                     (int)n, 0};
        seg[r] = rq;
        max_ni_ = std::max(max_ni_, ni);
        max_n_ = std::max<int>(max_n_, (int)n);
        if (j.cfg.gpu_capacity <= 0) max_on_ = std::max<int>(max_on_, (int)n);
        rq += n;
        if (r_ans[r] > INT_MAX) throw std::invalid_argument("replica answer tokens exceed 2^31");
        ans += r_ans[r];
        q += 2ll * ni * (n + 1);
        bt += (long long)ni * std::max<long long>(n, 1);
        hp += n + ni + 2;
        lg += log_cap_;
    }
    // Instance-parallel engine: few replicas (latency shapes: each gets a
    // whole SM), more than one instance, no decision log (record arrays are
    // kept: records-only parity dumps run on it),
    // enqueue seqs (k * ni + i) within 32 bits, a positive lookahead for
    // Pascal. PB_PDES=0 disables it (experiment hook / A-B).
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const char* pe = std::getenv("PB_PDES");
        bool ok = !(pe && std::atoi(pe) == 0) && log_cap_ == 0 && n_rep_ >= 1 &&
                  n_rep_ <= sms && max_ni_ >= 2;
        long long ph = 0;
        for (int r = 0; ok && r < n_rep_; ++r) {
            const pb::ReplicaDesc& d = desc_[r];
            // enqueues per request <= 4 (arrival, demotion, phase boundary, transfer)
            if ((4.0 * d.n + 8.0) * (double)d.ni >= 4294967295.0) ok = false;
            if (d.policy == pb::kPascal && !(d.lookahead > 0.0)) ok = false;
        }
        if (ok) {
            pdes_w_ = std::min(pb::kPdesMaxWarps, max_ni_);
            for (int r = 0; r < n_rep_; ++r) {
                desc_[r].pheap_base = ph;
                ph += (long long)desc_[r].ni * (desc_[r].n + 2);
            }
            for (pb::ReplicaDesc& od : odesc_) {  // pre-runs share their replica's layout
                for (int r = 0; r < n_rep_; ++r)
                    if (desc_[r].req_base == od.req_base) od.pheap_base = desc_[r].pheap_base;
            }
            pheap_total_ = ph;
        }
    }
    seg[n_rep_] = rq;
    if (rq > (long long)INT_MAX)  // the per-replica TTFT sort (CUB) counts items in int
        throw std::invalid_argument("batch exceeds 2^31 - 1 requests in total; split it");
    total_req_ = rq;
    total_ans_ = ans;
    total_q_ = q;
    total_batch_ = bt;
    total_heap_ = hp;
    total_log_ = lg;

    // ---- host staging of the read-only trace (replicas in parallel, each
    // into its own request range; arrays left uninitialised: every slot is
    // written)
    std::unique_ptr<double[]> arrival(new double[std::max<long long>(rq, 1)]);
    std::unique_ptr<int4[]> spec(new int4[std::max<long long>(rq, 1)]);
    std::unique_ptr<long long[]> aoff(new long long[std::max<long long>(rq, 1)]);
    std::unique_ptr<int[]> aoff32(new int[std::max<long long>(rq, 1)]);
    std::unique_ptr<int[]> rid(new int[std::max<long long>(rq, 1)]);
    {
        std::vector<long long> abase(n_rep_ + 1, 0);
        for (int r = 0; r < n_rep_; ++r) abase[r + 1] = abase[r] + r_ans[r];
        parallel_replicas(n_rep_, [&](int r) {
            long long g = seg[r], a = abase[r];
            const long long a0 = a;
            for (const Spec& s : *jobs_[r].trace) {
                arrival[g] = s.arrival;
                spec[g] = make_int4((int)s.prompt, (int)s.reasoning, (int)s.answering,
                                    s.preloaded ? 1 : 0);
                aoff[g] = a;
                aoff32[g] = (int)(a - a0);
                rid[g] = r;
                a += s.answering;
                ++g;
            }
        });
    }

    // ---- device arenas
    d_desc_.ensure(n_rep_);
    d_desc_init_.ensure(n_rep_);
    d_out_.ensure(n_rep_);
    d_odesc_.ensure(odesc_.size());
    d_oout_.ensure(odesc_.size());
    d_omap_.ensure(omap_.size());
    d_oref_.ensure(oref_.size());
    d_work_.ensure(2);
    d_arrival_.ensure(rq);
    d_spec_.ensure(rq);
    d_aoff_.ensure(rq);
    d_rid_.ensure(rq);
    d_rs_.ensure(rq);
    d_aoff32_.ensure(rq);
    d_blocked_.ensure(rq);
    d_pfrom_.ensure(rq);
    d_plog_.ensure(std::max<long long>(pl, 1));
    d_rec_.ensure(rq);
    // per-warp planner scratch: one copy per warp of a replica under the
    // instance-parallel engine
    const long long scr = rq * std::max(1, pdes_w_);
    d_cand_.ensure(scr);
    d_tmp_.ensure(scr);
    d_tmpq_.ensure(scr);
    d_cstat_.ensure(scr);
    d_elist_.ensure(scr);
    d_stack_.ensure(scr);
    d_ph_.ensure(rq);
    d_bpv_.ensure(ans);
    d_bpk_.ensure(ans);
    d_dig_.ensure(records_ ? ans : 1);
    d_del_.ensure(records_ ? ans : 1);
    d_qent_.ensure(q);
    d_batch_.ensure(bt);
    d_heap_.ensure(std::max(hp, pheap_total_));
    d_log_.ensure(std::max<long long>(lg, 1));
    d_params_.ensure(n_rep_);
    d_frac_.ensure(n_rep_);
    d_biggest_.ensure(n_rep_);
    d_echo_.ensure(n_rep_);
    d_seg_.ensure(n_rep_ + 1);
    d_ttft_.ensure(rq);
    d_tpot_.ensure(rq);
    d_ttfat_.ensure(rq);
    d_qoe_.ensure(rq);
    d_block_.ensure(rq);
    d_slo_.ensure(rq);
    d_sorted_.ensure(rq);
    d_sum_.ensure(n_rep_);

    pb::RowArrays rows{d_ttft_.p, d_ttfat_.p, d_qoe_.p, d_block_.p, d_slo_.p, d_sorted_.p,
                       d_tpot_.p};
    pb::Arena ar = arena(false);
    size_t bytes = 0;
    if (pb::launch_metrics(ar, d_params_.p, d_seg_.p, d_rid_.p, rq, n_rep_, rows, d_sum_.p,
                           d_echo_.p, nullptr, &bytes, st_) != 0)
        throw std::logic_error("CUB size query failed");
    sort_bytes_ = std::max<size_t>(bytes, 16);
    d_sort_tmp_.ensure(sort_bytes_);

    // ---- uploads (timed as h2d)
    ck(cudaEventRecord(ev_[0], st_), "event");
    long long hb = 0;
    auto up = [&](void* dst, const void* src, size_t b) {
        if (b == 0) return;
        ck(cudaMemcpyAsync(dst, src, b, cudaMemcpyHostToDevice, st_), "h2d");
        hb += (long long)b;
    };
    up(d_desc_init_.p, desc_.data(), desc_.size() * sizeof(pb::ReplicaDesc));
    up(d_odesc_.p, odesc_.data(), odesc_.size() * sizeof(pb::ReplicaDesc));
    up(d_omap_.p, omap_.data(), omap_.size() * sizeof(int));
    up(d_oref_.p, oref_.data(), oref_.size() * sizeof(int));
    // Longest-predicted-first hand-out order for the work-stealing loop (the
    // step ends with its slowest warp): cost ~ request-iterations, doubled
    // for the queue-scanning policies.
    {
        auto cost = [&](int r) {
            double c = (double)r_iters[r];
            return jobs_[r].cfg.policy == pb::kPascal || jobs_[r].cfg.policy == pb::kRr ? 2 * c : c;
        };
        std::vector<double> cr(n_rep_);
        for (int r = 0; r < n_rep_; ++r) cr[r] = cost(r);
        order_.resize(n_rep_);
        std::iota(order_.begin(), order_.end(), 0);
        std::stable_sort(order_.begin(), order_.end(), [&](int a, int b) { return cr[a] > cr[b]; });
        oorder_.resize(odesc_.size());
        std::iota(oorder_.begin(), oorder_.end(), 0);
        std::stable_sort(oorder_.begin(), oorder_.end(),
                         [&](int a, int b) { return cr[orep_[a]] > cr[orep_[b]]; });
        d_order_.ensure(n_rep_);
        d_oorder_.ensure(oorder_.size());
        up(d_order_.p, order_.data(), order_.size() * sizeof(int));
        up(d_oorder_.p, oorder_.data(), oorder_.size() * sizeof(int));
    }
    up(d_arrival_.p, arrival.get(), rq * sizeof(double));
    up(d_spec_.p, spec.get(), rq * sizeof(int4));
    up(d_aoff_.p, aoff.get(), rq * sizeof(long long));
    up(d_aoff32_.p, aoff32.get(), rq * sizeof(int));
    up(d_rid_.p, rid.get(), rq * sizeof(int));
    up(d_params_.p, params.data(), params.size() * sizeof(pb::MetricParams));
    up(d_frac_.p, frac.data(), frac.size() * sizeof(double));
    up(d_biggest_.p, biggest.data(), biggest.size() * sizeof(long long));
    up(d_echo_.p, echo_static_.data(), echo_static_.size() * sizeof(long long));
    up(d_seg_.p, seg.data(), seg.size() * sizeof(long long));
    ck(cudaEventRecord(ev_[1], st_), "event");
    ck(cudaEventSynchronize(ev_[1]), "sync");
    float ms = 0;
    cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
    tm.h2d_ms = ms;
    tm.h2d_bytes = hb;
}

pb::Arena Batch::arena(bool oracle) const {
    pb::Arena a{};
    a.desc = oracle ? d_odesc_.p : d_desc_.p;
    a.out = oracle ? d_oout_.p : d_out_.p;
    a.n_rep = oracle ? (int)odesc_.size() : n_rep_;
    a.work = d_work_.p + (oracle ? 0 : 1);
    a.order = oracle ? d_oorder_.p : d_order_.p;
    a.arrival = d_arrival_.p;
    a.spec = d_spec_.p;
    a.aoff = d_aoff_.p;
    a.aoff32 = d_aoff32_.p;
    a.blocked = d_blocked_.p;
    a.rs = d_rs_.p;
    a.rec = d_rec_.p;
    a.ph = d_ph_.p;
    a.bpv = d_bpv_.p;
    a.bpk = d_bpk_.p;
    a.dig = d_dig_.p;
    a.del = d_del_.p;
    a.qent = d_qent_.p;
    a.batch = d_batch_.p;
    a.heap = d_heap_.p;
    a.cand = d_cand_.p;
    a.tmp = d_tmp_.p;
    a.tmpq = d_tmpq_.p;
    a.cstat = d_cstat_.p;
    a.elist = d_elist_.p;
    a.stack = d_stack_.p;
    a.log = d_log_.p;
    a.plog = d_plog_.p;
    a.pfrom = d_pfrom_.p;
    a.prec = d_prec_.p;
    a.pord = d_pord_.p;
    a.wstride = total_req_;
    return a;
}

void Batch::execute() {
    build();
    ScopedDevice sd(dev_);
    Timing& tm = g_timing;
    const char* penv = std::getenv("PB_NO_POLICY_SPECIALISATION");  // experiment hook
    const bool spec = !(penv && std::atoi(penv));
    // the policy all replicas share (-1: mixed)
    int common = desc_.empty() ? -1 : desc_[0].policy;
    for (const pb::ReplicaDesc& d : desc_)
        if (d.policy != common) common = -1;
    using Launcher = int (*)(const pb::Arena&, int, int, int, int, int, int, int, void*);
    auto lean_for = [](int policy) -> Launcher {
        switch (policy) {
            case pb::kPascal: return pb::pascal_lean::launch_engine;
            case pb::kOracle: return pb::oracle_lean::launch_engine;
            case pb::kFcfs: return pb::fcfs_lean::launch_engine;
            case pb::kRr: return pb::rr_lean::launch_engine;
            default: return pb::nolog::launch_engine;
        }
    };
    // `pre_run`: the oracle capacity pre-run (never logs or records)
    auto launch = [&](const pb::Arena& ar, int reps, int max_n, bool pre_run) {
        const Shape sh = pick_shape(reps, max_ni_, max_n);
        Launcher eng = pre_run                        ? (spec ? lean_for(pb::kOracle)
                                                              : pb::nolog::launch_engine)
                       : (log_cap_ > 0 || records_)   ? pb::logging::launch_engine
                       : spec                          ? lean_for(common)
                                                       : pb::nolog::launch_engine;
        return eng(ar, max_ni_, sh.n_smem, sh.c_smem, sh.h_slots, sh.b_smem, sh.wpb, sh.blocks,
                   st_);
    };
    int launches = 0;
    // Instance-parallel engine (engine_pdes.cuh) for few, large replicas; the
    // replicas it declines (kErrPdes) are re-run by the serial engine on the
    // same stream before anything reads their results.
    using PLauncher = int (*)(const pb::Arena&, int, int, int, int, int, void*);
    auto run = [&](bool pre_run) {
        pb::Arena ar = arena(pre_run);
        const int reps = ar.n_rep;
        const int max_n = pre_run ? max_on_ : max_n_;
        if (pdes_w_ == 0) {
            if (!pre_run) tm.instance_parallel = 0;
            if (launch(ar, reps, max_n, pre_run))
                throw std::logic_error(pre_run ? "engine launch failed (oracle pre-run)"
                                               : "engine launch failed");
            launches += 1;
            return;
        }
        int dev = 0, sms = 148, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        // dynamic shared memory beside the kernel's static 4 KB merge scratch
        const int budget = std::max(48 * 1024, optin) - 6 * 1024;
        int c = std::max(32, std::min(max_n, 512)), hs = 32;
        while (pb::pdes_smem(max_ni_, hs, c, pdes_w_) > budget && c > 32) c /= 2;
        while (pb::pdes_smem(max_ni_, hs, c, pdes_w_) > budget && hs > 4) hs /= 2;
        const int blocks = std::min(reps, sms);
        d_prec_.ensure((size_t)blocks * pb::kPdesMaxWarps * pb::kPdesRecCap);
        d_pord_.ensure((size_t)blocks * pb::kPdesMaxWarps * pb::kPdesRecCap);
        ar.prec = d_prec_.p;
        ar.pord = d_pord_.p;
        PLauncher eng = pre_run ? (spec ? pb::pdes_oracle::launch_engine : pb::pdes::launch_engine)
                                : (spec && common == pb::kPascal ? pb::pdes_pascal::launch_engine
                                                                 : pb::pdes::launch_engine);
        if (eng(ar, max_ni_, hs, c, pdes_w_, blocks, st_))
            throw std::logic_error("instance-parallel engine launch failed");
        launches += 1;
        std::vector<pb::ReplicaOut> outs(reps);
        ck(cudaMemcpyAsync(outs.data(), ar.out, reps * sizeof(pb::ReplicaOut),
                           cudaMemcpyDeviceToHost, st_),
           "d2h");
        ck(cudaStreamSynchronize(st_), "instance-parallel engine");
        std::vector<int> sub;
        static const bool dbg = std::getenv("PB_PDES_DEBUG") != nullptr;
        if (dbg)
            for (int r = 0; r < std::min(reps, 4); ++r)
                std::fprintf(stderr, "[pdes] %s replica %d: events %lld rounds %.0f serialised %lld\n",
                             pre_run ? "oracle" : "policy", r, outs[r].events, outs[r].now,
                             outs[r].nlog);
        for (int r = 0; r < reps; ++r)
            if (outs[r].status == pb::kErrPdes) {
                sub.push_back(r);
                if (dbg)  // ReplicaOut::pad carries the decline reason (engine_pdes.cuh)
                    std::fprintf(stderr, "[pdes] %s replica %d declined, reason %d\n",
                                 pre_run ? "oracle" : "policy", r, outs[r].pad);
            }
        if (!pre_run) {
            declined_ = sub;
            tm.instance_parallel = reps - (int)sub.size();
        }
        if (sub.empty()) return;
        d_sub_.ensure(sub.size());
        ck(cudaMemcpyAsync(d_sub_.p, sub.data(), sub.size() * sizeof(int), cudaMemcpyHostToDevice,
                           st_),
           "h2d");
        ck(cudaMemsetAsync(const_cast<int*>(ar.work), 0, sizeof(int), st_), "memset");
        pb::Arena sa = ar;
        sa.order = d_sub_.p;
        sa.n_rep = (int)sub.size();
        if (launch(sa, sa.n_rep, max_n, pre_run))
            throw std::logic_error("engine launch failed (serial re-run)");
        launches += 1;
        ck(cudaStreamSynchronize(st_), "serial re-run");  // d_sub_ is reused by the next run
    };
    ck(cudaEventRecord(ev_[0], st_), "event");
    ck(cudaMemcpyAsync(d_desc_.p, d_desc_init_.p, n_rep_ * sizeof(pb::ReplicaDesc),
                       cudaMemcpyDeviceToDevice, st_),
       "desc reset");
    ck(cudaMemsetAsync(d_work_.p, 0, 2 * sizeof(int), st_), "memset");
    if (!odesc_.empty()) {
        run(true);
        if (pb::launch_capacity(d_desc_.p, d_oout_.p, d_omap_.p, d_oref_.p, d_frac_.p,
                                d_biggest_.p, d_echo_.p, (int)omap_.size(), st_))
            throw std::logic_error("capacity kernel launch failed");
        launches += 1;
    }
    ck(cudaEventRecord(ev_[1], st_), "event");
    pb::Arena pa = arena(false);
    run(false);
    ck(cudaEventRecord(ev_[2], st_), "event");
    pb::RowArrays rows{d_ttft_.p, d_ttfat_.p, d_qoe_.p, d_block_.p, d_slo_.p, d_sorted_.p,
                       d_tpot_.p};
    size_t bytes = sort_bytes_;
    if (pb::launch_metrics(pa, d_params_.p, d_seg_.p, d_rid_.p, total_req_, n_rep_, rows,
                           d_sum_.p, d_echo_.p, d_sort_tmp_.p, &bytes, st_) != 0)
        throw std::logic_error("metrics launch failed");
    launches += total_req_ > 0 ? 3 : 1;
    if (n_groups_ > 0) {
        if (pb::launch_histograms(d_rid_.p, d_group_.p, rows, d_out_.p, total_req_, n_groups_,
                                  d_hist_.p, d_slo_hist_.p, st_))
            throw std::logic_error("histogram launch failed");
        launches += 1;
    }
    ck(cudaEventRecord(ev_[3], st_), "event");
    ck(cudaEventSynchronize(ev_[3]), "engine sync");
    ck(cudaGetLastError(), "engine");
    float a = 0, b = 0, c = 0, t = 0;
    cudaEventElapsedTime(&a, ev_[0], ev_[1]);
    cudaEventElapsedTime(&b, ev_[1], ev_[2]);
    cudaEventElapsedTime(&c, ev_[2], ev_[3]);
    cudaEventElapsedTime(&t, ev_[0], ev_[3]);
    tm.derive_ms = a;
    tm.engine_ms = b;
    tm.metrics_ms = c;
    tm.total_ms = t;
    tm.launches = launches;
}

void Batch::fetch_summaries(std::vector<DeviceSummary>& out) {
    ScopedDevice sd(dev_);
    static_assert(sizeof(DeviceSummary) == sizeof(pb::DevSummary), "summary layout");
    out.resize(n_rep_);
    ck(cudaEventRecord(ev_[0], st_), "event");
    ck(cudaMemcpyAsync(out.data(), d_sum_.p, n_rep_ * sizeof(pb::DevSummary),
                       cudaMemcpyDeviceToHost, st_),
       "d2h");
    ck(cudaEventRecord(ev_[1], st_), "event");
    ck(cudaEventSynchronize(ev_[1]), "sync");
    float ms = 0;
    cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
    g_timing.d2h_ms = ms;
    g_timing.d2h_bytes = (long long)(n_rep_ * sizeof(pb::DevSummary));
}

void Batch::fetch_single(RunOutputs& o, bool records, bool log) {
    ScopedDevice sd(dev_);
    std::vector<DeviceSummary> s;
    fetch_summaries(s);
    o.summary = s[0];
    o.status = s[0].status;
    o.capacity = s[0].capacity;
    const long long n = total_req_;
    std::vector<double> ttft(n), ttfat(n), qoe(n), blk(n), tpot(n);
    std::vector<unsigned char> slo(n);
    auto down = [&](void* dst, const void* src, size_t b) {
        if (b) ck(cudaMemcpy(dst, src, b, cudaMemcpyDeviceToHost), "d2h");
    };
    down(ttft.data(), d_ttft_.p, n * sizeof(double));
    down(ttfat.data(), d_ttfat_.p, n * sizeof(double));
    down(qoe.data(), d_qoe_.p, n * sizeof(double));
    down(blk.data(), d_block_.p, n * sizeof(double));
    down(tpot.data(), d_tpot_.p, n * sizeof(double));
    down(slo.data(), d_slo_.p, n);
    const Trace& t = *jobs_[0].trace;
    o.rows.resize(n);
    for (long long k = 0; k < n; ++k) {
        Row& w = o.rows[k];
        w.id = t[k].id;
        w.reasoning = t[k].reasoning;
        w.answering = t[k].answering;
        w.ttft = ttft[k];
        w.ttfat = ttfat[k];
        w.qoe = qoe[k];
        w.slo = slo[k] != 0;
        w.blocking = blk[k];
        w.tpot = tpot[k];
    }
    if (records) {
        o.rec.resize(n);
        down(o.rec.data(), d_rec_.p, n * sizeof(pb::RecOut));
        o.dig.resize(total_ans_);
        down(o.dig.data(), d_dig_.p, total_ans_ * sizeof(double));
        if (records_) {
            o.del.resize(total_ans_);
            down(o.del.data(), d_del_.p, total_ans_ * sizeof(double));
        }
        o.aoff.resize(n);
        down(o.aoff.data(), d_aoff_.p, n * sizeof(long long));
        std::vector<pb::ReqState> rs(n);
        down(rs.data(), d_rs_.p, n * sizeof(pb::ReqState));
        // the delivered count travels in rec.pad for the dump writer
        for (long long k = 0; k < n; ++k) o.rec[k].pad = rs[k].ndel;
    }
    if (log) {
        pb::ReplicaOut ro;
        down(&ro, d_out_.p, sizeof ro);
        long long cnt = std::min<long long>(ro.nlog, log_cap_);
        o.log.resize(cnt);
        down(o.log.data(), d_log_.p, cnt * sizeof(pb::LogEnt));
        if (ro.nlog > log_cap_) o.log.resize(0), o.capacity = -ro.nlog;  // caller retries
    }
}

// Per-request metric rows of every replica (trace order within a replica).
void Batch::fetch_rows(std::vector<std::vector<Row>>& rows) {
    ScopedDevice sd(dev_);
    const long long n = total_req_;
    std::vector<double> ttft(n), ttfat(n), qoe(n), blk(n), tpot(n);
    std::vector<unsigned char> slo(n);
    auto down = [&](void* dst, const void* src, size_t b) {
        if (b) ck(cudaMemcpy(dst, src, b, cudaMemcpyDeviceToHost), "d2h");
    };
    down(ttft.data(), d_ttft_.p, n * sizeof(double));
    down(ttfat.data(), d_ttfat_.p, n * sizeof(double));
    down(qoe.data(), d_qoe_.p, n * sizeof(double));
    down(blk.data(), d_block_.p, n * sizeof(double));
    down(tpot.data(), d_tpot_.p, n * sizeof(double));
    down(slo.data(), d_slo_.p, n);
    rows.assign(n_rep_, {});
    long long g = 0;
    for (int r = 0; r < n_rep_; ++r) {
        const Trace& t = *jobs_[r].trace;
        rows[r].resize(t.size());
        for (size_t k = 0; k < t.size(); ++k, ++g) {
            Row& w = rows[r][k];
            w.id = t[k].id;
            w.reasoning = t[k].reasoning;
            w.answering = t[k].answering;
            w.ttft = ttft[g];
            w.ttfat = ttfat[g];
            w.qoe = qoe[g];
            w.slo = slo[g] != 0;
            w.blocking = blk[g];
            w.tpot = tpot[g];
        }
    }
}

void batch_rows(Batch* b, std::vector<std::vector<Row>>& rows) { b->fetch_rows(rows); }

Batch* batch_create(const std::vector<Job>& jobs) {
    auto* b = new Batch(jobs);
    try {
        b->build();
    } catch (...) {
        delete b;
        throw;
    }
    return b;
}
void batch_execute(Batch* b) { b->execute(); }
void batch_summaries(Batch* b, std::vector<DeviceSummary>& out) { b->fetch_summaries(out); }
void batch_free(Batch* b) { delete b; }

void batch_set_groups(Batch* b, const int* group_of_replica, int n_groups) {
    if (n_groups < 1) throw std::invalid_argument("n_groups must be >= 1");
    ScopedDevice sd(b->dev_);
    for (int r = 0; r < b->n_rep_; ++r)
        if (group_of_replica[r] < 0 || group_of_replica[r] >= n_groups)
            throw std::invalid_argument("group id out of range");
    b->n_groups_ = n_groups;
    b->d_group_.ensure(b->n_rep_);
    b->d_hist_.ensure((size_t)n_groups * (pb::kHistBins + 2));
    b->d_slo_hist_.ensure((size_t)n_groups * 2);
    ck(cudaMemcpy(b->d_group_.p, group_of_replica, b->n_rep_ * sizeof(int),
                  cudaMemcpyHostToDevice),
       "h2d");
}

void batch_histograms(Batch* b, unsigned long long* hist, unsigned long long* slo) {
    if (b->n_groups_ == 0) throw std::invalid_argument("no groups set on this batch");
    ScopedDevice sd(b->dev_);
    ck(cudaMemcpy(hist, b->d_hist_.p,
                  sizeof(unsigned long long) * b->n_groups_ * (pb::kHistBins + 2),
                  cudaMemcpyDeviceToHost),
       "d2h");
    ck(cudaMemcpy(slo, b->d_slo_hist_.p, sizeof(unsigned long long) * b->n_groups_ * 2,
                  cudaMemcpyDeviceToHost),
       "d2h");
}

RunOutputs run_single(const Job& job, bool want_records, bool want_log) {
    if (!device_available()) throw std::logic_error("no CUDA device available for the B200 engine");
    long long cap = want_log ? std::max<long long>(1024, 8 * request_iterations(*job.trace) +
                                                             64 * (long long)job.trace->size())
                             : 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        if (want_log) {
            // the decision log is kept on the device for the whole run (one
            // 24-byte entry per line): refuse up front with a clear message
            // instead of failing inside the allocator
            size_t free_b = 0, total_b = 0;
            if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess &&
                (double)cap * sizeof(pb::LogEnt) > 0.8 * (double)free_b)
                throw std::runtime_error(
                    "decision log of " + std::to_string(cap) + " entries (" +
                    std::to_string((double)cap * sizeof(pb::LogEnt) / 1e9) +
                    " GB) does not fit in device memory; run without an event log or split "
                    "the trace");
        }
        Batch b({job});
        if (want_records) b.enable_records();
        if (want_log) b.enable_log(cap);
        b.execute();
        RunOutputs o;
        b.fetch_single(o, want_records, want_log);
        if (o.status != 0) throw std::logic_error(status_message(o.status));
        if (want_log && o.capacity < 0) {  // decision log larger than the first guess
            cap = -o.capacity;
            continue;
        }
        return o;
    }
    throw std::logic_error("event log sizing failed");
}

long long derive_capacity_dev(const Job& job) {
    if (job.cfg.instances < 1) throw std::invalid_argument("instance_count must be >= 1");
    long long big = 0;
    for (const Spec& s : *job.trace) big = std::max(big, (long long)s.max_kv());
    if (job.cfg.gpu_capacity > 0) return std::max<long long>(job.cfg.gpu_capacity, big);
    if (!device_available()) throw std::logic_error("no CUDA device available for the B200 engine");
    Batch b({job});
    b.execute();
    std::vector<DeviceSummary> s;
    b.fetch_summaries(s);
    return s[0].capacity;
}

}  // namespace pbh
