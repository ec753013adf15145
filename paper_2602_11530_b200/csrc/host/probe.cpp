// probe.cpp — unit-parity seams of libpascal.so (pascal_probe_* in
// include/pascal_b200.h).
//
// The reference's unit tests drive pure C++ functions with hand-built states:
// apply_demotion + plan_iteration + Simulator::maybe_start's plan application
// (proj/src/instance.cpp:39-57,103-282, proj/src/engine.cpp:192-258) and the
// placement rules (proj/src/cluster.cpp:27-44,59-62). The device engine fuses
// them into its event loop, so these entries pack a hand-built state into the
// engine's own layout (engine.h ReqState / queues / instance counters), run
// the logging build's planner or select_instance for one step on the current
// device (engine.cu plan_probe_kernel / select_probe_kernel), and unpack the
// decision log, the pushed events and the counters into the reference's
// terms.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/pascal_b200.h"
#include "common.hpp"

namespace pbh {
namespace {

void cu(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::logic_error(std::string("CUDA error (") + what + "): " + cudaGetErrorString(e));
}

// Scratch device buffers of one probe call (freed on every exit path).
class Scratch {
public:
    ~Scratch() {
        for (void* p : ptrs_) cudaFree(p);
    }
    template <class T>
    T* get(size_t count) {
        void* p = nullptr;
        cu(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
        ptrs_.push_back(p);
        cu(cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T)), "cudaMemset");
        return static_cast<T*>(p);
    }
    template <class T>
    T* put(const std::vector<T>& v) {
        T* p = get<T>(v.size());
        if (!v.empty()) cu(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "h2d");
        return p;
    }

private:
    std::vector<void*> ptrs_;
};

template <class T>
std::vector<T> fetch(const T* d, size_t count) {
    std::vector<T> h(count);
    if (count) cu(cudaMemcpy(h.data(), d, count * sizeof(T), cudaMemcpyDeviceToHost), "d2h");
    return h;
}

void need(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

}  // namespace

void probe_maybe_start(const pascal_probe_state& st, const pb::Profile& prof,
                       pascal_probe_plan& out) {
    const long n = st.n_requests;
    need(n >= 0 && n < (1L << 24), "n_requests out of range");
    need(n == 0 || st.requests != nullptr, "requests is null");
    need(st.n_high >= 0 && st.n_low >= 0, "negative queue length");
    need((st.n_high == 0 || st.high_queue) && (st.n_low == 0 || st.low_queue), "queue is null");
    need(st.policy != nullptr, "policy is null");
    const int policy = parse_policy(st.policy);
    need(policy == pb::kPascal || st.n_low == 0,
         "only pascal uses the low queue (baselines keep every request in the high queue)");
    // queued requests and the engine's queue invariant: each queue is in
    // (enqueue_seq, id) order (engine.cpp:111-116 appends with a growing
    // counter), a request sits in at most one queue
    std::vector<int> where(n, 0);  // 0 none, 1 high, 2 low
    std::vector<std::pair<unsigned long long, long>> queued;
    auto scan = [&](const long* q, long len, int tag) {
        for (long k = 0; k < len; ++k) {
            const long idx = q[k];
            need(idx >= 0 && idx < n, "queue entry out of range");
            need(where[idx] == 0, "request queued twice");
            where[idx] = tag;
            const pascal_probe_request& r = st.requests[idx];
            if (k > 0) {
                const pascal_probe_request& p = st.requests[q[k - 1]];
                need(p.enqueue_seq < r.enqueue_seq || (p.enqueue_seq == r.enqueue_seq && q[k - 1] < idx),
                     "queue not in (enqueue_seq, id) order");
            }
            if (tag == 2)
                need(r.enqueue_seq <= st.enqueue_counter,
                     "low-queue seq above the enqueue counter");
            queued.emplace_back(r.enqueue_seq, idx);
        }
    };
    scan(st.high_queue, st.n_high, 1);
    scan(st.low_queue, st.n_low, 2);
    // baselines enqueue only at arrival (engine.cpp:111-116,260-283), so their
    // queue is in arrival order; the engine's FCFS / oracle order is the queue
    // order
    if (policy != pb::kPascal)
        for (long k = 1; k < st.n_high; ++k)
            need(st.high_queue[k - 1] < st.high_queue[k],
                 "baseline queue not in arrival order (baselines enqueue only at arrival)");
    std::sort(queued.begin(), queued.end());
    std::vector<unsigned> dseq(n, 0);  // engine seqs: unique, same relative order
    for (size_t k = 0; k < queued.size(); ++k) dseq[queued[k].second] = (unsigned)(k + 1);

    std::vector<pb::ReqState> rs(n);
    std::vector<int4> spec(n);
    std::vector<double> arrival(n);
    for (long k = 0; k < n; ++k) {
        const pascal_probe_request& r = st.requests[k];
        need(k == 0 || st.requests[k - 1].arrival_time <= r.arrival_time,
             "requests not in arrival order");
        need(r.prompt_tokens >= 0 && r.reasoning_tokens >= 0 && r.answering_tokens >= 0 &&
                 r.prompt_tokens + r.reasoning_tokens + r.answering_tokens < (1L << 26),
             "token counts out of range");
        need(r.kv_tokens >= 0 && r.kv_tokens < (1L << 26) && r.tokens_generated >= 0 &&
                 r.tokens_generated < (1L << 26) && r.quanta_exhausted >= 0 &&
                 r.quanta_exhausted < (1L << 30) && r.quantum_used_in_round >= 0 &&
                 r.quantum_used_in_round < (1L << 30),
             "request state out of range");
        unsigned ph;
        switch (r.phase) {
            case 0: ph = 0; break;
            case 1: ph = 1; break;
            case 2: ph = 2; break;
            case 4: ph = 3; break;
            default: throw std::invalid_argument("phase must be 0, 1, 2 or 4");
        }
        need(r.kv_location >= 0 && r.kv_location <= 2, "kv_location must be 0, 1 or 2");
        pb::ReqState s{};
        s.h = make_int4((int)r.kv_tokens, (int)r.tokens_generated, (int)dseq[k],
                        (int)r.quanta_exhausted);
        unsigned m = ph | ((unsigned)r.kv_location << 2) | ((unsigned)(r.swapping_in != 0) << 4) |
                     ((unsigned)(r.swapping_out != 0) << 5) | ((unsigned)(where[k] == 2) << 6);
        s.meta = m;  // owner 0
        s.qused = (int)r.quantum_used_in_round;
        rs[k] = s;
        spec[k] = make_int4((int)r.prompt_tokens, (int)r.reasoning_tokens,
                            (int)r.answering_tokens, 0);
        arrival[k] = r.arrival_time;
    }
    std::vector<uint2> qent(2 * (size_t)(n + 1));
    const long long qcap = n + 1;
    for (long k = 0; k < st.n_high; ++k)
        qent[k] = make_uint2((unsigned)st.high_queue[k], dseq[st.high_queue[k]]);
    for (long k = 0; k < st.n_low; ++k)
        qent[qcap + k] = make_uint2((unsigned)st.low_queue[k], dseq[st.low_queue[k]]);

    Scratch sc;
    pb::PlanProbe p{};
    p.n = (int)n;
    p.ni = 1;
    p.inst = 0;
    p.policy = policy;
    p.cap = st.gpu_capacity;
    p.quantum = 500;
    p.demotion = st.demotion_threshold;
    p.now = st.now;
    p.prof = prof;
    p.enq = (unsigned)queued.size();
    p.c_smem = std::max(0, std::min(st.candidate_scratch, 4096));
    p.rs = sc.put(rs);
    p.spec = sc.put(spec);
    p.arrival = sc.put(arrival);
    p.blocked = sc.get<double>(n);
    p.rec = sc.get<pb::RecOut>(n);
    p.ph = sc.get<pb::PacerHot>(n);
    p.aoff = sc.get<int>(n);
    p.qent = sc.put(qent);
    p.qcap = qcap;
    p.qlen = sc.put(std::vector<int>{(int)st.n_high, (int)st.n_low});
    p.used = sc.put(std::vector<long long>{st.gpu_used, st.cpu_used});
    p.batch = sc.get<unsigned>(n);
    p.heap_cap = 2 * (long long)n + 8;
    p.heap = sc.get<pb::HeapEnt>(p.heap_cap);
    p.log_cap = 4 * (long long)n + 8;
    p.log = sc.get<pb::LogEnt>(p.log_cap);
    p.cand = sc.get<int4>(n + 1);
    p.tmp = sc.get<int4>(n + 1);
    p.tmpq = sc.get<unsigned>(n + 1);
    p.cstat = sc.get<unsigned char>(n + 1);
    p.elist = sc.get<unsigned>(n + 1);
    p.stack = sc.get<unsigned>(n + 1);
    p.out_used = sc.get<long long>(2);
    p.out_scal = sc.get<int>(5);
    if (pb::logging::launch_plan_probe(p, nullptr))
        throw std::logic_error("plan probe launch failed");
    cu(cudaDeviceSynchronize(), "plan probe");
    const std::vector<int> scal = fetch(p.out_scal, 5);
    const std::vector<long long> used = fetch(p.out_used, 2);
    const int status = scal[0];
    if (status != 0 && status != pb::kErrCapacity) throw std::logic_error(status_message(status));
    const std::vector<pb::LogEnt> log = fetch(p.log, (size_t)std::min<long long>(scal[2], p.log_cap));
    const std::vector<pb::HeapEnt> heap = fetch(p.heap + 1, (size_t)scal[1]);
    const std::vector<unsigned> batch = fetch(p.batch, (size_t)scal[3]);
    const std::vector<double> blocked = fetch(p.blocked, (size_t)n);

    out.kind = 0;
    out.over_capacity = status == pb::kErrCapacity;
    out.prefill_request = -1;
    out.completion_time = 0.0;
    out.gpu_used = (long)used[0];
    out.cpu_used = (long)used[1];
    out.n_demoted = out.n_evictions = out.n_swap_ins = out.n_immediate_swap_ins = 0;
    out.n_denied = out.n_batch = out.n_swap_events = 0;
    auto add = [](long* arr, long& cnt, long v) {
        if (arr) arr[cnt] = v;
        ++cnt;
    };
    for (const pb::LogEnt& e : log) {
        switch (e.kind) {
            case pb::kLDemote: add(out.demoted, out.n_demoted, e.req); break;
            case pb::kLEvict: add(out.evictions, out.n_evictions, e.req); break;
            case pb::kLSwapIn: {
                const long kv = st.requests[e.req].kv_tokens;
                // instance.cpp:259: zero-latency reloads join the batch immediately
                if (kv == 0 || std::isinf(prof.swap_bandwidth))
                    add(out.immediate_swap_ins, out.n_immediate_swap_ins, e.req);
                else add(out.swap_ins, out.n_swap_ins, e.req);
                break;
            }
            case pb::kLBlock: add(out.denied, out.n_denied, e.req); break;
            case pb::kLPrefillStart:
                out.kind = 1;
                out.prefill_request = e.req;
                break;
            case pb::kLDecodeStart: out.kind = 2; break;
            default: throw std::logic_error("unexpected decision-log entry in a plan step");
        }
    }
    for (unsigned v : batch) add(out.batch, out.n_batch, (long)v);
    // pushed events in push order (the key's event seq)
    std::vector<pb::HeapEnt> ev = heap;
    std::sort(ev.begin(), ev.end(),
              [](const pb::HeapEnt& a, const pb::HeapEnt& b) { return (a.key >> 29) < (b.key >> 29); });
    for (const pb::HeapEnt& e : ev) {
        const unsigned kind = (unsigned)(e.key >> 26) & 7u;
        const long id = (long)(e.key & ((1u << 26) - 1u));
        if (kind == 3) {  // EV_SWAP
            if (out.swap_event_request) out.swap_event_request[out.n_swap_events] = id;
            if (out.swap_event_time) out.swap_event_time[out.n_swap_events] = e.t;
            ++out.n_swap_events;
        } else {
            out.completion_time = e.t;
        }
    }
    if (out.blocked)
        for (long k = 0; k < n; ++k) out.blocked[k] = blocked[k];
}

void probe_select(int mode, long count, int n, const unsigned char* t, const long* k1,
                  const long* k2, int* out) {
    need(mode >= 0 && mode <= 2, "mode must be 0, 1 or 2");
    need(n >= 1 && n <= 32, "instances per vector must be in [1, 32]");
    need(count >= 0, "negative count");
    need(count == 0 || (t && k1 && out && (mode != 1 || k2)), "null argument");
    if (count == 0) return;
    const size_t m = (size_t)count * n;
    for (size_t k = 0; k < m; ++k) {
        need(k1[k] >= 0 && k1[k] < (1L << 40), "key out of range");
        if (mode == 1) need(k2[k] >= 0 && k2[k] < (1L << 30), "key out of range");
    }
    Scratch sc;
    pb::SelectProbe p{};
    p.mode = mode;
    p.n = n;
    p.count = count;
    p.t = sc.put(std::vector<unsigned char>(t, t + m));
    std::vector<long long> a(k1, k1 + m), b(mode == 1 ? m : 1, 0);
    if (mode == 1) std::copy(k2, k2 + m, b.begin());
    p.k1 = sc.put(a);
    p.k2 = sc.put(b);
    p.out = sc.get<int>((size_t)count);
    // the behind-schedule answering member: one delivery at t0 = 0, its
    // digest known, A = 50 tokens, so at now = 100 with tpot 1 it is 49
    // digests short (instance.cpp:22-33)
    pb::ReqState r{};
    r.h = make_int4(0, 0, 1, 0);
    r.meta = 2u;  // Answering, on the GPU, low queue
    r.ndel = 1;
    r.cursor = 1;
    p.rs = sc.put(std::vector<pb::ReqState>{r});
    p.spec = sc.put(std::vector<int4>{make_int4(0, 0, 50, 0)});
    p.ph = sc.get<pb::PacerHot>(1);
    p.aoff = sc.get<int>(1);
    p.bpk = sc.get<int>(1);
    p.bpv = sc.get<double>(1);
    if (pb::logging::launch_select_probe(p, nullptr))
        throw std::logic_error("select probe launch failed");
    cu(cudaDeviceSynchronize(), "select probe");
    cu(cudaMemcpy(out, p.out, (size_t)count * sizeof(int), cudaMemcpyDeviceToHost), "d2h");
}

}  // namespace pbh
