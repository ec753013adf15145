// engine.h — layout shared by the host driver (engine_host.cpp) and the
// sm_100a scheduling engine (engine.cu).
//
// One warp simulates one replica (one trace under one policy/config) end to
// end: the reference's serial (time, seq) event chain (proj/src/engine.cpp:
// 392-404) stays serial, and each handler's inner loops (queue scans, priority
// partition, admission, plan application, batch retire, monitor snapshots)
// run across the 32 lanes. Many replicas run side by side, one per warp, so a
// replica sweep fills all 148 SMs.
//
// All per-request state is struct-of-arrays in HBM, indexed by
// g = ReplicaDesc::req_base + i (i = trace index). Per-instance state lives in
// shared memory for the lifetime of the replica.
#pragma once

#include <cstdint>

#include <vector_types.h>  // int4 / uint2 (CUDA vector types, host and device)

namespace pb {

enum Policy : int { kFcfs = 0, kRr = 1, kOracle = 2, kPascal = 3 };

// ReplicaDesc::flags
enum : int {
    kNoMigration = 1,   // Ablations::no_migration (proj/include/pascalsim/cluster.hpp:13-16)
    kNonAdaptive = 2,   // Ablations::non_adaptive
    kRecordDeliv = 4,   // keep every answer delivery time (records / parity mode)
    kLogEvents = 8,     // write the decision log (pascal-events-v1 entries)
};

// proj/include/pascalsim/costmodel.hpp:12-21
struct Profile {
    double prefill_base, prefill_per_token;
    double decode_base, decode_per_request, decode_per_kv_token;
    double swap_bandwidth, fabric_bandwidth, fabric_latency;
};

struct ReplicaDesc {
    int n;        // requests
    int ni;       // instances
    int policy;
    int flags;
    long long capacity;  // per-instance KV capacity (tokens)
    long long quantum, demotion, slack;
    double tpot;
    Profile prof;
    long long req_base;    // into request arrays
    long long ans_base;    // into digest/delivery arenas (unused: aoff is absolute)
    long long queue_base;  // into qent: 2 queues per instance, qcap entries each
    long long qcap;
    long long batch_base;  // into batch: ni * n entries
    long long heap_base;   // into heap: n + ni + 2 entries
    long long log_base, log_cap;
    long long plog_base;   // into plog: ni * kParkLog entries (lean Pascal build, parked tails)
    // instance-parallel (PDES) engine only
    long long pheap_base;  // into heap: ni * (n + 2) entries (per-instance heaps)
    double lookahead;      // lower bound on the duration of an event that can create a
                           // cross-instance interaction (Pascal phase boundary)
};

// Counters the device reports per replica (roofline accounting).
struct ReplicaOut {
    int status;      // 0 ok, else kErr*
    int pad;
    long long peak;  // peak sum of gpu_used (engine.cpp:75-79)
    long long nlog;  // log entries produced (may exceed log_cap)
    long long events, plans, visits, req_iters, answer_tokens, health_checks;
    long long adm_rounds, adm_slow;
    double now;      // clock at the end of the run
};

enum : int {
    kErrNone = 0,
    kErrPast = 1,      // "event scheduled in the past"      engine.cpp:86-87
    kErrClock = 2,     // "clock moved backwards"            engine.cpp:395
    kErrCapacity = 3,  // "instance over GPU capacity"       engine.cpp:255-256
    kErrStall = 4,     // "simulation stalled with unfinished requests"  :424
    kErrHeap = 5,      // device heap overflow (internal)
    kErrPdes = 6,      // instance-parallel engine declined (cross-instance time tie or a
                       // bounded buffer overflow): the host re-runs the replica serially
};

// Per-request record, proj/include/pascalsim/metrics.hpp:15-28 (vectors live
// in the digest/delivery arenas; at most one migration per request).
struct RecOut {
    double arrival, prefill_complete, reasoning_end, first_answer_delivery,
        first_answer_iter_start, blocked, completion, mig_start, mig_end;
    int nmig, pad;
};

struct HeapEnt {
    double t;
    unsigned long long key;  // seq(35) | kind(3) | id(26)
};

struct LogEnt {
    double t;
    int req;  // trace index or -1
    int inst;
    int kind;
    int detail;
};

enum LogKind : int {
    kLArrival = 0, kLDemote, kLEvict, kLSwapIn, kLBlock, kLPrefillStart, kLDecodeStart,
    kLPrefillComplete, kLToken, kLTransition, kLMigrate, kLFinish, kLSwapComplete,
    kLTransferComplete
};

// Mutable per-request scheduling state, packed into one 32-byte sector so a
// queue scan touches one sector per request (RequestState,
// proj/include/pascalsim/instance.hpp:41-62).
struct __align__(16) ReqState {
    int4 h;           // {kv_tokens, tokens_generated, enqueue_seq (0 = not queued), quanta_exhausted}
    unsigned meta;    // phase:2 | loc:2 | swin:1 | swout:1 | qlow:1 | owner:16 (<<8)
    int qused;        // quantum_used_in_round
    int ndel;         // delivered answer tokens
    int cursor;       // digests known <= a past `now` (pacer health cursor)
};

// Pacer state of an answering request (PacerState, instance.hpp:22-39) in
// breakpoint form. Digest k is d_k = max(gen_k, d_{k-1} + tpot) with d_0 =
// gen_0 (instance.cpp:10-20); it equals gen_k only at "breakpoints" (the
// first token and tokens generated after the pacing lead ran out) and is
// d_{k-1} + tpot otherwise, so the digest sequence is stored as its
// breakpoints {k, gen_k} (bpk / bpv arenas, ~3 per request on C2 instead of
// one double per answer token) and replayed with the same double additions.
struct __align__(16) PacerHot {
    double dlast;  // d_{nd-1}: last digest (the QoE horizon at finish)
    double dcur;   // d_{cursor-1}: last digest known <= a past `now`
    double t0;     // first delivery (health's t0)
    int nbp;       // breakpoints recorded
    int jn;        // breakpoints consumed by the health cursor
};

// Batch-wide device arenas.
struct Arena {
    const ReplicaDesc* desc;
    ReplicaOut* out;
    int n_rep;
    int* work;  // work-stealing counter
    const int* order;  // replicas in hand-out order (longest predicted first)
    // read-only trace
    const double* arrival;
    const int4* spec;       // {prompt, reasoning, answering, kv_preloaded}
    const long long* aoff;  // absolute offset of the request's answer slots
    const int* aoff32;      // same, relative to the replica's first request
    // mutable request state
    ReqState* rs;     // per-request scheduling state (one 32-byte sector each)
    double* blocked;  // blocked_interval_total accumulator (global-resident replicas)
    RecOut* rec;
    PacerHot* ph;     // per-request pacer state
    double* bpv;      // digest breakpoint values (answer-slot arena)
    int* bpk;         // digest breakpoint token indices (answer-slot arena)
    double* dig;      // full digest times (kRecordDeliv)
    double* del;      // delivery times (kRecordDeliv)
    // queues / batches / events
    uint2* qent;      // {request index, enqueue_seq}
    unsigned* batch;
    HeapEnt* heap;
    // per-replica scratch, n entries each (indexed by req_base)
    int4* cand;
    int4* tmp;
    unsigned* tmpq;
    unsigned char* cstat;
    unsigned* elist;
    unsigned* stack;
    LogEnt* log;
    // lean Pascal build: durations of the plans that skipped an instance's parked
    // tail (kParkLog per instance) and the log index each parked request joined at
    double* plog;
    int* pfrom;
    struct PdesRec* prec;  // PDES: kPdesMaxWarps * kPdesRecCap records per CTA
    int* pord;             // PDES: the same count of ints per CTA (records by rank)
    long long wstride;  // PDES: per-warp scratch copies (cand / tmp / tmpq / cstat / elist /
                        // stack) are wstride entries apart
};

// Per-replica metric parameters (RunConfig fields used by build_report).
struct MetricParams {
    double tpot, qoe_threshold, ttfat_target;
    long long req_base;
    int n;
    int pad;
};

// Device-computed build_report aggregates + counters; same layout as
// pascal_summary in include/pascal_b200.h.
struct DevSummary {
    double ttft_mean, ttft_p50, ttft_p90, ttft_p95, ttft_p99;
    double slo_rate, ttfat_attain, throughput;
    long long capacity, requests, req_iters, answer_tokens, events, plans, visits, health;
    long long slo_violations;
    long long adm_rounds, adm_slow;
    int status, pad;
    double tpot_mean;        // over requests with A > 1
    long long tpot_requests;
};

// Per-request metric outputs (trace order), proj/include/pascalsim/metrics.hpp:58-67.
struct RowArrays {
    double* ttft;
    double* ttfat;
    double* qoe;
    double* blocking;
    unsigned char* slo;
    double* ttft_sorted;
    double* tpot;  // (completion - first answer delivery) / (A - 1); 0 when A <= 1
};

#ifdef __CUDACC__
#define PB_HD __host__ __device__
#else
#define PB_HD
#endif

// Dynamic shared memory per warp: instance state for ni instances; for
// replicas with n <= n_smem also the hot per-request state (60 B each: hot,
// spec, blocked, meta, quantum_used, delivered, cursor, answer offset) and
// the event heap (n + ni + 2 entries of 16 B); and a candidate scratch of
// c_smem entries (37 B each). Larger replicas keep request state and heap in
// HBM; plans with more queued requests than c_smem use the HBM scratch.
// (+32: the replica's fixed-divisor reciprocals, engine.cu rcp_of, ahead of
// the instance arrays)
// (+20 per instance: the parked-tail summary of the lean Pascal build, engine.cu PB_PARK)
PB_HD inline int smem_inst_bytes(int ni) { return ((ni * 84 + 16 + 32) + 15) / 16 * 16; }
// Parked tails (engine.cu PB_PARK): plans an instance may skip its parked
// requests in before they are materialised.
constexpr int kParkLog = 1024;
PB_HD inline int smem_req_bytes(int n_smem) { return (n_smem * 60 + 15) / 16 * 16; }  // rs 32 + spec 16 + blocked 8 + aoff 4
// Shared-memory event heap: sized for every pending event of a resident
// replica; HBM-resident replicas start with h_slots slots (default 128) and
// move their heap to HBM if it ever grows past them.
constexpr int kSmemHeapSlots = 128;
PB_HD inline int smem_heap_bytes(int n_smem, int ni, int h_slots = kSmemHeapSlots) {
    return n_smem ? (n_smem + ni + 2) * 16 : h_slots * 16;
}
// (+ 32 ints of per-warp bucket scratch for the planner's quanta partition,
// engine.cu warp_hist)
PB_HD inline int smem_cand_bytes(int c_smem) { return (c_smem * 37 + 15) / 16 * 16 + 128; }
// HBM-resident replicas with n <= b_smem keep their blocked-time totals (the
// most frequently written per-request value: one read-modify-write per denial)
// in shared memory.
PB_HD inline int smem_blocked_bytes(int b_smem) { return (b_smem * 8 + 15) / 16 * 16; }
PB_HD inline int smem_per_warp(int ni, int n_smem, int c_smem, int h_slots = kSmemHeapSlots,
                               int b_smem = 0) {
    return smem_inst_bytes(ni) + smem_req_bytes(n_smem) + smem_heap_bytes(n_smem, ni, h_slots) +
           smem_cand_bytes(c_smem) + smem_blocked_bytes(b_smem);
}

// Instance-parallel engine (one CTA per replica, W warps, instance i owned by
// warp i % W): shared memory = instance state + per-instance scalars
// (pending cross-instance event time, merge head {time, key}, heap size,
// spill flag, enqueue counter, tokens-to-boundary bound, merge cursor / end:
// 48 B) + per-instance heap slots + per warp a candidate scratch + round
// control. Per warp an HBM buffer of kPdesRecCap event records per round.
constexpr int kPdesMaxWarps = 8;
constexpr int kPdesRecCap = 4096;  // events one warp may process in one round
PB_HD inline int pdes_inst_bytes(int ni, int hs) {
    return smem_inst_bytes(ni) + ni * 48 + ni * hs * 16;
}
// One phase-A event: what the end-of-phase merge needs to assign the exact
// global push sequence numbers (and the oracle's Σ gpu_used samples) in the
// reference's (time, seq) order.
struct PdesRec {
    double t;
    unsigned long long key;  // the event's heap key (global seq, or provisional)
    long long d1, d2;        // change of Σ gpu_used before / after its peak sample
    int inst;                // bit 31: sampled
    int npush;               // heap pushes made while processing it
    unsigned long long gbase;  // merge: global seq before its first push
    int rank;                // merge: position in the round's global order
    int pad;
};
PB_HD inline int pdes_warp_bytes(int c_smem) { return smem_cand_bytes(c_smem); }
PB_HD inline int pdes_ctl_bytes() { return 512; }
PB_HD inline int pdes_smem(int ni, int hs, int c_smem, int warps) {
    return pdes_inst_bytes(ni, hs) + warps * pdes_warp_bytes(c_smem) + pdes_ctl_bytes();
}

// Unit-parity seams (pascal_probe_* in include/pascal_b200.h): one
// maybe_start on a hand-built instance state, run by the logging build's own
// planner (one warp). The host fills the request / queue / instance arrays in
// the engine's layout; the outputs are the decision log, the heap (pushed
// events), the batch list and the instance counters.
struct PlanProbe {
    int n, ni, inst, policy;
    long long cap, quantum, demotion;
    double now;
    Profile prof;
    unsigned enq;  // enqueue seqs handed out so far (demotions take the next ones)
    int c_smem;    // shared-memory candidate slots
    ReqState* rs;
    int4* spec;
    double* arrival;
    double* blocked;
    RecOut* rec;
    PacerHot* ph;
    int* aoff;
    uint2* qent;  // 2 * ni queues of qcap entries
    long long qcap;
    const int* qlen;         // [2 * ni] {high, low} live lengths
    const long long* used;   // [2 * ni] {gpu_used, cpu_used}
    unsigned* batch;         // ni * n
    HeapEnt* heap;           // heap_cap slots (1-based)
    long long heap_cap;
    LogEnt* log;
    long long log_cap;
    int4* cand;
    int4* tmp;
    unsigned* tmpq;
    unsigned char* cstat;
    unsigned* elist;
    unsigned* stack;
    long long* out_used;     // [2 * ni] after the step
    int* out_scal;           // {status, heap entries, log entries, batch length, busy}
};
// Batched Alg. 1 / Alg. 2 evaluation through the engine's select_instance:
// vector v has n instances with on-track flags t[v*n+i] and keys k1 (m_i for
// modes 0 / 2, r_i for mode 1) and k2 (a_i, mode 1).
struct SelectProbe {
    int mode;  // 0 select_instance_reasoning, 1 select_instance_answering, 2 argmin m_i
    int n;
    long long count;
    const unsigned char* t;
    const long long* k1;
    const long long* k2;
    int* out;
    ReqState* rs;  // one behind-schedule answering request (the unhealthy member)
    int4* spec;
    PacerHot* ph;
    int* aoff;
    int* bpk;
    double* bpv;
};

constexpr int kHistBins = 128;  // PASCAL_HIST_BINS

// Host entries (engine.cu / metrics.cu). All enqueue on `stream`.
// Two builds of the engine: `logging` writes the pascal-events-v1 decision
// log (kLogEvents) and the full delivery / digest arrays (kRecordDeliv);
// `nolog` has every log and record site compiled out.
namespace logging {
int launch_engine(const Arena& a, int max_ni, int n_smem, int c_smem, int h_slots, int b_smem,
                  int warps_per_block, int blocks, void* stream);
int launch_plan_probe(const PlanProbe& p, void* stream);
int launch_select_probe(const SelectProbe& p, void* stream);
}
namespace nolog {
int launch_engine(const Arena& a, int max_ni, int n_smem, int c_smem, int h_slots, int b_smem,
                  int warps_per_block, int blocks, void* stream);
}
// Instance-parallel engine for few, large replicas (no decision log): one CTA
// per replica; replicas that return kErrPdes must be re-run serially.
namespace pdes {
int launch_engine(const Arena& a, int max_ni, int hs, int c_smem, int warps, int blocks,
                  void* stream);
}
namespace pdes_pascal {
int launch_engine(const Arena& a, int max_ni, int hs, int c_smem, int warps, int blocks,
                  void* stream);
}
namespace pdes_oracle {
int launch_engine(const Arena& a, int max_ni, int hs, int c_smem, int warps, int blocks,
                  void* stream);
}
// `nolog` specialised to batches whose replicas all run one policy (Pascal,
// Oracle — also the capacity pre-run —, FCFS, RR).
namespace pascal_lean {
int launch_engine(const Arena& a, int max_ni, int n_smem, int c_smem, int h_slots, int b_smem,
                  int warps_per_block, int blocks, void* stream);
}
namespace oracle_lean {
int launch_engine(const Arena& a, int max_ni, int n_smem, int c_smem, int h_slots, int b_smem,
                  int warps_per_block, int blocks, void* stream);
}
namespace fcfs_lean {
int launch_engine(const Arena& a, int max_ni, int n_smem, int c_smem, int h_slots, int b_smem,
                  int warps_per_block, int blocks, void* stream);
}
namespace rr_lean {
int launch_engine(const Arena& a, int max_ni, int n_smem, int c_smem, int h_slots, int b_smem,
                  int warps_per_block, int blocks, void* stream);
}
// capacity = max(ceil(fraction * peak / ni), biggest) for the replicas listed
// in `map`, peak from oracle pre-run oref[k] (derive_capacity,
// proj/src/engine.cpp:466-470); writes echo[r] and, unless the replica runs
// the oracle policy, desc[r].capacity.
int launch_capacity(ReplicaDesc* desc, const ReplicaOut* oracle_out, const int* map,
                    const int* oref, const double* fraction, const long long* biggest,
                    long long* echo, int count, void* stream);
int launch_histograms(const int* rid, const int* group, const RowArrays rows,
                      const ReplicaOut* out, long long total, int n_groups,
                      unsigned long long* hist, unsigned long long* slo, void* stream);
int launch_metrics(const Arena& a, const MetricParams* params, const long long* seg,
                   const int* rid, long long total, int n_rep, RowArrays rows,
                   DevSummary* out, const long long* echo_capacity, void* sort_tmp,
                   size_t* sort_tmp_bytes, void* stream);

}  // namespace pb
