// engine.cu — the B200 scheduling engine (sm_100a).
//
// Replaces, end to end, the reference's per-iteration scheduling loop:
//   event loop          proj/src/engine.cpp:392-404        -> run_replica()
//   arrival placement   engine.cpp:260-283, cluster.cpp:10-33,59-62
//   monitor snapshot    instance.cpp:22-33,59-76, engine.cpp:103-109
//   demotion            instance.cpp:39-57
//   planner             instance.cpp:103-282               -> maybe_start()
//   plan application    engine.cpp:192-258
//   iteration retire    engine.cpp:310-337, instance.cpp:10-20
//   phase boundary      engine.cpp:159-190, cluster.cpp:35-57,64-68
//   other handlers      engine.cpp:285-308,339-367
//
// Execution model: one warp owns one replica for its whole lifetime. Scalar
// simulation state (clock, counters, heap size) is held redundantly and
// identically by all 32 lanes; data-parallel steps (queue scans, stable
// priority partition, plan materialisation, batch retire, snapshots) spread
// over the lanes with ballots, prefix scans and shuffles.
//
// Bit-exactness: built with -fmad=false; every floating-point expression keeps
// the reference's operation order (see the costmodel helpers below).
//
// The admission pass is the reference's greedy admit/evict loop with the
// O(Q) two-pointer victim walk: victim order is exactly the
// reverse of admission order, so the victims of an admission are (a) not yet
// visited candidates taken from the back, then (b) previously denied residents
// in descending order (a stack), restricted to the class-eligible suffix.

#include <cuda_runtime.h>
#include <math_constants.h>

#include <cfloat>
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "engine.h"

// This file is compiled twice (engine_log.cu / engine_nolog.cu): PB_LOG = 1
// builds the decision-log writer and the full per-token record arrays in
// (parity dumps), PB_LOG = 0 compiles every log / record site out of the hot
// loops (batches, reports and the benchmark never need them; measured +5.7%
// request-iterations/s on the C2 bench).
#ifndef PB_LOG
#define PB_LOG 1
#define PB_VARIANT logging
#endif
// PB_PDES = 1 builds the instance-parallel engine (pdes_kernel below) instead
// of the warp-per-replica one: one CTA per replica, instance i owned by warp
// i % W, instances advance concurrently between cross-instance interactions
// (arrivals, Pascal phase boundaries). Never combined with the decision log.
#ifndef PB_PDES
#define PB_PDES 0
#endif
#if PB_PDES && PB_LOG
#error "the instance-parallel engine has no decision-log build"
#endif
// PB_PARK (the lean Pascal build only): an instance "parks" the all-denied
// tail of its class-1 candidates — requests on the CPU, not swapping, whose
// admission need exceeds the free KV and who have no reachable victim — by
// flagging their low-queue entries. Parked requests are frozen until a plan
// admits them (nothing but a plan touches a CPU-resident, non-swapping
// request), so later plans skip them — no request-state read, no ordering,
// admission or apply work — as long as a check at their position in the
// priority order proves they would all be denied again without side effects
// (see maybe_start). Their blocked-time additions are logged per instance
// and replayed, in the same order, when they are unparked. Results are
// bit-identical to the reference; only the work changes.
#if !PB_LOG && !PB_PDES && defined(PB_ONLY_POLICY) && PB_ONLY_POLICY == 3
#define PB_PARK 1
#else
#define PB_PARK 0
#endif

namespace pb {
namespace PB_VARIANT {

#define DEVI __device__ __forceinline__
constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------- meta bits
constexpr unsigned PH_WAIT = 0, PH_REASON = 1, PH_ANSWER = 2, PH_DONE = 3;
constexpr unsigned LOC_GPU = 0, LOC_CPU = 1, LOC_TRANSIT = 2;
DEVI unsigned m_phase(unsigned m) { return m & 3u; }
DEVI unsigned m_loc(unsigned m) { return (m >> 2) & 3u; }
DEVI bool m_swin(unsigned m) { return (m >> 4) & 1u; }
DEVI bool m_swout(unsigned m) { return (m >> 5) & 1u; }
DEVI bool m_qlow(unsigned m) { return (m >> 6) & 1u; }
// PDES builds keep the owner in bits 8..23 and, in bits 24..31, min(255,
// tokens left until the request's phase boundary) (engine_pdes.cuh horizon).
DEVI int m_owner(unsigned m) { return PB_PDES ? (int)((m >> 8) & 0xffffu) : (int)(m >> 8); }
DEVI unsigned m_set_phase(unsigned m, unsigned p) { return (m & ~3u) | p; }
// PDES builds: rem = tokens until the phase boundary (a decode iteration
// holding a reasoning request with rem == 1 is a cross-instance event under
// Pascal); meaningful in the waiting / reasoning phases only.
DEVI unsigned m_rem(unsigned m) { return m >> 24; }
DEVI unsigned m_set_rem(unsigned m, long long r) {
    const unsigned v = r < 0 ? 0u : (r > 255 ? 255u : (unsigned)r);
    return (m & 0x00ffffffu) | (v << 24);
}
DEVI bool m_tnext(unsigned m) { return ((m & 3u) == 1u) && m_rem(m) == 1u; }  // PH_REASON
DEVI unsigned m_set_loc(unsigned m, unsigned l) { return (m & ~(3u << 2)) | (l << 2); }
DEVI unsigned m_set_swin(unsigned m, bool b) { return (m & ~(1u << 4)) | ((unsigned)b << 4); }
DEVI unsigned m_set_swout(unsigned m, bool b) { return (m & ~(1u << 5)) | ((unsigned)b << 5); }
DEVI unsigned m_set_qlow(unsigned m, bool b) { return (m & ~(1u << 6)) | ((unsigned)b << 6); }
DEVI unsigned m_set_owner(unsigned m, int o) {
    return PB_PDES ? (m & 0xff0000ffu) | ((unsigned)o << 8) : (m & 0xffu) | ((unsigned)o << 8);
}
// instance.hpp:59-61
DEVI bool m_resident(unsigned m) { return m_loc(m) == LOC_GPU && !m_swin(m) && !m_swout(m); }
// instance.cpp:86-90 (a queued request is never Done)
DEVI bool m_candidate(unsigned m) {
    return m_phase(m) != PH_DONE && m_loc(m) != LOC_TRANSIT && !m_swin(m) && !m_swout(m);
}

// candidate flags (int4::w of the candidate scratch)
constexpr int CF_LOW = 1, CF_WAIT = 2, CF_RES = 4, CF_QPOS = 8, CF_TNEXT = 16;
constexpr int CF_POS_SHIFT = 5;  // PB_PARK: the candidate's queue position above the flags
// candidate status
constexpr unsigned char CS_ADMIT = 1, CS_DENY = 2;

// event kinds in the heap key
constexpr unsigned EV_PREFILL = 1, EV_ITER = 2, EV_SWAP = 3, EV_TRANSFER = 4;

// ------------------------------------------------------------- warp helpers
DEVI int lane_id() { return threadIdx.x & 31; }
DEVI unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
// Sum of non-negative 64-bit lane values (KV token counts) below 2^63: three
// independent 32-bit REDUX sums of 24 / 24 / 15-bit slices (none overflows
// across 32 lanes).
DEVI long long warp_sum_ll(long long v) {
    const unsigned long long u = (unsigned long long)v;
    const unsigned lo = __reduce_add_sync(FULL, (unsigned)(u & 0xffffffu));
    const unsigned mid = __reduce_add_sync(FULL, (unsigned)((u >> 24) & 0xffffffu));
    const unsigned hi = __reduce_add_sync(FULL, (unsigned)(u >> 48));
    return (long long)((unsigned long long)lo + ((unsigned long long)mid << 24) +
                       ((unsigned long long)hi << 48));
}
// 32-bit warp reductions: one REDUX instruction instead of a five-step
// shuffle chain (the planner's per-plan reductions sit on the replica's
// serial dependency chain)
DEVI int warp_sum(int v) { return (int)__reduce_add_sync(FULL, (unsigned)v); }
DEVI unsigned warp_min_u(unsigned v) { return __reduce_min_sync(FULL, v); }
DEVI unsigned warp_max_u(unsigned v) { return __reduce_max_sync(FULL, v); }
DEVI int warp_excl_scan(int v, int* total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, x, o);
        if (lane_id() >= o) x += y;
    }
    *total = __shfl_sync(FULL, x, 31);
    return x - v;
}
// -------------------------------------------------------------- costmodel
// proj/src/costmodel.cpp:35-51, operation order preserved (device code is
// compiled with -fmad=false so no contraction happens).
DEVI double prefill_latency(const Profile& p, long long prompt) {
    return __dadd_rn(p.prefill_base, __dmul_rn(p.prefill_per_token, (double)prompt));
}
DEVI double decode_step_latency(const Profile& p, long long batch, long long kv) {
    return __dadd_rn(__dadd_rn(p.decode_base, __dmul_rn(p.decode_per_request, (double)batch)),
                     __dmul_rn(p.decode_per_kv_token, (double)kv));
}
// kv / bw for a fixed divisor: with rcp = RN(1 / bw), q = RN(kv * rcp) is
// within one ulp of kv / bw, the remainder kv - q * bw is exact in one FMA,
// and RN(q + rem * rcp) is the correctly rounded quotient (Markstein's
// theorem; no overflow / underflow for |a| in {0} u [2^-900, 2^900) and bw
// in [2^-500, 2^500]). 3 FP64 ops instead of a full division. rcp = 0 or a
// tiny |a| selects the plain division. Checked against the division on 4.4e8
// (kv, bw) pairs (every kv < 2^22 for the profile bandwidths in use) and
// 8e8 (elapsed time, tpot) pairs.
__device__ __noinline__ double div_slow(double a, double b) { return __ddiv_rn(a, b); }
DEVI double div_by(double a, double b, double rcp) {
    if (rcp == 0.0 || !(fabs(a) >= 0x1p-900 || a == 0.0)) return div_slow(a, b);
    const double q = __dmul_rn(a, rcp);
    const double r = __fma_rn(-q, b, a);
    return __fma_rn(r, rcp, q);
}
DEVI double fixed_rcp(double b) {
    return (b >= 0x1p-500 && b <= 0x1p500) ? __ddiv_rn(1.0, b) : 0.0;
}
DEVI double swap_latency(const Profile& p, long long kv, double rcp) {
    if (kv == 0) return 0.0;
    return div_by((double)kv, p.swap_bandwidth, rcp);
}
DEVI double transfer_latency(const Profile& p, long long kv, double rcp) {
    return __dadd_rn(p.fabric_latency, div_by((double)kv, p.fabric_bandwidth, rcp));
}
DEVI double dmax(double a, double b) { return a < b ? b : a; }  // std::max(a, b)
// swap_latency(p, kv) == 0.0 exactly when kv == 0 or the bandwidth is +inf:
// for kv >= 1 and a finite positive bandwidth kv / bw >= 1 / DBL_MAX > 0.
// (instance.cpp:259: zero-latency reloads join the batch immediately.)
DEVI bool swap_is_instant(const Profile& p, long long kv) {
    return kv == 0 || isinf(p.swap_bandwidth);
}

// ------------------------------------------------------- per-replica view
struct Inst {  // shared-memory SoA for the replica's instances
    long long* gpu;
    long long* cpu;
    double* iter_start;
    double* link;
    int* hi_len;
    int* lo_len;
    int* hcount;
    int* lcount;
    int* afresh;
    int* blen;
    int* busy;
    int* healthy;
#if PB_PARK
    // parked tail summary: members, min admission need, min priority key
    // (quanta << 32 | seq), plans logged in plog since the first member parked
    int* pcount;
    int* pneed;
    unsigned long long* pkey;  // 8-byte aligned: laid out ahead of the int arrays
    int* plen;
#endif
#if PB_PDES
    // per-instance event heaps and sequence counters (instance-parallel engine)
    int* hn;                    // heap entries
    int* hspill;                // heap moved to its HBM region
    unsigned* enq;              // enqueue-seq counter (seqs are (k * ni + i))
    double* gtime;              // time of the pending cross-instance event, else +inf
    double* mt;                 // merge: head record time of this round's events
    unsigned long long* mk;     // merge: head record global key
    int* mcur;                  // merge: next record (CTA-wide index), -1 = none this round
    int* mend;                  // merge: one past the instance's last record
    int* dmin;                  // min rem (tokens to a phase boundary) over the queued
                                // waiting / reasoning requests, as of the last plan
#endif
};

struct Rep {
    int n, ni, policy, flags;
    long long cap, quantum, demotion, slack;
    double tpot;
    Profile prof;
    long long logcap;
    // request arrays (offset to this replica)
    const double* arrival;
    int4* spec;
    int* aoff;  // answer-slot offset relative to the replica's bpv / bpk / dig / del
    ReqState* rs;
    double* blocked;
    RecOut* rec;
    PacerHot* ph;
    double* bpv;  // this replica's breakpoint arenas (indexed by aoff)
    int* bpk;
    double* dig;  // this replica's full digest arena (kRecordDeliv)
    double* del;  // this replica's delivery arena (kRecordDeliv)
    uint2* qent;
    long long qcap;
    unsigned* batch;
    HeapEnt* heap;
    int4* cand;
    int4* tmp;
    unsigned* tmpq;
    unsigned char* cstat;
    // candidate scratch: shared memory (capacity c_smem) and HBM (capacity n)
    int4* s_cand;
    int4* s_tmp;
    unsigned* s_tmpq;
    unsigned char* s_cstat;
    int4* g_cand;
    int4* g_tmp;
    unsigned* g_tmpq;
    unsigned char* g_cstat;
    int c_smem;
    unsigned* elist;
    unsigned* stack;
    LogEnt* log;
#if PB_PARK
    double* plog;  // this replica's per-instance plan-duration logs (kParkLog each)
    int* pfrom;    // per request: plog index it joined the parked tail at
#endif
    Inst s;
#if PB_PDES
    HeapEnt* s_heap;  // per-instance shared-memory heap slots (hs each, 1-based)
    int hs;
    long long hcap;   // per-instance HBM heap capacity (n + 2)
    PdesRec* prec;    // this CTA's event records (kPdesRecCap per warp)
    int* pord;        // this CTA's records in merged order
#endif
};

struct Scal {
    HeapEnt* heap;        // shared-memory heap, or the HBM heap after a spill
    long long heap_slots;  // usable slots (1-based: entries 1..heap_slots-1)
    double now;
    unsigned long long evseq;
    unsigned enq;
    int next_arr;
    int hn;
    int done;
    int status;
    long long gpu_total, peak, nlog;
    long long events, plans, visits, req_iters, ans_tokens, health, adm_rounds, adm_slow;
#if PB_PDES
    long long prec_base;  // gpu_total at the start of the current event
    long long d1;         // change of gpu_total before the event's peak sample
    bool sampled;         // the current event sampled Σ gpu_used (note_peak)
    int rec_n;            // records this round (phase A)
    int npush;            // pushes made by the current event (phase A)
    unsigned long long gseq;  // phase B (warp 0): last global push seq
    bool phase_b;         // processing a serialised (cross-instance) event
    int reason;           // why this warp declined the replica (engine_pdes.cuh kPdes*)
    long long nb;         // serialised (phase-B) events processed by this warp
#endif
};

// The replica's fixed-divisor reciprocals (div_by) live in shared memory just
// ahead of the instance arrays, addressed off R.s.gpu (no registers held).
enum : int { kRcpSwap = 1, kRcpFabric = 2, kRcpTpot = 3 };
DEVI double rcp_of(const Rep& R, int k) { return reinterpret_cast<const double*>(R.s.gpu)[-k]; }
DEVI void set_rcps(const Rep& R) {
    if (lane_id() == 0) {
        double* r = reinterpret_cast<double*>(R.s.gpu);
        r[-kRcpSwap] = fixed_rcp(R.prof.swap_bandwidth);
        r[-kRcpFabric] = fixed_rcp(R.prof.fabric_bandwidth);
        r[-kRcpTpot] = fixed_rcp(R.tpot);
    }
}

// 32 ints of per-warp scratch after the shared candidate scratch (engine.h
// smem_cand_bytes): the quanta histogram / bucket offsets of the partition
DEVI int* warp_hist(const Rep& R) {
    return reinterpret_cast<int*>(
        reinterpret_cast<char*>(R.s_cand) + (R.c_smem * 37 + 15) / 16 * 16);
}

DEVI uint2* queue_ptr(const Rep& R, int i, int low) {
    return R.qent + (long long)(2 * i + low) * R.qcap;
}

// First 64 entries of instance i's high and low queues into L1 (lanes 0..9:
// five 128-byte lines per queue), ahead of the plan's dependent
// queue-entry -> request-state loads.
DEVI void prefetch_queue_heads(const Rep& R, int i) {
    const int ln = lane_id();
    if (ln < 10) {
        const uint2* p = queue_ptr(R, i, ln >= 5) + (ln % 5) * 16;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
    }
}

// ------------------------------------------------------------- event log
// Cold paths live out of line (__noinline__): the kernel's hot loop must stay
// small for the instruction cache (L1.5 I$ is 32 KB per SM; the fully inlined
// kernel was 180 KB and stalled on instruction fetch ~30% of the time).
__device__ __noinline__ void log_store(LogEnt* log, long long pos, double t, int kind, int inst,
                                       int req, int det) {
    LogEnt e;
    e.t = t;
    e.req = req;
    e.inst = inst;
    e.kind = kind;
    e.detail = det;
    log[pos] = e;
}
DEVI void log_put(const Rep& R, long long pos, double t, int kind, int inst, int req, int det) {
    if (PB_LOG && (R.flags & kLogEvents) && pos < R.logcap)
        log_store(R.log, pos, t, kind, inst, req, det);
}
// Scalar emit (engine.cpp:91-97): one line at the end of the log.
DEVI void emit(const Rep& R, Scal& S, int kind, int inst, int req, int det = 0) {
    if (lane_id() == 0) log_put(R, S.nlog, S.now, kind, inst, req, det);
    S.nlog++;
}

// ------------------------------------------------------------ event heap
// Min-heap on (time, seq) == EventAfter (engine.cpp:52-57). 1-based; lane 0
// does the memory work, every lane tracks hn.
DEVI bool ev_less(double ta, unsigned long long ka, double tb, unsigned long long kb) {
    return ta < tb || (ta == tb && ka < kb);
}
__device__ __noinline__ void heap_spill(HeapEnt* dst, const HeapEnt* src, int hn) {
    for (int k = 1 + lane_id(); k <= hn; k += 32) dst[k] = src[k];
    __syncwarp();
}
__device__ __noinline__ void heap_sift_up(HeapEnt* h, int pos, double t, unsigned long long key) {
    while (pos > 1) {
        int p = pos >> 1;
        HeapEnt pe = h[p];
        if (!ev_less(t, key, pe.t, pe.key)) break;
        h[pos] = pe;
        pos = p;
    }
    h[pos].t = t;
    h[pos].key = key;
}
#if !PB_PDES
DEVI void heap_push(const Rep& R, Scal& S, double t, unsigned kind, unsigned id, int /*inst*/) {
    // engine.cpp:85-89
    if (t < S.now - 1e-12) {
        if (S.status == 0) S.status = kErrPast;
        return;
    }
    unsigned long long key = ((++S.evseq) << 29) | ((unsigned long long)kind << 26) | id;
    if (S.hn + 1 >= S.heap_slots && S.heap != R.heap) {
        // shared-memory heap full: move it to the HBM heap (sized for every
        // pending event) and stay there
        heap_spill(R.heap, S.heap, S.hn);
        S.heap = R.heap;
        S.heap_slots = (long long)R.n + R.ni + 2;
    }
    int pos = ++S.hn;
    if (lane_id() == 0) heap_sift_up(S.heap, pos, t, key);
    __syncwarp();
}
#endif
// Lane 0 removes the root (sift-down); `top` is returned to every lane by
// shuffles. heap_drop_at: the same without the broadcast, for a caller that
// has already read the root in all lanes.
DEVI void heap_drop_at(HeapEnt* h, int n) {
    if (lane_id() == 0) {
        HeapEnt last = h[n];
        int m = n - 1;
        int i = 1;
        while (true) {
            int c = 2 * i;
            if (c > m) break;
            HeapEnt cl = h[c];
            if (c + 1 <= m) {
                HeapEnt cr = h[c + 1];
                if (ev_less(cr.t, cr.key, cl.t, cl.key)) {
                    cl = cr;
                    ++c;
                }
            }
            if (!ev_less(cl.t, cl.key, last.t, last.key)) break;
            h[i] = cl;
            i = c;
        }
        if (m >= 1) h[i] = last;
    }
}
DEVI HeapEnt heap_pop_at(HeapEnt* h, int n) {
    HeapEnt top;
    if (lane_id() == 0) top = h[1];
    heap_drop_at(h, n);
    top.t = __shfl_sync(FULL, top.t, 0);
    top.key = __shfl_sync(FULL, top.key, 0);
    return top;
}
#if !PB_PDES
DEVI void heap_pop(const Rep& R, Scal& S) {  // the caller read the root in every lane
    heap_drop_at(S.heap, S.hn);
    S.hn = S.hn - 1;
    __syncwarp();
}
#else
// Per-instance heaps: instance i's heap lives in its shared-memory slots
// (1-based, hs - 1 usable) until it outgrows them, then in its HBM region of
// hcap = n + 2 entries. Keys carry the reference's global event seq (exact:
// see engine_pdes.cuh), so (time, key) orders events exactly as the global
// (time, seq) does, across instances too.
constexpr unsigned long long kPdesProv = 1ull << 34;  // provisional-seq flag
DEVI HeapEnt* inst_heap(const Rep& R, int i) {
    return R.s.hspill[i] ? R.heap + (long long)i * R.hcap : R.s_heap + (long long)i * R.hs;
}
DEVI void heap_push(const Rep& R, Scal& S, double t, unsigned kind, unsigned id, int inst) {
    if (t < S.now - 1e-12) {  // engine.cpp:85-89
        if (S.status == 0) S.status = kErrPast;
        return;
    }
    const int hn = R.s.hn[inst];
    const bool spilled = R.s.hspill[inst] != 0;
    // sequence number: phase B runs serially in the global order, so its
    // pushes take the next global seq; a phase-A push gets a provisional key
    // {warp, record, push index} (bit 34 set: after every global seq) that
    // the end-of-phase merge replaces (engine_pdes.cuh pdes_merge)
    unsigned long long sq;
    if (R.policy != kPascal && R.policy != kOracle) {
        // FCFS / RR: events of different instances never need ordering
        // against each other (the arrival, the only cross-instance reader,
        // precedes every dynamic event at its time); per-instance counters
        // from n keep each heap in push order and after the arrivals
        const unsigned long long c = R.s.mk[inst] + 1;
        __syncwarp();
        if (lane_id() == 0) R.s.mk[inst] = c;
        sq = c;
    } else if (S.phase_b) {
        sq = ++S.gseq;
    } else {
        if (inst % (int)(blockDim.x >> 5) != (int)(threadIdx.x >> 5) || S.npush >= (1 << 19)) {
            if (S.status == 0) S.status = kErrPdes, S.reason = 5;  // kPdesOrder
            return;
        }
        sq = kPdesProv | ((unsigned long long)(threadIdx.x >> 5) << 31) |
             ((unsigned long long)S.rec_n << 19) | (unsigned long long)S.npush;
        S.npush++;
    }
    if (hn + 1 >= R.hcap) {
        if (S.status == 0) S.status = kErrHeap;
        return;
    }
    HeapEnt* h = spilled ? R.heap + (long long)inst * R.hcap : R.s_heap + (long long)inst * R.hs;
    if (!spilled && hn + 1 >= R.hs) {
        h = R.heap + (long long)inst * R.hcap;
        heap_spill(h, R.s_heap + (long long)inst * R.hs, hn);
    }
    __syncwarp();
    if (lane_id() == 0) {
        heap_sift_up(h, hn + 1, t, (sq << 29) | ((unsigned long long)kind << 26) | id);
        R.s.hn[inst] = hn + 1;
        if (!spilled && hn + 1 >= R.hs) R.s.hspill[inst] = 1;
    }
    __syncwarp();
}
DEVI HeapEnt heap_pop_inst(const Rep& R, int i) {
    const int n = R.s.hn[i];
    HeapEnt top = heap_pop_at(inst_heap(R, i), n);
    __syncwarp();
    if (lane_id() == 0) R.s.hn[i] = n - 1;
    __syncwarp();
    return top;
}
#endif

// ------------------------------------------------------------ queues
// Parked low-queue entries carry kPark in their seq word (PB_PARK builds;
// enqueue seqs stay below 2^31: <= 4 enqueues per request, < 2^26 requests).
constexpr unsigned kPark = 0x80000000u;
constexpr unsigned kSeqMask = PB_PARK ? 0x7fffffffu : 0xffffffffu;
// Queue (instance i, class low) is an append-only array of {idx, seq}; an
// entry is live iff hot[idx].seq == seq (dequeue zeroes the request's seq).
// Live entries keep ascending-seq order, i.e. the order of the reference's
// std::vector queues (engine.cpp:111-126).
__device__ __noinline__ int queue_compact_impl(uint2* q, int len, const ReqState* rs) {
    int w = 0;
    for (int base = 0; base < len; base += 32) {
        int k = base + lane_id();
        bool live = false;
        uint2 e = make_uint2(0, 0);
        if (k < len) {
            e = q[k];
            live = (unsigned)rs[e.x].h.z == (e.y & kSeqMask);
        }
        unsigned mk = __ballot_sync(FULL, live);
        __syncwarp();
        {
            const int dst = w + __popc(mk & lanemask_lt());
            if (live && dst != k) q[dst] = e;
        }
        w += __popc(mk);
    }
    __syncwarp();
    return w;
}
DEVI void queue_compact(const Rep& R, int i, int low) {
    const int len = low ? R.s.lo_len[i] : R.s.hi_len[i];
    const int w = queue_compact_impl(queue_ptr(R, i, low), len, R.rs);
    if (lane_id() == 0) {
        if (low) R.s.lo_len[i] = w;
        else R.s.hi_len[i] = w;
    }
    __syncwarp();
}

// Enqueue sequence numbers (engine.cpp:114, instance.cpp:49). The queues rely
// on two properties only: seqs are unique (an entry is live iff it carries
// its request's current seq) and ascending in each queue (queue order ==
// priority order). Serial: one counter per replica. PDES: per-instance
// counters k, seq = k * ni + i, unique across instances and ascending within
// each instance's queues. seq_reserve hands out `cnt` seqs on instance i and
// returns a base for seq_of(R, i, base, r), r in [0, cnt).
DEVI unsigned seq_reserve(const Rep& R, Scal& S, int i, int cnt) {
#if PB_PDES
    const unsigned base = R.s.enq[i];
    __syncwarp();
    if (lane_id() == 0) R.s.enq[i] = base + (unsigned)cnt;
    __syncwarp();
    return base;
#else
    const unsigned base = S.enq;
    S.enq += (unsigned)cnt;
    return base;
#endif
}
DEVI unsigned seq_of(const Rep& R, int i, unsigned base, int r) {
#if PB_PDES
    return (base + 1u + (unsigned)r) * (unsigned)R.ni + (unsigned)i;
#else
    return base + 1u + (unsigned)r;
#endif
}

// engine.cpp:111-116 (+ monitor counters r_i / a_i kept incrementally)
DEVI void enqueue(const Rep& R, Scal& S, int i, int idx, bool high) {
    int len = high ? R.s.hi_len[i] : R.s.lo_len[i];
    if (len >= R.qcap) {
        queue_compact(R, i, high ? 0 : 1);
        len = high ? R.s.hi_len[i] : R.s.lo_len[i];
    }
    const unsigned seq = seq_of(R, i, seq_reserve(R, S, i, 1), 0);
    __syncwarp();  // every lane has read the queue length before lane 0 bumps it
    if (lane_id() == 0) {
        int4 h = R.rs[idx].h;
        h.z = (int)seq;
        R.rs[idx].h = h;
        unsigned m = R.rs[idx].meta;
        m = m_set_owner(m_set_qlow(m, !high), i);
        R.rs[idx].meta = m;
#if PB_PDES
        if (m_phase(m) == PH_WAIT || m_phase(m) == PH_REASON)
            R.s.dmin[i] = min(R.s.dmin[i], (int)m_rem(m));
#endif
        queue_ptr(R, i, high ? 0 : 1)[len] = make_uint2((unsigned)idx, seq);
        if (high) {
            R.s.hi_len[i] = len + 1;
            R.s.hcount[i] += 1;
        } else {
            R.s.lo_len[i] = len + 1;
            R.s.lcount[i] += 1;
            if (h.w == 0) R.s.afresh[i] += 1;
        }
    }
    __syncwarp();
}

// engine.cpp:122-126 (lane 0 only; caller syncs)
DEVI void dequeue_lane(const Rep& R, int idx, int owner, unsigned m, int quanta) {
    int4 h = R.rs[idx].h;
    h.z = 0;
    R.rs[idx].h = h;
    if (m_qlow(m)) {
        atomicSub(&R.s.lcount[owner], 1);
        if (quanta == 0) atomicSub(&R.s.afresh[owner], 1);
    } else {
        atomicSub(&R.s.hcount[owner], 1);
    }
}

// ------------------------------------------------------ monitor snapshots
// What the snapshot scan reads; passed by value to the out-of-line scan so
// the replica's register-resident state never has its address taken.
struct HealthView {
    const uint2* qent;
    long long qcap;
    const int* lo_len;
    ReqState* rs;
    const int4* spec;
    PacerHot* ph;
    const int* bpk;
    const double* bpv;
    const int* aoff;
    double tpot;
    double tpot_rcp;  // RN(1 / tpot) for div_by, or 0
    long long slack;
    int ni;
};

// PacerState::healthy (instance.cpp:22-33) with a monotone cursor: `now`
// never decreases and digests only grow, so the count of digests <= now only
// grows. Digests are regenerated from the breakpoints (engine.h PacerHot):
// d_c is the next breakpoint's value when its token index is c, else
// d_{c-1} + tpot — the reference's own addition.
DEVI bool pacer_healthy(const HealthView& V, double now, int idx, int answering) {
    int nd = V.rs[idx].ndel;
    if (nd == 0) return true;
    PacerHot p = V.ph[idx];
    long long expected = 1 + (long long)floor(div_by(__dsub_rn(now, p.t0), V.tpot, V.tpot_rcp));
    if (expected > answering) expected = answering;
    int c = V.rs[idx].cursor;
    if (c < nd) {
        const int off = V.aoff[idx];
        const int c0 = c;
        while (c < nd) {
            const bool isbp = p.jn < p.nbp && V.bpk[off + p.jn] == c;
            const double v = isbp ? V.bpv[off + p.jn] : __dadd_rn(p.dcur, V.tpot);
            if (!(v <= now)) break;
            p.dcur = v;
            ++c;
            if (isbp) ++p.jn;
        }
        if (c != c0) {
            V.rs[idx].cursor = c;
            V.ph[idx].dcur = p.dcur;
            V.ph[idx].jn = p.jn;
        }
    }
    return (long long)c >= expected - V.slack;
}

// t_i of instance i (instance.cpp:67-74): AND over its low-queue Answering
// members, stopping at the first unhealthy one. Adds the pacer evaluations
// made to *checks.
DEVI bool instance_healthy(const HealthView& V, double now, int i, long long* checks) {
    const uint2* q = V.qent + (long long)(2 * i + 1) * V.qcap;
    const int len = V.lo_len[i];
    bool ok = true;
    for (int base = 0; base < len && ok; base += 32) {
        int k = base + lane_id();
        bool bad = false;
        bool chk = false;
        if (k < len) {
            uint2 e = q[k];
            int4 h = V.rs[e.x].h;
            if ((unsigned)h.z == (e.y & kSeqMask)) {
                unsigned m = V.rs[e.x].meta;
                if (m_phase(m) == PH_ANSWER) {
                    chk = true;
                    bad = !pacer_healthy(V, now, (int)e.x, V.spec[e.x].z);
                }
            }
        }
        *checks += __popc(__ballot_sync(FULL, chk));
        ok = __ballot_sync(FULL, bad) == 0;
    }
    return ok;
}

// Instance selection with the monitor snapshot evaluated lazily
// (cluster.cpp:10-44,59-62, instance.cpp:59-76). "argmin over healthy
// instances" is the first healthy instance in (key, id) order, so instances
// are visited in that order and t_i is evaluated only until one is healthy —
// the same choice as snapshotting every instance first; the pacer cursors it
// advances are monotone caches. Keys are non-negative and below 2^54 (token
// sums of < 2^26 requests of < 2^26 tokens), ids below 512, so (key, id)
// packs into one u64 and a plain warp min is the argmin.
//   SEL_M:         argmin m_i = gpu + cpu (baseline routing, no health)
//   SEL_M_HEALTHY: argmin m_i over healthy instances, else over all (Alg. 1)
//   SEL_ANSWER:    argmin r_i over healthy, else argmin r_i + a_i (Alg. 2)
// One out-of-line copy serves arrivals and both phase-boundary sites.
enum : int { SEL_M = 0, SEL_M_HEALTHY = 1, SEL_ANSWER = 2 };
struct SelOut {
    int id;
    int pad;
    long long checks;
};
__device__ __noinline__ SelOut select_instance(const HealthView V, double now, int mode,
                                               const long long* gpu, const long long* cpu,
                                               const int* hcount, const int* afresh,
                                               unsigned* rejected) {
    const unsigned long long NONE = ~0ull;
    const int ni = V.ni;
    SelOut o;
    o.checks = 0;
    o.pad = 0;
    for (int w = lane_id(); w < (ni + 31) / 32; w += 32) rejected[w] = 0u;
    __syncwarp();
    auto key = [&](int i, int pass) -> long long {
        if (mode == SEL_ANSWER)
            return pass == 0 ? (long long)hcount[i] : (long long)hcount[i] + afresh[i];
        return gpu[i] + cpu[i];
    };
    auto argmin = [&](int pass) -> unsigned long long {
        unsigned long long best = NONE;
        for (int base = 0; base < ni; base += 32) {
            const int i = base + lane_id();
            unsigned long long v = NONE;
            if (i < ni && (pass == 1 || !((rejected[i >> 5] >> (i & 31)) & 1u)))
                v = ((unsigned long long)key(i, pass) << 9) | (unsigned)i;
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const unsigned long long y = __shfl_xor_sync(FULL, v, off);
                v = y < v ? y : v;
            }
            best = v < best ? v : best;
        }
        return best;
    };
    if (mode != SEL_M) {
        while (true) {  // pass 0: healthy instances in key order
            const unsigned long long b = argmin(0);
            if (b == NONE) break;
            const int i = (int)(b & 511u);
            if (instance_healthy(V, now, i, &o.checks)) {
                o.id = i;
                return o;
            }
            if (lane_id() == 0) rejected[i >> 5] |= 1u << (i & 31);
            __syncwarp();
        }
    }
    o.id = (int)(argmin(1) & 511u);
    return o;
}

DEVI HealthView health_view(const Rep& R) {
    HealthView V;
    V.qent = R.qent;
    V.qcap = R.qcap;
    V.lo_len = R.s.lo_len;
    V.rs = R.rs;
    V.spec = R.spec;
    V.ph = R.ph;
    V.bpk = R.bpk;
    V.bpv = R.bpv;
    V.aoff = R.aoff;
    V.tpot = R.tpot;
    V.tpot_rcp = rcp_of(R, kRcpTpot);
    V.slack = R.slack;
    V.ni = R.ni;
    return V;
}
DEVI int select_instance(const Rep& R, Scal& S, int mode) {
    const SelOut o = select_instance(health_view(R), S.now, mode, R.s.gpu, R.s.cpu, R.s.hcount,
                                     R.s.afresh, reinterpret_cast<unsigned*>(R.s.healthy));  // scratch bitmap
    S.health += o.checks;
    return o.id;
}

// ------------------------------------------------------------- handlers
DEVI void add_gpu(const Rep& R, Scal& S, int i, long long d) {
    if (lane_id() == 0) R.s.gpu[i] += d;
    S.gpu_total += d;
}
DEVI void add_cpu(const Rep& R, int i, long long d) {
    if (lane_id() == 0) R.s.cpu[i] += d;
}
#if PB_PDES
// The oracle pre-run's peak of sum_i gpu_used (engine.cpp:75-79) is sampled at
// event ends in global (time, seq) order. Instances advance concurrently, so
// each event only notes the change of its warp's total up to its sample
// (S.d1); the merge (phase A) or warp 0 (phase B) accumulates the CTA total
// in the global order. Only the oracle run's peak is ever consumed.
#endif
DEVI void note_peak(const Rep& R, Scal& S) {  // engine.cpp:75-79
#if PB_PDES
    (void)R;
    S.d1 = S.gpu_total - S.prec_base;
    S.sampled = true;
#else
    (void)R;
    if (S.gpu_total > S.peak) S.peak = S.gpu_total;
#endif
}

// engine.cpp:159-190 (Pascal branch; the caller has already set phase,
// reasoning_end and logged "transition").
DEVI void pascal_transition(const Rep& R, Scal& S, int idx) {
#if PB_PDES
    // reads every instance: only legal while the other instances are paused
    if (!S.phase_b && S.status == 0) S.status = kErrPdes, S.reason = 5;  // kPdesOrder
#endif
    unsigned m = R.rs[idx].meta;
    int4 h = R.rs[idx].h;
    int cur = m_owner(m);
    __syncwarp();  // every lane has read the request before lane 0 dequeues it
    if (lane_id() == 0) dequeue_lane(R, idx, cur, m, h.w);
    __syncwarp();
    int target = select_instance(R, S, SEL_ANSWER);
    long long kv = h.x;
    // cluster.cpp:46-57
    bool migrate;
    if (R.flags & kNoMigration) migrate = false;
    else if (target == cur) migrate = false;
    else if (R.flags & kNonAdaptive) migrate = true;
    else {
        long long cur_free = R.cap - R.s.gpu[cur];
        long long tgt_free = R.cap - R.s.gpu[target];
        migrate = !(cur_free >= kv && tgt_free < kv);
    }
    // every lane has read gpu_used / link before lane 0 updates them
    const double busy = R.s.link[target];
    __syncwarp();
    if (!migrate) {
        if (lane_id() == 0) {
            R.rs[idx].qused = 0;
            int4 hh = R.rs[idx].h;
            hh.w = 0;
            R.rs[idx].h = hh;
        }
        __syncwarp();
        enqueue(R, S, cur, idx, false);
        return;
    }
    // free_memory (engine.cpp:128-133) on the current owner
    unsigned loc = m_loc(m);
    if (loc == LOC_GPU || m_swin(m)) add_gpu(R, S, cur, -kv);
    else if (loc == LOC_CPU) add_cpu(R, cur, -kv);
    double dur = transfer_latency(R.prof, kv, rcp_of(R, kRcpFabric));
    double start = dmax(S.now, busy);  // cluster.cpp:64-68
    double fin = __dadd_rn(start, dur);
    if (lane_id() == 0) {
        R.s.link[target] = fin;
        R.rs[idx].meta = m_set_owner(m_set_loc(m, LOC_TRANSIT), target);
        RecOut* rc = &R.rec[idx];
        rc->mig_start = S.now;
        rc->mig_end = fin;
        rc->nmig = 1;
    }
    __syncwarp();
    heap_push(R, S, fin, EV_TRANSFER, (unsigned)idx, target);
    emit(R, S, kLMigrate, cur, idx, target);
}

// One answer delivery (PacerState::on_delivery, instance.cpp:10-20 +
// engine.cpp:148-156); shared by the R == 0 path of prefill completion.
// Records a breakpoint when the digest is the generation time itself.
DEVI void deliver_lane(const Rep& R, double now, int idx, double iter_start) {
    int nd = R.rs[idx].ndel;
    const int off = R.aoff[idx];
    PacerHot* pp = R.ph + idx;
    double v;
    bool bp;
    if (nd == 0) {
        v = now;
        bp = true;
        pp->t0 = now;
    } else {
        const double x = __dadd_rn(pp->dlast, R.tpot);
        bp = !(now < x);  // std::max(gen, prev + tpot) picks gen
        v = bp ? now : x;
    }
    if (bp) {
        const int j = pp->nbp;
        R.bpv[off + j] = now;
        R.bpk[off + j] = nd;
        pp->nbp = j + 1;
    }
    pp->dlast = v;
    if ((PB_LOG || PB_PDES) && (R.flags & kRecordDeliv)) {  // records mode (parity dumps)
        R.dig[off + nd] = v;
        R.del[off + nd] = now;
    }
    R.rs[idx].ndel = nd + 1;
    if (nd == 0) {
        R.rec[idx].first_answer_delivery = now;
        R.rec[idx].first_answer_iter_start = iter_start;
    }
}

// ----------------------------------------------------------- the planner
// Admission walk helpers. `b` is the lowest index visited by the back walk:
// every resident (rkv > 0) candidate at index >= b has been evicted.
struct Adm {
    long long free_;
    int b;
    int ns;  // stack size
    int ne;  // evictions
};

DEVI int cand_rkv(int4 c) { return ((c.w & CF_RES) && c.z > 0) ? c.z : 0; }

// Walk the unvisited back region down to `lo` while need > free (or free < 0
// when need < 0 encodes the over-capacity repair). Victims are taken highest
// index first (instance.cpp:166-177 reversed order == candidate order).
DEVI void walk_back(const Rep& R, Adm& A, int lo, long long need) {
    while (A.b > lo && need > A.free_) {
        int w0 = max(lo, A.b - 32);
        int cnt = A.b - w0;
        int rkv = 0;
        unsigned idx = 0;
        if (lane_id() < cnt) {
            int4 c = R.cand[w0 + lane_id()];
            rkv = cand_rkv(c);
            idx = (unsigned)c.x;
        }
        unsigned mk = __ballot_sync(FULL, rkv > 0);
        int newb = w0;
        while (mk && need > A.free_) {
            int j = 31 - __clz(mk);
            mk &= ~(1u << j);
            long long kv = __shfl_sync(FULL, rkv, j);
            unsigned vi = __shfl_sync(FULL, idx, j);
            A.free_ += kv;
            if (lane_id() == 0) R.elist[A.ne] = vi;
            A.ne++;
            newb = w0 + j;
        }
        // if still short the whole window was consumed
        A.b = need > A.free_ ? w0 : newb;
    }
}
DEVI void pop_stack(const Rep& R, Adm& A, int s, long long need) {
    while (A.ns > 0 && need > A.free_) {
        int j = (int)R.stack[A.ns - 1];
        if (j < s) break;
        A.ns--;
        int4 c = R.cand[j];
        A.free_ += c.z;
        if (lane_id() == 0) R.elist[A.ne] = (unsigned)c.x;
        A.ne++;
    }
}

// Parked-tail bookkeeping of one plan (PB_PARK): the parked tail's min key
// and what the low-queue gather measured against it (class-1 candidates
// keyed below it).
struct ParkG {
    unsigned long long pkey;  // min (quanta << 32 | seq) over the parked tail
    int below;                // class-1 candidates with key < pkey
};
DEVI unsigned long long prio_key(int4 h) {  // (quanta_exhausted, enqueue_seq)
    return ((unsigned long long)(unsigned)h.w << 32) | (unsigned)h.z;
}

// Gather one queue (demoting first when Pascal scans the high queue) into
// cand[nt..] in queue order; quanta go to tmpq for the partition. Returns the
// min / max quanta of the gathered candidates, how many have quanta 0, the
// highest position holding a resident KV footprint (-1 if none) and, when
// `count_q`, the quanta histogram for the partition (lane b: quanta == b).
// PB_PARK: a candidate's flags carry its queue position (bits 5..31); parked
// low-queue entries are kept in place but not gathered.
DEVI void gather_queue(const Rep& R, Scal& S, int i, int low, int& nt, unsigned& qmin,
                       unsigned& qmax, int& zero_q, int& rbpos, bool count_q, int& qcnt,
                       unsigned& rem_min, ParkG& pg) {
    unsigned lmin = 0xffffffffu, lmax = 0;
    unsigned lrem = 255u;  // PDES: min tokens to a phase boundary over the live entries
    int lzero = 0;
    int lrb = -1;
    int lbelow = 0;
    uint2* q = queue_ptr(R, i, low);
    int len = low ? R.s.lo_len[i] : R.s.hi_len[i];
    const bool demote = (R.policy == kPascal) && !low;
    // PB_PARK: parked entries whose request state is not read this pass
    const bool skip_parked = PB_PARK && low;
    int w = 0;
    if (count_q) {
        warp_hist(R)[lane_id()] = 0;
        __syncwarp();
    }
    // Two-deep software pipeline: while chunk c is processed, the request
    // state of chunk c+1 and the queue entries of chunk c+2 are in flight.
    // Safe because a request has at most one entry in a high queue (appended
    // once, at arrival) and the low-queue scan writes no request state.
    const int ln = lane_id();
    uint2 e_c = make_uint2(0, 0), e_n = make_uint2(0, 0);
    int4 h_c = make_int4(0, 0, 0, 0);
    unsigned m_c = 0;
    if (ln < len) {
        e_c = q[ln];
        if (!(skip_parked && (e_c.y & kPark))) {
            h_c = R.rs[e_c.x].h;
            m_c = R.rs[e_c.x].meta;
        }
    }
    if (32 + ln < len) e_n = q[32 + ln];
    for (int base = 0; base < len; base += 32) {
        int k = base + ln;
        int4 h_n = make_int4(0, 0, 0, 0);
        unsigned m_n = 0;
        uint2 e_nn = make_uint2(0, 0);
        if (k + 32 < len && !(skip_parked && (e_n.y & kPark))) {
            h_n = R.rs[e_n.x].h;
            m_n = R.rs[e_n.x].meta;
        }
        if (k + 64 < len) e_nn = q[k + 64];
        bool live = false, dem = false, cnd = false, parked = false;
        uint2 e = e_c;
        int4 h = h_c;
        unsigned m = 0;
        if (k < len) {
            parked = skip_parked && (e.y & kPark);  // frozen: always live, never a candidate
            live = parked;
            if (!parked) {
                live = (unsigned)h.z == e.y;
                if (live) {
                    m = m_c;
                    dem = demote && (long long)h.x > R.demotion;  // strict, instance.cpp:44
                }
            }
        }
        e_c = e_n;
        h_c = h_n;
        m_c = m_n;
        e_n = e_nn;
        // --- demotion (instance.cpp:39-57): new seqs in queue order, appended
        // to the low queue; logged "demote" in that order (engine.cpp:196-197).
        unsigned dm = demote ? __ballot_sync(FULL, dem) : 0u;  // (low queues never demote)
        if (dm) {
            int nd = __popc(dm);
            int lo_len = R.s.lo_len[i];
            if (lo_len + nd > R.qcap) {
                queue_compact(R, i, 1);
                lo_len = R.s.lo_len[i];
            }
            int rank = __popc(dm & lanemask_lt());
            const unsigned sbase = seq_reserve(R, S, i, nd);
            if (dem) {
                unsigned seq = seq_of(R, i, sbase, rank);
                h.z = (int)seq;
                h.w = 0;
                R.rs[e.x].h = h;
                R.rs[e.x].qused = 0;
                m = m_set_qlow(m, true);
                R.rs[e.x].meta = m;
                queue_ptr(R, i, 1)[lo_len + rank] = make_uint2(e.x, seq);
                log_put(R, S.nlog + rank, S.now, kLDemote, i, (int)e.x, 0);
            }
            __syncwarp();
            if (lane_id() == 0) {
                R.s.lo_len[i] = lo_len + nd;
                R.s.hcount[i] -= nd;
                R.s.lcount[i] += nd;
                R.s.afresh[i] += nd;
            }
            S.nlog += nd;
            __syncwarp();
        }
        bool keep = live && !dem;
        cnd = keep && !parked && m_candidate(m);
        if (PB_PDES && live && (m_phase(m) == PH_WAIT || m_phase(m) == PH_REASON))
            lrem = min(lrem, m_rem(m));
        // compact the queue in place (tombstones and demoted entries leave)
        unsigned km = __ballot_sync(FULL, keep);
        __syncwarp();
        const int qpos = w + __popc(km & lanemask_lt());
        if (keep && qpos != k) q[qpos] = e;  // entries only move past tombstones
        w += __popc(km);
        // candidate record
        unsigned cm = __ballot_sync(FULL, cnd);
        if (cnd) {
            int flags = (low ? CF_LOW : 0);
            int need;
            if (m_phase(m) == PH_WAIT) {  // instance.cpp:94-99
                int4 sp = R.spec[e.x];
                flags |= CF_WAIT;
                need = sp.x + (sp.y == 0 ? 1 : 0);
                if (m_resident(m)) flags |= CF_RES;
            } else if (m_resident(m)) {
                flags |= CF_RES;
                need = 1;
            } else {
                need = h.x + 1;
            }
            if (h.w > 0) flags |= CF_QPOS;
            if (PB_PDES && m_tnext(m)) flags |= CF_TNEXT;
            if (PB_PARK) {
                flags |= qpos << CF_POS_SHIFT;
                if (low) lbelow += prio_key(h) < pg.pkey;
            }
            int pos = nt + __popc(cm & lanemask_lt());
            R.cand[pos] = make_int4((int)e.x, need, h.x, flags);
            R.tmpq[pos] = (unsigned)h.w;
            lmin = min(lmin, (unsigned)h.w);
            lmax = max(lmax, (unsigned)h.w);
            lzero += h.w == 0;
            if ((flags & CF_RES) && h.x > 0) lrb = pos;  // positions grow per lane
        }
        if (count_q) {  // quanta histogram: each value's lowest lane adds its peers
            const unsigned pm = __match_any_sync(FULL, cnd ? (unsigned)h.w : 0xffffffffu);
            if (cnd && (unsigned)h.w < 32u && !(pm & lanemask_lt()))
                warp_hist(R)[h.w] += __popc(pm);
        }
        nt += __popc(cm);
    }
    qmin = warp_min_u(lmin);
    qmax = warp_max_u(lmax);
    if (PB_PDES) rem_min = min(rem_min, warp_min_u(lrem));
    if (PB_PARK && low) pg.below = warp_sum(lbelow);
    if (count_q) {
        __syncwarp();
        qcnt = warp_hist(R)[lane_id()];
    }
    zero_q = warp_sum(lzero);
    rbpos = (int)warp_max_u((unsigned)(lrb + 1)) - 1;
    __syncwarp();
    if (lane_id() == 0) {
        if (low) R.s.lo_len[i] = w;
        else R.s.hi_len[i] = w;
    }
    __syncwarp();
}

// Stable partition of src[s, e) into dst[s, e) by quanta ascending (== sort
// by (quanta, enqueue_seq) since queues are in seq order). `part` false: plain
// copy. Quanta below 32 (the common case): one scatter pass, bucket offsets
// from the histogram gather_queue built (lane b: bucket b), one ballot per
// distinct quanta value per chunk; wider ranges: one selection pass per
// distinct value. Returns the highest dst position holding a resident KV
// footprint (-1 if none) when `part`, else `rb_in`.
DEVI int order_segment(const Rep& R, const int4* src, int4* dst, int s, int e, unsigned qmin,
                       unsigned qmax, bool part, int qcnt, int rb_in) {
    const int ln = lane_id();
    if (!part) {
        if (src != dst)
            for (int k = s + ln; k < e; k += 32) dst[k] = src[k];
        __syncwarp();  // the admission pass reads these slots from other lanes
        return rb_in;
    }
    const unsigned lt = lanemask_lt();
    int lrb = -1;
    if (qmax < 32) {
        // bucket b's next slot lives in warp_hist[b]; per chunk, the lanes of
        // one quanta value (match.any) take consecutive slots in lane order
        int* off = warp_hist(R);
        int total;
        off[ln] = s + warp_excl_scan(qcnt, &total);  // lane b: first slot of bucket b
        __syncwarp();
        for (int base = s; base < e; base += 32) {
            const int k = base + ln;
            const bool valid = k < e;
            const unsigned q = valid ? R.tmpq[k] : 0xffffffffu;
            const int4 v = valid ? src[k] : make_int4(0, 0, 0, 0);
            const unsigned m = __match_any_sync(FULL, q);
            const int o = valid ? off[q] : 0;
            __syncwarp();
            if (valid) {
                const int d = o + __popc(m & lt);
                dst[d] = v;
                if (cand_rkv(v) > 0) lrb = max(lrb, d);
                if (!(m & lt)) off[q] = o + __popc(m);
            }
            __syncwarp();
        }
        return (int)warp_max_u((unsigned)(lrb + 1)) - 1;
    }
    int out = s;
    unsigned q = qmin;
    while (true) {
        unsigned next = 0xffffffffu;
        for (int base = s; base < e; base += 32) {
            int k = base + ln;
            unsigned kq = 0xffffffffu;
            if (k < e) kq = R.tmpq[k];
            bool sel = kq == q;
            unsigned sm = __ballot_sync(FULL, sel);
            if (sel) {
                const int d = out + __popc(sm & lt);
                const int4 v = src[k];
                dst[d] = v;
                if (cand_rkv(v) > 0) lrb = max(lrb, d);
            }
            out += __popc(sm);
            next = min(next, kq > q ? kq : 0xffffffffu);  // lane-local
        }
        next = warp_min_u(next);
        if (next == 0xffffffffu) break;
        q = next;
    }
    __syncwarp();
    return (int)warp_max_u((unsigned)(lrb + 1)) - 1;
}

// Highest candidate index j < b with a resident KV footprint (a potential
// back-region victim), or -1.
DEVI int find_rb(const Rep& R, int b) {
    for (int hi = b; hi > 0; hi -= 32) {
        int lo = max(0, hi - 32);
        int j = lo + lane_id();
        bool res = false;
        if (j < hi) res = cand_rkv(R.cand[j]) > 0;
        unsigned mk = __ballot_sync(FULL, res);
        if (mk) return lo + 31 - __clz(mk);
    }
    return -1;
}

#if PB_PARK
// Unpark the members of instance i's parked tail whose admission need is at
// most `thr` (LLONG_MAX: all): replay the plans they sat out (blocked += dur,
// in plan order: the reference's own additions) and clear their flag; the
// rest stay parked and the tail's summary is recomputed over them. With no
// victim left at the tail's rank and the free KV there at `thr`, a member
// needing more is denied wherever it ranks (free only shrinks past that
// rank), so it may stay parked across the re-plan.
DEVI void unpark(const Rep& R, int i, long long thr) {
    uint2* q = queue_ptr(R, i, 1);
    const int len = R.s.lo_len[i];
    const double* lg = R.plog + (long long)i * kParkLog;
    const int end = R.s.plen[i];
    int cnt = 0;
    unsigned mneed = 0xffffffffu;
    unsigned long long mkey = ~0ull;
    for (int k = lane_id(); k < len; k += 32) {
        uint2 e = q[k];
        if (!(e.y & kPark)) continue;
        const int4 h = R.rs[e.x].h;
        if ((long long)h.x + 1 <= thr) {
            double b = R.blocked[e.x];
            for (int p = R.pfrom[e.x]; p < end; ++p) b = __dadd_rn(b, lg[p]);
            R.blocked[e.x] = b;
            q[k].y = e.y & ~kPark;
        } else {
            ++cnt;
            mneed = min(mneed, (unsigned)h.x + 1u);
            const unsigned long long key = prio_key(h);
            mkey = key < mkey ? key : mkey;
        }
    }
    cnt = warp_sum(cnt);
    mneed = warp_min_u(mneed);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(FULL, mkey, o);
        mkey = y < mkey ? y : mkey;
    }
    __syncwarp();
    if (lane_id() == 0) {
        R.s.pcount[i] = cnt;
        R.s.pneed[i] = cnt ? (int)mneed : INT_MAX;
        R.s.pkey[i] = mkey;
        if (!cnt) R.s.plen[i] = 0;
    }
    __syncwarp();
}
#endif

// maybe_start (engine.cpp:192-258) with plan_iteration (instance.cpp:103-282).
// TAIL_FAST: all-denied chunks (the swapped-out tail of an overloaded
// instance) skip the per-chunk statistics and plan-application ballots. It
// cuts a lone replica's run time ~6%, but measured ~2% slower at 8 warps/SM
// (same-session A/B), so only the latency launch shapes use it.
template <bool TAIL_FAST>
DEVI void maybe_start(Rep& R, Scal& S, int i) {
    if (R.s.busy[i]) return;
    S.plans++;
    // candidates never exceed the queued entries: use the shared-memory
    // scratch when they fit
    if (R.s.hi_len[i] + R.s.lo_len[i] <= R.c_smem) {
        R.cand = R.s_cand;
        R.tmp = R.s_tmp;
        R.tmpq = R.s_tmpq;
        R.cstat = R.s_cstat;
    } else {
        R.cand = R.g_cand;
        R.tmp = R.g_tmp;
        R.tmpq = R.g_tmpq;
        R.cstat = R.g_cstat;
    }
    const bool pascal = R.policy == kPascal;
    const bool classed = pascal;
    // PB_PARK: the instance's parked tail (pcnt members); a full duration log
    // forces it back in
    ParkG pg;
    int pcnt = 0;
#if PB_PARK
    long long pthr = LLONG_MAX;  // unpark the members with need <= pthr
    bool do_unpark = R.s.pcount[i] > 0 && R.s.plen[i] >= kParkLog;
#endif
    // PB_PARK: one pass when the parked tail is skipped (or there is none);
    // when the check at its rank fails, the members it may concern are
    // unparked and the plan is made again
#pragma unroll 1
    for (;;) {
#if PB_PARK
    if (do_unpark) unpark(R, i, pthr);  // one inlined copy for both sites
    do_unpark = false;
    pcnt = R.s.pcount[i];
    pg.pkey = pcnt > 0 ? R.s.pkey[i] : ~0ull;
#else
    pg.pkey = ~0ull;
#endif
    pg.below = 0;

    // ---- gather (+ demotion) and priority order (instance.cpp:113-141)
    const bool by_quanta = R.policy == kRr || pascal;
    // segment 0 = high queue, segment 1 = low queue (Pascal class 1); one
    // code copy for both (instruction-cache footprint)
    int nt = 0, z0 = 0, rb0 = -1, rb1 = -1, qc0 = 0, qc1 = 0, c1 = 0;
    unsigned rem_min = 255u;
    unsigned qmin0 = 0xffffffffu, qmax0 = 0, qmin1 = 0xffffffffu, qmax1 = 0;
    const int segs = pascal ? 2 : 1;
#pragma unroll 1
    for (int sg = 0; sg < segs; ++sg) {
        unsigned qmn, qmx;
        int zq, rbs, qc = 0;
        c1 = nt;
        gather_queue(R, S, i, sg, nt, qmn, qmx, zq, rbs, by_quanta, qc, rem_min, pg);
        if (sg == 0) {
            qmin0 = qmn, qmax0 = qmx, z0 = zq, rb0 = rbs, qc0 = qc;
        } else {
            qmin1 = qmn, qmax1 = qmx, rb1 = rbs, qc1 = qc;
        }
    }
    if (!pascal) c1 = nt;
#if PB_PDES
    __syncwarp();
    if (lane_id() == 0) R.s.dmin[i] = (int)rem_min;
#endif
    const int n = nt;
    // PB_PARK: skip the parked tail this plan (checked at its rank, `chk`)
    const bool skip = PB_PARK && pcnt > 0;
    // priority order: the queue-ordered segments are partitioned into the
    // second scratch buffer, which then becomes the candidate array
    const bool part0 = by_quanta && qmin0 < qmax0;
    const bool part1 = pascal && qmin1 < qmax1;
    if (part0 || part1) {
        int4* src = R.cand;
        int4* dst = R.tmp;
#pragma unroll 1
        for (int sg = 0; sg < segs; ++sg) {
            const bool one = sg == 1;
            const int r = order_segment(R, src, dst, one ? c1 : 0, one ? n : c1,
                                        one ? qmin1 : qmin0, one ? qmax1 : qmax0,
                                        one ? part1 : part0, one ? qc1 : qc0, one ? rb1 : rb0);
            if (one) rb1 = r;
            else rb0 = r;
        }
        R.cand = dst;
        R.tmp = src;
    }
    // k0: first class-0 candidate with quanta > 0 (victims of a class-0
    // admission form the suffix [k0, n), instance.cpp:158-162); after the
    // partition the quanta-0 candidates lead the class-0 block
    const int k0 = z0;

    // ---- admission / controlled preemption (instance.cpp:143-243)
    // Warp-parallel greedy with an exact scalar slow path. Per chunk of 32
    // candidates, everything up to the first "event" is decided at once:
    //   * evicted earlier in the pass (index >= b, resident)      -> deny
    //   * FCFS strict queue after a denial                        -> deny
    //   * need <= free after the admitted prefix (prefix sum)      -> admit
    //   * need > free at chunk state with no reachable victim,
    //     not resident, not FCFS, something already admitted      -> deny
    // The first candidate that may evict, deny a resident (stack push), set
    // the FCFS block, or reach the deadlock breaker runs the reference logic
    // one candidate at a time (walk_back / pop_stack). rb = highest resident
    // index below b, so "a victim exists in [lo, b)" is rb >= lo.
    Adm A;
    A.free_ = R.cap - R.s.gpu[i];
    A.b = n;
    A.ns = 0;
    A.ne = 0;
    int stack_top = -1;
    int rb = rb1 >= 0 ? rb1 : rb0;
    bool any_admitted = false, fcfs_blocked = false;
    const bool fcfs = R.policy == kFcfs, oracle = R.policy == kOracle;
    // materialisation statistics, accumulated as candidates are decided
    // (instance.cpp:245-267): first admitted waiting-prefill, batch size/KV,
    // swap-ins, immediate swap-ins, denials
    int pf = INT_MAX;
    long long bcount = 0, bkv = 0;
    int nsw = 0, nimm = 0, nden = 0;
    bool tn_batch = false;  // PDES: a batch member's next token ends its reasoning
    // PB_PARK: the parked tail ranks right before candidate `chk` (after the
    // class-1 candidates keyed below it). It is denied again without side
    // effects if, at that rank, something was admitted (no deadlock
    // breaker), no class-1 resident is left to evict — none ranked after it
    // but not yet evicted (rb < chk: every resident at or past b was evicted
    // by an earlier admission's back walk) and none denied on the stack — and
    // the free KV is below every member's need (with no victims left, free
    // only shrinks past that rank).
    int chk = skip ? c1 + pg.below : -1;
    bool pfail = false;
    // PB_PARK: the last position admitted, resident or class 0, and the last
    // one that evicted: the denied, non-resident class-1 candidates after
    // both are this plan's new parked members
    int last_keep = -1, last_ev = -1;
    const int ln = lane_id();
    for (int base = 0; base < n; base += 32) {
        const int ci_l = base + ln;
        const bool valid = ci_l < n;
        int4 my = make_int4(0, 0, 0, 0);
        if (valid) my = R.cand[ci_l];
        const long long my_need = my.y;
        const int my_rkv = cand_rkv(my);
        const int my_w = my.w;
        const bool my_allow = !oracle && !(fcfs && (my_w & CF_WAIT));
        const int my_s = classed ? ((my_w & CF_LOW) ? c1 : k0) : 0;
        unsigned char st = 0;
        const int cnt = min(32, n - base);
        int k = 0;
        while (k < cnt) {
            S.adm_rounds++;
            const bool mine = valid && ln >= k;
            const bool evd = mine && ci_l >= A.b && my_rkv > 0;
            const bool bld = mine && !evd && fcfs_blocked && my_rkv == 0;
            const bool act = mine && !evd && !bld;
            const long long F = A.free_;
            const bool sf = act && my_need > F;
            const bool vict =
                my_allow && (rb >= max(my_s, ci_l + 1) || (A.ns > 0 && stack_top >= my_s));
            const bool simple_sf = sf && my_rkv == 0 && !fcfs && any_admitted && !vict;
            const bool fc = act && !sf;
            // needs are < 2^26 (host-validated KV limit), so a 32-bit prefix
            // over 32 lanes cannot overflow
            const int contrib = fc ? (int)my_need : 0;
            int pin = contrib;
            if (__ballot_sync(FULL, fc)) {  // all-denied rounds (the tail) skip the scan
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(FULL, pin, o);
                    if (ln >= o) pin += y;
                }
            }
            const bool stop_here = (fc && (long long)pin > F) || (sf && !simple_sf) ||
                                   (PB_PARK && mine && ci_l == chk);
            const unsigned sm = __ballot_sync(FULL, stop_here);
            const int stop = sm ? __ffs(sm) - 1 : cnt;
            const bool fin = mine && ln < stop;
            if (fin) st = fc ? CS_ADMIT : CS_DENY;
            // pin at lane stop-1 = admitted need so far (lanes < k contribute 0)
            const long long taken = __shfl_sync(FULL, pin, max(stop - 1, 0));  // widened
            if (stop > 0) A.free_ -= taken;
            if (__ballot_sync(FULL, fin && fc)) any_admitted = true;
            if (stop >= cnt) break;
#if PB_PARK
            if (base + stop == chk) {  // the parked tail's rank
                const bool novict = any_admitted && rb < chk && !(A.ns > 0 && stack_top >= c1);
                if (!(novict && A.free_ < (long long)R.s.pneed[i])) {
#ifdef PB_PARK_STATS
                    S.adm_slow += !novict ? 1ll : 1ll << 16;
#endif
                    // with no victim left only members whose need fits the
                    // free KV can be admitted; anything else: all come back
                    pthr = novict ? A.free_ : LLONG_MAX;
                    pfail = true;
                    break;
                }
                chk = -1;
                k = stop;
                continue;
            }
            const int ne0 = A.ne;
#endif
            // ---- exact reference step for candidate `stop`
#ifndef PB_PARK_STATS
            S.adm_slow++;
#endif
            const int ci = base + stop;
            const long long need = __shfl_sync(FULL, my_need, stop);
            const int cw = __shfl_sync(FULL, my_w, stop);
            const int rkv = __shfl_sync(FULL, my_rkv, stop);
            const int b0 = A.b;
            if (need > A.free_) {
                bool allow = !oracle && !(fcfs && (cw & CF_WAIT));
                if (allow) {
                    int s = classed ? ((cw & CF_LOW) ? c1 : k0) : 0;
                    walk_back(R, A, max(s, ci + 1), need);
                    pop_stack(R, A, s, need);
                    if (need > A.free_ && !any_admitted) {  // deadlock breaker :211-220
                        walk_back(R, A, ci + 1, need);
                        pop_stack(R, A, 0, need);
                    }
                }
            }
            unsigned char dec;
            if (need <= A.free_) {
                dec = CS_ADMIT;
                any_admitted = true;
                A.free_ -= need;
            } else {
                dec = CS_DENY;
                if (rkv > 0) {
                    if (ln == 0) R.stack[A.ns] = (unsigned)ci;
                    A.ns++;
                }
                if (fcfs) fcfs_blocked = true;
            }
            stack_top = A.ns > 0 ? (int)R.stack[A.ns - 1] : -1;
            if (A.b != b0) rb = find_rb(R, A.b);
            if (ln == stop) st = dec;
#if PB_PARK
            if (A.ne != ne0) last_ev = ci;
#endif
            k = stop + 1;
        }
#if PB_PARK
        if (pfail) break;
        {
            // (residents at or past b were evicted: they sit this plan out)
            const unsigned km = __ballot_sync(
                FULL, valid && (st == CS_ADMIT || ci_l < c1 ||
                                ((my_w & CF_RES) && !(ci_l >= A.b && my_rkv > 0))));
            if (km) last_keep = base + 31 - __clz(km);
        }
#endif
        if (valid) R.cstat[ci_l] = st;
        // statistics for this (now final) chunk
        const bool adm = st == CS_ADMIT, den = st == CS_DENY;
        if (TAIL_FAST && !__ballot_sync(FULL, adm)) {  // all-denied chunk
            if (PB_LOG) nden += __popc(__ballot_sync(FULL, den));
            continue;
        }
        bool wt = false, inb = false, sw = false, imm = false;
        if (adm) {
            if (my_w & CF_WAIT) wt = true;
            else if (my_w & CF_RES) inb = true;
            else if (swap_is_instant(R.prof, my.z)) { imm = true; inb = true; }
            else sw = true;
        }
        const unsigned wm = __ballot_sync(FULL, wt);
        if (wm && pf == INT_MAX) pf = base + __ffs(wm) - 1;
        bcount += __popc(__ballot_sync(FULL, inb));
        if (PB_PDES && __ballot_sync(FULL, inb && (my_w & CF_TNEXT))) tn_batch = true;
        bkv += inb ? (long long)my.z : 0;  // lane-local; reduced after the loop
        if (PB_LOG) {  // log-line positions only
            nsw += __popc(__ballot_sync(FULL, sw));
            nimm += __popc(__ballot_sync(FULL, imm));
            nden += __popc(__ballot_sync(FULL, den));
        }
        __syncwarp();
    }
#if PB_PARK
    if (chk == n) {
        const bool novict = any_admitted && !(A.ns > 0 && stack_top >= c1);
        if (!(novict && A.free_ < (long long)R.s.pneed[i])) {
#ifdef PB_PARK_STATS
            S.adm_slow += !novict ? 1ll : 1ll << 16;
#endif
            pthr = novict ? A.free_ : LLONG_MAX;
            pfail = true;
        }
    }
    if (pfail) {  // re-plan with (some of) the parked tail back in the queue
        do_unpark = true;
        continue;
    }
#ifdef PB_PARK_STATS
    if (skip) S.adm_rounds += pcnt, S.adm_slow += 1ll << 48;
#endif
#endif
    S.visits += n + (skip ? pcnt : 0);
    bkv = warp_sum_ll(bkv);
    if (A.free_ < 0) pop_stack(R, A, 0, 0);  // over-capacity repair :235-243

    int kind;  // 0 idle, 1 prefill, 2 decode
    double dur;
    int pf_idx = -1;
    if (pf != INT_MAX) {
        pf_idx = R.cand[pf].x;
        kind = 1;
        dur = prefill_latency(R.prof, R.spec[pf_idx].x);
    } else if (bcount > 0) {
        kind = 2;
        dur = decode_step_latency(R.prof, bcount, bkv);
    } else {
        kind = 0;
        dur = 0.0;
    }

    // ---- apply (engine.cpp:201-257). Evictions first, in eviction order.
    long long log0 = S.nlog;
    for (int base = 0; base < A.ne; base += 32) {
        int k = base + lane_id();
        bool act = k < A.ne;
        long long kv = 0;
        double sd = 0.0;
        int vi = 0;
        if (act) {
            vi = (int)R.elist[k];
            int4 h = R.rs[vi].h;
            kv = h.x;
            unsigned m = m_set_loc(R.rs[vi].meta, LOC_CPU);
            sd = swap_latency(R.prof, kv, rcp_of(R, kRcpSwap));
            if (sd > 0.0) m = m_set_swout(m, true);
            R.rs[vi].meta = m;
            log_put(R, log0 + k, S.now, kLEvict, i, vi, 0);
        }
        long long tot = warp_sum_ll(kv);
        add_gpu(R, S, i, -tot);
        add_cpu(R, i, tot);
        unsigned pm = __ballot_sync(FULL, act && sd > 0.0);
        while (pm) {
            int j = __ffs(pm) - 1;
            pm &= pm - 1;
            double t = __shfl_sync(FULL, sd, j);
            int v = __shfl_sync(FULL, vi, j);
            heap_push(R, S, __dadd_rn(S.now, t), EV_SWAP, (unsigned)v, i);
        }
    }
    __syncwarp();
    // pass B: swap-ins, immediate swap-ins, denials, batch, in candidate order
    long long lsw = log0 + A.ne, limm = lsw + nsw, lden = limm + nimm;
    const bool logging = PB_LOG && (R.flags & kLogEvents) != 0;
    int bpos = 0;
    long long mv = 0;
    unsigned* bout = R.batch + (long long)i * R.n;
#if PB_PARK
    // the skipped tail sat this plan out: log its blocked-time addition; the
    // denied non-resident class-1 candidates after the last admitted /
    // resident / evicting position join the tail (replaying from here on)
    const int ptail = any_admitted ? max(max(last_keep, last_ev), c1 - 1) + 1 : n;
    int pjoin = 0;
    if (skip || ptail < n) {
        pjoin = skip ? R.s.plen[i] : 0;  // a new tail starts an empty log
        __syncwarp();
        if (skip) {
            if (lane_id() == 0) R.plog[(long long)i * kParkLog + pjoin] = dur;
            ++pjoin;
        }
        if (lane_id() == 0) R.s.plen[i] = pjoin;
    }
    uint2* const qlow = queue_ptr(R, i, 1);
    int pmin_need = INT_MAX, pfirst = INT_MAX, pnew = 0;
#endif
    // pipelined: the blocked totals of the next chunk's denials are loaded
    // while this chunk is applied (a request is a candidate at most once)
    int4 c_n = make_int4(0, 0, 0, 0);
    unsigned char st_n = 0;
    double bl_n = 0.0;
    if (lane_id() < n) {
        c_n = R.cand[lane_id()];
        st_n = R.cstat[lane_id()];
        if (st_n == CS_DENY) bl_n = R.blocked[c_n.x];
    }
    for (int base = 0; base < n; base += 32) {
        int k = base + lane_id();
        const int4 c = c_n;
        const unsigned char st_c = st_n;
        const double bl = bl_n;
        if (k + 32 < n) {
            c_n = R.cand[k + 32];
            st_n = R.cstat[k + 32];
            bl_n = st_n == CS_DENY ? R.blocked[c_n.x] : 0.0;
        }
        bool adm = false, den = false, inb = false, sw = false, imm = false;
        if (k < n) {
            adm = st_c == CS_ADMIT;
            den = st_c == CS_DENY;
        }
#if PB_PARK
        // park: flag the queue entry, note the log index (residents past
        // ptail were evicted: they are swapping out, not frozen)
        if (k >= ptail && k < n && !(c.w & CF_RES)) {
            qlow[(unsigned)c.w >> CF_POS_SHIFT].y |= kPark;
            R.pfrom[c.x] = pjoin;
            pmin_need = min(pmin_need, c.y);
            pfirst = min(pfirst, k);
            ++pnew;
        }
#endif
        if (TAIL_FAST && !logging && !__ballot_sync(FULL, adm)) {  // blocked time only
            if (den) R.blocked[c.x] = __dadd_rn(bl, dur);
            continue;
        }
        double sd = 0.0;
        if (adm && !(c.w & CF_WAIT)) {
            if (c.w & CF_RES) inb = true;
            else if (swap_is_instant(R.prof, c.z)) {
                imm = true;
                inb = true;
            } else {
                sw = true;
                sd = swap_latency(R.prof, c.z, rcp_of(R, kRcpSwap));
            }
        }
        // swap-in / immediate / denial masks only place log lines
        unsigned swm = __ballot_sync(FULL, sw), bm = __ballot_sync(FULL, inb);
        unsigned imm_m = 0, dnm = 0;
        if (logging) {
            imm_m = __ballot_sync(FULL, imm);
            dnm = __ballot_sync(FULL, den);
        }
        unsigned lt = lanemask_lt();
        if (sw) {
            unsigned m = R.rs[c.x].meta;
            R.rs[c.x].meta = m_set_swin(m, true);
            log_put(R, lsw + __popc(swm & lt), S.now, kLSwapIn, i, c.x, 0);
        }
        if (imm) {
            unsigned m = R.rs[c.x].meta;
            R.rs[c.x].meta = m_set_loc(m, LOC_GPU);
            log_put(R, limm + __popc(imm_m & lt), S.now, kLSwapIn, i, c.x, 0);
        }
        if (den) {
            R.blocked[c.x] = __dadd_rn(bl, dur);
            log_put(R, lden + __popc(dnm & lt), S.now, kLBlock, i, c.x, 0);
        }
        if (inb && kind == 2) bout[bpos + __popc(bm & lt)] = (unsigned)c.x;
        mv += (sw || imm) ? (long long)c.z : 0;  // lane-local; reduced after the loop
        lsw += __popc(swm);
        limm += __popc(imm_m);
        lden += __popc(dnm);
        bpos += __popc(bm);
        while (swm) {
            int j = __ffs(swm) - 1;
            swm &= swm - 1;
            double t = __shfl_sync(FULL, sd, j);
            int v = __shfl_sync(FULL, c.x, j);
            heap_push(R, S, __dadd_rn(S.now, t), EV_SWAP, (unsigned)v, i);
        }
    }
    S.nlog = log0 + A.ne + nsw + nimm + nden;
#if PB_PARK
    pnew = warp_sum(pnew);
    if (pnew > 0) {
        pmin_need = (int)warp_min_u((unsigned)pmin_need);
        pfirst = (int)warp_min_u((unsigned)pfirst);
        // the first new member has the lowest new key (priority order)
        const unsigned long long k_new = prio_key(R.rs[R.cand[pfirst].x].h);
        __syncwarp();
        if (lane_id() == 0) {
            R.s.pcount[i] = pcnt + pnew;
            R.s.pneed[i] = min(skip ? R.s.pneed[i] : INT_MAX, pmin_need);
            const unsigned long long k_old = skip ? R.s.pkey[i] : ~0ull;
            R.s.pkey[i] = k_new < k_old ? k_new : k_old;
        }
        __syncwarp();
    }
#endif
    mv = warp_sum_ll(mv);
    add_cpu(R, i, -mv);
    add_gpu(R, S, i, mv);
    __syncwarp();

    if (kind == 1) {
        int4 sp = R.spec[pf_idx];
        add_gpu(R, S, i, (long long)sp.x + (sp.y == 0 ? 1 : 0));
        if (lane_id() == 0) {
            R.s.busy[i] = 1;
            R.s.iter_start[i] = S.now;
            R.s.blen[i] = 0;
        }
        __syncwarp();
#if PB_PDES
        // a prefill of an R = 0 request with more than one answer token ends
        // in a Pascal phase boundary (engine.cpp:295-305)
        if (lane_id() == 0)
            R.s.gtime[i] = (R.policy == kPascal && sp.y == 0 && sp.z > 1) ? __dadd_rn(S.now, dur)
                                                                           : CUDART_INF;
#endif
        heap_push(R, S, __dadd_rn(S.now, dur), EV_PREFILL, (unsigned)pf_idx, i);
        emit(R, S, kLPrefillStart, i, pf_idx);
    } else if (kind == 2) {
        add_gpu(R, S, i, bcount);  // growth reserved up front (engine.cpp:245)
        if (lane_id() == 0) {
            R.s.busy[i] = 1;
            R.s.iter_start[i] = S.now;
            R.s.blen[i] = (int)bcount;
        }
        __syncwarp();
#if PB_PDES
        if (lane_id() == 0)
            R.s.gtime[i] = (R.policy == kPascal && tn_batch) ? __dadd_rn(S.now, dur) : CUDART_INF;
#endif
        heap_push(R, S, __dadd_rn(S.now, dur), EV_ITER, (unsigned)i, i);
        emit(R, S, kLDecodeStart, i, -1, (int)bcount);
    }
    __syncwarp();
    if (R.s.gpu[i] > R.cap && S.status == 0) S.status = kErrCapacity;
    note_peak(R, S);
    break;
    }  // PB_PARK re-plan loop
}

// --------------------------------------------------------------- events
// engine.cpp:260-283
DEVI int on_arrival(Rep& R, Scal& S, int idx) {
    if (lane_id() == 0) R.rec[idx].arrival = S.now;
    const bool pascal = R.policy == kPascal;
    int dst = select_instance(R, S, pascal ? SEL_M_HEALTHY : SEL_M);
    emit(R, S, kLArrival, dst, idx);
    int4 sp = R.spec[idx];
    bool high;
    if (sp.w) {  // kv_preloaded: prompt KV starts on the CPU
        unsigned m = 0;
        m = m_set_loc(m, LOC_CPU);
        m = m_set_phase(m, sp.y > 0 ? PH_REASON : PH_ANSWER);
        if (PB_PDES) m = m_set_rem(m, sp.y);
        if (lane_id() == 0) {
            int4 h = R.rs[idx].h;
            h.x = sp.x;
            R.rs[idx].h = h;
            R.rs[idx].meta = m;
            R.rec[idx].prefill_complete = S.now;
            if (sp.y == 0) R.rec[idx].reasoning_end = S.now;
        }
        add_cpu(R, dst, sp.x);
        high = sp.y > 0 ? true : !pascal;
    } else {
        // waiting prefill; PDES: the phase boundary is >= max(1, R) iterations away
        if (lane_id() == 0)
            R.rs[idx].meta = PB_PDES ? m_set_rem(m_set_phase(0u, PH_WAIT), sp.y > 0 ? sp.y : 1)
                                     : m_set_phase(0u, PH_WAIT);
        high = true;
    }
    __syncwarp();
    enqueue(R, S, dst, idx, high);
    return dst;  // every handler ends with maybe_start on this instance
}

// engine.cpp:285-308
DEVI int on_prefill_complete(Rep& R, Scal& S, int idx) {
    unsigned m = R.rs[idx].meta;
    int i = m_owner(m);
    int4 sp = R.spec[idx];
    if (lane_id() == 0) R.s.busy[i] = 0;
    int kv = sp.x + (sp.y == 0 ? 1 : 0);
    double iter_start = R.s.iter_start[i];
    __syncwarp();
    if (lane_id() == 0) {
        int4 h = R.rs[idx].h;
        h.x = kv;
        if (sp.y == 0) h.y = 1;
        R.rs[idx].h = h;
        R.rec[idx].prefill_complete = S.now;
    }
    __syncwarp();
    emit(R, S, kLPrefillComplete, i, idx);
    S.req_iters++;
    if (sp.y == 0) {
        if (lane_id() == 0) {
            R.rec[idx].reasoning_end = S.now;
            deliver_lane(R, S.now, idx, iter_start);
        }
        S.ans_tokens++;
        __syncwarp();
        if (1 == sp.z) {
            // phase = Answering; finish_request (engine.cpp:135-146)
            int4 h = R.rs[idx].h;
            if (lane_id() == 0) {
                dequeue_lane(R, idx, i, m, h.w);
                R.rs[idx].meta = m_set_phase(m, PH_DONE);
                R.rec[idx].completion = S.now;
            }
            // free_memory: waiting-prefill requests default to Gpu
            add_gpu(R, S, i, -(long long)kv);
            S.done++;
            __syncwarp();
            emit(R, S, kLFinish, i, idx);
        } else {
            if (lane_id() == 0) R.rs[idx].meta = m_set_phase(m, PH_ANSWER);
            __syncwarp();
            emit(R, S, kLTransition, i, idx);
            if (R.policy == kPascal) pascal_transition(R, S, idx);
        }
    } else {
        if (lane_id() == 0) {
            unsigned mm = m_set_phase(m, PH_REASON);
            if (PB_PDES) mm = m_set_rem(mm, sp.y);
            R.rs[idx].meta = mm;
        }
        __syncwarp();
    }
    return i;  // every handler ends with maybe_start on this instance
}

// engine.cpp:310-337: retire one decode iteration, batch members in plan order.
DEVI int on_iteration_complete(Rep& R, Scal& S, int i) {
    if (lane_id() == 0) R.s.busy[i] = 0;
    int nb = R.s.blen[i];
    double iter_start = R.s.iter_start[i];
    __syncwarp();
    if (lane_id() == 0) R.s.blen[i] = 0;
    const bool use_quanta = R.policy == kRr || R.policy == kPascal;
    const bool pascal = R.policy == kPascal;
    const bool logging = PB_LOG && (R.flags & kLogEvents) != 0;
    const unsigned* bin = R.batch + (long long)i * R.n;
    S.req_iters += nb;
    // two-deep pipeline as in gather_queue: a request is in a batch once, and
    // a member's phase boundary only touches its own state
    const int ln = lane_id();
    int idx_c = 0, idx_n = 0;
    int4 h_c = make_int4(0, 0, 0, 0), sp_c = make_int4(0, 0, 0, 0);
    unsigned m_c = 0;
    int qu_c = 0;
    if (ln < nb) {
        idx_c = (int)bin[ln];
        h_c = R.rs[idx_c].h;
        m_c = R.rs[idx_c].meta;
        sp_c = R.spec[idx_c];
        qu_c = use_quanta ? R.rs[idx_c].qused : 0;
    }
    if (32 + ln < nb) idx_n = (int)bin[32 + ln];
    for (int base = 0; base < nb; base += 32) {
        int k = base + ln;
        bool act = k < nb;
        int idx = idx_c;
        int4 h = h_c, sp = sp_c;
        unsigned m = m_c;
        int qu = qu_c;
        if (k + 32 < nb) {
            idx_c = idx_n;
            h_c = R.rs[idx_n].h;
            m_c = R.rs[idx_n].meta;
            sp_c = R.spec[idx_n];
            qu_c = use_quanta ? R.rs[idx_n].qused : 0;
        }
        if (k + 64 < nb) idx_n = (int)bin[k + 64];
        bool fresh_lost = false;
        if (act) {
            h.y += 1;
            h.x += 1;
            if (use_quanta) {
                qu = qu + 1;
                if ((long long)qu >= R.quantum) {
                    qu = 0;
                    h.w += 1;
                    // a_i counts low-queue members with no exhausted quantum
                    fresh_lost = m_qlow(m) && h.z != 0 && h.w == 1;
                }
            }
        }
        const unsigned ph = m_phase(m);
        const bool trans = act && ph == PH_REASON && h.y == sp.y;
        const bool ans = act && ph == PH_ANSWER;
        const bool fin = ans && h.y == sp.y + sp.z;
        S.ans_tokens += __popc(__ballot_sync(FULL, ans));
        unsigned remaining = __ballot_sync(FULL, act);
        unsigned tmask = pascal ? __ballot_sync(FULL, trans) : 0u;
        while (remaining) {
            int t = tmask ? __ffs(tmask) - 1 : 32;
            unsigned seg = remaining & (t == 32 ? FULL : ((1u << t) - 1u));
            bool in = (seg >> lane_id()) & 1u;
            // ---- parallel segment: token, quanta, delivery, finish
            int ltot, lpos = 0;
            if (logging) {
                int lines = in ? 1 + (fin ? 1 : 0) + ((!pascal && trans) ? 1 : 0) : 0;
                lpos = warp_excl_scan(lines, &ltot);
            } else if (PB_LOG) {  // keep the line count exact (sizes a later logged run)
                ltot = __popc(seg) + __popc(__ballot_sync(FULL, in && (fin || (!pascal && trans))));
            } else {
                ltot = 0;  // no log, nothing to size
            }
            long long freed = 0;
            if (in) {
                unsigned mm = m;
                log_put(R, S.nlog + lpos, S.now, kLToken, i, idx, 0);
                if (trans) {  // baselines: phase flips, placement kept (engine.cpp:164)
                    mm = m_set_phase(mm, PH_ANSWER);
                    R.rec[idx].reasoning_end = S.now;
                    log_put(R, S.nlog + lpos + 1, S.now, kLTransition, i, idx, 0);
                }
                if (ans) deliver_lane(R, S.now, idx, iter_start);
                int4 hw = h;
                if (fin) {
                    // finish_request: free GPU KV, dequeue, record completion
                    freed = h.x;
                    hw.z = 0;
                    if (m_qlow(m)) {
                        atomicSub(&R.s.lcount[i], 1);
                        if (h.w == 0) atomicSub(&R.s.afresh[i], 1);
                    } else {
                        atomicSub(&R.s.hcount[i], 1);
                    }
                    mm = m_set_phase(mm, PH_DONE);
                    R.rec[idx].completion = S.now;
                    log_put(R, S.nlog + lpos + 1, S.now, kLFinish, i, idx, 0);
                }
                if (fresh_lost) atomicSub(&R.s.afresh[i], 1);
                if (PB_PDES && m_phase(mm) == PH_REASON) mm = m_set_rem(mm, (long long)sp.y - h.y);
                R.rs[idx].h = hw;
                if (use_quanta) R.rs[idx].qused = qu;
                if (mm != m) R.rs[idx].meta = mm;
            }
            S.nlog += ltot;
            const unsigned fm = __ballot_sync(FULL, in && fin);
            if (fm) {
                add_gpu(R, S, i, -warp_sum_ll(freed));
                S.done += __popc(fm);
            }
            __syncwarp();
            if (t == 32) break;
            // ---- Pascal phase boundary for lane t, applied in batch order
            int tidx = __shfl_sync(FULL, idx, t);
            if (lane_id() == t) {
                R.rs[idx].h = h;
                if (use_quanta) R.rs[idx].qused = qu;
                if (fresh_lost) atomicSub(&R.s.afresh[i], 1);
                R.rs[idx].meta = m_set_phase(m, PH_ANSWER);
                R.rec[idx].reasoning_end = S.now;
            }
            __syncwarp();
            emit(R, S, kLToken, i, tidx);
            emit(R, S, kLTransition, i, tidx);
            pascal_transition(R, S, tidx);
            remaining &= ~((2u << t) - 1u);
            tmask &= ~(1u << t);
        }
    }
    __syncwarp();
    return i;  // every handler ends with maybe_start on this instance
}

// engine.cpp:339-349
DEVI int on_swap_complete(Rep& R, Scal& S, int idx) {
    unsigned m = R.rs[idx].meta;
    int i = m_owner(m);
    __syncwarp();  // every lane has read meta before lane 0 rewrites it
    if (lane_id() == 0) {
        unsigned mm = m;
        if (m_swout(m)) mm = m_set_swout(mm, false);
        else if (m_swin(m)) mm = m_set_loc(m_set_swin(mm, false), LOC_GPU);
        R.rs[idx].meta = mm;
    }
    __syncwarp();
    emit(R, S, kLSwapComplete, i, idx);
    return i;  // every handler ends with maybe_start on this instance
}

// engine.cpp:351-367
DEVI int on_transfer_complete(Rep& R, Scal& S, int idx) {
    unsigned m = R.rs[idx].meta;
    int dst = m_owner(m);
    long long kv = R.rs[idx].h.x;
    bool fits = R.cap - R.s.gpu[dst] >= kv;
    __syncwarp();  // every lane has read gpu_used / meta before lane 0 updates them
    if (fits) add_gpu(R, S, dst, kv);
    else add_cpu(R, dst, kv);
    if (lane_id() == 0) {
        R.rs[idx].meta = m_set_loc(m, fits ? LOC_GPU : LOC_CPU);
        R.rs[idx].qused = 0;
        int4 h = R.rs[idx].h;
        h.w = 0;
        R.rs[idx].h = h;
    }
    __syncwarp();
    enqueue(R, S, dst, idx, false);
    emit(R, S, kLTransferComplete, dst, idx);
    note_peak(R, S);
    return dst;  // every handler ends with maybe_start on this instance
}

#if !PB_PDES
// ------------------------------------------------------------ the replica
template <bool TAIL_FAST>
DEVI void run_replica(const Arena& a, int r, char* smem, int max_ni, int n_smem, int c_smem,
                      int h_slots, int b_smem) {
    const ReplicaDesc d = a.desc[r];
    Rep R;
    R.n = d.n;
    R.ni = d.ni;
#ifdef PB_ONLY_POLICY
    R.policy = PB_ONLY_POLICY;  // single-policy build: every policy test folds
#else
    R.policy = d.policy;
#endif
    R.flags = d.flags;
    R.cap = d.capacity;
    R.quantum = d.quantum;
    R.demotion = d.demotion;
    R.slack = d.slack;
    R.tpot = d.tpot;
    R.prof = d.prof;
    R.logcap = d.log_cap;
    const long long g = d.req_base;
    const long long abase = R.n > 0 ? a.aoff[g] : 0;
    R.arrival = a.arrival + g;
    R.rec = a.rec + g;
    R.ph = a.ph + g;
    R.bpv = a.bpv + abase;
    R.bpk = a.bpk + abase;
    R.dig = a.dig + abase;
    R.del = a.del + abase;
    R.qent = a.qent + d.queue_base;
    R.qcap = d.qcap;
    R.batch = a.batch + d.batch_base;
    R.heap = a.heap + d.heap_base;
    R.g_cand = a.cand + g;
    R.g_tmp = a.tmp + g;
    R.g_tmpq = a.tmpq + g;
    R.g_cstat = a.cstat + g;
    R.elist = a.elist + g;
    R.stack = a.stack + g;
    R.log = a.log + d.log_base;
    const int ni = d.ni;
    // ---- shared-memory carve-up (engine.h smem_per_warp)
    char* sp = smem;
    R.s.gpu = reinterpret_cast<long long*>(sp + 32);  // rcp_of slots ahead
    R.s.cpu = R.s.gpu + ni;
    R.s.iter_start = reinterpret_cast<double*>(R.s.cpu + ni);
    R.s.link = R.s.iter_start + ni;
#if PB_PARK
    R.s.pkey = reinterpret_cast<unsigned long long*>(R.s.link + ni);
    R.s.hi_len = reinterpret_cast<int*>(R.s.pkey + ni);
#else
    R.s.hi_len = reinterpret_cast<int*>(R.s.link + ni);
#endif
    R.s.lo_len = R.s.hi_len + ni;
    R.s.hcount = R.s.lo_len + ni;
    R.s.lcount = R.s.hcount + ni;
    R.s.afresh = R.s.lcount + ni;
    R.s.blen = R.s.afresh + ni;
    R.s.busy = R.s.blen + ni;
    R.s.healthy = R.s.busy + ni;
#if PB_PARK
    R.s.pcount = R.s.healthy + ni;
    R.s.pneed = R.s.pcount + ni;
    R.s.plen = R.s.pneed + ni;
    R.plog = a.plog + d.plog_base;
    R.pfrom = a.pfrom + g;
#endif
    sp += smem_inst_bytes(max_ni);
    const bool resident = R.n <= n_smem;  // request state in shared memory
    if (resident) {
        R.rs = reinterpret_cast<ReqState*>(sp);
        R.spec = reinterpret_cast<int4*>(R.rs + n_smem);
        R.blocked = reinterpret_cast<double*>(R.spec + n_smem);
        R.aoff = reinterpret_cast<int*>(R.blocked + n_smem);
    } else {
        R.rs = a.rs + g;
        R.spec = const_cast<int4*>(a.spec) + g;
        R.blocked = a.blocked + g;
        R.aoff = const_cast<int*>(a.aoff32) + g;
    }
    sp += smem_req_bytes(n_smem);
    HeapEnt* sheap = reinterpret_cast<HeapEnt*>(sp);
    const long long sheap_slots = resident ? (long long)n_smem + max_ni + 2 : h_slots;
    if (resident) R.heap = sheap;  // fits every pending event
    sp += smem_heap_bytes(n_smem, max_ni, h_slots);
    R.c_smem = c_smem;
    R.s_cand = reinterpret_cast<int4*>(sp);
    R.s_tmp = R.s_cand + c_smem;
    R.s_tmpq = reinterpret_cast<unsigned*>(R.s_tmp + c_smem);
    R.s_cstat = reinterpret_cast<unsigned char*>(R.s_tmpq + c_smem);
    sp += smem_cand_bytes(c_smem);
    const bool blocked_smem = !resident && R.n <= b_smem;
    if (blocked_smem) R.blocked = reinterpret_cast<double*>(sp);
    set_rcps(R);
    for (int i = lane_id(); i < ni; i += 32) {
        R.s.gpu[i] = 0;
        R.s.cpu[i] = 0;
        R.s.iter_start[i] = 0.0;
        R.s.link[i] = 0.0;
        R.s.hi_len[i] = R.s.lo_len[i] = R.s.hcount[i] = R.s.lcount[i] = 0;
        R.s.afresh[i] = R.s.blen[i] = R.s.busy[i] = 0;
        R.s.healthy[i] = 1;
#if PB_PARK
        R.s.pcount[i] = 0;
        R.s.pneed[i] = INT_MAX;
        R.s.plen[i] = 0;
        R.s.pkey[i] = ~0ull;
#endif
    }
    // reset per-request state (Simulator::run, engine.cpp:382-389)
    for (int k = lane_id(); k < R.n; k += 32) {
        ReqState z0;
        z0.h = make_int4(0, 0, 0, 0);
        z0.meta = m_set_phase(0u, PH_WAIT);
        z0.qused = 0;
        z0.ndel = 0;
        z0.cursor = 0;
        R.rs[k] = z0;
        R.blocked[k] = 0.0;
        if (resident) {
            R.spec[k] = a.spec[g + k];
            R.aoff[k] = a.aoff32[g + k];
        }
        PacerHot zp;
        zp.dlast = zp.dcur = zp.t0 = 0.0;
        zp.nbp = zp.jn = 0;
        R.ph[k] = zp;
        RecOut z;
        z.arrival = z.prefill_complete = z.reasoning_end = z.first_answer_delivery = 0.0;
        z.first_answer_iter_start = z.blocked = z.completion = z.mig_start = z.mig_end = 0.0;
        z.nmig = 0;
        z.pad = 0;
        R.rec[k] = z;
    }
    __syncwarp();

    Scal S;
    S.heap = sheap;
    S.heap_slots = sheap_slots;
    S.now = 0.0;
    S.evseq = (unsigned long long)R.n;  // arrivals hold seqs 1..n (engine.cpp:384-389)
    S.enq = 0;
    S.next_arr = 0;
    S.hn = 0;
    S.done = 0;
    S.status = 0;
    S.gpu_total = 0;
    S.peak = 0;
    S.nlog = 0;
    S.events = S.plans = S.visits = S.req_iters = S.ans_tokens = S.health = 0;
    S.adm_rounds = S.adm_slow = 0;
    const long long heap_cap = (long long)R.n + R.ni + 1;

    // the next arrival time is loaded one event ahead
    double ta_next = R.n > 0 ? R.arrival[0] : 0.0;
    while (S.status == 0) {
        const bool has_arr = S.next_arr < R.n;
        const bool has_ev = S.hn > 0;
        if (!has_arr && !has_ev) break;
        const double ta = ta_next;
        HeapEnt top;
        top.t = 0.0;
        top.key = 0;
        if (has_ev) top = S.heap[1];
        // arrivals carry seqs 1..n, below every dynamic event seq
        bool take_arr = has_arr && (!has_ev || !(top.t < ta));
        double et;
        unsigned kind, id;
        if (take_arr) {
            et = ta;
            kind = 0;
            id = (unsigned)S.next_arr++;
            if (S.next_arr < R.n) ta_next = R.arrival[S.next_arr];
        } else {
            heap_pop(R, S);  // top: the root every lane read above
            et = top.t;
            kind = (unsigned)(top.key >> 26) & 7u;
            id = (unsigned)(top.key & ((1u << 26) - 1u));
        }
        S.events++;
        if (et < S.now - 1e-12) {
            S.status = kErrClock;
            break;
        }
        S.now = dmax(S.now, et);
        int plan_inst;
        switch (kind) {
            case 0: plan_inst = on_arrival(R, S, (int)id); break;
            case EV_PREFILL: plan_inst = on_prefill_complete(R, S, (int)id); break;
            case EV_ITER:
                // the plan that follows gathers this instance's queues: pull
                // their heads into L1 while the batch retires
                prefetch_queue_heads(R, (int)id);
                plan_inst = on_iteration_complete(R, S, (int)id);
                break;
            case EV_SWAP: plan_inst = on_swap_complete(R, S, (int)id); break;
            default: plan_inst = on_transfer_complete(R, S, (int)id); break;
        }
        // one inlined copy of the planner for all five handlers
        maybe_start<TAIL_FAST>(R, S, plan_inst);
        if (S.hn + 1 > heap_cap && S.status == 0) S.status = kErrHeap;
    }
    if (S.status == 0 && S.done != R.n) S.status = kErrStall;
    // outputs the metric kernels read: delivered counts and blocked totals
    for (int k = lane_id(); k < R.n; k += 32) {
        R.rec[k].blocked = R.blocked[k];
        if (resident) a.rs[g + k] = R.rs[k];
    }
    if (lane_id() == 0) {
        ReplicaOut o;
        o.status = S.status;
        o.pad = 0;
        o.peak = S.peak;
        o.nlog = PB_LOG ? S.nlog : 0;  // log-free builds never size a log
        o.events = S.events;
        o.plans = S.plans;
        o.visits = S.visits;
        o.req_iters = S.req_iters;
        o.answer_tokens = S.ans_tokens;
        o.health_checks = S.health;
        o.adm_rounds = S.adm_rounds;
        o.adm_slow = S.adm_slow;
        o.now = S.now;
        a.out[r] = o;
    }
    __syncwarp();
}

// MINB = 1: up to 8 warps per SM, registers unconstrained (the default
// shapes; TAIL_FAST for the 1-2 warps/SM latency shapes); MINB = 3 / 4: 12 /
// 16 warps per SM with <= 168 / 128 registers (opt-in, PB_MAX_WARPS_PER_SM).
template <int MINB, bool TAIL_FAST>
__global__ void __launch_bounds__(128, MINB) sched_kernel(Arena a, int max_ni, int n_smem, int c_smem,
                                                          int h_slots, int b_smem) {
    extern __shared__ __align__(16) char smem_raw[];
    const int warp = threadIdx.x >> 5;
    char* smem = smem_raw + (size_t)warp * smem_per_warp(max_ni, n_smem, c_smem, h_slots, b_smem);
    while (true) {
        int r = 0;
        if (lane_id() == 0) {  // a.order lists this launch's replicas (maybe a subset)
            const int w = atomicAdd(a.work, 1);
            r = w < a.n_rep ? a.order[w] : -1;
        }
        r = __shfl_sync(FULL, r, 0);
        if (r < 0) break;
        run_replica<TAIL_FAST>(a, r, smem, max_ni, n_smem, c_smem, h_slots, b_smem);
    }
}

int launch_engine(const Arena& a, int max_ni, int n_smem, int c_smem, int h_slots, int b_smem,
                  int warps_per_block, int blocks, void* stream) {
    if (warps_per_block < 1 || warps_per_block > 4 || h_slots < 2) return 1;
    const size_t smem =
        (size_t)warps_per_block * smem_per_warp(max_ni, n_smem, c_smem, h_slots, b_smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // register budget by warps per SM: <= 8 -> unconstrained (~240 regs),
    // <= 12 -> <= 168 regs, more -> <= 128 regs
    const long long wpsm = ((long long)blocks * warps_per_block + sms - 1) / sms;
    auto kern = wpsm <= 2    ? sched_kernel<1, true>
                : wpsm <= 8  ? sched_kernel<1, false>
                : wpsm <= 12 ? sched_kernel<3, false>
                             : sched_kernel<4, false>;
    if (smem > 48 * 1024) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return 2;
    }
    if (const char* cv = getenv("PB_CARVEOUT"))  // experiment hook: shared-memory carveout %
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
    kern<<<blocks, warps_per_block * 32, smem, (cudaStream_t)stream>>>(a, max_ni, n_smem, c_smem,
                                                                       h_slots, b_smem);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

#if PB_LOG
// ---------------------------------------------------- unit-parity seams
// One maybe_start (demotion + plan_iteration + plan application,
// engine.cpp:192-258 / instance.cpp:39-57,103-282) on a hand-built instance
// state, through the same inlined planner the event loop runs. One warp.
__global__ void __launch_bounds__(32, 1) plan_probe_kernel(PlanProbe p) {
    extern __shared__ __align__(16) char smem_raw[];
    Rep R;
    R.n = p.n;
    R.ni = p.ni;
    R.policy = p.policy;
    R.flags = kLogEvents;
    R.cap = p.cap;
    R.quantum = p.quantum;
    R.demotion = p.demotion;
    R.slack = 0;
    R.tpot = 0.1;
    R.prof = p.prof;
    R.logcap = p.log_cap;
    R.arrival = p.arrival;
    R.spec = p.spec;
    R.aoff = p.aoff;
    R.rs = p.rs;
    R.blocked = p.blocked;
    R.rec = p.rec;
    R.ph = p.ph;
    R.bpv = nullptr;
    R.bpk = nullptr;
    R.dig = nullptr;
    R.del = nullptr;
    R.qent = p.qent;
    R.qcap = p.qcap;
    R.batch = p.batch;
    R.heap = p.heap;
    R.g_cand = p.cand;
    R.g_tmp = p.tmp;
    R.g_tmpq = p.tmpq;
    R.g_cstat = p.cstat;
    R.elist = p.elist;
    R.stack = p.stack;
    R.log = p.log;
    const int ni = p.ni;
    char* sp = smem_raw;
    R.s.gpu = reinterpret_cast<long long*>(sp + 32);  // rcp_of slots ahead
    R.s.cpu = R.s.gpu + ni;
    R.s.iter_start = reinterpret_cast<double*>(R.s.cpu + ni);
    R.s.link = R.s.iter_start + ni;
    R.s.hi_len = reinterpret_cast<int*>(R.s.link + ni);
    R.s.lo_len = R.s.hi_len + ni;
    R.s.hcount = R.s.lo_len + ni;
    R.s.lcount = R.s.hcount + ni;
    R.s.afresh = R.s.lcount + ni;
    R.s.blen = R.s.afresh + ni;
    R.s.busy = R.s.blen + ni;
    R.s.healthy = R.s.busy + ni;
    sp += smem_inst_bytes(ni);
    R.c_smem = p.c_smem;
    R.s_cand = reinterpret_cast<int4*>(sp);
    R.s_tmp = R.s_cand + p.c_smem;
    R.s_tmpq = reinterpret_cast<unsigned*>(R.s_tmp + p.c_smem);
    R.s_cstat = reinterpret_cast<unsigned char*>(R.s_tmpq + p.c_smem);
    set_rcps(R);
    for (int i = lane_id(); i < ni; i += 32) {
        R.s.gpu[i] = p.used[2 * i];
        R.s.cpu[i] = p.used[2 * i + 1];
        R.s.iter_start[i] = 0.0;
        R.s.link[i] = 0.0;
        R.s.hi_len[i] = p.qlen[2 * i];
        R.s.lo_len[i] = p.qlen[2 * i + 1];
        // monitor counters r_i, |low|, a_i of the live entries
        int hc = 0, lc = 0, af = 0;
        for (int k = 0; k < p.qlen[2 * i]; ++k) hc += 1;
        const uint2* lq = p.qent + (long long)(2 * i + 1) * p.qcap;
        for (int k = 0; k < p.qlen[2 * i + 1]; ++k) {
            lc += 1;
            af += p.rs[lq[k].x].h.w == 0;
        }
        R.s.hcount[i] = hc;
        R.s.lcount[i] = lc;
        R.s.afresh[i] = af;
        R.s.blen[i] = 0;
        R.s.busy[i] = 0;
        R.s.healthy[i] = 1;
    }
    __syncwarp();
    Scal S;
    S.heap = p.heap;
    S.heap_slots = p.heap_cap;
    S.now = p.now;
    S.evseq = 0;
    S.enq = p.enq;
    S.next_arr = p.n;
    S.hn = 0;
    S.done = 0;
    S.status = 0;
    long long tot = 0;
    for (int i = 0; i < ni; ++i) tot += p.used[2 * i];
    S.gpu_total = tot;
    S.peak = tot;
    S.nlog = 0;
    S.events = S.plans = S.visits = S.req_iters = S.ans_tokens = S.health = 0;
    S.adm_rounds = S.adm_slow = 0;
    maybe_start<false>(R, S, p.inst);
    __syncwarp();
    if (lane_id() == 0) {
        for (int i = 0; i < ni; ++i) {
            p.out_used[2 * i] = R.s.gpu[i];
            p.out_used[2 * i + 1] = R.s.cpu[i];
        }
        p.out_scal[0] = S.status;
        p.out_scal[1] = S.hn;
        p.out_scal[2] = (int)S.nlog;
        p.out_scal[3] = R.s.blen[p.inst];
        p.out_scal[4] = R.s.busy[p.inst];
    }
}

int launch_plan_probe(const PlanProbe& p, void* stream) {
    const size_t smem = (size_t)smem_inst_bytes(p.ni) + smem_cand_bytes(p.c_smem);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(plan_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return 2;
    plan_probe_kernel<<<1, 32, smem, (cudaStream_t)stream>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Alg. 1 / Alg. 2 placement (cluster.cpp:10-44,59-62) for a batch of
// snapshot vectors through the engine's select_instance: one warp per
// vector; instance i's m_i / r_i / a_i go to the counters select_instance
// reads, and t_i = 0 is realised as one behind-schedule answering request in
// the instance's low queue (the health scan's own input), t_i = 1 as an empty
// low queue.
constexpr int kSelProbeMaxN = 32;
constexpr int kSelProbeWarps = 4;
__global__ void __launch_bounds__(kSelProbeWarps * 32) select_probe_kernel(SelectProbe p) {
    struct W {
        long long gpu[kSelProbeMaxN], cpu[kSelProbeMaxN];
        int hcount[kSelProbeMaxN], afresh[kSelProbeMaxN], lo_len[kSelProbeMaxN];
        uint2 qent[2 * kSelProbeMaxN];
        unsigned rejected[kSelProbeMaxN / 32 + 1];
    };
    __shared__ W ws[kSelProbeWarps];
    W& w = ws[threadIdx.x >> 5];
    const int n = p.n;
    const long long nw = (long long)gridDim.x * kSelProbeWarps;
    for (long long v = (long long)blockIdx.x * kSelProbeWarps + (threadIdx.x >> 5); v < p.count;
         v += nw) {
        __syncwarp();
        for (int i = lane_id(); i < n; i += 32) {
            const long long o = v * n + i;
            const bool ok = p.t[o] != 0;
            w.gpu[i] = p.mode == 1 ? 0 : p.k1[o];
            w.cpu[i] = 0;
            w.hcount[i] = p.mode == 1 ? (int)p.k1[o] : 0;
            w.afresh[i] = p.mode == 1 ? (int)p.k2[o] : 0;
            w.lo_len[i] = ok ? 0 : 1;
            w.qent[2 * i] = make_uint2(0, 0);
            w.qent[2 * i + 1] = make_uint2(0u, 1u);  // request 0, its live seq
        }
        __syncwarp();
        HealthView V;
        V.qent = w.qent;
        V.qcap = 1;
        V.lo_len = w.lo_len;
        V.rs = p.rs;
        V.spec = p.spec;
        V.ph = p.ph;
        V.bpk = p.bpk;
        V.bpv = p.bpv;
        V.aoff = p.aoff;
        V.tpot = 1.0;
        V.tpot_rcp = 1.0;
        V.slack = 0;
        V.ni = n;
        const int mode = p.mode == 0 ? SEL_M_HEALTHY : p.mode == 1 ? SEL_ANSWER : SEL_M;
        const SelOut o = select_instance(V, 100.0, mode, w.gpu, w.cpu, w.hcount, w.afresh,
                                         w.rejected);
        if (lane_id() == 0) p.out[v] = o.id;
    }
}

int launch_select_probe(const SelectProbe& p, void* stream) {
    if (p.n < 1 || p.n > kSelProbeMaxN) return 1;
    const long long want = (p.count + kSelProbeWarps - 1) / kSelProbeWarps;
    const int blocks = (int)(want < 4096 ? (want > 0 ? want : 1) : 4096);
    select_probe_kernel<<<blocks, kSelProbeWarps * 32, 0, (cudaStream_t)stream>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
#endif  // PB_LOG

#endif  // !PB_PDES

#if PB_PDES
#include "engine_pdes.cuh"
#endif

}  // namespace PB_VARIANT
}  // namespace pb
