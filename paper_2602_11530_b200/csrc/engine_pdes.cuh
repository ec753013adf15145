// engine_pdes.cuh — the instance-parallel engine (included by engine.cu when
// PB_PDES = 1; shares every handler and the planner with the serial engine).
//
// One CTA simulates one replica; instance i is owned by warp i % W. The
// reference's event chain (proj/src/engine.cpp:392-404) is global in
// (time, seq) order, but most events touch one instance only: an iteration /
// prefill / swap / transfer completion and the plan that follows it
// (engine.cpp:192-258,285-367, instance.cpp:103-282) read and write that
// instance's queues, batch and counters and the requests it owns. The events
// that read other instances are
//   * arrivals (Alg. 1 over every instance's snapshot, engine.cpp:260-283), and
//   * Pascal phase boundaries (Alg. 2 + migration, engine.cpp:159-190): an
//     iteration whose batch holds a request at its last reasoning token, or
//     the prefill of an R = 0 request (flagged when the plan is made:
//     meta bit 7 / Inst::gtime).
// The engine advances in rounds. Round horizon
//   H = min(next arrival, earliest pending cross-instance event,
//           earliest pending event + lookahead)
// where lookahead (ReplicaDesc::lookahead, host-computed) bounds from below
// the duration of any iteration / prefill, so no event processed in the round
// can create a cross-instance event before H. Phase A: every warp processes
// its instances' events with time < H, concurrently (they commute: disjoint
// state). Phase B: warp 0 processes the event at H — the arrival (arrival
// seqs 1..n precede every dynamic event at equal times), or the instance's
// events at H up to its cross-instance one while every other instance is
// paused exactly at H. An exact time tie between a cross-instance event and
// another instance's pending event would need the global push order to
// break, so the replica is declined (kErrPdes) and the host re-runs it with
// the serial engine; likewise for a bounded-buffer overflow.
//
// The oracle pre-run's peak of sum_i gpu_used (engine.cpp:75-79, sampled at
// event ends in global order) is merged per round from per-warp records
// {time, delta, sampled, instance} (peak_record).

struct PdesCtl {
    double wmin[kPdesMaxWarps];  // per warp: earliest pending event time
    double wg[kPdesMaxWarps];    // per warp: earliest pending cross-instance event time
    double web[kPdesMaxWarps];   // per warp: earliest possible new cross-instance event
    int wstat[kPdesMaxWarps];
    int wrec[kPdesMaxWarps];
    int next_arr;
    int pad0;
    long long total;  // oracle: sum_i gpu_used at the start of the round
    long long peak;
    long long cnt[10];  // events plans visits req_iters ans_tokens health adm_rounds adm_slow done
                        // phase-B events
    int status;
    int reason;  // why the replica was declined (kPdes* below), for diagnostics
};
enum : int {
    kPdesTieB = 1,       // cross-instance event tied with another instance's event
    kPdesTiePeak = 2,    // oracle peak records of two instances at the same time
    kPdesRecs = 3,       // peak-record buffer overflow
    kPdesNoProgress = 4, // horizon does not advance (lookahead below the clock's ulp)
    kPdesOrder = 5,      // a phase boundary outside phase B (flagging bug guard)
};
static_assert(sizeof(PdesCtl) <= 512, "pdes_ctl_bytes");

// Merge this round's peak records (all threads of the CTA; called between
// barriers): the total after record k is the round-start total plus the
// deltas of every record before it in (time, instance order); a sampled
// record is a candidate peak. Records of different instances at the same
// time cannot be ordered without the global seq: declined.
DEVI const PeakRec& prec_at(const char* base, int stride, int w, int j) {
    return reinterpret_cast<const PeakRec*>(base + (size_t)w * stride)[j];
}
DEVI void pdes_merge_peak(PdesCtl* ctl, const char* prec_all, int stride, int W) {
    int off[kPdesMaxWarps + 1];
    off[0] = 0;
    for (int w = 0; w < W; ++w) off[w + 1] = off[w] + ctl->wrec[w];
    const int M = off[W];
    if (M == 0) return;
    long long best = LLONG_MIN;
    for (int k = threadIdx.x; k < M; k += blockDim.x) {
        int wk = 0;
        while (off[wk + 1] <= k) ++wk;
        const int jk = k - off[wk];
        const PeakRec rk = prec_at(prec_all, stride, wk, jk);
        if (!rk.sampled) continue;
        long long v = ctl->total;
        bool tie = false;
        for (int w = 0; w < W; ++w) {
            for (int j = 0; j < ctl->wrec[w]; ++j) {
                const PeakRec rs = prec_at(prec_all, stride, w, j);
                bool before;
                if (rs.t < rk.t) before = true;
                else if (rs.t > rk.t) before = false;
                else if (rs.inst != rk.inst) {
                    tie = true;
                    before = false;
                } else {
                    before = (w < wk) || (w == wk && j <= jk);  // same instance: processing order
                }
                if (before) v += rs.d;
            }
        }
        if (tie) {
            atomicCAS(&ctl->reason, 0, kPdesTiePeak);
            atomicMax(&ctl->status, kErrPdes);
        }
        best = max(best, v);
    }
    if (best != LLONG_MIN) atomicMax(&ctl->peak, best);
}

template <bool TAIL_FAST>
DEVI void run_replica_pdes(const Arena& a, int r, char* smem, int max_ni, int hs, int c_smem,
                           int W) {
    const ReplicaDesc d = a.desc[r];
    const int warp = threadIdx.x >> 5;
    Rep R;
    R.n = d.n;
    R.ni = d.ni;
#ifdef PB_ONLY_POLICY
    R.policy = PB_ONLY_POLICY;
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
    R.logcap = 0;
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
    R.heap = a.heap + d.pheap_base;
    R.hs = hs;
    R.hcap = (long long)R.n + 2;
    const long long wo = (long long)warp * a.wstride;
    R.g_cand = a.cand + wo + g;
    R.g_tmp = a.tmp + wo + g;
    R.g_tmpq = a.tmpq + wo + g;
    R.g_cstat = a.cstat + wo + g;
    R.elist = a.elist + wo + g;
    R.stack = a.stack + wo + g;
    R.log = a.log;
    R.rs = a.rs + g;
    R.spec = const_cast<int4*>(a.spec) + g;
    R.blocked = a.blocked + g;
    R.aoff = const_cast<int*>(a.aoff32) + g;
    const int ni = d.ni;
    // ---- shared-memory carve-up (engine.h pdes_smem)
    char* sp = smem;
    R.s.gpu = reinterpret_cast<long long*>(sp);
    R.s.cpu = R.s.gpu + max_ni;
    R.s.iter_start = reinterpret_cast<double*>(R.s.cpu + max_ni);
    R.s.link = R.s.iter_start + max_ni;
    R.s.hi_len = reinterpret_cast<int*>(R.s.link + max_ni);
    R.s.lo_len = R.s.hi_len + max_ni;
    R.s.hcount = R.s.lo_len + max_ni;
    R.s.lcount = R.s.hcount + max_ni;
    R.s.afresh = R.s.lcount + max_ni;
    R.s.blen = R.s.afresh + max_ni;
    R.s.busy = R.s.blen + max_ni;
    R.s.healthy = R.s.busy + max_ni;
    sp += smem_inst_bytes(max_ni);
    R.s.evseq = reinterpret_cast<unsigned long long*>(sp);
    R.s.gtime = reinterpret_cast<double*>(R.s.evseq + max_ni);
    R.s.hn = reinterpret_cast<int*>(R.s.gtime + max_ni);
    R.s.hspill = R.s.hn + max_ni;
    R.s.enq = reinterpret_cast<unsigned*>(R.s.hspill + max_ni);
    R.s.dmin = reinterpret_cast<int*>(R.s.enq + max_ni);
    sp += max_ni * 32;
    R.s_heap = reinterpret_cast<HeapEnt*>(sp);
    sp += max_ni * hs * 16;
    char* wbase = sp;
    const int wbytes = pdes_warp_bytes(c_smem);
    char* wsp = wbase + warp * wbytes;
    R.c_smem = c_smem;
    R.s_cand = reinterpret_cast<int4*>(wsp);
    R.s_tmp = R.s_cand + c_smem;
    R.s_tmpq = reinterpret_cast<unsigned*>(R.s_tmp + c_smem);
    R.s_cstat = reinterpret_cast<unsigned char*>(R.s_tmpq + c_smem);
    R.prec = reinterpret_cast<PeakRec*>(wsp + smem_cand_bytes(c_smem));
    const char* prec_all = wbase + smem_cand_bytes(c_smem);
    const int prec_stride = wbytes;  // bytes between warps' record buffers
    PdesCtl* ctl = reinterpret_cast<PdesCtl*>(wbase + W * wbytes);

    for (int i = threadIdx.x; i < ni; i += blockDim.x) {
        R.s.gpu[i] = 0;
        R.s.cpu[i] = 0;
        R.s.iter_start[i] = 0.0;
        R.s.link[i] = 0.0;
        R.s.hi_len[i] = R.s.lo_len[i] = R.s.hcount[i] = R.s.lcount[i] = 0;
        R.s.afresh[i] = R.s.blen[i] = R.s.busy[i] = 0;
        R.s.healthy[i] = 1;
        R.s.evseq[i] = 0;
        R.s.gtime[i] = CUDART_INF;
        R.s.hn[i] = R.s.hspill[i] = 0;
        R.s.enq[i] = 0;
        R.s.dmin[i] = 255;
    }
    for (int k = threadIdx.x; k < R.n; k += blockDim.x) {  // engine.cpp:382-389
        ReqState z0;
        z0.h = make_int4(0, 0, 0, 0);
        z0.meta = m_set_phase(0u, PH_WAIT);
        z0.qused = 0;
        z0.ndel = 0;
        z0.cursor = 0;
        R.rs[k] = z0;
        R.blocked[k] = 0.0;
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
    if (threadIdx.x == 0) {
        ctl->next_arr = 0;
        ctl->total = 0;
        ctl->peak = 0;
        for (int c = 0; c < 10; ++c) ctl->cnt[c] = 0;
        ctl->status = 0;
        ctl->reason = 0;
    }
    __syncthreads();

    Scal S;
    S.heap = nullptr;
    S.heap_slots = 0;
    S.now = 0.0;
    S.evseq = 0;
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
    S.prec_base = 0;
    S.prec_n = 0;
    S.cur_inst = 0;
    S.phase_b = false;
    S.reason = 0;
    S.nb = 0;
    const bool pascal = R.policy == kPascal;
    const bool oracle = R.policy == kOracle;
    const double L = d.lookahead;

    long long rounds = 0;
    while (true) {
        ++rounds;
        // ---- round start: every warp publishes its instances' earliest
        // pending event, earliest pending cross-instance event and earliest
        // time a new cross-instance event could be created (Pascal: an
        // instance whose queued requests are >= d tokens from a phase
        // boundary cannot end one before its next event + max(1, d-1)
        // iterations of >= lookahead each; the oracle bounds its rounds by
        // one lookahead to bound its peak records)
        double mn = CUDART_INF, gg = CUDART_INF, eb = CUDART_INF;
        for (int i = warp; i < ni; i += W) {
            if (R.s.hn[i] > 0) {
                const double t = inst_heap(R, i)[1].t;
                mn = fmin(mn, t);
                if (pascal) {
                    const int dk = max(1, R.s.dmin[i] - 1);
                    // (1 - 1e-9) covers the rounding of dk repeated additions
                    eb = fmin(eb, __dadd_rn(t, __dmul_rn((double)dk * L, 1.0 - 1e-9)));
                }
            }
            gg = fmin(gg, R.s.gtime[i]);
        }
        if (oracle && mn < CUDART_INF && L > 0.0) eb = __dadd_rn(mn, L);
        if (lane_id() == 0) {
            ctl->wmin[warp] = mn;
            ctl->wg[warp] = gg;
            ctl->web[warp] = eb;
            ctl->wstat[warp] = S.status;
        }
        __syncthreads();
        double MN = CUDART_INF, G = CUDART_INF, EB = CUDART_INF;
        int st = ctl->status;
        for (int w = 0; w < W; ++w) {
            MN = fmin(MN, ctl->wmin[w]);
            G = fmin(G, ctl->wg[w]);
            EB = fmin(EB, ctl->web[w]);
            if (st == 0) st = ctl->wstat[w];
        }
        const int na = ctl->next_arr;
        __syncthreads();  // everyone has read the round-start state
        if (st != 0) break;
        const double TA = na < R.n ? R.arrival[na] : CUDART_INF;
        if (MN == CUDART_INF && TA == CUDART_INF) break;
        const double H = fmin(fmin(TA, G), EB);
        // Phase B action (warp 0, after every warp finished phase A):
        // 1 = the arrival at H, 2 = instance gi's cross-instance event at H
        int bact = 0, gi = -1;
        if (TA == H && TA <= G && TA < CUDART_INF) bact = 1;
        else if (G == H && G < CUDART_INF) bact = 2;
        if (bact == 0 && !(MN < H)) {  // no event can advance: decline
            if (threadIdx.x == 0) {
                ctl->status = kErrPdes;
                ctl->reason = kPdesNoProgress;
            }
            __syncthreads();
            continue;
        }

        // ---- one event loop (a single inlined copy of the handlers and the
        // planner) run in two passes: pass 0 = phase A (every warp, its own
        // instances' events before H), pass 1 = phase B (warp 0: the event at
        // H). The CTA barrier between the passes (one PC for every warp)
        // orders every warp's phase-A shared-memory writes before warp 0's
        // phase-B reads, and phase B's writes before the next round.
        S.prec_n = 0;
        int ii = warp;
        bool b_started = false, b_over = false;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          S.phase_b = pass == 1;
          while (true) {
            HeapEnt e;
            int inst = -1;
            if (!S.phase_b) {
                while (ii < ni && !(S.status == 0 && R.s.hn[ii] > 0 && inst_heap(R, ii)[1].t < H))
                    ii += W;
                if (ii >= ni) break;
                inst = ii;
                e = heap_pop_inst(R, ii);
            } else {
                if (warp != 0 || bact == 0 || S.status != 0 || b_over) break;
                if (bact == 1) {
                    b_over = true;
                    e.t = TA;
                    e.key = (unsigned long long)na;  // kind 0 = arrival
                    if (lane_id() == 0) ctl->next_arr = na + 1;
                } else {
                    if (!b_started) {
                        // the cross-instance event's instance; any other
                        // instance with a pending event at exactly H (or a
                        // second cross-instance event) would need the global
                        // seq order: decline
                        int cnt = 0, who = -1;
                        for (int i = lane_id(); i < ni; i += 32) {
                            if (R.s.gtime[i] == H) {
                                ++cnt;
                                who = i;
                            } else if (R.s.hn[i] > 0 && inst_heap(R, i)[1].t == H) {
                                ++cnt;
                            }
                        }
                        cnt = warp_sum(cnt);
                        who = (int)warp_max_u((unsigned)(who + 1)) - 1;
                        b_started = true;
                        if (cnt != 1 || who < 0) {
                            if (S.status == 0) S.status = kErrPdes;
                            if (lane_id() == 0) atomicCAS(&ctl->reason, 0, kPdesTieB);
                            break;
                        }
                        gi = who;
                    }
                    if (R.s.hn[gi] == 0) {  // cannot happen: the event is pending
                        if (S.status == 0) S.status = kErrPdes;
                        break;
                    }
                    inst = gi;
                    e = heap_pop_inst(R, gi);
                    const unsigned k = (unsigned)(e.key >> 26) & 7u;
                    if (k == EV_ITER || k == EV_PREFILL) b_over = true;
                }
            }
            // ---- process one event (engine.cpp:392-404 loop body)
            const unsigned kind = (unsigned)(e.key >> 26) & 7u;
            const unsigned id = (unsigned)(e.key & ((1u << 26) - 1u));
            S.events++;
            S.now = e.t;  // an instance's events pop in (time, seq) order
            if (kind == EV_ITER || kind == EV_PREFILL) {
                if (lane_id() == 0) R.s.gtime[inst] = CUDART_INF;
                __syncwarp();
            }
            int plan_inst;
            switch (kind) {
                case 0:
                    plan_inst = on_arrival(R, S, (int)id);
                    break;
                case EV_PREFILL: plan_inst = on_prefill_complete(R, S, (int)id); break;
                case EV_ITER: plan_inst = on_iteration_complete(R, S, (int)id); break;
                case EV_SWAP: plan_inst = on_swap_complete(R, S, (int)id); break;
                default: plan_inst = on_transfer_complete(R, S, (int)id); break;
            }
            S.cur_inst = plan_inst;
            if (S.phase_b) S.nb++;
            maybe_start<TAIL_FAST>(R, S, plan_inst);
            if (oracle) peak_record(R, S, false);
            if (S.status != 0 && !S.phase_b && warp != 0) break;
          }
          __syncthreads();
        }
        if (lane_id() == 0) {
            ctl->wrec[warp] = S.prec_n;
            if (S.status != 0) atomicCAS(&ctl->status, 0, S.status);
            if (S.reason != 0) atomicCAS(&ctl->reason, 0, S.reason);
        }
        __syncthreads();
        if (oracle) {
            pdes_merge_peak(ctl, prec_all, prec_stride, W);
            __syncthreads();
            if (threadIdx.x == 0) {
                long long tot = ctl->total;
                for (int w = 0; w < W; ++w)
                    for (int j = 0; j < ctl->wrec[w]; ++j)
                        tot += prec_at(prec_all, prec_stride, w, j).d;
                ctl->total = tot;
            }
        }
        __syncthreads();
    }

    // ---- epilogue: counters, status, outputs the metric kernels read
    if (lane_id() == 0) {
        atomicAdd((unsigned long long*)&ctl->cnt[0], (unsigned long long)S.events);
        atomicAdd((unsigned long long*)&ctl->cnt[1], (unsigned long long)S.plans);
        atomicAdd((unsigned long long*)&ctl->cnt[2], (unsigned long long)S.visits);
        atomicAdd((unsigned long long*)&ctl->cnt[3], (unsigned long long)S.req_iters);
        atomicAdd((unsigned long long*)&ctl->cnt[4], (unsigned long long)S.ans_tokens);
        atomicAdd((unsigned long long*)&ctl->cnt[5], (unsigned long long)S.health);
        atomicAdd((unsigned long long*)&ctl->cnt[6], (unsigned long long)S.adm_rounds);
        atomicAdd((unsigned long long*)&ctl->cnt[7], (unsigned long long)S.adm_slow);
        atomicAdd((unsigned long long*)&ctl->cnt[8], (unsigned long long)S.done);
        atomicAdd((unsigned long long*)&ctl->cnt[9], (unsigned long long)S.nb);
        if (S.status != 0) atomicCAS(&ctl->status, 0, S.status);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < R.n; k += blockDim.x) R.rec[k].blocked = R.blocked[k];
    if (threadIdx.x == 0) {
        ReplicaOut o;
        o.status = ctl->status;
        if (o.status == 0 && ctl->cnt[8] != R.n) o.status = kErrStall;
        o.pad = o.status == kErrPdes ? (ctl->reason ? ctl->reason : -1) : 0;
        o.peak = ctl->peak;
        o.nlog = ctl->cnt[9];     // PDES: serialised (phase-B) events
        o.now = (double)rounds;   // PDES: rounds
        o.events = ctl->cnt[0];
        o.plans = ctl->cnt[1];
        o.visits = ctl->cnt[2];
        o.req_iters = ctl->cnt[3];
        o.answer_tokens = ctl->cnt[4];
        o.health_checks = ctl->cnt[5];
        o.adm_rounds = ctl->cnt[6];
        o.adm_slow = ctl->cnt[7];
        o.now = 0.0;
        a.out[r] = o;
    }
    __syncthreads();
}

// One CTA per replica (work-stolen), W warps; 255 registers per thread at
// W <= 8 (one CTA per SM).
__global__ void __launch_bounds__(kPdesMaxWarps * 32, 1)
    pdes_kernel(Arena a, int max_ni, int hs, int c_smem, int W) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ int rsel;
    while (true) {
        if (threadIdx.x == 0) {
            const int w = atomicAdd(a.work, 1);
            rsel = w < a.n_rep ? a.order[w] : -1;
        }
        __syncthreads();
        const int r = rsel;
        __syncthreads();
        if (r < 0) break;
        run_replica_pdes<false>(a, r, smem_raw, max_ni, hs, c_smem, W);
    }
}

int launch_engine(const Arena& a, int max_ni, int hs, int c_smem, int warps, int blocks,
                  void* stream) {
    if (warps < 1 || warps > kPdesMaxWarps || hs < 2) return 1;
    const size_t smem = (size_t)pdes_smem(max_ni, hs, c_smem, warps);
    if (smem > 48 * 1024) {
        if (cudaFuncSetAttribute(pdes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return 2;
    }
    pdes_kernel<<<blocks, warps * 32, smem, (cudaStream_t)stream>>>(a, max_ni, hs, c_smem, warps);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
