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
//     Inst::gtime).
// The engine advances in rounds. Round horizon
//   H = min(next arrival, earliest pending cross-instance event,
//           earliest pending event + lookahead bound)
// where the lookahead (ReplicaDesc::lookahead, host-computed) bounds from
// below the duration of any iteration / prefill, so no event processed in the
// round can create a cross-instance event before H.
//   Phase A: every warp processes its instances' events with time < H,
//     concurrently (they commute: disjoint state), recording each event.
//   Merge (warp 0): the reference's seq of every push is its rank in the
//     global push order, and pushes happen in the global processing order
//     (time, seq). Phase-A pushes carry provisional keys {warp, record, push
//     index}; merging the round's records by (time, exact seq) — an event's
//     seq is known once the event that pushed it has been merged — assigns
//     every push its exact global seq, which then replaces the provisional
//     keys still in the heaps. The oracle's Σ gpu_used samples
//     (engine.cpp:75-79) are accumulated in the same order.
//   Phase B (warp 0): every event at exactly H, across instances, in
//     (time, seq) order — the arrival (seqs 1..n precede every dynamic event)
//     and the cross-instance events with every other instance paused at H.
// So ties between instances are broken exactly as the reference breaks them.
// A record-buffer overflow or a horizon that cannot advance makes the engine
// decline the replica (kErrPdes); the host re-runs it on the serial engine.

struct PdesCtl {
    double wmin[kPdesMaxWarps];  // per warp: earliest pending event time
    double wg[kPdesMaxWarps];    // per warp: earliest pending cross-instance event time
    double web[kPdesMaxWarps];   // per warp: earliest possible new cross-instance event
    int wstat[kPdesMaxWarps];
    int wrec[kPdesMaxWarps];     // per warp: phase-A records this round
    int next_arr;
    int tie;                     // merge: the round has a cross-instance time tie
    unsigned long long gseq;  // last global push seq (arrivals hold 1..n)
    long long total;          // oracle: Σ gpu_used after the merged events
    long long peak;
    long long cnt[10];  // events plans visits req_iters ans_tokens health adm_rounds adm_slow done
                        // phase-B events
    int status;
    int reason;  // why the replica was declined (kPdes* below), for diagnostics
};
enum : int {
    kPdesRecs = 3,       // record buffer or push-index overflow
    kPdesNoProgress = 4, // horizon does not advance (lookahead below the clock's ulp)
    kPdesOrder = 5,      // a cross-instance action outside phase B (flagging bug guard)
};
static_assert(sizeof(PdesCtl) <= 512, "pdes_ctl_bytes");

// Global key of a record / heap key: provisional keys {warp, record, push
// index} resolve through the pushing event's merged gbase.
DEVI unsigned long long pdes_global_key(const PdesRec* prec, unsigned long long key) {
    const unsigned long long sq = key >> 29;
    if (!(sq & kPdesProv)) return key;
    const int w = (int)((sq >> 31) & 7u);
    const int r = (int)((sq >> 19) & 4095u);
    const unsigned long long p = sq & ((1ull << 19) - 1u);
    const unsigned long long g = prec[(long long)w * kPdesRecCap + r].gbase + 1 + p;
    return (g << 29) | (key & ((1ull << 29) - 1u));
}

// Merge of the round's phase-A records (warp 0; every instance's records are
// contiguous and in its processing order, R.s.mcur / mend). Repeatedly takes
// the instance whose next record has the smallest (time, global key), gives
// that event's pushes the next global seqs, and adds its Σ gpu_used changes.
DEVI void pdes_merge(const Rep& R, PdesCtl* ctl, int ni, bool oracle) {
    const int ln = lane_id();
    for (int i = ln; i < ni; i += 32) {  // heads
        if (R.s.mcur[i] >= 0 && R.s.mcur[i] < R.s.mend[i]) {
            const PdesRec& h = R.prec[R.s.mcur[i]];
            R.s.mt[i] = h.t;
            R.s.mk[i] = pdes_global_key(R.prec, h.key);
        }
    }
    __syncwarp();
    unsigned long long G = ctl->gseq;
    long long total = ctl->total, peak = ctl->peak;
    while (true) {
        double bt = CUDART_INF;
        unsigned long long bk = ~0ull;
        int bi = -1;
        for (int i = ln; i < ni; i += 32) {
            if (R.s.mcur[i] < 0 || R.s.mcur[i] >= R.s.mend[i]) continue;
            const double t = R.s.mt[i];
            const unsigned long long k = R.s.mk[i];
            if (t < bt || (t == bt && k < bk)) bt = t, bk = k, bi = i;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double t2 = __shfl_xor_sync(FULL, bt, o);
            const unsigned long long k2 = __shfl_xor_sync(FULL, bk, o);
            const int i2 = __shfl_xor_sync(FULL, bi, o);
            if (t2 < bt || (t2 == bt && k2 < bk)) bt = t2, bk = k2, bi = i2;
        }
        if (bi < 0) break;
        const int rix = R.s.mcur[bi];
        const PdesRec& e = R.prec[rix];
        const int npush = e.npush;
        if (oracle) {
            total += e.d1;
            if (e.inst < 0 && total > peak) peak = total;  // bit 31: sampled
            total += e.d2;
        }
        __syncwarp();
        if (ln == 0) {
            R.prec[rix].gbase = G;
            R.s.mcur[bi] = rix + 1;
        }
        G += (unsigned long long)npush;
        __syncwarp();
        if (ln == (bi & 31) && rix + 1 < R.s.mend[bi]) {  // the owning lane loads the next head
            const PdesRec& h = R.prec[rix + 1];
            R.s.mt[bi] = h.t;
            R.s.mk[bi] = pdes_global_key(R.prec, h.key);
        }
        __syncwarp();
    }
    __syncwarp();
    if (ln == 0) {
        ctl->gseq = G;
        ctl->total = total;
        ctl->peak = peak;
    }
}

// The same merge, CTA-parallel, for rounds without a cross-instance time tie
// (the common case): then the global order is the time order, each record's
// rank is its position in its instance's list plus, per other instance, the
// number of its records with a smaller time (binary search); the pushes' seqs
// and the running Σ gpu_used follow from prefix sums in rank order. Returns
// false (nothing written) when a tie exists; the caller then runs the serial
// merge. All threads of the CTA call it.
DEVI bool pdes_merge_par(const Rep& R, PdesCtl* ctl, int ni, int W, bool oracle) {
    __shared__ long long s_np[kPdesMaxWarps * 32], s_d[kPdesMaxWarps * 32];
    __shared__ long long s_pk[kPdesMaxWarps];
    int off[kPdesMaxWarps + 1];
    off[0] = 0;
    for (int w = 0; w < W; ++w) off[w + 1] = off[w] + ctl->wrec[w];
    const int M = off[W];
    const int T = blockDim.x, tid = threadIdx.x;
    if (tid == 0) ctl->tie = 0;
    __syncthreads();
    if (M == 0) return true;
    for (int f = tid; f < M; f += T) {
        int w = 0;
        while (off[w + 1] <= f) ++w;
        const int r = w * kPdesRecCap + (f - off[w]);
        const double t = R.prec[r].t;
        const int i = R.prec[r].inst & 0x7fffffff;
        int rank = r - R.s.mcur[i];
        bool tie = false;
        for (int q = 0; q < ni; ++q) {
            const int lo0 = R.s.mcur[q];
            if (q == i || lo0 < 0) continue;
            int lo = lo0, hi = R.s.mend[q];  // first record with time >= t
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (R.prec[mid].t < t) lo = mid + 1;
                else hi = mid;
            }
            if (lo < R.s.mend[q] && R.prec[lo].t == t) tie = true;
            rank += lo - lo0;
        }
        if (tie) ctl->tie = 1;
        R.prec[r].rank = rank;
        R.pord[rank] = r;
    }
    __syncthreads();
    if (ctl->tie) return false;
    // prefix sums in rank order: thread tid owns ranks [tid*C, tid*C + C)
    const int C = (M + T - 1) / T;
    const int k0 = min(M, tid * C), k1 = min(M, k0 + C);
    long long np = 0, dd = 0;
    for (int k = k0; k < k1; ++k) {
        const PdesRec& e = R.prec[R.pord[k]];
        np += e.npush;
        dd += e.d1 + e.d2;
    }
    s_np[tid] = np;
    s_d[tid] = dd;
    __syncthreads();
    if (tid == 0) {  // exclusive scan of the T partial sums
        long long a = 0, b = 0;
        for (int u = 0; u < T; ++u) {
            const long long x = s_np[u], y = s_d[u];
            s_np[u] = a;
            s_d[u] = b;
            a += x;
            b += y;
        }
        s_pk[0] = a;  // totals
        s_pk[1] = b;
    }
    __syncthreads();
    const unsigned long long G0 = ctl->gseq;
    const long long tot0 = ctl->total;
    unsigned long long gb = G0 + (unsigned long long)s_np[tid];
    long long tot = tot0 + s_d[tid], pk = LLONG_MIN;
    for (int k = k0; k < k1; ++k) {
        const int r = R.pord[k];
        const PdesRec e = R.prec[r];
        R.prec[r].gbase = gb;
        gb += (unsigned long long)e.npush;
        if (oracle) {
            tot += e.d1;
            if (e.inst < 0 && tot > pk) pk = tot;
            tot += e.d2;
        }
    }
    const long long ntot = s_pk[0], dtot = s_pk[1];
    __syncthreads();
    // CTA max of the sampled totals
    for (int o = 16; o; o >>= 1) pk = max(pk, __shfl_xor_sync(FULL, pk, o));
    if (lane_id() == 0) s_pk[tid >> 5] = pk;
    __syncthreads();
    if (tid == 0) {
        long long m = ctl->peak;
        for (int w = 0; w < (T >> 5); ++w) m = max(m, s_pk[w]);
        ctl->peak = m;
        ctl->gseq = G0 + (unsigned long long)ntot;
        ctl->total = tot0 + dtot;
    }
    __syncthreads();
    return true;
}

// Replace the provisional keys left in instance i's heap by the merged global
// seqs (the relative order of the heap's keys is unchanged: provisional keys
// follow every global one and keep their push order, so do their seqs).
DEVI void pdes_fix_heap(const Rep& R, int i) {
    HeapEnt* h = inst_heap(R, i);
    const int hn = R.s.hn[i];
    for (int k = 1 + lane_id(); k <= hn; k += 32) {
        const unsigned long long key = h[k].key;
        if ((key >> 29) & kPdesProv) h[k].key = pdes_global_key(R.prec, key);
    }
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
    R.s.gpu = reinterpret_cast<long long*>(sp + 32);  // rcp_of slots ahead
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
    R.s.gtime = reinterpret_cast<double*>(sp);
    R.s.mt = R.s.gtime + max_ni;
    R.s.mk = reinterpret_cast<unsigned long long*>(R.s.mt + max_ni);
    R.s.hn = reinterpret_cast<int*>(R.s.mk + max_ni);
    R.s.hspill = R.s.hn + max_ni;
    R.s.enq = reinterpret_cast<unsigned*>(R.s.hspill + max_ni);
    R.s.dmin = reinterpret_cast<int*>(R.s.enq + max_ni);
    R.s.mcur = R.s.dmin + max_ni;
    R.s.mend = R.s.mcur + max_ni;
    sp += max_ni * 48;
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
    R.prec = a.prec + (long long)blockIdx.x * kPdesMaxWarps * kPdesRecCap;
    R.pord = a.pord + (long long)blockIdx.x * kPdesMaxWarps * kPdesRecCap;
    PdesRec* const myrec = R.prec + (long long)warp * kPdesRecCap;
    PdesCtl* ctl = reinterpret_cast<PdesCtl*>(wbase + W * wbytes);

    if (threadIdx.x < 32) set_rcps(R);  // thread 0 writes
    for (int i = threadIdx.x; i < ni; i += blockDim.x) {
        R.s.gpu[i] = 0;
        R.s.cpu[i] = 0;
        R.s.iter_start[i] = 0.0;
        R.s.link[i] = 0.0;
        R.s.hi_len[i] = R.s.lo_len[i] = R.s.hcount[i] = R.s.lcount[i] = 0;
        R.s.afresh[i] = R.s.blen[i] = R.s.busy[i] = 0;
        R.s.healthy[i] = 1;
        R.s.gtime[i] = CUDART_INF;
        R.s.hn[i] = R.s.hspill[i] = 0;
        R.s.enq[i] = 0;
        R.s.dmin[i] = 255;
        R.s.mcur[i] = R.s.mend[i] = -1;
        R.s.mk[i] = (unsigned long long)R.n;  // FCFS / RR: per-instance push seqs after the arrivals
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
        ctl->gseq = (unsigned long long)R.n;  // arrivals hold seqs 1..n (engine.cpp:384-389)
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
    S.d1 = 0;
    S.sampled = false;
    S.rec_n = 0;
    S.npush = 0;
    S.gseq = 0;
    S.phase_b = false;
    S.reason = 0;
    S.nb = 0;
    const bool pascal = R.policy == kPascal;
    const bool oracle = R.policy == kOracle;
    // exact global seqs (records + merge) where cross-instance order matters:
    // Pascal (boundaries read every instance) and the oracle (Σ gpu_used
    // samples); FCFS / RR order per instance only (heap_push)
    const bool exact = pascal || oracle;
    const double L = d.lookahead;

    long long rounds = 0;
    while (true) {
        ++rounds;
        // ---- round start: every warp publishes its instances' earliest
        // pending event, earliest pending cross-instance event and earliest
        // time a new cross-instance event could be created (Pascal: an
        // instance whose queued requests are >= d tokens from a phase
        // boundary cannot end one before its next event + max(1, d-1)
        // iterations of >= lookahead each, d capped so a round stays within
        // the record buffers; the oracle bounds its rounds by one lookahead)
        double mn = CUDART_INF, gg = CUDART_INF, eb = CUDART_INF;
        for (int i = warp; i < ni; i += W) {
            if (R.s.hn[i] > 0) {
                const double t = inst_heap(R, i)[1].t;
                mn = fmin(mn, t);
                if (pascal) {
                    const int dk = min(64, max(1, R.s.dmin[i] - 1));
                    // (1 - 1e-9) covers the rounding of dk repeated additions
                    eb = fmin(eb, __dadd_rn(t, __dmul_rn((double)dk * L, 1.0 - 1e-9)));
                }
            }
            gg = fmin(gg, R.s.gtime[i]);
            if (lane_id() == 0) R.s.mcur[i] = R.s.mend[i] = -1;
        }
        if (oracle && mn < CUDART_INF && L > 0.0)  // no boundaries: bound the round's size
            eb = __dadd_rn(mn, __dmul_rn(64.0 * L, 1.0 - 1e-9));
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
        const int na0 = ctl->next_arr;
        __syncthreads();  // everyone has read the round-start state
        if (st != 0) break;
        const double TA = na0 < R.n ? R.arrival[na0] : CUDART_INF;
        if (MN == CUDART_INF && TA == CUDART_INF) break;
        const double H = fmin(fmin(TA, G), EB);
        if (!(MN < H) && !(TA == H) && !(G == H)) {  // no event can advance: decline
            if (threadIdx.x == 0) {
                ctl->status = kErrPdes;
                ctl->reason = kPdesNoProgress;
            }
            __syncthreads();
            continue;
        }

        // ---- one event loop (a single inlined copy of the handlers and the
        // planner) run in two passes: pass 0 = phase A (every warp, its own
        // instances' events before H), pass 1 = phase B (warp 0: every event
        // at H in (time, seq) order). CTA barriers between the phases order
        // the shared-memory writes of one phase before the reads of the next.
        S.rec_n = 0;
        int ii = warp;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          S.phase_b = pass == 1;
          if (S.phase_b) S.gseq = ctl->gseq;
          while (true) {
            HeapEnt e;
            int inst = -1;
            if (!S.phase_b) {
                while (ii < ni && !(S.status == 0 && R.s.hn[ii] > 0 && inst_heap(R, ii)[1].t < H))
                    ii += W;
                if (ii >= ni) break;
                if (exact && S.rec_n >= kPdesRecCap) {
                    if (S.status == 0) S.status = kErrPdes, S.reason = kPdesRecs;
                    break;
                }
                inst = ii;
                if (exact && lane_id() == 0 && R.s.mcur[ii] < 0)
                    R.s.mcur[ii] = warp * kPdesRecCap + S.rec_n;
                e = heap_pop_inst(R, ii);
            } else {
                if (warp != 0 || S.status != 0) break;
                // the next event at exactly H: the arrival (seq k + 1) or the
                // heap top with the smallest global key
                const int na = ctl->next_arr;
                const bool arr = na < R.n && R.arrival[na] == H;
                unsigned long long bk = ~0ull;
                int bi = -1;
                for (int i = lane_id(); i < ni; i += 32) {
                    if (R.s.hn[i] > 0) {
                        const HeapEnt top = inst_heap(R, i)[1];
                        if (top.t == H && top.key < bk) bk = top.key, bi = i;
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long k2 = __shfl_xor_sync(FULL, bk, o);
                    const int i2 = __shfl_xor_sync(FULL, bi, o);
                    if (k2 < bk) bk = k2, bi = i2;
                }
                if (arr && (bi < 0 || ((unsigned long long)na + 1) < (bk >> 29))) {
                    e.t = H;
                    e.key = (unsigned long long)na;  // kind 0 = arrival
                    __syncwarp();
                    if (lane_id() == 0) ctl->next_arr = na + 1;
                    __syncwarp();
                } else if (bi >= 0) {
                    inst = bi;
                    e = heap_pop_inst(R, bi);
                } else {
                    break;
                }
            }
            // ---- process one event (engine.cpp:392-404 loop body)
            const unsigned kind = (unsigned)(e.key >> 26) & 7u;
            const unsigned id = (unsigned)(e.key & ((1u << 26) - 1u));
            S.events++;
            S.now = e.t;  // an instance's events pop in (time, seq) order
            S.npush = 0;
            S.sampled = false;
            S.prec_base = S.gpu_total;
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
            maybe_start<TAIL_FAST>(R, S, plan_inst);
            // the event's changes of Σ gpu_used before / after its sample
            const long long dt = S.gpu_total - S.prec_base;
            const long long d1 = S.sampled ? S.d1 : dt;
            const long long d2 = dt - d1;
            if (!S.phase_b) {
                if (exact && lane_id() == 0) {
                    PdesRec rc;
                    rc.t = e.t;
                    rc.key = e.key;
                    rc.d1 = d1;
                    rc.d2 = d2;
                    rc.inst = inst | (S.sampled ? (int)0x80000000u : 0);
                    rc.npush = S.npush;
                    rc.gbase = 0;
                    rc.rank = 0;
                    rc.pad = 0;
                    myrec[S.rec_n] = rc;
                    R.s.mend[inst] = warp * kPdesRecCap + S.rec_n + 1;
                }
                S.rec_n++;
                __syncwarp();
            } else {
                S.nb++;
                if (oracle && lane_id() == 0) {  // serial: the exact global order
                    long long tot = ctl->total + d1;
                    if (S.sampled && tot > ctl->peak) ctl->peak = tot;
                    ctl->total = tot + d2;
                }
                __syncwarp();
            }
            if (S.status != 0 && !S.phase_b && warp != 0) break;
          }
          if (pass == 0 && lane_id() == 0) ctl->wrec[warp] = S.rec_n;
          __syncthreads();
          if (pass == 0 && exact) {
              // exact global seqs for the phase-A pushes, then the heaps
              if (!pdes_merge_par(R, ctl, ni, W, oracle)) {  // a time tie: serial merge
                  if (warp == 0) pdes_merge(R, ctl, ni, oracle);
                  __syncthreads();
              }
              for (int i = warp; i < ni; i += W) pdes_fix_heap(R, i);
              __syncthreads();
          } else if (pass == 1 && warp == 0 && lane_id() == 0) {
              ctl->gseq = S.gseq;
          }
        }
        if (lane_id() == 0) {
            if (S.status != 0) atomicCAS(&ctl->status, 0, S.status);
            if (S.reason != 0) atomicCAS(&ctl->reason, 0, S.reason);
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
