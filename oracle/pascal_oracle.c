/* pascal_oracle.c — TEST INFRASTRUCTURE ONLY (see pascal_oracle.h).
 *
 * Literal C restatement of the reference scheduling loop. Every function names
 * the reference lines it restates. Nothing here is on the product path; the
 * product is the CUDA engine in paper_2602_11530_b200/csrc/.
 */
#include "pascal_oracle.h"

#include <limits.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- defaults */

void po_profile_default(po_profile* p) { /* costmodel.hpp:12-21 */
    p->prefill_base = 0.0;
    p->prefill_per_token = 0.00025;
    p->decode_base = 0.03;
    p->decode_per_request = 0.0;
    p->decode_per_kv_token = 0.0;
    p->swap_bandwidth = 51200.0;
    p->fabric_bandwidth = 51200.0;
    p->fabric_latency = 0.0;
}

void po_config_default(po_config* c) { /* engine.hpp:18-33 */
    c->instance_count = 8;
    c->gpu_capacity = 0;
    c->capacity_fraction = 0.0;
    c->token_quantum = 500;
    c->demotion_threshold = 5000;
    c->policy = PO_PASCAL;
    c->no_migration = 0;
    c->non_adaptive = 0;
    c->target_tpot = 0.1;
    c->ttfat_target = 0.25;
    c->qoe_threshold = 0.95;
    c->pacer_slack_tokens = 0;
}

/* --------------------------------------------------------------- costmodel */
/* costmodel.cpp:35-51 */
static double prefill_latency(const po_profile* p, long prompt) {
    return p->prefill_base + p->prefill_per_token * (double)prompt;
}
static double decode_step_latency(const po_profile* p, long batch, long kv) {
    return p->decode_base + p->decode_per_request * (double)batch +
           p->decode_per_kv_token * (double)kv;
}
static double swap_latency(const po_profile* p, long kv) {
    if (kv == 0) return 0.0;
    return (double)kv / p->swap_bandwidth;
}
static double transfer_latency(const po_profile* p, long kv) {
    return p->fabric_latency + (double)kv / p->fabric_bandwidth;
}

/* ------------------------------------------------------------------ vectors */
typedef struct {
    long* v;
    long n, cap;
} lvec;
static void lv_push(lvec* a, long x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 16;
        a->v = (long*)realloc(a->v, (size_t)a->cap * sizeof(long));
    }
    a->v[a->n++] = x;
}
static void lv_remove(lvec* a, long x) { /* erase(remove(...)) engine.cpp:118-120 */
    long w = 0;
    for (long r = 0; r < a->n; ++r)
        if (a->v[r] != x) a->v[w++] = a->v[r];
    a->n = w;
}
typedef struct {
    double* v;
    long n, cap;
} dvec;
static void dv_push(dvec* a, double x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 16;
        a->v = (double*)realloc(a->v, (size_t)a->cap * sizeof(double));
    }
    a->v[a->n++] = x;
}

/* ------------------------------------------------------------------- state */
enum { PH_WAIT = 0, PH_REASON = 1, PH_ANSWER = 2, PH_MIGRATING = 3, PH_DONE = 4 };
enum { LOC_GPU = 0, LOC_CPU = 1, LOC_TRANSIT = 2 };

typedef struct { /* instance.hpp:41-62 */
    po_spec spec;
    int phase;
    long tokens, kv;
    int loc;
    long qused, quanta;
    dvec deliv, digest; /* PacerState, instance.hpp:22-39 */
    int owner;
    uint64_t seq;
    int demoted, swout, swin;
} req_t;

typedef struct { /* instance.hpp:74-88 */
    int id;
    long cap, gpu, cpu;
    lvec hi, lo, batch;
    int busy;
    double iter_start, iter_dur;
} inst_t;

typedef struct { /* engine.cpp:44-50 */
    double time;
    uint64_t seq;
    int kind, inst;
    long req;
} event_t;
enum { EV_ARRIVAL, EV_PREFILL, EV_ITER, EV_SWAP, EV_TRANSFER };

typedef struct { /* instance.hpp:65-72 */
    int id, healthy;
    long total_kv, r, a, free;
} snap_t;

typedef struct {
    const po_spec* trace;
    long n;
    const po_config* cfg;
    const po_profile* prof;
    int policy;
    FILE* log;
    req_t* reqs;
    po_record* recs;
    inst_t* inst;
    double* link_busy;
    event_t* heap;
    long hn, hcap;
    uint64_t event_seq, enq_counter;
    double now;
    long done, peak;
    int failed;
    char* err;
    size_t errlen;
} sim_t;

static void fail(sim_t* s, const char* msg) {
    if (!s->failed) {
        s->failed = 1;
        if (s->err && s->errlen) snprintf(s->err, s->errlen, "%s", msg);
    }
}

/* ---------------------------------------------------------- event queue */
/* std::priority_queue with EventAfter (engine.cpp:52-57,68): min (time,seq). */
static int ev_less(const event_t* a, const event_t* b) {
    if (a->time != b->time) return a->time < b->time;
    return a->seq < b->seq;
}
static void push_event(sim_t* s, double t, int kind, int inst, long req) { /* engine.cpp:85-89 */
    if (t < s->now - 1e-12) {
        fail(s, "event scheduled in the past");
        return;
    }
    if (s->hn == s->hcap) {
        s->hcap = s->hcap ? 2 * s->hcap : 64;
        s->heap = (event_t*)realloc(s->heap, (size_t)s->hcap * sizeof(event_t));
    }
    event_t e = {t, ++s->event_seq, kind, inst, req};
    long i = s->hn++;
    while (i > 0) {
        long p = (i - 1) / 2;
        if (!ev_less(&e, &s->heap[p])) break;
        s->heap[i] = s->heap[p];
        i = p;
    }
    s->heap[i] = e;
}
static event_t pop_event(sim_t* s) {
    event_t top = s->heap[0];
    event_t last = s->heap[--s->hn];
    long i = 0;
    for (;;) {
        long l = 2 * i + 1, r = l + 1, m = i;
        const event_t* best = &last;
        if (l < s->hn && ev_less(&s->heap[l], best)) { m = l; best = &s->heap[l]; }
        if (r < s->hn && ev_less(&s->heap[r], best)) { m = r; best = &s->heap[r]; }
        if (m == i) break;
        s->heap[i] = s->heap[m];
        i = m;
    }
    if (s->hn > 0) s->heap[i] = last;
    return top;
}

/* ------------------------------------------------------------- event log */
static void emit(sim_t* s, const char* kind, int inst, long req, const char* detail) {
    /* engine.cpp:91-97 */
    if (!s->log) return;
    fprintf(s->log, "%.9f,%s,%d,%ld,%s\n", s->now, kind, inst,
            req >= 0 ? s->reqs[req].spec.id : -1L, detail ? detail : "");
}

/* ------------------------------------------------------------------ pacer */
static void pacer_deliver(req_t* r, double t, double tpot) { /* instance.cpp:10-20 */
    dv_push(&r->deliv, t);
    if (r->digest.n == 0) dv_push(&r->digest, t);
    else {
        double prev = r->digest.v[r->digest.n - 1] + tpot;
        dv_push(&r->digest, t > prev ? t : prev); /* std::max(gen, prev+tpot) */
    }
}
static int pacer_healthy(const req_t* r, double now, long total, long slack,
                         double tpot) { /* instance.cpp:22-33 */
    if (r->deliv.n == 0) return 1;
    double t0 = r->deliv.v[0];
    long expected = 1 + (long)floor((now - t0) / tpot);
    if (expected > total) expected = total;
    long digested = 0;
    for (long k = 0; k < r->digest.n; ++k) {
        if (r->digest.v[k] <= now) ++digested;
        else break;
    }
    return digested >= expected - slack;
}

/* -------------------------------------------------------------- monitor */
static snap_t monitor_snapshot(sim_t* s, int i) { /* instance.cpp:59-76 */
    inst_t* st = &s->inst[i];
    snap_t sn;
    sn.id = st->id;
    sn.healthy = 1;
    sn.total_kv = st->gpu + st->cpu;
    sn.r = st->hi.n;
    sn.a = 0;
    sn.free = st->cap - st->gpu;
    for (long k = 0; k < st->lo.n; ++k) {
        const req_t* r = &s->reqs[st->lo.v[k]];
        if (r->quanta == 0) ++sn.a;
        if (r->phase == PH_ANSWER &&
            !pacer_healthy(r, s->now, r->spec.answering_tokens, s->cfg->pacer_slack_tokens,
                           s->cfg->target_tpot))
            sn.healthy = 0;
    }
    return sn;
}

/* ------------------------------------------------------------ placement */
/* cluster.cpp:10-23 argmin_by; key selects m_i / r_i / r_i+a_i */
static long snap_key(const snap_t* sn, int which) {
    return which == 0 ? sn->total_kv : which == 1 ? sn->r : sn->r + sn->a;
}
static int argmin_by(const snap_t* sn, int n, int healthy_only, int which) {
    int best = -1;
    long bk = 0;
    for (int i = 0; i < n; ++i) {
        if (healthy_only && !sn[i].healthy) continue;
        long k = snap_key(&sn[i], which);
        if (best < 0 || k < bk) {
            best = sn[i].id;
            bk = k;
        }
    }
    return best;
}
static int select_reasoning(const snap_t* sn, int n) { /* cluster.cpp:27-33 */
    int b = argmin_by(sn, n, 1, 0);
    if (b < 0) b = argmin_by(sn, n, 0, 0);
    return b;
}
static int select_answering(const snap_t* sn, int n) { /* cluster.cpp:35-44 */
    int b = argmin_by(sn, n, 1, 1);
    if (b < 0) b = argmin_by(sn, n, 0, 2);
    return b;
}
/* cluster.cpp:46-57: returns 1 for Migrate */
static int decide_migration(const snap_t* cur, const snap_t* tgt, long kv, const po_config* c) {
    if (c->no_migration) return 0;
    if (tgt->id == cur->id) return 0;
    if (c->non_adaptive) return 1;
    if (cur->free >= kv && tgt->free < kv) return 0;
    return 1;
}

/* ------------------------------------------------------------------ planner */
typedef struct {
    long idx;
    int cls;
} cand_t;
typedef struct { /* instance.hpp:90-100 */
    int kind; /* 0 idle 1 prefill 2 decode */
    long prefill_request;
    lvec batch, swap_ins, immediate, evictions, denied;
    double duration;
} plan_t;

static int is_candidate(const req_t* r) { /* instance.cpp:86-90 */
    if (r->phase == PH_DONE || r->loc == LOC_TRANSIT) return 0;
    if (r->swout || r->swin) return 0;
    return 1;
}
static int gpu_resident(const req_t* r) { /* instance.hpp:59-61 */
    return r->loc == LOC_GPU && !r->swout && !r->swin;
}
static long admission_need(const req_t* r) { /* instance.cpp:94-99 */
    if (r->phase == PH_WAIT) return r->spec.prompt_tokens + (r->spec.reasoning_tokens == 0 ? 1 : 0);
    if (gpu_resident(r)) return 1;
    return r->kv + 1;
}

/* Sorting context (qsort has no closure argument). */
static const req_t* g_reqs;
static int g_classed;
static int cmp_arrival(const void* A, const void* B) { /* instance.cpp:127-133 */
    const req_t* a = &g_reqs[((const cand_t*)A)->idx];
    const req_t* b = &g_reqs[((const cand_t*)B)->idx];
    if (a->spec.arrival_time != b->spec.arrival_time)
        return a->spec.arrival_time < b->spec.arrival_time ? -1 : 1;
    return a->spec.id < b->spec.id ? -1 : a->spec.id > b->spec.id ? 1 : 0;
}
static int cmp_rr(const void* A, const void* B) { /* instance.cpp:82-84,135-140 */
    const cand_t* ca = (const cand_t*)A;
    const cand_t* cb = (const cand_t*)B;
    const req_t* a = &g_reqs[ca->idx];
    const req_t* b = &g_reqs[cb->idx];
    int xa = g_classed ? ca->cls : 0, xb = g_classed ? cb->cls : 0;
    if (xa != xb) return xa < xb ? -1 : 1;
    if (a->quanta != b->quanta) return a->quanta < b->quanta ? -1 : 1;
    if (a->seq != b->seq) return a->seq < b->seq ? -1 : 1;
    return a->spec.id < b->spec.id ? -1 : a->spec.id > b->spec.id ? 1 : 0;
}

/* victim_order, instance.cpp:151-179, restated literally (scan + sort). */
typedef struct {
    const cand_t* c;
    const req_t* reqs;
    int policy, classed;
} vctx_t;
static vctx_t g_v;
static int cmp_victim(const void* A, const void* B) { /* descending priority */
    long ia = *(const long*)A, ib = *(const long*)B;
    const req_t* a = &g_v.reqs[g_v.c[ia].idx];
    const req_t* b = &g_v.reqs[g_v.c[ib].idx];
    if (g_v.policy == PO_FCFS || g_v.policy == PO_ORACLE) {
        if (a->spec.arrival_time != b->spec.arrival_time)
            return a->spec.arrival_time > b->spec.arrival_time ? -1 : 1;
        return a->spec.id > b->spec.id ? -1 : a->spec.id < b->spec.id ? 1 : 0;
    }
    int xa = g_v.classed ? g_v.c[ia].cls : 0, xb = g_v.classed ? g_v.c[ib].cls : 0;
    if (xa != xb) return xa > xb ? -1 : 1;
    if (a->quanta != b->quanta) return a->quanta > b->quanta ? -1 : 1;
    if (a->seq != b->seq) return a->seq > b->seq ? -1 : 1;
    return a->spec.id > b->spec.id ? -1 : a->spec.id < b->spec.id ? 1 : 0;
}
static long victim_order(const cand_t* c, long nc, const req_t* reqs, const char* admitted,
                         const char* evicted, int policy, int classed, int repair,
                         int admitting_cls, long admitting_idx, long* out) {
    long nv = 0;
    for (long i = 0; i < nc; ++i) {
        if (admitted[i] || i == admitting_idx) continue;
        const req_t* r = &reqs[c[i].idx];
        if (!gpu_resident(r) || r->kv == 0 || evicted[c[i].idx]) continue;
        if (!repair && classed) {
            int ev = c[i].cls == 1 || (admitting_cls == 0 && r->quanta > 0);
            if (admitting_cls == 1 && c[i].cls == 0) ev = 0;
            if (!ev) continue;
        }
        out[nv++] = i;
    }
    g_v.c = c;
    g_v.reqs = reqs;
    g_v.policy = policy;
    g_v.classed = classed;
    qsort(out, (size_t)nv, sizeof(long), cmp_victim);
    return nv;
}

/* plan_iteration, instance.cpp:103-282. */
static void plan_iteration(sim_t* s, int ii, plan_t* plan) {
    inst_t* st = &s->inst[ii];
    const req_t* reqs = s->reqs;
    int policy = s->policy;
    int classed = policy == PO_PASCAL;
    memset(plan, 0, sizeof(*plan));
    plan->prefill_request = -1;

    long nc = 0;
    cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)(st->hi.n + st->lo.n + 1));
    for (long k = 0; k < st->hi.n; ++k)
        if (is_candidate(&reqs[st->hi.v[k]])) c[nc++] = (cand_t){st->hi.v[k], 0};
    for (long k = 0; k < st->lo.n; ++k)
        if (is_candidate(&reqs[st->lo.v[k]])) c[nc++] = (cand_t){st->lo.v[k], 1};
    g_reqs = reqs;
    g_classed = classed;
    qsort(c, (size_t)nc, sizeof(cand_t),
          (policy == PO_FCFS || policy == PO_ORACLE) ? cmp_arrival : cmp_rr);

    long free_ = st->cap - st->gpu;
    char* admitted = (char*)calloc((size_t)nc + 1, 1);
    char* evicted = (char*)calloc((size_t)s->n + 1, 1);
    long* vs = (long*)malloc(sizeof(long) * (size_t)(nc + 1));
    int fcfs_blocked = 0, any_admitted = 0;

    for (long i = 0; i < nc; ++i) {
        const req_t* r = &reqs[c[i].idx];
        if ((fcfs_blocked && !(gpu_resident(r) && r->kv > 0)) || evicted[c[i].idx]) {
            lv_push(&plan->denied, c[i].idx);
            continue;
        }
        long need = admission_need(r);
        if (need > free_) {
            int allow = policy != PO_ORACLE && !(policy == PO_FCFS && r->phase == PH_WAIT);
            if (allow) {
                long nv = victim_order(c, nc, reqs, admitted, evicted, policy, classed, 0,
                                       c[i].cls, i, vs);
                for (long k = 0; k < nv; ++k) {
                    if (need <= free_) break;
                    free_ += reqs[c[vs[k]].idx].kv;
                    evicted[c[vs[k]].idx] = 1;
                    lv_push(&plan->evictions, c[vs[k]].idx);
                }
                if (need > free_ && !any_admitted) { /* deadlock breaker :211-220 */
                    nv = victim_order(c, nc, reqs, admitted, evicted, policy, classed, 1,
                                      c[i].cls, i, vs);
                    for (long k = 0; k < nv; ++k) {
                        if (need <= free_) break;
                        if (evicted[c[vs[k]].idx]) continue;
                        free_ += reqs[c[vs[k]].idx].kv;
                        evicted[c[vs[k]].idx] = 1;
                        lv_push(&plan->evictions, c[vs[k]].idx);
                    }
                }
            }
        }
        if (need <= free_) {
            admitted[i] = 1;
            any_admitted = 1;
            free_ -= need;
        } else {
            lv_push(&plan->denied, c[i].idx);
            if (policy == PO_FCFS) fcfs_blocked = 1;
        }
    }
    if (free_ < 0) { /* over-capacity repair :235-243 */
        long nv = victim_order(c, nc, reqs, admitted, evicted, policy, classed, 1, 0, nc, vs);
        for (long k = 0; k < nv; ++k) {
            if (free_ >= 0) break;
            free_ += reqs[c[vs[k]].idx].kv;
            evicted[c[vs[k]].idx] = 1;
            lv_push(&plan->evictions, c[vs[k]].idx);
        }
    }
    /* materialise :247-281 */
    long total_kv = 0;
    for (long i = 0; i < nc; ++i) {
        if (!admitted[i]) continue;
        const req_t* r = &reqs[c[i].idx];
        if (r->phase == PH_WAIT) {
            if (plan->prefill_request < 0) plan->prefill_request = c[i].idx;
            continue;
        }
        if (gpu_resident(r)) {
            lv_push(&plan->batch, c[i].idx);
            total_kv += r->kv;
        } else if (swap_latency(s->prof, r->kv) == 0.0) {
            lv_push(&plan->immediate, c[i].idx);
            lv_push(&plan->batch, c[i].idx);
            total_kv += r->kv;
        } else {
            lv_push(&plan->swap_ins, c[i].idx);
        }
    }
    if (plan->prefill_request >= 0) {
        plan->kind = 1;
        plan->batch.n = 0;
        plan->duration = prefill_latency(s->prof, reqs[plan->prefill_request].spec.prompt_tokens);
    } else if (plan->batch.n > 0) {
        plan->kind = 2;
        plan->duration = decode_step_latency(s->prof, plan->batch.n, total_kv);
    } else {
        plan->kind = 0;
    }
    free(c);
    free(admitted);
    free(evicted);
    free(vs);
}

static void plan_free(plan_t* p) {
    free(p->batch.v);
    free(p->swap_ins.v);
    free(p->immediate.v);
    free(p->evictions.v);
    free(p->denied.v);
}

/* ------------------------------------------------------------------ engine */
static void note_peak(sim_t* s) { /* engine.cpp:75-79 */
    long total = 0;
    for (int i = 0; i < s->cfg->instance_count; ++i) total += s->inst[i].gpu;
    if (total > s->peak) s->peak = total;
}
static void enqueue(sim_t* s, int i, long idx, int high) { /* engine.cpp:111-116 */
    s->reqs[idx].owner = i;
    s->reqs[idx].seq = ++s->enq_counter;
    lv_push(high ? &s->inst[i].hi : &s->inst[i].lo, idx);
}
static void dequeue(sim_t* s, long idx) { /* engine.cpp:122-126 */
    inst_t* st = &s->inst[s->reqs[idx].owner];
    lv_remove(&st->hi, idx);
    lv_remove(&st->lo, idx);
}
static void free_memory(sim_t* s, long idx) { /* engine.cpp:128-133 */
    req_t* r = &s->reqs[idx];
    inst_t* st = &s->inst[r->owner];
    if (r->loc == LOC_GPU || r->swin) st->gpu -= r->kv;
    else if (r->loc == LOC_CPU) st->cpu -= r->kv;
}
static void finish_request(sim_t* s, long idx) { /* engine.cpp:135-146 */
    req_t* r = &s->reqs[idx];
    po_record* rc = &s->recs[idx];
    free_memory(s, idx);
    dequeue(s, idx);
    r->phase = PH_DONE;
    rc->completion = s->now;
    ++s->done;
    emit(s, "finish", r->owner, idx, "");
}
static void deliver_answer_token(sim_t* s, long idx, double iter_start) { /* :148-156 */
    req_t* r = &s->reqs[idx];
    long k = r->deliv.n;
    pacer_deliver(r, s->now, s->cfg->target_tpot);
    if (k == 0) {
        s->recs[idx].first_answer_delivery = s->now;
        s->recs[idx].first_answer_iter_start = iter_start;
    }
}
static void all_snapshots(sim_t* s, snap_t* out) { /* engine.cpp:103-109 */
    for (int i = 0; i < s->cfg->instance_count; ++i) out[i] = monitor_snapshot(s, i);
}
static void phase_transition(sim_t* s, long idx) { /* engine.cpp:159-190 */
    req_t* r = &s->reqs[idx];
    r->phase = PH_ANSWER;
    s->recs[idx].reasoning_end = s->now;
    emit(s, "transition", r->owner, idx, "");
    if (s->policy != PO_PASCAL) return;
    int cur = r->owner;
    dequeue(s, idx);
    int ni = s->cfg->instance_count;
    snap_t* sn = (snap_t*)malloc(sizeof(snap_t) * (size_t)ni);
    all_snapshots(s, sn);
    int target = select_answering(sn, ni);
    int mig = decide_migration(&sn[cur], &sn[target], r->kv, s->cfg);
    free(sn);
    if (!mig || target == cur) {
        r->qused = 0;
        r->quanta = 0;
        enqueue(s, cur, idx, 0);
        return;
    }
    free_memory(s, idx);
    r->loc = LOC_TRANSIT;
    r->owner = target;
    double dur = transfer_latency(s->prof, r->kv);
    double start = s->now > s->link_busy[target] ? s->now : s->link_busy[target]; /* cluster.cpp:64-68 */
    s->link_busy[target] = start + dur;
    double finish = s->link_busy[target];
    po_record* rc = &s->recs[idx];
    rc->mig = (double*)realloc(rc->mig, sizeof(double) * (size_t)(2 * (rc->n_mig + 1)));
    rc->mig[2 * rc->n_mig] = s->now;
    rc->mig[2 * rc->n_mig + 1] = finish;
    rc->n_mig++;
    push_event(s, finish, EV_TRANSFER, target, idx);
    char d[64];
    snprintf(d, sizeof d, "to=%d", target);
    emit(s, "migrate", cur, idx, d);
}
static void apply_demotion(sim_t* s, int i) { /* instance.cpp:39-57 + engine.cpp:195-198 */
    inst_t* st = &s->inst[i];
    long w = 0;
    long n = st->hi.n;
    long* dem = (long*)malloc(sizeof(long) * (size_t)(n + 1));
    long nd = 0;
    for (long k = 0; k < n; ++k) {
        long idx = st->hi.v[k];
        req_t* r = &s->reqs[idx];
        if (r->kv > s->cfg->demotion_threshold) {
            dem[nd++] = idx;
            r->demoted = 1;
            r->qused = 0;
            r->quanta = 0;
            r->seq = ++s->enq_counter;
            lv_push(&st->lo, idx);
        } else {
            st->hi.v[w++] = idx;
        }
    }
    st->hi.n = w;
    for (long k = 0; k < nd; ++k) emit(s, "demote", i, dem[k], "");
    free(dem);
}
static void maybe_start(sim_t* s, int i) { /* engine.cpp:192-258 */
    inst_t* st = &s->inst[i];
    if (st->busy || s->failed) return;
    if (s->policy == PO_PASCAL) apply_demotion(s, i);
    plan_t plan;
    plan_iteration(s, i, &plan);
    for (long k = 0; k < plan.evictions.n; ++k) {
        long v = plan.evictions.v[k];
        req_t* r = &s->reqs[v];
        st->gpu -= r->kv;
        st->cpu += r->kv;
        r->loc = LOC_CPU;
        double dur = swap_latency(s->prof, r->kv);
        if (dur > 0.0) {
            r->swout = 1;
            push_event(s, s->now + dur, EV_SWAP, i, v);
        }
        emit(s, "evict", i, v, "");
    }
    for (long k = 0; k < plan.swap_ins.n; ++k) {
        long v = plan.swap_ins.v[k];
        req_t* r = &s->reqs[v];
        st->cpu -= r->kv;
        st->gpu += r->kv;
        r->swin = 1;
        push_event(s, s->now + swap_latency(s->prof, r->kv), EV_SWAP, i, v);
        emit(s, "swap_in", i, v, "");
    }
    for (long k = 0; k < plan.immediate.n; ++k) {
        long v = plan.immediate.v[k];
        req_t* r = &s->reqs[v];
        st->cpu -= r->kv;
        st->gpu += r->kv;
        r->loc = LOC_GPU;
        emit(s, "swap_in", i, v, "");
    }
    for (long k = 0; k < plan.denied.n; ++k) {
        s->recs[plan.denied.v[k]].blocked_interval_total += plan.duration;
        emit(s, "block", i, plan.denied.v[k], "");
    }
    if (plan.kind == 1) {
        req_t* r = &s->reqs[plan.prefill_request];
        long extra = r->spec.reasoning_tokens == 0 ? 1 : 0;
        st->gpu += r->spec.prompt_tokens + extra;
        st->busy = 1;
        st->iter_start = s->now;
        st->iter_dur = plan.duration;
        st->batch.n = 0;
        push_event(s, s->now + plan.duration, EV_PREFILL, i, plan.prefill_request);
        emit(s, "prefill_start", i, plan.prefill_request, "");
    } else if (plan.kind == 2) {
        st->gpu += plan.batch.n;
        st->busy = 1;
        st->iter_start = s->now;
        st->iter_dur = plan.duration;
        st->batch.n = 0;
        for (long k = 0; k < plan.batch.n; ++k) lv_push(&st->batch, plan.batch.v[k]);
        push_event(s, s->now + plan.duration, EV_ITER, i, -1);
        char d[64];
        snprintf(d, sizeof d, "batch=%ld", plan.batch.n);
        emit(s, "decode_start", i, -1, d);
    }
    if (st->gpu > st->cap) fail(s, "instance over GPU capacity");
    note_peak(s);
    plan_free(&plan);
}
static void on_arrival(sim_t* s, long idx) { /* engine.cpp:260-283 */
    req_t* r = &s->reqs[idx];
    s->recs[idx].arrival = s->now;
    int ni = s->cfg->instance_count;
    snap_t* sn = (snap_t*)malloc(sizeof(snap_t) * (size_t)ni);
    all_snapshots(s, sn);
    int dst = s->policy == PO_PASCAL ? select_reasoning(sn, ni) : argmin_by(sn, ni, 0, 0);
    free(sn);
    emit(s, "arrival", dst, idx, "");
    if (r->spec.kv_preloaded) {
        r->kv = r->spec.prompt_tokens;
        r->loc = LOC_CPU;
        s->inst[dst].cpu += r->kv;
        s->recs[idx].prefill_complete = s->now;
        if (r->spec.reasoning_tokens > 0) {
            r->phase = PH_REASON;
            enqueue(s, dst, idx, 1);
        } else {
            r->phase = PH_ANSWER;
            s->recs[idx].reasoning_end = s->now;
            enqueue(s, dst, idx, s->policy == PO_PASCAL ? 0 : 1);
        }
    } else {
        r->phase = PH_WAIT;
        enqueue(s, dst, idx, 1);
    }
    maybe_start(s, dst);
}
static void on_prefill_complete(sim_t* s, int i, long idx) { /* engine.cpp:285-308 */
    inst_t* st = &s->inst[i];
    st->busy = 0;
    req_t* r = &s->reqs[idx];
    long extra = r->spec.reasoning_tokens == 0 ? 1 : 0;
    r->kv = r->spec.prompt_tokens + extra;
    s->recs[idx].prefill_complete = s->now;
    emit(s, "prefill_complete", i, idx, "");
    if (r->spec.reasoning_tokens == 0) {
        r->tokens = 1;
        s->recs[idx].reasoning_end = s->now;
        deliver_answer_token(s, idx, st->iter_start);
        if (r->tokens == r->spec.answering_tokens) {
            r->phase = PH_ANSWER;
            finish_request(s, idx);
        } else {
            phase_transition(s, idx);
        }
    } else {
        r->phase = PH_REASON;
    }
    maybe_start(s, i);
}
static void on_iteration_complete(sim_t* s, int i) { /* engine.cpp:310-337 */
    inst_t* st = &s->inst[i];
    st->busy = 0;
    long nb = st->batch.n;
    long* batch = (long*)malloc(sizeof(long) * (size_t)(nb + 1));
    memcpy(batch, st->batch.v, sizeof(long) * (size_t)nb);
    st->batch.n = 0;
    int use_quanta = s->policy == PO_RR || s->policy == PO_PASCAL;
    for (long k = 0; k < nb; ++k) {
        long idx = batch[k];
        req_t* r = &s->reqs[idx];
        r->tokens += 1;
        r->kv += 1;
        emit(s, "token", i, idx, "");
        if (use_quanta) {
            r->qused += 1;
            if (r->qused >= s->cfg->token_quantum) {
                r->qused = 0;
                r->quanta += 1;
            }
        }
        if (r->phase == PH_REASON) {
            if (r->tokens == r->spec.reasoning_tokens) phase_transition(s, idx);
        } else if (r->phase == PH_ANSWER) {
            deliver_answer_token(s, idx, st->iter_start);
            if (r->tokens == r->spec.reasoning_tokens + r->spec.answering_tokens)
                finish_request(s, idx);
        }
    }
    free(batch);
    maybe_start(s, i);
}
static void on_swap_complete(sim_t* s, int i, long idx) { /* engine.cpp:339-349 */
    req_t* r = &s->reqs[idx];
    if (r->swout) r->swout = 0;
    else if (r->swin) {
        r->swin = 0;
        r->loc = LOC_GPU;
    }
    emit(s, "swap_complete", i, idx, "");
    maybe_start(s, i);
}
static void on_transfer_complete(sim_t* s, int dst, long idx) { /* engine.cpp:351-367 */
    req_t* r = &s->reqs[idx];
    inst_t* st = &s->inst[dst];
    if (st->cap - st->gpu >= r->kv) {
        st->gpu += r->kv;
        r->loc = LOC_GPU;
    } else {
        st->cpu += r->kv;
        r->loc = LOC_CPU;
    }
    r->qused = 0;
    r->quanta = 0;
    enqueue(s, dst, idx, 0);
    emit(s, "transfer_complete", dst, idx, "");
    note_peak(s);
    maybe_start(s, dst);
}

/* ---------------------------------------------------------------- validate */
static int validate_trace(const po_spec* t, long n, char* err, size_t errlen) {
    /* workload.cpp:200-219; the id set is an open-addressing hash table */
    double prev_a = -1.0;
    long prev_id = -1;
    size_t hcap = 16;
    while (hcap < (size_t)n * 2 + 2) hcap <<= 1;
    long* seen = (long*)malloc(hcap * sizeof(long));
    for (size_t k = 0; k < hcap; ++k) seen[k] = -1;
    for (long i = 0; i < n; ++i) {
        const po_spec* r = &t[i];
        const char* what = NULL;
        int dup = 0;
        if (r->id >= 0) {
            size_t h = ((uint64_t)r->id * 0x9E3779B97F4A7C15ull) & (hcap - 1);
            while (seen[h] >= 0 && seen[h] != r->id) h = (h + 1) & (hcap - 1);
            if (seen[h] == r->id) dup = 1;
            else seen[h] = r->id;
        }
        if (r->id < 0) what = "id must be non-negative";
        else if (r->arrival_time < 0.0) what = "arrival_time must be >= 0";
        else if (r->prompt_tokens < 1) what = "prompt_tokens must be >= 1";
        else if (r->reasoning_tokens < 0) what = "reasoning_tokens must be >= 0";
        else if (r->answering_tokens < 1) what = "answering_tokens must be >= 1";
        else if (dup) what = "duplicate id";
        else if (r->arrival_time < prev_a || (r->arrival_time == prev_a && r->id < prev_id))
            what = "trace not sorted by (arrival_time, id)";
        if (what) {
            snprintf(err, errlen, "%s (request %ld)", what, r->id);
            free(seen);
            return 1;
        }
        prev_a = r->arrival_time;
        prev_id = r->id;
    }
    free(seen);
    return 0;
}
static int validate_profile(const po_profile* p, char* err, size_t errlen) { /* costmodel.cpp:21-33 */
    const char* bad = NULL;
    if (!(p->prefill_base >= 0.0)) bad = "prefill_base must be >= 0";
    else if (!(p->prefill_per_token >= 0.0)) bad = "prefill_per_token must be >= 0";
    else if (!(p->decode_base >= 0.0)) bad = "decode_base must be >= 0";
    else if (!(p->decode_per_request >= 0.0)) bad = "decode_per_request must be >= 0";
    else if (!(p->decode_per_kv_token >= 0.0)) bad = "decode_per_kv_token must be >= 0";
    else if (!(p->fabric_latency >= 0.0)) bad = "fabric_latency must be >= 0";
    else if (!(p->swap_bandwidth > 0.0)) bad = "swap_bandwidth must be > 0";
    else if (!(p->fabric_bandwidth > 0.0)) bad = "fabric_bandwidth must be > 0";
    if (bad) {
        snprintf(err, errlen, "%s", bad);
        return 1;
    }
    return 0;
}

/* -------------------------------------------------------------------- run */
static int cmp_rec_id(const void* A, const void* B) {
    long a = ((const po_record*)A)->spec.id, b = ((const po_record*)B)->spec.id;
    return a < b ? -1 : a > b;
}

static int sim_run(const po_spec* trace, long n, const po_config* cfg, const po_profile* prof,
                   int policy, long capacity, FILE* log, po_record** out, long* peak_out,
                   char* err, size_t errlen) { /* engine.cpp:369-432 */
    sim_t s;
    memset(&s, 0, sizeof s);
    s.trace = trace;
    s.n = n;
    s.cfg = cfg;
    s.prof = prof;
    s.policy = policy;
    s.log = log;
    s.err = err;
    s.errlen = errlen;
    int ni = cfg->instance_count;
    s.inst = (inst_t*)calloc((size_t)ni, sizeof(inst_t));
    s.link_busy = (double*)calloc((size_t)ni, sizeof(double));
    for (int i = 0; i < ni; ++i) {
        s.inst[i].id = i;
        s.inst[i].cap = capacity;
    }
    s.reqs = (req_t*)calloc((size_t)n + 1, sizeof(req_t));
    s.recs = (po_record*)calloc((size_t)n + 1, sizeof(po_record));
    for (long i = 0; i < n; ++i) {
        s.reqs[i].spec = trace[i];
        s.reqs[i].owner = -1;
        s.recs[i].spec = trace[i];
        push_event(&s, trace[i].arrival_time, EV_ARRIVAL, -1, i);
    }
    if (log) fprintf(log, "pascal-events-v1\n");
    while (s.hn > 0 && !s.failed) {
        event_t ev = pop_event(&s);
        if (ev.time < s.now - 1e-12) {
            fail(&s, "clock moved backwards");
            break;
        }
        if (ev.time > s.now) s.now = ev.time;
        switch (ev.kind) {
            case EV_ARRIVAL: on_arrival(&s, ev.req); break;
            case EV_PREFILL: on_prefill_complete(&s, ev.inst, ev.req); break;
            case EV_ITER: on_iteration_complete(&s, ev.inst); break;
            case EV_SWAP: on_swap_complete(&s, ev.inst, ev.req); break;
            case EV_TRANSFER: on_transfer_complete(&s, ev.inst, ev.req); break;
        }
    }
    if (!s.failed && s.done != n) fail(&s, "simulation stalled with unfinished requests");
    int rc = s.failed ? 3 : 0;
    for (long i = 0; i < n; ++i) {
        po_record* r = &s.recs[i];
        r->n_del = s.reqs[i].deliv.n;
        r->delivery = s.reqs[i].deliv.v;
        r->n_dig = s.reqs[i].digest.n;
        r->digest = s.reqs[i].digest.v;
    }
    for (int i = 0; i < ni; ++i) {
        free(s.inst[i].hi.v);
        free(s.inst[i].lo.v);
        free(s.inst[i].batch.v);
    }
    free(s.inst);
    free(s.link_busy);
    free(s.heap);
    free(s.reqs);
    if (peak_out) *peak_out = s.peak;
    if (rc == 0 && out) {
        qsort(s.recs, (size_t)n, sizeof(po_record), cmp_rec_id);
        *out = s.recs;
    } else {
        po_records_free(s.recs, n);
    }
    return rc;
}

int po_derive_capacity(const po_spec* trace, long n, const po_config* cfg,
                       const po_profile* prof, long* out, char* err, size_t errlen) {
    /* engine.cpp:449-471 */
    if (cfg->instance_count < 1) {
        snprintf(err, errlen, "instance_count must be >= 1");
        return 1;
    }
    long biggest = 0;
    for (long i = 0; i < n; ++i) {
        long m = trace[i].prompt_tokens + trace[i].reasoning_tokens + trace[i].answering_tokens;
        if (m > biggest) biggest = m;
    }
    if (cfg->gpu_capacity > 0) {
        *out = cfg->gpu_capacity > biggest ? cfg->gpu_capacity : biggest;
        return 0;
    }
    long peak = 0;
    int rc = sim_run(trace, n, cfg, prof, PO_ORACLE, LONG_MAX / 4, NULL, NULL, &peak, err, errlen);
    if (rc) return rc;
    double fraction = cfg->capacity_fraction > 0.0 ? cfg->capacity_fraction : 1.0;
    long cap = (long)ceil(fraction * (double)peak / (double)cfg->instance_count);
    *out = cap > biggest ? cap : biggest;
    return 0;
}

int po_run(const po_spec* trace, long n, const po_config* cfg, const po_profile* prof,
           FILE* log, po_record** out, char* err, size_t errlen) { /* engine.cpp:437-447 */
    if (validate_trace(trace, n, err, errlen)) return 1;
    if (validate_profile(prof, err, errlen)) return 1;
    long capacity = LONG_MAX / 4;
    if (cfg->policy != PO_ORACLE) {
        int rc = po_derive_capacity(trace, n, cfg, prof, &capacity, err, errlen);
        if (rc) return rc;
    } else if (cfg->instance_count < 1) {
        snprintf(err, errlen, "instance_count must be >= 1");
        return 1;
    }
    return sim_run(trace, n, cfg, prof, cfg->policy, capacity, log, out, NULL, err, errlen);
}

void po_records_free(po_record* recs, long n) {
    if (!recs) return;
    for (long i = 0; i < n; ++i) {
        free(recs[i].mig);
        free(recs[i].delivery);
        free(recs[i].digest);
    }
    free(recs);
}

void po_dump_records(const po_record* recs, long n, FILE* f) {
    for (long i = 0; i < n; ++i) {
        const po_record* r = &recs[i];
        fprintf(f, "R %ld %a %a %a %a %a %a %a %ld", r->spec.id, r->arrival, r->prefill_complete,
                r->reasoning_end, r->first_answer_delivery, r->first_answer_iter_start,
                r->blocked_interval_total, r->completion, r->n_mig);
        for (long k = 0; k < r->n_mig; ++k) fprintf(f, " %a %a", r->mig[2 * k], r->mig[2 * k + 1]);
        fprintf(f, " %ld", r->n_del);
        for (long k = 0; k < r->n_del; ++k) fprintf(f, " %a", r->delivery[k]);
        fprintf(f, " %ld", r->n_dig);
        for (long k = 0; k < r->n_dig; ++k) fprintf(f, " %a", r->digest[k]);
        fprintf(f, "\n");
    }
}

/* ----------------------------------------------------------------- metrics */
double po_qoe(const po_record* r, double tpot) { /* metrics.cpp:38-52 */
    long n = r->spec.answering_tokens;
    if (n < 1 || r->n_dig == 0) return 1.0;
    double t0 = r->first_answer_delivery;
    double horizon = r->digest[r->n_dig - 1];
    if (horizon <= t0) return 1.0;
    double da = 0.0;
    for (long k = 0; k < r->n_dig; ++k) {
        double d = horizon - r->digest[k];
        da += d > 0.0 ? d : 0.0;
    }
    double ea = 0.0;
    for (long k = 0; k < n; ++k) {
        double d = horizon - (t0 + (double)k * tpot);
        ea += d > 0.0 ? d : 0.0;
    }
    if (ea <= 0.0) return 1.0;
    return da / ea;
}

double po_blocking_latency(const po_record* r) { /* metrics.cpp:58-68 */
    double lo = r->reasoning_end, hi = r->first_answer_iter_start, mig = 0.0;
    for (long k = 0; k < r->n_mig; ++k) {
        double a = r->mig[2 * k] > lo ? r->mig[2 * k] : lo;
        double b = r->mig[2 * k + 1] < hi ? r->mig[2 * k + 1] : hi;
        if (b > a) mig += b - a;
    }
    double v = hi - lo - mig;
    return v > 0.0 ? v : 0.0;
}
