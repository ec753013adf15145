/* oracle_dump — TEST INFRASTRUCTURE. Same CLI/output formats as ref_dump.cpp,
 * but driving the C restatement (pascal_oracle.c) instead of the reference:
 *
 *   oracle_dump run  TRACE.hex CFG RECORDS_OUT EVENTS_OUT|-
 *   oracle_dump capacity TRACE.hex CFG
 *   oracle_dump time TRACE.hex CFG REPEATS
 */
#define _POSIX_C_SOURCE 199309L
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <time.h>

#include "pascal_oracle.h"

static po_spec* read_hex_trace(const char* path, long* n_out) {
    FILE* f = fopen(path, "r");
    if (!f) return NULL;
    char line[512];
    if (!fgets(line, sizeof line, f) || strncmp(line, "pascal-trace-hex-v1", 19) != 0) {
        fclose(f);
        return NULL;
    }
    long cap = 1024, n = 0;
    po_spec* t = (po_spec*)malloc(sizeof(po_spec) * (size_t)cap);
    while (fgets(line, sizeof line, f)) {
        char arr[128];
        po_spec r;
        if (sscanf(line, "%ld %127s %ld %ld %ld %d", &r.id, arr, &r.prompt_tokens,
                   &r.reasoning_tokens, &r.answering_tokens, &r.kv_preloaded) != 6)
            continue;
        r.arrival_time = strtod(arr, NULL);
        if (n == cap) {
            cap *= 2;
            t = (po_spec*)realloc(t, sizeof(po_spec) * (size_t)cap);
        }
        t[n++] = r;
    }
    fclose(f);
    *n_out = n;
    return t;
}

static int read_cfg(const char* path, po_config* c, po_profile* p) {
    po_config_default(c);
    po_profile_default(p);
    FILE* f = fopen(path, "r");
    if (!f) return 1;
    char line[512];
    while (fgets(line, sizeof line, f)) {
        char* eq = strchr(line, '=');
        if (!eq) continue;
        *eq = 0;
        char* k = line;
        char* v = eq + 1;
        v[strcspn(v, "\r\n")] = 0;
        double d = strtod(v, NULL);
        long l = strtol(v, NULL, 10);
        if (!strcmp(k, "instance_count")) c->instance_count = (int)l;
        else if (!strcmp(k, "gpu_capacity")) c->gpu_capacity = l;
        else if (!strcmp(k, "capacity_fraction")) c->capacity_fraction = d;
        else if (!strcmp(k, "token_quantum")) c->token_quantum = l;
        else if (!strcmp(k, "demotion_threshold")) c->demotion_threshold = l;
        else if (!strcmp(k, "policy")) {
            if (!strcmp(v, "fcfs")) c->policy = PO_FCFS;
            else if (!strcmp(v, "rr")) c->policy = PO_RR;
            else if (!strcmp(v, "oracle")) c->policy = PO_ORACLE;
            else if (!strcmp(v, "pascal")) c->policy = PO_PASCAL;
            else return 1;
        } else if (!strcmp(k, "no_migration")) c->no_migration = l != 0;
        else if (!strcmp(k, "non_adaptive")) c->non_adaptive = l != 0;
        else if (!strcmp(k, "target_tpot")) c->target_tpot = d;
        else if (!strcmp(k, "ttfat_target")) c->ttfat_target = d;
        else if (!strcmp(k, "qoe_threshold")) c->qoe_threshold = d;
        else if (!strcmp(k, "pacer_slack_tokens")) c->pacer_slack_tokens = l;
        else if (!strcmp(k, "prefill_base")) p->prefill_base = d;
        else if (!strcmp(k, "prefill_per_token")) p->prefill_per_token = d;
        else if (!strcmp(k, "decode_base")) p->decode_base = d;
        else if (!strcmp(k, "decode_per_request")) p->decode_per_request = d;
        else if (!strcmp(k, "decode_per_kv_token")) p->decode_per_kv_token = d;
        else if (!strcmp(k, "swap_bandwidth")) p->swap_bandwidth = d;
        else if (!strcmp(k, "fabric_bandwidth")) p->fabric_bandwidth = d;
        else if (!strcmp(k, "fabric_latency")) p->fabric_latency = d;
        else return 1;
    }
    fclose(f);
    return 0;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int main(int argc, char** argv) {
    if (argc < 4) {
        fprintf(stderr, "usage: oracle_dump run|capacity|time TRACE.hex CFG ...\n");
        return 2;
    }
    long n = 0;
    po_spec* t = read_hex_trace(argv[2], &n);
    po_config c;
    po_profile p;
    if (!t || read_cfg(argv[3], &c, &p)) {
        fprintf(stderr, "oracle_dump: bad trace or config\n");
        return 2;
    }
    char err[256] = {0};
    if (!strcmp(argv[1], "run") && argc == 6) {
        FILE* log = strcmp(argv[5], "-") ? fopen(argv[5], "w") : NULL;
        po_record* recs = NULL;
        int rc = po_run(t, n, &c, &p, log, &recs, err, sizeof err);
        if (log) fclose(log);
        if (rc) {
            fprintf(stderr, "oracle_dump: %s\n", err);
            return 1;
        }
        FILE* f = fopen(argv[4], "w");
        po_dump_records(recs, n, f);
        fclose(f);
        po_records_free(recs, n);
    } else if (!strcmp(argv[1], "sim")) {
        po_record* recs = NULL;
        if (po_run(t, n, &c, &p, NULL, &recs, err, sizeof err)) {
            fprintf(stderr, "oracle_dump: %s\n", err);
            return 1;
        }
        /* P99 TTFT (nearest rank), SLO-violation rate, mean TTFT (metrics.cpp:115-153) */
        double* tt = (double*)malloc(sizeof(double) * (size_t)(n + 1));
        long viol = 0;
        for (long k = 0; k < n; ++k) {
            tt[k] = recs[k].first_answer_delivery - recs[k].arrival;
            if (po_qoe(&recs[k], c.target_tpot) < c.qoe_threshold) ++viol;
        }
        for (long a = 1; a < n; ++a) { /* insertion sort: small n, test infrastructure */
            double x = tt[a];
            long b = a - 1;
            while (b >= 0 && tt[b] > x) { tt[b + 1] = tt[b]; --b; }
            tt[b + 1] = x;
        }
        double sum = 0.0;
        for (long k = 0; k < n; ++k) sum += tt[k];
        long rank = n ? (long)ceil(0.99 * (double)n) : 1;
        if (rank < 1) rank = 1;
        if (rank > n) rank = n;
        printf("%ld %a %a %a\n", n, n ? tt[rank - 1] : 0.0, n ? (double)viol / (double)n : 0.0,
               n ? sum / (double)n : 0.0);
        free(tt);
        po_records_free(recs, n);
    } else if (!strcmp(argv[1], "capacity")) {
        long cap = 0;
        if (po_derive_capacity(t, n, &c, &p, &cap, err, sizeof err)) {
            fprintf(stderr, "oracle_dump: %s\n", err);
            return 1;
        }
        printf("%ld\n", cap);
    } else if (!strcmp(argv[1], "time") && argc == 5) {
        int reps = atoi(argv[4]);
        double t0 = now_s();
        long cap = 0;
        if (po_derive_capacity(t, n, &c, &p, &cap, err, sizeof err)) {
            fprintf(stderr, "oracle_dump: %s\n", err);
            return 1;
        }
        double t1 = now_s();
        c.gpu_capacity = cap;
        double run_s = 0.0;
        for (int i = 0; i < reps; ++i) {
            po_record* recs = NULL;
            double a = now_s();
            if (po_run(t, n, &c, &p, NULL, &recs, err, sizeof err)) {
                fprintf(stderr, "oracle_dump: %s\n", err);
                return 1;
            }
            run_s += now_s() - a;
            po_records_free(recs, n);
        }
        printf("{\"capacity\": %ld, \"derive_s\": %.6f, \"run_s\": %.6f, \"reps\": %d}\n", cap,
               t1 - t0, run_s / reps, reps);
    } else {
        fprintf(stderr, "oracle_dump: bad arguments\n");
        return 2;
    }
    free(t);
    return 0;
}
