/* pascal_oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's per-iteration scheduling loop
 * (/root/reference/proj/src/{engine,instance,cluster,costmodel,metrics}.cpp).
 * It exists to check the CUDA product path; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. It is deliberately literal (the
 * O(Q^2) victim rescan of proj/src/instance.cpp:151-179 is kept as is) so that
 * it is easy to audit line by line against the reference.
 *
 * Parity pinning: validated against the real reference (oracle/_ref, built by
 * oracle/Makefile from the read-only sources) and against the committed golden
 * fixtures under tests/golden/ (tests/test_oracle.py).
 */
#ifndef PASCAL_ORACLE_H
#define PASCAL_ORACLE_H

#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/include/pascalsim/workload.hpp:14-28 */
typedef struct {
    long id;
    double arrival_time;
    long prompt_tokens;
    long reasoning_tokens;
    long answering_tokens;
    int kv_preloaded;
} po_spec;

/* proj/include/pascalsim/costmodel.hpp:12-21 */
typedef struct {
    double prefill_base, prefill_per_token;
    double decode_base, decode_per_request, decode_per_kv_token;
    double swap_bandwidth, fabric_bandwidth, fabric_latency;
} po_profile;

enum { PO_FCFS = 0, PO_RR = 1, PO_ORACLE = 2, PO_PASCAL = 3 };

/* proj/include/pascalsim/engine.hpp:18-33 */
typedef struct {
    int instance_count;
    long gpu_capacity;
    double capacity_fraction;
    long token_quantum;
    long demotion_threshold;
    int policy;
    int no_migration, non_adaptive;
    double target_tpot, ttfat_target, qoe_threshold;
    long pacer_slack_tokens;
} po_config;

/* proj/include/pascalsim/metrics.hpp:15-28 */
typedef struct {
    po_spec spec;
    double arrival, prefill_complete, reasoning_end, first_answer_delivery,
        first_answer_iter_start, blocked_interval_total, completion;
    long n_mig;
    double* mig; /* 2*n_mig: start,end pairs */
    long n_del;
    double* delivery;
    long n_dig;
    double* digest;
} po_record;

void po_profile_default(po_profile* p);
void po_config_default(po_config* c);

/* Returns 0 on success; on failure a nonzero code (1 invalid argument,
 * 3 internal invariant) and a message in err. *out receives n records sorted
 * by id (free with po_records_free). log may be NULL. */
int po_run(const po_spec* trace, long n, const po_config* cfg, const po_profile* prof,
           FILE* log, po_record** out, char* err, size_t errlen);
int po_derive_capacity(const po_spec* trace, long n, const po_config* cfg,
                       const po_profile* prof, long* out, char* err, size_t errlen);
void po_records_free(po_record* recs, long n);

/* Record dump in the exact text format of oracle/ref_dump.cpp. */
void po_dump_records(const po_record* recs, long n, FILE* f);

/* Per-request metrics, proj/src/metrics.cpp:34-68 */
double po_qoe(const po_record* r, double target_tpot);
double po_blocking_latency(const po_record* r);

#ifdef __cplusplus
}
#endif
#endif
