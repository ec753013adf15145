/* pascal_b200.h — additive entry points of libpascal.so (B200 build).
 *
 * None of these exist in the reference; they sit beside the 19 drop-in
 * symbols of pascal.h without changing them (SURVEY.md §8b "Additive
 * extension"). They serve the replica sweep (many independent simulations
 * per GPU, one process per GPU), the parity tests (full per-request records
 * and the decision log in exact-text form) and the benchmark (device-resident
 * batches timed with CUDA events).
 */
#ifndef PASCAL_B200_H
#define PASCAL_B200_H

#include "pascal.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One replica's outcome: metrics::build_report aggregates
 * (proj/src/metrics.cpp:115-153) computed on the device, plus the work
 * counters used for roofline accounting. */
typedef struct {
    double ttft_mean, ttft_p50, ttft_p90, ttft_p95, ttft_p99;
    double slo_violation_rate, ttfat_attainment, throughput;
    long long capacity;            /* resolved per-instance KV capacity */
    long long requests;
    long long request_iterations;  /* prefills + decode participations */
    long long answer_tokens;
    long long events, plans, candidate_visits, health_checks;
    long long slo_violations;
    long long admission_rounds;    /* warp-parallel admission rounds */
    long long admission_slow_steps; /* candidates decided by the exact scalar step */
    int status;                    /* pascal_status of this replica */
    int pad;
    /* time per output token, not a reference output: per request
     * (completion - first answer delivery) / (A - 1) for A > 1 answer tokens;
     * the mean over those requests, and how many there are */
    double tpot_mean;
    long long tpot_requests;
} pascal_summary;

/* One request's latency-model outputs (metrics::RequestRow,
 * proj/include/pascalsim/metrics.hpp:58-67) plus its TPOT. */
typedef struct {
    long id;
    double ttft, ttfat, qoe, blocking_latency;
    double tpot; /* (completion - first answer delivery) / (A - 1); 0 when A <= 1 */
    int slo_violated;
    int pad;
} pascal_request_row;

/* Device-side timing of the most recent batch execution on this thread. */
typedef struct {
    double derive_ms;   /* oracle pre-run (engine.cpp:449-471) */
    double engine_ms;   /* policy run */
    double metrics_ms;  /* per-request metrics + per-replica summary */
    double total_ms;    /* whole device step (CUDA events on the launch stream) */
    double h2d_ms, d2h_ms;
    long long h2d_bytes, d2h_bytes;
    int kernel_launches;
    int instance_parallel; /* policy-run replicas completed by the instance-parallel engine
                              (the rest ran on the warp-per-replica engine) */
} pascal_timing;

typedef struct pascal_batch pascal_batch;

/* Uploads `count` replicas (trace k under cfgs[k] / profiles[k]) to the
 * current device. Inputs are borrowed. */
pascal_status pascal_batch_create(const pascal_trace* const* traces,
                                  const pascal_profile* const* profiles,
                                  const pascal_run_config* cfgs, size_t count,
                                  pascal_batch** out);
/* Runs every replica to completion on the device (capacity derivation,
 * policy run, metrics); inputs stay resident. */
pascal_status pascal_batch_execute(pascal_batch* b);
/* Copies the per-replica summaries to host memory. */
pascal_status pascal_batch_summaries(pascal_batch* b, pascal_summary* out);
void pascal_batch_free(pascal_batch* b);
/* Per-request rows of replica `replica` after an execute, trace order;
 * `out` holds pascal_trace_size(trace of that replica) entries. */
pascal_status pascal_batch_rows(pascal_batch* b, size_t replica, pascal_request_row* out);

/* Sweep reduction on the device: per-group TTFT histograms over every request
 * of the group's replicas (PASCAL_HIST_BINS log-spaced bins over
 * [1e-4, 1e5) s plus an underflow and an overflow bin) and SLO counters
 * {violations, requests}. Groups are assigned once; the histograms are
 * rebuilt by every pascal_batch_execute. */
#define PASCAL_HIST_BINS 128
pascal_status pascal_batch_set_groups(pascal_batch* b, const int* group_of_replica,
                                      int n_groups);
pascal_status pascal_batch_histograms(pascal_batch* b, unsigned long long* hist,
                                      unsigned long long* slo);

/* create + execute + summaries + free: the end-to-end replica-sweep call
 * with host buffers. */
pascal_status pascal_run_batch(const pascal_trace* const* traces,
                               const pascal_profile* const* profiles,
                               const pascal_run_config* cfgs, size_t count,
                               pascal_summary* out);

pascal_status pascal_last_timing(pascal_timing* out);

/* ---- Several GPUs of one process (replicas shard, no
 * data-path collective). Replicas are split into cost-balanced parts
 * (longest-first greedy over predicted work = request-iterations x a
 * per-policy factor, ties to the lowest part; deterministic), one part per
 * listed device, each run as one device batch by its own host thread.
 * devices = NULL / n_devices = 0: the current device only. */
pascal_status pascal_partition_replicas(const pascal_trace* const* traces,
                                        const pascal_run_config* cfgs, size_t count, int n_parts,
                                        int* part_of_replica);
pascal_status pascal_run_batch_devices(const pascal_trace* const* traces,
                                       const pascal_profile* const* profiles,
                                       const pascal_run_config* cfgs, size_t count,
                                       const int* devices, int n_devices, pascal_summary* out);

/* The reference CLI's `pascalsim sweep` (proj/tools/pascalsim_cli.cpp:
 * 299-342) as one device batch: every (policy, capacity fraction) point of
 * the grid is simulated side by side, then <out_dir>/<policy>_f<%.2f>.{
 * requests.csv,summary.txt,bins.csv} and <out_dir>/sweep.csv are written
 * byte-identically to the sequential CLI loop. `base` supplies every other
 * run-config field. */
pascal_status pascal_sweep(const pascal_trace* t, const pascal_profile* p,
                           const pascal_run_config* base, const char* const* policies,
                           size_t n_policies, const double* fractions, size_t n_fractions,
                           const char* out_dir);
/* pascal_sweep with the grid points spread over `devices` (as above);
 * outputs are identical for any device list. */
pascal_status pascal_sweep_devices(const pascal_trace* t, const pascal_profile* p,
                                   const pascal_run_config* base, const char* const* policies,
                                   size_t n_policies, const double* fractions, size_t n_fractions,
                                   const char* out_dir, const int* devices, int n_devices);

/* Parity: per-request records in the hex-float dump format of
 * oracle/ref_dump.cpp (id order) and, when event_log_path is non-NULL, the
 * pascal-events-v1 decision log. */
pascal_status pascal_run_dump(const pascal_trace* t, const pascal_profile* p,
                              const pascal_run_config* cfg, const char* records_path,
                              const char* event_log_path);

/* engine::derive_capacity (proj/src/engine.cpp:449-471), oracle pre-run on
 * the device. */
pascal_status pascal_derive_capacity(const pascal_trace* t, const pascal_profile* p,
                                     const pascal_run_config* cfg, long* out);

/* Lossless trace files (one line per request, arrival as %a). */
pascal_status pascal_trace_load_hex(const char* path, pascal_trace** out);
pascal_status pascal_trace_save_hex(const pascal_trace* t, const char* path);

/* Array views for bindings. */
pascal_status pascal_trace_from_arrays(long n, const long* ids, const double* arrivals,
                                       const long* prompt, const long* reasoning,
                                       const long* answering, const int* preloaded,
                                       pascal_trace** out);
pascal_status pascal_trace_get(const pascal_trace* t, long i, long* id, double* arrival,
                               long* prompt, long* reasoning, long* answering,
                               int* preloaded);
/* Request-iterations of the trace: sum(R + A - [R==0 and not preloaded] +
 * [not preloaded]). */
long long pascal_trace_request_iterations(const pascal_trace* t);

/* Releases every idle device block the library's caching allocator holds
 * (on every device). Blocks in use by live batches are not affected. The
 * idle cache is also bounded by PB_POOL_CACHE_MB (default 16384) per device. */
pascal_status pascal_release_cached_memory(void);

/* ---- Unit-parity seams ------------------------------------------------
 * The reference keeps its planner and placement rules as pure C++ functions
 * that its unit tests drive with hand-built states: instance::apply_demotion
 * + instance::plan_iteration + the plan application in Simulator::maybe_start
 * (proj/src/instance.cpp:39-57,103-282, proj/src/engine.cpp:192-258;
 * fixtures proj/tests/test_instance.cpp:84-306) and
 * cluster::select_instance_reasoning / _answering / route_arrival
 * (proj/src/cluster.cpp:27-44,59-62; proj/tests/test_cluster.cpp:67-107,
 * proj/tests/acceptance.cpp:137-216). The device engine fuses them into its
 * event loop; these entries run the engine's own code (the same inlined
 * planner and the same select_instance) for one step on a hand-built state,
 * on the current device. */

/* RequestState (proj/include/pascalsim/instance.hpp:41-62); request k's id is
 * k and requests must be in arrival order (as a trace is). */
typedef struct {
    double arrival_time;
    long prompt_tokens, reasoning_tokens, answering_tokens;
    int phase;        /* 0 WaitingPrefill, 1 Reasoning, 2 Answering, 4 Done (Phase) */
    int kv_location;  /* 0 Gpu, 1 Cpu, 2 InTransit (KvLocation) */
    int swapping_in, swapping_out;
    long tokens_generated, kv_tokens, quantum_used_in_round, quanta_exhausted;
    unsigned long long enqueue_seq;
} pascal_probe_request;

/* InstanceState (instance.hpp:74-88) of the instance being planned, plus the
 * engine inputs maybe_start reads: policy, demotion threshold, the enqueue
 * counter demotions draw from, and the clock. */
typedef struct {
    const pascal_probe_request* requests;
    long n_requests;
    const long* high_queue;
    long n_high;
    const long* low_queue;
    long n_low;
    long gpu_capacity, gpu_used, cpu_used;
    unsigned long long enqueue_counter;
    long demotion_threshold;
    const char* policy; /* "fcfs" | "rr" | "oracle" | "pascal" */
    double now;
    int candidate_scratch; /* device shared-memory candidate slots (0: all in HBM) */
} pascal_probe_state;

/* What maybe_start did, in the reference's order. List arrays are caller
 * buffers of n_requests entries (NULL to skip); the counts are always set.
 * Completion / swap event times are the times the step pushed
 * (now + duration), as the event queue holds them. */
typedef struct {
    int kind;           /* 0 Idle, 1 Prefill, 2 Decode (IterationPlan::Kind) */
    int over_capacity;  /* "instance over GPU capacity" (engine.cpp:255-256) fired */
    long prefill_request;
    double completion_time; /* PrefillComplete / IterationComplete time; 0 when idle */
    long gpu_used, cpu_used;
    long *demoted, *evictions, *swap_ins, *immediate_swap_ins, *denied, *batch;
    long n_demoted, n_evictions, n_swap_ins, n_immediate_swap_ins, n_denied, n_batch;
    long* swap_event_request;  /* SwapComplete pushes, in push order */
    double* swap_event_time;
    long n_swap_events;
    double* blocked;           /* per request: blocked time this step added */
} pascal_probe_plan;

pascal_status pascal_probe_maybe_start(const pascal_probe_state* st, const pascal_profile* p,
                                       pascal_probe_plan* out);

/* `count` snapshot vectors of n instances each (n <= 32), instance i of
 * vector v at v*n+i: on_track = t_i, key1 = m_i (modes 0, 2) or r_i (mode 1),
 * key2 = a_i (mode 1). mode 0: select_instance_reasoning (Alg. 1), 1:
 * select_instance_answering (Alg. 2), 2: baseline route_arrival (argmin
 * m_i). Writes the chosen instance of every vector to out[v]. */
pascal_status pascal_probe_select(int mode, long count, int n, const unsigned char* on_track,
                                  const long* key1, const long* key2, int* out);

/* One process per GPU: selects the CUDA device for this thread. */
pascal_status pascal_set_device(int device);
/* 1 when a usable CUDA device is present (no kernels are launched). */
int pascal_device_available(void);

#ifdef __cplusplus
}
#endif
#endif /* PASCAL_B200_H */
