"""ctypes binding of libpascal.so (the C ABI in include/pascal.h + pascal_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (make -C
paper_2602_11530_b200/csrc). Loading fails loudly when it is missing: there is
no Python or CPU implementation of the scheduling loop behind this module.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpascal.so")

OK, INVALID_ARGUMENT, IO, INTERNAL = 0, 1, 2, 3

# Every symbol include/*.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = (
    # pascal.h — the 19 drop-in entry points (reference proj/include/pascal.h:27-102)
    "pascal_last_error", "pascal_trace_load", "pascal_trace_save", "pascal_trace_generate",
    "pascal_trace_mix", "pascal_trace_size", "pascal_trace_free", "pascal_profile_default",
    "pascal_profile_load", "pascal_profile_save", "pascal_profile_set",
    "pascal_profile_calibrate", "pascal_profile_free", "pascal_run_config_init", "pascal_run",
    "pascal_report_load", "pascal_report_summary_value", "pascal_report_free", "pascal_compare",
    # pascal_b200.h — additive extensions
    "pascal_batch_create", "pascal_batch_execute", "pascal_batch_summaries", "pascal_batch_free",
    "pascal_run_batch", "pascal_last_timing", "pascal_run_dump", "pascal_derive_capacity",
    "pascal_trace_load_hex", "pascal_trace_save_hex", "pascal_trace_from_arrays",
    "pascal_trace_get", "pascal_trace_request_iterations", "pascal_set_device",
    "pascal_device_available", "pascal_release_cached_memory", "pascal_batch_set_groups",
    "pascal_batch_histograms",
    "pascal_sweep",
    "pascal_probe_maybe_start", "pascal_probe_select", "pascal_batch_rows",
    "pascal_partition_replicas", "pascal_run_batch_devices", "pascal_sweep_devices",
)
HIST_BINS = 128


class RunConfig(C.Structure):
    """pascal_run_config (reference proj/include/pascal.h:65-78)."""

    _fields_ = [
        ("instance_count", C.c_int),
        ("gpu_capacity", C.c_long),
        ("capacity_fraction", C.c_double),
        ("token_quantum", C.c_long),
        ("demotion_threshold", C.c_long),
        ("policy", C.c_char_p),
        ("no_migration", C.c_int),
        ("non_adaptive", C.c_int),
        ("target_tpot", C.c_double),
        ("ttfat_target", C.c_double),
        ("qoe_threshold", C.c_double),
        ("pacer_slack_tokens", C.c_long),
    ]


class Summary(C.Structure):
    """pascal_summary (include/pascal_b200.h)."""

    _fields_ = [
        ("ttft_mean", C.c_double), ("ttft_p50", C.c_double), ("ttft_p90", C.c_double),
        ("ttft_p95", C.c_double), ("ttft_p99", C.c_double),
        ("slo_violation_rate", C.c_double), ("ttfat_attainment", C.c_double),
        ("throughput", C.c_double),
        ("capacity", C.c_longlong), ("requests", C.c_longlong),
        ("request_iterations", C.c_longlong), ("answer_tokens", C.c_longlong),
        ("events", C.c_longlong), ("plans", C.c_longlong),
        ("candidate_visits", C.c_longlong), ("health_checks", C.c_longlong),
        ("slo_violations", C.c_longlong),
        ("admission_rounds", C.c_longlong), ("admission_slow_steps", C.c_longlong),
        ("status", C.c_int), ("pad", C.c_int),
        ("tpot_mean", C.c_double), ("tpot_requests", C.c_longlong),
    ]


class RequestRow(C.Structure):
    """pascal_request_row (include/pascal_b200.h)."""

    _fields_ = [
        ("id", C.c_long), ("ttft", C.c_double), ("ttfat", C.c_double), ("qoe", C.c_double),
        ("blocking_latency", C.c_double), ("tpot", C.c_double),
        ("slo_violated", C.c_int), ("pad", C.c_int),
    ]


class Timing(C.Structure):
    """pascal_timing (include/pascal_b200.h)."""

    _fields_ = [
        ("derive_ms", C.c_double), ("engine_ms", C.c_double), ("metrics_ms", C.c_double),
        ("total_ms", C.c_double), ("h2d_ms", C.c_double), ("d2h_ms", C.c_double),
        ("h2d_bytes", C.c_longlong), ("d2h_bytes", C.c_longlong),
        ("kernel_launches", C.c_int), ("instance_parallel", C.c_int),
    ]


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libpascal.so (once). Raises if the native library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    _lib = bind(C.CDLL(path))
    return _lib


class ProbeRequest(C.Structure):
    """pascal_probe_request (include/pascal_b200.h; RequestState,
    proj/include/pascalsim/instance.hpp:41-62)."""

    _fields_ = [
        ("arrival_time", C.c_double),
        ("prompt_tokens", C.c_long), ("reasoning_tokens", C.c_long),
        ("answering_tokens", C.c_long),
        ("phase", C.c_int), ("kv_location", C.c_int),
        ("swapping_in", C.c_int), ("swapping_out", C.c_int),
        ("tokens_generated", C.c_long), ("kv_tokens", C.c_long),
        ("quantum_used_in_round", C.c_long), ("quanta_exhausted", C.c_long),
        ("enqueue_seq", C.c_ulonglong),
    ]


class ProbeState(C.Structure):
    """pascal_probe_state (include/pascal_b200.h)."""

    _fields_ = [
        ("requests", C.POINTER(ProbeRequest)), ("n_requests", C.c_long),
        ("high_queue", C.POINTER(C.c_long)), ("n_high", C.c_long),
        ("low_queue", C.POINTER(C.c_long)), ("n_low", C.c_long),
        ("gpu_capacity", C.c_long), ("gpu_used", C.c_long), ("cpu_used", C.c_long),
        ("enqueue_counter", C.c_ulonglong), ("demotion_threshold", C.c_long),
        ("policy", C.c_char_p), ("now", C.c_double), ("candidate_scratch", C.c_int),
    ]


class ProbePlan(C.Structure):
    """pascal_probe_plan (include/pascal_b200.h)."""

    _LISTS = ("demoted", "evictions", "swap_ins", "immediate_swap_ins", "denied", "batch")
    _fields_ = [
        ("kind", C.c_int), ("over_capacity", C.c_int), ("prefill_request", C.c_long),
        ("completion_time", C.c_double), ("gpu_used", C.c_long), ("cpu_used", C.c_long),
    ] + [(k, C.POINTER(C.c_long)) for k in _LISTS] + [
        ("n_" + k, C.c_long) for k in _LISTS] + [
        ("swap_event_request", C.POINTER(C.c_long)),
        ("swap_event_time", C.POINTER(C.c_double)), ("n_swap_events", C.c_long),
        ("blocked", C.POINTER(C.c_double)),
    ]


def bind(lib: C.CDLL, extensions: bool = True) -> C.CDLL:
    """Attach argument/return types for every ABI symbol present in `lib`.
    Also used by the tests on oracle/_ref/libpascal_ref.so (19 symbols only)."""
    P = C.c_void_p
    PP = C.POINTER(C.c_void_p)
    st = C.c_int
    sig = {
        "pascal_last_error": (C.c_char_p, []),
        "pascal_trace_load": (st, [C.c_char_p, PP]),
        "pascal_trace_save": (st, [P, C.c_char_p]),
        "pascal_trace_generate": (st, [C.c_long, C.c_double, C.c_char_p, C.c_char_p, C.c_char_p,
                                       C.c_uint64, C.c_int, PP]),
        "pascal_trace_mix": (st, [P, P, C.c_double, C.c_uint64, PP]),
        "pascal_trace_size": (C.c_long, [P]),
        "pascal_trace_free": (None, [P]),
        "pascal_profile_default": (st, [PP]),
        "pascal_profile_load": (st, [C.c_char_p, PP]),
        "pascal_profile_save": (st, [P, C.c_char_p]),
        "pascal_profile_set": (st, [P, C.c_char_p, C.c_double]),
        "pascal_profile_calibrate": (st, [C.c_char_p, P, C.POINTER(C.c_double)]),
        "pascal_profile_free": (None, [P]),
        "pascal_run_config_init": (None, [C.POINTER(RunConfig)]),
        "pascal_run": (st, [P, P, C.POINTER(RunConfig), C.c_char_p, C.c_char_p]),
        "pascal_report_load": (st, [C.c_char_p, PP]),
        "pascal_report_summary_value": (st, [P, C.c_char_p, C.POINTER(C.c_double)]),
        "pascal_report_free": (None, [P]),
        "pascal_compare": (st, [C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), C.c_size_t,
                                C.c_char_p]),
        "pascal_batch_create": (st, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                     C.POINTER(RunConfig), C.c_size_t, PP]),
        "pascal_batch_execute": (st, [P]),
        "pascal_batch_summaries": (st, [P, C.POINTER(Summary)]),
        "pascal_batch_free": (None, [P]),
        "pascal_batch_rows": (st, [P, C.c_size_t, C.POINTER(RequestRow)]),
        "pascal_partition_replicas": (st, [C.POINTER(C.c_void_p), C.POINTER(RunConfig),
                                           C.c_size_t, C.c_int, C.POINTER(C.c_int)]),
        "pascal_run_batch_devices": (st, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                          C.POINTER(RunConfig), C.c_size_t,
                                          C.POINTER(C.c_int), C.c_int, C.POINTER(Summary)]),
        "pascal_sweep_devices": (st, [P, P, C.POINTER(RunConfig), C.POINTER(C.c_char_p),
                                      C.c_size_t, C.POINTER(C.c_double), C.c_size_t, C.c_char_p,
                                      C.POINTER(C.c_int), C.c_int]),
        "pascal_run_batch": (st, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                  C.POINTER(RunConfig), C.c_size_t, C.POINTER(Summary)]),
        "pascal_last_timing": (st, [C.POINTER(Timing)]),
        "pascal_run_dump": (st, [P, P, C.POINTER(RunConfig), C.c_char_p, C.c_char_p]),
        "pascal_derive_capacity": (st, [P, P, C.POINTER(RunConfig), C.POINTER(C.c_long)]),
        "pascal_trace_load_hex": (st, [C.c_char_p, PP]),
        "pascal_trace_save_hex": (st, [P, C.c_char_p]),
        "pascal_trace_from_arrays": (st, [C.c_long, C.POINTER(C.c_long), C.POINTER(C.c_double),
                                          C.POINTER(C.c_long), C.POINTER(C.c_long),
                                          C.POINTER(C.c_long), C.POINTER(C.c_int), PP]),
        "pascal_trace_get": (st, [P, C.c_long, C.POINTER(C.c_long), C.POINTER(C.c_double),
                                  C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_long),
                                  C.POINTER(C.c_int)]),
        "pascal_trace_request_iterations": (C.c_longlong, [P]),
        "pascal_set_device": (st, [C.c_int]),
        "pascal_device_available": (C.c_int, []),
        "pascal_release_cached_memory": (st, []),
        "pascal_batch_set_groups": (st, [P, C.POINTER(C.c_int), C.c_int]),
        "pascal_batch_histograms": (st, [P, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
        "pascal_sweep": (st, [P, P, C.POINTER(RunConfig), C.POINTER(C.c_char_p), C.c_size_t,
                              C.POINTER(C.c_double), C.c_size_t, C.c_char_p]),
        "pascal_probe_maybe_start": (st, [C.POINTER(ProbeState), P, C.POINTER(ProbePlan)]),
        "pascal_probe_select": (st, [C.c_int, C.c_long, C.c_int, C.POINTER(C.c_ubyte),
                                     C.POINTER(C.c_long), C.POINTER(C.c_long),
                                     C.POINTER(C.c_int)]),
    }
    for name, (res, args) in sig.items():
        if not extensions and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
