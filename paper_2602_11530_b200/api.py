"""Python mirror of the reference's public C interface for the scheduling path.

Names, argument meaning and error behaviour follow /root/reference/proj/
include/pascal.h (trace / profile / run / report / compare), so tests read like
the reference's own (proj/tests/test_capi.cpp). Every call goes through
libpascal.so; simulations run on the GPU (sm_100a kernels in csrc/).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Iterable, List, Optional, Sequence

from . import _lib

POLICIES = ("fcfs", "rr", "oracle", "pascal")

# Length presets of the reference CLI (proj/tools/pascalsim_cli.cpp:41-49).
PRESETS = {
    "reasoning-char": ("constant:128", "uniform:128:2048", "constant:1", False),
    "answering-char": ("constant:128", "constant:0", "uniform:128:2048", True),
    "chat": ("uniform:64:512",
             "hist:256=0.35,512=0.30,768=0.20,1024=0.10,1536=0.04,2048=0.01",
             "uniform:256:1024", False),
    "reasoning-heavy": ("uniform:64:512", "uniform:2048:8192", "uniform:128:512", False),
}


class PascalError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[status {status}] {message}")
        self.status = status
        self.message = message


def _lib_():
    return _lib.load()


def _check(status: int) -> None:
    if status != _lib.OK:
        msg = _lib_().pascal_last_error()
        raise PascalError(status, msg.decode() if msg else "")


def _b(s: Optional[str]) -> Optional[bytes]:
    return None if s is None else os.fsencode(s)


class Trace:
    """Opaque pascal_trace handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib_().pascal_trace_free(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @classmethod
    def generate(cls, count: int, arrival_rate: float, prompt: str, reasoning: str,
                 answering: str, seed: int, kv_preloaded: bool = False) -> "Trace":
        out = C.c_void_p()
        _check(_lib_().pascal_trace_generate(count, arrival_rate, _b(prompt), _b(reasoning),
                                             _b(answering), seed, int(kv_preloaded),
                                             C.byref(out)))
        return cls(out.value)

    @classmethod
    def preset(cls, name: str, count: int, arrival_rate: float, seed: int,
               mix_fraction: float = 0.25) -> "Trace":
        """`pascalsim gen --preset` (proj/tools/pascalsim_cli.cpp:169-222)."""
        if name == "mixed":
            base = cls.preset("chat", count, arrival_rate, seed)
            heavy = cls.preset("reasoning-heavy", count, arrival_rate, seed + 1)
            return cls.mix(base, heavy, mix_fraction, seed + 2)
        p, r, a, pre = PRESETS[name]
        return cls.generate(count, arrival_rate, p, r, a, seed, pre)

    @classmethod
    def mix(cls, base: "Trace", replacement: "Trace", fraction: float, seed: int) -> "Trace":
        out = C.c_void_p()
        _check(_lib_().pascal_trace_mix(base._h, replacement._h, fraction, seed, C.byref(out)))
        return cls(out.value)

    @classmethod
    def load(cls, path: str) -> "Trace":
        out = C.c_void_p()
        _check(_lib_().pascal_trace_load(_b(path), C.byref(out)))
        return cls(out.value)

    @classmethod
    def load_hex(cls, path: str) -> "Trace":
        out = C.c_void_p()
        _check(_lib_().pascal_trace_load_hex(_b(path), C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_arrays(cls, ids, arrivals, prompt, reasoning, answering, preloaded=None) -> "Trace":
        n = len(ids)
        L = C.c_long * n
        D = C.c_double * n
        I = C.c_int * n
        out = C.c_void_p()
        pre = I(*[int(x) for x in preloaded]) if preloaded is not None else None
        _check(_lib_().pascal_trace_from_arrays(
            n, L(*ids), D(*arrivals), L(*prompt), L(*reasoning), L(*answering), pre,
            C.byref(out)))
        return cls(out.value)

    def save(self, path: str) -> None:
        _check(_lib_().pascal_trace_save(self._h, _b(path)))

    def save_hex(self, path: str) -> None:
        _check(_lib_().pascal_trace_save_hex(self._h, _b(path)))

    def __len__(self) -> int:
        return int(_lib_().pascal_trace_size(self._h))

    def request_iterations(self) -> int:
        return int(_lib_().pascal_trace_request_iterations(self._h))

    def specs(self) -> List[tuple]:
        lib = _lib_()
        out = []
        i_, p_, r_, a_ = C.c_long(), C.c_long(), C.c_long(), C.c_long()
        t_ = C.c_double()
        pre = C.c_int()
        for k in range(len(self)):
            _check(lib.pascal_trace_get(self._h, k, C.byref(i_), C.byref(t_), C.byref(p_),
                                        C.byref(r_), C.byref(a_), C.byref(pre)))
            out.append((i_.value, t_.value, p_.value, r_.value, a_.value, bool(pre.value)))
        return out


class Profile:
    """Opaque pascal_profile handle (LatencyProfile, costmodel.hpp:12-21)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib_().pascal_profile_free(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @classmethod
    def default(cls, **fields) -> "Profile":
        out = C.c_void_p()
        _check(_lib_().pascal_profile_default(C.byref(out)))
        p = cls(out.value)
        for k, v in fields.items():
            p.set(k, v)
        return p

    @classmethod
    def load(cls, path: str) -> "Profile":
        out = C.c_void_p()
        _check(_lib_().pascal_profile_load(_b(path), C.byref(out)))
        return cls(out.value)

    def save(self, path: str) -> None:
        _check(_lib_().pascal_profile_save(self._h, _b(path)))

    def set(self, key: str, value: float) -> None:
        _check(_lib_().pascal_profile_set(self._h, _b(key), float(value)))

    def calibrate(self, samples_path: str) -> float:
        rmse = C.c_double()
        _check(_lib_().pascal_profile_calibrate(_b(samples_path), self._h, C.byref(rmse)))
        return rmse.value


def run_config(policy: str = "pascal", **fields) -> _lib.RunConfig:
    """pascal_run_config with the reference defaults (pascal_run_config_init)."""
    cfg = _lib.RunConfig()
    _lib_().pascal_run_config_init(C.byref(cfg))
    cfg.policy = policy.encode()
    for k, v in fields.items():
        if not hasattr(cfg, k):
            raise AttributeError(k)
        setattr(cfg, k, v)
    return cfg


def run(trace: Trace, profile: Profile, cfg, report_prefix: str,
        event_log: Optional[str] = None) -> None:
    """pascal_run: simulate on the GPU, write the pascal-report-v1 files."""
    _check(_lib_().pascal_run(trace.handle, profile.handle, C.byref(cfg), _b(report_prefix),
                              _b(event_log)))


def run_dump(trace: Trace, profile: Profile, cfg, records_path: str,
             event_log: Optional[str] = None) -> None:
    """Full per-request records (hex-float dump) + optional decision log."""
    _check(_lib_().pascal_run_dump(trace.handle, profile.handle, C.byref(cfg),
                                   _b(records_path), _b(event_log)))


def derive_capacity(trace: Trace, profile: Profile, cfg) -> int:
    out = C.c_long()
    _check(_lib_().pascal_derive_capacity(trace.handle, profile.handle, C.byref(cfg),
                                          C.byref(out)))
    return out.value


class Report:
    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib_().pascal_report_free(h)
            self._h = None

    @classmethod
    def load(cls, prefix: str) -> "Report":
        out = C.c_void_p()
        _check(_lib_().pascal_report_load(_b(prefix), C.byref(out)))
        return cls(out.value)

    def summary_value(self, key: str) -> float:
        out = C.c_double()
        _check(_lib_().pascal_report_summary_value(self._h, _b(key), C.byref(out)))
        return out.value


def compare(prefixes: Sequence[str], names: Sequence[str], out_path: str) -> None:
    n = len(prefixes)
    P = C.c_char_p * max(n, 1)
    _check(_lib_().pascal_compare(P(*[_b(p) for p in prefixes]), P(*[_b(x) for x in names]),
                                  n, _b(out_path)))


def _arrays(traces, profiles, cfgs):
    n = len(traces)
    T = C.c_void_p * n
    R = _lib.RunConfig * n
    return n, T(*[t.handle.value for t in traces]), T(*[p.handle.value for p in profiles]), \
        R(*cfgs)


class Batch:
    """Device-resident replica batch (pascal_batch_*)."""

    def __init__(self, traces: Sequence[Trace], profiles: Sequence[Profile], cfgs: Sequence):
        n, tt, pp, cc = _arrays(traces, profiles, cfgs)
        out = C.c_void_p()
        _check(_lib_().pascal_batch_create(tt, pp, cc, n, C.byref(out)))
        self._h = out
        self.n = n

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib_().pascal_batch_free(h)
            self._h = None

    def execute(self) -> None:
        _check(_lib_().pascal_batch_execute(self._h))

    def summaries(self) -> List[_lib.Summary]:
        out = (_lib.Summary * self.n)()
        _check(_lib_().pascal_batch_summaries(self._h, out))
        return list(out)

    def rows(self, replica: int, n_requests: int) -> List[_lib.RequestRow]:
        """Per-request TTFT / TTFAT / QoE / blocking / TPOT of one replica
        (trace order), pascal_batch_rows."""
        out = (_lib.RequestRow * max(n_requests, 1))()
        _check(_lib_().pascal_batch_rows(self._h, replica, out))
        return list(out)[:n_requests]

    def set_groups(self, group_of_replica: Sequence[int], n_groups: int) -> None:
        self.n_groups = n_groups
        arr = (C.c_int * self.n)(*group_of_replica)
        _check(_lib_().pascal_batch_set_groups(self._h, arr, n_groups))

    def histograms(self):
        """(hist[n_groups][HIST_BINS + 2], slo[n_groups][2]) as nested lists."""
        nb = _lib.HIST_BINS + 2
        h = (C.c_ulonglong * (self.n_groups * nb))()
        s = (C.c_ulonglong * (self.n_groups * 2))()
        _check(_lib_().pascal_batch_histograms(self._h, h, s))
        return ([list(h[g * nb:(g + 1) * nb]) for g in range(self.n_groups)],
                [list(s[2 * g:2 * g + 2]) for g in range(self.n_groups)])


def run_batch(traces, profiles, cfgs) -> List[_lib.Summary]:
    n, tt, pp, cc = _arrays(traces, profiles, cfgs)
    out = (_lib.Summary * n)()
    _check(_lib_().pascal_run_batch(tt, pp, cc, n, out))
    return list(out)


def run_batch_devices(traces, profiles, cfgs, devices: Sequence[int]) -> List[_lib.Summary]:
    """pascal_run_batch over several GPUs of this process (cost-balanced
    replica parts, one host thread per device)."""
    n, tt, pp, cc = _arrays(traces, profiles, cfgs)
    out = (_lib.Summary * n)()
    dv = (C.c_int * max(len(devices), 1))(*devices)
    _check(_lib_().pascal_run_batch_devices(tt, pp, cc, n, dv, len(devices), out))
    return list(out)


def partition_replicas(traces, cfgs, n_parts: int) -> List[int]:
    """pascal_partition_replicas: the device part of every replica (host-only)."""
    n = len(traces)
    tt = (C.c_void_p * n)(*[t.handle.value for t in traces])
    cc = (_lib.RunConfig * n)(*cfgs)
    out = (C.c_int * max(n, 1))()
    _check(_lib_().pascal_partition_replicas(tt, cc, n, n_parts, out))
    return list(out)[:n]


def run_sweep(trace: Trace, profile: Profile, base_cfg, policies: Sequence[str],
              fractions: Sequence[float], out_dir: str,
              devices: Optional[Sequence[int]] = None) -> None:
    """`pascalsim sweep` (proj/tools/pascalsim_cli.cpp:299-342) as device
    batches: per-point reports <out_dir>/<policy>_f<frac>.* and sweep.csv;
    `devices` spreads the grid over several GPUs."""
    pols = (C.c_char_p * len(policies))(*[_b(x) for x in policies])
    fr = (C.c_double * len(fractions))(*fractions)
    dv = (C.c_int * max(len(devices or []), 1))(*(devices or []))
    _check(_lib_().pascal_sweep_devices(trace.handle, profile.handle, C.byref(base_cfg), pols,
                                        len(policies), fr, len(fractions), _b(out_dir), dv,
                                        len(devices or [])))


def last_timing() -> _lib.Timing:
    t = _lib.Timing()
    _check(_lib_().pascal_last_timing(C.byref(t)))
    return t


def set_device(device: int) -> None:
    _check(_lib_().pascal_set_device(device))


def device_available() -> bool:
    return bool(_lib_().pascal_device_available())


# ---- unit-parity seams (pascal_probe_*; include/pascal_b200.h) -----------
PHASES = {"waiting": 0, "reasoning": 1, "answering": 2, "done": 4}
LOCATIONS = {"gpu": 0, "cpu": 1, "transit": 2}


def probe_maybe_start(requests: Sequence[dict], high: Sequence[int], low: Sequence[int],
                      gpu_capacity: int, gpu_used: int = 0, cpu_used: int = 0,
                      policy: str = "pascal", profile: Optional[Profile] = None,
                      enqueue_counter: int = 0, demotion_threshold: int = 5000,
                      now: float = 0.0, candidate_scratch: int = 256) -> dict:
    """One maybe_start step (apply_demotion + plan_iteration + plan application,
    proj/src/engine.cpp:192-258) on a hand-built instance state, run by the
    device engine's planner. `requests[k]` (id k) holds RequestState fields:
    prompt/reasoning/answering, phase ("waiting"|"reasoning"|"answering"|
    "done"), loc ("gpu"|"cpu"|"transit"), swapping_in/out, tokens, kv, qused,
    quanta, seq, arrival (default k)."""
    n = len(requests)
    arr = (_lib.ProbeRequest * max(n, 1))()
    for k, r in enumerate(requests):
        a = arr[k]
        a.arrival_time = float(r.get("arrival", k))
        a.prompt_tokens = r.get("prompt", 1)
        a.reasoning_tokens = r.get("reasoning", 0)
        a.answering_tokens = r.get("answering", 1)
        a.phase = PHASES[r.get("phase", "waiting")]
        a.kv_location = LOCATIONS[r.get("loc", "gpu")]
        a.swapping_in = int(bool(r.get("swapping_in", False)))
        a.swapping_out = int(bool(r.get("swapping_out", False)))
        a.tokens_generated = r.get("tokens", 0)
        a.kv_tokens = r.get("kv", 0)
        a.quantum_used_in_round = r.get("qused", 0)
        a.quanta_exhausted = r.get("quanta", 0)
        a.enqueue_seq = r.get("seq", 0)
    hq = (C.c_long * max(len(high), 1))(*high)
    lq = (C.c_long * max(len(low), 1))(*low)
    st = _lib.ProbeState(arr, n, hq, len(high), lq, len(low), gpu_capacity, gpu_used, cpu_used,
                         enqueue_counter, demotion_threshold, policy.encode(), float(now),
                         candidate_scratch)
    out = _lib.ProbePlan()
    bufs = {}
    for name in _lib.ProbePlan._LISTS + ("swap_event_request",):
        bufs[name] = (C.c_long * max(n, 1))()
        setattr(out, name, bufs[name])
    times = (C.c_double * max(2 * n, 1))()
    blocked = (C.c_double * max(n, 1))()
    evreq = (C.c_long * max(2 * n, 1))()
    out.swap_event_request = evreq
    out.swap_event_time = times
    out.blocked = blocked
    prof = profile if profile is not None else Profile.default()
    _check(_lib_().pascal_probe_maybe_start(C.byref(st), prof.handle, C.byref(out)))
    res = {"kind": ("idle", "prefill", "decode")[out.kind],
           "prefill_request": out.prefill_request, "completion_time": out.completion_time,
           "gpu_used": out.gpu_used, "cpu_used": out.cpu_used,
           "over_capacity": bool(out.over_capacity),
           "swap_events": [(evreq[k], times[k]) for k in range(out.n_swap_events)],
           "blocked": [blocked[k] for k in range(n)]}
    for name in _lib.ProbePlan._LISTS:
        res[name] = [bufs[name][k] for k in range(getattr(out, "n_" + name))]
    return res


def probe_select(mode: int, on_track, key1, key2=None):
    """Alg. 1 (mode 0: select_instance_reasoning), Alg. 2 (mode 1:
    select_instance_answering) or the baseline route (mode 2: argmin m_i) for
    a batch of snapshot vectors, through the device engine's
    select_instance. Arrays are (count, n): on_track t_i, key1 m_i or r_i,
    key2 a_i. Returns the chosen instance per vector (numpy int32)."""
    import numpy as np
    t = np.ascontiguousarray(on_track, dtype=np.uint8)
    count, n = t.shape
    k1 = np.ascontiguousarray(key1, dtype=np.int64)
    k2 = np.ascontiguousarray(key2 if key2 is not None else np.zeros_like(k1), dtype=np.int64)
    out = np.zeros(count, dtype=np.int32)
    _check(_lib_().pascal_probe_select(
        mode, count, n, t.ctypes.data_as(C.POINTER(C.c_ubyte)),
        k1.ctypes.data_as(C.POINTER(C.c_long)), k2.ctypes.data_as(C.POINTER(C.c_long)),
        out.ctypes.data_as(C.POINTER(C.c_int))))
    return out
