"""B200-native PASCAL scheduling loop (arXiv 2602.11530), drop-in for the
reference's pascal.h path. See DESIGN.md."""
from .api import (  # noqa: F401
    POLICIES,
    PRESETS,
    Batch,
    PascalError,
    Profile,
    Report,
    Trace,
    compare,
    derive_capacity,
    probe_maybe_start,
    probe_select,
    device_available,
    last_timing,
    run,
    run_batch,
    run_config,
    run_dump,
    run_sweep,
    set_device,
)
