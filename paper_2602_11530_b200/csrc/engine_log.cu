// The engine with the decision-log writer (pascal_run_dump / pascal_run with
// an event log). See engine.cu.
#define PB_LOG 1
#define PB_VARIANT logging
#include "engine.cu"
