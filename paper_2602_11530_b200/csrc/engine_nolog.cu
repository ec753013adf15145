// The engine with every decision-log site compiled out (batches, reports,
// the benchmark). See engine.cu.
#define PB_LOG 0
#define PB_VARIANT nolog
#include "engine.cu"
