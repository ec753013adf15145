// The lean engine specialised to the Oracle policy: the capacity pre-run of
// derive_capacity (proj/src/engine.cpp:449-471) never logs, never records and
// never evicts. See engine.cu.
#define PB_LOG 0
#define PB_VARIANT oracle_lean
#define PB_ONLY_POLICY 2  // pb::kOracle
#include "engine.cu"
