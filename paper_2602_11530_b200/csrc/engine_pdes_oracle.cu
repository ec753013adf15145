// The instance-parallel engine specialised to the oracle (the capacity
// pre-run), see engine_pdes.cuh.
#define PB_LOG 0
#define PB_PDES 1
#define PB_VARIANT pdes_oracle
#define PB_ONLY_POLICY 2  // pb::kOracle
#include "engine.cu"
