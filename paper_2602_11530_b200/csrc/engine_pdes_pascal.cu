// The instance-parallel engine specialised to Pascal batches, see engine_pdes.cuh.
#define PB_LOG 0
#define PB_PDES 1
#define PB_VARIANT pdes_pascal
#define PB_ONLY_POLICY 3  // pb::kPascal
#include "engine.cu"
