// The instance-parallel engine (generic policy), see engine_pdes.cuh.
#define PB_LOG 0
#define PB_PDES 1
#define PB_VARIANT pdes
#include "engine.cu"
