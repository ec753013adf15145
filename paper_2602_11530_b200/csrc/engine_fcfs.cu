// The lean engine specialised to the FCFS policy (batches whose policy
// runs all use it): every policy test folds at compile time. See engine.cu.
#define PB_LOG 0
#define PB_VARIANT fcfs_lean
#define PB_ONLY_POLICY 0  // pb::kFcfs
#include "engine.cu"
