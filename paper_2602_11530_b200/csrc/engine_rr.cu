// The lean engine specialised to the RR policy (batches whose policy
// runs all use it): every policy test folds at compile time. See engine.cu.
#define PB_LOG 0
#define PB_VARIANT rr_lean
#define PB_ONLY_POLICY 1  // pb::kRr
#include "engine.cu"
