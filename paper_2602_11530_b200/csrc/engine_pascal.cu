// The lean engine (no decision log / record arrays) specialised for batches
// whose policy runs are all Pascal (with or without ablations): every policy
// test folds at compile time. See engine.cu.
#define PB_LOG 0
#define PB_VARIANT pascal_lean
#define PB_ONLY_POLICY 3  // pb::kPascal
#include "engine.cu"
