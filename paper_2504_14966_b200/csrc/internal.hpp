// Library-internal helpers shared by the host translation units (not part of the public API).
#ifndef SLOSCHED_INTERNAL_HPP
#define SLOSCHED_INTERNAL_HPP

#include "slosched_b200.hpp"
#include "slosched_gpu.h"

namespace slosched::detail {

// engine contexts from the per-device pool (host.cpp); release only a context whose last call
// succeeded
slo_ctx* acquire_ctx(int device);
void release_ctx(int device, slo_ctx* ctx);
int resolve_device(int requested);
// slo_status -> the reference's exception types (EngineError for CUDA / state failures)
void check(int rc);

}  // namespace slosched::detail

#endif
