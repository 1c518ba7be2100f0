// Context accessors shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>

#include "../../include/ebcc_gpu.h"

namespace ebcc {
cudaStream_t ctx_stream(ebcc_ctx* c);
int ctx_device(ebcc_ctx* c);
int ctx_fail(ebcc_ctx* c, int code, const char* msg);
// metrics.cu: per-context scratch, released by ebcc_destroy
void metrics_release(ebcc_ctx* c);
}  // namespace ebcc
