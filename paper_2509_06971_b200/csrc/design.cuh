// design.cuh -- design-subsystem kernels (placeholder until the device loop lands).
#pragma once

#include "context.hpp"

namespace petto_b200 {

inline void design_free(petto_ctx* ctx) {
    cudaFree(ctx->phases);
    cudaFree(ctx->gc);
    cudaFree(ctx->scratch1);
    cudaFree(ctx->scratch2);
    cudaFree(ctx->region_dev);
    ctx->phases = ctx->gc = ctx->scratch1 = ctx->scratch2 = nullptr;
    ctx->region_dev = nullptr;
}

}  // namespace petto_b200
