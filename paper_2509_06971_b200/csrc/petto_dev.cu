// petto_dev.cu -- C-ABI implementation: device context, uploads, and the state
// solver (hybrid_solve / iterate_to_tolerance / residual) on B200.
//
// Reference seam: include/petto/state_solver.hpp (StateOperator, hybrid_solve,
// iterate_to_tolerance).  Every step loop runs without host synchronisation:
// non-finite detection and the tolerance test are evaluated by the kernels
// themselves through the context's DeviceStatus block.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

#include "comm.hpp"
#include "context.hpp"
#include "design.cuh"
#include "elastic3d.cuh"
#include "fast2d.cuh"
#include "replica.cuh"
#include "stiffness.hpp"
#include "writers.cuh"

#include <cub/device/device_scan.cuh>
#include <nvtx3/nvToolsExt.h>

using namespace petto_b200;

namespace {

thread_local std::string g_err;  // errors before a context exists

int fail(petto_ctx* ctx, int code, const std::string& msg) {
    (ctx ? ctx->err : g_err) = msg;
    return code;
}

#define CK(expr)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess) return fail(ctx, PETTO_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define CKL()                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = cudaGetLastError();                                                  \
        if (e_ != cudaSuccess) return fail(ctx, PETTO_ERROR, std::string("launch: ") + cudaGetErrorString(e_)); \
    } while (0)

long long global_nodes(const petto_ctx* ctx) {
    return (long long)ctx->g.nx * ctx->g.ny * ctx->g.nz;
}

long long owned_nodes(const petto_ctx* ctx) {
    return (long long)ctx->g.nx * ctx->g.ny * (ctx->g.ke - ctx->g.kb);
}

int blocks_for(long long n, int threads = 256) { return (int)std::max(1LL, (n + threads - 1) / threads); }

// launch shape of the z-streamed 3D sensitivity kernel
constexpr int SENS_ZC = 16;
dim3 sens_grid(const petto_ctx* x) {
    const Geo& g = x->g;
    return dim3((g.nx + 31) / 32, (g.ny + 3) / 4, (g.ke - g.kb + SENS_ZC - 1) / SENS_ZC);
}


// ------------------------------------------------- x-outermost permutation
// Host layout x-fastest (grid.hpp:47); device layout of a permuted context: axes
// (y, z, x).  A rank's stored x planes [ks0, ks0 + nzs) of `comps` host components
// sit in the staging buffer as [c][z][y][x - ks0]; these kernels move them to /
// from the pitched device layout with 32 x 32 shared-memory tiles (coalesced on
// both sides).  Host extents: nxh = stored (or owned) x planes, ny = g.nx, nz =
// g.ny.  cperm: device component of host component c is (c + 2) % 3.
__global__ void k_perm_in(Geo g, const double* __restrict__ stage, int nxh, int comps, bool cperm,
                          double* __restrict__ dst) {
    __shared__ double tile[32][33];
    const int z = blockIdx.z;                       // host z = device j
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int c = 0; c < comps; ++c) {
        const double* sc = stage + (long long)c * g.nx * g.ny * nxh;
        double* dc = dst + (long long)(cperm ? (c + 2) % 3 : c) * g.Ns;
        for (int r = ty; r < 32; r += 8) {
            const int y = y0 + r, x = x0 + tx;      // read along host x
            if (y < g.nx && x < nxh) tile[r][tx] = sc[((long long)z * g.nx + y) * nxh + x];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int x = x0 + r, y = y0 + tx;      // write along device x (= host y)
            if (y < g.nx && x < nxh) dc[((long long)x * g.ny + z) * g.px + y] = tile[tx][r];
        }
        __syncthreads();
    }
}

// device planes [k0, k0 + nxh) -> staging [c][z][y][x - k0]
__global__ void k_perm_out(Geo g, const double* __restrict__ src, int k0, int nxh, int comps, bool cperm,
                           double* __restrict__ stage) {
    __shared__ double tile[32][33];
    const int z = blockIdx.z;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int c = 0; c < comps; ++c) {
        const double* sc = src + (long long)(cperm ? (c + 2) % 3 : c) * g.Ns;
        double* dc = stage + (long long)c * g.nx * g.ny * nxh;
        for (int r = ty; r < 32; r += 8) {
            const int x = x0 + r, y = y0 + tx;      // read along device x (= host y)
            if (y < g.nx && x < nxh) tile[r][tx] = sc[((long long)(k0 - g.ks0 + x) * g.ny + z) * g.px + y];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int y = y0 + r, x = x0 + tx;      // write along host x
            if (y < g.nx && x < nxh) dc[((long long)z * g.nx + y) * nxh + x] = tile[tx][r];
        }
        __syncthreads();
    }
}

// staging buffer for the next permuted transfer (alternating between two)
double* stage_reserve(petto_ctx* ctx, size_t elems) {
    if (!ctx->xstream) {
        // the permutations run on a high-priority stream: when several contexts share
        // the GPU (a pipelined caller), they slip in between another context's steps
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) hi = 0;
        if (const char* e = std::getenv("PETTO_XPRIO")) hi = e[0] == '0' ? lo : hi;  // A/B of the priority
        if (
            cudaStreamCreateWithPriority(&ctx->xstream, cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->xev[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->xev[1], cudaEventDisableTiming) != cudaSuccess) {
            fail(ctx, PETTO_ERROR, "permutation stream creation failed");
            return nullptr;
        }
    }
    if (ctx->stage_elems < elems) {
        for (double*& b : ctx->stage) {
            cudaFree(b);
            b = nullptr;
        }
        ctx->stage_elems = 0;
        for (double*& b : ctx->stage)
            if (cudaMalloc(&b, sizeof(double) * elems) != cudaSuccess) {
                fail(ctx, PETTO_ERROR, "out of device memory (staging)");
                return nullptr;
            }
        ctx->stage_elems = elems;
    }
    double* b = ctx->stage[ctx->stage_next];
    ctx->stage_next ^= 1;
    return b;
}

// main stream -> permutation stream -> main stream
int xfer_fork(petto_ctx* ctx) {
    CK(cudaEventRecord(ctx->xev[0], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->xstream, ctx->xev[0], 0));
    return PETTO_OK;
}
int xfer_join(petto_ctx* ctx) {
    CK(cudaEventRecord(ctx->xev[1], ctx->xstream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->xev[1], 0));
    return PETTO_OK;
}

// device component of host component c of a displacement-like field (3D elasticity)
int dev_comp(const petto_ctx* ctx, int c, bool vec) { return ctx->perm && vec && ctx->comps == 3 ? (c + 2) % 3 : c; }

// Host (global, dense) <-> device (local, pitched) copies of `comps` components;
// vec: a displacement-like field whose components follow the axes.
int upload(petto_ctx* ctx, double* dst, const double* host, int comps, bool vec = false) {
    const Geo& g = ctx->g;
    const long long N = global_nodes(ctx);
    if (ctx->perm) {
        // host x planes [ks0, ks0 + nzs) of every component into the staging buffer
        // (rows of nzs doubles, host pitch nx_host = g.nz), then one permutation
        const size_t elems = (size_t)g.nzs * g.nx * g.ny;
        double* stage = stage_reserve(ctx, elems * comps);
        if (!stage) return PETTO_ERROR;
        if (g.nzs == g.nz)
            CK(cudaMemcpyAsync(stage, host, sizeof(double) * elems * comps, cudaMemcpyHostToDevice, ctx->stream));
        else
            for (int c = 0; c < comps; ++c)
                CK(cudaMemcpy2DAsync(stage + c * elems, (size_t)g.nzs * 8, host + c * N + g.ks0,
                                     (size_t)g.nz * 8, (size_t)g.nzs * 8, (size_t)g.nx * g.ny, cudaMemcpyHostToDevice,
                                     ctx->stream));
        if (int rc = xfer_fork(ctx)) return rc;
        const dim3 grid((g.nzs + 31) / 32, (g.nx + 31) / 32, g.ny), blk(32, 8);
        k_perm_in<<<grid, blk, 0, ctx->xstream>>>(g, stage, g.nzs, comps, vec && ctx->comps == 3, dst);
        ctx->launches++;
        CKL();
        return xfer_join(ctx);
    }
    for (int c = 0; c < comps; ++c) {
        const double* src = host + c * N + (long long)g.ks0 * g.nx * g.ny;
        if (g.px == g.nx)  // unpadded rows: one linear copy (full copy-engine rate)
            CK(cudaMemcpyAsync(dst + c * g.Ns, src, sizeof(double) * (size_t)g.nx * g.ny * g.nzs,
                               cudaMemcpyHostToDevice, ctx->stream));
        else
            CK(cudaMemcpy2DAsync(dst + c * g.Ns, (size_t)g.px * 8, src, (size_t)g.nx * 8, (size_t)g.nx * 8,
                                 (size_t)g.ny * g.nzs, cudaMemcpyHostToDevice, ctx->stream));
    }
    return PETTO_OK;
}

int download(petto_ctx* ctx, double* host, const double* src, int comps, bool vec = false) {
    const Geo& g = ctx->g;
    const long long N = global_nodes(ctx);
    if (ctx->perm) {
        const int nxo = g.ke - g.kb;
        const size_t elems = (size_t)nxo * g.nx * g.ny;
        double* stage = stage_reserve(ctx, elems * comps);
        if (!stage) return PETTO_ERROR;
        if (int rc = xfer_fork(ctx)) return rc;
        const dim3 grid((nxo + 31) / 32, (g.nx + 31) / 32, g.ny), blk(32, 8);
        k_perm_out<<<grid, blk, 0, ctx->xstream>>>(g, src, g.kb, nxo, comps, vec && ctx->comps == 3, stage);
        ctx->launches++;
        CKL();
        if (int rc = xfer_join(ctx)) return rc;
        if (nxo == g.nz)
            CK(cudaMemcpyAsync(host, stage, sizeof(double) * elems * comps, cudaMemcpyDeviceToHost, ctx->stream));
        else
            for (int c = 0; c < comps; ++c)
                CK(cudaMemcpy2DAsync(host + c * N + g.kb, (size_t)g.nz * 8, stage + c * elems, (size_t)nxo * 8,
                                     (size_t)nxo * 8, (size_t)g.nx * g.ny, cudaMemcpyDeviceToHost, ctx->stream));
        return PETTO_OK;
    }
    for (int c = 0; c < comps; ++c) {
        double* dst = host + c * N + (long long)g.kb * g.nx * g.ny;
        const double* s = src + c * g.Ns + lidx(g, 0, 0, g.kb);
        if (g.px == g.nx)
            CK(cudaMemcpyAsync(dst, s, sizeof(double) * (size_t)g.nx * g.ny * (g.ke - g.kb), cudaMemcpyDeviceToHost,
                               ctx->stream));
        else
            CK(cudaMemcpy2DAsync(dst, (size_t)g.nx * 8, s, (size_t)g.px * 8, (size_t)g.nx * 8,
                                 (size_t)g.ny * (g.ke - g.kb), cudaMemcpyDeviceToHost, ctx->stream));
    }
    return PETTO_OK;
}

// Host global node -> device (i, j, k) of the device grid.
void host_to_dev(const petto_ctx* ctx, long long node, int& i, int& j, int& k) {
    const Geo& g = ctx->g;
    if (ctx->perm) {  // host dims (nz, nx, ny) of the device grid
        const long long plane = (long long)g.nz * g.nx;
        const int hk = (int)(node / plane);
        const long long r = node - (long long)hk * plane;
        const int hj = (int)(r / g.nz), hi = (int)(r - (long long)hj * g.nz);
        i = hj;
        j = hk;
        k = hi;
        return;
    }
    const long long plane = (long long)g.nx * g.ny;
    k = (int)(node / plane);
    const long long r = node - (long long)k * plane;
    j = (int)(r / g.nx);
    i = (int)(r - (long long)j * g.nx);
}

// Global entry comp*N + node -> local entry comp*Ns + lidx, or -1 if the node is
// not on an owned plane of this rank.
long long local_entry(const petto_ctx* ctx, long long e, int* comp = nullptr, long long* node_out = nullptr) {
    const Geo& g = ctx->g;
    const long long N = global_nodes(ctx);
    const int c = (int)(e / N);
    int i, j, k;
    host_to_dev(ctx, e - (long long)c * N, i, j, k);
    if (k < g.kb || k >= g.ke) return -1;
    const int cd = dev_comp(ctx, c, true);
    if (comp) *comp = cd;
    if (node_out) *node_out = lidx(g, i, j, k);
    return cd * g.Ns + lidx(g, i, j, k);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// Stream memory operations (driver API): stream-ordered waits on / writes of
// 64-bit flags, used by the peer halo to order neighbouring slabs' steps without
// the host and without occupying SMs.
typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

StreamValueFn driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        return reinterpret_cast<StreamValueFn>(p);
    return nullptr;
}

int stream_wait_geq(petto_ctx* ctx, unsigned long long* addr, unsigned long long v) {
    static StreamValueFn fn = driver_fn("cuStreamWaitValue64");
    if (!fn) return fail(ctx, PETTO_ERROR, "cuStreamWaitValue64 unavailable");
    if (fn(reinterpret_cast<CUstream>(ctx->stream), reinterpret_cast<CUdeviceptr>(addr), v, 0x0 /*GEQ*/) !=
        CUDA_SUCCESS)
        return fail(ctx, PETTO_ERROR, "cuStreamWaitValue64 failed");
    return PETTO_OK;
}

int stream_write(petto_ctx* ctx, unsigned long long* addr, unsigned long long v) {
    static StreamValueFn fn = driver_fn("cuStreamWriteValue64");
    if (!fn) return fail(ctx, PETTO_ERROR, "cuStreamWriteValue64 unavailable");
    if (fn(reinterpret_cast<CUstream>(ctx->stream), reinterpret_cast<CUdeviceptr>(addr), v, 0x0 /*DEFAULT*/) !=
        CUDA_SUCCESS)
        return fail(ctx, PETTO_ERROR, "cuStreamWriteValue64 failed");
    return PETTO_OK;
}

// Peer halo, per fused step `seq`: wait until both neighbours finished step seq-1
// (their stores into our ghost planes are complete, and they no longer read the
// ghost planes of theirs that this step overwrites) ...
int peer_wait(petto_ctx* ctx, unsigned long long seq) {
    if (ctx->peer_lo.st[0])
        if (int rc = stream_wait_geq(ctx, ctx->inbox + 0, seq - 1)) return rc;
    if (ctx->peer_hi.st[0])
        if (int rc = stream_wait_geq(ctx, ctx->inbox + 1, seq - 1)) return rc;
    return PETTO_OK;
}

// ... and after the step's kernel tell them step `seq` is done.
int peer_signal(petto_ctx* ctx, unsigned long long seq) {
    if (ctx->peer_lo.flag)
        if (int rc = stream_write(ctx, ctx->peer_lo.flag, seq)) return rc;
    if (ctx->peer_hi.flag)
        if (int rc = stream_write(ctx, ctx->peer_hi.flag, seq)) return rc;
    return PETTO_OK;
}

// TMA descriptors of the fused 3D kernel (and its cell-modulus field).  No L2
// sector promotion: the 34-column U boxes start 256 B-aligned and would drag a
// second 256 B block each, and the 32-byte mask rows a full 256 B block
// (measured: 1.6x the algorithmic reads).
int make_tmaps(petto_ctx* ctx) {
    const Geo& g = ctx->g;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return fail(ctx, PETTO_ERROR, "cuTensorMapEncodeTiled unavailable");
    if (!ctx->ecell && cudaMalloc(&ctx->ecell, (size_t)g.Ns * sizeof(double)) != cudaSuccess)
        return fail(ctx, PETTO_ERROR, "out of device memory (cell modulus)");
    const cuuint64_t d4[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nzs, 3};
    const cuuint64_t s4[3] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.px * g.ny * 8, (cuuint64_t)g.Ns * 8};
    const cuuint32_t boxU[4] = {e3::LBOXX, e3::LROWS, e3::ZP, 3};
    const cuuint32_t boxP[4] = {32, e3::W, e3::ZP, 3};
    const cuuint32_t one[4] = {1, 1, 1, 1};
    auto map4 = [&](CUtensorMap* m, double* base, const cuuint32_t* box) {
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, d4, s4, box, one, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    const cuuint32_t boxO[4] = {32, e3::W, 1, 3};
    for (int b = 0; b < 3; ++b)
        if (!map4(&ctx->tU[b], ctx->st[b], boxU) || !map4(&ctx->tP[b], ctx->st[b], boxP) ||
            !map4(&ctx->tO[b], ctx->st[b], boxO))
            return fail(ctx, PETTO_ERROR, "tensor map (state) encode failed");
    if (!map4(&ctx->tO[3], ctx->r, boxO)) return fail(ctx, PETTO_ERROR, "tensor map (residual) encode failed");
    const cuuint64_t d3[3] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nzs};
    const cuuint64_t s3[2] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.px * g.ny * 8};
    const cuuint32_t boxC[3] = {32, e3::NWARP, e3::ZP};
    if (enc(&ctx->tC, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ctx->ecell, d3, s3, boxC, one,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(ctx, PETTO_ERROR, "tensor map (cell modulus) encode failed");
    const cuuint64_t sm[2] = {(cuuint64_t)g.px, (cuuint64_t)g.px * g.ny};
    const cuuint32_t boxM[3] = {32, e3::W, e3::ZP};
    if (enc(&ctx->tM, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, ctx->mask, d3, sm, boxM, one,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(ctx, PETTO_ERROR, "tensor map (mask) encode failed");
    ctx->tmaps = true;
    return PETTO_OK;
}

// ------------------------------------------------------------------- kernels

__global__ void k_scatter_bytes(const long long* __restrict__ idx, const unsigned char* __restrict__ v, long long n,
                                unsigned char* out) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[idx[t]] = v[t];
}

__global__ void k_scatter_values(const long long* __restrict__ idx, const double* __restrict__ v, long long n,
                                 double* out) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[idx[t]] = v[t];
}

// Lame positivity check of the ElasticityOperator constructor
// (state_solver.hpp:295-297) and kappa > 0 of variable_diffusion (stencil.hpp:145).
__global__ void k_check_positive(Geo g, const double* __restrict__ p, double c1, double c2, unsigned* flag) {
    int i, j, k;
    if (!owned_node(g, (long long)blockIdx.x * blockDim.x + threadIdx.x, i, j, k)) return;
    const double v = p[lidx(g, i, j, k)];
    if (!(c1 * v > 0.0) || !(c2 * v > 0.0)) atomicOr(flag, 1u);
}

// iterate_to_tolerance bookkeeping after residual #iter (state_solver.hpp:517-539):
// r = sqrt(sum r^2)/N; record, test, and raise the stop flag on the device.
__global__ void k_iter_finish(DeviceStatus* s, const double* __restrict__ partials, int n) {
    __shared__ double scratch[32];
    if (s->done) return;
    double v = 0.0;
    if (partials)
        for (int t = threadIdx.x; t < n; t += blockDim.x) v += partials[t];
    const double tot = block_sum<8>(v, scratch);
    if (threadIdx.x != 0) return;
    const double sq = partials ? tot : s->sumsq;
    const double r = sqrt(sq) / s->nodes;
    const long long k = s->iter;
    if (k == 0) {
        s->r_initial = r;
        s->r_final = r;
        if (r < s->target) {
            s->done = 1;
            s->converged = 1;
        } else if (s->max_iters <= 0) {
            s->done = 1;
        }
    } else {
        s->iterations = k;
        s->r_final = r;
        if (!isfinite(r)) {
            s->done = 1;
            s->aborted = 1;
        } else if (r < s->target) {
            s->done = 1;
            s->converged = 1;
        } else if (k >= s->max_iters) {
            s->done = 1;
        }
    }
    s->iter = k + 1;
}

__global__ void k_sum_to(const double* __restrict__ partials, int n, double* out) {
    __shared__ double scratch[32];
    double v = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) v += partials[t];
    const double tot = block_sum<8>(v, scratch);
    if (threadIdx.x == 0) *out = tot;
}

// ------------------------------------------------------------- state launches

struct StepCoef {
    int form;  // 0 APT explicit, 1 APT semi, 2 PT, 3 residual
    double dt, a, b, inv;
};

StepCoef coef(int form, double dt, double theta) {
    StepCoef c{form, dt, 0.0, 0.0, 1.0};
    if (form <= 1) {  // apt_step_inplace (state_solver.hpp:423-435)
        c.a = dt * dt / theta;
        c.b = dt / theta;
        c.inv = 1.0 / (1.0 + c.b);
    }
    return c;
}

// Work plan of the fused 3D kernel: items = strips x z-chunks, one CTA per SM.
// Chunks are as few as fill the SMs (each chunk restarts the z stream: two extra
// planes), at least 8 planes long, at most LMAX.
double step_bytes(const petto_ctx* ctx, int form);

void plan_3d(const petto_ctx* ctx, int nstrips, int& chunk, int& nitems, int& grid) {
    // Work items = y-strips x z-chunks of an even length L <= LMAX, one CTA per SM.
    // A CTA's time is (items per CTA) x (x tiles) x (a prologue, ~0.6 of a two-plane
    // task -- measured with the slot probe, tools/cta_times.py -- + L/2 tasks): pick
    // the L that minimises it (a partial second wave costs a whole wave; shorter
    // chunks restart the z stream more often).
    const int nzo = ctx->g.ke - ctx->g.kb;
    double best = 1e300;
    chunk = 2;
    // Grids far larger than L2: chunks of at most 32 planes, so that the line of
    // the next x-tile that a tile's halo columns pull in is still in L2 when the
    // CTA reaches that tile (16 tasks later instead of 32).  At C5 this cuts the
    // HBM reads per launch from 2.39 to 2.09 GB for 1.6% more SM cycles -- a net
    // gain under the power cap, where the clock follows the board power
    // (profiles/README.md, round 2).
    const double footprint = (double)owned_nodes(ctx) * step_bytes(ctx, 0);
    const int lmax = footprint > 512e6 ? 32 : e3::LMAX;
    for (int L = 2; L <= std::max(2, std::min(lmax, nzo + (nzo & 1))); L += 2) {
        const int items = nstrips * ((nzo + L - 1) / L);
        const int waves = (items + ctx->nsm - 1) / ctx->nsm;
        const double t = waves * (0.6 + 0.5 * L);
        if (t < best - 1e-9) {
            best = t;
            chunk = L;
        }
    }
    if (const char* e = std::getenv("PETTO_CHUNK")) chunk = std::max(2, std::min(e3::LMAX, std::atoi(e) & ~1));  // A/B
    nitems = nstrips * ((nzo + chunk - 1) / chunk);
    grid = std::min(ctx->nsm, nitems);
}

// Algorithmic HBM bytes per node and pseudo-time step: every
// array touched once -- state levels, the property, the new level.  Loads, pins
// and 1/V are O(surface) or computed and not counted.
double step_bytes(const petto_ctx* ctx, int form) {
    const int c = ctx->comps;
    const double lvl = 8.0 * c;                   // one state level
    if (form == 3) return lvl + 8.0 + lvl;        // residual: u_n, property, r
    if (form == 2) return lvl + 8.0 + lvl;        // PT: u_n, property, u_{n+1}
    return lvl + lvl + 8.0 + lvl;                 // APT: u_n, u_{n-1}, property, u_{n+1}
}

void timing_begin(petto_ctx* ctx, cudaEvent_t* ev) {
    ev[0] = ev[1] = nullptr;
    if (!ctx->timing) return;
    if (ctx->timing_seq++ % ctx->timing_stride) return;  // sample every timing_stride-th launch
    if (ctx->ev_used + 2 > (int)ctx->ev_pool.size()) {
        // drain the pool
        cudaStreamSynchronize(ctx->stream);
        for (int e = 0; e + 1 < ctx->ev_used; e += 2) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ctx->ev_pool[e], ctx->ev_pool[e + 1]);
            ctx->kernel_ms += ms;
        }
        ctx->ev_used = 0;
    }
    ev[0] = ctx->ev_pool[ctx->ev_used];
    ev[1] = ctx->ev_pool[ctx->ev_used + 1];
    ctx->ev_used += 2;
    cudaEventRecord(ev[0], ctx->stream);
}

void timing_end(petto_ctx* ctx, cudaEvent_t* ev, const char* name, double bytes) {
    if (!ctx->timing || !ev[0]) return;
    cudaEventRecord(ev[1], ctx->stream);
    ctx->kernel_launches += 1;
    ctx->bytes_per_launch = bytes;
    ctx->kernel_name = name;
}

// Parameters of the small fused kernels (heat 2D/3D, 2D elasticity) for one step.
FusedParams fused_params(const petto_ctx* ctx, const StepCoef& k, int cur, int prev, double* next, double* partials,
                         long long step, long long nsteps) {
    const Geo& g = ctx->g;
    FusedParams P{};
    P.g = g;
    P.form = k.form;
    P.dt = k.dt;
    P.a = k.a;
    P.b = k.b;
    P.inv = k.inv;
    P.cur = ctx->st[cur];
    P.prev = ctx->st[prev];
    P.next = next;
    P.prop = ctx->prop;
    P.mask = ctx->mask;
    P.aux = ctx->aux;
    P.src = ctx->src_uniform ? nullptr : ctx->src;
    P.src_uniform = ctx->src_value;
    for (int i = 0; i < 10 && i < (int)ctx->kh.size(); ++i) P.kh[i] = ctx->kh[i];
    const double nu = ctx->desc.poisson_ratio;
    P.e_scale = (ctx->prop_is_mu ? 1.0 : 1.0 / (2.0 * (1.0 + nu))) * (2.0 * (1.0 + ctx->nu_op) / 4.0);
    P.inv_base = g.dim == 3 ? 1.0 / (g.h[0] * g.h[1] * g.h[2]) : 1.0 / (g.h[0] * g.h[1]);
    for (int a = 0; a < 3; ++a) P.hih2[a] = 0.5 / (g.h[a] * g.h[a]);
    P.partials = partials;
    P.status = ctx->status;
    P.step = step;
    P.nsteps = nsteps;
    return P;
}

// The fused 3D elasticity step (k_elastic3d_fast): one step, or with nloc > 1 a
// persistent launch of steps step .. step + nloc - 1 (single domain, output =
// st[prev], no r^2 partials).  With `rot` (the tolerance loop's buffer rotation:
// u_it in st[rot[it % 3]]) a persistent launch of the tolerance loop's
// iterations step .. step + nloc - 1 with the stop test on the device.
int e3_launch(petto_ctx* ctx, const StepCoef& k, int cur, int prev, double* next, long long step,
              long long nsteps, double* partials, int nloc, const int* rot = nullptr) {
    const Geo& g = ctx->g;
    cudaEvent_t ev[2];
    const long long owned = owned_nodes(ctx);
    if (!ctx->tmaps && make_tmaps(ctx)) return PETTO_ERROR;
    const double nu = ctx->desc.poisson_ratio;
    const double e_scale =
        (ctx->prop_is_mu ? 1.0 : 1.0 / (2.0 * (1.0 + nu))) * (2.0 * (1.0 + ctx->nu_op) / 8.0);
    if (!ctx->ecell_valid || ctx->ecell_scale != e_scale) {
        e3::k_cell_modulus<<<4 * ctx->nsm, 256, 0, ctx->stream>>>(g, ctx->prop, e_scale, ctx->ecell);
        ctx->launches++;
        CKL();
        ctx->ecell_valid = true;
        ctx->ecell_scale = e_scale;
    }
    e3::Params P{};
    P.g = g;
    for (int i = 0; i < 45; ++i) P.kh[i] = ctx->kh[i];
    P.inv_base = 1.0 / (g.h[0] * g.h[1] * g.h[2]);
    if (k.form == 0) {  // 2u - u_prev + a r - b (u - u_prev)
        P.c1 = 2.0 - k.b;
        P.c2 = 1.0 - k.b;
        P.c3 = k.a;
    } else if (k.form == 1) {  // (2u - u_prev + b u + a r) / (1 + b)
        P.c1 = (2.0 + k.b) * k.inv;
        P.c2 = k.inv;
        P.c3 = k.a * k.inv;
    }
    P.dt = k.dt;
    P.next = next;
    if (ctx->peer_step) {
        int ob = -1;
        for (int b = 0; b < 3; ++b)
            if (next == ctx->st[b]) ob = b;
        if (ob < 0) return fail(ctx, PETTO_ERROR, "peer halo: output is not a state buffer");
        const long long plane = (long long)g.px * g.ny;
        if (ctx->peer_lo.st[0]) {
            P.peer_lo = ctx->peer_lo.st[ob] + (long long)(g.ks0 - ctx->peer_lo.ks0) * plane;
            P.peer_lo_Ns = ctx->peer_lo.Ns;
        }
        if (ctx->peer_hi.st[0]) {
            P.peer_hi = ctx->peer_hi.st[ob] + (long long)(g.ks0 - ctx->peer_hi.ks0) * plane;
            P.peer_hi_Ns = ctx->peer_hi.Ns;
        }
    }
    P.aux = ctx->aux;
#ifdef E3_CTA_TIMING
    {
        static unsigned long long* probe = nullptr;
        if (!probe) cudaMalloc(&probe, sizeof(unsigned long long) * 4 * 1024);
        P.cta_ns = probe;
        ctx->cta_probe = probe;
    }
#endif
    P.partials = partials;
    P.status = ctx->status;
    P.step = step;
    P.nsteps = nsteps;
    P.ntx = (g.nx + 31) / 32;
    P.nstrips = (g.ny + e3::W - 1) / e3::W;
    int grid = 0;
    plan_3d(ctx, P.nstrips, P.chunk, P.nitems, grid);
    if (partials && grid * (rot ? 2 : 1) > ctx->npartials) return fail(ctx, PETTO_ERROR, "partials buffer too small");
    e3::MapSet<3> MT;  // tolerance loop: iteration it reads st[rot[it % 3]], st[rot[(it + 2) % 3]]
    if (rot) {
        for (int j = 0; j < 3; ++j) {
            MT.m[j].u = ctx->tU[rot[j]];
            MT.m[j].c = ctx->tC;
            MT.m[j].p = ctx->tP[rot[(j + 2) % 3]];
            MT.m[j].m = ctx->tM;
            MT.m[j].o = ctx->tO[rot[(j + 1) % 3]];
        }
        P.nloc = nloc;
        P.gbar = ctx->gbar;
        CK(cudaMemsetAsync(ctx->gbar, 0, sizeof(unsigned), ctx->stream));
    }
    e3::MapSet<2> MS;
    int ob = next == ctx->r ? 3 : -1;
    for (int b = 0; b < 3; ++b)
        if (next == ctx->st[b]) ob = b;
    if (ob < 0) return fail(ctx, PETTO_ERROR, "fused 3D step: output is not a context buffer");
    MS.m[0].u = ctx->tU[cur];
    MS.m[0].c = ctx->tC;
    MS.m[0].p = ctx->tP[prev];
    MS.m[0].m = ctx->tM;
    MS.m[0].o = ctx->tO[ob];
    if (nloc > 1 && !rot) {
        // u_{n+1} overwrites u_{n-1}; the next step reads it as u_n
        if (ob != prev || partials || ctx->peer_step) return fail(ctx, PETTO_ERROR, "persistent 3D launch: bad plan");
        MS.m[1] = MS.m[0];
        MS.m[1].u = ctx->tU[prev];
        MS.m[1].p = ctx->tP[cur];
        MS.m[1].o = ctx->tO[cur];
        P.nloc = nloc;
        P.gbar = ctx->gbar;
        CK(cudaMemsetAsync(ctx->gbar, 0, sizeof(unsigned), ctx->stream));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(e3::WS_THREADS);
    cfg.dynamicSmemBytes = e3::SMEM_BYTES;
    cfg.stream = ctx->stream;
    timing_begin(ctx, ev);
    // Programmatic dependent launch: step s+1's CTAs become resident on the SMs
    // step s leaves idle and finish their setup (TMEM, barriers, tensor maps)
    // before griddepcontrol.wait releases them at step s's completion.  Only
    // when the plan leaves SMs idle (C4: 110 of 148; at C5 every SM is busy
    // and it measured 0.7% slower), not on a launch whose duration is sampled,
    // and not on slab ranks, whose steps are separated by stream memory
    // operations.
    cudaLaunchAttribute la[1];
    if (nloc > 1 || rot) {  // every CTA resident (the grid barrier), or the launch fails
        la[0].id = cudaLaunchAttributeCooperative;
        la[0].val.cooperative = 1;
        cfg.attrs = la;
        cfg.numAttrs = 1;
    } else if (!ctx->no_pdl && !ctx->peer_step && grid < ctx->nsm && !ev[0]) {
        la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        la[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = la;
        cfg.numAttrs = 1;
    }
    cudaError_t le;
    // r^2 partials only when a caller reads them (iterate_to_tolerance, residual)
    if (rot) {
        switch (k.form) {
            case 0: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_persist<0, true>, P, MT); break;
            case 1: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_persist<1, true>, P, MT); break;
            default: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_persist<2, true>, P, MT); break;
        }
    } else if (nloc > 1) {
        switch (k.form) {
            case 0: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_persist<0, false>, P, MS); break;
            case 1: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_persist<1, false>, P, MS); break;
            default: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_persist<2, false>, P, MS); break;
        }
    } else
    switch (k.form * 2 + (partials ? 1 : 0)) {
        case 0: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_fast<0, false>, P, MS.m[0]); break;
        case 1: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_fast<0, true>, P, MS.m[0]); break;
        case 2: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_fast<1, false>, P, MS.m[0]); break;
        case 3: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_fast<1, true>, P, MS.m[0]); break;
        case 4: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_fast<2, false>, P, MS.m[0]); break;
        case 5: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_fast<2, true>, P, MS.m[0]); break;
        case 6: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_fast<3, false>, P, MS.m[0]); break;
        default: le = cudaLaunchKernelEx(&cfg, e3::k_elastic3d_fast<3, true>, P, MS.m[0]); break;
    }
    if (le != cudaSuccess) return fail(ctx, PETTO_ERROR, std::string("fused 3D launch: ") + cudaGetErrorString(le));
    timing_end(ctx, ev, nloc > 1 || rot ? "k_elastic3d_persist" : "k_elastic3d_fast",
               (double)owned * step_bytes(ctx, k.form) * nloc);
    ctx->launches++;
    CKL();
    if (partials) ctx->npartials_used = grid;
    return PETTO_OK;
}

// One fused (fast) or replica state step: reads st[cur] (and st[prev]), writes
// `next` (a state buffer or the residual scratch for form 3).
int state_step(petto_ctx* ctx, const StepCoef& k, int cur, int prev, double* next, long long step, long long nsteps,
               bool want_partials) {
    const Geo& g = ctx->g;
    double* partials = want_partials ? ctx->partials : nullptr;
    if (ctx->mode == PETTO_MODE_FAST) {
        cudaEvent_t ev[2];
        const long long owned = owned_nodes(ctx);
        if (g.dim == 3 && ctx->desc.physics == 1) return e3_launch(ctx, k, cur, prev, next, step, nsteps, partials, 1);
        FusedParams P = fused_params(ctx, k, cur, prev, next, partials, step, nsteps);
        const int grid = (int)std::min<long long>(ctx->npartials, blocks_for(owned));
        timing_begin(ctx, ev);
        if (ctx->desc.physics == 0) {
            k_heat_fast<<<grid, 256, 0, ctx->stream>>>(P);
            timing_end(ctx, ev, "k_heat_fast", (double)owned * step_bytes(ctx, k.form));
        } else {
            k_elastic2d_fast<<<grid, 256, 0, ctx->stream>>>(P);
            timing_end(ctx, ev, "k_elastic2d_fast", (double)owned * step_bytes(ctx, k.form));
        }
        ctx->launches++;
        CKL();
        if (partials) ctx->npartials_used = grid;
        return PETTO_OK;
    }
    // replica: residual, [zero constrained], update, apply constraints
    const long long owned = owned_nodes(ctx);
    const int nb = blocks_for(owned);
    double* r = k.form == 3 ? next : ctx->r;
    if (ctx->desc.physics == 1) {
        // mu per corner: the stored Lame field, or cm * E as update_lame forms it
        const double cm = ctx->prop_is_mu ? 1.0 : 1.0 / (2.0 * (1.0 + ctx->desc.poisson_ratio));
        k_elastic_residual_replica<<<nb, 256, 0, ctx->stream>>>(g, ctx->st[cur], ctx->prop, cm, ctx->src,
                                                                ctx->Kdev, 2.0 * (1.0 + ctx->nu_op) / (1 << g.dim),
                                                                r, ctx->status, step, nsteps);
    } else {
        k_heat_residual_replica<<<nb, 256, 0, ctx->stream>>>(g, ctx->st[cur], ctx->prop, ctx->src, ctx->src_value,
                                                             ctx->src_uniform ? 0 : 1, r, ctx->status, step,
                                                             nsteps);
    }
    ctx->launches++;
    CKL();
    if (k.form == 3 || want_partials) {
        // zero_constrained then the serial r^2 (residual_norm in threads == 1 order)
        if (ctx->ncons) {
            k_zero_entries<<<blocks_for(ctx->ncons), 256, 0, ctx->stream>>>(ctx->cons_ent, ctx->ncons, r,
                                                                           ctx->status, step, nsteps);
            ctx->launches++;
        }
        if (want_partials) {
            k_sumsq_serial<<<1, 32, 0, ctx->stream>>>(g, ctx->comps, r, &ctx->status->sumsq);
            ctx->launches++;
        }
        CKL();
        if (k.form == 3) return PETTO_OK;
    }
    k_update_replica<<<nb, 256, 0, ctx->stream>>>(g, ctx->comps, k.form, ctx->st[cur], ctx->st[prev], r, next, k.dt,
                                                  k.a, k.b, k.inv, ctx->status, step, nsteps);
    ctx->launches++;
    if (ctx->ncons) {
        k_apply_constraints<<<blocks_for(ctx->ncons), 256, 0, ctx->stream>>>(ctx->cons_ent, ctx->cons_val,
                                                                             ctx->ncons, next, ctx->status, step,
                                                                             nsteps);
        ctx->launches++;
    }
    CKL();
    return PETTO_OK;
}

int reset_status(petto_ctx* ctx) {
    DeviceStatus s{};
    s.first_bad = PETTO_NO_BAD;
    s.nodes = (double)global_nodes(ctx);
    *ctx->status_h = s;
    CK(cudaMemcpyAsync(ctx->status, ctx->status_h, sizeof(DeviceStatus), cudaMemcpyHostToDevice, ctx->stream));
    return PETTO_OK;
}

int read_status(petto_ctx* ctx) {
    CK(cudaMemcpyAsync(ctx->status_h, ctx->status, sizeof(DeviceStatus), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return PETTO_OK;
}

int require_ready(petto_ctx* ctx) {
    if (!ctx->state_set) return fail(ctx, PETTO_INVALID, "state not set");
    if (ctx->desc.physics == 1 && !ctx->op_ready)
        return fail(ctx, PETTO_INVALID, "elasticity operator not initialised (petto_dev_init_operator)");
    return PETTO_OK;
}

// ------------------------------------------------------------ slab transport

enum FieldSel { F_STATE = 0, F_PROP = 1, F_PHASES = 2, F_SCRATCH1 = 3 };

double* field_of(petto_ctx* c, FieldSel s, int buf) {
    switch (s) {
        case F_STATE: return c->st[buf];
        case F_PROP: return c->prop;
        case F_PHASES: return c->phases;
        default: return c->scratch1;
    }
}

int comps_of(const petto_ctx* c, FieldSel s) {
    return s == F_STATE ? c->comps : (s == F_PHASES ? c->mat.nphases : 1);
}

int nccl_check(petto_ctx* ctx, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return PETTO_OK;
    const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error";
    return fail(ctx, PETTO_ERROR, std::string(what) + ": " + m);
}

// Ghost planes of `field` from the +-1 ranks (NCCL transport), stream ordered after
// the kernel that wrote the owned planes.  No-op on a single rank.
int halo_ptr(petto_ctx* ctx, double* f, int comps) {
    if (!ctx->nccl_comm) return PETTO_OK;
    NcclApi& N = nccl();
    const ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl_comm);
    const Geo& g = ctx->g;
    const size_t plane = (size_t)g.px * g.ny;
    N.GroupStart();
    for (int c = 0; c < comps; ++c) {
        double* fc = f + c * g.Ns;
        if (ctx->rank > 0) {
            N.Send(fc + lidx(g, 0, 0, g.kb), plane, ncclDouble, ctx->rank - 1, comm, ctx->stream);
            N.Recv(fc + lidx(g, 0, 0, g.kb - 1), plane, ncclDouble, ctx->rank - 1, comm, ctx->stream);
        }
        if (ctx->rank < ctx->nranks - 1) {
            N.Send(fc + lidx(g, 0, 0, g.ke - 1), plane, ncclDouble, ctx->rank + 1, comm, ctx->stream);
            N.Recv(fc + lidx(g, 0, 0, g.ke), plane, ncclDouble, ctx->rank + 1, comm, ctx->stream);
        }
    }
    return nccl_check(ctx, N.GroupEnd(), "halo exchange");
}

int halo(petto_ctx* ctx, FieldSel s, int buf) { return halo_ptr(ctx, field_of(ctx, s, buf), comps_of(ctx, s)); }

// In-place all-reduce of device scalars across the ranks (no-op on one rank).
int allreduce(petto_ctx* ctx, void* p, size_t n, ncclDataType_t t, ncclRedOp_t op) {
    if (!ctx->nccl_comm) return PETTO_OK;
    return nccl_check(ctx, nccl().AllReduce(p, p, n, t, op, static_cast<ncclComm_t>(ctx->nccl_comm), ctx->stream),
                      "all-reduce");
}

// Local group: pull this context's ghost planes of state buffer `buf` from the
// neighbours' owned planes once their step has finished.
int group_pull(petto_ctx* ctx, int buf) {
    const Geo& g = ctx->g;
    const size_t bytes = sizeof(double) * (size_t)g.px * g.ny;
    for (petto_ctx* nb : {ctx->nb_lo, ctx->nb_hi}) {
        if (!nb) continue;
        CK(cudaStreamWaitEvent(ctx->stream, nb->ev_step, 0));
        const int k = nb == ctx->nb_lo ? g.kb - 1 : g.ke;  // ghost plane = neighbour's owned plane
        for (int c = 0; c < ctx->comps; ++c)
            CK(cudaMemcpyAsync(ctx->st[buf] + c * g.Ns + lidx(g, 0, 0, k),
                               nb->st[buf] + c * nb->g.Ns + lidx(nb->g, 0, 0, k), bytes, cudaMemcpyDefault,
                               ctx->stream));
    }
    CK(cudaEventRecord(ctx->ev_pull, ctx->stream));
    return PETTO_OK;
}

// kappa > 0 guard of variable_diffusion_into (stencil.hpp:145-157), checked once per
// call because kappa is constant within a solve.
int check_kappa(petto_ctx* ctx) {
    if (ctx->desc.physics != 0) return PETTO_OK;
    CK(cudaMemsetAsync(&ctx->status->flags, 0, sizeof(unsigned), ctx->stream));
    k_check_positive<<<blocks_for(owned_nodes(ctx)), 256, 0, ctx->stream>>>(ctx->g, ctx->prop, 1.0, 1.0,
                                                                            &ctx->status->flags);
    ctx->launches++;
    CKL();
    if (int rc = read_status(ctx)) return rc;
    if (ctx->status_h->flags & 1u)
        return fail(ctx, PETTO_INVALID, "variable_diffusion: kappa must be positive everywhere");
    return PETTO_OK;
}

}  // namespace

// ======================================================================= C-ABI

namespace {
constexpr long long WCHUNK = 8LL << 20;  // values per chunk
constexpr long long WBLOCKS = WCHUNK / wr::TB;

int writer_buffers(petto_ctx* ctx) {
    if (ctx->wtext[0]) return PETTO_OK;
    const size_t cap = (size_t)WCHUNK * wr::MAXB;
    for (int b = 0; b < 2; ++b) {
        CK(cudaMalloc(&ctx->wtext[b], cap));
        CK(cudaMallocHost(&ctx->htext[b], cap));
    }
    CK(cudaMalloc(&ctx->wblk, sizeof(long long) * 2 * (WBLOCKS + 1)));
    CK(cudaMallocHost(&ctx->wcount, sizeof(long long) * 2));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, ctx->wscan_bytes, ctx->wblk, ctx->wblk, (int)(WBLOCKS + 1)));
    CK(cudaMalloc(&ctx->wscan, ctx->wscan_bytes));
    return PETTO_OK;
}

// The field a writer reads: component/phase `index` of the context's state,
// phases or property, in the reference's node order.
int writer_source(petto_ctx* ctx, int field, int index, wr::Src* out) {
    const Geo& g = ctx->g;
    if (g.kb != 0 || g.ke != g.nz)
        return fail(ctx, PETTO_INVALID, "writers need the whole grid in one context (slab rank: gather first)");
    if (ctx->perm)
        return fail(ctx, PETTO_INVALID, "writers need the reference layout (x_outermost context: download first)");
    const double* base = nullptr;
    if (field == PETTO_FIELD_STATE) {
        if (index < 0 || index >= ctx->comps) return fail(ctx, PETTO_INVALID, "writer: state component out of range");
        base = ctx->st[ctx->cur] + (long long)index * g.Ns;
    } else if (field == PETTO_FIELD_PHASE) {
        if (!ctx->design_set) return fail(ctx, PETTO_INVALID, "design not set (petto_dev_set_design)");
        if (index < 0 || index >= ctx->mat.nphases) return fail(ctx, PETTO_INVALID, "writer: phase out of range");
        base = ctx->phases + (long long)index * g.Ns;
    } else if (field == PETTO_FIELD_PROPERTY) {
        base = ctx->prop;
    } else {
        return fail(ctx, PETTO_INVALID, "writer: unknown field");
    }
    *out = wr::Src{base, g.nx, g.ny, g.px, (long long)g.px * g.ny, (long long)g.nx * g.ny * g.nz};
    return PETTO_OK;
}

// Formats src's values ("%.17g" + separator) chunk by chunk and hands the bytes
// to sink(const char*, size_t) in order.
template <class Sink>
int format_stream(petto_ctx* ctx, const wr::Src& src, int sep_mode, Sink&& sink) {
    if (int rc = writer_buffers(ctx)) return rc;
    cudaEvent_t ev[2];
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    int rc = PETTO_OK;
    long long c = 0;
    for (long long i0 = 0; i0 < src.n && rc == PETTO_OK; i0 += WCHUNK, ++c) {
        const int b = (int)(c & 1);
        const long long n = std::min(WCHUNK, src.n - i0);
        const int blocks = (int)((n + wr::TB - 1) / wr::TB);
        long long* bytes = ctx->wblk + (size_t)b * (WBLOCKS + 1);
        wr::k_block_bytes<<<blocks, wr::TB, 0, ctx->stream>>>(src, i0, n, bytes);
        cudaMemsetAsync(bytes + blocks, 0, sizeof(long long), ctx->stream);
        size_t tb = ctx->wscan_bytes;
        // exclusive scan in place: bytes[blocks] becomes the chunk's total
        if (cub::DeviceScan::ExclusiveSum(ctx->wscan, tb, bytes, bytes, blocks + 1, ctx->stream) != cudaSuccess) {
            rc = fail(ctx, PETTO_ERROR, "writer: scan failed");
            break;
        }
        wr::k_block_write<<<blocks, wr::TB, 0, ctx->stream>>>(src, i0, n, sep_mode, bytes, ctx->wtext[b]);
        ctx->launches += 3;
        if (cudaGetLastError() != cudaSuccess) {
            rc = fail(ctx, PETTO_ERROR, "writer: launch failed");
            break;
        }
        cudaMemcpyAsync(&ctx->wcount[b], bytes + blocks, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(ctx->htext[b], ctx->wtext[b], (size_t)n * wr::MAXB, cudaMemcpyDeviceToHost, ctx->stream);
        cudaEventRecord(ev[b], ctx->stream);
        if (c > 0) {  // the previous chunk while this one formats and copies
            cudaEventSynchronize(ev[1 - b]);
            rc = sink(ctx->htext[1 - b], (size_t)ctx->wcount[1 - b]);
        }
    }
    if (rc == PETTO_OK && c > 0) {
        const int b = (int)((c - 1) & 1);
        if (cudaEventSynchronize(ev[b]) != cudaSuccess) rc = fail(ctx, PETTO_ERROR, "writer: copy failed");
        else rc = sink(ctx->htext[b], (size_t)ctx->wcount[b]);
    }
    cudaStreamSynchronize(ctx->stream);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    return rc;
}

std::string fmt17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

struct OutFile {
    FILE* f = nullptr;
    ~OutFile() {
        if (f) std::fclose(f);
    }
};

int open_out(petto_ctx* ctx, OutFile& o, const char* path, bool binary) {
    o.f = std::fopen(path, binary ? "wb" : "w");
    if (!o.f) return fail(ctx, PETTO_IO, std::string("cannot open '") + path + "' for writing");
    std::setvbuf(o.f, nullptr, _IOFBF, 1 << 22);
    return PETTO_OK;
}

int close_out(petto_ctx* ctx, OutFile& o, const char* path) {
    const bool bad = std::ferror(o.f) != 0;
    const int rc = std::fclose(o.f);
    o.f = nullptr;
    if (bad || rc) return fail(ctx, PETTO_IO, std::string("write failed for '") + path + "'");
    return PETTO_OK;
}

std::string grid_dims(const Geo& g) {
    return std::to_string(g.nx) + " " + std::to_string(g.ny) + " " + std::to_string(g.nz);
}
}  // namespace

extern "C" {

const char* petto_dev_version(void) { return "petto_b200 0.1 (sm_100a)"; }

int petto_dev_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

const char* petto_dev_last_error(const petto_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

void* petto_dev_stream(petto_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int petto_dev_create(const petto_grid_desc* d, petto_ctx** out) {
    petto_ctx* ctx = nullptr;
    *out = nullptr;
    if (d->dim != 2 && d->dim != 3) return fail(nullptr, PETTO_INVALID, "grid: dim must be 2 or 3");
    for (int a = 0; a < d->dim; ++a) {
        if (d->n[a] < 3) return fail(nullptr, PETTO_INVALID, "grid: need at least 3 nodes per axis");
        if (!(d->length[a] > 0.0)) return fail(nullptr, PETTO_INVALID, "grid: axis length must be positive");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= d->device)
        return fail(nullptr, PETTO_ERROR, "no CUDA device available (the B200 path has no CPU fallback)");
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, d->device) != cudaSuccess || prop.major < 10)
        return fail(nullptr, PETTO_ERROR, "device is not sm_100-class (Blackwell) -- no fallback");
    if (cudaSetDevice(d->device) != cudaSuccess) return fail(nullptr, PETTO_ERROR, "cudaSetDevice failed");

    ctx = new petto_ctx();
    ctx->desc = *d;
    ctx->device = d->device;
    ctx->nsm = prop.multiProcessorCount;
    ctx->mode = d->mode;
    ctx->comps = d->physics ? d->dim : 1;
    Geo& g = ctx->g;
    g.dim = d->dim;
    g.nx = (int)d->n[0];
    g.ny = (int)d->n[1];
    g.nz = d->dim == 3 ? (int)d->n[2] : 1;
    for (int a = 0; a < 3; ++a) g.h[a] = 1.0;
    for (int a = 0; a < d->dim; ++a) g.h[a] = d->length[a] / (double)(d->n[a] - 1);
    if (d->x_outermost) {
        // device axes (y, z, x): the unit-cell stiffness, lumped volumes and every
        // kernel follow from the device spacings (an axis relabelling of an
        // isotropic operator); the reference's operation order is not kept, so
        // REPLICA mode is refused
        if (d->dim != 3 || d->mode != PETTO_MODE_FAST) {
            delete ctx;
            return fail(nullptr, PETTO_INVALID, "x_outermost: 3D grids in FAST mode only");
        }
        ctx->perm = true;
        const double h[3] = {g.h[0], g.h[1], g.h[2]};
        g.nx = (int)d->n[1];
        g.ny = (int)d->n[2];
        g.nz = (int)d->n[0];
        g.h[0] = h[1];
        g.h[1] = h[2];
        g.h[2] = h[0];
    }
    g.kb = (int)(d->k_end > d->k_begin ? d->k_begin : 0);
    g.ke = (int)(d->k_end > d->k_begin ? d->k_end : g.nz);
    if (g.kb < 0 || g.ke > g.nz || g.kb >= g.ke) {
        delete ctx;
        return fail(nullptr, PETTO_INVALID, "slab: need 0 <= k_begin < k_end <= nz");
    }
    geo_factors(g);
    g.ks0 = std::max(0, g.kb - 1);
    g.nzs = std::min(g.nz, g.ke + 1) - g.ks0;
    g.px = (g.nx + 15) / 16 * 16;
    if (const char* e = std::getenv("PETTO_PITCH_PAD")) g.px += (std::atoi(e) + 15) / 16 * 16;  // layout A/B
    g.Ns = (long long)g.px * g.ny * g.nzs;

    auto cleanup = [&](const std::string& m) {
        petto_dev_destroy(ctx);
        return fail(nullptr, PETTO_ERROR, m);
    };
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup("stream creation failed");
    const size_t fb = sizeof(double) * (size_t)g.Ns;
    for (int b = 0; b < 3; ++b)
        if (cudaMalloc(&ctx->st[b], fb * ctx->comps) != cudaSuccess) return cleanup("out of device memory (state)");
    if (cudaMalloc(&ctx->prop, fb) != cudaSuccess || cudaMalloc(&ctx->aux, fb * ctx->comps) != cudaSuccess ||
        cudaMalloc(&ctx->mask, (size_t)g.Ns) != cudaSuccess || cudaMalloc(&ctx->src, fb * ctx->comps) != cudaSuccess ||
        cudaMalloc(&ctx->r, fb * ctx->comps) != cudaSuccess)
        return cleanup("out of device memory (fields)");
    for (int b = 0; b < 3; ++b) cudaMemsetAsync(ctx->st[b], 0, fb * ctx->comps, ctx->stream);
    cudaMemsetAsync(ctx->prop, 0, fb, ctx->stream);
    cudaMemsetAsync(ctx->aux, 0, fb * ctx->comps, ctx->stream);
    cudaMemsetAsync(ctx->mask, 0, (size_t)g.Ns, ctx->stream);
    cudaMemsetAsync(ctx->src, 0, fb * ctx->comps, ctx->stream);
    cudaMemsetAsync(ctx->r, 0, fb * ctx->comps, ctx->stream);
    // block partials of the reductions: enough blocks (32 per SM) for the design
    // loop's grid-stride passes to keep HBM busy, one partial each
    ctx->npartials = std::max(32 * ctx->nsm, 1024);
    if (const char* e = std::getenv("PETTO_NO_TBLOCK")) ctx->no_tblock = e[0] == '1';  // A/B of the 2D solves
    if (const char* e = std::getenv("PETTO_NO_PDL")) ctx->no_pdl = e[0] == '1';        // A/B of the 3D step overlap
    if (const char* e = std::getenv("PETTO_MULTI")) ctx->multi = e[0] - '0';          // A/B of persistent 3D solves
    if (cudaMalloc(&ctx->partials, sizeof(double) * ctx->npartials) != cudaSuccess ||
        cudaMalloc(&ctx->status, sizeof(DeviceStatus)) != cudaSuccess ||
        cudaMallocHost(&ctx->status_h, sizeof(DeviceStatus)) != cudaSuccess ||
        cudaMalloc(&ctx->dscal, sizeof(double) * 256) != cudaSuccess ||
        cudaMallocHost(&ctx->hpin, sizeof(double) * 1024) != cudaSuccess ||
        cudaMalloc(&ctx->Kdev, sizeof(double) * 576) != cudaSuccess ||
        cudaMalloc(&ctx->gbar, sizeof(unsigned) * 32) != cudaSuccess)
        return cleanup("out of device memory (scalars)");
    const cudaFuncAttribute smattr = cudaFuncAttributeMaxDynamicSharedMemorySize;
#define E3_KERNEL e3::k_elastic3d_fast
    if (cudaFuncSetAttribute(E3_KERNEL<0, false>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(E3_KERNEL<0, true>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(E3_KERNEL<1, false>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(E3_KERNEL<1, true>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(E3_KERNEL<2, false>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(E3_KERNEL<2, true>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(E3_KERNEL<3, false>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(E3_KERNEL<3, true>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(e3::k_elastic3d_persist<0, false>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(e3::k_elastic3d_persist<1, false>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(e3::k_elastic3d_persist<2, false>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(e3::k_elastic3d_persist<0, true>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(e3::k_elastic3d_persist<1, true>, smattr, e3::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(e3::k_elastic3d_persist<2, true>, smattr, e3::SMEM_BYTES) != cudaSuccess)
        return cleanup("cannot configure shared memory for k_elastic3d_fast");
    if (reset_status(ctx)) return cleanup(ctx->err);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return cleanup("device initialisation failed");
    *out = ctx;
    return PETTO_OK;
}

void petto_dev_destroy(petto_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->nccl_comm && nccl().CommDestroy) nccl().CommDestroy(static_cast<ncclComm_t>(ctx->nccl_comm));
    for (petto_ctx* nb : {ctx->nb_lo, ctx->nb_hi})  // unlink from a local group
        if (nb) (nb->nb_lo == ctx ? nb->nb_lo : nb->nb_hi) = nullptr;
    if (ctx->ev_step) cudaEventDestroy(ctx->ev_step);
    if (ctx->ev_pull) cudaEventDestroy(ctx->ev_pull);
    if (ctx->ev_team) cudaEventDestroy(ctx->ev_team);
    cudaFree(ctx->team_buf);
    for (double* b : ctx->stage) cudaFree(b);
    if (ctx->xstream) cudaStreamDestroy(ctx->xstream);
    for (cudaEvent_t e : ctx->xev)
        if (e) cudaEventDestroy(e);
    for (int b = 0; b < 3; ++b) cudaFree(ctx->st[b]);
    cudaFree(ctx->prop);
    cudaFree(ctx->ecell);
    for (petto_b200::PeerSlab* ps : {&ctx->peer_lo, &ctx->peer_hi}) {
        if (!ps->ipc) continue;
        for (double* p : ps->st) cudaIpcCloseMemHandle(p);
        cudaIpcCloseMemHandle(ps->ipc_inbox);
    }
    cudaFree(ctx->inbox);
    cudaFree(ctx->aux);
    cudaFree(ctx->mask);
    cudaFree(ctx->src);
    cudaFree(ctx->r);
    cudaFree(ctx->cons_ent);
    cudaFree(ctx->cons_val);
    cudaFree(ctx->Kdev);
    cudaFree(ctx->gbar);
    cudaFree(ctx->partials);
    cudaFree(ctx->status);
    cudaFree(ctx->dscal);
    if (ctx->hpin) cudaFreeHost(ctx->hpin);
    if (ctx->status_h) cudaFreeHost(ctx->status_h);
    for (int b = 0; b < 2; ++b) {
        cudaFree(ctx->wtext[b]);
        if (ctx->htext[b]) cudaFreeHost(ctx->htext[b]);
    }
    cudaFree(ctx->wblk);
    if (ctx->wcount) cudaFreeHost(ctx->wcount);
    cudaFree(ctx->wscan);
    cudaFree(ctx->wmm);
    design_free(ctx);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int petto_dev_set_mode(petto_ctx* ctx, int mode) {
    if (mode != PETTO_MODE_FAST && mode != PETTO_MODE_REPLICA) return fail(ctx, PETTO_INVALID, "unknown mode");
    if (ctx->perm && mode != PETTO_MODE_FAST) return fail(ctx, PETTO_INVALID, "x_outermost: FAST mode only");
    ctx->mode = mode;
    return PETTO_OK;
}

// aux and mask from the context's constraint list and loads (whatever the order of
// set_constraints / set_source): mask bit c = component c pinned, bit 3 = a load
// at the node; aux = the pinned value at a constrained entry (apply_constraints,
// grid.hpp:234-238), the load at the other entries.
static int rebuild_aux_mask(petto_ctx* ctx) {
    const Geo& g = ctx->g;
    std::vector<unsigned char> hmask((size_t)g.Ns, 0);
    std::vector<double> haux;
    std::vector<long long> hidx;
    for (long long le : ctx->cons_host) hmask[le % g.Ns] |= (unsigned char)(1u << (le / g.Ns));
    for (size_t t = 0; t < ctx->load_host.size(); ++t) {
        const long long le = ctx->load_host[t];
        const long long node = le % g.Ns;
        if (!((hmask[node] >> (le / g.Ns)) & 1u)) {
            hidx.push_back(le);
            haux.push_back(ctx->load_vhost[t]);
        }
    }
    for (long long le : ctx->load_host) hmask[le % g.Ns] |= 8u;
    hidx.insert(hidx.end(), ctx->cons_host.begin(), ctx->cons_host.end());
    haux.insert(haux.end(), ctx->cons_vhost.begin(), ctx->cons_vhost.end());
    CK(cudaMemcpyAsync(ctx->mask, hmask.data(), (size_t)g.Ns, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->aux, 0, sizeof(double) * (size_t)g.Ns * ctx->comps, ctx->stream));
    if (!hidx.empty()) {
        long long* di = nullptr;
        double* dv = nullptr;
        CK(cudaMalloc(&di, sizeof(long long) * hidx.size()));
        CK(cudaMalloc(&dv, sizeof(double) * haux.size()));
        CK(cudaMemcpyAsync(di, hidx.data(), sizeof(long long) * hidx.size(), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(dv, haux.data(), sizeof(double) * haux.size(), cudaMemcpyHostToDevice, ctx->stream));
        k_scatter_values<<<blocks_for((long long)hidx.size()), 256, 0, ctx->stream>>>(di, dv, (long long)hidx.size(),
                                                                                      ctx->aux);
        ctx->launches++;
        CKL();
        CK(cudaStreamSynchronize(ctx->stream));
        cudaFree(di);
        cudaFree(dv);
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return PETTO_OK;
}

int petto_dev_set_constraints(petto_ctx* ctx, const int64_t* entry, const double* value, int64_t count) {
    CK(cudaSetDevice(ctx->device));
    std::vector<long long> ent;
    std::vector<double> val;
    for (int64_t t = 0; t < count; ++t) {
        if (entry[t] < 0 || entry[t] >= global_nodes(ctx) * ctx->comps)
            return fail(ctx, PETTO_INVALID, "constraint entry outside the field");
        const long long le = local_entry(ctx, entry[t]);
        if (le < 0) continue;
        ent.push_back(le);
        val.push_back(value[t]);
    }
    cudaFree(ctx->cons_ent);
    cudaFree(ctx->cons_val);
    ctx->cons_ent = nullptr;
    ctx->cons_val = nullptr;
    ctx->ncons = (long long)ent.size();
    if (ctx->ncons) {
        CK(cudaMalloc(&ctx->cons_ent, sizeof(long long) * ent.size()));
        CK(cudaMalloc(&ctx->cons_val, sizeof(double) * val.size()));
        CK(cudaMemcpyAsync(ctx->cons_ent, ent.data(), sizeof(long long) * ent.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaMemcpyAsync(ctx->cons_val, val.data(), sizeof(double) * val.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
    }
    ctx->cons_host = std::move(ent);
    ctx->cons_vhost = std::move(val);
    return rebuild_aux_mask(ctx);
}

int petto_dev_set_source(petto_ctx* ctx, const double* source) {
    CK(cudaSetDevice(ctx->device));
    const long long N = global_nodes(ctx);
    if (int rc = upload(ctx, ctx->src, source, ctx->comps, true)) return rc;
    if (ctx->desc.physics == 0) {
        // uniform source: the fused kernel reads a scalar instead of a field
        bool uni = true;
        for (long long n = 1; n < N && uni; ++n) uni = source[n] == source[0];
        ctx->src_uniform = uni;
        ctx->src_value = source[0];
        CK(cudaStreamSynchronize(ctx->stream));
        return PETTO_OK;
    }
    // elasticity: the nonzero loads of the owned planes (sparse in every preset)
    ctx->load_host.clear();
    ctx->load_vhost.clear();
    for (long long e = 0; e < ctx->comps * N; ++e) {
        const double v = source[e];
        if (v == 0.0) continue;
        const long long le = local_entry(ctx, e);
        if (le < 0) continue;
        ctx->load_host.push_back(le);
        ctx->load_vhost.push_back(v);
    }
    return rebuild_aux_mask(ctx);
}

int petto_dev_set_property(petto_ctx* ctx, const double* property) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = upload(ctx, ctx->prop, property, 1)) return rc;
    ctx->ecell_valid = false;
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->prop_node0 = property[0];
    ctx->prop_node0_valid = true;
    ctx->prop_is_mu = false;
    return PETTO_OK;
}

int petto_dev_set_lame(petto_ctx* ctx, const double* lambda, const double* mu) {
    CK(cudaSetDevice(ctx->device));
    if (ctx->desc.physics != 1) return fail(ctx, PETTO_INVALID, "set_lame: not an elasticity context");
    // positivity of both Lame fields (state_solver.hpp:295-297), lambda staged in the residual scratch
    if (int rc = upload(ctx, ctx->r, lambda, 1)) return rc;
    if (int rc = upload(ctx, ctx->prop, mu, 1)) return rc;
    ctx->ecell_valid = false;
    CK(cudaMemsetAsync(&ctx->status->flags, 0, sizeof(unsigned), ctx->stream));
    k_check_positive<<<blocks_for(owned_nodes(ctx)), 256, 0, ctx->stream>>>(ctx->g, ctx->r, 1.0, 1.0,
                                                                            &ctx->status->flags);
    k_check_positive<<<blocks_for(owned_nodes(ctx)), 256, 0, ctx->stream>>>(ctx->g, ctx->prop, 1.0, 1.0,
                                                                            &ctx->status->flags);
    ctx->launches += 2;
    CKL();
    if (int rc = read_status(ctx)) return rc;
    ctx->lame_bad = (ctx->status_h->flags & 1u) != 0;
    ctx->lame0[0] = lambda[0];
    ctx->lame0[1] = mu[0];
    ctx->prop_is_mu = true;
    ctx->prop_node0_valid = true;
    return PETTO_OK;
}

int petto_dev_init_operator(petto_ctx* ctx) {
    CK(cudaSetDevice(ctx->device));
    if (ctx->desc.physics == 0) {
        ctx->op_ready = true;
        return PETTO_OK;
    }
    const double nu = ctx->desc.poisson_ratio;
    const double cl = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double cm = 1.0 / (2.0 * (1.0 + nu));
    double l0, m0;
    if (ctx->prop_is_mu) {
        if (ctx->lame_bad) return fail(ctx, PETTO_INVALID, "elasticity: Lame fields must be positive");
        l0 = ctx->lame0[0];
        m0 = ctx->lame0[1];
    } else {
        CK(cudaMemsetAsync(&ctx->status->flags, 0, sizeof(unsigned), ctx->stream));
        k_check_positive<<<blocks_for(owned_nodes(ctx)), 256, 0, ctx->stream>>>(ctx->g, ctx->prop, cl, cm,
                                                                                &ctx->status->flags);
        ctx->launches++;
        CKL();
        if (int rc = read_status(ctx)) return rc;
        if (ctx->status_h->flags & 1u) return fail(ctx, PETTO_INVALID, "elasticity: Lame fields must be positive");
        // Lame pair of node 0 as make_lame / update_lame store it
        double e0 = ctx->prop_node0;
        if (!ctx->prop_node0_valid) {
            if (ctx->g.kb != 0) return fail(ctx, PETTO_INVALID, "node 0 property unknown on this rank");
            CK(cudaMemcpyAsync(ctx->hpin, ctx->prop + lidx(ctx->g, 0, 0, 0), sizeof(double), cudaMemcpyDeviceToHost,
                               ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            e0 = ctx->hpin[0];
        }
        l0 = cl * e0;
        m0 = cm * e0;
    }
    // nu from node 0's Lame pair (state_solver.hpp:299-301)
    ctx->nu_op = l0 / (2.0 * (l0 + m0));
    ctx->K = unit_cell_stiffness(ctx->g.dim, ctx->g.h, ctx->nu_op);
    try {
        ctx->kh = modal_stiffness(ctx->g.dim, ctx->K);
    } catch (const std::exception& e) {
        return fail(ctx, PETTO_ERROR, e.what());
    }
    // Kdev (576 doubles, allocated with the context): no allocation here -- this runs
    // inside run(), where a device-synchronising call could wait on another rank
    std::memcpy(ctx->hpin, ctx->K.data(), sizeof(double) * ctx->K.size());
    CK(cudaMemcpyAsync(ctx->Kdev, ctx->hpin, sizeof(double) * ctx->K.size(), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->op_ready = true;
    return PETTO_OK;
}

int petto_dev_set_state(petto_ctx* ctx, const double* current, const double* previous) {
    CK(cudaSetDevice(ctx->device));
    ctx->cur = 0;
    ctx->prev = 1;
    // peer halo: the upload (ghost planes included) is a step of the neighbour
    // protocol -- it waits until the neighbours stopped storing into our ghosts and
    // tells them when their next stores may land
    const unsigned long long seq = ctx->peer_halo ? ++ctx->peer_seq : 0;
    if (seq)
        if (int rc = peer_wait(ctx, seq)) return rc;
    if (int rc = upload(ctx, ctx->st[0], current, ctx->comps, true)) return rc;
    if (int rc = upload(ctx, ctx->st[1], previous ? previous : current, ctx->comps, true)) return rc;
    if (seq)
        if (int rc = peer_signal(ctx, seq)) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->state_set = true;
    return PETTO_OK;
}

int petto_dev_get_state(petto_ctx* ctx, double* current, double* previous) {
    CK(cudaSetDevice(ctx->device));
    if (current)
        if (int rc = download(ctx, current, ctx->st[ctx->cur], ctx->comps, true)) return rc;
    if (previous)
        if (int rc = download(ctx, previous, ctx->st[ctx->prev], ctx->comps, true)) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    return PETTO_OK;
}

// Inbox of the peer halo: two step counters written by the neighbours.
int peer_prepare(petto_ctx* ctx) {
    if (!ctx->inbox) {
        CK(cudaMalloc(&ctx->inbox, 2 * sizeof(unsigned long long)));
    }
    CK(cudaMemset(ctx->inbox, 0, 2 * sizeof(unsigned long long)));
    ctx->peer_seq = 0;
    return PETTO_OK;
}

// One step of hybrid_solve: next := previous buffer, written in place; then swap
// (state_solver.hpp:421, 440).  Slab ranks then refresh their ghost planes: with
// the peer halo the fused kernel already stored its boundary planes into the
// neighbours' ghosts and the step is ordered by stream flags; otherwise NCCL.
bool use_peer(const petto_ctx* ctx) {
    return ctx->peer_halo && ctx->mode == PETTO_MODE_FAST && ctx->g.dim == 3 && ctx->desc.physics == 1;
}

int hybrid_step(petto_ctx* ctx, const StepCoef& k, long long step, long long nsteps) {
    const bool peer = use_peer(ctx);
    unsigned long long seq = 0;
    if (peer) {
        seq = ++ctx->peer_seq;
        if (int rc = peer_wait(ctx, seq)) return rc;
        ctx->peer_step = true;
    }
    const int rc = state_step(ctx, k, ctx->cur, ctx->prev, ctx->st[ctx->prev], step, nsteps, false);
    ctx->peer_step = false;
    if (rc) return rc;
    std::swap(ctx->cur, ctx->prev);
    if (peer) return peer_signal(ctx, seq);
    return halo(ctx, F_STATE, ctx->cur);
}

// Persistent 3D elasticity solves (e3::k_elastic3d_persist): one domain, fast
// mode, grids whose per-step launch overhead is not negligible (<= 16 M nodes,
// e.g. C4); PETTO_MULTI=0/1 forces it off/on (A/B).
bool persistent_3d_ok(const petto_ctx* ctx) {
    const Geo& g = ctx->g;
    if (ctx->mode != PETTO_MODE_FAST || g.dim != 3 || ctx->desc.physics != 1 || ctx->nccl_comm || ctx->nb_lo ||
        ctx->nb_hi || ctx->peer_halo || ctx->multi == 0)
        return false;
    return ctx->multi == 1 || owned_nodes(ctx) <= (16LL << 20);
}

// Small grids of the heat / 2D-elasticity operators: the whole hybrid_solve runs
// as one cooperative launch (k_small_solve) instead of one launch per step.
bool small_solve_ok(const petto_ctx* ctx) {
    const Geo& g = ctx->g;
    const bool small_op = ctx->desc.physics == 0 || g.dim == 2;
    return ctx->mode == PETTO_MODE_FAST && small_op && !ctx->nccl_comm && !ctx->nb_lo && !ctx->nb_hi &&
           owned_nodes(ctx) <= (16LL << 20);
}

int small_solve(petto_ctx* ctx, const StepCoef& ka, const StepCoef& kp, long long n_apt, long long n_pt) {
    SolveParams S{};
    S.base = fused_params(ctx, ka, ctx->cur, ctx->prev, ctx->st[ctx->prev], nullptr, 0, n_apt + n_pt);
    S.st[0] = ctx->st[ctx->cur];
    S.st[1] = ctx->st[ctx->prev];
    S.c0 = 0;
    S.n_apt = n_apt;
    S.n_pt = n_pt;
    S.form_apt = ka.form;
    S.a = ka.a;
    S.b = ka.b;
    S.inv = ka.inv;
    S.dt_pt = kp.dt;
    const bool heat = ctx->desc.physics == 0;
    if (ctx->g.dim == 2 && !ctx->no_tblock) {
        // temporal blocking: TBK (heat) / EK (elasticity) steps per grid barrier on
        // shared-memory tiles; the first shape whose tiles are all co-resident
        const Geo& g = ctx->g;
        struct Shape {
            const void* fn;
            int tw, th, nthr;
            size_t smem;
            const char* name;
        };
        const Shape shapes[] = {
            heat ? Shape{(const void*)k_heat2d_tb, TBX, TBY, TB_THREADS, (size_t)TRN * (6 * sizeof(double) + 1),
                         "k_heat2d_tb"}
                 : Shape{(const void*)k_elastic2d_tb<1>, ETX, e_ty(1), ETHREADS, e_smem(1), "k_elastic2d_tb"},
            heat ? Shape{nullptr, 0, 0, 0, 0, nullptr}
                 : Shape{(const void*)k_elastic2d_tb<2>, ETX, e_ty(2), ETHREADS, e_smem(2), "k_elastic2d_tb"},
        };
        for (const Shape& sh : shapes) {
            if (!sh.fn) continue;
            const int tx = (g.nx + sh.tw - 1) / sh.tw, ty = (g.ny + sh.th - 1) / sh.th;
            CK(cudaFuncSetAttribute(sh.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem));
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sh.fn, sh.nthr, sh.smem));
            if ((long long)tx * ty > (long long)per_sm * ctx->nsm) continue;
            TBParams T{};
            T.base = S.base;
            T.pair[0][0] = S.st[0];
            T.pair[0][1] = S.st[1];
            T.pair[1][0] = ctx->st[3 - ctx->cur - ctx->prev];  // the spare state buffer
            T.pair[1][1] = ctx->r;
            T.n_apt = n_apt;
            T.n_pt = n_pt;
            T.form_apt = ka.form;
            T.a = ka.a;
            T.b = ka.b;
            T.inv = ka.inv;
            T.dt_pt = kp.dt;
            T.tiles_x = tx;
            void* targs[] = {&T};
            cudaEvent_t ev[2];
            timing_begin(ctx, ev);
            CK(cudaLaunchCooperativeKernel(sh.fn, dim3(tx * ty), dim3(sh.nthr), targs, sh.smem, ctx->stream));
            timing_end(ctx, ev, sh.name,
                       (double)owned_nodes(ctx) * (step_bytes(ctx, ka.form) * n_apt + step_bytes(ctx, 2) * n_pt));
            ctx->launches++;
            CKL();
            return PETTO_OK;
        }
    }
    const void* fn = heat ? (const void*)k_small_solve<0> : (const void*)k_small_solve<1>;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
    const int grid = (int)std::min<long long>((long long)std::max(per_sm, 1) * ctx->nsm, blocks_for(owned_nodes(ctx)));
    void* args[] = {&S};
    cudaEvent_t ev[2];
    timing_begin(ctx, ev);
    CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, 0, ctx->stream));
    timing_end(ctx, ev, "k_small_solve",
               (double)owned_nodes(ctx) * (step_bytes(ctx, ka.form) * n_apt + step_bytes(ctx, 2) * n_pt));
    ctx->launches++;
    CKL();
    return PETTO_OK;
}

// PTParams::validate (state_solver.hpp:25-33)
static int validate_params(petto_ctx* ctx, const petto_pt_params* p) {
    if (!(p->dt_pt > 0.0) && p->n_pt > 0) return fail(ctx, PETTO_INVALID, "pt params: dt_pt must be positive");
    if (!(p->dt_apt > 0.0) && p->n_apt > 0) return fail(ctx, PETTO_INVALID, "pt params: dt_apt must be positive");
    if (!(p->theta > 0.0)) return fail(ctx, PETTO_INVALID, "pt params: theta must be positive");
    if (p->n_apt < 0 || p->n_pt < 0 || p->n_apt + p->n_pt < 1)
        return fail(ctx, PETTO_INVALID, "pt params: need at least one step per loop");
    return PETTO_OK;
}

// ---------------------------------------------------------------- design (a19-a26)

// MaterialModel::validate (objectives.hpp:26-33) / ObjectiveWeights::validate (:44-51)
static int validate_design(petto_ctx* ctx, const petto_material* m, const petto_weights* w) {
    if (m->nphases < 1 || m->nphases > PETTO_MAX_PHASES)
        return fail(ctx, PETTO_INVALID, "material: one property value per phase required");
    for (int i = 0; i < m->nphases; ++i)
        if (!(m->properties[i] > 0.0)) return fail(ctx, PETTO_INVALID, "material: properties must be positive");
    if (m->penalty < 1.0) return fail(ctx, PETTO_INVALID, "material: penalty must be >= 1");
    if (!(m->void_floor > 0.0)) return fail(ctx, PETTO_INVALID, "material: void floor must be positive");
    if (w->alpha_compliance < 0 || w->alpha_volume < 0 || w->alpha_unity < 0 || w->alpha_region < 0)
        return fail(ctx, PETTO_INVALID, "weights: must be non-negative");
    if (w->alpha_compliance + w->alpha_volume + w->alpha_unity + w->alpha_region <= 0)
        return fail(ctx, PETTO_INVALID, "weights: at least one weight must be positive");
    if (w->compliance_sign != 1 && w->compliance_sign != -1)
        return fail(ctx, PETTO_INVALID, "weights: compliance sign must be +1 or -1");
    return PETTO_OK;
}

static DesignP design_params(const petto_ctx* ctx) {
    DesignP d{};
    d.np = ctx->mat.nphases;
    for (int i = 0; i < d.np; ++i) d.props[i] = ctx->mat.properties[i];
    d.penalty = ctx->mat.penalty;
    auto ipow = [](double e) {
        const int ei = (int)e;
        return (e == (double)ei && ei >= 0 && ei <= 8) ? ei : -1;
    };
    d.ipen = ipow(d.penalty);
    d.ipen1 = ipow(d.penalty - 1.0);
    d.floor_v = ctx->mat.void_floor;
    return d;
}

static double domain_volume(const petto_ctx* ctx) {
    double v = 1.0;
    for (int a = 0; a < ctx->g.dim; ++a) v *= ctx->desc.length[a];
    return v;
}

int petto_dev_set_design(petto_ctx* ctx, const petto_material* m, const petto_targets* t, const petto_weights* w) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = validate_design(ctx, m, w)) return rc;
    if (t->has_region && t->nregion <= 0)
        return fail(ctx, PETTO_INVALID, "region_objective: region mask covers no nodes");
    const Geo& g = ctx->g;
    ctx->mat = *m;
    ctx->tgt = *t;
    ctx->wts = *w;
    ctx->region_nodes.assign(t->region_nodes, t->region_nodes + (t->has_region ? t->nregion : 0));
    ctx->tgt.region_nodes = nullptr;
    design_free(ctx);
    const size_t P = (size_t)m->nphases;
    const long long owned = owned_nodes(ctx);
    CK(cudaMalloc(&ctx->phases, sizeof(double) * P * g.Ns));
    CK(cudaMalloc(&ctx->gc, sizeof(double) * P * g.Ns));
    CK(cudaMalloc(&ctx->scratch1, sizeof(double) * g.Ns));
    CK(cudaMalloc(&ctx->term1, sizeof(double) * std::max<long long>(owned, (long long)ctx->region_nodes.size() + 1)));
    CK(cudaMalloc(&ctx->term2, sizeof(double) * owned));
    {
        const dim3 sg = sens_grid(ctx);  // block maxima of the sensitivity kernels, partials of the FAST sums
        CK(cudaMalloc(&ctx->pmax, sizeof(double) * 8 * std::max<long long>(ctx->npartials, (long long)sg.x * sg.y * sg.z)));
    }
    CK(cudaMalloc(&ctx->count, sizeof(unsigned long long)));
    CK(cudaMemsetAsync(ctx->phases, 0, sizeof(double) * P * g.Ns, ctx->stream));
    CK(cudaMemsetAsync(ctx->gc, 0, sizeof(double) * P * g.Ns, ctx->stream));
    CK(cudaMemsetAsync(ctx->scratch1, 0, sizeof(double) * g.Ns, ctx->stream));
    CK(cudaMemsetAsync(ctx->dscal, 0, sizeof(double) * 256, ctx->stream));
    // region: per stored node mask, and the owned region nodes in list order as
    // device-grid node ids (k_region_terms decodes them with the device dims)
    std::vector<unsigned char> mask((size_t)g.Ns, 0);
    std::vector<long long> own;
    for (int64_t node : ctx->region_nodes) {
        if (node < 0 || node >= global_nodes(ctx)) return fail(ctx, PETTO_INVALID, "region node outside the grid");
        int i, j, k;
        host_to_dev(ctx, node, i, j, k);
        if (k >= g.ks0 && k < g.ks0 + g.nzs) mask[lidx(g, i, j, k)] = 1;
        if (k >= g.kb && k < g.ke) own.push_back(((long long)k * g.ny + j) * g.nx + i);
    }
    CK(cudaMalloc(&ctx->region_mask, (size_t)g.Ns));
    CK(cudaMemcpyAsync(ctx->region_mask, mask.data(), (size_t)g.Ns, cudaMemcpyHostToDevice, ctx->stream));
    if (!ctx->region_nodes.empty()) {
        ctx->region_nodes.assign(own.begin(), own.end());
        CK(cudaMalloc(&ctx->region_dev, sizeof(long long) * std::max<size_t>(own.size(), 1)));
        if (!own.empty())
            CK(cudaMemcpyAsync(ctx->region_dev, own.data(), sizeof(long long) * own.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->design_set = true;
    return PETTO_OK;
}

int petto_dev_set_phases(petto_ctx* ctx, const double* phases) {
    CK(cudaSetDevice(ctx->device));
    if (!ctx->design_set) return fail(ctx, PETTO_INVALID, "design not set (petto_dev_set_design)");
    if (int rc = upload(ctx, ctx->phases, phases, ctx->mat.nphases)) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    return PETTO_OK;
}

int petto_dev_get_phases(petto_ctx* ctx, double* phases) {
    CK(cudaSetDevice(ctx->device));
    if (!ctx->design_set) return fail(ctx, PETTO_INVALID, "design not set (petto_dev_set_design)");
    if (int rc = download(ctx, phases, ctx->phases, ctx->mat.nphases)) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    return PETTO_OK;
}

// ================================================================= teams
// A slab decomposition as one host thread drives it: the contexts that thread
// owns -- every slab of a local group (one process, one or several GPUs), or this
// rank's single context under NCCL -- and the transport between the slabs.  The
// solver and design-loop routines below run the same code for one domain, a local
// group and an NCCL rank.  Every collective is stream ordered, with
// no host synchronisation, and exists twice:
//   NCCL  -- all-reduce / send-recv / broadcast on the context's stream;
//   group -- peer copies between the contexts' streams ordered by events, values
//            combined on the lead context in rank order (deterministic), ghost
//            planes pulled from the neighbours' owned planes.
// REPLICA-mode sums (the reference's threads == 1 order, parallel.hpp:22-24) are
// chained across the slabs in rank order, so a split run stays bit-identical to
// the single domain; FAST sums are per-slab trees plus one reduction.
namespace {

// NVTX range over one phase of the path (header-only NVTX v3: free unless a
// profiler attaches) -- nsys / ncu timelines show hybrid_solve, the design-loop
// phases, the halo exchanges and the slab reductions by name.
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
    Range(const Range&) = delete;
    Range& operator=(const Range&) = delete;
};

struct Team {
    petto_ctx** c;
    int n;
    petto_ctx* lead() const { return c[0]; }
    bool nccl() const { return n == 1 && c[0]->nccl_comm != nullptr; }
    bool split() const { return n > 1 || nccl(); }
    bool replica() const { return c[0]->mode == PETTO_MODE_REPLICA; }
};

using PtrOf = std::function<void*(petto_ctx*)>;
using DblOf = std::function<double*(petto_ctx*)>;

bool is_slab(const petto_ctx* ctx) { return ctx->g.kb != 0 || ctx->g.ke != ctx->g.nz; }

// A context used on its own: a slab needs its communicator for the collectives.
// (A lone slab may still run the state solve: its ghost planes then stay as
// uploaded, or follow the peer halo -- used for timing one rank's share.)
int solo_ok(petto_ctx* ctx, bool solve_only) {
    if (ctx->nb_lo || ctx->nb_hi)
        return fail(ctx, PETTO_INVALID, "slab context is linked in a local group: use the petto_dev_group_* calls");
    if (is_slab(ctx) && !ctx->nccl_comm && !solve_only)
        return fail(ctx, PETTO_INVALID, "slab context without a communicator (petto_dev_comm_init)");
    return PETTO_OK;
}

int team_check(Team t) {
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        if (t.n > 1 && (ctx->nb_lo != (i ? t.c[i - 1] : nullptr) || ctx->nb_hi != (i + 1 < t.n ? t.c[i + 1] : nullptr)))
            return fail(ctx, PETTO_INVALID, "group: call petto_dev_group_link first");
        if (ctx->mode != t.lead()->mode) return fail(ctx, PETTO_INVALID, "group: contexts differ in mode");
    }
    return PETTO_OK;
}

// every stream of the group waits until every other one reached this point
int team_sync(Team t) {
    if (t.n == 1) return PETTO_OK;
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        CK(cudaEventRecord(ctx->ev_team, ctx->stream));
    }
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        for (int j = 0; j < t.n; ++j)
            if (j != i) CK(cudaStreamWaitEvent(ctx->stream, t.c[j]->ev_team, 0));
    }
    return PETTO_OK;
}

enum { RED_SUM = 0, RED_MAX = 1, RED_MIN_I64 = 2, RED_SUM_U64 = 3, RED_MAX_U32 = 4 };
constexpr int TEAM_MAX = 64;

// in-place reduction of `count` device values at at(ctx) over the slabs
int team_reduce(Team t, const PtrOf& at, int count, int op) {
    Range nv("petto.team_reduce");
    const size_t es = op == RED_MAX_U32 ? 4 : 8;
    if (t.n == 1) {
        petto_ctx* ctx = t.c[0];
        static const ncclDataType_t ty[5] = {ncclDouble, ncclDouble, ncclInt64, ncclUint64, ncclUint32};
        static const ncclRedOp_t ro[5] = {ncclSum, ncclMax, ncclMin, ncclSum, ncclMax};
        return allreduce(ctx, at(ctx), (size_t)count, ty[op], ro[op]);
    }
    petto_ctx* ctx = t.lead();
    if (count > TEAM_MAX || t.n > TEAM_MAX) return fail(ctx, PETTO_INVALID, "group: too many slabs or values");
    CK(cudaSetDevice(ctx->device));
    if (!ctx->team_buf) CK(cudaMalloc(&ctx->team_buf, 8 * TEAM_MAX * TEAM_MAX));
    if (int rc = team_sync(t)) return rc;
    CK(cudaSetDevice(ctx->device));
    for (int i = 0; i < t.n; ++i)
        CK(cudaMemcpyAsync(static_cast<char*>(ctx->team_buf) + (size_t)i * count * es, at(t.c[i]), count * es,
                           cudaMemcpyDefault, ctx->stream));
    k_team_combine<<<1, TEAM_MAX, 0, ctx->stream>>>(ctx->team_buf, t.n, count, op, at(ctx));
    ctx->launches++;
    CKL();
    if (int rc = team_sync(t)) return rc;
    for (int i = 1; i < t.n; ++i) {
        petto_ctx* x = t.c[i];
        CK(cudaSetDevice(x->device));
        if (cudaMemcpyAsync(at(x), at(ctx), count * es, cudaMemcpyDefault, x->stream) != cudaSuccess)
            return fail(x, PETTO_ERROR, "group: reduction broadcast failed");
    }
    return team_sync(t);  // the lead may overwrite its value only after every copy
}

// Ordered sum over the slabs: segment s of every slab in rank order, s = 0..nseg-1
// (the components of a vector field are segments: entry order c*N + node).
// seg(ctx, s, init, out) launches one segment on ctx's stream continuing from
// *init (nullptr: from zero).  The total lands in dst(ctx) of every context.
using SegFn = std::function<int(petto_ctx*, int, const double*, double*)>;

int team_chain(Team t, int nseg, const SegFn& seg, const DblOf& dst) {
    Range nv("petto.team_chain");
    petto_ctx* ctx = t.lead();
    const bool ranks = t.nccl() && ctx->nranks > 1;
    if (t.n == 1 && !ranks) {
        for (int s = 0; s < nseg; ++s)
            if (int rc = seg(ctx, s, s ? ctx->dscal + DS_CHAIN : nullptr, ctx->dscal + DS_CHAIN)) return rc;
        CK(cudaMemcpyAsync(dst(ctx), ctx->dscal + DS_CHAIN, 8, cudaMemcpyDeviceToDevice, ctx->stream));
        return PETTO_OK;
    }
    if (ranks) {
        NcclApi& N = nccl();
        const ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl_comm);
        const int r = ctx->rank, R = ctx->nranks;
        for (int s = 0; s < nseg; ++s) {
            const bool has_prev = r > 0 || s > 0, has_next = !(s == nseg - 1 && r == R - 1);
            if (has_prev)
                if (int rc = nccl_check(ctx, N.Recv(ctx->dscal + DS_CHAIN_IN, 1, ncclDouble, (r + R - 1) % R, comm,
                                                    ctx->stream), "chain recv"))
                    return rc;
            if (int rc = seg(ctx, s, has_prev ? ctx->dscal + DS_CHAIN_IN : nullptr, ctx->dscal + DS_CHAIN)) return rc;
            if (has_next)
                if (int rc = nccl_check(ctx, N.Send(ctx->dscal + DS_CHAIN, 1, ncclDouble, (r + 1) % R, comm,
                                                    ctx->stream), "chain send"))
                    return rc;
        }
        if (int rc = nccl_check(ctx, N.Broadcast(ctx->dscal + DS_CHAIN, ctx->dscal + DS_CHAIN, 1, ncclDouble, R - 1,
                                                 comm, ctx->stream), "chain broadcast"))
            return rc;
        CK(cudaMemcpyAsync(dst(ctx), ctx->dscal + DS_CHAIN, 8, cudaMemcpyDeviceToDevice, ctx->stream));
        return PETTO_OK;
    }
    if (int rc = team_sync(t)) return rc;
    petto_ctx* before = nullptr;
    for (int s = 0; s < nseg; ++s)
        for (int i = 0; i < t.n; ++i) {
            petto_ctx* x = t.c[i];
            CK(cudaSetDevice(x->device));
            if (before) {
                if (cudaStreamWaitEvent(x->stream, before->ev_team, 0) != cudaSuccess ||
                    cudaMemcpyAsync(x->dscal + DS_CHAIN_IN, before->dscal + DS_CHAIN, 8, cudaMemcpyDefault,
                                    x->stream) != cudaSuccess)
                    return fail(x, PETTO_ERROR, "group: chain hand-off failed");
            }
            if (int rc = seg(x, s, before ? x->dscal + DS_CHAIN_IN : nullptr, x->dscal + DS_CHAIN)) return rc;
            if (cudaEventRecord(x->ev_team, x->stream) != cudaSuccess)
                return fail(x, PETTO_ERROR, "group: chain event failed");
            before = x;
        }
    if (int rc = team_sync(t)) return rc;
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* x = t.c[i];
        CK(cudaSetDevice(x->device));
        if (cudaMemcpyAsync(dst(x), before->dscal + DS_CHAIN, 8, cudaMemcpyDefault, x->stream) != cudaSuccess)
            return fail(x, PETTO_ERROR, "group: chain broadcast failed");
    }
    return team_sync(t);
}

// Sum over all slabs of the per-node terms every context left in term(ctx)[0,
// len(ctx)) (owned nodes in k, j, i order, or region-list order), into dst(ctx).
int team_sum_terms(Team t, const DblOf& term, const std::function<long long(petto_ctx*)>& len, const DblOf& dst) {
    if (t.replica())
        return team_chain(
            t, 1,
            [&](petto_ctx* ctx, int, const double* init, double* out) {
                k_sum_serial<<<1, 32, 0, ctx->stream>>>(term(ctx), len(ctx), out, init);
                ctx->launches++;
                CKL();
                return PETTO_OK;
            },
            dst);
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        const long long n = len(ctx);
        const int nb = (int)std::min<long long>(ctx->npartials, blocks_for(n));
        k_sum_partials<<<nb, 256, 0, ctx->stream>>>(term(ctx), n, ctx->partials);
        k_sum_finish<<<1, 256, 0, ctx->stream>>>(ctx->partials, nb, dst(ctx));
        ctx->launches += 2;
        CKL();
    }
    return team_reduce(t, [&](petto_ctx* x) -> void* { return dst(x); }, 1, RED_SUM);
}

// FAST: the sum of block partials a kernel left in partials(ctx)[0, nparts(ctx)),
// into dst(ctx) of every context (same tree as team_sum_terms' FAST branch).
int team_sum_partials(Team t, const DblOf& partials, const std::function<int(petto_ctx*)>& nparts,
                      const DblOf& dst) {
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        k_sum_finish<<<1, 256, 0, ctx->stream>>>(partials(ctx), nparts(ctx), dst(ctx));
        ctx->launches++;
        CKL();
    }
    return team_reduce(t, [&](petto_ctx* x) -> void* { return dst(x); }, 1, RED_SUM);
}

// grid of the FAST partial-sum kernels: the partition k_sum_partials uses
int sum_grid(const petto_ctx* ctx) { return (int)std::min<long long>(ctx->npartials, blocks_for(owned_nodes(ctx))); }

// Ghost planes of `comps` fields starting at f(ctx) (component stride Ns).
int team_halo(Team t, const DblOf& f, int comps) {
    Range nv("petto.halo");
    if (t.n == 1) return t.nccl() ? halo_ptr(t.lead(), f(t.lead()), comps) : PETTO_OK;
    if (int rc = team_sync(t)) return rc;
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        const Geo& g = ctx->g;
        const size_t bytes = sizeof(double) * (size_t)g.px * g.ny;
        for (petto_ctx* nb : {ctx->nb_lo, ctx->nb_hi}) {
            if (!nb) continue;
            const int k = nb == ctx->nb_lo ? g.kb - 1 : g.ke;
            for (int c = 0; c < comps; ++c)
                CK(cudaMemcpyAsync(f(ctx) + c * g.Ns + lidx(g, 0, 0, k), f(nb) + c * nb->g.Ns + lidx(nb->g, 0, 0, k),
                                   bytes, cudaMemcpyDefault, ctx->stream));
        }
    }
    return team_sync(t);
}

int team_phase_ghosts(Team t) {
    bool stale = false;
    for (int i = 0; i < t.n; ++i) stale |= t.c[i]->phi_ghosts_stale;
    if (stale && t.split())
        if (int rc = team_halo(t, [](petto_ctx* x) { return x->phases; }, t.lead()->mat.nphases)) return rc;
    for (int i = 0; i < t.n; ++i) t.c[i]->phi_ghosts_stale = false;
    return PETTO_OK;
}

// ------------------------------------------------------------ state solver

int team_hybrid_solve(Team t, const petto_pt_params* p, int64_t* abort_step) {
    Range nv("petto.hybrid_solve");
    if (int rc = team_check(t)) return rc;
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        if (int rc = validate_params(ctx, p)) return rc;
        if (int rc = require_ready(ctx)) return rc;
        if (int rc = check_kappa(ctx)) return rc;
        if (int rc = reset_status(ctx)) return rc;
    }
    petto_ctx* ctx = t.lead();
    const long long nsteps = p->n_apt + p->n_pt;
    const StepCoef ka = coef(p->form ? 1 : 0, p->dt_apt, p->theta);
    const StepCoef kp = coef(2, p->dt_pt, p->theta);
    auto first_bad = [](petto_ctx* x) -> void* { return &x->status->first_bad; };
    if (t.n == 1 && small_solve_ok(ctx)) {
        if (int rc = small_solve(ctx, ka, kp, p->n_apt, p->n_pt)) return rc;
        if (nsteps % 2) std::swap(ctx->cur, ctx->prev);  // the kernel swapped nsteps times
    } else if (t.n == 1 && persistent_3d_ok(ctx)) {
        // one persistent launch per form segment (APT, then PT)
        for (int seg = 0; seg < 2; ++seg) {
            const long long n = seg ? p->n_pt : p->n_apt, s0 = seg ? p->n_apt + 1 : 1;
            if (n <= 0) continue;
            if (int rc = e3_launch(ctx, seg ? kp : ka, ctx->cur, ctx->prev, ctx->st[ctx->prev], s0, nsteps, nullptr,
                                   (int)n))
                return rc;
            if (n % 2) std::swap(ctx->cur, ctx->prev);
        }
    } else {
        for (long long step = 1; step <= nsteps; ++step) {
            const StepCoef& k = step <= p->n_apt ? ka : kp;
            if (t.n == 1 || use_peer(ctx)) {
                // one context (its halo, peer or NCCL, inside), or a group whose fused
                // steps store their boundary planes into the neighbours' ghosts
                for (int i = 0; i < t.n; ++i) {
                    CK(cudaSetDevice(t.c[i]->device));
                    if (int rc = hybrid_step(t.c[i], k, step, nsteps)) return rc;
                }
            } else {
                // group, other kernels: step every slab, then pull the ghost planes
                for (int i = 0; i < t.n; ++i) {
                    petto_ctx* x = t.c[i];
                    CK(cudaSetDevice(x->device));
                    // the buffer written now was read by the neighbours' pulls of the last step
                    for (petto_ctx* nb : {x->nb_lo, x->nb_hi})
                        if (nb) CK(cudaStreamWaitEvent(x->stream, nb->ev_pull, 0));
                    if (int rc = state_step(x, k, x->cur, x->prev, x->st[x->prev], step, nsteps, false)) return rc;
                    std::swap(x->cur, x->prev);
                    CK(cudaEventRecord(x->ev_step, x->stream));
                }
                for (int i = 0; i < t.n; ++i) {
                    CK(cudaSetDevice(t.c[i]->device));
                    if (int rc = group_pull(t.c[i], t.c[i]->cur)) return rc;
                }
            }
            // check_finite cadence (state_solver.hpp:490): every slab learns the
            // first non-finite step of any slab at each check, so all skip alike
            if (t.split() && step % 100 == 0 && step < nsteps)
                if (int rc = team_reduce(t, first_bad, 1, RED_MIN_I64)) return rc;
        }
    }
    if (int rc = team_reduce(t, first_bad, 1, RED_MIN_I64)) return rc;
    long long fb = PETTO_NO_BAD;
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* x = t.c[i];
        CK(cudaSetDevice(x->device));
        if (int rc = read_status(x)) return rc;
        fb = std::min(fb, x->status_h->first_bad);
    }
    if (fb != PETTO_NO_BAD) {
        const long long at = std::min(((fb + 99) / 100) * 100, nsteps);
        // the kernels after `at` were skipped: the buffers still hold the state of
        // step `at`, but the cur/prev indices advanced past it -- rewind the swaps
        const std::string msg = "numerical abort in 'state' at step " + std::to_string(at) +
                                ": non-finite values (time step too large?)";
        for (int i = 0; i < t.n; ++i) {
            if ((nsteps - at) % 2) std::swap(t.c[i]->cur, t.c[i]->prev);
            fail(t.c[i], PETTO_ABORT, msg);
        }
        if (abort_step) *abort_step = at;
        return PETTO_ABORT;
    }
    return PETTO_OK;
}

// residual + residual_norm (state_solver.hpp:49-58, 327-385): sqrt(sum r^2) / N
int team_residual(Team t, double* r_pde) {
    Range nv("petto.residual");
    if (int rc = team_check(t)) return rc;
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        if (int rc = require_ready(ctx)) return rc;
        if (int rc = check_kappa(ctx)) return rc;
        if (int rc = reset_status(ctx)) return rc;
        const StepCoef k = coef(3, 0.0, 1.0);
        if (int rc = state_step(ctx, k, ctx->cur, ctx->prev, ctx->r, 0, 0, !t.replica())) return rc;
        if (!t.replica()) {
            k_sum_to<<<1, 256, 0, ctx->stream>>>(ctx->partials, ctx->npartials_used, &ctx->status->sumsq);
            ctx->launches++;
            CKL();
        }
    }
    auto sumsq = [](petto_ctx* x) -> double* { return &x->status->sumsq; };
    if (t.replica()) {
        // entry order c*N + node: component after component, each over the slabs
        if (int rc = team_chain(
                t, t.lead()->comps,
                [](petto_ctx* ctx, int c, const double* init, double* out) {
                    k_sumsq_serial<<<1, 32, 0, ctx->stream>>>(ctx->g, ctx->comps, ctx->r, out, c, init);
                    ctx->launches++;
                    CKL();
                    return PETTO_OK;
                },
                sumsq))
            return rc;
    } else if (int rc = team_reduce(t, [&](petto_ctx* x) -> void* { return sumsq(x); }, 1, RED_SUM)) {
        return rc;
    }
    petto_ctx* ctx = t.lead();
    CK(cudaSetDevice(ctx->device));
    if (int rc = read_status(ctx)) return rc;
    if (r_pde) *r_pde = std::sqrt(ctx->status_h->sumsq) / (double)global_nodes(ctx);
    return PETTO_OK;
}

// iterate_to_tolerance (state_solver.hpp:511-541): step, re-evaluate the residual,
// stop below the absolute target -- the stop test on the device (k_iter_finish),
// the host reading the status once per chunk of steps.  On slabs the r^2 of every
// step is reduced over the slabs (REPLICA: the serial sum chained across them) and
// the new state's ghost planes are exchanged before the next step.
int team_iterate_to_tolerance(Team t, int mode, const petto_pt_params* p, double target, long max_iters,
                              petto_solve_stats* stats) {
    if (int rc = team_check(t)) return rc;
    Range nv("petto.iterate_to_tolerance");
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        if (int rc = require_ready(ctx)) return rc;
        if (int rc = check_kappa(ctx)) return rc;
        if (int rc = reset_status(ctx)) return rc;
        ctx->status_h->target = target;
        ctx->status_h->max_iters = max_iters;
        CK(cudaMemcpyAsync(ctx->status, ctx->status_h, sizeof(DeviceStatus), cudaMemcpyHostToDevice, ctx->stream));
    }
    petto_ctx* ctx = t.lead();
    // u_k lives in b[k % 3] (the same rotation on every slab)
    std::vector<std::array<int, 3>> b(t.n);
    for (int i = 0; i < t.n; ++i) b[i] = {t.c[i]->cur, 3 - t.c[i]->cur - t.c[i]->prev, t.c[i]->prev};
    const StepCoef k = mode == 0 ? coef(2, p->dt_pt, p->theta) : coef(p->form ? 1 : 0, p->dt_apt, p->theta);
    const long long never = LLONG_MAX;
    auto sumsq = [](petto_ctx* x) -> double* { return &x->status->sumsq; };
    long long launched = 0;  // residual evaluations issued
    long long chunk = 32;
    const bool persist = t.n == 1 && persistent_3d_ok(ctx);
    while (persist) {
        // persistent launches of up to 16384 iterations, the stop test inside
        const long long n = std::min<long long>(max_iters + 1 - launched, 16384);
        if (int rc = e3_launch(ctx, k, 0, 0, ctx->st[b[0][1]], launched, never, ctx->partials, (int)n, b[0].data()))
            return rc;
        launched += n;
        if (int rc = read_status(ctx)) return rc;
        if (ctx->status_h->done || launched > max_iters) break;
    }
    while (!persist) {
        for (long long c = 0; c < chunk && launched <= max_iters; ++c, ++launched) {
            const long long it = launched;
            for (int i = 0; i < t.n; ++i) {
                petto_ctx* x = t.c[i];
                CK(cudaSetDevice(x->device));
                if (int rc = state_step(x, k, b[i][it % 3], b[i][(it + 2) % 3], x->st[b[i][(it + 1) % 3]], it + 1,
                                        never, true))
                    return rc;
            }
            if (!t.split()) {  // one domain: the partials straight into the stop test
                k_iter_finish<<<1, 256, 0, ctx->stream>>>(ctx->status, t.replica() ? nullptr : ctx->partials,
                                                          ctx->npartials_used);
                ctx->launches++;
                CKL();
                continue;
            }
            if (t.replica()) {
                if (int rc = team_chain(
                        t, ctx->comps,
                        [](petto_ctx* ctx, int cc, const double* init, double* out) {
                            k_sumsq_serial<<<1, 32, 0, ctx->stream>>>(ctx->g, ctx->comps, ctx->r, out, cc, init);
                            ctx->launches++;
                            CKL();
                            return PETTO_OK;
                        },
                        sumsq))
                    return rc;
            } else {
                for (int i = 0; i < t.n; ++i) {
                    petto_ctx* x = t.c[i];
                    CK(cudaSetDevice(x->device));
                    k_sum_to<<<1, 256, 0, x->stream>>>(x->partials, x->npartials_used, &x->status->sumsq);
                    x->launches++;
                }
                if (int rc = team_reduce(t, [&](petto_ctx* x) -> void* { return sumsq(x); }, 1, RED_SUM)) return rc;
            }
            for (int i = 0; i < t.n; ++i) {
                petto_ctx* x = t.c[i];
                CK(cudaSetDevice(x->device));
                k_iter_finish<<<1, 256, 0, x->stream>>>(x->status, nullptr, 0);
                x->launches++;
                CKL();
            }
            // the new state's ghost planes (u_{it+1} lives in b[(it+1) % 3])
            for (int i = 0; i < t.n; ++i) t.c[i]->cur = b[i][(it + 1) % 3];
            if (int rc = team_halo(t, [](petto_ctx* x) { return x->st[x->cur]; }, t.lead()->comps)) return rc;
        }
        CK(cudaSetDevice(ctx->device));
        if (int rc = read_status(ctx)) return rc;
        if (ctx->status_h->done || launched > max_iters) break;
        chunk = std::min<long long>(chunk * 2, 4096);
    }
    const DeviceStatus s = *ctx->status_h;
    const long long n = s.iterations;
    for (int i = 0; i < t.n; ++i) {
        t.c[i]->cur = b[i][n % 3];
        t.c[i]->prev = b[i][(n + 2) % 3];
    }
    stats->iterations = (long)n;
    stats->r_initial = s.r_initial;
    stats->r_final = s.r_final;
    stats->converged = s.converged;
    if (s.aborted) {
        for (int i = 0; i < t.n; ++i)
            fail(t.c[i], PETTO_ABORT,
                 "numerical abort in 'state' at step " + std::to_string(n) + ": residual norm diverged");
        return PETTO_ABORT;
    }
    return PETTO_OK;
}

// ------------------------------------------------------------ design loop

int team_require_design(Team t, bool need_state) {
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        if (!ctx->design_set) return fail(ctx, PETTO_INVALID, "design not set (petto_dev_set_design)");
        if (need_state && !ctx->state_set) return fail(ctx, PETTO_INVALID, "state not set");
    }
    return team_check(t);
}

long long owned_of(petto_ctx* x) { return owned_nodes(x); }

// phase_mass per phase (phase_field.hpp:83-102) into dscal[slot + q]
int team_phase_masses(Team t, int slot) {
    for (int q = 0; q < t.lead()->mat.nphases; ++q) {
        if (!t.replica()) {  // block partials straight from phi (no term array)
            for (int i = 0; i < t.n; ++i) {
                petto_ctx* ctx = t.c[i];
                CK(cudaSetDevice(ctx->device));
                k_mass_partials<<<sum_grid(ctx), 256, 0, ctx->stream>>>(ctx->g, ctx->phases + q * ctx->g.Ns,
                                                                        ctx->pmax);
                ctx->launches++;
                CKL();
            }
            if (int rc = team_sum_partials(t, [](petto_ctx* x) { return x->pmax; }, sum_grid,
                                           [&](petto_ctx* x) { return x->dscal + slot + q; }))
                return rc;
            continue;
        }
        for (int i = 0; i < t.n; ++i) {
            petto_ctx* ctx = t.c[i];
            CK(cudaSetDevice(ctx->device));
            k_term_mass<<<blocks_for(owned_nodes(ctx)), 256, 0, ctx->stream>>>(ctx->g, ctx->phases + q * ctx->g.Ns,
                                                                               ctx->term1);
            ctx->launches++;
            CKL();
        }
        if (int rc = team_sum_terms(t, [](petto_ctx* x) { return x->term1; }, owned_of,
                                    [&](petto_ctx* x) { return x->dscal + slot + q; }))
            return rc;
    }
    return PETTO_OK;
}

// region volume and per-phase region masses (objectives.hpp:251-288), list order
int team_region_sums(Team t) {
    if (!t.lead()->tgt.has_region) return PETTO_OK;
    auto len = [](petto_ctx* x) { return (long long)x->region_nodes.size(); };
    for (int q = -1; q < t.lead()->mat.nphases; ++q) {
        for (int i = 0; i < t.n; ++i) {
            petto_ctx* ctx = t.c[i];
            CK(cudaSetDevice(ctx->device));
            k_region_terms<<<blocks_for(len(ctx)), 256, 0, ctx->stream>>>(
                ctx->g, ctx->region_dev, len(ctx), q < 0 ? nullptr : ctx->phases + q * ctx->g.Ns, ctx->term1);
            ctx->launches++;
            CKL();
        }
        if (int rc = team_sum_terms(t, [](petto_ctx* x) { return x->term1; }, len,
                                    [&](petto_ctx* x) { return x->dscal + (q < 0 ? DS_RVOL : DS_RACC + q); }))
            return rc;
    }
    return PETTO_OK;
}

// interpolate_into (objectives.hpp:95-116) over every stored plane (the ghost
// planes too: the operator reads the property of the cells across a slab face)
int team_interpolate(Team t) {
    Range nv("petto.interpolate");
    if (int rc = team_require_design(t, false)) return rc;
    if (int rc = team_phase_ghosts(t)) return rc;
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* ctx = t.c[i];
        CK(cudaSetDevice(ctx->device));
        const long long n = (long long)ctx->g.nx * ctx->g.ny * ctx->g.nzs;
        k_interpolate<<<blocks_for(n), 256, 0, ctx->stream>>>(ctx->g, design_params(ctx), ctx->phases, ctx->prop);
        ctx->launches++;
        CKL();
        ctx->ecell_valid = false;
        ctx->prop_node0_valid = false;
        ctx->prop_is_mu = false;
    }
    return PETTO_OK;
}

// The elasticity operator's nu comes from node 0's Lame pair (state_solver.hpp:
// 299-301); node 0 lives on the first slab, whose value every slab takes.
int team_init_operator(Team t) {
    petto_ctx* ctx = t.lead();
    if (ctx->desc.physics == 1) {
        double e0 = 0.0;
        CK(cudaSetDevice(ctx->device));
        if (t.nccl() && ctx->nranks > 1) {
            if (ctx->rank == 0)
                CK(cudaMemcpyAsync(ctx->dscal + DS_CHAIN_IN, ctx->prop + lidx(ctx->g, 0, 0, 0), 8,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
            if (int rc = nccl_check(ctx, nccl().Broadcast(ctx->dscal + DS_CHAIN_IN, ctx->dscal + DS_CHAIN_IN, 1,
                                                          ncclDouble, 0, static_cast<ncclComm_t>(ctx->nccl_comm),
                                                          ctx->stream), "node-0 broadcast"))
                return rc;
            CK(cudaMemcpyAsync(ctx->hpin, ctx->dscal + DS_CHAIN_IN, 8, cudaMemcpyDeviceToHost, ctx->stream));
        } else {
            CK(cudaMemcpyAsync(ctx->hpin, ctx->prop + lidx(ctx->g, 0, 0, 0), 8, cudaMemcpyDeviceToHost, ctx->stream));
        }
        CK(cudaStreamSynchronize(ctx->stream));
        e0 = ctx->hpin[0];
        for (int i = 0; i < t.n; ++i) {
            t.c[i]->prop_node0 = e0;
            t.c[i]->prop_node0_valid = true;
        }
    }
    for (int i = 0; i < t.n; ++i)
        if (int rc = petto_dev_init_operator(t.c[i])) return rc;
    return PETTO_OK;
}

// sensitivities (objectives.hpp:336-439) + design_update_inplace (:444-480)
int team_design_update(Team t) {
    Range nv("petto.design_update");
    if (int rc = team_require_design(t, true)) return rc;
    petto_ctx* ctx = t.lead();
    const DesignP d = design_params(ctx);
    if (int rc = team_phase_masses(t, DS_MASS)) return rc;  // volume_fractions of the pre-update design
    if (int rc = team_region_sums(t)) return rc;
    const double nu = ctx->mat.poisson_ratio;
    const double ctr = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double cec = 1.0 / (1.0 + nu);
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* x = t.c[i];
        CK(cudaSetDevice(x->device));
        int nb = (int)std::min<long long>(x->npartials, blocks_for(owned_nodes(x)));
        if (x->g.dim == 3 && d.np <= 4) {
            // z-streamed (every node of u read once), one block per 32 x 4 columns x SENS_ZC planes
            const dim3 grid3 = sens_grid(x), blk(32, 4);
            nb = (int)(grid3.x * grid3.y * grid3.z);
            auto launch = [&](auto np_c, auto kind_c) {
                k_sens_gc3<decltype(np_c)::value, decltype(kind_c)::value><<<grid3, blk, 0, x->stream>>>(
                    x->g, d, ctr, cec, x->phases, x->st[x->cur], x->gc, x->pmax, SENS_ZC);
            };
            auto by_kind = [&](auto np_c) {
                if (x->mat.kind == 0) launch(np_c, std::integral_constant<int, 0>{});
                else launch(np_c, std::integral_constant<int, 1>{});
            };
            switch (d.np) {
                case 1: by_kind(std::integral_constant<int, 1>{}); break;
                case 2: by_kind(std::integral_constant<int, 2>{}); break;
                case 3: by_kind(std::integral_constant<int, 3>{}); break;
                default: by_kind(std::integral_constant<int, 4>{}); break;
            }
        } else if (x->g.dim == 3) {
            k_sens_gc<3><<<nb, 256, 0, x->stream>>>(x->g, d, x->mat.kind, ctr, cec, x->phases, x->st[x->cur], x->gc,
                                                    x->pmax);
        } else {
            k_sens_gc<2><<<nb, 256, 0, x->stream>>>(x->g, d, x->mat.kind, ctr, cec, x->phases, x->st[x->cur], x->gc,
                                                    x->pmax);
        }
        k_local_gmax<<<1, 32 * d.np, 0, x->stream>>>(d.np, x->pmax, nb, x->dscal);
        x->launches += 2;
        if (cudaGetLastError() != cudaSuccess) return fail(x, PETTO_ERROR, "sensitivity launch failed");
    }
    // max_abs_nodes over the whole grid (parallel.hpp:33-42, objectives.hpp:459-461)
    if (int rc = team_reduce(t, [](petto_ctx* x) -> void* { return x->dscal + DS_GMAX; }, d.np, RED_MAX)) return rc;
    UpdateScal u{};
    u.inv_vol = 1.0 / domain_volume(ctx);
    for (int q = 0; q < d.np; ++q) {
        u.fractions[q] = ctx->tgt.fractions[q];
        u.region_fractions[q] = ctx->tgt.region_fractions[q];
    }
    u.has_region = ctx->tgt.has_region;
    u.alpha_c = ctx->wts.alpha_compliance;
    u.alpha_v = ctx->wts.alpha_volume;
    u.alpha_u = ctx->wts.alpha_unity;
    u.alpha_r = ctx->wts.alpha_region;
    u.normalize = ctx->wts.normalize_compliance;
    u.sign = ctx->wts.compliance_sign;
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* x = t.c[i];
        CK(cudaSetDevice(x->device));
        k_design_scalars<<<1, 32, 0, x->stream>>>(d.np, u, x->dscal);
        const int nbu = blocks_for(owned_nodes(x));
        switch (d.np) {
#define PETTO_UPD(NP)                                                                                   \
    case NP:                                                                                            \
        k_design_update<NP><<<nbu, 256, 0, x->stream>>>(x->g, u, x->dscal, x->gc, x->region_mask, x->phases); \
        break;
            PETTO_UPD(1) PETTO_UPD(2) PETTO_UPD(3) PETTO_UPD(4) PETTO_UPD(5) PETTO_UPD(6) PETTO_UPD(7) PETTO_UPD(8)
#undef PETTO_UPD
        }
        x->launches += 2;
        if (cudaGetLastError() != cudaSuccess) return fail(x, PETTO_ERROR, "design update launch failed");
        x->phi_ghosts_stale = true;
    }
    return PETTO_OK;
}

// ch_step_multi_inplace (phase_field.hpp:136-176): per phase, mass before, mu on
// the owned planes from phi with fresh ghosts, phi += dt D lap(mu) with fresh mu
// ghosts (the 2-plane footprint as two 1-plane exchanges), mass pre, clamp, mass post
int team_ch_step(Team t, const petto_ch_params* p, petto_ch_stats* stats) {
    Range nv("petto.ch_step");
    if (int rc = team_require_design(t, false)) return rc;
    petto_ctx* ctx = t.lead();
    // CahnHilliardParams::validate (phase_field.hpp:17-21)
    if (!(p->mobility > 0.0)) return fail(ctx, PETTO_INVALID, "cahn-hilliard: mobility must be positive");
    if (!(p->gamma > 0.0)) return fail(ctx, PETTO_INVALID, "cahn-hilliard: gamma must be positive");
    if (!(p->dt > 0.0)) return fail(ctx, PETTO_INVALID, "cahn-hilliard: dt must be positive");
    const double step = p->dt * p->mobility;
    auto term1 = [](petto_ctx* x) { return x->term1; };
    for (int q = 0; q < ctx->mat.nphases; ++q) {
        auto phi = [q](petto_ctx* x) { return x->phases + q * x->g.Ns; };
        auto slot = [q](int k) { return [q, k](petto_ctx* x) { return x->dscal + DS_CH + 3 * q + k; }; };
        if (!t.replica()) {
            // FAST: two passes per phase -- mu + mass before, then update + clamp +
            // both masses -- with the sums as block partials (bit-identical to the
            // term-array route, a third of the HBM traffic)
            auto part = [](int k) { return [k](petto_ctx* x) { return x->pmax + k * x->npartials; }; };
            if (t.split())
                if (int rc = team_halo(t, phi, 1)) return rc;
            for (int i = 0; i < t.n; ++i) {
                petto_ctx* x = t.c[i];
                CK(cudaSetDevice(x->device));
                k_chem_potential_mass<<<sum_grid(x), 256, 0, x->stream>>>(x->g, phi(x), p->gamma, x->scratch1,
                                                                           part(0)(x));
                x->launches++;
            }
            if (int rc = team_sum_partials(t, part(0), sum_grid, slot(0))) return rc;
            if (t.split())
                if (int rc = team_halo(t, [](petto_ctx* x) { return x->scratch1; }, 1)) return rc;
            for (int i = 0; i < t.n; ++i) {
                petto_ctx* x = t.c[i];
                CK(cudaSetDevice(x->device));
                k_ch_update_clamp<<<sum_grid(x), 256, 0, x->stream>>>(x->g, x->scratch1, step, phi(x), part(1)(x),
                                                                       part(2)(x), &x->status->flags);
                x->launches++;
                if (cudaGetLastError() != cudaSuccess) return fail(x, PETTO_ERROR, "cahn-hilliard launch failed");
            }
            if (int rc = team_sum_partials(t, part(1), sum_grid, slot(1))) return rc;
            if (int rc = team_sum_partials(t, part(2), sum_grid, slot(2))) return rc;
            continue;
        }
        for (int i = 0; i < t.n; ++i) {
            petto_ctx* x = t.c[i];
            CK(cudaSetDevice(x->device));
            k_term_mass<<<blocks_for(owned_nodes(x)), 256, 0, x->stream>>>(x->g, phi(x), x->term1);
            x->launches++;
        }
        if (int rc = team_sum_terms(t, term1, owned_of, slot(0))) return rc;
        if (t.split())
            if (int rc = team_halo(t, phi, 1)) return rc;
        for (int i = 0; i < t.n; ++i) {
            petto_ctx* x = t.c[i];
            CK(cudaSetDevice(x->device));
            k_chem_potential<<<blocks_for(owned_nodes(x)), 256, 0, x->stream>>>(x->g, phi(x), p->gamma, x->scratch1);
            x->launches++;
        }
        if (t.split())
            if (int rc = team_halo(t, [](petto_ctx* x) { return x->scratch1; }, 1)) return rc;
        for (int i = 0; i < t.n; ++i) {
            petto_ctx* x = t.c[i];
            CK(cudaSetDevice(x->device));
            k_ch_update<<<blocks_for(owned_nodes(x)), 256, 0, x->stream>>>(x->g, x->scratch1, step, phi(x), x->term1);
            x->launches++;
        }
        if (int rc = team_sum_terms(t, term1, owned_of, slot(1))) return rc;
        for (int i = 0; i < t.n; ++i) {
            petto_ctx* x = t.c[i];
            CK(cudaSetDevice(x->device));
            k_ch_clamp<<<blocks_for(owned_nodes(x)), 256, 0, x->stream>>>(x->g, phi(x), x->term1, &x->status->flags);
            x->launches++;
            if (cudaGetLastError() != cudaSuccess) return fail(x, PETTO_ERROR, "cahn-hilliard launch failed");
        }
        if (int rc = team_sum_terms(t, term1, owned_of, slot(2))) return rc;
    }
    for (int i = 0; i < t.n; ++i) t.c[i]->phi_ghosts_stale = true;
    if (stats) {
        double* h = ctx->hpin;
        CK(cudaSetDevice(ctx->device));
        CK(cudaMemcpyAsync(h, ctx->dscal + DS_CH, sizeof(double) * 3 * ctx->mat.nphases, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (int q = 0; q < ctx->mat.nphases; ++q) {
            stats[q].mass_before = h[3 * q];
            stats[q].mass_preclamp = h[3 * q + 1];
            stats[q].mass_postclamp = h[3 * q + 2];
        }
    }
    return PETTO_OK;
}

// evaluate_objectives (objectives.hpp:304-320) + the separation metric
// (optimizer.hpp:95-112) of the current design and state
int team_objectives(Team t, petto_report* rep, double* separation) {
    Range nv("petto.objectives");
    if (int rc = team_require_design(t, true)) return rc;
    petto_ctx* ctx = t.lead();
    const int np = ctx->mat.nphases;
    const double nu = ctx->mat.poisson_ratio;
    const double cl = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double cm = 1.0 / (2.0 * (1.0 + nu));
    for (int i = 0; i < t.n; ++i) {
        petto_ctx* x = t.c[i];
        CK(cudaSetDevice(x->device));
        CK(cudaMemsetAsync(x->count, 0, sizeof(unsigned long long), x->stream));
        if (x->g.dim == 3)
            k_objective_terms<3><<<blocks_for(owned_nodes(x)), 256, 0, x->stream>>>(
                x->g, design_params(x), x->mat.kind, cl, cm, x->phases, x->st[x->cur], x->term1, x->term2, x->count);
        else
            k_objective_terms<2><<<blocks_for(owned_nodes(x)), 256, 0, x->stream>>>(
                x->g, design_params(x), x->mat.kind, cl, cm, x->phases, x->st[x->cur], x->term1, x->term2, x->count);
        x->launches++;
        if (cudaGetLastError() != cudaSuccess) return fail(x, PETTO_ERROR, "objective launch failed");
    }
    if (int rc = team_sum_terms(t, [](petto_ctx* x) { return x->term1; }, owned_of,
                                [](petto_ctx* x) { return x->dscal + DS_OBJ; }))
        return rc;
    if (int rc = team_sum_terms(t, [](petto_ctx* x) { return x->term2; }, owned_of,
                                [](petto_ctx* x) { return x->dscal + DS_OBJ + 1; }))
        return rc;
    if (int rc = team_reduce(t, [](petto_ctx* x) -> void* { return x->count; }, 1, RED_SUM_U64)) return rc;
    if (int rc = team_phase_masses(t, DS_TMP)) return rc;
    if (int rc = team_region_sums(t)) return rc;
    double* h = ctx->hpin;
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(h, ctx->dscal, sizeof(double) * DS_COUNT, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(h + DS_COUNT, ctx->count, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    unsigned long long cnt;
    std::memcpy(&cnt, h + DS_COUNT, sizeof(cnt));
    // scalar parts on the host, as the reference forms them
    const double inv_vol = 1.0 / domain_volume(ctx);
    petto_report r{};
    r.compliance = h[DS_OBJ];
    r.unity = h[DS_OBJ + 1];
    double jv = 0.0;
    for (int q = 0; q < np; ++q) {
        r.volume_fractions[q] = h[DS_TMP + q] * inv_vol;
        const double dd = r.volume_fractions[q] - ctx->tgt.fractions[q];
        jv += dd * dd;
    }
    r.volume = jv;
    r.region = 0.0;
    if (ctx->tgt.has_region) {
        double jr = 0.0;
        for (int q = 0; q < np; ++q) {
            const double dd = h[DS_RACC + q] / h[DS_RVOL] - ctx->tgt.region_fractions[q];
            jr += dd * dd;
        }
        r.region = jr;
    }
    if (rep) *rep = r;
    if (separation) *separation = (double)cnt / (double)global_nodes(ctx);
    return PETTO_OK;
}

// run() (optimizer.hpp:120-223): the coupled loop with every field resident in HBM;
// the host only sees scalars (records, CH mass stats, abort flags).
int team_run(Team t, const petto_schedule* s, petto_record_cb cb, void* user, petto_run_result* result) {
    petto_ctx* ctx = t.lead();
    CK(cudaSetDevice(ctx->device));
    // LoopSchedule::validate (optimizer.hpp:23-33)
    if (int rc = validate_params(ctx, &s->pt)) return rc;
    if (!(s->ch.mobility > 0.0)) return fail(ctx, PETTO_INVALID, "cahn-hilliard: mobility must be positive");
    if (!(s->ch.gamma > 0.0)) return fail(ctx, PETTO_INVALID, "cahn-hilliard: gamma must be positive");
    if (!(s->ch.dt > 0.0)) return fail(ctx, PETTO_INVALID, "cahn-hilliard: dt must be positive");
    if (s->max_loops < 1) return fail(ctx, PETTO_INVALID, "schedule: max_loops must be >= 1");
    if (!(s->convergence_tol > 0.0))
        return fail(ctx, PETTO_INVALID, "schedule: convergence tolerance must be positive");
    if (s->convergence_window < 2) return fail(ctx, PETTO_INVALID, "schedule: convergence window must be >= 2");
    if (s->report_every < 1) return fail(ctx, PETTO_INVALID, "schedule: report_every must be >= 1");
    if (int rc = team_require_design(t, true)) return rc;
    if (int rc = validate_design(ctx, &ctx->mat, &ctx->wts)) return rc;

    petto_run_result res{};
    // operator construction on the initial design (optimizer.hpp:131-138)
    if (int rc = team_interpolate(t)) return rc;
    if (int rc = team_init_operator(t)) return rc;
    std::vector<double> comp_hist;
    const auto t0 = std::chrono::steady_clock::now();
    res.termination = 1;
    std::vector<petto_ch_stats> chs(ctx->mat.nphases);
    auto flags = [](petto_ctx* x) -> void* { return &x->status->flags; };
    for (long loop = 1; loop <= s->max_loops; ++loop) {
        Range nv("petto.loop");
        res.loops = loop;
        if (int rc = team_interpolate(t)) return rc;
        int64_t astep = 0;
        int rc = team_hybrid_solve(t, &s->pt, &astep);
        if (rc == PETTO_ABORT) {
            res.termination = 2;
            std::snprintf(res.abort_detail, sizeof res.abort_detail, "loop %ld: %s", loop, ctx->err.c_str());
            break;
        }
        if (rc) return rc;
        res.apt_steps += s->pt.n_apt;
        res.pt_steps += s->pt.n_pt;
        if ((rc = team_design_update(t))) return rc;
        ++res.design_updates;
        for (int i = 0; i < t.n; ++i) {
            petto_ctx* x = t.c[i];
            CK(cudaSetDevice(x->device));
            CK(cudaMemsetAsync(&x->status->flags, 0, sizeof(unsigned), x->stream));
        }
        if ((rc = team_ch_step(t, &s->ch, chs.data()))) return rc;
        ++res.ch_steps;
        for (const petto_ch_stats& st : chs) res.clamp_mass_drift += std::abs(st.mass_postclamp - st.mass_preclamp);
        // all_finite of the phases (optimizer.hpp:203-205), any slab
        if ((rc = team_reduce(t, flags, 1, RED_MAX_U32))) return rc;
        CK(cudaSetDevice(ctx->device));
        if ((rc = read_status(ctx))) return rc;
        if (ctx->status_h->flags & 4u) {
            res.termination = 2;
            std::snprintf(res.abort_detail, sizeof res.abort_detail,
                          "loop %ld: numerical abort in 'phi' at step %ld: design field turned non-finite", loop,
                          loop);
            break;
        }
        if (loop % s->report_every == 0 || loop == 1 || loop == s->max_loops) {
            petto_record rec{};
            petto_report rep{};
            double sep = 0.0;
            if ((rc = team_objectives(t, &rep, &sep))) return rc;
            rec.loop = loop;
            rec.apt_steps = res.apt_steps;
            rec.pt_steps = res.pt_steps;
            rec.compliance = rep.compliance;
            rec.volume = rep.volume;
            rec.unity = rep.unity;
            rec.region = rep.region;
            for (int q = 0; q < ctx->mat.nphases; ++q) rec.volume_fractions[q] = rep.volume_fractions[q];
            // the operator sees the property of the updated design (optimizer.hpp:157-162)
            if ((rc = team_interpolate(t))) return rc;
            if ((rc = team_residual(t, &rec.r_pde))) return rc;
            rec.separation = sep;
            rec.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            comp_hist.push_back(rec.compliance);
            if (cb) cb(&rec, user);
            // converged() (optimizer.hpp:170-181)
            const int w = s->convergence_window;
            if ((int)comp_hist.size() >= w) {
                double lo = comp_hist.back(), hi = lo;
                for (int i = 0; i < w; ++i) {
                    const double v = comp_hist[comp_hist.size() - 1 - i];
                    lo = std::min(lo, v);
                    hi = std::max(hi, v);
                }
                const double scale = std::max(std::abs(hi), 1e-300);
                if ((hi - lo) / scale < s->convergence_tol) {
                    res.termination = 0;
                    break;
                }
            }
        }
    }
    if (result) *result = res;
    return PETTO_OK;
}

}  // namespace

// ----------------------------------------------------- C-ABI over the teams

int petto_dev_hybrid_solve(petto_ctx* ctx, const petto_pt_params* p, int64_t* abort_step) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = solo_ok(ctx, true)) return rc;
    return team_hybrid_solve(Team{&ctx, 1}, p, abort_step);
}

int petto_dev_iterate_to_tolerance(petto_ctx* ctx, int mode, const petto_pt_params* p, double target,
                                   long max_iters, petto_solve_stats* stats) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = solo_ok(ctx, false)) return rc;
    return team_iterate_to_tolerance(Team{&ctx, 1}, mode, p, target, max_iters, stats);
}

int petto_dev_group_iterate_to_tolerance(petto_ctx** c, int n, int mode, const petto_pt_params* p, double target,
                                         long max_iters, petto_solve_stats* stats) {
    return team_iterate_to_tolerance(Team{c, n}, mode, p, target, max_iters, stats);
}

int petto_dev_residual(petto_ctx* ctx, double* out, double* r_pde) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = solo_ok(ctx, false)) return rc;
    if (int rc = team_residual(Team{&ctx, 1}, r_pde)) return rc;
    if (out) {
        if (int rc = download(ctx, out, ctx->r, ctx->comps, true)) return rc;
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return PETTO_OK;
}

int petto_dev_interpolate(petto_ctx* ctx, double* property_out) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = solo_ok(ctx, false)) return rc;
    if (int rc = team_interpolate(Team{&ctx, 1})) return rc;
    if (property_out) {
        if (int rc = download(ctx, property_out, ctx->prop, 1)) return rc;
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return PETTO_OK;
}

int petto_dev_design_update(petto_ctx* ctx) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = solo_ok(ctx, false)) return rc;
    return team_design_update(Team{&ctx, 1});
}

int petto_dev_ch_step(petto_ctx* ctx, const petto_ch_params* p, petto_ch_stats* stats) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = solo_ok(ctx, false)) return rc;
    return team_ch_step(Team{&ctx, 1}, p, stats);
}

int petto_dev_objectives(petto_ctx* ctx, petto_report* rep, double* separation) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = solo_ok(ctx, false)) return rc;
    return team_objectives(Team{&ctx, 1}, rep, separation);
}

int petto_dev_run(petto_ctx* ctx, const petto_schedule* s, petto_record_cb cb, void* user,
                  petto_run_result* result) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = solo_ok(ctx, false)) return rc;
    return team_run(Team{&ctx, 1}, s, cb, user, result);
}

int petto_dev_group_hybrid_solve(petto_ctx** c, int n, const petto_pt_params* p, int64_t* abort_step) {
    return team_hybrid_solve(Team{c, n}, p, abort_step);
}

int petto_dev_group_residual(petto_ctx** c, int n, double* r_pde) { return team_residual(Team{c, n}, r_pde); }

int petto_dev_group_interpolate(petto_ctx** c, int n) { return team_interpolate(Team{c, n}); }

int petto_dev_group_init_operator(petto_ctx** c, int n) {
    if (int rc = team_check(Team{c, n})) return rc;
    return team_init_operator(Team{c, n});
}

int petto_dev_group_design_update(petto_ctx** c, int n) { return team_design_update(Team{c, n}); }

int petto_dev_group_ch_step(petto_ctx** c, int n, const petto_ch_params* p, petto_ch_stats* stats) {
    return team_ch_step(Team{c, n}, p, stats);
}

int petto_dev_group_objectives(petto_ctx** c, int n, petto_report* rep, double* separation) {
    return team_objectives(Team{c, n}, rep, separation);
}

int petto_dev_group_run(petto_ctx** c, int n, const petto_schedule* s, petto_record_cb cb, void* user,
                        petto_run_result* result) {
    return team_run(Team{c, n}, s, cb, user, result);
}

// ------------------------------------------------------------ slab decomposition

int petto_dev_comm_unique_id(void* id128) {
    std::string err;
    if (!nccl().load(err)) return fail(nullptr, PETTO_ERROR, err);
    ncclUniqueId id;
    if (nccl().GetUniqueId(&id) != ncclSuccess) return fail(nullptr, PETTO_ERROR, "ncclGetUniqueId failed");
    std::memcpy(id128, &id, sizeof(id));
    return PETTO_OK;
}

int petto_dev_comm_init(petto_ctx* ctx, const void* id128, int rank, int nranks) {
    CK(cudaSetDevice(ctx->device));
    std::string err;
    if (!nccl().load(err)) return fail(ctx, PETTO_ERROR, err);
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, PETTO_INVALID, "comm: bad rank / size");
    if ((rank > 0) != (ctx->g.kb > 0) || (rank < nranks - 1) != (ctx->g.ke < ctx->g.nz))
        return fail(ctx, PETTO_INVALID, "comm: the context's plane range does not match the rank order");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    if (int rc = nccl_check(ctx, nccl().CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank")) return rc;
    ctx->nccl_comm = comm;
    ctx->rank = rank;
    ctx->nranks = nranks;
    return PETTO_OK;
}

namespace {
struct PeerBlob {
    uint32_t magic;
    int32_t ks0, kb, ke;
    int64_t Ns;
    cudaIpcMemHandle_t st[3];
    cudaIpcMemHandle_t inbox;
};
static_assert(sizeof(PeerBlob) <= PETTO_PEER_BLOB_BYTES, "peer blob size");
constexpr uint32_t PEER_MAGIC = 0x50455452u;
}  // namespace

int petto_dev_peer_export(petto_ctx* ctx, void* blob) {
    CK(cudaSetDevice(ctx->device));
    if (int rc = peer_prepare(ctx)) return rc;
    PeerBlob b{};
    b.magic = PEER_MAGIC;
    b.ks0 = ctx->g.ks0;
    b.kb = ctx->g.kb;
    b.ke = ctx->g.ke;
    b.Ns = ctx->g.Ns;
    for (int i = 0; i < 3; ++i) CK(cudaIpcGetMemHandle(&b.st[i], ctx->st[i]));
    CK(cudaIpcGetMemHandle(&b.inbox, ctx->inbox));
    std::memset(blob, 0, PETTO_PEER_BLOB_BYTES);
    std::memcpy(blob, &b, sizeof(b));
    return PETTO_OK;
}

int petto_dev_peer_import(petto_ctx* ctx, const void* lo_blob, const void* hi_blob) {
    CK(cudaSetDevice(ctx->device));
    if (!ctx->inbox) return fail(ctx, PETTO_INVALID, "peer halo: call petto_dev_peer_export first");
    auto open = [&](petto_b200::PeerSlab& ps, const void* raw, bool lo) -> int {
        ps = petto_b200::PeerSlab{};
        if (!raw) return PETTO_OK;
        PeerBlob b;
        std::memcpy(&b, raw, sizeof(b));
        if (b.magic != PEER_MAGIC) return fail(ctx, PETTO_INVALID, "peer halo: not a peer blob");
        if ((lo && b.ke != ctx->g.kb) || (!lo && b.kb != ctx->g.ke))
            return fail(ctx, PETTO_INVALID, "peer halo: the neighbour's planes do not adjoin this slab");
        for (int i = 0; i < 3; ++i) {
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, b.st[i], cudaIpcMemLazyEnablePeerAccess));
            ps.st[i] = static_cast<double*>(p);
        }
        void* q = nullptr;
        CK(cudaIpcOpenMemHandle(&q, b.inbox, cudaIpcMemLazyEnablePeerAccess));
        ps.ipc = true;
        ps.ipc_inbox = static_cast<unsigned long long*>(q);
        ps.flag = ps.ipc_inbox + (lo ? 1 : 0);  // our slot in the neighbour's inbox
        ps.Ns = b.Ns;
        ps.ks0 = b.ks0;
        return PETTO_OK;
    };
    if (int rc = open(ctx->peer_lo, lo_blob, true)) return rc;
    if (int rc = open(ctx->peer_hi, hi_blob, false)) return rc;
    ctx->peer_halo = lo_blob || hi_blob;
    ctx->peer_seq = 0;
    return PETTO_OK;
}

int petto_dev_group_link(petto_ctx** c, int n) {
    for (int i = 0; i < n; ++i) {
        petto_ctx* x = c[i];
        petto_ctx* ctx = x;  // error sink of CK()
        if (i + 1 < n && (x->g.ke != c[i + 1]->g.kb || x->g.nx != c[i + 1]->g.nx || x->g.ny != c[i + 1]->g.ny))
            return fail(x, PETTO_INVALID, "group: contexts must hold consecutive slabs of one grid");
        x->nb_lo = i > 0 ? c[i - 1] : nullptr;
        x->nb_hi = i + 1 < n ? c[i + 1] : nullptr;
        x->rank = i;
        x->nranks = n;
        CK(cudaSetDevice(x->device));
        if (!x->ev_step) CK(cudaEventCreateWithFlags(&x->ev_step, cudaEventDisableTiming));
        if (!x->ev_pull) CK(cudaEventCreateWithFlags(&x->ev_pull, cudaEventDisableTiming));
        if (!x->ev_team) CK(cudaEventCreateWithFlags(&x->ev_team, cudaEventDisableTiming));
        CK(cudaEventRecord(x->ev_step, x->stream));
        CK(cudaEventRecord(x->ev_pull, x->stream));
        if (int rc = peer_prepare(x)) return rc;
        for (petto_ctx* nb : {x->nb_lo, x->nb_hi}) {
            if (!nb || nb->device == x->device) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, x->device, nb->device);
            if (can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(nb->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                cudaGetLastError();
            }
        }
    }
    // peer halo between the group's slabs: direct pointers (same process)
    for (int i = 0; i < n; ++i) {
        petto_ctx* ctx = c[i];  // error sink of CK()
        CK(cudaSetDevice(ctx->device));
        CK(cudaDeviceSynchronize());
    }
    for (int i = 0; i < n; ++i) {
        petto_ctx* x = c[i];
        auto fill = [&](petto_b200::PeerSlab& ps, petto_ctx* nb, int slot) {
            ps = petto_b200::PeerSlab{};
            if (!nb) return;
            for (int b = 0; b < 3; ++b) ps.st[b] = nb->st[b];
            ps.Ns = nb->g.Ns;
            ps.ks0 = nb->g.ks0;
            ps.flag = nb->inbox + slot;
        };
        fill(x->peer_lo, x->nb_lo, 1);  // we are the lo neighbour's hi neighbour
        fill(x->peer_hi, x->nb_hi, 0);
        x->peer_halo = n > 1;
        x->peer_seq = 0;
    }
    return PETTO_OK;
}

void petto_dev_unit_cell_stiffness(int dim, const double h[3], double nu, double* ke) {
    const std::vector<double> K = unit_cell_stiffness(dim, h, nu);
    std::memcpy(ke, K.data(), sizeof(double) * K.size());
}

double petto_dev_spectral_bound(int dim, const int64_t n[3], const double length[3], double nu, double e_max) {
    double h[3] = {1.0, 1.0, 1.0};
    for (int a = 0; a < dim; ++a) h[a] = length[a] / (double)(n[a] - 1);
    return spectral_bound(dim, h, nu, e_max);
}

#ifdef E3_CTA_TIMING
// probe builds only: the last fused launch's per-CTA globaltimer start/end and SM id
int petto_dev_probe_cta_times(petto_ctx* ctx, uint64_t* out, int n) {
    if (!ctx->cta_probe) return fail(ctx, PETTO_INVALID, "no fused launch yet");
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(out, ctx->cta_probe, sizeof(uint64_t) * (size_t)n, cudaMemcpyDeviceToHost));
    return PETTO_OK;
}
#endif

int64_t petto_dev_launch_count(const petto_ctx* ctx) { return ctx->launches; }

int petto_dev_kernel_timing(petto_ctx* ctx, int enable) {
    CK(cudaSetDevice(ctx->device));
    if (enable && ctx->ev_pool.empty()) {
        ctx->ev_pool.resize(512);
        for (auto& e : ctx->ev_pool) CK(cudaEventCreate(&e));
    }
    ctx->timing = enable != 0;
    ctx->timing_stride = enable > 1 ? enable : 1;
    ctx->timing_seq = 0;
    ctx->kernel_ms = 0.0;
    ctx->kernel_launches = 0;
    ctx->ev_used = 0;
    return PETTO_OK;
}

int petto_dev_kernel_stats(petto_ctx* ctx, double* total_ms, int64_t* launches, double* bytes_per_launch,
                           char* name, int name_cap) {
    CK(cudaStreamSynchronize(ctx->stream));
    for (int e = 0; e + 1 < ctx->ev_used; e += 2) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev_pool[e], ctx->ev_pool[e + 1]));
        ctx->kernel_ms += ms;
    }
    ctx->ev_used = 0;
    if (total_ms) *total_ms = ctx->kernel_ms;
    if (launches) *launches = ctx->kernel_launches;
    if (bytes_per_launch) *bytes_per_launch = ctx->bytes_per_launch;
    if (name && name_cap > 0) std::snprintf(name, (size_t)name_cap, "%s", ctx->kernel_name.c_str());
    return PETTO_OK;
}


// ------------------------------------------------------------------ writers
// the reference's writers (field_io.cpp:29-126) from
// device buffers, byte-identical.  Values are formatted on the device
// (writers.cuh); chunks of WCHUNK values alternate between two text buffers so
// that the copy of chunk c and the host write of chunk c-1 overlap.

int petto_dev_format_values(petto_ctx* ctx, const double* values, int64_t n, int sep_mode, int64_t row,
                            char* out, int64_t cap, int64_t* len) {
    CK(cudaSetDevice(ctx->device));
    if (n < 0 || row <= 0 || (sep_mode != 0 && sep_mode != 1))
        return fail(ctx, PETTO_INVALID, "format_values: bad arguments");
    cudaPointerAttributes at{};
    const bool dev = cudaPointerGetAttributes(&at, values) == cudaSuccess && at.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    double* tmp = nullptr;
    if (!dev && n) {
        CK(cudaMalloc(&tmp, sizeof(double) * (size_t)n));
        CK(cudaMemcpyAsync(tmp, values, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (sep_mode == 1 && row > (1LL << 30)) return fail(ctx, PETTO_INVALID, "format_values: row too long");
    const long long nx = sep_mode == 1 ? row : (1LL << 20);  // the separator of mode 0 ignores rows
    const wr::Src src{dev ? values : tmp, (int)nx, 1, nx, nx, (long long)n};
    int64_t used = 0;
    const int rc = format_stream(ctx, src, sep_mode, [&](const char* p, size_t k) {
        if (used + (int64_t)k > cap) return fail(ctx, PETTO_INVALID, "format_values: output buffer too small");
        std::memcpy(out + used, p, k);
        used += (int64_t)k;
        return PETTO_OK;
    });
    cudaFree(tmp);
    if (len) *len = used;
    return rc;
}

int petto_dev_write_field_csv(petto_ctx* ctx, int field, int index, const char* path) {
    CK(cudaSetDevice(ctx->device));
    wr::Src src;
    if (int rc = writer_source(ctx, field, index, &src)) return rc;
    const Geo& g = ctx->g;
    OutFile o;
    if (int rc = open_out(ctx, o, path, false)) return rc;
    const std::string head = "# nx=" + std::to_string(g.nx) + " ny=" + std::to_string(g.ny) +
                             " nz=" + std::to_string(g.nz) + " dx=" + fmt17(g.h[0]) + " dy=" + fmt17(g.h[1]) +
                             " dz=" + fmt17(g.h[2]) + "\n";
    std::fwrite(head.data(), 1, head.size(), o.f);
    if (int rc = format_stream(ctx, src, 1, [&](const char* p, size_t k) {
            std::fwrite(p, 1, k, o.f);
            return PETTO_OK;
        }))
        return rc;
    return close_out(ctx, o, path);
}

int petto_dev_write_vtk(petto_ctx* ctx, const petto_array* arrays, int narrays, const char* path) {
    CK(cudaSetDevice(ctx->device));
    std::vector<wr::Src> src((size_t)std::max(narrays, 0));
    for (int a = 0; a < narrays; ++a)
        if (int rc = writer_source(ctx, arrays[a].field, arrays[a].index, &src[a])) return rc;
    const Geo& g = ctx->g;
    OutFile o;
    if (int rc = open_out(ctx, o, path, false)) return rc;
    const std::string head = "# vtk DataFile Version 3.0\nstructured point fields\nASCII\nDATASET STRUCTURED_POINTS\n"
                             "DIMENSIONS " + grid_dims(g) + "\nORIGIN 0 0 0\nSPACING " + fmt17(g.h[0]) + " " +
                             fmt17(g.h[1]) + " " + fmt17(g.h[2]) + "\nPOINT_DATA " +
                             std::to_string((long long)g.nx * g.ny * g.nz) + "\n";
    std::fwrite(head.data(), 1, head.size(), o.f);
    for (int a = 0; a < narrays; ++a) {
        const std::string sh = std::string("SCALARS ") + arrays[a].name + " double 1\nLOOKUP_TABLE default\n";
        std::fwrite(sh.data(), 1, sh.size(), o.f);
        if (int rc = format_stream(ctx, src[a], 0, [&](const char* p, size_t k) {
                std::fwrite(p, 1, k, o.f);
                return PETTO_OK;
            }))
            return rc;
    }
    return close_out(ctx, o, path);
}

int petto_dev_write_pgm(petto_ctx* ctx, int field, int index, const char* path) {
    CK(cudaSetDevice(ctx->device));
    const Geo& g = ctx->g;
    if (g.dim != 2) return fail(ctx, PETTO_INVALID, "write_pgm: only 2D fields");
    wr::Src src;
    if (int rc = writer_source(ctx, field, index, &src)) return rc;
    const int nb = 2 * ctx->nsm;
    if (!ctx->wmm) CK(cudaMalloc(&ctx->wmm, sizeof(wr::MinMax) * (size_t)nb));
    wr::MinMax* mm = static_cast<wr::MinMax*>(ctx->wmm);
    unsigned char* dbytes = nullptr;
    const size_t nbytes = (size_t)g.nx * g.ny;
    CK(cudaMalloc(&dbytes, nbytes));
    wr::k_minmax<<<nb, wr::TB, 0, ctx->stream>>>(src, mm);
    wr::k_minmax_final<<<1, 32, 0, ctx->stream>>>(mm, nb);
    wr::k_pgm_bytes<<<blocks_for((long long)nbytes), 256, 0, ctx->stream>>>(src, mm, dbytes);
    ctx->launches += 3;
    CKL();
    std::vector<unsigned char> bytes(nbytes);
    wr::MinMax h{};
    CK(cudaMemcpyAsync(bytes.data(), dbytes, nbytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&h, mm, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(dbytes);
    const bool any = h.ilo != 0x7fffffffffffffffLL;
    const double lo = any ? h.lo : 0.0, hi = any ? h.hi : 0.0;
    {
        OutFile o;
        if (int rc = open_out(ctx, o, path, true)) return rc;
        const std::string head = "P5\n" + std::to_string(g.nx) + " " + std::to_string(g.ny) + "\n255\n";
        std::fwrite(head.data(), 1, head.size(), o.f);
        std::fwrite(bytes.data(), 1, nbytes, o.f);
        if (int rc = close_out(ctx, o, path)) return rc;
    }
    const std::string side = std::string(path) + ".scale.txt";
    OutFile o;
    if (int rc = open_out(ctx, o, side.c_str(), false)) return rc;
    const std::string body = "min = " + fmt17(lo) + "\nmax = " + fmt17(hi) + "\nrows = top_to_bottom\n";
    std::fwrite(body.data(), 1, body.size(), o.f);
    return close_out(ctx, o, side.c_str());
}

}  // extern "C"
