// common.cuh -- device-side layout, arithmetic and sm_100a PTX helpers.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace petto_b200 {

// HBM layout of one rank's fields.  Rows are padded to a pitch of px doubles
// (px % 16 == 0) so every TMA global stride is 16-byte aligned; the rank stores
// global node planes [ks0, ks0 + nzs) (owned planes [kb, ke) plus one ghost
// plane per interior slab face).  Component c of a vector field starts at c*Ns.
struct Geo {
    int dim;
    int nx, ny, nz;  // global node counts (nz = 1 in 2D)
    int kb, ke;      // owned global planes
    int ks0, nzs;    // stored planes
    int px;          // row pitch (elements)
    long long Ns;    // stored nodes incl. padding = px * ny * nzs
    double h[3];
    double hih[3];   // 0.5 / h  (stencil.hpp:23-31 derivative factor; host IEEE division = the device's)
    double ilap[3];  // 1 / (h h) (stencil.hpp:109-116 Laplacian factor)
};

// The per-axis stencil factors the design kernels need at every node, computed
// once (same IEEE operations as the reference's per-call expressions).
inline void geo_factors(Geo& g) {
    for (int a = 0; a < 3; ++a) {
        g.hih[a] = 0.5 / g.h[a];
        const double h2 = g.h[a] * g.h[a];
        g.ilap[a] = 1.0 / h2;
    }
}

// Device-resident control block of a context: non-finite detection with the
// reference's check_finite cadence (state_solver.hpp:463-497) and the
// iterate_to_tolerance stop logic (:511-541), evaluated on the device so the
// step loops never synchronise with the host.
struct DeviceStatus {
    unsigned flags;        // bit 0 non-finite written, bit 1 non-positive kappa
    int done;              // iterate_to_tolerance: stop flag
    long long first_bad;   // first step that wrote a non-finite value (LLONG_MAX: none)
    int converged;
    int aborted;
    long long iter;        // iterate_to_tolerance: index of the residual being evaluated
    long long iterations;
    double r_initial, r_final;
    double target;
    long long max_iters;
    double nodes;
    double sumsq;
};

#define PETTO_NO_BAD 0x7fffffffffffffffLL

// True when the kernel of pseudo-time step `step` (1-based) must not run: the
// reference would already have aborted at the check_finite following the first
// non-finite write (every 100 steps and at the last step), or the tolerance
// loop has stopped.
__device__ __forceinline__ bool skip_step(const DeviceStatus* s, long long step, long long nsteps) {
    if (s->done) return true;
    const long long fb = s->first_bad;
    if (fb == PETTO_NO_BAD) return false;
    long long lim = ((fb + 99) / 100) * 100;
    if (lim > nsteps) lim = nsteps;
    return step > lim;
}

__device__ __forceinline__ void mark_bad(DeviceStatus* s, long long step) {
    atomicOr(&s->flags, 1u);
    atomicMin(reinterpret_cast<unsigned long long*>(&s->first_bad), (unsigned long long)step);
}

__host__ __device__ inline long long lidx(const Geo& g, int i, int j, int k) {
    return ((long long)(k - g.ks0) * g.ny + j) * g.px + i;
}

// Round-to-nearest IEEE operations that the compiler never contracts into FMA:
// the replica kernels spell the reference's expressions with these.
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }

// Lumped extent along an axis (grid.hpp:64-67).
__device__ __forceinline__ double cell_extent(const Geo& g, int axis, int i) {
    const int n = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
    if (n == 1) return 1.0;
    return (i == 0 || i == n - 1) ? rmul(0.5, g.h[axis]) : g.h[axis];
}

// cell_volume (grid.hpp:69-73), reference multiplication order.
__device__ __forceinline__ double cell_volume(const Geo& g, int i, int j, int k) {
    double v = rmul(cell_extent(g, 0, i), cell_extent(g, 1, j));
    if (g.dim == 3) v = rmul(v, cell_extent(g, 2, k));
    return v;
}

// Power-of-two boundary factor of 1/cell_volume: 1/(h_x h_y h_z) * 2^(#end axes),
// which is exact because halving is exact.
__device__ __forceinline__ double inv_volume_fast(const Geo& g, double inv_base, int i, int j, int k) {
    int e = (i == 0 || i == g.nx - 1) + (j == 0 || j == g.ny - 1);
    if (g.dim == 3) e += (k == 0 || k == g.nz - 1);
    return inv_base * (double)(1 << e);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum in a fixed order (warp butterflies, then warp 0 over the warp
// partials): deterministic for a fixed launch shape.  Result valid in thread 0.
template <int NWARPS>
__device__ double block_sum(double v, double* scratch) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = l < NWARPS ? scratch[l] : 0.0;
        r = warp_sum(r);
    }
    return r;
}

// ----------------------------------------------------------- mbarrier / TMA

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(addr),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
        "%6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// TMA tensor store (shared -> global, bulk-group completion); the threads that
// wrote the shared source fence it into the async proxy first
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                             int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------ tensor memory
// TMEM as a per-warp scratch: warp w reaches lanes 32 (w % 4) .. +31 only; the
// 32x32b shape moves one 32-bit column per thread (thread l <-> lane base + l).

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols));
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// one double (two columns) per thread: a register pair as it is, no marshalling
__device__ __forceinline__ void tmem_st1(uint32_t taddr, double a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(__double2loint(a)),
                 "r"(__double2hiint(a))
                 : "memory");
}
// twelve doubles (24 columns at taddr): three loads and the wait in one block, so
// no consumer can be scheduled between the load and its completion
__device__ __forceinline__ void tmem_ld12(uint32_t taddr, double (&v)[12]) {
    uint32_t r[24];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%24];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8, %9, %10, %11, %12, %13, %14, %15}, [%25];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16, %17, %18, %19, %20, %21, %22, %23}, [%26];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23])
        : "r"(taddr), "r"(taddr + 8), "r"(taddr + 16)
        : "memory");
#pragma unroll
    for (int k = 0; k < 12; ++k) v[k] = __hiloint2double(r[2 * k + 1], r[2 * k]);
}

template <uint32_t N>
__device__ __forceinline__ void regs_grow() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <uint32_t N>
__device__ __forceinline__ void regs_shrink() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace petto_b200
