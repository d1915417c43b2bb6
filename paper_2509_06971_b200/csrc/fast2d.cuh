// fast2d.cuh -- fused residual + PT/APT update kernels for the small operators:
// heat conduction (2D/3D, HeatOperator::residual -> variable_diffusion_into,
// stencil.hpp:123-158) and 2D plane-strain elasticity (modal form, 10 nonzeros).
// One thread per owned node; neighbours come through L1/L2 (the C1-C3 working
// sets are L2-resident, so these are latency/launch-bound rather than HBM-bound).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace petto_b200 {

struct FusedParams {
    Geo g;
    int form;           // 0 APT explicit, 1 APT semi-implicit, 2 PT, 3 residual only
    double dt, a, b, inv;
    const double* cur;
    const double* prev;
    double* next;       // may alias prev
    const double* prop; // kappa (heat) / Young's modulus E (elasticity)
    const unsigned char* mask;  // bit c: component c pinned; bit 3: load present
    const double* aux;  // pinned values / loads
    const double* src;  // heat: dense source (nullable -> src_uniform)
    double src_uniform;
    double kh[10];      // 2D modal stiffness
    double e_scale;     // sum of 4 corner E -> E_cell
    double hih2[3];     // heat: 0.5 / h_a^2
    double inv_base;    // 1/(hx hy [hz])
    double* partials;   // per-block r^2 (nullable)
    DeviceStatus* status;
    long long step, nsteps;
};

__device__ __forceinline__ double fused_update(const FusedParams& P, double r, double cu, long long e, int c,
                                               unsigned char mk, double& rsq) {
    if ((mk >> c) & 1) return P.form == 3 ? 0.0 : P.aux[e];
    rsq += r * r;
    switch (P.form) {
        case 0: {
            const double pp = P.prev[e];
            return 2.0 * cu - pp + P.a * r - P.b * (cu - pp);
        }
        case 1: {
            const double pp = P.prev[e];
            return (2.0 * cu - pp + P.b * cu + P.a * r) * P.inv;
        }
        case 2:
            return cu + P.dt * r;
        default:
            return r;
    }
}

__device__ __forceinline__ double flux_fast(const double* f, const double* kp, int t, int n, long long s,
                                            double hih2) {
    if (n == 1) return 0.0;
    const double f0 = f[0], k0 = kp[0];
    if (t == 0) return (k0 + kp[s]) * (f[s] - f0) * (2.0 * hih2);
    if (t == n - 1) return (k0 + kp[-s]) * (f[-s] - f0) * (2.0 * hih2);
    return ((k0 + kp[s]) * (f[s] - f0) - (kp[-s] + k0) * (f0 - f[-s])) * hih2;
}

template <int NT>
__device__ __forceinline__ void finish_block(const FusedParams& P, double rsq, unsigned bad) {
    __shared__ double scratch[32];
    const double s = block_sum<NT / 32>(rsq, scratch);
    if (threadIdx.x == 0 && P.partials) P.partials[blockIdx.x] = s;
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) {
        if (bad & 2u) atomicOr(&P.status->flags, 2u);
        if (bad & 1u) mark_bad(P.status, P.step);
    }
}

// Heat: one owned node t (HeatOperator::residual + the update).
__device__ __forceinline__ void heat_node(const FusedParams& P, long long t, double& rsq, unsigned& bad) {
    const Geo& g = P.g;
    const long long plane = (long long)g.nx * g.ny;
    const int k = g.kb + (int)(t / plane);
    const long long rr = t - (long long)(k - g.kb) * plane;
    const int j = (int)(rr / g.nx);
    const int i = (int)(rr - (long long)j * g.nx);
    const long long node = lidx(g, i, j, k);
    const double* T = P.cur + node;
    const double* kp = P.prop + node;
    if (!(kp[0] > 0.0)) bad |= 2u;
    double acc = flux_fast(T, kp, i, g.nx, 1, P.hih2[0]) + flux_fast(T, kp, j, g.ny, g.px, P.hih2[1]);
    if (g.nz > 1) acc += flux_fast(T, kp, k, g.nz, (long long)g.px * g.ny, P.hih2[2]);
    const double r = acc + (P.src ? P.src[node] : P.src_uniform);
    const double nv = fused_update(P, r, T[0], node, 0, P.mask[node], rsq);
    bad |= !isfinite(nv);
    P.next[node] = nv;
}

// Heat: grid-stride over owned nodes (fixed grid => deterministic partials).
__global__ void __launch_bounds__(256) k_heat_fast(const FusedParams P) {
    const Geo& g = P.g;
    if (skip_step(P.status, P.step, P.nsteps)) return;
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    double rsq = 0.0;
    unsigned bad = 0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < owned;
         t += (long long)gridDim.x * blockDim.x)
        heat_node(P, t, rsq, bad);
    finish_block<256>(P, rsq, bad);
}

// 2D plane-strain elasticity: each node gathers the corner forces of its (up to)
// four cells, evaluated in the modal basis (stiffness.hpp pattern order).
__device__ __forceinline__ void elastic2d_node(const FusedParams& P, long long t, double& rsq, unsigned& bad) {
    const Geo& g = P.g;
    const double* k = P.kh;
    const int j = (int)(t / g.nx);
    const int i = (int)(t - (long long)j * g.nx);
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int m = 0; m < 4; ++m) {  // this node is corner m of cell (i - bx, j - by)
        const int ci = i - (m & 1), cj = j - (m >> 1);
        if (ci < 0 || ci > g.nx - 2 || cj < 0 || cj > g.ny - 2) continue;
        const long long b = lidx(g, ci, cj, 0);
        const long long o[4] = {b, b + 1, b + g.px, b + g.px + 1};
        double C[4][2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const double* u = P.cur + c * g.Ns;
            const double v0 = u[o[0]], v1 = u[o[1]], v2 = u[o[2]], v3 = u[o[3]];
            C[1][c] = (v0 - v1) + (v2 - v3);
            C[2][c] = (v0 + v1) - (v2 + v3);
            C[3][c] = (v0 - v1) - (v2 - v3);
        }
        const double ec = ((P.prop[o[0]] + P.prop[o[1]]) + (P.prop[o[2]] + P.prop[o[3]])) * P.e_scale;
        const double F10 = ec * (k[0] * C[1][0] + k[1] * C[2][1]);
        const double F11 = ec * (k[2] * C[1][1] + k[3] * C[2][0]);
        const double F20 = ec * (k[4] * C[1][1] + k[5] * C[2][0]);
        const double F21 = ec * (k[6] * C[1][0] + k[7] * C[2][1]);
        const double F30 = ec * (k[8] * C[3][0]);
        const double F31 = ec * (k[9] * C[3][1]);
        const double s1 = (m & 1) ? -1.0 : 1.0, s2 = (m & 2) ? -1.0 : 1.0, s3 = s1 * s2;
        acc[0] += s1 * F10 + s2 * F20 + s3 * F30;
        acc[1] += s1 * F11 + s2 * F21 + s3 * F31;
    }
    const long long node = lidx(g, i, j, 0);
    const double invv = inv_volume_fast(g, P.inv_base, i, j, 0);
    const unsigned char mk = P.mask[node];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const long long e = c * g.Ns + node;
        const double f = ((mk & 8) && !((mk >> c) & 1)) ? P.aux[e] : 0.0;
        const double r = -acc[c] * invv - f;
        const double nv = fused_update(P, r, P.cur[e], e, c, mk, rsq);
        bad |= !isfinite(nv);
        P.next[e] = nv;
    }
}

__global__ void __launch_bounds__(256) k_elastic2d_fast(const FusedParams P) {
    const Geo& g = P.g;
    if (skip_step(P.status, P.step, P.nsteps)) return;
    const long long owned = (long long)g.nx * g.ny;
    double rsq = 0.0;
    unsigned bad = 0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < owned;
         t += (long long)gridDim.x * blockDim.x)
        elastic2d_node(P, t, rsq, bad);
    finish_block<256>(P, rsq, bad);
}

// Whole hybrid_solve (state_solver.hpp:480-498) of a small grid in ONE cooperative
// launch: the per-step kernels of C1-C3 last a few microseconds, so launch and
// drain dominate; here the steps are separated by grid-wide barriers instead.
// Buffers swap exactly as in the host loop (next := previous, then swap); the
// check_finite cadence is kept through skip_step, read after each barrier.
struct SolveParams {
    FusedParams base;     // geometry, fields and constants (cur/prev/next per step)
    double* st[2];        // history: current = st[c], previous = st[1 - c]
    int c0;               // current buffer at step 1
    long long n_apt, n_pt;
    int form_apt;         // 0 explicit, 1 semi-implicit
    double a, b, inv;     // APT coefficients
    double dt_pt;         // PT step
};

template <int PHYS>  // 0 heat, 1 2D elasticity
__global__ void __launch_bounds__(256) k_small_solve(const SolveParams S) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    FusedParams P = S.base;
    const Geo& g = P.g;
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    const long long nsteps = S.n_apt + S.n_pt;
    int c = S.c0;
    for (long long step = 1; step <= nsteps; ++step) {
        if (skip_step(P.status, step, nsteps)) break;  // same value in every CTA (read after the barrier)
        const bool apt = step <= S.n_apt;
        P.form = apt ? S.form_apt : 2;
        P.a = S.a;
        P.b = S.b;
        P.inv = S.inv;
        P.dt = S.dt_pt;
        P.cur = S.st[c];
        P.prev = S.st[1 - c];
        P.next = S.st[1 - c];
        P.step = step;
        double rsq = 0.0;
        unsigned bad = 0;
        for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < owned;
             t += (long long)gridDim.x * blockDim.x) {
            if (PHYS == 0) heat_node(P, t, rsq, bad);
            else elastic2d_node(P, t, rsq, bad);
        }
        bad = __reduce_or_sync(0xffffffffu, bad);
        if (bad && (threadIdx.x & 31) == 0) {
            if (bad & 2u) atomicOr(&P.status->flags, 2u);
            if (bad & 1u) mark_bad(P.status, step);
        }
        c ^= 1;
        grid.sync();
    }
}

// ---------------------------------------------------------------------------
// Temporal blocking for small 2D heat grids: the whole hybrid_solve in one
// cooperative launch, K steps per grid barrier.  A CTA owns a TBX x TBY tile; per
// round it loads the tile plus a K-node halo of T_n, T_{n-1}, kappa, mask,
// pinned values and source into shared memory, advances it k <= K steps there
// (the halo's outer layers go stale one node per step, never reaching the tile),
// writes the tile's two time levels back, and waits at one grid barrier.  The
// per-node arithmetic is heat_node + fused_update's (stencil.hpp:123-158,
// state_solver.hpp:400-442).  Rounds never cross a multiple of 100 steps, so the
// check_finite abort (state_solver.hpp:463-497) stops exactly where the per-step
// solve does; global levels alternate between two buffer pairs so no CTA
// overwrites a tile another CTA is still reading.
constexpr int TBK = 10;                          // steps per round (divides 100)
constexpr int TRX = 64, TRY = 32, TRN = TRX * TRY; // shared region: a thread per column, rows ty and ty + 16
constexpr int TBX = TRX - 2 * TBK, TBY = TRY - 2 * TBK;  // owned tile 44 x 12
constexpr int TB_THREADS = 1024;

struct TBParams {
    FusedParams base;
    double* pair[2][2];   // [pair][0 current, 1 previous]; pair 0 = the caller's (current, previous)
    long long n_apt, n_pt;
    int form_apt;
    double a, b, inv, dt_pt;
    int tiles_x;
};

__device__ __forceinline__ double tb_flux(const double* f, const double* kp, int t, int n, int s, double hih2) {
    const double f0 = f[0], k0 = kp[0];
    if (t == 0) return (k0 + kp[s]) * (f[s] - f0) * (2.0 * hih2);
    if (t == n - 1) return (k0 + kp[-s]) * (f[-s] - f0) * (2.0 * hih2);
    return ((k0 + kp[s]) * (f[s] - f0) - (kp[-s] + k0) * (f0 - f[-s])) * hih2;
}

__global__ void __launch_bounds__(TB_THREADS, 1) k_heat2d_tb(const TBParams S) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    extern __shared__ __align__(16) unsigned char tb_smem[];
    double* buf[3] = {reinterpret_cast<double*>(tb_smem), reinterpret_cast<double*>(tb_smem) + TRN,
                      reinterpret_cast<double*>(tb_smem) + 2 * TRN};
    double* kap = reinterpret_cast<double*>(tb_smem) + 3 * TRN;
    double* pin = kap + TRN;
    double* src = pin + TRN;
    unsigned char* msk = reinterpret_cast<unsigned char*>(src + TRN);
    const FusedParams& P = S.base;
    const Geo& g = P.g;
    const long long nsteps = S.n_apt + S.n_pt;
    const int x0 = (blockIdx.x % S.tiles_x) * TBX, y0 = (blockIdx.x / S.tiles_x) * TBY;
    const int rx0 = x0 - TBK, ry0 = y0 - TBK;
    // this thread: region column lx, rows ly[0], ly[1]
    const int lx = threadIdx.x & (TRX - 1), gx = rx0 + lx;
    const int ly[2] = {(int)(threadIdx.x >> 6), (int)(threadIdx.x >> 6) + 16};
    const bool colin = gx >= 0 && gx < g.nx;
    bool in[2], own[2];
    long long node[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int gy = ry0 + ly[h];
        in[h] = colin && gy >= 0 && gy < g.ny;
        own[h] = in[h] && lx >= TBK && lx < TBK + TBX && ly[h] >= TBK && ly[h] < TBK + TBY;
        node[h] = in[h] ? (long long)gy * g.px + gx : 0;
    }
    // kappa, mask, pinned values, source: constant through the solve
    unsigned bad = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int q = ly[h] * TRX + lx;
        kap[q] = in[h] ? P.prop[node[h]] : 1.0;
        const unsigned char m = in[h] ? P.mask[node[h]] : 0;
        msk[q] = m;
        pin[q] = (m & 1) ? P.aux[node[h]] : 0.0;
        src[q] = in[h] ? (P.src ? P.src[node[h]] : P.src_uniform) : 0.0;
        if (own[h] && !(kap[q] > 0.0)) bad |= 2u;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(&P.status->flags, 2u);
    __syncthreads();
    // per node: the two face sums of each axis, (k0 + k+) and (k- + k0) as the
    // reference adds them (stencil.hpp:123-158), and the source / pinned value --
    // constant through the solve, so held in registers (shared memory then only
    // serves the temperature levels)
    double cxp[2], cxm[2], cyp[2], cym[2], sr[2], pv[2];
    int ex[2], ey[2];  // 0 interior, 1 at the low end, 2 at the high end
    bool pinned[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int q = ly[h] * TRX + lx;
        const int gy = ry0 + ly[h];
        const bool interior = lx > 0 && lx < TRX - 1 && ly[h] > 0 && ly[h] < TRY - 1;
        const double k0 = kap[q];
        ex[h] = gx == 0 ? 1 : (gx == g.nx - 1 ? 2 : 0);
        ey[h] = gy == 0 ? 1 : (gy == g.ny - 1 ? 2 : 0);
        cxp[h] = interior ? k0 + kap[q + 1] : 0.0;
        cxm[h] = interior ? kap[q - 1] + k0 : 0.0;
        cyp[h] = interior ? k0 + kap[q + TRX] : 0.0;
        cym[h] = interior ? kap[q - TRX] + k0 : 0.0;
        if (ex[h] == 2) cxp[h] = interior ? k0 + kap[q - 1] : 0.0;  // the one neighbour at the high end
        if (ey[h] == 2) cyp[h] = interior ? k0 + kap[q - TRX] : 0.0;
        sr[h] = src[q];
        pinned[h] = msk[q] & 1;
        pv[h] = pin[q];
    }
    long long s0 = 0;  // steps completed
    int rd = 0;        // pair holding the levels at step s0
    while (s0 < nsteps) {
        if (skip_step(P.status, s0 + 1, nsteps)) break;  // read after the barrier: the same in every CTA
        const int k = (int)min((long long)TBK, min(nsteps - s0, 100 - s0 % 100));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = ly[h] * TRX + lx;
            buf[0][q] = in[h] ? S.pair[rd][0][node[h]] : 0.0;
            buf[1][q] = in[h] ? S.pair[rd][1][node[h]] : 0.0;
        }
        __syncthreads();
        int ic = 0, ip = 1, in_ = 2;
        long long first_bad = PETTO_NO_BAD;
        for (int sub = 1; sub <= k; ++sub) {
            const long long step = s0 + sub;
            const int form = step <= S.n_apt ? S.form_apt : 2;
            const double* T = buf[ic];
            const double* Tp = buf[ip];
            double* Tn = buf[in_];
            // nodes whose dependencies are still fresh: the region shrinks by one per step
            const bool colok = lx >= sub && lx < TRX - sub;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (!in[h] || !colok || ly[h] < sub || ly[h] >= TRY - sub) continue;
                const int q = ly[h] * TRX + lx;
                const double f0 = T[q];
                double fx, fy;  // flux_fast / tb_flux with the face sums from registers
                if (ex[h] == 0) fx = (cxp[h] * (T[q + 1] - f0) - cxm[h] * (f0 - T[q - 1])) * P.hih2[0];
                else if (ex[h] == 1) fx = cxp[h] * (T[q + 1] - f0) * (2.0 * P.hih2[0]);
                else fx = cxp[h] * (T[q - 1] - f0) * (2.0 * P.hih2[0]);
                if (ey[h] == 0) fy = (cyp[h] * (T[q + TRX] - f0) - cym[h] * (f0 - T[q - TRX])) * P.hih2[1];
                else if (ey[h] == 1) fy = cyp[h] * (T[q + TRX] - f0) * (2.0 * P.hih2[1]);
                else fy = cyp[h] * (T[q - TRX] - f0) * (2.0 * P.hih2[1]);
                const double acc = fx + fy;
                const double r = acc + sr[h];
                const double cu = f0;
                double nv;
                if (pinned[h]) {
                    nv = pv[h];
                } else if (form == 0) {
                    const double pp = Tp[q];
                    nv = 2.0 * cu - pp + S.a * r - S.b * (cu - pp);
                } else if (form == 1) {
                    const double pp = Tp[q];
                    nv = (2.0 * cu - pp + S.b * cu + S.a * r) * S.inv;
                } else {
                    nv = cu + S.dt_pt * r;
                }
                Tn[q] = nv;
                if (own[h] && !isfinite(nv) && step < first_bad) first_bad = step;
            }
            __syncthreads();
            const int t = ip;  // previous <- current <- next
            ip = ic;
            ic = in_;
            in_ = t;
        }
        if (first_bad != PETTO_NO_BAD) mark_bad(P.status, first_bad);
        // the tile's two levels into the other pair
        const int wr = rd ^ 1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!own[h]) continue;
            const int q = ly[h] * TRX + lx;
            S.pair[wr][0][node[h]] = buf[ic][q];
            S.pair[wr][1][node[h]] = buf[ip][q];
        }
        s0 += k;
        rd = wr;
        grid.sync();
    }
    // the caller's convention (k_small_solve): after s0 steps the current level is
    // in the caller's buffer (s0 & 1), the previous one in the other
    const int cur_slot = (int)(s0 & 1);
    if (rd == 0 && cur_slot == 0) return;  // already in place
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!own[h]) continue;
        const double c = S.pair[rd][0][node[h]], pv = S.pair[rd][1][node[h]];
        S.pair[0][cur_slot][node[h]] = c;
        S.pair[0][cur_slot ^ 1][node[h]] = pv;
    }
}

// ---------------------------------------------------------------------------
// Temporal blocking for small 2D elasticity grids (plane strain): the same scheme
// as k_heat2d_tb -- EK steps per grid barrier on a shared-memory region with an
// EK-node halo -- with elastic2d_node's arithmetic per node (the four cells
// around it in the modal basis, state_solver.hpp:327-385 via stiffness.hpp).
// Shared memory holds the three displacement levels, the cell moduli (corner sum
// x scale, once per solve), the pinned values / loads and the mask.
constexpr int EK = 4;                              // steps per round (divides 100)
// Region 64 x 16 ER: a thread per column and ER consecutive rows.  ER = 2 (tile
// 56 x 24) for grids up to ~148 such tiles; ER = 1 (tile 56 x 8) halves each
// thread's per-step chain for grids that fit in 148 of the smaller tiles (C1).
constexpr int ERX = 64, ETX = ERX - 2 * EK, ETHREADS = 1024;
__host__ __device__ constexpr int e_ry(int er) { return 16 * er; }
__host__ __device__ constexpr int e_ty(int er) { return e_ry(er) - 2 * EK; }
__host__ __device__ constexpr size_t e_smem(int er) {
    return (size_t)ERX * e_ry(er) * (sizeof(double) * (3 * 2 + 1 + 2) + 1);
}

template <int ER>
__global__ void __launch_bounds__(ETHREADS, 1) k_elastic2d_tb(const TBParams S) {
    constexpr int ERY = e_ry(ER), ERN = ERX * ERY, ETY = e_ty(ER), EROWS = ER;
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    extern __shared__ __align__(16) unsigned char tb_smem[];
    double* U = reinterpret_cast<double*>(tb_smem);  // [3 levels][2 comps][ERN]
    double* EC = U + 6 * ERN;                        // cell whose low corner is the node
    double* AX = EC + ERN;                           // [2][ERN] pinned value / load
    unsigned char* MK = reinterpret_cast<unsigned char*>(AX + 2 * ERN);
    const FusedParams& P = S.base;
    const Geo& g = P.g;
    const double* kh = P.kh;
    const long long nsteps = S.n_apt + S.n_pt;
    const int x0 = (blockIdx.x % S.tiles_x) * ETX, y0 = (blockIdx.x / S.tiles_x) * ETY;
    const int rx0 = x0 - EK, ry0 = y0 - EK;
    const int lx = threadIdx.x & (ERX - 1), gx = rx0 + lx;
    const int ly0 = (threadIdx.x / ERX) * EROWS;  // rows ly0 .. ly0 + EROWS - 1
    const bool colin = gx >= 0 && gx < g.nx;
    bool in[EROWS], own[EROWS];
    long long node[EROWS];
    double invv[EROWS];
#pragma unroll
    for (int h = 0; h < EROWS; ++h) {
        const int ly = ly0 + h, gy = ry0 + ly;
        in[h] = colin && gy >= 0 && gy < g.ny;
        own[h] = in[h] && lx >= EK && lx < EK + ETX && ly >= EK && ly < EK + ETY;
        node[h] = in[h] ? (long long)gy * g.px + gx : 0;
        invv[h] = in[h] ? inv_volume_fast(g, P.inv_base, gx, gy, 0) : 0.0;
        const int q = ly * ERX + lx;
        const bool cell = gx >= 0 && gy >= 0 && gx <= g.nx - 2 && gy <= g.ny - 2;
        if (cell) {
            const long long b = (long long)gy * g.px + gx;
            EC[q] = ((P.prop[b] + P.prop[b + 1]) + (P.prop[b + g.px] + P.prop[b + g.px + 1])) * P.e_scale;
        } else {
            EC[q] = 0.0;
        }
        const unsigned char m = in[h] ? P.mask[node[h]] : 0;
        MK[q] = m;
        AX[q] = m ? P.aux[node[h]] : 0.0;
        AX[ERN + q] = m ? P.aux[g.Ns + node[h]] : 0.0;
    }
    long long s0 = 0;
    int rd = 0;
    while (s0 < nsteps) {
        if (skip_step(P.status, s0 + 1, nsteps)) break;  // read after the barrier: the same in every CTA
        const int k = (int)min((long long)EK, min(nsteps - s0, 100 - s0 % 100));
#pragma unroll
        for (int h = 0; h < EROWS; ++h) {
            const int q = (ly0 + h) * ERX + lx;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                U[(0 * 2 + c) * ERN + q] = in[h] ? S.pair[rd][0][c * g.Ns + node[h]] : 0.0;
                U[(1 * 2 + c) * ERN + q] = in[h] ? S.pair[rd][1][c * g.Ns + node[h]] : 0.0;
            }
        }
        __syncthreads();
        int ic = 0, ip = 1, in_ = 2;
        long long first_bad = PETTO_NO_BAD;
        for (int sub = 1; sub <= k; ++sub) {
            const long long step = s0 + sub;
            const int form = step <= S.n_apt ? S.form_apt : 2;
            const double* Ux = U + (ic * 2) * ERN;
            const double* Uy = Ux + ERN;
            // Column-of-cells sweep: this thread's four nodes (lx, ly0..ly0+3) touch
            // the cells of columns lx-1, lx in rows ly0-1..ly0+3; each cell is evaluated
            // once and its corner forces go to the (up to) two nodes of this column
            // it touches.  Rows run top-down and the x+ cell first, so every node
            // sums its cells in elastic2d_node's order (m = 0, 1, 2, 3).
            if (lx >= sub && lx < ERX - sub) {
                double acc[EROWS][2];
#pragma unroll
                for (int h = 0; h < EROWS; ++h) acc[h][0] = acc[h][1] = 0.0;
                // per row and component: the differences and sums of horizontally
                // adjacent nodes (u[x] - u[x+1], u[x] + u[x+1] for x = lx-1, lx), the
                // operands of the modal coefficients, shared by the cells above and below
                double hd[2][2], hs[2][2], ld[2][2], ls[2][2];
                auto row_terms = [&](int row, double (&dd)[2][2], double (&sd)[2][2]) {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const double* u = (c ? Uy : Ux) + row * ERX + lx - 1;
                        const double w0 = u[0], w1 = u[1], w2 = u[2];
                        dd[0][c] = w0 - w1;
                        sd[0][c] = w0 + w1;
                        dd[1][c] = w1 - w2;
                        sd[1][c] = w1 + w2;
                    }
                };
                row_terms(min(ly0 + EROWS, ERY - 1), hd, hs);
#pragma unroll
                for (int cr = EROWS; cr >= 0; --cr) {
                    const int lcj = ly0 - 1 + cr;
                    const int row = max(lcj, 0);
                    row_terms(row, ld, ls);
                    const int gcj = ry0 + lcj;
                    const bool row_ok = lcj >= sub - 1 && lcj + 1 <= ERY - sub && gcj >= 0 && gcj <= g.ny - 2;
#pragma unroll
                    for (int cc = 1; cc >= 0; --cc) {
                        const int gci = gx - 1 + cc;
                        if (!row_ok || gci < 0 || gci > g.nx - 2) continue;
                        double C[4][2];
#pragma unroll
                        for (int c = 0; c < 2; ++c) {  // corners v0 v1 (row lcj), v2 v3 (row lcj + 1)
                            C[1][c] = ld[cc][c] + hd[cc][c];  // (v0 - v1) + (v2 - v3)
                            C[2][c] = ls[cc][c] - hs[cc][c];  // (v0 + v1) - (v2 + v3)
                            C[3][c] = ld[cc][c] - hd[cc][c];  // (v0 - v1) - (v2 - v3)
                        }
                        const double ec = EC[row * ERX + lx - 1 + cc];
                        const double F10 = ec * (kh[0] * C[1][0] + kh[1] * C[2][1]);
                        const double F11 = ec * (kh[2] * C[1][1] + kh[3] * C[2][0]);
                        const double F20 = ec * (kh[4] * C[1][1] + kh[5] * C[2][0]);
                        const double F21 = ec * (kh[6] * C[1][0] + kh[7] * C[2][1]);
                        const double F30 = ec * (kh[8] * C[3][0]);
                        const double F31 = ec * (kh[9] * C[3][1]);
                        const double s1 = cc ? 1.0 : -1.0;  // m & 1 = 1 - cc
                        if (cr >= 1) {  // node row lcj: corner m = 1 - cc
                            acc[cr - 1][0] += s1 * F10 + 1.0 * F20 + s1 * F30;
                            acc[cr - 1][1] += s1 * F11 + 1.0 * F21 + s1 * F31;
                        }
                        if (cr < EROWS) {  // node row lcj + 1: corner m = (1 - cc) | 2
                            acc[cr][0] += s1 * F10 + -1.0 * F20 + -s1 * F30;
                            acc[cr][1] += s1 * F11 + -1.0 * F21 + -s1 * F31;
                        }
                    }
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2)
#pragma unroll
                        for (int c = 0; c < 2; ++c) hd[k2][c] = ld[k2][c], hs[k2][c] = ls[k2][c];
                }
#pragma unroll
                for (int h = 0; h < EROWS; ++h) {
                    const int ly = ly0 + h;
                    if (!in[h] || ly < sub || ly >= ERY - sub) continue;
                    const int q = ly * ERX + lx;
                    const unsigned char mk = MK[q];
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const double cu = U[(ic * 2 + c) * ERN + q];
                        double nv;
                        if ((mk >> c) & 1) {
                            nv = AX[c * ERN + q];
                        } else {
                            const double f = (mk & 8) ? AX[c * ERN + q] : 0.0;
                            const double r = -acc[h][c] * invv[h] - f;
                            if (form == 0) {
                                const double pp = U[(ip * 2 + c) * ERN + q];
                                nv = 2.0 * cu - pp + S.a * r - S.b * (cu - pp);
                            } else if (form == 1) {
                                const double pp = U[(ip * 2 + c) * ERN + q];
                                nv = (2.0 * cu - pp + S.b * cu + S.a * r) * S.inv;
                            } else {
                                nv = cu + S.dt_pt * r;
                            }
                        }
                        U[(in_ * 2 + c) * ERN + q] = nv;
                        if (own[h] && !isfinite(nv) && step < first_bad) first_bad = step;
                    }
                }
            }
            __syncthreads();
            const int t = ip;
            ip = ic;
            ic = in_;
            in_ = t;
        }
        if (first_bad != PETTO_NO_BAD) mark_bad(P.status, first_bad);
        const int wr = rd ^ 1;
#pragma unroll
        for (int h = 0; h < EROWS; ++h) {
            if (!own[h]) continue;
            const int q = (ly0 + h) * ERX + lx;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                S.pair[wr][0][c * g.Ns + node[h]] = U[(ic * 2 + c) * ERN + q];
                S.pair[wr][1][c * g.Ns + node[h]] = U[(ip * 2 + c) * ERN + q];
            }
        }
        s0 += k;
        rd = wr;
        grid.sync();
    }
    const int cur_slot = (int)(s0 & 1);
    if (rd == 0 && cur_slot == 0) return;
#pragma unroll
    for (int h = 0; h < EROWS; ++h) {
        if (!own[h]) continue;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const long long e = c * g.Ns + node[h];
            const double cv = S.pair[rd][0][e], pv = S.pair[rd][1][e];
            S.pair[0][cur_slot][e] = cv;
            S.pair[0][cur_slot ^ 1][e] = pv;
        }
    }
}

}  // namespace petto_b200
