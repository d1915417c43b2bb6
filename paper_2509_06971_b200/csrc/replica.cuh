// replica.cuh -- reference-order ("replica") kernels.
//
// Each kernel restates one reference loop with the same operation order and no
// FMA contraction (radd/rmul = __dadd_rn/__dmul_rn), so the device reproduces
// the reference bit for bit on every input.  They are the parity anchor for the
// fast fused kernels and the PETTO_MODE_REPLICA execution mode; one thread per
// owned node, no tiling.
#pragma once

#include "common.cuh"

namespace petto_b200 {

__device__ __forceinline__ double tree_sum(double* v, int count) {
    // detail::mirror_tree_sum (state_solver.hpp:242-247)
    for (int width = count; width > 1; width /= 2)
        for (int i = 0; i < width / 2; ++i) v[i] = radd(v[2 * i], v[2 * i + 1]);
    return v[0];
}

__device__ __forceinline__ bool owned_node(const Geo& g, long long t, int& i, int& j, int& k) {
    const long long plane = (long long)g.nx * g.ny;
    const long long owned = plane * (g.ke - g.kb);
    if (t >= owned) return false;
    k = g.kb + (int)(t / plane);
    const long long r = t - (long long)(k - g.kb) * plane;
    j = (int)(r / g.nx);
    i = (int)(r - (long long)j * g.nx);
    return true;
}

// ElasticityOperator::residual (state_solver.hpp:327-385) without the final
// zero_constrained (applied by k_zero_entries).  mu = cm * E as make_lame /
// update_lame store it; e_from_mu = 2(1+nu_op)/2^dim.
__global__ void k_elastic_residual_replica(Geo g, const double* __restrict__ u, const double* __restrict__ E,
                                           double cm, const double* __restrict__ src,
                                           const double* __restrict__ K, double e_from_mu,
                                           double* __restrict__ out, const DeviceStatus* st, long long step,
                                           long long nsteps) {
    int i, j, k;
    if (skip_step(st, step, nsteps)) return;
    if (!owned_node(g, (long long)blockIdx.x * blockDim.x + threadIdx.x, i, j, k)) return;
    const int d = g.dim;
    const int cn = 1 << d;
    const int dofs = cn * d;
    double lanes[3][8];
    for (int c = 0; c < d; ++c)
        for (int m = 0; m < cn; ++m) lanes[c][m] = 0.0;
    for (int m = 0; m < cn; ++m) {
        const int ci = i - (m & 1);
        const int cj = j - ((m >> 1) & 1);
        const int ck = d == 3 ? k - ((m >> 2) & 1) : 0;
        if (ci < 0 || ci > g.nx - 2 || cj < 0 || cj > g.ny - 2) continue;
        if (d == 3 && (ck < 0 || ck > g.nz - 2)) continue;
        long long corners[8];
        double ev[8];
        for (int m2 = 0; m2 < cn; ++m2) {
            corners[m2] = lidx(g, ci + (m2 & 1), cj + ((m2 >> 1) & 1), d == 3 ? ck + ((m2 >> 2) & 1) : 0);
            ev[m2] = rmul(cm, E[corners[m2]]);
        }
        const double e_cell = rmul(tree_sum(ev, cn), e_from_mu);
        const int l = m;
        for (int c = 0; c < d; ++c) {
            const double* kr = K + (l * d + c) * dofs;
            double tv[8];
            for (int m2 = 0; m2 < cn; ++m2) {
                double t = 0.0;
                for (int b = 0; b < d; ++b) t = radd(t, rmul(__ldg(kr + m2 * d + b), u[b * g.Ns + corners[m2]]));
                tv[m2] = t;
            }
            lanes[c][m] = rmul(e_cell, tree_sum(tv, cn));
        }
    }
    const long long node = lidx(g, i, j, k);
    const double invv = rdiv(1.0, cell_volume(g, i, j, k));
    for (int c = 0; c < d; ++c)
        out[c * g.Ns + node] = rsub(rmul(-tree_sum(lanes[c], cn), invv), src[c * g.Ns + node]);
}

// detail::flux_along (stencil.hpp:97-107) with pointer offsets in elements.
__device__ __forceinline__ double flux_along(const double* f, const double* kp, int t, int n, long long s,
                                             double hih2) {
    if (n == 1) return 0.0;
    if (t == 0) return rmul(rmul(radd(kp[0], kp[s]), rsub(f[s], f[0])), rmul(2.0, hih2));
    if (t == n - 1) return rmul(rmul(radd(kp[0], kp[-s]), rsub(f[-s], f[0])), rmul(2.0, hih2));
    return rmul(rsub(rmul(radd(kp[0], kp[s]), rsub(f[s], f[0])), rmul(radd(kp[-s], kp[0]), rsub(f[0], f[-s]))),
                hih2);
}

// HeatOperator::residual -> variable_diffusion_into with fused source
// (stencil.hpp:123-158); non-positive kappa raises the bad flag.
__global__ void k_heat_residual_replica(Geo g, const double* __restrict__ T, const double* __restrict__ kap,
                                        const double* __restrict__ src, double src_uniform, int src_dense,
                                        double* __restrict__ out, DeviceStatus* st, long long step,
                                        long long nsteps) {
    int i, j, k;
    if (skip_step(st, step, nsteps)) return;
    if (!owned_node(g, (long long)blockIdx.x * blockDim.x + threadIdx.x, i, j, k)) return;
    const long long node = lidx(g, i, j, k);
    double hih2[3];
    for (int a = 0; a < 3; ++a) hih2[a] = rdiv(0.5, rmul(g.h[a], g.h[a]));
    if (!(kap[node] > 0.0)) atomicOr(&st->flags, 2u);
    double acc = flux_along(T + node, kap + node, i, g.nx, 1, hih2[0]);
    acc = radd(acc, flux_along(T + node, kap + node, j, g.ny, g.px, hih2[1]));
    if (g.nz > 1) acc = radd(acc, flux_along(T + node, kap + node, k, g.nz, (long long)g.px * g.ny, hih2[2]));
    out[node] = radd(acc, src_dense ? src[node] : src_uniform);
}

// zero_constrained (grid.hpp:240-243) / apply_constraints (grid.hpp:234-238).
__global__ void k_zero_entries(const long long* __restrict__ ent, long long n, double* f, const DeviceStatus* st,
                               long long step, long long nsteps) {
    if (skip_step(st, step, nsteps)) return;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) f[ent[t]] = 0.0;
}

__global__ void k_apply_constraints(const long long* __restrict__ ent, const double* __restrict__ val, long long n,
                                    double* f, const DeviceStatus* st, long long step, long long nsteps) {
    if (skip_step(st, step, nsteps)) return;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) f[ent[t]] = val[t];
}

// pt_step_inplace / apt_step_inplace node loops (state_solver.hpp:400-442).
// form: 0 explicit APT, 1 semi-implicit APT, 2 PT.  next may alias prev.
// Non-finite results are flagged for the check_finite cadence (the constraint
// scatter that follows only writes finite pinned values, and the reference's
// Sum|x| is non-finite iff some free entry is).
__global__ void k_update_replica(Geo g, int comps, int form, const double* __restrict__ cur, const double* prev,
                                 const double* __restrict__ r, double* next, double dt, double a, double b,
                                 double inv, DeviceStatus* st, long long step, long long nsteps) {
    int i, j, k;
    if (skip_step(st, step, nsteps)) return;
    if (!owned_node(g, (long long)blockIdx.x * blockDim.x + threadIdx.x, i, j, k)) return;
    const long long node = lidx(g, i, j, k);
    bool bad = false;
    for (int c = 0; c < comps; ++c) {
        const long long e = c * g.Ns + node;
        const double cc = cur[e];
        if (form == 2) {
            next[e] = radd(cc, rmul(dt, r[e]));
        } else if (form == 0) {
            const double pp = prev[e];
            const double first = rsub(cc, pp);
            next[e] = rsub(radd(rsub(rmul(2.0, cc), pp), rmul(a, r[e])), rmul(b, first));
        } else {
            const double pp = prev[e];
            next[e] = rmul(radd(radd(rsub(rmul(2.0, cc), pp), rmul(b, cc)), rmul(a, r[e])), inv);
        }
        bad |= !isfinite(next[e]);
    }
    if (bad) mark_bad(st, step);
}

// par::sum_nodes serial branch (parallel.hpp:22-24) of r^2 in entry order
// (entry = c*N + node, node in k, j, i order): one thread, bit-exact.  With
// c0 >= 0 only component c0, continuing from *init (the team chain over slabs).
__global__ void k_sumsq_serial(Geo g, int comps, const double* __restrict__ r, double* out, int c0 = -1,
                               const double* init = nullptr) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    double s = init ? *init : 0.0;
    for (int c = c0 < 0 ? 0 : c0; c < (c0 < 0 ? comps : c0 + 1); ++c)
        for (int k = g.kb; k < g.ke; ++k)
            for (int j = 0; j < g.ny; ++j) {
                const double* row = r + c * g.Ns + lidx(g, 0, j, k);
                for (int i = 0; i < g.nx; ++i) {
                    const double v = row[i];
                    s = radd(s, rmul(v, v));
                }
            }
    *out = s;
}

// Order-free partial sums of r^2 and |x| over owned entries (fixed launch
// shape => deterministic); one partial per block, summed by k_finish_sum.
template <int MODE>  // 0: r^2, 1: |x|
__global__ void k_partial_sum(Geo g, int comps, const double* __restrict__ f, double* partials) {
    __shared__ double scratch[32];
    const long long plane = (long long)g.nx * g.ny;
    const long long owned = plane * (g.ke - g.kb);
    double s = 0.0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < owned;
         t += (long long)gridDim.x * blockDim.x) {
        const int k = g.kb + (int)(t / plane);
        const long long rr = t - (long long)(k - g.kb) * plane;
        const int j = (int)(rr / g.nx);
        const int i = (int)(rr - (long long)j * g.nx);
        const long long node = lidx(g, i, j, k);
        for (int c = 0; c < comps; ++c) {
            const double v = f[c * g.Ns + node];
            s += MODE == 0 ? v * v : fabs(v);
        }
    }
    const double b = block_sum<8>(s, scratch);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
}

__global__ void k_finish_sum(const double* __restrict__ partials, int n, double* out) {
    __shared__ double scratch[32];
    double s = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) s += partials[t];
    const double b = block_sum<8>(s, scratch);
    if (threadIdx.x == 0) *out = b;
}

}  // namespace petto_b200
