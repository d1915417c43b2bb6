// design.cuh -- design-subsystem kernels: property interpolation, sensitivities
// + clamped design update, Cahn-Hilliard step, record-time objectives.
//
// Reference: include/petto/objectives.hpp:80-480, phase_field.hpp:50-176,
// optimizer.hpp:95-112.  Per-node terms are computed in parallel with the
// reference's expression order (radd/rmul: no contraction), and every
// order-sensitive sum goes through sum_terms(): a single-thread k,j,i-order sum in
// REPLICA mode (bit-exact with the reference's threads == 1 path) or a fixed-shape
// tree in FAST mode.  Max-reductions and counts are order-free.
#pragma once

#include "common.cuh"
#include "context.hpp"

namespace petto_b200 {

#define PETTO_PI 3.141592653589793238462643383279502884

struct DesignP {
    int np;
    double props[8];
    double penalty;
    int ipen;          // integer exponent 0..8 of pow_penalty, or -1
    int ipen1;         // same for penalty - 1
    double floor_v;
};

// detail::pow_penalty (objectives.hpp:80-89)
__device__ __forceinline__ double pow_pen(double x, double e, int ie) {
    if (ie >= 0) {
        double r = 1.0;
        for (int i = 0; i < ie; ++i) r = rmul(r, x);
        return r;
    }
    return pow(x, e);
}

// compact owned index t -> (i, j, k) and the stored (pitched) index (32-bit
// divisions: a slab holds fewer than 2^32 owned nodes)
__device__ __forceinline__ long long owned_ijk(const Geo& g, long long t, int& i, int& j, int& k) {
    const unsigned plane = (unsigned)g.nx * (unsigned)g.ny;
    const unsigned tt = (unsigned)t;
    const unsigned kl = tt / plane;
    const unsigned r = tt - kl * plane;
    j = (int)(r / (unsigned)g.nx);
    i = (int)(r - (unsigned)j * (unsigned)g.nx);
    k = g.kb + (int)kl;
    return lidx(g, i, j, k);
}

// sum_i props_i pow_penalty(phi_i) (objectives.hpp:110-115) in phase order; the
// phase loop is unrolled over PETTO_MAX_PHASES so nothing is indexed at run time
// (no local-memory copies of the parameter arrays)
__device__ __forceinline__ double mix_property(const DesignP& d, const double* ph, long long Ns, long long node) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (q < d.np) acc = radd(acc, rmul(d.props[q], pow_pen(ph[q * Ns + node], d.penalty, d.ipen)));
    return acc;
}

// interpolate_into (objectives.hpp:95-116) over every stored plane.
__global__ void k_interpolate(Geo g, DesignP d, const double* __restrict__ ph, double* __restrict__ prop) {
    const unsigned plane = (unsigned)g.nx * (unsigned)g.ny;
    const long long n = (long long)plane * g.nzs;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const unsigned kl = (unsigned)t / plane;
    const unsigned r = (unsigned)t - kl * plane;
    const int j = (int)(r / (unsigned)g.nx), i = (int)(r - (unsigned)j * (unsigned)g.nx);
    const long long node = lidx(g, i, j, g.ks0 + (int)kl);
    const double acc = mix_property(d, ph, g.Ns, node);
    prop[node] = acc > d.floor_v ? acc : d.floor_v;
}

// detail::d1_along (stencil.hpp:23-31) on the pitched layout.
__device__ __forceinline__ double d1(const double* f, int t, int n, long long s, double hih) {
    if (n == 1) return 0.0;
    if (t == 0) return rmul(rsub(radd(rmul(-3.0, f[0]), rmul(4.0, f[s])), f[2 * s]), hih);
    if (t == n - 1) return rmul(radd(rsub(rmul(3.0, f[0]), rmul(4.0, f[-s])), f[-2 * s]), hih);
    return rmul(rsub(f[s], f[-s]), hih);
}

// Displacement gradient du[c][a] = d u_c / d x_a (strain_invariants' derivative_into
// calls, objectives.hpp:158-160), DIM fixed at compile time so the small arrays
// stay in registers.
template <int DIM>
__device__ __forceinline__ void grad_u(const Geo& g, const double* st, long long node, int i, int j, int k,
                                       double (&du)[DIM][DIM]) {
    const long long s[3] = {1, g.px, (long long)g.px * g.ny};
    const int idx[3] = {i, j, k};
    const int n[3] = {g.nx, g.ny, g.nz};
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int a = 0; a < DIM; ++a) du[c][a] = d1(st + c * g.Ns + node, idx[a], n[a], s[a], g.hih[a]);
}

// strain invariants (tr eps, eps:eps) (objectives.hpp:163-179)
template <int DIM>
__device__ __forceinline__ void invariants(const double (&du)[DIM][DIM], double& t, double& c2) {
    t = 0.0;
    c2 = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const double eaa = du[a][a];
        t = radd(t, eaa);
        c2 = radd(c2, rmul(eaa, eaa));
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int b = a + 1; b < DIM; ++b) {
            const double eab = rmul(0.5, radd(du[a][b], du[b][a]));
            c2 = radd(c2, rmul(rmul(2.0, eab), eab));
        }
}

// Energy-density factor of sensitivities (objectives.hpp:345-375): |grad T|^2 or
// ctr tr(eps)^2 + cec eps:eps.
template <int DIM>
__device__ __forceinline__ double energy_factor(const Geo& g, int kind, const double* st, long long node, int i,
                                                int j, int k, double ctr, double cec) {
    if (kind == 0) {
        const long long s[3] = {1, g.px, (long long)g.px * g.ny};
        const int idx[3] = {i, j, k};
        const int n[3] = {g.nx, g.ny, g.nz};
        double gsq = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const double v = d1(st + node, idx[a], n[a], s[a], g.hih[a]);
            gsq = radd(gsq, rmul(v, v));
        }
        return gsq;
    }
    double du[DIM][DIM];
    grad_u<DIM>(g, st, node, i, j, k, du);
    double t, c2;
    invariants<DIM>(du, t, c2);
    return radd(rmul(rmul(ctr, t), t), rmul(cec, c2));
}

// term[t] = phi * cell_volume (phase_mass, phase_field.hpp:84-101), compact order.
__global__ void k_term_mass(Geo g, const double* __restrict__ phi, double* __restrict__ term) {
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= owned) return;
    int i, j, k;
    const long long node = owned_ijk(g, t, i, j, k);
    term[t] = rmul(phi[node], cell_volume(g, i, j, k));
}

// single-thread ordered sum (par::serial() branch) / fixed-shape tree partials.
// `init` continues a sum over the previous slabs (the team chain, REPLICA mode).
__global__ void k_sum_serial(const double* __restrict__ term, long long n, double* out,
                             const double* init = nullptr) {
    if (threadIdx.x || blockIdx.x) return;
    double s = init ? *init : 0.0;
    for (long long t = 0; t < n; ++t) s = radd(s, term[t]);
    *out = s;
}

__global__ void k_sum_partials(const double* __restrict__ term, long long n, double* partials) {
    __shared__ double scratch[32];
    double s = 0.0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
        s += term[t];
    const double b = block_sum<8>(s, scratch);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
}

__global__ void k_sum_finish(const double* __restrict__ partials, int n, double* out) {
    __shared__ double scratch[32];
    double s = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) s += partials[t];
    const double b = block_sum<8>(s, scratch);
    if (threadIdx.x == 0) *out = b;
}

// ------------------------------------------------------------- sensitivities

// gc_i = dprop_i * factor * vol (objectives.hpp:393-420) for every phase, plus
// block partial maxima of |gc_i| (par::max_abs_nodes, order-free).
template <int DIM>
__global__ void k_sens_gc(Geo g, DesignP d, int kind, double ctr, double cec, const double* __restrict__ ph,
                          const double* __restrict__ st, double* __restrict__ gc, double* __restrict__ pmax) {
    __shared__ double smax[8][8];
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    double lmax[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) lmax[q] = 0.0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < owned;
         t += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        const long long node = owned_ijk(g, t, i, j, k);
        const double fac = energy_factor<DIM>(g, kind, st, node, i, j, k, ctr, cec);
        const double vol = cell_volume(g, i, j, k);
        const double mix = mix_property(d, ph, g.Ns, node);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q >= d.np) continue;
            const double dprop =
                mix > d.floor_v ? rmul(rmul(d.penalty, d.props[q]), pow_pen(ph[q * g.Ns + node], d.penalty - 1.0, d.ipen1))
                                : 0.0;
            const double v = rmul(rmul(dprop, fac), vol);
            gc[q * g.Ns + node] = v;
            lmax[q] = fmax(lmax[q], fabs(v));
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (q >= d.np) continue;
        const double m = warp_max(lmax[q]);
        if (l == 0) smax[q][w] = m;
    }
    __syncthreads();
    if (threadIdx.x < d.np) {
        double m = 0.0;
        for (int ww = 0; ww < 8; ++ww) m = fmax(m, smax[threadIdx.x][ww]);
        pmax[blockIdx.x * 8 + threadIdx.x] = m;
    }
}

// detail::d1_along (stencil.hpp:23-31) from values: f(t-2) .. f(t+2) along the axis
__device__ __forceinline__ double d1v(int t, int n, double fm2, double fm1, double f0, double fp1, double fp2,
                                      double hih) {
    if (n == 1) return 0.0;
    if (t == 0) return rmul(rsub(radd(rmul(-3.0, f0), rmul(4.0, fp1)), fp2), hih);
    if (t == n - 1) return rmul(radd(rsub(rmul(3.0, f0), rmul(4.0, fm1)), fm2), hih);
    return rmul(rsub(fp1, fm1), hih);
}

// 3D sensitivities streamed along z: a thread owns one (i, j) column of a z-chunk
// and slides a window of u over planes k-1, k, k+1, so every node of u comes from
// HBM once (the x / y neighbours hit L1).  Same per-node expressions as k_sens_gc
// (bit-identical gc); block maxima of |gc_q| into pmax[block][8].
template <int NP, int KIND>
__global__ void __launch_bounds__(128) k_sens_gc3(Geo g, DesignP d, double ctr, double cec,
                                                  const double* __restrict__ ph, const double* __restrict__ st,
                                                  double* __restrict__ gc, double* __restrict__ pmax, int zc) {
    __shared__ double smax[4][NP];
    const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 4 + threadIdx.y;
    const int k0 = g.kb + blockIdx.z * zc, k1 = min(k0 + zc, g.ke);
    const bool valid = i < g.nx && j < g.ny;
    constexpr int comps = KIND == 0 ? 1 : 3;
    const long long sz = (long long)g.px * g.ny;
    double lmax[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) lmax[q] = 0.0;
    double wm[3] = {0.0, 0.0, 0.0}, w0[3] = {0.0, 0.0, 0.0}, wp[3] = {0.0, 0.0, 0.0};  // u at k-1, k, k+1
    if (valid) {
        const long long n0 = lidx(g, i, j, k0);
#pragma unroll
        for (int c = 0; c < comps; ++c) {
            if (k0 > 0) wm[c] = st[c * g.Ns + n0 - sz];
            w0[c] = st[c * g.Ns + n0];
        }
    }
    for (int k = k0; k < k1; ++k) {
        if (!valid) continue;
        const long long node = lidx(g, i, j, k);
#pragma unroll
        for (int c = 0; c < comps; ++c) wp[c] = k + 1 < g.nz ? st[c * g.Ns + node + sz] : 0.0;
        double fac;
        if (KIND == 0) {
            const double gx = d1(st + node, i, g.nx, 1, g.hih[0]);
            const double gy = d1(st + node, j, g.ny, g.px, g.hih[1]);
            const double fp2 = k == 0 ? st[node + 2 * sz] : 0.0, fm2 = k == g.nz - 1 ? st[node - 2 * sz] : 0.0;
            const double gz = d1v(k, g.nz, fm2, wm[0], w0[0], wp[0], fp2, g.hih[2]);
            fac = radd(radd(radd(0.0, rmul(gx, gx)), rmul(gy, gy)), rmul(gz, gz));
        } else {
            double du[3][3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double* f = st + c * g.Ns + node;
                du[c][0] = d1(f, i, g.nx, 1, g.hih[0]);
                du[c][1] = d1(f, j, g.ny, g.px, g.hih[1]);
                const double fp2 = k == 0 ? f[2 * sz] : 0.0, fm2 = k == g.nz - 1 ? f[-2 * sz] : 0.0;
                du[c][2] = d1v(k, g.nz, fm2, wm[c], w0[c], wp[c], fp2, g.hih[2]);
            }
            double t, c2;
            invariants<3>(du, t, c2);
            fac = radd(rmul(rmul(ctr, t), t), rmul(cec, c2));
        }
        const double vol = cell_volume(g, i, j, k);
        double mix = 0.0;
        double pq[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            pq[q] = ph[q * g.Ns + node];
            mix = radd(mix, rmul(d.props[q], pow_pen(pq[q], d.penalty, d.ipen)));
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double dprop =
                mix > d.floor_v ? rmul(rmul(d.penalty, d.props[q]), pow_pen(pq[q], d.penalty - 1.0, d.ipen1)) : 0.0;
            const double v = rmul(rmul(dprop, fac), vol);
            gc[q * g.Ns + node] = v;
            lmax[q] = fmax(lmax[q], fabs(v));
        }
#pragma unroll
        for (int c = 0; c < comps; ++c) {
            wm[c] = w0[c];
            w0[c] = wp[c];
        }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const double m = warp_max(lmax[q]);
        if (threadIdx.x == 0) smax[threadIdx.y][q] = m;
    }
    __syncthreads();
    const int tid = threadIdx.y * 32 + threadIdx.x;
    if (tid < NP) {
        const double m = fmax(fmax(smax[0][tid], smax[1][tid]), fmax(smax[2][tid], smax[3][tid]));
        const long long b = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        pmax[b * 8 + tid] = m;
    }
}

// Scalars of the update (objectives.hpp:386-398, 424-436, 456-468), computed on
// the device from the reduced masses / maxima.  dsc layout: see DS_* below.
enum {
    DS_MASS = 0,     // [8] phase masses (pre-update)
    DS_GMAX = 8,     // [8]
    DS_RACC = 16,    // [8] region sums of phi*vol
    DS_RVOL = 24,    // region volume
    DS_CSCALE = 32,  // [8]
    DS_DM = 40,      // [8]
    DS_RCOEFF = 48,  // [8]
    DS_TMP = 56,     // [8] scratch sums
    DS_DRIFT = 64,   // accumulated clamp mass drift
    DS_CH = 72,      // [8][3] ch masses: before, pre, post
    DS_OBJ = 104,    // [4] compliance, unity, separation count, spare
    DS_CHAIN = 108,  // running value of a team chain sum (REPLICA)
    DS_CHAIN_IN = 109,
    DS_COUNT = 128
};

struct UpdateScal {
    double inv_vol;
    double fractions[8];
    double region_fractions[8];
    int has_region;
    double alpha_c, alpha_v, alpha_u, alpha_r;
    int normalize, sign;
};

// this slab's max|gc_i| (par::max_abs_nodes, parallel.hpp:33-42) from the block maxima
// (one warp per phase; a maximum is order-free)
__global__ void k_local_gmax(int np, const double* __restrict__ pmax, int nblocks, double* dsc) {
    const int q = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (blockIdx.x || q >= np) return;
    double m = 0.0;
    for (int b = l; b < nblocks; b += 32) m = fmax(m, pmax[b * 8 + q]);
    m = warp_max(m);
    if (l == 0) dsc[DS_GMAX + q] = m;
}

// dsc[DS_GMAX] holds the global maxima (team-reduced), dsc[DS_MASS] the masses
__global__ void k_design_scalars(int np, UpdateScal u, double* dsc) {
    if (threadIdx.x || blockIdx.x) return;
    for (int q = 0; q < np; ++q) {
        const double m = dsc[DS_GMAX + q];
        const double mean = dsc[DS_MASS + q] * u.inv_vol;  // volume_fractions
        dsc[DS_DM + q] = (2.0 * (mean - u.fractions[q])) * u.inv_vol;
        double cs = 0.0;
        if (u.alpha_c > 0) {
            if (u.normalize)
                cs = m > 0 ? (double)u.sign * u.alpha_c / m : 0.0;
            else
                cs = (double)u.sign * u.alpha_c;
        }
        dsc[DS_CSCALE + q] = cs;
        if (u.has_region) {
            const double vb = dsc[DS_RVOL];
            const double mb = dsc[DS_RACC + q] / vb;
            dsc[DS_RCOEFF + q] = (2.0 * (mb - u.region_fractions[q])) / vb;
        }
    }
}

// design_update_inplace (objectives.hpp:444-480) with gv/gu/gr formed on the fly
// from the pre-update phases of the node.
template <int NP>
__global__ void k_design_update(Geo g, UpdateScal u, const double* __restrict__ dsc, const double* __restrict__ gc,
                                const unsigned char* __restrict__ region, double* ph) {
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= owned) return;
    int i, j, k;
    const long long node = owned_ijk(g, t, i, j, k);
    const double vol = cell_volume(g, i, j, k);
    double p[NP];
    double ssum = -1.0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        p[q] = ph[q * g.Ns + node];
        ssum = radd(ssum, p[q]);
    }
    const double gu = rmul(rmul(2.0, ssum), vol);
    const bool in_region = u.has_region && region[node];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const double gv = rmul(dsc[DS_DM + q], vol);
        double step = radd(radd(rmul(dsc[DS_CSCALE + q], gc[q * g.Ns + node]), rmul(u.alpha_v, gv)), rmul(u.alpha_u, gu));
        if (u.has_region) {
            const double gr = in_region ? rmul(dsc[DS_RCOEFF + q], vol) : 0.0;
            step = radd(step, rmul(u.alpha_r, gr));
        }
        const double v = rsub(p[q], step);
        ph[q * g.Ns + node] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
}

// region sums (region_fractions_measured / region_volume, objectives.hpp:251-288):
// terms in the region list order.
__global__ void k_region_terms(Geo g, const long long* __restrict__ nodes, long long n, const double* __restrict__ phi,
                               double* __restrict__ term) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const long long gn = nodes[t];
    const long long plane = (long long)g.nx * g.ny;
    const int k = (int)(gn / plane);
    const long long r = gn - (long long)k * plane;
    const int j = (int)(r / g.nx), i = (int)(r - (long long)j * g.nx);
    const double cv = cell_volume(g, i, j, k);
    term[t] = phi ? rmul(phi[lidx(g, i, j, k)], cv) : cv;
}

// --------------------------------------------------------------- Cahn-Hilliard

// dwell (phase_field.hpp:56-60)
__device__ __forceinline__ double dwell(double p) {
    return rmul(PETTO_PI / 64.0, sin(rmul(2.0 * PETTO_PI, p)));
}

// detail::lap_along (stencil.hpp:109-116)
__device__ __forceinline__ double lap_along(const double* f, int t, int n, long long s, double inv_h2) {
    if (n == 1) return 0.0;
    if (t == 0) return rmul(rmul(2.0, rsub(f[s], f[0])), inv_h2);
    if (n - 1 == t) return rmul(rmul(2.0, rsub(f[-s], f[0])), inv_h2);
    return rmul(radd(rsub(f[s], f[0]), rsub(f[-s], f[0])), inv_h2);
}

__device__ __forceinline__ double lap_noflux(const Geo& g, const double* f, long long node, int i, int j, int k) {
    // g.ilap[a] = rdiv(1.0, rmul(h, h))
    double acc = lap_along(f + node, i, g.nx, 1, g.ilap[0]);
    acc = radd(acc, lap_along(f + node, j, g.ny, g.px, g.ilap[1]));
    if (g.nz > 1) acc = radd(acc, lap_along(f + node, k, g.nz, (long long)g.px * g.ny, g.ilap[2]));
    return acc;
}

// chemical_potential_into (phase_field.hpp:63-72): mu = dwell(phi) - gamma lap(phi)
__global__ void k_chem_potential(Geo g, const double* __restrict__ phi, double gamma, double* __restrict__ mu) {
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= owned) return;
    int i, j, k;
    const long long node = owned_ijk(g, t, i, j, k);
    mu[node] = rsub(dwell(phi[node]), rmul(gamma, lap_noflux(g, phi, node, i, j, k)));
}

// phi += dt D lap(mu) (phase_field.hpp:147-149); pre-clamp mass terms
__global__ void k_ch_update(Geo g, const double* __restrict__ mu, double step, double* phi, double* __restrict__ term) {
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= owned) return;
    int i, j, k;
    const long long node = owned_ijk(g, t, i, j, k);
    const double v = radd(phi[node], rmul(step, lap_noflux(g, mu, node, i, j, k)));
    phi[node] = v;
    term[t] = rmul(v, cell_volume(g, i, j, k));
}

// clamp to [0, 1] (phase_field.hpp:151-153); post-clamp mass terms, non-finite flag
__global__ void k_ch_clamp(Geo g, double* phi, double* __restrict__ term, unsigned* flag) {
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= owned) return;
    int i, j, k;
    const long long node = owned_ijk(g, t, i, j, k);
    const double p = phi[node];
    const double v = p < 0.0 ? 0.0 : (p > 1.0 ? 1.0 : p);
    phi[node] = v;
    if (!isfinite(v)) atomicOr(flag, 4u);
    term[t] = rmul(v, cell_volume(g, i, j, k));
}

// ------------------------------------------------- FAST: sums as block partials
// The FAST-mode sums of the design loop without the per-node term arrays: each
// kernel walks the owned nodes with the same grid-stride partition as
// k_sum_partials over a term array (grid = min(npartials, blocks), 256 threads) and
// leaves one block_sum per block, so the totals (k_sum_finish) are bit-identical
// to the term-array route while the terms never touch HBM.

// phase_mass partials of phi (phase_field.hpp:84-101)
__global__ void k_mass_partials(Geo g, const double* __restrict__ phi, double* __restrict__ partials) {
    __shared__ double scratch[32];
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    double s = 0.0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < owned;
         t += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        const long long node = owned_ijk(g, t, i, j, k);
        s += rmul(phi[node], cell_volume(g, i, j, k));
    }
    const double b = block_sum<8>(s, scratch);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
}

// chemical_potential_into (phase_field.hpp:63-72) + the mass before the step
__global__ void k_chem_potential_mass(Geo g, const double* __restrict__ phi, double gamma, double* __restrict__ mu,
                                      double* __restrict__ partials) {
    __shared__ double scratch[32];
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    double s = 0.0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < owned;
         t += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        const long long node = owned_ijk(g, t, i, j, k);
        const double p = phi[node];
        mu[node] = rsub(dwell(p), rmul(gamma, lap_noflux(g, phi, node, i, j, k)));
        s += rmul(p, cell_volume(g, i, j, k));
    }
    const double b = block_sum<8>(s, scratch);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
}

// phi += dt D lap(mu), pre-clamp mass, clamp to [0, 1], post-clamp mass, non-finite
// flag (phase_field.hpp:147-155) in one pass
__global__ void k_ch_update_clamp(Geo g, const double* __restrict__ mu, double step, double* phi,
                                  double* __restrict__ pre, double* __restrict__ post, unsigned* flag) {
    __shared__ double scratch[32];
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    double sp = 0.0, sq = 0.0;
    bool bad = false;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < owned;
         t += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        const long long node = owned_ijk(g, t, i, j, k);
        const double cv = cell_volume(g, i, j, k);
        const double v = radd(phi[node], rmul(step, lap_noflux(g, mu, node, i, j, k)));
        const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        phi[node] = c;
        bad |= !isfinite(c);
        sp += rmul(v, cv);
        sq += rmul(c, cv);
    }
    if (bad) atomicOr(flag, 4u);
    const double bp = block_sum<8>(sp, scratch);
    const double bq = block_sum<8>(sq, scratch);
    if (threadIdx.x == 0) {
        pre[blockIdx.x] = bp;
        post[blockIdx.x] = bq;
    }
}

// ------------------------------------------------------------------ objectives

// Per-node terms of evaluate_objectives (objectives.hpp:126-247, 304-320):
// compliance (thermal: kappa |grad T|^2 dV, elastic: (lam tr^2 + 2 mu eps:eps) dV with
// make_lame of the re-interpolated property), unity (sum phi - 1)^2 dV, and the
// phase-separation indicator (optimizer.hpp:95-112).
template <int DIM>
__global__ void k_objective_terms(Geo g, DesignP d, int kind, double cl, double cm, const double* __restrict__ ph,
                                  const double* __restrict__ st, double* __restrict__ tcomp,
                                  double* __restrict__ tunity, unsigned long long* sep_count) {
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool near = false;
    if (t < owned) {
        int i, j, k;
        const long long node = owned_ijk(g, t, i, j, k);
        const double cv = cell_volume(g, i, j, k);
        double acc = 0.0, s = -1.0, worst = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q >= d.np) continue;
            const double p = ph[q * g.Ns + node];
            acc = radd(acc, rmul(d.props[q], pow_pen(p, d.penalty, d.ipen)));
            s = radd(s, p);
            const double dd = p < rsub(1.0, p) ? p : rsub(1.0, p);
            if (dd > worst) worst = dd;
        }
        near = worst < 0.1;
        const double E = acc > d.floor_v ? acc : d.floor_v;
        double c;
        if (kind == 0) {
            c = rmul(rmul(E, energy_factor<DIM>(g, 0, st, node, i, j, k, 0.0, 0.0)), cv);
        } else {
            double du[DIM][DIM], tr, c2;
            grad_u<DIM>(g, st, node, i, j, k, du);
            invariants<DIM>(du, tr, c2);
            const double lam = rmul(cl, E), mu = rmul(cm, E);
            c = rmul(radd(rmul(rmul(lam, tr), tr), rmul(rmul(2.0, mu), c2)), cv);
        }
        tcomp[t] = c;
        tunity[t] = rmul(rmul(s, s), cv);
    }
    const unsigned cnt = __popc(__ballot_sync(0xffffffffu, near));
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(sep_count, (unsigned long long)cnt);
}

// Team reduction on the group lead: n contexts' values gathered rank after rank,
// combined in rank order (deterministic).  op: 0 sum f64, 1 max f64, 2 min i64,
// 3 sum u64, 4 max u32.
__global__ void k_team_combine(const void* __restrict__ buf, int n, int count, int op, void* out) {
    const int v = threadIdx.x;
    if (blockIdx.x || v >= count) return;
    if (op == 0 || op == 1) {
        const double* b = static_cast<const double*>(buf);
        double a = b[v];
        for (int r = 1; r < n; ++r) a = op == 0 ? radd(a, b[r * count + v]) : fmax(a, b[r * count + v]);
        static_cast<double*>(out)[v] = a;
    } else if (op == 2) {
        const long long* b = static_cast<const long long*>(buf);
        long long a = b[v];
        for (int r = 1; r < n; ++r) a = min(a, b[r * count + v]);
        static_cast<long long*>(out)[v] = a;
    } else if (op == 3) {
        const unsigned long long* b = static_cast<const unsigned long long*>(buf);
        unsigned long long a = b[v];
        for (int r = 1; r < n; ++r) a += b[r * count + v];
        static_cast<unsigned long long*>(out)[v] = a;
    } else {
        const unsigned* b = static_cast<const unsigned*>(buf);
        unsigned a = b[v];
        for (int r = 1; r < n; ++r) a = max(a, b[r * count + v]);
        static_cast<unsigned*>(out)[v] = a;
    }
}

__global__ void k_check_finite_phases(Geo g, int np, const double* __restrict__ ph, unsigned* flag) {
    const long long owned = (long long)g.nx * g.ny * (g.ke - g.kb);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= owned) return;
    int i, j, k;
    const long long node = owned_ijk(g, t, i, j, k);
    for (int q = 0; q < np; ++q)
        if (!isfinite(ph[q * g.Ns + node])) atomicOr(flag, 4u);
}

inline void design_free(petto_ctx* ctx) {
    cudaFree(ctx->phases);
    cudaFree(ctx->gc);
    cudaFree(ctx->scratch1);
    cudaFree(ctx->scratch2);
    cudaFree(ctx->region_dev);
    cudaFree(ctx->region_mask);
    cudaFree(ctx->term1);
    cudaFree(ctx->term2);
    cudaFree(ctx->pmax);
    cudaFree(ctx->count);
    ctx->count = nullptr;
    ctx->phases = ctx->gc = ctx->scratch1 = ctx->scratch2 = nullptr;
    ctx->term1 = ctx->term2 = ctx->pmax = nullptr;
    ctx->region_dev = nullptr;
    ctx->region_mask = nullptr;
}

}  // namespace petto_b200
