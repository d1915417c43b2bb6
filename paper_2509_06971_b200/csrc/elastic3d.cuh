// elastic3d.cuh -- fused 3D elasticity residual + PT/APT update (fast mode).
//
// Computes, for every owned node, r = -(sum_cells E_c K_e u_c)/V_node - f
// (ElasticityOperator::residual, state_solver.hpp:327-385) and immediately the
// pseudo-time update (pt_step_inplace / apt_step_inplace, :400-442) with the
// constraint overwrite (apply_constraints, grid.hpp:234-238): one HBM pass per
// step instead of the reference's three.
//
// Algorithm (cell-centric, modal):
//   * the unit-cell stiffness is applied in the Walsh-Hadamard corner-parity
//     basis, where it has 45 structural nonzeros (stiffness.hpp); the forward and
//     inverse transforms factor into x/y/z butterflies;
//   * CTA = 9 warps: lane l <-> x = i0 + l (32 nodes), warp w <-> row j0-1+w
//     (warp 0 is the y-halo row of cells whose top corners feed row j0);
//   * each CTA streams along z (the outermost axis): per cell plane it keeps the
//     previous plane's y/x-butterflies (12+1 doubles) and the top-face
//     contributions (12 doubles) in registers;
//   * node planes arrive by TMA (cp.async.bulk.tensor, zero-filled outside the
//     grid) into a 5-stage shared-memory ring guarded by mbarriers, issued 4
//     tasks ahead by one elected thread;
//   * x-neighbour contributions travel by warp shuffle, y-neighbour ones through
//     a double-buffered shared tile, and the contribution of the previous x-tile's
//     last column through a small shared "x-halo" array -- CTAs walk the x-tiles
//     of their (strip, z-run) sequentially, so no cell is computed twice in x;
//   * work = (y-strip, plane) units split evenly over a persistent grid.
// Algorithmic HBM bytes per node-update: u_n 24 + u_{n-1} 24 + E 8 + u_{n+1} 24
// (+1 mask byte); PT drops u_{n-1}.
#pragma once

#include "common.cuh"

namespace petto_b200 {
namespace e3 {

constexpr int W = 7;           // owned node rows per tile
constexpr int NWARP = W + 1;   // + y-halo warp
constexpr int NTHREADS = NWARP * 32;
constexpr int BOXX = 34;       // TMA box width (33 columns used; 16-byte multiple)
constexpr int UROWS = W + 2;   // rows j0-1 .. j0+W
constexpr int S = 5;           // pipeline depth
constexpr int LMAX = 64;       // longest z sub-run (x-halo buffer)

constexpr int r128(int b) { return (b + 127) / 128 * 128; }
constexpr int OFF_U = 0;                                    // [3][UROWS][BOXX] f64
constexpr int OFF_E = r128(3 * UROWS * BOXX * 8);           // [UROWS][BOXX] f64
constexpr int OFF_P = OFF_E + r128(UROWS * BOXX * 8);       // [3][W][32] f64
constexpr int OFF_M = OFF_P + r128(3 * W * 32 * 8);         // [W][32] u8
constexpr int STAGE_BYTES = OFF_M + r128(W * 32);
constexpr uint32_t BYTES_UE = 3 * UROWS * BOXX * 8 + UROWS * BOXX * 8;
constexpr uint32_t BYTES_P = 3 * W * 32 * 8;
constexpr uint32_t BYTES_M = W * 32;

constexpr int OFF_Y = S * STAGE_BYTES;                      // [2][NWARP][6][32] f64
constexpr int OFF_X = OFF_Y + 2 * NWARP * 6 * 32 * 8;       // [2][LMAX][NWARP][3] f64
constexpr int OFF_BAR = OFF_X + 2 * LMAX * NWARP * 3 * 8;   // [S] mbarriers
constexpr int OFF_RED = OFF_BAR + S * 8;                    // [NWARP] f64
constexpr int OFF_PIT = OFF_RED + 16 * 8;                   // producer cursor
constexpr int SMEM_BYTES = OFF_PIT + 64;

struct Params {
    Geo g;
    double kh[45];     // modal stiffness (stiffness.hpp pattern order)
    double e_scale;    // (sum of 8 corner E) -> E_cell: cm * 2(1+nu_op) / 8
    double inv_base;   // 1 / (hx hy hz)
    int form;          // 0 APT explicit, 1 APT semi-implicit, 2 PT, 3 residual only
    double dt, a, b, inv;
    double* next;      // output field (may alias the previous iterate)
    const double* aux; // pinned values / loads (3 x Ns)
    double* partials;  // per-CTA sum of r^2 over unconstrained entries (nullable)
    DeviceStatus* status;
    long long step, nsteps;  // 1-based step index within the solve, total steps
    int ntx;           // x tiles
    int nzo;           // owned planes
    long long units;   // strips * nzo
};

struct TaskIt {
    long long u, u_end;
    int s, ka, len, t, kk;
    bool valid;

    __device__ void subrun(const Params& P) {
        if (u >= u_end) {
            valid = false;
            return;
        }
        s = (int)(u / P.nzo);
        ka = P.g.kb + (int)(u - (long long)s * P.nzo);
        long long lim = (long long)(s + 1) * P.nzo;
        if (lim > u_end) lim = u_end;
        long long l = lim - u;
        len = (int)(l < LMAX ? l : LMAX);
        t = 0;
        kk = 0;
        valid = true;
    }
    __device__ void init(const Params& P) {
        u = (long long)blockIdx.x * P.units / gridDim.x;
        u_end = (long long)(blockIdx.x + 1) * P.units / gridDim.x;
        subrun(P);
    }
    __device__ void next(const Params& P) {
        if (++kk == len + 2) {
            kk = 0;
            if (++t == P.ntx) {
                u += len;
                subrun(P);
            }
        }
    }
    __device__ int kc() const { return ka - 2 + kk; }
};

__device__ __forceinline__ void issue(const Params& P, const TaskIt& it, unsigned char* smem, uint64_t* bars,
                                      int stage, const CUtensorMap* tU, const CUtensorMap* tE,
                                      const CUtensorMap* tP, const CUtensorMap* tM) {
    unsigned char* st = smem + stage * STAGE_BYTES;
    const bool own = it.kk >= 2;
    const bool need_p = own && P.form <= 1;
    uint32_t bytes = BYTES_UE + (own ? BYTES_M : 0) + (need_p ? BYTES_P : 0);
    mbar_expect_tx(&bars[stage], bytes);
    const int i0 = it.t * 32, j0 = it.s * W;
    const int zn = it.kc() + 1 - P.g.ks0;
    tma_load_4d(st + OFF_U, tU, &bars[stage], i0, j0 - 1, zn, 0);
    tma_load_3d(st + OFF_E, tE, &bars[stage], i0, j0 - 1, zn);
    if (own) {
        const int zc = it.kc() - P.g.ks0;
        tma_load_3d(st + OFF_M, tM, &bars[stage], i0, j0, zc);
        if (need_p) tma_load_4d(st + OFF_P, tP, &bars[stage], i0, j0, zc, 0);
    }
}

__global__ void __launch_bounds__(NTHREADS, 1)
    k_elastic3d_fast(const __grid_constant__ Params P, const __grid_constant__ CUtensorMap tU,
                     const __grid_constant__ CUtensorMap tE, const __grid_constant__ CUtensorMap tP,
                     const __grid_constant__ CUtensorMap tM) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    double* sY = reinterpret_cast<double*>(smem + OFF_Y);
    double* sX = reinterpret_cast<double*>(smem + OFF_X);
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const Geo& g = P.g;
    if (skip_step(P.status, P.step, P.nsteps)) return;

    TaskIt it;
    it.init(P);
    if (threadIdx.x == 0) {
        prefetch_tmap(&tU);
        prefetch_tmap(&tE);
        prefetch_tmap(&tP);
        prefetch_tmap(&tM);
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // producer cursor, S-1 tasks ahead; lives in shared memory (thread 0 only)
    TaskIt& pit = *reinterpret_cast<TaskIt*>(smem + OFF_PIT);
    if (threadIdx.x == 0) {
        pit = it;
        for (int s = 0; s < S - 1 && pit.valid; ++s) {
            issue(P, pit, smem, bars, s, &tU, &tE, &tP, &tM);
            pit.next(P);
        }
    }

    double Bc[4][3], Ec = 0.0, top[4][3], ucar[3];
    double rsq = 0.0;
    unsigned bad = 0;
    long long q = 0;
    for (; it.valid; it.next(P), ++q) {
        const int st = (int)(q % S);
        mbar_wait(&bars[st], (uint32_t)((q / S) & 1));
        const unsigned char* sb = smem + st * STAGE_BYTES;
        const double* su = reinterpret_cast<const double*>(sb + OFF_U);
        const double* se = reinterpret_cast<const double*>(sb + OFF_E);
        const int kc = it.kc();
        const int i = it.t * 32 + l;
        const int j = it.s * W - 1 + w;

        // ---- forward butterflies of node plane kc+1 for cell (i, j)
        double Bn[4][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double* r0 = su + (c * UROWS + w) * BOXX + l;
            const double a = r0[0], b = r0[1], cc = r0[BOXX], d = r0[BOXX + 1];
            const double A0 = a + b, A1 = a - b, A0n = cc + d, A1n = cc - d;
            Bn[0][c] = A0 + A0n;
            Bn[1][c] = A1 + A1n;
            Bn[2][c] = A0 - A0n;
            Bn[3][c] = A1 - A1n;
        }
        const double* e0 = se + w * BOXX + l;
        const double En = (e0[0] + e0[1]) + (e0[BOXX] + e0[BOXX + 1]);

        const int kind = it.kk;  // 0 prologue, 1 first cell plane, >= 2 owned node plane
        double face[4][3];
        if (kind == 0) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    Bc[q4][c] = Bn[q4][c];
                    top[q4][c] = 0.0;
                }
            Ec = En;
        } else {
            // z butterflies -> modal coefficients C[s][c], s = sx + 2 sy + 4 sz
            double C[8][3];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    C[q4][c] = Bc[q4][c] + Bn[q4][c];
                    C[q4 + 4][c] = Bc[q4][c] - Bn[q4][c];
                    Bc[q4][c] = Bn[q4][c];
                }
            const bool valid = i <= g.nx - 2 && j >= 0 && j <= g.ny - 2 && kc >= 0 && kc <= g.nz - 2;
            const double ecell = valid ? (Ec + En) * P.e_scale : 0.0;
            Ec = En;
#pragma unroll
            for (int s = 1; s < 8; ++s)
#pragma unroll
                for (int c = 0; c < 3; ++c) C[s][c] *= ecell;
            const double* k = P.kh;
            double F[8][3];
            F[0][0] = F[0][1] = F[0][2] = 0.0;
            F[1][0] = k[0] * C[1][0] + k[1] * C[2][1] + k[2] * C[4][2];
            F[1][1] = k[3] * C[1][1] + k[4] * C[2][0];
            F[1][2] = k[5] * C[1][2] + k[6] * C[4][0];
            F[2][0] = k[7] * C[1][1] + k[8] * C[2][0];
            F[2][1] = k[9] * C[1][0] + k[10] * C[2][1] + k[11] * C[4][2];
            F[2][2] = k[12] * C[2][2] + k[13] * C[4][1];
            F[4][0] = k[14] * C[1][2] + k[15] * C[4][0];
            F[4][1] = k[16] * C[2][2] + k[17] * C[4][1];
            F[4][2] = k[18] * C[1][0] + k[19] * C[2][1] + k[20] * C[4][2];
            F[3][0] = k[21] * C[3][0] + k[22] * C[6][2];
            F[3][1] = k[23] * C[3][1] + k[24] * C[5][2];
            F[3][2] = k[25] * C[3][2] + k[26] * C[5][1] + k[27] * C[6][0];
            F[5][0] = k[28] * C[5][0] + k[29] * C[6][1];
            F[5][1] = k[30] * C[3][2] + k[31] * C[5][1] + k[32] * C[6][0];
            F[5][2] = k[33] * C[3][1] + k[34] * C[5][2];
            F[6][0] = k[35] * C[3][2] + k[36] * C[5][1] + k[37] * C[6][0];
            F[6][1] = k[38] * C[5][0] + k[39] * C[6][1];
            F[6][2] = k[40] * C[3][0] + k[41] * C[6][2];
            F[7][0] = k[42] * C[7][0];
            F[7][1] = k[43] * C[7][1];
            F[7][2] = k[44] * C[7][2];
            // inverse z butterflies: bottom face (node plane kc), top face (kc+1)
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    face[q4][c] = top[q4][c] + (F[q4][c] + F[q4 + 4][c]);
                    top[q4][c] = F[q4][c] - F[q4 + 4][c];
                }
        }

        // inverse y butterflies of the face; row j+1's share goes to warp w+1
        double Yj[2][3];
        double* sYw = sY + ((size_t)(q & 1) * NWARP * 6 * 32);
        if (kind >= 2) {
#pragma unroll
            for (int sx = 0; sx < 2; ++sx)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    Yj[sx][c] = face[sx][c] + face[sx + 2][c];
                    sYw[(w * 6 + sx * 3 + c) * 32 + l] = face[sx][c] - face[sx + 2][c];
                }
        }
        __syncthreads();
        if (threadIdx.x == 0 && pit.valid) {
            issue(P, pit, smem, bars, (int)((q + S - 1) % S), &tU, &tE, &tP, &tM);
            pit.next(P);
        }
        if (kind >= 2) {
            // edge sums, inverse x butterflies, node assembly
            double Xi[3], Xn[3];
            if (w >= 1) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double e0v = Yj[0][c] + sYw[((w - 1) * 6 + c) * 32 + l];
                    const double e1v = Yj[1][c] + sYw[((w - 1) * 6 + 3 + c) * 32 + l];
                    Xi[c] = e0v + e1v;
                    Xn[c] = e0v - e1v;
                }
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) Xi[c] = Xn[c] = 0.0;
            }
            const int zi = kc - it.ka;
            double* xw = sX + ((size_t)(it.t & 1) * LMAX + zi) * NWARP * 3 + w * 3;
            const double* xr = sX + ((size_t)((it.t + 1) & 1) * LMAX + zi) * NWARP * 3 + w * 3;
            double acc[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double nb = __shfl_up_sync(0xffffffffu, Xn[c], 1);
                acc[c] = Xi[c] + (l > 0 ? nb : (it.t > 0 ? xr[c] : 0.0));
            }
            if (l == 31) {
#pragma unroll
                for (int c = 0; c < 3; ++c) xw[c] = Xn[c];
            }
            if (w >= 1 && i < g.nx && j < g.ny) {
                const double* sp = reinterpret_cast<const double*>(sb + OFF_P);
                const unsigned char mk = (sb + OFF_M)[(w - 1) * 32 + l];
                const double invv = inv_volume_fast(g, P.inv_base, i, j, kc);
                const long long node = lidx(g, i, j, kc);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const bool pinned = (mk >> c) & 1;
                    const double f = ((mk & 8) && !pinned) ? P.aux[c * g.Ns + node] : 0.0;
                    const double r = -acc[c] * invv - f;
                    double nv;
                    if (pinned) {
                        nv = P.form == 3 ? 0.0 : P.aux[c * g.Ns + node];
                    } else {
                        rsq += r * r;
                        const double cu = ucar[c];
                        if (P.form == 0) {
                            const double pp = sp[(c * W + (w - 1)) * 32 + l];
                            nv = 2.0 * cu - pp + P.a * r - P.b * (cu - pp);
                        } else if (P.form == 1) {
                            const double pp = sp[(c * W + (w - 1)) * 32 + l];
                            nv = (2.0 * cu - pp + P.b * cu + P.a * r) * P.inv;
                        } else if (P.form == 2) {
                            nv = cu + P.dt * r;
                        } else {
                            nv = r;
                        }
                    }
                    bad |= !isfinite(nv);
                    P.next[c * g.Ns + node] = nv;
                }
            }
        }
        // own node of plane kc+1 feeds next task's update (this stage is only
        // recycled after the next task's barrier)
#pragma unroll
        for (int c = 0; c < 3; ++c) ucar[c] = su[(c * UROWS + w) * BOXX + l];
    }

    // CTA reduction of r^2 (fixed order) and the non-finite flag
    double* red = reinterpret_cast<double*>(smem + OFF_RED);
    rsq = warp_sum(rsq);
    bad = __any_sync(0xffffffffu, bad);
    __syncthreads();
    if (l == 0) red[w] = rsq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < NWARP; ++k) s += red[k];
        if (P.partials) P.partials[blockIdx.x] = s;
    }
    if (bad && l == 0) mark_bad(P.status, P.step);
}

}  // namespace e3
}  // namespace petto_b200
