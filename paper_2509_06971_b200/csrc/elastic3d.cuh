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
//   * CTA = 8 warps: lane l <-> x = i0 + l (32 nodes), warp w <-> row j0-1+w
//     (warp 0 is the y-halo row of cells whose top corners feed row j0);
//   * each CTA streams along z (the outermost axis): per cell plane it keeps the
//     previous plane's y/x-butterflies (12+1 doubles) and the top-face
//     contributions (12 doubles) in registers, alternating two register sets so
//     the stream needs no copies;
//   * node planes arrive by TMA (cp.async.bulk.tensor, zero-filled outside the
//     grid) into a 5-stage shared-memory ring guarded by mbarriers, issued 4
//     tasks ahead by one elected thread;
//   * x-neighbour contributions travel by warp shuffle, y-neighbour ones through
//     a double-buffered shared tile, and the previous x-tile's last column through
//     a small shared "x-halo" array -- a CTA walks the x-tiles of its
//     (strip, z-chunk) item sequentially, so no cell is computed twice in x;
//   * work item = (y-strip, z-chunk); item b -> CTA b with strips fastest, so the
//     CTAs sharing a strip boundary stream the same planes at the same time and
//     the halo rows are served from L2.
// Algorithmic HBM bytes per node-update: u_n 24 + u_{n-1} 24 + E 8 + u_{n+1} 24
// (+1 mask byte); PT drops u_{n-1}.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace petto_b200 {
namespace e3 {

// Build-time knobs (A/B variants: -DE3_W=11 -DE3_S=4 -DE3_TOP_SMEM=1 ...).
#ifndef E3_W
#define E3_W 7
#endif
#ifndef E3_S
#define E3_S 5
#endif
#ifndef E3_TOP_SMEM
#define E3_TOP_SMEM 0
#endif
#ifndef E3_DESYNC
#define E3_DESYNC 0
#endif
#ifndef E3_CONST_KH
#define E3_CONST_KH 0
#endif
constexpr int W = E3_W;        // owned node rows per tile
constexpr int NWARP = W + 1;   // + y-halo warp
constexpr int NTHREADS = NWARP * 32;
constexpr int BOXX = 34;       // TMA box width (33 columns used; 16-byte multiple)
constexpr int UROWS = W + 2;   // rows j0-1 .. j0+W
constexpr int S = E3_S;        // pipeline depth
constexpr int LMAX = 64;       // longest z chunk (x-halo buffer)
constexpr bool TOP_SMEM = E3_TOP_SMEM != 0;  // carried top-face sums in shared memory
// DESYNC: no CTA-wide barrier per task.  Warp w hands its row-(j+1) face shares to
// warp w+1 through a pairwise named barrier, and each warp releases a TMA stage
// through an "empty" mbarrier; warps drift apart by up to a task, so the FP64
// phase of one warp overlaps the load/exchange phase of another.
constexpr bool DESYNC = E3_DESYNC != 0;
constexpr int YD = DESYNC ? S : 2;  // depth of the y-exchange ring (>= the drift bound)

constexpr int r128(int b) { return (b + 127) / 128 * 128; }
constexpr int OFF_U = 0;                                    // [3][UROWS][BOXX] f64
constexpr int OFF_E = r128(3 * UROWS * BOXX * 8);           // [UROWS][BOXX] f64
constexpr int OFF_P = OFF_E + r128(UROWS * BOXX * 8);       // [3][W][32] f64
constexpr int OFF_M = OFF_P + r128(3 * W * 32 * 8);         // [W][32] u8
constexpr int STAGE_BYTES = OFF_M + r128(W * 32);
constexpr uint32_t BYTES_UE = 3 * UROWS * BOXX * 8 + UROWS * BOXX * 8;
constexpr uint32_t BYTES_P = 3 * W * 32 * 8;
constexpr uint32_t BYTES_M = W * 32;

constexpr int OFF_Y = S * STAGE_BYTES;                      // [YD][NWARP][6][32] f64
constexpr int OFF_X = OFF_Y + YD * NWARP * 6 * 32 * 8;      // [2][LMAX][NWARP][3] f64
constexpr int OFF_BAR = OFF_X + 2 * LMAX * NWARP * 3 * 8;   // [S] full, [S] empty, [W][S] y-ready
constexpr int OFF_RED = OFF_BAR + (2 * S + W * S) * 8;      // [NWARP] f64
constexpr int OFF_CUR = OFF_RED + 16 * 8;                   // producer cursor
constexpr int OFF_TOP = OFF_CUR + 128;                      // [12][NTHREADS] f64 (TOP_SMEM)
constexpr int SMEM_BYTES = OFF_TOP + (TOP_SMEM ? 12 * NTHREADS * 8 : 0);

// Carried top-face contributions of the previous cell plane: 12 doubles per
// thread, in registers or in the thread's own shared-memory column.
struct TopRegs {
    double v[4][3];
    __device__ __forceinline__ double& at(int q, int c) { return v[q][c]; }
};
struct TopSmem {
    double* p;  // this thread's column
    __device__ __forceinline__ double& at(int q, int c) { return p[(q * 3 + c) * NTHREADS]; }
};
using Top = typename std::conditional<TOP_SMEM, TopSmem, TopRegs>::type;
__device__ __forceinline__ void bind_top(TopRegs&, unsigned char*) {}
__device__ __forceinline__ void bind_top(TopSmem& t, unsigned char* smem) {
    t.p = reinterpret_cast<double*>(smem + OFF_TOP) + threadIdx.x;
}

// Modal stiffness operands: from the kernel parameters (default) or from a
// __constant__ bank refreshed on the launching stream before each launch.
__constant__ double c_kh[48];
#if E3_CONST_KH
#define KH c_kh
#else
#define KH P.kh
#endif

struct Params {
    Geo g;
    double kh[45];     // modal stiffness (stiffness.hpp pattern order)
    double e_scale;    // (sum of 8 corner E) -> E_cell: cm * 2(1+nu_op) / 8
    double inv_base;   // 1 / (hx hy hz)
    double dt, a, b, inv;
    double* next;      // output field (may alias the previous iterate)
    const double* aux; // pinned values / loads (3 x Ns)
    double* partials;  // per-CTA sum of r^2 over unconstrained entries (nullable)
    DeviceStatus* status;
    long long step, nsteps;  // 1-based step index within the solve, total steps
    int ntx;           // x tiles of 32 nodes
    int nstrips;       // y strips of W rows
    int chunk;         // owned planes per z chunk (<= LMAX)
    int nitems;        // nstrips * chunks
};

// Producer cursor over the CTA's task sequence: items (b, b+grid, ...), x tiles,
// tasks kc = ka-2 (prologue), ka-1 (first cell plane), ka .. kb-1 (owned planes).
struct Cursor {
    int item, t, kk, s, ka, len;
    bool valid;
    __device__ void set(const Params& P) {
        valid = item < P.nitems;
        if (!valid) return;
        s = item % P.nstrips;
        ka = P.g.kb + (item / P.nstrips) * P.chunk;
        len = min(P.chunk, P.g.ke - ka);
    }
    __device__ void next(const Params& P) {
        if (++kk == len + 2) {
            kk = 0;
            if (++t == P.ntx) {
                t = 0;
                item += gridDim.x;
                set(P);
            }
        }
    }
};

template <int FORM>
__device__ __forceinline__ void issue(const Params& P, const Cursor& c, unsigned char* smem, uint64_t* bars,
                                      int stage, const CUtensorMap* tU, const CUtensorMap* tE,
                                      const CUtensorMap* tP, const CUtensorMap* tM) {
    unsigned char* st = smem + stage * STAGE_BYTES;
    const bool own = c.kk >= 2;
    const bool need_p = own && FORM <= 1;
    const uint32_t bytes = BYTES_UE + (own ? BYTES_M : 0) + (need_p ? BYTES_P : 0);
    mbar_expect_tx(&bars[stage], bytes);
    const int i0 = c.t * 32, j0 = c.s * W, kc = c.ka - 2 + c.kk;
    const int zn = kc + 1 - P.g.ks0;
    tma_load_4d(st + OFF_U, tU, &bars[stage], i0, j0 - 1, zn, 0);
    tma_load_3d(st + OFF_E, tE, &bars[stage], i0, j0 - 1, zn);
    if (own) {
        tma_load_3d(st + OFF_M, tM, &bars[stage], i0, j0, kc - P.g.ks0);
        if (need_p) tma_load_4d(st + OFF_P, tP, &bars[stage], i0, j0, kc - P.g.ks0, 0);
    }
}

// Everything a task needs that is fixed for one x-tile of one item.
struct Tile {
    int i, j, t;
    bool upd;            // this thread owns a grid node of the tile
    double escale;       // e_scale, or 0 where the cell (i, j) is outside the grid
    double invv_xy;      // 1/V without the z-end factor
    long long node0;     // lidx(i, j, 0)
    double* xw;          // x-halo out (lane 31) / in (lane 0)
    const double* xr;
};

struct Pipe {
    unsigned char* smem;
    uint64_t* bars;
    int st, q;
    uint32_t phase;
};

// forward x/y butterflies of node plane kc+1 for cell (i, j): B[sx + 2 sy][c], E sum
__device__ __forceinline__ void forward(const unsigned char* sb, int w, int l, double (&B)[4][3], double& E) {
    const double* su = reinterpret_cast<const double*>(sb + OFF_U) + w * BOXX + l;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double* r0 = su + c * UROWS * BOXX;
        const double a = r0[0], b = r0[1], cc = r0[BOXX], d = r0[BOXX + 1];
        const double A0 = a + b, A1 = a - b, A0n = cc + d, A1n = cc - d;
        B[0][c] = A0 + A0n;
        B[1][c] = A1 + A1n;
        B[2][c] = A0 - A0n;
        B[3][c] = A1 - A1n;
    }
    const double* e0 = reinterpret_cast<const double*>(sb + OFF_E) + w * BOXX + l;
    E = (e0[0] + e0[1]) + (e0[BOXX] + e0[BOXX + 1]);
}

// z butterflies, modal stiffness, inverse z butterflies: bottom face (node plane
// kc) returned in face (added to the carried top), new top carried out.
template <bool EMIT>
__device__ __forceinline__ void cell(const Params& P, const double (&Bc)[4][3], double Ec, const double (&Bn)[4][3],
                                     double En, double escale, Top& top, double (&Yj)[2][3], double* sYw) {
    const double ec = (Ec + En) * escale;
    // modal coefficients C[s] = E_cell * (z butterfly), s = sx + 2 sy + 4 sz; the
    // modal stiffness decouples into blocks {1,2,4}, {3,5,6}, {7}, evaluated and
    // consumed one after the other to keep few values live.
    auto Cp = [&](int q, int c) { return (Bc[q][c] + Bn[q][c]) * ec; };  // sz = 0
    auto Cm = [&](int q, int c) { return (Bc[q][c] - Bn[q][c]) * ec; };  // sz = 1
    // block A: linear modes 1 (x), 2 (y), 4 (z)
    const double c10 = Cp(1, 0), c11 = Cp(1, 1), c12 = Cp(1, 2);
    const double c20 = Cp(2, 0), c21 = Cp(2, 1), c22 = Cp(2, 2);
    const double c40 = Cm(0, 0), c41 = Cm(0, 1), c42 = Cm(0, 2);
    const double F10 = KH[0] * c10 + KH[1] * c21 + KH[2] * c42;
    const double F11 = KH[3] * c11 + KH[4] * c20;
    const double F12 = KH[5] * c12 + KH[6] * c40;
    const double F20 = KH[7] * c11 + KH[8] * c20;
    const double F21 = KH[9] * c10 + KH[10] * c21 + KH[11] * c42;
    const double F22 = KH[12] * c22 + KH[13] * c41;
    const double F40 = KH[14] * c12 + KH[15] * c40;
    const double F41 = KH[16] * c22 + KH[17] * c41;
    const double F42 = KH[18] * c10 + KH[19] * c21 + KH[20] * c42;
    // pair (0, 4): mode 0 (rigid translation) carries no force
    double f0[3];
    f0[0] = top.at(0, 0) + F40;
    f0[1] = top.at(0, 1) + F41;
    f0[2] = top.at(0, 2) + F42;
    top.at(0, 0) = -F40;
    top.at(0, 1) = -F41;
    top.at(0, 2) = -F42;
    // block B: bilinear modes 3 (xy), 5 (xz), 6 (yz)
    const double c30 = Cp(3, 0), c31 = Cp(3, 1), c32 = Cp(3, 2);
    const double c50 = Cm(1, 0), c51 = Cm(1, 1), c52 = Cm(1, 2);
    const double c60 = Cm(2, 0), c61 = Cm(2, 1), c62 = Cm(2, 2);
    const double F30 = KH[21] * c30 + KH[22] * c62;
    const double F31 = KH[23] * c31 + KH[24] * c52;
    const double F32 = KH[25] * c32 + KH[26] * c51 + KH[27] * c60;
    const double F50 = KH[28] * c50 + KH[29] * c61;
    const double F51 = KH[30] * c32 + KH[31] * c51 + KH[32] * c60;
    const double F52 = KH[33] * c31 + KH[34] * c52;
    const double F60 = KH[35] * c32 + KH[36] * c51 + KH[37] * c60;
    const double F61 = KH[38] * c50 + KH[39] * c61;
    const double F62 = KH[40] * c30 + KH[41] * c62;
    // pairs (1, 5) and (2, 6)
    double f1[3];
    f1[0] = top.at(1, 0) + (F10 + F50);
    f1[1] = top.at(1, 1) + (F11 + F51);
    f1[2] = top.at(1, 2) + (F12 + F52);
    top.at(1, 0) = F10 - F50;
    top.at(1, 1) = F11 - F51;
    top.at(1, 2) = F12 - F52;
    const double f20 = top.at(2, 0) + (F20 + F60);
    const double f21 = top.at(2, 1) + (F21 + F61);
    const double f22 = top.at(2, 2) + (F22 + F62);
    top.at(2, 0) = F20 - F60;
    top.at(2, 1) = F21 - F61;
    top.at(2, 2) = F22 - F62;
    // inverse y butterflies of the sx = 0 face modes: row j keeps the sum, row j+1
    // (warp w+1) gets the difference through shared memory
    if (EMIT) {
        Yj[0][0] = f0[0] + f20;
        Yj[0][1] = f0[1] + f21;
        Yj[0][2] = f0[2] + f22;
        sYw[0 * 32] = f0[0] - f20;
        sYw[1 * 32] = f0[1] - f21;
        sYw[2 * 32] = f0[2] - f22;
    }
    // block C: trilinear mode 7, pair (3, 7), then the sx = 1 face modes
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double F7 = KH[42 + c] * Cm(3, c);
        const double F3 = c == 0 ? F30 : (c == 1 ? F31 : F32);
        const double f3 = top.at(3, c) + (F3 + F7);
        top.at(3, c) = F3 - F7;
        if (EMIT) {
            Yj[1][c] = f1[c] + f3;
            sYw[(3 + c) * 32] = f1[c] - f3;
        }
    }
}

// Mid-task hand-off (after the y shares are written).  Synchronous mode: one CTA
// barrier, then the producer refills the stage of the previous task.
template <int FORM>
__device__ __forceinline__ void end_task(const Params& P, Pipe& pp, Cursor* pc, const CUtensorMap* tU,
                                         const CUtensorMap* tE, const CUtensorMap* tP, const CUtensorMap* tM) {
    if (DESYNC) return;
    __syncthreads();
    if (threadIdx.x == 0 && pc->valid) {
        issue<FORM>(P, *pc, pp.smem, pp.bars, pp.st == 0 ? S - 1 : pp.st - 1, tU, tE, tP, tM);
        pc->next(P);
    }
}

// End of a task (after the warp's last read of the stage).  Desync mode: the warp
// releases the stage; thread 0 refills the stage of the previous task once every
// warp has released it.
template <int FORM>
__device__ __forceinline__ void release(const Params& P, Pipe& pp, Cursor* pc, const CUtensorMap* tU,
                                        const CUtensorMap* tE, const CUtensorMap* tP, const CUtensorMap* tM) {
    if (!DESYNC) return;
    __syncwarp();
    uint64_t* empty = pp.bars + S;
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[pp.st]);
    if (threadIdx.x == 0 && pc->valid) {
        const int prev = pp.st == 0 ? S - 1 : pp.st - 1;
        if (pp.q >= 1) mbar_wait(&empty[prev], pp.st == 0 ? pp.phase ^ 1u : pp.phase);
        issue<FORM>(P, *pc, pp.smem, pp.bars, prev, tU, tE, tP, tM);
        pc->next(P);
    }
}

// The y-ready barriers complete one phase per task, so tasks without a y exchange
// (prologue, first cell plane) still hand off to keep the phases aligned with the
// task counter.
__device__ __forceinline__ void y_handoff(Pipe& pp) {
    if (!DESYNC) return;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t* yready = pp.bars + 2 * S;
    if (w < W) {
        __syncwarp();
        if (l == 0) mbar_arrive(&yready[w * S + pp.st]);
    }
    if (w > 0) mbar_wait(&yready[(w - 1) * S + pp.st], pp.phase);
}

__device__ __forceinline__ void advance(Pipe& pp) {
    ++pp.q;
    if (++pp.st == S) {
        pp.st = 0;
        pp.phase ^= 1u;
    }
}

// One owned node plane kc: forward of plane kc+1 into Bn, cell plane kc, face
// assembly, node update of (i, j, kc).
template <int FORM>
__device__ __forceinline__ void own_task(const Params& P, Pipe& pp, Cursor* pc, const Tile& T, int kc, int zi,
                                         const double (&Bc)[4][3], double Ec, double (&Bn)[4][3], double& En,
                                         Top& top, double (&ucar)[3], double& rsq, unsigned& bad,
                                         double* sY, const CUtensorMap* tU, const CUtensorMap* tE,
                                         const CUtensorMap* tP, const CUtensorMap* tM) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const Geo& g = P.g;
    mbar_wait(&pp.bars[pp.st], pp.phase);
    const unsigned char* sb = pp.smem + pp.st * STAGE_BYTES;
    forward(sb, w, l, Bn, En);
    // cell plane kc with the inverse y butterflies: row j's sums in Yj, row j+1's
    // shares to warp w+1 through shared memory
    double* sYw = sY + (DESYNC ? pp.st : (pp.q & 1)) * (NWARP * 6 * 32);
    double Yj[2][3];
    cell<true>(P, Bc, Ec, Bn, En, kc <= g.nz - 2 ? T.escale : 0.0, top, Yj, sYw + w * 6 * 32 + l);
    uint64_t* yready = pp.bars + 2 * S;  // [W][S]: warp w's shares of task q ready
    if (DESYNC && w < W) {
        __syncwarp();
        if (l == 0) mbar_arrive(&yready[w * S + pp.st]);
    }
    end_task<FORM>(P, pp, pc, tU, tE, tP, tM);
    // edge sums (w >= 1), inverse x butterflies, node assembly
    double Xi[3], Xn[3];
    if (w > 0) {  // warp-uniform
        if (DESYNC) mbar_wait(&yready[(w - 1) * S + pp.st], pp.phase);
        const double* below = sYw + (w - 1) * 6 * 32 + l;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double e0v = Yj[0][c] + below[c * 32];
            const double e1v = Yj[1][c] + below[(3 + c) * 32];
            Xi[c] = e0v + e1v;
            Xn[c] = e0v - e1v;
        }
    } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            Xi[c] = Yj[0][c] + Yj[1][c];
            Xn[c] = Yj[0][c] - Yj[1][c];
        }
    }
    double acc[3];
    const double* xr = T.xr + zi * (NWARP * 3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double nb = __shfl_up_sync(0xffffffffu, Xn[c], 1);
        acc[c] = Xi[c] + (l > 0 ? nb : (T.t > 0 ? xr[c] : 0.0));
    }
    if (l == 31) {
        double* xw = T.xw + zi * (NWARP * 3);
#pragma unroll
        for (int c = 0; c < 3; ++c) xw[c] = Xn[c];
    }
    if (T.upd) {
        const unsigned char mk = (sb + OFF_M)[(w - 1) * 32 + l];
        const double* sp = reinterpret_cast<const double*>(sb + OFF_P) + (w - 1) * 32 + l;
        const double invv = (kc == 0 || kc == g.nz - 1) ? 2.0 * T.invv_xy : T.invv_xy;
        const long long node = T.node0 + (long long)(kc - g.ks0) * g.ny * g.px;
        auto update = [&](int c, double r) {
            if (FORM == 0) {
                const double cu = ucar[c], pv = sp[c * W * 32];
                return 2.0 * cu - pv + P.a * r - P.b * (cu - pv);
            } else if (FORM == 1) {
                const double cu = ucar[c], pv = sp[c * W * 32];
                return (2.0 * cu - pv + P.b * cu + P.a * r) * P.inv;
            } else if (FORM == 2) {
                return ucar[c] + P.dt * r;
            }
            return r;
        };
        double nv[3];
        if (!mk) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double r = -acc[c] * invv;
                nv[c] = update(c, r);
                rsq += r * r;
            }
        } else {  // rare: pinned components and/or a load on this node
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const bool pinned = (mk >> c) & 1;
                const double f = ((mk & 8) && !pinned) ? P.aux[c * g.Ns + node] : 0.0;
                const double r = -acc[c] * invv - f;
                if (pinned) {
                    nv[c] = FORM == 3 ? 0.0 : P.aux[c * g.Ns + node];
                } else {
                    rsq += r * r;
                    nv[c] = update(c, r);
                }
            }
        }
        // non-finite iff the exponent field is all ones (integer pipe, no FP64 work)
        unsigned ex = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            ex |= ((__double2hiint(nv[c]) & 0x7ff00000) == 0x7ff00000);
            P.next[c * g.Ns + node] = nv[c];
        }
        bad |= ex;
    }
    // own node of plane kc+1 feeds the next task's update (this stage is only
    // recycled after the next task's barrier)
    const double* su = reinterpret_cast<const double*>(sb + OFF_U) + w * BOXX + l;
#pragma unroll
    for (int c = 0; c < 3; ++c) ucar[c] = su[c * UROWS * BOXX];
    release<FORM>(P, pp, pc, tU, tE, tP, tM);
    advance(pp);
}

template <int FORM>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_elastic3d_fast(const __grid_constant__ Params P, const __grid_constant__ CUtensorMap tU,
                     const __grid_constant__ CUtensorMap tE, const __grid_constant__ CUtensorMap tP,
                     const __grid_constant__ CUtensorMap tM) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const Geo& g = P.g;
    if (skip_step(P.status, P.step, P.nsteps)) return;
    Pipe pp{smem, reinterpret_cast<uint64_t*>(smem + OFF_BAR), 0, 0, 0u};
    double* sY = reinterpret_cast<double*>(smem + OFF_Y);
    double* sX = reinterpret_cast<double*>(smem + OFF_X);
    Cursor* pc = reinterpret_cast<Cursor*>(smem + OFF_CUR);
    if (threadIdx.x == 0) {
        prefetch_tmap(&tU);
        prefetch_tmap(&tE);
        prefetch_tmap(&tP);
        prefetch_tmap(&tM);
        for (int s = 0; s < S; ++s) {
            mbar_init(&pp.bars[s], 1);          // full: the producer's expect_tx + TMA bytes
            mbar_init(&pp.bars[S + s], NWARP);  // empty: one arrival per warp
        }
        for (int b = 0; b < W * S; ++b) mbar_init(&pp.bars[2 * S + b], 1);  // y-ready: producer lane 0
        fence_mbar_init();
        pc->item = blockIdx.x;
        pc->t = 0;
        pc->kk = 0;
        pc->set(P);
        for (int s = 0; s < S - 1 && pc->valid; ++s) {
            issue<FORM>(P, *pc, smem, pp.bars, s, &tU, &tE, &tP, &tM);
            pc->next(P);
        }
    }
    __syncthreads();

    double BA[4][3], BB[4][3], EA = 0.0, EB = 0.0, ucar[3] = {0.0, 0.0, 0.0};
    Top top;
    bind_top(top, smem);
    double rsq = 0.0;
    unsigned bad = 0;
    for (int item = blockIdx.x; item < P.nitems; item += gridDim.x) {
        const int s = item % P.nstrips;
        const int ka = g.kb + (item / P.nstrips) * P.chunk;
        const int kb = min(ka + P.chunk, g.ke);
        for (int t = 0; t < P.ntx; ++t) {
            Tile T;
            T.t = t;
            T.i = t * 32 + l;
            T.j = s * W - 1 + w;
            T.upd = w >= 1 && T.i < g.nx && T.j < g.ny;
            const bool cxy = T.i <= g.nx - 2 && T.j >= 0 && T.j <= g.ny - 2;
            T.escale = cxy ? P.e_scale : 0.0;
            const int ends = (T.i == 0 || T.i == g.nx - 1) + (T.j == 0 || T.j == g.ny - 1);
            T.invv_xy = P.inv_base * (double)(1 << ends);
            T.node0 = (long long)max(T.j, 0) * g.px + T.i;
            T.xw = sX + (t & 1) * (LMAX * NWARP * 3) + w * 3;
            T.xr = sX + ((t + 1) & 1) * (LMAX * NWARP * 3) + w * 3;

            // prologue: butterflies of node plane ka-1
            mbar_wait(&pp.bars[pp.st], pp.phase);
            forward(pp.smem + pp.st * STAGE_BYTES, w, l, BA, EA);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                for (int c = 0; c < 3; ++c) top.at(q4, c) = 0.0;
            end_task<FORM>(P, pp, pc, &tU, &tE, &tP, &tM);
            y_handoff(pp);
            release<FORM>(P, pp, pc, &tU, &tE, &tP, &tM);
            advance(pp);
            // first cell plane ka-1: its top face feeds node plane ka
            {
                mbar_wait(&pp.bars[pp.st], pp.phase);
                const unsigned char* sb = pp.smem + pp.st * STAGE_BYTES;
                forward(sb, w, l, BB, EB);
                double Yj[2][3];
                cell<false>(P, BA, EA, BB, EB, ka - 1 >= 0 ? T.escale : 0.0, top, Yj, nullptr);
                end_task<FORM>(P, pp, pc, &tU, &tE, &tP, &tM);
                const double* su = reinterpret_cast<const double*>(sb + OFF_U) + w * BOXX + l;
#pragma unroll
                for (int c = 0; c < 3; ++c) ucar[c] = su[c * UROWS * BOXX];
                y_handoff(pp);
                release<FORM>(P, pp, pc, &tU, &tE, &tP, &tM);
                advance(pp);
            }
            // owned planes, two per iteration with alternating register roles
            int kc = ka;
            for (; kc + 1 < kb; kc += 2) {
                own_task<FORM>(P, pp, pc, T, kc, kc - ka, BB, EB, BA, EA, top, ucar, rsq, bad, sY, &tU, &tE, &tP,
                               &tM);
                own_task<FORM>(P, pp, pc, T, kc + 1, kc + 1 - ka, BA, EA, BB, EB, top, ucar, rsq, bad, sY, &tU,
                               &tE, &tP, &tM);
            }
            if (kc < kb)
                own_task<FORM>(P, pp, pc, T, kc, kc - ka, BB, EB, BA, EA, top, ucar, rsq, bad, sY, &tU, &tE, &tP,
                               &tM);
        }
    }

    // CTA reduction of r^2 (fixed order) and the non-finite flag
    double* red = reinterpret_cast<double*>(smem + OFF_RED);
    rsq = warp_sum(rsq);
    bad = __any_sync(0xffffffffu, bad);
    __syncthreads();
    if (l == 0) red[w] = rsq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (int k = 0; k < NWARP; ++k) sum += red[k];
        if (P.partials) P.partials[blockIdx.x] = sum;
    }
    if (bad && l == 0) mark_bad(P.status, P.step);
}

}  // namespace e3
}  // namespace petto_b200
