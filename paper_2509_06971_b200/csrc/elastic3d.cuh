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
//   * the cell modulus E_cell (the corner tree sum times the operator scale,
//     state_solver.hpp:336-343) is a per-cell field computed once per property
//     change (k_cell_modulus), so a cell costs one load instead of eight;
//   * a tile = 32 x-columns (lane l <-> x = i0 + l) by 8 rows j0-1 .. j0+6 (row
//     j0-1 is the y-halo row of cells whose top corners feed row j0); the CTA is
//     warp-specialised (16 warps, see k_elastic3d_fast): 8 cell warps, one per
//     row, stream the z axis (the outermost), ZP node planes per task, keeping
//     the previous plane's y/x-butterflies (12 doubles) and the top-face sums
//     (12 doubles) in registers; 7 node warps assemble and update the owned rows
//     one task behind; one producer warp;
//   * node planes arrive by TMA (cp.async.bulk.tensor, zero-filled outside the
//     grid) into an S-stage shared-memory ring guarded by mbarriers, issued S-1
//     tasks ahead by the producer;
//   * x-neighbour contributions travel by warp shuffle, a row's face sums to its
//     node warp through tensor memory, the row-(j+1) shares through a
//     double-buffered shared tile (one CTA barrier per task, i.e. per ZP planes),
//     and the previous x-tile's last column through a small shared "x-halo"
//     array -- a CTA walks the x-tiles of its (strip, z-chunk) item
//     sequentially, so no cell is computed twice in x;
//   * work item = (y-strip, z-chunk); item b -> CTA b with strips fastest, so the
//     CTAs sharing a strip boundary stream the same planes at the same time and
//     the halo rows are served from L2.
// Algorithmic HBM bytes per node-update: u_n 24 + u_{n-1} 24 + E_cell 8 +
// u_{n+1} 24 (+1 mask byte); PT drops u_{n-1}.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace petto_b200 {
namespace e3 {

// Build-time knobs (A/B variants: -DE3_W=7 -DE3_S=4 ...).
#ifndef E3_W
#define E3_W 7
#endif
#ifndef E3_S
#define E3_S 4
#endif
#ifndef E3_EXPERIMENT
#define E3_EXPERIMENT 0  // 1: no TMA traffic (compute only), 2: no cell math (traffic only)
#endif
constexpr int W = E3_W;        // owned node rows per tile
constexpr int NWARP = W + 1;   // cell rows per tile (+ y-halo row)
constexpr int NTHREADS = NWARP * 32;
constexpr int ZP = 2;          // node planes per task
constexpr int BOXX = 34;       // TMA box width of U (33 columns used; 16-byte multiple)
constexpr int UROWS = W + 2;   // rows j0-1 .. j0+W
constexpr int S = E3_S;        // pipeline depth (tasks)
constexpr int LMAX = 64;       // longest z chunk (x-halo buffer)

constexpr int r128(int b) { return (b + 127) / 128 * 128; }
constexpr int OFF_U = 0;                                      // [3][ZP][UROWS][BOXX] f64
constexpr int OFF_C = r128(3 * ZP * UROWS * BOXX * 8);        // [ZP][NWARP][32] f64 cell modulus
constexpr int OFF_P = OFF_C + r128(ZP * NWARP * 32 * 8);      // [3][ZP][W][32] f64
constexpr int OFF_M = OFF_P + r128(3 * ZP * W * 32 * 8);      // [ZP][W][32] u8
constexpr int STAGE_BYTES = OFF_M + r128(ZP * W * 32);
constexpr uint32_t BYTES_U = 3 * ZP * UROWS * BOXX * 8;
// Traffic-attribution probes (wrong results, ncu only): load U boxes without the
// y-halo rows (E3_PROBE_UROWS=7) and / or the x-halo columns (E3_PROBE_UBOXX=32).
#ifndef E3_PROBE_UROWS
#define E3_PROBE_UROWS (E3_W + 2)
#endif
#ifndef E3_PROBE_UBOXX
#define E3_PROBE_UBOXX 34
#endif
constexpr int LROWS = E3_PROBE_UROWS, LBOXX = E3_PROBE_UBOXX;
constexpr uint32_t BYTES_U_LOAD = 3 * ZP * LROWS * LBOXX * 8;
constexpr uint32_t BYTES_C = ZP * NWARP * 32 * 8;
constexpr uint32_t BYTES_P = 3 * ZP * W * 32 * 8;
constexpr uint32_t BYTES_M = ZP * W * 32;
constexpr int USTRIDE = ZP * UROWS * BOXX;  // component stride of the U tile
constexpr int PSTRIDE = ZP * W * 32;        // component stride of the P tile
constexpr int YS = ZP * 6 * 32;             // one warp's y shares of one task

constexpr int OFF_Y = S * STAGE_BYTES;                      // [2][NWARP][ZP][6][32] f64
constexpr int OFF_X = OFF_Y + 2 * NWARP * YS * 8;           // [2][LMAX][NWARP][3] f64
constexpr int OSTRIDE = 3 * W * 32;                         // one node plane of the output staging
constexpr int OFF_O = OFF_X + 2 * LMAX * NWARP * 3 * 8;     // [2][ZP][3][W][32] f64 output staging
constexpr int OFF_BAR = OFF_O + 2 * ZP * OSTRIDE * 8;       // [S] full
constexpr int OFF_RED = OFF_BAR + S * 8;                    // [2 NWARP] f64
constexpr int OFF_CUR = OFF_RED + 16 * 8;                   // producer cursor
constexpr int SMEM_BYTES = OFF_CUR + 128;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");

struct Params {
    Geo g;
    double kh[45];     // modal stiffness (stiffness.hpp pattern order)
    double inv_base;   // 1 / (hx hy hz)
    // update coefficients: APT u' = c1 u - c2 u_prev + c3 r; PT u' = u + dt r
    double c1, c2, c3, dt;
    double* next;      // output field (may alias the previous iterate)
    // peer halo: the neighbours' buffers of this step's output, offset so that this
    // slab's local node index addresses them (null: no neighbour / not in use)
    double* peer_lo;
    double* peer_hi;
    long long peer_lo_Ns, peer_hi_Ns;
    const double* aux; // pinned values / loads (3 x Ns)
    double* partials;  // per-CTA sum of r^2 over unconstrained entries (nullable)
    DeviceStatus* status;
    unsigned long long* cta_ns;  // probe builds (E3_CTA_TIMING): [grid][2] globaltimer at start / end
    long long step, nsteps;  // 1-based step index within the solve (of the launch's first step), total steps
    int nloc;          // steps of this launch (persistent launches, NM = 2; else 1)
    unsigned* gbar;    // grid barrier counter of a persistent launch (zeroed before it)
    int ntx;           // x tiles of 32 nodes
    int nstrips;       // y strips of W rows
    int chunk;         // owned planes per z chunk (<= LMAX)
    int nitems;        // nstrips * chunks
};
#define KH P.kh

// The tensor maps of one launch (kernel parameters, 64-byte aligned).
struct Maps {
    CUtensorMap u;     // state u_n: box [3][ZP][UROWS][BOXX]
    CUtensorMap c;     // cell modulus: box [ZP][NWARP][32]
    CUtensorMap p;     // previous iterate: box [3][ZP][W][32]
    CUtensorMap m;     // node mask: box [ZP][W][32]
    CUtensorMap o;     // output field: box [3][1][W][32] (TMA store, one node plane)
};

// The tensor maps of a persistent launch: step si uses m[si % NM] (u_n and u_{n-1}
// trade places every step; the output overwrites u_{n-1}).
template <int NM>
struct MapSet {
    Maps m[NM];
};

// Producer cursor over the CTA's task sequence: items (b, b+grid, ...), x tiles,
// tasks kk = 0 (prologue: node planes ka-1, ka) and kk >= 1 (owned planes
// kc = ka + ZP (kk-1) ..., loading node planes kc+1 .. kc+ZP).
struct Cursor {
    int item, t, kk, s, ka, ntask;
    bool valid;
    __device__ void set(const Params& P) {
        valid = item < P.nitems;
        if (!valid) return;
        s = item % P.nstrips;
        ka = P.g.kb + (item / P.nstrips) * P.chunk;
        ntask = 1 + (min(P.chunk, P.g.ke - ka) + ZP - 1) / ZP;
    }
    __device__ void next(const Params& P) {
        if (++kk == ntask) {
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
                                      int stage, const Maps& T) {
    unsigned char* st = smem + stage * STAGE_BYTES;
    const bool own = c.kk >= 1;
    const bool need_p = own && FORM <= 1;
    const uint32_t bytes = BYTES_U_LOAD + BYTES_C + (own ? BYTES_M : 0) + (need_p ? BYTES_P : 0);
    if (E3_EXPERIMENT == 1) {
        mbar_arrive(&bars[stage]);
        return;
    }
    mbar_expect_tx(&bars[stage], bytes);
    const int i0 = c.t * 32, j0 = c.s * W;
    // first cell plane of the task; the node planes loaded are kc+1, kc+2 for an
    // owned task and kc, kc+1 (= ka-1, ka) for the prologue
    const int kc = own ? c.ka + ZP * (c.kk - 1) : c.ka - 1;
    tma_load_4d(st + OFF_U, &T.u, &bars[stage], i0, j0 - 1 + (UROWS - LROWS) / 2, kc + (own ? 1 : 0) - P.g.ks0, 0);
    tma_load_3d(st + OFF_C, &T.c, &bars[stage], i0, j0 - 1, kc - P.g.ks0);
    if (own) {
        tma_load_3d(st + OFF_M, &T.m, &bars[stage], i0, j0, kc - P.g.ks0);
        if (need_p) tma_load_4d(st + OFF_P, &T.p, &bars[stage], i0, j0, kc - P.g.ks0, 0);
    }
}

// Everything a task needs that is fixed for one x-tile of one item.
struct Tile {
    bool upd;            // this thread owns a grid node of the tile (peer stores)
    double ninv;         // -1/V at an interior z plane (x2 at z = 0 or nz-1)
    double ca;           // coefficient of the face sum in the update: c3/dt/1 times ninv
    long long node0;     // lidx(i, j, 0) (loads, pinned values, peer stores)
    double* xw;          // x-halo out (lane 31) / in (lane 0; zeros at an item's first tile)
    const double* xr;
};

// forward x/y butterflies of stage plane z for cell (i, j): B[sx + 2 sy][c]
__device__ __forceinline__ void forward(const unsigned char* sb, int z, int w, int l, double (&B)[4][3]) {
    const double* su = reinterpret_cast<const double*>(sb + OFF_U) + (z * UROWS + w) * BOXX + l;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double* r0 = su + c * USTRIDE;
        const double a = r0[0], b = r0[1], cc = r0[BOXX], d = r0[BOXX + 1];
        const double A0 = a + b, A1 = a - b, A0n = cc + d, A1n = cc - d;
        B[0][c] = A0 + A0n;
        B[1][c] = A1 + A1n;
        B[2][c] = A0 - A0n;
        B[3][c] = A1 - A1n;
    }
}

// z butterflies, modal stiffness, inverse z butterflies of one cell with modulus
// ec: bottom face (node plane kc) assembled with the carried top, new top carried
// out; with EMIT the inverse y butterflies of the face: row j's sums in Yj, row
// j+1's shares to sYw.  The modulus multiplies the modal forces inside the face
// sums (fused multiply-adds) instead of the 21 modal inputs.
template <bool EMIT>
__device__ __forceinline__ void cell(const Params& P, const double (&Bc)[4][3], const double (&Bn)[4][3], double ec,
                                     double (&top)[4][3], double (&Yj)[2][3], double* sYw) {
    if (E3_EXPERIMENT == 2) {
        if (EMIT) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                Yj[0][c] = Bc[0][c] + Bn[1][c];
                Yj[1][c] = Bc[2][c] + Bn[3][c] + ec;
                sYw[c * 32] = Bc[1][c];
                sYw[(3 + c) * 32] = Bn[2][c];
            }
        }
        return;
    }
    // The modal stiffness is symmetric: a mirrored entry reads its partner's
    // operand (KH[1] for entry 9, ...), so one uniform-register load serves both.
    // modal coefficients C[s] (z butterflies), s = sx + 2 sy + 4 sz; the modal
    // stiffness decouples into blocks {1,2,4}, {3,5,6}, {7}, evaluated and consumed
    // one after the other to keep few values live.
    auto Cp = [&](int q, int c) { return Bc[q][c] + Bn[q][c]; };  // sz = 0
    auto Cm = [&](int q, int c) { return Bc[q][c] - Bn[q][c]; };  // sz = 1
    // block A: linear modes 1 (x), 2 (y), 4 (z)
    const double c10 = Cp(1, 0), c11 = Cp(1, 1), c12 = Cp(1, 2);
    const double c20 = Cp(2, 0), c21 = Cp(2, 1), c22 = Cp(2, 2);
    const double c40 = Cm(0, 0), c41 = Cm(0, 1), c42 = Cm(0, 2);
    const double F10 = KH[0] * c10 + KH[1] * c21 + KH[2] * c42;
    const double F11 = KH[3] * c11 + KH[4] * c20;
    const double F12 = KH[5] * c12 + KH[6] * c40;
    const double F20 = KH[4] * c11 + KH[8] * c20;
    const double F21 = KH[1] * c10 + KH[10] * c21 + KH[11] * c42;
    const double F22 = KH[12] * c22 + KH[13] * c41;
    const double F40 = KH[6] * c12 + KH[15] * c40;
    const double F41 = KH[13] * c22 + KH[17] * c41;
    const double F42 = KH[2] * c10 + KH[11] * c21 + KH[20] * c42;
    // pair (0, 4): mode 0 (rigid translation) carries no force; the carried top
    // of this pair is stored with the opposite sign
    double f0[3];
    {
        const double F4[3] = {F40, F41, F42};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            f0[c] = fma(ec, F4[c], -top[0][c]);
            top[0][c] = ec * F4[c];
        }
    }
    // block B: bilinear modes 3 (xy), 5 (xz), 6 (yz)
    const double c30 = Cp(3, 0), c31 = Cp(3, 1), c32 = Cp(3, 2);
    const double c50 = Cm(1, 0), c51 = Cm(1, 1), c52 = Cm(1, 2);
    const double c60 = Cm(2, 0), c61 = Cm(2, 1), c62 = Cm(2, 2);
    const double F30 = KH[21] * c30 + KH[22] * c62;
    const double F31 = KH[23] * c31 + KH[24] * c52;
    const double F32 = KH[25] * c32 + KH[26] * c51 + KH[27] * c60;
    const double F50 = KH[28] * c50 + KH[29] * c61;
    const double F51 = KH[26] * c32 + KH[31] * c51 + KH[32] * c60;
    const double F52 = KH[24] * c31 + KH[34] * c52;
    const double F60 = KH[27] * c32 + KH[32] * c51 + KH[37] * c60;
    const double F61 = KH[29] * c50 + KH[39] * c61;
    const double F62 = KH[22] * c30 + KH[41] * c62;
    // pairs (1, 5) and (2, 6)
    double f1[3], f2[3];
    {
        const double F1[3] = {F10, F11, F12}, F5[3] = {F50, F51, F52};
        const double F2[3] = {F20, F21, F22}, F6[3] = {F60, F61, F62};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            f1[c] = fma(ec, F1[c] + F5[c], top[1][c]);
            top[1][c] = ec * (F1[c] - F5[c]);
            f2[c] = fma(ec, F2[c] + F6[c], top[2][c]);
            top[2][c] = ec * (F2[c] - F6[c]);
        }
    }
    if (EMIT) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            Yj[0][c] = f0[c] + f2[c];
            sYw[c * 32] = f0[c] - f2[c];
        }
    }
    // block C: trilinear mode 7, pair (3, 7), then the sx = 1 face modes
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double F7 = KH[42 + c] * Cm(3, c);
        const double F3 = c == 0 ? F30 : (c == 1 ? F31 : F32);
        const double f3 = fma(ec, F3 + F7, top[3][c]);
        top[3][c] = ec * (F3 - F7);
        if (EMIT) {
            Yj[1][c] = f1[c] + f3;
            sYw[(3 + c) * 32] = f1[c] - f3;
        }
    }
}

// Node (i, j, kc): edge sums with warp w-1's shares, inverse x butterflies (x-halo
// for lane 0), then the residual, the update and the value into the output
// staging (so, one node plane) -- the producer stores it with TMA.  u_n arrives
// in u.  RSQ: accumulate r^2 (only the tolerance loop reads it).  ZEND: the task
// holds the plane z = 0 or nz-1 (twice the volume weight there).  exm: running
// minimum of (~hi & exponent mask) over the values written -- 0 iff one of them
// is not finite.
template <int FORM, bool RSQ, bool ZEND>
__device__ __forceinline__ void node(const Params& P, const Tile& T, int kc, int zi, const double (&Yj)[2][3],
                                     const double* below, const double (&u)[3], const double* sp,
                                     unsigned char mk, double* so, double& rsq, unsigned& exm) {
    const int l = threadIdx.x & 31;
    const Geo& g = P.g;
    double Xi[3], Xn[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double e0v = Yj[0][c] + below[c * 32];
        const double e1v = Yj[1][c] + below[(3 + c) * 32];
        Xi[c] = e0v + e1v;
        Xn[c] = e0v - e1v;
    }
    double acc[3];
    const double* xr = T.xr + zi * (NWARP * 3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double nb = __shfl_up_sync(0xffffffffu, Xn[c], 1);
        if (l == 0) nb = xr[c];
        acc[c] = Xi[c] + nb;
    }
    if (l == 31) {
        double* xw = T.xw + zi * (NWARP * 3);
#pragma unroll
        for (int c = 0; c < 3; ++c) xw[c] = Xn[c];
    }
    // nodes outside the grid (TMA zero-filled inputs, zero cell moduli) compute 0.0;
    // the TMA store clips them
    const bool endz = ZEND && (kc == 0 || kc == g.nz - 1);  // warp-uniform
    double nv[3];
    if (!mk) {
        double ca = T.ca, ninv = T.ninv;
        if (ZEND && endz) {
            ca += ca;
            ninv += ninv;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (FORM <= 1) nv[c] = fma(P.c1, u[c], fma(-P.c2, sp[c * PSTRIDE], ca * acc[c]));
            else if (FORM == 2) nv[c] = fma(ca, acc[c], u[c]);
            else nv[c] = acc[c] * ninv;
            if (RSQ) {
                const double r = acc[c] * ninv;
                rsq = fma(r, r, rsq);
            }
        }
    } else {  // rare: pinned components and/or a load on this node
        const double ninv = endz ? 2.0 * T.ninv : T.ninv;
        const long long node = T.node0 + (long long)(kc - g.ks0) * g.ny * g.px;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const bool pinned = (mk >> c) & 1;
            const double f = ((mk & 8) && !pinned) ? P.aux[c * g.Ns + node] : 0.0;
            const double r = acc[c] * ninv - f;
            if (pinned) {
                nv[c] = FORM == 3 ? 0.0 : P.aux[c * g.Ns + node];
            } else {
                if (RSQ) rsq = fma(r, r, rsq);
                if (FORM <= 1) nv[c] = fma(P.c1, u[c], fma(-P.c2, sp[c * PSTRIDE], P.c3 * r));
                else if (FORM == 2) nv[c] = fma(P.dt, r, u[c]);
                else nv[c] = r;
            }
        }
    }
    // non-finite iff the exponent field is all ones (integer pipe, no FP64 work)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        exm = min(exm, ~(unsigned)__double2hiint(nv[c]) & 0x7ff00000u);
        so[c * W * 32] = nv[c];
    }
    // a boundary plane is also the neighbour's ghost plane: store it there directly
    // (NVLink / same-device stores, overlapped with the rest of the step)
    if (kc == g.kb && P.peer_lo && T.upd) {
        const long long local = T.node0 + (long long)(kc - g.ks0) * g.ny * g.px;
#pragma unroll
        for (int c = 0; c < 3; ++c) P.peer_lo[c * P.peer_lo_Ns + local] = nv[c];
    }
    if (kc == g.ke - 1 && P.peer_hi && T.upd) {
        const long long local = T.node0 + (long long)(kc - g.ks0) * g.ny * g.px;
#pragma unroll
        for (int c = 0; c < 3; ++c) P.peer_hi[c * P.peer_hi_Ns + local] = nv[c];
    }
}

// ---------------------------------------------------------------------------
// The kernel is warp-specialised: 16 warps per CTA.  Warps 0-7 ("cell warps",
// rows j0-1 .. j0+6, 184 registers each via setmaxnreg) stream the forward
// butterflies and the cell stiffness of task q; warps 9-15 ("node warps", rows
// j0 .. j0+6, 72 registers) assemble and update the nodes of task q-1 at the
// same time; warp 8 is the producer (TMA loads).  A cell warp
// hands its row-j face sums to the node warp of the same row through tensor
// memory (same TMEM lane quarter: warp % 4) and its row-(j+1) shares through
// shared memory; one CTA barrier per task separates the phases.  The FP64-heavy
// cell work and the latency-bound node work of different tasks overlap on every
// scheduler.
constexpr int WS_THREADS = 2 * NTHREADS;
#ifndef E3_REG_CELL
#define E3_REG_CELL 184
#endif
constexpr uint32_t REG_CELL = E3_REG_CELL, REG_NODE = 256 - E3_REG_CELL;  // 8 (cell + node) = 2048 = 64K / 32
constexpr uint32_t TMEM_COLS = 128;                // [2 warp halves][2 parities][32 columns]
constexpr int OFF_TMEM = OFF_CUR + 64;             // TMEM base address (u32)
static_assert(NWARP == 8, "warp roles assume 8 cell warps");

// Calls f(own, s, t, ka, kc, two) for every task of the CTA in order: per x tile
// the prologue (own = false, cell plane ka-1), then the owned two-plane tasks.
template <class F>
__device__ __forceinline__ void walk(const Params& P, F&& f) {
    const Geo& g = P.g;
    for (int item = blockIdx.x; item < P.nitems; item += gridDim.x) {
        const int s = item % P.nstrips;
        const int ka = g.kb + (item / P.nstrips) * P.chunk;
        const int kb = min(ka + P.chunk, g.ke);
        for (int t = 0; t < P.ntx; ++t) {
            f(false, s, t, ka, ka - 1, false);
            for (int kc = ka; kc < kb; kc += ZP) f(true, s, t, ka, kc, kc + 1 < kb);
        }
    }
}

// Grid-wide barrier of a persistent launch (cooperative: every CTA is resident),
// called by one thread per CTA between __syncthreads.  The output of a step is
// written by TMA (the async proxy) and read by the next step's TMA loads: the
// bulk stores are complete (wait_group 0) before the proxy fence and the release.
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        if (v >= target) break;
        __nanosleep(64);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) __trap();  // 20 s: never hang the device
    }
    __threadfence();
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int FORM, bool RSQ>
__global__ void __launch_bounds__(WS_THREADS, 1)
    k_elastic3d_fast(const __grid_constant__ Params P, const __grid_constant__ Maps M) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const Geo& g = P.g;
    // Programmatic dependent launch: the next step may launch now; this one waits
    // until the previous step has completed and its stores are visible (a no-op
    // without the launch attribute).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (skip_step(P.status, P.step, P.nsteps)) return;
#ifdef E3_CTA_TIMING
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    double* sY = reinterpret_cast<double*>(smem + OFF_Y);
    double* sX = reinterpret_cast<double*>(smem + OFF_X);
    Cursor* pc = reinterpret_cast<Cursor*>(smem + OFF_CUR);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
    if (w == 0) tmem_alloc(tslot, TMEM_COLS);
    if (w == 8 && l == 0) {
        prefetch_tmap(&M.u);
        prefetch_tmap(&M.c);
        prefetch_tmap(&M.p);
        prefetch_tmap(&M.m);
        prefetch_tmap(&M.o);
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        pc->item = blockIdx.x;
        pc->t = 0;
        pc->kk = 0;
        pc->set(P);
        for (int s = 0; s < S - 1 && pc->valid; ++s) {
            issue<FORM>(P, *pc, smem, bars, s, M);
            pc->next(P);
        }
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tbase = *tslot;
    double rsq = 0.0;
    unsigned bad = 0;

    if (w < NWARP) {
        // ------------------------------------------------------------ cell warps
        regs_grow<REG_CELL>();
        double Bc[4][3], top[4][3];
        uint32_t st = 0, phase = 0, q = 0;
        const uint32_t tq = tbase + ((32u * (w & 3)) << 16) + (w >> 2) * 64;
        walk(P, [&](bool own, int, int, int, int, bool two) {
            mbar_wait(&bars[st], phase);
            const unsigned char* sb = smem + st * STAGE_BYTES;
            const double* sc = reinterpret_cast<const double*>(sb + OFF_C) + w * 32 + l;
            if (!own) {  // prologue: node planes ka-1, ka and cell plane ka-1
                double B0[4][3], Yd[2][3];
                forward(sb, 0, w, l, B0);
                forward(sb, 1, w, l, Bc);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                    for (int c = 0; c < 3; ++c) top[q4][c] = 0.0;
#ifndef E3_PROBE_NOPROLOGUE  // probe build (wrong results): no cell work in the prologue
                cell<false>(P, B0, Bc, sc[0], top, Yd, nullptr);
#endif
            } else {
                double* sYw = sY + (q & 1) * (NWARP * YS) + w * YS + l;
                double B1[4][3], Y0[2][3], Y1[2][3];
                forward(sb, 0, w, l, B1);
                cell<true>(P, Bc, B1, sc[0], top, Y0, sYw);
                if (two) {
                    forward(sb, 1, w, l, Bc);
                    cell<true>(P, B1, Bc, sc[NWARP * 32], top, Y1, sYw + 6 * 32);
                } else {
#pragma unroll
                    for (int k = 0; k < 6; ++k) Y1[k / 3][k % 3] = 0.0;
                }
                if (w > 0) {  // the y-halo row's own sums are not needed
                    const uint32_t ta = tq + (q & 1) * 32;
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        tmem_st1(ta + 2 * k, Y0[k / 3][k % 3]);
                        tmem_st1(ta + 12 + 2 * k, Y1[k / 3][k % 3]);
                    }
                    tmem_wait_st();
                }
            }
            tmem_fence_before();
#ifdef E3_SLOT_TIMING  // probe: warp 1 of CTA 0 records when it reaches / leaves each barrier
            unsigned long long t_arrive;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_arrive));
#endif
            __syncthreads();  // task q's shares and sums are complete
#ifdef E3_SLOT_TIMING
            if (blockIdx.x == 0 && w == 1 && l == 0 && P.cta_ns && q < 1000) {
                unsigned long long t_leave;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_leave));
                P.cta_ns[1024 + 3 * q] = t_arrive;
                P.cta_ns[1024 + 3 * q + 1] = t_leave;
                P.cta_ns[1024 + 3 * q + 2] = own ? 1 : 0;
            }
#endif
            ++q;
            if (++st == S) {
                st = 0;
                phase ^= 1u;
            }
        });
        __syncthreads();  // the node warps' last task
    } else if (w == NWARP) {
        // ------------------------------------------------------------- producer
        regs_shrink<REG_NODE>();
        uint32_t st = 0, q = 0;
        // the node output of the previous task (stored once the node warps are done with it)
        bool pown = false, ptwo = false;
        int pi0 = 0, pj0 = 0, pk = 0;
        auto store_prev = [&]() {
            if (l == 0 && pown) {
                const double* so = reinterpret_cast<const double*>(smem + OFF_O) + ((q - 1) & 1) * (ZP * OSTRIDE);
                tma_store_4d(&M.o, so, pi0, pj0, pk, 0);
                if (ptwo) tma_store_4d(&M.o, so + OSTRIDE, pi0, pj0, pk + 1, 0);
                bulk_commit();
            }
        };
        walk(P, [&](bool own, int s, int t, int, int kc, bool two) {
            if (l == 0) bulk_wait_read_all();  // staging (q-2) & 1 is free before the node warps refill it
            __syncthreads();  // cell warps done with task q, node warps with task q-1
            if (l == 0 && pc->valid) {  // refill the stage of task q-1
                issue<FORM>(P, *pc, smem, bars, st == 0 ? S - 1 : st - 1, M);
                pc->next(P);
            }
            store_prev();
            pown = own;
            ptwo = two;
            pi0 = t * 32;
            pj0 = s * W;
            pk = kc - g.ks0;
            ++q;
            if (++st == S) st = 0;
        });
        __syncthreads();
        store_prev();
        if (l == 0) bulk_wait_all();
    } else {
        // ------------------------------------------------------------ node warps
        regs_shrink<REG_NODE>();
        const int v = w - NWARP;  // row j0-1+v, v = 1..7
        double ucar[3] = {0.0, 0.0, 0.0};
        uint32_t st = 0, q = 0;
        const uint32_t tq = tbase + ((32u * (w & 3)) << 16) + (v >> 2) * 64;
        Tile T{};  // set at each x tile's prologue task
        int ntile = 0;
        unsigned exm = 0xffffffffu;
        walk(P, [&](bool own, int s, int t, int ka, int kc, bool two) {
            __syncthreads();  // the cell warps finished task q
            tmem_fence_after();
            const unsigned char* sb = smem + st * STAGE_BYTES;
            const double* su = reinterpret_cast<const double*>(sb + OFF_U) + v * BOXX + l;  // plane 0, row v
            if (!own) {
                const int i = t * 32 + l, j = s * W - 1 + v;
                T.upd = i < g.nx && j < g.ny;
                const int ends = (i == 0 || i == g.nx - 1) + (j == 0 || j == g.ny - 1);
                T.ninv = -P.inv_base * (double)(1 << ends);
                T.ca = (FORM <= 1 ? P.c3 : FORM == 2 ? P.dt : 1.0) * T.ninv;
                T.node0 = (long long)j * g.px + i;
                // x-halo buffers alternate per tile of the CTA; the first tile of an
                // item reads zeros (no cell to the left of x = 0)
                T.xw = sX + (ntile & 1) * (LMAX * NWARP * 3) + v * 3;
                T.xr = sX + ((ntile + 1) & 1) * (LMAX * NWARP * 3) + v * 3;
                if (t == 0) {
                    for (int k = l; k < LMAX * 3; k += 32) const_cast<double*>(T.xr)[(k / 3) * (NWARP * 3) + k % 3] = 0.0;
                    __syncwarp();
                }
                ++ntile;
            } else {
                double Yv[12];
                tmem_ld12(tq + (q & 1) * 32, Yv);
                const double Y0[2][3] = {{Yv[0], Yv[1], Yv[2]}, {Yv[3], Yv[4], Yv[5]}};
                const double Y1[2][3] = {{Yv[6], Yv[7], Yv[8]}, {Yv[9], Yv[10], Yv[11]}};
                const double* below = sY + (q & 1) * (NWARP * YS) + (v - 1) * YS + l;
                const unsigned char* mk = sb + OFF_M + (v - 1) * 32 + l;
                const double* sp = reinterpret_cast<const double*>(sb + OFF_P) + (v - 1) * 32 + l;
                double* so = reinterpret_cast<double*>(smem + OFF_O) + (q & 1) * (ZP * OSTRIDE) + (v - 1) * 32 + l;
                auto planes = [&](auto zend) {
                    constexpr bool ZE = decltype(zend)::value;
                    node<FORM, RSQ, ZE>(P, T, kc, kc - ka, Y0, below, ucar, sp, mk[0], so, rsq, exm);
                    if (two) {
                        double u1[3];
#pragma unroll
                        for (int c = 0; c < 3; ++c) u1[c] = su[c * USTRIDE];
                        node<FORM, RSQ, ZE>(P, T, kc + 1, kc + 1 - ka, Y1, below + 6 * 32, u1, sp + W * 32,
                                            mk[W * 32], so + OSTRIDE, rsq, exm);
                    }
                };
#ifndef E3_PROBE_NONODE  // probe build (wrong results): node warps skip the node work
                if (kc == 0 || kc + 1 >= g.nz - 1) planes(std::true_type{});
                else planes(std::false_type{});
#else
                (void)planes;
#endif
                fence_async_smem();  // the staging is read by the producer's TMA store
            }
            // u_n of the next task's first node plane (stage plane 1)
#pragma unroll
            for (int c = 0; c < 3; ++c) ucar[c] = su[c * USTRIDE + UROWS * BOXX];
            ++q;
            if (++st == S) st = 0;
        });
        if (P.peer_lo || P.peer_hi) __threadfence_system();  // peer stores before the step's signal
#ifndef E3_PROBE_NOMARK  // probe builds that compute garbage: keep every step running
        bad = exm == 0;
#endif
        __syncthreads();
    }

    // CTA reduction of r^2 (fixed order) and the non-finite flag
    double* red = reinterpret_cast<double*>(smem + OFF_RED);
    rsq = warp_sum(rsq);
    bad = __any_sync(0xffffffffu, bad);
    if (l == 0) red[w] = rsq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (int k = 0; k < 2 * NWARP; ++k) sum += red[k];
        if (P.partials) P.partials[blockIdx.x] = sum;
    }
    if (bad && l == 0) mark_bad(P.status, P.step);
    if (w == 0) tmem_dealloc(tbase, TMEM_COLS);
#ifdef E3_CTA_TIMING
    if (threadIdx.x == 0 && P.cta_ns) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        P.cta_ns[3 * blockIdx.x] = t_start;
        P.cta_ns[3 * blockIdx.x + 1] = t_end;
        P.cta_ns[3 * blockIdx.x + 2] = smid;
    }
#endif
}

// The persistent variant: P.nloc steps in one cooperative launch (single domain),
// separated by grid barriers -- the launch, the CTA setup and the tail of every
// step but the last disappear (small grids such as C4).  The same roles and task
// walk as k_elastic3d_fast, each role looping over the steps (its register budget
// set once); a separate kernel because folding the step loop into
// k_elastic3d_fast cost its single-step launches 5% more cycles at C5.
//   TOL = false: hybrid_solve's steps P.step .. (u_{n+1} overwrites u_{n-1}).
//   TOL = true: iterate_to_tolerance's iterations it = P.step .. (u_it in
//   MS.m[it % 3], u_{it+1} into a third buffer), each with its r^2 partials
//   (double-buffered by iteration parity); after the grid barrier every CTA sums
//   them in k_iter_finish's order and applies its stop test, so all stop at the
//   same iteration with the status k_iter_finish would have written.
template <int FORM, bool TOL>
__global__ void __launch_bounds__(WS_THREADS, 1)
    k_elastic3d_persist(const __grid_constant__ Params P, const __grid_constant__ MapSet<TOL ? 3 : 2> MS) {
    constexpr int NM = TOL ? 3 : 2;
    constexpr bool RSQ = TOL;  // r^2 partials (node() template argument)
    extern __shared__ __align__(128) unsigned char smem[];
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const Geo& g = P.g;
    if (TOL ? P.status->done != 0 : skip_step(P.status, P.step, P.nsteps)) return;
    // the stop test's constants (iterate_to_tolerance)
    const double target = P.status->target, nodes = P.status->nodes;
    const long long max_iters = P.status->max_iters;
    bool stop = false;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    double* sY = reinterpret_cast<double*>(smem + OFF_Y);
    double* sX = reinterpret_cast<double*>(smem + OFF_X);
    Cursor* pc = reinterpret_cast<Cursor*>(smem + OFF_CUR);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
    if (w == 0) tmem_alloc(tslot, TMEM_COLS);
    if (w == 8 && l == 0) {
        for (int m = 0; m < NM; ++m) {
            prefetch_tmap(&MS.m[m].u);
            prefetch_tmap(&MS.m[m].p);
            prefetch_tmap(&MS.m[m].o);
        }
        prefetch_tmap(&MS.m[0].c);
        prefetch_tmap(&MS.m[0].m);
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tbase = *tslot;
    double rsq = 0.0;
    // Per step: the roles walk the same tasks (one CTA barrier each, plus one after
    // the last); then the step's non-finite mark and, between steps, the grid
    // barrier.  Each role loops over the steps itself (its register budget is set
    // once, by setmaxnreg).
    const int nloc = P.nloc;
    auto skip = [&](int si) {  // uniform over the grid: marks in flight are for steps >= this one
        return TOL ? stop : si > 0 && skip_step(P.status, P.step + si, P.nsteps);
    };
    auto step_end = [&](int si, unsigned bad) {
        bad = __any_sync(0xffffffffu, bad);
        const long long it = P.step + si;
        if (bad && l == 0) mark_bad(P.status, TOL ? it + 1 : it);
        if (TOL) {
            // the CTA's r^2 partial, in k_elastic3d_fast's order
            double* red = reinterpret_cast<double*>(smem + OFF_RED);
            const double v = warp_sum(rsq);
            rsq = 0.0;
            if (l == 0) red[w] = v;
            __syncthreads();
            double* part = P.partials + (it & 1) * gridDim.x;
            if (threadIdx.x == 0) {
                double sum = 0.0;
                for (int k = 0; k < 2 * NWARP; ++k) sum += red[k];
                part[blockIdx.x] = sum;
            }
            __syncthreads();  // the partial and (producer) the completed stores
            if (w == NWARP && l == 0) grid_barrier(P.gbar, (unsigned)(si + 1) * gridDim.x);
            __syncthreads();
            // k_iter_finish: 256 threads stride over the partials, block_sum<8>
            if (w < 8) {
                double x = 0.0;
                for (int t = threadIdx.x; t < (int)gridDim.x; t += 256) x += __ldcg(part + t);
                x = warp_sum(x);
                if (l == 0) red[w] = x;
            }
            __syncthreads();
            if (w == 0) {
                double x = l < 8 ? red[l] : 0.0;
                x = warp_sum(x);
                if (l == 0) red[8] = x;
            }
            __syncthreads();
            const double r = sqrt(red[8]) / nodes;
            const bool first = it == 0;
            const bool aborted = !first && !isfinite(r);
            const bool converged = !aborted && r < target;
            stop = aborted || converged || it >= max_iters;
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                DeviceStatus* s = P.status;
                if (first) s->r_initial = r;
                else s->iterations = it;
                s->r_final = r;
                if (stop) s->done = 1;
                if (converged) s->converged = 1;
                if (aborted) s->aborted = 1;
                s->iter = it + 1;
            }
        } else if (si + 1 < nloc) {
            __syncthreads();  // the CTA's marks and (producer) completed stores
            if (w == NWARP && l == 0) grid_barrier(P.gbar, (unsigned)(si + 1) * gridDim.x);
            __syncthreads();
        }
    };
    // ring position and task parity: continue across the steps of a launch
    uint32_t st = 0, phase = 0, q = 0;

    if (w < NWARP) {
        // ------------------------------------------------------------ cell warps
        regs_grow<REG_CELL>();
        for (int si = 0; si < nloc && !skip(si); ++si) {
            double Bc[4][3], top[4][3];
            const uint32_t tq = tbase + ((32u * (w & 3)) << 16) + (w >> 2) * 64;
            walk(P, [&](bool own, int, int, int, int, bool two) {
                mbar_wait(&bars[st], phase);
                const unsigned char* sb = smem + st * STAGE_BYTES;
                const double* sc = reinterpret_cast<const double*>(sb + OFF_C) + w * 32 + l;
                if (!own) {  // prologue: node planes ka-1, ka and cell plane ka-1
                    double B0[4][3], Yd[2][3];
                    forward(sb, 0, w, l, B0);
                    forward(sb, 1, w, l, Bc);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                        for (int c = 0; c < 3; ++c) top[q4][c] = 0.0;
#ifndef E3_PROBE_NOPROLOGUE  // probe build (wrong results): no cell work in the prologue
                    cell<false>(P, B0, Bc, sc[0], top, Yd, nullptr);
#endif
                } else {
                    double* sYw = sY + (q & 1) * (NWARP * YS) + w * YS + l;
                    double B1[4][3], Y0[2][3], Y1[2][3];
                    forward(sb, 0, w, l, B1);
                    cell<true>(P, Bc, B1, sc[0], top, Y0, sYw);
                    if (two) {
                        forward(sb, 1, w, l, Bc);
                        cell<true>(P, B1, Bc, sc[NWARP * 32], top, Y1, sYw + 6 * 32);
                    } else {
#pragma unroll
                        for (int k = 0; k < 6; ++k) Y1[k / 3][k % 3] = 0.0;
                    }
                    if (w > 0) {  // the y-halo row's own sums are not needed
                        const uint32_t ta = tq + (q & 1) * 32;
#pragma unroll
                        for (int k = 0; k < 6; ++k) {
                            tmem_st1(ta + 2 * k, Y0[k / 3][k % 3]);
                            tmem_st1(ta + 12 + 2 * k, Y1[k / 3][k % 3]);
                        }
                        tmem_wait_st();
                    }
                }
                tmem_fence_before();
#ifdef E3_SLOT_TIMING  // probe: warp 1 of CTA 0 records when it reaches / leaves each barrier
                unsigned long long t_arrive;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_arrive));
#endif
                __syncthreads();  // task q's shares and sums are complete
#ifdef E3_SLOT_TIMING
                if (blockIdx.x == 0 && w == 1 && l == 0 && P.cta_ns && q < 1000) {
                    unsigned long long t_leave;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_leave));
                    P.cta_ns[1024 + 3 * q] = t_arrive;
                    P.cta_ns[1024 + 3 * q + 1] = t_leave;
                    P.cta_ns[1024 + 3 * q + 2] = own ? 1 : 0;
                }
#endif
                ++q;
                if (++st == S) {
                    st = 0;
                    phase ^= 1u;
                }
            });
            __syncthreads();  // the node warps' last task
            step_end(si, 0);
        }
    } else if (w == NWARP) {
        // ------------------------------------------------------------- producer
        regs_shrink<REG_NODE>();
        for (int si = 0; si < nloc && !skip(si); ++si) {
            const Maps& M = MS.m[TOL ? (P.step + si) % 3 : (si & 1)];
            if (l == 0) {  // the first S-1 tasks of the step, from the ring position on
                pc->item = blockIdx.x;
                pc->t = 0;
                pc->kk = 0;
                pc->set(P);
                for (int s = 0; s < S - 1 && pc->valid; ++s) {
                    issue<FORM>(P, *pc, smem, bars, (st + s) % S, M);
                    pc->next(P);
                }
            }
            // the node output of the previous task (stored once the node warps are done with it)
            bool pown = false, ptwo = false;
            int pi0 = 0, pj0 = 0, pk = 0;
            auto store_prev = [&]() {
                if (l == 0 && pown) {
                    const double* so = reinterpret_cast<const double*>(smem + OFF_O) + ((q - 1) & 1) * (ZP * OSTRIDE);
                    tma_store_4d(&M.o, so, pi0, pj0, pk, 0);
                    if (ptwo) tma_store_4d(&M.o, so + OSTRIDE, pi0, pj0, pk + 1, 0);
                    bulk_commit();
                }
            };
            walk(P, [&](bool own, int s, int t, int, int kc, bool two) {
                if (l == 0) bulk_wait_read_all();  // staging (q-2) & 1 is free before the node warps refill it
                __syncthreads();  // cell warps done with task q, node warps with task q-1
                if (l == 0 && pc->valid) {  // refill the stage of task q-1
                    issue<FORM>(P, *pc, smem, bars, st == 0 ? S - 1 : st - 1, M);
                    pc->next(P);
                }
                store_prev();
                pown = own;
                ptwo = two;
                pi0 = t * 32;
                pj0 = s * W;
                pk = kc - g.ks0;
                ++q;
                if (++st == S) st = 0;
            });
            __syncthreads();
            store_prev();
            if (l == 0) bulk_wait_all();
            step_end(si, 0);
        }
    } else {
        // ------------------------------------------------------------ node warps
        regs_shrink<REG_NODE>();
        const int v = w - NWARP;  // row j0-1+v, v = 1..7
        const uint32_t tq = tbase + ((32u * (w & 3)) << 16) + (v >> 2) * 64;
        int ntile = 0;  // x tiles so far (x-halo buffer parity)
        for (int si = 0; si < nloc && !skip(si); ++si) {
            double ucar[3] = {0.0, 0.0, 0.0};
            Tile T{};  // set at each x tile's prologue task
            unsigned exm = 0xffffffffu;
            walk(P, [&](bool own, int s, int t, int ka, int kc, bool two) {
                __syncthreads();  // the cell warps finished task q
                tmem_fence_after();
                const unsigned char* sb = smem + st * STAGE_BYTES;
                const double* su = reinterpret_cast<const double*>(sb + OFF_U) + v * BOXX + l;  // plane 0, row v
                if (!own) {
                    const int i = t * 32 + l, j = s * W - 1 + v;
                    T.upd = i < g.nx && j < g.ny;
                    const int ends = (i == 0 || i == g.nx - 1) + (j == 0 || j == g.ny - 1);
                    T.ninv = -P.inv_base * (double)(1 << ends);
                    T.ca = (FORM <= 1 ? P.c3 : FORM == 2 ? P.dt : 1.0) * T.ninv;
                    T.node0 = (long long)j * g.px + i;
                    // x-halo buffers alternate per tile of the CTA; the first tile of an
                    // item reads zeros (no cell to the left of x = 0)
                    T.xw = sX + (ntile & 1) * (LMAX * NWARP * 3) + v * 3;
                    T.xr = sX + ((ntile + 1) & 1) * (LMAX * NWARP * 3) + v * 3;
                    if (t == 0) {
                        for (int k = l; k < LMAX * 3; k += 32)
                            const_cast<double*>(T.xr)[(k / 3) * (NWARP * 3) + k % 3] = 0.0;
                        __syncwarp();
                    }
                    ++ntile;
                } else {
                    double Yv[12];
                    tmem_ld12(tq + (q & 1) * 32, Yv);
                    const double Y0[2][3] = {{Yv[0], Yv[1], Yv[2]}, {Yv[3], Yv[4], Yv[5]}};
                    const double Y1[2][3] = {{Yv[6], Yv[7], Yv[8]}, {Yv[9], Yv[10], Yv[11]}};
                    const double* below = sY + (q & 1) * (NWARP * YS) + (v - 1) * YS + l;
                    const unsigned char* mk = sb + OFF_M + (v - 1) * 32 + l;
                    const double* sp = reinterpret_cast<const double*>(sb + OFF_P) + (v - 1) * 32 + l;
                    double* so = reinterpret_cast<double*>(smem + OFF_O) + (q & 1) * (ZP * OSTRIDE) + (v - 1) * 32 + l;
                    auto planes = [&](auto zend) {
                        constexpr bool ZE = decltype(zend)::value;
                        node<FORM, RSQ, ZE>(P, T, kc, kc - ka, Y0, below, ucar, sp, mk[0], so, rsq, exm);
                        if (two) {
                            double u1[3];
#pragma unroll
                            for (int c = 0; c < 3; ++c) u1[c] = su[c * USTRIDE];
                            node<FORM, RSQ, ZE>(P, T, kc + 1, kc + 1 - ka, Y1, below + 6 * 32, u1, sp + W * 32,
                                                mk[W * 32], so + OSTRIDE, rsq, exm);
                        }
                    };
#ifndef E3_PROBE_NONODE  // probe build (wrong results): node warps skip the node work
                    if (kc == 0 || kc + 1 >= g.nz - 1) planes(std::true_type{});
                    else planes(std::false_type{});
#else
                    (void)planes;
#endif
                    fence_async_smem();  // the staging is read by the producer's TMA store
                }
                // u_n of the next task's first node plane (stage plane 1)
#pragma unroll
                for (int c = 0; c < 3; ++c) ucar[c] = su[c * USTRIDE + UROWS * BOXX];
                ++q;
                if (++st == S) st = 0;
            });
            if (P.peer_lo || P.peer_hi) __threadfence_system();  // peer stores before the step's signal
            __syncthreads();
            step_end(si, exm == 0);
        }
    }

    __syncthreads();
    if (w == 0) tmem_dealloc(tbase, TMEM_COLS);
}

// Cell modulus of every stored cell (i, j, k), k = ks0 + kl: the operator scale
// times the corner sum (the association of the fused kernel's former in-tile
// sum), 0 where the cell lies outside the grid or its top plane is not stored.
__global__ void k_cell_modulus(Geo g, const double* __restrict__ prop, double scale, double* __restrict__ ec) {
    const long long n = (long long)g.px * g.ny * g.nzs;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t % g.px);
        const int j = (int)((t / g.px) % g.ny);
        const int kl = (int)(t / ((long long)g.px * g.ny));
        const int k = g.ks0 + kl;
        double v = 0.0;
        if (i <= g.nx - 2 && j <= g.ny - 2 && k <= g.nz - 2 && kl + 1 < g.nzs) {
            const double* e0 = prop + t;
            const double* e1 = e0 + (long long)g.px * g.ny;
            const double a = (e0[0] + e0[1]) + (e0[g.px] + e0[g.px + 1]);
            const double b = (e1[0] + e1[1]) + (e1[g.px] + e1[g.px + 1]);
            v = (a + b) * scale;
        }
        ec[t] = v;
    }
}

}  // namespace e3
}  // namespace petto_b200
