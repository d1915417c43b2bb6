/*
 * petto_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference
 * algorithms on the hot path (the parity checker; the product never links it).
 *
 * Every function restates one reference function in the reference's own
 * floating-point operation order, so that with -ffp-contract=off it rounds
 * exactly like the reference's non-FMA x86-64 build (bitwise equality is checked
 * against oracle/_ref and the golden fixtures in tests/golden/).  Serial only:
 * reductions follow the reference's threads == 1 order (parallel.hpp:19-29,
 * phase_field.hpp:89-95).  Citations are to /root/reference/proj/.
 */
#include "petto_oracle.h"

#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <time.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define PI 3.141592653589793238462643383279502884

static char g_err[512];
static int g_threads = 1;

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }
const char* orc_impl_name(void) { return "port"; }
void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int orc_threads(void) { return g_threads; }

/* ------------------------------------------------------------------ grid.hpp */

typedef struct {
    int dim;
    int64_t n[3];
    double length[3];
    double h[3];
} grid_t;

/* Grid::make2d/make3d + finalize (grid.hpp:27-43, 76-89). */
static int grid_init(grid_t* g, const orc_grid* o) {
    g->dim = o->dim;
    if (g->dim != 2 && g->dim != 3) return fail(2, "grid: dim must be 2 or 3");
    for (int a = 0; a < 3; ++a) {
        g->n[a] = o->n[a];
        g->length[a] = o->length[a];
        g->h[a] = 1.0;
    }
    if (g->dim == 2) {
        g->n[2] = 1;
        g->length[2] = 0.0;
    }
    for (int a = 0; a < g->dim; ++a) {
        if (g->n[a] < 3) return fail(2, "grid: need at least 3 nodes per axis");
        if (!(g->length[a] > 0.0)) return fail(2, "grid: axis length must be positive");
        g->h[a] = g->length[a] / (double)(g->n[a] - 1);
    }
    return 0;
}

static int64_t nnodes(const grid_t* g) { return g->n[0] * g->n[1] * g->n[2]; }

/* grid.hpp:64-73 */
static double cell_extent(const grid_t* g, int axis, int64_t i) {
    if (g->n[axis] == 1) return 1.0;
    return (i == 0 || i == g->n[axis] - 1) ? 0.5 * g->h[axis] : g->h[axis];
}

static double cell_volume(const grid_t* g, int64_t i, int64_t j, int64_t k) {
    double v = cell_extent(g, 0, i) * cell_extent(g, 1, j);
    if (g->dim == 3) v *= cell_extent(g, 2, k);
    return v;
}

static double domain_volume(const grid_t* g) {
    double v = 1.0;
    for (int a = 0; a < g->dim; ++a) v *= g->length[a];
    return v;
}

int64_t orc_num_nodes(const orc_grid* o) {
    grid_t g;
    return grid_init(&g, o) ? -1 : nnodes(&g);
}

double orc_spacing(const orc_grid* o, int axis) {
    grid_t g;
    return grid_init(&g, o) ? NAN : g.h[axis];
}

double orc_cell_volume(const orc_grid* o, int64_t i, int64_t j, int64_t k) {
    grid_t g;
    return grid_init(&g, o) ? NAN : cell_volume(&g, i, j, k);
}

/* make_constraints (grid.hpp:185-232): faces in order, later assignments win
 * (unordered_map operator[]), pins last, entries sorted ascending. */
typedef struct {
    int64_t n;
    int64_t* entry;
    double* value;
} cset_t;

static void cset_free(cset_t* c) {
    free(c->entry);
    free(c->value);
    c->entry = NULL;
    c->value = NULL;
    c->n = 0;
}

static int make_constraints(const grid_t* g, const orc_bc* bc, int comps, cset_t* out) {
    const int64_t nn = nnodes(g);
    const int64_t total = nn * comps;
    unsigned char* has = (unsigned char*)calloc((size_t)total, 1);
    double* val = (double*)malloc(sizeof(double) * (size_t)total);
    out->n = 0;
    out->entry = NULL;
    out->value = NULL;
    const int nfaces = g->dim * 2;
    for (int f = 0; f < nfaces; ++f) {
        const int kind = bc->kind[f];
        if (kind != 0 /*Dirichlet*/ && kind != 3 /*Roller*/) continue;
        const int a = f / 2;
        const int64_t fixed = (f % 2) ? g->n[a] - 1 : 0;
        const int b = (a + 1) % 3, c = (a + 2) % 3;
        int64_t idx[3];
        idx[a] = fixed;
        for (int64_t p = 0; p < g->n[b]; ++p) {
            idx[b] = p;
            for (int64_t q = 0; q < g->n[c]; ++q) {
                idx[c] = q;
                const int64_t node = (idx[2] * g->n[1] + idx[1]) * g->n[0] + idx[0];
                if (kind == 0) {
                    for (int comp = 0; comp < comps; ++comp) {
                        has[comp * nn + node] = 1;
                        val[comp * nn + node] = bc->value[f];
                    }
                } else if (bc->component[f] < comps) {
                    has[bc->component[f] * nn + node] = 1;
                    val[bc->component[f] * nn + node] = bc->value[f];
                }
            }
        }
    }
    for (int64_t p = 0; p < bc->npins; ++p) {
        if (bc->pin_node[p] < 0 || bc->pin_node[p] >= nn) {
            free(has);
            free(val);
            return fail(2, "boundary: pin references a node outside the grid");
        }
        if (bc->pin_comp[p] < 0 || bc->pin_comp[p] >= comps) {
            free(has);
            free(val);
            return fail(2, "boundary: pin references an invalid component");
        }
        const int64_t e = (int64_t)bc->pin_comp[p] * nn + bc->pin_node[p];
        has[e] = 1;
        val[e] = bc->pin_value[p];
    }
    int64_t cnt = 0;
    for (int64_t e = 0; e < total; ++e) cnt += has[e];
    out->entry = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cnt ? cnt : 1));
    out->value = (double*)malloc(sizeof(double) * (size_t)(cnt ? cnt : 1));
    for (int64_t e = 0; e < total; ++e)
        if (has[e]) {
            out->entry[out->n] = e;
            out->value[out->n] = val[e];
            ++out->n;
        }
    free(has);
    free(val);
    return 0;
}

int64_t orc_make_constraints(const orc_grid* o, const orc_bc* bc, int comps, int64_t* entry,
                             double* value, int64_t cap) {
    grid_t g;
    int rc = grid_init(&g, o);
    if (rc) return -1 - rc;
    cset_t cs;
    rc = make_constraints(&g, bc, comps, &cs);
    if (rc) return -1 - rc;
    for (int64_t i = 0; i < cs.n && i < cap; ++i) {
        entry[i] = cs.entry[i];
        value[i] = cs.value[i];
    }
    const int64_t n = cs.n;
    cset_free(&cs);
    return n;
}

/* grid.hpp:234-243 */
static void apply_constraints(double* f, const cset_t* cs) {
    for (int64_t i = 0; i < cs->n; ++i) f[cs->entry[i]] = cs->value[i];
}

static void zero_constrained(double* f, const cset_t* cs) {
    for (int64_t i = 0; i < cs->n; ++i) f[cs->entry[i]] = 0.0;
}

/* ----------------------------------------------------- state_solver.hpp (a9) */

/* detail::unit_cell_stiffness (state_solver.hpp:149-237). */
static void unit_cell_stiffness(int dim, const double h[3], double nu, double* canon) {
    const int nodes = 1 << dim;
    const int dofs = nodes * dim;
    const int voigt = dim * (dim + 1) / 2;
    const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double mu = 1.0 / (2.0 * (1.0 + nu));
    double ke[24 * 24];
    double dmat[6 * 6];
    double bmat[6 * 24];
    memset(ke, 0, sizeof ke);
    memset(dmat, 0, sizeof dmat);
    for (int a = 0; a < dim; ++a)
        for (int b = 0; b < dim; ++b) dmat[a * voigt + b] = lam + (a == b ? 2.0 * mu : 0.0);
    for (int s = dim; s < voigt; ++s) dmat[s * voigt + s] = mu;

    double cvol = 1.0;
    for (int a = 0; a < dim; ++a) cvol *= h[a];
    const double weight = cvol / nodes;
    const double gauss[2] = {0.5 - 0.5 / sqrt(3.0), 0.5 + 0.5 / sqrt(3.0)};

    for (int gp = 0; gp < nodes; ++gp) {
        const double xi[3] = {gauss[gp & 1], gauss[(gp >> 1) & 1], gauss[(gp >> 2) & 1]};
        double ds[8][3]; /* dshape(l, a) */
        for (int l = 0; l < nodes; ++l)
            for (int a = 0; a < dim; ++a) {
                double v = 1.0;
                for (int b = 0; b < dim; ++b) {
                    const int bit = (l >> b) & 1;
                    if (b == a)
                        v *= (bit ? 1.0 : -1.0) / h[b];
                    else
                        v *= bit ? xi[b] : 1.0 - xi[b];
                }
                ds[l][a] = v;
            }
        for (int i = 0; i < voigt * dofs; ++i) bmat[i] = 0.0;
        for (int l = 0; l < nodes; ++l)
            for (int c = 0; c < dim; ++c) {
                const int dof = l * dim + c;
                bmat[c * dofs + dof] = ds[l][c];
                int row = dim;
                for (int a = 0; a < dim; ++a)
                    for (int b = a + 1; b < dim; ++b, ++row) {
                        if (c == a) bmat[row * dofs + dof] += ds[l][b];
                        if (c == b) bmat[row * dofs + dof] += ds[l][a];
                    }
            }
        for (int p = 0; p < dofs; ++p)
            for (int q = 0; q < dofs; ++q) {
                double acc = 0.0;
                for (int r = 0; r < voigt; ++r) {
                    double db = 0.0;
                    for (int s = 0; s < voigt; ++s) db += dmat[r * voigt + s] * bmat[s * dofs + q];
                    acc += bmat[r * dofs + p] * db;
                }
                ke[p * dofs + q] += weight * acc;
            }
    }
    /* canonicalisation over transposition and the axis-mirror group (:214-235) */
    for (int p = 0; p < dofs; ++p)
        for (int q = 0; q < dofs; ++q) {
            int best_p = p, best_q = q;
            double best_sign = 1.0;
            for (int flips = 0; flips < nodes; ++flips)
                for (int tr = 0; tr < 2; ++tr) {
                    int pp = ((p / dim) ^ flips) * dim + p % dim;
                    int qq = ((q / dim) ^ flips) * dim + q % dim;
                    double sign = 1.0;
                    if ((flips >> (p % dim)) & 1) sign = -sign;
                    if ((flips >> (q % dim)) & 1) sign = -sign;
                    if (tr) {
                        const int t = pp;
                        pp = qq;
                        qq = t;
                    }
                    if (pp < best_p || (pp == best_p && qq < best_q)) {
                        best_p = pp;
                        best_q = qq;
                        best_sign = sign;
                    }
                }
            canon[p * dofs + q] = best_sign * ke[best_p * dofs + best_q];
        }
}

void orc_unit_cell_stiffness(int dim, const double h[3], double nu, double* ke) {
    unit_cell_stiffness(dim, h, nu, ke);
}

/* elasticity_spectral_bound (state_solver.hpp:254-279) */
double orc_elasticity_spectral_bound(const orc_grid* o, double nu, double e_max) {
    grid_t g;
    if (grid_init(&g, o)) return NAN;
    const int dim = g.dim;
    const int dofs = (1 << dim) * dim;
    double ke[24 * 24], v[24], w[24];
    unit_cell_stiffness(dim, g.h, nu, ke);
    for (int p = 0; p < dofs; ++p) v[p] = 1.0;
    double lmax = 0.0;
    for (int it = 0; it < 200; ++it) {
        double norm = 0.0;
        for (int p = 0; p < dofs; ++p) {
            double acc = 0.0;
            for (int q = 0; q < dofs; ++q) acc += ke[p * dofs + q] * v[q];
            w[p] = acc;
            norm += acc * acc;
        }
        norm = sqrt(norm);
        if (norm == 0.0) break;
        lmax = norm;
        for (int p = 0; p < dofs; ++p) v[p] = w[p] / norm;
    }
    double cvol = 1.0;
    for (int a = 0; a < dim; ++a) cvol *= g.h[a];
    return lmax * e_max * (1 << dim) / cvol;
}

/* ch_stable_dt (phase_field.hpp:26-31) */
double orc_ch_stable_dt(const orc_grid* o, double mobility, double gamma) {
    grid_t g;
    if (grid_init(&g, o)) return NAN;
    double s = 0.0;
    for (int a = 0; a < g.dim; ++a) s += 4.0 / (g.h[a] * g.h[a]);
    const double wpp_max = PI * PI / 32.0;
    return 2.0 / (mobility * (gamma * s * s + wpp_max * s));
}

/* ---------------------------------------------------------- operators (a7, a12) */

typedef struct {
    int physics; /* 0 heat, 1 elasticity */
    grid_t g;
    int comps;
    cset_t cs;
    const double* property; /* kappa (heat) */
    double* mu;             /* elasticity: Lame mu = cm * E (make_lame) */
    const double* source;
    double nu_op; /* nu derived from node 0 (state_solver.hpp:299-301) */
    double ke[24 * 24];
    double* inv_volume;
} op_t;

static void op_free(op_t* op) {
    cset_free(&op->cs);
    free(op->mu);
    free(op->inv_volume);
    op->mu = NULL;
    op->inv_volume = NULL;
}

/* HeatOperator ctor (state_solver.hpp:79-81) / make_lame + ElasticityOperator ctor
 * (state_solver.hpp:113-127, 292-310). */
static int op_init(op_t* op, int physics, const orc_grid* o, const orc_bc* bc,
                   const double* property, double nu, const double* source) {
    memset(op, 0, sizeof *op);
    int rc = grid_init(&op->g, o);
    if (rc) return rc;
    op->physics = physics;
    op->comps = physics ? op->g.dim : 1;
    op->property = property;
    op->source = source;
    rc = make_constraints(&op->g, bc, op->comps, &op->cs);
    if (rc) return rc;
    if (!physics) return 0;
    const int64_t nn = nnodes(&op->g);
    const double cl = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double cm = 1.0 / (2.0 * (1.0 + nu));
    op->mu = (double*)malloc(sizeof(double) * (size_t)nn);
    int bad = 0;
    for (int64_t i = 0; i < nn; ++i) {
        const double l = cl * property[i];
        op->mu[i] = cm * property[i];
        if (!(l > 0.0) || !(op->mu[i] > 0.0)) bad = 1;
    }
    if (bad) {
        op_free(op);
        return fail(2, "elasticity: Lame fields must be positive");
    }
    const double l0 = cl * property[0];
    const double m0 = op->mu[0];
    op->nu_op = l0 / (2.0 * (l0 + m0));
    unit_cell_stiffness(op->g.dim, op->g.h, op->nu_op, op->ke);
    op->inv_volume = (double*)malloc(sizeof(double) * (size_t)nn);
    for (int64_t k = 0; k < op->g.n[2]; ++k)
        for (int64_t j = 0; j < op->g.n[1]; ++j)
            for (int64_t i = 0; i < op->g.n[0]; ++i)
                op->inv_volume[(k * op->g.n[1] + j) * op->g.n[0] + i] =
                    1.0 / cell_volume(&op->g, i, j, k);
    return 0;
}

/* detail::flux_along (stencil.hpp:97-107) */
static double flux_along(const double* f, const double* kp, int64_t t, int64_t nn,
                         int64_t stride, double half_inv_h2) {
    if (nn == 1) return 0.0;
    if (t == 0) return (kp[0] + kp[stride]) * (f[stride] - f[0]) * (2.0 * half_inv_h2);
    if (t == nn - 1) return (kp[0] + kp[-stride]) * (f[-stride] - f[0]) * (2.0 * half_inv_h2);
    return ((kp[0] + kp[stride]) * (f[stride] - f[0]) - (kp[-stride] + kp[0]) * (f[0] - f[-stride])) *
           half_inv_h2;
}

/* variable_diffusion_into with fused source (stencil.hpp:123-158). */
static int variable_diffusion(const grid_t* g, const double* fd, const double* kd, double* od,
                              const double* source) {
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    double hih2[3];
    for (int a = 0; a < 3; ++a) hih2[a] = 0.5 / (g->h[a] * g->h[a]);
    int bad = 0;
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j) {
            const int64_t row = (k * ny + j) * nx;
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t node = row + i;
                if (!(kd[node] > 0.0)) bad = 1;
                double acc = flux_along(fd + node, kd + node, i, nx, 1, hih2[0]);
                acc += flux_along(fd + node, kd + node, j, ny, nx, hih2[1]);
                if (nz > 1) acc += flux_along(fd + node, kd + node, k, nz, nx * ny, hih2[2]);
                od[node] = source ? acc + source[node] : acc;
            }
        }
    if (bad) return fail(2, "variable_diffusion: kappa must be positive everywhere");
    return 0;
}

/* detail::mirror_tree_sum (state_solver.hpp:242-247) */
static double tree_sum(double* v, int count) {
    for (int width = count; width > 1; width /= 2)
        for (int i = 0; i < width / 2; ++i) v[i] = v[2 * i] + v[2 * i + 1];
    return v[0];
}

/* ElasticityOperator::residual (state_solver.hpp:327-385) */
static void elasticity_residual(const op_t* op, const double* u, double* out) {
    const grid_t* g = &op->g;
    const int d = g->dim;
    const int cn = 1 << d;
    const int dofs = cn * d;
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    const int64_t nn = nnodes(g);
    const double* mu = op->mu;
    const double e_from_mu = 2.0 * (1.0 + op->nu_op) / cn;
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j) {
            const int64_t row = (k * ny + j) * nx;
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t node = row + i;
                double lanes[3][8];
                for (int c = 0; c < d; ++c)
                    for (int m = 0; m < cn; ++m) lanes[c][m] = 0.0;
                for (int m = 0; m < cn; ++m) {
                    const int64_t ci = i - (m & 1);
                    const int64_t cj = j - ((m >> 1) & 1);
                    const int64_t ck = d == 3 ? k - ((m >> 2) & 1) : 0;
                    if (ci < 0 || ci > nx - 2 || cj < 0 || cj > ny - 2) continue;
                    if (d == 3 && (ck < 0 || ck > nz - 2)) continue;
                    const int64_t base = (ck * ny + cj) * nx + ci;
                    int64_t corners[8];
                    double ev[8];
                    for (int m2 = 0; m2 < cn; ++m2) {
                        corners[m2] = base + (m2 & 1) + nx * ((m2 >> 1) & 1) +
                                      (d == 3 ? nx * ny * ((m2 >> 2) & 1) : 0);
                        ev[m2] = mu[corners[m2]];
                    }
                    const double e_cell = tree_sum(ev, cn) * e_from_mu;
                    const int l = m;
                    for (int c = 0; c < d; ++c) {
                        const double* kr = op->ke + (l * d + c) * dofs;
                        double tv[8];
                        for (int m2 = 0; m2 < cn; ++m2) {
                            double t = 0.0;
                            for (int b = 0; b < d; ++b) t += kr[m2 * d + b] * u[b * nn + corners[m2]];
                            tv[m2] = t;
                        }
                        lanes[c][m] = e_cell * tree_sum(tv, cn);
                    }
                }
                const double invv = op->inv_volume[node];
                for (int c = 0; c < d; ++c)
                    out[c * nn + node] = -tree_sum(lanes[c], cn) * invv - op->source[c * nn + node];
            }
        }
    zero_constrained(out, &op->cs);
}

static int op_residual(const op_t* op, const double* state, double* out) {
    if (op->physics) {
        elasticity_residual(op, state, out);
        return 0;
    }
    const int rc = variable_diffusion(&op->g, state, op->property, out, op->source);
    if (rc) return rc;
    zero_constrained(out, &op->cs); /* HeatOperator::residual (state_solver.hpp:83-86) */
    return 0;
}

int orc_heat_residual(const orc_grid* o, const orc_bc* bc, const double* kappa,
                      const double* source, const double* T, double* out) {
    op_t op;
    int rc = op_init(&op, 0, o, bc, kappa, 0.0, source);
    if (!rc) rc = op_residual(&op, T, out);
    op_free(&op);
    return rc;
}

int orc_elasticity_residual(const orc_grid* o, const orc_bc* bc, const double* modulus,
                            double nu, const double* loads, const double* u, double* out) {
    op_t op;
    int rc = op_init(&op, 1, o, bc, modulus, nu, loads);
    if (!rc) rc = op_residual(&op, u, out);
    op_free(&op);
    return rc;
}

/* residual_norm (state_solver.hpp:49-58), serial sum_nodes (parallel.hpp:22-24) */
double orc_residual_norm(const double* r, int64_t nodes, int comps) {
    double sq = 0.0;
    const int64_t n = nodes * comps;
    for (int64_t i = 0; i < n; ++i) sq += r[i] * r[i];
    return sqrt(sq) / (double)nodes;
}

/* ------------------------------------------------- pseudo-time steps (a13-a17) */

typedef struct {
    double* cur;
    double* prev;
} hist_t;

static void swap_hist(hist_t* h) {
    double* t = h->cur;
    h->cur = h->prev;
    h->prev = t;
}

/* pt_step_inplace (state_solver.hpp:400-412) */
static void pt_step(hist_t* h, const double* r, double dt, const cset_t* cs, int64_t n) {
    const double* c = h->cur;
    double* next = h->prev;
    for (int64_t i = 0; i < n; ++i) next[i] = c[i] + dt * r[i];
    swap_hist(h);
    apply_constraints(h->cur, cs);
}

/* apt_step_inplace (state_solver.hpp:414-442) */
static void apt_step(hist_t* h, const double* r, double dt, double theta, int form,
                     const cset_t* cs, int64_t n) {
    const double* c = h->cur;
    const double* p = h->prev;
    double* next = h->prev;
    const double a = dt * dt / theta;
    const double b = dt / theta;
    if (form == 0) {
        for (int64_t i = 0; i < n; ++i) {
            const double first = c[i] - p[i];
            next[i] = 2.0 * c[i] - p[i] + a * r[i] - b * first;
        }
    } else {
        const double inv = 1.0 / (1.0 + b);
        for (int64_t i = 0; i < n; ++i) next[i] = (2.0 * c[i] - p[i] + b * c[i] + a * r[i]) * inv;
    }
    swap_hist(h);
    apply_constraints(h->cur, cs);
}

/* PTParams::validate (state_solver.hpp:25-33) */
static int validate_params(const orc_pt_params* p) {
    if (!(p->dt_pt > 0.0) && p->n_pt > 0) return fail(2, "pt params: dt_pt must be positive");
    if (!(p->dt_apt > 0.0) && p->n_apt > 0) return fail(2, "pt params: dt_apt must be positive");
    if (!(p->theta > 0.0)) return fail(2, "pt params: theta must be positive");
    if (p->n_apt < 0 || p->n_pt < 0 || p->n_apt + p->n_pt < 1)
        return fail(2, "pt params: need at least one step per loop");
    return 0;
}

/* detail::check_finite (state_solver.hpp:463-473) */
static int check_finite(const double* f, int64_t n, long long step, int64_t* abort_step) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double v = f[i];
        s += v < 0 ? -v : v;
    }
    if (!isfinite(s)) {
        if (abort_step) *abort_step = step;
        snprintf(g_err, sizeof g_err,
                 "numerical abort in 'state' at step %lld: non-finite values (time step too "
                 "large?)",
                 step);
        return 1;
    }
    return 0;
}

/* hybrid_solve (state_solver.hpp:480-498); the history buffers are the caller's
 * two arrays, swapped in place like StateHistory's Fields. */
static int hybrid_solve(hist_t* h, const op_t* op, const orc_pt_params* p, double* r,
                        int64_t* abort_step) {
    int rc = validate_params(p);
    if (rc) return rc;
    const int64_t n = nnodes(&op->g) * op->comps;
    long long step = 0;
    for (long s = 0; s < p->n_apt; ++s) {
        if ((rc = op_residual(op, h->cur, r))) return rc;
        apt_step(h, r, p->dt_apt, p->theta, p->form, &op->cs, n);
        if (++step % 100 == 0 && check_finite(h->cur, n, step, abort_step)) return 1;
    }
    for (long s = 0; s < p->n_pt; ++s) {
        if ((rc = op_residual(op, h->cur, r))) return rc;
        pt_step(h, r, p->dt_pt, &op->cs, n);
        if (++step % 100 == 0 && check_finite(h->cur, n, step, abort_step)) return 1;
    }
    return check_finite(h->cur, n, step, abort_step);
}

/* Copy the history back so that (cur, prev) hold StateHistory's (current, previous). */
static void hist_writeback(const hist_t* h, double* cur, double* prev, double* spare_a,
                           double* spare_b, int64_t n) {
    (void)spare_a;
    (void)spare_b;
    if (h->cur != cur) {
        /* buffers swapped an odd number of times: exchange contents */
        for (int64_t i = 0; i < n; ++i) {
            const double t = cur[i];
            cur[i] = prev[i];
            prev[i] = t;
        }
    }
}

int orc_hybrid_solve(int physics, const orc_grid* o, const orc_bc* bc, const double* property,
                     double nu, const double* source, double* cur, double* prev,
                     const orc_pt_params* p, int64_t* abort_step) {
    op_t op;
    int rc = op_init(&op, physics, o, bc, property, nu, source);
    if (rc) return rc;
    const int64_t n = nnodes(&op.g) * op.comps;
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    hist_t h = {cur, prev};
    rc = hybrid_solve(&h, &op, p, r, abort_step);
    hist_writeback(&h, cur, prev, NULL, NULL, n);
    free(r);
    op_free(&op);
    return rc;
}

int orc_time_hybrid(int physics, const orc_grid* o, const orc_bc* bc, const double* property, double nu,
                    const double* source, double* cur, double* prev, const orc_pt_params* p,
                    double* seconds) {
    op_t op;
    int rc = op_init(&op, physics, o, bc, property, nu, source);
    if (rc) return rc;
    const int64_t n = nnodes(&op.g) * op.comps;
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    hist_t h = {cur, prev};
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    rc = hybrid_solve(&h, &op, p, r, NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    hist_writeback(&h, cur, prev, NULL, NULL, n);
    free(r);
    op_free(&op);
    return rc;
}

/* iterate_to_tolerance (state_solver.hpp:511-541) */
int orc_iterate_to_tolerance(int physics, const orc_grid* o, const orc_bc* bc,
                             const double* property, double nu, const double* source,
                             double* cur, double* prev, int mode, const orc_pt_params* p,
                             double target, long max_iters, orc_solve_stats* st) {
    op_t op;
    int rc = op_init(&op, physics, o, bc, property, nu, source);
    if (rc) return rc;
    const int64_t nn = nnodes(&op.g);
    const int64_t n = nn * op.comps;
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    hist_t h = {cur, prev};
    st->iterations = 0;
    st->converged = 0;
    rc = op_residual(&op, h.cur, r);
    if (!rc) {
        st->r_initial = orc_residual_norm(r, nn, op.comps);
        st->r_final = st->r_initial;
        if (st->r_final < target) {
            st->converged = 1;
        } else {
            for (long it = 0; it < max_iters; ++it) {
                if (mode == 0)
                    pt_step(&h, r, p->dt_pt, &op.cs, n);
                else
                    apt_step(&h, r, p->dt_apt, p->theta, p->form, &op.cs, n);
                if ((rc = op_residual(&op, h.cur, r))) break;
                st->iterations = it + 1;
                st->r_final = orc_residual_norm(r, nn, op.comps);
                if (!isfinite(st->r_final)) {
                    snprintf(g_err, sizeof g_err,
                             "numerical abort in 'state' at step %ld: residual norm diverged",
                             it + 1);
                    rc = 1;
                    break;
                }
                if (st->r_final < target) {
                    st->converged = 1;
                    break;
                }
            }
        }
    }
    hist_writeback(&h, cur, prev, NULL, NULL, n);
    free(r);
    op_free(&op);
    return rc;
}

/* ------------------------------------------------ design subsystems (a19-a26) */

/* MaterialModel::validate (objectives.hpp:26-33) */
static int validate_material(const orc_material* m, int phase_count) {
    if (m->nphases != phase_count)
        return fail(2, "material: one property value per phase required");
    for (int i = 0; i < m->nphases; ++i)
        if (!(m->properties[i] > 0.0)) return fail(2, "material: properties must be positive");
    if (m->penalty < 1.0) return fail(2, "material: penalty must be >= 1");
    if (!(m->void_floor > 0.0)) return fail(2, "material: void floor must be positive");
    return 0;
}

/* detail::pow_penalty (objectives.hpp:80-89) */
static double pow_penalty(double x, double e) {
    const int ei = (int)e;
    if (e == (double)ei && ei >= 0 && ei <= 8) {
        double r = 1.0;
        for (int i = 0; i < ei; ++i) r *= x;
        return r;
    }
    return pow(x, e);
}

/* interpolate_into (objectives.hpp:95-116) */
static void interpolate(const grid_t* g, const orc_material* m, const double* phases, double* o) {
    const int64_t n = nnodes(g);
    const double floor_v = m->void_floor;
    const double e = m->penalty;
    for (int64_t node = 0; node < n; ++node) {
        double acc = 0.0;
        for (int i = 0; i < m->nphases; ++i)
            acc += m->properties[i] * pow_penalty(phases[i * n + node], e);
        o[node] = acc > floor_v ? acc : floor_v;
    }
}

int orc_interpolate(const orc_grid* o, const orc_material* m, const double* phases,
                    double* out) {
    grid_t g;
    int rc = grid_init(&g, o);
    if (!rc) rc = validate_material(m, m->nphases);
    if (rc) return rc;
    interpolate(&g, m, phases, out);
    return 0;
}

/* detail::d1_along + derivative_into (stencil.hpp:23-52) */
static void derivative(const grid_t* g, const double* f, int axis, double* out) {
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    const int64_t stride = axis == 0 ? 1 : (axis == 1 ? nx : nx * ny);
    const int64_t nn = g->n[axis];
    const double hih = 0.5 / g->h[axis];
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t node = (k * ny + j) * nx + i;
                const int64_t t = axis == 0 ? i : (axis == 1 ? j : k);
                const double* q = f + node;
                double v;
                if (nn == 1)
                    v = 0.0;
                else if (t == 0)
                    v = (-3.0 * q[0] + 4.0 * q[stride] - q[2 * stride]) * hih;
                else if (t == nn - 1)
                    v = (3.0 * q[0] - 4.0 * q[-stride] + q[-2 * stride]) * hih;
                else
                    v = (q[stride] - q[-stride]) * hih;
                out[node] = v;
            }
}

/* strain_invariants (objectives.hpp:151-180) */
static void strain_invariants(const grid_t* g, const double* u, double* tr, double* ec) {
    const int d = g->dim;
    const int64_t nn = nnodes(g);
    double* du = (double*)malloc(sizeof(double) * (size_t)(d * d * nn));
    for (int c = 0; c < d; ++c)
        for (int a = 0; a < d; ++a) derivative(g, u + c * nn, a, du + (c * d + a) * nn);
    for (int64_t node = 0; node < nn; ++node) {
        double t = 0.0, c2 = 0.0;
        for (int a = 0; a < d; ++a) {
            const double eaa = du[(a * d + a) * nn + node];
            t += eaa;
            c2 += eaa * eaa;
        }
        for (int a = 0; a < d; ++a)
            for (int b = a + 1; b < d; ++b) {
                const double eab = 0.5 * (du[(a * d + b) * nn + node] + du[(b * d + a) * nn + node]);
                c2 += 2.0 * eab * eab;
            }
        tr[node] = t;
        ec[node] = c2;
    }
    free(du);
}

/* thermal factor |grad T|^2 (objectives.hpp:348-361) */
static void grad_sq(const grid_t* g, const double* T, double* out) {
    const int64_t nn = nnodes(g);
    double* grad = (double*)malloc(sizeof(double) * (size_t)(g->dim * nn));
    for (int a = 0; a < g->dim; ++a) derivative(g, T, a, grad + a * nn);
    for (int64_t node = 0; node < nn; ++node) {
        double gsq = 0.0;
        for (int a = 0; a < g->dim; ++a) {
            const double dd = grad[a * nn + node];
            gsq += dd * dd;
        }
        out[node] = gsq;
    }
    free(grad);
}

/* phase_mass, serial branch (phase_field.hpp:84-95) */
static double phase_mass(const grid_t* g, const double* p) {
    double total = 0.0;
    for (int64_t k = 0; k < g->n[2]; ++k)
        for (int64_t j = 0; j < g->n[1]; ++j)
            for (int64_t i = 0; i < g->n[0]; ++i)
                total += p[(k * g->n[1] + j) * g->n[0] + i] * cell_volume(g, i, j, k);
    return total;
}

double orc_phase_mass(const orc_grid* o, const double* phi) {
    grid_t g;
    return grid_init(&g, o) ? NAN : phase_mass(&g, phi);
}

/* volume_fractions (objectives.hpp:207-214) */
static void volume_fractions(const grid_t* g, int np, const double* phases, double* out) {
    const double inv_vol = 1.0 / domain_volume(g);
    const int64_t n = nnodes(g);
    for (int i = 0; i < np; ++i) out[i] = phase_mass(g, phases + i * n) * inv_vol;
}

static void node_ijk(const grid_t* g, int64_t node, int64_t* i, int64_t* j, int64_t* k) {
    const int64_t nx = g->n[0], ny = g->n[1];
    *k = node / (nx * ny);
    *j = (node - *k * nx * ny) / nx;
    *i = node - (*k * ny + *j) * nx;
}

/* detail::region_volume (objectives.hpp:251-262) */
static double region_volume(const grid_t* g, const orc_targets* t) {
    double vol = 0.0;
    for (int64_t r = 0; r < t->nregion; ++r) {
        int64_t i, j, k;
        node_ijk(g, t->region_nodes[r], &i, &j, &k);
        vol += cell_volume(g, i, j, k);
    }
    return vol;
}

/* region_fractions_measured (objectives.hpp:267-288) */
static int region_fractions_measured(const grid_t* g, const orc_targets* t, int np,
                                     const double* phases, double* m) {
    if (t->nregion == 0) return fail(2, "region_objective: region mask covers no nodes");
    const double vol_b = region_volume(g, t);
    const int64_t n = nnodes(g);
    for (int q = 0; q < np; ++q) {
        double acc = 0.0;
        for (int64_t r = 0; r < t->nregion; ++r) {
            int64_t i, j, k;
            const int64_t node = t->region_nodes[r];
            node_ijk(g, node, &i, &j, &k);
            acc += phases[q * n + node] * cell_volume(g, i, j, k);
        }
        m[q] = acc / vol_b;
    }
    return 0;
}

/* sensitivities (objectives.hpp:336-439) */
static int sensitivities(const grid_t* g, const orc_material* m, const orc_targets* t,
                         const double* phases, const double* state, double* gc, double* gv,
                         double* gu, double* gr) {
    int rc = validate_material(m, m->nphases);
    if (rc) return rc;
    const int np = m->nphases;
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    const int64_t nn = nnodes(g);
    const double e = m->penalty;
    double* factor = (double*)malloc(sizeof(double) * (size_t)nn);
    if (m->kind == 0) {
        grad_sq(g, state, factor);
    } else {
        double* tr = (double*)malloc(sizeof(double) * (size_t)nn);
        double* ec = (double*)malloc(sizeof(double) * (size_t)nn);
        strain_invariants(g, state, tr, ec);
        const double nu = m->poisson_ratio;
        const double ctr = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
        const double cec = 1.0 / (1.0 + nu);
        for (int64_t node = 0; node < nn; ++node)
            factor[node] = ctr * tr[node] * tr[node] + cec * ec[node];
        free(tr);
        free(ec);
    }
    double means[ORC_MAX_PHASES];
    volume_fractions(g, np, phases, means);
    const double inv_vol = 1.0 / domain_volume(g);
    const double floor_v = m->void_floor;
    for (int i = 0; i < np; ++i) {
        double* gci = gc + i * nn;
        double* gvi = gv + i * nn;
        double* gui = gu + i * nn;
        const double prop = m->properties[i];
        const double dm = 2.0 * (means[i] - t->fractions[i]) * inv_vol;
        for (int64_t k = 0; k < nz; ++k)
            for (int64_t j = 0; j < ny; ++j)
                for (int64_t ii = 0; ii < nx; ++ii) {
                    const int64_t node = (k * ny + j) * nx + ii;
                    const double vol = cell_volume(g, ii, j, k);
                    double mix = 0.0;
                    double ssum = -1.0;
                    for (int q = 0; q < np; ++q) {
                        mix += m->properties[q] * pow_penalty(phases[q * nn + node], e);
                        ssum += phases[q * nn + node];
                    }
                    const double dprop =
                        mix > floor_v ? e * prop * pow_penalty(phases[i * nn + node], e - 1.0) : 0.0;
                    gci[node] = dprop * factor[node] * vol;
                    gvi[node] = dm * vol;
                    gui[node] = 2.0 * ssum * vol;
                }
    }
    if (t->region_fractions && gr) {
        double mb[ORC_MAX_PHASES];
        rc = region_fractions_measured(g, t, np, phases, mb);
        if (rc) {
            free(factor);
            return rc;
        }
        const double vol_b = region_volume(g, t);
        for (int i = 0; i < np; ++i) {
            double* gri = gr + i * nn;
            for (int64_t node = 0; node < nn; ++node) gri[node] = 0.0;
            const double coeff = 2.0 * (mb[i] - t->region_fractions[i]) / vol_b;
            for (int64_t r = 0; r < t->nregion; ++r) {
                int64_t ri, rj, rk;
                const int64_t node = t->region_nodes[r];
                node_ijk(g, node, &ri, &rj, &rk);
                gri[node] = coeff * cell_volume(g, ri, rj, rk);
            }
        }
    }
    free(factor);
    return 0;
}

int orc_sensitivities(const orc_grid* o, const orc_material* m, const orc_targets* t,
                      const double* phases, const double* state, double* gc, double* gv,
                      double* gu, double* gr) {
    grid_t g;
    const int rc = grid_init(&g, o);
    return rc ? rc : sensitivities(&g, m, t, phases, state, gc, gv, gu, gr);
}

/* ObjectiveWeights::validate (objectives.hpp:44-51) */
static int validate_weights(const orc_weights* w) {
    if (w->alpha_compliance < 0 || w->alpha_volume < 0 || w->alpha_unity < 0 ||
        w->alpha_region < 0)
        return fail(2, "weights: must be non-negative");
    if (w->alpha_compliance + w->alpha_volume + w->alpha_unity + w->alpha_region <= 0)
        return fail(2, "weights: at least one weight must be positive");
    if (w->compliance_sign != 1 && w->compliance_sign != -1)
        return fail(2, "weights: compliance sign must be +1 or -1");
    return 0;
}

/* design_update_inplace (objectives.hpp:444-480) with par::max_abs_nodes
 * (parallel.hpp:33-42) */
static int design_update(const grid_t* g, int np, const orc_weights* w, double* phases,
                         const double* gc, const double* gv, const double* gu, const double* gr) {
    const int rc = validate_weights(w);
    if (rc) return rc;
    const int64_t nn = nnodes(g);
    for (int i = 0; i < np; ++i) {
        double* phi = phases + i * nn;
        const double* gci = gc + i * nn;
        const double* gvi = gv + i * nn;
        const double* gui = gu + i * nn;
        const double* gri = gr ? gr + i * nn : NULL;
        double cscale = 0.0;
        if (w->alpha_compliance > 0) {
            if (w->normalize_compliance) {
                double gmax = 0.0;
                for (int64_t q = 0; q < nn; ++q) {
                    const double v = gci[q];
                    const double a = v < 0 ? -v : v;
                    if (a > gmax) gmax = a;
                }
                cscale = gmax > 0 ? w->compliance_sign * w->alpha_compliance / gmax : 0.0;
            } else {
                cscale = w->compliance_sign * w->alpha_compliance;
            }
        }
        const double av = w->alpha_volume, au = w->alpha_unity, ar = w->alpha_region;
        for (int64_t q = 0; q < nn; ++q) {
            double step = cscale * gci[q] + av * gvi[q] + au * gui[q];
            if (gri) step += ar * gri[q];
            const double v = phi[q] - step;
            phi[q] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        }
    }
    return 0;
}

int orc_design_update(const orc_grid* o, int np, const orc_weights* w, double* phases,
                      const double* gc, const double* gv, const double* gu, const double* gr) {
    grid_t g;
    const int rc = grid_init(&g, o);
    return rc ? rc : design_update(&g, np, w, phases, gc, gv, gu, gr);
}

/* laplacian_noflux_into (stencil.hpp:109-116, 169-191) */
static double lap_along(const double* f, int64_t t, int64_t nn, int64_t stride, double inv_h2) {
    if (nn == 1) return 0.0;
    if (t == 0) return 2.0 * (f[stride] - f[0]) * inv_h2;
    if (nn - 1 == t) return 2.0 * (f[-stride] - f[0]) * inv_h2;
    return ((f[stride] - f[0]) + (f[-stride] - f[0])) * inv_h2;
}

static void laplacian_noflux(const grid_t* g, const double* fd, double* od) {
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    double inv_h2[3];
    for (int a = 0; a < 3; ++a) inv_h2[a] = 1.0 / (g->h[a] * g->h[a]);
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j) {
            const int64_t row = (k * ny + j) * nx;
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t node = row + i;
                double acc = lap_along(fd + node, i, nx, 1, inv_h2[0]);
                acc += lap_along(fd + node, j, ny, nx, inv_h2[1]);
                if (nz > 1) acc += lap_along(fd + node, k, nz, nx * ny, inv_h2[2]);
                od[node] = acc;
            }
        }
}

/* dwell (phase_field.hpp:56-60) */
static double dwell(double p) { return (PI / 64.0) * sin(2.0 * PI * p); }

/* ch_step_inplace (phase_field.hpp:136-155) */
static int ch_step(const grid_t* g, const orc_ch_params* p, double* phi, double* mu,
                   double* lap, orc_ch_stats* st) {
    if (!(p->mobility > 0.0)) return fail(2, "cahn-hilliard: mobility must be positive");
    if (!(p->gamma > 0.0)) return fail(2, "cahn-hilliard: gamma must be positive");
    if (!(p->dt > 0.0)) return fail(2, "cahn-hilliard: dt must be positive");
    const int64_t n = nnodes(g);
    if (st) st->mass_before = phase_mass(g, phi);
    laplacian_noflux(g, phi, mu); /* chemical_potential_into (:63-72) */
    for (int64_t i = 0; i < n; ++i) mu[i] = dwell(phi[i]) - p->gamma * mu[i];
    laplacian_noflux(g, mu, lap);
    const double step = p->dt * p->mobility;
    for (int64_t i = 0; i < n; ++i) phi[i] += step * lap[i];
    if (st) st->mass_preclamp = phase_mass(g, phi);
    for (int64_t i = 0; i < n; ++i) phi[i] = phi[i] < 0.0 ? 0.0 : (phi[i] > 1.0 ? 1.0 : phi[i]);
    if (st) st->mass_postclamp = phase_mass(g, phi);
    return 0;
}

int orc_ch_step(const orc_grid* o, const orc_ch_params* p, double* phi, orc_ch_stats* st) {
    grid_t g;
    int rc = grid_init(&g, o);
    if (rc) return rc;
    const int64_t n = nnodes(&g);
    double* mu = (double*)malloc(sizeof(double) * (size_t)n);
    double* lap = (double*)malloc(sizeof(double) * (size_t)n);
    rc = ch_step(&g, p, phi, mu, lap, st);
    free(mu);
    free(lap);
    return rc;
}

/* gl_energy (phase_field.hpp:105-125) */
double orc_gl_energy(const orc_grid* o, const double* phi, double gamma) {
    grid_t g;
    if (grid_init(&g, o)) return NAN;
    const int64_t nn = nnodes(&g);
    double* gs = (double*)malloc(sizeof(double) * (size_t)nn);
    grad_sq(&g, phi, gs);
    double total = 0.0;
    for (int64_t k = 0; k < g.n[2]; ++k)
        for (int64_t j = 0; j < g.n[1]; ++j)
            for (int64_t i = 0; i < g.n[0]; ++i) {
                const int64_t node = (k * g.n[1] + j) * g.n[0] + i;
                const double s = sin(PI * phi[node]);
                const double w = s * s / 64.0;
                total += (w + 0.5 * gamma * gs[node]) * cell_volume(&g, i, j, k);
            }
    free(gs);
    return total;
}

/* phase_separation_metric (optimizer.hpp:95-112) */
static double separation(const grid_t* g, int np, const double* phases) {
    const int64_t nn = nnodes(g);
    int64_t near = 0;
    for (int64_t node = 0; node < nn; ++node) {
        double worst = 0.0;
        for (int i = 0; i < np; ++i) {
            const double v = phases[i * nn + node];
            const double d = v < 1.0 - v ? v : 1.0 - v;
            if (d > worst) worst = d;
        }
        if (worst < 0.1) ++near;
    }
    return (double)near / (double)nn;
}

double orc_separation(const orc_grid* o, int np, const double* phases) {
    grid_t g;
    return grid_init(&g, o) ? NAN : separation(&g, np, phases);
}

/* thermal_compliance (objectives.hpp:126-147) */
static double thermal_compliance(const grid_t* g, const double* T, const double* kd) {
    const int64_t nn = nnodes(g);
    double* gs = (double*)malloc(sizeof(double) * (size_t)nn);
    grad_sq(g, T, gs);
    double total = 0.0;
    for (int64_t k = 0; k < g->n[2]; ++k)
        for (int64_t j = 0; j < g->n[1]; ++j)
            for (int64_t i = 0; i < g->n[0]; ++i) {
                const int64_t node = (k * g->n[1] + j) * g->n[0] + i;
                total += kd[node] * gs[node] * cell_volume(g, i, j, k);
            }
    free(gs);
    return total;
}

/* mechanical_compliance (objectives.hpp:183-204) with make_lame (state_solver.hpp:113-127) */
static double mechanical_compliance(const grid_t* g, const double* u, const double* modulus,
                                    double nu) {
    const int64_t nn = nnodes(g);
    const double cl = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double cm = 1.0 / (2.0 * (1.0 + nu));
    double* tr = (double*)malloc(sizeof(double) * (size_t)nn);
    double* ec = (double*)malloc(sizeof(double) * (size_t)nn);
    strain_invariants(g, u, tr, ec);
    double total = 0.0;
    for (int64_t k = 0; k < g->n[2]; ++k)
        for (int64_t j = 0; j < g->n[1]; ++j)
            for (int64_t i = 0; i < g->n[0]; ++i) {
                const int64_t node = (k * g->n[1] + j) * g->n[0] + i;
                const double t = tr[node];
                const double lam = cl * modulus[node];
                const double mu = cm * modulus[node];
                total += (lam * t * t + 2.0 * mu * ec[node]) * cell_volume(g, i, j, k);
            }
    free(tr);
    free(ec);
    return total;
}

/* unity_objective (objectives.hpp:229-247) */
static double unity_objective(const grid_t* g, int np, const double* phases) {
    const int64_t nn = nnodes(g);
    double total = 0.0;
    for (int64_t k = 0; k < g->n[2]; ++k)
        for (int64_t j = 0; j < g->n[1]; ++j)
            for (int64_t i = 0; i < g->n[0]; ++i) {
                const int64_t node = (k * g->n[1] + j) * g->n[0] + i;
                double s = -1.0;
                for (int q = 0; q < np; ++q) s += phases[q * nn + node];
                total += s * s * cell_volume(g, i, j, k);
            }
    return total;
}

/* evaluate_objectives (objectives.hpp:304-320) */
static int evaluate_objectives(const grid_t* g, const orc_material* m, const orc_targets* t,
                               const double* phases, const double* state, orc_report* out) {
    int rc = validate_material(m, m->nphases);
    if (rc) return rc;
    const int np = m->nphases;
    const int64_t nn = nnodes(g);
    double* prop = (double*)malloc(sizeof(double) * (size_t)nn);
    interpolate(g, m, phases, prop);
    out->compliance = m->kind == 0 ? thermal_compliance(g, state, prop)
                                   : mechanical_compliance(g, state, prop, m->poisson_ratio);
    free(prop);
    double vf[ORC_MAX_PHASES];
    volume_fractions(g, np, phases, vf);
    double j = 0.0;
    for (int i = 0; i < np; ++i) {
        const double d = vf[i] - t->fractions[i];
        j += d * d;
    }
    out->volume = j;
    out->unity = unity_objective(g, np, phases);
    out->region = 0.0;
    if (t->region_fractions) {
        double mb[ORC_MAX_PHASES];
        if ((rc = region_fractions_measured(g, t, np, phases, mb))) return rc;
        double jr = 0.0;
        for (int i = 0; i < np; ++i) {
            const double d = mb[i] - t->region_fractions[i];
            jr += d * d;
        }
        out->region = jr;
    }
    for (int i = 0; i < np; ++i) out->volume_fractions[i] = vf[i];
    return 0;
}

int orc_evaluate_objectives(const orc_grid* o, const orc_material* m, const orc_targets* t,
                            const double* phases, const double* state, orc_report* out) {
    grid_t g;
    const int rc = grid_init(&g, o);
    return rc ? rc : evaluate_objectives(&g, m, t, phases, state, out);
}

/* ----------------------------------------------------------------- run() (a25) */

/* LoopSchedule::validate (optimizer.hpp:23-33) + CahnHilliardParams::validate */
static int validate_schedule(const orc_schedule* s) {
    int rc = validate_params(&s->pt);
    if (rc) return rc;
    if (!(s->ch.mobility > 0.0)) return fail(2, "cahn-hilliard: mobility must be positive");
    if (!(s->ch.gamma > 0.0)) return fail(2, "cahn-hilliard: gamma must be positive");
    if (!(s->ch.dt > 0.0)) return fail(2, "cahn-hilliard: dt must be positive");
    if (s->max_loops < 1) return fail(2, "schedule: max_loops must be >= 1");
    if (!(s->convergence_tol > 0.0))
        return fail(2, "schedule: convergence tolerance must be positive");
    if (s->convergence_window < 2) return fail(2, "schedule: convergence window must be >= 2");
    if (s->report_every < 1) return fail(2, "schedule: report_every must be >= 1");
    return 0;
}

/* run() (optimizer.hpp:120-223) */
int orc_run(const orc_problem* pr, const orc_schedule* sc, double* phases_out,
            double* state_out, orc_record* records, long records_cap, long* nrecords,
            orc_run_result* res) {
    int rc = validate_schedule(sc);
    if (!rc) rc = validate_weights(&pr->weights);
    if (rc) return rc;
    grid_t g;
    if ((rc = grid_init(&g, &pr->grid))) return rc;
    const int np = pr->material.nphases;
    const int64_t nn = nnodes(&g);
    const int comps = pr->physics ? g.dim : 1;
    const int64_t ns = nn * comps;

    memset(res, 0, sizeof *res);
    double* phases = (double*)malloc(sizeof(double) * (size_t)(np * nn));
    memcpy(phases, pr->initial_phases, sizeof(double) * (size_t)(np * nn));
    double* cur = (double*)malloc(sizeof(double) * (size_t)ns);
    double* prev = (double*)malloc(sizeof(double) * (size_t)ns);
    memcpy(cur, pr->initial_state, sizeof(double) * (size_t)ns);
    memcpy(prev, pr->initial_state, sizeof(double) * (size_t)ns);
    hist_t h = {cur, prev};
    double* property = (double*)malloc(sizeof(double) * (size_t)nn);
    double* r = (double*)malloc(sizeof(double) * (size_t)ns);
    double* gc = (double*)malloc(sizeof(double) * (size_t)(np * nn));
    double* gv = (double*)malloc(sizeof(double) * (size_t)(np * nn));
    double* gu = (double*)malloc(sizeof(double) * (size_t)(np * nn));
    double* gr = pr->targets.region_fractions ? (double*)malloc(sizeof(double) * (size_t)(np * nn))
                                              : NULL;
    double* mu_s = (double*)malloc(sizeof(double) * (size_t)nn);
    double* lap_s = (double*)malloc(sizeof(double) * (size_t)nn);
    double* comp_hist = (double*)malloc(sizeof(double) * (size_t)(sc->max_loops + 2));
    long nrec = 0;

    if ((rc = validate_material(&pr->material, np))) goto done;
    interpolate(&g, &pr->material, phases, property);
    op_t op;
    if ((rc = op_init(&op, pr->physics, &pr->grid, &pr->bc, property, pr->material.poisson_ratio,
                      pr->source)))
        goto done;
    const double nu = pr->material.poisson_ratio;
    const double cm = 1.0 / (2.0 * (1.0 + nu));

    res->termination = 1;
    for (long loop = 1; loop <= sc->max_loops; ++loop) {
        res->loops = loop;
        /* interpolate_into + update_lame (:187-189); op reads property / mu */
        interpolate(&g, &pr->material, phases, property);
        if (pr->physics)
            for (int64_t i = 0; i < nn; ++i) op.mu[i] = cm * property[i];
        int64_t abort_step = 0;
        rc = hybrid_solve(&h, &op, &sc->pt, r, &abort_step);
        if (rc == 1) {
            res->termination = 2;
            snprintf(res->abort_detail, sizeof res->abort_detail, "loop %ld: %s", loop, g_err);
            rc = 0;
            break;
        }
        if (rc) break;
        res->apt_steps += sc->pt.n_apt;
        res->pt_steps += sc->pt.n_pt;
        if ((rc = sensitivities(&g, &pr->material, &pr->targets, phases, h.cur, gc, gv, gu, gr)))
            break;
        if ((rc = design_update(&g, np, &pr->weights, phases, gc, gv, gu, gr))) break;
        ++res->design_updates;
        double pre[ORC_MAX_PHASES], post[ORC_MAX_PHASES];
        for (int i = 0; i < np; ++i) {
            orc_ch_stats st;
            if ((rc = ch_step(&g, &sc->ch, phases + i * nn, mu_s, lap_s, &st))) break;
            pre[i] = st.mass_preclamp;
            post[i] = st.mass_postclamp;
        }
        if (rc) break;
        ++res->ch_steps;
        for (int i = 0; i < np; ++i) res->clamp_mass_drift += fabs(post[i] - pre[i]);
        int nonfinite = 0;
        for (int64_t q = 0; q < np * nn; ++q)
            if (!isfinite(phases[q])) nonfinite = 1;
        if (nonfinite) {
            res->termination = 2;
            snprintf(res->abort_detail, sizeof res->abort_detail,
                     "loop %ld: numerical abort in 'phi' at step %ld: design field turned "
                     "non-finite",
                     loop, loop);
            break;
        }
        if (loop % sc->report_every == 0 || loop == 1 || loop == sc->max_loops) {
            /* record lambda (:145-168) */
            orc_report rep;
            if ((rc = evaluate_objectives(&g, &pr->material, &pr->targets, phases, h.cur, &rep)))
                break;
            interpolate(&g, &pr->material, phases, property);
            if (pr->physics)
                for (int64_t i = 0; i < nn; ++i) op.mu[i] = cm * property[i];
            if ((rc = op_residual(&op, h.cur, r))) break;
            if (nrec < records_cap) {
                orc_record* o = &records[nrec];
                memset(o, 0, sizeof *o);
                o->loop = loop;
                o->apt_steps = res->apt_steps;
                o->pt_steps = res->pt_steps;
                o->compliance = rep.compliance;
                o->volume = rep.volume;
                o->unity = rep.unity;
                o->region = rep.region;
                for (int i = 0; i < np; ++i) o->volume_fractions[i] = rep.volume_fractions[i];
                o->r_pde = orc_residual_norm(r, nn, comps);
                o->separation = separation(&g, np, phases);
            }
            comp_hist[nrec] = rep.compliance;
            ++nrec;
            /* converged() (:170-181) */
            const int w = sc->convergence_window;
            if (nrec >= w) {
                double lo = comp_hist[nrec - 1], hi = lo;
                for (int i = 0; i < w; ++i) {
                    const double v = comp_hist[nrec - 1 - i];
                    lo = v < lo ? v : lo;
                    hi = v > hi ? v : hi;
                }
                const double ah = fabs(hi);
                const double scale = ah > 1e-300 ? ah : 1e-300;
                if ((hi - lo) / scale < sc->convergence_tol) {
                    res->termination = 0;
                    break;
                }
            }
        }
    }
    op_free(&op);
done:
    if (!rc) {
        if (phases_out) memcpy(phases_out, phases, sizeof(double) * (size_t)(np * nn));
        if (state_out) memcpy(state_out, h.cur, sizeof(double) * (size_t)ns);
        if (nrecords) *nrecords = nrec;
    }
    free(phases);
    free(cur);
    free(prev);
    free(property);
    free(r);
    free(gc);
    free(gv);
    free(gu);
    free(gr);
    free(mu_s);
    free(lap_s);
    free(comp_hist);
    return rc;
}

/* ------------------------------------------------------------------ writers */
/* field_io.cpp:15-19: every double through snprintf("%.17g"). */
static int io_fail(const char* what, const char* path) {
    char m[600];
    snprintf(m, sizeof m, "%s '%s'%s", what, path, strcmp(what, "cannot open") == 0 ? " for writing" : "");
    return fail(4, m);
}

/* write_field_csv (field_io.cpp:29-47): header line, then one line per (k, j) row. */
int orc_write_field_csv(const orc_grid* o, const double* values, const char* path) {
    grid_t g;
    if (grid_init(&g, o)) return 2;
    FILE* f = fopen(path, "w");
    if (!f) return io_fail("cannot open", path);
    fprintf(f, "# nx=%lld ny=%lld nz=%lld dx=%.17g dy=%.17g dz=%.17g\n", (long long)g.n[0], (long long)g.n[1],
            (long long)g.n[2], g.h[0], g.h[1], g.h[2]);
    for (int64_t k = 0; k < g.n[2]; ++k)
        for (int64_t j = 0; j < g.n[1]; ++j) {
            const int64_t row = (k * g.n[1] + j) * g.n[0];
            for (int64_t i = 0; i < g.n[0]; ++i) fprintf(f, i ? ",%.17g" : "%.17g", values[row + i]);
            fputc('\n', f);
        }
    const int bad = ferror(f);
    if (fclose(f) || bad) return io_fail("write failed for", path);
    return 0;
}

/* write_pgm (field_io.cpp:68-101): finite min/max, rows top-down, lround(255 v). */
int orc_write_pgm(const orc_grid* o, const double* values, const char* path) {
    grid_t g;
    if (grid_init(&g, o)) return 2;
    if (g.dim != 2) return fail(2, "write_pgm: only 2D fields");
    const int64_t n = nnodes(&g);
    double lo = 0.0, hi = 0.0;
    int first = 1;
    for (int64_t i = 0; i < n; ++i) {
        const double v = values[i];
        if (!isfinite(v)) continue;
        lo = first ? v : (v < lo ? v : lo); /* std::min(lo, v): lo unless v < lo */
        hi = first ? v : (hi < v ? v : hi); /* std::max(hi, v): hi unless hi < v */
        first = 0;
    }
    const double span = hi > lo ? hi - lo : 1.0;
    FILE* f = fopen(path, "wb");
    if (!f) return io_fail("cannot open", path);
    fprintf(f, "P5\n%lld %lld\n255\n", (long long)g.n[0], (long long)g.n[1]);
    unsigned char* row = (unsigned char*)malloc((size_t)g.n[0]);
    for (int64_t j = g.n[1] - 1; j >= 0; --j) {
        for (int64_t i = 0; i < g.n[0]; ++i) {
            const double raw = values[j * g.n[0] + i];
            const double v = isfinite(raw) ? (raw - lo) / span : 0.0;
            const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); /* std::clamp */
            row[i] = (unsigned char)lround(255.0 * c);
        }
        fwrite(row, 1, (size_t)g.n[0], f);
    }
    free(row);
    const int bad = ferror(f);
    if (fclose(f) || bad) return io_fail("write failed for", path);
    char side[1100];
    snprintf(side, sizeof side, "%s.scale.txt", path);
    FILE* s = fopen(side, "w");
    if (!s) return fail(4, "cannot open side file for writing");
    fprintf(s, "min = %.17g\nmax = %.17g\nrows = top_to_bottom\n", lo, hi);
    fclose(s);
    return 0;
}

/* write_vtk_structured_points (field_io.cpp:103-126): legacy ASCII, one value per line. */
int orc_write_vtk(const orc_grid* o, int narrays, const char* const* names, const double* values,
                  const char* path) {
    grid_t g;
    if (grid_init(&g, o)) return 2;
    FILE* f = fopen(path, "w");
    if (!f) return io_fail("cannot open", path);
    const int64_t n = nnodes(&g);
    fprintf(f,
            "# vtk DataFile Version 3.0\nstructured point fields\nASCII\nDATASET STRUCTURED_POINTS\n"
            "DIMENSIONS %lld %lld %lld\nORIGIN 0 0 0\nSPACING %.17g %.17g %.17g\nPOINT_DATA %lld\n",
            (long long)g.n[0], (long long)g.n[1], (long long)g.n[2], g.h[0], g.h[1], g.h[2], (long long)n);
    for (int a = 0; a < narrays; ++a) {
        fprintf(f, "SCALARS %s double 1\nLOOKUP_TABLE default\n", names[a]);
        for (int64_t i = 0; i < n; ++i) fprintf(f, "%.17g\n", values[(int64_t)a * n + i]);
    }
    const int bad = ferror(f);
    if (fclose(f) || bad) return io_fail("write failed for", path);
    return 0;
}
