/*
 * petto_dev.h -- C-ABI of the B200 (sm_100a) PeTTO hot path.
 *
 * Drop-in boundary for the reference's state-solver seam
 * (/root/reference/proj/include/petto/state_solver.hpp): a device context owns
 * every field of one problem in HBM (structure-of-arrays FP64, the reference's
 * x-fastest, component-major layout) and exposes the reference entry points as
 * POD-only calls.  The C++ adapter include/petto_dev.hpp maps these onto the
 * reference's own types (StateOperator, StateHistory, PTParams, run()), and
 * INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *   - Host arrays are caller-owned; every upload/download is a copy.
 *   - Fields: node = (k*ny + j)*nx + i (grid.hpp:47); component c of a
 *     vector field occupies [c*N, (c+1)*N) (grid.hpp:93); P phases are P
 *     consecutive N-blocks.
 *   - Status codes (every int-returning call):
 *       PETTO_OK 0, PETTO_ABORT 1 (NumericalAbort, errors.hpp:10-23),
 *       PETTO_INVALID 2 (std::invalid_argument), PETTO_ERROR 3 (CUDA/other).
 *     petto_dev_last_error() holds the message, worded like the reference's.
 *   - A context is not thread-safe (same as the reference's globals).
 *   - No CPU fallback: creating a context without a usable sm_100 device
 *     fails with PETTO_ERROR.
 */
#ifndef PETTO_DEV_H
#define PETTO_DEV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PETTO_OK 0
#define PETTO_ABORT 1
#define PETTO_INVALID 2
#define PETTO_ERROR 3
#define PETTO_IO 4  /* IoError (errors.hpp): cannot open / write failed (CLI exit code 4) */

#define PETTO_MAX_PHASES 8

typedef struct petto_ctx petto_ctx;

/* Execution mode of the state kernels.
 *   FAST:    fused residual+update kernels (modal cell-centric elasticity,
 *            FMA contraction, tree reductions); per step <= 1e-12 relative to
 *            the reference.
 *   REPLICA: the reference's operation order, no FMA contraction, serial-order
 *            reductions -- bit-identical to the reference for parity tests. */
#define PETTO_MODE_FAST 0
#define PETTO_MODE_REPLICA 1

/* Grid + operator description.  Replaces Grid::make2d/make3d (grid.hpp:27-43)
 * plus the operator choice of run() (optimizer.hpp:133-138). */
typedef struct {
    int dim;           /* 2 or 3 */
    int64_t n[3];      /* nodes per axis; n[2] = 1 in 2D */
    double length[3];  /* domain extents; spacing = length/(n-1) */
    int physics;       /* 0 heat (HeatOperator), 1 elasticity (ElasticityOperator) */
    double poisson_ratio; /* make_lame / update_lame nu (state_solver.hpp:113-142) */
    int mode;          /* PETTO_MODE_FAST or PETTO_MODE_REPLICA */
    int device;        /* CUDA ordinal */
    /* slab decomposition along the outermost axis (k): this rank owns node
     * planes [k_begin, k_end) of the global grid.  Single GPU: 0, n[2]. */
    int64_t k_begin, k_end;
    /* 3D, FAST mode: keep the grid in HBM with x as the outermost (slab) axis --
     * device axes (y, z, x), displacement components permuted alike; uploads and
     * downloads permute, the host side keeps the reference's x-fastest layout
     * (grid.hpp:47).  Then k_begin/k_end are x planes: slabs along the longest
     * axis of an x-elongated grid.  0: the reference layout. */
    int x_outermost;
} petto_grid_desc;

/* PTParams (state_solver.hpp:17-34); form 0 ExplicitDamping, 1 SemiImplicitDamping. */
typedef struct {
    double dt_pt, dt_apt, theta;
    long n_apt, n_pt;
    int form;
} petto_pt_params;

/* SolveStats (state_solver.hpp:502-507). */
typedef struct {
    long iterations;
    double r_initial, r_final;
    int converged;
} petto_solve_stats;

/* MaterialModel (objectives.hpp:19-34); kind 0 Thermal, 1 Elastic. */
typedef struct {
    int kind;
    int nphases;
    double properties[PETTO_MAX_PHASES];
    double poisson_ratio, penalty, void_floor;
} petto_material;

/* VolumeTargets (objectives.hpp:56-62); region_nodes sorted, has_region 0/1. */
typedef struct {
    double fractions[PETTO_MAX_PHASES];
    int has_region;
    double region_fractions[PETTO_MAX_PHASES];
    int64_t nregion;
    const int64_t* region_nodes;
} petto_targets;

/* ObjectiveWeights (objectives.hpp:36-52), already effective for the grid. */
typedef struct {
    double alpha_compliance, alpha_volume, alpha_unity, alpha_region;
    int normalize_compliance;
    int compliance_sign;
} petto_weights;

/* CahnHilliardParams / ChStepStats (phase_field.hpp:12-22, 127-131). */
typedef struct { double mobility, gamma, dt; } petto_ch_params;
typedef struct { double mass_before, mass_preclamp, mass_postclamp; } petto_ch_stats;

/* ObjectiveReport (objectives.hpp:64-72). */
typedef struct {
    double compliance, volume, unity, region;
    double volume_fractions[PETTO_MAX_PHASES];
} petto_report;

/* LoopSchedule (optimizer.hpp:15-34). */
typedef struct {
    petto_pt_params pt;
    petto_ch_params ch;
    long max_loops;
    double convergence_tol;
    int convergence_window;
    int report_every;
} petto_schedule;

/* HistoryRecord (optimizer.hpp:49-61). */
typedef struct {
    long loop;
    long long apt_steps, pt_steps;
    double compliance, volume, unity, region, r_pde, separation;
    double volume_fractions[PETTO_MAX_PHASES];
    double wall_seconds;
} petto_record;

/* OptimizationResult counters (optimizer.hpp:79-92); termination 0 Converged,
 * 1 MaxLoops, 2 AbortedNaN. */
typedef struct {
    long loops;
    long long apt_steps, pt_steps, design_updates, ch_steps;
    double clamp_mass_drift;
    int termination;
    char abort_detail[256];
} petto_run_result;

typedef void (*petto_record_cb)(const petto_record* rec, void* user);

/* ------------------------------------------------------------ lifecycle */

const char* petto_dev_version(void);
int petto_dev_device_count(void);
/* Allocates the device fields.  Replaces constructing Grid + Fields. */
int petto_dev_create(const petto_grid_desc* desc, petto_ctx** out);
void petto_dev_destroy(petto_ctx* ctx);
const char* petto_dev_last_error(const petto_ctx* ctx);
/* The CUDA stream every call of this context is ordered on (cudaStream_t). */
void* petto_dev_stream(petto_ctx* ctx);
int petto_dev_set_mode(petto_ctx* ctx, int mode);

/* ------------------------------------------------------------- uploads */

/* ConstraintSet (grid.hpp:176-181): sorted entries comp*N + node, values.
 * Replaces make_constraints' product being handed to the operator. */
int petto_dev_set_constraints(petto_ctx* ctx, const int64_t* entry, const double* value,
                              int64_t count);
/* Heat source (1 x N) or elastic loads (dim x N), the operator's source_/loads_. */
int petto_dev_set_source(petto_ctx* ctx, const double* source);
/* Property field: conductivity (heat) or Young's modulus (elasticity, stored
 * as Lame mu = E/(2(1+nu)) like update_lame, state_solver.hpp:129-142). */
int petto_dev_set_property(petto_ctx* ctx, const double* property);
/* Elasticity from the Lame pair the reference's ElasticityOperator takes
 * (ElasticMaterialField, state_solver.hpp:106-110, 292-297): mu drives the
 * residual, lambda only the positivity check and the operator's nu. */
int petto_dev_set_lame(petto_ctx* ctx, const double* lambda, const double* mu);
/* ElasticityOperator constructor semantics (state_solver.hpp:292-310): checks
 * the Lame fields are positive, derives nu from node 0 and builds the unit-cell
 * stiffness.  Heat: validates nothing (kappa is checked per residual). */
int petto_dev_init_operator(petto_ctx* ctx);
/* StateHistory (state_solver.hpp:37-45): current and previous iterates. */
int petto_dev_set_state(petto_ctx* ctx, const double* current, const double* previous);
int petto_dev_get_state(petto_ctx* ctx, double* current, double* previous);

/* ------------------------------------------------------- state solve (a12-a17) */

/* op.residual(current, out) (state_solver.hpp:83-86 / 327-385) with zeroed
 * constrained entries; out may be NULL; r_pde = residual_norm(out) (:49-58). */
int petto_dev_residual(petto_ctx* ctx, double* out, double* r_pde);
/* hybrid_solve (state_solver.hpp:480-498).  On PETTO_ABORT *abort_step holds the
 * reference's check_finite step index. */
int petto_dev_hybrid_solve(petto_ctx* ctx, const petto_pt_params* p, int64_t* abort_step);
/* iterate_to_tolerance (state_solver.hpp:511-541); mode 0 PT, 1 APT. */
int petto_dev_iterate_to_tolerance(petto_ctx* ctx, int mode, const petto_pt_params* p,
                                   double target, long max_iters, petto_solve_stats* stats);

/* ------------------------------------------------ design subsystems (a19-a26) */

int petto_dev_set_design(petto_ctx* ctx, const petto_material* m, const petto_targets* t,
                         const petto_weights* w);
int petto_dev_set_phases(petto_ctx* ctx, const double* phases);
int petto_dev_get_phases(petto_ctx* ctx, double* phases);
/* interpolate_into + update_lame (objectives.hpp:95-116, state_solver.hpp:129-142):
 * property := interpolate(phases); optionally downloaded. */
int petto_dev_interpolate(petto_ctx* ctx, double* property_out);
/* sensitivities + design_update_inplace (objectives.hpp:336-480) on the device
 * phases with the current state held fixed. */
int petto_dev_design_update(petto_ctx* ctx);
/* ch_step_multi_inplace (phase_field.hpp:168-176); stats: one per phase. */
int petto_dev_ch_step(petto_ctx* ctx, const petto_ch_params* p, petto_ch_stats* stats);
/* evaluate_objectives (objectives.hpp:304-320) and the separation metric
 * (optimizer.hpp:95-112) of the current phases/state. */
int petto_dev_objectives(petto_ctx* ctx, petto_report* rep, double* separation);
/* The coupled loop run() (optimizer.hpp:120-223), device resident; the
 * callback fires at every record like RecordCallback.  Expects the state, the
 * phases (initial), source, constraints and design already set. */
int petto_dev_run(petto_ctx* ctx, const petto_schedule* s, petto_record_cb cb, void* user,
                  petto_run_result* result);

/* ------------------------------------------- slab decomposition */

/* A rank's context is created with petto_grid_desc.k_begin/k_end = its planes of
 * the outermost axis and receives the GLOBAL host arrays on upload (it keeps its
 * planes plus one ghost plane per interior face); downloads fill its owned planes.
 *
 * Multi-process (one GPU per rank): rank 0 creates a 128-byte NCCL unique id, the
 * caller broadcasts it, every rank calls petto_dev_comm_init.  From then on the
 * state solves exchange ghost planes with the +-1 ranks after every step, the
 * design loop exchanges the ghost planes of phi and mu around the Cahn-Hilliard
 * kernels, and every global scalar (r^2, the first non-finite step at each
 * check_finite, masses, max|gc|, compliance/unity/region sums, the separation
 * count) is all-reduced -- REPLICA sums as one serial sum passed rank to rank. */
int petto_dev_comm_unique_id(void* id128);
int petto_dev_comm_init(petto_ctx* ctx, const void* id128, int rank, int nranks);

/* Peer halo (optional, after comm_init): each rank exports the IPC handles of
 * its state buffers and step inbox (PETTO_PEER_BLOB_BYTES bytes), the caller
 * all-gathers the blobs, and every rank imports its -1 / +1 neighbours' (NULL
 * at a physical end).  From then on the fused 3D steps of hybrid_solve store
 * their boundary planes straight into the neighbours' ghost planes over
 * NVLink and order the steps with stream-ordered flags (no NCCL call and no
 * SM time for the halo); set_state takes part in the same step protocol. */
#define PETTO_PEER_BLOB_BYTES 512
int petto_dev_peer_export(petto_ctx* ctx, void* blob);
int petto_dev_peer_import(petto_ctx* ctx, const void* lo_blob, const void* hi_blob);

/* Single process driving several contexts (several GPUs, or one GPU in tests):
 * link the contexts of consecutive slabs, then run them in lock step -- the same
 * solver and design-loop code as one context or one NCCL rank, with the group's
 * own transport: fused 3D steps use the peer halo (direct pointers), the other
 * kernels stream-ordered peer copies of the ghost planes, and every reduction
 * (r^2, first non-finite step, masses, max|gc|, compliance/unity/region sums,
 * the separation count) is combined on the first context in slab order
 * (REPLICA: one serial sum chained across the slabs, bit-identical to one
 * domain).  A linked or communicator-less slab context is refused by the
 * single-context entry points (PETTO_INVALID).  Results land in ctxs[0]. */
int petto_dev_group_link(petto_ctx** ctxs, int n);
int petto_dev_group_hybrid_solve(petto_ctx** ctxs, int n, const petto_pt_params* p, int64_t* abort_step);
int petto_dev_group_residual(petto_ctx** ctxs, int n, double* r_pde);
int petto_dev_group_iterate_to_tolerance(petto_ctx** ctxs, int n, int mode, const petto_pt_params* p,
                                         double target, long max_iters, petto_solve_stats* stats);
int petto_dev_group_interpolate(petto_ctx** ctxs, int n);
int petto_dev_group_init_operator(petto_ctx** ctxs, int n); /* nu from node 0 on the first slab */
int petto_dev_group_design_update(petto_ctx** ctxs, int n);
int petto_dev_group_ch_step(petto_ctx** ctxs, int n, const petto_ch_params* p, petto_ch_stats* stats);
int petto_dev_group_objectives(petto_ctx** ctxs, int n, petto_report* rep, double* separation);
int petto_dev_group_run(petto_ctx** ctxs, int n, const petto_schedule* s, petto_record_cb cb, void* user,
                        petto_run_result* result);

/* --------------------------------------------------------------- utilities */

/* detail::unit_cell_stiffness (state_solver.hpp:149-237), node-major dofs. */
void petto_dev_unit_cell_stiffness(int dim, const double h[3], double nu, double* ke);
/* elasticity_spectral_bound (state_solver.hpp:254-279). */
double petto_dev_spectral_bound(int dim, const int64_t n[3], const double length[3], double nu,
                                double e_max);

/* Instrumentation for bench.py: kernel launches issued by this context, and
 * (when enabled) CUDA-event time of the dominant state kernel. */
/* ---- Output writers --------------------------------
 * The reference's writers from device buffers, byte-identical to its files:
 * every value formatted on the device exactly as snprintf("%.17g")
 * (field_io.cpp:15-19), the text assembled in HBM and written in chunks.
 * Single-domain contexts only (a slab rank returns PETTO_INVALID).  Errors:
 * PETTO_IO with the reference's IoError message. */
#define PETTO_FIELD_STATE 0    /* component `index` of the current state */
#define PETTO_FIELD_PHASE 1    /* phase `index` (after petto_dev_set_design) */
#define PETTO_FIELD_PROPERTY 2 /* the property field (E / kappa; petto_dev_interpolate refreshes it) */
typedef struct {
    int field;
    int index;
    const char* name;  /* VTK array name, e.g. "phase_0", "modulus", "displacement_x" */
} petto_array;
/* write_field_csv (field_io.cpp:29-47) */
int petto_dev_write_field_csv(petto_ctx* ctx, int field, int index, const char* path);
/* write_vtk_structured_points (field_io.cpp:103-126), arrays in file order */
int petto_dev_write_vtk(petto_ctx* ctx, const petto_array* arrays, int narrays, const char* path);
/* write_pgm (field_io.cpp:68-101), 2D only; also writes "<path>.scale.txt" */
int petto_dev_write_pgm(petto_ctx* ctx, int field, int index, const char* path);
/* The formatter alone: n doubles (host or device memory) as "%.17g" each followed
 * by '\n' (sep_mode 0) or by ',' / '\n' at the end of every `row` values
 * (sep_mode 1) into out[0, cap); *len = bytes written. */
int petto_dev_format_values(petto_ctx* ctx, const double* values, int64_t n, int sep_mode, int64_t row,
                            char* out, int64_t cap, int64_t* len);

int64_t petto_dev_launch_count(const petto_ctx* ctx);
/* Instrumentation: CUDA events around the hot launches (0 off; n >= 1: around
 * every n-th launch, so a timed region can sample launch durations cheaply). */
int petto_dev_kernel_timing(petto_ctx* ctx, int enable);
int petto_dev_kernel_stats(petto_ctx* ctx, double* total_ms, int64_t* launches,
                           double* bytes_per_launch, char* name, int name_cap);

#ifdef __cplusplus
}
#endif

#endif /* PETTO_DEV_H */
