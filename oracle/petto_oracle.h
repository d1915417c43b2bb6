/*
 * petto_oracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * One C interface, two implementations:
 *   oracle/petto_oracle.c   -> oracle/liboracle.so       plain-C restatement of the
 *                                                         reference algorithms ("port")
 *   oracle/ref_shim.cpp     -> oracle/_ref/libpetto_ref.so the UNMODIFIED reference
 *                                                         headers/sources compiled from
 *                                                         /root/reference ("reference")
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load either library.  The product path (libpetto_b200.so) never links them.
 *
 * All fields use the reference layout: x-fastest nodes, node = (k*ny + j)*nx + i
 * (grid.hpp:47), component-major SoA (grid.hpp:93).  Multi-phase fields are P
 * consecutive N-blocks.
 */
#ifndef PETTO_ORACLE_H
#define PETTO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Grid: grid.hpp:21-90.  length[2] ignored in 2D; n[2] must be 1 in 2D. */
typedef struct {
    int dim;
    int64_t n[3];
    double length[3];
} orc_grid;

/* BoundarySpec: grid.hpp:149-172.  kind: 0 Dirichlet, 1 NeumannZero,
 * 2 TractionFree, 3 Roller (CondKind order). */
typedef struct {
    int kind[6];
    double value[6];
    int component[6];
    int64_t npins;
    const int64_t* pin_node;
    const int32_t* pin_comp;
    const double* pin_value;
} orc_bc;

/* PTParams: state_solver.hpp:17-34.  form: 0 ExplicitDamping, 1 SemiImplicitDamping. */
typedef struct {
    double dt_pt, dt_apt, theta;
    long n_apt, n_pt;
    int form;
} orc_pt_params;

/* SolveStats: state_solver.hpp:502-507. */
typedef struct {
    long iterations;
    double r_initial, r_final;
    int converged;
} orc_solve_stats;

/* MaterialModel: objectives.hpp:19-34.  kind: 0 Thermal, 1 Elastic. */
typedef struct {
    int kind;
    int nphases;
    const double* properties;
    double poisson_ratio, penalty, void_floor;
} orc_material;

/* VolumeTargets: objectives.hpp:56-62 (region_fractions NULL = no region). */
typedef struct {
    const double* fractions;
    int64_t nregion;
    const int64_t* region_nodes;
    const double* region_fractions;
} orc_targets;

/* ObjectiveWeights: objectives.hpp:36-52. */
typedef struct {
    double alpha_compliance, alpha_volume, alpha_unity, alpha_region;
    int normalize_compliance;
    int compliance_sign;
} orc_weights;

/* CahnHilliardParams / ChStepStats: phase_field.hpp:12-22, 127-131. */
typedef struct { double mobility, gamma, dt; } orc_ch_params;
typedef struct { double mass_before, mass_preclamp, mass_postclamp; } orc_ch_stats;

#define ORC_MAX_PHASES 8

/* ObjectiveReport: objectives.hpp:64-72. */
typedef struct {
    double compliance, volume, unity, region;
    double volume_fractions[ORC_MAX_PHASES];
} orc_report;

/* Problem<Real>: optimizer.hpp:66-77 (physics 0 heat, 1 elasticity). */
typedef struct {
    orc_grid grid;
    int physics;
    orc_bc bc;
    orc_material material;
    orc_targets targets;
    orc_weights weights;
    const double* source;         /* comps x N */
    const double* initial_phases; /* P x N */
    const double* initial_state;  /* comps x N */
} orc_problem;

/* LoopSchedule: optimizer.hpp:15-34. */
typedef struct {
    orc_pt_params pt;
    orc_ch_params ch;
    long max_loops;
    double convergence_tol;
    int convergence_window;
    int report_every;
} orc_schedule;

/* HistoryRecord: optimizer.hpp:49-61 (wall_seconds omitted: not deterministic). */
typedef struct {
    long loop;
    long long apt_steps, pt_steps;
    double compliance, volume, unity, region, r_pde, separation;
    double volume_fractions[ORC_MAX_PHASES];
} orc_record;

/* OptimizationResult: optimizer.hpp:79-92.  termination: 0 Converged, 1 MaxLoops,
 * 2 AbortedNaN. */
typedef struct {
    long loops;
    long long apt_steps, pt_steps, design_updates, ch_steps;
    double clamp_mass_drift;
    int termination;
    char abort_detail[256];
} orc_run_result;

/* Return codes of the int functions: 0 ok, 1 NumericalAbort, 2 std::invalid_argument,
 * 3 other error.  orc_last_error() holds the exception text. */
const char* orc_last_error(void);
const char* orc_impl_name(void);           /* "port" or "reference" */

void orc_set_threads(int n);                /* parallel.hpp:11 (port: serial only) */
int orc_threads(void);

int64_t orc_num_nodes(const orc_grid* g);
double orc_spacing(const orc_grid* g, int axis);
double orc_cell_volume(const orc_grid* g, int64_t i, int64_t j, int64_t k);

int64_t orc_make_constraints(const orc_grid* g, const orc_bc* bc, int comps,
                             int64_t* entry, double* value, int64_t cap);
void orc_unit_cell_stiffness(int dim, const double h[3], double nu, double* ke);
double orc_elasticity_spectral_bound(const orc_grid* g, double nu, double e_max);
double orc_ch_stable_dt(const orc_grid* g, double mobility, double gamma);

int orc_heat_residual(const orc_grid* g, const orc_bc* bc, const double* kappa,
                      const double* source, const double* T, double* out);
int orc_elasticity_residual(const orc_grid* g, const orc_bc* bc, const double* modulus,
                            double nu, const double* loads, const double* u, double* out);
double orc_residual_norm(const double* r, int64_t nodes, int comps);

/* property: conductivity (heat) or Young's modulus (elasticity; Lame via make_lame). */
int orc_hybrid_solve(int physics, const orc_grid* g, const orc_bc* bc, const double* property,
                     double nu, const double* source, double* cur, double* prev,
                     const orc_pt_params* p, int64_t* abort_step);
/* hybrid_solve timed alone (operator construction excluded): wall seconds of the
 * solve itself, for the CPU baseline legs of bench.py. */
int orc_time_hybrid(int physics, const orc_grid* g, const orc_bc* bc, const double* property,
                    double nu, const double* source, double* cur, double* prev,
                    const orc_pt_params* p, double* seconds);
int orc_iterate_to_tolerance(int physics, const orc_grid* g, const orc_bc* bc,
                             const double* property, double nu, const double* source,
                             double* cur, double* prev, int mode /*0 PT, 1 APT*/,
                             const orc_pt_params* p, double target, long max_iters,
                             orc_solve_stats* stats);

int orc_interpolate(const orc_grid* g, const orc_material* m, const double* phases,
                    double* out);
int orc_sensitivities(const orc_grid* g, const orc_material* m, const orc_targets* t,
                      const double* phases, const double* state, double* gc, double* gv,
                      double* gu, double* gr);
int orc_design_update(const orc_grid* g, int nphases, const orc_weights* w, double* phases,
                      const double* gc, const double* gv, const double* gu, const double* gr);
int orc_ch_step(const orc_grid* g, const orc_ch_params* p, double* phi, orc_ch_stats* stats);
double orc_phase_mass(const orc_grid* g, const double* phi);
double orc_gl_energy(const orc_grid* g, const double* phi, double gamma);
double orc_separation(const orc_grid* g, int nphases, const double* phases);
int orc_evaluate_objectives(const orc_grid* g, const orc_material* m, const orc_targets* t,
                            const double* phases, const double* state, orc_report* out);

int orc_run(const orc_problem* prob, const orc_schedule* sched, double* phases_out,
            double* state_out, orc_record* records, long records_cap, long* nrecords,
            orc_run_result* result);

/* Output writers (field_io.cpp): write_field_csv (:29-47), write_pgm (:68-101,
 * 2D only, plus "<path>.scale.txt"), write_vtk_structured_points (:103-126) with
 * narrays consecutive N-blocks named names[i].  Errors: 2 invalid argument,
 * 4 IoError (cannot open / write failed). */
int orc_write_field_csv(const orc_grid* g, const double* values, const char* path);
int orc_write_pgm(const orc_grid* g, const double* values, const char* path);
int orc_write_vtk(const orc_grid* g, int narrays, const char* const* names, const double* values,
                  const char* path);

#ifdef __cplusplus
}
#endif

#endif /* PETTO_ORACLE_H */
