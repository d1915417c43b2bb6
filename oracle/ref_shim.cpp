// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference implementation (headers and sources read in
// place from /root/reference/proj, never copied) through the plain-C interface of
// petto_oracle.h, so the parity tests can drive the reference and the C
// restatement (petto_oracle.c) through one ctypes binding.  Built by
// oracle/Makefile into oracle/_ref/libpetto_ref.so with the reference's own
// release flags (g++ -O3 -fopenmp, no -march => no FMA contraction on x86-64).
//
// Every function is a thin marshalling layer: build the reference's Grid /
// BoundarySpec / Field objects from the POD arguments, call the reference entry
// point named in the comment, copy results back.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "petto/config_io.hpp"
#include "petto/errors.hpp"
#include "petto/field_io.hpp"
#include "petto/engine.hpp"
#include "petto/objectives.hpp"
#include "petto/optimizer.hpp"
#include "petto/parallel.hpp"
#include "petto/phase_field.hpp"
#include "petto/state_solver.hpp"

#include "petto_oracle.h"

using namespace petto;

namespace {

thread_local std::string g_err;

Grid make_grid(const orc_grid* g) {
    if (g->dim == 3) return Grid::make3d(g->n[0], g->n[1], g->n[2], g->length[0], g->length[1],
                                         g->length[2]);
    return Grid::make2d(g->n[0], g->n[1], g->length[0], g->length[1]);
}

BoundarySpec make_bc(const orc_bc* b) {
    BoundarySpec bc;
    for (int f = 0; f < 6; ++f)
        bc.face[f] = {static_cast<CondKind>(b->kind[f]), b->value[f], b->component[f]};
    for (int64_t p = 0; p < b->npins; ++p)
        bc.pins.push_back({b->pin_node[p], b->pin_comp[p], b->pin_value[p]});
    return bc;
}

Field<double> field_from(const Grid& g, int comps, const double* src) {
    Field<double> f(g, comps);
    if (src) std::memcpy(f.data.data(), src, sizeof(double) * f.data.size());
    return f;
}

void field_to(const Field<double>& f, double* dst) {
    std::memcpy(dst, f.data.data(), sizeof(double) * f.data.size());
}

PTParams make_params(const orc_pt_params* p) {
    PTParams q;
    q.dt_pt = p->dt_pt;
    q.dt_apt = p->dt_apt;
    q.theta = p->theta;
    q.n_apt = p->n_apt;
    q.n_pt = p->n_pt;
    q.form = p->form ? AptForm::SemiImplicitDamping : AptForm::ExplicitDamping;
    return q;
}

MaterialModel make_material(const orc_material* m) {
    MaterialModel mm;
    mm.kind = m->kind ? MaterialKind::Elastic : MaterialKind::Thermal;
    mm.properties.assign(m->properties, m->properties + m->nphases);
    mm.poisson_ratio = m->poisson_ratio;
    mm.penalty = m->penalty;
    mm.void_floor = m->void_floor;
    return mm;
}

VolumeTargets make_targets(const orc_targets* t, int np) {
    VolumeTargets vt;
    vt.fractions.assign(t->fractions, t->fractions + np);
    if (t->region_fractions) {
        vt.region_nodes.assign(t->region_nodes, t->region_nodes + t->nregion);
        vt.region_fractions.assign(t->region_fractions, t->region_fractions + np);
    }
    return vt;
}

PhaseSet<double> phases_from(const Grid& g, int np, const double* src) {
    PhaseSet<double> ps(g, np, 0.0);
    const Index n = g.num_nodes();
    for (int i = 0; i < np; ++i)
        std::memcpy(ps.phases[i].data.data(), src + i * n, sizeof(double) * n);
    return ps;
}

void phases_to(const PhaseSet<double>& ps, double* dst) {
    const Index n = ps.grid().num_nodes();
    for (int i = 0; i < ps.count(); ++i)
        std::memcpy(dst + i * n, ps.phases[i].data.data(), sizeof(double) * n);
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const NumericalAbort& e) {
        g_err = e.what();
        return 1;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// IoError -> 4 (the CLI's exit code for it, src/engine.cpp:259-268)
template <class F>
int guarded_io(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// Operator bundle owning the fields the reference operators point at.
struct OpBundle {
    Grid grid;
    BoundarySpec bc;
    Field<double> property, source;
    ElasticMaterialField<double> lame;
    std::unique_ptr<StateOperator<double>> op;

    OpBundle(int physics, const orc_grid* g, const orc_bc* b, const double* prop, double nu,
             const double* src)
        : grid(make_grid(g)), bc(make_bc(b)) {
        const int comps = physics ? grid.dim : 1;
        property = field_from(grid, 1, prop);
        source = field_from(grid, comps, src);
        if (physics) {
            lame = make_lame(property, nu);
            op = std::make_unique<ElasticityOperator<double>>(grid, lame, source, bc);
        } else {
            op = std::make_unique<HeatOperator<double>>(grid, property, source, bc);
        }
    }
};

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_impl_name(void) { return "reference"; }
void orc_set_threads(int n) { par::set_threads(n); }
int orc_threads(void) { return par::threads(); }

int64_t orc_num_nodes(const orc_grid* g) { return make_grid(g).num_nodes(); }
double orc_spacing(const orc_grid* g, int axis) { return make_grid(g).spacing[axis]; }
double orc_cell_volume(const orc_grid* g, int64_t i, int64_t j, int64_t k) {
    return make_grid(g).cell_volume(i, j, k);
}

int64_t orc_make_constraints(const orc_grid* g, const orc_bc* b, int comps, int64_t* entry,
                             double* value, int64_t cap) {
    int64_t count = -1;
    const int rc = guarded([&] {
        const Grid grid = make_grid(g);
        const ConstraintSet cs = make_constraints(grid, make_bc(b), comps);
        count = static_cast<int64_t>(cs.size());
        for (int64_t i = 0; i < std::min<int64_t>(count, cap); ++i) {
            entry[i] = cs.entry[i];
            value[i] = cs.value[i];
        }
    });
    return rc ? -1 - rc : count;
}

void orc_unit_cell_stiffness(int dim, const double h[3], double nu, double* ke) {
    const std::vector<double> k = detail::unit_cell_stiffness(dim, {h[0], h[1], h[2]}, nu);
    std::memcpy(ke, k.data(), sizeof(double) * k.size());
}

double orc_elasticity_spectral_bound(const orc_grid* g, double nu, double e_max) {
    return elasticity_spectral_bound(make_grid(g), nu, e_max);
}

double orc_ch_stable_dt(const orc_grid* g, double mobility, double gamma) {
    return ch_stable_dt(make_grid(g), mobility, gamma);
}

int orc_heat_residual(const orc_grid* g, const orc_bc* b, const double* kappa,
                      const double* source, const double* T, double* out) {
    return guarded([&] {
        OpBundle ob(0, g, b, kappa, 0.0, source);
        const Field<double> t = field_from(ob.grid, 1, T);
        Field<double> r(ob.grid, 1);
        ob.op->residual(t, r);
        field_to(r, out);
    });
}

int orc_elasticity_residual(const orc_grid* g, const orc_bc* b, const double* modulus,
                            double nu, const double* loads, const double* u, double* out) {
    return guarded([&] {
        OpBundle ob(1, g, b, modulus, nu, loads);
        const Field<double> uu = field_from(ob.grid, ob.grid.dim, u);
        Field<double> r(ob.grid, ob.grid.dim);
        ob.op->residual(uu, r);
        field_to(r, out);
    });
}

double orc_residual_norm(const double* r, int64_t nodes, int comps) {
    // residual_norm(Field) (state_solver.hpp:50-58) needs a Grid; the same
    // par::sum_nodes reduction is applied to the raw entries here.
    const double sq = par::sum_nodes(nodes * comps, [r](Index i) {
        const double v = r[i];
        return v * v;
    });
    return std::sqrt(sq) / static_cast<double>(nodes);
}

int orc_hybrid_solve(int physics, const orc_grid* g, const orc_bc* b, const double* property,
                     double nu, const double* source, double* cur, double* prev,
                     const orc_pt_params* p, int64_t* abort_step) {
    OpBundle* keep = nullptr;
    int rc = guarded([&] {
        keep = new OpBundle(physics, g, b, property, nu, source);
        const int comps = keep->op->components();
        StateHistory<double> hist(field_from(keep->grid, comps, cur),
                                  field_from(keep->grid, comps, prev));
        try {
            hybrid_solve(hist, *keep->op, make_params(p));
        } catch (const NumericalAbort& e) {
            if (abort_step) *abort_step = e.step();
            field_to(hist.current, cur);
            field_to(hist.previous, prev);
            throw;
        }
        field_to(hist.current, cur);
        field_to(hist.previous, prev);
    });
    delete keep;
    return rc;
}

int orc_time_hybrid(int physics, const orc_grid* g, const orc_bc* b, const double* property, double nu,
                    const double* source, double* cur, double* prev, const orc_pt_params* p, double* seconds) {
    return guarded([&] {
        OpBundle ob(physics, g, b, property, nu, source);
        const int comps = ob.op->components();
        StateHistory<double> hist(field_from(ob.grid, comps, cur), field_from(ob.grid, comps, prev));
        const auto t0 = std::chrono::steady_clock::now();
        hybrid_solve(hist, *ob.op, make_params(p));
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        field_to(hist.current, cur);
        field_to(hist.previous, prev);
    });
}

int orc_iterate_to_tolerance(int physics, const orc_grid* g, const orc_bc* b,
                             const double* property, double nu, const double* source,
                             double* cur, double* prev, int mode, const orc_pt_params* p,
                             double target, long max_iters, orc_solve_stats* stats) {
    return guarded([&] {
        OpBundle ob(physics, g, b, property, nu, source);
        const int comps = ob.op->components();
        StateHistory<double> hist(field_from(ob.grid, comps, cur),
                                  field_from(ob.grid, comps, prev));
        const SolveStats s =
            iterate_to_tolerance(hist, *ob.op, mode ? IterationMode::APT : IterationMode::PT,
                                 make_params(p), target, max_iters);
        stats->iterations = s.iterations;
        stats->r_initial = s.r_initial;
        stats->r_final = s.r_final;
        stats->converged = s.converged ? 1 : 0;
        field_to(hist.current, cur);
        field_to(hist.previous, prev);
    });
}

int orc_interpolate(const orc_grid* g, const orc_material* m, const double* phases,
                    double* out) {
    return guarded([&] {
        const Grid grid = make_grid(g);
        const PhaseSet<double> ps = phases_from(grid, m->nphases, phases);
        field_to(interpolate(ps, make_material(m)), out);
    });
}

int orc_sensitivities(const orc_grid* g, const orc_material* m, const orc_targets* t,
                      const double* phases, const double* state, double* gc, double* gv,
                      double* gu, double* gr) {
    return guarded([&] {
        const Grid grid = make_grid(g);
        const PhaseSet<double> ps = phases_from(grid, m->nphases, phases);
        const int comps = m->kind ? grid.dim : 1;
        const Field<double> st = field_from(grid, comps, state);
        const SensitivityFields<double> s =
            sensitivities(ps, st, make_material(m), make_targets(t, m->nphases));
        const Index n = grid.num_nodes();
        for (int i = 0; i < m->nphases; ++i) {
            field_to(s.compliance[i], gc + i * n);
            field_to(s.volume[i], gv + i * n);
            field_to(s.unity[i], gu + i * n);
            if (gr && !s.region.empty()) field_to(s.region[i], gr + i * n);
        }
    });
}

int orc_design_update(const orc_grid* g, int nphases, const orc_weights* w, double* phases,
                      const double* gc, const double* gv, const double* gu, const double* gr) {
    return guarded([&] {
        const Grid grid = make_grid(g);
        PhaseSet<double> ps = phases_from(grid, nphases, phases);
        const Index n = grid.num_nodes();
        SensitivityFields<double> s;
        for (int i = 0; i < nphases; ++i) {
            s.compliance.push_back(field_from(grid, 1, gc + i * n));
            s.volume.push_back(field_from(grid, 1, gv + i * n));
            s.unity.push_back(field_from(grid, 1, gu + i * n));
            if (gr) s.region.push_back(field_from(grid, 1, gr + i * n));
        }
        ObjectiveWeights ow;
        ow.alpha_compliance = w->alpha_compliance;
        ow.alpha_volume = w->alpha_volume;
        ow.alpha_unity = w->alpha_unity;
        ow.alpha_region = w->alpha_region;
        ow.normalize_compliance = w->normalize_compliance != 0;
        ow.compliance_sign = w->compliance_sign;
        design_update_inplace(ps, s, ow);
        phases_to(ps, phases);
    });
}

int orc_ch_step(const orc_grid* g, const orc_ch_params* p, double* phi, orc_ch_stats* stats) {
    return guarded([&] {
        const Grid grid = make_grid(g);
        Field<double> f = field_from(grid, 1, phi);
        Field<double> mu(grid, 1), lap(grid, 1);
        CahnHilliardParams cp;
        cp.mobility = p->mobility;
        cp.gamma = p->gamma;
        cp.dt = p->dt;
        ChStepStats st;
        ch_step_inplace(f, cp, mu, lap, &st);
        if (stats) {
            stats->mass_before = st.mass_before;
            stats->mass_preclamp = st.mass_preclamp;
            stats->mass_postclamp = st.mass_postclamp;
        }
        field_to(f, phi);
    });
}

double orc_phase_mass(const orc_grid* g, const double* phi) {
    const Grid grid = make_grid(g);
    return phase_mass(field_from(grid, 1, phi));
}

double orc_gl_energy(const orc_grid* g, const double* phi, double gamma) {
    const Grid grid = make_grid(g);
    return gl_energy(field_from(grid, 1, phi), gamma);
}

double orc_separation(const orc_grid* g, int nphases, const double* phases) {
    const Grid grid = make_grid(g);
    return phase_separation_metric(phases_from(grid, nphases, phases));
}

int orc_evaluate_objectives(const orc_grid* g, const orc_material* m, const orc_targets* t,
                            const double* phases, const double* state, orc_report* out) {
    return guarded([&] {
        const Grid grid = make_grid(g);
        const PhaseSet<double> ps = phases_from(grid, m->nphases, phases);
        const int comps = m->kind ? grid.dim : 1;
        const ObjectiveReport r = evaluate_objectives(
            ps, field_from(grid, comps, state), make_material(m), make_targets(t, m->nphases));
        out->compliance = r.compliance;
        out->volume = r.volume;
        out->unity = r.unity;
        out->region = r.region;
        for (std::size_t i = 0; i < r.volume_fractions.size() && i < ORC_MAX_PHASES; ++i)
            out->volume_fractions[i] = r.volume_fractions[i];
    });
}

int orc_run(const orc_problem* pr, const orc_schedule* sc, double* phases_out,
            double* state_out, orc_record* records, long records_cap, long* nrecords,
            orc_run_result* result) {
    return guarded([&] {
        Problem<double> prob;
        prob.grid = std::make_unique<Grid>(make_grid(&pr->grid));
        const Grid& g = *prob.grid;
        const int comps = pr->physics ? g.dim : 1;
        prob.kind = pr->physics ? MaterialKind::Elastic : MaterialKind::Thermal;
        prob.bc = make_bc(&pr->bc);
        prob.material = make_material(&pr->material);
        prob.targets = make_targets(&pr->targets, pr->material.nphases);
        prob.weights.alpha_compliance = pr->weights.alpha_compliance;
        prob.weights.alpha_volume = pr->weights.alpha_volume;
        prob.weights.alpha_unity = pr->weights.alpha_unity;
        prob.weights.alpha_region = pr->weights.alpha_region;
        prob.weights.normalize_compliance = pr->weights.normalize_compliance != 0;
        prob.weights.compliance_sign = pr->weights.compliance_sign;
        prob.source = field_from(g, comps, pr->source);
        prob.initial_phases = phases_from(g, pr->material.nphases, pr->initial_phases);
        prob.initial_state = field_from(g, comps, pr->initial_state);

        LoopSchedule s;
        s.pt = make_params(&sc->pt);
        s.ch.mobility = sc->ch.mobility;
        s.ch.gamma = sc->ch.gamma;
        s.ch.dt = sc->ch.dt;
        s.max_loops = sc->max_loops;
        s.convergence_tol = sc->convergence_tol;
        s.convergence_window = sc->convergence_window;
        s.report_every = sc->report_every;

        const OptimizationResult<double> res = run(prob, s);
        if (phases_out) phases_to(res.phases, phases_out);
        if (state_out) field_to(res.state, state_out);
        long nr = 0;
        for (const HistoryRecord& h : res.history) {
            if (nr < records_cap) {
                orc_record& o = records[nr];
                o.loop = h.loop;
                o.apt_steps = h.apt_steps;
                o.pt_steps = h.pt_steps;
                o.compliance = h.compliance;
                o.volume = h.volume;
                o.unity = h.unity;
                o.region = h.region;
                o.r_pde = h.r_pde;
                o.separation = h.separation;
                for (std::size_t i = 0; i < h.volume_fractions.size() && i < ORC_MAX_PHASES; ++i)
                    o.volume_fractions[i] = h.volume_fractions[i];
            }
            ++nr;
        }
        if (nrecords) *nrecords = nr;
        result->loops = res.loops;
        result->apt_steps = res.apt_steps;
        result->pt_steps = res.pt_steps;
        result->design_updates = res.design_updates;
        result->ch_steps = res.ch_steps;
        result->clamp_mass_drift = res.clamp_mass_drift;
        result->termination = static_cast<int>(res.termination);
        std::snprintf(result->abort_detail, sizeof result->abort_detail, "%s",
                      res.abort_detail.c_str());
    });
}

// ---------------------------------------------------------------------------
// Reference-only extras: problem assembly from the reference's config format
// (config_io.cpp:206-240, engine.hpp:27-97, engine.cpp:39-96), serialised as
// JSON so the Python assembly mirror used by tests/bench can be pinned to it.

static std::string g_json;

static std::string num(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

// parse_config + validate_config of a config text: 0, or 3 with the ConfigError message
int ref_check_config(const char* text) {
    return guarded([&] {
        std::istringstream in(text);
        (void)parse_config(in, "<text>");
    });
}

const char* ref_config_json(const char* text) {
    g_json.clear();
    const int rc = guarded([&] {
        std::istringstream in(text);
        const ProblemConfig cfg = parse_config(in, "<text>");
        const Problem<double> prob = build_problem<double>(cfg);
        const Grid& g = *prob.grid;
        const LoopSchedule s = build_schedule(cfg, g);
        std::ostringstream o;
        o << "{\"dim\": " << g.dim << ", \"n\": [" << g.n[0] << ", " << g.n[1] << ", " << g.n[2]
          << "], \"length\": [" << num(g.length[0]) << ", " << num(g.length[1]) << ", "
          << num(g.length[2]) << "], \"spacing\": [" << num(g.spacing[0]) << ", "
          << num(g.spacing[1]) << ", " << num(g.spacing[2]) << "]";
        o << ", \"physics\": " << (prob.kind == MaterialKind::Elastic ? 1 : 0);
        o << ", \"properties\": [";
        for (std::size_t i = 0; i < prob.material.properties.size(); ++i)
            o << (i ? ", " : "") << num(prob.material.properties[i]);
        o << "], \"poisson_ratio\": " << num(prob.material.poisson_ratio)
          << ", \"penalty\": " << num(prob.material.penalty)
          << ", \"void_floor\": " << num(prob.material.void_floor);
        o << ", \"fractions\": [";
        for (std::size_t i = 0; i < prob.targets.fractions.size(); ++i)
            o << (i ? ", " : "") << num(prob.targets.fractions[i]);
        o << "], \"region_fractions\": [";
        for (std::size_t i = 0; i < prob.targets.region_fractions.size(); ++i)
            o << (i ? ", " : "") << num(prob.targets.region_fractions[i]);
        o << "], \"region_nodes\": [";
        for (std::size_t i = 0; i < prob.targets.region_nodes.size(); ++i)
            o << (i ? ", " : "") << prob.targets.region_nodes[i];
        o << "], \"weights\": {\"alpha_compliance\": " << num(prob.weights.alpha_compliance)
          << ", \"alpha_volume\": " << num(prob.weights.alpha_volume)
          << ", \"alpha_unity\": " << num(prob.weights.alpha_unity)
          << ", \"alpha_region\": " << num(prob.weights.alpha_region)
          << ", \"normalize_compliance\": " << (prob.weights.normalize_compliance ? 1 : 0)
          << ", \"compliance_sign\": " << prob.weights.compliance_sign << "}";
        o << ", \"faces\": [";
        for (int f = 0; f < 6; ++f)
            o << (f ? ", " : "") << "[" << static_cast<int>(prob.bc.face[f].kind) << ", "
              << num(prob.bc.face[f].value) << ", " << prob.bc.face[f].component << "]";
        o << "], \"pins\": [";
        for (std::size_t i = 0; i < prob.bc.pins.size(); ++i)
            o << (i ? ", " : "") << "[" << prob.bc.pins[i].node << ", "
              << prob.bc.pins[i].component << ", " << num(prob.bc.pins[i].value) << "]";
        o << "], \"schedule\": {\"dt_pt\": " << num(s.pt.dt_pt) << ", \"dt_apt\": "
          << num(s.pt.dt_apt) << ", \"theta\": " << num(s.pt.theta)
          << ", \"n_apt\": " << s.pt.n_apt << ", \"n_pt\": " << s.pt.n_pt
          << ", \"form\": " << (s.pt.form == AptForm::SemiImplicitDamping ? 1 : 0)
          << ", \"ch_mobility\": " << num(s.ch.mobility) << ", \"ch_gamma\": "
          << num(s.ch.gamma) << ", \"dt_ch\": " << num(s.ch.dt)
          << ", \"max_loops\": " << s.max_loops << ", \"convergence_tol\": "
          << num(s.convergence_tol) << ", \"convergence_window\": " << s.convergence_window
          << ", \"report_every\": " << s.report_every << "}";
        o << ", \"initial_phase\": " << num(cfg.initial_phase)
          << ", \"initial_state\": " << num(cfg.initial_state);
        // nonzero source entries (sparse for elasticity loads)
        o << ", \"source_value\": " << num(cfg.source);
        o << ", \"source_nonzero\": [";
        bool first = true;
        for (std::size_t e = 0; e < prob.source.data.size(); ++e)
            if (prob.kind == MaterialKind::Elastic && prob.source.data[e] != 0.0) {
                o << (first ? "" : ", ") << "[" << e << ", " << num(prob.source.data[e]) << "]";
                first = false;
            }
        o << "], \"initial_state_constrained\": [";
        first = true;
        for (std::size_t e = 0; e < prob.initial_state.data.size(); ++e)
            if (prob.initial_state.data[e] != cfg.initial_state) {
                o << (first ? "" : ", ") << "[" << e << ", " << num(prob.initial_state.data[e])
                  << "]";
                first = false;
            }
        o << "]}";
        g_json = o.str();
    });
    if (rc) g_json = std::string("{\"error\": ") + std::to_string(rc) + "}";
    return g_json.c_str();
}

int orc_write_field_csv(const orc_grid* g, const double* values, const char* path) {
    return guarded_io([&] {
        const Grid grid = make_grid(g);
        write_field_csv(grid, std::vector<double>(values, values + grid.num_nodes()), path);
    });
}

int orc_write_pgm(const orc_grid* g, const double* values, const char* path) {
    return guarded_io([&] {
        const Grid grid = make_grid(g);
        write_pgm(grid, std::vector<double>(values, values + grid.num_nodes()), path);
    });
}

int orc_write_vtk(const orc_grid* g, int narrays, const char* const* names, const double* values,
                  const char* path) {
    return guarded_io([&] {
        const Grid grid = make_grid(g);
        const Index n = grid.num_nodes();
        std::vector<std::pair<std::string, std::vector<double>>> arrays;
        for (int a = 0; a < narrays; ++a)
            arrays.emplace_back(names[a], std::vector<double>(values + a * n, values + (a + 1) * n));
        write_vtk_structured_points(grid, arrays, path);
    });
}

}  // extern "C"
