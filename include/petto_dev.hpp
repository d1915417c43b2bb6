// petto_dev.hpp -- C++ drop-in for the reference's state-solver seam.
//
// Include AFTER the reference's headers (it is written against the reference's own
// types: petto::Grid, Field<double>, BoundarySpec, StateOperator<double>,
// StateHistory<double>, PTParams, Problem<double>, LoopSchedule,
// OptimizationResult<double>).  Everything here is a thin, header-only layer over the
// POD C-ABI in petto_dev.h; link with libpetto_b200.so.
//
//   reference (state_solver.hpp / optimizer.hpp)      drop-in (this header)
//   ElasticityOperator<double>(g, lame, loads, bc)    dev::ElasticityOperator(g, lame, loads, bc)
//   HeatOperator<double>(g, kappa, source, bc)        dev::HeatOperator(g, kappa, source, bc)
//   hybrid_solve(hist, op, params)                     dev::hybrid_solve(hist, op, params)
//   iterate_to_tolerance(hist, op, mode, p, tgt, n)    dev::iterate_to_tolerance(...)
//   run(prob, sched, cb)                               dev::run(prob, sched, cb)
//   write_outputs(cfg, prob, result)                   dev::write_outputs(cfg, prob, result)
//
// Errors come back as the reference's exception types: NumericalAbort (with the
// step index), std::invalid_argument, and std::runtime_error for device failures.
#pragma once

#include <filesystem>
#include <fstream>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "petto/engine.hpp"
#include "petto/errors.hpp"
#include "petto/field_io.hpp"
#include "petto/optimizer.hpp"
#include "petto_dev.h"

namespace petto::dev {

inline void check(petto_ctx* ctx, int rc, long long step = -1) {
    if (rc == PETTO_OK) return;
    const std::string msg = petto_dev_last_error(ctx);
    if (rc == PETTO_ABORT) {
        // message is "numerical abort in 'F' at step S: detail": rebuild the same exception
        const auto a = msg.find("'"), b = msg.find("'", a + 1), c = msg.find(": ", b);
        const std::string field = a != std::string::npos ? msg.substr(a + 1, b - a - 1) : "state";
        const std::string detail = c != std::string::npos ? msg.substr(c + 2) : msg;
        throw NumericalAbort(field, step, detail);
    }
    if (rc == PETTO_INVALID) throw std::invalid_argument(msg);
    if (rc == PETTO_IO) throw IoError(msg);
    throw std::runtime_error(msg);
}

// One problem resident in HBM.
class Context {
public:
    Context(const Grid& g, int physics, double nu, int mode = PETTO_MODE_FAST, int device = 0,
            bool x_outermost = false) {
        petto_grid_desc d{};
        d.dim = g.dim;
        for (int a = 0; a < 3; ++a) {
            d.n[a] = g.n[a];
            d.length[a] = g.length[a];
        }
        d.physics = physics;
        d.poisson_ratio = nu;
        d.mode = mode;
        d.device = device;
        d.x_outermost = x_outermost ? 1 : 0;
        check(nullptr, petto_dev_create(&d, &ctx_));
    }
    // The device layout run() picks: x outermost for a FAST 3D elasticity grid whose
    // longest axis is x (the cantilever configs; measured faster)
    static bool prefer_x_outermost(const Grid& g, int physics, int mode) {
        return g.dim == 3 && physics == 1 && mode == PETTO_MODE_FAST && g.n[0] >= g.n[1] && g.n[0] >= g.n[2];
    }
    ~Context() { petto_dev_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    petto_ctx* get() const { return ctx_; }

private:
    petto_ctx* ctx_ = nullptr;
};

// A StateOperator whose residual runs on the B200.  residual() is the host-buffer
// path (upload, evaluate, download); the solvers below keep the state resident.
//
// Like the reference operators (state_solver.hpp:91-94, 318-324), a DeviceOperator
// aliases the caller's material field (kappa, or the Lame pair): the field must
// outlive the operator, and every residual / hybrid_solve / iterate_to_tolerance
// re-reads it, so a loop that updates the field in place between solves
// (interpolate_into + update_lame, optimizer.hpp:187-189) is seen by the device.
// The loads / source are read once, at construction (run() never changes them);
// call refresh_loads() after changing them in place.  set_static_material(true)
// skips the per-call material upload when the caller knows the field is fixed.
class DeviceOperator : public StateOperator<double> {
public:
    int components() const override { return comps_; }
    const ConstraintSet& constraints() const override { return cs_; }
    void residual(const Field<double>& state, Field<double>& out) const override {
        petto_ctx* c = ctx_->get();
        refresh();
        check(c, petto_dev_set_state(c, state.data.data(), state.data.data()));
        double r = 0.0;
        check(c, petto_dev_residual(c, out.data.data(), &r));
    }
    petto_ctx* ctx() const { return ctx_->get(); }
    // upload the aliased material field again (no-op with a static material)
    void refresh() const {
        if (!static_material_ && upload_material_) upload_material_();
    }
    void refresh_loads() const {
        if (upload_loads_) upload_loads_();
    }
    void set_static_material(bool on) { static_material_ = on; }

protected:
    DeviceOperator(const Grid& g, int physics, double nu, const BoundarySpec& bc, int mode)
        : ctx_(std::make_unique<Context>(g, physics, nu, mode)),
          comps_(physics ? g.dim : 1),
          cs_(make_constraints(g, bc, comps_)) {
        check(ctx(), petto_dev_set_constraints(ctx(), cs_.entry.data(), cs_.value.data(),
                                               static_cast<int64_t>(cs_.size())));
    }
    std::unique_ptr<Context> ctx_;
    int comps_;
    ConstraintSet cs_;
    std::function<void()> upload_material_, upload_loads_;
    bool static_material_ = false;
};

// HeatOperator (state_solver.hpp:76-95)
class HeatOperator final : public DeviceOperator {
public:
    HeatOperator(const Grid& g, const Field<double>& kappa, const Field<double>& source, const BoundarySpec& bc,
                 int mode = PETTO_MODE_FAST)
        : DeviceOperator(g, 0, 0.3, bc, mode) {
        const Field<double>* k = &kappa;
        const Field<double>* f = &source;
        upload_material_ = [this, k] { check(ctx(), petto_dev_set_property(ctx(), k->data.data())); };
        upload_loads_ = [this, f] { check(ctx(), petto_dev_set_source(ctx(), f->data.data())); };
        upload_loads_();
        upload_material_();
        check(ctx(), petto_dev_init_operator(ctx()));
    }
};

// ElasticityOperator (state_solver.hpp:289-325)
class ElasticityOperator final : public DeviceOperator {
public:
    ElasticityOperator(const Grid& g, const ElasticMaterialField<double>& mat, const Field<double>& loads,
                       const BoundarySpec& bc, int mode = PETTO_MODE_FAST)
        : DeviceOperator(g, 1, nu_of(mat), bc, mode) {
        const ElasticMaterialField<double>* m = &mat;
        const Field<double>* f = &loads;
        upload_material_ = [this, m] {
            check(ctx(), petto_dev_set_lame(ctx(), m->lambda.data.data(), m->mu.data.data()));
        };
        upload_loads_ = [this, f] { check(ctx(), petto_dev_set_source(ctx(), f->data.data())); };
        upload_loads_();
        upload_material_();
        check(ctx(), petto_dev_init_operator(ctx()));
    }

private:
    static double nu_of(const ElasticMaterialField<double>& m) {
        const double l0 = m.lambda.data.at(0), m0 = m.mu.data.at(0);
        return l0 / (2.0 * (l0 + m0));
    }
};

inline petto_pt_params params(const PTParams& p) {
    return {p.dt_pt, p.dt_apt, p.theta, p.n_apt, p.n_pt, p.form == AptForm::SemiImplicitDamping ? 1 : 0};
}

// hybrid_solve (state_solver.hpp:480-498)
inline void hybrid_solve(StateHistory<double>& hist, const DeviceOperator& op, const PTParams& p) {
    petto_ctx* c = op.ctx();
    op.refresh();
    check(c, petto_dev_set_state(c, hist.current.data.data(), hist.previous.data.data()));
    const petto_pt_params pp = params(p);
    int64_t step = 0;
    const int rc = petto_dev_hybrid_solve(c, &pp, &step);
    check(c, petto_dev_get_state(c, hist.current.data.data(), hist.previous.data.data()));
    check(c, rc, step);
}

// iterate_to_tolerance (state_solver.hpp:511-541)
inline SolveStats iterate_to_tolerance(StateHistory<double>& hist, const DeviceOperator& op, IterationMode mode,
                                       const PTParams& p, double target, long max_iters) {
    petto_ctx* c = op.ctx();
    op.refresh();
    check(c, petto_dev_set_state(c, hist.current.data.data(), hist.previous.data.data()));
    const petto_pt_params pp = params(p);
    petto_solve_stats st{};
    const int rc = petto_dev_iterate_to_tolerance(c, mode == IterationMode::APT ? 1 : 0, &pp, target, max_iters, &st);
    check(c, petto_dev_get_state(c, hist.current.data.data(), hist.previous.data.data()));
    check(c, rc, st.iterations);
    SolveStats out;
    out.iterations = st.iterations;
    out.r_initial = st.r_initial;
    out.r_final = st.r_final;
    out.converged = st.converged != 0;
    return out;
}

// run() (optimizer.hpp:120-223) with the whole loop resident on the device.
inline OptimizationResult<double> run(const Problem<double>& prob, const LoopSchedule& sched,
                                      const RecordCallback& on_record = {}, int mode = PETTO_MODE_FAST) {
    sched.validate();
    prob.weights.validate();
    const Grid& g = *prob.grid;
    const int physics = prob.kind == MaterialKind::Elastic ? 1 : 0;
    const int comps = physics ? g.dim : 1;
    Context cx(g, physics, prob.material.poisson_ratio, mode, 0, Context::prefer_x_outermost(g, physics, mode));
    petto_ctx* c = cx.get();
    const ConstraintSet cs = make_constraints(g, prob.bc, comps);
    check(c, petto_dev_set_constraints(c, cs.entry.data(), cs.value.data(), static_cast<int64_t>(cs.size())));
    check(c, petto_dev_set_source(c, prob.source.data.data()));
    petto_material m{};
    m.kind = physics;
    m.nphases = static_cast<int>(prob.material.properties.size());
    if (m.nphases > PETTO_MAX_PHASES) throw std::invalid_argument("petto_dev: at most 8 phases");
    for (int i = 0; i < m.nphases; ++i) m.properties[i] = prob.material.properties[i];
    m.poisson_ratio = prob.material.poisson_ratio;
    m.penalty = prob.material.penalty;
    m.void_floor = prob.material.void_floor;
    petto_targets t{};
    for (int i = 0; i < m.nphases; ++i) t.fractions[i] = prob.targets.fractions.at(i);
    t.has_region = prob.targets.has_region() ? 1 : 0;
    for (int i = 0; t.has_region && i < m.nphases; ++i) t.region_fractions[i] = prob.targets.region_fractions[i];
    t.nregion = static_cast<int64_t>(prob.targets.region_nodes.size());
    t.region_nodes = prob.targets.region_nodes.data();
    const petto_weights w{prob.weights.alpha_compliance, prob.weights.alpha_volume, prob.weights.alpha_unity,
                          prob.weights.alpha_region, prob.weights.normalize_compliance ? 1 : 0,
                          prob.weights.compliance_sign};
    check(c, petto_dev_set_design(c, &m, &t, &w));
    const Index N = g.num_nodes();
    std::vector<double> phases(static_cast<size_t>(N) * m.nphases);
    for (int i = 0; i < m.nphases; ++i)
        std::copy(prob.initial_phases.phases[i].data.begin(), prob.initial_phases.phases[i].data.end(),
                  phases.begin() + static_cast<size_t>(i) * N);
    check(c, petto_dev_set_phases(c, phases.data()));
    check(c, petto_dev_set_state(c, prob.initial_state.data.data(), prob.initial_state.data.data()));

    OptimizationResult<double> result;
    struct Sink {
        OptimizationResult<double>* res;
        const RecordCallback* cb;
        int np;
    } sink{&result, &on_record, m.nphases};
    auto trampoline = [](const petto_record* r, void* user) {
        auto* s = static_cast<Sink*>(user);
        HistoryRecord h;
        h.loop = r->loop;
        h.apt_steps = r->apt_steps;
        h.pt_steps = r->pt_steps;
        h.compliance = r->compliance;
        h.volume = r->volume;
        h.unity = r->unity;
        h.region = r->region;
        h.r_pde = r->r_pde;
        h.separation = r->separation;
        h.volume_fractions.assign(r->volume_fractions, r->volume_fractions + s->np);
        h.wall_seconds = r->wall_seconds;
        s->res->history.push_back(h);
        if (*s->cb) (*s->cb)(h);
    };
    const petto_schedule s{params(sched.pt), {sched.ch.mobility, sched.ch.gamma, sched.ch.dt}, sched.max_loops,
                           sched.convergence_tol, sched.convergence_window, sched.report_every};
    petto_run_result rr{};
    check(c, petto_dev_run(c, &s, trampoline, &sink, &rr));
    result.loops = rr.loops;
    result.apt_steps = rr.apt_steps;
    result.pt_steps = rr.pt_steps;
    result.design_updates = rr.design_updates;
    result.ch_steps = rr.ch_steps;
    result.clamp_mass_drift = rr.clamp_mass_drift;
    result.termination = rr.termination == 0   ? Termination::Converged
                         : rr.termination == 2 ? Termination::AbortedNaN
                                               : Termination::MaxLoops;
    result.abort_detail = rr.abort_detail;
    check(c, petto_dev_get_phases(c, phases.data()));
    result.phases = PhaseSet<double>(g, m.nphases, 0.0);
    for (int i = 0; i < m.nphases; ++i)
        std::copy(phases.begin() + static_cast<size_t>(i) * N, phases.begin() + static_cast<size_t>(i + 1) * N,
                  result.phases.phases[i].data.begin());
    result.state = Field<double>(g, comps);
    std::vector<double> prev(result.state.data.size());
    check(c, petto_dev_get_state(c, result.state.data.data(), prev.data()));
    return result;
}

// write_outputs (engine.cpp:145-217) with the field files formatted on the device
// (petto_dev_write_field_csv / _pgm / _vtk): the result's phases and state are
// uploaded once, the property is interpolated on the device, and every field file
// is byte-identical to the reference's.  history.csv and summary.txt are a few
// lines of host text, written as the reference writes them.
inline void write_outputs(const ProblemConfig& cfg, const Problem<double>& prob,
                          const OptimizationResult<double>& result, int device = 0) {
    namespace fs = std::filesystem;
    const fs::path dir(cfg.out_dir);
    std::error_code ec;
    fs::create_directories(dir, ec);
    if (ec) throw IoError("cannot create output directory '" + cfg.out_dir + "'");
    auto path = [&](const std::string& name) { return (dir / name).string(); };
    auto wants = [&](const char* f) {
        for (const std::string& x : cfg.formats)
            if (x == f) return true;
        return false;
    };
    const Grid& g = *prob.grid;
    write_history_csv(result.history, path("history.csv"));

    const bool thermal = prob.kind == MaterialKind::Thermal;
    Context cx(g, thermal ? 0 : 1, prob.material.poisson_ratio, PETTO_MODE_FAST, device);
    petto_ctx* c = cx.get();
    petto_material m{};
    m.kind = thermal ? 0 : 1;
    m.nphases = result.phases.count();
    if (m.nphases > PETTO_MAX_PHASES) throw std::invalid_argument("petto_dev: at most 8 phases");
    for (int i = 0; i < m.nphases; ++i) m.properties[i] = prob.material.properties[i];
    m.poisson_ratio = prob.material.poisson_ratio;
    m.penalty = prob.material.penalty;
    m.void_floor = prob.material.void_floor;
    petto_targets t{};
    for (int i = 0; i < m.nphases; ++i) t.fractions[i] = prob.targets.fractions.at(i);
    const petto_weights w{1.0, 0.0, 0.0, 0.0, 0, -1};
    check(c, petto_dev_set_design(c, &m, &t, &w));
    const Index N = g.num_nodes();
    std::vector<double> buf(static_cast<size_t>(N) * m.nphases);
    for (int i = 0; i < m.nphases; ++i)
        std::copy(result.phases.phases[i].data.begin(), result.phases.phases[i].data.end(),
                  buf.begin() + static_cast<size_t>(i) * N);
    check(c, petto_dev_set_phases(c, buf.data()));
    check(c, petto_dev_interpolate(c, nullptr));  // interpolate(result.phases, prob.material)
    check(c, petto_dev_set_state(c, result.state.data.data(), result.state.data.data()));
    const char* prop_name = thermal ? "conductivity" : "modulus";

    if (g.dim == 2) {
        for (int i = 0; i < m.nphases; ++i) {
            const std::string base = "phase_" + std::to_string(i);
            if (wants("csv")) check(c, petto_dev_write_field_csv(c, PETTO_FIELD_PHASE, i, path(base + ".csv").c_str()));
            if (wants("pgm")) check(c, petto_dev_write_pgm(c, PETTO_FIELD_PHASE, i, path(base + ".pgm").c_str()));
        }
        const std::string pn(prop_name);
        if (wants("csv")) check(c, petto_dev_write_field_csv(c, PETTO_FIELD_PROPERTY, 0, path(pn + ".csv").c_str()));
        if (wants("pgm")) check(c, petto_dev_write_pgm(c, PETTO_FIELD_PROPERTY, 0, path(pn + ".pgm").c_str()));
        if (thermal) {
            check(c, petto_dev_write_field_csv(c, PETTO_FIELD_STATE, 0, path("temperature.csv").c_str()));
        } else {
            for (int k = 0; k < g.dim; ++k)
                check(c, petto_dev_write_field_csv(c, PETTO_FIELD_STATE, k,
                                                   path("displacement_" + component_name(k) + ".csv").c_str()));
        }
    } else {
        std::vector<std::string> names;
        std::vector<petto_array> arrays;
        for (int i = 0; i < m.nphases; ++i) names.push_back("phase_" + std::to_string(i));
        names.push_back(prop_name);
        for (int k = 0; k < result.state.components; ++k) names.push_back("displacement_" + component_name(k));
        for (int i = 0; i < m.nphases; ++i) arrays.push_back({PETTO_FIELD_PHASE, i, nullptr});
        arrays.push_back({PETTO_FIELD_PROPERTY, 0, nullptr});
        for (int k = 0; k < result.state.components; ++k) arrays.push_back({PETTO_FIELD_STATE, k, nullptr});
        for (size_t a = 0; a < arrays.size(); ++a) arrays[a].name = names[a].c_str();
        check(c, petto_dev_write_vtk(c, arrays.data(), static_cast<int>(arrays.size()), path("fields.vtk").c_str()));
    }

    std::ofstream sum(path("summary.txt"));
    if (!sum) throw IoError("cannot write run summary");
    sum << "preset = " << (cfg.preset.empty() ? "(custom)" : cfg.preset) << "\n";
    sum << "termination = " << to_string(result.termination) << "\n";
    if (!result.abort_detail.empty()) sum << "abort_detail = " << result.abort_detail << "\n";
    sum << "loops = " << result.loops << "\n";
    sum << "apt_steps = " << result.apt_steps << "\n";
    sum << "pt_steps = " << result.pt_steps << "\n";
    sum << "design_updates = " << result.design_updates << "\n";
    sum << "ch_steps = " << result.ch_steps << "\n";
    sum << "clamp_mass_drift = " << result.clamp_mass_drift << "\n";
    const LoopSchedule sched = build_schedule(cfg, g);
    sum << "dt_pt = " << sched.pt.dt_pt << "\n";
    sum << "dt_apt = " << sched.pt.dt_apt << "\n";
    sum << "dt_ch = " << sched.ch.dt << "\n";
    const ObjectiveWeights ew = effective_weights(cfg, g);
    sum << "alpha_volume_effective = " << ew.alpha_volume << "\n";
    sum << "alpha_unity_effective = " << ew.alpha_unity << "\n";
    sum << "alpha_region_effective = " << ew.alpha_region << "\n";
    if (!result.history.empty()) {
        const HistoryRecord& r = result.history.back();
        sum << "final_compliance = " << r.compliance << "\n";
        sum << "final_r_pde = " << r.r_pde << "\n";
        sum << "final_separation = " << r.separation << "\n";
        for (std::size_t i = 0; i < r.volume_fractions.size(); ++i)
            sum << "final_volfrac_" << i << " = " << r.volume_fractions[i] << "\n";
        sum << "wall_seconds = " << r.wall_seconds << "\n";
    }
}

}  // namespace petto::dev
