// test_dropin.cpp -- the reference's own C++ API with the B200 drop-in.
//
// Built against the reference headers/sources (tests/cpp/Makefile); the same
// problem goes through petto::run (CPU reference) and petto::dev::run (B200), and
// through hybrid_solve / iterate_to_tolerance with the reference's operator types.
// Prints one line per check and exits non-zero on failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <sstream>
#include <string>

#include "petto/config_io.hpp"
#include "petto/engine.hpp"
#include "petto/parallel.hpp"
#include "petto_dev.hpp"

using namespace petto;

static int failures = 0;

static void expect(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

static double rel(double a, double b) { return std::abs(a - b) / std::max(std::abs(b), 1e-300); }

static ProblemConfig cfg_of(const char* text) {
    std::istringstream in(text);
    return parse_config(in, "<test>");
}

int main() {
    par::set_threads(1);
    // 1. run() on a small cantilever3d (replica mode must track the reference closely)
    const char* c4 =
        "preset = cantilever3d\nnx = 24\nny = 10\nnz = 10\nlength_x = 2\nlength_y = 1\nlength_z = 1\n"
        "properties = 1, 1e-6\ntarget_fractions = 0.3, 0.7\nload_count = 1\nload_0_box = 0,0,0.5,0,1,0.5\n"
        "load_0_direction = 0,0,1\nload_0_magnitude = 1\nmax_loops = 3\nreport_every = 1\nn_apt = 40\nn_pt = 40\n";
    for (int mode : {PETTO_MODE_REPLICA, PETTO_MODE_FAST}) {
        const ProblemConfig cfg = cfg_of(c4);
        const Problem<double> prob = build_problem<double>(cfg);
        const LoopSchedule sched = build_schedule(cfg, *prob.grid);
        const OptimizationResult<double> a = run(prob, sched);
        const OptimizationResult<double> b = dev::run(prob, sched, {}, mode);
        bool ok = a.history.size() == b.history.size() && a.loops == b.loops;
        double worst = 0.0;
        for (size_t i = 0; ok && i < a.history.size(); ++i) {
            worst = std::max(worst, rel(b.history[i].compliance, a.history[i].compliance));
            worst = std::max(worst, rel(b.history[i].volume_fractions[0], a.history[i].volume_fractions[0]));
        }
        char buf[160];
        std::snprintf(buf, sizeof buf, "dev::run %s vs run: worst rel diff %.3e", mode ? "replica" : "fast", worst);
        expect(ok && worst < (mode ? 1e-12 : 1e-9), buf);
    }
    // 2. hybrid_solve with the reference's ElasticityOperator inputs (Lame fields)
    {
        const Grid g = Grid::make3d(20, 9, 8, 2.0, 1.0, 0.8);
        BoundarySpec bc;
        for (int f = 0; f < 6; ++f) bc.face[f] = {CondKind::TractionFree, 0.0, 0};
        bc.face[XHi] = {CondKind::Dirichlet, 0.0, 0};
        Field<double> E(g, 1);
        for (Index i = 0; i < g.num_nodes(); ++i) E.data[i] = 0.2 + 0.8 * std::fmod(0.37 * i, 1.0);
        const ElasticMaterialField<double> lame = make_lame(E, 0.3);
        Field<double> loads(g, 3, 0.0);
        loads.at(2, g.node(0, 4, 4)) = -1.0;
        PTParams p;
        p.dt_pt = g.min_spacing() * g.min_spacing() / 8;
        p.dt_apt = 0.1 * g.min_spacing();
        p.n_apt = 30;
        p.n_pt = 10;
        p.form = AptForm::SemiImplicitDamping;
        const ElasticityOperator<double> ref_op(g, lame, loads, bc);
        StateHistory<double> h1(Field<double>(g, 3, 0.0));
        hybrid_solve(h1, ref_op, p);
        const dev::ElasticityOperator dev_op(g, lame, loads, bc, PETTO_MODE_REPLICA);
        StateHistory<double> h2(Field<double>(g, 3, 0.0));
        dev::hybrid_solve(h2, dev_op, p);
        expect(h1.current.data == h2.current.data && h1.previous.data == h2.previous.data,
               "dev::hybrid_solve (replica, Lame input) bit-identical to hybrid_solve");
        Field<double> r1(g, 3), r2(g, 3);
        ref_op.residual(h1.current, r1);
        dev_op.residual(h1.current, r2);
        expect(r1.data == r2.data, "DeviceOperator::residual bit-identical to ElasticityOperator::residual");
    }
    // 2b. the operators alias the caller's Lame fields, as run() relies on
    // (optimizer.hpp:187-190): update_lame in place between two solves
    {
        const Grid g = Grid::make3d(20, 9, 8, 2.0, 1.0, 0.8);
        BoundarySpec bc;
        for (int f = 0; f < 6; ++f) bc.face[f] = {CondKind::TractionFree, 0.0, 0};
        bc.face[XHi] = {CondKind::Dirichlet, 0.0, 0};
        Field<double> E(g, 1);
        for (Index i = 0; i < g.num_nodes(); ++i) E.data[i] = 0.2 + 0.8 * std::fmod(0.37 * i, 1.0);
        ElasticMaterialField<double> lame_ref = make_lame(E, 0.3), lame_dev = make_lame(E, 0.3);
        Field<double> loads(g, 3, 0.0);
        loads.at(2, g.node(0, 4, 4)) = -1.0;
        PTParams p;
        p.dt_pt = g.min_spacing() * g.min_spacing() / 8;
        p.dt_apt = 0.1 * g.min_spacing();
        p.n_apt = 20;
        p.n_pt = 5;
        p.form = AptForm::SemiImplicitDamping;
        const ElasticityOperator<double> ref_op(g, lame_ref, loads, bc);
        const dev::ElasticityOperator dev_op(g, lame_dev, loads, bc, PETTO_MODE_REPLICA);
        StateHistory<double> h1(Field<double>(g, 3, 0.0)), h2(Field<double>(g, 3, 0.0));
        for (int loop = 0; loop < 3; ++loop) {
            for (Index i = 0; i < g.num_nodes(); ++i) E.data[i] = 0.1 + 0.9 * std::fmod(0.53 * i + 0.17 * loop, 1.0);
            update_lame(E, 0.3, lame_ref);
            update_lame(E, 0.3, lame_dev);
            hybrid_solve(h1, ref_op, p);
            dev::hybrid_solve(h2, dev_op, p);
        }
        expect(h1.current.data == h2.current.data && h1.previous.data == h2.previous.data,
               "dev::hybrid_solve sees in-place update_lame between solves (aliased material, replica)");
    }
    // 3. iterate_to_tolerance on the criterion-1 Poisson box (n = 32)
    {
        const Grid g = Grid::make2d(32, 32, 1.0, 1.0);
        BoundarySpec bc;
        for (int f = 0; f < 4; ++f) bc.face[f] = {CondKind::Dirichlet, 0.0, 0};
        Field<double> kappa(g, 1, 1.0), src(g, 1);
        for (Index j = 0; j < g.n[1]; ++j)
            for (Index i = 0; i < g.n[0]; ++i)
                src.at(0, g.node(i, j)) = std::sin(M_PI * g.coord(0, i)) * std::sin(M_PI * g.coord(1, j));
        const HeatOperator<double> ref_op(g, kappa, src, bc);
        PTParams p;
        p.dt_pt = g.min_spacing() * g.min_spacing() / 4;
        p.dt_apt = g.min_spacing() / 2;
        Field<double> r0(g, 1);
        ref_op.residual(Field<double>(g, 1, 0.0), r0);
        const double target = 1e-8 * residual_norm(r0);
        StateHistory<double> h1(Field<double>(g, 1, 0.0));
        const SolveStats s1 = iterate_to_tolerance(h1, ref_op, IterationMode::APT, p, target, 100000);
        for (int mode : {PETTO_MODE_REPLICA, PETTO_MODE_FAST}) {
            const dev::HeatOperator dev_op(g, kappa, src, bc, mode);
            StateHistory<double> h2(Field<double>(g, 1, 0.0));
            const SolveStats s2 = dev::iterate_to_tolerance(h2, dev_op, IterationMode::APT, p, target, 100000);
            char buf[160];
            std::snprintf(buf, sizeof buf, "dev::iterate_to_tolerance %s: %ld vs %ld iterations",
                          mode ? "replica" : "fast", s2.iterations, s1.iterations);
            expect(mode ? s2.iterations == s1.iterations && h2.current.data == h1.current.data
                        : std::labs(s2.iterations - s1.iterations) <= 1,
                   buf);
        }
    }
    // 4. error behaviour: reckless dt -> NumericalAbort at the first check
    {
        const Grid g = Grid::make2d(16, 16, 1.0, 1.0);
        BoundarySpec bc;
        for (int f = 0; f < 4; ++f) bc.face[f] = {CondKind::Dirichlet, 0.0, 0};
        Field<double> kappa(g, 1, 1.0), f(g, 1, 1.0);
        const dev::HeatOperator op(g, kappa, f, bc);
        PTParams p;
        p.dt_pt = 1e6;
        p.dt_apt = 0.1;
        p.n_pt = 5000;
        StateHistory<double> h(Field<double>(g, 1, 0.0));
        bool caught = false;
        try {
            dev::hybrid_solve(h, op, p);
        } catch (const NumericalAbort& e) {
            caught = e.step() == 100 && e.field() == "state";
        }
        expect(caught, "dev::hybrid_solve raises NumericalAbort(state, 100)");
    }
    // 4. write_outputs: the reference's files and the device writers' files for the
    //    same result are byte-identical (2D: CSV + PGM per field; 3D: fields.vtk)
    {
        namespace fs = std::filesystem;
        char tmpl[] = "/tmp/petto_dropin_XXXXXX";
        const fs::path root = mkdtemp(tmpl);
        auto slurp = [](const fs::path& p) {
            std::ifstream in(p, std::ios::binary);
            return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        };
        const char* cases[] = {
            "preset = mbb2d\nnx = 40\nny = 16\nproperties = 1, 0.55, 1e-6\ntarget_fractions = 0.2, 0.2, 0.6\n"
            "max_loops = 2\nn_apt = 20\nn_pt = 20\n",
            "preset = heat2d\nnx = 33\nny = 29\nmax_loops = 2\nn_apt = 30\nn_pt = 30\n",
            "preset = cantilever3d\nnx = 20\nny = 9\nnz = 7\nlength_x = 2\nlength_y = 1\nlength_z = 1\n"
            "properties = 1, 1e-6\ntarget_fractions = 0.3, 0.7\nmax_loops = 2\nn_apt = 20\nn_pt = 20\n"};
        int k = 0;
        for (const char* text : cases) {
            ProblemConfig cfg = cfg_of(text);
            const Problem<double> prob = build_problem<double>(cfg);
            const OptimizationResult<double> res = run(prob, build_schedule(cfg, *prob.grid));
            const fs::path a = root / ("ref" + std::to_string(k)), b = root / ("dev" + std::to_string(k));
            cfg.out_dir = a.string();
            write_outputs(cfg, prob, res);
            cfg.out_dir = b.string();
            dev::write_outputs(cfg, prob, res);
            int files = 0, same = 0;
            for (const auto& e : fs::directory_iterator(a)) {
                ++files;
                if (slurp(e.path()) == slurp(b / e.path().filename())) ++same;
                else std::printf("  differs: %s\n", e.path().filename().c_str());
            }
            char buf[160];
            std::snprintf(buf, sizeof buf, "dev::write_outputs vs write_outputs (%s): %d/%d files identical",
                          cfg.preset.c_str(), same, files);
            expect(files > 2 && same == files, buf);
            ++k;
        }
        fs::remove_all(root);
    }
    std::printf("%s\n", failures ? "FAILED" : "ALL PASSED");
    return failures ? 1 : 0;
}
