// Drop-in check of the C++ shim (include/magfd_b200/simulation.hpp): ONE driver
// body, written against the reference's own API and types (magfd::SimSpec,
// magfd::Backend, Simulation<T>(spec, backend), step(), step(&StepTiming),
// sampleNow(), state().step / state().M.cast<double>(), relax(),
// io::writeTrajectoryCsv), instantiated twice: with the reference's
// magfd::Simulation<T> (sim.hpp:15-72, running on the host) and with
// magfd_b200::Simulation<T> (the B200 engine) — the namespace swap a reference
// driver needs.  Test infrastructure: built by oracle/Makefile (target refapi)
// against /root/reference/proj into oracle/_ref/, run by tests/test_cpp_shim.py.
//
// usage: refapi_driver <32|64> <ref|b200> <outdir>
// prints torque / sample / relax lines and writes <outdir>/<engine>.csv through
// the reference's io::writeTrajectoryCsv.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "magfd/config.hpp"
#include "magfd/io.hpp"
#include "magfd/sim.hpp"
#include "magfd_b200/simulation.hpp"

template <template <class> class Sim, class T>
int drive(const magfd::SimSpec& spec, long steps, const std::string& csv) {
    magfd::Backend backend(spec.backend, spec.threads);
    Sim<T> sim(spec, backend);
    std::vector<magfd::dynamics::TrajectorySample> log;
    for (long i = 0; i < steps; ++i) {
        if (sim.state().step % spec.sampleEvery == 0) log.push_back(sim.sampleNow());
        std::printf("torque %ld %.17g\n", i, sim.step());
    }
    magfd::StepTiming timing;
    std::printf("torque %ld %.17g\n", steps, sim.step(&timing));
    std::printf("timing_positive %d\n", timing.total > 0 ? 1 : 0);
    log.push_back(sim.sampleNow());
    for (const auto& s : log)
        std::printf("sample %ld %.17g %.17g %.17g %.17g %.17g %.17g\n", s.step, s.t, s.m.x, s.m.y, s.m.z,
                    s.energy.total, s.maxTorqueDegPerNs);
    const magfd::VectorField<double> M = sim.state().M.template cast<double>();
    double sx = 0, sy = 0, sz = 0;
    for (std::size_t c = 0; c < M.size(); ++c) {
        sx += M.x[c];
        sy += M.y[c];
        sz += M.z[c];
    }
    std::printf("msum %.17g %.17g %.17g\n", sx, sy, sz);
    magfd::io::writeTrajectoryCsv(csv, log);
    auto res = sim.relax();
    std::printf("relax %d %zu %ld %ld %.17g\n", res.converged ? 1 : 0, res.log.size(), res.log.back().step,
                res.state.step, res.state.M.template cast<double>().x[0]);
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const int prec = std::atoi(argv[1]);
    const std::string engine = argv[2], out = argv[3];
    magfd::SimSpec spec;
    spec.nx = 24; spec.ny = 16; spec.nz = 4;
    spec.dx = spec.dy = 3e-9; spec.dz = 2e-9;
    spec.A = 1.3e-11; spec.Ku = 4e4; spec.Ms = 8e5; spec.alpha = 0.5;
    spec.easyAxis = {0, 0, 1};
    spec.externField = {1e4, -5e3, 0};
    spec.initKind = magfd::InitKind::vortex;
    spec.vortexAxis = magfd::SignedAxis::zPlus;
    spec.dt = 2e-14;
    spec.maxSteps = 400;
    spec.torqueTol = 300.0;
    spec.sampleEvery = 4;
    spec.backend = magfd::BackendKind::serial;
    spec.precision = prec == 32 ? magfd::Precision::f32 : magfd::Precision::f64;
    const std::string csv = out + "/" + engine + ".csv";
    try {
        if (engine == "ref")
            return prec == 32 ? drive<magfd::Simulation, float>(spec, 10, csv) : drive<magfd::Simulation, double>(spec, 10, csv);
        return prec == 32 ? drive<magfd_b200::Simulation, float>(spec, 10, csv)
                          : drive<magfd_b200::Simulation, double>(spec, 10, csv);
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
}
