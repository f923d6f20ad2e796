// A driver written the way the reference's drivers use magfd::Simulation<T>
// (cli.cpp:63-67 runImpl, acceptance.cpp), compiled against the B200 shim.
// Prints: torque of each step, final <m>, relax result; used by
// tests/test_gpu_cpp_shim.py, which compares against the oracle.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "magfd_b200/simulation.hpp"

int main(int argc, char** argv) {
    const int prec = argc > 1 ? std::atoi(argv[1]) : 64;
    mfd_grid g{16, 8, 4, 3e-9, 3e-9, 3e-9};
    mfd_material m{1.3e-11, 4e4, 8e5, 0.5, 1.760859630e11, {0, 0, 1}};
    mfd_terms t{1, 1, 1, 1, {1e4, 0, 0}};
    mfd_stepper s{1e-14, 1, 300, 500.0, 100};
    const double dir[3] = {1 / std::sqrt(3.0), 1 / std::sqrt(3.0), 1 / std::sqrt(3.0)};
    auto run = [&](auto tag) {
        using T = decltype(tag);
        magfd_b200::Simulation<T> sim(g, m, t, s);
        sim.set_uniform(dir);
        for (int i = 0; i < 3; ++i) std::printf("torque %.17g\n", sim.step());
        auto smp = sim.sample_now();
        std::printf("m %.17g %.17g %.17g\n", smp.m[0], smp.m[1], smp.m[2]);
        auto r = sim.relax();
        std::printf("relax %d %zu %ld\n", r.converged ? 1 : 0, r.log.size(), r.log.empty() ? -1L : r.log.back().step);
        try {
            mfd_grid bad{0, 1, 1, 1e-9, 1e-9, 1e-9};
            magfd_b200::Simulation<T> b(bad, m, t, s);
        } catch (const std::invalid_argument& e) {
            std::printf("invalid_argument %s\n", e.what());
        }
    };
    if (prec == 32) run(float{});
    else run(double{});
    return 0;
}
