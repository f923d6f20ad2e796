// magfd-b200: the reference CLI's relax / run / bench subcommands
// (tools/magfd.cpp, cli.cpp:40-200) driving the B200 engine through the C ABI.
// Same config format, same outputs (trajectory CSV, field dump, bench CSV),
// same summary text and exit codes (0 ok, 1 error, 2 unconverged; cli.hpp:13-16).
//
//   magfd-b200 relax --config FILE [--device D]
//   magfd-b200 run   --config FILE --steps N [--device D]
//   magfd-b200 bench [--sizes 8,16,32,64] [--config FILE] [--with-128] [--csv bench.csv] [--device D]
//
// Bench phases map onto the fused passes: pad = 0 (fused into the x pass),
// forward FFT = K1 + K2, multiply = K3 (z transforms + tensor product),
// inverse FFT = K4, local = K5 (inverse x + H_eff + LLG + Euler), integrate = 0
// (fused into K5).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/mfd.h"
#include "../../../include/mfd_host.h"

namespace {

constexpr int kOk = 0, kError = 1, kUnconverged = 2;

std::string sci(double x, int prec = 6) {
    char b[48];
    std::snprintf(b, sizeof b, "%.*g", prec, x);
    return b;
}

struct Ctx {
    mfd_ctx* c = nullptr;
    ~Ctx() { if (c) mfd_destroy(c); }
};

[[noreturn]] void fail(const std::string& msg) { throw std::runtime_error(msg); }

void check(mfd_status s, mfd_ctx* c) {
    if (s != MFD_OK) fail(mfd_last_error(c));
}

// Simulation(spec): engine + initial state (sim.hpp:17-24, state.hpp:71-108)
void create(const mfd_spec& spec, int device, Ctx& ctx) {
    mfd_exec ex{};
    ex.precision_bits = spec.precision_bits;
    ex.device = device;
    ex.world = 1;
    if (mfd_create(&spec.grid, &spec.material, &spec.terms, &spec.stepper, &ex, &ctx.c) != MFD_OK)
        fail(mfd_last_error(nullptr));
    if (spec.init_kind == 0) check(mfd_set_m_uniform(ctx.c, spec.init_direction), ctx.c);
    else check(mfd_set_m_vortex(ctx.c, spec.vortex_axis), ctx.c);
}

void summary(const mfd_sample& s, bool converged) {   // cli.cpp:24-37
    std::printf("final: step %ld, t %s s, %s\n", s.step, sci(s.t).c_str(), converged ? "converged" : "NOT converged");
    std::printf("  <m> = (%s, %s, %s)\n", sci(s.m[0], 9).c_str(), sci(s.m[1], 9).c_str(), sci(s.m[2], 9).c_str());
    std::printf("  E_exch %s J, E_anis %s J, E_demag %s J, E_zeeman %s J, E_total %s J\n", sci(s.e_exchange).c_str(),
                sci(s.e_anisotropy).c_str(), sci(s.e_demag).c_str(), sci(s.e_zeeman).c_str(), sci(s.e_total).c_str());
    std::printf("  max torque %s deg/ns\n", sci(s.torque_deg_per_ns).c_str());
}

// trajectory CSV + final dump; false (after printing) on an IO error
bool outputs(const mfd_spec& spec, mfd_ctx* c, const std::vector<mfd_sample>& log) {
    if (spec.csv_path[0] && mfd_trajectory_csv_write(spec.csv_path, log.data(), (long)log.size()) != MFD_OK) {
        std::printf("error: %s\n", mfd_host_last_error());
        return false;
    }
    if (spec.dump_path[0]) {
        const size_t n = (size_t)spec.grid.nx * spec.grid.ny * spec.grid.nz;
        std::vector<double> m(3 * n);
        check(mfd_get_m_f64(c, m.data(), m.data() + n, m.data() + 2 * n), c);
        if (mfd_dump_write(spec.dump_path, &spec.grid, spec.material.Ms, spec.precision_bits, m.data(), m.data() + n,
                           m.data() + 2 * n) != MFD_OK) {
            std::printf("error: %s\n", mfd_host_last_error());
            return false;
        }
    }
    return true;
}

int cmd_relax(const mfd_spec& spec, int device) try {
    Ctx ctx;
    create(spec, device, ctx);
    const double lim = mfd_stability_dt_limit(&spec.material, &spec.grid);
    if (spec.stepper.dt > lim)
        std::printf("warning: stepper.dt %s s exceeds the stability heuristic %s s\n", sci(spec.stepper.dt).c_str(),
                    sci(lim).c_str());
    std::vector<mfd_sample> log;
    int conv = 0;
    check(mfd_relax(ctx.c, &conv,
                    [](const mfd_sample* s, void* u) { static_cast<std::vector<mfd_sample>*>(u)->push_back(*s); },
                    &log),
          ctx.c);
    if (!outputs(spec, ctx.c, log)) return kError;
    summary(log.back(), conv != 0);
    return conv ? kOk : kUnconverged;
} catch (const std::exception& e) {   // cli.cpp:123-131: engine errors go to the command's stream
    std::printf("error: %s\n", e.what());
    return kError;
}

int cmd_run(const mfd_spec& spec, long steps, int device) try {
    if (steps < 0) {
        std::printf("error: steps must be >= 0\n");
        return kError;
    }
    Ctx ctx;
    create(spec, device, ctx);
    std::vector<mfd_sample> log;
    const long every = spec.stepper.sample_every;
    mfd_sample s;
    for (long done = 0; done < steps;) {   // sample when step % sampleEvery == 0, then step (cli.cpp:63-67)
        double t;
        long cur;
        check(mfd_get_time(ctx.c, &t, &cur), ctx.c);
        if (cur % every == 0) {
            check(mfd_sample_now(ctx.c, &s), ctx.c);
            log.push_back(s);
        }
        const long adv = std::min(steps - done, every - cur % every);
        double last;
        check(mfd_step(ctx.c, adv, &last, nullptr), ctx.c);
        done += adv;
    }
    check(mfd_sample_now(ctx.c, &s), ctx.c);
    log.push_back(s);
    if (!outputs(spec, ctx.c, log)) return kError;
    summary(log.back(), false);
    return kOk;
} catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return kError;
}

double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

int cmd_bench(const std::vector<int>& sizes, const mfd_spec& tmpl, const std::string& csv, int device,
              int measured = 20) {
    std::printf("backend: b200 sm_100a (device %d), precision: %s\n", device, tmpl.precision_bits == 32 ? "f32" : "f64");
    std::printf("  size    ms/step        pad    fwd-fft   multiply    inv-fft      local  integrate\n");
    std::vector<mfd_bench_row> rows;
    for (int size : sizes) {
        mfd_spec s = tmpl;
        s.grid.nx = s.grid.ny = s.grid.nz = size;
        s.init_kind = 0;
        const double r3 = 1.0 / std::sqrt(3.0);
        s.init_direction[0] = s.init_direction[1] = s.init_direction[2] = r3;   // normalized(1,1,1)
        Ctx ctx;
        try {
            create(s, device, ctx);
        } catch (const std::exception& e) {
            if (std::strstr(e.what(), "bad_alloc") || std::strstr(e.what(), "out of memory")) {
                std::printf("warning: size %d^3 skipped (allocation failure)\n", size);
                continue;
            }
            std::printf("error: size %d: %s\n", size, e.what());
            return kError;
        }
        double last;
        check(mfd_step(ctx.c, 3, &last, nullptr), ctx.c);   // warm-up, discarded
        std::vector<double> ph[6];
        for (int i = 0; i < measured; ++i) {
            double ms[7];
            check(mfd_last_step_timing(ctx.c, ms), ctx.c);
            for (int p = 0; p < 6; ++p) ph[p].push_back(ms[p]);
        }
        mfd_bench_row r{};
        r.size = size;
        r.ms_per_step = median(ph[5]);
        r.pad_ms = 0;
        r.forward_fft_ms = median(ph[0]) + median(ph[1]);
        r.spectral_multiply_ms = median(ph[2]);
        r.inverse_fft_ms = median(ph[3]);
        r.local_fields_ms = median(ph[4]);
        r.integrate_ms = 0;
        rows.push_back(r);
        std::printf("%6d %10.4f %10.4f %10.4f %10.4f %10.4f %10.4f %10.4f\n", size, r.ms_per_step, r.pad_ms,
                    r.forward_fft_ms, r.spectral_multiply_ms, r.inverse_fft_ms, r.local_fields_ms, r.integrate_ms);
    }
    if (rows.empty()) {
        std::printf("error: no bench size succeeded\n");
        return kError;
    }
    if (!csv.empty() && mfd_bench_csv_write(csv.c_str(), rows.data(), (long)rows.size()) != MFD_OK) {
        std::printf("error: %s\n", mfd_host_last_error());
        return kError;
    }
    return kOk;
}

mfd_spec load_spec(const std::string& path) {   // tools/magfd.cpp:14-19
    mfd_spec s;
    std::vector<char> defaults(1 << 16);
    if (mfd_config_load(path.c_str(), &s, defaults.data(), defaults.size()) != MFD_OK) fail(mfd_host_last_error());
    const char* p = defaults.data();
    while (*p) {
        const char* e = std::strchr(p, '\n');
        std::printf("default applied: %.*s\n", (int)(e - p), p);
        p = e + 1;
    }
    return s;
}

int usage() {
    std::fprintf(stderr,
                 "magfd-b200: finite-difference LLG micromagnetics with FFT demag on B200\n"
                 "usage: magfd-b200 relax --config FILE [--device D]\n"
                 "       magfd-b200 run --config FILE --steps N [--device D]\n"
                 "       magfd-b200 bench [--sizes 8,16,32,64] [--config FILE] [--with-128] [--csv PATH] "
                 "[--device D]\n");
    return kError;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    std::string config, csv = "bench.csv";
    long steps = 0;
    bool have_steps = false, with128 = false;
    int device = 0;
    std::vector<int> sizes{8, 16, 32, 64};
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string a = argv[i];
            auto val = [&]() -> std::string {
                if (i + 1 >= argc) fail(a + ": value expected");
                return argv[++i];
            };
            if (a == "--config") config = val();
            else if (a == "--steps") { steps = std::stol(val()); have_steps = true; }
            else if (a == "--device") device = std::stoi(val());
            else if (a == "--csv") csv = val();
            else if (a == "--with-128") with128 = true;
            else if (a == "--sizes") {
                sizes.clear();
                std::string v = val();
                for (size_t p = 0; p <= v.size();) {
                    const size_t q = std::min(v.find(',', p), v.size());
                    if (q > p) sizes.push_back(std::stoi(v.substr(p, q - p)));
                    p = q + 1;
                }
                while (i + 1 < argc && argv[i + 1][0] != '-') sizes.push_back(std::stoi(argv[++i]));
            } else fail("unknown option " + a);
        }
        if (cmd == "relax") {
            if (config.empty()) fail("--config is required");
            return cmd_relax(load_spec(config), device);
        }
        if (cmd == "run") {
            if (config.empty() || !have_steps) fail("--config and --steps are required");
            return cmd_run(load_spec(config), steps, device);
        }
        if (cmd == "bench") {
            mfd_spec tmpl;
            if (!config.empty()) {
                tmpl = load_spec(config);
            } else {   // default bench problem (tools/magfd.cpp:62-67)
                mfd_spec_default(&tmpl);
                tmpl.grid.dx = tmpl.grid.dy = tmpl.grid.dz = 2.5e-9;
                tmpl.material.Ms = 8e5;
                tmpl.material.A = 1.3e-11;
                tmpl.material.Ku = 4e4;
                tmpl.backend_kind = 1;
            }
            if (with128) sizes.push_back(128);
            return cmd_bench(sizes, tmpl, csv, device);
        }
        return usage();
    } catch (const std::exception& e) {   // config / usage errors: stderr (tools/magfd.cpp:76-79)
        std::fflush(stdout);
        std::fprintf(stderr, "error: %s\n", e.what());
        return kError;
    }
}
