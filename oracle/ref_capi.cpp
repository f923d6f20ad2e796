// TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// C entry points over the UNMODIFIED reference solver (/root/reference/proj),
// compiled from the reference's own sources by oracle/Makefile into
// oracle/_ref/libmagfd_ref.so.  Used by tests/ (parity checker), by
// __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
// leg.  No reference source is copied here: this file only #includes the
// reference headers at build time and calls their public API.
//
// Every wrapper follows the reference call it names:
//   ref_sim_step        -> Simulation<T>::step            (sim.hpp:33-42)
//   ref_sim_relax       -> Simulation<T>::relax / dynamics::relax (dynamics.hpp:157-198)
//   ref_sim_heff        -> EffectiveFieldProvider<T>::compute (fields.hpp:220-253)
//   ref_sim_hdemag      -> EffectiveFieldProvider<T>::lastDemagField (fields.hpp:264-268)
//   ref_tensor_entry    -> newell::demagTensorEntry      (newell.cpp:188-209)
//   ref_direct_demag    -> oracle::directDemag           (oracle.hpp:26-70)
//   ref_spectrum_octant -> demag::precomputeSpectrum     (demag.hpp:105-119)
//   ref_config_format   -> parseConfig + formatConfig    (config.cpp:76-276)
//   ref_dump_write/read -> io::writeFieldDump / readFieldDump (io.cpp:18-100)
//   ref_trajectory_csv  -> io::writeTrajectoryCsv        (io.cpp:102-117)
//   ref_vortex_state    -> makeVortexState               (state.hpp:83-108)
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "magfd/backend.hpp"
#include "magfd/config.hpp"
#include "magfd/io.hpp"
#include "magfd/demag.hpp"
#include "magfd/dynamics.hpp"
#include "magfd/fields.hpp"
#include "magfd/newell.hpp"
#include "magfd/oracle.hpp"
#include "magfd/sim.hpp"
#include "magfd/state.hpp"

using namespace magfd;

extern "C" {

// Flat mirror of the SimSpec fields the hot path uses (config.hpp:35-80).
typedef struct {
    int nx, ny, nz;
    double dx, dy, dz;
    double A, Ku, Ms, alpha, gamma;
    double easy_axis[3];
    int exchange, anisotropy, demag, zeeman;
    double h_ext[3];
    double dt;
    int renorm_every;
    long max_steps;
    double torque_tol;
    long sample_every;
    int parallel;   // 0 serial, 1 thread pool
    int threads;    // 0 = hardware concurrency
} ref_spec;

typedef struct {
    long step;
    double t, m[3];
    double e_exch, e_anis, e_demag, e_zeeman, e_total;
    double torque;
} ref_sample;

static thread_local std::string g_err;
const char* ref_last_error(void) { return g_err.c_str(); }
}

namespace {

struct Base {
    virtual ~Base() = default;
    virtual void setM(const double*, const double*, const double*) = 0;
    virtual void getM(double*, double*, double*) const = 0;
    virtual double step() = 0;
    virtual void heff(double*, double*, double*) = 0;
    virtual void hdemag(double*, double*, double*) = 0;
    virtual int relax(ref_sample*, long cap, long* nsamples) = 0;
    virtual void time(double* t, long* step) const = 0;
    virtual void setTime(double t, long step) = 0;
    virtual void energies(double out[5]) = 0;
    virtual void setStepThreads(int threads) = 0;
};

template <class T>
struct Handle final : Base {
    Backend backend;
    Grid grid;
    MaterialParams mat;
    dynamics::StepperConfig stepper;
    fields::EffectiveFieldProvider<T> provider;
    SimState<T> state;
    VectorField<T> heffF, rhs;
    // Backend the per-step calls use.  Simulation<T> takes its backend by
    // pointer (sim.hpp:20,70) and every hot-path call receives it per call
    // (fields.hpp:220, demag.hpp:194), so the setup can run on all threads and
    // the steps on another pool (the CPU baseline's 1-thread row).
    std::unique_ptr<Backend> alt;
    const Backend* sb = &backend;

    Handle(const ref_spec& s, Grid g, MaterialParams m, fields::FieldConfig fc)
        : backend(s.parallel ? BackendKind::parallel : BackendKind::serial,
                  static_cast<unsigned>(s.threads)),
          grid(g), mat(m), provider(g, m, fc, backend), state(g), heffF(g), rhs(g) {
        stepper.dt = s.dt;
        stepper.renormalizeEvery = s.renorm_every;
        stepper.maxSteps = s.max_steps;
        stepper.torqueTolDegPerNs = s.torque_tol;
        stepper.sampleEvery = s.sample_every;
        stepper.validate();
    }
    void setM(const double* x, const double* y, const double* z) override {
        for (std::size_t c = 0; c < state.M.size(); ++c) {
            state.M.x[c] = static_cast<T>(x[c]);
            state.M.y[c] = static_cast<T>(y[c]);
            state.M.z[c] = static_cast<T>(z[c]);
        }
        state.energy.reset();
    }
    void getM(double* x, double* y, double* z) const override {
        for (std::size_t c = 0; c < state.M.size(); ++c) {
            x[c] = state.M.x[c];
            y[c] = state.M.y[c];
            z[c] = state.M.z[c];
        }
    }
    // Same sequence as Simulation<T>::step (sim.hpp:33-42).
    double step() override {
        provider.compute(state.M, heffF, *sb, nullptr);
        dynamics::llgRhs(state.M, heffF, mat, *sb, rhs);
        const double torque = dynamics::maxTorqueRate(rhs, mat.Ms, *sb);
        const bool renorm = (state.step + 1) % stepper.renormalizeEvery == 0;
        dynamics::eulerUpdate(state, rhs, stepper.dt, mat.Ms, renorm, *sb);
        return torque;
    }
    void heff(double* x, double* y, double* z) override {
        provider.compute(state.M, heffF, *sb, nullptr);
        for (std::size_t c = 0; c < heffF.size(); ++c) {
            x[c] = heffF.x[c];
            y[c] = heffF.y[c];
            z[c] = heffF.z[c];
        }
    }
    void hdemag(double* x, double* y, double* z) override {
        provider.compute(state.M, heffF, *sb, nullptr);
        const auto& h = provider.lastDemagField();
        for (std::size_t c = 0; c < h.size(); ++c) {
            x[c] = h.x[c];
            y[c] = h.y[c];
            z[c] = h.z[c];
        }
    }
    int relax(ref_sample* out, long cap, long* n) override {
        auto res = dynamics::relax(state, provider, stepper, mat, *sb, nullptr);
        state = res.state;
        long k = 0;
        for (const auto& s : res.log) {
            if (k < cap) {
                ref_sample& o = out[k];
                o.step = s.step;
                o.t = s.t;
                o.m[0] = s.m.x;
                o.m[1] = s.m.y;
                o.m[2] = s.m.z;
                o.e_exch = s.energy.exchange;
                o.e_anis = s.energy.anisotropy;
                o.e_demag = s.energy.demag;
                o.e_zeeman = s.energy.zeeman;
                o.e_total = s.energy.total;
                o.torque = s.maxTorqueDegPerNs;
            }
            ++k;
        }
        *n = k;
        return res.converged ? 1 : 0;
    }
    void time(double* t, long* s) const override {
        *t = state.t;
        *s = state.step;
    }
    void setTime(double t, long s) override {
        state.t = t;
        state.step = s;
    }
    void energies(double out[5]) override {
        provider.compute(state.M, heffF, *sb, nullptr);
        const EnergyBreakdown e = provider.energies(state.M, *sb);
        out[0] = e.exchange;
        out[1] = e.anisotropy;
        out[2] = e.demag;
        out[3] = e.zeeman;
        out[4] = e.total;
    }
    void setStepThreads(int threads) override {
        if (threads <= 0) {
            alt.reset();
            sb = &backend;
            return;
        }
        alt = std::make_unique<Backend>(threads == 1 ? BackendKind::serial : BackendKind::parallel,
                                        static_cast<unsigned>(threads));
        sb = alt.get();
    }
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

} // namespace

extern "C" {

void* ref_sim_create(int precision_bits, const ref_spec* s) {
    Base* out = nullptr;
    const int rc = guard([&] {
        Grid g(s->nx, s->ny, s->nz, s->dx, s->dy, s->dz);
        MaterialParams m;
        m.A = s->A;
        m.Ku = s->Ku;
        m.Ms = s->Ms;
        m.alpha = s->alpha;
        m.gamma = s->gamma;
        m.easyAxis = {s->easy_axis[0], s->easy_axis[1], s->easy_axis[2]};
        fields::FieldConfig fc{s->exchange != 0, s->anisotropy != 0, s->demag != 0,
                               s->zeeman != 0, {s->h_ext[0], s->h_ext[1], s->h_ext[2]}};
        if (precision_bits == 32)
            out = new Handle<float>(*s, g, m, fc);
        else
            out = new Handle<double>(*s, g, m, fc);
    });
    return rc == 0 ? out : nullptr;
}

void ref_sim_destroy(void* h) { delete static_cast<Base*>(h); }

int ref_sim_set_m(void* h, const double* x, const double* y, const double* z) {
    return guard([&] { static_cast<Base*>(h)->setM(x, y, z); });
}
int ref_sim_get_m(void* h, double* x, double* y, double* z) {
    return guard([&] { static_cast<Base*>(h)->getM(x, y, z); });
}
int ref_sim_set_time(void* h, double t, long step) {
    return guard([&] { static_cast<Base*>(h)->setTime(t, step); });
}
int ref_sim_get_time(void* h, double* t, long* step) {
    return guard([&] { static_cast<Base*>(h)->time(t, step); });
}
// n steps; torques[i] = pre-step torque of step i (may be null).
int ref_sim_step(void* h, long n, double* torques) {
    return guard([&] {
        for (long i = 0; i < n; ++i) {
            const double t = static_cast<Base*>(h)->step();
            if (torques) torques[i] = t;
        }
    });
}
int ref_sim_heff(void* h, double* x, double* y, double* z) {
    return guard([&] { static_cast<Base*>(h)->heff(x, y, z); });
}
int ref_sim_hdemag(void* h, double* x, double* y, double* z) {
    return guard([&] { static_cast<Base*>(h)->hdemag(x, y, z); });
}
// Step on a `threads`-thread backend from now on (<= 0: back to the creation backend).
int ref_sim_set_step_threads(void* h, int threads) {
    return guard([&] { static_cast<Base*>(h)->setStepThreads(threads); });
}
int ref_sim_energies(void* h, double out[5]) {
    return guard([&] { static_cast<Base*>(h)->energies(out); });
}
// Returns converged (0/1) or -code on error; samples copied up to cap.
int ref_sim_relax(void* h, ref_sample* samples, long cap, long* nsamples) {
    int conv = 0;
    const int rc = guard([&] { conv = static_cast<Base*>(h)->relax(samples, cap, nsamples); });
    return rc ? -rc : conv;
}

void ref_tensor_entry(int di, int dj, int dk, double dx, double dy, double dz, double out[6]) {
    const newell::TensorEntry e = newell::demagTensorEntry(di, dj, dk, dx, dy, dz);
    out[0] = e.xx;
    out[1] = e.yy;
    out[2] = e.zz;
    out[3] = e.xy;
    out[4] = e.xz;
    out[5] = e.yz;
}
double ref_newell_nxx(double X, double Y, double Z, double dx, double dy, double dz) {
    return static_cast<double>(newell::demagNxx(X, Y, Z, dx, dy, dz));
}
double ref_newell_nxy(double X, double Y, double Z, double dx, double dy, double dz) {
    return static_cast<double>(newell::demagNxy(X, Y, Z, dx, dy, dz));
}

// Octant of tensor entries over [0,n)^3, layout [comp][k][j][i]
// (buildDemagTensor's per-cell evaluation, demag.hpp:66-70).
int ref_tensor_octant(int nx, int ny, int nz, double dx, double dy, double dz, int threads,
                      double* out) {
    return guard([&] {
        Grid g(nx, ny, nz, dx, dy, dz);
        Backend b(threads > 0 ? BackendKind::parallel : BackendKind::serial,
                  static_cast<unsigned>(threads > 0 ? threads : 0));
        const std::size_t n = g.cellCount();
        b.forEach(n, [&](std::size_t c) {
            int i, j, k;
            g.unindex(c, i, j, k);
            const newell::TensorEntry e = newell::demagTensorEntry(i, j, k, dx, dy, dz);
            out[0 * n + c] = e.xx;
            out[1 * n + c] = e.yy;
            out[2 * n + c] = e.zz;
            out[3 * n + c] = e.xy;
            out[4 * n + c] = e.xz;
            out[5 * n + c] = e.yz;
        });
    });
}

// Real parts of the six f64 tensor spectra on the non-negative-frequency
// octant [0,Px/2]x[0,Py/2]x[0,Pz/2], layout [comp][w][v][u]; plus the max
// |imag| over the whole spectrum in *max_imag.
int ref_spectrum_octant(int nx, int ny, int nz, double dx, double dy, double dz, double* out,
                        double* max_imag) {
    return guard([&] {
        Grid g(nx, ny, nz, dx, dy, dz);
        Backend b(BackendKind::serial);
        const auto pd = demag::paddedDimsFor(g);
        auto plan = fft::FftPlan<double>::create(pd);
        auto spec = demag::precomputeSpectrum(demag::buildDemagTensor<double>(g, pd, b), plan, b);
        const int hx = pd.x / 2 + 1, hy = pd.y / 2 + 1, hz = pd.z / 2 + 1;
        const std::size_t oct = static_cast<std::size_t>(hx) * hy * hz;
        const fft::Spectrum<double>* comps[6] = {&spec.xx, &spec.yy, &spec.zz,
                                                 &spec.xy, &spec.xz, &spec.yz};
        double mi = 0;
        for (int c = 0; c < 6; ++c) {
            for (const auto& v : comps[c]->data) mi = std::max(mi, std::abs(v.imag()));
            for (int w = 0; w < hz; ++w)
                for (int v = 0; v < hy; ++v)
                    for (int u = 0; u < hx; ++u)
                        out[c * oct + (static_cast<std::size_t>(w) * hy + v) * hx + u] =
                            comps[c]->data[u + static_cast<std::size_t>(pd.x) *
                                                   (v + static_cast<std::size_t>(pd.y) * w)]
                                .real();
        }
        *max_imag = mi;
    });
}

// Brute-force long-double direct demag sum (oracle.hpp:26-70), f64 input.
int ref_direct_demag(int nx, int ny, int nz, double dx, double dy, double dz,
                     const double* mx, const double* my, const double* mz, double* hx,
                     double* hy, double* hz) {
    return guard([&] {
        Grid g(nx, ny, nz, dx, dy, dz);
        VectorField<double> M(g);
        for (std::size_t c = 0; c < M.size(); ++c) {
            M.x[c] = mx[c];
            M.y[c] = my[c];
            M.z[c] = mz[c];
        }
        auto H = oracle::directDemag(M, g, g.cellCount());
        for (std::size_t c = 0; c < H.size(); ++c) {
            hx[c] = H.x[c];
            hy[c] = H.y[c];
            hz[c] = H.z[c];
        }
    });
}

double ref_stability_dt_limit(double A, double Ms, double alpha, double gamma, double dx,
                              double dy, double dz) {
    MaterialParams m;
    m.A = A;
    m.Ms = Ms;
    m.alpha = alpha;
    m.gamma = gamma;
    return dynamics::stabilityDtLimit(m, Grid(1, 1, 1, dx, dy, dz));
}

// parseConfig(text, &defaults) -> formatConfig.  Returns 0 (out = canonical
// text, defaults = applied-default lines) or 7 (out = ConfigError text).
static void put(const std::string& s, char* out, size_t cap) {
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(out, s.data(), n);
    out[n] = 0;
}
int ref_config_format(const char* text, char* out, size_t cap, char* defaults, size_t dcap) {
    try {
        std::vector<std::string> d;
        const SimSpec spec = parseConfig(text, &d);
        put(formatConfig(spec), out, cap);
        std::string all;
        for (const auto& l : d) all += l + "\n";
        put(all, defaults, dcap);
        return 0;
    } catch (const ConfigError& e) {
        put(e.what(), out, cap);
        return 7;
    }
}

int ref_dump_write(const char* path, int nx, int ny, int nz, double dx, double dy, double dz, double Ms, int prec,
                   const double* mx, const double* my, const double* mz) {
    try {
        Grid g(nx, ny, nz, dx, dy, dz);
        VectorField<double> M(g);
        for (std::size_t c = 0; c < M.size(); ++c) M.set(c, {mx[c], my[c], mz[c]});
        io::writeFieldDump(path, M, Ms, prec == 32 ? Precision::f32 : Precision::f64);
        return 0;
    } catch (const io::IoError& e) {
        g_err = e.what();
        return 8;
    }
}

// hdr = {nx, ny, nz, dx, dy, dz, Ms, precision_bits}; m = 3 x N (may be null: header only)
int ref_dump_read(const char* path, double* hdr, double* m, long long cap) {
    try {
        const io::FieldDump d = io::readFieldDump(path);
        const Grid& g = d.grid;
        const double h[8] = {(double)g.nx, (double)g.ny, (double)g.nz, g.dx, g.dy, g.dz, d.Ms,
                             d.precision == Precision::f32 ? 32.0 : 64.0};
        std::memcpy(hdr, h, sizeof h);
        const long long n = (long long)g.cellCount();
        if (m && cap >= 3 * n)
            for (long long c = 0; c < n; ++c) {
                m[c] = d.M.x[c];
                m[c + n] = d.M.y[c];
                m[c + 2 * n] = d.M.z[c];
            }
        return 0;
    } catch (const io::IoError& e) {
        g_err = e.what();
        return 8;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// rows: n x 11 {step, t, mx, my, mz, E_exch, E_anis, E_demag, E_zeeman, E_total, torque}
int ref_trajectory_csv(const char* path, const double* rows, long n) {
    try {
        std::vector<dynamics::TrajectorySample> log(n);
        for (long r = 0; r < n; ++r) {
            const double* x = rows + 11 * r;
            auto& s = log[r];
            s.step = (long)x[0];
            s.t = x[1];
            s.m = {x[2], x[3], x[4]};
            s.energy.exchange = x[5];
            s.energy.anisotropy = x[6];
            s.energy.demag = x[7];
            s.energy.zeeman = x[8];
            s.energy.total = x[9];
            s.maxTorqueDegPerNs = x[10];
        }
        io::writeTrajectoryCsv(path, log);
        return 0;
    } catch (const io::IoError& e) {
        g_err = e.what();
        return 8;
    }
}

// makeVortexState<T>(grid, axis, Ms) -> 3 x N (as double)
int ref_vortex_state(int precision_bits, int nx, int ny, int nz, double dx, double dy, double dz, int axis, double Ms,
                     double* m) {
    return guard([&] {
        Grid g(nx, ny, nz, dx, dy, dz);
        const SignedAxis a = static_cast<SignedAxis>(axis);
        const std::size_t n = g.cellCount();
        auto emit = [&](const auto& st) {
            for (std::size_t c = 0; c < n; ++c) {
                m[c] = (double)st.M.x[c];
                m[c + n] = (double)st.M.y[c];
                m[c + 2 * n] = (double)st.M.z[c];
            }
        };
        if (precision_bits == 32) emit(makeVortexState<float>(g, a, Ms));
        else emit(makeVortexState<double>(g, a, Ms));
    });
}

} // extern "C"
