// Header-only C++ shim over the C ABI (include/mfd.h) that re-exposes the
// reference's Simulation<T> surface (/root/reference/proj/include/magfd/sim.hpp:15-72)
// and maps mfd_status back to the reference exception types and messages.
//
// Drop-in form (the reference's own signatures; a driver recompiles with only a
// namespace swap, magfd::Simulation<T> -> magfd_b200::Simulation<T>):
//
//   Simulation(const SimSpec&, const Backend&)       sim.hpp:17-24 (initial state from
//                                                    spec.initKind: makeUniformState /
//                                                    makeVortexState, state.hpp:71-108)
//   double step(StepTiming* = nullptr)               sim.hpp:33-42 (pre-step torque, deg/ns)
//   TrajectorySample sampleNow()                     sim.hpp:45-55
//   RelaxResult<T> relax(StepTiming* = nullptr)      sim.hpp:57-62
//   grid() / material() / stepper()                  sim.hpp:26-28
//   state()                                          sim.hpp:29-30: the state lives on the
//                                                    device; state() returns a view with
//                                                    .step, .t and .M (M.cast<U>(), M.size(),
//                                                    M.x / .y / .z are downloaded on use)
//
// When the reference headers are on the include path (the integration build,
// INTEGRATION.md section 1) TrajectorySample, RelaxResult<T>, SimState<T>,
// VectorField<T>, Vec3d and EnergyBreakdown ARE the reference's types, so the
// results flow into io::writeTrajectoryCsv / io::writeFieldDump unchanged.
// Without them the shim uses member-compatible mirrors of those types.  The
// Backend argument is accepted for signature compatibility (the device is
// MFD_DEVICE, default 0); SimSpec / Backend / StepTiming are duck-typed.
//
// Plain-struct form (no reference types): Simulation(mfd_grid, mfd_material,
// mfd_terms, mfd_stepper) with set_m / get_m / step(n) / sample_now / relax /
// effective_field / demag_field.
#pragma once

#include <cstdlib>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../mfd.h"
#include "../mfd_host.h"

#if __has_include("magfd/dynamics.hpp") && __has_include("magfd/state.hpp")
#include "magfd/dynamics.hpp"
#include "magfd/state.hpp"
#define MAGFD_B200_REFERENCE_TYPES 1
#else
#define MAGFD_B200_REFERENCE_TYPES 0
#endif

namespace magfd_b200 {

[[noreturn]] inline void raise(mfd_status st, const char* msg) {
    switch (st) {
        case MFD_EINVAL: throw std::invalid_argument(msg);
        case MFD_ENONFINITE: throw std::runtime_error(msg);
        case MFD_ELOGIC: throw std::logic_error(msg);
        case MFD_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(std::string("magfd-b200: ") + msg);
    }
}

// ------------------------------------------------ reference-compatible types
#if MAGFD_B200_REFERENCE_TYPES
using Vec3d = magfd::Vec3d;
using EnergyBreakdown = magfd::EnergyBreakdown;
using TrajectorySample = magfd::dynamics::TrajectorySample;
template <class T> using VectorField = magfd::VectorField<T>;
template <class T> using SimState = magfd::SimState<T>;
template <class T> using RelaxResult = magfd::dynamics::RelaxResult<T>;
template <class T> inline VectorField<T> make_field(const mfd_grid& g) {
    return VectorField<T>(magfd::Grid(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz));
}
#else
struct Vec3d { double x = 0, y = 0, z = 0; };
struct EnergyBreakdown { double exchange = 0, anisotropy = 0, demag = 0, zeeman = 0, total = 0; };
struct TrajectorySample {                      // dynamics.hpp:138-144
    long step = 0;
    double t = 0;
    Vec3d m{};
    EnergyBreakdown energy{};
    double maxTorqueDegPerNs = 0;
};
template <class T>
struct VectorField {                           // vector_field.hpp:14-43 (grid omitted)
    std::vector<T> x, y, z;
    VectorField() = default;
    explicit VectorField(std::size_t n) : x(n), y(n), z(n) {}
    std::size_t size() const { return x.size(); }
    template <class U>
    VectorField<U> cast() const {
        VectorField<U> o(size());
        for (std::size_t i = 0; i < size(); ++i) {
            o.x[i] = static_cast<U>(x[i]);
            o.y[i] = static_cast<U>(y[i]);
            o.z[i] = static_cast<U>(z[i]);
        }
        return o;
    }
};
template <class T>
struct SimState {                              // state.hpp:23-32
    VectorField<T> M;
    double t = 0;
    long step = 0;
};
template <class T>
struct RelaxResult {                           // dynamics.hpp:146-151
    SimState<T> state;
    bool converged = false;
    std::vector<TrajectorySample> log;
};
template <class T> inline VectorField<T> make_field(const mfd_grid& g) {
    return VectorField<T>(static_cast<std::size_t>(g.nx) * g.ny * g.nz);
}
#endif

// Plain-struct sample (the C ABI's mfd_sample with named energies).
struct Sample {
    long step;
    double t;
    double m[3];
    double e_exchange, e_anisotropy, e_demag, e_zeeman, e_total;
    double max_torque_deg_per_ns;
};

struct PlainRelaxResult {
    bool converged = false;
    std::vector<Sample> log;
};

// Field data are SoA vectors like VectorField<T> (vector_field.hpp:14-43).
template <class T>
struct HostField {
    std::vector<T> x, y, z;
    explicit HostField(std::size_t n = 0) : x(n), y(n), z(n) {}
};

template <class T>
class Simulation;

// state() of the drop-in form: the magnetisation stays on the device; .step and
// .t are copied, M downloads when it is read (cast<U>(), x / y / z, size()).
template <class T>
struct DeviceField {
    Simulation<T>* sim;
    std::size_t size() const { return sim->cell_count(); }
    template <class U>
    VectorField<U> cast() const { return sim->template download<U>(); }
    VectorField<T> get() const { return sim->template download<T>(); }
};
template <class T>
struct StateView {
    long step;
    double t;
    DeviceField<T> M;
};

template <class T>
class Simulation {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "T must be float or double");

public:
    // --- plain-struct form
    Simulation(const mfd_grid& grid, const mfd_material& mat, const mfd_terms& terms,
               const mfd_stepper& stepper, int device = 0)
        : grid_(grid), mat_(mat), stepper_(stepper), n_(static_cast<std::size_t>(grid.nx) * grid.ny * grid.nz) {
        create(terms, device);
    }

    // --- drop-in form: magfd::Simulation<T>(const SimSpec&, const Backend&) (sim.hpp:17-24)
    template <class Spec, class Backend, class = decltype(std::declval<const Spec&>().toGrid())>
    Simulation(const Spec& s, const Backend& /*backend*/)
        : grid_{s.nx, s.ny, s.nz, s.dx, s.dy, s.dz},
          mat_{s.A, s.Ku, s.Ms, s.alpha, s.gamma, {s.easyAxis.x, s.easyAxis.y, s.easyAxis.z}},
          stepper_{s.dt, s.renormEvery, s.maxSteps, s.torqueTol, s.sampleEvery},
          n_(static_cast<std::size_t>(s.nx > 0 ? s.nx : 0) * (s.ny > 0 ? s.ny : 0) * (s.nz > 0 ? s.nz : 0)) {
        const mfd_terms terms{s.termExchange, s.termAnisotropy, s.termDemag, s.termZeeman,
                              {s.externField.x, s.externField.y, s.externField.z}};
        const char* dev = std::getenv("MFD_DEVICE");
        create(terms, dev ? std::atoi(dev) : 0);
        if (static_cast<int>(s.initKind) == 0) {   // InitKind::uniform -> makeUniformState
            const double d[3] = {s.initDirection.x, s.initDirection.y, s.initDirection.z};
            check(mfd_set_m_uniform(ctx_, d));
        } else {                                   // InitKind::vortex -> makeVortexState
            check(mfd_set_m_vortex(ctx_, static_cast<int>(s.vortexAxis)));
        }
    }

    ~Simulation() { mfd_destroy(ctx_); }
    Simulation(const Simulation&) = delete;
    Simulation& operator=(const Simulation&) = delete;

    std::size_t cell_count() const { return n_; }
    const mfd_grid& grid() const { return grid_; }
    const mfd_material& material() const { return mat_; }
    const mfd_stepper& stepper() const { return stepper_; }

    // ---- reference-named methods (sim.hpp:26-62)
    // One Euler step; returns the pre-step max torque rate (deg/ns).  With a
    // timing record the step runs on the instrumented path and the device time
    // of its passes is added in seconds (pad and the x pass share the first
    // pass; the local fields and the integrator share the last).
    template <class Timing = void>
    double step(Timing* timing = nullptr) {
        if constexpr (std::is_void_v<Timing>) {
            return step(1L);
        } else {
            if (!timing) return step(1L);
            double ms[7];
            check(mfd_last_step_timing(ctx_, ms));
            timing->pad += 0.0;
            timing->forwardFft += (ms[0] + ms[1]) * 1e-3;
            timing->spectralMultiply += ms[2] * 1e-3;
            timing->inverseFft += ms[3] * 1e-3;
            timing->localFields += ms[4] * 1e-3;
            timing->total += ms[5] * 1e-3;
            return ms[6];
        }
    }
    TrajectorySample sampleNow() {
        mfd_sample s{};
        check(mfd_sample_now(ctx_, &s));
        return to_ref(s);
    }
    template <class Timing = void>
    RelaxResult<T> relax(Timing* = nullptr) {
        RelaxResult<T> r;
        int conv = 0;
        check(mfd_relax(ctx_, &conv, &Simulation::on_ref_sample, &r.log));
        r.converged = conv != 0;
        r.state.M = download<T>();
        double t;
        long st;
        mfd_get_time(ctx_, &t, &st);
        r.state.t = t;
        r.state.step = st;
        return r;
    }
    StateView<T> state() {
        double t;
        long st;
        mfd_get_time(ctx_, &t, &st);
        return StateView<T>{st, t, DeviceField<T>{this}};
    }
    template <class U>
    VectorField<U> download() {
        VectorField<T> m = make_field<T>(grid_);
        if constexpr (std::is_same_v<T, float>) check(mfd_get_m_f32(ctx_, m.x.data(), m.y.data(), m.z.data()));
        else check(mfd_get_m_f64(ctx_, m.x.data(), m.y.data(), m.z.data()));
        if constexpr (std::is_same_v<U, T>) return m;
        else return m.template cast<U>();
    }
    // Replace the device state (the drop-in for writing state().M).
    void setState(const VectorField<T>& m) {
        if constexpr (std::is_same_v<T, float>) check(mfd_set_m_f32(ctx_, m.x.data(), m.y.data(), m.z.data()));
        else check(mfd_set_m_f64(ctx_, m.x.data(), m.y.data(), m.z.data()));
    }

    // ---- plain-struct methods
    void set_uniform(const double dir[3]) { check(mfd_set_m_uniform(ctx_, dir)); }
    void set_m(const HostField<T>& m) {
        if constexpr (std::is_same_v<T, float>) check(mfd_set_m_f32(ctx_, m.x.data(), m.y.data(), m.z.data()));
        else check(mfd_set_m_f64(ctx_, m.x.data(), m.y.data(), m.z.data()));
    }
    HostField<T> get_m() {
        HostField<T> m(n_);
        if constexpr (std::is_same_v<T, float>) check(mfd_get_m_f32(ctx_, m.x.data(), m.y.data(), m.z.data()));
        else check(mfd_get_m_f64(ctx_, m.x.data(), m.y.data(), m.z.data()));
        return m;
    }
    double t() const { double t; long s; mfd_get_time(ctx_, &t, &s); return t; }
    long step_count() const { double t; long s; mfd_get_time(ctx_, &t, &s); return s; }
    double step(long n) {
        double torque = 0;
        check(mfd_step(ctx_, n, &torque, nullptr));
        return torque;
    }
    Sample sample_now() {
        mfd_sample s{};
        check(mfd_sample_now(ctx_, &s));
        return convert(s);
    }
    PlainRelaxResult relax_plain() {
        PlainRelaxResult r;
        int conv = 0;
        check(mfd_relax(ctx_, &conv, &Simulation::on_sample, &r));
        r.converged = conv != 0;
        return r;
    }
    HostField<double> effective_field() {
        HostField<double> h(n_);
        check(mfd_effective_field_f64(ctx_, h.x.data(), h.y.data(), h.z.data()));
        return h;
    }
    HostField<double> demag_field() {
        HostField<double> h(n_);
        check(mfd_demag_field_f64(ctx_, h.x.data(), h.y.data(), h.z.data()));
        return h;
    }
    HostField<T> effective_field_t() {
        HostField<T> h(n_);
        if constexpr (std::is_same_v<T, float>) check(mfd_effective_field_f32(ctx_, h.x.data(), h.y.data(), h.z.data()));
        else check(mfd_effective_field_f64(ctx_, h.x.data(), h.y.data(), h.z.data()));
        return h;
    }

private:
    void create(const mfd_terms& terms, int device) {
        mfd_exec ex{};
        ex.precision_bits = sizeof(T) == 4 ? 32 : 64;
        ex.device = device;
        const mfd_status st = mfd_create(&grid_, &mat_, &terms, &stepper_, &ex, &ctx_);
        if (st != MFD_OK) raise(st, mfd_last_error(nullptr));
    }
    static Sample convert(const mfd_sample& s) {
        return Sample{s.step, s.t, {s.m[0], s.m[1], s.m[2]}, s.e_exchange, s.e_anisotropy,
                      s.e_demag, s.e_zeeman, s.e_total, s.torque_deg_per_ns};
    }
    static TrajectorySample to_ref(const mfd_sample& s) {
        TrajectorySample o{};
        o.step = s.step;
        o.t = s.t;
        o.m.x = s.m[0];
        o.m.y = s.m[1];
        o.m.z = s.m[2];
        o.energy.exchange = s.e_exchange;
        o.energy.anisotropy = s.e_anisotropy;
        o.energy.demag = s.e_demag;
        o.energy.zeeman = s.e_zeeman;
        o.energy.total = s.e_total;
        o.maxTorqueDegPerNs = s.torque_deg_per_ns;
        return o;
    }
    static void on_sample(const mfd_sample* s, void* user) {
        static_cast<PlainRelaxResult*>(user)->log.push_back(convert(*s));
    }
    static void on_ref_sample(const mfd_sample* s, void* user) {
        static_cast<std::vector<TrajectorySample>*>(user)->push_back(to_ref(*s));
    }
    void check(mfd_status st) {
        if (st != MFD_OK) raise(st, mfd_last_error(ctx_));
    }

    mfd_ctx* ctx_ = nullptr;
    mfd_grid grid_;
    mfd_material mat_;
    mfd_stepper stepper_;
    std::size_t n_;
};

} // namespace magfd_b200
