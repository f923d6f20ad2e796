// Header-only C++ shim over the C ABI (include/mfd.h) that re-exposes the
// reference's Simulation<T> surface (/root/reference/proj/include/magfd/sim.hpp:15-72)
// and maps mfd_status back to the reference exception types and messages, so a
// driver written against magfd::Simulation<T> recompiles against
// magfd_b200::Simulation<T> with the field data resident on the B200.
//
//   magfd::Simulation<T>(spec, backend)      -> magfd_b200::Simulation<T>(grid, mat, terms, stepper)
//   double step(StepTiming*)                 -> double step()            (sim.hpp:33-42)
//   TrajectorySample sampleNow()             -> Sample sample_now()      (sim.hpp:45-55)
//   RelaxResult<T> relax()                   -> RelaxResult relax()      (sim.hpp:57-62)
//   state().M  (read / write)                -> get_m / set_m            (state.hpp:23-32)
//   EffectiveFieldProvider::compute          -> effective_field()        (fields.hpp:220-253)
//   EffectiveFieldProvider::lastDemagField   -> demag_field()            (fields.hpp:264-268)
#pragma once

#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../mfd.h"

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

struct Sample {
    long step;
    double t;
    double m[3];
    double e_exchange, e_anisotropy, e_demag, e_zeeman, e_total;
    double max_torque_deg_per_ns;
};

struct RelaxResult {
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
class Simulation {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "T must be float or double");

public:
    Simulation(const mfd_grid& grid, const mfd_material& mat, const mfd_terms& terms,
               const mfd_stepper& stepper, int device = 0)
        : n_(static_cast<std::size_t>(grid.nx) * grid.ny * grid.nz) {
        mfd_exec ex{};
        ex.precision_bits = sizeof(T) == 4 ? 32 : 64;
        ex.device = device;
        const mfd_status st = mfd_create(&grid, &mat, &terms, &stepper, &ex, &ctx_);
        if (st != MFD_OK) raise(st, mfd_last_error(nullptr));
    }
    ~Simulation() { mfd_destroy(ctx_); }
    Simulation(const Simulation&) = delete;
    Simulation& operator=(const Simulation&) = delete;

    std::size_t cell_count() const { return n_; }

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

    // One Euler step; returns the pre-step max torque rate (deg/ns) (sim.hpp:32-42).
    double step() {
        double torque = 0;
        check(mfd_step(ctx_, 1, &torque, nullptr));
        return torque;
    }
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

    RelaxResult relax() {
        RelaxResult r;
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

private:
    static Sample convert(const mfd_sample& s) {
        return Sample{s.step, s.t, {s.m[0], s.m[1], s.m[2]}, s.e_exchange, s.e_anisotropy,
                      s.e_demag, s.e_zeeman, s.e_total, s.torque_deg_per_ns};
    }
    static void on_sample(const mfd_sample* s, void* user) {
        static_cast<RelaxResult*>(user)->log.push_back(convert(*s));
    }
    void check(mfd_status st) {
        if (st != MFD_OK) raise(st, mfd_last_error(ctx_));
    }

    mfd_ctx* ctx_ = nullptr;
    std::size_t n_;
};

} // namespace magfd_b200
