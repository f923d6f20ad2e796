// C ABI of libmagfd_b200.so (include/mfd.h).  Validation mirrors the
// reference constructors and their exception messages; no exception crosses
// the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "engine.cuh"
#include "../../include/mfd_host.h"

struct mfd_ctx {
    std::unique_ptr<mfd::EngineBase> eng;
    std::string err;
    mfd_stepper st{};
};

namespace {
thread_local std::string g_create_err;

template <class F>
mfd_status guard(mfd_ctx* c, F&& f) {
    try {
        f();
        return MFD_OK;
    } catch (const mfd::Error& e) {
        if (c) c->err = e.what();
        else g_create_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        if (c) c->err = "std::bad_alloc";
        else g_create_err = "std::bad_alloc";
        return MFD_ENOMEM;
    } catch (const std::exception& e) {
        if (c) c->err = e.what();
        else g_create_err = e.what();
        return MFD_ECUDA;
    }
}

void validate(const mfd_grid& g, const mfd_material& m, const mfd_stepper& s) {
    using mfd::Error;
    if (g.nx < 1 || g.ny < 1 || g.nz < 1) throw Error(MFD_EINVAL, "Grid: cell counts must be >= 1");
    if (!(g.dx > 0) || !(g.dy > 0) || !(g.dz > 0)) throw Error(MFD_EINVAL, "Grid: cell sizes must be > 0");
    if (!(m.Ms > 0)) throw Error(MFD_EINVAL, "MaterialParams: Ms must be > 0");
    if (m.A < 0) throw Error(MFD_EINVAL, "MaterialParams: A must be >= 0");
    if (m.alpha < 0) throw Error(MFD_EINVAL, "MaterialParams: alpha must be >= 0");
    if (!(m.gamma > 0)) throw Error(MFD_EINVAL, "MaterialParams: gamma must be > 0");
    const double an = std::sqrt(m.easy_axis[0] * m.easy_axis[0] + m.easy_axis[1] * m.easy_axis[1] +
                                m.easy_axis[2] * m.easy_axis[2]);
    if (std::abs(an - 1.0) > 1e-12) throw Error(MFD_EINVAL, "MaterialParams: easyAxis must be a unit vector");
    if (!(s.dt > 0)) throw Error(MFD_EINVAL, "StepperConfig: dt must be > 0");
    if (s.renorm_every < 1) throw Error(MFD_EINVAL, "StepperConfig: renormalizeEvery must be >= 1");
    if (!(s.torque_tol_deg_per_ns > 0)) throw Error(MFD_EINVAL, "StepperConfig: torque tolerance must be > 0");
}
} // namespace

extern "C" {

const char* mfd_version(void) { return "magfd-b200 0.1 (sm_100a)"; }

mfd_status mfd_nccl_unique_id(unsigned char id[128]) {
    return guard(nullptr, [&] { mfd::nccl_unique_id(id); });
}

mfd_status mfd_create(const mfd_grid* grid, const mfd_material* mat, const mfd_terms* terms,
                      const mfd_stepper* stepper, const mfd_exec* exec, mfd_ctx** out) {
    *out = nullptr;
    return guard(nullptr, [&] {
        if (!grid || !mat || !terms || !stepper) throw mfd::Error(MFD_EINVAL, "mfd_create: null argument");
        validate(*grid, *mat, *stepper);
        const int prec = exec ? exec->precision_bits : 64;
        const int dev = exec ? exec->device : 0;
        if (prec != 32 && prec != 64) throw mfd::Error(MFD_EINVAL, "mfd_create: precision_bits must be 32 or 64");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw mfd::Error(MFD_ECUDA, "magfd-b200: no CUDA device (the engine has no CPU fallback)");
        cudaDeviceProp p{};
        mfd::ck(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
        if (p.major != 10) throw mfd::Error(MFD_ECUDA, "magfd-b200: built for sm_100a, device is sm_" +
                                                           std::to_string(p.major) + std::to_string(p.minor));
        const int world = exec && exec->world > 1 ? exec->world : 1;
        const int rank = exec ? exec->rank : 0;
        if (world > 1 && grid->nz % world != 0)
            throw mfd::Error(MFD_EINVAL, "magfd-b200: nz must be divisible by the number of GPUs (z-slab decomposition)");
        if (world > 1 && (rank < 0 || rank >= world)) throw mfd::Error(MFD_EINVAL, "mfd_create: rank out of range");
        auto c = std::make_unique<mfd_ctx>();
        c->st = *stepper;
        if (world > 1 && exec->virtual_ranks) {
            c->eng.reset(prec == 32 ? mfd::make_virtual_group<float>(*grid, *mat, *terms, *stepper, dev, world)
                                    : mfd::make_virtual_group<double>(*grid, *mat, *terms, *stepper, dev, world));
        } else {
            if (world > 1 && exec->transport != 0 && exec->transport != 1)
                throw mfd::Error(MFD_EINVAL, "mfd_create: transport must be 0 (NCCL) or 1 (shared memory)");
            std::unique_ptr<mfd::Transport> tr;
            if (world > 1)
                tr.reset(exec->transport == 1 ? mfd::make_shm_transport(exec->nccl_id, rank, world)
                                              : mfd::make_nccl_transport(exec->nccl_id, rank, world, dev));
            // ownership of the transport passes to the engine (released by it on failure too)
            mfd::Transport* t = tr.release();
            c->eng.reset(prec == 32 ? mfd::make_engine<float>(*grid, *mat, *terms, *stepper, dev, rank, world, t)
                                    : mfd::make_engine<double>(*grid, *mat, *terms, *stepper, dev, rank, world, t));
        }
        *out = c.release();
    });
}

void mfd_destroy(mfd_ctx* ctx) { delete ctx; }

const char* mfd_last_error(const mfd_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

#define ENG(ctx) (ctx)->eng

mfd_status mfd_set_m_f64(mfd_ctx* c, const double* x, const double* y, const double* z) {
    return guard(c, [&] { ENG(c)->set_m(x, y, z); });
}
mfd_status mfd_get_m_f64(mfd_ctx* c, double* x, double* y, double* z) {
    return guard(c, [&] { ENG(c)->get_m(x, y, z); });
}
mfd_status mfd_set_m_f32(mfd_ctx* c, const float* x, const float* y, const float* z) {
    return guard(c, [&] { ENG(c)->set_m32(x, y, z); });
}
mfd_status mfd_get_m_f32(mfd_ctx* c, float* x, float* y, float* z) {
    return guard(c, [&] { ENG(c)->get_m32(x, y, z); });
}
mfd_status mfd_stage_m_f64(mfd_ctx* c, const double* x, const double* y, const double* z) {
    return guard(c, [&] { ENG(c)->stage_m(x, y, z, 64); });
}
mfd_status mfd_stage_m_f32(mfd_ctx* c, const float* x, const float* y, const float* z) {
    return guard(c, [&] { ENG(c)->stage_m(x, y, z, 32); });
}
mfd_status mfd_set_m_uniform(mfd_ctx* c, const double dir[3]) {
    return guard(c, [&] {
        const double n = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
        if (std::abs(n - 1.0) > 1e-9)
            throw mfd::Error(MFD_EINVAL, "makeUniformState: direction must be a unit vector");
        ENG(c)->set_uniform(dir);
    });
}
mfd_status mfd_set_m_vortex(mfd_ctx* c, int axis) {
    return guard(c, [&] { ENG(c)->set_vortex(axis); });
}
mfd_status mfd_set_time(mfd_ctx* c, double t, long step) {
    return guard(c, [&] {
        ENG(c)->t = t;
        ENG(c)->stepno = step;
    });
}
mfd_status mfd_get_time(const mfd_ctx* c, double* t, long* step) {
    *t = c->eng->t;
    *step = c->eng->stepno;
    return MFD_OK;
}
mfd_status mfd_effective_field_f64(mfd_ctx* c, double* x, double* y, double* z) {
    return guard(c, [&] { ENG(c)->field(1, x, y, z); });
}
mfd_status mfd_demag_field_f64(mfd_ctx* c, double* x, double* y, double* z) {
    return guard(c, [&] { ENG(c)->field(2, x, y, z); });
}
mfd_status mfd_effective_field_f32(mfd_ctx* c, float* x, float* y, float* z) {
    return guard(c, [&] { ENG(c)->field32(1, x, y, z); });
}
mfd_status mfd_demag_field_f32(mfd_ctx* c, float* x, float* y, float* z) {
    return guard(c, [&] { ENG(c)->field32(2, x, y, z); });
}
mfd_status mfd_set_stepper(mfd_ctx* c, const mfd_stepper* s) {
    return guard(c, [&] {
        if (!s) throw mfd::Error(MFD_EINVAL, "mfd_set_stepper: null argument");
        if (!(s->dt > 0)) throw mfd::Error(MFD_EINVAL, "StepperConfig: dt must be > 0");
        if (s->renorm_every < 1) throw mfd::Error(MFD_EINVAL, "StepperConfig: renormalizeEvery must be >= 1");
        if (!(s->torque_tol_deg_per_ns > 0))
            throw mfd::Error(MFD_EINVAL, "StepperConfig: torque tolerance must be > 0");
        c->st = *s;
        ENG(c)->set_stepper(*s);
    });
}
mfd_status mfd_step(mfd_ctx* c, long n, double* last, double* all) {
    return guard(c, [&] {
        if (n < 0) throw mfd::Error(MFD_EINVAL, "mfd_step: nsteps must be >= 0");
        ENG(c)->step(n, last, all);
    });
}
mfd_status mfd_step_async(mfd_ctx* c, long n) { return guard(c, [&] { ENG(c)->step_async(n); }); }
mfd_status mfd_prepare_async(mfd_ctx* c, long n, long* launches) {
    return guard(c, [&] {
        const long k = ENG(c)->prepare_async(n);
        if (launches) *launches = k;
    });
}
mfd_status mfd_sync(mfd_ctx* c) { return guard(c, [&] { ENG(c)->sync(); }); }
mfd_status mfd_sync_torque(mfd_ctx* c, double* last_torque) {
    return guard(c, [&] { *last_torque = ENG(c)->sync_torque(); });
}
void* mfd_stream(mfd_ctx* c) { return (void*)c->eng->stream(); }
mfd_status mfd_relax(mfd_ctx* c, int* converged, mfd_sample_cb cb, void* user) {
    return guard(c, [&] { *converged = ENG(c)->relax(cb, user) ? 1 : 0; });
}
mfd_status mfd_sample_now(mfd_ctx* c, mfd_sample* out) {
    return guard(c, [&] { *out = ENG(c)->sample_now(); });
}
mfd_status mfd_reduced_mean(mfd_ctx* c, double m[3]) {
    return guard(c, [&] {
        const mfd_sample s = ENG(c)->sample_now();
        m[0] = s.m[0];
        m[1] = s.m[1];
        m[2] = s.m[2];
    });
}
mfd_status mfd_energies(mfd_ctx* c, double e[5]) {
    return guard(c, [&] {
        const mfd_sample s = ENG(c)->sample_now();
        e[0] = s.e_exchange;
        e[1] = s.e_anisotropy;
        e[2] = s.e_demag;
        e[3] = s.e_zeeman;
        e[4] = s.e_total;
    });
}
mfd_status mfd_last_step_timing(mfd_ctx* c, double ms[7]) { return guard(c, [&] { ENG(c)->timing(ms); }); }
double mfd_stability_dt_limit(const mfd_material* m, const mfd_grid* g) {
    // dynamics.hpp:39-45
    if (m->A <= 0) return INFINITY;
    const double dmin = std::fmin(std::fmin(g->dx, g->dy), g->dz);
    return (1.0 + m->alpha * m->alpha) * m->Ms * dmin * dmin / (m->gamma * 4.0 * m->A * 10.0);
}
mfd_status mfd_set_demag_octant_f64(mfd_ctx* c, const double* o) { return guard(c, [&] { ENG(c)->set_octant(o); }); }
mfd_status mfd_get_demag_octant_f64(mfd_ctx* c, double* o) { return guard(c, [&] { ENG(c)->get_octant(o); }); }
mfd_status mfd_get_spectrum_octant_f64(mfd_ctx* c, double* o) { return guard(c, [&] { ENG(c)->get_spectrum(o); }); }
mfd_status mfd_debug_stage_f64(mfd_ctx* c, int stage, double* out) {
    return guard(c, [&] { ENG(c)->debug_stage(stage, out); });
}
mfd_status mfd_device_state(mfd_ctx* c, void** m, long long* n, int* prec) {
    return guard(c, [&] {
        *m = ENG(c)->state_ptr();
        *n = ENG(c)->ncell;
        *prec = ENG(c)->precision;
    });
}
int mfd_launches_per_step(const mfd_ctx* c) { return c->eng->launches_per_step(); }
long long mfd_debug_guard_check(mfd_ctx* c) {
    long long r = -2;
    guard(c, [&] { r = ENG(c)->guard_check(); });
    return r;
}
int mfd_debug_variants(const mfd_ctx* c, char* buf, int len) {
    const std::string v = c->eng->variants();
    if (buf && len > 0) {
        const size_t n = std::min<size_t>(v.size(), (size_t)len - 1);
        std::memcpy(buf, v.data(), n);
        buf[n] = 0;
    }
    return (int)v.size() + 1;
}
double mfd_model_bytes_per_step(const mfd_ctx* c) { return c->eng->model_bytes(); }

} // extern "C"
