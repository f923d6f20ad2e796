/*
 * mfd.h — C ABI of libmagfd_b200.so, the B200 (sm_100a) engine for the
 * per-step effective-field + LLG hot path of the reference solver "magfd"
 * (/root/reference/proj, arXiv:1406.7459).
 *
 * The reference has no FFI; its drop-in seams are C++ classes.  Each entry
 * point below replaces one reference call (file:line in the reference):
 *
 *   mfd_create               Simulation<T>::Simulation (sim.hpp:17-24): builds the
 *                            EffectiveFieldProvider + DemagConvolution (fields.hpp:207-215,
 *                            demag.hpp:184-188) — tensor (newell.cpp:188-209,
 *                            demag.hpp:49-90) and spectra (demag.hpp:105-119) on device
 *   mfd_set_m_* / mfd_get_m_* Simulation<T>::state().M read/write (sim.hpp:29-30,
 *                            state.hpp:23-32); host SoA, N values per component, A/m
 *   mfd_set_time/mfd_get_time SimState<T>::t / ::step (state.hpp:25-26)
 *   mfd_effective_field_*    EffectiveFieldProvider<T>::compute (fields.hpp:220-253)
 *   mfd_demag_field_*        DemagConvolution<T>::field / lastDemagField
 *                            (demag.hpp:194-251, fields.hpp:264-268)
 *   mfd_step                 Simulation<T>::step (sim.hpp:33-42), n times; returns the
 *                            pre-step max torque of the last step
 *   mfd_relax                Simulation<T>::relax -> dynamics::relax (dynamics.hpp:157-198)
 *   mfd_sample               Simulation<T>::sampleNow (sim.hpp:45-55)
 *   mfd_reduced_mean         reducedMean (state.hpp:113-124)
 *   mfd_energies             EffectiveFieldProvider<T>::energies (fields.hpp:256-262)
 *   mfd_last_step_timing     StepTiming phases of one step (backend.hpp:147-164)
 *   mfd_last_error           text of the reference exception the call maps to
 *
 * Conventions (the reference's, SPEC.md / README): SI units, M and H in A/m,
 * H = K * M with K = -N, cell index i + nx*(j + ny*k), padded FFT sizes
 * nextPow2(2n) (n = 1 -> 2).  M stays resident on the device between calls;
 * host pointers are borrowed for the duration of a call only.  No call
 * throws; errors come back as mfd_status with the reference message in
 * mfd_last_error().  One context must not be used by two threads at once
 * (DemagConvolution "must not run concurrently with itself", demag.hpp:176).
 */
#ifndef MFD_H
#define MFD_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mfd_ctx mfd_ctx;

typedef enum {
    MFD_OK = 0,
    MFD_EINVAL = 1,     /* std::invalid_argument (grid.hpp:19-22, material.hpp:20-28, ...) */
    MFD_ENONFINITE = 2, /* std::runtime_error from eulerUpdate (dynamics.hpp:115-117) */
    MFD_ELOGIC = 3,     /* std::logic_error (fields.hpp:264-267) */
    MFD_ENOMEM = 4,     /* std::bad_alloc */
    MFD_ECUDA = 5,      /* device failure / no sm_100 device */
    MFD_ENCCL = 6       /* multi-GPU transport failure */
} mfd_status;

/* Grid (grid.hpp:12-48). */
typedef struct { int nx, ny, nz; double dx, dy, dz; } mfd_grid;

/* MaterialParams (material.hpp:12-33). */
typedef struct { double A, Ku, Ms, alpha, gamma; double easy_axis[3]; } mfd_material;

/* FieldConfig (fields.hpp:193-199). */
typedef struct { int exchange, anisotropy, demag, zeeman; double h_ext[3]; } mfd_terms;

/* StepperConfig (dynamics.hpp:18-32). */
typedef struct {
    double dt;
    int renorm_every;
    long max_steps;
    double torque_tol_deg_per_ns;
    long sample_every;
} mfd_stepper;

/* Execution: precision 32 (float) or 64 (double); device ordinal; z-slab
 * decomposition over `world` ranks.
 *   world = 1                    single GPU (the reference has no distribution)
 *   world > 1, virtual_ranks = 1 all slabs on `device` (correctness harness)
 *   world > 1, virtual_ranks = 0 one process per GPU, NCCL over NVLink; every rank
 *                                passes the same nccl_id (mfd_nccl_unique_id on rank
 *                                0, broadcast by the caller).  In this mode
 *                                mfd_set_m_* / mfd_get_m_* move the rank's slab
 *                                (planes [rank*nz/world, (rank+1)*nz/world)); all
 *                                other calls are collective.
 * nz must be divisible by world. */
typedef struct {
    int precision_bits;
    int device;
    int world;
    int rank;
    int virtual_ranks;
    /* world > 1, virtual_ranks = 0: 0 = NCCL over NVLink (production); 1 = host-staged
     * shared-memory transport (test harness: the one-process-per-GPU path with several
     * processes on ONE GPU, which NCCL refuses; the first 16 bytes of nccl_id name the
     * segment, any random bytes shared by the ranks). */
    int transport;
    int reserved[2];
    unsigned char nccl_id[128];
} mfd_exec;

/* NCCL unique id for a multi-GPU context (call on rank 0). */
mfd_status mfd_nccl_unique_id(unsigned char id[128]);

/* TrajectorySample (dynamics.hpp:138-144). */
typedef struct {
    long step;
    double t;
    double m[3];
    double e_exchange, e_anisotropy, e_demag, e_zeeman, e_total;
    double torque_deg_per_ns;
} mfd_sample;

typedef void (*mfd_sample_cb)(const mfd_sample* s, void* user);

mfd_status mfd_create(const mfd_grid* grid, const mfd_material* mat, const mfd_terms* terms,
                      const mfd_stepper* stepper, const mfd_exec* exec, mfd_ctx** out);
void mfd_destroy(mfd_ctx* ctx);

mfd_status mfd_set_m_f64(mfd_ctx* ctx, const double* mx, const double* my, const double* mz);
mfd_status mfd_get_m_f64(mfd_ctx* ctx, double* mx, double* my, double* mz);
mfd_status mfd_set_m_f32(mfd_ctx* ctx, const float* mx, const float* my, const float* mz);
mfd_status mfd_get_m_f32(mfd_ctx* ctx, float* mx, float* my, float* mz);
/* Overlapped state upload: queue M from host memory on a copy stream and return at
 * once; the next call that reads the state (step, step_async, relax, fields, get_m, ...)
 * installs every queued state in order (the last one wins).  With pinned host arrays
 * the transfer overlaps a step already enqueued by mfd_step_async (the arrays must stay
 * untouched until the installing call returns); at most two states in flight.
 * Pipelined use: stage(in_0); for each i: step_async(1); stage(in_{i+1}); sync_torque. */
mfd_status mfd_stage_m_f64(mfd_ctx* ctx, const double* mx, const double* my, const double* mz);
mfd_status mfd_stage_m_f32(mfd_ctx* ctx, const float* mx, const float* my, const float* mz);
/* Uniform initial state M = Ms * dir (makeUniformState, state.hpp:71-78). */
mfd_status mfd_set_m_uniform(mfd_ctx* ctx, const double dir[3]);

mfd_status mfd_set_time(mfd_ctx* ctx, double t, long step);
mfd_status mfd_get_time(const mfd_ctx* ctx, double* t, long* step);

mfd_status mfd_effective_field_f64(mfd_ctx* ctx, double* hx, double* hy, double* hz);
mfd_status mfd_demag_field_f64(mfd_ctx* ctx, double* hx, double* hy, double* hz);
/* The same in float (the f32 engine copies its fields out unconverted). */
mfd_status mfd_effective_field_f32(mfd_ctx* ctx, float* hx, float* hy, float* hz);
mfd_status mfd_demag_field_f32(mfd_ctx* ctx, float* hx, float* hy, float* hz);

/* Replace the StepperConfig (dt, renormalizeEvery, maxSteps, torque tolerance,
 * sampleEvery) of a live context (dynamics::relax takes its config per call,
 * dynamics.hpp:157-160); validation as StepperConfig::validate (dynamics.hpp:26-30). */
mfd_status mfd_set_stepper(mfd_ctx* ctx, const mfd_stepper* stepper);

/* nsteps x Simulation::step; *last_torque = pre-step max torque (deg/ns) of the last
 * step; torques (optional, nsteps entries) receives every step's value. */
mfd_status mfd_step(mfd_ctx* ctx, long nsteps, double* last_torque, double* torques);

/* dynamics::relax with the context's stepper config.  Samples are delivered through
 * on_sample in order (may be NULL); *converged set on return. */
mfd_status mfd_relax(mfd_ctx* ctx, int* converged, mfd_sample_cb on_sample, void* user);

mfd_status mfd_sample_now(mfd_ctx* ctx, mfd_sample* out);
mfd_status mfd_reduced_mean(mfd_ctx* ctx, double m[3]);
mfd_status mfd_energies(mfd_ctx* ctx, double e[5]);

/* One real Simulation::step, instrumented: device time of its passes, ms, and its torque:
 * [pad+forward x, forward y, z + multiply, inverse y, inverse x + local + integrate, total,
 *  pre-step max torque in deg/ns]. */
mfd_status mfd_last_step_timing(mfd_ctx* ctx, double ms[7]);

/* Stability heuristic (dynamics.hpp:39-45). */
double mfd_stability_dt_limit(const mfd_material* mat, const mfd_grid* grid);

const char* mfd_last_error(const mfd_ctx* ctx);
const char* mfd_version(void);

/* ---- test / bench hooks (not part of the reference surface) ---- */
/* Replace the device tensor octant by host-supplied entries (layout [6][nz][ny][nx],
 * K convention) and re-transform; lets tests feed the reference's own tensor. */
mfd_status mfd_set_demag_octant_f64(mfd_ctx* ctx, const double* octant6);
/* Read the device tensor octant (fp64 entries, [6][nz][ny][nx]). */
mfd_status mfd_get_demag_octant_f64(mfd_ctx* ctx, double* octant6);
/* Read the real tensor spectrum octant as T widened to f64, layout [6][Py/2+1][Pz/2+1][Px/2+1]. */
mfd_status mfd_get_spectrum_octant_f64(mfd_ctx* ctx, double* out);
/* Run the pipeline up to pass `stage` (1..4) on the current M and copy the intermediate
 * spectrum (1,4: [3][nz][ny][Hp]; 2,3: [3][nz][Py][Hp], Hp = pitch) as interleaved (re, im). */
mfd_status mfd_debug_stage_f64(mfd_ctx* ctx, int stage, double* out);
/* Device pointers of the resident state for zero-copy benchmarking:
 * m = current M (3 x N SoA of float or double). */
mfd_status mfd_device_state(mfd_ctx* ctx, void** m, long long* ncell, int* precision_bits);
/* Run nsteps via CUDA graph on the context stream without host sync; pair with mfd_sync. */
mfd_status mfd_step_async(mfd_ctx* ctx, long nsteps);
/* Capture (without running) the CUDA graphs the next mfd_step_async(ctx, nsteps) will
 * launch, so a timed region contains no capture / instantiation; *launches (may be
 * NULL) = the kernel launches those graphs contain. */
mfd_status mfd_prepare_async(mfd_ctx* ctx, long nsteps, long* launches);
mfd_status mfd_sync(mfd_ctx* ctx);
/* mfd_sync + the pre-step max torque (deg/ns) of the last step of the last mfd_step_async. */
mfd_status mfd_sync_torque(mfd_ctx* ctx, double* last_torque);
/* The context's CUDA stream (cudaStream_t) for event timing. */
void* mfd_stream(mfd_ctx* ctx);
/* Kernel launches per step of the hot path (for bench accounting). */
int mfd_launches_per_step(const mfd_ctx* ctx);
/* Algorithmic HBM bytes per step of the 5-pass model. */
double mfd_model_bytes_per_step(const mfd_ctx* ctx);
/* Kernel template instantiations this context has enqueued since creation, one per
 * line ("K5 k_c2r_x_llg_v<f32,256,SUMS=0,RS=0,FWD=1,MULTI=0>", ...).  Copies at most
 * len-1 bytes + NUL into buf (may be NULL) and returns the full length + 1. */
int mfd_debug_variants(const mfd_ctx* ctx, char* buf, int len);
/* With MFD_GUARD=1 in the environment at mfd_create, every device buffer is bracketed by
 * 4 KB guard bands of 0xA5; returns the number of guard bytes overwritten so far
 * (-1: guards off, -2: error).  A write-overrun check for the tests. */
long long mfd_debug_guard_check(mfd_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* MFD_H */
