/*
 * mfd_host.h — host-side formats around the B200 hot path (SURVEY.md section 8f,
 * rows f3 / f4), exported by the same libmagfd_b200.so as mfd.h:
 *
 *   mfd_config_parse / _load   parseConfig / loadConfigFile (config.hpp:97-103,
 *                              config.cpp:76-246, 278-284): the `key = value` SimSpec format,
 *                              same validation order and error texts ("config line N: ...")
 *   mfd_config_format          formatConfig (config.cpp:248-276): canonical rendering,
 *                              parse(format(s)) == s
 *   mfd_dump_write / _read     writeFieldDump / readFieldDump (io.hpp:21-30, io.cpp:18-100):
 *                              text dump v1, %.17g, bitwise f64 round trip
 *   mfd_trajectory_csv_write   writeTrajectoryCsv (io.hpp:40-42, io.cpp:102-117)
 *   mfd_bench_csv_write        the bench CSV of cli::cmdBench (cli.cpp:187-200)
 *   mfd_set_m_vortex           makeVortexState (state.hpp:83-108), evaluated on the device
 *                              in fp64 with the reference's operation order (bitwise)
 *
 * These are host code (no kernels) except mfd_set_m_vortex.  Calls without a
 * context report errors through mfd_host_last_error() (thread-local text of
 * the reference exception: ConfigError / IoError / std::invalid_argument).
 */
#ifndef MFD_HOST_H
#define MFD_HOST_H
#include <stddef.h>

#include "mfd.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Extra status codes of the host formats (mfd_status values 1..6 in mfd.h). */
#define MFD_ECONFIG 7 /* magfd::ConfigError (config.hpp:21-23) */
#define MFD_EIO 8     /* magfd::io::IoError (io.hpp:14-16) */

/* SimSpec (config.hpp:26-80), flat.  init_kind: 0 uniform, 1 vortex.
 * vortex_axis: 0 +x, 1 -x, 2 +y, 3 -y, 4 +z, 5 -z (SignedAxis, state.hpp:36).
 * backend_kind: 0 serial, 1 parallel (the reference's CPU backend; recorded and
 * round-tripped, the B200 engine ignores it).  sample_every lives in stepper. */
typedef struct {
    mfd_grid grid;
    mfd_material material;
    mfd_terms terms;
    mfd_stepper stepper;
    int init_kind;
    double init_direction[3];
    int vortex_axis;
    int backend_kind;
    unsigned threads;
    int precision_bits;
    char csv_path[1024];
    char dump_path[1024];
} mfd_spec;

/* SimSpec{} defaults (config.hpp:27-70). */
void mfd_spec_default(mfd_spec* out);
/* parseConfig(text, &appliedDefaults).  defaults (optional) receives the
 * `key = value` lines of the defaulted optional keys, '\n'-separated,
 * truncated to cap bytes (NUL-terminated). */
int mfd_config_parse(const char* text, mfd_spec* out, char* defaults, size_t cap);
int mfd_config_load(const char* path, mfd_spec* out, char* defaults, size_t cap);
/* formatConfig: writes up to cap bytes (NUL-terminated); returns the full length. */
long mfd_config_format(const mfd_spec* spec, char* buf, size_t cap);

/* Field dump v1.  precision_bits: 32 | 64 (the `# precision` header). */
int mfd_dump_write(const char* path, const mfd_grid* grid, double Ms, int precision_bits, const double* mx,
                   const double* my, const double* mz);
/* Header only (sizes for the caller's buffers). */
int mfd_dump_read_header(const char* path, mfd_grid* grid, double* Ms, int* precision_bits);
/* Full parse and validation; mx/my/mz hold nx*ny*nz values each. */
int mfd_dump_read(const char* path, mfd_grid* grid, double* Ms, int* precision_bits, double* mx, double* my,
                  double* mz);

int mfd_trajectory_csv_write(const char* path, const mfd_sample* samples, long n);

/* One row of the bench sweep, milliseconds (cli.hpp:30-34). */
typedef struct {
    int size;
    double ms_per_step, pad_ms, forward_fft_ms, spectral_multiply_ms, inverse_fft_ms, local_fields_ms,
        integrate_ms;
} mfd_bench_row;
int mfd_bench_csv_write(const char* path, const mfd_bench_row* rows, long n);

/* makeVortexState(grid, axis, Ms) into the context's M (device kernel). */
mfd_status mfd_set_m_vortex(mfd_ctx* ctx, int axis);

const char* mfd_host_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MFD_HOST_H */
