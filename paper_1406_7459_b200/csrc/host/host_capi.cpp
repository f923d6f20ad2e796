// C ABI of the host formats (include/mfd_host.h).  Nothing throws across
// the boundary: exceptions become a status + thread-local message.
#include <cstring>
#include <new>

#include "host_common.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        return MFD_OK;
    } catch (const mfd::host::ConfigError& e) {
        g_err = e.what();
        return MFD_ECONFIG;
    } catch (const mfd::host::IoError& e) {
        g_err = e.what();
        return MFD_EIO;
    } catch (const std::bad_alloc&) {
        g_err = "std::bad_alloc";
        return MFD_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MFD_EINVAL;
    }
}

void put_lines(const std::vector<std::string>& lines, char* buf, size_t cap) {
    if (!buf || cap == 0) return;
    std::string all;
    for (const auto& l : lines) all += l + "\n";
    const size_t n = all.size() < cap - 1 ? all.size() : cap - 1;
    std::memcpy(buf, all.data(), n);
    buf[n] = 0;
}
} // namespace

extern "C" {

void mfd_spec_default(mfd_spec* out) {
    if (out) mfd::host::spec_default(*out);
}

int mfd_config_parse(const char* text, mfd_spec* out, char* defaults, size_t cap) {
    return guard([&] {
        if (!text || !out) throw std::invalid_argument("mfd_config_parse: null argument");
        std::vector<std::string> d;
        *out = mfd::host::parse_config(text, &d);
        put_lines(d, defaults, cap);
    });
}

int mfd_config_load(const char* path, mfd_spec* out, char* defaults, size_t cap) {
    return guard([&] {
        if (!path || !out) throw std::invalid_argument("mfd_config_load: null argument");
        std::vector<std::string> d;
        *out = mfd::host::load_config(path, &d);
        put_lines(d, defaults, cap);
    });
}

long mfd_config_format(const mfd_spec* spec, char* buf, size_t cap) {
    if (!spec) return -1;
    const std::string s = mfd::host::format_config(*spec);
    if (buf && cap > 0) {
        const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return (long)s.size();
}

int mfd_dump_write(const char* path, const mfd_grid* grid, double Ms, int precision_bits, const double* mx,
                   const double* my, const double* mz) {
    return guard([&] {
        if (!path || !grid || !mx || !my || !mz) throw std::invalid_argument("mfd_dump_write: null argument");
        mfd::host::write_dump(path, *grid, Ms, precision_bits, mx, my, mz);
    });
}

int mfd_dump_read_header(const char* path, mfd_grid* grid, double* Ms, int* precision_bits) {
    return guard([&] {
        if (!path) throw std::invalid_argument("mfd_dump_read_header: null path");
        const auto d = mfd::host::read_dump(path, true);
        if (grid) *grid = d.grid;
        if (Ms) *Ms = d.Ms;
        if (precision_bits) *precision_bits = d.precision_bits;
    });
}

int mfd_dump_read(const char* path, mfd_grid* grid, double* Ms, int* precision_bits, double* mx, double* my,
                  double* mz) {
    return guard([&] {
        if (!path || !mx || !my || !mz) throw std::invalid_argument("mfd_dump_read: null argument");
        const auto d = mfd::host::read_dump(path, false);
        if (grid) *grid = d.grid;
        if (Ms) *Ms = d.Ms;
        if (precision_bits) *precision_bits = d.precision_bits;
        std::memcpy(mx, d.mx.data(), d.mx.size() * sizeof(double));
        std::memcpy(my, d.my.data(), d.my.size() * sizeof(double));
        std::memcpy(mz, d.mz.data(), d.mz.size() * sizeof(double));
    });
}

int mfd_trajectory_csv_write(const char* path, const mfd_sample* samples, long n) {
    return guard([&] {
        if (!path || (n > 0 && !samples)) throw std::invalid_argument("mfd_trajectory_csv_write: null argument");
        mfd::host::write_trajectory_csv(path, samples, n);
    });
}

int mfd_bench_csv_write(const char* path, const mfd_bench_row* rows, long n) {
    return guard([&] {
        if (!path || (n > 0 && !rows)) throw std::invalid_argument("mfd_bench_csv_write: null argument");
        mfd::host::write_bench_csv(path, rows, n);
    });
}

const char* mfd_host_last_error(void) { return g_err.c_str(); }

} // extern "C"
