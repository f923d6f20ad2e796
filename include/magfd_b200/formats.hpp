// Header-only C++ shim over include/mfd_host.h: the reference's config and IO
// surface (config.hpp:97-103, io.hpp:21-42) with its exception types, so
// drivers that load magfd configs and write dumps / trajectory CSVs keep their
// code and messages when they move to the B200 engine.
//
//   magfd::parseConfig / loadConfigFile / formatConfig -> parse_config / load_config / format_config
//   magfd::io::writeFieldDump / readFieldDump         -> write_field_dump / read_field_dump
//   magfd::io::writeTrajectoryCsv                     -> write_trajectory_csv
//   makeVortexState (state.hpp:83-108)                -> Simulation<T>::set_vortex (device)
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "../mfd_host.h"
#include "simulation.hpp"

namespace magfd_b200 {

struct ConfigError : std::runtime_error {   // config.hpp:21-23
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {       // io.hpp:14-16
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void host_check(int st) {
    if (st == 0) return;
    const char* m = mfd_host_last_error();
    if (st == MFD_ECONFIG) throw ConfigError(m);
    if (st == MFD_EIO) throw IoError(m);
    raise(static_cast<mfd_status>(st), m);
}
inline std::vector<std::string> split_lines(const std::vector<char>& buf) {
    std::vector<std::string> out;
    std::string cur;
    for (const char* p = buf.data(); *p; ++p) {
        if (*p == '\n') { out.push_back(cur); cur.clear(); }
        else cur += *p;
    }
    return out;
}
} // namespace detail

inline mfd_spec parse_config(const std::string& text, std::vector<std::string>* applied_defaults = nullptr) {
    mfd_spec s;
    std::vector<char> d(1 << 16);
    detail::host_check(mfd_config_parse(text.c_str(), &s, d.data(), d.size()));
    if (applied_defaults) *applied_defaults = detail::split_lines(d);
    return s;
}

inline mfd_spec load_config(const std::string& path, std::vector<std::string>* applied_defaults = nullptr) {
    mfd_spec s;
    std::vector<char> d(1 << 16);
    detail::host_check(mfd_config_load(path.c_str(), &s, d.data(), d.size()));
    if (applied_defaults) *applied_defaults = detail::split_lines(d);
    return s;
}

inline std::string format_config(const mfd_spec& s) {
    const long n = mfd_config_format(&s, nullptr, 0);
    std::string out(static_cast<std::size_t>(n) + 1, '\0');
    mfd_config_format(&s, out.data(), out.size());
    out.resize(static_cast<std::size_t>(n));
    return out;
}

inline void write_field_dump(const std::string& path, const HostField<double>& M, const mfd_grid& g, double Ms,
                             int precision_bits) {
    detail::host_check(mfd_dump_write(path.c_str(), &g, Ms, precision_bits, M.x.data(), M.y.data(), M.z.data()));
}

struct FieldDump {   // io.hpp:21-26
    mfd_grid grid{};
    double Ms = 0;
    int precision_bits = 64;
    HostField<double> M;
};

inline FieldDump read_field_dump(const std::string& path) {
    FieldDump d;
    detail::host_check(mfd_dump_read_header(path.c_str(), &d.grid, &d.Ms, &d.precision_bits));
    d.M = HostField<double>(static_cast<std::size_t>(d.grid.nx) * d.grid.ny * d.grid.nz);
    detail::host_check(
        mfd_dump_read(path.c_str(), &d.grid, &d.Ms, &d.precision_bits, d.M.x.data(), d.M.y.data(), d.M.z.data()));
    return d;
}

inline void write_trajectory_csv(const std::string& path, const std::vector<Sample>& log) {
    std::vector<mfd_sample> rows(log.size());
    for (std::size_t i = 0; i < log.size(); ++i) {
        const Sample& s = log[i];
        rows[i] = mfd_sample{s.step, s.t, {s.m[0], s.m[1], s.m[2]}, s.e_exchange, s.e_anisotropy, s.e_demag,
                             s.e_zeeman, s.e_total, s.max_torque_deg_per_ns};
    }
    detail::host_check(mfd_trajectory_csv_write(path.c_str(), rows.data(), static_cast<long>(rows.size())));
}

} // namespace magfd_b200
