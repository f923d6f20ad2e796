// Shared declarations of the host-side formats (config, IO, CLI support).
#pragma once
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/mfd_host.h"

namespace mfd::host {

struct ConfigError : std::runtime_error {   // config.hpp:21-23
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {       // io.hpp:14-16
    using std::runtime_error::runtime_error;
};

// %.17g: the reference's round-trip number format (io.cpp:9-13, config.cpp:66-70)
inline std::string g17(double x) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", x);
    return buf;
}

void spec_default(mfd_spec& s);
mfd_spec parse_config(const std::string& text, std::vector<std::string>* defaults);
std::string format_config(const mfd_spec& s);
mfd_spec load_config(const std::string& path, std::vector<std::string>* defaults);

struct Dump {
    mfd_grid grid{};
    double Ms = 0;
    int precision_bits = 64;
    std::vector<double> mx, my, mz;
};
void write_dump(const std::string& path, const mfd_grid& g, double Ms, int precision_bits, const double* mx,
                const double* my, const double* mz);
Dump read_dump(const std::string& path, bool header_only);
void write_trajectory_csv(const std::string& path, const mfd_sample* s, long n);
void write_bench_csv(const std::string& path, const mfd_bench_row* rows, long n);

} // namespace mfd::host
