// Reference-style host driver over include/magfd_b200/formats.hpp (no GPU
// needed): parse / format a config, dump round trip, trajectory CSV, errors.
#include <cstdio>
#include <string>
#include <vector>

#include "magfd_b200/formats.hpp"

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    std::vector<std::string> defaults;
    const mfd_spec s = magfd_b200::parse_config(
        "grid.nx = 3\ngrid.ny = 2\ngrid.nz = 1\ngrid.dx = 1e-9\ngrid.dy = 1e-9\ngrid.dz = 1e-9\nmaterial.Ms = 8e5\n"
        "init.kind = vortex\n", &defaults);
    std::printf("defaults %zu\n", defaults.size());
    std::printf("%s", magfd_b200::format_config(s).c_str());
    magfd_b200::HostField<double> M(6);
    for (int c = 0; c < 6; ++c) { M.x[c] = 0.1 * c; M.y[c] = 1.0 / (c + 3); M.z[c] = -c * 1e5; }
    magfd_b200::write_field_dump(dir + "/d.dump", M, s.grid, s.material.Ms, 64);
    const auto d = magfd_b200::read_field_dump(dir + "/d.dump");
    bool same = d.M.x == M.x && d.M.y == M.y && d.M.z == M.z && d.grid.nx == 3;
    std::printf("dump round trip %s\n", same ? "bitwise" : "DIFFERS");
    magfd_b200::write_trajectory_csv(dir + "/t.csv", {magfd_b200::Sample{0, 0.0, {1, 0, 0}, 1, 2, 3, 4, 10, 0.5}});
    try {
        magfd_b200::parse_config("grid.nx = 0\n");
    } catch (const magfd_b200::ConfigError& e) {
        std::printf("ConfigError %s\n", e.what());
    }
    try {
        magfd_b200::read_field_dump(dir + "/missing.dump");
    } catch (const magfd_b200::IoError& e) {
        std::printf("IoError %s\n", e.what());
    }
    return 0;
}
