// SimSpec config format: parser, canonical
// formatter and the applied-defaults echo of the reference's
// parseConfig / formatConfig / loadConfigFile (config.cpp:76-284).  Same
// accepted syntax, same validation order, same error texts; the spec lands in
// the flat C struct mfd_spec (include/mfd_host.h).
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_common.hpp"

namespace mfd::host {
namespace {

std::string trim(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && std::isspace((unsigned char)s[a])) ++a;
    while (b > a && std::isspace((unsigned char)s[b - 1])) --b;
    return s.substr(a, b - a);
}

struct LineError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Value readers; each throws LineError with the reference's wording
// (config.cpp:26-64).
double read_double(const std::string& v, const std::string& key) {
    size_t used = 0;
    double x = 0;
    try {
        x = std::stod(v, &used);
    } catch (const std::exception&) {
        throw LineError("malformed number for " + key + ": '" + v + "'");
    }
    if (!trim(v.substr(used)).empty()) throw LineError("trailing characters for " + key + ": '" + v + "'");
    if (!std::isfinite(x)) throw LineError("non-finite value for " + key);
    return x;
}

long read_long(const std::string& v, const std::string& key) {
    size_t used = 0;
    long x = 0;
    try {
        x = std::stol(v, &used);
    } catch (const std::exception&) {
        throw LineError("malformed integer for " + key + ": '" + v + "'");
    }
    if (!trim(v.substr(used)).empty()) throw LineError("trailing characters for " + key + ": '" + v + "'");
    return x;
}

bool read_bool(const std::string& v, const std::string& key) {
    static const char* yes[] = {"true", "on", "1"};
    static const char* no[] = {"false", "off", "0"};
    for (const char* s : yes)
        if (v == s) return true;
    for (const char* s : no)
        if (v == s) return false;
    throw LineError("malformed boolean for " + key + ": '" + v + "' (use true/false)");
}

void read_vec3(const std::string& v, const std::string& key, double out[3]) {
    std::istringstream is(v);
    double a = 0, b = 0, c = 0;
    std::string extra;
    if (!(is >> a >> b >> c)) throw LineError("malformed 3-vector for " + key + ": '" + v + "'");
    if (is >> extra) throw LineError("trailing characters for " + key + ": '" + v + "'");
    out[0] = a; out[1] = b; out[2] = c;
}

int read_pos_int(const std::string& v, const std::string& key) {
    const long x = read_long(v, key);
    if (x < 1) throw LineError(key + " must be >= 1, got " + v);
    return (int)x;
}
double read_pos_double(const std::string& v, const std::string& key) {
    const double x = read_double(v, key);
    if (!(x > 0)) throw LineError(key + " must be > 0, got " + v);
    return x;
}
double read_nonneg_double(const std::string& v, const std::string& key) {
    const double x = read_double(v, key);
    if (x < 0) throw LineError(key + " must be >= 0, got " + v);
    return x;
}

// Vec3 helpers with the reference's operation order (vec3.hpp:20-25).
double vnorm(const double v[3]) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }
void vnormalize(double v[3]) {
    const double n = vnorm(v);
    v[0] = v[0] / n; v[1] = v[1] / n; v[2] = v[2] / n;
}

const char* kAxisNames[6] = {"+x", "-x", "+y", "-y", "+z", "-z"};
int parse_axis(const std::string& s) {   // state.hpp:60-68: bare x/y/z mean +
    for (int a = 0; a < 6; ++a)
        if (s == kAxisNames[a]) return a;
    if (s == "x") return 0;
    if (s == "y") return 2;
    if (s == "z") return 4;
    return -1;
}

void copy_path(char* dst, const std::string& v) {
    if (v.size() >= 1024) throw LineError("path too long");
    std::memcpy(dst, v.c_str(), v.size() + 1);
}

// Key table, in the reference's canonical order (formatConfig, config.cpp:248-276).
enum class K {
    nx, ny, nz, dx, dy, dz, A, Ku, Ms, alpha, gamma, easy_axis, t_exch, t_anis, t_demag, t_zee, extern_field,
    init_kind, init_dir, init_axis, dt, max_steps, torque_tol, renorm, backend, threads, precision, csv, dump,
    sample_every
};
struct KeyDef { const char* name; K k; };
const KeyDef kKeys[] = {
    {"grid.nx", K::nx}, {"grid.ny", K::ny}, {"grid.nz", K::nz}, {"grid.dx", K::dx}, {"grid.dy", K::dy},
    {"grid.dz", K::dz}, {"material.A", K::A}, {"material.Ku", K::Ku}, {"material.Ms", K::Ms},
    {"material.alpha", K::alpha}, {"material.gamma", K::gamma}, {"material.easy_axis", K::easy_axis},
    {"terms.exchange", K::t_exch}, {"terms.anisotropy", K::t_anis}, {"terms.demag", K::t_demag},
    {"terms.zeeman", K::t_zee}, {"field.extern", K::extern_field}, {"init.kind", K::init_kind},
    {"init.direction", K::init_dir}, {"init.axis", K::init_axis}, {"stepper.dt", K::dt},
    {"stepper.max_steps", K::max_steps}, {"stepper.torque_tol", K::torque_tol},
    {"stepper.renorm_every", K::renorm}, {"backend.kind", K::backend}, {"backend.threads", K::threads},
    {"precision", K::precision}, {"output.csv", K::csv}, {"output.dump", K::dump},
    {"output.sample_every", K::sample_every},
};

void assign(mfd_spec& s, K k, const std::string& key, const std::string& v) {
    switch (k) {
        case K::nx: s.grid.nx = read_pos_int(v, key); break;
        case K::ny: s.grid.ny = read_pos_int(v, key); break;
        case K::nz: s.grid.nz = read_pos_int(v, key); break;
        case K::dx: s.grid.dx = read_pos_double(v, key); break;
        case K::dy: s.grid.dy = read_pos_double(v, key); break;
        case K::dz: s.grid.dz = read_pos_double(v, key); break;
        case K::A: s.material.A = read_nonneg_double(v, key); break;
        case K::Ku: s.material.Ku = read_double(v, key); break;
        case K::Ms: s.material.Ms = read_pos_double(v, key); break;
        case K::alpha: s.material.alpha = read_nonneg_double(v, key); break;
        case K::gamma: s.material.gamma = read_pos_double(v, key); break;
        case K::easy_axis: {
            double a[3];
            read_vec3(v, key, a);
            if (!(vnorm(a) > 0)) throw LineError("material.easy_axis must be nonzero");
            vnormalize(a);
            std::memcpy(s.material.easy_axis, a, sizeof a);
            break;
        }
        case K::t_exch: s.terms.exchange = read_bool(v, key); break;
        case K::t_anis: s.terms.anisotropy = read_bool(v, key); break;
        case K::t_demag: s.terms.demag = read_bool(v, key); break;
        case K::t_zee: s.terms.zeeman = read_bool(v, key); break;
        case K::extern_field: read_vec3(v, key, s.terms.h_ext); break;
        case K::init_kind:
            if (v == "uniform") s.init_kind = 0;
            else if (v == "vortex") s.init_kind = 1;
            else throw LineError("init.kind must be uniform or vortex, got '" + v + "'");
            break;
        case K::init_dir: {
            double d[3];
            read_vec3(v, key, d);
            if (!(vnorm(d) > 0)) throw LineError("init.direction must be nonzero");
            vnormalize(d);
            std::memcpy(s.init_direction, d, sizeof d);
            break;
        }
        case K::init_axis: {
            const int a = parse_axis(v);
            if (a < 0) throw LineError("init.axis must be one of +x -x +y -y +z -z, got '" + v + "'");
            s.vortex_axis = a;
            break;
        }
        case K::dt: s.stepper.dt = read_pos_double(v, key); break;
        case K::max_steps:
            s.stepper.max_steps = read_long(v, key);
            if (s.stepper.max_steps < 0) throw LineError("stepper.max_steps must be >= 0");
            break;
        case K::torque_tol: s.stepper.torque_tol_deg_per_ns = read_pos_double(v, key); break;
        case K::renorm: s.stepper.renorm_every = read_pos_int(v, key); break;
        case K::backend:
            if (v == "serial") s.backend_kind = 0;
            else if (v == "parallel") s.backend_kind = 1;
            else throw LineError("backend.kind must be serial or parallel, got '" + v + "'");
            break;
        case K::threads: {
            const long t = read_long(v, key);
            if (t < 0) throw LineError("backend.threads must be >= 0");
            s.threads = (unsigned)t;
            break;
        }
        case K::precision:
            if (v == "f32") s.precision_bits = 32;
            else if (v == "f64") s.precision_bits = 64;
            else throw LineError("precision must be f32 or f64, got '" + v + "'");
            break;
        case K::csv: copy_path(s.csv_path, v); break;
        case K::dump: copy_path(s.dump_path, v); break;
        case K::sample_every: s.stepper.sample_every = read_pos_int(v, key); break;
    }
}

std::string vec_text(const double v[3]) { return g17(v[0]) + " " + g17(v[1]) + " " + g17(v[2]); }
const char* tf(int b) { return b ? "true" : "false"; }

// Value text of one key in the canonical rendering.
std::string value_text(const mfd_spec& s, K k) {
    switch (k) {
        case K::nx: return std::to_string(s.grid.nx);
        case K::ny: return std::to_string(s.grid.ny);
        case K::nz: return std::to_string(s.grid.nz);
        case K::dx: return g17(s.grid.dx);
        case K::dy: return g17(s.grid.dy);
        case K::dz: return g17(s.grid.dz);
        case K::A: return g17(s.material.A);
        case K::Ku: return g17(s.material.Ku);
        case K::Ms: return g17(s.material.Ms);
        case K::alpha: return g17(s.material.alpha);
        case K::gamma: return g17(s.material.gamma);
        case K::easy_axis: return vec_text(s.material.easy_axis);
        case K::t_exch: return tf(s.terms.exchange);
        case K::t_anis: return tf(s.terms.anisotropy);
        case K::t_demag: return tf(s.terms.demag);
        case K::t_zee: return tf(s.terms.zeeman);
        case K::extern_field: return vec_text(s.terms.h_ext);
        case K::init_kind: return s.init_kind == 0 ? "uniform" : "vortex";
        case K::init_dir: return vec_text(s.init_direction);
        case K::init_axis: return kAxisNames[s.vortex_axis < 0 || s.vortex_axis > 5 ? 4 : s.vortex_axis];
        case K::dt: return g17(s.stepper.dt);
        case K::max_steps: return std::to_string(s.stepper.max_steps);
        case K::torque_tol: return g17(s.stepper.torque_tol_deg_per_ns);
        case K::renorm: return std::to_string(s.stepper.renorm_every);
        case K::backend: return s.backend_kind == 0 ? "serial" : "parallel";
        case K::threads: return std::to_string(s.threads);
        case K::precision: return s.precision_bits == 32 ? "f32" : "f64";
        case K::csv: return s.csv_path;
        case K::dump: return s.dump_path;
        case K::sample_every: return std::to_string(s.stepper.sample_every);
    }
    return "";
}

} // namespace

void spec_default(mfd_spec& s) {
    std::memset(&s, 0, sizeof s);
    s.material.alpha = 1.0;
    s.material.gamma = 1.760859630e11;   // constants::gamma_e (constants.hpp:16)
    s.material.easy_axis[2] = 1.0;
    s.terms.exchange = s.terms.anisotropy = s.terms.demag = s.terms.zeeman = 1;
    s.init_kind = 0;
    s.init_direction[2] = 1.0;
    s.vortex_axis = 4;                   // +z
    s.stepper.dt = 1e-14;
    s.stepper.max_steps = 500000;
    s.stepper.torque_tol_deg_per_ns = 0.01;
    s.stepper.renorm_every = 1;
    s.stepper.sample_every = 100;
    s.backend_kind = 0;
    s.threads = 0;
    s.precision_bits = 64;
    std::strcpy(s.csv_path, "trajectory.csv");
    std::strcpy(s.dump_path, "final_state.dump");
}

mfd_spec parse_config(const std::string& text, std::vector<std::string>* defaults) {
    mfd_spec s;
    spec_default(s);
    std::set<std::string> seen;
    std::istringstream in(text);
    std::string raw;
    for (int line_no = 1; std::getline(in, raw); ++line_no) {
        std::string line = raw.substr(0, raw.find('#'));
        line = trim(line);
        if (line.empty()) continue;
        auto where = [&](const std::string& msg) {
            return ConfigError("config line " + std::to_string(line_no) + ": " + msg);
        };
        const size_t eq = line.find('=');
        if (eq == std::string::npos) throw where("expected key = value, got '" + trim(raw) + "'");
        const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
        const KeyDef* def = nullptr;
        for (const KeyDef& d : kKeys)
            if (key == d.name) def = &d;
        if (!def) throw where("unknown key '" + key + "'");
        if (!seen.insert(key).second) throw where("duplicate key '" + key + "'");
        if (value.empty() && def->k != K::csv && def->k != K::dump) throw where("empty value for " + key);
        try {
            assign(s, def->k, key, value);
        } catch (const LineError& e) {
            throw where(e.what());
        }
    }
    for (const char* req : {"grid.nx", "grid.ny", "grid.nz", "grid.dx", "grid.dy", "grid.dz", "material.Ms"})
        if (!seen.count(req)) throw ConfigError(std::string("config: missing required key '") + req + "'");
    if (s.init_kind == 1) {   // vortex: two perpendicular extents >= 2 (config.cpp:211-218)
        const bool along_x = s.vortex_axis <= 1, along_y = s.vortex_axis == 2 || s.vortex_axis == 3;
        const int p1 = along_x ? s.grid.ny : s.grid.nx;
        const int p2 = (along_x || along_y) ? s.grid.nz : s.grid.ny;
        if (p1 < 2 || p2 < 2)
            throw ConfigError("config: vortex init needs >= 2 cells along each axis perpendicular to init.axis");
    }
    if (defaults) {
        mfd_spec d;
        spec_default(d);
        // optional keys in canonical order, skipping the required ones
        for (const KeyDef& k : kKeys) {
            if (k.k <= K::dz || k.k == K::Ms || seen.count(k.name)) continue;
            defaults->push_back(std::string(k.name) + " = " + value_text(d, k.k));
        }
    }
    return s;
}

std::string format_config(const mfd_spec& s) {
    std::string out;
    for (const KeyDef& k : kKeys) out += std::string(k.name) + " = " + value_text(s, k.k) + "\n";
    return out;
}

mfd_spec load_config(const std::string& path, std::vector<std::string>* defaults) {
    std::ifstream f(path);
    if (!f) throw ConfigError("cannot open config file: " + path);
    std::ostringstream buf;
    buf << f.rdbuf();
    return parse_config(buf.str(), defaults);
}

} // namespace mfd::host
