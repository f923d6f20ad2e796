"""Host-side formats around the hot path,
mirroring the reference's magfd::parseConfig / formatConfig / loadConfigFile
(config.hpp:97-103) and magfd::io (io.hpp:21-42) over the C ABI of
libmagfd_b200.so (include/mfd_host.h).  Errors raise ConfigError / IoError
with the reference's message text.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from . import (GAMMA_E, FieldConfig, Grid, Material, Sample, Simulation, StepperConfig, _Grid, _Material,
               _Sample, _Stepper, _Terms, load_library)

__all__ = ["ConfigError", "IoError", "SimSpec", "parse_config", "format_config", "load_config",
           "FieldDump", "write_field_dump", "read_field_dump", "write_trajectory_csv", "BenchRow",
           "write_bench_csv", "AXES", "simulation_from_spec"]

AXES = ("+x", "-x", "+y", "-y", "+z", "-z")          # SignedAxis (state.hpp:36)


class ConfigError(RuntimeError):
    """magfd::ConfigError (config.hpp:21-23)."""


class IoError(RuntimeError):
    """magfd::io::IoError (io.hpp:14-16)."""


class _Spec(C.Structure):
    _fields_ = [("grid", _Grid), ("material", _Material), ("terms", _Terms), ("stepper", _Stepper),
                ("init_kind", C.c_int), ("init_direction", C.c_double * 3), ("vortex_axis", C.c_int),
                ("backend_kind", C.c_int), ("threads", C.c_uint), ("precision_bits", C.c_int),
                ("csv_path", C.c_char * 1024), ("dump_path", C.c_char * 1024)]


class _BenchRow(C.Structure):
    _fields_ = [("size", C.c_int)] + [(n, C.c_double) for n in (
        "ms_per_step", "pad_ms", "forward_fft_ms", "spectral_multiply_ms", "inverse_fft_ms", "local_fields_ms",
        "integrate_ms")]


_PD = C.POINTER(C.c_double)
_sig_done = False


def _lib():
    global _sig_done
    lib = load_library()
    if not _sig_done:
        sig = {
            "mfd_spec_default": (None, [C.POINTER(_Spec)]),
            "mfd_config_parse": (C.c_int, [C.c_char_p, C.POINTER(_Spec), C.c_char_p, C.c_size_t]),
            "mfd_config_load": (C.c_int, [C.c_char_p, C.POINTER(_Spec), C.c_char_p, C.c_size_t]),
            "mfd_config_format": (C.c_long, [C.POINTER(_Spec), C.c_char_p, C.c_size_t]),
            "mfd_dump_write": (C.c_int, [C.c_char_p, C.POINTER(_Grid), C.c_double, C.c_int, _PD, _PD, _PD]),
            "mfd_dump_read_header": (C.c_int, [C.c_char_p, C.POINTER(_Grid), _PD, C.POINTER(C.c_int)]),
            "mfd_dump_read": (C.c_int, [C.c_char_p, C.POINTER(_Grid), _PD, C.POINTER(C.c_int), _PD, _PD, _PD]),
            "mfd_trajectory_csv_write": (C.c_int, [C.c_char_p, C.POINTER(_Sample), C.c_long]),
            "mfd_bench_csv_write": (C.c_int, [C.c_char_p, C.POINTER(_BenchRow), C.c_long]),
            "mfd_set_m_vortex": (C.c_int, [C.c_void_p, C.c_int]),
            "mfd_host_last_error": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _sig_done = True
    return lib


def _raise(rc: int):
    if rc == 0:
        return
    msg = _lib().mfd_host_last_error().decode()
    raise {7: ConfigError, 8: IoError, 1: ValueError, 4: MemoryError}.get(rc, RuntimeError)(msg)


@dataclass
class SimSpec:
    """SimSpec (config.hpp:26-80): the parsed config, reference field names."""
    grid: Grid
    material: Material
    fields: FieldConfig
    stepper: StepperConfig
    init_kind: str = "uniform"                              # uniform | vortex
    init_direction: Tuple[float, float, float] = (0.0, 0.0, 1.0)
    vortex_axis: str = "+z"
    backend: str = "serial"                                  # recorded; the B200 engine ignores it
    threads: int = 0
    precision: str = "f64"
    csv_path: str = "trajectory.csv"
    dump_path: str = "final_state.dump"

    @staticmethod
    def _from(s: _Spec) -> "SimSpec":
        g, m, t, st = s.grid, s.material, s.terms, s.stepper
        return SimSpec(Grid(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz),
                       Material(m.A, m.Ku, m.Ms, m.alpha, m.gamma, tuple(m.easy_axis)),
                       FieldConfig(bool(t.exchange), bool(t.anisotropy), bool(t.demag), bool(t.zeeman),
                                   tuple(t.h_ext)),
                       StepperConfig(st.dt, st.renorm_every, st.max_steps, st.torque_tol_deg_per_ns,
                                     st.sample_every),
                       "uniform" if s.init_kind == 0 else "vortex", tuple(s.init_direction), AXES[s.vortex_axis],
                       "serial" if s.backend_kind == 0 else "parallel", int(s.threads),
                       "f32" if s.precision_bits == 32 else "f64", s.csv_path.decode(), s.dump_path.decode())

    def _to(self) -> _Spec:
        s = _Spec()
        g, m, f, st = self.grid, self.material, self.fields, self.stepper
        s.grid = _Grid(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz)
        s.material = _Material(m.A, m.Ku, m.Ms, m.alpha, m.gamma, (C.c_double * 3)(*m.easy_axis))
        s.terms = _Terms(int(f.exchange), int(f.anisotropy), int(f.demag), int(f.zeeman),
                         (C.c_double * 3)(*f.extern_field))
        s.stepper = _Stepper(st.dt, st.renormalize_every, st.max_steps, st.torque_tol_deg_per_ns, st.sample_every)
        s.init_kind = 0 if self.init_kind == "uniform" else 1
        s.init_direction = (C.c_double * 3)(*self.init_direction)
        s.vortex_axis = AXES.index(self.vortex_axis)
        s.backend_kind = 0 if self.backend == "serial" else 1
        s.threads = self.threads
        s.precision_bits = 32 if self.precision == "f32" else 64
        s.csv_path = self.csv_path.encode()
        s.dump_path = self.dump_path.encode()
        return s


def _defaults(buf) -> List[str]:
    return [l for l in buf.value.decode().split("\n") if l]


def parse_config(text: str) -> Tuple[SimSpec, List[str]]:
    """parseConfig(text, &appliedDefaults) (config.cpp:76-246)."""
    s, buf = _Spec(), C.create_string_buffer(1 << 16)
    _raise(_lib().mfd_config_parse(text.encode(), C.byref(s), buf, len(buf)))
    return SimSpec._from(s), _defaults(buf)


def load_config(path: str) -> Tuple[SimSpec, List[str]]:
    """loadConfigFile (config.cpp:278-284)."""
    s, buf = _Spec(), C.create_string_buffer(1 << 16)
    _raise(_lib().mfd_config_load(str(path).encode(), C.byref(s), buf, len(buf)))
    return SimSpec._from(s), _defaults(buf)


def format_config(spec: SimSpec) -> str:
    """formatConfig (config.cpp:248-276): parse_config(format_config(s))[0] == s."""
    s = spec._to()
    n = _lib().mfd_config_format(C.byref(s), None, 0)
    buf = C.create_string_buffer(n + 1)
    _lib().mfd_config_format(C.byref(s), buf, len(buf))
    return buf.value.decode()


@dataclass
class FieldDump:
    """io::FieldDump (io.hpp:21-26); M is 3 x N float64, A/m."""
    grid: Grid
    Ms: float
    precision: str
    M: np.ndarray = field(repr=False)


def write_field_dump(path: str, M: np.ndarray, grid: Grid, Ms: float, precision: str = "f64"):
    """io::writeFieldDump (io.cpp:18-36)."""
    M = np.ascontiguousarray(np.asarray(M, dtype=np.float64).reshape(3, -1))
    g = _Grid(grid.nx, grid.ny, grid.nz, grid.dx, grid.dy, grid.dz)
    p = [M[i].ctypes.data_as(_PD) for i in range(3)]
    _raise(_lib().mfd_dump_write(str(path).encode(), C.byref(g), Ms, 32 if precision == "f32" else 64, *p))


def read_field_dump(path: str) -> FieldDump:
    """io::readFieldDump (io.cpp:38-100)."""
    g, ms, prec = _Grid(), C.c_double(), C.c_int()
    lib = _lib()
    _raise(lib.mfd_dump_read_header(str(path).encode(), C.byref(g), C.byref(ms), C.byref(prec)))
    M = np.zeros((3, g.nx * g.ny * g.nz))
    p = [M[i].ctypes.data_as(_PD) for i in range(3)]
    _raise(lib.mfd_dump_read(str(path).encode(), C.byref(g), C.byref(ms), C.byref(prec), *p))
    return FieldDump(Grid(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz), ms.value, "f32" if prec.value == 32 else "f64", M)


def write_trajectory_csv(path: str, log: Sequence[Sample]):
    """io::writeTrajectoryCsv (io.cpp:102-117)."""
    arr = (_Sample * max(1, len(log)))()
    for i, s in enumerate(log):
        arr[i] = _Sample(s.step, s.t, (C.c_double * 3)(*s.m), s.e_exchange, s.e_anisotropy, s.e_demag,
                         s.e_zeeman, s.e_total, s.max_torque_deg_per_ns)
    _raise(_lib().mfd_trajectory_csv_write(str(path).encode(), arr, len(log)))


@dataclass
class BenchRow:
    """cli::BenchRow (cli.hpp:30-34), milliseconds."""
    size: int
    ms_per_step: float
    pad_ms: float = 0.0
    forward_fft_ms: float = 0.0
    spectral_multiply_ms: float = 0.0
    inverse_fft_ms: float = 0.0
    local_fields_ms: float = 0.0
    integrate_ms: float = 0.0


def write_bench_csv(path: str, rows: Sequence[BenchRow]):
    """The bench CSV of cli::cmdBench (cli.cpp:187-200)."""
    arr = (_BenchRow * max(1, len(rows)))()
    for i, r in enumerate(rows):
        arr[i] = _BenchRow(r.size, r.ms_per_step, r.pad_ms, r.forward_fft_ms, r.spectral_multiply_ms,
                           r.inverse_fft_ms, r.local_fields_ms, r.integrate_ms)
    _raise(_lib().mfd_bench_csv_write(str(path).encode(), arr, len(rows)))


def simulation_from_spec(spec: SimSpec, device: int = 0) -> Simulation:
    """Simulation<T>(spec) (sim.hpp:17-24): engine + initial state from init.*
    (makeUniformState / makeVortexState on the device)."""
    sim = Simulation(spec.grid, spec.material, spec.fields, spec.stepper,
                     precision=32 if spec.precision == "f32" else 64, device=device,
                     init_direction=spec.init_direction)
    if spec.init_kind == "vortex":
        sim._check(_lib().mfd_set_m_vortex(sim.h, AXES.index(spec.vortex_axis)))
    return sim
