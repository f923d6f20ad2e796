"""magfd-b200: B200-native (sm_100a) engine for the per-step effective-field +
LLG hot path of the reference micromagnetic solver "magfd" (arXiv:1406.7459).

Python mirror of the reference C++ API over the C ABI of libmagfd_b200.so
(include/mfd.h).  ``Simulation`` follows ``magfd::Simulation<T>``
(/root/reference/proj/include/magfd/sim.hpp:15-72): ``step()`` returns the
pre-step max torque in deg/ns, ``sample_now()`` returns a TrajectorySample,
``relax()`` runs dynamics::relax (dynamics.hpp:157-198).  Errors map to the
reference exception types: ValueError (std::invalid_argument), RuntimeError
(std::runtime_error), LookupError (std::logic_error).

There is no CPU fallback: importing works anywhere, but constructing a
Simulation without the built library or without an sm_100 GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MFD_LIB") or os.path.join(HERE, "libmagfd_b200.so")   # MFD_LIB: A/B builds (tools/build_variant.sh)

MU0 = 4.0e-7 * 3.14159265358979323846      # constants.hpp:9
GAMMA_E = 1.760859630e11                    # constants.hpp:12

__all__ = ["Grid", "Material", "FieldConfig", "StepperConfig", "Sample", "Simulation",
           "build", "load_library", "MU0", "GAMMA_E"]


def build(jobs: int = 4) -> str:
    """Compile libmagfd_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", HERE], check=True)
    return LIB_PATH


# ----------------------------------------------------------------- ABI types
class _Grid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double)]


class _Material(C.Structure):
    _fields_ = [("A", C.c_double), ("Ku", C.c_double), ("Ms", C.c_double),
                ("alpha", C.c_double), ("gamma", C.c_double), ("easy_axis", C.c_double * 3)]


class _Terms(C.Structure):
    _fields_ = [("exchange", C.c_int), ("anisotropy", C.c_int), ("demag", C.c_int),
                ("zeeman", C.c_int), ("h_ext", C.c_double * 3)]


class _Stepper(C.Structure):
    _fields_ = [("dt", C.c_double), ("renorm_every", C.c_int), ("max_steps", C.c_long),
                ("torque_tol_deg_per_ns", C.c_double), ("sample_every", C.c_long)]


class _Exec(C.Structure):
    _fields_ = [("precision_bits", C.c_int), ("device", C.c_int), ("world", C.c_int), ("rank", C.c_int),
                ("virtual_ranks", C.c_int), ("transport", C.c_int), ("reserved", C.c_int * 2),
                ("nccl_id", C.c_ubyte * 128)]


class _Sample(C.Structure):
    _fields_ = [("step", C.c_long), ("t", C.c_double), ("m", C.c_double * 3),
                ("e_exchange", C.c_double), ("e_anisotropy", C.c_double), ("e_demag", C.c_double),
                ("e_zeeman", C.c_double), ("e_total", C.c_double), ("torque_deg_per_ns", C.c_double)]


_SampleCB = C.CFUNCTYPE(None, C.POINTER(_Sample), C.c_void_p)
_PD = C.POINTER(C.c_double)
_PF = C.POINTER(C.c_float)

_lib = None


def load_library() -> C.CDLL:
    """Load libmagfd_b200.so; fails loudly if it was not built (no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with paper_1406_7459_b200.build() "
                          "(the engine has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    V = C.c_void_p
    sig = {
        "mfd_create": (C.c_int, [C.POINTER(_Grid), C.POINTER(_Material), C.POINTER(_Terms),
                                 C.POINTER(_Stepper), C.POINTER(_Exec), C.POINTER(V)]),
        "mfd_destroy": (None, [V]),
        "mfd_set_m_f64": (C.c_int, [V, _PD, _PD, _PD]),
        "mfd_get_m_f64": (C.c_int, [V, _PD, _PD, _PD]),
        "mfd_set_m_f32": (C.c_int, [V, _PF, _PF, _PF]),
        "mfd_get_m_f32": (C.c_int, [V, _PF, _PF, _PF]),
        "mfd_set_m_uniform": (C.c_int, [V, _PD]),
        "mfd_stage_m_f64": (C.c_int, [V, _PD, _PD, _PD]),
        "mfd_stage_m_f32": (C.c_int, [V, _PF, _PF, _PF]),
        "mfd_set_time": (C.c_int, [V, C.c_double, C.c_long]),
        "mfd_get_time": (C.c_int, [V, _PD, C.POINTER(C.c_long)]),
        "mfd_effective_field_f64": (C.c_int, [V, _PD, _PD, _PD]),
        "mfd_demag_field_f64": (C.c_int, [V, _PD, _PD, _PD]),
        "mfd_step": (C.c_int, [V, C.c_long, _PD, _PD]),
        "mfd_step_async": (C.c_int, [V, C.c_long]),
        "mfd_prepare_async": (C.c_int, [V, C.c_long, C.POINTER(C.c_long)]),
        "mfd_sync": (C.c_int, [V]),
        "mfd_sync_torque": (C.c_int, [V, _PD]),
        "mfd_stream": (V, [V]),
        "mfd_relax": (C.c_int, [V, C.POINTER(C.c_int), _SampleCB, V]),
        "mfd_sample_now": (C.c_int, [V, C.POINTER(_Sample)]),
        "mfd_reduced_mean": (C.c_int, [V, _PD]),
        "mfd_energies": (C.c_int, [V, _PD]),
        "mfd_last_step_timing": (C.c_int, [V, _PD]),
        "mfd_stability_dt_limit": (C.c_double, [C.POINTER(_Material), C.POINTER(_Grid)]),
        "mfd_last_error": (C.c_char_p, [V]),
        "mfd_version": (C.c_char_p, []),
        "mfd_nccl_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
        "mfd_set_demag_octant_f64": (C.c_int, [V, _PD]),
        "mfd_get_demag_octant_f64": (C.c_int, [V, _PD]),
        "mfd_get_spectrum_octant_f64": (C.c_int, [V, _PD]),
        "mfd_debug_stage_f64": (C.c_int, [V, C.c_int, _PD]),
        "mfd_device_state": (C.c_int, [V, C.POINTER(V), C.POINTER(C.c_longlong), C.POINTER(C.c_int)]),
        "mfd_launches_per_step": (C.c_int, [V]),
        "mfd_model_bytes_per_step": (C.c_double, [V]),
        "mfd_debug_variants": (C.c_int, [V, C.c_char_p, C.c_int]),
        "mfd_debug_guard_check": (C.c_longlong, [V]),
        "mfd_effective_field_f32": (C.c_int, [V, _PF, _PF, _PF]),
        "mfd_demag_field_f32": (C.c_int, [V, _PF, _PF, _PF]),
        "mfd_set_stepper": (C.c_int, [V, C.POINTER(_Stepper)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


# ----------------------------------------------------------- reference mirror
@dataclass
class Grid:
    """grid.hpp:12-48."""
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float

    @property
    def cell_count(self) -> int:
        return self.nx * self.ny * self.nz

    def cell_volume(self) -> float:
        return self.dx * self.dy * self.dz


@dataclass
class Material:
    """MaterialParams (material.hpp:12-33)."""
    A: float = 0.0
    Ku: float = 0.0
    Ms: float = 0.0
    alpha: float = 1.0
    gamma: float = GAMMA_E
    easy_axis: Sequence[float] = (0.0, 0.0, 1.0)


@dataclass
class FieldConfig:
    """FieldConfig (fields.hpp:193-199)."""
    exchange: bool = True
    anisotropy: bool = True
    demag: bool = True
    zeeman: bool = True
    extern_field: Sequence[float] = (0.0, 0.0, 0.0)


@dataclass
class StepperConfig:
    """StepperConfig (dynamics.hpp:18-32)."""
    dt: float = 1e-14
    renormalize_every: int = 1
    max_steps: int = 500000
    torque_tol_deg_per_ns: float = 0.01
    sample_every: int = 100


@dataclass
class Sample:
    """TrajectorySample (dynamics.hpp:138-144)."""
    step: int
    t: float
    m: np.ndarray
    e_exchange: float
    e_anisotropy: float
    e_demag: float
    e_zeeman: float
    e_total: float
    max_torque_deg_per_ns: float

    @staticmethod
    def _from(s: _Sample) -> "Sample":
        return Sample(s.step, s.t, np.array(s.m[:]), s.e_exchange, s.e_anisotropy, s.e_demag,
                      s.e_zeeman, s.e_total, s.torque_deg_per_ns)


_ERR = {1: ValueError, 2: RuntimeError, 3: LookupError, 4: MemoryError, 5: OSError, 6: OSError}


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_PD if a.dtype == np.float64 else _PF)


class Simulation:
    """Device-resident simulation: the B200 counterpart of magfd::Simulation<T>.

    ``precision`` is 32 (float) or 64 (double), the reference's template T.
    The initial state is uniform along ``init_direction`` (makeUniformState);
    use ``set_m`` for any other start (the reference seeds from SimState)."""

    def __init__(self, grid: Grid, material: Material, fields: FieldConfig = FieldConfig(),
                 stepper: StepperConfig = StepperConfig(), precision: int = 64, device: int = 0,
                 init_direction: Sequence[float] = (0.0, 0.0, 1.0), world: int = 1, rank: int = 0,
                 virtual_ranks: bool = False, nccl_id: Optional[bytes] = None, transport: str = "nccl"):
        """world > 1: z-slab decomposition (mfd.h mfd_exec).  virtual_ranks runs
        all slabs on `device`; otherwise one process per rank, with set_m / get_m
        moving this rank's slab, over NCCL (transport="nccl", one GPU each) or the
        host-staged shared-memory test transport (transport="shm", any number of
        processes on one GPU; nccl_id = shared random bytes naming the segment)."""
        self.lib = load_library()
        self.grid, self.material, self.fields, self.stepper = grid, material, fields, stepper
        self.precision = precision
        self.world, self.rank = world, rank
        self.local = world > 1 and not virtual_ranks
        self._g = _Grid(grid.nx, grid.ny, grid.nz, grid.dx, grid.dy, grid.dz)
        self._m = _Material(material.A, material.Ku, material.Ms, material.alpha, material.gamma,
                            (C.c_double * 3)(*material.easy_axis))
        self._t = _Terms(int(fields.exchange), int(fields.anisotropy), int(fields.demag),
                         int(fields.zeeman), (C.c_double * 3)(*fields.extern_field))
        self._s = _Stepper(stepper.dt, stepper.renormalize_every, stepper.max_steps,
                           stepper.torque_tol_deg_per_ns, stepper.sample_every)
        if transport not in ("nccl", "shm"):
            raise ValueError("transport must be 'nccl' or 'shm'")
        self._e = _Exec(precision, device, world, rank, int(virtual_ranks), 1 if transport == "shm" else 0)
        if nccl_id is not None:
            C.memmove(self._e.nccl_id, bytes(nccl_id), 128)
        h = C.c_void_p()
        rc = self.lib.mfd_create(C.byref(self._g), C.byref(self._m), C.byref(self._t),
                                 C.byref(self._s), C.byref(self._e), C.byref(h))
        if rc != 0:
            raise _ERR.get(rc, RuntimeError)(self.lib.mfd_last_error(None).decode())
        self.h = h
        self.n = grid.cell_count // world if self.local else grid.cell_count
        d = np.asarray(init_direction, dtype=np.float64)
        self._check(self.lib.mfd_set_m_uniform(self.h, _ptr(d)))

    def _check(self, rc: int):
        if rc != 0:
            raise _ERR.get(rc, RuntimeError)(self.lib.mfd_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.mfd_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # -- state (SimState<T>, state.hpp:23-32)
    def set_m(self, m: np.ndarray):
        m = np.asarray(m).reshape(3, -1)
        if m.shape[1] != self.n:
            raise ValueError("set_m: expected 3 x N values")
        if m.dtype == np.float32:
            x, y, z = (np.ascontiguousarray(m[i]) for i in range(3))
            self._check(self.lib.mfd_set_m_f32(self.h, _ptr(x), _ptr(y), _ptr(z)))
        else:
            x, y, z = (np.ascontiguousarray(m[i], dtype=np.float64) for i in range(3))
            self._check(self.lib.mfd_set_m_f64(self.h, _ptr(x), _ptr(y), _ptr(z)))

    def stage_m(self, m: np.ndarray):
        """Queue a new state (3 x N, float32 or float64) for the next step; the upload
        overlaps a running step when m lives in pinned memory.  m must stay
        untouched until the next call that reads the state returns."""
        m = np.asarray(m).reshape(3, -1)
        if m.shape[1] != self.n:
            raise ValueError("stage_m: expected 3 x N values")
        if m.dtype == np.float32:
            if not m.flags.c_contiguous:
                raise ValueError("stage_m: m must be C-contiguous")
            self._check(self.lib.mfd_stage_m_f32(self.h, _ptr(m[0]), _ptr(m[1]), _ptr(m[2])))
        else:
            if m.dtype != np.float64 or not m.flags.c_contiguous:
                raise ValueError("stage_m: m must be a C-contiguous float32 / float64 array")
            self._check(self.lib.mfd_stage_m_f64(self.h, _ptr(m[0]), _ptr(m[1]), _ptr(m[2])))
        # keep the host arrays of the (at most two) states in flight alive
        self._staged = (getattr(self, "_staged", (None, None))[1], m)

    def get_m(self, dtype=np.float64) -> np.ndarray:
        out = np.zeros((3, self.n), dtype=dtype)
        x, y, z = out[0], out[1], out[2]
        if dtype == np.float32:
            self._check(self.lib.mfd_get_m_f32(self.h, _ptr(x), _ptr(y), _ptr(z)))
        else:
            self._check(self.lib.mfd_get_m_f64(self.h, _ptr(x), _ptr(y), _ptr(z)))
        return out

    @property
    def t(self) -> float:
        return self.time()[0]

    @property
    def step_count(self) -> int:
        return self.time()[1]

    def time(self):
        t, s = C.c_double(), C.c_long()
        self._check(self.lib.mfd_get_time(self.h, C.byref(t), C.byref(s)))
        return t.value, s.value

    def set_time(self, t: float, step: int):
        self._check(self.lib.mfd_set_time(self.h, t, step))

    # -- field evaluation (EffectiveFieldProvider, fields.hpp:220-268)
    def effective_field(self, dtype=np.float64) -> np.ndarray:
        out = np.zeros((3, self.n), dtype=dtype)
        f = self.lib.mfd_effective_field_f32 if dtype == np.float32 else self.lib.mfd_effective_field_f64
        self._check(f(self.h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    def demag_field(self, dtype=np.float64) -> np.ndarray:
        out = np.zeros((3, self.n), dtype=dtype)
        f = self.lib.mfd_demag_field_f32 if dtype == np.float32 else self.lib.mfd_demag_field_f64
        self._check(f(self.h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    # -- dynamics
    def step(self, n: int = 1, return_all: bool = False):
        """n x Simulation::step (sim.hpp:33-42); returns the last pre-step torque (deg/ns)."""
        last = C.c_double()
        allv = np.zeros(max(n, 1)) if return_all else None
        self._check(self.lib.mfd_step(self.h, n, C.byref(last), _ptr(allv) if return_all else None))
        return allv[:n] if return_all else last.value

    def step_async(self, n: int):
        self._check(self.lib.mfd_step_async(self.h, n))

    def prepare_async(self, n: int) -> int:
        """Capture the graphs of the next step_async(n) without running them; returns
        the kernel launches they contain."""
        k = C.c_long()
        self._check(self.lib.mfd_prepare_async(self.h, n, C.byref(k)))
        return k.value

    def sync(self):
        self._check(self.lib.mfd_sync(self.h))

    def sync_torque(self) -> float:
        """sync() + the pre-step torque (deg/ns) of the last asynchronous step."""
        t = C.c_double()
        self._check(self.lib.mfd_sync_torque(self.h, C.byref(t)))
        return t.value

    def sample_now(self) -> Sample:
        s = _Sample()
        self._check(self.lib.mfd_sample_now(self.h, C.byref(s)))
        return Sample._from(s)

    def reduced_mean(self) -> np.ndarray:
        m = np.zeros(3)
        self._check(self.lib.mfd_reduced_mean(self.h, _ptr(m)))
        return m

    def energies(self) -> np.ndarray:
        e = np.zeros(5)
        self._check(self.lib.mfd_energies(self.h, _ptr(e)))
        return e

    def relax(self, on_sample: Optional[Callable[[Sample], None]] = None):
        """dynamics::relax; returns (converged, [Sample, ...])."""
        log: List[Sample] = []

        def cb(p, _u):
            s = Sample._from(p.contents)
            log.append(s)
            if on_sample:
                on_sample(s)

        cfun = _SampleCB(cb)
        conv = C.c_int()
        self._check(self.lib.mfd_relax(self.h, C.byref(conv), cfun, None))
        return bool(conv.value), log

    def step_timing(self) -> np.ndarray:
        ms = np.zeros(7)
        self._check(self.lib.mfd_last_step_timing(self.h, _ptr(ms)))
        return ms

    # -- test / bench hooks
    def set_demag_octant(self, oct6: np.ndarray):
        o = np.ascontiguousarray(oct6, dtype=np.float64)
        self._check(self.lib.mfd_set_demag_octant_f64(self.h, _ptr(o)))

    def demag_octant(self) -> np.ndarray:
        g = self.grid
        o = np.zeros((6, g.nz, g.ny, g.nx))
        self._check(self.lib.mfd_get_demag_octant_f64(self.h, _ptr(o)))
        return o

    def spectrum_octant(self) -> np.ndarray:
        g = self.grid
        px, py, pz = (padded_size(v) for v in (g.nx, g.ny, g.nz))
        o = np.zeros((6, py // 2 + 1, pz // 2 + 1, px // 2 + 1))
        self._check(self.lib.mfd_get_spectrum_octant_f64(self.h, _ptr(o)))
        return o

    def debug_stage(self, stage: int) -> np.ndarray:
        """Intermediate spectrum after pass K<stage> (test hook), complex, pitch included."""
        g = self.grid
        hp = (padded_size(g.nx) // 2 + 1 + 15) // 16 * 16
        rows = g.ny if stage in (1, 4) else padded_size(g.ny)
        out = np.zeros(2 * 3 * g.nz * rows * hp)
        self._check(self.lib.mfd_debug_stage_f64(self.h, stage, _ptr(out)))
        return (out[0::2] + 1j * out[1::2]).reshape(3, g.nz, rows, hp)

    def device_state(self):
        p, n, prec = C.c_void_p(), C.c_longlong(), C.c_int()
        self._check(self.lib.mfd_device_state(self.h, C.byref(p), C.byref(n), C.byref(prec)))
        return p.value, n.value, prec.value

    def stream_handle(self) -> int:
        return self.lib.mfd_stream(self.h)

    def launches_per_step(self) -> int:
        return self.lib.mfd_launches_per_step(self.h)

    def model_bytes_per_step(self) -> float:
        return self.lib.mfd_model_bytes_per_step(self.h)

    def guard_check(self) -> int:
        """Guard-band bytes overwritten (MFD_GUARD=1 at creation; -1 when off)."""
        return int(self.lib.mfd_debug_guard_check(self.h))

    def set_stepper(self, stepper: StepperConfig):
        """Replace the StepperConfig of the live simulation."""
        self.stepper = stepper
        self._s = _Stepper(stepper.dt, stepper.renormalize_every, stepper.max_steps,
                           stepper.torque_tol_deg_per_ns, stepper.sample_every)
        self._check(self.lib.mfd_set_stepper(self.h, C.byref(self._s)))

    def variants(self) -> List[str]:
        """Kernel template instantiations this context has enqueued (test hook)."""
        n = self.lib.mfd_debug_variants(self.h, None, 0)
        buf = C.create_string_buffer(n)
        self.lib.mfd_debug_variants(self.h, buf, n)
        return [l for l in buf.value.decode().split("\n") if l]

    @staticmethod
    def stability_dt_limit(grid: Grid, material: Material) -> float:
        lib = load_library()
        g = _Grid(grid.nx, grid.ny, grid.nz, grid.dx, grid.dy, grid.dz)
        m = _Material(material.A, material.Ku, material.Ms, material.alpha, material.gamma,
                      (C.c_double * 3)(*material.easy_axis))
        return lib.mfd_stability_dt_limit(C.byref(m), C.byref(g))


def nccl_unique_id() -> bytes:
    """NCCL unique id for a multi-GPU context (rank 0; broadcast it to the other ranks)."""
    lib = load_library()
    buf = (C.c_ubyte * 128)()
    rc = lib.mfd_nccl_unique_id(buf)
    if rc != 0:
        raise OSError(lib.mfd_last_error(None).decode())
    return bytes(buf)


def padded_size(n: int) -> int:
    """nextPow2(2n), n = 1 -> 2 (demag.hpp:24)."""
    p = 1
    while p < 2 * n:
        p <<= 1
    return p
