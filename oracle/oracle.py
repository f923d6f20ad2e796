"""TEST INFRASTRUCTURE ONLY — ctypes front-end to the CPU oracles.

Two checkers, both built by oracle/Makefile:

* ``Port``: the plain-C restatement oracle/magfd_oracle.c
  (oracle/build/libmagfd_oracle_{f32,f64}.so).  Always available.
* ``Ref``: the unmodified reference solver compiled from /root/reference/proj
  (oracle/_ref/libmagfd_ref.so) — present wherever it was built (it travels to
  the GPU box as a prebuilt .so).  ``ref_available()`` says whether it is.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module.  The product (paper_1406_7459_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmagfd_ref.so")
QUAD_SO = os.path.join(HERE, "_ref", "libnewell_quad.so")
PORT_SO = {32: os.path.join(HERE, "build", "libmagfd_oracle_f32.so"),
           64: os.path.join(HERE, "build", "libmagfd_oracle_f64.so")}

MU0 = 4.0e-7 * 3.14159265358979323846
GAMMA_E = 1.760859630e11


def build(ref: bool | None = None) -> None:
    """Compile the C restatement (always) and oracle/_ref (when /root/reference exists)."""
    targets = ["port"]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj")
    if ref:
        targets += ["ref", "refapi"]   # refapi links libmagfd_b200.so: build the package first
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def quad_available() -> bool:
    return os.path.exists(QUAD_SO)


@dataclass
class Spec:
    """Mirror of the reference SimSpec hot-path fields (config.hpp:35-80)."""
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    A: float = 0.0
    Ku: float = 0.0
    Ms: float = 8e5
    alpha: float = 1.0
    gamma: float = GAMMA_E
    easy_axis: tuple = (0.0, 0.0, 1.0)
    exchange: bool = True
    anisotropy: bool = True
    demag: bool = True
    zeeman: bool = True
    h_ext: tuple = (0.0, 0.0, 0.0)
    dt: float = 1e-14
    renorm_every: int = 1
    max_steps: int = 500000
    torque_tol: float = 0.01
    sample_every: int = 100
    parallel: bool = False
    threads: int = 0

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz


class _RefSpec(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("A", C.c_double), ("Ku", C.c_double), ("Ms", C.c_double),
                ("alpha", C.c_double), ("gamma", C.c_double), ("easy_axis", C.c_double * 3),
                ("exchange", C.c_int), ("anisotropy", C.c_int), ("demag", C.c_int),
                ("zeeman", C.c_int), ("h_ext", C.c_double * 3), ("dt", C.c_double),
                ("renorm_every", C.c_int), ("max_steps", C.c_long), ("torque_tol", C.c_double),
                ("sample_every", C.c_long), ("parallel", C.c_int), ("threads", C.c_int)]


class _OrcSpec(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("A", C.c_double), ("Ku", C.c_double), ("Ms", C.c_double),
                ("alpha", C.c_double), ("gamma", C.c_double), ("easy_axis", C.c_double * 3),
                ("exchange", C.c_int), ("anisotropy", C.c_int), ("demag", C.c_int),
                ("zeeman", C.c_int), ("h_ext", C.c_double * 3), ("dt", C.c_double),
                ("renorm_every", C.c_int)]


class RefSample(C.Structure):
    _fields_ = [("step", C.c_long), ("t", C.c_double), ("m", C.c_double * 3),
                ("e_exch", C.c_double), ("e_anis", C.c_double), ("e_demag", C.c_double),
                ("e_zeeman", C.c_double), ("e_total", C.c_double), ("torque", C.c_double)]


def _fill(st, s: Spec):
    for f, _ in st._fields_:
        v = getattr(s, f)
        if f in ("easy_axis", "h_ext"):
            setattr(st, f, (C.c_double * 3)(*v))
        else:
            setattr(st, f, int(v) if isinstance(v, bool) else v)
    return st


_P = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_P)


_lib_cache: dict = {}


def _load(path):
    if path not in _lib_cache:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run oracle.build())")
        _lib_cache[path] = C.CDLL(path)
    return _lib_cache[path]


class _Sim:
    precision: int
    spec: Spec

    def _vec(self):
        n = self.spec.n
        return np.zeros(n), np.zeros(n), np.zeros(n)

    def set_m(self, m: np.ndarray):
        m = np.ascontiguousarray(m, dtype=np.float64).reshape(3, -1)
        x, y, z = (np.ascontiguousarray(m[i]) for i in range(3))
        self._call("set_m", _ptr(x), _ptr(y), _ptr(z))

    def get_m(self) -> np.ndarray:
        x, y, z = self._vec()
        self._call("get_m", _ptr(x), _ptr(y), _ptr(z))
        return np.stack([x, y, z])

    def heff(self) -> np.ndarray:
        x, y, z = self._vec()
        self._call("heff", _ptr(x), _ptr(y), _ptr(z))
        return np.stack([x, y, z])

    def hdemag(self) -> np.ndarray:
        x, y, z = self._vec()
        self._call("hdemag", _ptr(x), _ptr(y), _ptr(z))
        return np.stack([x, y, z])

    def step(self, n: int = 1) -> np.ndarray:
        t = np.zeros(max(n, 1))
        self._call("step", C.c_long(n), _ptr(t))
        return t[:n]

    def time(self):
        t = C.c_double()
        s = C.c_long()
        self._call("get_time", C.byref(t), C.byref(s))
        return t.value, s.value

    def set_time(self, t: float, step: int):
        self._call("set_time", C.c_double(t), C.c_long(step))

    def energies(self) -> np.ndarray:
        e = np.zeros(5)
        self._call("energies", _ptr(e))
        return e


class Ref(_Sim):
    """The reference solver itself (oracle/_ref/libmagfd_ref.so)."""

    def __init__(self, spec: Spec, precision: int = 64):
        self.lib = _load(REF_SO)
        self.lib.ref_sim_create.restype = C.c_void_p
        self.lib.ref_last_error.restype = C.c_char_p
        self.spec, self.precision = spec, precision
        self._s = _fill(_RefSpec(), spec)
        self.h = self.lib.ref_sim_create(precision, C.byref(self._s))
        if not self.h:
            raise ValueError(self.lib.ref_last_error().decode())

    def _call(self, name, *args):
        rc = getattr(self.lib, "ref_sim_" + name)(C.c_void_p(self.h), *args)
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            raise {1: ValueError, 2: RuntimeError, 3: LookupError}.get(rc, RuntimeError)(msg)

    def set_step_threads(self, threads: int):
        """Run the per-step calls on a `threads`-thread backend (setup stays on the
        creation backend; <= 0 restores it)."""
        self._call("set_step_threads", C.c_int(threads))

    def relax(self, cap: int = 100000):
        buf = (RefSample * cap)()
        n = C.c_long()
        rc = self.lib.ref_sim_relax(C.c_void_p(self.h), buf, C.c_long(cap), C.byref(n))
        if rc < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return bool(rc), [buf[i] for i in range(min(n.value, cap))]

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_sim_destroy(C.c_void_p(self.h))
            self.h = None


class Port(_Sim):
    """The plain-C restatement (oracle/magfd_oracle.c)."""

    def __init__(self, spec: Spec, precision: int = 64):
        self.lib = _load(PORT_SO[precision])
        self.sfx = "_f32" if precision == 32 else "_f64"
        getattr(self.lib, "orc_create" + self.sfx).restype = C.c_void_p
        self.spec, self.precision = spec, precision
        self._s = _fill(_OrcSpec(), spec)
        self.h = getattr(self.lib, "orc_create" + self.sfx)(C.byref(self._s))

    def _call(self, name, *args):
        fn = getattr(self.lib, "orc_" + name + self.sfx)
        rc = fn(C.c_void_p(self.h), *args)
        if name in ("step", "hdemag") and rc:
            raise {2: RuntimeError, 3: LookupError}[rc](
                "eulerUpdate: non-finite magnetization after step (time step too large?)"
                if rc == 2 else "lastDemagField: demag term is disabled")

    def reduced_mean(self) -> np.ndarray:
        m = np.zeros(3)
        getattr(self.lib, "orc_reduced_mean" + self.sfx)(C.c_void_p(self.h), _ptr(m))
        return m

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.lib, "orc_destroy" + self.sfx)(C.c_void_p(self.h))
            self.h = None


def tensor_entry(di, dj, dk, dx, dy, dz, which: str = "port") -> np.ndarray:
    """K = -N entries (xx,yy,zz,xy,xz,yz) at an integer displacement."""
    out = (C.c_double * 6)()
    args = (C.c_int(di), C.c_int(dj), C.c_int(dk), C.c_double(dx), C.c_double(dy), C.c_double(dz), out)
    if which == "port":
        _load(PORT_SO[64]).orc_tensor_entry_f64(*args)
    elif which == "ref":
        _load(REF_SO).ref_tensor_entry(*args)
    elif which == "quad":
        _load(QUAD_SO).quad_tensor_entry(*args)
    else:
        raise ValueError(which)
    return np.array(out[:])


def newell_nxx(X, Y, Z, dx, dy, dz, which: str = "port") -> float:
    if which == "port":
        f = _load(PORT_SO[64]).orc_nxx_f64
    else:
        f = _load(REF_SO).ref_newell_nxx
    f.restype = C.c_double
    return f(*(C.c_double(v) for v in (X, Y, Z, dx, dy, dz)))


def newell_nxy(X, Y, Z, dx, dy, dz, which: str = "port") -> float:
    if which == "port":
        f = _load(PORT_SO[64]).orc_nxy_f64
    else:
        f = _load(REF_SO).ref_newell_nxy
    f.restype = C.c_double
    return f(*(C.c_double(v) for v in (X, Y, Z, dx, dy, dz)))


def tensor_octant(nx, ny, nz, dx, dy, dz, which: str = "quad", threads: int = 0) -> np.ndarray:
    """Entries over [0,n)^3, shape (6, nz, ny, nx)."""
    out = np.zeros(6 * nx * ny * nz)
    d = (C.c_double(dx), C.c_double(dy), C.c_double(dz))
    if which == "quad":
        _load(QUAD_SO).quad_tensor_octant(nx, ny, nz, *d, _ptr(out))
    elif which == "ref":
        rc = _load(REF_SO).ref_tensor_octant(nx, ny, nz, *d, threads or os.cpu_count(), _ptr(out))
        assert rc == 0
    else:
        for q, (k, j, i) in enumerate(np.ndindex(nz, ny, nx)):
            e = tensor_entry(i, j, k, dx, dy, dz, "port")
            out[q::nx * ny * nz] = e
    return out.reshape(6, nz, ny, nx)


def ref_spectrum_octant(nx, ny, nz, dx, dy, dz):
    """Reference f64 tensor spectra (real parts) on [0,P/2] per axis, shape (6,Hz,Hy,Hx)."""
    px, py, pz = (padded(n) for n in (nx, ny, nz))
    hx, hy, hz = px // 2 + 1, py // 2 + 1, pz // 2 + 1
    out = np.zeros(6 * hx * hy * hz)
    mi = C.c_double()
    rc = _load(REF_SO).ref_spectrum_octant(nx, ny, nz, C.c_double(dx), C.c_double(dy),
                                           C.c_double(dz), _ptr(out), C.byref(mi))
    assert rc == 0
    return out.reshape(6, hz, hy, hx), mi.value


def direct_demag(spec: Spec, m: np.ndarray, which: str = "port") -> np.ndarray:
    m = np.ascontiguousarray(m, dtype=np.float64).reshape(3, -1)
    x, y, z = (np.ascontiguousarray(m[i]) for i in range(3))
    hx, hy, hz = np.zeros(spec.n), np.zeros(spec.n), np.zeros(spec.n)
    d = (C.c_double(spec.dx), C.c_double(spec.dy), C.c_double(spec.dz))
    if which == "port":
        _load(PORT_SO[64]).orc_direct_demag_f64(spec.nx, spec.ny, spec.nz, *d, _ptr(x), _ptr(y),
                                                _ptr(z), _ptr(hx), _ptr(hy), _ptr(hz))
    else:
        rc = _load(REF_SO).ref_direct_demag(spec.nx, spec.ny, spec.nz, *d, _ptr(x), _ptr(y),
                                            _ptr(z), _ptr(hx), _ptr(hy), _ptr(hz))
        assert rc == 0
    return np.stack([hx, hy, hz])


def padded(n: int) -> int:
    """nextPow2(2n), n = 1 -> 2 (demag.hpp:24)."""
    p = 1
    while p < 2 * n:
        p <<= 1
    return p


def random_unit_field(n: int, Ms: float, seed: int) -> np.ndarray:
    """Random unit directions x Ms (testutil.hpp:23-34 analogue; numpy RNG)."""
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(3, n))
    v /= np.linalg.norm(v, axis=0)
    return v * Ms


def rel_linf(a: np.ndarray, b: np.ndarray) -> float:
    """max|a-b| / max|b| over all components (testutil.hpp:36-47)."""
    d = np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)))
    r = np.max(np.abs(b))
    return float(d / r) if r > 0 else float(d)


# ---- host formats: the reference's own
# parseConfig / formatConfig, io::writeFieldDump / readFieldDump,
# io::writeTrajectoryCsv and makeVortexState, for byte-level parity tests.
def ref_config_format(text: str):
    """parseConfig + formatConfig (config.cpp:76-276) -> (rc, canonical text or
    ConfigError text, applied-default lines); rc 0 ok, 7 ConfigError."""
    lib = _load(REF_SO)
    out, dflt = C.create_string_buffer(1 << 16), C.create_string_buffer(1 << 16)
    rc = lib.ref_config_format(text.encode(), out, C.c_size_t(len(out)), dflt, C.c_size_t(len(dflt)))
    return rc, out.value.decode(), [l for l in dflt.value.decode().split("\n") if l]


def ref_last_error() -> str:
    lib = _load(REF_SO)
    lib.ref_last_error.restype = C.c_char_p
    return lib.ref_last_error().decode()


def ref_dump_write(path: str, m: np.ndarray, nx, ny, nz, dx, dy, dz, Ms, precision_bits=64) -> int:
    m = np.ascontiguousarray(m, dtype=np.float64).reshape(3, -1)
    x, y, z = (np.ascontiguousarray(m[i]) for i in range(3))
    return _load(REF_SO).ref_dump_write(str(path).encode(), nx, ny, nz, C.c_double(dx), C.c_double(dy),
                                        C.c_double(dz), C.c_double(Ms), precision_bits, _ptr(x), _ptr(y), _ptr(z))


def ref_dump_read(path: str):
    """-> (rc, header [nx, ny, nz, dx, dy, dz, Ms, precision_bits], M 3 x N or None)."""
    lib = _load(REF_SO)
    hdr = np.zeros(8)
    rc = lib.ref_dump_read(str(path).encode(), _ptr(hdr), None, C.c_longlong(0))
    if rc != 0:
        return rc, None, None
    n = int(hdr[0] * hdr[1] * hdr[2])
    m = np.zeros(3 * n)
    rc = lib.ref_dump_read(str(path).encode(), _ptr(hdr), _ptr(m), C.c_longlong(3 * n))
    return rc, hdr, m.reshape(3, n)


def ref_trajectory_csv(path: str, rows: np.ndarray) -> int:
    """rows: n x 11 {step, t, mx, my, mz, E_exch, E_anis, E_demag, E_zeeman, E_total, torque}."""
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    return _load(REF_SO).ref_trajectory_csv(str(path).encode(), _ptr(rows), C.c_long(len(rows)))


def ref_vortex_state(precision_bits, nx, ny, nz, dx, dy, dz, axis: int, Ms: float) -> np.ndarray:
    """makeVortexState<T> (state.hpp:83-108) widened to f64, 3 x N."""
    m = np.zeros(3 * nx * ny * nz)
    rc = _load(REF_SO).ref_vortex_state(precision_bits, nx, ny, nz, C.c_double(dx), C.c_double(dy),
                                        C.c_double(dz), axis, C.c_double(Ms), _ptr(m))
    assert rc == 0, ref_last_error()
    return m.reshape(3, -1)
