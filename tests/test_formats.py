"""Host formats around the hot path, byte
for byte against the reference's own implementations (oracle/_ref):

* parseConfig / formatConfig / applied defaults (config.cpp:76-276), including
  every validation error text;
* io::writeFieldDump / readFieldDump (io.cpp:18-100) and writeTrajectoryCsv
  (io.cpp:102-117);
* the bench CSV of cli::cmdBench (cli.cpp:187-200).

CPU-only: these are host code paths of libmagfd_b200.so (no kernel calls).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

F = pytest.importorskip("paper_1406_7459_b200.formats")

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

BASE = """grid.nx = 4
grid.ny = 3
grid.nz = 2
grid.dx = 2e-9
grid.dy = 2.5e-9
grid.dz = 3e-9
material.Ms = 8e5
"""

FULL = BASE + """# every optional key, odd spacing and trailing comments
material.A=1.3e-11   # exchange
material.Ku = -4e4
material.alpha = 0.02
material.gamma = 1.76e11
material.easy_axis = 1 1 0
terms.exchange = on
terms.anisotropy = 0
terms.demag = true
terms.zeeman = off
field.extern = 1e4 -2e3 0.5
init.kind = vortex
init.direction = 0 3 4
init.axis = y
stepper.dt = 5e-14
stepper.max_steps = 1234
stepper.torque_tol = 0.5
stepper.renorm_every = 7
backend.kind = parallel
backend.threads = 3
precision = f32
output.csv =
output.dump = out dir/final.dump
output.sample_every = 25
"""

VALID = [BASE, FULL, "\n\n# header only comment\n" + BASE + "\n   \n", BASE.replace("= ", "=   \t"),
         BASE + "stepper.max_steps = 0\n", BASE + "init.axis = -x\n", BASE.replace("2e-9", "0x1p-30"),
         BASE + "material.Ku = 1e-300\n"]

BAD = [
    "",                                                # missing grid.nx
    BASE.replace("material.Ms = 8e5\n", ""),            # missing Ms
    BASE + "bogus.key = 1\n",
    BASE + "grid.nx = 5\n",                            # duplicate
    BASE + "material.A\n",                             # no '='
    BASE + "material.A =\n",                           # empty value
    BASE.replace("grid.nx = 4", "grid.nx = 0"),
    BASE.replace("grid.nx = 4", "grid.nx = 4.5"),
    BASE.replace("grid.nx = 4", "grid.nx = four"),
    BASE.replace("grid.nx = 4", "grid.nx = 99999999999999999999999"),
    BASE.replace("grid.dx = 2e-9", "grid.dx = -1"),
    BASE.replace("grid.dx = 2e-9", "grid.dx = 2e-9 m"),
    BASE.replace("grid.dx = 2e-9", "grid.dx = nan"),
    BASE.replace("grid.dx = 2e-9", "grid.dx = inf"),
    BASE.replace("grid.dx = 2e-9", "grid.dx = 1e999"),
    BASE + "material.A = -1\n",
    BASE + "material.alpha = -0.1\n",
    BASE + "material.easy_axis = 0 0 0\n",
    BASE + "material.easy_axis = 1 2\n",
    BASE + "material.easy_axis = 1 2 3 4\n",
    BASE + "field.extern = 0x1p-3 2 0\n",
    BASE + "terms.demag = yes\n",
    BASE + "init.kind = spiral\n",
    BASE + "init.direction = 0 0 0\n",
    BASE + "init.axis = +w\n",
    BASE + "stepper.max_steps = -1\n",
    BASE + "stepper.dt = 0\n",
    BASE + "stepper.torque_tol = -1\n",
    BASE + "stepper.renorm_every = 0\n",
    BASE + "backend.kind = gpu\n",
    BASE + "backend.threads = -2\n",
    BASE + "precision = f16\n",
    BASE + "output.sample_every = 0\n",
    BASE.replace("grid.ny = 3", "grid.ny = 1") + "init.kind = vortex\n",   # vortex needs 2 perpendicular cells
    BASE.replace("grid.nz = 2", "grid.nz = 1") + "init.kind = vortex\ninit.axis = x\n",
]


@needs_ref
@pytest.mark.parametrize("text", VALID)
def test_config_parse_format_matches_reference(text):
    rc, ref_text, ref_defaults = O.ref_config_format(text)
    assert rc == 0, ref_text
    spec, defaults = F.parse_config(text)
    assert F.format_config(spec) == ref_text
    assert defaults == ref_defaults


@needs_ref
@pytest.mark.parametrize("text", BAD)
def test_config_errors_match_reference(text):
    rc, ref_msg, _ = O.ref_config_format(text)
    assert rc == 7
    with pytest.raises(F.ConfigError) as e:
        F.parse_config(text)
    assert str(e.value) == ref_msg


def test_config_round_trip():
    # (re-normalising a %.17g-printed unit vector can move its last bit, in the
    # reference as here, so the round trip uses exactly normalisable vectors)
    for text in (BASE, FULL.replace("1 1 0", "0 0 -2")):
        spec, _ = F.parse_config(text)
        again, defaults = F.parse_config(F.format_config(spec))
        assert again == spec
        assert defaults == []
    spec, _ = F.parse_config(FULL)
    assert spec.init_kind == "vortex" and spec.vortex_axis == "+y" and spec.precision == "f32"
    assert spec.init_direction == (0.0, 0.6, 0.8) and spec.dump_path == "out dir/final.dump" and spec.csv_path == ""


def test_config_load_file(tmp_path):
    p = tmp_path / "a.cfg"
    p.write_text(BASE)
    spec, d = F.load_config(str(p))
    assert spec.grid.nx == 4 and "stepper.dt = %.17g" % 1e-14 in d
    with pytest.raises(F.ConfigError, match="cannot open config file: "):
        F.load_config(str(tmp_path / "missing.cfg"))


def _field(n, seed):
    rng = np.random.default_rng(seed)
    m = rng.normal(size=(3, n)) * 8e5
    m[:, 0] = [0.1, -0.0, 1e-300]      # awkward values: %.17g must round-trip them
    m[:, -1] = [8e5 / 3, np.nextafter(8e5, 1e6), -123.456]
    return m


@needs_ref
@pytest.mark.parametrize("prec", [32, 64])
def test_dump_bytes_and_round_trip(tmp_path, prec):
    g = F.Grid(5, 3, 2, 1e-9, 2.5e-9, 3.0000000000000004e-9)
    m = _field(g.cell_count, 7)
    mine, ref = tmp_path / "mine.dump", tmp_path / "ref.dump"
    F.write_field_dump(str(mine), m, g, 8e5, "f32" if prec == 32 else "f64")
    assert O.ref_dump_write(str(ref), m, 5, 3, 2, g.dx, g.dy, g.dz, 8e5, prec) == 0
    assert mine.read_bytes() == ref.read_bytes()
    d = F.read_field_dump(str(ref))
    assert (d.grid.nx, d.grid.ny, d.grid.nz) == (5, 3, 2) and d.grid.dz == g.dz and d.Ms == 8e5
    assert d.precision == ("f32" if prec == 32 else "f64")
    assert np.array_equal(d.M.view(np.uint64), m.view(np.uint64))     # bitwise
    rc, hdr, mr = O.ref_dump_read(str(mine))
    assert rc == 0 and np.array_equal(mr.view(np.uint64), m.view(np.uint64))


def _dump_text(lines=None, header=None):
    h = header if header is not None else [
        "# magfd-dump v1", "# nx 2", "# ny 1", "# nz 1", "# dx 1e-9", "# dy 1e-9", "# dz 1e-9", "# Ms 8e5",
        "# precision f64"]
    body = lines if lines is not None else ["0 0 0 1 2 3", "1 0 0 4 5 6"]
    return "\n".join(h + body) + "\n"


BAD_DUMPS = [
    _dump_text(header=["# magfd-dump v1", "# nx 2", "# ny 1", "# nz 1", "# dx 1e-9", "# dy 1e-9", "# dz 1e-9",
                       "# Ms 8e5"]),                                   # no precision
    _dump_text(header=["# nx 2", "# ny 1", "# nz 1", "# dx 1e-9", "# dy 1e-9", "# dz 1e-9", "# Ms 8e5",
                       "# precision f16"]),
    _dump_text(header=["# nx two", "# ny 1", "# nz 1", "# dx 1e-9", "# dy 1e-9", "# dz 1e-9", "# Ms 8e5",
                       "# precision f32"]),
    _dump_text(lines=["0 0 0 1 2 3"]),                                 # too few lines
    _dump_text(lines=["0 0 0 1 2 3", "1 0 0 4 5"]),                    # short line
    _dump_text(lines=["0 0 0 1 2 3", "2 0 0 4 5 6"]),                  # out of range
    _dump_text(lines=["0 0 0 1 2 3", "1 0 0 4 5 6", "1 0 0 4 5 6"]),   # too many lines
]
GOOD_DUMPS = [
    _dump_text(),
    _dump_text(header=["", "# a comment", "# nx 2", "#ny 1", "# nz 1 trailing", "# dx 1e-9", "# dy 1e-9",
                       "# dz 1e-9", "# Ms 8e5", "", "# precision f32"]),
    _dump_text(lines=["1 0 0 4 5 6", "# mid comment", "", "0 0 0 1 2 3 extra"]),
]


@needs_ref
@pytest.mark.parametrize("i", range(len(BAD_DUMPS)))
def test_dump_errors_match_reference(tmp_path, i):
    p = tmp_path / "x.dump"
    p.write_text(BAD_DUMPS[i])
    rc, _, _ = O.ref_dump_read(str(p))
    assert rc == 8
    with pytest.raises(F.IoError) as e:
        F.read_field_dump(str(p))
    assert str(e.value) == O.ref_last_error()


@needs_ref
@pytest.mark.parametrize("i", range(len(GOOD_DUMPS)))
def test_dump_tolerant_reads_match_reference(tmp_path, i):
    p = tmp_path / "x.dump"
    p.write_text(GOOD_DUMPS[i])
    rc, hdr, mr = O.ref_dump_read(str(p))
    assert rc == 0
    d = F.read_field_dump(str(p))
    assert np.array_equal(d.M, mr) and d.precision == ("f32" if hdr[7] == 32 else "f64")


def test_dump_missing_file(tmp_path):
    with pytest.raises(F.IoError, match="cannot open for reading: "):
        F.read_field_dump(str(tmp_path / "nope.dump"))
    with pytest.raises(F.IoError, match="cannot open for writing: "):
        F.write_field_dump(str(tmp_path / "no" / "dir.dump"), np.zeros((3, 1)), F.Grid(1, 1, 1, 1, 1, 1), 1.0)


@needs_ref
def test_trajectory_csv_bytes(tmp_path):
    rng = np.random.default_rng(3)
    rows = rng.normal(size=(6, 11))
    rows[:, 0] = [0, 100, 200, 300, 12345678901, 7]
    rows[0, 1:] = [0.0, 1 / 3, -0.0, 1e-300, 5e-324, 1e300, -2.5, 0.1, 0.2, 0.3]
    log = [F.Sample(int(r[0]), r[1], r[2:5], *r[5:11]) for r in rows]
    mine, ref = tmp_path / "m.csv", tmp_path / "r.csv"
    F.write_trajectory_csv(str(mine), log)
    assert O.ref_trajectory_csv(str(ref), rows) == 0
    assert mine.read_bytes() == ref.read_bytes()


def test_bench_csv_format(tmp_path):
    p = tmp_path / "b.csv"
    F.write_bench_csv(str(p), [F.BenchRow(8, 0.123456789, 0.0, 1.5, 2e-5, 3.25, 100.0, 0.0),
                               F.BenchRow(64, 1234567.0)])
    lines = p.read_text().splitlines()
    assert lines[0] == ("size,ms_per_step,pad_ms,forward_fft_ms,spectral_multiply_ms,inverse_fft_ms,"
                        "local_fields_ms,integrate_ms")
    assert lines[1] == "8,0.123457,0,1.5,2e-05,3.25,100,0"     # ostream default (%g, precision 6)
    assert lines[2] == "64,1.23457e+06,0,0,0,0,0,0"
