"""The magfd-b200 CLI (relax / run / bench over the C ABI) and the device
initialisers, against the reference:

* makeVortexState on the device is bitwise the reference's host state
  (state.hpp:83-108), f32 and f64, every axis family;
* `run` writes the reference's trajectory CSV / field dump formats with the
  reference's sampling cadence (cli.cpp:57-73), values at f64 parity;
* `relax` reproduces dynamics::relax's stop step and summary (cli.cpp:40-55);
* `bench` writes the bench CSV; bad configs fail like the reference CLI.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

F = pytest.importorskip("paper_1406_7459_b200.formats")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1406_7459_b200", "magfd-b200")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def cli(*args, cwd=None):
    return subprocess.run([CLI, *args], capture_output=True, text=True, cwd=cwd, timeout=300)


@needs_ref
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("axis,dims", [("+z", (7, 6, 3)), ("-x", (2, 5, 4)), ("y", (6, 1, 5)), ("-z", (8, 8, 1))])
def test_vortex_state_bitwise(prec, axis, dims):
    nx, ny, nz = dims
    text = (f"grid.nx = {nx}\ngrid.ny = {ny}\ngrid.nz = {nz}\ngrid.dx = 2e-9\ngrid.dy = 3e-9\ngrid.dz = 2.5e-9\n"
            f"material.Ms = 8e5\ninit.kind = vortex\ninit.axis = {axis}\nprecision = f{prec}\nterms.demag = false\n")
    spec, _ = F.parse_config(text)
    sim = F.simulation_from_spec(spec)
    mine = sim.get_m(np.float32 if prec == 32 else np.float64).astype(np.float64)
    ref = O.ref_vortex_state(prec, nx, ny, nz, 2e-9, 3e-9, 2.5e-9, F.AXES.index(spec.vortex_axis), 8e5)
    assert np.array_equal(mine, ref)


CFG = """# small film, all four terms
grid.nx = 16
grid.ny = 8
grid.nz = 2
grid.dx = 2.5e-9
grid.dy = 2.5e-9
grid.dz = 3e-9
material.Ms = 8e5
material.A = 1.3e-11
material.Ku = 4e4
material.alpha = 0.1
field.extern = 1e4 0 0
init.direction = 1 1 1
stepper.dt = 1e-14
output.csv = traj.csv
output.dump = final.dump
output.sample_every = 100
"""


@needs_ref
def test_cli_run_matches_reference(tmp_path):
    (tmp_path / "a.cfg").write_text(CFG)
    r = cli("run", "--config", "a.cfg", "--steps", "250", cwd=tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout.splitlines()
    assert "default applied: material.gamma = 176085963000" in out
    assert out[-4].startswith("final: step 250, t 2.5e-12 s, NOT converged")
    rows = np.loadtxt(tmp_path / "traj.csv", delimiter=",", skiprows=1)
    assert (tmp_path / "traj.csv").read_text().splitlines()[0].startswith("step,t_s,mx,my,mz,E_exch_J")
    assert list(rows[:, 0]) == [0, 100, 200, 250]                 # sample at step % 100 == 0, then final
    # the reference, same spec, from the same state
    spec = O.Spec(16, 8, 2, 2.5e-9, 2.5e-9, 3e-9, A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.1, h_ext=(1e4, 0, 0), dt=1e-14)
    ref = O.Ref(spec, 64)
    u = np.full((3, spec.n), 8e5 / np.sqrt(3.0))
    ref.set_m(u)
    done = 0
    for row in rows:
        k = int(row[0]) - done
        if k > 0:
            ref.step(k)
            done += k
        m = ref.get_m()
        np.testing.assert_allclose(row[2:5], m.mean(axis=1) / 8e5, rtol=0, atol=1e-12)
        e = ref.energies()
        np.testing.assert_allclose(row[5:10], e, rtol=1e-9, atol=1e-30)
        t0 = ref.time()
        tq = ref.step(1)[0]      # the sample's torque = the next step's pre-step value
        ref.set_m(m)
        ref.set_time(*t0)
        np.testing.assert_allclose(row[10], tq, rtol=1e-9)
    d = F.read_field_dump(str(tmp_path / "final.dump"))
    assert d.precision == "f64" and d.grid.nx == 16 and d.Ms == 8e5
    np.testing.assert_allclose(d.M, m, rtol=0, atol=1e-9 * 8e5)


ZEEMAN = """grid.nx = 1
grid.ny = 1
grid.nz = 1
grid.dx = 2e-9
grid.dy = 2e-9
grid.dz = 2e-9
material.Ms = 8e5
material.alpha = 0.5
terms.exchange = false
terms.anisotropy = false
terms.demag = false
field.extern = 0 0 1e5
init.kind = uniform
init.direction = 1 0 0
stepper.dt = 1e-12
stepper.max_steps = 100000
stepper.torque_tol = 0.05
output.csv = z.csv
output.dump = z.dump
output.sample_every = 50
"""


@needs_ref
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_cli_relax_single_cell(tmp_path, prec):
    (tmp_path / "z.cfg").write_text(ZEEMAN + f"precision = {prec}\n")
    r = cli("relax", "--config", "z.cfg", cwd=tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    spec = O.Spec(1, 1, 1, 2e-9, 2e-9, 2e-9, Ms=8e5, alpha=0.5, exchange=False, anisotropy=False, demag=False,
                  h_ext=(0, 0, 1e5), dt=1e-12, max_steps=100000, torque_tol=0.05, sample_every=50)
    ref = O.Ref(spec, 32 if prec == "f32" else 64)
    ref.set_m(np.array([[8e5], [0.0], [0.0]]))
    conv, log = ref.relax()
    assert conv
    rows = np.loadtxt(tmp_path / "z.csv", delimiter=",", skiprows=1, ndmin=2)
    assert [int(s.step) for s in log] == [int(x) for x in rows[:, 0]]      # same cadence and stop step
    last = log[-1]
    assert f"final: step {last.step}, t " in r.stdout and ", converged" in r.stdout
    np.testing.assert_allclose(rows[-1, 2:5], list(last.m), atol=1e-6 if prec == "f32" else 1e-12)
    assert "max torque " in r.stdout.splitlines()[-1]


def test_cli_bench_csv(tmp_path):
    r = cli("bench", "--sizes", "8,16", "--csv", "b.csv", cwd=tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = (tmp_path / "b.csv").read_text().splitlines()
    assert lines[0].startswith("size,ms_per_step,pad_ms") and len(lines) == 3
    assert [l.split(",")[0] for l in lines[1:]] == ["8", "16"]
    assert all(float(l.split(",")[1]) > 0 for l in lines[1:])


def test_cli_errors(tmp_path):
    (tmp_path / "bad.cfg").write_text("grid.nx = 4\ngrid.nx = 5\n")
    r = cli("run", "--config", "bad.cfg", "--steps", "1", cwd=tmp_path)
    assert r.returncode == 1 and "error: config line 2: duplicate key 'grid.nx'" in r.stderr
    r = cli("relax", "--config", "missing.cfg", cwd=tmp_path)
    assert r.returncode == 1 and "error: cannot open config file: missing.cfg" in r.stderr
    (tmp_path / "ok.cfg").write_text(ZEEMAN)
    r = cli("run", "--config", "ok.cfg", "--steps", "-1", cwd=tmp_path)
    assert r.returncode == 1 and "error: steps must be >= 0" in r.stdout
