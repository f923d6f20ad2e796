"""The one-process-per-GPU engine path (mfd_exec.world > 1, virtual_ranks = 0),
run as 2 and 4 processes on ONE B200 through the host-staged shared-memory
transport (transport="shm").

Everything but the byte mover is the production multi-GPU code: each process
owns its z slab (rank-local set/get), builds only its x-bin block of the
tensor spectrum, runs K1 -> all-to-all #1 per component on a second stream
overlapping K2 -> K3 -> K4 overlapping all-to-all #2 -> K5 after the
one-plane halo, all captured into the step graphs together with the torque /
error / sample allreduces, and relax decides its stop step from the
allreduced torque.  NCCL itself refuses two ranks on one device, so the
transfers go D2H -> shared file -> H2D with host barriers (no kernel waits on
another process).  Fields, torques and trajectories must equal the one-rank
engine bitwise; the fp64 sample sums reassociate (rank order).
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

MS = 8e5
TIMEOUT = 240


def make(g, prec, world=1, rank=0, idb=None, **kw):
    import paper_1406_7459_b200 as E
    nx, ny, nz, dx, dy, dz = g
    mat = E.Material(A=1.3e-11, Ku=4e4, Ms=MS, alpha=kw.get("alpha", 0.5), easy_axis=(0.6, 0.0, 0.8))
    fields = E.FieldConfig(True, True, kw.get("demag", True), True, (2e4, -1e4, 3e4))
    st = E.StepperConfig(dt=kw.get("dt", 1e-14), max_steps=kw.get("max_steps", 500000),
                         torque_tol_deg_per_ns=kw.get("torque_tol", 0.01), sample_every=kw.get("sample_every", 100))
    extra = dict(world=world, rank=rank, nccl_id=idb, transport="shm") if world > 1 else {}
    return E.Simulation(E.Grid(nx, ny, nz, dx, dy, dz), mat, fields, st, precision=prec, **extra)


def _steps_job(sim, m, n):
    out = {"m0": sim.get_m()}
    sim.set_m(m)
    out["m0"] = sim.get_m()
    out["hd"] = sim.demag_field() if sim.fields.demag else None
    out["he"] = sim.effective_field()
    out["t"] = sim.step(6, return_all=True)
    out["m"] = sim.get_m()
    out["time"] = sim.time()
    sim.step_async(70)          # graph chunks of 64 + 6 steps, no host sync inside
    sim.sync()
    out["m2"] = sim.get_m()
    out["time2"] = sim.time()
    s = sim.sample_now()
    out["smp"] = (np.array(s.m), s.e_total, s.max_torque_deg_per_ns)
    out["variants"] = sim.variants()
    return out


def _relax_job(sim, m, n):
    sim.set_m(m)
    conv, log = sim.relax()
    return {"conv": conv, "steps": [x.step for x in log], "ms": [np.array(x.m) for x in log],
            "torques": [x.max_torque_deg_per_ns for x in log], "m": sim.get_m(), "time": sim.time()}


JOBS = {"steps": _steps_job, "relax": _relax_job}


def _worker(rank, world, idb, g, prec, kw, m, job, q):
    try:
        sim = make(g, prec, world, rank, idb, **kw)
        n = sim.n
        res = JOBS[job](sim, np.ascontiguousarray(m[:, rank * n:(rank + 1) * n]), n)
        sim.close()
        q.put((rank, res, None))
    except BaseException:
        import traceback
        q.put((rank, None, traceback.format_exc()))


def run_ranks(world, g, prec, m, job, **kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    idb = os.urandom(16) + bytes(112)
    ps = [ctx.Process(target=_worker, args=(r, world, idb, g, prec, kw, m, job, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    try:
        for _ in range(world):
            rank, res, err = q.get(timeout=TIMEOUT)
            assert err is None, f"rank {rank} failed:\n{err}"
            out[rank] = res
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    return [out[r] for r in range(world)]


def cat(parts, key):
    return np.concatenate([p[key] for p in parts], axis=1)


GRIDS = [(16, 12, 8, 2e-9, 2e-9, 2e-9), (33, 17, 4, 2e-9, 3e-9, 2e-9), (64, 32, 16, 2e-9, 2e-9, 2e-9)]


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("world,g", [(2, GRIDS[0]), (2, GRIDS[1]), (4, GRIDS[2]), (2, GRIDS[2])])
def test_processes_match_single_rank(world, g, prec):
    m = O.random_unit_field(g[0] * g[1] * g[2], MS, 23)
    one = make(g, prec)
    ref = _steps_job(one, m, one.n)
    parts = run_ranks(world, g, prec, m, "steps")
    for key in ("m0", "hd", "he", "m", "m2"):
        assert np.array_equal(cat(parts, key), ref[key]), key
    for p in parts:
        assert np.array_equal(p["t"], ref["t"])
        assert p["time"] == ref["time"] and p["time2"] == ref["time2"]
        assert np.allclose(p["smp"][0], ref["smp"][0], rtol=0, atol=1e-13)
        assert abs(p["smp"][1] - ref["smp"][1]) <= 1e-12 * abs(ref["smp"][1])
        assert p["smp"][2] == ref["smp"][2]   # torque max is exact (integer max of the bit pattern)
    # the multi-process K1 / K5 variants (blocked x-bin layout) actually ran
    assert any("MULTI=1" in v and v.startswith("K1") for v in parts[0]["variants"])
    assert any("MULTI=1" in v and v.startswith("K5") for v in parts[0]["variants"])


def test_processes_demag_off_halo():
    """demag off: only the one-plane halo crosses processes (exchange stencil)."""
    g = (20, 10, 8, 2e-9, 2e-9, 2e-9)
    m = O.random_unit_field(g[0] * g[1] * g[2], MS, 29)
    one = make(g, 64, demag=False)
    ref = _steps_job(one, m, one.n)
    parts = run_ranks(2, g, 64, m, "steps", demag=False)
    for key in ("he", "m", "m2"):
        assert np.array_equal(cat(parts, key), ref[key]), key


def test_processes_relax_stop_step():
    """dynamics::relax on two processes: the allreduced torque gives every rank the
    reference's stop step; the state equals the one-rank relax bitwise."""
    g = (8, 8, 4, 5e-9, 5e-9, 5e-9)
    kw = dict(alpha=1.0, dt=1e-13, torque_tol=50.0, max_steps=3000, sample_every=50)
    m = O.random_unit_field(g[0] * g[1] * g[2], MS, 31)
    one = make(g, 64, **kw)
    ref = _relax_job(one, m, one.n)
    parts = run_ranks(2, g, 64, m, "relax", **kw)
    for p in parts:
        assert p["conv"] == ref["conv"] and p["steps"] == ref["steps"] and p["time"] == ref["time"]
        assert p["torques"] == ref["torques"]
        for a, b in zip(p["ms"], ref["ms"]):
            assert np.allclose(a, b, rtol=0, atol=1e-13)
    assert np.array_equal(cat(parts, "m"), ref["m"])
