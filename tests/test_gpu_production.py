"""GPU parity on the kernel instantiations the benchmark times.

The small-grid parity tests (test_gpu_parity.py) pick the few-row x-pass
variants and non-FZ z passes; the BASELINE configs run different template
instantiations.  Every case here (a) checks against the reference itself
(oracle/_ref: DemagConvolution::field, EffectiveFieldProvider::compute and
Simulation<T>::step, demag.hpp:194-251, fields.hpp:220-253, sim.hpp:33-42) and
(b) asserts through mfd_debug_variants that the production variant of every
pass actually ran.

Production variants (ncu launch list of bench.py, profiles/r1/launches_v6_summary.txt):
  C4 512x512x64 f32: k_r2c_x<f32,512,RS=0>, k_fft_y_fwd_tma<f32,1024,FY=1>,
  k_fft_z_conv2<f32,128,FZ=1,SROW=1>, k_fft_y_inv_tma<f32,1024,FY=1>,
  k_c2r_x_llg_v<f32,512,SUMS=0,RS=0,FWD=0>.
Grids: 128x128x64 (the bench's old CPU sample; fused K1-in-K5 at N=128, the C4 K3,
K4 TMA at L=256), 512x512x4 (every C4 x/y instantiation, K5 unfused via
MFD_FUSE_K1=0), C2 512x128x4, C3 128^3, and C4 itself (slow).

Tolerances: f32 H rel L-inf <= 1e-5 with the device
tensor; f64 <= 1e-11 with the reference's own tensor injected
(set_demag_octant: the reference's long-double Newell is itself only ~1e-7
accurate at >= 100 cells).  20 steps: torques and M within
2e-5 (f32) / 1e-10 (f64).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import engine_sim

pytestmark = pytest.mark.gpu

BENCH = dict(A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.02, easy_axis=(0.0, 0.0, 1.0), h_ext=(1e4, 0.0, 0.0), dt=1e-14)


def bench_spec(nx, ny, nz, d=2.5e-9, **kw):
    p = dict(BENCH)
    p.update(kw)
    return O.Spec(nx, ny, nz, d, d, d, parallel=True, threads=0, **p)


def need_ref():
    if not O.ref_available():
        pytest.skip("reference .so (oracle/_ref) not built")


def run_case(spec, prec, expect, env=None, steps=20, seed=31):
    need_ref()
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        sim = engine_sim(spec, prec)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ref = O.Ref(spec, prec)
    if prec == 64:
        sim.set_demag_octant(O.tensor_octant(spec.nx, spec.ny, spec.nz, spec.dx, spec.dy, spec.dz, which="ref"))
    m = O.random_unit_field(spec.n, spec.Ms, seed)
    if prec == 32:
        m = m.astype(np.float32).astype(np.float64)
    sim.set_m(m)
    ref.set_m(m)
    tol_h = 1e-5 if prec == 32 else 1e-11
    assert O.rel_linf(sim.demag_field(), ref.hdemag()) <= tol_h
    assert O.rel_linf(sim.effective_field(), ref.heff()) <= tol_h
    t_mine = sim.step(steps, return_all=True)
    t_ref = ref.step(steps)
    tol_s = 2e-5 if prec == 32 else 1e-10
    assert np.max(np.abs(t_mine - t_ref) / np.abs(t_ref)) <= tol_s
    assert O.rel_linf(sim.get_m(), ref.get_m()) <= tol_s
    assert sim.time() == ref.time()
    ran = sim.variants()
    print("\n".join(ran))
    missing = [v for v in expect if v not in ran]
    assert not missing, (missing, ran)
    return sim, ran


def test_film_128x128x64_f32():
    """fused K1-in-K5 RS=0 at N=128, the C4 K3 (FZ, one y row per CTA), K4 TMA at L=256."""
    run_case(bench_spec(128, 128, 64), 32, [
        "K1 k_r2c_x<f32,128,RS=0,MULTI=0>",
        "K2 k_fft_y_fwd<f32,256,FY=1>",
        "K3 k_fft_z_conv2<f32,128,FZ=1,SROW=1>",
        "K4 k_fft_y_inv_tma<f32,256,FY=1>",
        "K5 k_c2r_x_llg_v<f32,128,SUMS=0,RS=0,FWD=1,MULTI=0>",
        "K5 k_c2r_x_llg_v<f32,128,SUMS=0,RS=0,FWD=0,MULTI=0>",
    ])


def test_film_128x128x64_f64():
    """f64: the pair form of K3 (SROW=0), f64 K4 TMA at L=256."""
    run_case(bench_spec(128, 128, 64), 64, [
        "K1 k_r2c_x<f64,128,RS=0,MULTI=0>",
        "K3 k_fft_z_conv2<f64,128,FZ=1,SROW=0>",
        "K5 k_c2r_x_llg_v<f64,128,SUMS=0,RS=0,FWD=1,MULTI=0>",
    ])


@pytest.mark.parametrize("prec", [32, 64])
def test_c4_xy_passes_512x512x4(prec):
    """Every x/y instantiation of C4 (N=512 K1/K5 RS=0, y passes at L=1024), K5 unfused as at C4."""
    t = "f32" if prec == 32 else "f64"
    expect = [f"K1 k_r2c_x<{t},512,RS=0,MULTI=0>",
              f"K5 k_c2r_x_llg_v<{t},512,SUMS=0,RS=0,FWD=0,MULTI=0>"]
    if prec == 32:
        expect += ["K2 k_fft_y_fwd_tma<f32,1024,FY=1>", "K4 k_fft_y_inv_tma<f32,1024,FY=1>"]
    else:   # three-stage plan
        expect += ["K2 k_fft_y_fwd_tma<f64,1024,FY=1>", "K4 k_fft_y_inv_tma<f64,1024,FY=1>"]
    run_case(bench_spec(512, 512, 4), prec, expect, env={"MFD_FUSE_K1": "0"}, steps=12)


def test_sp4_refined_c2_f32():
    """C2: SP4 refined 512x128x4 (permalloy, no anisotropy), the bench's sp4fine workload."""
    s = bench_spec(512, 128, 4, Ku=0.0, h_ext=(-19576.1, 3421.8, 0.0), dt=4e-15)
    s.dx, s.dy, s.dz = 500e-9 / 512, 125e-9 / 128, 0.75e-9
    run_case(s, 32, ["K1 k_r2c_x<f32,512,RS=2,MULTI=0>",
                     "K5 k_c2r_x_llg_v<f32,512,SUMS=0,RS=1,FWD=1,MULTI=0>"])


def test_sp4_refined_c2_f64():
    s = bench_spec(512, 128, 4, Ku=0.0, h_ext=(-19576.1, 3421.8, 0.0), dt=4e-15)
    s.dx, s.dy, s.dz = 500e-9 / 512, 125e-9 / 128, 0.75e-9
    # f64 K5 runs one row per CTA at N = 512, so 512 rows fill the SMs without the 1-2-row variants
    run_case(s, 64, ["K1 k_r2c_x<f64,512,RS=0,MULTI=0>", "K5 k_c2r_x_llg_v<f64,512,SUMS=0,RS=0,FWD=1,MULTI=0>"],
             steps=10)


def test_cube_c3_f32():
    """C3 128^3: K3 at Pz=256 (radix 32 x 8, 16 columns), fused K1 at N=128."""
    run_case(bench_spec(128, 128, 128), 32, [
        "K1 k_r2c_x<f32,128,RS=0,MULTI=0>",
        "K3 k_fft_z_conv2<f32,256,FZ=1,SROW=1>",
        "K4 k_fft_y_inv_tma<f32,256,FY=1>",
        "K5 k_c2r_x_llg_v<f32,128,SUMS=0,RS=0,FWD=1,MULTI=0>",
    ], steps=10)


@pytest.mark.slow
def test_film_c4_f32_full():
    """C4 512x512x64 itself, f32, against the reference (setup ~1-3 min on the host)."""
    run_case(bench_spec(512, 512, 64), 32, [
        "K1 k_r2c_x<f32,512,RS=0,MULTI=0>",
        "K2 k_fft_y_fwd_tma<f32,1024,FY=1>",
        "K3 k_fft_z_conv2<f32,128,FZ=1,SROW=1>",
        "K4 k_fft_y_inv_tma<f32,1024,FY=1>",
        "K5 k_c2r_x_llg_v<f32,512,SUMS=0,RS=0,FWD=0,MULTI=0>",
    ], steps=5)


def test_sample_sums_production_k5():
    """SUMS=1 K5 at N=512 RS=0 (<m>, energies) against the reference's sampleNow."""
    need_ref()
    s = bench_spec(512, 512, 4)
    sim = engine_sim(s, 64)
    ref = O.Ref(s, 64)
    sim.set_demag_octant(O.tensor_octant(s.nx, s.ny, s.nz, s.dx, s.dy, s.dz, which="ref"))
    m = O.random_unit_field(s.n, s.Ms, 5)
    sim.set_m(m)
    ref.set_m(m)
    smp = sim.sample_now()
    e_ref = ref.energies()
    got = np.array([smp.e_exchange, smp.e_anisotropy, smp.e_demag, smp.e_zeeman, smp.e_total])
    assert np.allclose(got, e_ref, rtol=1e-10, atol=0)
    assert np.allclose(smp.m, m.sum(axis=1) / (s.Ms * s.n), rtol=0, atol=1e-14)
    assert "K5 k_c2r_x_llg_v<f64,512,SUMS=1,RS=0,FWD=0,MULTI=0>" in sim.variants()
