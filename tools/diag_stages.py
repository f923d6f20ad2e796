"""Localise FFT-pipeline errors: compare every intermediate buffer with numpy."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from tests.helpers import engine_sim
from tests.test_gpu_parity import spec_of

PLANS = {32: {1: [1], 2: [2], 4: [4], 8: [8], 16: [16], 32: [32], 64: [8, 8], 128: [16, 8], 256: [16, 16],
              512: [32, 16], 1024: [32, 32], 2048: [16, 16, 8]},
         64: {1: [1], 2: [2], 4: [4], 8: [8], 16: [16], 32: [8, 4], 64: [8, 8], 128: [16, 8], 256: [16, 16],
              512: [16, 8, 4], 1024: [16, 8, 8], 2048: [16, 16, 8]}}


def bufpos(prec, L, f):
    rs = PLANS[prec][L]
    if len(rs) <= 1:
        return f
    pos, rem, pre = 0, f, 1
    for s, R in enumerate(rs):
        k = rem % R
        rem //= R
        pre *= R
        pos += k * (L // pre)
    return pos


def full_kernel(g):
    nx, ny, nz = g[:3]
    px, py, pz = (O.padded(n) for n in (nx, ny, nz))
    oct6 = O.tensor_octant(*g, which="ref")
    K = np.zeros((6, pz, py, px))
    sgn = [(1, 1, 1), (1, 1, 1), (1, 1, 1), (-1, -1, 1), (-1, 1, -1), (1, -1, -1)]
    for c in range(6):
        for sx in (0, 1):
            for sy in (0, 1):
                for sz in (0, 1):
                    ii = np.arange(nx) if not sx else (px - np.arange(1, nx)) % px
                    jj = np.arange(ny) if not sy else (py - np.arange(1, ny)) % py
                    kk = np.arange(nz) if not sz else (pz - np.arange(1, nz)) % pz
                    src = oct6[c][(slice(None) if not sz else slice(1, None)),
                                  (slice(None) if not sy else slice(1, None)),
                                  (slice(None) if not sx else slice(1, None))]
                    f = (sgn[c][0] if sx else 1) * (sgn[c][1] if sy else 1) * (sgn[c][2] if sz else 1)
                    K[c][np.ix_(kk, jj, ii)] = f * src
    return np.fft.fftn(K, axes=(1, 2, 3)), oct6


def run(g, prec):
    nx, ny, nz = g[:3]
    px, py, pz = (O.padded(n) for n in (nx, ny, nz))
    hx = px // 2 + 1
    s = spec_of(g)
    sim = engine_sim(s, prec)
    Kf, oct6 = full_kernel(g)
    sim.set_demag_octant(oct6)
    m = O.random_unit_field(s.n, s.Ms, 3)
    sim.set_m(m)
    M = m.reshape(3, nz, ny, nx)
    A = np.fft.rfft(M, n=px, axis=3)                         # [3][nz][ny][hx]
    By = np.fft.fft(A, n=py, axis=2)                         # [3][nz][py][hx]
    Bz = np.fft.fft(By, n=pz, axis=1)                        # [3][pz][py][hx]
    Kh = Kf[:, :, :, :hx]
    xx, yy, zz, xy, xz, yz = Kh
    H = np.stack([xx * Bz[0] + xy * Bz[1] + xz * Bz[2], xy * Bz[0] + yy * Bz[1] + yz * Bz[2],
                  xz * Bz[0] + yz * Bz[1] + zz * Bz[2]])
    B3 = np.fft.ifft(H, axis=1)[:, :nz] * pz
    A4 = (np.fft.ifft(B3, axis=2) * py)[:, :, :ny]
    perm = [bufpos(prec, py, v) for v in range(py)]
    inv = np.argsort(perm)
    out = {}
    for st, want in ((1, A), (2, By), (3, B3), (4, A4)):
        got = sim.debug_stage(st)[..., :hx]
        if st in (2, 3):
            got = got[:, :, perm, :]        # buffer row b(v) -> natural v
        err = np.max(np.abs(got - want)) / np.max(np.abs(want))
        out[st] = err
    hd = sim.demag_field()
    href = O.Ref(s, 64)
    href.set_m(m)
    print(g[:3], prec, ' '.join(f'K{k}:{v:.1e}' for k, v in out.items()),
          f'H:{O.rel_linf(hd, href.hdemag()):.1e}', flush=True)


for prec in (64, 32):
    for g in [(2, 2, 2, 2e-9, 2e-9, 2e-9), (4, 4, 4, 2e-9, 2e-9, 2e-9), (5, 3, 2, 1e-9, 2e-9, 3e-9),
              (8, 8, 1, 2e-9, 2e-9, 2e-9), (16, 8, 4, 3e-9, 2e-9, 1e-9), (64, 48, 40, 2e-9, 2e-9, 2e-9)]:
        try:
            run(g, prec)
        except Exception as e:
            print(g[:3], prec, 'EXC', e, flush=True)
            break
