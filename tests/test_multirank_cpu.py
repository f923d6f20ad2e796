"""World-size-2 CPU (gloo) test of the multi-GPU decomposition logic.

Two processes run the z-slab algorithm of the engine in numpy with the exact
block layout of the device path (paper_1406_7459_b200/decomposition.py ==
csrc Slab/Geo): local x (R2C) FFT on the slab into [block][3][nzl][ny][Wb],
all_to_all, y FFT + z FFT + tensor product + inverse z / y on the rank's
x-bin block of every plane, all_to_all back, inverse x; and the one-plane M
halo for the exchange stencil.  The gathered fields must equal the
single-process oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1406_7459_b200 import decomposition as D

GRID = (10, 6, 8, 2e-9, 3e-9, 2e-9)
MS = 8e5


def _spec(**kw):
    base = dict(A=1.3e-11, Ku=0.0, Ms=MS, alpha=0.5, h_ext=(0.0, 0.0, 0.0), zeeman=False, anisotropy=False)
    base.update(kw)
    return O.Spec(*GRID, **base)


def full_kernel_spectrum(nx, ny, nz, dx, dy, dz):
    """K~ over the full padded lattice from the (port) tensor octant, mirrored with
    the parity signs of demag.hpp:71-87."""
    px, py, pz = (D.padded_size(n) for n in (nx, ny, nz))
    oct6 = O.tensor_octant(nx, ny, nz, dx, dy, dz, which="port")
    K = np.zeros((6, pz, py, px))
    sgn = [(1, 1, 1)] * 3 + [(-1, -1, 1), (-1, 1, -1), (1, -1, -1)]
    for c in range(6):
        for sz in (0, 1):
            for sy in (0, 1):
                for sx in (0, 1):
                    kk = np.arange(nz) if not sz else (pz - np.arange(1, nz)) % pz
                    jj = np.arange(ny) if not sy else (py - np.arange(1, ny)) % py
                    ii = np.arange(nx) if not sx else (px - np.arange(1, nx)) % px
                    src = oct6[c][slice(1, None) if sz else slice(None), slice(1, None) if sy else slice(None),
                                  slice(1, None) if sx else slice(None)]
                    f = (sgn[c][0] if sx else 1) * (sgn[c][1] if sy else 1) * (sgn[c][2] if sz else 1)
                    K[c][np.ix_(kk, jj, ii)] = f * src
    return np.fft.fftn(K, axes=(1, 2, 3)).real


def alltoall(send: np.ndarray, world: int) -> np.ndarray:
    """[G][...] complex blocks -> [G][...] (block g from rank g)."""
    s = torch.from_numpy(np.ascontiguousarray(send).view(np.float64).reshape(-1))
    r = torch.empty_like(s)
    dist.all_to_all_single(r, s)
    return r.numpy().view(np.complex128).reshape(send.shape)


def worker(rank, world, port, m, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz = GRID[:3]
    sl = D.slab(nz, rank, world)
    bl = D.blocks(nx, ny, nz, world)
    px, py, pz = (D.padded_size(n) for n in (nx, ny, nz))
    Kf = full_kernel_spectrum(*GRID)
    M = m.reshape(3, nz, ny, nx)[:, sl.k0:sl.k0 + sl.nzl]          # this rank's slab

    # K1 on the slab, packed by destination block (bin u -> block_of(u))
    A = np.fft.rfft(M, n=px, axis=3)                               # [3][nzl][ny][Hx]
    send = np.zeros((world, 3, sl.nzl, ny, bl.Wb), complex)
    for u in range(bl.Hx):
        p = bl.block_of(u)
        send[p, ..., u - p * bl.Wb] = A[..., u]
    recv = alltoall(send, world)                                   # block g: planes of rank g

    # K2 + K3 + K4 on this rank's x-bin block of every plane
    hv, u0 = bl.valid(rank), rank * bl.Wb
    Z = np.concatenate([recv[g] for g in range(world)], axis=1)    # [3][nz][ny][Wb]
    Zf = np.fft.fft(np.fft.fft(Z, n=py, axis=2), n=pz, axis=1)     # [3][Pz][Py][Wb]
    k = Kf[:, :, :, u0:u0 + hv]
    xx, yy, zz, xy, xz, yz = k
    a, b, c = Zf[0, ..., :hv], Zf[1, ..., :hv], Zf[2, ..., :hv]
    H = np.zeros_like(Zf)
    H[0, ..., :hv] = xx * a + xy * b + xz * c
    H[1, ..., :hv] = xy * a + yy * b + yz * c
    H[2, ..., :hv] = xz * a + yz * b + zz * c
    Hyz = (np.fft.ifft(np.fft.ifft(H, axis=1)[:, :nz] * pz, axis=2) * py)[:, :, :ny]
    back = np.stack([Hyz[:, g * sl.nzl:(g + 1) * sl.nzl] for g in range(world)])
    mine = alltoall(back, world)                                   # block p: my planes, x-bins of rank p

    # K5 (demag part) on the slab
    Hs = np.zeros((3, sl.nzl, ny, bl.Hx), complex)
    for p in range(world):
        hvp = bl.valid(p)
        Hs[..., p * bl.Wb:p * bl.Wb + hvp] = mine[p, ..., :hvp]
    hd = np.fft.irfft(Hs, n=px, axis=3)[..., :nx] * px / (px * py * pz)

    # one-plane halo of M for the exchange stencil (Neumann at the global ends)
    lo = np.zeros((3, ny, nx))
    hi = np.zeros((3, ny, nx))
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(M[:, 0])), rank - 1))
        t_lo = torch.empty(3, ny, nx, dtype=torch.float64)
        reqs.append(dist.irecv(t_lo, rank - 1))
    if rank < world - 1:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(M[:, -1])), rank + 1))
        t_hi = torch.empty(3, ny, nx, dtype=torch.float64)
        reqs.append(dist.irecv(t_hi, rank + 1))
    for r in reqs:
        r.wait()
    if rank > 0:
        lo = t_lo.numpy()
    if rank < world - 1:
        hi = t_hi.numpy()
    ext = np.concatenate([lo[:, None], M, hi[:, None]], axis=1)    # [3][nzl+2][ny][nx]
    w = 2 * 1.3e-11 / (O.MU0 * MS * MS) / np.array(GRID[3:]) ** 2
    h = np.zeros_like(M)
    kg = sl.k0 + np.arange(sl.nzl)
    for kk in range(sl.nzl):
        cen = ext[:, kk + 1]
        hh = np.zeros_like(cen)
        hh[:, :, 1:] += w[0] * (cen[:, :, :-1] - cen[:, :, 1:])
        hh[:, :, :-1] += w[0] * (cen[:, :, 1:] - cen[:, :, :-1])
        hh[:, 1:] += w[1] * (cen[:, :-1] - cen[:, 1:])
        hh[:, :-1] += w[1] * (cen[:, 1:] - cen[:, :-1])
        if kg[kk] > 0:
            hh += w[2] * (ext[:, kk] - cen)
        if kg[kk] < nz - 1:
            hh += w[2] * (ext[:, kk + 2] - cen)
        h[:, kk] = hh

    parts = [None] * world
    dist.all_gather_object(parts, (rank, hd, h))
    if rank == 0:
        parts.sort(key=lambda x: x[0])
        np.savez(out_path, hd=np.concatenate([p[1] for p in parts], axis=1),
                 hx=np.concatenate([p[2] for p in parts], axis=1))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_slab_decomposition_gloo(world, tmp_path):
    n = GRID[0] * GRID[1] * GRID[2]
    m = O.random_unit_field(n, MS, 37)
    out = str(tmp_path / "fields.npz")
    mp.spawn(worker, args=(world, free_port(), m, out), nprocs=world, join=True)
    z = np.load(out)
    ref = O.Port(_spec(exchange=False), 64)
    ref.set_m(m)
    assert O.rel_linf(z["hd"].reshape(3, -1), ref.hdemag()) <= 1e-12
    ex = O.Port(_spec(demag=False), 64)
    ex.set_m(m)
    assert O.rel_linf(z["hx"].reshape(3, -1), ex.heff()) <= 1e-12


def test_partition_math_matches_device_rules():
    b = D.blocks(512, 512, 64, 8)
    assert (b.Hx, b.Wb, b.nzl) == (513, 80, 8)
    assert sum(b.valid(r) for r in range(8)) == 513
    assert b.Wb % 16 == 0 and 8 * b.Wb >= b.Hx
    one = D.blocks(512, 512, 64, 1)
    assert one.Wb == 528 and one.S_c == 64 * 1024 * 528     # single GPU: [3][nz][Py][Hp]
    assert one.SA == 3 * 64 * 512 * 528                     # single GPU: A = [3][nz][ny][Hp]
    # the device's reciprocal block index equals u // Wb for every bin
    for G in (2, 4, 8):
        for n in (16, 100, 512, 1024, 2048):
            bb = D.blocks(n, 8, 8 * G, G)
            assert all(bb.block_of(u) == u // bb.Wb for u in range(bb.Hx))
    with pytest.raises(ValueError, match="divisible"):
        D.slab(64, 0, 3)
    # per-rank transpose volume at 8 GPUs, fp32: 2 transposes x 7 remote blocks of
    # 3*nzl*ny*Wb complex (the x-spectrum is moved)
    assert D.alltoall_bytes_per_rank(512, 512, 64, 8) == 2 * 7 * 3 * 8 * 512 * 80 * 8
