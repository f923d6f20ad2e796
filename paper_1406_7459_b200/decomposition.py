"""Host-side partition logic of the z-slab decomposition (mirrors the C++ in
csrc/engine.cuh Slab::of and csrc/engine_impl.cuh).

Rank r of G owns z-planes [k0, k0 + nz/G) for the x passes (K1, K5) and the
LLG update, and x-bin block r (width Wb, a multiple of 16) of every plane for
the y and z passes (K2-K4).  The x-spectrum A is laid out
[block][3][nzl][ny][Wb], so each of the two all-to-all transposes (after K1,
before K5) moves G contiguous blocks of SA elements; it has ny rows, not the
Py = 2 ny of the y-spectrum, so it moves half the bytes of a transpose after
the y pass.  The y-spectrum B = [3][nz][Py][Wb] is rank-local.
"""
from dataclasses import dataclass


def padded_size(n: int) -> int:
    p = 1
    while p < 2 * n:
        p <<= 1
    return p


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    k0: int
    nzl: int


def slab(nz: int, rank: int, world: int) -> Slab:
    if nz % world:
        raise ValueError("magfd-b200: nz must be divisible by the number of GPUs (z-slab decomposition)")
    nzl = nz // world
    return Slab(rank, world, rank * nzl, nzl)


@dataclass(frozen=True)
class Blocks:
    Hx: int      # x bins (Px/2 + 1)
    Wb: int      # block width (= A row pitch)
    Py: int
    nzl: int
    ny: int
    nz: int

    def valid(self, rank: int) -> int:
        """Valid x bins in block `rank` (Hv)."""
        return max(0, min(self.Wb, self.Hx - rank * self.Wb))

    @property
    def S_k(self) -> int:
        return self.Py * self.Wb

    @property
    def S_c(self) -> int:
        """B component stride: all nz planes of the rank's x-bin block."""
        return self.nz * self.S_k

    @property
    def SA(self) -> int:
        """A block (one destination rank): 3 x nzl x ny rows of Wb bins."""
        return 3 * self.nzl * self.ny * self.Wb

    def block_of(self, u: int) -> int:
        """Block of x-bin u, as the device computes it: (u * ceil(2^24 / Wb)) >> 24."""
        binv = ((1 << 24) + self.Wb - 1) // self.Wb
        return (u * binv) >> 24


def blocks(nx: int, ny: int, nz: int, world: int) -> Blocks:
    Hx = padded_size(nx) // 2 + 1
    Hp = (Hx + 15) // 16 * 16
    Wb = Hp if world == 1 else ((Hx + world - 1) // world + 15) // 16 * 16
    return Blocks(Hx, Wb, padded_size(ny), nz // world, ny, nz)


def alltoall_bytes_per_rank(nx: int, ny: int, nz: int, world: int, itemsize: int = 4) -> int:
    """Bytes a rank sends per step (both transposes), excluding its own block."""
    b = blocks(nx, ny, nz, world)
    return 2 * (world - 1) * b.SA * 2 * itemsize
