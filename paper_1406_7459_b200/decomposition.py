"""Host-side partition logic of the z-slab decomposition (mirrors the C++ in
csrc/engine.cuh Slab::of and csrc/engine_impl.cuh).

Rank r of G owns z-planes [k0, k0 + nz/G) for the x/y passes and the LLG
update, and x-bin block r (width Wb, a multiple of 16) of every z column for
the z pass.  The y-spectrum is laid out [block][3][nzl][Py][Wb] so each of the
two all-to-all transposes moves G contiguous blocks of S_blk elements.
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
    Wb: int      # block width
    Py: int
    nzl: int

    def valid(self, rank: int) -> int:
        """Valid x bins in block `rank` (Hv)."""
        return max(0, min(self.Wb, self.Hx - rank * self.Wb))

    @property
    def S_k(self) -> int:
        return self.Py * self.Wb

    @property
    def S_c(self) -> int:
        return self.nzl * self.S_k

    @property
    def S_blk(self) -> int:
        return 3 * self.S_c


def blocks(nx: int, ny: int, nz: int, world: int) -> Blocks:
    Hx = padded_size(nx) // 2 + 1
    Hp = (Hx + 15) // 16 * 16
    Wb = Hp if world == 1 else ((Hx + world - 1) // world + 15) // 16 * 16
    return Blocks(Hx, Wb, padded_size(ny), nz // world)


def alltoall_bytes_per_rank(nx: int, ny: int, nz: int, world: int, itemsize: int = 4) -> int:
    """Bytes a rank sends per step (both transposes), excluding its own block."""
    b = blocks(nx, ny, nz, world)
    return 2 * (world - 1) * b.S_blk * 2 * itemsize
