"""Morton-subtree partition plan.

The finest Morton range is split into G contiguous ranges of level-R subtrees
(R = L - min(L, 6), the engine's subtree level): partition g owns subtrees
[g*4^R/G, (g+1)*4^R/G), i.e. the finest Morton codes [g*4^L/G, (g+1)*4^L/G)
and a contiguous slice of every level n >= R; levels above R are replicated.
This module is the host-side statement of that plan (the kernels' owner_of()
in csrc/hwfv1_kernels.cuh is its device twin); the tests check it with a
world-size-2 gloo group.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Plan:
    L: int
    G: int

    @property
    def R(self) -> int:
        return self.L - min(self.L, 6)

    @property
    def tiles(self) -> int:
        return 1 << (2 * self.R)

    @property
    def tiles_per_part(self) -> int:
        return self.tiles // self.G

    def valid(self) -> bool:
        return 1 <= self.G <= 8 and self.tiles % self.G == 0

    def tile_range(self, g: int) -> tuple[int, int]:
        t = self.tiles_per_part
        return g * t, (g + 1) * t

    def finest_range(self, g: int) -> tuple[int, int]:
        """Contiguous finest Morton codes owned by partition g."""
        lo, hi = self.tile_range(g)
        s = 2 * (self.L - self.R)
        return lo << s, hi << s

    def owner(self, n: int, m: int) -> int:
        """Partition holding cell (n, m): its (first) level-R subtree's owner."""
        t = m >> (2 * (n - self.R)) if n >= self.R else m << (2 * (self.R - n))
        return t // self.tiles_per_part

    def level_slice(self, g: int, n: int) -> tuple[int, int]:
        """Morton codes of level n >= R owned by partition g (contiguous)."""
        assert n >= self.R
        lo, hi = self.tile_range(g)
        s = 2 * (n - self.R)
        return lo << s, hi << s
