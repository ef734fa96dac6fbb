"""Host-side sharding of a midpoint line across ranks (BASELINE multi-GPU).

CMP gathers are independent: rank r scans a contiguous block.  CRS midpoints
need their +-aperture neighbours: rank r receives its block plus a replicated
halo on each side and restricts its outputs to the block (the 1-D case of the
reference's partition + strip_of, crs_pipeline.hpp:92-158,341-347, with the
halo replicated up front instead of exchanged).  There is no collective on
the data path; results are gathered to rank 0 at the end.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def block_range(n: int, world: int, rank: int) -> tuple:
    """Contiguous block [b, e) of n rows for rank (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    q, r = divmod(n, world)
    b = rank * q + min(rank, r)
    return b, b + q + (1 if rank < r else 0)


@dataclass
class Shard:
    rank: int
    block: tuple   # own output rows [b, e) in line order
    gathers: tuple  # gathers [lo, hi) this rank holds (block + halo)

    @property
    def row_first(self) -> int:
        return self.block[0] - self.gathers[0]

    @property
    def row_count(self) -> int:
        return self.block[1] - self.block[0]


def line_shards(mx: np.ndarray, world: int, apm: float = 0.0) -> list:
    """Shards of a line whose midpoint x coordinates ``mx`` are sorted
    ascending.  The halo holds every gather within apm (plus a float margin;
    the exact closed-ball test runs in the library) of the block's ends."""
    mx = np.asarray(mx, np.float64)
    n = len(mx)
    if n and np.any(np.diff(mx) < 0):
        raise ValueError("line_shards: midpoints must be sorted by x")
    out = []
    margin = apm * 1e-5 + 1e-3 if apm > 0 else 0.0
    for r in range(world):
        b, e = block_range(n, world, r)
        if apm > 0 and e > b:
            lo = int(np.searchsorted(mx, mx[b] - apm - margin, "left"))
            hi = int(np.searchsorted(mx, mx[e - 1] + apm + margin, "right"))
        else:
            lo, hi = b, e
        out.append(Shard(r, (b, e), (lo, hi)))
    return out


def weak_shard(n_per_rank: int, rank: int, halo: int = 0, world: int = 1) -> Shard:
    """Weak scaling: rank r owns gathers [r n, (r+1) n) of a world*n line and
    holds `halo` extra gathers on each side (clipped to the line)."""
    b, e = rank * n_per_rank, (rank + 1) * n_per_rank
    lo, hi = max(0, b - halo), min(world * n_per_rank, e + halo)
    return Shard(rank, (b, e), (lo, hi))
