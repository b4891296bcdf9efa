"""Slab domain decomposition for the multi-GPU path — host logic only.

Each rank owns a contiguous range of global cell ids (z-slabs of the cubes, x-slabs of the
BFS: the meshes are ordered so that these are contiguous; C5 at 8 ranks is exactly the
survey's 124,928 cells per rank).  The cells across partition faces are the rank's ghosts.
Exchange protocol (implemented by libdgvv.so, mirrored here for the CPU tests):
  * ghosts are stored in (owner rank, global id) order; the block of ghosts owned by peer r
    is received from r in that order;
  * rank r sends to peer q its owned cells that have a face neighbour owned by q, in
    ascending global id — the same set and order q expects.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class LocalMesh:
    n_cells: int                # rows = owned + ghosts (binding convention: mesh.n_cells rows)
    n_owned: int
    first: int
    neighbor: np.ndarray        # int64 [n_owned + n_ghost, 6] global ids / -1-bc
    nodes: np.ndarray           # [n_owned + n_ghost, (m+1)^3, 3]
    map_degree: int
    ghost_global_id: np.ndarray  # int64 [n_ghost], sorted by (owner, gid)
    ghost_owner: np.ndarray      # int32 [n_ghost]
    periods: tuple = (0.0, 0.0, 0.0)

    @property
    def n_ghost(self):
        return len(self.ghost_global_id)


def bounds(n_cells: int, nranks: int) -> np.ndarray:
    return np.array([(n_cells * r) // nranks for r in range(nranks + 1)], dtype=np.int64)


def owner_of(gids, b):
    return (np.searchsorted(b, gids, side="right") - 1).astype(np.int32)


def slab_partition(mesh, nranks: int, rank: int) -> LocalMesh:
    b = bounds(mesh.n_cells, nranks)
    first, last = int(b[rank]), int(b[rank + 1])
    owned = np.arange(first, last)
    nb = mesh.neighbor[owned]
    cand = nb[nb >= 0]
    ghosts = np.unique(cand[(cand < first) | (cand >= last)])
    own = owner_of(ghosts, b)
    order = np.lexsort((ghosts, own))
    ghosts, own = ghosts[order], own[order]
    rows = np.concatenate([owned, ghosts])
    return LocalMesh(len(rows), len(owned), first, mesh.neighbor[rows], mesh.nodes[rows], mesh.map_degree,
                     ghosts.astype(np.int64), own.astype(np.int32), mesh.periods)


def send_lists(local: LocalMesh):
    """{peer: owned global ids to send}, ascending (the library's rule)."""
    out = {}
    first = local.first
    nb = local.neighbor[:local.n_owned]
    gset = {int(g): int(o) for g, o in zip(local.ghost_global_id, local.ghost_owner)}
    for c in range(local.n_owned):
        peers = {gset[int(g)] for g in nb[c] if int(g) in gset}
        for q in peers:
            out.setdefault(q, []).append(first + c)
    return {q: np.array(v, dtype=np.int64) for q, v in out.items()}


def recv_blocks(local: LocalMesh):
    """{peer: (offset, count)} of the ghost rows received from each peer."""
    out = {}
    for q in np.unique(local.ghost_owner):
        idx = np.nonzero(local.ghost_owner == q)[0]
        out[int(q)] = (int(idx[0]), len(idx))
    return out
