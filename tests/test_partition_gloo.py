"""CPU (gloo, world_size 2) tests of the multi-GPU host logic: slab partition, ghost lists
and the exchange protocol (ordering by (owner, global id) / ascending send lists) — the
same rule libdgvv.so implements.  After the exchange every rank holds exactly the global
vector's entries at its ghost ids."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from inputs import bfs, cube, deformed_cube, uniform
from paper_2506_14424_b200.partition import recv_blocks, send_lists, slab_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


MESHES = {"cube5": lambda: cube(5), "deformed4": lambda: deformed_cube(4, 2),
          "bfs": lambda: bfs(nx_in=4, ny_in=2, nx_out=8, nz=3)}


def _worker(rank, world, port, mesh_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = MESHES[mesh_name]()
        loc = slab_partition(m, world, rank)
        per = 8
        glob = uniform(0, m.n_cells * per).reshape(m.n_cells, per)
        mine = torch.from_numpy(glob[loc.first:loc.first + loc.n_owned].copy())
        sends = send_lists(loc)
        recvs = recv_blocks(loc)
        ghost = torch.zeros(loc.n_ghost, per, dtype=torch.float64)
        reqs = []
        for peer in sorted(set(sends) | set(recvs)):
            if peer in sends:
                idx = torch.from_numpy(sends[peer] - loc.first)
                reqs.append(dist.isend(mine[idx].contiguous(), peer))
            if peer in recvs:
                o, cnt = recvs[peer]
                buf = torch.empty(cnt, per, dtype=torch.float64)
                reqs.append((dist.irecv(buf, peer), o, buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                ghost[r[1]:r[1] + len(r[2])] = r[2]
            else:
                r.wait()
        ok = np.array_equal(ghost.numpy(), glob[loc.ghost_global_id])
        # every face neighbour of an owned cell is owned or a ghost
        nb = loc.neighbor[:loc.n_owned]
        known = set(range(loc.first, loc.first + loc.n_owned)) | set(loc.ghost_global_id.tolist())
        cover = all(int(g) in known for g in nb[nb >= 0])
        q.put((rank, ok, cover, loc.n_owned, loc.n_ghost))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mesh_name", list(MESHES))
def test_ghost_exchange_world2(mesh_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mesh_name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, cover, no, ng in res:
        assert ok and cover and no > 0 and ng > 0, (rank, ok, cover)


def test_c5_partition_matches_survey():
    """C5 at 8 ranks: 124,928 cells each, rank 0 = inlet block + 21 outlet layers; every cut
    is a 64 x 32 = 2048-face outlet cross-section."""
    m = bfs()
    for r in (0, 3, 7):
        loc = slab_partition(m, 8, r)
        assert loc.n_owned == 124928
        assert loc.n_ghost == (2048 if r in (0, 7) else 4096)
