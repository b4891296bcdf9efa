"""The NCCL data plane across two GPUs: two processes, one per GPU, each owning a
z-slab of the mesh, with the library's own NCCL communicator (unique id broadcast over
torch.distributed).  The gathered viscous apply must equal the CPU oracle within 1e-12 and the
one-GPU apply bitwise; a V-cycle-preconditioned CG must converge with allreduced dots.  Needs two
GPUs: skipped (with the reason) on a one-GPU box, where test_gpu_threads_comm.py runs the same
multi-rank library path through the in-process communicator instead."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from inputs import cube, uniform
    from oracle import laws
    from paper_2506_14424_b200 import _abi
    from paper_2506_14424_b200.dgvv import Context, nccl_comm_init, nccl_unique_id
    from paper_2506_14424_b200.partition import slab_partition
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = nccl_comm_init(bytes(uid.cpu().numpy().tobytes()), world, rank)
        m = cube(6)
        k = 3
        per = 3 * (k + 1) ** 3
        p = slab_partition(m, world, rank)
        ctx = Context(p, k, visc_law=laws.C2_LAW, degrees=[3, 2, 1], n_owned=p.n_owned, n_ghost=p.n_ghost,
                      ghost_global_id=p.ghost_global_id, ghost_owner=p.ghost_owner, first_global_cell=p.first,
                      nccl_comm=comm)
        u = uniform(0, m.n_cells * per)
        x = torch.from_numpy(u[p.first * per:(p.first + p.n_owned) * per].copy()).cuda()
        y = torch.empty_like(x)
        ctx.apply_viscous(x, y)
        ctx.set_mass(0, 10.0)
        lams = [1.2 * ctx.estimate_lambda_max(0, torch.ones(3 * p.n_owned * (kk + 1) ** 3, dtype=torch.float64, device="cuda"),
                                              level=l, steps=15) for l, kk in enumerate([3, 2, 1])]
        z = torch.zeros_like(x)
        it, rr = ctx.cg_solve(0, x, z, rtol=1e-9, maxit=500, precond="vcycle", lam_hi_per_level=lams)
        torch.cuda.synchronize()
        q.put((rank, p.first, y.cpu().numpy(), it, rr))
        ctx.close()
        _abi.lib().dgvv_nccl_comm_destroy(comm)
        dist.destroy_process_group()
    except BaseException as e:              # noqa: BLE001 - reported to the parent
        q.put((rank, "error", repr(e), 0, 0))


def test_nccl_two_gpus_apply_and_cg():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun and the round-end tests have one; the in-process "
                    "communicator test covers the multi-rank path on one GPU)")
    import torch.multiprocessing as mp

    from inputs import cube, uniform
    from oracle import dg, laws
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx_mp.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
    for r in res:
        assert r[1] != "error", r[2]
    m = cube(6)
    d = dg.Disc(m, 3)
    u = uniform(0, m.n_cells * 3 * d.N)
    y = np.concatenate([r[2] for r in sorted(res, key=lambda t: t[1])])
    ref = dg.viscous_apply(d, u, dg.AnalyticNu(d, laws.C2_LAW))
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) < 1e-12
    assert res[0][3] == res[1][3] and max(r[4] for r in res) <= 1e-9
