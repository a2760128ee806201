"""The subtree partition over NCCL, one process per GPU (include/dh2.h dh2_dist with an
ncclUniqueId): the recompressed matrix must be bitwise the single-GPU one, on the full and on the
memory-lean plan.  Needs >= 2 visible GPUs (skipped otherwise: every GPU run of this build so far
had one GPU; the same partition runs on one GPU in the virtual mode, tests/test_gpu_shard.py and
tests/test_gpu_lean.py)."""
import os
import socket

import numpy as np
import pytest

from synth import get_config, mesh_for, seeded_vector

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _worker(rank, world, port, name, chunks, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1809_04384_b200 import DH2, nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], device=rank, world=world, rank=rank,
            nccl_uid=obj[0])
    h.recompress(cfg["eps"])
    y = h.matvec(seeded_vector(h.n, 1), 1)
    st = h.stats()
    if rank == 0:
        q.put((y, st["E_row"], st["far2"], st["transport"], h.storage(1)))
    h.close()
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpus() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("name", ["C1", "P2"])
def test_nccl_two_gpus_bitwise(name):
    import torch.multiprocessing as mp
    from paper_1809_04384_b200 import DH2
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], device=0)
    h.recompress(cfg["eps"])
    y1 = h.matvec(seeded_vector(h.n, 1), 1)
    s1 = h.stats()
    st1 = h.storage(1)
    h.close()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, 0, q)) for r in range(2)]
    for p in procs:
        p.start()
    y2, e_row, far2, transport, st2 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert transport == "nccl"
    assert np.array_equal(y1, y2)
    assert e_row == pytest.approx(s1["E_row"], rel=1e-14) and far2 == pytest.approx(s1["far2"], rel=1e-14)
    assert st1 == st2
