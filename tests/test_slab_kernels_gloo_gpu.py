"""Two processes (gloo, world size 2) run the REAL slab kernels on the one GPU:
each rank's grfc_slab_pass_a, the block exchange staged through host memory
with dist.all_to_all_single (gloo), and grfc_slab_pass_b. The assembled field
must be bit-identical to the single-GPU grfc_generate field. No kernel of one
rank waits on the other's (the exchange is host-side between the passes), so
sharing the GPU changes timing only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

COUNTS = (256, 128, 256)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1105_2737_b200 import grfc

    plan = grfc.Plan(COUNTS, (1.0, 1.0, 1.0), grfc.Density.gaussian_cov(3, 0.03), grfc.ONE_FFT_OVERWRITE, grfc.F32)
    buf, block, pts = plan.slab_sizes(world)
    send = torch.empty(buf, dtype=torch.complex64, device="cuda")
    plan.slab_pass_a(world, rank, 9, 2, send.data_ptr())
    torch.cuda.synchronize()
    recv_h = torch.empty(buf, dtype=torch.complex64)
    dist.all_to_all_single(torch.view_as_real(recv_h), torch.view_as_real(send.cpu()))
    recv = recv_h.cuda()
    out = torch.empty(pts, dtype=torch.float32, device="cuda")
    plan.slab_pass_b(world, recv.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    q.put((rank, out.cpu().numpy()))  # by value: a shared-memory tensor would die with this process
    dist.barrier()
    dist.destroy_process_group()


def test_slab_kernels_world2_gloo_bit_identical():
    from paper_1105_2737_b200 import grfc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    field = torch.from_numpy(np.concatenate([got[r] for r in range(world)])).reshape(COUNTS)
    plan = grfc.Plan(COUNTS, (1.0, 1.0, 1.0), grfc.Density.gaussian_cov(3, 0.03), grfc.ONE_FFT_OVERWRITE, grfc.F32)
    want = plan.generate_tensor(9, 2, 1)[0].cpu()
    assert torch.equal(field, want)
