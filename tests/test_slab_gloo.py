"""CPU, world_size 2 over gloo: the slab decomposition of one 3D field
(include/grfc.h grfc_slab_*), restated in numpy on the oracle's spectrum and
run as two real processes with a point-to-point block exchange. Checks the
decomposition math and the contiguous-block all-to-all layout the device
path uses against the oracle's single-process field (rel-L2 <= 1e-12).

Pass A (rank r): Zh(k0,k1,k) = (X + conj X(-k0,-k1,M-k)) + i e^{2pi i k/N2}
(X - conj X(-k0,-k1,M-k)) for k1 in the rank's slab, exp(+) FFT along axis 0;
send block q = planes j0 in slab q. Pass B (rank q): axis-1 and axis-2 exp(+)
FFTs of its planes; z(j0,j1,m) = x(j0,j1,2m) + i x(j0,j1,2m+1).
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

COUNTS, LENGTHS = (8, 4, 6), (1.0, 2.0, 1.5)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spectrum_x(seed):
    from oracle import pyoracle as po

    port = po.Port()
    dens = po.density("matern", 3, nu=1.5, ell=0.3)
    draws = np.random.default_rng(seed).standard_normal(port.count_draws(COUNTS, po.ONE_FFT_OVERWRITE))
    V = port.spectrum(COUNTS, LENGTHS, dens, 1, draws)
    scale = math.sqrt((2 * math.pi) ** 3 / np.prod(LENGTHS))
    field, _ = port.synthesize(COUNTS, LENGTHS, dens, po.ONE_FFT_OVERWRITE, draws)
    return np.conj(V) * scale, field


def _pass_a(X, rank, world):
    n0, n1, n2 = X.shape
    m, n1p = n2 // 2, n1 // world
    k0 = np.arange(n0)[:, None, None]
    k1 = (rank * n1p + np.arange(n1p))[None, :, None]
    k = np.arange(m)[None, None, :]
    Xs = X[k0, k1, k]
    P = np.conj(X[(-k0) % n0, (-k1) % n1, (m - k) % n2])
    w = np.exp(2j * np.pi * k / n2)
    Zh = (Xs + P) + 1j * w * (Xs - P)
    return np.fft.ifft(Zh, axis=0) * n0  # exp(+), [j0][k1 local][k]


def _pass_b(recv, world, n0, n1, n2):
    m, n0p, n1p = n2 // 2, n0 // world, n1 // world
    planes = np.concatenate([recv[r] for r in range(world)], axis=1)  # [j0 local][k1][k]
    assert planes.shape == (n0p, n1, m)
    z = np.fft.ifft(np.fft.ifft(planes, axis=1) * n1, axis=2) * m
    out = np.empty((n0p, n1, n2))
    out[:, :, 0::2], out[:, :, 1::2] = z.real, z.imag
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    X, _ = _spectrum_x(123)
    n0, n1, n2 = X.shape
    W = _pass_a(X, rank, world)
    n0p = n0 // world
    send = [np.ascontiguousarray(W[r * n0p:(r + 1) * n0p]) for r in range(world)]  # block r
    recv = [None] * world
    recv[rank] = send[rank]
    reqs = []
    bufs = {}
    for peer in range(world):
        if peer == rank:
            continue
        t_out = torch.from_numpy(np.stack([send[peer].real, send[peer].imag]))
        t_in = torch.empty_like(t_out)
        bufs[peer] = t_in
        if rank < peer:
            dist.send(t_out, peer)
            dist.recv(t_in, peer)
        else:
            dist.recv(t_in, peer)
            dist.send(t_out, peer)
    for peer, t_in in bufs.items():
        a = t_in.numpy()
        recv[peer] = a[0] + 1j * a[1]
    slab = _pass_b(recv, world, n0, n1, n2)
    gathered = [torch.empty(slab.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(slab))
    if rank == 0:
        q.put(np.concatenate([g.numpy() for g in gathered], axis=0))
    dist.destroy_process_group()


def test_slab_decomposition_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, want = _spectrum_x(123)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel < 1e-12, rel


@pytest.mark.parametrize("world", [1, 2])
def test_slab_math_single_process(world):
    """The same decomposition without processes, every world size dividing N0, N1."""
    X, want = _spectrum_x(7)
    n0, n1, n2 = X.shape
    W = [_pass_a(X, r, world) for r in range(world)]
    n0p = n0 // world
    slabs = [_pass_b([W[r][q * n0p:(q + 1) * n0p] for r in range(world)], world, n0, n1, n2) for q in range(world)]
    got = np.concatenate(slabs, axis=0)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
