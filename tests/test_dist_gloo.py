"""CPU, world_size 2 over gloo: the multi-rank plumbing of paper_1105_2737_b200.dist.

* covariance estimator: ranks own contiguous chunk ranges, gather their
  partials, and merge in chunk order — bit-identical to the single-process
  estimate (the reference's worker-count invariance, test_stats.cpp:43-56).
  Partials are computed here from oracle-port fields (numpy), so the test
  exercises the partition, the collective and the ordered merge without a GPU.
* batch sharding: the field ranges of all ranks tile [0, world * per_rank).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

COUNTS, LENGTHS = (6, 4), (1.0, 2.0)
SAMPLES, REF = 2600, 7  # 3 chunks of 1024 (the last partial)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fields(samples=SAMPLES):
    from oracle import pyoracle as po

    port = po.Port()
    dens = po.density("matern", 2, nu=1.5, ell=0.3)
    n = port.count_draws(COUNTS, po.ONE_FFT_OVERWRITE)
    draws = np.random.default_rng(11).standard_normal((samples, n))
    return np.stack([port.synthesize(COUNTS, LENGTHS, dens, po.ONE_FFT_OVERWRITE, d)[0].ravel() for d in draws])


def _partials(fields, c0, n, chunk=1024):
    out = np.zeros((n, fields.shape[1]))
    for k in range(n):
        for j in range((c0 + k) * chunk, min((c0 + k + 1) * chunk, fields.shape[0])):
            out[k] = out[k] + fields[j, REF] * fields[j]
    return torch.from_numpy(out)


def _merge(parts, m):
    from paper_1105_2737_b200 import dist as gd

    return torch.from_numpy(gd.kahan_merge_numpy(parts.numpy(), m))


def _worker(rank, world, port, q, samples):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1105_2737_b200 import dist as gd

    fields = _fields(samples)
    est = gd.estimate_covariance_distributed(None, 0, samples, REF, partials_fn=lambda c0, n: _partials(fields, c0, n),
                                             merge_fn=_merge, points=fields.shape[1])
    q.put((rank, est.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("samples", [SAMPLES, 1000])
def test_covariance_partials_world2_bit_identical(samples):
    """2600 samples: 3 chunks over 2 ranks; 1000 samples: one chunk, so rank 1
    owns none and joins the all_gather with padding only."""
    from paper_1105_2737_b200 import dist as gd

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, samples)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    fields = _fields(samples)
    nch = (samples + 1023) // 1024
    single = gd.kahan_merge_numpy(_partials(fields, 0, nch).numpy(), samples)
    for r in range(world):
        assert np.array_equal(got[r], single)  # bitwise, on every rank
    # and the estimate is the plain covariance sum up to rounding
    direct = (fields[:, REF:REF + 1] * fields).sum(0) / samples
    assert np.abs(single - direct).max() < 1e-12 * np.abs(direct).max()


def test_partitions():
    from paper_1105_2737_b200 import dist as gd

    for samples in (1, 1024, 1025, 10_000, 123_457):
        total = (samples + 1023) // 1024
        for world in (1, 2, 3, 8):
            rs = [gd.chunk_range(r, world, samples) for r in range(world)]
            assert sum(n for _, n in rs) == total
            pos = 0
            for first, n in rs:
                assert first == pos
                pos += n
    assert [gd.field_range(r, 4, 32) for r in range(4)] == [(0, 32), (32, 32), (64, 32), (96, 32)]
