"""GPU: the device covariance estimator (grfc_estimate_covariance & co.) vs the
reference's own grf::estimate_covariance (oracle/_ref, src/stats.cpp:39-97)
fed the same per-sample noise through its StreamFactory overload, plus the
determinism contract (chunking, batch size and device count never change a
bit) and the statistical gate of SURVEY.md §8d run through the estimator.
"""
import math

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_1105_2737_b200 import grfc

pytestmark = pytest.mark.gpu


def odens(g: grfc.Density):
    d = po.Density()
    d.family, d.dim = g.family, g.dim
    for k in range(8):
        d.r[k], d.i[k] = g.r[k], g.i[k]
    return d


def kahan_merge(partials, samples):
    """numpy restatement of the chunk-ordered Kahan merge (stats.cpp:84-93)."""
    est = np.zeros_like(partials[0])
    comp = np.zeros_like(partials[0])
    for acc in partials:
        y = acc - comp
        t = est + y
        comp = (t - est) - y
        est = t
    return est * (1.0 / samples)


@pytest.fixture(scope="module")
def ref():
    if not po.reference_available():
        pytest.skip("oracle/_ref not built")
    return po.Reference()


@pytest.mark.parametrize("alg", [grfc.ONE_FFT_OVERWRITE, grfc.TWO_FFT, grfc.ONE_FFT_RECURSIVE])
def test_estimate_matches_reference_estimator(ref, alg):
    counts, lengths = (16, 8), (1.0, 2.0)
    dens = grfc.Density.matern(2, 1.5, 0.2)
    plan = grfc.Plan(counts, lengths, dens, alg, grfc.F64)
    M, seed, refpt = 2500, 7, (3, 5)  # 3 chunks, the last one partial
    got = plan.estimate_covariance_host(seed, M, refpt)
    draws = np.stack([plan.dump_noise(seed, j) for j in range(M)])
    want = ref.estimate_covariance_fixed(counts, lengths, odens(dens), alg, refpt, draws, threads=4)
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err < 1e-12, err


def test_estimate_fp32_matches_reference_estimator(ref):
    counts, lengths = (512, 256), (1.0, 1.0)
    dens = grfc.Density.gaussian_cov(2, 0.05)
    plan = grfc.Plan(counts, lengths, dens, grfc.ONE_FFT_OVERWRITE, grfc.F32)
    assert plan.path.startswith("pow2-2d")
    M, seed, refpt = 40, 3, (100, 7)
    got = plan.estimate_covariance_host(seed, M, refpt)
    draws = np.stack([plan.dump_noise(seed, j) for j in range(M)])
    want = ref.estimate_covariance_fixed(counts, lengths, odens(dens), grfc.ONE_FFT_OVERWRITE, refpt, draws)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 1e-5, err


def test_determinism_batch_chunks_and_devices(monkeypatch):
    """Bit-identical for any generation batch size, and partials split over
    'devices' (chunk ranges) + the ordered merge == the single-device estimate."""
    counts = (64, 32)
    plan = grfc.Plan(counts, (1.0, 1.0), grfc.Density.matern(2, 0.5, 0.1), grfc.ONE_FFT_OVERWRITE, grfc.F32)
    M, seed, refpt = 3000, 11, (10, 20)
    base = plan.estimate_covariance_tensor(seed, M, refpt)
    monkeypatch.setenv("GRFC_COV_BATCH", "37")
    assert torch.equal(plan.estimate_covariance_tensor(seed, M, refpt), base)
    monkeypatch.delenv("GRFC_COV_BATCH")
    nch = (M + grfc.COV_CHUNK - 1) // grfc.COV_CHUNK
    parts = torch.cat([plan.covariance_partials_tensor(seed, M, 0, 1, refpt),
                       plan.covariance_partials_tensor(seed, M, 1, nch - 1, refpt)])
    assert torch.equal(plan.covariance_merge_tensor(parts, M), base)
    # the device merge is the numpy restatement bit for bit
    host = kahan_merge([p.cpu().numpy() for p in parts], M)
    assert np.array_equal(host, base.cpu().numpy())
    # and the chunk partials are the plain ordered sums of the fields' products
    f = plan.generate_tensor(seed, 0, grfc.COV_CHUNK).reshape(grfc.COV_CHUNK, -1).double()
    lin = plan.linear_index(refpt)
    direct = (f[:, lin:lin + 1] * f).sum(0)
    assert torch.allclose(direct, parts[0].reshape(-1), rtol=1e-12, atol=1e-12)


def test_injected_chunk_matches_seeded_partial(ref):
    counts = (32, 16)
    plan = grfc.Plan(counts, (1.0, 1.0), grfc.Density.gaussian_cov(2, 0.1), grfc.ONE_FFT_RECURSIVE, grfc.F64)
    M, seed, refpt = 300, 5, (0, 0)
    draws = np.stack([plan.dump_noise(seed, j) for j in range(M)])
    inj = plan.covariance_chunk_injected_host(draws, refpt)
    seeded = plan.covariance_partials_tensor(seed, M, 0, 1, refpt)[0].cpu().numpy().ravel()
    assert np.abs(inj - seeded).max() < 1e-12 * np.abs(seeded).max()


def test_errors():
    plan = grfc.Plan((8, 8), (1.0, 1.0), grfc.Density.gaussian_cov(2, 0.1), grfc.ONE_FFT_OVERWRITE, grfc.F64)
    with pytest.raises(ValueError, match="at least one sample"):
        plan.estimate_covariance_host(0, 0, (0, 0))
    with pytest.raises(ValueError, match="out of range"):
        plan.estimate_covariance_host(0, 10, 64)
    with pytest.raises(ValueError, match="chunk range"):
        plan.covariance_partials(0, 1000, 1, 1, 0, 0)


def test_statistical_gate_through_estimator(ref):
    """10^4 fields at 64^2: the device estimator vs exact_discrete_covariance_all
    within 5 (2/sqrt(M)) C(0) (acceptance.cpp:98 form), every algorithm."""
    counts, lengths = (64, 64), (1.0, 1.0)
    dens = grfc.Density.gaussian_cov(2, 0.05)
    exact = ref.exact_cov_all(counts, lengths, odens(dens))
    M = 10000
    for alg in (grfc.TWO_FFT, grfc.ONE_FFT_OVERWRITE, grfc.ONE_FFT_RECURSIVE):
        plan = grfc.Plan(counts, lengths, dens, alg, grfc.F32)
        est = plan.estimate_covariance_host(123, M, (0, 0))
        tol = 5 * 2 / math.sqrt(M) * exact.flat[0]
        assert np.abs(est - exact).max() < tol, (alg, np.abs(est - exact).max(), tol)


def test_distributed_helper_single_rank_matches_estimate():
    """paper_1105_2737_b200.dist on one rank (no process group): device partials +
    device merge == grfc_estimate_covariance, bit for bit."""
    from paper_1105_2737_b200 import dist as gd

    plan = grfc.Plan((128, 64), (1.0, 1.0), grfc.Density.matern(2, 1.5, 0.1), grfc.ONE_FFT_OVERWRITE, grfc.F64)
    est = gd.estimate_covariance_distributed(plan, 3, 2500, (5, 9))
    assert torch.equal(est.reshape(plan.counts), plan.estimate_covariance_tensor(3, 2500, (5, 9)))
