"""Config-size parity: the BASELINE workloads at the batch sizes the bench runs.

* c1 and c2 (fields 0 and 1023 of the full 1024-field batch, Algorithms 1 and 2)
  are compared directly with the reference's own ``grf::synthesize`` compiled
  unmodified in ``oracle/_ref`` (FixedStream fed the dumped device noise:
  synth.cpp:68-127, hermitian.cpp:178-202).
* c3 (64 fields of 4096^2) and c5 (512 steps of 1024^2) run at the bench's
  batch size: first and last field against the plain-C oracle, plus
  bit-identity with single-field launches (the persistent ring reuses slots
  many times over at these batch sizes).
* c4 at the full 512^3: four planes j0 of the device field against the
  oracle's spectrum (the reference's overwrite rule, pinned to oracle/_ref)
  summed along axis 0 and transformed by numpy (synth.cpp:118-126).

Tolerances: north_star's rel-L2 <= 1e-12 (fp64) and <= 1e-5 (fp32).
"""
import math
import os

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import pyoracle as po
from paper_1105_2737_b200 import grfc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def port():
    return po.Port()


@pytest.fixture(scope="module")
def ref():
    assert os.path.exists(po.REF_LIB), "oracle/_ref/libgrf_ref.so missing: run __graft_entry__.build()"
    return po.Reference()


def odens(name, d, **kw):
    return po.density(name, d, **kw)


def test_c1_against_reference_build(ref):
    counts, lengths = (512, 512), (1.0, 1.0)
    plan = grfc.Plan(counts, lengths, grfc.Density.gaussian_cov(2, 0.05), grfc.ONE_FFT_OVERWRITE, grfc.F64)
    got = plan.generate_tensor(0, 0, 1)[0].cpu().numpy()
    draws = plan.dump_noise(0, 0)
    want, residue, used = ref.synthesize(counts, lengths, odens("gauss", 2, ell=0.05), grfc.ONE_FFT_OVERWRITE, draws)
    assert used == len(draws) == 263164  # count_draws(512^2, overwrite) = 2|H| - 2^d
    assert rel_l2(got, want) <= 1e-12, rel_l2(got, want)


@pytest.mark.parametrize("alg", [grfc.ONE_FFT_OVERWRITE, grfc.TWO_FFT])
def test_c2_full_batch_first_and_last_against_reference_build(ref, alg):
    counts, lengths = (512, 512), (1.0, 1.0)
    plan = grfc.Plan(counts, lengths, grfc.Density.matern(2, 1.5, 0.1), alg, grfc.F32)
    batch = plan.generate_tensor(0, 0, 1024)
    torch.cuda.synchronize()
    for f in (0, 1023):
        want, _, _ = ref.synthesize(counts, lengths, odens("matern", 2, nu=1.5, ell=0.1), alg, plan.dump_noise(0, f))
        got = batch[f].double().cpu().numpy()
        assert rel_l2(got, want) <= 1e-5, (alg, f, rel_l2(got, want))
    assert torch.equal(batch[1023], plan.generate_tensor(0, 1023, 1)[0])
    assert torch.isfinite(batch).all()


def _batch_check(port, counts, dens_g, dens_o, n, first, singles):
    plan = grfc.Plan(counts, (1.0, 1.0), dens_g, grfc.ONE_FFT_OVERWRITE, grfc.F32)
    assert plan.path == "pow2-2d-f32", plan.path
    batch = plan.generate_tensor(0, first, n)
    torch.cuda.synchronize()
    for f in (0, n - 1):
        want, _ = port.synthesize(counts, (1.0, 1.0), dens_o, grfc.ONE_FFT_OVERWRITE, plan.dump_noise(0, first + f))
        got = batch[f].double().cpu().numpy()
        assert rel_l2(got, want) <= 1e-5, (counts, f, rel_l2(got, want))
    for f in singles:
        assert torch.equal(batch[f], plan.generate_tensor(0, first + f, 1)[0]), (counts, f)
    assert torch.isfinite(batch).all()


def test_c3_full_batch_64_fields(port):
    _batch_check(port, (4096, 4096), grfc.Density.matern(2, 0.5, 0.02), odens("matern", 2, nu=0.5, ell=0.02), 64, 0,
                 (0, 31, 63))


def test_c5_full_batch_512_steps(port):
    # the bench's per-GPU batch: steps [3584, 4096) (rank 7 of 8 in the 8-GPU split)
    _batch_check(port, (1024, 1024), grfc.Density.matern(2, 2.5, 0.05), odens("matern", 2, nu=2.5, ell=0.05), 512,
                 3584, (0, 1, 255, 510, 511))


def test_c4_512cubed_planes_against_oracle(port):
    counts, lengths = (512, 512, 512), (1.0, 1.0, 1.0)
    plan = grfc.Plan(counts, lengths, grfc.Density.gaussian_cov(3, 0.03), grfc.ONE_FFT_OVERWRITE, grfc.F32)
    assert plan.path == "pow2-3d-f32", plan.path
    field = plan.generate_tensor(0, 0, 1)[0]
    planes = (0, 1, 255, 511)
    got = field[list(planes)].double().cpu().numpy()
    del field
    draws = plan.dump_noise(0, 0)
    V = port.spectrum(counts, lengths, odens("gauss", 3, ell=0.03), 1, draws)  # overwrite rule, full lattice
    del draws
    # B(J) = sqrt((2 pi)^3/|A|) sum_K V(K) e^{-2 pi i K.J/N}: axis 0 by a phase matrix, axes 1-2 by fft2 (exp(-))
    k0 = np.arange(counts[0])
    ph = np.exp(-2j * np.pi * np.outer(planes, k0) / counts[0])
    S = (ph @ V.reshape(counts[0], -1)).reshape(len(planes), counts[1], counts[2])
    del V
    want = np.real(np.fft.fft2(S)) * math.sqrt((2 * math.pi) ** 3)
    for i, j0 in enumerate(planes):
        assert rel_l2(got[i], want[i]) <= 1e-5, (j0, rel_l2(got[i], want[i]))
