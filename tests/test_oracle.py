"""CPU: pins the plain-C oracle (oracle/grf_oracle.c) to the reference.

* against the committed golden fixtures, generated from the reference's own
  proj/core compiled unmodified (tests/golden/make_golden.py);
* against the reference build itself when oracle/_ref is present;
* against the known-answer tests of the reference's own suite
  (/root/reference/proj/tests/*.cpp, lines cited per test).
"""
import math

import numpy as np
import pytest

from conftest import golden_cases, rel_l2
from oracle import pyoracle as po


@pytest.fixture(scope="module")
def port():
    return po.Port()


def _dens(family, r, i, dim):
    d = po.Density()
    d.family, d.dim = family, dim
    for k in range(8):
        d.r[k], d.i[k] = float(r[k]), int(i[k])
    return d


def test_port_matches_golden_fields(port, golden):
    n = 0
    for key, counts, lengths, fam, r, i, alg, draws, field in golden_cases(golden):
        got, residue = port.synthesize(counts, lengths, _dens(fam, r, i, len(counts)), alg, draws)
        assert rel_l2(got, field) < 1e-13, key
        assert residue < 1e-10
        n += 1
    assert n >= 30


def test_port_matches_golden_reps_and_covariance(port, golden):
    for c in range(11):
        counts = tuple(golden[f"c{c}_a0_counts"])
        lin, self_ = port.conjugate_reps(counts)
        assert np.array_equal(lin, golden[f"c{c}_reps"])
        assert np.array_equal(self_, golden[f"c{c}_reps_self"])
        fam, r, i = int(golden[f"c{c}_a0_family"]), golden[f"c{c}_a0_r"], golden[f"c{c}_a0_i"]
        cov = port.exact_cov_all(counts, tuple(golden[f"c{c}_a0_lengths"]), _dens(fam, r, i, len(counts)))
        assert rel_l2(cov, golden[f"c{c}_cov"]) < 1e-12


@pytest.mark.skipif(not po.reference_available(), reason="oracle/_ref not built")
def test_port_matches_live_reference_random_grids(port):
    ref = po.Reference()
    rng = np.random.default_rng(5)
    for t in range(25):
        d = int(rng.integers(1, 5))
        counts = tuple(int(2 * rng.integers(1, 6)) for _ in range(d))
        lengths = tuple(float(x) for x in rng.uniform(0.5, 3.0, d))
        dens = po.density("matern", d, nu=float(rng.uniform(0.3, 3)), ell=float(rng.uniform(0.05, 0.5)))
        for alg in po.ALGORITHMS:
            nd = ref.count_draws(counts, alg)
            assert nd == port.count_draws(counts, alg)
            draws = rng.standard_normal(nd)
            a, _, used = ref.synthesize(counts, lengths, dens, alg, draws)
            b, _ = port.synthesize(counts, lengths, dens, alg, draws)
            assert used == nd
            assert rel_l2(b, a) < 1e-13
            # the reference's own naive DFT backend agrees (test_synth.cpp:159-174)
            c, _, _ = ref.synthesize(counts, lengths, dens, alg, draws, backend=1)
            assert np.abs(a - c).max() <= 1e-9 * np.abs(c).max()
        for alg in (po.ONE_FFT_OVERWRITE, po.ONE_FFT_RECURSIVE):
            mode = 1 if alg == po.ONE_FFT_OVERWRITE else 0
            draws = rng.standard_normal(ref.count_draws(counts, alg))
            assert np.array_equal(ref.spectrum(counts, lengths, dens, mode, draws),
                                  port.spectrum(counts, lengths, dens, mode, draws))


def test_draw_counts_known_answers(port):
    # test_synth.cpp:150-156, test_hermitian.cpp:106-119
    assert port.count_draws((4, 4), po.TWO_FFT) == 16
    assert port.count_draws((4, 4), po.ONE_FFT_RECURSIVE) == 16
    assert port.count_draws((4, 4), po.ONE_FFT_OVERWRITE) == 20
    assert port.count_draws((6, 2), po.ONE_FFT_OVERWRITE) == 6 * 2 + 2 * 6 - 4
    # BASELINE configs
    assert port.count_draws((512, 512), po.ONE_FFT_OVERWRITE) == 263164
    assert port.count_draws((1024, 1024), po.ONE_FFT_OVERWRITE) == 1050620
    assert port.count_draws((4096, 4096), po.ONE_FFT_OVERWRITE) == 16785404
    assert port.count_draws((512, 512, 512), po.ONE_FFT_OVERWRITE) == 134742008


def test_representative_set_known_answers(port):
    lin, self_ = port.conjugate_reps((4,))  # test_hermitian.cpp:44-53
    assert list(lin) == [0, 2, 1] and list(self_) == [True, True, False]
    assert len(port.conjugate_reps((4, 4))[0]) == 10  # :55-58
    lin, _ = port.conjugate_reps((8, 8))
    assert len(lin) == 34
    blocks = {(a, b) for a in range(5) for b in range(5)} | {(a, b) for a in range(1, 4) for b in range(5, 8)}
    assert {(int(x) // 8, int(x) % 8) for x in lin} == blocks  # :60-71


@pytest.mark.parametrize("counts", [(2,), (12,), (4, 4), (2, 10), (4, 2, 6), (2, 4, 2, 6)])
def test_partition_property(port, counts):
    # test_hermitian.cpp:17-41,73-80: reps and the negations of paired reps tile the lattice
    lin, self_ = port.conjugate_reps(counts)
    P = int(np.prod(counts))
    assert self_.sum() == 2 ** len(counts)
    assert len(lin) == 2 ** len(counts) + (P - 2 ** len(counts)) // 2
    seen = np.zeros(P, bool)
    for l, s in zip(lin, self_):
        k = np.unravel_index(int(l), counts)
        neg = np.ravel_multi_index(tuple((-np.array(k)) % np.array(counts)), counts)
        assert not seen[l]
        seen[l] = True
        if not s:
            assert not seen[neg]
            seen[neg] = True
    assert seen.all()


def test_density_goldens(port):
    # test_spectral.cpp:14-41
    assert port.density_eval(po.density("poly", 2, m=1.0, k=1, l=1, n=1), [0.0, 0.0]) == pytest.approx(1.0)
    assert port.density_eval(po.density("poly", 2, m=1.0, k=1, l=1, n=1), [1.0, 0.0]) == pytest.approx(0.5)
    assert port.density_eval(po.density("poly", 1, m=2.0, k=2, l=3, n=1), [0.0]) == pytest.approx(1 / 64)
    t = po.density("test1d", 1)
    assert port.density_eval(t, [0.0]) == pytest.approx(0.10185916357881303, rel=1e-14)
    assert port.density_eval(t, [10.0]) == pytest.approx((32e6 / math.pi) / 200.0 ** 4, rel=1e-14)
    # Matern / Gaussian normalisation: C(0) = integral of g = 1 (1D quadrature)
    w = np.linspace(-4000, 4000, 800001)
    for dens in (po.density("matern", 1, nu=1.5, ell=0.1), po.density("gauss", 1, ell=0.05)):
        g = np.array([port.density_eval(dens, [x]) for x in w[::100]])
        assert np.trapezoid(g, w[::100]) == pytest.approx(1.0, rel=2e-3)


def test_zero_stream_and_impulse(port):
    # test_synth.cpp:50-73
    dens = po.density("constant", 2, c=2.0)
    for alg in po.ALGORITHMS:
        f, res = port.synthesize((4, 6), (1.0, 1.0), dens, alg, np.zeros(port.count_draws((4, 6), alg)))
        assert (f == 0).all() and res == 0.0
    c = 2.25
    draws = np.zeros(port.count_draws((4, 4), po.ONE_FFT_RECURSIVE))
    draws[0] = 1.0
    f, _ = port.synthesize((4, 4), (1.0, 1.0), po.density("constant", 2, c=c), po.ONE_FFT_RECURSIVE, draws)
    np.testing.assert_allclose(f, math.sqrt((2 * math.pi) ** 2 * c), rtol=1e-12)


def test_flat_density_covariance(port):
    # test_synth.cpp:75-87 (via the transform-at-once form, synth.cpp:188-209)
    counts, lengths, c = (4, 6), (1.0, 2.0), 0.7
    cov = port.exact_cov_all(counts, lengths, po.density("constant", 2, c=c)).ravel()
    at0 = c * (2 * math.pi) ** 2 * 24 / 2.0
    assert cov[0] == pytest.approx(at0, rel=1e-12)
    assert np.abs(cov[1:]).max() < 1e-12 * at0


def test_errors(port):
    with pytest.raises(po.OracleError) as e:
        port.synthesize((3, 4), (1.0, 1.0), po.density("constant", 2, c=1.0), 0, np.zeros(12))
    assert e.value.code == 1
    with pytest.raises(po.OracleError) as e:
        port.synthesize((8,), (1.0,), po.density("constant", 2, c=1.0), 0, np.zeros(8))
    assert e.value.code == 1  # density dimension mismatch, synth.cpp:70-71
    with pytest.raises(po.OracleError) as e:
        port.synthesize((8,), (1.0,), po.density("constant", 1, c=1.0), 2, np.zeros(3))
    assert e.value.code == 2  # FixedStream exhaustion, random.hpp:56
    with pytest.raises(po.OracleError) as e:
        port.synthesize((8,), (1.0,), po.density("constant", 1, c=float("nan")), 0, np.zeros(8))
    assert e.value.code == 2  # NaN density, synth.cpp:105-106


def test_dft_round_trip_and_naive(port):
    # test_synth.cpp:21-48 on the oracle FFT
    rng = np.random.default_rng(7)
    for counts in [(8,), (4, 6), (2, 4, 6), (10, 12)]:
        x = rng.standard_normal(counts) + 1j * rng.standard_normal(counts)
        fwd = port.dft(counts, x, +1)
        back = port.dft(counts, fwd, -1)
        assert np.abs(back - x).max() <= 1e-12 * np.abs(x).max()
        # numpy's ifftn * P is the exp(+) unnormalised sum
        np.testing.assert_allclose(fwd, np.fft.ifftn(x) * x.size, rtol=0, atol=1e-11 * np.abs(fwd).max())


def estimate_covariance_restated(fields, ref_lin, samples, chunk=1024):
    """numpy restatement of grf::estimate_covariance's arithmetic
    (src/stats.cpp:60-96): per chunk, acc += f[ref] * f in sample order; chunk
    partials merged in order with Kahan compensation; times 1/M."""
    est = np.zeros(fields.shape[1])
    comp = np.zeros_like(est)
    for c0 in range(0, samples, chunk):
        acc = np.zeros_like(est)
        for j in range(c0, min(c0 + chunk, samples)):
            acc = acc + fields[j, ref_lin] * fields[j]
        y = acc - comp
        t = est + y
        comp = (t - est) - y
        est = t
    return est * (1.0 / samples)


@pytest.mark.skipif(not po.reference_available(), reason="oracle/_ref not built")
def test_covariance_estimator_restatement_matches_reference(port):
    """The reference estimator (StreamFactory overload, FixedStream per sample)
    equals the restated chunk/Kahan arithmetic on the port's fields; worker
    count never changes a bit (test_stats.cpp:43-56)."""
    ref = po.Reference()
    counts, lengths = (6, 4), (1.0, 2.0)
    dens = po.density("matern", 2, nu=1.5, ell=0.3)
    M, refpt = 2100, (2, 1)
    n = port.count_draws(counts, po.ONE_FFT_OVERWRITE)
    draws = np.random.default_rng(3).standard_normal((M, n))
    fields = np.stack([port.synthesize(counts, lengths, dens, po.ONE_FFT_OVERWRITE, d)[0].ravel() for d in draws])
    want = estimate_covariance_restated(fields, refpt[0] * counts[1] + refpt[1], M)
    a = ref.estimate_covariance_fixed(counts, lengths, dens, po.ONE_FFT_OVERWRITE, refpt, draws, threads=1).ravel()
    b = ref.estimate_covariance_fixed(counts, lengths, dens, po.ONE_FFT_OVERWRITE, refpt, draws, threads=3).ravel()
    assert np.array_equal(a, b)
    assert np.abs(a - want).max() < 1e-13 * np.abs(want).max()
