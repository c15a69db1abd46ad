"""TEST / BASELINE INFRASTRUCTURE — NOT PRODUCT CODE.

CPU FFT-library check for the bench's cpu_baseline (SURVEY.md §8d asks for an
"FFTW-class" line): the inverse real 2D FFT of Algorithm 2 (half-spectrum ->
field) through a production multithreaded CPU FFT library (scipy.fft /
pocketfft, all host threads), timed alone. The reference's own path is timed
through oracle/_ref on the FFTW API stand-in (FFTW is absent from the image);
this line shows how a library transform compares with that stand-in. On the
B200 box's host (round-1 bench, 16 threads) the FFT alone ran at 0.72 Gpts/s
against 0.33 Gpts/s for the reference's whole path: the transform is not the
reference's bottleneck (its per-cell spectrum walk, ziggurat draws and virtual
density calls are), so the reported baseline is the reference path, and this
line only bounds what a production CPU FFT would add.
"""
import math
import time

import numpy as np
import scipy.fft


def _sqrt_density(counts, lengths, density):
    n1, n2 = counts
    k1 = np.fft.fftfreq(n1, d=1.0 / n1)  # wrapped integer frequencies
    k2 = np.arange(n2 // 2 + 1, dtype=np.float64)
    w1 = 2 * math.pi * k1 / lengths[0]
    w2 = 2 * math.pi * k2 / lengths[1]
    r2 = w1[:, None] ** 2 + w2[None, :] ** 2
    if density[0] == "gauss":
        ell = density[1]
        g = (ell / math.sqrt(2 * math.pi)) ** 2 * np.exp(-0.5 * ell * ell * r2)
    else:
        nu, ell = density[1], density[2]
        c = ell ** 2 * math.gamma(nu + 1) / (math.pi * math.gamma(nu))
        g = c * (1 + ell * ell * r2) ** (-(nu + 1))
    return np.sqrt(g) * math.sqrt((2 * math.pi) ** 2 / (lengths[0] * lengths[1]))


def rate(counts, lengths, density, nfields, workers):
    """Gpts/s of the FFT-only stage of nfields syntheses: the Hermitian
    half-spectra (noise x sqrt(g), built once) go through
    scipy.fft.irfft2 (pocketfft) with `workers` threads, 16 fields per call.
    Noise generation and the density are excluded."""
    sg = _sqrt_density(counts, lengths, density)
    rng = np.random.default_rng(0)
    batch = 16
    z = rng.standard_normal((batch,) + sg.shape) + 1j * rng.standard_normal((batch,) + sg.shape)
    v = z * (sg * math.sqrt(0.5))
    P = counts[0] * counts[1]
    scipy.fft.irfft2(v, s=counts, workers=workers, norm="forward")  # plan / warm-up
    t0 = time.perf_counter()
    done = 0
    while done < nfields:
        scipy.fft.irfft2(v, s=counts, workers=workers, norm="forward")
        done += batch
    secs = time.perf_counter() - t0
    return done * P / secs / 1e9, secs
