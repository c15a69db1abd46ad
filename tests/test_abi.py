"""CPU: the C-ABI library loads, exports every symbol include/grfc.h declares,
and its host-side logic (draw counts, grid validation, the noise bridge)
matches the oracle — no device calls."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden_cases
from oracle import pyoracle as po
from paper_1105_2737_b200 import grfc

HEADER = os.path.join(ROOT, "include", "grfc.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(grfc_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 13
    lib = ctypes.CDLL(grfc.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in grfc.h but not exported"
    assert set(syms) == set(grfc.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", grfc.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s


def test_no_unresolved_internal_symbols():
    # a shared library links with undefined symbols; catch a missing definition here
    out = subprocess.run(["nm", "-C", "-u", grfc.LIB_PATH], capture_output=True, text=True).stdout
    assert not [ln for ln in out.splitlines() if "grfc::" in ln or " grfc_" in ln], out


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", grfc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_count_draws_matches_oracle():
    port = po.Port()
    rng = np.random.default_rng(1)
    for _ in range(40):
        d = int(rng.integers(1, 5))
        counts = tuple(int(2 * rng.integers(1, 9)) for _ in range(d))
        for alg in po.ALGORITHMS:
            assert grfc.count_draws(counts, alg) == port.count_draws(counts, alg)
    assert grfc.count_draws((512, 512), grfc.ONE_FFT_OVERWRITE) == 263164
    assert grfc.half_cells((512, 512)) == 512 * 257


def test_grid_validation_errors():
    with pytest.raises(grfc.GrfcInvalidArgument, match="even"):
        grfc.count_draws((3, 4), 1)
    with pytest.raises(grfc.GrfcInvalidArgument):
        grfc.count_draws((), 1)
    with pytest.raises(grfc.GrfcInvalidArgument, match="lengths"):
        grfc.Plan((4, 4), (1.0, -1.0), grfc.Density.constant(2, 1.0))
    with pytest.raises(grfc.GrfcInvalidArgument, match="dimension mismatch"):
        grfc.Plan((8,), (1.0,), grfc.Density.constant(2, 1.0))
    with pytest.raises(grfc.GrfcInvalidArgument):
        grfc.Plan((8,), (1.0,), grfc.Density.constant(1, 1.0), algorithm=7)
    with pytest.raises(grfc.GrfcRuntimeError, match="NaN"):
        grfc.Plan((8,), (1.0,), grfc.Density.constant(1, float("nan")))
    with pytest.raises(grfc.GrfcInvalidArgument):
        grfc.Plan((8,), (1.0,), grfc.Density.poly(1, m=-1.0))


def _dens(family, r, i, dim):
    d = po.Density()
    d.family, d.dim = family, dim
    for k in range(8):
        d.r[k], d.i[k] = float(r[k]), int(i[k])
    return d


def test_noise_bridge_reproduces_reference_spectra(golden):
    """w(K) * sqrt(g) on the half-lattice == the reference's own spectrum
    (hermitian.cpp:128-203) for both one-FFT modes."""
    port = po.Port()
    ref = po.Reference() if po.reference_available() else None
    for key, counts, lengths, fam, r, i, alg, draws, _ in golden_cases(golden):
        if alg == po.TWO_FFT:
            continue
        dens = _dens(fam, r, i, len(counts))
        w = grfc.half_noise_from_draws(counts, alg, draws)
        mode = 1 if alg == po.ONE_FFT_OVERWRITE else 0
        spec = (ref or port).spectrum(counts, lengths, dens, mode, draws)
        half = spec[..., : counts[-1] // 2 + 1]
        d = len(counts)
        omegas = np.meshgrid(*[2 * np.pi * np.where(np.arange(n if a < d - 1 else n // 2 + 1) <= n // 2,
                                                      np.arange(n if a < d - 1 else n // 2 + 1),
                                                      np.arange(n if a < d - 1 else n // 2 + 1) - n) / lengths[a]
                               for a, n in enumerate(counts)], indexing="ij")
        g = np.vectorize(lambda *wv: port.density_eval(dens, list(wv)))(*omegas)
        np.testing.assert_allclose(w * np.sqrt(g), half, rtol=1e-14, atol=1e-15 * np.abs(half).max(), err_msg=key)


def test_noise_bridge_exhaustion():
    with pytest.raises(grfc.GrfcRuntimeError, match="exhausted"):
        grfc.half_noise_from_draws((8,), grfc.ONE_FFT_RECURSIVE, np.array([0.1, 0.2, 0.3]))
