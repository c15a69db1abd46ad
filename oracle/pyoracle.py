"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes bindings to the two CPU checkers built by oracle/Makefile:

* ``Port``      — oracle/_build/libgrf_oracle.so, the plain-C restatement
                  (oracle/grf_oracle.c) of the reference's synthesis path.
* ``Reference`` — oracle/_ref/libgrf_ref.so, the reference's own proj/core
                  compiled unmodified (FFTW replaced by the API stand-in).

Only tests/, bench.py's cpu_baseline / --impl reference legs and
__graft_entry__.smoke() import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libgrf_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libgrf_ref.so")

TWO_FFT, ONE_FFT_OVERWRITE, ONE_FFT_RECURSIVE = 0, 1, 2
ALGORITHMS = (TWO_FFT, ONE_FFT_OVERWRITE, ONE_FFT_RECURSIVE)
FAMILY = {"poly": 0, "aniso": 1, "test1d": 2, "gauss": 3, "matern": 4, "constant": 5}


class Density(C.Structure):
    """POD density descriptor shared by the oracle, the reference harness and
    (field for field) the product C-ABI ``grfc_density``."""

    _fields_ = [("family", C.c_int), ("dim", C.c_int), ("r", C.c_double * 8), ("i", C.c_int * 8)]


def density(name: str, dim: int, **kw) -> Density:
    d = Density()
    d.family = FAMILY[name]
    d.dim = dim
    if name == "poly":
        d.r[0] = kw.get("m", 1.0)
        d.i[0], d.i[1], d.i[2] = kw.get("k", 1), kw.get("l", 1), kw.get("n", 1)
    elif name == "aniso":
        d.r[0] = kw.get("m", 1.0)
        d.i[0] = kw.get("n", 1)
        for a, k in enumerate(kw["ks"]):
            d.i[1 + a] = k
    elif name == "gauss":
        d.r[0] = kw["ell"]
    elif name == "matern":
        d.r[0], d.r[1] = kw["nu"], kw["ell"]
    elif name == "constant":
        d.r[0] = kw.get("c", 1.0)
    return d


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _i64(a: Sequence[int]):
    arr = (C.c_int64 * len(a))(*a)
    return arr


def _f64(a: Sequence[float]):
    return (C.c_double * len(a))(*a)


def _ptr(x: np.ndarray, ctype=C.c_double):
    return x.ctypes.data_as(C.POINTER(ctype))


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise FileNotFoundError(f"{self.path} missing: run `make -C oracle` (or __graft_entry__.build())")
        self.lib = C.CDLL(self.path)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, getattr(self.lib, self.prefix + "last_error")().decode())


class Port(_Lib):
    prefix = "gro_"
    path = PORT_LIB

    def __init__(self):
        super().__init__()
        L = self.lib
        L.gro_count_draws.restype = C.c_uint64
        L.gro_density_eval.restype = C.c_double
        L.gro_conjugate_reps.restype = C.c_int64

    def count_draws(self, counts, alg) -> int:
        return int(self.lib.gro_count_draws(len(counts), _i64(counts), alg))

    def density_eval(self, dens: Density, omega) -> float:
        return float(self.lib.gro_density_eval(C.byref(dens), _f64(omega)))

    def conjugate_reps(self, counts):
        P = int(np.prod(counts))
        lin = np.zeros(P, np.int64)
        self_ = np.zeros(P, np.uint8)
        n = self.lib.gro_conjugate_reps(len(counts), _i64(counts), _ptr(lin, C.c_int64),
                                        _ptr(self_, C.c_uint8), C.c_int64(P))
        if n < 0:
            raise OracleError(1, "invalid grid")
        return lin[:n], self_[:n].astype(bool)

    def spectrum(self, counts, lengths, dens, mode, draws):
        P = int(np.prod(counts))
        out = np.zeros(2 * P)
        draws = np.ascontiguousarray(draws, np.float64)
        self._check(self.lib.gro_spectrum(len(counts), _i64(counts), _f64(lengths), C.byref(dens), mode,
                                          _ptr(draws), C.c_uint64(len(draws)), _ptr(out)))
        return out.view(np.complex128).reshape(counts)

    def dft(self, counts, x, sign):
        x = np.ascontiguousarray(x, np.complex128)
        out = np.zeros_like(x)
        self.lib.gro_dft(len(counts), _i64(counts), _ptr(x.view(np.float64)), _ptr(out.view(np.float64)), sign)
        return out

    def synthesize(self, counts, lengths, dens, alg, draws):
        P = int(np.prod(counts))
        out = np.zeros(P)
        res = C.c_double(0)
        draws = np.ascontiguousarray(draws, np.float64)
        self._check(self.lib.gro_synthesize(len(counts), _i64(counts), _f64(lengths), C.byref(dens), alg,
                                            _ptr(draws), C.c_uint64(len(draws)), _ptr(out), C.byref(res)))
        return out.reshape(counts), res.value

    def exact_cov_all(self, counts, lengths, dens):
        out = np.zeros(int(np.prod(counts)))
        self._check(self.lib.gro_exact_cov_all(len(counts), _i64(counts), _f64(lengths), C.byref(dens), _ptr(out)))
        return out.reshape(counts)


class Reference(_Lib):
    prefix = "ref_"
    path = REF_LIB

    def __init__(self):
        super().__init__()
        L = self.lib
        L.ref_density_eval.restype = C.c_double
        L.ref_conjugate_reps.restype = C.c_int64

    def count_draws(self, counts, alg) -> int:
        out = C.c_uint64(0)
        self._check(self.lib.ref_count_draws(len(counts), _i64(counts), alg, C.byref(out)))
        return int(out.value)

    def density_eval(self, dens: Density, omega) -> float:
        return float(self.lib.ref_density_eval(C.byref(dens), _f64(omega)))

    def conjugate_reps(self, counts):
        P = int(np.prod(counts))
        lin = np.zeros(P, np.int64)
        self_ = np.zeros(P, np.uint8)
        n = self.lib.ref_conjugate_reps(len(counts), _i64(counts), _ptr(lin, C.c_int64),
                                        _ptr(self_, C.c_uint8), C.c_int64(P))
        if n < 0:
            raise OracleError(1, self.lib.ref_last_error().decode())
        return lin[:n], self_[:n].astype(bool)

    def spectrum(self, counts, lengths, dens, mode, draws):
        P = int(np.prod(counts))
        out = np.zeros(2 * P)
        draws = np.ascontiguousarray(draws, np.float64)
        self._check(self.lib.ref_spectrum(len(counts), _i64(counts), _f64(lengths), C.byref(dens), mode,
                                          _ptr(draws), C.c_uint64(len(draws)), _ptr(out)))
        return out.view(np.complex128).reshape(counts)

    def synthesize(self, counts, lengths, dens, alg, draws, backend=0):
        """backend 0 = FftwBackend (stand-in FFT), 1 = NaiveDftBackend."""
        P = int(np.prod(counts))
        out = np.zeros(P)
        res = C.c_double(0)
        used = C.c_uint64(0)
        draws = np.ascontiguousarray(draws, np.float64)
        self._check(self.lib.ref_synthesize_draws(len(counts), _i64(counts), _f64(lengths), C.byref(dens), alg,
                                                  _ptr(draws), C.c_uint64(len(draws)), backend, _ptr(out),
                                                  C.byref(res), C.byref(used)))
        return out.reshape(counts), res.value, int(used.value)

    def xoshiro(self, seed, substream, n):
        """n normals and n raw u64 words of the reference's Xoshiro256Stream(seed, substream)."""
        normals = np.zeros(n)
        words = np.zeros(n, np.uint64)
        self._check(self.lib.ref_xoshiro(C.c_uint64(seed), C.c_uint64(substream), C.c_uint64(n), _ptr(normals),
                                         _ptr(words, C.c_uint64)))
        return normals, words

    def synthesize_seed(self, counts, lengths, dens, alg, seed):
        out = np.zeros(int(np.prod(counts)))
        self._check(self.lib.ref_synthesize_seed(len(counts), _i64(counts), _f64(lengths), C.byref(dens), alg,
                                                 C.c_uint64(seed), _ptr(out)))
        return out.reshape(counts)

    def exact_cov_all(self, counts, lengths, dens, backend=0):
        out = np.zeros(int(np.prod(counts)))
        self._check(self.lib.ref_exact_cov_all(len(counts), _i64(counts), _f64(lengths), C.byref(dens), backend,
                                               _ptr(out)))
        return out.reshape(counts)

    def bench_batch(self, counts, lengths, dens, alg, seed, nfields, threads):
        secs = C.c_double(0)
        chk = C.c_double(0)
        self._check(self.lib.ref_bench_batch(len(counts), _i64(counts), _f64(lengths), C.byref(dens), alg,
                                             C.c_uint64(seed), C.c_uint64(nfields), threads, C.byref(secs),
                                             C.byref(chk)))
        return secs.value, chk.value


    def estimate_covariance_fixed(self, counts, lengths, dens, alg, reference, draws, threads=0):
        """grf::estimate_covariance with per-sample FixedStreams: draws is (samples, ndraws)."""
        draws = np.ascontiguousarray(draws, np.float64)
        out = np.zeros(int(np.prod(counts)))
        self._check(self.lib.ref_estimate_covariance_fixed(
            len(counts), _i64(counts), _f64(lengths), C.byref(dens), alg, C.c_uint64(draws.shape[0]),
            _i64(reference), _ptr(draws), C.c_uint64(draws.shape[1]), threads, _ptr(out)))
        return out.reshape(counts)

    def convergence_study(self, level_min, level_max, samples, alg, seed, threads=0):
        rows = np.zeros(4 * 16)
        n = C.c_int(0)
        slope = C.c_double(0)
        self._check(self.lib.ref_convergence_study(level_min, level_max, C.c_uint64(samples), alg,
                                                   C.c_uint64(seed), threads, _ptr(rows), C.byref(n),
                                                   C.byref(slope)))
        return rows[:4 * n.value].reshape(n.value, 4), slope.value


    def write_grf1(self, path, counts, lengths, values):
        v = np.ascontiguousarray(values, np.float64).ravel()
        self._check(self.lib.ref_write_grf1(str(path).encode(), len(counts), _i64(counts), _f64(lengths), _ptr(v)))

    def read_grf1(self, path, cap=1 << 24):
        dim = C.c_int(0)
        counts = np.zeros(16, np.int64)
        lengths = np.zeros(16)
        vals = np.zeros(cap)
        self._check(self.lib.ref_read_grf1(str(path).encode(), C.byref(dim), _ptr(counts, C.c_int64), _ptr(lengths),
                                           _ptr(vals), C.c_uint64(cap)))
        d = dim.value
        P = int(np.prod(counts[:d]))
        return tuple(int(c) for c in counts[:d]), tuple(lengths[:d]), vals[:P].reshape(counts[:d])


def reference_available() -> bool:
    return os.path.exists(REF_LIB)
