"""ctypes binding of the grfc C-ABI (include/grfc.h).

This is the Python face of the drop-in boundary: ``Plan`` wraps
``grfc_plan_*``/``grfc_generate*``; errors map like the reference's
exceptions (``GrfcInvalidArgument`` <- std::invalid_argument,
``GrfcRuntimeError`` <- std::runtime_error; see
/root/reference/proj/core/src/synth.cpp:70-71,105-106 and grid.cpp:13-28).

The shared library is built in-tree by ``__graft_entry__.build()``; if it is
missing this module raises at import — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GRFC_LIB") or os.path.join(_HERE, "lib", "libgrfc.so")

OK, EINVAL, ERUNTIME, ECUDA, ENCCL = 0, 1, 2, 3, 4
F32, F64 = 0, 1
TWO_FFT, ONE_FFT_OVERWRITE, ONE_FFT_RECURSIVE = 0, 1, 2
ALGORITHM_NAMES = {"two-fft": TWO_FFT, "one-fft": ONE_FFT_OVERWRITE, "recursive": ONE_FFT_RECURSIVE}
POLY, ANISO, TEST1D, GAUSSIAN_COV, MATERN, CONSTANT, TABLE = range(7)


class GrfcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class GrfcInvalidArgument(GrfcError, ValueError):
    pass


class GrfcRuntimeError(GrfcError):
    pass


class Density(C.Structure):
    """POD image of grfc_density (same field layout)."""

    _fields_ = [("family", C.c_int), ("dim", C.c_int), ("r", C.c_double * 8), ("i", C.c_int * 8)]

    @classmethod
    def poly(cls, dim, m=1.0, k=1, l=1, n=1):
        d = cls(family=POLY, dim=dim)
        d.r[0] = m
        d.i[0], d.i[1], d.i[2] = k, l, n
        return d

    @classmethod
    def aniso(cls, m, ks: Sequence[int], n):
        d = cls(family=ANISO, dim=len(ks))
        d.r[0] = m
        d.i[0] = n
        for a, k in enumerate(ks):
            d.i[1 + a] = k
        return d

    @classmethod
    def test1d(cls):
        return cls(family=TEST1D, dim=1)

    @classmethod
    def gaussian_cov(cls, dim, ell):
        d = cls(family=GAUSSIAN_COV, dim=dim)
        d.r[0] = ell
        return d

    @classmethod
    def matern(cls, dim, nu, ell):
        d = cls(family=MATERN, dim=dim)
        d.r[0], d.r[1] = nu, ell
        return d

    @classmethod
    def constant(cls, dim, c):
        d = cls(family=CONSTANT, dim=dim)
        d.r[0] = c
        return d

    @classmethod
    def table(cls, dim):
        return cls(family=TABLE, dim=dim)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    lib.grfc_last_error.restype = C.c_char_p
    lib.grfc_last_launch_count.restype = C.c_uint64
    P = C.c_void_p
    sigs = {
        "grfc_count_draws": [C.c_int, P, C.c_int, P],
        "grfc_half_lattice_cells": [C.c_int, P, P],
        "grfc_plan_create": [P, C.c_int, P, P, C.c_int, C.c_int, P, C.c_int],
        "grfc_plan_set_sqrt_gamma_table": [P, P],
        "grfc_generate": [P, C.c_uint64, C.c_uint64, C.c_uint64, P, C.c_uint64, P],
        "grfc_generate_host": [P, C.c_uint64, C.c_uint64, C.c_uint64, P, P],
        "grfc_generate_injected": [P, P, C.c_uint64, P, P],
        "grfc_dump_noise": [P, C.c_uint64, C.c_uint64, P, C.c_uint64],
        "grfc_dft_c2c": [C.c_int, P, P, P, C.c_int, P],
        "grfc_plan_info": [P, P, P, P],
        "grfc_half_noise_from_draws": [C.c_int, P, C.c_int, P, C.c_uint64, P],
        "grfc_kernel_timing_read": [C.c_int, P, P, P],
        "grfc_generate_injected_host": [P, P, C.c_uint64, P],
        "grfc_dft_c2c_host": [C.c_int, P, P, P, C.c_int, C.c_int],
        "grfc_dft_naive_c2c": [C.c_int, P, P, P, C.c_int, P],
        "grfc_grid_check": [C.c_int, P, P, P],
        "grfc_comm_unique_id": [P],
        "grfc_comm_create": [P, P, C.c_int, C.c_int, C.c_int],
        "grfc_comm_info": [P, P, P, P],
        "grfc_slab_exchange": [P, P, P, P, P],
        "grfc_slab_generate": [P, P, C.c_uint64, C.c_uint64, P, P],
        "grfc_dft_naive_c2c_host": [C.c_int, P, P, P, C.c_int, C.c_int],
        "grfc_conjugate_reps": [C.c_int, P, P, P, C.c_uint64, P],
        "grfc_slab_sizes": [P, C.c_int, P, P, P],
        "grfc_slab_pass_a": [P, C.c_int, C.c_int, C.c_uint64, C.c_uint64, P, P],
        "grfc_slab_pass_b": [P, C.c_int, P, P, P],
        "grfc_estimate_covariance": [P, C.c_uint64, C.c_uint64, C.c_int64, P, P],
        "grfc_estimate_covariance_host": [P, C.c_uint64, C.c_uint64, C.c_int64, P],
        "grfc_covariance_partials": [P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, P, P],
        "grfc_covariance_merge": [P, P, C.c_uint64, C.c_uint64, P, P],
        "grfc_covariance_accumulate": [P, P, C.c_uint64, C.c_uint64, C.c_int64, P, P],
        "grfc_covariance_chunk_injected_host": [P, P, C.c_uint64, C.c_uint64, C.c_int64, P],
        "grfc_plan_grid": [P, P, P, P, P, P],
        "grfc_write_grf1": [P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_char_p],
        "grfc_measure_fp32_peak": [C.c_int, P],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.grfc_plan_destroy.argtypes = [P]
    lib.grfc_plan_destroy.restype = None
    lib.grfc_comm_destroy.argtypes = [P]
    lib.grfc_comm_destroy.restype = None
    lib.grfc_kernel_timing_enable.argtypes = [C.c_int]
    lib.grfc_kernel_timing_enable.restype = None
    return lib


_lib = _load()

#: Every symbol include/grfc.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "grfc_last_error", "grfc_count_draws", "grfc_half_lattice_cells", "grfc_plan_create",
    "grfc_plan_set_sqrt_gamma_table", "grfc_plan_destroy", "grfc_generate", "grfc_generate_host",
    "grfc_generate_injected", "grfc_half_noise_from_draws", "grfc_dump_noise", "grfc_dft_c2c", "grfc_plan_info",
    "grfc_last_launch_count", "grfc_kernel_timing_enable", "grfc_kernel_timing_read",
    "grfc_generate_injected_host", "grfc_dft_c2c_host", "grfc_conjugate_reps", "grfc_slab_sizes",
    "grfc_slab_pass_a", "grfc_slab_pass_b", "grfc_estimate_covariance", "grfc_estimate_covariance_host",
    "grfc_covariance_partials", "grfc_covariance_merge", "grfc_covariance_accumulate",
    "grfc_covariance_chunk_injected_host", "grfc_plan_grid", "grfc_write_grf1", "grfc_measure_fp32_peak",
    "grfc_dft_naive_c2c", "grfc_dft_naive_c2c_host", "grfc_grid_check",
    "grfc_comm_unique_id", "grfc_comm_create", "grfc_comm_destroy", "grfc_comm_info", "grfc_slab_exchange",
    "grfc_slab_generate",
)


def measure_fp32_peak(device: int = 0) -> float:
    """Measured dense FP32 TFLOP/s of the device (FFMA2 probe)."""
    v = C.c_double(0)
    _check(_lib.grfc_measure_fp32_peak(device, C.byref(v)))
    return v.value

#: Samples per accumulation chunk of the covariance estimator (GRFC_COV_CHUNK; src/stats.cpp:18).
COV_CHUNK = 1024


def grf1_bytes(counts: Sequence[int], lengths: Sequence[float], values) -> bytes:
    """GRF1 image (include/grf/field_io.hpp:10-14): "GRF1" | u32 1 | u32 d | (u64 N, f64 l)* | P f64, LE."""
    import struct

    head = b"GRF1" + struct.pack("<II", 1, len(counts))
    head += b"".join(struct.pack("<Qd", int(n), float(l)) for n, l in zip(counts, lengths))
    return head + np.ascontiguousarray(values, dtype="<f8").tobytes()


def read_grf1(path):
    """(counts, lengths, values) of a GRF1 file, validated like src/field_io.cpp:82-107."""
    import struct

    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 12:
        raise RuntimeError("read_grf1: truncated file")
    if data[:4] != b"GRF1":
        raise RuntimeError("read_grf1: bad magic")
    version, d = struct.unpack_from("<II", data, 4)
    if version != 1:
        raise RuntimeError("read_grf1: unsupported version")
    if not 1 <= d <= 16:
        raise RuntimeError("read_grf1: implausible dimension")
    off = 12 + 16 * d
    if len(data) < off:
        raise RuntimeError("read_grf1: truncated file")
    axes = [struct.unpack_from("<Qd", data, 12 + 16 * a) for a in range(d)]
    counts = tuple(int(n) for n, _ in axes)
    lengths = tuple(float(l) for _, l in axes)
    P = int(np.prod(counts))
    if len(data) < off + 8 * P:
        raise RuntimeError("read_grf1: truncated file")
    if len(data) > off + 8 * P:
        raise RuntimeError("read_grf1: trailing bytes after payload")
    return counts, lengths, np.frombuffer(data, dtype="<f8", count=P, offset=off).reshape(counts)


def conjugate_reps(counts: Sequence[int]):
    """(linear indices, self-conjugate flags) of the representative set, Appendix order."""
    P = int(np.prod(counts))
    lin = np.zeros(P, np.int64)
    flg = np.zeros(P, np.uint8)
    n = C.c_uint64(0)
    _check(_lib.grfc_conjugate_reps(len(counts), _i64(counts), lin.ctypes.data_as(C.c_void_p),
                                    flg.ctypes.data_as(C.c_void_p), P, C.byref(n)))
    return lin[: n.value], flg[: n.value].astype(bool)


def kernel_timing_enable(on: bool):
    _lib.grfc_kernel_timing_enable(1 if on else 0)


def kernel_timing_read():
    """{kernel name: (total device ms, launches)} recorded on this thread since enable."""
    rows = {}
    i = 0
    name, ms, n = C.c_char_p(), C.c_double(0), C.c_uint64(0)
    while _lib.grfc_kernel_timing_read(i, C.byref(name), C.byref(ms), C.byref(n)) == OK:
        rows[name.value.decode()] = (ms.value, int(n.value))
        i += 1
    return rows


def lib():
    return _lib


def _check(rc: int):
    if rc == OK:
        return
    msg = _lib.grfc_last_error().decode()
    if rc == EINVAL:
        raise GrfcInvalidArgument(rc, msg)
    if rc == ERUNTIME:
        raise GrfcRuntimeError(rc, msg)
    raise GrfcError(rc, msg)


def _i64(a):
    return (C.c_int64 * len(a))(*[int(x) for x in a])


def _f64(a):
    return (C.c_double * len(a))(*[float(x) for x in a])


def count_draws(counts: Sequence[int], algorithm: int) -> int:
    out = C.c_uint64(0)
    _check(_lib.grfc_count_draws(len(counts), _i64(counts), algorithm, C.byref(out)))
    return int(out.value)


def half_cells(counts: Sequence[int]) -> int:
    out = C.c_uint64(0)
    _check(_lib.grfc_half_lattice_cells(len(counts), _i64(counts), C.byref(out)))
    return int(out.value)


def half_noise_from_draws(counts: Sequence[int], algorithm: int, draws: np.ndarray) -> np.ndarray:
    """Host noise bridge: unit-variance Hermitian noise per half-lattice cell (complex128, shape H)."""
    d = np.ascontiguousarray(draws, np.float64)
    out = np.zeros(2 * half_cells(counts), np.float64)
    _check(_lib.grfc_half_noise_from_draws(len(counts), _i64(counts), algorithm, d.ctypes.data_as(C.c_void_p),
                                           d.size, out.ctypes.data_as(C.c_void_p)))
    return out.view(np.complex128).reshape(tuple(counts[:-1]) + (counts[-1] // 2 + 1,))


def last_launch_count() -> int:
    return int(_lib.grfc_last_launch_count())


def dft_naive_c2c(counts, d_in: int, d_out: int, sign: int, stream: int = 0):
    """Direct-sum O(P^2) DFT (the drop-in's NaiveDftBackend), same conventions as dft_c2c."""
    _check(_lib.grfc_dft_naive_c2c(len(counts), _i64(counts), C.c_void_p(d_in), C.c_void_p(d_out), sign,
                                   C.c_void_p(stream)))


def dft_c2c(counts, d_in: int, d_out: int, sign: int, stream: int = 0):
    """Device fp64 complex DFT with the reference DftBackend contract."""
    _check(_lib.grfc_dft_c2c(len(counts), _i64(counts), C.c_void_p(d_in), C.c_void_p(d_out), sign,
                             C.c_void_p(stream)))


UNIQUE_ID_BYTES = 128


def comm_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0; broadcast the bytes to every rank)."""
    buf = (C.c_ubyte * UNIQUE_ID_BYTES)()
    _check(_lib.grfc_comm_unique_id(buf))
    return bytes(buf)


class Comm:
    """NCCL communicator of the slab path (grfc_comm_create: one per rank and GPU)."""

    def __init__(self, unique_id: bytes, world: int, rank: int, device: int = 0):
        if len(unique_id) != UNIQUE_ID_BYTES:
            raise ValueError("unique id must be %d bytes" % UNIQUE_ID_BYTES)
        buf = (C.c_ubyte * UNIQUE_ID_BYTES).from_buffer_copy(unique_id)
        h = C.c_void_p()
        _check(_lib.grfc_comm_create(C.byref(h), buf, world, rank, device))
        self._h = h
        self.world, self.rank, self.device = world, rank, device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.grfc_comm_destroy(h)
            self._h = None


class Plan:
    """One (grid, density, algorithm, precision) bound to a device."""

    def __init__(self, counts: Sequence[int], lengths: Sequence[float], density: Density,
                 algorithm: int = ONE_FFT_OVERWRITE, dtype: int = F32, device: int = 0):
        self.counts = tuple(int(c) for c in counts)
        self.lengths = tuple(float(x) for x in lengths)
        self.algorithm = algorithm
        self.dtype = dtype
        self.device = device
        self._h = C.c_void_p(None)
        self._density = density
        _check(_lib.grfc_plan_create(C.byref(self._h), len(self.counts), _i64(self.counts), _f64(self.lengths),
                                     dtype, algorithm, C.byref(density), device))
        cells, points, path = C.c_uint64(0), C.c_uint64(0), C.c_char_p()
        _check(_lib.grfc_plan_info(self._h, C.byref(cells), C.byref(points), C.byref(path)))
        self.cells, self.points, self.path = int(cells.value), int(points.value), path.value.decode()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.grfc_plan_destroy(h)
            self._h = C.c_void_p(None)

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == F64 else np.float32

    def count_draws(self) -> int:
        return count_draws(self.counts, self.algorithm)

    def set_sqrt_gamma_table(self, sqrt_gamma: np.ndarray):
        t = np.ascontiguousarray(sqrt_gamma, np.float64).ravel()
        if t.size != self.cells:
            raise GrfcInvalidArgument(EINVAL, f"table needs {self.cells} half-lattice cells, got {t.size}")
        _check(_lib.grfc_plan_set_sqrt_gamma_table(self._h, t.ctypes.data_as(C.c_void_p)))

    def generate(self, seed: int, first_field: int, nfields: int, d_out: int, field_stride: Optional[int] = None,
                 stream: int = 0):
        """Device pointers/streams as ints (e.g. tensor.data_ptr(), torch stream.cuda_stream)."""
        stride = self.points if field_stride is None else field_stride
        _check(_lib.grfc_generate(self._h, seed, first_field, nfields, C.c_void_p(d_out), stride,
                                  C.c_void_p(stream)))

    def generate_host(self, seed: int, first_field: int, nfields: int, h_out: np.ndarray, stream: int = 0):
        if h_out.dtype != self.np_dtype or h_out.size < nfields * self.points or not h_out.flags.c_contiguous:
            raise GrfcInvalidArgument(EINVAL, "host buffer has the wrong dtype/size")
        _check(_lib.grfc_generate_host(self._h, seed, first_field, nfields, C.c_void_p(h_out.ctypes.data),
                                       C.c_void_p(stream)))

    def generate_host_ptr(self, seed: int, first_field: int, nfields: int, h_ptr: int, stream: int = 0):
        _check(_lib.grfc_generate_host(self._h, seed, first_field, nfields, C.c_void_p(h_ptr), C.c_void_p(stream)))

    def generate_injected(self, draws: np.ndarray, d_out: int, stream: int = 0):
        d = np.ascontiguousarray(draws, np.float64)
        _check(_lib.grfc_generate_injected(self._h, d.ctypes.data_as(C.c_void_p), d.size, C.c_void_p(d_out),
                                           C.c_void_p(stream)))

    def dump_noise(self, seed: int, field: int) -> np.ndarray:
        n = self.count_draws()
        out = np.zeros(n, np.float64)
        _check(_lib.grfc_dump_noise(self._h, seed, field, out.ctypes.data_as(C.c_void_p), n))
        return out

    # ---- slab decomposition of one 3D field (include/grfc.h grfc_slab_*)
    def slab_sizes(self, world: int):
        """(buffer complex elements, block complex elements, slab points) per rank."""
        b, k, s = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        _check(_lib.grfc_slab_sizes(self._h, world, C.byref(b), C.byref(k), C.byref(s)))
        return int(b.value), int(k.value), int(s.value)

    def slab_pass_a(self, world: int, rank: int, seed: int, field: int, d_send: int, stream: int = 0):
        _check(_lib.grfc_slab_pass_a(self._h, world, rank, seed, field, C.c_void_p(d_send), C.c_void_p(stream)))

    def slab_generate(self, comm: "Comm", seed: int, field: int, d_out: int, stream: int = 0):
        """One field over all ranks of comm (pass A -> NCCL all-to-all -> pass B); d_out = this
        rank's planes (slab_sizes(world)[2] reals)."""
        _check(_lib.grfc_slab_generate(self._h, comm._h, seed, field, C.c_void_p(d_out), C.c_void_p(stream)))

    def slab_exchange(self, comm: "Comm", d_send: int, d_recv: int, stream: int = 0):
        _check(_lib.grfc_slab_exchange(self._h, comm._h, C.c_void_p(d_send), C.c_void_p(d_recv),
                                       C.c_void_p(stream)))

    def slab_pass_b(self, world: int, d_recv: int, d_out: int, stream: int = 0):
        _check(_lib.grfc_slab_pass_b(self._h, world, C.c_void_p(d_recv), C.c_void_p(d_out), C.c_void_p(stream)))

    # ---- GRF1 output (grf::write_grf1, src/field_io.cpp:60-80)
    def write_grf1(self, seed: int, first_field: int, nfields: int, path_format: str):
        """Fields (seed, first_field + i) -> one GRF1 file each; "{field}" in the path is the field index."""
        _check(_lib.grfc_write_grf1(self._h, seed, first_field, nfields, str(path_format).encode()))

    # ---- Monte-Carlo covariance (grf::estimate_covariance, src/stats.cpp:39-97)
    def linear_index(self, index) -> int:
        """Row-major linear index of a grid multi-index (GridSpec::linear_index)."""
        if isinstance(index, (int, np.integer)):
            return int(index)
        lin = 0
        for i, n in zip(index, self.counts):
            lin = lin * n + int(i)
        return lin

    def estimate_covariance(self, seed: int, samples: int, reference, d_out: int, stream: int = 0):
        _check(_lib.grfc_estimate_covariance(self._h, seed, samples, self.linear_index(reference), C.c_void_p(d_out),
                                             C.c_void_p(stream)))

    def estimate_covariance_host(self, seed: int, samples: int, reference) -> np.ndarray:
        out = np.empty(self.points, dtype=np.float64)
        _check(_lib.grfc_estimate_covariance_host(self._h, seed, samples, self.linear_index(reference),
                                                  out.ctypes.data_as(C.c_void_p)))
        return out.reshape(self.counts)

    def covariance_partials(self, seed: int, samples: int, chunk0: int, nchunks: int, reference, d_partials: int,
                            stream: int = 0):
        _check(_lib.grfc_covariance_partials(self._h, seed, samples, chunk0, nchunks, self.linear_index(reference),
                                             C.c_void_p(d_partials), C.c_void_p(stream)))

    def covariance_merge(self, d_partials: int, nchunks: int, samples: int, d_out: int, stream: int = 0):
        _check(_lib.grfc_covariance_merge(self._h, C.c_void_p(d_partials), nchunks, samples, C.c_void_p(d_out),
                                          C.c_void_p(stream)))

    def covariance_accumulate(self, d_fields: int, nfields: int, field_stride: int, reference, d_acc: int,
                              stream: int = 0):
        _check(_lib.grfc_covariance_accumulate(self._h, C.c_void_p(d_fields), nfields, field_stride,
                                               self.linear_index(reference), C.c_void_p(d_acc), C.c_void_p(stream)))

    def covariance_chunk_injected_host(self, draws: np.ndarray, reference) -> np.ndarray:
        """Partial sum of one chunk whose samples are given as draw rows (reference draw order)."""
        d = np.ascontiguousarray(draws, dtype=np.float64)
        if d.ndim != 2:
            raise ValueError("draws must be (nsamples, ndraws)")
        out = np.empty(self.points, dtype=np.float64)
        _check(_lib.grfc_covariance_chunk_injected_host(self._h, d.ctypes.data_as(C.c_void_p), d.shape[0], d.shape[1],
                                                        self.linear_index(reference), out.ctypes.data_as(C.c_void_p)))
        return out

    def estimate_covariance_tensor(self, seed: int, samples: int, reference, stream=None):
        import torch

        out = torch.empty(self.counts, dtype=torch.float64, device=f"cuda:{self.device}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.estimate_covariance(seed, samples, reference, out.data_ptr(), s.cuda_stream)
        return out

    def covariance_partials_tensor(self, seed: int, samples: int, chunk0: int, nchunks: int, reference, stream=None):
        import torch

        out = torch.empty((nchunks,) + self.counts, dtype=torch.float64, device=f"cuda:{self.device}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.covariance_partials(seed, samples, chunk0, nchunks, reference, out.data_ptr(), s.cuda_stream)
        return out

    def covariance_merge_tensor(self, partials, samples: int, stream=None):
        import torch

        p = partials.contiguous()
        out = torch.empty(self.counts, dtype=torch.float64, device=p.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.covariance_merge(p.data_ptr(), p.shape[0], samples, out.data_ptr(), s.cuda_stream)
        return out

    # ---- torch conveniences (torch is plumbing: device memory and streams)
    def generate_tensor(self, seed: int, first_field: int = 0, nfields: int = 1, out=None, stream=None):
        import torch

        if out is None:
            out = torch.empty((nfields,) + self.counts, dtype=torch.float64 if self.dtype == F64 else torch.float32,
                              device=f"cuda:{self.device}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.generate(seed, first_field, nfields, out.data_ptr(), self.points, s.cuda_stream)
        return out

    def generate_injected_tensor(self, draws: np.ndarray, stream=None):
        import torch

        out = torch.empty(self.counts, dtype=torch.float64 if self.dtype == F64 else torch.float32,
                          device=f"cuda:{self.device}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.generate_injected(draws, out.data_ptr(), s.cuda_stream)
        return out
