/*
 * grfc — C-ABI of the B200-native Gaussian-random-field generator.
 *
 * This is the drop-in boundary for the reference's core generator
 * (/root/reference/proj/core). Every entry point names the reference
 * interface it replaces; the C++ drop-in (paper_1105_2737_b200/cpp, namespace
 * grf) and the Python mirror (paper_1105_2737_b200/grfc.py) sit on top.
 *
 * Conventions (all from the reference code, which is authoritative over its
 * SPEC/PAPER — SURVEY.md §A):
 *   - grids are row-major, last index fastest (include/grf/grid.hpp:36);
 *   - densities are evaluated at angular frequency w = 2 pi k~ / l with the
 *     Nyquist index wrapping to +N/2 (src/grid.cpp:96-111);
 *   - the field law is E[B B'] = (2 pi)^d/|A| sum_K g(w_K) cos(...)
 *     (include/grf/synth.hpp:47-51).
 *
 * Pointers are plain; no torch/CUDA types cross the boundary (streams are
 * passed as void* = cudaStream_t). All functions are thread-safe; a plan is
 * immutable after creation (grfc_plan_set_sqrt_gamma_table must precede any
 * generate call), and every call allocates its scratch stream-ordered, so one
 * plan may serve concurrent calls on different streams.
 */
#ifndef GRFC_H
#define GRFC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRFC_MAX_DIM 8

typedef enum {
  GRFC_OK = 0,
  GRFC_EINVAL = 1,   /* reference: std::invalid_argument */
  GRFC_ERUNTIME = 2, /* reference: std::runtime_error (NaN density, exhaustion) */
  GRFC_ECUDA = 3,    /* CUDA runtime failure (no reference analogue) */
  GRFC_ENCCL = 4     /* collective failure (slab path) */
} grfc_status;

typedef enum { GRFC_F32 = 0, GRFC_F64 = 1 } grfc_dtype;

/* Same order as grf::Algorithm (include/grf/synth.hpp:18-25). */
typedef enum {
  GRFC_TWO_FFT = 0,
  GRFC_ONE_FFT_OVERWRITE = 1,
  GRFC_ONE_FFT_RECURSIVE = 2
} grfc_algorithm;

/* Spectral-density descriptor: the POD image of a grf::SpectralDensity
 * (include/grf/spectral.hpp:14-85) that the device can evaluate in-kernel.
 *   POLY     r[0]=m, i[0]=k, i[1]=l, i[2]=n        (spectral.cpp:42-55)
 *   ANISO    r[0]=m, i[0]=n, i[1+a]=k_a            (spectral.cpp:65-78)
 *   TEST1D   -                                     (spectral.cpp:88-93)
 *   GAUSSIAN_COV r[0]=ell: (ell/sqrt(2pi))^d exp(-ell^2|w|^2/2)
 *   MATERN   r[0]=nu, r[1]=ell: c (1+ell^2|w|^2)^-(nu+d/2),
 *            c = ell^d Gamma(nu+d/2)/(pi^{d/2} Gamma(nu))
 *   CONSTANT r[0]=c
 *   TABLE    any user density: sqrt(g) supplied per half-lattice cell by
 *            grfc_plan_set_sqrt_gamma_table (host-evaluated, NaN-checked). */
typedef enum {
  GRFC_DENSITY_POLY = 0,
  GRFC_DENSITY_ANISO = 1,
  GRFC_DENSITY_TEST1D = 2,
  GRFC_DENSITY_GAUSSIAN_COV = 3,
  GRFC_DENSITY_MATERN = 4,
  GRFC_DENSITY_CONSTANT = 5,
  GRFC_DENSITY_TABLE = 6
} grfc_density_family;

typedef struct {
  int family;
  int dim;
  double r[8];
  int i[8];
} grfc_density;

typedef struct grfc_plan_s* grfc_plan;

/* Last error message of the calling thread ("" if none). */
const char* grfc_last_error(void);

/* Exact number of N(0,1) draws one field consumes.
 * Replaces grf::count_draws (src/synth.cpp:211-218) and
 * grf::spectrum_draw_count (src/hermitian.cpp:228-236). */
grfc_status grfc_count_draws(int dim, const int64_t* counts, int algorithm, uint64_t* out);

/* Half-lattice size |H| = N_1..N_{d-1} (N_d/2+1): the length of the table
 * grfc_plan_set_sqrt_gamma_table expects (row-major over H). */
grfc_status grfc_half_lattice_cells(int dim, const int64_t* counts, uint64_t* out);

/* Representative set of the lattice in the paper-Appendix order — the
 * reference's for_each_conjugate_rep (src/hermitian.cpp:39-84,308-311) and the
 * Alg-3 draw order: row-major linear index and self-conjugate flag of each
 * rep, written up to `cap` entries; *count = |L| = 2^d + (P - 2^d)/2. */
grfc_status grfc_conjugate_reps(int dim, const int64_t* counts, int64_t* lin, uint8_t* self_flag, uint64_t cap,
                                uint64_t* count);

/* Plan = GridSpec (include/grf/grid.hpp:16-47, validated as src/grid.cpp:10-30)
 * + density + algorithm + precision, bound to one device. Replaces the
 * per-call setup of grf::synthesize (src/synth.cpp:68-80) and the FFTW plan
 * cache (src/dft.cpp:27-69). */
grfc_status grfc_plan_create(grfc_plan* plan, int dim, const int64_t* counts,
                             const double* lengths, int dtype, int algorithm,
                             const grfc_density* density, int device);
/* sqrt(g(w_K)) for every K of the half-lattice H, row-major; required for
 * GRFC_DENSITY_TABLE (user SpectralDensity subclasses). Rejects NaN/negative
 * with GRFC_ERUNTIME like src/hermitian.cpp:147-148. */
grfc_status grfc_plan_set_sqrt_gamma_table(grfc_plan plan, const double* sqrt_gamma);
void grfc_plan_destroy(grfc_plan plan);

/* Seeded batch generation — the device form of
 * grf::synthesize(grid, density, seed, algorithm) (src/synth.cpp:129-135),
 * extended to a batch the way the reference's stats.cpp:105 derives
 * substreams (seed, j). Field f (f = first_field .. first_field+nfields-1) is
 * a pure function of (seed, f): Philox4x32-10 keyed by seed, counter
 * (cell, f). Output: nfields fields of P elements (dtype), field i at
 * d_out + i*field_stride elements. Asynchronous on `stream`. */
grfc_status grfc_generate(grfc_plan plan, uint64_t seed, uint64_t first_field, uint64_t nfields,
                          void* d_out, uint64_t field_stride, void* stream);

/* Same as grfc_generate but writes to HOST memory (pinned or pageable):
 * generation of chunk i+1 overlaps the D2H copy of chunk i. Synchronous.
 * This is the end-to-end form of grf::synthesize returning RealField.values. */
grfc_status grfc_generate_host(grfc_plan plan, uint64_t seed, uint64_t first_field,
                               uint64_t nfields, void* h_out, void* stream);

/* Injected-noise synthesis of one field: `draws` are the N(0,1) values in
 * the reference's own draw order (exactly count_draws of them) — i.e. what
 * grf::synthesize(grid, density, GaussianStream&, algorithm)
 * (src/synth.cpp:68-127) would pull from a FixedStream. The Hermitian
 * arrangement of src/hermitian.cpp:128-203 is resolved on the host; FFTs run
 * on device. This is the parity path and the stream-overload drop-in. */
grfc_status grfc_generate_injected(grfc_plan plan, const double* draws, uint64_t ndraws,
                                   void* d_out, void* stream);

/* grfc_generate_injected with a HOST output buffer (P elements of the plan's
 * dtype); synchronous. What the C++ drop-in's stream overload calls. */
grfc_status grfc_generate_injected_host(grfc_plan plan, const double* draws, uint64_t ndraws, void* h_out);

/* Host-only noise bridge (no device): the unit-variance Hermitian noise w(K)
 * the reference would assemble from `draws` (its own draw order) for every
 * half-lattice cell K, row-major over H, interleaved (re, im) — i.e. the
 * spectrum of src/hermitian.cpp:128-203 divided by sqrt(g). w_half holds
 * 2*|H| doubles. algorithm must be ONE_FFT_OVERWRITE or ONE_FFT_RECURSIVE. */
grfc_status grfc_half_noise_from_draws(int dim, const int64_t* counts, int algorithm, const double* draws,
                                       uint64_t ndraws, double* w_half);

/* The Philox noise grfc_generate uses for field (seed, field), in the
 * reference's draw order (count_draws values, as doubles; fp32 plans give
 * fp32-valued noise). Feeding it to the reference through a FixedStream
 * reproduces grfc_generate's field. Synchronous. */
grfc_status grfc_dump_noise(grfc_plan plan, uint64_t seed, uint64_t field, double* draws,
                            uint64_t ndraws);

/* Device complex DFT with the reference DftBackend contract
 * (include/grf/dft.hpp:11-25): sign=+1 "forward" out[K] = sum in[J] e^{+...};
 * sign=-1 "inverse" out[J] = P^-1 sum in[K] e^{-...}. fp64 interleaved,
 * device pointers, out-of-place (in == out rejected as src/dft.cpp:21-22). */
grfc_status grfc_dft_c2c(int dim, const int64_t* counts, const double* d_in, double* d_out,
                         int sign, void* stream);
/* Same with host buffers on `device` (synchronous): the CudaDftBackend of
 * the C++ drop-in (replaces FftwBackend::forward/inverse, src/dft.cpp:95-108). */
grfc_status grfc_dft_c2c_host(int dim, const int64_t* counts, const double* h_in, double* h_out, int sign,
                              int device);

/* Direct-sum complex DFT, O(P^2), same conventions and errors as grfc_dft_c2c:
 * the drop-in's NaiveDftBackend (replaces NaiveDftBackend::forward/inverse,
 * src/dft.cpp:113-165 — the reference's cross-check backend for small grids).
 * Device pointers, synchronous on `stream`. */
grfc_status grfc_dft_naive_c2c(int dim, const int64_t* counts, const double* d_in, double* d_out, int sign,
                               void* stream);
/* Same with host buffers on `device` (synchronous). */
grfc_status grfc_dft_naive_c2c_host(int dim, const int64_t* counts, const double* h_in, double* h_out, int sign,
                                    int device);

/* Slab decomposition of one 3D field over `world` ranks (pow2 3D plans;
 * world divides N0 and N1) — the multi-GPU form of grfc_generate for a
 * single large field. Per field and rank:
 *   grfc_slab_pass_a  generation + axis-0 FFT of the rank's spectrum slab
 *                     (k1 in [rank N1/world, (rank+1) N1/world)) into d_send;
 *   all-to-all        block q of every rank's d_send (elements
 *                     [q*block, (q+1)*block), complex) goes to block r of
 *                     rank q's d_recv — contiguous blocks, no packing (NCCL
 *                     ncclAlltoAll / grouped ncclSend-ncclRecv, or
 *                     torch.distributed.all_to_all_single);
 *   grfc_slab_pass_b  axis-1 + axis-2 transforms of the rank's field planes
 *                     j0 in [rank N0/world, ...) into d_out (slab_points reals).
 * Mirror partners that live on other ranks are regenerated locally from the
 * counter-based noise, never exchanged. Results are bit-identical for every
 * world size. Buffer sizes are in complex elements of the plan's dtype. */
grfc_status grfc_slab_sizes(grfc_plan plan, int world, uint64_t* buf_elems, uint64_t* block_elems,
                            uint64_t* slab_points);
grfc_status grfc_slab_pass_a(grfc_plan plan, int world, int rank, uint64_t seed, uint64_t field, void* d_send,
                             void* stream);
grfc_status grfc_slab_pass_b(grfc_plan plan, int world, const void* d_recv, void* d_out, void* stream);

/* NCCL communicator of the slab path (one process per GPU). Bootstrap: rank 0
 * calls grfc_comm_unique_id, the host framework broadcasts the
 * GRFC_UNIQUE_ID_BYTES bytes, every rank calls grfc_comm_create with its rank
 * and CUDA device (ncclGetUniqueId / ncclCommInitRank; NCCL is loaded at run
 * time, GRFC_ENCCL if it is absent). */
#define GRFC_UNIQUE_ID_BYTES 128
typedef struct grfc_comm_s* grfc_comm;
grfc_status grfc_comm_unique_id(unsigned char* id);
grfc_status grfc_comm_create(grfc_comm* out, const unsigned char* id, int world, int rank, int device);
void grfc_comm_destroy(grfc_comm comm);
grfc_status grfc_comm_info(grfc_comm comm, int* world, int* rank, int* device);
/* The all-to-all step above over `comm` (grouped ncclSend/ncclRecv; the
 * rank's own block is a device copy), enqueued on `stream`. */
grfc_status grfc_slab_exchange(grfc_plan plan, grfc_comm comm, const void* d_send, void* d_recv, void* stream);
/* One field (seed, field) over all ranks of `comm`: pass A -> exchange ->
 * pass B; d_out = this rank's planes j0 in [rank N0/world, ...) (slab_points
 * reals). Scratch is stream-ordered; asynchronous on `stream`. Fields are
 * bit-identical to grfc_generate's for every world size. */
grfc_status grfc_slab_generate(grfc_plan plan, grfc_comm comm, uint64_t seed, uint64_t field, void* d_out,
                               void* stream);

/* GridSpec validation (replaces GridSpec::GridSpec's checks, src/grid.cpp:10-30):
 * dim >= 1, every counts[i] even and >= 2, every lengths[i] finite and > 0
 * (lengths may be NULL: counts only), prod counts fits int64. GRFC_EINVAL with
 * the reason in grfc_last_error(); *points = prod counts on success (may be
 * NULL). Any dim (plans additionally need dim <= 8). Host-only. */
grfc_status grfc_grid_check(int dim, const int64_t* counts, const double* lengths, int64_t* points);

/* Plan grid: dim, counts[dim], lengths[dim], dtype and device (any output may be NULL). */
grfc_status grfc_plan_grid(grfc_plan plan, int* dim, int64_t* counts, double* lengths, int* dtype, int* device);

/* Batch GRF1 writer — the reference's write_grf1 (src/field_io.cpp:60-80,
 * format include/grf/field_io.hpp:10-14: "GRF1" | u32 1 | u32 dim |
 * (u64 N_i, f64 l_i)... | P f64, little-endian) applied to fields
 * (seed, first_field + i), i < nfields, streamed device -> pinned host ->
 * file with generation, copies and file writes overlapped. Field f goes to
 * path_format with "{field}" replaced by f (required when nfields > 1).
 * fp32 plans are widened exactly to f64. Synchronous. Errors: unopenable or
 * short write -> GRFC_ERUNTIME with the reference's messages. */
grfc_status grfc_write_grf1(grfc_plan plan, uint64_t seed, uint64_t first_field, uint64_t nfields,
                            const char* path_format);

/* Monte-Carlo covariance against one reference grid point — the device form
 * of grf::estimate_covariance (src/stats.cpp:39-97, include/grf/stats.hpp):
 *   est[K] = M^-1 sum_{j<M} f_j[ref] f_j[K],   f_j = field (seed, j) of grfc_generate
 * (the reference's substream (seed, j), stats.cpp:105). Determinism as the
 * reference (stats.cpp:17-18,60-93): samples in fixed chunks of
 * GRFC_COV_CHUNK; per chunk and point, fp64 multiply-then-add in ascending j;
 * chunk partials merged in chunk order with Kahan compensation; then x (1/M).
 * Bit-identical for any generation batch size and any number of devices.
 * `ref` is the row-major linear index of the reference point
 * (GridSpec::linear_index). Errors: samples == 0 or ref out of range ->
 * GRFC_EINVAL with the reference's messages (stats.cpp:43-45). Output: P
 * doubles. */
#define GRFC_COV_CHUNK 1024
grfc_status grfc_estimate_covariance(grfc_plan plan, uint64_t seed, uint64_t samples, int64_t ref, double* d_out,
                                     void* stream);
/* Same, HOST output; synchronous (what the C++ drop-in calls). */
grfc_status grfc_estimate_covariance_host(grfc_plan plan, uint64_t seed, uint64_t samples, int64_t ref,
                                          double* h_out);
/* Multi-device form: the partial sums of chunks [chunk0, chunk0+nchunks) of a
 * `samples`-sample estimate (nchunks*P doubles, chunk-major) ... */
grfc_status grfc_covariance_partials(grfc_plan plan, uint64_t seed, uint64_t samples, uint64_t chunk0,
                                     uint64_t nchunks, int64_t ref, double* d_partials, void* stream);
/* ... and their chunk-ordered Kahan merge scaled by 1/samples (all chunks, in
 * order, gathered on one device): equals grfc_estimate_covariance bit for bit. */
grfc_status grfc_covariance_merge(grfc_plan plan, const double* d_partials, uint64_t nchunks, uint64_t samples,
                                  double* d_out, void* stream);
/* Building block for caller-made fields (device, plan dtype, field j at
 * d_fields + j*field_stride): d_acc[K] += sum_j f_j[ref] f_j[K], ascending j. */
grfc_status grfc_covariance_accumulate(grfc_plan plan, const void* d_fields, uint64_t nfields,
                                       uint64_t field_stride, int64_t ref, double* d_acc, void* stream);
/* One chunk of the StreamFactory overload (stats.cpp:39-82): sample i is
 * synthesized from draws + i*ndraws (reference draw order, as
 * grfc_generate_injected); h_partial (P doubles, host) receives the chunk's
 * partial sum. The caller merges chunks in order (Kahan) and scales by 1/M. */
grfc_status grfc_covariance_chunk_injected_host(grfc_plan plan, const double* draws, uint64_t nsamples,
                                                uint64_t ndraws, int64_t ref, double* h_partial);

/* Plan introspection for benchmarks: bytes of workspace per field and the
 * kernel path chosen ("pow2-2d", "generic", ...). */
grfc_status grfc_plan_info(grfc_plan plan, uint64_t* cells_half, uint64_t* points,
                           const char** path);

/* Benchmark helper: measured dense FP32 throughput of `device` in TFLOP/s
 * (packed FFMA2 chains on every SM; FMA = 2 flops) — the compute-roofline
 * denominator bench.py reports beside the HBM one. */
grfc_status grfc_measure_fp32_peak(int device, double* tflops);

/* Number of kernel launches the last generate call on this thread issued. */
uint64_t grfc_last_launch_count(void);

/* Per-kernel timing for benchmarks, per calling thread: while enabled, every
 * kernel the library launches is bracketed by CUDA events recorded on the
 * stream it is launched on. Enabling clears previous records. */
void grfc_kernel_timing_enable(int on);
/* Records aggregated by kernel name (synchronises the events): the index-th
 * kernel's name, summed device milliseconds and launch count. GRFC_EINVAL
 * past the last kernel. */
grfc_status grfc_kernel_timing_read(int index, const char** name, double* total_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif

#endif
