/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's GRF synthesis path
 * (/root/reference/proj/core/src/{grid,hermitian,spectral,synth}.cpp), used
 * only as the checker for the CUDA path: tests/, bench.py's cpu_baseline leg
 * and __graft_entry__.smoke() may call it; the product never does.
 *
 * Parity pin: tests/test_oracle.py checks every function here against the
 * reference itself compiled unmodified into oracle/_ref (oracle/Makefile) and
 * against the golden fixtures in tests/golden/ generated from it.
 */
#ifndef GRF_ORACLE_H
#define GRF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Density descriptor (families: 0 poly, 1 aniso, 2 test1d, 3 gaussian-cov,
 * 4 matern, 5 constant). r/i parameter slots are documented per family in
 * gro_density_eval. Same layout as the harness' ref_density. */
typedef struct {
  int family;
  int dim;
  double r[8];
  int i[8];
} gro_density;

enum { GRO_OK = 0, GRO_EINVAL = 1, GRO_ERUNTIME = 2 };
enum { GRO_TWO_FFT = 0, GRO_ONE_FFT_OVERWRITE = 1, GRO_ONE_FFT_RECURSIVE = 2 };
enum { GRO_EXACT_SET = 0, GRO_OVERWRITE = 1 };

const char* gro_last_error(void);
int gro_validate_grid(int d, const int64_t* n, const double* l);
uint64_t gro_count_draws(int d, const int64_t* n, int alg);
double gro_density_eval(const gro_density* g, const double* omega);
int64_t gro_conjugate_reps(int d, const int64_t* n, int64_t* lin, uint8_t* self, int64_t cap);
int gro_spectrum(int d, const int64_t* n, const double* l, const gro_density* g, int mode,
                 const double* draws, uint64_t ndraws, double* out);
/* sign = +1: reference "forward" (exp(+), unnormalised); -1: "inverse"
 * (exp(-), x 1/P) — /root/reference/proj/core/include/grf/dft.hpp:11-14. */
void gro_dft(int d, const int64_t* n, const double* in, double* out, int sign);
int gro_synthesize(int d, const int64_t* n, const double* l, const gro_density* g, int alg,
                   const double* draws, uint64_t ndraws, double* field, double* residue);
int gro_exact_cov_all(int d, const int64_t* n, const double* l, const gro_density* g, double* out);

#ifdef __cplusplus
}
#endif

#endif
