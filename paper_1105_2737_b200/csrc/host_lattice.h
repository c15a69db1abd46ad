// Host-side lattice logic of the grfc C-ABI (pure C++, no CUDA): grid
// validation, draw counts, the representative-set enumeration order, and the
// noise bridge between the reference's sequential draw order and the
// device's per-cell layout. Citations relative to /root/reference/proj/core.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace grfc {

// GridSpec validation, src/grid.cpp:10-30 (lengths may be null: counts only);
// any d >= 1. *points = prod N_i when valid (points may be null).
bool check_grid_spec(int d, const int64_t* counts, const double* lengths, int64_t* points, std::string& err);
// check_grid_spec plus the device path's d <= 8.
bool validate_grid(int d, const int64_t* counts, const double* lengths, std::string& err);

// count_draws, src/synth.cpp:211-218 + src/hermitian.cpp:228-236.
uint64_t count_draws(int d, const int64_t* counts, int algorithm);

// |H| = N_1 .. N_{d-1} (N_d/2 + 1).
uint64_t half_cells(int d, const int64_t* counts);

// Representative set in the paper-Appendix order of src/hermitian.cpp:39-84:
// L0 = {0,M}^d row-major, then blocks n = 1..d over lexicographic n-subsets
// of axes (first chosen axis [1,M-1], further chosen [1,M-1] u [M+1,N-1],
// unchosen {0,M}), row-major within a block. fn(k, self_conjugate).
void for_each_rep(int d, const int64_t* counts, const std::function<void(const int64_t*, bool)>& fn);

// Noise bridge, injected direction: resolves the reference's Hermitian
// arrangement of `draws` (its own draw order) into the unit-variance noise
// w(K) for every half-lattice cell K (row-major over H), as interleaved
// (re, im) doubles. Self-conjugate: w = a; paired: w = (a + i b)/sqrt(2) with
// the mirror conj — overwrite mode replays the half-lattice sweep with later
// visits winning (hermitian.cpp:178-202), exact-set mode the rep walk
// (hermitian.cpp:173-177). Returns false (err set) if draws run out, like
// FixedStream (include/grf/random.hpp:56).
bool arrange_half_noise(int d, const int64_t* counts, int algorithm, const double* draws, uint64_t ndraws,
                        std::vector<double>& w_half, std::string& err);

// Noise bridge, dump direction: the Philox counters in the reference's draw
// order and how many draws (1 or 2) each contributes. Alg 1: counter J/2 per
// pair of grid points (2 draws); Alg 2: H cell index c; Alg 3: full-lattice
// index of each rep.
void reference_order_counters(int d, const int64_t* counts, int algorithm, std::vector<uint64_t>& counters,
                              std::vector<uint8_t>& ndraw);

}  // namespace grfc
