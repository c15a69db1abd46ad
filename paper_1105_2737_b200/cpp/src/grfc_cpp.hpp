// Internal glue between the grf:: drop-in and the grfc C-ABI: status ->
// exception mapping (std::invalid_argument / std::runtime_error as the
// reference throws them), RAII plans and density descriptors.
#pragma once

#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/grfc.h"
#include "grf/grid.hpp"
#include "grf/spectral.hpp"

namespace grf::detail {

inline void check(grfc_status st) {
  if (st == GRFC_OK) return;
  const std::string msg = grfc_last_error();
  if (st == GRFC_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct PlanDeleter {
  void operator()(grfc_plan_s* p) const { grfc_plan_destroy(p); }
};
using PlanPtr = std::unique_ptr<grfc_plan_s, PlanDeleter>;

/// The POD descriptor of a density the device evaluates in-kernel, or a
/// GRFC_DENSITY_TABLE descriptor for any other subclass.
grfc_density describe(const SpectralDensity& density);

/// sqrt(g) over the half-lattice, evaluated on the host at the angular
/// frequencies the reference's synthesis uses ((2 pi k~) / l).
/// Throws std::runtime_error on NaN / negative values.
std::vector<double> sqrt_gamma_table(const GridSpec& grid, const SpectralDensity& density);

using SharedPlan = std::shared_ptr<grfc_plan_s>;

/// fp64 plan for (grid, density, algorithm); the table is filled when needed.
/// Plans of in-kernel density families come from a process-wide LRU cache.
SharedPlan make_plan(const GridSpec& grid, const SpectralDensity& density, int algorithm, int dtype = GRFC_F64);
std::mutex& plan_cache_mutex();
std::list<std::pair<std::string, SharedPlan>>& plan_cache();

}  // namespace grf::detail
