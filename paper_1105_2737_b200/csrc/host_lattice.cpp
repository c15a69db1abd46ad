#include "host_lattice.h"

#include <cmath>
#include <limits>

namespace grfc {

// GridSpec rules (reference grid.cpp:10-30): d >= 1; every N_i even and >= 2;
// every l_i finite and > 0 (skipped when l is null); prod N_i fits int64.
bool check_grid_spec(int d, const int64_t* n, const double* l, int64_t* points, std::string& err) {
  if (d < 1) return err = "GridSpec: dimension must be >= 1", false;
  int64_t p = 1;
  for (int a = 0; a < d; ++a) {
    if (n[a] < 2 || (n[a] & 1)) return err = "GridSpec: point counts must be even and >= 2", false;
    if (l && !(std::isfinite(l[a]) && l[a] > 0.0))
      return err = "GridSpec: edge lengths must be positive and finite", false;
    if (p > std::numeric_limits<int64_t>::max() / n[a]) return err = "GridSpec: total point count overflows", false;
    p *= n[a];
  }
  if (points) *points = p;
  return true;
}

bool validate_grid(int d, const int64_t* n, const double* l, std::string& err) {
  if (!check_grid_spec(d, n, l, nullptr, err)) return false;
  if (d > 8) return err = "grfc: dimension > 8 not supported", false;
  return true;
}

uint64_t half_cells(int d, const int64_t* n) {
  uint64_t c = (uint64_t)(n[d - 1] / 2 + 1);
  for (int a = 0; a + 1 < d; ++a) c *= (uint64_t)n[a];
  return c;
}

uint64_t count_draws(int d, const int64_t* n, int alg) {
  uint64_t p = 1;
  for (int a = 0; a < d; ++a) p *= (uint64_t)n[a];
  if (alg != 1) return p;  // two_fft and exact set: P real degrees of freedom
  return 2 * half_cells(d, n) - (uint64_t{1} << d);
}

namespace {

// Row-major product walk over per-axis value lists (skipped if any is empty).
void walk_lists(int d, const std::vector<std::vector<int64_t>>& v, bool self,
                const std::function<void(const int64_t*, bool)>& fn) {
  for (int a = 0; a < d; ++a)
    if (v[a].empty()) return;
  std::vector<size_t> pos(d, 0);
  std::vector<int64_t> k(d);
  for (int a = 0; a < d; ++a) k[a] = v[a][0];
  for (;;) {
    fn(k.data(), self);
    int a = d - 1;
    for (; a >= 0; --a) {
      if (++pos[a] < v[a].size()) {
        k[a] = v[a][pos[a]];
        break;
      }
      pos[a] = 0;
      k[a] = v[a][0];
    }
    if (a < 0) return;
  }
}

bool is_self(int d, const int64_t* n, const int64_t* k) {
  for (int a = 0; a < d; ++a)
    if (k[a] != 0 && k[a] != n[a] / 2) return false;
  return true;
}

}  // namespace

void for_each_rep(int d, const int64_t* n, const std::function<void(const int64_t*, bool)>& fn) {
  std::vector<std::vector<int64_t>> v(d);
  for (int a = 0; a < d; ++a) v[a] = {0, n[a] / 2};
  walk_lists(d, v, true, fn);
  std::vector<int> chosen;
  for (int m = 1; m <= d; ++m) {
    chosen.assign(m, 0);
    for (int i = 0; i < m; ++i) chosen[i] = i;
    for (;;) {
      for (int a = 0, c = 0; a < d; ++a) {
        const int64_t half = n[a] / 2;
        v[a].clear();
        if (c < m && chosen[c] == a) {
          for (int64_t x = 1; x < half; ++x) v[a].push_back(x);
          if (c > 0)
            for (int64_t x = half + 1; x < n[a]; ++x) v[a].push_back(x);
          ++c;
        } else {
          v[a] = {0, half};
        }
      }
      walk_lists(d, v, false, fn);
      int i = m - 1;
      while (i >= 0 && chosen[i] == d - m + i) --i;
      if (i < 0) break;
      ++chosen[i];
      for (int j = i + 1; j < m; ++j) chosen[j] = chosen[j - 1] + 1;
    }
  }
}

bool arrange_half_noise(int d, const int64_t* n, int alg, const double* draws, uint64_t ndraws,
                        std::vector<double>& w, std::string& err) {
  const uint64_t cells = half_cells(d, n);
  const int64_t hd = n[d - 1] / 2 + 1;
  w.assign(2 * cells, 0.0);
  const double r = 1.0 / std::sqrt(2.0);
  uint64_t pos = 0;
  bool ok = true;
  auto next = [&]() -> double {
    if (pos >= ndraws) {
      ok = false;
      return 0.0;
    }
    return draws[pos++];
  };
  // H index of a full-lattice multi-index, or -1 when outside H.
  auto h_index = [&](const int64_t* k) -> int64_t {
    if (k[d - 1] > n[d - 1] / 2) return -1;
    int64_t h = 0;
    for (int a = 0; a < d - 1; ++a) h = h * n[a] + k[a];
    return h * hd + k[d - 1];
  };
  std::vector<int64_t> neg(d);
  auto set_cell = [&](const int64_t* k, bool self) {
    if (!ok) return;
    if (self) {
      const double a = next();
      const int64_t h = h_index(k);
      w[2 * h] = a;
      w[2 * h + 1] = 0.0;
      return;
    }
    const double a = next(), b = next();
    for (int x = 0; x < d; ++x) neg[x] = k[x] == 0 ? 0 : n[x] - k[x];
    const int64_t h = h_index(k), hm = h_index(neg.data());
    if (h >= 0) {
      w[2 * h] = r * a;
      w[2 * h + 1] = r * b;
    }
    if (hm >= 0) {
      w[2 * hm] = r * a;
      w[2 * hm + 1] = -r * b;
    }
  };
  if (alg == 2) {
    for_each_rep(d, n, set_cell);
  } else {
    std::vector<std::vector<int64_t>> v(d);
    for (int a = 0; a < d; ++a) {
      const int64_t len = (a == d - 1) ? hd : n[a];
      for (int64_t x = 0; x < len; ++x) v[a].push_back(x);
    }
    walk_lists(d, v, false, [&](const int64_t* k, bool) { set_cell(k, is_self(d, n, k)); });
  }
  if (!ok) err = "FixedStream: stream exhausted";
  return ok;
}

void reference_order_counters(int d, const int64_t* n, int alg, std::vector<uint64_t>& ctr,
                              std::vector<uint8_t>& nd) {
  ctr.clear();
  nd.clear();
  if (alg == 0) {
    uint64_t p = 1;
    for (int a = 0; a < d; ++a) p *= (uint64_t)n[a];
    ctr.reserve(p / 2);
    for (uint64_t j = 0; j < p / 2; ++j) {
      ctr.push_back(j);
      nd.push_back(2);
    }
    return;
  }
  if (alg == 2) {
    for_each_rep(d, n, [&](const int64_t* k, bool self) {
      uint64_t lin = 0;
      for (int a = 0; a < d; ++a) lin = lin * (uint64_t)n[a] + (uint64_t)k[a];
      ctr.push_back(lin);
      nd.push_back(self ? 1 : 2);
    });
    return;
  }
  const uint64_t cells = half_cells(d, n);
  const int64_t hd = n[d - 1] / 2 + 1;
  std::vector<int64_t> k(d);
  for (uint64_t c = 0; c < cells; ++c) {
    uint64_t r = c;
    k[d - 1] = (int64_t)(r % (uint64_t)hd);
    r /= (uint64_t)hd;
    for (int a = d - 2; a >= 0; --a) {
      k[a] = (int64_t)(r % (uint64_t)n[a]);
      r /= (uint64_t)n[a];
    }
    ctr.push_back(c);
    nd.push_back(is_self(d, n, k.data()) ? 1 : 2);
  }
}

}  // namespace grfc
