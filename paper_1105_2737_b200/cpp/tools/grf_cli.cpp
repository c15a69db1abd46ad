// grf — command-line front end of the B200 generator, a drop-in for the
// reference's tools/grf.cpp (subcommands generate / cov / converge / bench,
// same flags, CSV layouts and exit codes: 0 ok, 1 usage or error, 2 criteria
// not met). Everything runs through the grf:: drop-in, i.e. on the device.
// B200 additions: generate --count N (batch of GRF1 files through the
// pipelined device writer, "{field}" in --out) and bench --batch N (fields
// per timed call, throughput on stderr); the stdout CSVs are unchanged.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <numbers>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "grf/field_io.hpp"
#include "grf/spectral.hpp"
#include "grf/stats.hpp"
#include "grf/synth.hpp"

namespace {

constexpr int kOk = 0, kUsage = 1, kCriteria = 2;

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --flag value / --flag=value parser; a flag may repeat (bench --points).
class Flags {
 public:
  Flags(int argc, char** argv, int first, const std::vector<std::string>& known) {
    for (int i = first; i < argc; ++i) {
      std::string a = argv[i];
      if (a.rfind("--", 0) != 0) throw Usage("unexpected argument '" + a + "'");
      std::string key = a.substr(2), val;
      const auto eq = key.find('=');
      if (eq != std::string::npos) {
        val = key.substr(eq + 1);
        key = key.substr(0, eq);
      } else {
        if (i + 1 >= argc) throw Usage("--" + key + " needs a value");
        val = argv[++i];
      }
      if (std::find(known.begin(), known.end(), key) == known.end()) throw Usage("unknown option --" + key);
      vals_[key].push_back(val);
    }
  }
  bool has(const std::string& k) const { return vals_.count(k) != 0; }
  std::string str(const std::string& k, const std::string& def) const { return has(k) ? vals_.at(k).back() : def; }
  std::string need(const std::string& k) const {
    if (!has(k)) throw Usage("--" + k + " is required");
    return vals_.at(k).back();
  }
  std::uint64_t u64(const std::string& k, std::uint64_t def) const {
    if (!has(k)) return def;
    const std::string s = vals_.at(k).back();
    if (s.empty() || s[0] == '-') throw Usage("--" + k + ": expected a non-negative integer");
    std::size_t pos = 0;
    const unsigned long long v = std::stoull(s, &pos);
    if (pos != s.size()) throw Usage("--" + k + ": expected an integer");
    return v;
  }
  const std::vector<std::string>& all(const std::string& k) const {
    static const std::vector<std::string> none;
    return has(k) ? vals_.at(k) : none;
  }

 private:
  std::map<std::string, std::vector<std::string>> vals_;
};

template <class T>
std::vector<T> split(const std::string& s, const std::function<T(const std::string&)>& conv) {
  std::vector<T> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ',')) out.push_back(conv(item));
  return out;
}
std::vector<std::int64_t> ints(const std::string& s) {
  return split<std::int64_t>(s, [](const std::string& t) { return std::stoll(t); });
}
std::vector<double> reals(const std::string& s) {
  return split<double>(s, [](const std::string& t) { return std::stod(t); });
}

std::string g17(double v) {
  std::ostringstream os;
  os.precision(17);
  os << v;
  return os.str();
}

grf::GridSpec make_grid(const Flags& f, std::vector<double> origin = {}) {
  const std::vector<std::int64_t> n = ints(f.need("points"));
  std::vector<double> l = f.has("lengths") ? reals(f.str("lengths", "")) : std::vector<double>(n.size(), 1.0);
  return grf::GridSpec(l, n, std::move(origin));
}

grf::Algorithm algorithm_of(const Flags& f) {
  const auto a = grf::parse_algorithm(f.str("algorithm", "recursive"));
  if (!a) throw Usage("--algorithm must be two-fft, one-fft or recursive");
  return *a;
}

const char* kDefaultDensity = "poly:m=1,k=1,l=1,n=2";

int cmd_generate(const Flags& f) {
  const grf::GridSpec grid = make_grid(f);
  const auto density = grf::parse_density(f.str("density", kDefaultDensity), grid.dim());
  const grf::Algorithm alg = algorithm_of(f);
  const std::string out = f.need("out"), format = f.str("format", "grf1");
  const std::uint64_t seed = f.u64("seed", 0), count = f.u64("count", 1);
  if (format == "pgm" && grid.dim() != 2) throw std::invalid_argument("pgm output requires a 2-dimensional grid");
  if (format != "grf1" && format != "csv" && format != "pgm")
    throw std::invalid_argument("unknown format '" + format + "'");
  if (count != 1 && format != "grf1") throw std::invalid_argument("--count > 1 needs --format grf1");
  const auto t0 = std::chrono::steady_clock::now();
  if (count != 1) {  // device -> pinned -> file pipeline
    grf::write_grf1_batch(grid, *density, seed, 0, count, alg, out);
  } else {
    const grf::RealField field = grf::synthesize(grid, *density, seed, alg);
    if (format == "grf1") {
      grf::write_grf1(out, field);
    } else if (format == "csv") {
      std::ofstream os(out, std::ios::trunc);
      if (!os) throw std::runtime_error("cannot open '" + out + "' for writing");
      grf::write_field_csv(os, field);
    } else {
      grf::write_field_pgm(out, field);
    }
  }
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::cerr << "generated " << grid.point_count() * static_cast<std::int64_t>(count) << " points with "
            << grf::algorithm_name(alg) << " in " << s << " s\n";
  return kOk;
}

int cmd_cov(const Flags& f) {
  const std::uint64_t samples = f.u64("samples", 10000);
  if (samples < 1) throw std::invalid_argument("--samples must be >= 1");
  const grf::GridSpec grid = make_grid(f);
  const auto density = grf::parse_density(f.str("density", kDefaultDensity), grid.dim());
  const grf::Algorithm alg = algorithm_of(f);
  grf::MultiIndex ref = f.has("ref-index") ? ints(f.str("ref-index", "")) : grf::MultiIndex(grid.counts().size(), 0);
  if (!grid.valid_index(ref)) throw std::invalid_argument("--ref-index out of range");
  const std::string oracle = f.str("oracle", "none");
  if (oracle != "closed-form" && oracle != "discrete" && oracle != "none")
    throw std::invalid_argument("--oracle must be closed-form, discrete or none");
  if (oracle == "closed-form" && density->spec_string() != "test1d")
    throw std::invalid_argument("closed-form oracle is only available for the test1d density");
  const grf::CovarianceEstimate est = grf::estimate_covariance(grid, *density, alg, samples, ref, f.u64("seed", 0));
  std::vector<double> discrete;
  if (oracle == "discrete") discrete = grf::exact_discrete_covariance_all(grid, *density);
  std::ostringstream csv;
  for (int a = 1; a <= grid.dim(); ++a) csv << "lag" << a << ',';
  csv << "estimate,oracle,abs_diff\n";
  for (std::int64_t i = 0; i < grid.point_count(); ++i) {
    const grf::MultiIndex k = grid.index_at(i);
    grf::MultiIndex lag(k.size());
    double r2 = 0.0;
    for (std::size_t a = 0; a < k.size(); ++a) {
      const std::int64_t n = grid.counts()[a];
      lag[a] = ((k[a] - ref[a]) % n + n) % n;
      const std::int64_t signed_lag = lag[a] <= n / 2 ? lag[a] : lag[a] - n;  // torus lag
      const double r = static_cast<double>(signed_lag) * grid.spacing(static_cast<int>(a));
      csv << g17(r) << ',';
      r2 += r * r;
    }
    const double e = est.estimates[static_cast<std::size_t>(i)];
    csv << g17(e);
    std::optional<double> o;
    if (oracle == "closed-form") o = grf::closed_form_c1d(std::sqrt(r2));
    if (oracle == "discrete") o = discrete[static_cast<std::size_t>(grid.linear_index(lag))];
    if (o)
      csv << ',' << g17(*o) << ',' << g17(std::abs(e - *o));
    else
      csv << ",,";
    csv << '\n';
  }
  const std::string out = f.str("out", "");
  if (out.empty()) {
    std::cout << csv.str();
  } else {
    std::ofstream os(out, std::ios::trunc);
    if (!os) throw std::runtime_error("cannot open '" + out + "' for writing");
    os << csv.str();
  }
  return kOk;
}

int cmd_converge(const Flags& f) {
  const std::uint64_t samples = f.u64("samples", 100000);
  if (samples < 1) throw std::invalid_argument("--samples must be >= 1");
  const std::string levels = f.str("levels", "2..6");
  const auto dots = levels.find("..");
  const int lo = std::stoi(levels.substr(0, dots));
  const int hi = dots == std::string::npos ? lo : std::stoi(levels.substr(dots + 2));
  const grf::ConvergenceReport rep = grf::convergence_study(lo, hi, samples, algorithm_of(f), f.u64("seed", 0));
  std::cout << "level,cells,max_error,mc_floor\n";
  for (const auto& r : rep.rows)
    std::cout << r.level << ',' << r.cells << ',' << g17(r.max_err) << ',' << g17(r.mc_floor) << '\n';
  if (rep.fitted_slope) {
    std::cout << "# fitted_slope=" << g17(*rep.fitted_slope) << " levels=" << rep.fitted_levels.front() << ".."
              << rep.fitted_levels.back() << '\n';
  } else {
    std::cout << "# warning: fewer than two levels above 3x the Monte Carlo floor; no slope fit\n";
    std::cerr << "warning: no slope fit possible for the requested levels\n";
  }
  return rep.fitted_slope && *rep.fitted_slope <= -3.0 ? kOk : kCriteria;
}

int cmd_bench(const Flags& f) {
  const std::uint64_t repeat = f.u64("repeat", 7), batch = f.u64("batch", 1), seed = f.u64("seed", 0);
  if (repeat < 5) throw std::invalid_argument("--repeat must be >= 5");
  if (batch < 1) throw std::invalid_argument("--batch must be >= 1");
  if (!f.has("points")) throw Usage("--points is required");
  const std::string spec = f.str("density", kDefaultDensity);
  std::cout << "algorithm,points,P,repeat,median_seconds,draws\n";
  bool met = true;
  for (const std::string& pts : f.all("points")) {
    const std::vector<std::int64_t> n = ints(pts);
    const grf::GridSpec grid(std::vector<double>(n.size(), 1.0), n);
    const auto density = grf::parse_density(spec, grid.dim());
    std::string label;
    for (std::size_t i = 0; i < n.size(); ++i) label += (i ? "x" : "") + std::to_string(n[i]);
    double two_fft = 0.0;
    std::vector<double> medians;
    for (const grf::Algorithm alg :
         {grf::Algorithm::two_fft, grf::Algorithm::one_fft_overwrite, grf::Algorithm::one_fft_recursive}) {
      const auto once = [&](std::uint64_t s) {  // one timed call: `batch` fields to host memory
        const auto t0 = std::chrono::steady_clock::now();
        if (batch == 1)
          (void)grf::synthesize(grid, *density, s, alg);
        else
          (void)grf::synthesize_batch(grid, *density, s, 0, batch, alg);
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      };
      once(seed);  // warm-up
      std::vector<double> t;
      for (std::uint64_t r = 0; r < repeat; ++r) t.push_back(once(seed + r + 1));
      std::sort(t.begin(), t.end());
      const double med = t[t.size() / 2];
      if (alg == grf::Algorithm::two_fft) two_fft = med;
      medians.push_back(med);
      std::cout << grf::algorithm_name(alg) << ',' << label << ',' << grid.point_count() << ',' << repeat << ','
                << g17(med) << ',' << grf::count_draws(grid, alg) << '\n';
      std::cerr << "# " << grf::algorithm_name(alg) << ' ' << label << " x" << batch << ": "
                << static_cast<double>(grid.point_count()) * static_cast<double>(batch) / med / 1e9
                << " Gpts/s end to end\n";
    }
    for (std::size_t i = 1; i < medians.size(); ++i) met = met && medians[i] <= 0.75 * two_fft;
  }
  return met ? kOk : kCriteria;
}

}  // namespace

int main(int argc, char** argv) {
  static const std::map<std::string, std::vector<std::string>> known = {
      {"generate", {"points", "lengths", "density", "algorithm", "seed", "out", "format", "count"}},
      {"cov", {"points", "lengths", "density", "algorithm", "seed", "samples", "ref-index", "oracle", "out"}},
      {"converge", {"levels", "samples", "algorithm", "seed"}},
      {"bench", {"points", "repeat", "density", "seed", "batch"}},
  };
  if (argc < 2 || known.count(argv[1]) == 0) {
    std::cerr << "usage: grf {generate|cov|converge|bench} [--option value ...]\n";
    return kUsage;
  }
  const std::string cmd = argv[1];
  try {
    const Flags f(argc, argv, 2, known.at(cmd));
    if (cmd == "generate") return cmd_generate(f);
    if (cmd == "cov") return cmd_cov(f);
    if (cmd == "converge") return cmd_converge(f);
    return cmd_bench(f);
  } catch (const Usage& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  }
}
