// C++ tests of the grf:: drop-in (paper_1105_2737_b200/cpp) on a GPU: the
// reference's own test cases restated (file:line cited per case), written
// against the same public API a reference user calls.
//
//   test_dropin                     run all cases, exit code = #failures
//   test_dropin --synth IN OUT      synthesize one field from a case file
//                                   (used by tests/test_dropin_gpu.py to
//                                   compare with the golden fixtures)
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <unistd.h>
#include <functional>
#include <numbers>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "grf/dft.hpp"
#include "grf/field_io.hpp"
#include "grf/hermitian.hpp"
#include "grf/stats.hpp"
#include "grf/synth.hpp"

using namespace grf;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                                               \
  do {                                                                                            \
    ++g_checks;                                                                                   \
    if (!(cond)) {                                                                                \
      ++g_fail;                                                                                   \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                             \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

bool near(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(std::abs(a), std::abs(b)) + 1e-300; }

class ConstantDensity final : public SpectralDensity {  // user subclass -> table path
 public:
  ConstantDensity(double c, int d) : c_(c), d_(d) {}
  int dim() const override { return d_; }
  double eval(std::span<const double> w) const override {
    check_dim(w);
    return c_;
  }
  std::string spec_string() const override { return "constant"; }

 private:
  double c_;
  int d_;
};

class RandomEvenDensity final : public SpectralDensity {
 public:
  RandomEvenDensity(std::vector<double> c, std::vector<int> e, int d) : c_(std::move(c)), e_(std::move(e)), d_(d) {}
  int dim() const override { return d_; }
  double eval(std::span<const double> w) const override {
    check_dim(w);
    double n2 = 0.0, s = 0.0;
    for (double v : w) n2 += v * v;
    for (std::size_t t = 0; t < c_.size(); ++t) {
      double mono = 1.0;
      for (double v : w)
        for (int q = 0; q < e_[t]; ++q) mono *= v * v;
      s += c_[t] * mono;
    }
    return s * std::exp(-n2);
  }
  std::string spec_string() const override { return "random-even"; }

 private:
  std::vector<double> c_;
  std::vector<int> e_;
  int d_;
};

class NanDensity final : public SpectralDensity {
 public:
  explicit NanDensity(int d) : d_(d) {}
  int dim() const override { return d_; }
  double eval(std::span<const double>) const override { return std::nan(""); }
  std::string spec_string() const override { return "nan"; }

 private:
  int d_;
};

const Algorithm kAll[] = {Algorithm::two_fft, Algorithm::one_fft_overwrite, Algorithm::one_fft_recursive};

void run(const char* name, const std::function<void()>& body) {
  g_case = name;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_fail;
    std::fprintf(stderr, "FAIL [%s] unexpected exception: %s\n", name, e.what());
  }
}

// --synth IN OUT: IN = int32 d, int64 counts[d], f64 lengths[d], int32 family,
// f64 r[8], int32 i[8], int32 alg, uint64 ndraws, f64 draws[ndraws]
int synth_file(const char* in, const char* out) {
  std::ifstream f(in, std::ios::binary);
  auto rd = [&](void* p, std::size_t n) { f.read(static_cast<char*>(p), static_cast<std::streamsize>(n)); };
  int32_t d = 0, fam = 0, alg = 0;
  rd(&d, 4);
  std::vector<std::int64_t> counts(d);
  std::vector<double> lengths(d);
  rd(counts.data(), 8 * d);
  rd(lengths.data(), 8 * d);
  rd(&fam, 4);
  double r[8];
  int32_t iv[8];
  rd(r, sizeof r);
  rd(iv, sizeof iv);
  rd(&alg, 4);
  uint64_t nd = 0;
  rd(&nd, 8);
  std::vector<double> draws(nd);
  rd(draws.data(), 8 * nd);
  GridSpec grid(lengths, counts);
  std::unique_ptr<SpectralDensity> dens;
  switch (fam) {
    case 0: dens = std::make_unique<PolyDecayDensity>(r[0], iv[0], iv[1], iv[2], d); break;
    case 1: dens = std::make_unique<AnisoPolyDensity>(r[0], std::vector<int>(iv + 1, iv + 1 + d), iv[0]); break;
    case 2: dens = std::make_unique<Test1dDensity>(); break;
    case 3: dens = std::make_unique<GaussianCovDensity>(r[0], d); break;
    case 4: dens = std::make_unique<MaternDensity>(r[0], r[1], d); break;
    default: dens = std::make_unique<ConstantDensity>(r[0], d); break;
  }
  FixedStream rng(draws);
  const RealField fld = synthesize(grid, *dens, rng, static_cast<Algorithm>(alg));
  std::ofstream o(out, std::ios::binary);
  o.write(reinterpret_cast<const char*>(fld.values.data()), static_cast<std::streamsize>(8 * fld.values.size()));
  return rng.draws_consumed() == nd ? 0 : 3;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc == 4 && std::string(argv[1]) == "--synth") return synth_file(argv[2], argv[3]);

  run("grid validation (test_grid.cpp:15-23)", [] {
    CHECK(throws<std::invalid_argument>([] { GridSpec({1.0, 1.0}, {3, 4}); }));
    CHECK(throws<std::invalid_argument>([] { GridSpec({1.0}, {0}); }));
    CHECK(throws<std::invalid_argument>([] { GridSpec({-1.0}, {4}); }));
    CHECK(throws<std::invalid_argument>([] { GridSpec({1.0, 2.0}, {4}); }));
    const GridSpec g({1.5, 2.5}, {6, 8});
    CHECK(g.point_count() == 48);
    CHECK(near(g.domain_volume(), 3.75, 1e-15));
  });

  run("neg_index and wrapped frequency (test_grid.cpp:56-98)", [] {
    const GridSpec g({2.0 * std::numbers::pi}, {8});
    CHECK(neg_index({3}, g) == MultiIndex{5});
    CHECK(neg_index({0}, g) == MultiIndex{0});
    CHECK(near(frequency({1}, g)[0], 0.15915494309189535, 1e-14));
    CHECK(near(frequency({5}, g)[0], -0.47746482927568601, 1e-14));
    CHECK(near(angular_frequency({5}, g)[0], -3.0, 1e-14));
    CHECK(near(frequency({4}, g)[0], 4.0 / (2.0 * std::numbers::pi), 1e-14));
    CHECK(is_self_conjugate({4}, g) && !is_self_conjugate({3}, g));
  });

  run("densities (test_spectral.cpp:14-41, 98-118)", [] {
    const PolyDecayDensity d(1.0, 1, 1, 1, 2);
    CHECK(near(d.eval(std::vector<double>{0.0, 0.0}), 1.0, 1e-15));
    CHECK(near(d.eval(std::vector<double>{1.0, 0.0}), 0.5, 1e-15));
    CHECK(near(PolyDecayDensity(2.0, 2, 3, 1, 1).eval(std::vector<double>{0.0}), 1.0 / 64.0, 1e-15));
    CHECK(near(Test1dDensity().eval(std::vector<double>{0.0}), 0.10185916357881303, 1e-14));
    CHECK(near(closed_form_c1d(0.1), 0.9074359548895577, 1e-14));
    CHECK(throws<std::invalid_argument>([&] { d.eval(std::vector<double>{1.0}); }));
    CHECK(throws<std::invalid_argument>([] { parse_density("gauss:m=1", 2); }));
    CHECK(throws<std::invalid_argument>([] { parse_density("poly:m=1,k=1", 2); }));
    CHECK(parse_density("poly:m=1,k=1,l=1,n=2", 2)->spec_string() == "poly:m=1,k=1,l=1,n=2");
    CHECK(parse_density("matern:nu=1.5,ell=0.1", 2)->dim() == 2);
    CHECK(throws<std::invalid_argument>([] { parse_density("test1d", 2); }));
  });

  run("representative set (test_hermitian.cpp:44-93)", [] {
    const ConjugateRepSet s = build_conjugate_reps(GridSpec({1.0}, {4}));
    CHECK(s.reps.size() == 3 && s.reps[0] == MultiIndex{0} && s.reps[1] == MultiIndex{2} && s.reps[2] == MultiIndex{1});
    CHECK(s.self_conjugate.size() == 2);
    CHECK(build_conjugate_reps(GridSpec({1.0, 1.0}, {4, 4})).reps.size() == 10);
    const GridSpec g88({1.0, 1.0}, {8, 8});
    std::set<std::pair<std::int64_t, std::int64_t>> want, got;
    for (int a = 0; a <= 4; ++a)
      for (int b = 0; b <= 4; ++b) want.insert({a, b});
    for (int a = 1; a <= 3; ++a)
      for (int b = 5; b <= 7; ++b) want.insert({a, b});
    for (const auto& k : build_conjugate_reps(g88).reps) got.insert({k[0], k[1]});
    CHECK(got == want);
    for (const GridSpec& g : {GridSpec({1.0}, {12}), GridSpec({1.0, 1.0}, {2, 10}), GridSpec({1.0, 1.0, 1.0}, {4, 2, 6}),
                              GridSpec({1.0, 1.0, 1.0, 1.0}, {2, 4, 2, 6})}) {
      const ConjugateRepSet r = build_conjugate_reps(g);
      std::vector<int> seen(static_cast<std::size_t>(g.point_count()), 0);
      for (std::size_t i = 0; i < r.reps.size(); ++i) {
        seen[static_cast<std::size_t>(g.linear_index(r.reps[i]))]++;
        if (i >= r.self_conjugate.size()) seen[static_cast<std::size_t>(g.linear_index(neg_index(r.reps[i], g)))]++;
      }
      bool ok = true;
      for (int v : seen) ok = ok && v == 1;
      CHECK(ok);
    }
  });

  run("draw counts (test_synth.cpp:150-156, test_hermitian.cpp:106-119)", [] {
    const GridSpec g44({1.0, 1.0}, {4, 4});
    CHECK(count_draws(g44, Algorithm::two_fft) == 16);
    CHECK(count_draws(g44, Algorithm::one_fft_recursive) == 16);
    CHECK(count_draws(g44, Algorithm::one_fft_overwrite) == 20);
    CHECK(count_draws(GridSpec({1.0, 1.0}, {6, 2}), Algorithm::one_fft_overwrite) == 20);
    for (Algorithm a : kAll) {  // instrumented: exactly count_draws values are pulled
      ConstantStream rng(0.5);
      synthesize(GridSpec({1.0, 1.0, 1.0}, {4, 2, 6}), ConstantDensity(1.0, 3), rng, a);
      CHECK(rng.draws_consumed() == count_draws(GridSpec({1.0, 1.0, 1.0}, {4, 2, 6}), a));
    }
  });

  run("zero stream -> zero field (test_synth.cpp:50-59)", [] {
    for (Algorithm a : kAll) {
      ConstantStream rng(0.0);
      const RealField f = synthesize(GridSpec({1.0, 1.0}, {4, 6}), ConstantDensity(2.0, 2), rng, a);
      bool zero = true;
      for (double v : f.values) zero = zero && v == 0.0;
      CHECK(zero);
      CHECK(f.imag_residue == 0.0);
    }
  });

  run("spectral impulse -> constant field (test_synth.cpp:61-73)", [] {
    const GridSpec g({1.0, 1.0}, {4, 4});
    const double c = 2.25;
    std::vector<double> draws(count_draws(g, Algorithm::one_fft_recursive), 0.0);
    draws[0] = 1.0;
    FixedStream rng(draws);
    const RealField f = synthesize(g, ConstantDensity(c, 2), rng, Algorithm::one_fft_recursive);
    const double want = std::sqrt(4.0 * std::numbers::pi * std::numbers::pi * c);
    bool ok = true;
    for (double v : f.values) ok = ok && near(v, want, 1e-12);
    CHECK(ok);
  });

  run("hermitian invariants + corruption (test_hermitian.cpp:121-148)", [] {
    Xoshiro256Stream shapes(99);
    const RandomEvenDensity dens({1.0, 0.4}, {0, 1}, 2);
    for (int t = 0; t < 50; ++t) {
      const std::int64_t n1 = 2 * (1 + static_cast<std::int64_t>(shapes.next_u64() % 4));
      const std::int64_t n2 = 2 * (1 + static_cast<std::int64_t>(shapes.next_u64() % 4));
      Xoshiro256Stream rng(static_cast<std::uint64_t>(t));
      const auto mode = t % 2 ? SpectrumMode::overwrite : SpectrumMode::exact_set;
      CHECK(verify_hermitian(synthesize_spectrum(GridSpec({1.0, 2.0}, {n1, n2}), dens, rng, mode)));
    }
    Xoshiro256Stream rng(5);
    const GridSpec g({1.0, 1.0}, {4, 4});
    HermitianSpectrum s = synthesize_spectrum(g, ConstantDensity(1.0, 2), rng, SpectrumMode::exact_set);
    CHECK(verify_hermitian(s));
    HermitianSpectrum bad = s;
    bad.values[static_cast<std::size_t>(g.linear_index({0, 2}))] += std::complex<double>(0.0, 1.0);
    CHECK(!verify_hermitian(bad));
  });

  run("covariance: flat density, evenness, transform-at-once (test_synth.cpp:75-126)", [] {
    const GridSpec g({1.0, 2.0}, {4, 6});
    const ConstantDensity flat(0.7, 2);
    const double at0 = 0.7 * 4.0 * std::numbers::pi * std::numbers::pi * 24.0 / 2.0;
    CHECK(near(exact_discrete_covariance(g, flat, MultiIndex{0, 0}), at0, 1e-12));
    CHECK(std::abs(exact_discrete_covariance(g, flat, MultiIndex{1, 3})) < 1e-12 * at0);
    const GridSpec g2({2.0, 3.0}, {8, 6});
    const PolyDecayDensity dens(0.75, 1, 2, 1, 2);
    const std::vector<double> all = exact_discrete_covariance_all(g2, dens);
    for (std::int64_t i = 0; i < g2.point_count(); i += 7)
      CHECK(near(all[static_cast<std::size_t>(i)], exact_discrete_covariance(g2, dens, g2.index_at(i)), 1e-10));
    const GridSpec g3({1.0, 1.0}, {6, 8});
    const PolyDecayDensity d3(1.0, 1, 1, 2, 2);
    CHECK(near(exact_discrete_covariance(g3, d3, MultiIndex{1, 2}),
               exact_discrete_covariance(g3, d3, neg_index({1, 2}, g3)), 1e-12));
  });

  run("CudaDftBackend round trip and naive sums (test_synth.cpp:21-48)", [] {
    CudaDftBackend dft;
    Xoshiro256Stream rng(7);
    for (const GridSpec& g : {GridSpec({1.0}, {8}), GridSpec({1.0, 1.0}, {4, 6}), GridSpec({1.0, 1.0, 1.0}, {2, 4, 6})}) {
      const auto p = static_cast<std::size_t>(g.point_count());
      std::vector<std::complex<double>> x(p), fwd(p), back(p);
      for (auto& v : x) v = {rng.next(), rng.next()};
      dft.forward(g, x, fwd);
      dft.inverse(g, fwd, back);
      double err = 0.0, mx = 0.0;
      for (std::size_t i = 0; i < p; ++i) {
        err = std::max(err, std::abs(back[i] - x[i]));
        mx = std::max(mx, std::abs(x[i]));
      }
      CHECK(err <= 1e-12 * mx);
      double diff = 0.0, sc = 0.0;  // forward vs the literal exp(+) sum
      for (std::int64_t kk = 0; kk < g.point_count(); ++kk) {
        const MultiIndex k = g.index_at(kk);
        std::complex<double> acc = 0.0;
        for (std::int64_t jj = 0; jj < g.point_count(); ++jj) {
          const MultiIndex j = g.index_at(jj);
          double t = 0.0;
          for (int a = 0; a < g.dim(); ++a)
            t += static_cast<double>((k[a] * j[a]) % g.counts()[a]) / static_cast<double>(g.counts()[a]);
          acc += x[static_cast<std::size_t>(jj)] * std::polar(1.0, 2.0 * std::numbers::pi * t);
        }
        diff = std::max(diff, std::abs(acc - fwd[static_cast<std::size_t>(kk)]));
        sc = std::max(sc, std::abs(acc));
      }
      CHECK(diff <= 1e-11 * sc);
    }
    std::vector<std::complex<double>> a(8);
    CHECK(throws<std::invalid_argument>([&] { dft.forward(GridSpec({1.0}, {8}), a, a); }));
  });

  run("seed overload determinism and batch substreams", [] {
    const GridSpec g({1.0, 1.0}, {64, 32});
    const MaternDensity m(1.5, 0.1, 2);
    const RealField a = synthesize(g, m, 42, Algorithm::one_fft_overwrite);
    const RealField b = synthesize(g, m, 42, Algorithm::one_fft_overwrite);
    CHECK(a.values == b.values);
    CHECK(a.provenance.seed == 42);
    const auto batch = synthesize_batch(g, m, 42, 0, 3, Algorithm::one_fft_overwrite);
    CHECK(batch[0].values == a.values);
    CHECK(synthesize_batch(g, m, 42, 2, 1, Algorithm::one_fft_overwrite)[0].values == batch[2].values);
    CHECK(batch[1].values != batch[0].values);
  });

  run("monte carlo covariance vs exact, quick (test_synth.cpp:185-197)", [] {
    const GridSpec g({2.0 * std::numbers::pi}, {8}, {-std::numbers::pi});
    const Test1dDensity dens;
    const std::vector<double> exact = exact_discrete_covariance_all(g, dens);
    const std::uint64_t m = 20000;
    const double tol = 5.0 * 2.0 / std::sqrt(static_cast<double>(m)) * exact[0];
    for (Algorithm a : kAll) {
      const auto fields = synthesize_batch(g, dens, 101, 0, m, a);
      std::vector<double> est(8, 0.0);
      for (const auto& f : fields)
        for (int i = 0; i < 8; ++i) est[i] += f.values[0] * f.values[i];
      bool ok = true;
      for (int i = 0; i < 8; ++i) ok = ok && std::abs(est[i] / m - exact[i]) < tol;
      CHECK(ok);
    }
  });

  run("error paths (test_synth.cpp:199-219)", [] {
    const GridSpec g({1.0}, {8});
    ConstantStream zero(0.0);
    CHECK(throws<std::invalid_argument>([&] { synthesize(g, ConstantDensity(1.0, 2), zero, Algorithm::two_fft); }));
    for (Algorithm a : kAll) {
      Xoshiro256Stream rng(1);
      CHECK(throws<std::runtime_error>([&] { synthesize(g, NanDensity(1), rng, a); }));
    }
    FixedStream short_stream({0.1, 0.2, 0.3});
    CHECK(throws<std::runtime_error>(
        [&] { synthesize(g, ConstantDensity(1.0, 1), short_stream, Algorithm::one_fft_recursive); }));
    CHECK(parse_algorithm("two-fft") == Algorithm::two_fft);
    CHECK(parse_algorithm("one-fft") == Algorithm::one_fft_overwrite);
    CHECK(parse_algorithm("recursive") == Algorithm::one_fft_recursive);
    CHECK(!parse_algorithm("three-fft").has_value());
    CHECK(throws<std::invalid_argument>([&] { exact_discrete_covariance(g, ConstantDensity(1.0, 1), MultiIndex{8}); }));
  });

  run("estimator: rigged constant fields estimate to c^2 (test_stats.cpp:12-27)", [] {
    const GridSpec g({1.0}, {8});
    const ConstantDensity dens(4.0, 1);
    const std::uint64_t nd = count_draws(g, Algorithm::one_fft_recursive);
    const StreamFactory impulse = [nd](std::uint64_t) {
      std::vector<double> v(static_cast<std::size_t>(nd), 0.0);
      v[0] = 1.0;
      return std::make_unique<FixedStream>(std::move(v));
    };
    const CovarianceEstimate e = estimate_covariance(g, dens, Algorithm::one_fft_recursive, 50, MultiIndex{3}, impulse);
    const double c = std::sqrt(2.0 * std::numbers::pi * 4.0 / g.domain_volume());
    bool ok = e.estimates.size() == 8 && e.sample_count == 50;
    for (double v : e.estimates) ok = ok && near(v, c * c, 1e-12);
    CHECK(ok);
    const StreamFactory short_streams = [](std::uint64_t) { return std::make_unique<FixedStream>(std::vector<double>{1.0}); };
    CHECK(throws<std::runtime_error>(
        [&] { estimate_covariance(g, dens, Algorithm::one_fft_recursive, 5, MultiIndex{0}, short_streams); }));
  });

  run("estimator: flat density decorrelates off the reference (test_stats.cpp:29-41)", [] {
    const GridSpec g({1.0}, {16});
    const double c = 1.5;
    const std::uint64_t m = 40000;
    const CovarianceEstimate e = estimate_covariance(g, ConstantDensity(c, 1), Algorithm::two_fft, m, MultiIndex{0}, 17);
    const double at0 = c * 2.0 * std::numbers::pi * 16.0 / g.domain_volume();
    const double tol = 5.0 * at0 / std::sqrt(static_cast<double>(m));
    CHECK(std::abs(e.estimates[0] - at0) < tol);
    bool ok = true;
    for (std::size_t i = 1; i < e.estimates.size(); ++i) ok = ok && std::abs(e.estimates[i]) < tol;
    CHECK(ok);
    CHECK(e.seed == 17);
  });

  run("estimator: reproducible for any worker count (test_stats.cpp:43-56)", [] {
    const GridSpec g({2.0 * std::numbers::pi}, {16}, {-std::numbers::pi});
    const Test1dDensity dens;
    const auto a = estimate_covariance(g, dens, Algorithm::one_fft_overwrite, 3000, MultiIndex{8}, 9, 1);
    const auto b = estimate_covariance(g, dens, Algorithm::one_fft_overwrite, 3000, MultiIndex{8}, 9, 4);
    const auto c = estimate_covariance(g, dens, Algorithm::one_fft_overwrite, 3000, MultiIndex{8}, 9, 7);
    CHECK(a.estimates == b.estimates && a.estimates == c.estimates);
    CHECK(throws<std::invalid_argument>(
        [&] { estimate_covariance(g, dens, Algorithm::two_fft, 0, MultiIndex{0}, 1); }));
    CHECK(throws<std::invalid_argument>(
        [&] { estimate_covariance(g, dens, Algorithm::two_fft, 10, MultiIndex{16}, 1); }));
  });

  run("max_error and slope fitting (test_stats.cpp:58-91)", [] {
    const GridSpec g({1.0}, {4});
    CovarianceEstimate e{g, {0}, {1.0, 2.0, 3.0, 4.0}, 1, 0};
    const auto lin = [](std::span<const double> x) { return 10.0 * x[0]; };
    CHECK(near(max_error(e, lin), 3.5, 1e-12));
    const auto same = [&](std::span<const double> x) { return e.estimates[static_cast<std::size_t>(std::lround(x[0] * 4.0))]; };
    CHECK(max_error(e, same) == 0.0);
    const std::vector<double> x{2.0, 3.0, 4.0, 5.0};
    std::vector<double> y;
    for (double v : x) y.push_back(-4.0 * v);
    const auto s = fit_slope(x, y);
    CHECK(s.has_value() && near(*s, -4.0, 1e-12));
    CHECK(!fit_slope(std::vector<double>{1.0}, std::vector<double>{2.0}).has_value());
    CHECK(!fit_slope(std::vector<double>{1.0, 1.0}, std::vector<double>{1.0, 2.0}).has_value());
  });

  run("convergence study basics (test_stats.cpp:93-123)", [] {
    CHECK(throws<std::invalid_argument>([] { convergence_study(1, 4, 100, Algorithm::two_fft, 0); }));
    CHECK(throws<std::invalid_argument>([] { convergence_study(2, 13, 100, Algorithm::two_fft, 0); }));
    CHECK(throws<std::invalid_argument>([] { convergence_study(5, 3, 100, Algorithm::two_fft, 0); }));
    const ConvergenceReport one = convergence_study(2, 2, 400, Algorithm::one_fft_recursive, 12);
    CHECK(one.rows.size() == 1 && one.rows[0].level == 2 && one.rows[0].cells == 4);
    CHECK(near(one.rows[0].mc_floor, 0.1, 1e-12));
    CHECK(!one.fitted_slope.has_value());
    const ConvergenceReport r = convergence_study(2, 4, 10000, Algorithm::one_fft_recursive, 12);
    CHECK(r.rows.size() == 3);
    CHECK(r.rows[0].max_err > r.rows[1].max_err && r.rows[1].max_err > r.rows[2].max_err);
    CHECK(std::abs(r.rows[0].max_err - 0.615) < 0.15 * 0.615);
    CHECK(std::abs(r.rows[1].max_err - 0.328) < 0.2 * 0.328);
    CHECK(std::abs(r.rows[2].max_err - 0.073) < 0.8 * 0.073);
    CHECK(r.fitted_slope.has_value() && r.fitted_levels.size() == 3);
  });

  run("GRF1 round trip, header, corrupt files (test_field_io.cpp:41-92)", [] {
    const auto tmp = std::filesystem::temp_directory_path() / ("grf_dropin_" + std::to_string(::getpid()));
    const auto slurp = [](const std::filesystem::path& p) {
      std::ifstream is(p, std::ios::binary);
      std::ostringstream os;
      os << is.rdbuf();
      return os.str();
    };
    const auto spit = [](const std::filesystem::path& p, const std::string& b) {
      std::ofstream os(p, std::ios::binary | std::ios::trunc);
      os.write(b.data(), static_cast<std::streamsize>(b.size()));
    };
    const GridSpec grid({1.5, 2.0}, {4, 6});
    const RealField field = synthesize(grid, PolyDecayDensity(1.0, 1, 1, 2, 2), 11, Algorithm::one_fft_recursive);
    write_grf1(tmp, field);
    const RealField back = read_grf1(tmp);
    CHECK(back.grid.counts() == grid.counts() && back.grid.lengths() == grid.lengths());
    CHECK(back.values.size() == field.values.size() &&
          std::memcmp(back.values.data(), field.values.data(), 8 * field.values.size()) == 0);
    write_grf1(tmp, RealField{GridSpec({1.0}, {2}), {0.5, -0.25}, {}, 0.0});
    const std::string h = slurp(tmp);
    CHECK(h.size() == 4 + 4 + 4 + 8 + 8 + 16 && h.substr(0, 4) == "GRF1" && h[4] == 1 && h[8] == 1 &&
          static_cast<unsigned char>(h[12]) == 2);
    write_grf1(tmp, RealField{GridSpec({1.0}, {4}), {1.0, 2.0, 3.0, 4.0}, {}, 0.0});
    const std::string good = slurp(tmp);
    spit(tmp, "GRG1" + good.substr(4));
    bool magic = false;
    try {
      read_grf1(tmp);
    } catch (const std::runtime_error& e) {
      magic = std::string(e.what()) == "read_grf1: bad magic";
    }
    CHECK(magic);
    std::string v2 = good;
    v2[4] = 2;
    spit(tmp, v2);
    CHECK(throws<std::runtime_error>([&] { read_grf1(tmp); }));
    spit(tmp, good.substr(0, good.size() - 3));
    CHECK(throws<std::runtime_error>([&] { read_grf1(tmp); }));
    spit(tmp, good + "x");
    CHECK(throws<std::runtime_error>([&] { read_grf1(tmp); }));
    CHECK(throws<std::runtime_error>([] { read_grf1("/nonexistent/grf1"); }));
    // device batch writer: bit-exact with the same fields through RealField
    const auto fmt = tmp.string() + "_{field}.grf1";
    write_grf1_batch(grid, MaternDensity(1.5, 0.2, 2), 4, 10, 3, Algorithm::one_fft_overwrite, fmt);
    const auto fields = synthesize_batch(grid, MaternDensity(1.5, 0.2, 2), 4, 10, 3, Algorithm::one_fft_overwrite);
    for (int i = 0; i < 3; ++i) {
      const auto p = tmp.string() + "_" + std::to_string(10 + i) + ".grf1";
      CHECK(read_grf1(p).values == fields[static_cast<std::size_t>(i)].values);
      std::filesystem::remove(p);
    }
    std::filesystem::remove(tmp);
  });

  run("PGM bytes and CSV dump (test_field_io.cpp:94-140)", [] {
    const auto tmp = std::filesystem::temp_directory_path() / ("grf_pgm_" + std::to_string(::getpid()));
    const GridSpec g({1.0, 1.0}, {2, 4});
    write_field_pgm(tmp, RealField{g, {0, 1, 2, 3, 4, 5, 6, 7}, {}, 0.0});
    std::ifstream is(tmp, std::ios::binary);
    const std::string b((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    const std::string hdr = "P5\n4 2\n255\n";
    const unsigned char want[8] = {0, 36, 73, 109, 146, 182, 219, 255};
    bool ok = b.size() == hdr.size() + 8 && b.substr(0, hdr.size()) == hdr;
    for (int i = 0; ok && i < 8; ++i) ok = static_cast<unsigned char>(b[hdr.size() + i]) == want[i];
    CHECK(ok);
    write_field_pgm(tmp, RealField{g, std::vector<double>(8, 3.0), {}, 0.0});
    std::ifstream is2(tmp, std::ios::binary);
    const std::string flat((std::istreambuf_iterator<char>(is2)), std::istreambuf_iterator<char>());
    CHECK(flat.size() == hdr.size() + 8 && flat.substr(hdr.size()) == std::string(8, '\0'));
    CHECK(throws<std::invalid_argument>([&] { write_field_pgm(tmp, RealField{GridSpec({1.0}, {4}), {1, 2, 3, 4}, {}, 0.0}); }));
    std::filesystem::remove(tmp);
    std::ostringstream os;
    write_field_csv(os, RealField{GridSpec({1.0, 2.0}, {2, 2}, {0.0, 1.0}), {1.0, 2.0, 3.0, 4.5}, {}, 0.0});
    std::istringstream in(os.str());
    std::string line;
    std::getline(in, line);
    CHECK(line == "x1,x2,value");
    int rows = 0;
    bool commas = true;
    while (std::getline(in, line)) ++rows, commas = commas && std::count(line.begin(), line.end(), ',') == 2;
    CHECK(rows == 4 && commas && os.str().find("4.5") != std::string::npos);
  });

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail;
}
