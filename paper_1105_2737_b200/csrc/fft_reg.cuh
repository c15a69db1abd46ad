// Register-resident small DFTs with compile-time twiddles.
//
//   dft<N, SIGN>(v):  v[q] <- sum_i v[i] exp(SIGN * 2 pi i * i q / N), in place,
//                      natural order, N in {1, 2, 4, 8, 16, 32, 64}.
//
// Twiddle constants are evaluated by constexpr Taylor series (double) and
// multiplications by the trivial angles (multiples of pi/4) are specialised,
// so the SASS holds only the FADD/FMUL/FFMA a hand-written butterfly would.
#pragma once

#include <type_traits>

#include "grfc_internal.cuh"

namespace grfc {

// ---------------------------------------------------------------- constexpr trig
constexpr double kPi = 3.14159265358979323846264338327950288;

constexpr double taylor_sin(double x) {
  double term = x, sum = x;
  for (int n = 1; n < 14; ++n) {
    term *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
    sum += term;
  }
  return sum;
}
constexpr double taylor_cos(double x) {
  double term = 1.0, sum = 1.0;
  for (int n = 1; n < 14; ++n) {
    term *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
    sum += term;
  }
  return sum;
}
// sin/cos of a in [0, pi/2) given as (pi/2) * r / N, via the nearer of a and pi/2 - a.
constexpr double qsin(long r, long N) {
  return (2 * r <= N) ? taylor_sin(0.5 * kPi * r / N) : taylor_cos(0.5 * kPi * (N - r) / N);
}
constexpr double qcos(long r, long N) {
  return (2 * r <= N) ? taylor_cos(0.5 * kPi * r / N) : taylor_sin(0.5 * kPi * (N - r) / N);
}
// cos/sin(2 pi K / N): exact quadrant q and remainder r on the integers
// (2 pi K/N = q pi/2 + (pi/2) r/N).
constexpr double cos_2pi(long K, long N) {
  const long k = ((K % N) + N) % N, q = (4 * k) / N, r = 4 * k - q * N;
  return q == 0 ? qcos(r, N) : q == 1 ? -qsin(r, N) : q == 2 ? -qcos(r, N) : qsin(r, N);
}
constexpr double sin_2pi(long K, long N) {
  const long k = ((K % N) + N) % N, q = (4 * k) / N, r = 4 * k - q * N;
  return q == 0 ? qsin(r, N) : q == 1 ? qcos(r, N) : q == 2 ? -qsin(r, N) : -qcos(r, N);
}

template <int I>
using ic = std::integral_constant<int, I>;

template <int I, int END>
struct Unroll {
  template <class F>
  __device__ __forceinline__ static void run(F&& f) {
    if constexpr (I < END) {
      f(ic<I>{});
      Unroll<I + 1, END>::run(f);
    }
  }
};

// v * exp(SIGN * 2 pi i K / N), K and N compile-time.
template <long K, long N, int SIGN, typename C>
__device__ __forceinline__ C twmul(C v) {
  using R = decltype(C{}.x);
  constexpr long k = ((K % N) + N) % N;
  if constexpr (k == 0) {
    return v;
  } else if constexpr (2 * k == N) {
    return mk<C>(-v.x, -v.y);
  } else if constexpr (4 * k == N) {
    return mul_si<SIGN>(v);
  } else if constexpr (4 * k == 3 * N) {
    return mul_si<-SIGN>(v);
  } else if constexpr ((8 * k) % N == 0) {
    // (c, s) = (+-1/sqrt2, +-1/sqrt2)
    constexpr R h = (R)0.70710678118654752440;
    constexpr R c = (R)(cos_2pi(k, N) > 0 ? 1 : -1) * h;
    constexpr R s = (R)(SIGN * (sin_2pi(k, N) > 0 ? 1 : -1)) * h;
    // (c + i s) v with |c| = |s|: c * (v + i (s/c) v)
    const C t = (c == s) ? mul_si<+1>(v) : mul_si<-1>(v);
    return cscale(cadd(v, t), c);
  } else {
    constexpr R c = (R)cos_2pi(k, N);
    constexpr R s = (R)(SIGN * sin_2pi(k, N));
    return cmul_cs(v, c, s);
  }
}

template <int SIGN, typename C>
__device__ __forceinline__ void bfly2(C& a, C& b) {
  const C t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int SIGN, typename C>
__device__ __forceinline__ void dft4(C& v0, C& v1, C& v2, C& v3) {
  const C t0 = cadd(v0, v2), t1 = csub(v0, v2);
  const C t2 = cadd(v1, v3), t3 = mul_si<SIGN>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}

// Generic N = A * B split (A the outer radix): inputs i = A a + b, outputs
// q = q1 + B q2; y[q1 + B q2] = sum_b w_A^{b q2} (w_N^{b q1} D_b[q1]).
template <int N, int SIGN, typename C>
__device__ __forceinline__ void dft(C* v);

template <int A, int B, int SIGN, typename C>
__device__ __forceinline__ void dft_split(C* v) {
  constexpr int N = A * B;
  C d[A][B];
  Unroll<0, A>::run([&](auto bb) {
    constexpr int b = decltype(bb)::value;
    Unroll<0, B>::run([&](auto aa) {
      constexpr int a = decltype(aa)::value;
      d[b][a] = v[A * a + b];
    });
    dft<B, SIGN>(d[b]);
    Unroll<1, B>::run([&](auto qq) {
      constexpr int q1 = decltype(qq)::value;
      d[b][q1] = twmul<(long)b * q1, N, SIGN>(d[b][q1]);
    });
  });
  Unroll<0, B>::run([&](auto qq) {
    constexpr int q1 = decltype(qq)::value;
    C e[A];
    Unroll<0, A>::run([&](auto bb) {
      constexpr int b = decltype(bb)::value;
      e[b] = d[b][q1];
    });
    dft<A, SIGN>(e);
    Unroll<0, A>::run([&](auto qq2) {
      constexpr int q2 = decltype(qq2)::value;
      v[q1 + B * q2] = e[q2];
    });
  });
}

template <int N, int SIGN, typename C>
__device__ __forceinline__ void dft(C* v) {
  if constexpr (N == 1) {
    return;
  } else if constexpr (N == 2) {
    bfly2<SIGN>(v[0], v[1]);
  } else if constexpr (N == 4) {
    dft4<SIGN>(v[0], v[1], v[2], v[3]);
  } else if constexpr (N == 8) {
    dft_split<2, 4, SIGN>(v);
  } else if constexpr (N == 16) {
    dft_split<4, 4, SIGN>(v);
  } else if constexpr (N == 32) {
    dft_split<4, 8, SIGN>(v);
  } else if constexpr (N == 64) {
    dft_split<8, 8, SIGN>(v);
  } else {
    static_assert(N <= 64, "register DFT supports N <= 64");
  }
}

}  // namespace grfc
