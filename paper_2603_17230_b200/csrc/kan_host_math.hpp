// kan_host_math.hpp -- host-side table construction for the engine.
//
// The engine builds its lookup tables once at configure time on the host, in
// fp64 with the reference's operation order, so the device-side integer path
// reproduces the reference's quantized quantities exactly:
//   GridSpec (grid.hpp:27-96), Cox-de Boor triangle (grid.hpp:124-172),
//   compute_quant_params / quantize_value (quant.hpp:33-54),
//   ActivationLattice (lut.hpp:21-56), build_bspline_lut (lut.hpp:103-131),
//   lut_basis_lookup (lut.hpp:136-160).
// Compiled with -ffp-contract=off (see __graft_entry__.py) so no FMA fusing
// changes a rounding.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace kan {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ShapeMismatch : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Grid {
  int G = 0, P = 0;
  double lo = -1.0, hi = 1.0, delta = 0.0;
  int nb() const { return G + P; }
  static Grid build(int G, int P, double lo, double hi) {
    if (G < 1) throw InvalidArgument("build_grid: intervals must be >= 1");
    if (P < 0) throw InvalidArgument("build_grid: degree must be >= 0");
    if (!(hi > lo)) throw InvalidArgument("build_grid: degenerate domain");
    Grid g;
    g.G = G;
    g.P = P;
    g.lo = lo;
    g.hi = hi;
    g.delta = (hi - lo) / G;
    return g;
  }
  double knot_coord(double x) const { return (x - lo) / delta + P; }
  double hi_open() const { return std::nextafter(hi, lo); }
  double clamp(double x) const {
    const double ho = hi_open();
    const double t = (x < lo) ? lo : x;
    x = (ho < t) ? ho : t;
    if (P == 0)
      while (x > lo && knot_coord(x) >= static_cast<double>(G + 2 * P)) x = std::nextafter(x, lo);
    return x;
  }
  // dense degree-P basis at knot coordinate xi (grid.hpp:124-172)
  int basis_at_coord(double xi, double* out) const {
    const int n0 = G + 2 * P;
    std::vector<double> buf(static_cast<size_t>(n0) + 1, 0.0);
    const double jf = std::floor(xi);
    if (jf >= 0.0 && jf < static_cast<double>(n0)) buf[static_cast<size_t>(jf)] = 1.0;
    for (int d = 1; d <= P; ++d) {
      const double r = 1.0 / d;
      for (int i = 0; i <= n0 - d; ++i) {
        const double d1 = xi - i;
        const double d2 = static_cast<double>(i + d + 1) - xi;
        buf[i] = (d1 * r) * buf[i] + (d2 * r) * buf[i + 1];
      }
    }
    for (int i = 0; i < nb(); ++i) out[i] = buf[i];
    if (jf < 0.0 || jf >= static_cast<double>(n0)) return 0;
    int j = static_cast<int>(jf) - P;
    return j < 0 ? 0 : (j > nb() - 1 ? nb() - 1 : j);
  }
};

struct QParams {
  double scale = 1.0;
  int64_t zp = 0;
  int64_t qhi = 0;
};

inline QParams quant_params(double alpha, double beta, int bits) {
  if (bits < 1 || bits > 8)
    throw InvalidArgument("compute_quant_params: bits must be in [1,8] or 32");
  if (!(beta > alpha)) throw InvalidArgument("compute_quant_params: degenerate range");
  QParams q;
  q.qhi = (int64_t{1} << bits) - 1;
  q.scale = (beta - alpha) / static_cast<double>(q.qhi);
  q.zp = std::llround((beta * 0.0 - alpha * static_cast<double>(q.qhi)) / (beta - alpha));
  return q;
}

inline int64_t quantize(double x, const QParams& q) {
  int64_t v = std::llround(x / q.scale + static_cast<double>(q.zp));
  return v < 0 ? 0 : (v > q.qhi ? q.qhi : v);
}

struct Lattice {
  int k = 0;
  int64_t L = 0;
  double lo = 0.0, step = 0.0;
  static Lattice of(const Grid& g, int k) {
    if (k < 1 || k > 8) throw InvalidArgument("ActivationLattice: bits per interval must be in [1,8]");
    Lattice l;
    l.k = k;
    l.L = static_cast<int64_t>(g.G) << k;
    l.lo = g.lo;
    l.step = std::ldexp(g.delta, -k);
    return l;
  }
  int64_t quantize(double x) const {
    int64_t a = std::llround((x - lo) / step);
    return a < 0 ? 0 : (a > L ? L : a);
  }
  double dequantize(int64_t a) const { return lo + static_cast<double>(a) * step; }
};

inline std::vector<uint8_t> build_lut(int P, int k, int h) {
  if (P < 1) throw InvalidArgument("build_bspline_lut: degree must be >= 1");
  if (k < 1 || k > 8) throw InvalidArgument("build_bspline_lut: k must be in [1,8]");
  if (h < 2 || h > 8) throw InvalidArgument("build_bspline_lut: h must be in [2,8]");
  const QParams vq = quant_params(0.0, 1.0, h);
  const Grid canon = Grid::build(1, P, 0.0, 1.0);
  std::vector<double> basis(static_cast<size_t>(canon.nb()));
  const int64_t half = (P + 2) / 2;
  const int64_t stored = half * (int64_t{1} << k) + 1;
  const int64_t fold = static_cast<int64_t>(P + 1) << (k - 1);
  std::vector<uint8_t> e(static_cast<size_t>(stored));
  for (int64_t m = 0; m < stored; ++m) {
    const int64_t pos = m < fold ? m : fold;
    canon.basis_at_coord(P + std::ldexp(static_cast<double>(pos), -k), basis.data());
    e[static_cast<size_t>(m)] = static_cast<uint8_t>(quantize(basis[P], vq));
  }
  e[0] = 0;
  return e;
}

// lut_basis_lookup: values of the supported bases, packed little-endian in a
// u32 (byte r = basis support_start + r); bytes beyond `count` are zero.
inline uint32_t lut_pack(const Grid& g, int k, const std::vector<uint8_t>& lut, int64_t a) {
  const int64_t jj = a >> k, frac = a - (jj << k);
  const int64_t fold = static_cast<int64_t>(g.P + 1) << (k - 1);
  const int64_t support = static_cast<int64_t>(g.P + 1) << k;
  uint32_t v = 0;
  for (int r = 0; r <= g.P; ++r) {
    if (jj + r >= g.nb()) break;
    const int64_t m = (static_cast<int64_t>(g.P - r) << k) + frac;
    const int64_t f = m > fold ? support - m : m;
    v |= static_cast<uint32_t>(lut[static_cast<size_t>(f)]) << (8 * r);
  }
  return v;
}

inline int64_t level_of(const Grid& g, const Lattice& lat, double x) {
  return lat.quantize(g.clamp(x));
}

// thr[n] = smallest fp32 x whose level is >= n (n = 1..L); thr[0] = -inf,
// thr[L+1] = NaN.  The level is monotone in x, so a bisection over the
// ordered fp32 bit patterns finds every step exactly.
inline std::vector<float> level_thresholds(const Grid& g, const Lattice& lat) {
  auto key_to_float = [](int64_t key) {
    // monotone map: key in [-(2^31-1) .. 2^31-1] over finite+inf floats
    uint32_t bits = key >= 0 ? static_cast<uint32_t>(key)
                             : (static_cast<uint32_t>(-key) | 0x80000000u);
    float f;
    std::memcpy(&f, &bits, 4);
    return f;
  };
  const int64_t kmin = -static_cast<int64_t>(0x7F800000u), kmax = 0x7F800000;  // -inf..+inf
  std::vector<float> thr(static_cast<size_t>(lat.L) + 2);
  thr[0] = -INFINITY;
  thr[static_cast<size_t>(lat.L) + 1] = NAN;
  for (int64_t n = 1; n <= lat.L; ++n) {
    int64_t lo = kmin, hi = kmax;  // level(key_to_float(hi)) >= n holds at +inf
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (level_of(g, lat, static_cast<double>(key_to_float(mid))) >= n)
        hi = mid;
      else
        lo = mid + 1;
    }
    thr[static_cast<size_t>(n)] = key_to_float(lo);
  }
  return thr;
}

// Spline-table input levels (spline_table.hpp:98, quantize_value on the grid
// bounds, no domain clamp): thr[n] = smallest fp32 x with level >= n for
// n = 1..qhi, thr[0] = -inf; the same bisection over ordered fp32 patterns.
// thr[qhi+1] = ovf, the smallest fp32 x with x/s + z >= 2^63: there (and at
// NaN) the reference's llround overflows to LLONG_MIN, which clamps to level 0
// on its x86-64 build, so the level is 0 for x >= ovf.
inline std::vector<float> quant_thresholds(const QParams& q) {
  auto key_to_float = [](int64_t key) {
    uint32_t bits = key >= 0 ? static_cast<uint32_t>(key)
                             : (static_cast<uint32_t>(-key) | 0x80000000u);
    float f;
    std::memcpy(&f, &bits, 4);
    return f;
  };
  const int64_t kmin = -static_cast<int64_t>(0x7F800000u);
  auto overflows = [&](float f) {
    return !(static_cast<double>(f) / q.scale + static_cast<double>(q.zp) < 9223372036854775808.0);
  };
  int64_t ovf = 0, top = 0x7F800000;  // smallest key that overflows (+inf does)
  while (ovf < top) {
    const int64_t mid = ovf + (top - ovf) / 2;
    if (overflows(key_to_float(mid)))
      top = mid;
    else
      ovf = mid + 1;
  }
  const int64_t kmax = ovf - 1;  // quantize is monotone below the overflow
  std::vector<float> thr(static_cast<size_t>(q.qhi) + 2);
  thr[0] = -INFINITY;
  thr[static_cast<size_t>(q.qhi) + 1] = key_to_float(ovf);
  for (int64_t n = 1; n <= q.qhi; ++n) {
    int64_t lo = kmin, hi = kmax;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (quantize(static_cast<double>(key_to_float(mid)), q) >= n)
        hi = mid;
      else
        lo = mid + 1;
    }
    thr[static_cast<size_t>(n)] = key_to_float(lo);
  }
  return thr;
}

}  // namespace kan
