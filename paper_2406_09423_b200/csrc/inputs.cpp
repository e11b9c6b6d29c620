// Host-side producers of the correction loop's inputs:
//   * the reference's deterministic synthetic fields (field.cpp:126-250),
//   * resolve_bound's value range (field.cpp:31-50),
//   * the base codec's reconstruction f̂ (base_codec.cpp:26-120, payload omitted),
// restated bit-exactly (same RNG draws, same double-precision operation order,
// built with -ffp-contract=off like the reference, core/CMakeLists.txt:21-23)
// but parallel: per-vertex evaluation with OpenMP, and the Lorenzo quantiser as
// a block wavefront (a vertex only depends on neighbours with smaller or equal
// coordinates on every axis, so blocks on one anti-diagonal are independent).
// tests/test_inputs.py pins every function against the reference library.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace {

struct Topo {
  int ndims;
  uint64_t d[3];
  uint64_t n;
};

bool make_topo(int ndims, const uint64_t* dims, Topo& t) {
  if (ndims != 2 && ndims != 3) return false;
  t.ndims = ndims;
  t.d[0] = t.d[1] = t.d[2] = 1;
  t.n = 1;
  for (int a = 0; a < ndims; ++a) {
    if (dims[a] < 2) return false;
    t.d[a] = dims[a];
    t.n *= dims[a];
  }
  return true;
}

// field.cpp:128-134
double next_unit(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
double next_in(std::mt19937_64& rng, double lo, double hi) { return lo + (hi - lo) * next_unit(rng); }

// field.cpp:136-172
void gaussian_mixture(const Topo& t, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  const int k = 5 + static_cast<int>(seed % 6);
  struct Bump {
    double c[3];
    double inv2s2;
    double amp;
  };
  std::vector<Bump> bumps(k);
  const double min_extent =
      static_cast<double>(std::min({t.d[0], t.d[1], t.ndims == 3 ? t.d[2] : t.d[1]}));
  for (auto& b : bumps) {
    for (int a = 0; a < 3; ++a) {
      const double extent = static_cast<double>(t.d[a]);
      b.c[a] = (t.ndims == 2 && a == 2) ? 0.0 : next_in(rng, 0.15, 0.85) * (extent - 1);
    }
    const double sigma = next_in(rng, 0.08, 0.25) * min_extent;
    b.inv2s2 = 1.0 / (2.0 * sigma * sigma);
    const double amp = next_in(rng, 0.4, 1.2);
    b.amp = (next_unit(rng) < 0.25) ? -amp : amp;
  }
  const uint64_t X = t.d[0], Y = t.d[1];
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < static_cast<int64_t>(t.n / X); ++row) {
    const uint64_t y = static_cast<uint64_t>(row) % Y, z = static_cast<uint64_t>(row) / Y;
    for (uint64_t x = 0; x < X; ++x) {
      const double c[3] = {static_cast<double>(x), static_cast<double>(y), static_cast<double>(z)};
      double sum = 0.0;
      for (const auto& b : bumps) {
        double d2 = 0.0;
        for (int a = 0; a < t.ndims; ++a) {
          const double dd = c[a] - b.c[a];
          d2 += dd * dd;
        }
        sum += b.amp * std::exp(-d2 * b.inv2s2);
      }
      out[static_cast<uint64_t>(row) * X + x] = sum;
    }
  }
}

// field.cpp:174-194
void trig(const Topo& t, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  const double two_pi = 6.283185307179586476925286766559;
  double freq[3], phase[3];
  for (int a = 0; a < 3; ++a) {
    freq[a] = 1.5 + 0.7 * static_cast<double>(seed % 5) + 0.3 * next_unit(rng);
    phase[a] = two_pi * next_unit(rng);
  }
  const uint64_t X = t.d[0], Y = t.d[1];
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < static_cast<int64_t>(t.n / X); ++row) {
    const uint64_t y = static_cast<uint64_t>(row) % Y, z = static_cast<uint64_t>(row) / Y;
    for (uint64_t x = 0; x < X; ++x) {
      const uint64_t c[3] = {x, y, z};
      double prod = 1.0;
      for (int a = 0; a < t.ndims; ++a) {
        const double xx = static_cast<double>(c[a]) / static_cast<double>(t.d[a] - 1);
        const double arg = two_pi * freq[a] * xx + phase[a];
        prod *= (a % 2 == 0) ? std::sin(arg) : std::cos(arg);
      }
      out[static_cast<uint64_t>(row) * X + x] = prod;
    }
  }
}

// field.cpp:196-225
void random_smooth(const Topo& t, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  for (uint64_t v = 0; v < t.n; ++v) out[v] = next_in(rng, -1.0, 1.0);
  std::vector<double> tmp(t.n);
  double* src = out;
  double* dst = tmp.data();
  for (int pass = 0; pass < 3; ++pass) {
    for (int axis = 0; axis < t.ndims; ++axis) {
      uint64_t stride = 1;
      for (int a = 0; a < axis; ++a) stride *= t.d[a];
      const uint64_t X = t.d[0], Y = t.d[1];
#pragma omp parallel for schedule(static)
      for (int64_t row = 0; row < static_cast<int64_t>(t.n / X); ++row) {
        const uint64_t y = static_cast<uint64_t>(row) % Y, z = static_cast<uint64_t>(row) / Y;
        for (uint64_t x = 0; x < X; ++x) {
          const uint64_t v = static_cast<uint64_t>(row) * X + x;
          const uint64_t c = axis == 0 ? x : (axis == 1 ? y : z);
          double sum = src[v];
          int cnt = 1;
          if (c > 0) {
            sum += src[v - stride];
            ++cnt;
          }
          if (c + 1 < t.d[axis]) {
            sum += src[v + stride];
            ++cnt;
          }
          dst[v] = sum / cnt;
        }
      }
      std::swap(src, dst);
    }
  }
  if (src != out) std::copy(src, src + t.n, out);
}

void generate_double(int kind, const Topo& t, uint64_t seed, double* out) {
  switch (kind) {
    case 0: gaussian_mixture(t, seed, out); break;
    case 1: trig(t, seed, out); break;
    default: random_smooth(t, seed, out); break;
  }
}

template <class T>
int generate(int kind, int ndims, const uint64_t* dims, uint64_t seed, double a, T* out) {
  Topo t;
  if (!make_topo(ndims, dims, t) || kind < 0 || kind > 3) return 2;
  std::vector<double> v(t.n);
  if (kind == 3) {
    // multi-scale: gaussian_mixture(seed) + a * random_smooth(seed + 1),
    // summed in double, then narrowed
    generate_double(0, t, seed, v.data());
    std::vector<double> r(t.n);
    generate_double(2, t, seed + 1, r.data());
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < static_cast<int64_t>(t.n); ++i) v[i] = v[i] + a * r[i];
  } else {
    generate_double(kind, t, seed, v.data());
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(t.n); ++i) out[i] = static_cast<T>(v[i]);
  return 0;
}

// field.cpp:31-40
template <class T>
void value_range(uint64_t n, const T* values, double* lo, double* hi) {
  double l = static_cast<double>(values[0]), h = l;
#pragma omp parallel for reduction(min : l) reduction(max : h) schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(n); ++i) {
    const double d = static_cast<double>(values[i]);
    l = std::min(l, d);
    h = std::max(h, d);
  }
  *lo = l;
  *hi = h;
}

constexpr int64_t kQuantRadius = 32766;  // base_codec.cpp:13

// one vertex of compress_base (base_codec.cpp:87-113): Lorenzo prediction from
// the reconstruction (:26-49), 2xi quantisation, escape to the literal value
template <class T>
inline bool quantise_vertex(const Topo& t, const T* values, T* recon, uint64_t v, uint64_t x,
                            uint64_t y, uint64_t z, double xi, double two_xi) {
  const double f = static_cast<double>(values[v]);
  const uint64_t sx = 1, sy = t.d[0], sz = t.d[0] * t.d[1];
  const bool hx = x > 0, hy = y > 0;
  auto at = [&](uint64_t off) { return static_cast<double>(recon[v - off]); };
  double p = 0.0;
  if (t.ndims == 2) {
    if (hx) p += at(sx);
    if (hy) p += at(sy);
    if (hx && hy) p -= at(sx + sy);
  } else {
    const bool hz = z > 0;
    if (hx) p += at(sx);
    if (hy) p += at(sy);
    if (hz) p += at(sz);
    if (hx && hy) p -= at(sx + sy);
    if (hy && hz) p -= at(sy + sz);
    if (hx && hz) p -= at(sx + sz);
    if (hx && hy && hz) p += at(sx + sy + sz);
  }
  const double residual_steps = (f - p) / two_xi;
  int64_t q = 0;
  bool escape = !(std::fabs(residual_steps) <= static_cast<double>(kQuantRadius) + 1.0);
  if (!escape) {
    q = std::llround(residual_steps);
    escape = std::llabs(q) > kQuantRadius;
  }
  T r{};
  if (!escape) {
    r = static_cast<T>(p + two_xi * static_cast<double>(q));
    escape = !(std::abs(f - static_cast<double>(r)) <= xi) || !std::isfinite(static_cast<double>(r));
  }
  recon[v] = escape ? values[v] : r;
  return escape;
}

template <class T>
int compress_base_recon(int ndims, const uint64_t* dims, const T* values, double xi, T* recon,
                        uint64_t* escapes_out) {
  Topo t;
  if (!make_topo(ndims, dims, t)) return 2;
  if (!(xi > 0.0)) return 2;
  for (uint64_t i = 0; i < t.n; ++i)
    if (!std::isfinite(static_cast<double>(values[i]))) return 3;
  const double two_xi = 2.0 * xi;
  const uint64_t B[3] = {64, 16, t.ndims == 3 ? 16u : 1u};
  const uint64_t nb[3] = {(t.d[0] + B[0] - 1) / B[0], (t.d[1] + B[1] - 1) / B[1],
                          (t.d[2] + B[2] - 1) / B[2]};
  uint64_t escapes = 0;
  for (uint64_t diag = 0; diag < nb[0] + nb[1] + nb[2] - 2; ++diag) {
    // blocks (i,j,k) with i+j+k == diag are independent
    std::vector<uint64_t> blocks;
    for (uint64_t k = 0; k < nb[2] && k <= diag; ++k)
      for (uint64_t j = 0; j < nb[1] && j + k <= diag; ++j) {
        const uint64_t i = diag - j - k;
        if (i < nb[0]) blocks.push_back(i | (j << 21) | (k << 42));
      }
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : escapes)
    for (int64_t bi = 0; bi < static_cast<int64_t>(blocks.size()); ++bi) {
      const uint64_t i = blocks[bi] & 0x1FFFFF, j = (blocks[bi] >> 21) & 0x1FFFFF,
                     k = blocks[bi] >> 42;
      const uint64_t x0 = i * B[0], y0 = j * B[1], z0 = k * B[2];
      const uint64_t x1 = std::min(x0 + B[0], t.d[0]), y1 = std::min(y0 + B[1], t.d[1]),
                     z1 = std::min(z0 + B[2], t.d[2]);
      for (uint64_t z = z0; z < z1; ++z)
        for (uint64_t y = y0; y < y1; ++y)
          for (uint64_t x = x0; x < x1; ++x) {
            const uint64_t v = x + t.d[0] * (y + t.d[1] * z);
            escapes += quantise_vertex(t, values, recon, v, x, y, z, xi, two_xi) ? 1 : 0;
          }
    }
  }
  if (escapes_out) *escapes_out = escapes;
  return 0;
}

}  // namespace

extern "C" {

int mssz_in_generate_f32(int kind, int ndims, const uint64_t* dims, uint64_t seed, double a, float* out) {
  return generate<float>(kind, ndims, dims, seed, a, out);
}
int mssz_in_generate_f64(int kind, int ndims, const uint64_t* dims, uint64_t seed, double a, double* out) {
  return generate<double>(kind, ndims, dims, seed, a, out);
}
void mssz_in_value_range_f32(uint64_t n, const float* v, double* lo, double* hi) { value_range(n, v, lo, hi); }
void mssz_in_value_range_f64(uint64_t n, const double* v, double* lo, double* hi) { value_range(n, v, lo, hi); }
int mssz_in_compress_base_recon_f32(int ndims, const uint64_t* dims, const float* v, double xi,
                                    float* recon, uint64_t* escapes) {
  return compress_base_recon<float>(ndims, dims, v, xi, recon, escapes);
}
int mssz_in_compress_base_recon_f64(int ndims, const uint64_t* dims, const double* v, double xi,
                                    double* recon, uint64_t* escapes) {
  return compress_base_recon<double>(ndims, dims, v, xi, recon, escapes);
}

}  // extern "C"
