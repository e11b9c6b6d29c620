// Reference-style caller of the B200 engine through include/mssz_b200.hpp:
// the same shape as the reference's run_fix (tools/mssz.cpp:197-232) and the
// end-to-end KAT of test_edit_engine.cpp:198-230 (postconditions from scratch).
// Exit 0 on success, the ErrKind code on an mssz_b200::Error, 1 on a failed check.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "mssz_b200.hpp"

int main() {
  try {
    const std::uint64_t dims[] = {48, 40, 12};
    auto topo = mssz_b200::build_topology(dims);
    std::vector<float> f(topo.vertex_count), fh(topo.vertex_count);
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (std::uint64_t v = 0; v < topo.vertex_count; ++v) {
      const double x = double(v % 48) / 47, y = double((v / 48) % 40) / 39, z = double(v / 1920) / 11;
      f[v] = float(std::sin(6.0 * x) * std::cos(5.0 * y) + 0.3 * z + 0.05 * u(rng));
    }
    const double xi = 0.02;
    for (std::uint64_t v = 0; v < topo.vertex_count; ++v)  // a quantiser-like perturbation
      fh[v] = float(std::round(double(f[v]) / (2 * xi)) * (2 * xi));
    for (std::uint64_t v = 0; v < topo.vertex_count; ++v)
      if (std::abs(double(f[v]) - double(fh[v])) > xi) fh[v] = f[v];
    mssz_b200::DeriveOptions<float> opts;
    mssz_b200::EditStats stats;
    auto edits = mssz_b200::derive_edits(topo, f.data(), fh.data(), xi, opts, &stats);
    auto g = mssz_b200::apply_edits(topo, fh.data(), edits);
    auto lf = mssz_b200::compute_labels(topo, mssz_b200::compute_directions(topo, f.data()));
    auto lg = mssz_b200::compute_labels(topo, mssz_b200::compute_directions(topo, g.data()));
    if (!(lf == lg)) {
      std::fprintf(stderr, "labels differ after correction\n");
      return 1;
    }
    for (std::uint64_t v = 0; v < topo.vertex_count; ++v)
      if (std::abs(double(f[v]) - double(g[v])) > xi) {
        std::fprintf(stderr, "bound violated at %llu\n", (unsigned long long)v);
        return 1;
      }
    std::printf("ok edits=%llu sub_iterations=%llu r_iterations=%llu\n",
                (unsigned long long)edits.size(), (unsigned long long)stats.sub_iterations_total(),
                (unsigned long long)stats.r_iterations);
    return 0;
  } catch (const mssz_b200::Error& e) {
    std::fprintf(stderr, "mssz_b200::Error(%d): %s\n", e.exit_code(), e.what());
    return e.exit_code();
  }
}
