// Reference-style caller of the B200 engine through include/mssz_b200.hpp:
// the same shape as the reference's run_fix (tools/mssz.cpp:197-232) and the
// end-to-end KAT of test_edit_engine.cpp:198-230 (postconditions from scratch).
// Exit 0 on success, the ErrKind code on an mssz_b200::Error, 1 on a failed check.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <random>
#include <span>
#include <vector>

#include "mssz_b200.hpp"

static bool write_file(const std::string& path, const void* p, size_t n) {
  FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) return false;
  const bool ok = std::fwrite(p, 1, n, fp) == n;
  return std::fclose(fp) == 0 && ok;
}

// argv[1] (optional): directory receiving the edit set and its encoded payload,
// so the test can compare the payload with the reference encoder byte for byte.
int main(int argc, char** argv) {
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
    // run_compress (tools/mssz.cpp:150-195): base codec first, then the correction.
    auto base = mssz_b200::compress_base(topo, f.data(), xi);
    fh = base.reconstruction;
    for (std::uint64_t v = 0; v < topo.vertex_count; ++v)
      if (std::abs(double(f[v]) - double(fh[v])) > xi) {
        std::fprintf(stderr, "base codec bound violated at %llu\n", (unsigned long long)v);
        return 1;
      }
    auto back = mssz_b200::decompress_base<float>(topo, base.symbols, base.literals, xi);
    if (std::memcmp(back.data(), fh.data(), fh.size() * sizeof(float)) != 0) {
      std::fprintf(stderr, "decompress_base differs from the compressor's reconstruction\n");
      return 1;
    }
    auto before = mssz_b200::build_report(topo, f.data(), fh.data(), xi);
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
    if (!(mssz_b200::segmentation(topo, g.data()) == lg)) {
      std::fprintf(stderr, "segmentation() differs from compute_labels(compute_directions())\n");
      return 1;
    }
    auto payload = mssz_b200::encode_edits(edits, mssz_b200::BackendCodec::deflate);
    std::uint64_t head = 0;
    if (payload.size() < 16 || (std::memcpy(&head, payload.data(), 8), head != edits.size())) {
      std::fprintf(stderr, "encode_edits header does not carry the edit count\n");
      return 1;
    }
    auto after = mssz_b200::build_report(topo, f.data(), g.data(), xi, edits.size(),
                                         payload.size() + base.literals.size() * sizeof(float));
    if (!mssz_b200::verified(after) || after.fp_max + after.fp_min + after.fn_max + after.fn_min) {
      std::fprintf(stderr, "report after correction: distortion %g violations %llu\n",
                   after.mss_distortion, (unsigned long long)after.bound_violations);
      return 1;
    }
    if (edits.size() && mssz_b200::verified(before)) {
      std::fprintf(stderr, "edits derived although the base reconstruction already verified\n");
      return 1;
    }
    // an exception thrown by on_batch propagates out of derive_edits, as in the
    // reference (edit_engine.cpp:275 calls the std::function inside the loop)
    {
      struct Stop {};
      int calls = 0;
      mssz_b200::DeriveOptions<float> o2;
      o2.on_batch = [&](std::span<const float>) {
        if (++calls == 3) throw Stop{};
      };
      bool propagated = false;
      try {
        mssz_b200::derive_edits(topo, f.data(), fh.data(), xi, o2);
      } catch (const Stop&) {
        propagated = true;
      }
      if (!propagated || calls != 3) {
        std::fprintf(stderr, "on_batch exception did not propagate (calls=%d)\n", calls);
        return 1;
      }
    }
    if (argc > 1) {
      const std::string dir = argv[1];
      if (!write_file(dir + "/indices.u64", edits.indices.data(), edits.size() * 8) ||
          !write_file(dir + "/values.f32", edits.values.data(), edits.size() * 4) ||
          !write_file(dir + "/payload.bin", payload.data(), payload.size())) {
        std::fprintf(stderr, "cannot write to %s\n", dir.c_str());
        return 1;
      }
    }
    std::printf("ok edits=%llu sub_iterations=%llu r_iterations=%llu distortion_before=%g "
                "payload=%zu\n",
                (unsigned long long)edits.size(), (unsigned long long)stats.sub_iterations_total(),
                (unsigned long long)stats.r_iterations, before.mss_distortion, payload.size());
    return 0;
  } catch (const mssz_b200::Error& e) {
    std::fprintf(stderr, "mssz_b200::Error(%d): %s\n", e.exit_code(), e.what());
    return e.exit_code();
  }
}
