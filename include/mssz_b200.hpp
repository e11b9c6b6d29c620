// mssz_b200.hpp — header-only C++ host binding over the C-ABI (mssz_cuda.h)
// with the reference's proj/core entry-point signatures, so a reference caller
// (tools/mssz.cpp run_compress / run_fix / run_bench) switches by changing the
// namespace it calls:
//
//   reference:  mssz::derive_edits<T>(topo, f, fhat, xi, opts, &stats)
//               (/root/reference/proj/core/include/mssz/edit_engine.hpp:183-186)
//   B200:       mssz_b200::derive_edits<T>(topo, f, fhat, xi, opts, &stats)
//
// Types mirror grid.hpp:25-47 (GridTopology), edit_engine.hpp:45-82 (EditSet,
// EditStats, DeriveOptions), mss.hpp:24-42 (DirectionField, SegmentationLabels)
// and errors.hpp:9-28 (ErrKind, Error); a nonzero C-ABI return becomes the
// same mssz_b200::Error{kind} the reference throws.
#pragma once

#include <array>
#include <cstdint>
#include <exception>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "mssz_cuda.h"

namespace mssz_b200 {

using VertexId = std::uint64_t;

enum class ErrKind : int {
  usage = 2,
  io = 3,
  bound_violation = 4,
  non_convergence = 5,
  corrupt_archive = 6,
  internal = 7,
  cuda = 99,
};

class Error : public std::runtime_error {
 public:
  Error(ErrKind kind, const std::string& msg) : std::runtime_error(msg), kind_(kind) {}
  ErrKind kind() const noexcept { return kind_; }
  int exit_code() const noexcept { return static_cast<int>(kind_); }

 private:
  ErrKind kind_;
};

inline void check(int rc) {
  if (rc != 0) throw Error(static_cast<ErrKind>(rc), mssz_cu_last_error());
}

struct GridTopology {
  int ndims = 0;
  std::array<std::uint64_t, 3> dims{1, 1, 1};
  std::uint64_t vertex_count = 0;
};

// build_topology (grid.cpp:39-55)
inline GridTopology build_topology(std::span<const std::uint64_t> dims) {
  if (dims.size() != 2 && dims.size() != 3)
    throw Error(ErrKind::usage, "dims must have 2 or 3 extents");
  GridTopology t;
  t.ndims = static_cast<int>(dims.size());
  std::uint64_t count = 1;
  for (size_t a = 0; a < dims.size(); ++a) {
    if (dims[a] < 2) throw Error(ErrKind::usage, "every grid extent must be >= 2");
    if (dims[a] > (std::uint64_t(1) << 40) / count)
      throw Error(ErrKind::usage, "grid exceeds the address-space cap");
    t.dims[a] = dims[a];
    count *= dims[a];
  }
  t.vertex_count = count;
  return t;
}

template <class T>
struct EditSet {
  std::vector<VertexId> indices;
  std::vector<T> values;
  std::uint64_t size() const { return indices.size(); }
  bool empty() const { return indices.empty(); }
};

struct EditStats : mssz_cu_stats {
  EditStats() : mssz_cu_stats{} {}
  std::uint64_t sub_iterations_total() const {
    return sub_iterations[0] + sub_iterations[1] + sub_iterations[2] + sub_iterations[3];
  }
};

template <class T>
struct DeriveOptions {
  int device = -1;  // replaces ExecPolicy: which GPU
  std::uint64_t outer_cap = 1000;
  std::uint64_t subloop_cap = 640;
  std::uint64_t r_cap = 100000;
  bool force = false;
  std::function<void(std::span<const T>)> on_batch;
};

struct DirectionField {
  std::vector<VertexId> asc, desc;
  bool is_max(VertexId v) const { return asc[v] == v; }
  bool is_min(VertexId v) const { return desc[v] == v; }
};

struct SegmentationLabels {
  std::vector<VertexId> max_label, min_label;
  bool operator==(const SegmentationLabels&) const = default;
};

namespace detail {
template <class T>
struct Api;
template <>
struct Api<float> {
  static constexpr auto derive = mssz_cu_derive_edits_f32;
  static constexpr auto directions = mssz_cu_compute_directions_f32;
  static constexpr auto apply = mssz_cu_apply_edits_f32;
  static constexpr auto verify = mssz_cu_verify_f32;
  static constexpr auto segmentation = mssz_cu_segmentation_f32;
  static constexpr auto compress_base = mssz_cu_compress_base_f32;
  static constexpr auto decompress_base = mssz_cu_decompress_base_f32;
  static constexpr auto encode_edits = mssz_cu_encode_edits_f32;
};
template <>
struct Api<double> {
  static constexpr auto derive = mssz_cu_derive_edits_f64;
  static constexpr auto directions = mssz_cu_compute_directions_f64;
  static constexpr auto apply = mssz_cu_apply_edits_f64;
  static constexpr auto verify = mssz_cu_verify_f64;
  static constexpr auto segmentation = mssz_cu_segmentation_f64;
  static constexpr auto compress_base = mssz_cu_compress_base_f64;
  static constexpr auto decompress_base = mssz_cu_decompress_base_f64;
  static constexpr auto encode_edits = mssz_cu_encode_edits_f64;
};
// on_batch across the C ABI: an exception thrown by the callback is caught
// here (it must not unwind through extern "C"), the engine is told to abort
// (nonzero), and derive_edits rethrows it -- the reference's exception
// propagation out of derive_edits (edit_engine.cpp:275, :364).
template <class T>
struct BatchCall {
  std::function<void(std::span<const T>)> fn;
  std::exception_ptr error;
};
template <class T>
int batch_trampoline(const void* g, std::uint64_t n, void* user) {
  auto* call = static_cast<BatchCall<T>*>(user);
  try {
    call->fn(std::span<const T>(static_cast<const T*>(g), n));
    return 0;
  } catch (...) {
    call->error = std::current_exception();
    return 1;
  }
}
}  // namespace detail

// derive_edits<T> (edit_engine.hpp:183-186) on the GPU.
template <class T>
EditSet<T> derive_edits(const GridTopology& topo, const T* original, const T* decompressed,
                        double xi, const DeriveOptions<T>& opts = {},
                        EditStats* stats_out = nullptr) {
  mssz_cu_options o;
  mssz_cu_default_options(&o);
  o.outer_cap = opts.outer_cap;
  o.subloop_cap = opts.subloop_cap;
  o.r_cap = opts.r_cap;
  o.force = opts.force ? 1 : 0;
  o.device = opts.device;
  detail::BatchCall<T> call{opts.on_batch, nullptr};
  if (call.fn) {
    o.on_batch = &detail::batch_trampoline<T>;
    o.on_batch_user = &call;
  }
  std::uint64_t* idx = nullptr;
  T* val = nullptr;
  std::uint64_t count = 0;
  EditStats st;
  const int rc = detail::Api<T>::derive(topo.ndims, topo.dims.data(), original, decompressed, xi,
                                        &o, &idx, &val, &count, &st);
  if (rc == MSSZ_CU_ERR_CALLBACK && call.error) std::rethrow_exception(call.error);
  check(rc);
  EditSet<T> set;
  set.indices.assign(idx, idx + count);
  set.values.assign(val, val + count);
  mssz_cu_free(idx);
  mssz_cu_free(val);
  if (stats_out) *stats_out = st;
  return set;
}

// compute_directions<T> (mss.hpp:44-50)
template <class T>
DirectionField compute_directions(const GridTopology& topo, const T* values) {
  DirectionField d;
  d.asc.resize(topo.vertex_count);
  d.desc.resize(topo.vertex_count);
  check(detail::Api<T>::directions(topo.ndims, topo.dims.data(), values, d.asc.data(),
                                   d.desc.data()));
  return d;
}

// compute_labels (mss.hpp:58-60)
inline SegmentationLabels compute_labels(const GridTopology& topo, const DirectionField& d) {
  SegmentationLabels l;
  l.max_label.resize(topo.vertex_count);
  l.min_label.resize(topo.vertex_count);
  check(mssz_cu_compute_labels(topo.ndims, topo.dims.data(), d.asc.data(), d.desc.data(),
                               l.max_label.data(), l.min_label.data()));
  return l;
}

// apply_edits<T> (edit_engine.hpp:188-190)
template <class T>
std::vector<T> apply_edits(const GridTopology& topo, const T* decompressed,
                           const EditSet<T>& edits) {
  if (edits.indices.size() != edits.values.size())
    throw Error(ErrKind::corrupt_archive, "edit set index/value length mismatch");
  std::vector<T> out(topo.vertex_count);
  check(detail::Api<T>::apply(topo.vertex_count, decompressed, edits.indices.data(),
                              edits.values.data(), edits.size(), out.data()));
  return out;
}

// ---- the `mss` subcommand (tools/mssz.cpp:260-266) -------------------------
// compute_labels(compute_directions(values)) as one device pass.
template <class T>
SegmentationLabels segmentation(const GridTopology& topo, const T* values) {
  SegmentationLabels l;
  l.max_label.resize(topo.vertex_count);
  l.min_label.resize(topo.vertex_count);
  check(detail::Api<T>::segmentation(topo.ndims, topo.dims.data(), values, l.max_label.data(),
                                     l.min_label.data()));
  return l;
}

// ---- verification report (metrics.hpp:14-24, tools/mssz.cpp:84-104) --------
struct VerificationReport {
  double mss_distortion = 0.0;
  double right_labeled_ratio = 1.0;
  double psnr = 0.0;
  double edit_ratio = 0.0;
  double ocr = 0.0;
  double obr = 0.0;
  std::uint64_t bound_violations = 0;
  std::uint64_t fp_max = 0, fp_min = 0, fn_max = 0, fn_min = 0;
  // B200 extras: raw mismatch count and the device time of the report.
  std::uint64_t mismatches = 0;
  double device_seconds = 0.0;
};

// build_report<T>(original, candidate, xi, edit_count, archive_bytes, policy)
// (tools/mssz.cpp:84-104); `device` replaces the ExecPolicy.
template <class T>
VerificationReport build_report(const GridTopology& topo, const T* original, const T* candidate,
                                double xi, std::uint64_t edit_count = 0,
                                std::uint64_t archive_bytes = 0, int device = -1) {
  mssz_cu_options o;
  mssz_cu_default_options(&o);
  o.device = device;
  mssz_cu_report r{};
  check(detail::Api<T>::verify(topo.ndims, topo.dims.data(), original, candidate, xi,
                               edit_count, archive_bytes, &o, &r));
  VerificationReport v;
  v.mss_distortion = r.mss_distortion;
  v.right_labeled_ratio = r.right_labeled_ratio;
  v.psnr = r.psnr;
  v.edit_ratio = r.edit_ratio;
  v.ocr = r.ocr;
  v.obr = r.obr;
  v.bound_violations = r.bound_violations;
  v.fp_max = r.fp_max;
  v.fp_min = r.fp_min;
  v.fn_max = r.fn_max;
  v.fn_min = r.fn_min;
  v.mismatches = r.mismatches;
  v.device_seconds = r.device_seconds;
  return v;
}

// The reference CLI's `verify` verdict (tools/mssz.cpp: exit 0 iff both are 0).
inline bool verified(const VerificationReport& r) {
  return r.mss_distortion == 0.0 && r.bound_violations == 0;
}

// ---- base codec (base_codec.hpp:29-40) --------------------------------------
// The reference's compress_base returns {payload, reconstruction}; the payload is
// huffman::encode_stream(symbols) followed by the literals.  The GPU computes the
// prediction/quantisation wavefront, so this returns the reconstruction together
// with the symbol stream (0 = escape, else 1 + zigzag(q)) and the escaped literals
// in index order — the inputs of the reference's Huffman framing.
template <class T>
struct BaseQuantization {
  std::vector<T> reconstruction;  // fhat, |f - fhat| <= xi pointwise
  std::vector<std::uint32_t> symbols;
  std::vector<T> literals;
  double device_ms = 0.0;
};

template <class T>
BaseQuantization<T> compress_base(const GridTopology& topo, const T* values, double xi) {
  BaseQuantization<T> q;
  q.reconstruction.resize(topo.vertex_count);
  q.symbols.resize(topo.vertex_count);
  std::uint64_t escapes = 0;
  check(detail::Api<T>::compress_base(topo.ndims, topo.dims.data(), values, xi,
                                      q.reconstruction.data(), q.symbols.data(), &escapes,
                                      &q.device_ms));
  q.literals.reserve(escapes);
  for (std::uint64_t v = 0; v < topo.vertex_count; ++v)
    if (q.symbols[v] == 0) q.literals.push_back(values[v]);
  if (q.literals.size() != escapes)
    throw Error(ErrKind::internal, "compress_base: escape count mismatch");
  return q;
}

// decompress_base<T> (base_codec.hpp:38-40) after the Huffman decode of the payload.
template <class T>
std::vector<T> decompress_base(const GridTopology& topo, std::span<const std::uint32_t> symbols,
                               std::span<const T> literals, double xi) {
  if (symbols.size() != topo.vertex_count)
    throw Error(ErrKind::corrupt_archive, "code count does not match the grid");
  std::vector<T> out(topo.vertex_count);
  check(detail::Api<T>::decompress_base(topo.ndims, topo.dims.data(), symbols.data(),
                                        literals.empty() ? nullptr : literals.data(),
                                        literals.size(), xi, out.data(), nullptr));
  return out;
}

// ---- edit-set encoding (edit_codec.hpp:29-43) --------------------------------
enum class BackendCodec : std::uint8_t { store = 0, deflate = 1 };

// encode_edits<T>(edits, codec): byte-identical to the reference's payload.
template <class T>
std::vector<std::uint8_t> encode_edits(const EditSet<T>& edits, BackendCodec codec) {
  if (edits.indices.size() != edits.values.size())
    throw Error(ErrKind::usage, "edit set index/value length mismatch");
  std::uint8_t* buf = nullptr;
  std::uint64_t len = 0;
  check(detail::Api<T>::encode_edits(edits.indices.empty() ? nullptr : edits.indices.data(),
                                     edits.values.empty() ? nullptr : edits.values.data(),
                                     edits.size(), static_cast<int>(codec), &buf, &len,
                                     nullptr));
  std::vector<std::uint8_t> out(buf, buf + len);
  mssz_cu_free(buf);
  return out;
}

}  // namespace mssz_b200
