// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference core compiled from
// /root/reference/proj/core/src (see oracle/Makefile).  It exposes the
// reference's own hot-path entry points to the parity harness (tests/,
// __graft_entry__.smoke(), bench.py's cpu_baseline leg) via ctypes:
//   derive_edits<T>        edit_engine.hpp:183-186 / edit_engine.cpp:386-435
//   compute_directions<T>  mss.hpp:44-50 / mss.cpp:11-30
//   compute_labels         mss.hpp:58-60 / mss.cpp:91-97
//   oracle_labels<T>       mss.hpp:66-67 / mss.cpp:99-120
//   EditState::detect_false_critical / lower_step / find_troublemaker
//                          edit_engine.hpp:95-120
//   run_r_loop's target collection (r_targets) edit_engine.cpp:336-352
//   generate_synthetic<T>  field.hpp:343-345 / field.cpp:229-250
//   compress_base<T>       base_codec.hpp:198-199 / base_codec.cpp:76-120
//   resolve_bound<T>       field.hpp:320-321 / field.cpp:42-50
// Errors come back as the ErrKind integer (errors.hpp:9-16); 0 = success.

#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "mssz/base_codec.hpp"
#include "mssz/edit_codec.hpp"
#include "mssz/edit_engine.hpp"
#include "mssz/field.hpp"
#include "mssz/grid.hpp"
#include "mssz/mss.hpp"

using namespace mssz;

namespace {

thread_local std::string g_last_error;

ExecPolicy make_policy(int threads) {
  if (threads == 1) return ExecPolicy::serial_policy();
  return ExecPolicy{threads < 0 ? 0 : threads, false};
}

GridTopology topo_of(int ndims, const uint64_t* dims) {
  return build_topology(std::span<const std::uint64_t>(dims, static_cast<size_t>(ndims)));
}

template <class F>
int guarded(F&& body) {
  try {
    body();
    g_last_error.clear();
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.exit_code();
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return static_cast<int>(ErrKind::internal);
  }
}

}  // namespace

extern "C" {

typedef struct {
  uint64_t outer_cap;
  uint64_t subloop_cap;
  uint64_t r_cap;
  int force;
  int threads;  // 1 = ExecPolicy::serial_policy(); 0 = OpenMP default; n = n threads
} mssz_ref_options;

typedef struct {
  uint64_t outer_iterations;
  uint64_t c_passes;
  uint64_t sub_iterations[4];
  uint64_t r_iterations;
  uint64_t effective_edits;
  uint64_t touched;
  uint64_t input_bound_violations;
  double direction_seconds;
  double label_seconds;
} mssz_ref_stats;

const char* mssz_ref_last_error(void) { return g_last_error.c_str(); }
void mssz_ref_free(void* p) { std::free(p); }

}  // extern "C"

namespace {

template <class T>
int derive_impl(int ndims, const uint64_t* dims, const T* f, const T* fhat, double xi,
                const mssz_ref_options* o, void (*on_batch)(const T*, uint64_t, void*),
                void* user, uint64_t** idx_out, T** val_out, uint64_t* count_out,
                mssz_ref_stats* st) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    DeriveOptions<T> opts;
    if (o) {
      opts.outer_cap = o->outer_cap;
      opts.subloop_cap = o->subloop_cap;
      opts.r_cap = o->r_cap;
      opts.force = o->force != 0;
      opts.policy = make_policy(o->threads);
    }
    if (on_batch) {
      opts.on_batch = [on_batch, user](std::span<const T> g) {
        on_batch(g.data(), g.size(), user);
      };
    }
    EditStats stats;
    EditSet<T> set = derive_edits<T>(topo, f, fhat, xi, opts, &stats);
    const uint64_t n = set.size();
    uint64_t* idx = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (n ? n : 1)));
    T* val = static_cast<T*>(std::malloc(sizeof(T) * (n ? n : 1)));
    if (n) {
      std::memcpy(idx, set.indices.data(), sizeof(uint64_t) * n);
      std::memcpy(val, set.values.data(), sizeof(T) * n);
    }
    *idx_out = idx;
    *val_out = val;
    *count_out = n;
    if (st) {
      st->outer_iterations = stats.outer_iterations;
      st->c_passes = stats.c_passes;
      for (int k = 0; k < 4; ++k) st->sub_iterations[k] = stats.sub_iterations[k];
      st->r_iterations = stats.r_iterations;
      st->effective_edits = stats.effective_edits;
      st->touched = stats.touched;
      st->input_bound_violations = stats.input_bound_violations;
      st->direction_seconds = stats.direction_seconds;
      st->label_seconds = stats.label_seconds;
    }
  });
}

template <class T>
int directions_impl(int ndims, const uint64_t* dims, const T* values, uint64_t* asc,
                    uint64_t* desc, int threads) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    DirectionField d = compute_directions<T>(topo, values, make_policy(threads));
    std::memcpy(asc, d.asc.data(), sizeof(uint64_t) * topo.vertex_count);
    std::memcpy(desc, d.desc.data(), sizeof(uint64_t) * topo.vertex_count);
  });
}

template <class T>
int oracle_labels_impl(int ndims, const uint64_t* dims, const T* values, uint64_t* M,
                       uint64_t* m) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    SegmentationLabels l = oracle_labels<T>(topo, values);
    std::memcpy(M, l.max_label.data(), sizeof(uint64_t) * topo.vertex_count);
    std::memcpy(m, l.min_label.data(), sizeof(uint64_t) * topo.vertex_count);
  });
}

// counts[4] per first-match class; lists is 4*N u64 (class k at lists + k*N)
template <class T>
int detect_impl(int ndims, const uint64_t* dims, const T* f, const T* g, double xi,
                uint64_t* counts, uint64_t* lists, int threads = 1) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    EditState<T> state(topo, f, g, xi, make_policy(threads));
    const FalseCriticalReport& r = state.detect_false_critical();
    const std::vector<VertexId>* ls[4] = {&r.fp_max, &r.fp_min, &r.fn_max, &r.fn_min};
    for (int k = 0; k < 4; ++k) {
      counts[k] = ls[k]->size();
      if (lists && !ls[k]->empty())
        std::memcpy(lists + k * topo.vertex_count, ls[k]->data(),
                    sizeof(uint64_t) * ls[k]->size());
    }
  });
}

// Applies lower_step to vertex v up to max_steps times; trace receives every
// value g takes (trace[0] = initial); returns the number of successful steps.
template <class T>
int lower_step_impl(int ndims, const uint64_t* dims, const T* f, const T* g, double xi,
                    uint64_t v, int max_steps, T* trace, int* steps_out, T* floor_out) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    EditState<T> state(topo, f, g, xi, ExecPolicy::serial_policy());
    int steps = 0;
    trace[0] = state.edited()[v];
    while (steps < max_steps && state.lower_step(v)) {
      ++steps;
      trace[steps] = state.edited()[v];
    }
    *steps_out = steps;
    *floor_out = state.floors()[v];
  });
}

template <class T>
int troublemaker_impl(int ndims, const uint64_t* dims, const T* f, const T* g, double xi,
                      uint64_t v, int descending, uint64_t* vi, uint64_t* vt) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    EditState<T> state(topo, f, g, xi, ExecPolicy::serial_policy());
    auto r = state.find_troublemaker(v, descending ? EditState<T>::LineKind::descending
                                                   : EditState<T>::LineKind::ascending);
    *vi = r.first;
    *vt = r.second;
  });
}

}  // namespace

// The reference grants its test suite access to EditState's private R-loop
// steps through this friend (edit_engine.hpp:173); the shim uses it to run
// one R batch's target collection exactly as run_r_loop does.
namespace mssz {
struct EditEngineTestAccess {
  template <class T>
  static void compute_g_labels(EditState<T>& s) { s.compute_g_labels(); }
  template <class T>
  static std::uint64_t collect_mismatched(const EditState<T>& s, std::vector<VertexId>& out) {
    return s.collect_mismatched(out);
  }
  template <class T>
  static const SegmentationLabels& g_labels(const EditState<T>& s) { return s.g_labels_; }
};
}  // namespace mssz

namespace {

// One R batch's target set, run_r_loop (edit_engine.cpp:336-352): labels of g,
// collect_mismatched, find_troublemaker per mismatched vertex and family; the
// claim dedupe becomes sort + unique.  info = {false critical points of (f, g)
// (the gate, :338), distinct (v_i, family) troublemaker sources, mismatched
// vertices}.  Behind the gate only: a pair with false critical points has no
// R batch (run_r_loop returns there), so its target set is empty.
template <class T>
int r_targets_impl(int ndims, const uint64_t* dims, const T* f, const T* g, int threads,
                   uint64_t* targets, uint64_t* count, uint64_t* info) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    EditState<T> state(topo, f, g, 1.0, make_policy(threads));
    state.refresh_directions();
    info[0] = state.detect_false_critical().total();
    if (info[0] != 0) {  // the gate (edit_engine.cpp:338): no R batch
      info[1] = info[2] = 0;
      *count = 0;
      return;
    }
    EditEngineTestAccess::compute_g_labels(state);
    std::vector<VertexId> mismatched;
    info[2] = EditEngineTestAccess::collect_mismatched(state, mismatched);
    const SegmentationLabels& gl = EditEngineTestAccess::g_labels(state);
    const SegmentationLabels& fl = state.original_labels();
    std::vector<VertexId> t, src;
    for (VertexId v : mismatched) {
      if (gl.max_label[v] != fl.max_label[v]) {
        auto [vi, vt] = state.find_troublemaker(v, EditState<T>::LineKind::ascending);
        t.push_back(vt);
        src.push_back(vi * 2);
      }
      if (gl.min_label[v] != fl.min_label[v]) {
        auto [vi, vt] = state.find_troublemaker(v, EditState<T>::LineKind::descending);
        t.push_back(vt);
        src.push_back(vi * 2 + 1);
      }
    }
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    std::sort(src.begin(), src.end());
    info[1] = static_cast<uint64_t>(std::unique(src.begin(), src.end()) - src.begin());
    std::copy(t.begin(), t.end(), targets);
    *count = t.size();
  });
}

template <class T>
int generate_impl(int kind, int ndims, const uint64_t* dims, uint64_t seed, T* out) {
  return guarded([&] {
    Field<T> fld = generate_synthetic<T>(static_cast<SyntheticKind>(kind),
                                         std::span<const std::uint64_t>(dims, ndims), seed);
    std::memcpy(out, fld.values.data(), sizeof(T) * fld.values.size());
  });
}

template <class T>
int compress_base_impl(int ndims, const uint64_t* dims, const T* values, double xi, T* recon,
                       uint64_t* payload_bytes) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    BaseCompressResult<T> r = compress_base<T>(topo, values, xi);
    std::memcpy(recon, r.reconstruction.data(), sizeof(T) * topo.vertex_count);
    if (payload_bytes) *payload_bytes = r.payload.size();
  });
}

template <class T>
int resolve_rel_impl(int ndims, const uint64_t* dims, const T* values, double magnitude,
                     double* xi) {
  return guarded([&] {
    Field<T> fld;
    fld.topo = topo_of(ndims, dims);
    fld.values.assign(values, values + fld.topo.vertex_count);
    *xi = resolve_bound<T>(ErrorBound{ErrorBound::Mode::relative, magnitude}, fld);
  });
}

}  // namespace

extern "C" {

#define MSSZ_REF_INSTANTIATE(SUF, T)                                                        \
  int mssz_ref_derive_edits_##SUF(int ndims, const uint64_t* dims, const T* f, const T* fh,  \
                                  double xi, const mssz_ref_options* o,                      \
                                  void (*cb)(const T*, uint64_t, void*), void* user,         \
                                  uint64_t** idx, T** val, uint64_t* count,                  \
                                  mssz_ref_stats* st) {                                      \
    return derive_impl<T>(ndims, dims, f, fh, xi, o, cb, user, idx, val, count, st);         \
  }                                                                                          \
  int mssz_ref_compute_directions_##SUF(int ndims, const uint64_t* dims, const T* v,         \
                                        uint64_t* asc, uint64_t* desc, int threads) {        \
    return directions_impl<T>(ndims, dims, v, asc, desc, threads);                           \
  }                                                                                          \
  int mssz_ref_oracle_labels_##SUF(int ndims, const uint64_t* dims, const T* v, uint64_t* M, \
                                   uint64_t* m) {                                            \
    return oracle_labels_impl<T>(ndims, dims, v, M, m);                                      \
  }                                                                                          \
  int mssz_ref_detect_false_critical_##SUF(int ndims, const uint64_t* dims, const T* f,      \
                                           const T* g, double xi, uint64_t* counts,          \
                                           uint64_t* lists) {                                \
    return detect_impl<T>(ndims, dims, f, g, xi, counts, lists);                             \
  }                                                                                          \
  int mssz_ref_detect_false_critical_mt_##SUF(int ndims, const uint64_t* dims, const T* f,   \
                                              const T* g, double xi, uint64_t* counts,       \
                                              uint64_t* lists, int threads) {                \
    return detect_impl<T>(ndims, dims, f, g, xi, counts, lists, threads);                    \
  }                                                                                          \
  int mssz_ref_lower_step_##SUF(int ndims, const uint64_t* dims, const T* f, const T* g,     \
                                double xi, uint64_t v, int max_steps, T* trace, int* steps,  \
                                T* floor_out) {                                              \
    return lower_step_impl<T>(ndims, dims, f, g, xi, v, max_steps, trace, steps, floor_out); \
  }                                                                                          \
  int mssz_ref_find_troublemaker_##SUF(int ndims, const uint64_t* dims, const T* f,          \
                                       const T* g, double xi, uint64_t v, int descending,    \
                                       uint64_t* vi, uint64_t* vt) {                         \
    return troublemaker_impl<T>(ndims, dims, f, g, xi, v, descending, vi, vt);               \
  }                                                                                          \
  int mssz_ref_r_targets_##SUF(int ndims, const uint64_t* dims, const T* f, const T* g,      \
                               int threads, uint64_t* targets, uint64_t* count,              \
                               uint64_t* info) {                                             \
    return r_targets_impl<T>(ndims, dims, f, g, threads, targets, count, info);              \
  }                                                                                          \
  int mssz_ref_generate_##SUF(int kind, int ndims, const uint64_t* dims, uint64_t seed,      \
                              T* out) {                                                      \
    return generate_impl<T>(kind, ndims, dims, seed, out);                                   \
  }                                                                                          \
  int mssz_ref_compress_base_##SUF(int ndims, const uint64_t* dims, const T* v, double xi,   \
                                   T* recon, uint64_t* payload_bytes) {                      \
    return compress_base_impl<T>(ndims, dims, v, xi, recon, payload_bytes);                  \
  }                                                                                          \
  int mssz_ref_resolve_rel_##SUF(int ndims, const uint64_t* dims, const T* v, double mag,    \
                                 double* xi) {                                               \
    return resolve_rel_impl<T>(ndims, dims, v, mag, xi);                                     \
  }

MSSZ_REF_INSTANTIATE(f32, float)
MSSZ_REF_INSTANTIATE(f64, double)

int mssz_ref_compute_labels(int ndims, const uint64_t* dims, const uint64_t* asc,
                            const uint64_t* desc, uint64_t* M, uint64_t* m, int threads) {
  return guarded([&] {
    GridTopology topo = topo_of(ndims, dims);
    DirectionField d;
    d.asc.assign(asc, asc + topo.vertex_count);
    d.desc.assign(desc, desc + topo.vertex_count);
    SegmentationLabels l = compute_labels(topo, d, make_policy(threads));
    std::memcpy(M, l.max_label.data(), sizeof(uint64_t) * topo.vertex_count);
    std::memcpy(m, l.min_label.data(), sizeof(uint64_t) * topo.vertex_count);
  });
}

// encode_edits<T> (edit_codec.cpp:188-222): callee-allocated payload (mssz_ref_free)
#define MSSZ_REF_CODEC(SUF, T)                                                                 \
  int mssz_ref_encode_edits_##SUF(const uint64_t* idx, const T* val, uint64_t count, int codec, \
                                  uint8_t** out, uint64_t* len) {                               \
    return guarded([&] {                                                                        \
      EditSet<T> e;                                                                             \
      e.indices.assign(idx, idx + count);                                                       \
      e.values.assign(val, val + count);                                                        \
      const auto bytes = encode_edits<T>(e, parse_backend(static_cast<std::uint8_t>(codec)));   \
      *out = static_cast<uint8_t*>(std::malloc(bytes.size() ? bytes.size() : 1));               \
      std::memcpy(*out, bytes.data(), bytes.size());                                            \
      *len = bytes.size();                                                                      \
    });                                                                                         \
  }
MSSZ_REF_CODEC(f32, float)
MSSZ_REF_CODEC(f64, double)

int mssz_ref_build_topology(int ndims, const uint64_t* dims, uint64_t* vertex_count) {
  return guarded([&] { *vertex_count = topo_of(ndims, dims).vertex_count; });
}

}  // extern "C"
