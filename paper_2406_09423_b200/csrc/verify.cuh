// Verification report on the GPU: build_report
// (tools/mssz.cpp:84-104) with metrics.cpp's definitions, over (f, candidate)
// resident in HBM.  Directions and labels reuse K1 / K3; one fused sweep then
// reduces, per vertex: label mismatch (segmentation_equal, mss.cpp:122-133),
// (f - g)^2 in double (psnr, metrics.cpp:18-32), min/max of f (value_range,
// field.cpp:31-40), |f - g| > xi (count_bound_violations, metrics.cpp:46-56)
// and the first-match false-extremum class (count_false_extrema,
// tools/mssz.cpp:69-82).  Integer outputs are exact; the sum of squares is a
// deterministic tree (the reference sums sequentially), so psnr agrees to the
// reference's own test tolerance (1e-12 relative, test_metrics.cpp:40).
#pragma once

namespace mssz_b200 {
namespace {

constexpr int kRepThreads = 256;

struct RepPart {  // per-block partials
  double sq, lo, hi;
  unsigned long long mism, viol, cls[4];
};

template <class T>
__global__ void __launch_bounds__(kRepThreads) k_report(const T* __restrict__ f, const T* __restrict__ g,
                                                        const uint8_t* __restrict__ fdir,
                                                        const uint8_t* __restrict__ gdir,
                                                        const uint32_t* __restrict__ fM, const uint32_t* __restrict__ fm,
                                                        const uint32_t* __restrict__ gM, const uint32_t* __restrict__ gm,
                                                        uint64_t n, double xi, RepPart* __restrict__ parts) {
  double sq = 0.0, lo = INFINITY, hi = -INFINITY;
  unsigned long long mism = 0, viol = 0, cls[4] = {0, 0, 0, 0};
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const double a = static_cast<double>(__ldg(f + v)), b = static_cast<double>(__ldg(g + v));
    const double d = __dsub_rn(a, b);
    sq = __dadd_rn(sq, __dmul_rn(d, d));
    lo = fmin(lo, a);
    hi = fmax(hi, a);
    viol += fabs(d) > xi ? 1 : 0;
    mism += (__ldg(fM + v) != __ldg(gM + v) || __ldg(fm + v) != __ldg(gm + v)) ? 1 : 0;
    const uint32_t c = first_class(__ldg(fdir + v), __ldg(gdir + v));
    if (c < 4) ++cls[c];
  }
  __shared__ RepPart sp[kRepThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    mism += __shfl_xor_sync(0xffffffffu, mism, o);
    viol += __shfl_xor_sync(0xffffffffu, viol, o);
#pragma unroll
    for (int k = 0; k < 4; ++k) cls[k] += __shfl_xor_sync(0xffffffffu, cls[k], o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sp[w] = RepPart{sq, lo, hi, mism, viol, {cls[0], cls[1], cls[2], cls[3]}};
  __syncthreads();
  if (threadIdx.x == 0) {
    RepPart r = sp[0];
    for (int k = 1; k < kRepThreads / 32; ++k) {  // fixed order: deterministic
      r.sq = __dadd_rn(r.sq, sp[k].sq);
      r.lo = fmin(r.lo, sp[k].lo);
      r.hi = fmax(r.hi, sp[k].hi);
      r.mism += sp[k].mism;
      r.viol += sp[k].viol;
      for (int c = 0; c < 4; ++c) r.cls[c] += sp[k].cls[c];
    }
    parts[blockIdx.x] = r;
  }
}

// Host side: f -> ws.f, candidate -> ws.g (device copies), then K1 x2, K3 x2, k_report.
template <class T>
void verify_run(Workspace& ws, const Geom& geo, const mssz_cu_options& opt, double xi, uint64_t edit_count,
                uint64_t archive_bytes, mssz_cu_report* out) {
  if (!(xi > 0.0)) fail(MSSZ_CU_ERR_USAGE, "verify requires xi > 0");
  Engine<T> eng(ws, geo, opt);
  eng.bind(ws.f.as<T>());
  cudaEvent_t t0, t1;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventRecord(t0, ws.stream));
  eng.directions(ws.f.as<T>(), ws.fdir.as<uint8_t>());
  eng.directions(ws.g.as<T>(), ws.gdir.as<uint8_t>());
  eng.label_pass(ws.fdir.as<uint8_t>(), eng.lab(0), eng.lab(1), false, true);
  eng.label_pass(ws.gdir.as<uint8_t>(), eng.lab(2), eng.lab(3), false, true);
  const uint32_t blocks = grid_for(geo.n, kRepThreads, ws.sms, 8);
  DevBuf parts;
  parts.ensure(sizeof(RepPart) * blocks);
  eng.pre(kProfCompact);
  k_report<T><<<blocks, kRepThreads, 0, ws.stream>>>(ws.f.as<T>(), ws.g.as<T>(), ws.fdir.as<uint8_t>(),
                                                     ws.gdir.as<uint8_t>(), eng.lab(0), eng.lab(1), eng.lab(2),
                                                     eng.lab(3), geo.n, xi, parts.as<RepPart>());
  eng.launched(kProfCompact);
  std::vector<RepPart> h(blocks);
  CK(cudaMemcpyAsync(h.data(), parts.p, sizeof(RepPart) * blocks, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaEventRecord(t1, ws.stream));
  ws.sync();
  parts.release();
  RepPart r = h[0];
  for (uint32_t b = 1; b < blocks; ++b) {
    r.sq += h[b].sq;
    r.lo = std::min(r.lo, h[b].lo);
    r.hi = std::max(r.hi, h[b].hi);
    r.mism += h[b].mism;
    r.viol += h[b].viol;
    for (int c = 0; c < 4; ++c) r.cls[c] += h[b].cls[c];
  }
  const double N = static_cast<double>(geo.n);
  mssz_cu_report rep{};
  rep.mismatches = r.mism;
  rep.mss_distortion = static_cast<double>(r.mism) / N;            // metrics.cpp:12-15
  rep.right_labeled_ratio = 1.0 - rep.mss_distortion;               // tools/mssz.cpp:92
  const double rmse = std::sqrt(r.sq / N);                           // metrics.cpp:27-31
  rep.psnr = rmse == 0.0 ? std::numeric_limits<double>::infinity() : 20.0 * std::log10((r.hi - r.lo) / rmse);
  rep.edit_ratio = static_cast<double>(edit_count) / N;             // metrics.cpp:34-36
  if (archive_bytes != 0) {                                          // metrics.cpp:38-44
    rep.ocr = static_cast<double>(geo.n * sizeof(T)) / static_cast<double>(archive_bytes);
    rep.obr = 8.0 * static_cast<double>(archive_bytes) / N;
  }
  rep.bound_violations = r.viol;
  rep.fp_max = r.cls[0];
  rep.fp_min = r.cls[1];
  rep.fn_max = r.cls[2];
  rep.fn_min = r.cls[3];
  rep.sum_sq = r.sq;
  rep.value_lo = r.lo;
  rep.value_hi = r.hi;
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, t0, t1));
  rep.device_seconds = ms * 1e-3;
  rep.kernel_launches = eng.st.kernel_launches;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  *out = rep;
}

template <class T>
void verify_entry(int ndims, const uint64_t* dims, const T* f, const T* g, double xi, uint64_t edit_count,
                  uint64_t archive_bytes, const mssz_cu_options* o, mssz_cu_report* out, bool device,
                  void* stream) {
  const Geom geo = make_geom(ndims, dims);
  if (!f || !g || !out) fail(MSSZ_CU_ERR_USAGE, "null pointer");
  const mssz_cu_options opt = resolve(o);
  Workspace& ws = workspace(opt.device);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, sizeof(T));
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  if (device && caller) {
    CK(cudaEventRecord(ws.ev[0], caller));
    CK(cudaStreamWaitEvent(ws.stream, ws.ev[0], 0));
  }
  const cudaMemcpyKind k = device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CK(cudaMemcpyAsync(ws.f.p, f, sizeof(T) * geo.n, k, ws.stream));
  CK(cudaMemcpyAsync(ws.g.p, g, sizeof(T) * geo.n, k, ws.stream));
  verify_run<T>(ws, geo, opt, xi, edit_count, archive_bytes, out);
  if (device && caller) {
    CK(cudaEventRecord(ws.ev[1], ws.stream));
    CK(cudaStreamWaitEvent(caller, ws.ev[1], 0));
  }
}

// The `mss` subcommand (tools/mssz.cpp:260-266): compute_labels(compute_directions(f))
// in one device pass (K1 + tiled K3 with its finish phase), u64 labels out.
template <class T>
void segmentation_entry(int ndims, const uint64_t* dims, const T* values, uint64_t* M, uint64_t* m) {
  const Geom geo = make_geom(ndims, dims);
  if (!values || !M || !m) fail(MSSZ_CU_ERR_USAGE, "null pointer");
  mssz_cu_options opt;
  mssz_cu_default_options(&opt);
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, sizeof(T));
  Engine<T> eng(ws, geo, opt);
  eng.bind(ws.f.as<T>());
  CK(cudaMemcpyAsync(ws.f.p, values, sizeof(T) * geo.n, cudaMemcpyHostToDevice, ws.stream));
  eng.directions(ws.f.as<T>(), ws.fdir.as<uint8_t>());
  eng.label_pass(ws.fdir.as<uint8_t>(), eng.lab(0), eng.lab(1), false, true);
  const uint64_t np = (geo.n + 63) & ~uint64_t(63);
  uint64_t* da = reinterpret_cast<uint64_t*>(ws.lists.p);
  uint64_t* dd = da + np;
  const uint32_t blocks = grid_for(geo.n, 256, ws.sms, 16);
  k_u32_to_u64<<<blocks, 256, 0, ws.stream>>>(eng.lab(0), da, geo.n);
  k_u32_to_u64<<<blocks, 256, 0, ws.stream>>>(eng.lab(1), dd, geo.n);
  CK_LAUNCH();
  CK(cudaMemcpyAsync(M, da, 8ull * geo.n, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaMemcpyAsync(m, dd, 8ull * geo.n, cudaMemcpyDeviceToHost, ws.stream));
  ws.sync();
}

}  // namespace
}  // namespace mssz_b200

extern "C" {
int mssz_cu_segmentation_f32(int ndims, const uint64_t* dims, const float* values, uint64_t* M, uint64_t* m) {
  return mssz_b200::guarded([&] { mssz_b200::segmentation_entry<float>(ndims, dims, values, M, m); });
}
int mssz_cu_segmentation_f64(int ndims, const uint64_t* dims, const double* values, uint64_t* M, uint64_t* m) {
  return mssz_b200::guarded([&] { mssz_b200::segmentation_entry<double>(ndims, dims, values, M, m); });
}
#define MSSZ_CU_DEFINE_VERIFY(SUF, T)                                                                  \
  int mssz_cu_verify_##SUF(int ndims, const uint64_t* dims, const T* original, const T* candidate,     \
                           double xi, uint64_t edit_count, uint64_t archive_bytes,                      \
                           const mssz_cu_options* opt, mssz_cu_report* out) {                           \
    return mssz_b200::guarded([&] {                                                                    \
      mssz_b200::verify_entry<T>(ndims, dims, original, candidate, xi, edit_count, archive_bytes, opt,  \
                                 out, false, nullptr);                                                  \
    });                                                                                                \
  }                                                                                                    \
  int mssz_cu_verify_device_##SUF(int ndims, const uint64_t* dims, const T* original,                  \
                                  const T* candidate, double xi, uint64_t edit_count,                   \
                                  uint64_t archive_bytes, const mssz_cu_options* opt,                   \
                                  mssz_cu_report* out, void* stream) {                                  \
    return mssz_b200::guarded([&] {                                                                    \
      mssz_b200::verify_entry<T>(ndims, dims, original, candidate, xi, edit_count, archive_bytes, opt,  \
                                 out, true, stream);                                                    \
    });                                                                                                \
  }
MSSZ_CU_DEFINE_VERIFY(f32, float)
MSSZ_CU_DEFINE_VERIFY(f64, double)
}  // extern "C"
