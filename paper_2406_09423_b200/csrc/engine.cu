// Host engine + C-ABI of the B200 correction loop (include/mssz_cuda.h).
//
// derive_edits orchestration mirrors edit_engine.cpp:386-435 (validation,
// EditState ctor, outer{C-loop; R-loop}, postcondition tripwire, edits()).
// The host only sees one small control block per subloop / R iteration: every
// detect → fix → refresh batch runs inside a cooperative persistent kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <limits>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mssz_cuda.h"
#include "kernels.cuh"
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

namespace mssz_b200 {
namespace {

thread_local std::string g_last_error;
// what the current on_batch call reports (mssz_cu_batch_phase): kind, outer
// iteration, 1-based C pass or R iteration within that outer iteration
thread_local uint64_t g_phase[3] = {0, 0, 0};

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Fail{code, buf};
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      fail(MSSZ_CU_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
           __FILE__, __LINE__);                                                         \
  } while (0)

#define CK_LAUNCH() CK(cudaGetLastError())

template <class F>
int guarded(F&& body) {
  try {
    body();
    g_last_error.clear();
    return MSSZ_CU_OK;
  } catch (const Fail& f) {
    g_last_error = f.msg;
    return f.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return MSSZ_CU_ERR_CUDA;
  } catch (...) {  // nothing may unwind through the C ABI
    g_last_error = "unexpected C++ exception inside the engine";
    return MSSZ_CU_ERR_INTERNAL;
  }
}

// Validates dims like build_topology (grid.cpp:39-55) plus the u32 id limit.
// TMA descriptor of a 3D direction field for k_label_tile's 32x16x16-byte tile
// loads (cuTensorMapEncodeTiled through the runtime's driver entry point).
// false (byte/vector loads instead): 2D, strides not 16-byte multiples, no
// driver entry point, or MSSZ_LABEL_TMA=0.
bool label_tile_map(const Geom& g, const uint8_t* dir, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  std::memset(map, 0, sizeof(*map));
  if (const char* e = std::getenv("MSSZ_LABEL_TMA"))
    if (std::atoi(e) == 0) return false;
  using TL = LabelTile<3>;
  if (!enc || g.ndims != 3 || g.X % 16 || g.XY % 16 || reinterpret_cast<uintptr_t>(dir) % 16 || g.X < TL::TX ||
      g.Y < TL::TY || g.Z < TL::TZ)
    return false;
  const cuuint64_t gdim[3] = {g.X, g.Y, g.Z};
  const cuuint64_t gstride[2] = {g.X, static_cast<cuuint64_t>(g.XY)};
  const cuuint32_t box[3] = {TL::TX, TL::TY, TL::TZ};
  const cuuint32_t estride[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(dir), gdim, gstride, box, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

Geom make_geom(int ndims, const uint64_t* dims) {
  if (ndims != 2 && ndims != 3) fail(MSSZ_CU_ERR_USAGE, "dims must have 2 or 3 extents");
  if (!dims) fail(MSSZ_CU_ERR_USAGE, "dims is null");
  const uint64_t cap = uint64_t(1) << 40;
  uint64_t count = 1;
  uint64_t d[3] = {1, 1, 1};
  for (int a = 0; a < ndims; ++a) {
    if (dims[a] < 2) fail(MSSZ_CU_ERR_USAGE, "every grid extent must be >= 2");
    if (dims[a] > cap / count) fail(MSSZ_CU_ERR_USAGE, "grid exceeds the address-space cap");
    d[a] = dims[a];
    count *= dims[a];
  }
  if (count >= 0xFFFFFFFFull)
    fail(MSSZ_CU_ERR_USAGE,
         "grid of %llu vertices exceeds the single-device u32 id space; shard it into z-slabs",
         (unsigned long long)count);
  Geom g{};
  g.ndims = ndims;
  g.nst = ndims == 2 ? 6 : 14;
  g.X = static_cast<uint32_t>(d[0]);
  g.Y = static_cast<uint32_t>(d[1]);
  g.Z = static_cast<uint32_t>(d[2]);
  g.XY = g.X * g.Y;
  g.n = static_cast<uint32_t>(count);
  for (int k = 0; k < 16; ++k) g.off[k] = 0;
  for (int k = 0; k < g.nst; ++k) {
    int dx, dy, dz;
    if (ndims == 2) stencil<2>(k, dx, dy, dz);
    else stencil<3>(k, dx, dy, dz);
    // kernels add offsets in u32 arithmetic (v + off wraps onto the right id for
    // every in-grid target), so only the value mod 2^32 matters: computed in
    // int64, stored two's-complement (X + XY + 1 may exceed INT32_MAX)
    const int64_t o = dx + dy * static_cast<int64_t>(g.X) + dz * static_cast<int64_t>(g.XY);
    g.off[k] = static_cast<int32_t>(static_cast<uint32_t>(static_cast<uint64_t>(o)));
  }
  return g;
}

int bit_width_u64(uint64_t x) {
  int w = 0;
  while (x) {
    ++w;
    x >>= 1;
  }
  return w;
}

uint32_t grid_for(uint64_t work, int threads, int sms, int per_sm = 8) {
  uint64_t b = (work + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(sms) * per_sm;
  if (b > cap) b = cap;
  if (b == 0) b = 1;
  return static_cast<uint32_t>(b);
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool ensure(size_t bytes) {  // returns true when (re)allocated
    if (bytes <= cap && p) return false;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    CK(cudaMalloc(&p, bytes ? bytes : 16));
    cap = bytes;
    return true;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class U>
  U* as() const {
    return static_cast<U*>(p);
  }
};

// Per-device cached workspace: device buffers grow monotonically, claim and
// frontier stamp ids keep increasing across calls so the stamp arrays are only
// cleared when (re)allocated.
struct Workspace {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D of fhat overlapping the f-side setup
  DevBuf f, g, fh, fdir, gdir, touched, stamp, fmark, lab, fin, lists, tiles;
  DevBuf tE, tEcnt, toldfin, tdirty, taffected, tbits, tcnt, tlist;  // label-tile store
  DevBuf xbuf;  // sparse R pass: crossing lists X (2 families x 2 buffers)
  DevBuf cstamp; // per 64-vertex chunk: mark of the last batch that changed a code (k_detect_dirty)
  Ctl* ctl = nullptr;
  Ctl* hctl = nullptr;  // pinned mirror
  uint32_t next_batch = 1, next_mark = 1;
  bool fmark_parked = false;  // a sharded C loop raised with parked items: fmark holds kParked
  cudaEvent_t ev[4] = {};
  std::vector<cudaEvent_t> pev;  // profiling event pool
  std::mutex mu;

  void prof_ev(size_t need) {
    while (pev.size() < need + 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      pev.push_back(e);
    }
  }
  uint64_t launches = 0;

  void init(int dev) {
    device = dev;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (const char* e = std::getenv("MSSZ_L2_FETCH"))  // experiment: L2 miss fetch granularity
      CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(std::atoi(e))));
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&ctl, sizeof(Ctl)));
    CK(cudaMallocHost(&hctl, sizeof(Ctl)));
    for (auto& e : ev) CK(cudaEventCreate(&e));
    CK(cudaFuncSetAttribute(k_label_tile<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(label_tile_smem<2>())));
    CK(cudaFuncSetAttribute(k_label_tile<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(label_tile_smem<3>())));
    CK(cudaFuncSetAttribute(k_directions_col3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(k1_smem_bytes())));
    CK(cudaFuncSetAttribute(k_directions_reg3<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(sizeof(D3Smem))));
    CK(cudaFuncSetAttribute(k_directions_reg3<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(sizeof(D3Smem))));
  }
  // private workspaces (virtual slab ranks) free everything, not just buffers
  void destroy() {
    release();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : pev) cudaEventDestroy(e);
    pev.clear();
    if (ctl) cudaFree(ctl);
    if (hctl) cudaFreeHost(hctl);
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    ctl = nullptr;
    hctl = nullptr;
    stream = nullptr;
  }
  void release() {
    for (DevBuf* b : {&f, &g, &fh, &fdir, &gdir, &touched, &stamp, &fmark, &lab, &fin, &lists, &tiles,
                      &tE, &tEcnt, &toldfin, &tdirty, &taffected, &tbits, &tcnt, &tlist, &xbuf, &cstamp})
      b->release();
    next_batch = next_mark = 1;
  }

  // Sizes every buffer for n vertices of element size es.
  void ensure(uint64_t n, size_t es) {
    const uint64_t np = (n + 63) & ~uint64_t(63);
    f.ensure(np * es);
    g.ensure(np * es);
    fdir.ensure(np);
    gdir.ensure(np);
    touched.ensure(np);
    bool fresh = stamp.ensure(np * 4);
    fresh |= fmark.ensure(np * 4);
    lab.ensure(np * 16);    // fM fm gM gm (u32)
    // exit finals (finM finm), see k_exit_*.  Zeroed when (re)allocated: an
    // incremental pass's k_exit_save reads fin at the exits of re-labelled tiles
    // that may never have been exits before (their saved value only feeds the
    // change test of a tile that is dirty, hence recomputed, anyway)
    if (fin.ensure(np * 8)) CK(cudaMemsetAsync(fin.p, 0, fin.cap, stream));
    fresh |= cstamp.ensure((n + 63) / 64 * 4 + 4);
    lists.ensure(np * 16);  // list0 list1 S F (u32); reused as the u64+T EditSet
    tiles.ensure(((n + kCompactTile - 1) / kCompactTile + 1) * 4);
    if (fresh || fmark_parked || next_batch > 0xF0000000u || next_mark > 0xF0000000u) {
      fmark_parked = false;
      CK(cudaMemsetAsync(stamp.p, 0, stamp.cap, stream));
      CK(cudaMemsetAsync(fmark.p, 0, fmark.cap, stream));
      CK(cudaMemsetAsync(cstamp.p, 0, cstamp.cap, stream));
      next_batch = next_mark = 1;
    }
  }

  // label-tile store for ntiles tiles of the given surface
  void ensure_tiles(uint32_t ntiles, uint32_t surface) {
    tE.ensure(size_t(ntiles) * 2 * surface * 4);
    toldfin.ensure(size_t(ntiles) * 2 * surface * 4);
    tEcnt.ensure(size_t(ntiles) * 2 * 4);
    tdirty.ensure(ntiles);
    taffected.ensure(ntiles);
    tbits.ensure(size_t(ntiles) * 2 * (kLabelTileN / 32) * 4);
    tcnt.ensure(size_t(ntiles) * 4);
    tlist.ensure(size_t(ntiles) * 3 * 4 + 16);
  }

  void push_ctl() { CK(cudaMemcpyAsync(ctl, hctl, sizeof(Ctl), cudaMemcpyHostToDevice, stream)); }
  void pull_ctl() {
    CK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }
  void sync() { CK(cudaStreamSynchronize(stream)); }
};

std::mutex g_ws_mu;
std::vector<std::unique_ptr<Workspace>> g_ws;

Workspace& workspace(int device) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    fail(MSSZ_CU_ERR_CUDA, "no CUDA device available (%s); the B200 engine has no CPU fallback",
         e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  if (device < 0) CK(cudaGetDevice(&device));
  if (device >= ndev) fail(MSSZ_CU_ERR_USAGE, "device %d out of range (%d devices)", device, ndev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if (g_ws.size() < static_cast<size_t>(ndev)) g_ws.resize(ndev);
  if (!g_ws[device]) {
    auto ws = std::make_unique<Workspace>();
    ws->init(device);
    g_ws[device] = std::move(ws);
  }
  CK(cudaSetDevice(device));
  return *g_ws[device];
}

// worklists up to this size run inside the leader CTA of k_subloop
uint32_t kSmallBatchMax = 256;  // tunable via MSSZ_SMALL_MAX (experiments)
// worklists above n / kHugeBatchDivisor are run by host-launched streaming kernels
uint32_t kHugeBatchDivisor = 64;  // tunable via MSSZ_HUGE_DIVISOR (experiments)
// R batches applying more than n / kRHugeDivisor edits refresh with a full sweep
uint32_t kRHugeDivisor = 256;     // tunable via MSSZ_RHUGE_DIVISOR (round-2 sweep: 128-256 best)
// R iterations after one with fewer than n / kSparseMismDivisor mismatches use the
// sparse pass; it gives up when Up(X) exceeds n / kSparseUpDivisor vertices
uint32_t kSparseMismDivisor = 64;
uint32_t kSparseUpDivisor = 16;
uint32_t kSparseMaxLevels = 256;  // deeper upstream trees go to the full pass

const char* kKindName[4] = {"FPmax", "FPmin", "FNmax", "FNmin"};

// kernel classes of mssz_cu_stats::kernel_ms / kernel_count (MSSZ_CU_PROF_*)
enum {
  kProfValidate = MSSZ_CU_PROF_VALIDATE,
  kProfDirections = MSSZ_CU_PROF_DIRECTIONS,
  kProfDetectKind = MSSZ_CU_PROF_DETECT_KIND,
  kProfDetectAll = MSSZ_CU_PROF_DETECT_ALL,
  kProfSubloop = MSSZ_CU_PROF_SUBLOOP,
  kProfLabelInit = MSSZ_CU_PROF_LABEL_INIT,
  kProfLabelJump = MSSZ_CU_PROF_LABEL_JUMP,
  kProfRfix = MSSZ_CU_PROF_RFIX,
  kProfFrontier = MSSZ_CU_PROF_FRONTIER,
  kProfCompact = MSSZ_CU_PROF_COMPACT,
  kProfLabelFinish = MSSZ_CU_PROF_LABEL_FINISH,
  kProfFix = MSSZ_CU_PROF_FIX,
  kProfSparse = MSSZ_CU_PROF_SPARSE,
  kProfDetectDirty = MSSZ_CU_PROF_DETECT_DIRTY,
};

// ---------------------------------------------------------------------------
template <class T>
struct Engine {
  Workspace& ws;
  Geom geo;
  mssz_cu_options opt;
  mssz_cu_stats st{};
  State<T> s{};
  uint32_t cur = 0;
  int coop_blocks = 0;
  std::vector<T> host_g;  // on_batch snapshots only
  bool trace = std::getenv("MSSZ_TRACE") != nullptr;  // per-iteration log on stderr
  bool k1_reg3 = std::getenv("MSSZ_K1_REG3") != nullptr;  // A/B: the shared-memory K1 (k_directions_reg3)
  bool exit_reset_forced = std::getenv("MSSZ_EXIT_RESET") != nullptr;  // A/B: k_exit_reset on full label passes
  uint64_t r_last_mism = ~uint64_t(0);  // mismatches of the latest R iteration
  bool r_full_valid = false;            // tile label state matches gdir (no C edits since)
  bool x_valid = false;                 // crossing lists X match gdir (for k_cross_update)
  uint32_t x_mark = 0;                  // first change mark issued after the current X
  int x_cur[2] = {0, 0};
  uint32_t x_n[2] = {0, 0};
  size_t prof_n = 0;
  std::vector<int> prof_cls;
  // incremental subloop detection: kind k's list was empty at mark end_mark[k]
  // and every g-code change since then stamped its chunk (k_detect_dirty);
  // a full direction sweep invalidates that (fresh[k] = false)
  uint32_t end_mark[4] = {0, 0, 0, 0};
  bool fresh[4] = {false, false, false, false};
  // code_epoch advances whenever g-codes may have changed (a subloop or R loop
  // with edits, a full sweep); a fresh kind whose list ran empty at epoch
  // epoch_end[k] still has an empty list while the epoch is unchanged, so its
  // subloop is skipped without a launch (no chunk can be stamped since)
  uint64_t code_epoch = 1;
  uint64_t epoch_end[4] = {0, 0, 0, 0};
  float dir_ms = 0.f, lab_ms = 0.f;
  SlabRes sres{};  // z-slab label resolution for k_rfix_tiles (tab == nullptr: single device)

  const T* fhat = nullptr;  // decompressed input on the device (derives touched at compaction)

  Engine(Workspace& w, const Geom& g, const mssz_cu_options& o) : ws(w), geo(g), opt(o) {}

  uint32_t n() const { return geo.n; }
  uint32_t* list(int k) const { return ws.lists.as<uint32_t>() + static_cast<uint64_t>(k) * ((n() + 63) & ~63u); }
  uint32_t* list_ptr(int k) const { return list(k); }
  uint32_t* lab(int k) const { return ws.lab.as<uint32_t>() + static_cast<uint64_t>(k) * ((n() + 63) & ~63u); }

  void bind(const T* d_f) {
    s.geo = geo;
    s.f = d_f;
    s.g = ws.g.as<T>();
    s.fdir = ws.fdir.as<uint8_t>();
    s.gdir = ws.gdir.as<uint8_t>();
    s.touched = ws.touched.as<uint8_t>();
    s.stamp = ws.stamp.as<uint32_t>();
    s.fmark = ws.fmark.as<uint32_t>();
    s.list[0] = list(0);
    s.list[1] = list(1);
    s.S = list(2);
    s.F = list(3);
    s.fM = lab(0);
    s.fm = lab(1);
    s.fM64 = s.fm64 = nullptr;
    s.gM = lab(2);
    s.gm = lab(3);
    s.xi = 0;
    s.ctl = ws.ctl;
    s.tdirty = nullptr;
    s.cstamp = ws.cstamp.as<uint32_t>();
    s.own_lo = s.act_lo = 0;
    s.own_n = s.act_n = geo.n;
  }

  // Per-kernel-class device time (CUDA events on the launching stream), only
  // when opt.profile is set: bench.py's roofline reads kernel_ms / kernel_count.
  // opt.profile: bit 0 = every class, bit (cls + 1) = class cls only
  bool profiled(int cls) const { return (opt.profile & 1) || ((opt.profile >> (cls + 1)) & 1); }
  void pre(int cls) {
    if (!profiled(cls)) return;
    ws.prof_ev(prof_n * 2);
    CK(cudaEventRecord(ws.pev[prof_n * 2], ws.stream));
    prof_cls.push_back(cls);
  }
  void launched(int cls) {
    ++ws.launches;
    ++st.kernel_launches;
    ++st.kernel_count[cls];
    CK_LAUNCH();
    if (!profiled(cls)) return;
    CK(cudaEventRecord(ws.pev[prof_n * 2 + 1], ws.stream));
    ++prof_n;
  }
  void resolve_profile() {
    if (!opt.profile) return;
    ws.sync();
    for (size_t i = 0; i < prof_n; ++i) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ws.pev[2 * i], ws.pev[2 * i + 1]));
      st.kernel_ms[prof_cls[i]] += ms;
    }
    prof_n = 0;
    prof_cls.clear();
  }

  // K1 full sweep: 2.5D smem-tiled, chunk of the streamed axis sized for >= 8 CTAs/SM.
  void directions(const T* vals, uint8_t* dir) {
    // every code may change: every chunk counts as changed for the next
    // incremental X (one pass over both families beats two full k_cross)
    if (dir == s.gdir) x_mark = 0;
    if (dir == s.gdir) {
      for (bool& f : fresh) f = false;
      ++code_epoch;
    }
    pre(kProfDirections);
    const uint64_t want = static_cast<uint64_t>(ws.sms) * 8;
    if (geo.ndims == 2) {
      using DT = DirTile<2>;
      const uint32_t bx = (geo.X + DT::BX - 1) / DT::BX;
      uint32_t chunk = static_cast<uint32_t>(std::max<uint64_t>(4, (uint64_t(geo.Y) * bx) / want));
      chunk = std::min<uint32_t>(chunk, 64);
      dim3 grid(bx, (geo.Y + chunk - 1) / chunk);
      k_directions_tiled<T, 2><<<grid, DT::BX * DT::BY, 0, ws.stream>>>(vals, dir, geo, chunk);
    } else if (sizeof(T) == 4 && !k1_reg3) {
      // register-column K1: >= ~4 waves of 2 CTAs/SM, chunks of >= 8 planes
      const uint32_t bx = (geo.X + kK1Cols - 1) / kK1Cols;
      const uint32_t by = (geo.Y + kK1Warps * kK1R - 1) / (kK1Warps * kK1R);
      const uint64_t tiles = uint64_t(bx) * by;
      const uint32_t zc = static_cast<uint32_t>(std::min<uint64_t>(
          std::max<uint64_t>(1, (uint64_t(ws.sms) * 8 + tiles - 1) / tiles), std::max<uint32_t>(1, geo.Z / 8)));
      const uint32_t chunk = (geo.Z + zc - 1) / zc;
      dim3 grid(bx, by, (geo.Z + chunk - 1) / chunk);
      k_directions_col3<<<grid, kK1Warps * 32, k1_smem_bytes(), ws.stream>>>(reinterpret_cast<const float*>(vals), dir, geo,
                                                              static_cast<int>(chunk));
    } else if (sizeof(T) == 4) {
      const uint32_t bx = (geo.X + kD3W - 1) / kD3W, by = (geo.Y + kD3H - 1) / kD3H;
      const uint64_t tiles = uint64_t(bx) * by;
      // >= ~4 waves of 2 CTAs/SM, chunks of >= 8 planes
      uint32_t zc = static_cast<uint32_t>(std::min<uint64_t>(
          std::max<uint64_t>(1, (uint64_t(ws.sms) * 8 + tiles - 1) / tiles), std::max<uint32_t>(1, geo.Z / 8)));
      const uint32_t chunk = (geo.Z + zc - 1) / zc;
      dim3 grid(bx, by, (geo.Z + chunk - 1) / chunk);
      const float* fv = reinterpret_cast<const float*>(vals);
      if (geo.X % 4 == 0)
        k_directions_reg3<true, 2><<<grid, kD3Warps * 32, sizeof(D3Smem), ws.stream>>>(fv, dir, geo, chunk);
      else
        k_directions_reg3<false, 2><<<grid, kD3Warps * 32, sizeof(D3Smem), ws.stream>>>(fv, dir, geo, chunk);
    } else {
      using DB = DirBlock3<T>;
      const uint32_t bx = (geo.X + DB::BX - 1) / DB::BX, by = (geo.Y + DB::BY - 1) / DB::BY;
      uint32_t chunk =
          static_cast<uint32_t>(std::max<uint64_t>(4, (uint64_t(geo.Z) * bx * by) / want));
      chunk = std::min<uint32_t>(chunk, 64);
      dim3 grid(bx, by, (geo.Z + chunk - 1) / chunk);
      k_directions_block3<T><<<grid, DB::BX * DB::BY, 0, ws.stream>>>(vals, dir, geo, chunk);
    }
    launched(kProfDirections);
  }

  // Pointer-jumping labels over arbitrary u32 parent arrays (compute_labels API).
  // Rounds are launched in groups of 4 and the group's last flag is read back.
  void jump_to_fixpoint(uint32_t* M, uint32_t* m) {
    const int cap = bit_width_u64(static_cast<uint64_t>(n()) - 1) + 2;
    const uint32_t blocks = grid_for(n(), 256, ws.sms, 16);
    int round = 0;
    for (;;) {
      const int group = 4;
      CK(cudaMemsetAsync(ws.ctl->flags, 0, sizeof(uint32_t) * group, ws.stream));
      for (int r = 0; r < group; ++r) {
        pre(kProfLabelJump);
        k_label_jump<<<blocks, 256, 0, ws.stream>>>(M, m, n(), &ws.ctl->flags[r]);
        launched(kProfLabelJump);
      }
      uint32_t flags[4];
      CK(cudaMemcpyAsync(flags, ws.ctl->flags, sizeof flags, cudaMemcpyDeviceToHost, ws.stream));
      ws.sync();
      int used = 0;
      while (used < group && flags[used]) ++used;
      round += used;
      st.label_rounds += used < group ? used + 1 : used;
      if (used < group) return;  // a round observed the fixpoint
      if (round > cap)
        fail(MSSZ_CU_ERR_INTERNAL,
             "path compression exceeded its round cap (corrupt direction field)");
    }
  }

  // Tiled labels (k_label_tile -> exit jumping -> k_label_finish).
  uint32_t label_tiles() const {
    if (geo.ndims == 2) {
      using TL = LabelTile<2>;
      return ((geo.X + TL::TX - 1) / TL::TX) * ((geo.Y + TL::TY - 1) / TL::TY);
    }
    using TL = LabelTile<3>;
    return ((geo.X + TL::TX - 1) / TL::TX) * ((geo.Y + TL::TY - 1) / TL::TY) *
           ((geo.Z + TL::TZ - 1) / TL::TZ);
  }

  TileStore tile_store() {
    TileStore t{};
    t.ntiles = label_tiles();
    t.surface = geo.ndims == 2 ? LabelTile<2>::kSurface : LabelTile<3>::kSurface;
    ws.ensure_tiles(t.ntiles, t.surface);
    t.E = ws.tE.as<uint32_t>();
    t.Ecnt = ws.tEcnt.as<uint32_t>();
    t.oldfin = ws.toldfin.as<uint32_t>();
    t.dirty = ws.tdirty.as<uint8_t>();
    t.affected = ws.taffected.as<uint8_t>();
    t.mis_bits = ws.tbits.as<uint32_t>();
    t.mis_cnt = ws.tcnt.as<uint32_t>();
    t.own_lo = s.own_n ? s.own_lo : 0u;
    t.own_hi = s.own_n ? s.own_lo + s.own_n : n();
    t.err = &ws.ctl->flags[63];
    return t;
  }
  uint32_t* tile_list(int k) const { return ws.tlist.as<uint32_t>() + size_t(k) * label_tiles(); }
  uint32_t* fin(int k) const { return ws.fin.as<uint32_t>() + size_t(k) * ((n() + 63) & ~63u); }

  // tiles selected by k_select_tiles(mode) into tile_list(slot); returns the count
  uint32_t select_tiles(const TileStore& ts, int mode, int slot) {
    CK(cudaMemsetAsync(&ws.ctl->cmd_n, 0, sizeof(uint32_t), ws.stream));
    k_select_tiles<<<grid_for(ts.ntiles, 256, ws.sms, 8), 256, 0, ws.stream>>>(ts, mode, tile_list(slot),
                                                                             &ws.ctl->cmd_n);
    CK_LAUNCH();
    uint32_t c = 0;
    CK(cudaMemcpyAsync(&c, &ws.ctl->cmd_n, 4, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    return c;
  }

  // Tiled labels: phase 1 on all tiles (or only dirty ones), phase 2 over every
  // tile's exits with change detection (-> ts.affected), optional phase 3.
  // Afterwards fin[prov[v]] is v's final label; with finish, prov[v] is final.
  void label_pass(const uint8_t* dir, uint32_t* M, uint32_t* m, bool only_dirty, bool finish) {
    CK(cudaEventRecord(ws.ev[2], ws.stream));
    TileStore ts = tile_store();
    uint32_t* fM = fin(0);
    uint32_t* fm = fin(1);
    uint32_t ntodo = ts.ntiles;
    const uint32_t* list = nullptr;
    if (only_dirty) {
      ntodo = select_tiles(ts, 0, 0);
      list = tile_list(0);
    }
    // a pass over every tile seeds the exits' fin entries itself (k_label_tile
    // writes fin on tile surfaces), so k_exit_reset is skipped; an incremental
    // pass keeps save -> reset so changed exit finals are detected
    const bool seed_exits = !only_dirty && !exit_reset_forced;
    if (ntodo) {
      CK(cudaMemsetAsync(ts.err, 0, sizeof(uint32_t), ws.stream));
      pre(kProfLabelInit);
      CUtensorMap dmap;
      const int use_tma = label_tile_map(geo, dir, &dmap) ? 1 : 0;
      if (geo.ndims == 2)
        k_label_tile<2><<<ntodo, kLabelTileThreads, label_tile_smem<2>(), ws.stream>>>(
            dir, geo, M, m, fM, fm, list, ts, dmap, 0, seed_exits ? 1 : 0);
      else
        k_label_tile<3><<<ntodo, kLabelTileThreads, label_tile_smem<3>(), ws.stream>>>(
            dir, geo, M, m, fM, fm, list, ts, dmap, use_tma, seed_exits ? 1 : 0);
      launched(kProfLabelInit);
    }
    st.label_tiles += ntodo;
    // phase 2: exits restart from their provisional label, then doubling.  Exit
    // chains cross at most ntiles tiles: <= bit_width(ntiles)+1 rounds, launched
    // blind (no host sync); each round compacts the unresolved exits.
    if (only_dirty) {  // old finals only matter for change detection
      pre(kProfLabelJump);
      k_exit_save<<<ts.ntiles, 256, 0, ws.stream>>>(ts, fM, fm);
      launched(kProfLabelJump);
    }
    if (!seed_exits) {
      pre(kProfLabelJump);
      k_exit_reset<<<ts.ntiles, 256, 0, ws.stream>>>(ts, M, m, fM, fm);
      launched(kProfLabelJump);
    }
    uint32_t* cnt[2] = {&ws.ctl->s_count, &ws.ctl->list_count[0]};  // (asc, desc) pairs
    uint32_t* la[2] = {list_ptr(2), list_ptr(0)};
    uint32_t* ld[2] = {list_ptr(3), list_ptr(1)};
    CK(cudaMemsetAsync(cnt[0], 0, 2 * sizeof(uint32_t), ws.stream));
    pre(kProfLabelJump);
    k_exit_jump_tiles<<<ts.ntiles, 256, 0, ws.stream>>>(ts, fM, fm, la[0], ld[0], cnt[0]);
    launched(kProfLabelJump);
    const int rounds = bit_width_u64(ts.ntiles) + 1;
    const uint32_t blocks = grid_for(n() / 8 + 1, 256, ws.sms, 16);
    for (int r = 0; r < rounds; ++r) {
      const int a = r & 1, b2 = a ^ 1;
      CK(cudaMemsetAsync(cnt[b2], 0, 2 * sizeof(uint32_t), ws.stream));
      pre(kProfLabelJump);
      k_label_exit_jump<<<blocks, 256, 0, ws.stream>>>(fM, fm, la[a], ld[a], la[b2], ld[b2], cnt[a],
                                                      cnt[b2]);
      launched(kProfLabelJump);
    }
    st.label_rounds += rounds + 1;
    CK(cudaMemsetAsync(ts.affected, 0, ts.ntiles, ws.stream));
    if (only_dirty) {
      pre(kProfLabelJump);
      k_exit_changed<<<ts.ntiles, 256, 0, ws.stream>>>(ts, fM, fm);
      launched(kProfLabelJump);
    }
    uint32_t left[2], tile_err = 0;
    CK(cudaMemcpyAsync(left, cnt[rounds & 1], sizeof left, cudaMemcpyDeviceToHost, ws.stream));
    if (ntodo) CK(cudaMemcpyAsync(&tile_err, ts.err, sizeof tile_err, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    if (left[0] || left[1] || tile_err)
      fail(MSSZ_CU_ERR_INTERNAL, "path compression exceeded its round cap (corrupt direction field)");
    if (finish) {
      pre(kProfLabelFinish);
      if (geo.ndims == 2)
        k_label_finish_tiles<2><<<ts.ntiles, 256, 0, ws.stream>>>(M, m, fM, fm, geo);
      else
        k_label_finish_tiles<3><<<ts.ntiles, 256, 0, ws.stream>>>(M, m, fM, fm, geo);
      launched(kProfLabelFinish);
    }
    CK(cudaEventRecord(ws.ev[3], ws.stream));
    CK(cudaEventSynchronize(ws.ev[3]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ws.ev[2], ws.ev[3]));
    lab_ms += ms;
    ++st.label_passes;
  }

  // R batch targets from the tile mismatch bitmaps (k_rfix_tiles on the given
  // tiles first); returns the total mismatch count, targets in list(0).
  // raise_trouble = false (z-slab ranks): the status word is all-gathered instead
  uint64_t r_targets(bool all_tiles, bool raise_trouble = true) {
    TileStore ts = tile_store();
    uint32_t nt = ts.ntiles;
    const uint32_t* list = nullptr;
    if (!all_tiles) {
      nt = select_tiles(ts, 1, 1);  // dirty or affected
      list = tile_list(1);
    }
    reset_ctl();
    ws.push_ctl();
    if (nt) {
      pre(kProfRfix);
      if (geo.ndims == 2)
        k_rfix_tiles<T, 2><<<nt, 256, 0, ws.stream>>>(s, list, ts, fin(0), fin(1), sres);
      else
        k_rfix_tiles<T, 3><<<nt, 256, 0, ws.stream>>>(s, list, ts, fin(0), fin(1), sres);
      launched(kProfRfix);
    }
    st.rfix_tiles += nt;
    const uint32_t nm = select_tiles(ts, 2, 2);  // tiles with mismatches
    if (nm) {
      pre(kProfRfix);
      if (geo.ndims == 2)
        k_expand_targets<T, 2><<<nm, 256, 0, ws.stream>>>(s, tile_list(2), ts, list_ptr(0),
                                                          &ws.ctl->list_count[0]);
      else
        k_expand_targets<T, 3><<<nm, 256, 0, ws.stream>>>(s, tile_list(2), ts, list_ptr(0),
                                                          &ws.ctl->list_count[0]);
      launched(kProfRfix);
    }
    CK(cudaMemsetAsync(ts.dirty, 0, ts.ntiles, ws.stream));
    ws.pull_ctl();
    st.rfix_divergent += ws.hctl->rfix_div;
    if (raise_trouble && ws.hctl->status == kStatusTroubleMax)
      fail(MSSZ_CU_ERR_INTERNAL, "troublemaker target is an extremum (stale critical report)");
    return ws.hctl->mism;
  }

  void reset_ctl() {
    std::memset(ws.hctl, 0, sizeof(Ctl));
    ws.hctl->cur = cur;
  }

  int coop_grid() {
    if (coop_blocks) return coop_blocks;
    if (const char* h = std::getenv("MSSZ_HUGE_DIVISOR")) kHugeBatchDivisor = std::max(1, std::atoi(h));
    if (const char* h = std::getenv("MSSZ_RHUGE_DIVISOR")) kRHugeDivisor = std::max(1, std::atoi(h));
    if (const char* h = std::getenv("MSSZ_SMALL_MAX")) kSmallBatchMax = static_cast<uint32_t>(std::max(0, std::atoi(h)));
    if (const char* h = std::getenv("MSSZ_SPARSE_DIVISOR")) kSparseMismDivisor = std::max(1, std::atoi(h));
    int occ = 0;
    if (geo.ndims == 2)
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_subloop<T, 2>, kSubThreads, 0));
    else
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_subloop<T, 3>, kSubThreads, 0));
    if (occ < 1) fail(MSSZ_CU_ERR_CUDA, "persistent subloop kernel cannot be co-resident");
    coop_blocks = ws.sms * std::min(occ, 3);
    return coop_blocks;
  }

  // per_batch: the device loop stops after every batch (reference call sites);
  // otherwise on_batch fires only at phase ends (MSSZ_CU_ON_BATCH_PHASES)
  bool per_batch() const { return opt.on_batch && opt.on_batch_mode == MSSZ_CU_ON_BATCH_EVERY; }
  uint64_t outer_it = 0, pass_it = 0, r_it = 0;  // phase counters of on_batch
  uint64_t huge_edits = 0;  // edits of host-driven huge C batches (not k_subloop's)
  // debug: every subloop skipped as provably empty is re-checked by a full sweep
  bool check_skips = std::getenv("MSSZ_CHECK_SKIPS") != nullptr;
  void on_batch(uint64_t kind = MSSZ_CU_PHASE_BATCH) {
    if (!opt.on_batch) return;
    g_phase[0] = kind;
    g_phase[1] = outer_it;
    g_phase[2] = kind == MSSZ_CU_PHASE_R_ITERATION ? r_it : kind == MSSZ_CU_PHASE_C_PASS ? pass_it : pass_it + 1;
    host_g.resize(n());
    CK(cudaMemcpyAsync(host_g.data(), s.g, sizeof(T) * n(), cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    if (opt.on_batch(host_g.data(), n(), opt.on_batch_user) != 0)
      fail(MSSZ_CU_ERR_CALLBACK, "on_batch aborted derive_edits");
  }
  void on_batch_batch() {  // a fix batch ended
    if (per_batch()) on_batch();
  }

  // One huge batch with streaming kernels (see k_subloop): fix_list, full
  // refresh_directions, detect_kind.  Returns false when the list was empty.
  // Mirrors one iteration of run_subloop (edit_engine.cpp:255-275).
  void huge_batch(int kind, uint32_t batch_base) {
    Ctl c = *ws.hctl;  // state handed back by k_subloop
    const uint32_t nl = c.list_count[cur];
    ++c.attempted;
    if (c.attempted > opt.subloop_cap)
      fail(MSSZ_CU_ERR_NON_CONVERGENCE, "%s subloop exceeded its iteration cap", kKindName[kind]);
    const uint32_t batch = batch_base + 2 * static_cast<uint32_t>(c.attempted);  // k_subloop's scheme
    const int rule = (kind == 0 || kind == 3) ? 0 : 1;
    CK(cudaMemsetAsync(&ws.ctl->s_count, 0, 2 * sizeof(uint32_t), ws.stream));
    pre(kProfFix);
    k_fix_list<T><<<grid_for(nl, 256, ws.sms, 16), 256, 0, ws.stream>>>(s, s.list[cur], nl, rule, batch);
    launched(kProfFix);
    uint32_t applied = 0;
    CK(cudaMemcpyAsync(&applied, &ws.ctl->s_count, 4, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    if (applied == 0 && kind == 1) {
      pre(kProfFix);
      k_fix_list<T><<<grid_for(nl, 256, ws.sms, 16), 256, 0, ws.stream>>>(s, s.list[cur], nl, 2, batch + 1);
      launched(kProfFix);
      CK(cudaMemcpyAsync(&applied, &ws.ctl->s_count, 4, cudaMemcpyDeviceToHost, ws.stream));
      ws.sync();
    }
    if (applied == 0)
      fail(MSSZ_CU_ERR_NON_CONVERGENCE, "%s subloop stalled at the float floor", kKindName[kind]);
    directions(s.g, s.gdir);
    CK(cudaMemsetAsync(&ws.ctl->list_count[cur ^ 1], 0, sizeof(uint32_t), ws.stream));
    pre(kProfDetectKind);
    k_detect_kind<<<grid_for((n() + 15) / 16, 256, ws.sms, 16), 256, 0, ws.stream>>>(
        s.fdir, s.gdir, n(), kind, s.list[cur ^ 1], &ws.ctl->list_count[cur ^ 1]);
    launched(kProfDetectKind);
    ++st.detect_sweeps;
    ++st.huge_batches;
    uint32_t next = 0;
    CK(cudaMemcpyAsync(&next, &ws.ctl->list_count[cur ^ 1], 4, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    // hand the loop state back to the persistent kernel
    cur ^= 1;
    c.cur = cur;
    c.list_count[cur] = next;
    c.list_count[cur ^ 1] = 0;
    c.iters += 1;
    c.edits += applied;
    huge_edits += applied;
    c.frontier += n();
    c.s_count = c.f_count = 0;
    c.status = kStatusOk;
    *ws.hctl = c;
    ws.push_ctl();
    on_batch_batch();
  }

  // run_subloop (edit_engine.cpp:246-278)
  uint64_t run_subloop(int kind) {
    if (fresh[kind] && epoch_end[kind] == code_epoch && !per_batch()) {  // list provably empty
      if (check_skips) {  // MSSZ_CHECK_SKIPS: prove it with a full detection sweep
        reset_ctl();
        ws.push_ctl();
        k_detect_kind<<<grid_for((n() + 15) / 16, 256, ws.sms, 16), 256, 0, ws.stream>>>(
            s.fdir, s.gdir, n(), kind, s.list[cur], &ws.ctl->list_count[cur]);
        CK_LAUNCH();
        ws.pull_ctl();
        if (ws.hctl->list_count[cur])
          fail(MSSZ_CU_ERR_INTERNAL, "skipped %s subloop has %u items (code epoch invariant broken)",
               kKindName[kind], ws.hctl->list_count[cur]);
      }
      ++st.skipped_subloops;
      return 0;
    }
    const uint64_t huge0 = huge_edits;
    reset_ctl();
    ws.push_ctl();
    const int dcls = fresh[kind] ? kProfDetectDirty : kProfDetectKind;
    pre(dcls);
    if (fresh[kind])
      k_detect_dirty<<<grid_for((n() + 15) / 16, 256, ws.sms, 16), 256, 0, ws.stream>>>(
          s.fdir, s.gdir, n(), s.cstamp, end_mark[kind], kind, s.list[cur], &ws.ctl->list_count[cur], 0u, n());
    else
      k_detect_kind<<<grid_for((n() + 15) / 16, 256, ws.sms, 16), 256, 0, ws.stream>>>(
          s.fdir, s.gdir, n(), kind, s.list[cur], &ws.ctl->list_count[cur]);
    launched(dcls);
    ++st.detect_sweeps;
    const uint32_t batch_base = ws.next_batch, mark_base = ws.next_mark;
    // stamp ids must never be reused, also when this subloop raises
    struct IdGuard {
      Workspace& ws;
      uint32_t bb, mb;
      ~IdGuard() {
        const uint32_t it = static_cast<uint32_t>(ws.hctl->attempted) + 2;
        ws.next_batch = std::max(ws.next_batch, bb + 2 * it + 4);
        ws.next_mark = std::max(ws.next_mark, mb + it + 2);
      }
    } id_guard{ws, batch_base, mark_base};
    uint64_t cap = opt.subloop_cap;
    uint32_t maxb = per_batch() ? 1u : 0xFFFFFFFFu;
    uint32_t small_max = kSmallBatchMax;
    uint32_t huge_min = std::max<uint32_t>(kSmallBatchMax, n() / kHugeBatchDivisor);
    uint32_t park_cap = (n() + 63) & ~63u;  // P lives in list(3) (State::F)
    void* args[] = {&s, &kind, &cap, (void*)&batch_base, (void*)&mark_base, &maxb, &small_max,
                    &huge_min, &park_cap};
    void* fn = geo.ndims == 2 ? (void*)k_subloop<T, 2> : (void*)k_subloop<T, 3>;
    const int blocks = coop_grid();
    uint64_t seen_iters = 0;
    for (;;) {
      CK(cudaMemsetAsync(&ws.ctl->cmd_seq, 0, sizeof(uint32_t), ws.stream));
      pre(kProfSubloop);
      CK(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kSubThreads), args, 0, ws.stream));
      launched(kProfSubloop);
      ws.pull_ctl();
      const Ctl& c = *ws.hctl;
      cur = c.cur;
      if (c.status == kStatusHuge) {
        huge_batch(kind, batch_base);
        seen_iters = ws.hctl->iters;
        continue;
      }
      if (!per_batch() || c.status != kStatusOk) break;
      if (c.iters == seen_iters) break;  // list empty
      seen_iters = c.iters;
      on_batch();
    }
    const Ctl& c = *ws.hctl;
    cur = c.cur;
    if (c.status == kStatusCap)
      fail(MSSZ_CU_ERR_NON_CONVERGENCE, "%s subloop exceeded its iteration cap", kKindName[kind]);
    if (c.status == kStatusStall)
      fail(MSSZ_CU_ERR_NON_CONVERGENCE, "%s subloop stalled at the float floor", kKindName[kind]);
    if (trace)
      std::fprintf(stderr,
                   "[mssz] C kind=%d iters=%llu edits=%llu items=%llu merges=%llu big=%llu frontier=%llu small_ms=%.2f big_ms=%.2f\n",
                   kind, (unsigned long long)c.iters, (unsigned long long)c.edits, (unsigned long long)c.items,
                   (unsigned long long)c.merges,
                   (unsigned long long)c.big_batches, (unsigned long long)c.frontier,
                   c.small_ns * 1e-6, c.big_ns * 1e-6);
    if (trace && c.big_batches)
      std::fprintf(stderr, "[mssz]   big phases fix=%.2f frontier=%.2f rebuild=%.2f ms\n",
                   c.phase_ns[0] * 1e-6, c.phase_ns[1] * 1e-6, c.phase_ns[2] * 1e-6);
    st.sub_iterations[kind] += c.iters;
    st.effective_edits += c.edits;
    st.subloop_items += c.items;
    st.subloop_edits += c.edits - (huge_edits - huge0);
    st.frontier_vertices += c.frontier;
    st.big_batches += c.big_batches;
    if (c.edits) ++code_epoch;
    return c.edits;
  }

  // run_c_loop (edit_engine.cpp:280-291)
  void run_c_loop() {
    for (;;) {
      ++st.c_passes;
      uint64_t pass_edits = 0;
      for (int kind = 0; kind < 4; ++kind) {
        pass_edits += run_subloop(kind);
        end_mark[kind] = ws.next_mark;  // every later batch uses marks >= this
        fresh[kind] = true;
        epoch_end[kind] = code_epoch;
      }
      if (pass_edits) r_full_valid = false;  // the tile store no longer matches gdir
      ++pass_it;
      if (opt.on_batch && !per_batch()) on_batch(MSSZ_CU_PHASE_C_PASS);  // a C pass ended
      if (pass_edits == 0) return;
    }
  }

  // frontier_only: count over the F list of the last k_frontier (its vertices
  // are the only ones whose codes changed since a state with no false CPs)
  uint64_t count_false_critical(bool frontier_only = false) {
    CK(cudaMemsetAsync(&ws.ctl->counts[0], 0, sizeof(uint64_t), ws.stream));
    pre(kProfDetectAll);
    if (frontier_only)
      k_count_false_list<<<grid_for(n() / 64 + 1, 256, ws.sms, 8), 256, 0, ws.stream>>>(
          s.fdir, s.gdir, s.F, &ws.ctl->f_count, &ws.ctl->counts[0]);
    else
      k_count_false<<<grid_for(n() / 16 + 1, 256, ws.sms, 16), 256, 0, ws.stream>>>(
          s.fdir, s.gdir, n(), &ws.ctl->counts[0]);
    launched(kProfDetectAll);
    ++st.detect_sweeps;
    uint64_t total = 0;
    CK(cudaMemcpyAsync(&total, &ws.ctl->counts[0], sizeof total, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    return total;
  }

  // run_r_loop (edit_engine.cpp:329-366).  Returns true when it stopped on
  // matching labels (the outer loop's postcondition), false on new false CPs.
  // Sparse R batch targets (k_cross -> k_upstream -> restricted jumping ->
  // k_up_targets, see kernels.cuh).  Returns false (nothing emitted) when
  // Up(X) grows past max_up, in which case the caller runs the full pass.
  uint32_t x_cap() const { return std::max<uint32_t>(1u << 16, n() / kSparseUpDivisor); }
  uint32_t* xlist(int fam, int k) {
    ws.xbuf.ensure(size_t(x_cap()) * 4 * 4);
    return ws.xbuf.as<uint32_t>() + size_t(fam * 2 + k) * x_cap();
  }

  bool sparse_targets(uint64_t& mism) {
    reset_ctl();
    ws.push_ctl();
    const uint32_t max_up = x_cap();
    uint32_t* fa = list(2);
    uint32_t* fb = list(3);
    uint32_t* up = lab(2);
    uint32_t* upidx = fin(0);
    uint64_t* pv = reinterpret_cast<uint64_t*>(list(2));
    // 1. crossing lists X for both families: re-evaluate only 64-vertex chunks
    //    whose codes changed since the last X (change marks cstamp >= x_mark)
    const bool incremental = x_valid;
    uint32_t nxs[2];
    CK(cudaMemsetAsync(ws.ctl->sp_count, 0, 4 * sizeof(uint32_t), ws.stream));
    {
      // from scratch (no X yet): every chunk is changed (since = 0) and there
      // are no old entries -- one pass for both families (round 2: -1.3 ms per
      // C4 step against one k_cross per family)
      const uint32_t since = incremental ? x_mark : 0u;
      const uint32_t na = incremental ? x_n[0] : 0u, nd = incremental ? x_n[1] : 0u;
      pre(kProfSparse);
      k_cross_chunks<<<grid_for(uint64_t(na) + nd + n() / 64, 256, ws.sms, 16), 256, 0,
                       ws.stream>>>(s.gdir, s.fM, s.fm, geo, s.cstamp, since, xlist(0, x_cur[0]), na,
                                    xlist(1, x_cur[1]), nd, xlist(0, x_cur[0] ^ 1),
                                    xlist(1, x_cur[1] ^ 1), ws.ctl->sp_count, x_cap());
      launched(kProfSparse);
    }
    x_mark = ws.next_mark;  // changes after this X carry marks >= x_mark
    CK(cudaMemcpyAsync(nxs, ws.ctl->sp_count, sizeof nxs, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    x_valid = false;
    for (int fam = 0; fam < 2; ++fam) {
      if (trace) std::fprintf(stderr, "[mssz] sparse fam=%d |X|=%u%s\n", fam, nxs[fam],
                              incremental ? " (incremental)" : "");
      if (nxs[fam] > max_up) return false;
    }
    for (int fam = 0; fam < 2; ++fam) {
      x_cur[fam] ^= 1;
      x_n[fam] = nxs[fam];
    }
    x_valid = true;
    // 2. per family: Up(X) by backward BFS, restricted labels, targets
    for (int fam = 0; fam < 2; ++fam) {
      const uint32_t mark = ws.next_mark++;
      const uint32_t* fL = fam ? s.fm : s.fM;
      const uint32_t nx = x_n[fam];
      if (nx == 0) continue;  // no crossing step: every label of this family matches
      CK(cudaMemsetAsync(ws.ctl->sp_count, 0, 4 * sizeof(uint32_t), ws.stream));
      CK(cudaMemcpyAsync(fa, xlist(fam, x_cur[fam]), size_t(nx) * 4, cudaMemcpyDeviceToDevice,
                         ws.stream));
      CK(cudaMemcpyAsync(&ws.ctl->sp_count[1], &x_n[fam], 4, cudaMemcpyHostToDevice, ws.stream));
      CK(cudaMemcpyAsync(&ws.ctl->sp_count[3], &nx, 4, cudaMemcpyHostToDevice, ws.stream));
      pre(kProfSparse);
      k_up_seed<<<grid_for(nx, 256, ws.sms, 16), 256, 0, ws.stream>>>(fa, nx, s.fmark, mark, up);
      launched(kProfSparse);
      // backward BFS (cooperative)
      int occ = 0;
      void* fn = geo.ndims == 2 ? (void*)k_upstream<2> : (void*)k_upstream<3>;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 512, 0));
      const int blocks = ws.sms * std::max(1, std::min(occ, 2));
      Geom gg = geo;
      const uint8_t* gd = s.gdir;
      uint32_t* fmk = s.fmark;
      uint32_t mk = mark, mu = max_up, ml = kSparseMaxLevels;
      Ctl* ctl = ws.ctl;
      void* args[] = {(void*)&gd, &gg, &fam, &fmk, &mk, &fa, &fb, &up, &mu, &ml, &ctl};
      if (trace) std::fprintf(stderr, "[mssz] sparse fam=%d nx=%u: k_upstream blocks=%d occ=%d\n", fam, nx, blocks, occ);
      pre(kProfSparse);
      CK(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(512), args, 0, ws.stream));
      launched(kProfSparse);
      ws.pull_ctl();
      if (trace)
        std::fprintf(stderr, "[mssz] sparse fam=%d |Up|=%u levels=%u abort=%u\n", fam,
                     ws.hctl->sp_count[3], ws.hctl->sp_levels, ws.hctl->sp_abort);
      if (ws.hctl->sp_abort) return false;
      const uint32_t nup = ws.hctl->sp_count[3];
      st.sparse_up += nup;
      pre(kProfSparse);
      k_up_index<<<grid_for(nup, 256, ws.sms, 16), 256, 0, ws.stream>>>(up, nup, upidx);
      launched(kProfSparse);
      pre(kProfSparse);
      k_up_parent<<<grid_for(nup, 256, ws.sms, 16), 256, 0, ws.stream>>>(up, nup, s.gdir, geo, fam,
                                                                         s.fmark, mark, upidx, fL, pv);
      launched(kProfSparse);
      for (int round = 0;; round += 4) {
        CK(cudaMemsetAsync(ws.ctl->flags, 0, 4 * sizeof(uint32_t), ws.stream));
        for (int r = 0; r < 4; ++r) {
          pre(kProfSparse);
          k_up_jump<<<grid_for(nup, 256, ws.sms, 16), 256, 0, ws.stream>>>(pv, nup, &ws.ctl->flags[r]);
          launched(kProfSparse);
        }
        uint32_t flags[4];
        CK(cudaMemcpyAsync(flags, ws.ctl->flags, sizeof flags, cudaMemcpyDeviceToHost, ws.stream));
        ws.sync();
        if (trace) std::fprintf(stderr, "[mssz] sparse fam=%d jump round %d flags %u%u%u%u\n", fam, round, flags[0], flags[1], flags[2], flags[3]);
        if (!flags[3]) break;
        if (round > 70) fail(MSSZ_CU_ERR_INTERNAL, "integral line cycle in the sparse R pass");
      }
      pre(kProfSparse);
      k_up_targets<T><<<grid_for(nup, 256, ws.sms, 16), 256, 0, ws.stream>>>(s, up, nup, fam, pv,
                                                                             list(0));
      launched(kProfSparse);
    }
    ws.pull_ctl();
    if (ws.hctl->status == kStatusTroubleMax)
      fail(MSSZ_CU_ERR_INTERNAL, "troublemaker target is an extremum (stale critical report)");
    mism = ws.hctl->mism;
    ++st.sparse_iterations;
    return true;
  }

  // run_r_loop (edit_engine.cpp:329-366).  Returns true when it stopped on
  // matching labels (the outer loop's postcondition), false on new false CPs.
  // Incremental after the first iteration: only label tiles whose direction
  // codes changed are re-resolved, and only tiles that are dirty or whose exits
  // changed their final label recompute their mismatch bits.
  bool run_r_loop() {
    ++code_epoch;  // conservatively: R batches refresh codes
    uint64_t iters = 0;
    bool first = true;
    TileStore ts = tile_store();
    struct DirtyOff {
      State<T>& s;
      ~DirtyOff() { s.tdirty = nullptr; }
    } dirty_off{s};
    s.tdirty = ts.dirty;
    uint64_t& last_mism = r_last_mism;  // persists across run_r_loop calls
    bool& full_valid = r_full_valid;     // incremental full-pass state is current
    bool last_frontier = false;          // the previous batch refreshed via k_frontier
    for (;;) {
      const auto t_it = std::chrono::steady_clock::now();
      // the C-loop that precedes this call ended with every kind empty, so the
      // gate (edit_engine.cpp:338) can only fire after one of our own batches
      if (!first && count_false_critical(/*frontier_only=*/last_frontier) != 0) return false;
      uint64_t mism = 0;
      bool done = false;
      const bool try_sparse = last_mism < n() / kSparseMismDivisor;
      if (trace)
        std::fprintf(stderr, "[mssz] R decide first=%d last_mism=%llu limit=%u sparse=%d\n", int(first),
                     (unsigned long long)last_mism, n() / kSparseMismDivisor, int(try_sparse));
      if (try_sparse) done = sparse_targets(mism);
      if (!done) {
        label_pass(s.gdir, lab(2), lab(3), /*only_dirty=*/full_valid, /*finish=*/false);
        mism = r_targets(/*all_tiles=*/!full_valid);
        full_valid = true;
      } else {
        full_valid = false;
        CK(cudaMemsetAsync(ts.dirty, 0, ts.ntiles, ws.stream));
      }
      first = false;
      last_mism = mism;
      if (mism == 0) return true;
      if (++iters > opt.r_cap) fail(MSSZ_CU_ERR_NON_CONVERGENCE, "R-loop exceeded its iteration cap");
      // claim each distinct target once and lower it (edit_engine.cpp:344-358)
      const uint32_t ntargets = ws.hctl->list_count[0];
      const uint32_t batch = ws.next_batch++;
      CK(cudaMemsetAsync(&ws.ctl->s_count, 0, 2 * sizeof(uint32_t), ws.stream));
      pre(kProfFix);
      k_fix_list<T><<<grid_for(ntargets, 256, ws.sms, 16), 256, 0, ws.stream>>>(s, list(0), ntargets,
                                                                                0, batch);
      launched(kProfFix);
      uint32_t applied = 0;
      CK(cudaMemcpyAsync(&applied, &ws.ctl->s_count, 4, cudaMemcpyDeviceToHost, ws.stream));
      ws.sync();
      if (applied == 0)
        fail(MSSZ_CU_ERR_NON_CONVERGENCE, "R-loop stalled: every troublemaker is at its floor");
      const uint32_t mark = ws.next_mark++;
      if (applied > n() / kRHugeDivisor) {
        directions(s.g, s.gdir);  // large batch: one streaming sweep beats 15 RMWs per edit
        CK(cudaMemsetAsync(ts.dirty, 1, ts.ntiles, ws.stream));
        last_frontier = false;
      } else {
        last_frontier = true;
        pre(kProfFrontier);
        if (geo.ndims == 2)
          k_frontier<T, 2><<<grid_for(uint64_t(applied) * 8, 256, ws.sms, 16), 256, 0, ws.stream>>>(s, applied, mark);
        else
          k_frontier<T, 3><<<grid_for(uint64_t(applied) * 16, 256, ws.sms, 16), 256, 0, ws.stream>>>(s, applied, mark);
        launched(kProfFrontier);
      }
      st.effective_edits += applied;
      ++st.r_iterations;
      if (trace)
        std::fprintf(stderr, "[mssz] R it=%llu mism=%llu targets=%u applied=%u tiles=%llu/%llu %.2f ms\n",
                     (unsigned long long)st.r_iterations, (unsigned long long)mism, ntargets,
                     applied, (unsigned long long)st.label_tiles, (unsigned long long)st.rfix_tiles,
                     1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t_it).count());
      ++r_it;
      on_batch(MSSZ_CU_PHASE_R_ITERATION);
    }
  }

  // Validation + EditState ctor + outer loop + tripwire (edit_engine.cpp:386-428).
  // d_f: original (device), g already holds fhat.
  // fh_ready (optional): g is still being filled (H2D of fhat on the copy
  // stream); the f-side setup -- f's directions and labels, which the
  // reference computes in the EditState ctor -- runs first and overlaps it.
  void run(const T* d_f, double xi, cudaEvent_t fh_ready = nullptr) {
    if (!(xi > 0.0)) fail(MSSZ_CU_ERR_USAGE, "derive_edits requires xi > 0");
    bind(d_f);
    s.xi = xi;
    if (fh_ready) {
      CK(cudaEventRecord(ws.ev[0], ws.stream));
      directions(d_f, ws.fdir.as<uint8_t>());
      CK(cudaEventRecord(ws.ev[1], ws.stream));
      label_pass(s.fdir, lab(0), lab(1), false, true);
      float ms = 0;
      CK(cudaEventSynchronize(ws.ev[1]));
      CK(cudaEventElapsedTime(&ms, ws.ev[0], ws.ev[1]));
      dir_ms += ms;
      CK(cudaStreamWaitEvent(ws.stream, fh_ready, 0));
    }
    reset_ctl();
    ws.push_ctl();
    pre(kProfValidate);
    k_validate<T><<<grid_for(n(), 256, ws.sms, 8), 256, 0, ws.stream>>>(d_f, s.g, n(), xi, ws.ctl);
    launched(kProfValidate);
    ws.pull_ctl();
    if (ws.hctl->nonfinite) fail(MSSZ_CU_ERR_IO, "derive_edits: non-finite input");
    const uint64_t violations = ws.hctl->violations;
    if (violations && !opt.force)
      fail(MSSZ_CU_ERR_BOUND_VIOLATION,
           "%llu vertices violate |f - fhat| <= xi; the preservation guarantee would not hold "
           "(pass force to proceed anyway)",
           (unsigned long long)violations);
    st.input_bound_violations = violations;

    // EditState ctor (edit_engine.cpp:36-56)
    s.touched = nullptr;  // touched == (g != fhat), derived by edit_flags()
    CK(cudaEventRecord(ws.ev[0], ws.stream));
    if (!fh_ready) directions(d_f, ws.fdir.as<uint8_t>());
    directions(s.g, s.gdir);
    CK(cudaEventRecord(ws.ev[1], ws.stream));
    if (!fh_ready) label_pass(s.fdir, lab(0), lab(1), false, true);
    {
      float ms = 0;
      CK(cudaEventSynchronize(ws.ev[1]));
      CK(cudaEventElapsedTime(&ms, ws.ev[0], ws.ev[1]));
      dir_ms += ms;
    }

    bool labels_verified = false;
    for (uint64_t outer = 0;; ++outer) {
      if (outer >= opt.outer_cap)
        fail(MSSZ_CU_ERR_NON_CONVERGENCE,
             "outer loop cap reached after %llu edits (%llu C sub-iterations, %llu R iterations)",
             (unsigned long long)st.effective_edits,
             (unsigned long long)(st.sub_iterations[0] + st.sub_iterations[1] +
                                  st.sub_iterations[2] + st.sub_iterations[3]),
             (unsigned long long)st.r_iterations);
      ++st.outer_iterations;
      outer_it = st.outer_iterations;
      pass_it = r_it = 0;
      const uint64_t before = st.effective_edits;
      run_c_loop();
      const uint64_t after_c = st.effective_edits;
      labels_verified = run_r_loop();
      // zero-edit R pass that ended on matching labels == the tripwire's state
      labels_verified = labels_verified && st.effective_edits == after_c;
      if (st.effective_edits == before) break;
    }
    // postcondition tripwire (edit_engine.cpp:423-428).  When the final outer
    // pass made no edits, its R-loop already evaluated exactly this state
    // (zero false critical points, zero mismatches); recompute otherwise.
    if (!labels_verified) {
      if (count_false_critical() != 0)
        fail(MSSZ_CU_ERR_INTERNAL, "converged with false critical points");
      label_pass(s.gdir, lab(2), lab(3), false, false);
      if (r_targets(true) != 0) fail(MSSZ_CU_ERR_INTERNAL, "converged with mismatched labels");
    }
  }

  // edits() (edit_engine.cpp:368-378) into device buffers; returns the count.
  uint64_t compact(const uint8_t* flag, uint8_t want, const T* vals, uint64_t* d_idx, T* d_val,
                   uint64_t base = 0) {
    const uint64_t ntiles = (static_cast<uint64_t>(n()) + kCompactTile - 1) / kCompactTile;
    uint32_t* tiles = ws.tiles.as<uint32_t>();
    pre(kProfCompact);
    k_compact_count<<<static_cast<uint32_t>(ntiles), kCompactThreads, 0, ws.stream>>>(flag, n(), want, tiles);
    launched(kProfCompact);
    pre(kProfCompact);
    k_scan_tiles<<<1, 1024, 0, ws.stream>>>(tiles, ntiles, &ws.ctl->mism);
    launched(kProfCompact);
    pre(kProfCompact);
    k_compact_write<T><<<static_cast<uint32_t>(ntiles), kCompactThreads, 0, ws.stream>>>(
        flag, n(), want, vals, tiles, d_idx, d_val, base);
    launched(kProfCompact);
    uint64_t total = 0;
    CK(cudaMemcpyAsync(&total, &ws.ctl->mism, sizeof total, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    return total;
  }

  // EditSet membership (edit_engine.cpp:368-378): g != fhat, into ws.touched
  const uint8_t* edit_flags() {
    uint8_t* flag = ws.touched.as<uint8_t>();
    pre(kProfCompact);
    k_flag_changed<T><<<grid_for(n() / 4 + 1, 256, ws.sms, 8), 256, 0, ws.stream>>>(s.g, fhat, n(), flag);
    launched(kProfCompact);
    return flag;
  }

  // device EditSet buffers inside the (now idle) worklist block
  uint64_t* edit_idx() const { return reinterpret_cast<uint64_t*>(ws.lists.p); }
  T* edit_val() const {
    return reinterpret_cast<T*>(static_cast<char*>(ws.lists.p) +
                                static_cast<uint64_t>((n() + 63) & ~63u) * 8);
  }

  void finish_stats() {
    resolve_profile();
    st.direction_seconds = dir_ms * 1e-3;
    st.label_seconds = lab_ms * 1e-3;
  }
};

mssz_cu_options resolve(const mssz_cu_options* o) {
  mssz_cu_options d;
  mssz_cu_default_options(&d);
  return o ? *o : d;
}

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms * 1e-3;
}

// Host-buffer entry shared by derive_edits / derive_edits_into.
template <class T>
void derive_host(int ndims, const uint64_t* dims, const T* f, const T* fh, double xi,
                 const mssz_cu_options* o, uint64_t** idx_alloc, T** val_alloc, uint64_t* idx_buf,
                 T* val_buf, uint64_t capacity, uint64_t* count_out, mssz_cu_stats* stats_out) {
  const Geom geo = make_geom(ndims, dims);
  if (!f || !fh || !count_out) fail(MSSZ_CU_ERR_USAGE, "null input/output pointer");
  const mssz_cu_options opt = resolve(o);
  Workspace& ws = workspace(opt.device);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, sizeof(T));
  Engine<T> eng(ws, geo, opt);
  cudaEvent_t t0, t1, t2, t3;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventCreate(&t2));
  CK(cudaEventCreate(&t3));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  };
  cudaEvent_t evs[4] = {t0, t1, t2, t3};
  EvGuard guard{evs};
  CK(cudaEventRecord(t0, ws.stream));
  ws.fh.ensure(sizeof(T) * ((geo.n + 63) & ~uint64_t(63)));
  // f first on the engine stream; fhat on the copy stream while f's directions
  // and labels are computed (Engine::run with fh_ready)
  CK(cudaMemcpyAsync(ws.f.p, f, sizeof(T) * geo.n, cudaMemcpyHostToDevice, ws.stream));
  CK(cudaEventRecord(t2, ws.stream));  // f is in: fhat follows on the copy engine
  CK(cudaStreamWaitEvent(ws.copy_stream, t2, 0));
  CK(cudaMemcpyAsync(ws.fh.p, fh, sizeof(T) * geo.n, cudaMemcpyHostToDevice, ws.copy_stream));
  CK(cudaMemcpyAsync(ws.g.p, ws.fh.p, sizeof(T) * geo.n, cudaMemcpyDeviceToDevice, ws.copy_stream));
  CK(cudaEventRecord(t1, ws.copy_stream));
  eng.fhat = ws.fh.as<T>();
  eng.run(ws.f.as<T>(), xi, t1);
  const uint64_t count = eng.compact(eng.edit_flags(), 1, eng.s.g, eng.edit_idx(), eng.edit_val());
  CK(cudaEventRecord(t2, ws.stream));
  uint64_t* hi = idx_buf;
  T* hv = val_buf;
  if (idx_alloc) {
    hi = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (count ? count : 1)));
    hv = static_cast<T*>(std::malloc(sizeof(T) * (count ? count : 1)));
    if (!hi || !hv) {
      std::free(hi);
      std::free(hv);
      throw std::bad_alloc();
    }
  } else if (count > capacity) {
    *count_out = count;
    fail(MSSZ_CU_ERR_USAGE, "output capacity %llu < %llu edits", (unsigned long long)capacity,
         (unsigned long long)count);
  }
  if (count) {
    CK(cudaMemcpyAsync(hi, eng.edit_idx(), sizeof(uint64_t) * count, cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaMemcpyAsync(hv, eng.edit_val(), sizeof(T) * count, cudaMemcpyDeviceToHost, ws.stream));
  }
  CK(cudaEventRecord(t3, ws.stream));
  ws.sync();
  eng.st.touched = count;
  eng.finish_stats();
  eng.st.h2d_seconds = elapsed_s(t0, t1);
  eng.st.device_seconds = elapsed_s(t1, t2);
  eng.st.d2h_seconds = elapsed_s(t2, t3);
  if (idx_alloc) {
    *idx_alloc = hi;
    *val_alloc = hv;
  }
  *count_out = count;
  if (stats_out) *stats_out = eng.st;
}

template <class T>
void derive_device(int ndims, const uint64_t* dims, const T* d_f, const T* d_fh, double xi,
                   const mssz_cu_options* o, uint64_t* d_idx, T* d_val, uint64_t capacity,
                   uint64_t* count_out, mssz_cu_stats* stats_out, void* stream) {
  const Geom geo = make_geom(ndims, dims);
  if (!d_f || !d_fh || !count_out) fail(MSSZ_CU_ERR_USAGE, "null input/output pointer");
  const mssz_cu_options opt = resolve(o);
  Workspace& ws = workspace(opt.device);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, sizeof(T));
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  if (caller) {
    CK(cudaEventRecord(ws.ev[0], caller));
    CK(cudaStreamWaitEvent(ws.stream, ws.ev[0], 0));
  }
  Engine<T> eng(ws, geo, opt);
  cudaEvent_t t0, t1;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventRecord(t0, ws.stream));
  CK(cudaMemcpyAsync(ws.g.p, d_fh, sizeof(T) * geo.n, cudaMemcpyDeviceToDevice, ws.stream));
  eng.fhat = d_fh;
  eng.run(d_f, xi);
  const uint64_t count = eng.compact(eng.edit_flags(), 1, eng.s.g, eng.edit_idx(), eng.edit_val());
  if (count > capacity) {
    *count_out = count;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    fail(MSSZ_CU_ERR_USAGE, "output capacity %llu < %llu edits", (unsigned long long)capacity,
         (unsigned long long)count);
  }
  if (count) {
    CK(cudaMemcpyAsync(d_idx, eng.edit_idx(), sizeof(uint64_t) * count, cudaMemcpyDeviceToDevice, ws.stream));
    CK(cudaMemcpyAsync(d_val, eng.edit_val(), sizeof(T) * count, cudaMemcpyDeviceToDevice, ws.stream));
  }
  CK(cudaEventRecord(t1, ws.stream));
  ws.sync();
  eng.st.device_seconds = elapsed_s(t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (caller) {
    CK(cudaEventRecord(ws.ev[1], ws.stream));
    CK(cudaStreamWaitEvent(caller, ws.ev[1], 0));
  }
  eng.st.touched = count;
  eng.finish_stats();
  *count_out = count;
  if (stats_out) *stats_out = eng.st;
}

// ---- stand-alone kernel exports (parity harness) ----

template <class T>
struct Scratch {  // host-in/host-out helper for the per-kernel exports
  Workspace& ws;
  Geom geo;
  Scratch(Workspace& w, const Geom& g) : ws(w), geo(g) {}
};

template <class T>
void compute_dirs_host(int ndims, const uint64_t* dims, const T* values, uint8_t* codes,
                       uint64_t* asc, uint64_t* desc) {
  const Geom geo = make_geom(ndims, dims);
  if (!values) fail(MSSZ_CU_ERR_USAGE, "null values");
  mssz_cu_options opt;
  mssz_cu_default_options(&opt);
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, sizeof(T));
  Engine<T> eng(ws, geo, opt);
  CK(cudaMemcpyAsync(ws.g.p, values, sizeof(T) * geo.n, cudaMemcpyHostToDevice, ws.stream));
  eng.directions(ws.g.as<T>(), ws.gdir.as<uint8_t>());
  if (codes)
    CK(cudaMemcpyAsync(codes, ws.gdir.p, geo.n, cudaMemcpyDeviceToHost, ws.stream));
  if (asc && desc) {
    uint64_t* da = reinterpret_cast<uint64_t*>(ws.lists.p);
    uint64_t* dd = da + ((geo.n + 63) & ~63u);
    k_codes_to_ids<<<grid_for(geo.n, 256, ws.sms, 16), 256, 0, ws.stream>>>(ws.gdir.as<uint8_t>(), geo, da, dd);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(asc, da, 8ull * geo.n, cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaMemcpyAsync(desc, dd, 8ull * geo.n, cudaMemcpyDeviceToHost, ws.stream));
  }
  ws.sync();
}

template <class T>
__global__ void k_kind_flags(const uint8_t* __restrict__ fdir, const uint8_t* __restrict__ gdir,
                             uint32_t n, int kind, uint8_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    out[v] = kind_match(kind, fdir[v], gdir[v]) ? 1 : 0;
}

template <class T>
void detect_host(int ndims, const uint64_t* dims, const T* f, const T* g, int kind,
                 uint64_t* counts, uint64_t* lists, uint64_t* count_out) {
  const Geom geo = make_geom(ndims, dims);
  if (!f || !g) fail(MSSZ_CU_ERR_USAGE, "null input");
  if (kind > 3) fail(MSSZ_CU_ERR_USAGE, "kind must be 0..3");
  mssz_cu_options opt;
  mssz_cu_default_options(&opt);
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, sizeof(T));
  Engine<T> eng(ws, geo, opt);
  eng.bind(ws.f.as<T>());
  CK(cudaMemcpyAsync(ws.f.p, f, sizeof(T) * geo.n, cudaMemcpyHostToDevice, ws.stream));
  CK(cudaMemcpyAsync(ws.g.p, g, sizeof(T) * geo.n, cudaMemcpyHostToDevice, ws.stream));
  eng.directions(ws.f.as<T>(), ws.fdir.as<uint8_t>());
  eng.directions(ws.g.as<T>(), ws.gdir.as<uint8_t>());
  uint8_t* cls = ws.touched.as<uint8_t>();
  uint64_t* d_idx = eng.edit_idx();
  if (kind < 0) {
    eng.reset_ctl();
    ws.push_ctl();
    k_detect_all<<<grid_for((geo.n + 15) / 16, 256, ws.sms, 16), 256, 0, ws.stream>>>(
        ws.fdir.as<uint8_t>(), ws.gdir.as<uint8_t>(), geo.n, ws.ctl->counts, cls);
    CK_LAUNCH();
    for (int k = 0; k < 4; ++k) {
      const uint64_t c = eng.compact(cls, static_cast<uint8_t>(k), static_cast<const T*>(nullptr), d_idx, nullptr);
      counts[k] = c;
      if (lists && c)
        CK(cudaMemcpyAsync(lists + static_cast<uint64_t>(k) * geo.n, d_idx, 8 * c, cudaMemcpyDeviceToHost, ws.stream));
      ws.sync();
    }
  } else {
    k_kind_flags<T><<<grid_for(geo.n, 256, ws.sms, 16), 256, 0, ws.stream>>>(
        ws.fdir.as<uint8_t>(), ws.gdir.as<uint8_t>(), geo.n, kind, cls);
    CK_LAUNCH();
    const uint64_t c = eng.compact(cls, 1, static_cast<const T*>(nullptr), d_idx, nullptr);
    if (c) CK(cudaMemcpyAsync(lists, d_idx, 8 * c, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    *count_out = c;
  }
}

// R-batch target set of run_r_loop (edit_engine.cpp:336-352) for one (f, g)
// pair behind the R gate (:338; a pair with false critical points has no R
// batch): the deduplicated troublemaker targets v_t of every mismatched vertex,
// through the engine's own tiled pass (k_rfix_tiles -> k_expand_targets) or its
// sparse Up(X) pass, sorted.  info = {false critical points (the R gate,
// :338), divergent mismatched (vertex, family) pairs = distinct troublemaker
// sources v_i, path used (0 tiled, 1 sparse)}.
template <class T>
void r_targets_host(int ndims, const uint64_t* dims, const T* f, const T* g, int mode,
                    uint64_t* targets, uint64_t* count_out, uint64_t* info) {
  const Geom geo = make_geom(ndims, dims);
  if (!f || !g || !targets || !count_out || !info) fail(MSSZ_CU_ERR_USAGE, "null pointer");
  if (mode != 0 && mode != 1) fail(MSSZ_CU_ERR_USAGE, "mode must be 0 (tiled) or 1 (sparse)");
  mssz_cu_options opt;
  mssz_cu_default_options(&opt);
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, sizeof(T));
  Engine<T> eng(ws, geo, opt);
  eng.bind(ws.f.as<T>());
  CK(cudaMemcpyAsync(ws.f.p, f, sizeof(T) * geo.n, cudaMemcpyHostToDevice, ws.stream));
  CK(cudaMemcpyAsync(ws.g.p, g, sizeof(T) * geo.n, cudaMemcpyHostToDevice, ws.stream));
  auto tr = [&](const char* what) {
    if (eng.trace) {
      CK(cudaStreamSynchronize(ws.stream));
      std::fprintf(stderr, "[mssz] r_targets mode=%d n=%u: %s\n", mode, geo.n, what);
    }
  };
  tr("start");
  eng.directions(ws.f.as<T>(), ws.fdir.as<uint8_t>());
  eng.directions(eng.s.g, eng.s.gdir);
  tr("directions");
  eng.label_pass(eng.s.fdir, eng.lab(0), eng.lab(1), false, true);
  tr("f labels");
  info[0] = eng.count_false_critical();
  tr("gate");
  if (info[0] != 0) {  // the R gate (edit_engine.cpp:338): run_r_loop hands back to the C loop
    *count_out = 0;
    info[1] = 0;
    info[2] = 0;
    return;
  }
  uint64_t mism = 0;
  int path = 0;
  if (mode == 1 && eng.sparse_targets(mism)) path = 1;
  tr(path ? "sparse done" : "sparse skipped");
  if (path == 0) {
    eng.label_pass(eng.s.gdir, eng.lab(2), eng.lab(3), false, false);
    tr("g labels");
    mism = eng.r_targets(true);
    tr("tiled targets");
  }
  const uint32_t nt = ws.hctl->list_count[0];
  std::vector<uint32_t> t(nt);
  if (nt) CK(cudaMemcpyAsync(t.data(), eng.list(0), 4ull * nt, cudaMemcpyDeviceToHost, ws.stream));
  ws.sync();
  std::sort(t.begin(), t.end());
  t.erase(std::unique(t.begin(), t.end()), t.end());
  for (size_t i = 0; i < t.size(); ++i) targets[i] = t[i];
  *count_out = t.size();
  info[1] = mism;
  info[2] = static_cast<uint64_t>(path);
}

template <class T>
void elementwise_host(uint64_t n, const T* g, const T* f, double xi, T* out, uint8_t* moved,
                      bool floor_only) {
  if (n == 0) return;
  if (!f || !out) fail(MSSZ_CU_ERR_USAGE, "null pointer");
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  DevBuf a, b, c, d;
  struct Rel {
    DevBuf* x[4];
    ~Rel() {
      for (auto* p : x) p->release();
    }
  } rel{{&a, &b, &c, &d}};
  a.ensure(sizeof(T) * n);
  b.ensure(sizeof(T) * n);
  c.ensure(sizeof(T) * n);
  d.ensure(n);
  CK(cudaMemcpyAsync(b.p, f, sizeof(T) * n, cudaMemcpyHostToDevice, ws.stream));
  const uint32_t blocks = grid_for(n, 256, ws.sms, 16);
  if (floor_only) {
    k_floor<T><<<blocks, 256, 0, ws.stream>>>(n, b.as<T>(), xi, c.as<T>());
  } else {
    CK(cudaMemcpyAsync(a.p, g, sizeof(T) * n, cudaMemcpyHostToDevice, ws.stream));
    k_lower_step<T><<<blocks, 256, 0, ws.stream>>>(n, a.as<T>(), b.as<T>(), xi, c.as<T>(), d.as<uint8_t>());
  }
  CK_LAUNCH();
  CK(cudaMemcpyAsync(out, c.p, sizeof(T) * n, cudaMemcpyDeviceToHost, ws.stream));
  if (moved && !floor_only) CK(cudaMemcpyAsync(moved, d.p, n, cudaMemcpyDeviceToHost, ws.stream));
  ws.sync();
}

// apply_edits (edit_engine.cpp:437-450)
template <class T>
void apply_host(uint64_t n, const T* fh, const uint64_t* idx, const T* vals, uint64_t count, T* out) {
  if (!fh || !out || (count && (!idx || !vals))) fail(MSSZ_CU_ERR_USAGE, "null pointer");
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  DevBuf a, b, c, d;
  struct Rel {
    DevBuf* x[4];
    ~Rel() {
      for (auto* p : x) p->release();
    }
  } rel{{&a, &b, &c, &d}};
  a.ensure(sizeof(T) * (n ? n : 1));
  b.ensure(8 * (count ? count : 1));
  c.ensure(sizeof(T) * (count ? count : 1));
  d.ensure(4);
  CK(cudaMemsetAsync(d.p, 0, 4, ws.stream));
  CK(cudaMemcpyAsync(a.p, fh, sizeof(T) * n, cudaMemcpyHostToDevice, ws.stream));
  // d = {bad index, indices not non-decreasing}.  The reference applies the
  // edits in order, so for a repeated index the LAST value wins: with sorted
  // indices that is the last element of each run (k_scatter), otherwise a
  // winner pass (atomicMax of position + 1 per vertex) picks it.
  uint32_t flags[2] = {0, 0};
  d.ensure(8);
  CK(cudaMemsetAsync(d.p, 0, 8, ws.stream));
  if (count) {
    CK(cudaMemcpyAsync(b.p, idx, 8 * count, cudaMemcpyHostToDevice, ws.stream));
    CK(cudaMemcpyAsync(c.p, vals, sizeof(T) * count, cudaMemcpyHostToDevice, ws.stream));
    k_scatter_check<<<grid_for(count, 256, ws.sms, 16), 256, 0, ws.stream>>>(count, b.as<uint64_t>(), n,
                                                                          d.as<uint32_t>());
    CK_LAUNCH();
    CK(cudaMemcpyAsync(flags, d.p, 8, cudaMemcpyDeviceToHost, ws.stream));
    ws.sync();
    if (flags[0]) fail(MSSZ_CU_ERR_CORRUPT_ARCHIVE, "edit index out of range");  // no output
    if (!flags[1]) {
      k_scatter<T><<<grid_for(count, 256, ws.sms, 16), 256, 0, ws.stream>>>(count, b.as<uint64_t>(), c.as<T>(),
                                                                           a.as<T>());
      CK_LAUNCH();
    } else {
      DevBuf win;
      struct RelW {
        DevBuf& w;
        ~RelW() { w.release(); }
      } relw{win};
      win.ensure(8 * (n ? n : 1));
      CK(cudaMemsetAsync(win.p, 0, 8 * n, ws.stream));
      k_scatter_winner<<<grid_for(count, 256, ws.sms, 16), 256, 0, ws.stream>>>(count, b.as<uint64_t>(),
                                                                               win.as<unsigned long long>());
      k_scatter_won<T><<<grid_for(count, 256, ws.sms, 16), 256, 0, ws.stream>>>(
          count, b.as<uint64_t>(), c.as<T>(), win.as<unsigned long long>(), a.as<T>());
      CK_LAUNCH();
      CK(cudaMemcpyAsync(out, a.p, sizeof(T) * n, cudaMemcpyDeviceToHost, ws.stream));
      ws.sync();
      return;
    }
  }
  CK(cudaMemcpyAsync(out, a.p, sizeof(T) * n, cudaMemcpyDeviceToHost, ws.stream));
  ws.sync();
}

void labels_host(int ndims, const uint64_t* dims, const uint64_t* asc, const uint64_t* desc,
                 uint64_t* M, uint64_t* m) {
  const Geom geo = make_geom(ndims, dims);
  if (!asc || !desc || !M || !m) fail(MSSZ_CU_ERR_USAGE, "null pointer");
  mssz_cu_options opt;
  mssz_cu_default_options(&opt);
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, 4);
  Engine<float> eng(ws, geo, opt);
  const uint64_t np = (geo.n + 63) & ~63u;
  uint64_t* da = reinterpret_cast<uint64_t*>(ws.lists.p);
  uint64_t* dd = da + np;
  uint32_t* LM = eng.lab(0);
  uint32_t* Lm = eng.lab(1);
  CK(cudaMemcpyAsync(da, asc, 8ull * geo.n, cudaMemcpyHostToDevice, ws.stream));
  CK(cudaMemcpyAsync(dd, desc, 8ull * geo.n, cudaMemcpyHostToDevice, ws.stream));
  eng.reset_ctl();
  ws.push_ctl();
  const uint32_t blocks = grid_for(geo.n, 256, ws.sms, 16);
  k_u64_to_u32<<<blocks, 256, 0, ws.stream>>>(da, LM, geo.n, &ws.ctl->status);
  k_u64_to_u32<<<blocks, 256, 0, ws.stream>>>(dd, Lm, geo.n, &ws.ctl->status);
  CK_LAUNCH();
  ws.pull_ctl();
  if (ws.hctl->status) fail(MSSZ_CU_ERR_INTERNAL, "direction field references a vertex out of range");
  eng.jump_to_fixpoint(LM, Lm);
  k_u32_to_u64<<<blocks, 256, 0, ws.stream>>>(LM, da, geo.n);
  k_u32_to_u64<<<blocks, 256, 0, ws.stream>>>(Lm, dd, geo.n);
  CK_LAUNCH();
  CK(cudaMemcpyAsync(M, da, 8ull * geo.n, cudaMemcpyDeviceToHost, ws.stream));
  CK(cudaMemcpyAsync(m, dd, 8ull * geo.n, cudaMemcpyDeviceToHost, ws.stream));
  ws.sync();
}

void classify_host(uint64_t n, const uint64_t* asc, const uint64_t* desc, uint64_t* maxima,
                   uint64_t* nmax, uint64_t* minima, uint64_t* nmin) {
  if (n == 0 || n >= 0xFFFFFFFFull) fail(MSSZ_CU_ERR_USAGE, "bad vertex count");
  const uint64_t dims[2] = {n, 1};
  Geom geo{};
  geo.ndims = 2;
  geo.X = static_cast<uint32_t>(n);
  geo.Y = 1;
  geo.Z = 1;
  geo.XY = geo.X;
  geo.n = static_cast<uint32_t>(n);
  (void)dims;
  mssz_cu_options opt;
  mssz_cu_default_options(&opt);
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, 4);
  Engine<float> eng(ws, geo, opt);
  const uint64_t np = (n + 63) & ~uint64_t(63);
  uint64_t* da = reinterpret_cast<uint64_t*>(ws.lists.p);
  uint64_t* dd = da + np;
  CK(cudaMemcpyAsync(da, asc, 8ull * n, cudaMemcpyHostToDevice, ws.stream));
  CK(cudaMemcpyAsync(dd, desc, 8ull * n, cudaMemcpyHostToDevice, ws.stream));
  k_extremum_flags<<<grid_for(n, 256, ws.sms, 16), 256, 0, ws.stream>>>(da, dd, n, ws.fdir.as<uint8_t>(), ws.gdir.as<uint8_t>());
  CK_LAUNCH();
  uint64_t* out = reinterpret_cast<uint64_t*>(ws.lab.p);
  *nmax = eng.compact(ws.fdir.as<uint8_t>(), 1, static_cast<const float*>(nullptr), out, nullptr);
  if (*nmax) CK(cudaMemcpyAsync(maxima, out, 8 * *nmax, cudaMemcpyDeviceToHost, ws.stream));
  ws.sync();
  *nmin = eng.compact(ws.gdir.as<uint8_t>(), 1, static_cast<const float*>(nullptr), out, nullptr);
  if (*nmin) CK(cudaMemcpyAsync(minima, out, 8 * *nmin, cudaMemcpyDeviceToHost, ws.stream));
  ws.sync();
}

}  // namespace
}  // namespace mssz_b200

using namespace mssz_b200;

extern "C" {

void mssz_cu_default_options(mssz_cu_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->outer_cap = 1000;
  o->subloop_cap = 640;
  o->r_cap = 100000;
  o->force = 0;
  o->device = -1;
}

const char* mssz_cu_last_error(void) { return g_last_error.c_str(); }
int mssz_cu_batch_phase(uint64_t out[3]) {
  if (!out) return MSSZ_CU_ERR_USAGE;
  for (int i = 0; i < 3; ++i) out[i] = g_phase[i];
  return MSSZ_CU_OK;
}
void mssz_cu_free(void* p) { std::free(p); }
const char* mssz_cu_version(void) { return "mssz-b200 0.1 (sm_100a)"; }

int mssz_cu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int mssz_cu_release_workspace(int device) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (device < 0) CK(cudaGetDevice(&device));
    if (device < static_cast<int>(g_ws.size()) && g_ws[device]) {
      std::lock_guard<std::mutex> lk2(g_ws[device]->mu);
      g_ws[device]->release();
    }
  });
}

#define MSSZ_CU_DEFINE_TYPED(SUF, T)                                                              \
  int mssz_cu_derive_edits_##SUF(int ndims, const uint64_t* dims, const T* f, const T* fh,        \
                                 double xi, const mssz_cu_options* opt, uint64_t** idx, T** val,  \
                                 uint64_t* count, mssz_cu_stats* st) {                            \
    return guarded([&] {                                                                          \
      if (!idx || !val) fail(MSSZ_CU_ERR_USAGE, "null output pointer");                          \
      derive_host<T>(ndims, dims, f, fh, xi, opt, idx, val, nullptr, nullptr, 0, count, st);     \
    });                                                                                           \
  }                                                                                               \
  int mssz_cu_derive_edits_into_##SUF(int ndims, const uint64_t* dims, const T* f, const T* fh,   \
                                      double xi, const mssz_cu_options* opt, uint64_t* idx,       \
                                      T* val, uint64_t cap, uint64_t* count, mssz_cu_stats* st) { \
    return guarded([&] {                                                                          \
      derive_host<T>(ndims, dims, f, fh, xi, opt, nullptr, nullptr, idx, val, cap, count, st);   \
    });                                                                                           \
  }                                                                                               \
  int mssz_cu_derive_edits_device_##SUF(int ndims, const uint64_t* dims, const T* f,              \
                                        const T* fh, double xi, const mssz_cu_options* opt,       \
                                        uint64_t* idx, T* val, uint64_t cap, uint64_t* count,     \
                                        mssz_cu_stats* st, void* stream) {                        \
    return guarded([&] {                                                                          \
      derive_device<T>(ndims, dims, f, fh, xi, opt, idx, val, cap, count, st, stream);           \
    });                                                                                           \
  }                                                                                               \
  int mssz_cu_compute_directions_##SUF(int ndims, const uint64_t* dims, const T* v,              \
                                       uint64_t* asc, uint64_t* desc) {                           \
    return guarded([&] {                                                                          \
      if (!asc || !desc) fail(MSSZ_CU_ERR_USAGE, "null output pointer");                         \
      compute_dirs_host<T>(ndims, dims, v, nullptr, asc, desc);                                   \
    });                                                                                           \
  }                                                                                               \
  int mssz_cu_compute_direction_codes_##SUF(int ndims, const uint64_t* dims, const T* v,         \
                                            uint8_t* codes) {                                     \
    return guarded([&] {                                                                          \
      if (!codes) fail(MSSZ_CU_ERR_USAGE, "null output pointer");                                \
      compute_dirs_host<T>(ndims, dims, v, codes, nullptr, nullptr);                              \
    });                                                                                           \
  }                                                                                               \
  int mssz_cu_detect_false_critical_##SUF(int ndims, const uint64_t* dims, const T* f,           \
                                          const T* g, uint64_t counts[4], uint64_t* lists) {      \
    return guarded([&] {                                                                          \
      if (!counts) fail(MSSZ_CU_ERR_USAGE, "null counts");                                       \
      detect_host<T>(ndims, dims, f, g, -1, counts, lists, nullptr);                              \
    });                                                                                           \
  }                                                                                               \
  int mssz_cu_detect_kind_##SUF(int ndims, const uint64_t* dims, const T* f, const T* g,         \
                                int kind, uint64_t* list, uint64_t* count) {                      \
    return guarded([&] {                                                                          \
      if (!list || !count || kind < 0) fail(MSSZ_CU_ERR_USAGE, "bad arguments");                 \
      detect_host<T>(ndims, dims, f, g, kind, nullptr, list, count);                              \
    });                                                                                           \
  }                                                                                               \
  int mssz_cu_lower_step_##SUF(uint64_t n, const T* g, const T* f, double xi, T* out,           \
                               uint8_t* moved) {                                                  \
    return guarded([&] {                                                                          \
      if (!g) fail(MSSZ_CU_ERR_USAGE, "null g");                                                 \
      elementwise_host<T>(n, g, f, xi, out, moved, false);                                        \
    });                                                                                           \
  }                                                                                               \
  int mssz_cu_representable_floor_##SUF(uint64_t n, const T* f, double xi, T* out) {            \
    return guarded([&] { elementwise_host<T>(n, nullptr, f, xi, out, nullptr, true); });          \
  }                                                                                               \
  int mssz_cu_apply_edits_##SUF(uint64_t n, const T* fh, const uint64_t* idx, const T* vals,     \
                                uint64_t count, T* out) {                                         \
    return guarded([&] { apply_host<T>(n, fh, idx, vals, count, out); });                         \
  }                                                                                               \
  int mssz_cu_r_targets_##SUF(int ndims, const uint64_t* dims, const T* f, const T* g, int mode, \
                              uint64_t* targets, uint64_t* count, uint64_t* info) {               \
    return guarded([&] { r_targets_host<T>(ndims, dims, f, g, mode, targets, count, info); });   \
  }

MSSZ_CU_DEFINE_TYPED(f32, float)
MSSZ_CU_DEFINE_TYPED(f64, double)

int mssz_cu_compute_labels(int ndims, const uint64_t* dims, const uint64_t* asc,
                           const uint64_t* desc, uint64_t* M, uint64_t* m) {
  return guarded([&] { labels_host(ndims, dims, asc, desc, M, m); });
}

int mssz_cu_classify_critical(uint64_t n, const uint64_t* asc, const uint64_t* desc,
                              uint64_t* maxima, uint64_t* n_max, uint64_t* minima,
                              uint64_t* n_min) {
  return guarded([&] {
    if (!asc || !desc || !maxima || !minima || !n_max || !n_min)
      fail(MSSZ_CU_ERR_USAGE, "null pointer");
    classify_host(n, asc, desc, maxima, n_max, minima, n_min);
  });
}

}  // extern "C"

#include "shard_api.cuh"
#include "verify.cuh"
#include "base_codec.cuh"
#include "edit_codec.cuh"
