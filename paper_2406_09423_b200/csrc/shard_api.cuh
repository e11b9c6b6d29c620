// C-ABI of the z-slab sharded engine (include/mssz_cuda.h, "z-slab sharding").
#pragma once

#include "shard.cuh"

namespace mssz_b200 {
namespace {

// Global geometry of a z-slab sharded field: extents validated as
// build_topology (grid.cpp:39-55, cap 2^40 vertices); the vertex count may
// exceed 2^32 -- global ids are u64 in the sharded engine -- but a plane and
// every rank's window must fit the device's u32 ids.  n is left 0 (the global
// count is XY * Z in u64; only windows carry a device-sized n).
Geom make_slab_geom(int ndims, const uint64_t* dims) {
  if (ndims != 3) fail(MSSZ_CU_ERR_USAGE, "z-slab sharding needs a 3D grid");
  if (!dims) fail(MSSZ_CU_ERR_USAGE, "dims is null");
  const uint64_t cap = uint64_t(1) << 40;
  uint64_t count = 1;
  for (int a = 0; a < 3; ++a) {
    if (dims[a] < 2) fail(MSSZ_CU_ERR_USAGE, "every grid extent must be >= 2");
    if (dims[a] > cap / count) fail(MSSZ_CU_ERR_USAGE, "grid exceeds the address-space cap");
    count *= dims[a];
  }
  if (dims[0] * dims[1] >= 0xFFFFFFFFull || dims[2] >= 0xFFFFFFFFull)
    fail(MSSZ_CU_ERR_USAGE, "a z plane of %llu vertices exceeds the device's u32 ids",
         (unsigned long long)(dims[0] * dims[1]));
  Geom g{};
  g.ndims = 3;
  g.nst = 14;
  g.X = static_cast<uint32_t>(dims[0]);
  g.Y = static_cast<uint32_t>(dims[1]);
  g.Z = static_cast<uint32_t>(dims[2]);
  g.XY = g.X * g.Y;
  g.n = 0;
  for (int k = 0; k < 16; ++k) g.off[k] = 0;
  for (int k = 0; k < g.nst; ++k) {
    int dx, dy, dz;
    stencil<3>(k, dx, dy, dz);
    const int64_t o = dx + dy * static_cast<int64_t>(g.X) + dz * static_cast<int64_t>(g.XY);
    g.off[k] = static_cast<int32_t>(static_cast<uint32_t>(static_cast<uint64_t>(o)));
  }
  return g;
}

Geom window_geom(const Geom& gg, const SlabPlan& pl) {
  const uint64_t d[3] = {gg.X, gg.Y, pl.wz1 - pl.wz0};
  return make_geom(3, d);
}

// One rank's derive_edits on its window.  Inputs are the window planes
// [wz0, wz1) (host or device); the slab's part of the EditSet (global ids) is
// written at out + (concat ? offset : 0).
template <class T>
void slab_run(Transport& tr, Workspace& ws, SlabBufs& sb, const Geom& gg, const SlabPlan& pl,
              const mssz_cu_options& opt, const T* f_win, const T* fh_win, bool host_io, double xi,
              uint64_t* idx_out, T* val_out, uint64_t capacity, bool concat, uint64_t* count_out,
              uint64_t* offset_out, mssz_cu_stats* st_out) {
  if (opt.on_batch) fail(MSSZ_CU_ERR_USAGE, "on_batch is not supported by the sharded engine");
  const Geom gw = window_geom(gg, pl);
  ws.ensure(gw.n, sizeof(T));
  SlabEngine<T> se(tr, ws, sb, pl, gg, gw, opt);
  cudaEvent_t ev[4];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  const cudaMemcpyKind in_kind = host_io ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  CK(cudaEventRecord(ev[0], ws.stream));
  CK(cudaMemcpyAsync(ws.f.p, f_win, sizeof(T) * gw.n, in_kind, ws.stream));
  CK(cudaMemcpyAsync(ws.g.p, fh_win, sizeof(T) * gw.n, in_kind, ws.stream));
  CK(cudaEventRecord(ev[1], ws.stream));
  se.run(ws.f.as<T>(), xi);
  uint64_t count = 0, offset = 0, total = 0;
  se.compact(se.eng.edit_idx(), se.eng.edit_val(), count, offset, total);
  CK(cudaEventRecord(ev[2], ws.stream));
  const uint64_t need = concat ? total : count;
  if (need > capacity) {
    *count_out = need;
    fail(MSSZ_CU_ERR_USAGE, "output capacity %llu < %llu edits", (unsigned long long)capacity,
         (unsigned long long)need);
  }
  const uint64_t at = concat ? offset : 0;
  const cudaMemcpyKind out_kind = host_io ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (count) {
    CK(cudaMemcpyAsync(idx_out + at, se.eng.edit_idx(), sizeof(uint64_t) * count, out_kind, ws.stream));
    CK(cudaMemcpyAsync(val_out + at, se.eng.edit_val(), sizeof(T) * count, out_kind, ws.stream));
  }
  CK(cudaEventRecord(ev[3], ws.stream));
  ws.sync();
  se.st().touched = total;
  se.eng.finish_stats();
  se.st().h2d_seconds = host_io ? elapsed_s(ev[0], ev[1]) : 0.0;
  se.st().device_seconds = elapsed_s(ev[1], ev[2]);
  se.st().d2h_seconds = host_io ? elapsed_s(ev[2], ev[3]) : 0.0;
  *count_out = concat ? total : count;
  if (offset_out) *offset_out = offset;
  if (st_out) *st_out = se.st();
}

// P virtual ranks as host threads (devices[r % ndevices]); the EditSet is the
// concatenation of the slab parts in rank order, i.e. globally sorted.
template <class T>
void slabs_local(int P, const int* devices, int ndevices, int ndims, const uint64_t* dims, const T* f,
                 const T* fh, double xi, const mssz_cu_options* o, uint64_t* idx, T* val, uint64_t capacity,
                 uint64_t* count_out, mssz_cu_stats* st_out) {
  if (ndims != 3) fail(MSSZ_CU_ERR_USAGE, "z-slab sharding needs a 3D grid");
  if (!f || !fh || !count_out || (capacity && (!idx || !val)))
    fail(MSSZ_CU_ERR_USAGE, "null input/output pointer");
  const Geom gg = make_slab_geom(ndims, dims);
  const mssz_cu_options opt = resolve(o);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(MSSZ_CU_ERR_CUDA, "no CUDA device available; the B200 engine has no CPU fallback");
  std::vector<int> devs;
  if (devices && ndevices > 0) {
    devs.assign(devices, devices + ndevices);
  } else {
    int d = opt.device;
    if (d < 0) CK(cudaGetDevice(&d));
    devs.push_back(d);
  }
  for (int d : devs)
    if (d < 0 || d >= ndev) fail(MSSZ_CU_ERR_USAGE, "device %d out of range (%d devices)", d, ndev);
  std::vector<SlabPlan> plans;
  for (int r = 0; r < P; ++r) plans.push_back(slab_plan(gg.Z, P, r));
  LocalHub hub(P);
  std::vector<Fail> errs(P);
  std::vector<int> failed(P, 0);
  std::vector<mssz_cu_stats> stats(P);
  std::vector<uint64_t> counts(P, 0);
  std::vector<std::thread> th;
  for (int r = 0; r < P; ++r) {
    th.emplace_back([&, r] {
      Workspace ws;
      SlabBufs sb;
      try {
        const int dev = devs[r % devs.size()];
        ws.init(dev);
        LocalTransport tr(&hub, r);
        const SlabPlan& pl = plans[r];
        const uint64_t off = uint64_t(pl.wz0) * gg.XY;
        mssz_cu_options ro = opt;
        ro.device = dev;
        slab_run<T>(tr, ws, sb, gg, pl, ro, f + off, fh + off, true, xi, idx, val, capacity, true,
                    &counts[r], nullptr, &stats[r]);
      } catch (const Fail& e) {
        errs[r] = e;
        failed[r] = 1;
        hub.abort();
      } catch (const std::bad_alloc&) {
        errs[r] = Fail{MSSZ_CU_ERR_CUDA, "host allocation failed"};
        failed[r] = 1;
        hub.abort();
      }
      sb.release();
      ws.destroy();
    });
  }
  for (auto& t : th) t.join();
  // report the root cause, not a peer's "another slab failed"
  int first = -1;
  for (int r = 0; r < P; ++r)
    if (failed[r] && (first < 0 || errs[first].msg == "another slab failed")) first = r;
  if (first >= 0) {
    if (errs[first].code == MSSZ_CU_ERR_USAGE && counts[first]) *count_out = counts[first];
    throw errs[first];
  }
  *count_out = counts[0];
  if (st_out) {
    mssz_cu_stats s = stats[0];
    s.kernel_launches = 0;
    for (int r = 0; r < P; ++r) s.kernel_launches += stats[r].kernel_launches;
    *st_out = s;
  }
}

}  // namespace
}  // namespace mssz_b200

struct mssz_cu_comm {
  mssz_b200::NcclTransport tr;
  int device = 0;
  mssz_b200::SlabBufs sb;
};

extern "C" {

int mssz_cu_slab_range(uint64_t Z, int nranks, int rank, uint64_t out[4]) {
  return mssz_b200::guarded([&] {
    if (!out) mssz_b200::fail(MSSZ_CU_ERR_USAGE, "null output");
    const mssz_b200::SlabPlan p = mssz_b200::slab_plan(Z, nranks, rank);
    out[0] = p.z0;
    out[1] = p.z1;
    out[2] = p.wz0;
    out[3] = p.wz1;
  });
}

int mssz_cu_comm_unique_id(uint8_t* id) {
  return mssz_b200::guarded([&] {
    if (!id) mssz_b200::fail(MSSZ_CU_ERR_USAGE, "null id");
    ncclUniqueId u;
    NK(mssz_b200::nccl().GetUniqueId(&u));
    static_assert(sizeof(u) == MSSZ_CU_UNIQUE_ID_BYTES, "NCCL unique id size");
    std::memcpy(id, &u, sizeof u);
  });
}

int mssz_cu_comm_init(const uint8_t* id, int nranks, int rank, int device, mssz_cu_comm** out) {
  return mssz_b200::guarded([&] {
    using namespace mssz_b200;
    if (!id || !out) fail(MSSZ_CU_ERR_USAGE, "null argument");
    if (nranks < 1 || nranks > kMaxSlabs || rank < 0 || rank >= nranks)
      fail(MSSZ_CU_ERR_USAGE, "bad rank %d of %d", rank, nranks);
    workspace(device);  // validates the device and makes it current
    auto c = std::make_unique<mssz_cu_comm>();
    CK(cudaGetDevice(&c->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    c->tr.rank = rank;
    c->tr.size = nranks;
    c->tr.device = c->device;
    NK(nccl().CommInitRank(&c->tr.comm, nranks, u, rank));
    *out = c.release();
  });
}

int mssz_cu_comm_destroy(mssz_cu_comm* c) {
  return mssz_b200::guarded([&] {
    if (!c) return;
    CK(cudaSetDevice(c->device));
    c->sb.release();
    delete c;
  });
}

#define MSSZ_CU_DEFINE_SLAB(SUF, T)                                                                  \
  int mssz_cu_derive_edits_slab_##SUF(mssz_cu_comm* c, int ndims, const uint64_t* dims, const T* f,  \
                                      const T* fh, double xi, const mssz_cu_options* o,              \
                                      uint64_t* idx, T* val, uint64_t cap, uint64_t* count,          \
                                      uint64_t* offset, mssz_cu_stats* st) {                         \
    return mssz_b200::guarded([&] {                                                                  \
      using namespace mssz_b200;                                                                     \
      if (!c) fail(MSSZ_CU_ERR_USAGE, "null communicator");                                          \
      if (ndims != 3) fail(MSSZ_CU_ERR_USAGE, "z-slab sharding needs a 3D grid");                    \
      if (!f || !fh || !count || (cap && (!idx || !val))) fail(MSSZ_CU_ERR_USAGE, "null pointer");   \
      const Geom gg = make_slab_geom(ndims, dims);                                                   \
      mssz_cu_options opt = resolve(o);                                                              \
      opt.device = c->device;                                                                        \
      Workspace& ws = workspace(c->device);                                                          \
      std::lock_guard<std::mutex> lk(ws.mu);                                                         \
      slab_run<T>(c->tr, ws, c->sb, gg, slab_plan(gg.Z, c->tr.size, c->tr.rank), opt, f, fh, true,   \
                  xi, idx, val, cap, false, count, offset, st);                                      \
    });                                                                                              \
  }                                                                                                  \
  int mssz_cu_derive_edits_slab_device_##SUF(                                                        \
      mssz_cu_comm* c, int ndims, const uint64_t* dims, const T* f, const T* fh, double xi,          \
      const mssz_cu_options* o, uint64_t* idx, T* val, uint64_t cap, uint64_t* count,                \
      uint64_t* offset, mssz_cu_stats* st, void* stream) {                                           \
    return mssz_b200::guarded([&] {                                                                  \
      using namespace mssz_b200;                                                                     \
      if (!c) fail(MSSZ_CU_ERR_USAGE, "null communicator");                                          \
      if (ndims != 3) fail(MSSZ_CU_ERR_USAGE, "z-slab sharding needs a 3D grid");                    \
      if (!f || !fh || !count || (cap && (!idx || !val))) fail(MSSZ_CU_ERR_USAGE, "null pointer");   \
      const Geom gg = make_slab_geom(ndims, dims);                                                   \
      mssz_cu_options opt = resolve(o);                                                              \
      opt.device = c->device;                                                                        \
      Workspace& ws = workspace(c->device);                                                          \
      std::lock_guard<std::mutex> lk(ws.mu);                                                         \
      cudaStream_t caller = static_cast<cudaStream_t>(stream);                                       \
      if (caller) {                                                                                  \
        CK(cudaEventRecord(ws.ev[0], caller));                                                       \
        CK(cudaStreamWaitEvent(ws.stream, ws.ev[0], 0));                                             \
      }                                                                                              \
      slab_run<T>(c->tr, ws, c->sb, gg, slab_plan(gg.Z, c->tr.size, c->tr.rank), opt, f, fh, false,  \
                  xi, idx, val, cap, false, count, offset, st);                                      \
      if (caller) {                                                                                  \
        CK(cudaEventRecord(ws.ev[1], ws.stream));                                                    \
        CK(cudaStreamWaitEvent(caller, ws.ev[1], 0));                                                \
      }                                                                                              \
    });                                                                                              \
  }                                                                                                  \
  int mssz_cu_derive_edits_slabs_local_##SUF(int nslabs, const int* devices, int ndevices, int ndims, \
                                             const uint64_t* dims, const T* f, const T* fh,          \
                                             double xi, const mssz_cu_options* o, uint64_t* idx,     \
                                             T* val, uint64_t cap, uint64_t* count,                  \
                                             mssz_cu_stats* st) {                                    \
    return mssz_b200::guarded([&] {                                                                  \
      mssz_b200::slabs_local<T>(nslabs, devices, ndevices, ndims, dims, f, fh, xi, o, idx, val, cap,  \
                                count, st);                                                          \
    });                                                                                              \
  }

MSSZ_CU_DEFINE_SLAB(f32, float)
MSSZ_CU_DEFINE_SLAB(f64, double)

}  // extern "C"
