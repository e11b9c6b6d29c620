// z-slab sharded correction loop: one rank per GPU, each owning a
// contiguous range of z planes of one 3D field.
//
// Layout per rank.  Rank r of P owns planes [z0, z1) (z0 = floor(Z r / P)) and
// keeps a WINDOW of planes [z0 - 2, z1 + 2) (clipped to the grid) in HBM: two
// halo planes of values per side.  Local vertex ids are window ids; the global
// id of local v is v + wz0 * XY (slabs are index-contiguous, grid.hpp:41-43).
//   * directions are computed over the whole window; they are exact on the
//     owned planes and on the first halo plane (the "active" range), whose
//     stencil stays inside the window;
//   * owner-computes: a fix batch runs over every listed item of the active
//     range (owned items and the neighbours' boundary-plane items) and lowers
//     only OWNED targets, from the pre-batch value, with the single-device claim
//     rule -- so every target is lowered by exactly one rank and Σ applied is the
//     reference's applied count;
//   * after each batch a rank sends the targets it lowered in its first / last
//     two owned planes, as (global id, new value) pairs, to rank-1 / rank+1,
//     which patch their halo values and add them to the refresh seed S;
//   * every control decision (list empty, cap, stall, FPmin fallback, gate,
//     mismatch count) is taken on values all-gathered across ranks, so all
//     ranks follow the same schedule and the P-rank run is bit-identical to the
//     single-device engine: same edit set, same EditStats.
// Labels (mss.cpp:51-97): each rank labels its window with the halo planes
// masked as extrema, so a chain that leaves the slab stops at its first
// off-slab vertex (an exit, always on a neighbour's boundary plane).  The ranks
// all-gather the provisional labels of their first and last owned planes and
// resolve every table entry to its chain terminus by pointer chasing on the
// gathered table; a vertex's final label is then its provisional label, or
// that label's table entry when the label lies on a boundary plane.  The R loop
// is incremental as on a single device (dirty label tiles, tile mismatch bits),
// plus tiles whose labels depend on a boundary-table entry that changed.
//
// Transports: NCCL (one process per GPU; ncclAllGather for the per-batch
// status records and the label tables, grouped ncclSend/ncclRecv with the z
// neighbours for boundary edits), and an in-process transport that runs P
// virtual ranks as host threads (on one or several devices) for testing the
// sharded schedule on a single GPU.
#pragma once

#include <dlfcn.h>
#include <nccl.h>  // types only: every NCCL entry point is resolved with dlsym

#include <condition_variable>
#include <thread>

namespace mssz_b200 {
namespace {

// (global id, lowered value) of a boundary target.
template <class T>
struct BEdit {
  uint64_t idx;
  T val;
};

// Per-batch status record, all-gathered across ranks.
struct alignas(8) Rec {
  uint64_t list;      // current worklist size (active range)
  uint64_t applied;   // targets this rank lowered
  uint64_t to_lo;     // boundary edits for rank - 1
  uint64_t to_hi;     // boundary edits for rank + 1
  uint64_t false_cnt; // false critical points (owned)
  uint64_t mism;      // divergent mismatched vertices (owned) / compaction count
  uint64_t status;
  uint64_t nonfinite;
  uint64_t violations;
  uint64_t err;       // label-table resolution hit a cycle
  uint64_t parked;    // C loop: parked worklist items (see k_subloop)
};

__global__ void k_rec(const Ctl* __restrict__ ctl, uint32_t cur, const uint32_t* __restrict__ err,
                      Rec* __restrict__ out) {
  if (threadIdx.x != 0) return;
  Rec r;
  r.list = ctl->list_count[cur];
  r.applied = ctl->s_count;
  r.to_lo = ctl->bnd[0];
  r.to_hi = ctl->bnd[1];
  r.false_cnt = ctl->counts[0];
  r.mism = ctl->mism;
  r.status = ctl->status;
  r.nonfinite = ctl->nonfinite;
  r.violations = ctl->violations;
  r.err = *err;
  r.parked = ctl->park_count;
  *out = r;
}

// fix over a device-sized list (run_subloop / run_r_loop batch, edit_engine.cpp:255-275, :344-358)
template <class T>
__global__ void __launch_bounds__(256) k_slab_fix(State<T> s, const uint32_t* __restrict__ list,
                                                  const uint32_t* count, int rule, uint32_t batch,
                                                  uint32_t* retry, uint32_t* retry_count, bool park) {
  fix_batch(s, list, *count, rule, batch, &s.ctl->s_count,
            static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
            static_cast<uint64_t>(gridDim.x) * blockDim.x, retry, retry_count, park ? s.F : nullptr,
            park ? &s.ctl->park_count : nullptr);
}

// Parked items (see k_subloop) of the host-driven C loop.  k_unpark_list clears
// the flag of the worklist items parked by the batch being redone;
// k_unpark_merge appends every still-parked P entry to the worklist (append =
// false: only clears the flags, after a streaming refresh rebuilt the list).
__global__ void __launch_bounds__(256) k_unpark_list(const uint32_t* __restrict__ list, const uint32_t* count,
                                                     uint32_t* __restrict__ fmark) {
  const uint32_t n = *count;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = list[i];
    if (__ldcg(fmark + v) == kParked) fmark[v] = 0u;
  }
}
__global__ void __launch_bounds__(256) k_unpark_merge(const uint32_t* __restrict__ P, const uint32_t* np_ptr,
                                                      uint32_t* __restrict__ fmark, uint32_t* list,
                                                      uint32_t* count, bool append) {
  const uint32_t np = *np_ptr;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t wb = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~uint64_t(31); wb < np;
       wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    bool keep = false;
    uint32_t v = 0;
    if (i < np) {
      v = __ldcg(P + i);
      keep = __ldcg(fmark + v) == kParked && atomicCAS(&fmark[v], kParked, 0u) == kParked;
    }
    if (append) warp_append(keep, v, list, count);
  }
}

// Owned targets lowered in this batch that lie on the first / last two owned
// planes -> (global id, value) for the neighbour below / above.
template <class T>
__global__ void __launch_bounds__(256) k_pack_boundary(State<T> s, uint32_t lo_end, uint32_t hi_begin,
                                                       int has_lo, int has_hi, uint64_t base,
                                                       BEdit<T>* __restrict__ to_lo,
                                                       BEdit<T>* __restrict__ to_hi) {
  const uint32_t n = s.ctl->s_count;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t wb = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~uint64_t(31);
       wb < n; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    uint32_t t = 0;
    bool a = false, b = false;
    if (i < n) {
      t = __ldcg(s.S + i);
      a = has_lo && t < lo_end;
      b = has_hi && t >= hi_begin;
    }
    const T v = (a || b) ? __ldcg(s.g + t) : T(0);
    const uint32_t pa = warp_reserve(a ? 1u : 0u, &s.ctl->bnd[0]);
    const uint32_t pb = warp_reserve(b ? 1u : 0u, &s.ctl->bnd[1]);
    if (a) to_lo[pa] = BEdit<T>{t + base, v};
    if (b) to_hi[pb] = BEdit<T>{t + base, v};
  }
}

// Received boundary edits: patch the halo values and append the halo vertices
// to the refresh seed S (after this rank's own targets).
template <class T>
__global__ void __launch_bounds__(256) k_unpack_boundary(State<T> s, const BEdit<T>* __restrict__ a,
                                                         uint32_t na, const BEdit<T>* __restrict__ b,
                                                         uint32_t nb, uint64_t base) {
  const uint64_t n = static_cast<uint64_t>(na) + nb;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t wb = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~uint64_t(31);
       wb < n; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    uint32_t v = 0;
    if (i < n) {
      const BEdit<T> e = i < na ? a[i] : b[i - na];
      v = static_cast<uint32_t>(e.idx - base);
      s.g[v] = e.val;
    }
    const uint32_t p = warp_reserve(i < n ? 1u : 0u, &s.ctl->s_count);
    if (i < n) s.S[p] = v;
  }
}

// frontier refresh of a C batch straight into the next worklist (see frontier_update)
template <class T, int DIM>
__global__ void __launch_bounds__(256) k_slab_frontier(State<T> s, uint32_t ns, uint32_t mark, int kind,
                                                       uint32_t* next, uint32_t* next_count) {
  frontier_update<T, DIM>(s, ns, mark, &s.ctl->f_count,
                          static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                          static_cast<uint64_t>(gridDim.x) * blockDim.x, kind, next, next_count);
}

__global__ void __launch_bounds__(256) k_slab_rebuild(const uint32_t* __restrict__ retry,
                                                      const uint32_t* nr, const uint32_t* __restrict__ fmark,
                                                      uint32_t mark, uint32_t* nxt, uint32_t* nxt_count) {
  rebuild_retry(retry, *nr, fmark, mark, nxt, nxt_count,
                static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

// detect_kind (edit_engine.cpp:104-132) over vertex range [lo, hi), 16 per thread.
__global__ void __launch_bounds__(256) k_detect_range(const uint8_t* __restrict__ fdir,
                                                      const uint8_t* __restrict__ gdir, uint32_t lo,
                                                      uint32_t hi, int kind, uint32_t* __restrict__ list,
                                                      uint32_t* count) {
  const uint64_t c0 = lo / 16, c1 = (static_cast<uint64_t>(hi) + 15) / 16;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t wb = c0 + ((static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~uint64_t(31));
       wb < c1; wb += stride) {
    const uint64_t c = wb + (threadIdx.x & 31);
    uint32_t mask = 0;
    if (c < c1) {
      const uint64_t v0 = c * 16;
      if (v0 >= lo && v0 + 16 <= hi) {
        const uint4 f = __ldg(reinterpret_cast<const uint4*>(fdir + v0));
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(gdir + v0));
        mask = bytes_to_nibble(kind_bytes(kind, f.x, g.x)) |
               bytes_to_nibble(kind_bytes(kind, f.y, g.y)) << 4 |
               bytes_to_nibble(kind_bytes(kind, f.z, g.z)) << 8 |
               bytes_to_nibble(kind_bytes(kind, f.w, g.w)) << 12;
      } else {
        for (int j = 0; j < 16; ++j)
          if (v0 + j >= lo && v0 + j < hi && kind_match(kind, fdir[v0 + j], gdir[v0 + j]))
            mask |= 1u << j;
      }
    }
    const uint32_t base = warp_reserve(__popc(mask), count);
    uint32_t pos = base;
    while (mask) {
      const int j = __ffs(mask) - 1;
      mask &= mask - 1;
      list[pos++] = static_cast<uint32_t>(c * 16 + j);
    }
  }
}

// First-match false-critical count (edit_engine.cpp:134-158) over [lo, hi), or
// over the frontier list F restricted to [lo, hi) when F != nullptr.
__global__ void __launch_bounds__(256) k_count_false_range(const uint8_t* __restrict__ fdir,
                                                           const uint8_t* __restrict__ gdir,
                                                           uint32_t lo, uint32_t hi,
                                                           const uint32_t* __restrict__ F,
                                                           const uint32_t* nF, uint64_t* total) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t c = 0;
  if (F) {
    const uint32_t n = *nF;
    for (uint64_t i = tid; i < n; i += stride) {
      const uint32_t u = F[i];
      if (u >= lo && u < hi) c += __popc(false_cp_bytes(fdir[u], gdir[u]) & 0xFFu);
    }
  } else {
    const uint64_t q0 = (static_cast<uint64_t>(lo) + 15) / 16, q1 = hi / 16;
    for (uint64_t q = q0 + tid; q < q1; q += stride) {
      const uint4 f = __ldg(reinterpret_cast<const uint4*>(fdir) + q);
      const uint4 gg = __ldg(reinterpret_cast<const uint4*>(gdir) + q);
      c += __popc(false_cp_bytes(f.x, gg.x)) + __popc(false_cp_bytes(f.y, gg.y)) +
           __popc(false_cp_bytes(f.z, gg.z)) + __popc(false_cp_bytes(f.w, gg.w));
    }
    if (tid < 32) {  // ragged head and tail (fewer than 16 vertices each)
      const uint64_t hend = q0 * 16 < hi ? q0 * 16 : hi;
      for (uint64_t v = lo + tid; v < hend; v += 32) c += __popc(false_cp_bytes(fdir[v], gdir[v]) & 0xFFu);
      for (uint64_t v = (q1 * 16 > hend ? q1 * 16 : hend) + tid; v < hi; v += 32)
        c += __popc(false_cp_bytes(fdir[v], gdir[v]) & 0xFFu);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c)
    atomicAdd(reinterpret_cast<unsigned long long*>(total), static_cast<unsigned long long>(c));
}

// Window labels of the first / last owned plane -> this rank's table part
// [family][side][xy] (global ids).  Label = fin[prov[v]] (label_pass without
// its finish phase: prov is a root or a resolved exit).
__global__ void __launch_bounds__(256) k_publish_labels(const uint32_t* __restrict__ M,
                                                        const uint32_t* __restrict__ m,
                                                        const uint32_t* __restrict__ finM,
                                                        const uint32_t* __restrict__ finm, uint32_t XY,
                                                        uint32_t own_lo, uint32_t own_hi, uint64_t base,
                                                        uint64_t* __restrict__ tab) {
  const uint64_t total = 4ull * XY;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int fam = static_cast<int>(i / (2ull * XY));
    const int side = static_cast<int>((i / XY) & 1);
    const uint32_t xy = static_cast<uint32_t>(i % XY);
    const uint32_t v = side ? own_hi - XY + xy : own_lo + xy;
    tab[i] = static_cast<uint64_t>(fam ? finm[m[v]] : finM[M[v]]) + base;
  }
}

// Resolves every gathered table entry to its chain terminus.  An entry's label
// is final when it is not on a boundary plane, or when its own entry holds
// itself (a boundary extremum).  Chasing writes every intermediate back, so
// concurrent chasers shorten each other's paths; any value written is an
// ancestor on the same chain, so the fixpoint is the unique terminus.
__global__ void __launch_bounds__(256) k_resolve_table(uint64_t* __restrict__ tab, SlabTable t,
                                                       uint32_t* err) {
  const uint64_t total = static_cast<uint64_t>(t.P) * 4 * t.XY;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int fam = static_cast<int>((e / (2ull * t.XY)) & 1);
    volatile uint64_t* vt = tab;
    uint64_t L = vt[e];
    uint64_t hops = 0;
    for (;;) {
      const int64_t sl = table_slot(t, L, fam);
      if (sl < 0) break;
      const uint64_t L2 = vt[sl];
      if (L2 == L) break;
      L = L2;
      if (++hops > total) {  // a cycle: corrupt direction field
        atomicExch(err, 1u);
        break;
      }
    }
    vt[e] = L;
  }
}

// Final global labels of the active range: provisional label, or its resolved
// table entry when it lies on a boundary plane (halo vertices: their own entry).
__global__ void __launch_bounds__(256) k_final_labels(const uint32_t* __restrict__ M,
                                                      const uint32_t* __restrict__ m,
                                                      const uint32_t* __restrict__ finM,
                                                      const uint32_t* __restrict__ finm,
                                                      const uint64_t* __restrict__ tab, SlabTable t,
                                                      uint32_t lo, uint32_t hi, uint64_t base,
                                                      int resolve, uint64_t* __restrict__ FM,
                                                      uint64_t* __restrict__ Fm) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = lo + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < hi; v += stride) {
    uint64_t a = finM[M[v]] + base, d = finm[m[v]] + base;
    if (resolve) {
      const int64_t sa = table_slot(t, a, 0), sd = table_slot(t, d, 1);
      if (sa >= 0) a = __ldg(tab + sa);
      if (sd >= 0) d = __ldg(tab + sd);
    }
    FM[v] = a;
    Fm[v] = d;
  }
}

// Boundary-table entries that changed since the previous R iteration (the
// resolved table is then kept as the reference for the next one).
__global__ void __launch_bounds__(256) k_table_diff(const uint64_t* __restrict__ tab, uint64_t* __restrict__ prev,
                                                    uint8_t* __restrict__ changed, uint64_t total,
                                                    uint32_t* any) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  bool c_any = false;
  for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const uint64_t a = tab[e];
    const bool c = a != prev[e];
    changed[e] = c ? 1 : 0;
    if (c) {
      prev[e] = a;
      c_any = true;
    }
  }
  if (__any_sync(0xffffffffu, c_any) && (threadIdx.x & 31) == 0) *any = 1u;
}

// Tiles whose final labels depend on changed table entries become "affected":
// tiles holding non-owned window planes (their vertices' labels are table
// entries or chains into them), and tiles with an exit whose final label is an
// off-slab vertex on a changed entry.  CTA per tile.
template <int DIM>
__global__ void __launch_bounds__(256) k_slab_affected(TileStore ts, const uint32_t* __restrict__ finM,
                                                       const uint32_t* __restrict__ finm,
                                                       const uint8_t* __restrict__ changed, const uint32_t* any,
                                                       SlabTable t, Geom g, uint64_t base) {
  using TL = LabelTile<DIM>;
  if (!*any) return;
  const uint32_t b = blockIdx.x;
  const uint32_t ntx = (g.X + TL::TX - 1) / TL::TX, nty = (g.Y + TL::TY - 1) / TL::TY;
  const uint32_t tz = b / (ntx * nty);
  const uint64_t zlo = static_cast<uint64_t>(tz) * TL::TZ, zhi = min(zlo + TL::TZ, static_cast<uint64_t>(g.Z));
  if (zlo * g.XY < ts.own_lo || zhi * g.XY > ts.own_hi) {
    if (threadIdx.x == 0) ts.affected[b] = 1;
    return;
  }
  bool hit = false;
#pragma unroll
  for (int fam = 0; fam < 2; ++fam) {
    const uint32_t* E = ts.E + (static_cast<size_t>(b) * 2 + fam) * ts.surface;
    const uint32_t ne = ts.Ecnt[b * 2 + fam];
    const uint32_t* fin = fam ? finm : finM;
    for (uint32_t k = threadIdx.x; k < ne; k += blockDim.x) {
      const uint32_t L = fin[E[k]];
      if (L < ts.own_lo || L >= ts.own_hi) {
        const int64_t sl = table_slot(t, L + base, fam);
        hit |= sl >= 0 && changed[sl];
      }
    }
  }
  if (__syncthreads_or(hit) && threadIdx.x == 0) ts.affected[b] = 1;
}

// ---------------------------------------------------------------------------
// Transports.

struct Transport {
  int rank = 0, size = 1;
  virtual ~Transport() = default;
  // all-gather of `bytes` per rank from device memory; result in host memory (blocking)
  virtual void allgather_status(const void* d_mine, void* d_all, void* h_all, size_t bytes,
                                cudaStream_t s) = 0;
  // device all-gather (stream-ordered)
  virtual void allgather_dev(const void* d_mine, void* d_all, size_t bytes, cudaStream_t s) = 0;
  // grouped send/recv with rank-1 (lo) and rank+1 (hi); sizes in bytes, 0 = skip
  virtual void neighbor_exchange(const void* to_lo, size_t b_to_lo, const void* to_hi, size_t b_to_hi,
                                 void* from_lo, size_t b_from_lo, void* from_hi, size_t b_from_hi,
                                 cudaStream_t s) = 0;
  virtual void abort() {}
};

// ---- in-process transport: P virtual ranks as host threads ----
struct LocalHub {
  int P;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  std::vector<const void*> p0, p1;
  std::vector<std::vector<uint8_t>> host;
  explicit LocalHub(int p) : P(p), p0(p), p1(p), host(p) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw Fail{MSSZ_CU_ERR_INTERNAL, "another slab failed"};
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
    }
    if (aborted) throw Fail{MSSZ_CU_ERR_INTERNAL, "another slab failed"};
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct LocalTransport : Transport {
  LocalHub* hub;
  std::vector<uint8_t> tmp;
  LocalTransport(LocalHub* h, int r) : hub(h) {
    rank = r;
    size = h->P;
  }
  void allgather_status(const void* d_mine, void*, void* h_all, size_t bytes, cudaStream_t s) override {
    tmp.resize(bytes);
    CK(cudaMemcpyAsync(tmp.data(), d_mine, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    hub->host[rank] = tmp;
    hub->barrier();
    for (int r = 0; r < size; ++r) std::memcpy(static_cast<uint8_t*>(h_all) + r * bytes, hub->host[r].data(), bytes);
    hub->barrier();
  }
  void allgather_dev(const void* d_mine, void* d_all, size_t bytes, cudaStream_t s) override {
    CK(cudaStreamSynchronize(s));
    hub->p0[rank] = d_mine;
    hub->barrier();
    for (int r = 0; r < size; ++r)
      CK(cudaMemcpyAsync(static_cast<uint8_t*>(d_all) + r * bytes, hub->p0[r], bytes, cudaMemcpyDefault, s));
    CK(cudaStreamSynchronize(s));
    hub->barrier();
  }
  void neighbor_exchange(const void* to_lo, size_t, const void* to_hi, size_t, void* from_lo,
                         size_t b_from_lo, void* from_hi, size_t b_from_hi, cudaStream_t s) override {
    CK(cudaStreamSynchronize(s));
    hub->p0[rank] = to_lo;
    hub->p1[rank] = to_hi;
    hub->barrier();
    if (rank > 0 && b_from_lo)
      CK(cudaMemcpyAsync(from_lo, hub->p1[rank - 1], b_from_lo, cudaMemcpyDefault, s));
    if (rank + 1 < size && b_from_hi)
      CK(cudaMemcpyAsync(from_hi, hub->p0[rank + 1], b_from_hi, cudaMemcpyDefault, s));
    CK(cudaStreamSynchronize(s));
    hub->barrier();
  }
  void abort() override { hub->abort(); }
};

// ---- NCCL transport (one process per GPU) ----
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the NCCL already in the process (torch's), else MSSZ_NCCL_LIBRARY (the
    // Python mirror points it at torch's bundled copy, so a later `import torch`
    // finds a compatible libnccl.so.2), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char* path = std::getenv("MSSZ_NCCL_LIBRARY");
    if (!h && path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(h, name)); };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommAbort, "ncclCommAbort");
    sym(api.AllGather, "ncclAllGather");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    if (api.GetUniqueId && api.CommInitRank && api.AllGather && api.Send && api.Recv &&
        api.GroupStart && api.GroupEnd && api.CommDestroy)
      api.h = h;
  });
  if (!api.h) fail(MSSZ_CU_ERR_CUDA, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}

#define NK(call)                                                                           \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      fail(MSSZ_CU_ERR_CUDA, "%s failed: %s", #call,                                       \
           nccl().GetErrorString ? nccl().GetErrorString(r_) : "nccl error");              \
  } while (0)

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  int device = 0;
  void allgather_status(const void* d_mine, void* d_all, void* h_all, size_t bytes, cudaStream_t s) override {
    NK(nccl().AllGather(d_mine, d_all, bytes, ncclUint8, comm, s));
    CK(cudaMemcpyAsync(h_all, d_all, bytes * size, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  void allgather_dev(const void* d_mine, void* d_all, size_t bytes, cudaStream_t s) override {
    NK(nccl().AllGather(d_mine, d_all, bytes, ncclUint8, comm, s));
  }
  void neighbor_exchange(const void* to_lo, size_t b_to_lo, const void* to_hi, size_t b_to_hi,
                         void* from_lo, size_t b_from_lo, void* from_hi, size_t b_from_hi,
                         cudaStream_t s) override {
    if (!b_to_lo && !b_to_hi && !b_from_lo && !b_from_hi) return;
    NK(nccl().GroupStart());
    if (rank > 0) {
      if (b_to_lo) NK(nccl().Send(to_lo, b_to_lo, ncclUint8, rank - 1, comm, s));
      if (b_from_lo) NK(nccl().Recv(from_lo, b_from_lo, ncclUint8, rank - 1, comm, s));
    }
    if (rank + 1 < size) {
      if (b_to_hi) NK(nccl().Send(to_hi, b_to_hi, ncclUint8, rank + 1, comm, s));
      if (b_from_hi) NK(nccl().Recv(from_hi, b_from_hi, ncclUint8, rank + 1, comm, s));
    }
    NK(nccl().GroupEnd());
  }
  void abort() override {
    if (comm && nccl().CommAbort) nccl().CommAbort(comm);
    comm = nullptr;
  }
  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
  }
};

// ---------------------------------------------------------------------------
struct SlabPlan {
  uint32_t P, r, Z;
  uint32_t z0, z1, wz0, wz1;
};

SlabPlan slab_plan(uint64_t Z, int P, int r) {
  if (P < 1 || P > kMaxSlabs) fail(MSSZ_CU_ERR_USAGE, "slab count must be in [1, %d]", kMaxSlabs);
  if (r < 0 || r >= P) fail(MSSZ_CU_ERR_USAGE, "rank %d out of range for %d slabs", r, P);
  if (Z < 2ull * P) fail(MSSZ_CU_ERR_USAGE, "z extent %llu too small for %d slabs (>= 2 planes each)",
                         (unsigned long long)Z, P);
  SlabPlan p{};
  p.P = P;
  p.r = r;
  p.Z = static_cast<uint32_t>(Z);
  p.z0 = static_cast<uint32_t>(Z * r / P);
  p.z1 = static_cast<uint32_t>(Z * (r + 1) / P);
  p.wz0 = p.z0 >= 2 ? p.z0 - 2 : 0;
  p.wz1 = std::min<uint32_t>(p.Z, p.z1 + 2);
  return p;
}

// Workspace extras of the sharded loop.
struct SlabBufs {
  DevBuf tab_mine, tab_all, tab_prev, tchanged, send[2], recv[2], rec, rec_all;
  DevBuf flab;   // final f labels of the window as u64 global ids (FM | Fm)
  DevBuf flags;  // [0] table resolution hit a cycle, [1] a table entry changed
  std::vector<Rec> hrec;
  void release() {
    for (DevBuf* b : {&tab_mine, &tab_all, &tab_prev, &tchanged, &flags, &send[0], &send[1], &recv[0], &recv[1], &rec, &rec_all, &flab})
      b->release();
  }
};

template <class T>
struct SlabEngine {
  Transport& tr;
  Workspace& ws;
  SlabBufs& sb;
  SlabPlan pl;
  Geom gglob;
  Engine<T> eng;
  uint32_t XY = 0, own_lo = 0, own_hi = 0, act_lo = 0, act_hi = 0;
  // global id of window vertex 0 (u64: a sharded field may exceed 2^32
  // vertices) and the same for the EditSet; they differ only under the test
  // bias MSSZ_SLAB_Z_BIAS, which places the field zbias planes deep inside a
  // larger virtual grid so every internal global id exceeds 2^32
  uint64_t base = 0, out_base = 0;
  uint32_t zbias = 0;
  uint64_t n_glob = 0;
  SlabTable stab{};
  bool labels_verified = false;

  SlabEngine(Transport& t, Workspace& w, SlabBufs& b, const SlabPlan& p, const Geom& gg, const Geom& gw,
             const mssz_cu_options& o)
      : tr(t), ws(w), sb(b), pl(p), gglob(gg), eng(w, gw, o) {
    XY = gg.XY;
    if (const char* b = std::getenv("MSSZ_SLAB_Z_BIAS")) zbias = static_cast<uint32_t>(std::strtoul(b, nullptr, 10));
    base = (uint64_t(pl.wz0) + zbias) * XY;
    out_base = uint64_t(pl.wz0) * XY;
    own_lo = (pl.z0 - pl.wz0) * XY;
    own_hi = (pl.z1 - pl.wz0) * XY;
    act_lo = ((pl.z0 > 0 ? pl.z0 - 1 : 0) - pl.wz0) * XY;
    act_hi = (std::min(pl.Z, pl.z1 + 1) - pl.wz0) * XY;
    n_glob = uint64_t(gg.XY) * gg.Z;
    stab.P = pl.P;
    stab.XY = XY;
    for (uint32_t r = 0; r <= pl.P; ++r) stab.z0[r] = static_cast<uint32_t>(uint64_t(pl.Z) * r / pl.P) + zbias;
    const size_t nw = eng.n();
    sb.tab_mine.ensure(size_t(4) * XY * 8);
    sb.tab_all.ensure(size_t(4) * XY * 8 * pl.P);
    sb.tab_prev.ensure(size_t(4) * XY * 8 * pl.P);
    sb.flab.ensure(size_t(2) * ((nw + 63) & ~size_t(63)) * 8);
    sb.tchanged.ensure(size_t(4) * XY * pl.P);
    for (int k = 0; k < 2; ++k) {
      sb.send[k].ensure(size_t(2) * XY * sizeof(BEdit<T>));
      sb.recv[k].ensure(size_t(2) * XY * sizeof(BEdit<T>));
    }
    sb.rec.ensure(sizeof(Rec));
    sb.flags.ensure(16);
    sb.rec_all.ensure(sizeof(Rec) * pl.P);
    sb.hrec.resize(pl.P);
  }

  uint32_t n() const { return eng.n(); }
  mssz_cu_stats& st() { return eng.st; }
  State<T>& s() { return eng.s; }
  uint32_t blocks(uint64_t work, int per_sm = 8) const { return grid_for(work, 256, ws.sms, per_sm); }

  // all-gathered status records of every rank (blocking)
  const std::vector<Rec>& gather() {
    k_rec<<<1, 32, 0, ws.stream>>>(ws.ctl, eng.cur, sb.flags.as<uint32_t>(), sb.rec.as<Rec>());
    CK_LAUNCH();
    tr.allgather_status(sb.rec.p, sb.rec_all.p, sb.hrec.data(), sizeof(Rec), ws.stream);
    return sb.hrec;
  }
  template <class F>
  uint64_t sum(F&& field) const {
    uint64_t t = 0;
    for (const Rec& r : sb.hrec) t += field(r);
    return t;
  }

  void reset_ctl() {
    eng.reset_ctl();
    ws.push_ctl();
  }

  // ---- boundary edits: pack after a fix, exchange, unpack into the halo + S ----
  void pack() {
    CK(cudaMemsetAsync(ws.ctl->bnd, 0, sizeof(uint32_t) * 2, ws.stream));
    const uint32_t lo_end = own_lo + 2 * XY, hi_begin = own_hi - 2 * XY;
    eng.pre(kProfFix);
    k_pack_boundary<T><<<ws.sms, 256, 0, ws.stream>>>(  // grid-stride over |S| (device count)
        s(), lo_end, hi_begin, pl.r > 0, pl.r + 1 < pl.P, base, sb.send[0].as<BEdit<T>>(),
        sb.send[1].as<BEdit<T>>());
    eng.launched(kProfFix);
  }
  // returns the number of received halo targets appended to S
  uint32_t exchange() {
    const std::vector<Rec>& R = sb.hrec;
    const size_t e = sizeof(BEdit<T>);
    const uint32_t n_lo = pl.r > 0 ? static_cast<uint32_t>(R[pl.r - 1].to_hi) : 0;
    const uint32_t n_hi = pl.r + 1 < pl.P ? static_cast<uint32_t>(R[pl.r + 1].to_lo) : 0;
    tr.neighbor_exchange(sb.send[0].p, pl.r > 0 ? R[pl.r].to_lo * e : 0, sb.send[1].p,
                         pl.r + 1 < pl.P ? R[pl.r].to_hi * e : 0, sb.recv[0].p, n_lo * e, sb.recv[1].p,
                         n_hi * e, ws.stream);
    if (n_lo + n_hi) {
      eng.pre(kProfFix);
      k_unpack_boundary<T><<<blocks(n_lo + n_hi), 256, 0, ws.stream>>>(
          s(), sb.recv[0].as<BEdit<T>>(), n_lo, sb.recv[1].as<BEdit<T>>(), n_hi, base);
      eng.launched(kProfFix);
    }
    return n_lo + n_hi;
  }

  // full sweep, or (kind's list empty since its last subloop, no full direction
  // sweep since) only the chunks whose codes changed (see Engine::run_subloop)
  void detect(int kind, uint32_t* list, uint32_t* count, bool allow_dirty = false) {
    if (allow_dirty && eng.fresh[kind]) {
      eng.pre(kProfDetectDirty);
      k_detect_dirty<<<blocks(n() / 16 + 1, 16), 256, 0, ws.stream>>>(s().fdir, s().gdir, n(), s().cstamp,
                                                                      eng.end_mark[kind], kind, list, count,
                                                                      act_lo, act_hi);
      eng.launched(kProfDetectDirty);
    } else {
      eng.pre(kProfDetectKind);
      k_detect_range<<<blocks((act_hi - act_lo) / 16 + 1, 16), 256, 0, ws.stream>>>(
          s().fdir, s().gdir, act_lo, act_hi, kind, list, count);
      eng.launched(kProfDetectKind);
    }
    ++st().detect_sweeps;
  }

  // ---- labels of one direction field (f at setup, g per R iteration) ----
  // Window labels with the off-slab vertices masked as extrema (TileStore own
  // range), then the boundary tables.  finals: also write final global labels of
  // the active range to FM / Fm (f); g labels are resolved per tile by
  // k_rfix_tiles through SlabRes.
  uint64_t* flab(int fam) const { return sb.flab.as<uint64_t>() + size_t(fam) * ((n() + 63) & ~uint32_t(63)); }
  void labels(const uint8_t* dir, uint64_t* FM, uint64_t* Fm, bool finals, bool only_dirty = false) {
    uint32_t* M = eng.lab(2);
    uint32_t* m = eng.lab(3);
    // the tile store masks vertices outside [own_lo, own_hi) as extrema
    eng.label_pass(dir, M, m, only_dirty, /*finish=*/false);
    const bool multi = pl.P > 1;
    if (multi) {
      eng.pre(kProfLabelJump);
      k_publish_labels<<<blocks(4ull * XY), 256, 0, ws.stream>>>(M, m, eng.fin(0), eng.fin(1), XY, own_lo,
                                                                  own_hi, base, sb.tab_mine.as<uint64_t>());
      eng.launched(kProfLabelJump);
      tr.allgather_dev(sb.tab_mine.p, sb.tab_all.p, size_t(4) * XY * 8, ws.stream);
      eng.pre(kProfLabelJump);
      k_resolve_table<<<blocks(4ull * XY * pl.P, 16), 256, 0, ws.stream>>>(sb.tab_all.as<uint64_t>(), stab,
                                                                            sb.flags.as<uint32_t>());
      eng.launched(kProfLabelJump);
    }
    if (!finals) return;
    eng.pre(kProfLabelFinish);
    k_final_labels<<<blocks(act_hi - act_lo, 16), 256, 0, ws.stream>>>(
        M, m, eng.fin(0), eng.fin(1), sb.tab_all.as<uint64_t>(), stab, act_lo, act_hi, base, multi ? 1 : 0,
        FM, Fm);
    eng.launched(kProfLabelFinish);
  }

  // ---- run_subloop (edit_engine.cpp:246-278), one host-driven batch at a time ----
  uint64_t run_subloop(int kind) {
    // provably empty on every rank (Engine::run_subloop): edit totals, hence
    // the epoch, are global
    if (eng.fresh[kind] && eng.epoch_end[kind] == eng.code_epoch && !eng.per_batch()) return 0;
    State<T>& S = s();
    uint32_t& cur = eng.cur;
    reset_ctl();
    detect(kind, S.list[cur], &ws.ctl->list_count[cur], /*allow_dirty=*/true);
    const uint32_t batch_base = ws.next_batch, mark_base = ws.next_mark;
    uint64_t attempted = 0, iters = 0, edits = 0;
    struct IdGuard {
      Workspace& ws;
      uint32_t bb, mb;
      uint64_t& it;
      ~IdGuard() {
        ws.next_batch = std::max<uint32_t>(ws.next_batch, bb + 2 * static_cast<uint32_t>(it) + 6);
        ws.next_mark = std::max<uint32_t>(ws.next_mark, mb + static_cast<uint32_t>(it) + 3);
      }
    } id_guard{ws, batch_base, mark_base, attempted};
    const int rule = (kind == 0 || kind == 3) ? 0 : 1;
    for (;;) {
      const uint32_t it = static_cast<uint32_t>(attempted + 1);
      const uint32_t batch = batch_base + 2 * it, mark = mark_base + it;
      // the fix runs before the global emptiness test: when every list is
      // empty it is a no-op, and the test then costs no extra round trip.
      // Items whose claimed target sits at its floor are parked (k_subloop):
      // the worklist is the active list plus the parked list P.
      fix(rule, batch, S.list[cur], &ws.ctl->list_count[cur], false, /*park=*/true);
      ws.fmark_parked = true;
      gather();
      const uint64_t parked = sum([](const Rec& r) { return r.parked; });
      const uint64_t total = sum([](const Rec& r) { return r.list; }) + parked;
      if (total == 0) break;
      ++attempted;
      if (attempted > eng.opt.subloop_cap)
        fail(MSSZ_CU_ERR_NON_CONVERGENCE, "%s subloop exceeded its iteration cap", kKindName[kind]);
      uint64_t applied = sum([](const Rec& r) { return r.applied; });
      if (applied == 0 && kind == 1) {  // FPmin fallback (edit_engine.cpp:262-268) over list ∪ P
        if (parked) unpark(cur, /*append=*/true);
        fix(2, batch + 1, S.list[cur], &ws.ctl->list_count[cur], false);
        gather();
        applied = sum([](const Rec& r) { return r.applied; });
      }
      if (applied == 0)
        fail(MSSZ_CU_ERR_NON_CONVERGENCE, "%s subloop stalled at the float floor", kKindName[kind]);
      const uint32_t nrecv = exchange();
      const uint32_t ns = static_cast<uint32_t>(sb.hrec[pl.r].applied) + nrecv;
      CK(cudaMemsetAsync(&ws.ctl->list_count[cur ^ 1], 0, sizeof(uint32_t), ws.stream));
      CK(cudaMemsetAsync(&ws.ctl->f_count, 0, sizeof(uint32_t), ws.stream));
      if (total > n_glob / kHugeBatchDivisor) {  // one streaming sweep beats ~15 RMWs per edit
        unpark(cur, /*append=*/false);  // the detect below rebuilds the whole list
        eng.directions(S.g, S.gdir);
        detect(kind, S.list[cur ^ 1], &ws.ctl->list_count[cur ^ 1]);
        ++st().huge_batches;
      } else {  // re-evaluate S ∪ N(S); keep the old items outside it
        eng.pre(kProfFrontier);
        k_slab_frontier<T, 3><<<blocks(uint64_t(ns) * 16, 16), 256, 0, ws.stream>>>(
            S, ns, mark, kind, S.list[cur ^ 1], &ws.ctl->list_count[cur ^ 1]);
        eng.launched(kProfFrontier);
        eng.pre(kProfFrontier);
        k_slab_rebuild<<<blocks(sb.hrec[pl.r].list, 8), 256, 0, ws.stream>>>(
            S.list[cur], &ws.ctl->list_count[cur], S.fmark, mark, S.list[cur ^ 1], &ws.ctl->list_count[cur ^ 1]);
        eng.launched(kProfFrontier);
      }
      st().frontier_vertices += ns;  // refresh seeds (own targets + received halo targets)
      cur ^= 1;
      ++iters;
      edits += applied;
    }
    ws.fmark_parked = false;  // the loop ends with list ∪ P empty
    st().sub_iterations[kind] += iters;
    st().effective_edits += edits;
    if (edits) ++eng.code_epoch;
    return edits;
  }

  // merge P back into list[cur] (append) or only clear its flags; P is emptied
  void unpark(uint32_t cur, bool append) {
    State<T>& S = s();
    if (append)
      k_unpark_list<<<2 * ws.sms, 256, 0, ws.stream>>>(S.list[cur], &ws.ctl->list_count[cur], S.fmark);
    k_unpark_merge<<<2 * ws.sms, 256, 0, ws.stream>>>(S.F, &ws.ctl->park_count, S.fmark, S.list[cur],
                                                      &ws.ctl->list_count[cur], append);
    CK_LAUNCH();
    CK(cudaMemsetAsync(&ws.ctl->park_count, 0, sizeof(uint32_t), ws.stream));
  }

  // one fix over a device-counted list; resets the batch counters first
  void fix(int rule, uint32_t batch, const uint32_t* list, const uint32_t* count, bool retry,
           bool park = false) {
    CK(cudaMemsetAsync(&ws.ctl->s_count, 0, sizeof(uint32_t) * 2, ws.stream));  // s_count, f_count
    CK(cudaMemsetAsync(&ws.ctl->retry_count, 0, sizeof(uint32_t), ws.stream));
    eng.pre(kProfFix);
    // grid-stride over a device-side count: 2 CTAs per SM whatever the batch size
    k_slab_fix<T><<<2 * ws.sms, 256, 0, ws.stream>>>(s(), list, count, rule, batch,
                                                                   retry ? s().F : nullptr,
                                                                   retry ? &ws.ctl->retry_count : nullptr,
                                                                   park);
    eng.launched(kProfFix);
    pack();
  }

  void run_c_loop() {
    for (;;) {
      ++st().c_passes;
      uint64_t pass_edits = 0;
      for (int kind = 0; kind < 4; ++kind) {
        pass_edits += run_subloop(kind);
        eng.end_mark[kind] = ws.next_mark;  // every later batch uses marks >= this
        eng.fresh[kind] = true;
        eng.epoch_end[kind] = eng.code_epoch;
      }
      if (pass_edits) r_full_valid = false;  // the C loop does not track dirty label tiles
      if (pass_edits == 0) return;
    }
  }

  // global first-match false-critical count (owned vertices; frontier list only when given)
  uint64_t count_false(bool frontier_only) {
    CK(cudaMemsetAsync(&ws.ctl->counts[0], 0, sizeof(uint64_t), ws.stream));
    eng.pre(kProfDetectAll);
    k_count_false_range<<<blocks(n() / 16 + 1, 16), 256, 0, ws.stream>>>(
        s().fdir, s().gdir, own_lo, own_hi, frontier_only ? s().F : nullptr, &ws.ctl->f_count,
        &ws.ctl->counts[0]);
    eng.launched(kProfDetectAll);
    ++st().detect_sweeps;
    gather();
    return sum([](const Rec& r) { return r.false_cnt; });
  }

  // g labels + R targets + (speculative) fix; returns the global mismatch count
  // Incremental R batch, as on a single device (Engine::run_r_loop): after a
  // full pass only label tiles whose codes changed are re-resolved, and only
  // tiles that are dirty or whose exits' finals changed recompute their
  // mismatch bits -- plus, across slabs, tiles whose labels depend on a
  // boundary-table entry that changed (k_slab_affected).
  bool r_full_valid = false;
  uint64_t r_batch(uint32_t batch) {
    const bool incr = r_full_valid;
    TileStore ts = eng.tile_store();
    CK(cudaMemsetAsync(sb.flags.p, 0, 8, ws.stream));
    labels(s().gdir, nullptr, nullptr, false, incr);
    if (pl.P > 1) {
      const uint64_t tot = 4ull * XY * pl.P;
      if (incr) {
        eng.pre(kProfLabelJump);
        k_table_diff<<<blocks(tot, 16), 256, 0, ws.stream>>>(sb.tab_all.as<uint64_t>(), sb.tab_prev.as<uint64_t>(),
                                                            sb.tchanged.as<uint8_t>(), tot,
                                                            sb.flags.as<uint32_t>() + 1);
        eng.launched(kProfLabelJump);
        eng.pre(kProfLabelJump);
        k_slab_affected<3><<<ts.ntiles, 256, 0, ws.stream>>>(ts, eng.fin(0), eng.fin(1), sb.tchanged.as<uint8_t>(),
                                                            sb.flags.as<uint32_t>() + 1, stab, eng.geo, base);
        eng.launched(kProfLabelJump);
      } else {
        CK(cudaMemcpyAsync(sb.tab_prev.p, sb.tab_all.p, tot * 8, cudaMemcpyDeviceToDevice, ws.stream));
      }
      eng.sres = SlabRes{sb.tab_all.as<uint64_t>(), stab, base};
    } else {
      eng.sres = SlabRes{nullptr, stab, base};  // one slab: window labels are final
    }
    eng.r_targets(/*all_tiles=*/!incr, /*raise_trouble=*/false);  // targets -> list(0), ctl->mism / status
    r_full_valid = true;
    fix(0, batch, eng.list(0), &ws.ctl->list_count[0], false);
    gather();
    if (sum([](const Rec& r) { return r.err; }))
      fail(MSSZ_CU_ERR_INTERNAL, "path compression exceeded its round cap (corrupt direction field)");
    if (sum([](const Rec& r) { return r.status == kStatusTroubleMax ? 1u : 0u; }))
      fail(MSSZ_CU_ERR_INTERNAL, "troublemaker target is an extremum (stale critical report)");
    return sum([](const Rec& r) { return r.mism; });
  }

  // run_r_loop (edit_engine.cpp:329-366)
  bool run_r_loop() {
    ++eng.code_epoch;  // conservatively: R batches refresh codes
    uint64_t iters = 0;
    bool first = true, last_frontier = false;
    TileStore ts = eng.tile_store();
    struct DirtyOff {
      State<T>& s;
      ~DirtyOff() { s.tdirty = nullptr; }
    } dirty_off{s()};
    s().tdirty = ts.dirty;  // the R-loop frontier marks the label tiles it changes
    for (;;) {
      if (!first && count_false(last_frontier) != 0) return false;
      first = false;
      const uint32_t batch = ws.next_batch++;
      const uint64_t mism = r_batch(batch);
      if (mism == 0) return true;
      if (++iters > eng.opt.r_cap) fail(MSSZ_CU_ERR_NON_CONVERGENCE, "R-loop exceeded its iteration cap");
      const uint64_t applied = sum([](const Rec& r) { return r.applied; });
      if (applied == 0) fail(MSSZ_CU_ERR_NON_CONVERGENCE, "R-loop stalled: every troublemaker is at its floor");
      const uint32_t nrecv = exchange();
      const uint32_t ns = static_cast<uint32_t>(sb.hrec[pl.r].applied) + nrecv;
      const uint32_t mark = ws.next_mark++;
      CK(cudaMemsetAsync(&ws.ctl->f_count, 0, sizeof(uint32_t), ws.stream));
      if (applied > n_glob / kRHugeDivisor) {
        eng.directions(s().g, s().gdir);
        CK(cudaMemsetAsync(ts.dirty, 1, ts.ntiles, ws.stream));  // every tile may have changed
        last_frontier = false;
      } else {
        last_frontier = true;
        if (ns) {
          eng.pre(kProfFrontier);
          k_frontier<T, 3><<<blocks(uint64_t(ns) * 16, 16), 256, 0, ws.stream>>>(s(), ns, mark);
          eng.launched(kProfFrontier);
        }
      }
      st().effective_edits += applied;
      ++st().r_iterations;
    }
  }

  // derive_edits (edit_engine.cpp:386-428) on this slab; ws.g holds the fhat window
  void run(const T* d_f, double xi) {
    if (!(xi > 0.0)) fail(MSSZ_CU_ERR_USAGE, "derive_edits requires xi > 0");
    eng.bind(d_f);
    State<T>& S = s();
    S.xi = xi;
    S.own_lo = own_lo;
    S.own_n = own_hi - own_lo;
    S.act_lo = act_lo;
    S.act_n = act_hi - act_lo;
    reset_ctl();
    eng.pre(kProfValidate);
    k_validate<T><<<blocks(own_hi - own_lo), 256, 0, ws.stream>>>(d_f + own_lo, S.g + own_lo, own_hi - own_lo,
                                                                   xi, ws.ctl);
    eng.launched(kProfValidate);
    gather();
    if (sum([](const Rec& r) { return r.nonfinite; })) fail(MSSZ_CU_ERR_IO, "derive_edits: non-finite input");
    const uint64_t violations = sum([](const Rec& r) { return r.violations; });
    if (violations && !eng.opt.force)
      fail(MSSZ_CU_ERR_BOUND_VIOLATION,
           "%llu vertices violate |f - fhat| <= xi; the preservation guarantee would not hold "
           "(pass force to proceed anyway)",
           (unsigned long long)violations);
    st().input_bound_violations = violations;

    CK(cudaMemsetAsync(S.touched, 0, n(), ws.stream));
    CK(cudaMemsetAsync(sb.flags.p, 0, 16, ws.stream));
    r_full_valid = false;
    CK(cudaEventRecord(ws.ev[0], ws.stream));
    eng.directions(d_f, ws.fdir.as<uint8_t>());
    eng.directions(S.g, S.gdir);
    CK(cudaEventRecord(ws.ev[1], ws.stream));
    S.fM64 = flab(0);
    S.fm64 = flab(1);
    labels(S.fdir, flab(0), flab(1), true);
    gather();
    if (sum([](const Rec& r) { return r.err; }))
      fail(MSSZ_CU_ERR_INTERNAL, "path compression exceeded its round cap (corrupt direction field)");
    {
      float ms = 0;
      CK(cudaEventSynchronize(ws.ev[1]));
      CK(cudaEventElapsedTime(&ms, ws.ev[0], ws.ev[1]));
      eng.dir_ms += ms;
    }
    labels_verified = false;
    for (uint64_t outer = 0;; ++outer) {
      if (outer >= eng.opt.outer_cap)
        fail(MSSZ_CU_ERR_NON_CONVERGENCE,
             "outer loop cap reached after %llu edits (%llu C sub-iterations, %llu R iterations)",
             (unsigned long long)st().effective_edits,
             (unsigned long long)(st().sub_iterations[0] + st().sub_iterations[1] + st().sub_iterations[2] +
                                  st().sub_iterations[3]),
             (unsigned long long)st().r_iterations);
      ++st().outer_iterations;
      const uint64_t before = st().effective_edits;
      run_c_loop();
      const uint64_t after_c = st().effective_edits;
      labels_verified = run_r_loop() && st().effective_edits == after_c;
      if (st().effective_edits == before) break;
    }
    if (!labels_verified) {  // postcondition tripwire (edit_engine.cpp:423-428)
      if (count_false(false) != 0) fail(MSSZ_CU_ERR_INTERNAL, "converged with false critical points");
      if (r_batch(ws.next_batch++) != 0) fail(MSSZ_CU_ERR_INTERNAL, "converged with mismatched labels");
    }
  }

  // this slab's part of edits() (edit_engine.cpp:368-378): global ids, sorted;
  // returns (local count, offset of this slab's part in the global EditSet, global count)
  void compact(uint64_t* d_idx, T* d_val, uint64_t& count, uint64_t& offset, uint64_t& total) {
    count = eng.compact(s().touched, 1, s().g, d_idx, d_val, out_base);  // touched is 0 off the owned range
    gather();  // ctl->mism holds the compaction count
    offset = 0;
    for (uint32_t r = 0; r < pl.r; ++r) offset += sb.hrec[r].mism;
    total = sum([](const Rec& r) { return r.mism; });
  }
};

}  // namespace
}  // namespace mssz_b200
