// Kernels of the B200 correction loop.  Each cites the reference code whose
// semantics it reproduces (paths relative to /root/reference/proj/core).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace mssz_b200 {

namespace cg = cooperative_groups;

// Device control block: counters and status words shared by the kernels of one
// derive_edits call.  The host reads it back once per subloop / R iteration.
struct Ctl {
  uint32_t list_count[2];
  uint32_t s_count;  // |S| edited targets of the last batch
  uint32_t f_count;  // |S ∪ N(S)| of the last batch
  uint32_t status;   // kStatus*
  uint32_t cur;      // which list buffer is current
  uint64_t attempted;  // iterations counted against subloop_cap (edit_engine.cpp:258)
  uint64_t iters;      // successful batches (EditStats::sub_iterations)
  uint64_t edits;      // applied edits (EditStats::effective_edits)
  uint64_t frontier;   // Σ |S ∪ N(S)|
  uint64_t counts[4];  // first-match false-critical counts (edit_engine.cpp:339-348)
  uint64_t mism;       // vertices with g labels != f labels (edit_engine.cpp:317-327)
  uint64_t nonfinite;  // input validation (edit_engine.cpp:390-397)
  uint64_t violations;
  uint32_t flags[64];  // pointer-jumping "changed" flags, one per round
};

enum : uint32_t {
  kStatusOk = 0,
  kStatusCap = 1,          // subloop cap (edit_engine.cpp:258-260)
  kStatusStall = 2,        // "stalled at the float floor" (:269-271)
  kStatusTroubleMax = 3,   // "troublemaker target is an extremum" (:305-306)
};

// ---------------------------------------------------------------------------
// K1: full direction sweep (compute_directions, mss.cpp:11-30).
// Grid (ceil(X/128), Y, Z): one thread per vertex, no div/mod; neighbours come
// through L1/L2 (each value is reused by up to 15 threads of nearby rows).
template <class T, int DIM>
__global__ void __launch_bounds__(128) k_directions(const T* __restrict__ vals,
                                                    uint8_t* __restrict__ dir, Geom g) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t y = blockIdx.y;
  const uint32_t z = blockIdx.z;
  if (x >= g.X) return;
  const uint32_t v = x + g.X * y + g.XY * z;
  dir[v] = static_cast<uint8_t>(direction_code<T, DIM, false>(vals, g, v, x, y, z));
}

// ---------------------------------------------------------------------------
// K1b: full detect sweep for one kind (detect_kind, edit_engine.cpp:104-132),
// 16 vertices per thread from two 16-byte loads, compacted with one atomic per
// warp.  List order is arbitrary: every consumer is order-independent.
__global__ void __launch_bounds__(256) k_detect_kind(const uint8_t* __restrict__ fdir,
                                                     const uint8_t* __restrict__ gdir,
                                                     uint32_t n, int kind,
                                                     uint32_t* __restrict__ list,
                                                     uint32_t* count) {
  const uint64_t nchunks = (static_cast<uint64_t>(n) + 15) / 16;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t wbase0 = tid & ~uint64_t(31);
  for (uint64_t wb = wbase0; wb < nchunks; wb += stride) {
    const uint64_t c = wb + (threadIdx.x & 31);
    uint32_t mask = 0;
    if (c < nchunks) {
      const uint64_t v0 = c * 16;
      uint8_t fb[16], gb[16];
      if (v0 + 16 <= n) {
        *reinterpret_cast<uint4*>(fb) = __ldg(reinterpret_cast<const uint4*>(fdir + v0));
        *reinterpret_cast<uint4*>(gb) = __ldg(reinterpret_cast<const uint4*>(gdir + v0));
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          fb[j] = (v0 + j < n) ? fdir[v0 + j] : 0xFF;
          gb[j] = (v0 + j < n) ? gdir[v0 + j] : 0xFF;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (kind_match(kind, fb[j], gb[j])) mask |= 1u << j;
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

// Counts of the first-match classes (detect_false_critical, edit_engine.cpp:134-158)
// into ctl->counts; optional per-vertex class bytes for the API export.
__global__ void __launch_bounds__(256) k_detect_all(const uint8_t* __restrict__ fdir,
                                                    const uint8_t* __restrict__ gdir, uint32_t n,
                                                    uint64_t* counts, uint8_t* cls_out) {
  __shared__ uint32_t sc[4];
  if (threadIdx.x < 4) sc[threadIdx.x] = 0;
  __syncthreads();
  uint32_t local[4] = {0, 0, 0, 0};
  const uint64_t nchunks = (static_cast<uint64_t>(n) + 15) / 16;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < nchunks;
       c += stride) {
    const uint64_t v0 = c * 16;
    uint8_t fb[16], gb[16];
    if (v0 + 16 <= n) {
      *reinterpret_cast<uint4*>(fb) = __ldg(reinterpret_cast<const uint4*>(fdir + v0));
      *reinterpret_cast<uint4*>(gb) = __ldg(reinterpret_cast<const uint4*>(gdir + v0));
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        fb[j] = (v0 + j < n) ? fdir[v0 + j] : 0xFF;
        gb[j] = (v0 + j < n) ? gdir[v0 + j] : 0xFF;
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t k = first_class(fb[j], gb[j]);
      if (k < 4) ++local[k];
      if (cls_out && v0 + j < n) cls_out[v0 + j] = static_cast<uint8_t>(k);
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t s = local[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(&sc[k], s);
  }
  __syncthreads();
  if (threadIdx.x < 4 && sc[threadIdx.x])
    atomicAdd(reinterpret_cast<unsigned long long*>(&counts[threadIdx.x]),
              static_cast<unsigned long long>(sc[threadIdx.x]));
}

// ---------------------------------------------------------------------------
// Fix / frontier building blocks used by the persistent subloop kernel and by
// the R-loop.  rule: 0 = self (FPmax, FNmin), 1 = g's ascending neighbour
// (FPmin, FNmax; equals g_argmax_neighbor at batch start, edit_engine.cpp:171-185),
// 2 = f's descending neighbour (FPmin fallback, edit_engine.cpp:187-195, :262-268).
template <class T>
struct State {
  Geom geo;
  const T* f;
  T* g;
  const uint8_t* fdir;
  uint8_t* gdir;
  uint8_t* touched;
  uint32_t* stamp;
  uint32_t* fmark;
  uint32_t* list[2];
  uint32_t* S;
  uint32_t* F;
  const uint32_t* fM;
  const uint32_t* fm;
  const uint32_t* gM;
  const uint32_t* gm;
  double xi;
  Ctl* ctl;
};

// claim (edit_engine.cpp:160-169) + lower_step (:75-86): the first claimant of
// t in this batch lowers it from the pre-batch value; exactly one winner per
// target, so Σ winners == the reference's applied count.
template <class T>
__device__ __forceinline__ bool claim_and_lower(const State<T>& s, uint32_t t, uint32_t batch) {
  if (atomicExch(&s.stamp[t], batch) == batch) return false;
  T nv;
  if (!lower_value<T>(__ldcg(s.g + t), __ldg(s.f + t), s.xi, nv)) return false;
  s.g[t] = nv;
  s.touched[t] = 1;
  return true;
}

template <class T>
__device__ __forceinline__ void fix_batch(const State<T>& s, const uint32_t* __restrict__ list,
                                          uint32_t n, int rule, uint32_t batch, uint64_t tid,
                                          uint64_t stride) {
  for (uint64_t wb = tid & ~uint64_t(31); wb < n; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    bool ok = false;
    uint32_t t = 0;
    if (i < n) {
      const uint32_t v = __ldcg(list + i);
      if (rule == 0) t = v;
      else if (rule == 1) t = v + s.geo.off[__ldcg(s.gdir + v) & 15u];
      else t = v + s.geo.off[__ldg(s.fdir + v) >> 4];
      ok = claim_and_lower(s, t, batch);
    }
    warp_append(ok, t, s.S, &s.ctl->s_count);
  }
}

// Re-evaluates gdir on S ∪ N(S) (the only vertices whose direction can change
// after a batch), each vertex once (fmark dedupe), and collects them in F.
template <class T, int DIM>
__device__ __forceinline__ void frontier_update(const State<T>& s, uint32_t ns, uint32_t mark,
                                                uint64_t tid, uint64_t stride) {
  constexpr int NS = StencilSize<DIM>::value;
  for (uint64_t wb = tid & ~uint64_t(31); wb < ns; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    uint32_t sv = 0, sx = 0, sy = 0, sz = 0;
    const bool live = i < ns;
    if (live) {
      sv = __ldcg(s.S + i);
      coords(s.geo, sv, sx, sy, sz);
    }
#pragma unroll
    for (int k = -1; k < NS; ++k) {
      bool mine = false;
      uint32_t u = sv;
      if (live) {
        uint32_t ux = sx, uy = sy, uz = sz;
        bool valid = true;
        if (k >= 0) {
          valid = in_grid<DIM>(s.geo, sx, sy, sz, k);
          int dx, dy, dz;
          stencil<DIM>(k, dx, dy, dz);
          ux = sx + dx;
          uy = sy + dy;
          uz = sz + dz;
          u = sv + slot_offset<DIM>(s.geo, k);
        }
        if (valid && atomicExch(&s.fmark[u], mark) != mark) {
          mine = true;
          s.gdir[u] = static_cast<uint8_t>(direction_code<T, DIM, true>(s.g, s.geo, u, ux, uy, uz));
        }
      }
      warp_append(mine, u, s.F, &s.ctl->f_count);
    }
  }
}

// New worklist = (old list minus frontier) ∪ {u in frontier : kind(u)}.
// Exact: only frontier vertices can change class after a batch.
template <class T>
__device__ __forceinline__ void rebuild_list(const State<T>& s, int kind, const uint32_t* old,
                                             uint32_t nold, uint32_t* nxt, uint32_t* nxt_count,
                                             uint32_t nf, uint32_t mark, uint64_t tid,
                                             uint64_t stride) {
  const uint64_t total = static_cast<uint64_t>(nf) + nold;
  for (uint64_t wb = tid & ~uint64_t(31); wb < total; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    bool keep = false;
    uint32_t v = 0;
    if (i < nf) {
      v = __ldcg(s.F + i);
      keep = kind_match(kind, __ldg(s.fdir + v), __ldcg(s.gdir + v));
    } else if (i < total) {
      v = __ldcg(old + (i - nf));
      keep = __ldcg(s.fmark + v) != mark;
    }
    warp_append(keep, v, nxt, nxt_count);
  }
}

// ---------------------------------------------------------------------------
// Persistent subloop (run_subloop, edit_engine.cpp:246-278): detect → fix →
// refresh until the kind's list is empty, entirely on the device.  One
// cooperative launch per subloop invocation; three grid barriers per batch.
// batch ids: batch_base + 2*it (+1 for the FPmin fallback); mark ids: mark_base + it.
template <class T, int DIM>
__global__ void __launch_bounds__(512, 1)
    k_subloop(State<T> s, int kind, uint64_t cap, uint32_t batch_base, uint32_t mark_base,
              uint32_t max_batches) {
  cg::grid_group grid = cg::this_grid();
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const bool leader = tid == 0;
  Ctl* ctl = s.ctl;
  const int rule = (kind == 0 || kind == 3) ? 0 : 1;

  uint32_t cur = *reinterpret_cast<volatile uint32_t*>(&ctl->cur);
  uint64_t attempted = *reinterpret_cast<volatile uint64_t*>(&ctl->attempted);
  uint64_t iters = 0, edits = 0, frontier = 0;
  uint32_t status = kStatusOk;
  uint32_t done_batches = 0;

  for (;;) {
    const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&ctl->list_count[cur]);
    if (n == 0 || done_batches >= max_batches) break;
    ++attempted;
    if (attempted > cap) {
      status = kStatusCap;
      break;
    }
    const uint32_t it = static_cast<uint32_t>(attempted);
    const uint32_t batch = batch_base + 2 * it;
    const uint32_t mark = mark_base + it;
    if (leader) {
      ctl->f_count = 0;
      ctl->list_count[cur ^ 1] = 0;
    }
    // phase F: fix (fix_list, edit_engine.cpp:197-227)
    fix_batch(s, s.list[cur], n, rule, batch, tid, stride);
    grid.sync();
    uint32_t applied = *reinterpret_cast<volatile uint32_t*>(&ctl->s_count);
    if (applied == 0 && kind == 1) {
      grid.sync();  // every thread has read applied == 0 before the fallback appends to S
      fix_batch(s, s.list[cur], n, 2, batch + 1, tid, stride);
      grid.sync();
      applied = *reinterpret_cast<volatile uint32_t*>(&ctl->s_count);
    }
    if (applied == 0) {
      status = kStatusStall;
      break;
    }
    ++iters;
    edits += applied;
    // phase D: refresh directions on S ∪ N(S) (refresh_directions, edit_engine.cpp:88-95)
    frontier_update<T, DIM>(s, applied, mark, tid, stride);
    grid.sync();
    const uint32_t nf = *reinterpret_cast<volatile uint32_t*>(&ctl->f_count);
    frontier += nf;
    // phase L: next worklist (detect_kind on the refreshed field)
    rebuild_list(s, kind, s.list[cur], n, s.list[cur ^ 1], &ctl->list_count[cur ^ 1], nf, mark,
                 tid, stride);
    if (leader) ctl->s_count = 0;
    grid.sync();
    cur ^= 1;
    ++done_batches;
  }
  grid.sync();
  if (leader) {
    ctl->cur = cur;
    ctl->attempted = attempted;
    ctl->iters += iters;
    ctl->edits += edits;
    ctl->frontier += frontier;
    ctl->status = status;
  }
}

// ---------------------------------------------------------------------------
// K3: extremum labels (compute_labels_into, mss.cpp:51-97) as u32 pointer
// jumping.  Init follows up to kChase direction codes (1-byte, spatially local
// gathers), then asynchronous in-place doubling rounds.  In-place doubling
// reaches the same unique fixpoint (the chain terminus) in no more rounds than
// the reference's round-synchronous version, so its round cap still applies.
constexpr int kChase = 8;

__global__ void __launch_bounds__(256) k_label_init(const uint8_t* __restrict__ dir, Geom g,
                                                    uint32_t* __restrict__ M,
                                                    uint32_t* __restrict__ m) {
  __shared__ int32_t off[16];
  if (threadIdx.x < 16) off[threadIdx.x] = g.off[threadIdx.x];
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < g.n;
       v += stride) {
    const uint32_t c = __ldg(dir + v);
    uint32_t a = static_cast<uint32_t>(v) + off[c & 15u];
    uint32_t d = static_cast<uint32_t>(v) + off[c >> 4];
#pragma unroll
    for (int h = 1; h < kChase; ++h) {
      a += off[__ldg(dir + a) & 15u];
      d += off[__ldg(dir + d) >> 4];
    }
    M[v] = a;
    m[v] = d;
  }
}

__global__ void __launch_bounds__(256) k_label_jump(uint32_t* __restrict__ M,
                                                    uint32_t* __restrict__ m, uint32_t n,
                                                    uint32_t* flag) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  bool changed = false;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += stride) {
    const uint32_t a = M[v];
    const uint32_t d = m[v];
    const uint32_t aa = M[a];
    const uint32_t dd = m[d];
    if (aa != a) {
      M[v] = aa;
      changed = true;
    }
    if (dd != d) {
      m[v] = dd;
      changed = true;
    }
  }
  if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) *flag = 1;
}

// Generic u64 parent arrays (the exported compute_labels API): copy to u32.
__global__ void k_u64_to_u32(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                             uint32_t n, uint32_t* bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const uint64_t p = in[i];
    if (p >= n) *bad = 1;
    out[i] = static_cast<uint32_t>(p < n ? p : i);
  }
}

__global__ void k_u32_to_u64(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                             uint32_t n) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    out[i] = in[i];
}

// ---------------------------------------------------------------------------
// K4+K5 fused R-loop batch (run_r_loop, edit_engine.cpp:329-366).
// For a mismatched vertex v, find_troublemaker (:293-315) walks f's line to the
// first vertex w whose g-direction diverges.  Up to w the g line equals the f
// line, so w carries v's labels: w is itself divergent AND mismatched, and its
// own walk stops at w.  Hence the set of troublemaker targets is exactly
//   { gasc(w) : gasc(w) != fasc(w), gM(w) != fM(w) } ∪
//   { fdesc(w) : gdesc(w) != fdesc(w), gm(w) != fm(w) }
// and one full sweep finds it without walking.  Targets are claimed once and
// lowered from the pre-batch g, which is the reference's batch semantics (claim
// stamps, then lower_step over the deduplicated targets).
template <class T>
__global__ void __launch_bounds__(256) k_rfix(State<T> s, uint32_t batch) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t mism = 0;
  const uint32_t n = s.geo.n;
  for (uint64_t wb = tid & ~uint64_t(31); wb < n; wb += stride) {
    const uint64_t v = wb + (threadIdx.x & 31);
    bool oka = false, okd = false;
    uint32_t ta = 0, td = 0;
    if (v < n) {
      const uint32_t fc = __ldg(s.fdir + v), gc = __ldg(s.gdir + v);
      const bool mM = __ldg(s.gM + v) != __ldg(s.fM + v);
      const bool mm = __ldg(s.gm + v) != __ldg(s.fm + v);
      mism += (mM || mm) ? 1u : 0u;
      if (mM && (gc & 15u) != (fc & 15u)) {
        if ((gc & 15u) == kSelf) atomicExch(&s.ctl->status, kStatusTroubleMax);
        else {
          ta = static_cast<uint32_t>(v) + s.geo.off[gc & 15u];
          oka = claim_and_lower(s, ta, batch);
        }
      }
      if (mm && (gc >> 4) != (fc >> 4)) {
        if ((fc >> 4) == kSelf) atomicExch(&s.ctl->status, kStatusTroubleMax);
        else {
          td = static_cast<uint32_t>(v) + s.geo.off[fc >> 4];
          okd = claim_and_lower(s, td, batch);
        }
      }
    }
    warp_append(oka, ta, s.S, &s.ctl->s_count);
    warp_append(okd, td, s.S, &s.ctl->s_count);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mism += __shfl_xor_sync(0xffffffffu, mism, o);
  if ((threadIdx.x & 31) == 0 && mism)
    atomicAdd(reinterpret_cast<unsigned long long*>(&s.ctl->mism),
              static_cast<unsigned long long>(mism));
}

// Non-persistent frontier refresh (after an R batch).
template <class T, int DIM>
__global__ void __launch_bounds__(256) k_frontier(State<T> s, uint32_t ns, uint32_t mark) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  frontier_update<T, DIM>(s, ns, mark, tid, stride);
}

// ---------------------------------------------------------------------------
// Input validation (derive_edits, edit_engine.cpp:389-402): non-finite values
// and |f - fhat| > xi counted in double.
template <class T>
__global__ void __launch_bounds__(256) k_validate(const T* __restrict__ f,
                                                  const T* __restrict__ fh, uint64_t n, double xi,
                                                  Ctl* ctl) {
  uint32_t bad = 0, viol = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const double a = static_cast<double>(__ldg(f + i));
    const double b = static_cast<double>(__ldg(fh + i));
    if (!isfinite(a) || !isfinite(b)) ++bad;
    else if (fabs(__dsub_rn(a, b)) > xi) ++viol;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    viol += __shfl_xor_sync(0xffffffffu, viol, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->nonfinite), (unsigned long long)bad);
    if (viol) atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->violations), (unsigned long long)viol);
  }
}

// ---------------------------------------------------------------------------
// K6: ordered stream compaction (EditState::edits, edit_engine.cpp:368-378):
// indices where flag[i] == want, strictly increasing, plus the value g[i].
// Pass 1 counts per tile, a single-CTA scan turns counts into offsets, pass 2
// writes.  Tile = 256 threads x 16 vertices.
constexpr int kCompactThreads = 256;
constexpr int kCompactPer = 16;
constexpr uint64_t kCompactTile = uint64_t(kCompactThreads) * kCompactPer;

__device__ __forceinline__ uint32_t tile_flags(const uint8_t* __restrict__ flag, uint64_t n,
                                               uint64_t v0, uint8_t want) {
  uint32_t bits = 0;
  if (v0 + 16 <= n) {
    uint8_t b[16];
    *reinterpret_cast<uint4*>(b) = __ldg(reinterpret_cast<const uint4*>(flag + v0));
#pragma unroll
    for (int j = 0; j < 16; ++j) bits |= (b[j] == want ? 1u : 0u) << j;
  } else {
    for (int j = 0; j < 16; ++j)
      if (v0 + j < n && flag[v0 + j] == want) bits |= 1u << j;
  }
  return bits;
}

__global__ void __launch_bounds__(kCompactThreads) k_compact_count(const uint8_t* __restrict__ flag,
                                                                   uint64_t n, uint8_t want,
                                                                   uint32_t* __restrict__ tile_counts) {
  __shared__ uint32_t wsum[kCompactThreads / 32];
  const uint64_t v0 = (static_cast<uint64_t>(blockIdx.x) * kCompactThreads + threadIdx.x) * kCompactPer;
  uint32_t c = v0 < n ? __popc(tile_flags(flag, n, v0, want)) : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kCompactThreads / 32; ++w) t += wsum[w];
    tile_counts[blockIdx.x] = t;
  }
}

// exclusive scan of tile counts in one CTA (tiles <= 2^32/4096), total -> *total
__global__ void __launch_bounds__(1024) k_scan_tiles(uint32_t* __restrict__ counts, uint64_t ntiles,
                                                     uint64_t* total) {
  __shared__ uint64_t wsum[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < ntiles; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t c = i < ntiles ? counts[i] : 0;
    uint64_t incl = c;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      uint64_t s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += t;
      }
      wsum[lane] = s;  // inclusive prefix over warps
    }
    __syncthreads();
    const uint64_t warp_excl = w ? wsum[w - 1] : 0;
    if (i < ntiles) counts[i] = static_cast<uint32_t>(carry + warp_excl + incl - c);
    __syncthreads();
    if (threadIdx.x == 0) carry += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

template <class T>
__global__ void __launch_bounds__(kCompactThreads) k_compact_write(
    const uint8_t* __restrict__ flag, uint64_t n, uint8_t want, const T* __restrict__ g,
    const uint32_t* __restrict__ tile_offsets, uint64_t* __restrict__ idx_out,
    T* __restrict__ val_out) {
  __shared__ uint32_t wsum[kCompactThreads / 32];
  const uint64_t v0 = (static_cast<uint64_t>(blockIdx.x) * kCompactThreads + threadIdx.x) * kCompactPer;
  uint32_t bits = v0 < n ? tile_flags(flag, n, v0, want) : 0u;
  const uint32_t c = __popc(bits);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t wex = 0;
  for (int k = 0; k < w; ++k) wex += wsum[k];
  uint64_t pos = static_cast<uint64_t>(tile_offsets[blockIdx.x]) + wex + incl - c;
  while (bits) {
    const int j = __ffs(bits) - 1;
    bits &= bits - 1;
    idx_out[pos] = v0 + j;
    if (val_out) val_out[pos] = g[v0 + j];
    ++pos;
  }
}

// ---------------------------------------------------------------------------
// Element-wise exports (lower_step / representable_floor / apply_edits).
template <class T>
__global__ void k_lower_step(uint64_t n, const T* __restrict__ g, const T* __restrict__ f,
                             double xi, T* __restrict__ out, uint8_t* __restrict__ moved) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    T nv;
    const bool ok = lower_value<T>(g[i], f[i], xi, nv);
    out[i] = ok ? nv : g[i];
    moved[i] = ok ? 1 : 0;
  }
}

template <class T>
__global__ void k_floor(uint64_t n, const T* __restrict__ f, double xi, T* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    out[i] = representable_floor<T>(f[i], xi);
}

template <class T>
__global__ void k_scatter(uint64_t count, const uint64_t* __restrict__ idx,
                          const T* __restrict__ vals, uint64_t n, T* __restrict__ out,
                          uint32_t* bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    const uint64_t v = idx[i];
    if (v >= n) *bad = 1;
    else out[v] = vals[i];
  }
}

// dir codes -> the reference's u64 vertex ids (DirectionField, mss.hpp:24-27)
__global__ void k_codes_to_ids(const uint8_t* __restrict__ dir, Geom g, uint64_t* __restrict__ asc,
                               uint64_t* __restrict__ desc) {
  __shared__ int32_t off[16];
  if (threadIdx.x < 16) off[threadIdx.x] = g.off[threadIdx.x];
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < g.n;
       v += stride) {
    const uint32_t c = dir[v];
    asc[v] = static_cast<uint64_t>(static_cast<int64_t>(v) + off[c & 15u]);
    desc[v] = static_cast<uint64_t>(static_cast<int64_t>(v) + off[c >> 4]);
  }
}

// extremum flags from u64 parent arrays (classify_critical, mss.cpp:40-47)
__global__ void k_extremum_flags(const uint64_t* __restrict__ asc, const uint64_t* __restrict__ desc,
                                 uint64_t n, uint8_t* __restrict__ fmax, uint8_t* __restrict__ fmin) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += stride) {
    fmax[v] = asc[v] == v ? 1 : 0;
    fmin[v] = desc[v] == v ? 1 : 0;
  }
}

}  // namespace mssz_b200
