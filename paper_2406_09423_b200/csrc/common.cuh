// Shared device helpers for the B200 correction loop.
//
// Data layout in HBM (one field of N vertices, row-major, axis 0 fastest as
// in the reference grid.hpp:32-43):
//   f, g        T[N]        original / edited values (g starts as fhat)
//   fdir, gdir  u8[N]       packed steepest directions: low nibble = ascending
//                           stencil slot, high nibble = descending slot,
//                           15 = SELF (extremum).  Slots follow the reference
//                           stencil order grid.cpp:8-16.
//   touched     u8[N]       1 once lower_step moved the vertex (edit_engine.cpp:84)
//   stamp       u32[N]      claim stamps, one id per fix batch (edit_engine.cpp:160-169)
//   fmark       u32[N]      frontier stamps, one id per batch (dedupes S ∪ N(S))
//   fM,fm,gM,gm u32[N]      extremum labels (mss.hpp:37-42), u32 instead of u64
//   lists       u32[N] x 4  current/next worklist, edited set S, frontier F
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mssz_b200 {

constexpr uint32_t kSelf = 15;
constexpr int kWarp = 32;

// Grid geometry passed by value to every kernel.
struct Geom {
  int ndims;   // 2 or 3
  int nst;     // 6 or 14 stencil slots
  uint32_t X, Y, Z;
  uint32_t XY;
  uint32_t n;
  int32_t off[16];  // linear offset per slot; off[15] = 0 (SELF)
};

// Freudenthal stencil (reference grid.cpp:8-16), slot order preserved so that
// direction codes map back to the reference's neighbour enumeration.
template <int DIM>
__host__ __device__ __forceinline__ void stencil(int k, int& dx, int& dy, int& dz) {
  if (DIM == 2) {
    const int t[6][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {1, 1}, {-1, -1}};
    dx = t[k][0];
    dy = t[k][1];
    dz = 0;
  } else {
    const int t[14][3] = {{1, 0, 0},  {-1, 0, 0},  {0, 1, 0},  {0, -1, 0}, {0, 0, 1},
                          {0, 0, -1}, {1, 1, 0},   {-1, -1, 0}, {0, 1, 1},  {0, -1, -1},
                          {1, 0, 1},  {-1, 0, -1}, {1, 1, 1},  {-1, -1, -1}};
    dx = t[k][0];
    dy = t[k][1];
    dz = t[k][2];
  }
}

template <int DIM>
struct StencilSize {
  static constexpr int value = DIM == 2 ? 6 : 14;
};

// ---- order-preserving keys (SoS, reference grid.hpp:53-63) ----
// value order first, index as tie-break; -0.0 and +0.0 compare equal in the
// reference (values[i] != values[j] is false), so both map to the same key.
__device__ __forceinline__ uint32_t okey(float x) {
  uint32_t b = __float_as_uint(x);
  if (b == 0x80000000u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint64_t okey(double x) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  if (b == 0x8000000000000000ull) b = 0ull;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <class T>
struct KeyOf;
template <>
struct KeyOf<float> {
  using type = uint32_t;
};
template <>
struct KeyOf<double> {
  using type = uint64_t;
};

// Loads: LDG (read-only path) for data that is constant during the launch;
// plain (weak, L1-cacheable) loads for data other CTAs of the same persistent
// launch wrote before the last grid/block barrier -- the barrier's gpu-scope
// fence orders those writes before these loads (and invalidates L1), so the
// 16 lanes re-reading one edited vertex's neighbourhood can hit in L1.
template <bool kCoherent, class T>
__device__ __forceinline__ T ld(const T* p) {
  if constexpr (kCoherent) return *p;
  else return __ldg(p);
}

__device__ __forceinline__ void coords(const Geom& g, uint32_t v, uint32_t& x, uint32_t& y,
                                       uint32_t& z) {
  x = v % g.X;
  const uint32_t r = v / g.X;
  y = r % g.Y;
  z = r / g.Y;
}

template <int DIM>
__device__ __forceinline__ bool in_grid(const Geom& g, uint32_t x, uint32_t y, uint32_t z, int k) {
  int dx, dy, dz;
  stencil<DIM>(k, dx, dy, dz);
  // unsigned wraparound rejects -1, exactly as grid.cpp:30-33
  const uint32_t xx = x + static_cast<uint32_t>(dx);
  const uint32_t yy = y + static_cast<uint32_t>(dy);
  const uint32_t zz = z + static_cast<uint32_t>(dz);
  return xx < g.X && yy < g.Y && (DIM == 2 || zz < g.Z);
}

template <int DIM>
__device__ __forceinline__ int32_t slot_offset(const Geom& g, int k) {
  int dx, dy, dz;
  stencil<DIM>(k, dx, dy, dz);
  return dx + dy * static_cast<int32_t>(g.X) + dz * static_cast<int32_t>(g.XY);
}

// Index-rank order of the stencil slots (plus SELF = 15): the linear offsets
// of grid.cpp:8-16 sort the same way for every grid with extents >= 2
//   3D: -1-X-XY < -X-XY < -1-XY < -XY < -1-X < -X < -1 < 0 < 1 < X < 1+X < XY
//       < 1+XY < X+XY < 1+X+XY
//   2D: -1-X < -X < -1 < 0 < 1 < X < 1+X
// so SoS (value, then index) reduces to comparing keys while scanning slots in
// this order: ascending uses >= (the highest index wins a tie), descending
// uses < (the lowest index wins), exactly sos_greater / sos_less (grid.hpp:53-63).
template <int DIM>
__host__ __device__ __forceinline__ constexpr int rank_slot(int r) {
  if (DIM == 2) {
    constexpr int t[7] = {5, 3, 1, 15, 0, 2, 4};
    return t[r];
  } else {
    constexpr int t[15] = {13, 9, 11, 5, 7, 3, 1, 15, 0, 2, 6, 4, 10, 8, 12};
    return t[r];
  }
}

// Steepest ascending / descending slot of v over self ∪ link (mss.cpp:11-30):
// returns (asc | desc << 4), SELF = 15.
template <class T, int DIM, bool kCoherent>
__device__ __forceinline__ uint32_t direction_code(const T* __restrict__ vals, const Geom& g,
                                                   uint32_t v, uint32_t x, uint32_t y,
                                                   uint32_t z) {
  using K = typename KeyOf<T>::type;
  constexpr int NR = StencilSize<DIM>::value + 1;
  const bool interior = x > 0 && x + 1 < g.X && y > 0 && y + 1 < g.Y &&
                        (DIM == 2 || (z > 0 && z + 1 < g.Z));
  // all loads first (out-of-grid slots re-read v and are masked below)
  K key[NR];
  bool ok[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int k = rank_slot<DIM>(r);
    ok[r] = k == 15 || interior || in_grid<DIM>(g, x, y, z, k);
    const uint32_t u = (k == 15 || !ok[r]) ? v : v + slot_offset<DIM>(g, k);
    key[r] = okey(ld<kCoherent>(vals + u));
  }
  K hi = 0, lo = ~K(0);
  uint32_t hc = kSelf, lc = kSelf;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const uint32_t k = static_cast<uint32_t>(rank_slot<DIM>(r));
    if (ok[r] && key[r] >= hi) {
      hi = key[r];
      hc = k;
    }
    if (ok[r] && key[r] < lo) {
      lo = key[r];
      lc = k;
    }
  }
  return hc | (lc << 4);
}

__device__ __forceinline__ bool is_max(uint32_t code) { return (code & 15u) == kSelf; }
__device__ __forceinline__ bool is_min(uint32_t code) { return (code >> 4) == kSelf; }

// detect_kind predicates (edit_engine.cpp:110-117) on packed codes.
__device__ __forceinline__ bool kind_match(int kind, uint32_t fc, uint32_t gc) {
  switch (kind) {
    case 0: return is_max(gc) && !is_max(fc);   // FPmax
    case 1: return is_min(gc) && !is_min(fc);   // FPmin
    case 2: return is_max(fc) && !is_max(gc);   // FNmax
    default: return is_min(fc) && !is_min(gc);  // FNmin
  }
}

// first-match class (edit_engine.cpp:339-348), 4 = none
__device__ __forceinline__ uint32_t first_class(uint32_t fc, uint32_t gc) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (kind_match(k, fc, gc)) return k;
  return 4;
}

// ---- bit-exact error-bounded halving (edit_engine.cpp:22-29, 75-86) ----
// Every double operation is an explicit round-to-nearest intrinsic so no FMA
// contraction can change the result (the reference builds with -ffp-contract=off).
__device__ __forceinline__ float narrow(double d, float) { return __double2float_rn(d); }
__device__ __forceinline__ double narrow(double d, double) { return d; }

template <class T>
__device__ __forceinline__ T representable_floor(T f, double xi) {
  const double lo = __dsub_rn(static_cast<double>(f), xi);
  T c = narrow(lo, T{});
  if (!(static_cast<double>(c) > lo)) {
    if constexpr (sizeof(T) == 4) c = nextafterf(c, __int_as_float(0x7f800000));
    else c = nextafter(c, __longlong_as_double(0x7ff0000000000000ll));
  }
  return c;
}

template <class T>
__device__ __forceinline__ bool lower_value(T g, T f, double xi, T& out) {
  const T lo = representable_floor(f, xi);
  if (!(g > lo)) return false;
  const double target = __dsub_rn(static_cast<double>(f), xi);
  T mid = narrow(__dmul_rn(0.5, __dadd_rn(static_cast<double>(g), target)), T{});
  if (!(mid < g) || mid < lo) mid = lo;
  out = mid;
  return true;
}

// ---- warp-aggregated append: one atomic per warp (ballot + popc) ----
// Must be called by all 32 lanes of the warp (full mask).
__device__ __forceinline__ void warp_append(bool pred, uint32_t val, uint32_t* __restrict__ list,
                                            uint32_t* count) {
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  if (b == 0) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(b) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(count, static_cast<uint32_t>(__popc(b)));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (pred) list[base + __popc(b & ((1u << lane) - 1u))] = val;
}

// warp_append variant that drops entries past `cap` (the count still grows,
// so the caller detects the overflow).
__device__ __forceinline__ void warp_append_cap(bool pred, uint32_t val, uint32_t* __restrict__ list,
                                                uint32_t* count, uint32_t cap) {
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  if (b == 0) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(b) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(count, static_cast<uint32_t>(__popc(b)));
  base = __shfl_sync(0xffffffffu, base, leader);
  const uint32_t pos = base + __popc(b & ((1u << lane) - 1u));
  if (pred && pos < cap) list[pos] = val;
}

// Per-lane staging buffer (in the warp's shared-memory slice `st`, K x 32
// words) for list appends inside warp-uniform loops: values are written with
// ONE warp reservation when some lane's buffer is full (and at the end)
// instead of one contended global atomic per loop iteration.  All calls must
// be made by the full warp.
template <int K>
struct WarpBuffer {
  uint32_t* st;  // st[j * 32 + lane]
  int n = 0;
  __device__ __forceinline__ explicit WarpBuffer(uint32_t* stage) : st(stage) {}
  __device__ __forceinline__ void flush(uint32_t* __restrict__ list, uint32_t* count);
  __device__ __forceinline__ void push(bool pred, uint32_t val, uint32_t* __restrict__ list,
                                       uint32_t* count) {
    if (__any_sync(0xffffffffu, n == K)) flush(list, count);
    if (pred) st[n * 32 + (threadIdx.x & 31)] = val;
    n += pred ? 1 : 0;
  }
};

// Per-lane count c -> returns this lane's slot base after a single warp atomic.
__device__ __forceinline__ uint32_t warp_reserve(uint32_t c, uint32_t* count) {
  const int lane = threadIdx.x & 31;
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  uint32_t base = 0;
  if (lane == 31 && total) base = atomicAdd(count, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - c;
}

template <int K>
__device__ __forceinline__ void WarpBuffer<K>::flush(uint32_t* __restrict__ list, uint32_t* count) {
  __syncwarp();
  const uint32_t pos = warp_reserve(static_cast<uint32_t>(n), count);
  for (int j = 0; j < n; ++j) list[pos + j] = st[j * 32 + (threadIdx.x & 31)];
  __syncwarp();
  n = 0;
}

// Block-wide reservation: every thread of the block calls it (block-uniform
// control flow) with its count c; one atomic per block instead of one per warp,
// so long appends from full sweeps do not serialise on the counter.
__device__ __forceinline__ uint32_t block_reserve(uint32_t c, uint32_t* count) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t bbase;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    const uint32_t v = lane < nw ? wsum[lane] : 0u;
    uint32_t s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    if (lane < nw) wsum[lane] = s - v;  // exclusive warp offsets
    if (lane == 31) bbase = s ? atomicAdd(count, s) : 0u;
  }
  __syncthreads();
  const uint32_t base = bbase + wsum[w] + incl - c;
  __syncthreads();  // wsum / bbase are reused by the next call
  return base;
}

constexpr int kStageK = 4;
constexpr int kStageWarps = 16;  // blocks of up to 512 threads
// per-warp staging slice of a [kStageWarps][kStageK * 32] shared array
__device__ __forceinline__ uint32_t* warp_stage(uint32_t (*arr)[kStageK * 32]) {
  return arr[threadIdx.x >> 5];
}

}  // namespace mssz_b200
