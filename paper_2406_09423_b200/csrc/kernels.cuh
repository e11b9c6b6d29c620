// Kernels of the B200 correction loop.  Each cites the reference code whose
// semantics it reproduces (paths relative to /root/reference/proj/core).
#pragma once

#include <cooperative_groups.h>
#include <cuda.h>  // CUtensorMap (TMA descriptor of the direction field)

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
  uint32_t cmd_seq;    // leader -> worker CTA command word (k_subloop)
  uint32_t cmd_type;
  uint32_t cmd_n;
  uint32_t cmd_cur;
  uint32_t cmd_it;
  uint32_t pad_;
  uint64_t big_batches;  // batches that ran grid-wide
  uint64_t small_ns, big_ns;  // k_subloop batch time by regime (%globaltimer, leader thread)
  uint64_t phase_ns[3];       // big batches: fix / frontier / rebuild
  uint32_t retry_count;       // k_subloop: old-list items whose target was not lowered
  uint32_t pad2_;
  uint32_t sp_count[4];  // sparse R-loop: X / frontier (2) / Up sizes
  uint32_t sp_abort;
  uint32_t sp_levels;
  uint32_t bnd[2];       // z-slab sharding: boundary edits packed for rank-1 / rank+1
  uint64_t items;        // Σ worklist sizes over the batches of a subloop (trace)
  uint64_t rfix_div;     // k_rfix_tiles: divergent (vertex, family) pairs evaluated
  uint32_t park_count;   // k_subloop: entries of the parked-item list (State::F)
  uint32_t merges;       // k_subloop: parked-list merges (trace)
};

enum : uint32_t {
  kStatusOk = 0,
  kStatusCap = 1,          // subloop cap (edit_engine.cpp:258-260)
  kStatusStall = 2,        // "stalled at the float floor" (:269-271)
  kStatusTroubleMax = 3,   // "troublemaker target is an extremum" (:305-306)
  kStatusHuge = 4,         // k_subloop handed a huge batch back to the host
};

// Label tiles (K3): 8192 vertices, power-of-two extents.
template <int DIM>
struct LabelTile;
template <>
struct LabelTile<2> {
  static constexpr int TX = 128, TY = 64, TZ = 1, LX = 7, LY = 6;
  static constexpr int kSurface = 2 * (TX + TY);
};
template <>
struct LabelTile<3> {
  static constexpr int TX = 32, TY = 16, TZ = 16, LX = 5, LY = 4;
  static constexpr int kSurface = 2 * (TX * TY + TY * TZ + TX * TZ);
};
template <int DIM>
__device__ __forceinline__ uint32_t label_tile_of(const Geom& g, uint32_t x, uint32_t y, uint32_t z) {
  using TL = LabelTile<DIM>;
  const uint32_t ntx = (g.X + TL::TX - 1) / TL::TX, nty = (g.Y + TL::TY - 1) / TL::TY;
  return x / TL::TX + ntx * (y / TL::TY + nty * (DIM == 2 ? 0u : z / TL::TZ));
}

// z-slab partition for label-table lookups on the device (shard.cuh)
constexpr int kMaxSlabs = 64;

struct SlabTable {  // the z partition, for label-table lookups on the device
  uint32_t P, XY;
  uint32_t z0[kMaxSlabs + 1];  // z0[P] = Z
};

__device__ __forceinline__ int slab_owner(const SlabTable& t, uint32_t z) {
  int lo = 0, hi = static_cast<int>(t.P) - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.z0[mid] <= z) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Slot of global vertex L in the gathered label table [rank][family][side][xy],
// or -1 when L is not on the first (side 0) or last (side 1) plane of its slab.
// Global ids are u64 (a sharded field may exceed 2^32 vertices; the reference
// caps grids at 2^40, grid.cpp:19); planes and window-local ids stay u32.
__device__ __forceinline__ int64_t table_slot(const SlabTable& t, uint64_t L, int fam) {
  const uint32_t z = static_cast<uint32_t>(L / t.XY);
  const int r = slab_owner(t, z);
  int side;
  if (z == t.z0[r]) side = 0;
  else if (z + 1 == t.z0[r + 1]) side = 1;
  else return -1;
  return ((static_cast<int64_t>(r) * 2 + fam) * 2 + side) * t.XY +
         static_cast<int64_t>(L - static_cast<uint64_t>(z) * t.XY);
}

// R target slot a rank does not own (z-slab windows): fix_batch's ownership test
// rejects it (ids are < 2^32 - 1)
constexpr uint32_t kNoTarget = 0xFFFFFFFFu;

// z-slab label resolution for the tile-based R kernels: a window-local final
// label lying on a slab boundary plane is replaced by its resolved table entry.
// tab == nullptr on a single device (labels are already final).
struct SlabRes {
  const uint64_t* tab;
  SlabTable t;
  uint64_t base;  // global id of window vertex 0
};
__device__ __forceinline__ uint64_t resolve_label(const SlabRes& r, uint32_t local, int fam) {
  if (!r.tab) return local + r.base;  // single device / one slab: base of the window (0 on a device)
  const uint64_t L = local + r.base;
  const int64_t sl = table_slot(r.t, L, fam);
  return sl >= 0 ? __ldg(r.tab + sl) : L;
}

template <class T>
struct State;

// ---------------------------------------------------------------------------
// K1: full direction sweep (compute_directions, mss.cpp:11-30) for f, f̂ and large batches.  2.5D
// streaming: a CTA owns a (BX x BY) column of the grid and walks it along the
// slowest axis with a ring of three shared-memory planes of SoS keys (halo 1),
// so every value is fetched once from L2/HBM and converted to its key once;
// each output direction then needs 15 shared-memory reads.
template <int DIM>
struct DirTile;
template <>
struct DirTile<2> {
  static constexpr int BX = 256, BY = 1;  // stream along y
};
template <>
struct DirTile<3> {
  static constexpr int BX = 64, BY = 8;  // stream along z
};

template <class T, int DIM>
__global__ void __launch_bounds__(DirTile<DIM>::BX * DirTile<DIM>::BY)
    k_directions_tiled(const T* __restrict__ vals, uint8_t* __restrict__ dir, Geom g, int chunk) {
  using K = typename KeyOf<T>::type;
  constexpr int BX = DirTile<DIM>::BX, BY = DirTile<DIM>::BY;
  constexpr int HX = BX + 2, HY = DIM == 2 ? 1 : BY + 2;
  constexpr int NT = BX * BY;
  constexpr int PL = (HX * HY + NT - 1) / NT;  // plane elements per thread
  constexpr int NR = StencilSize<DIM>::value + 1;
  __shared__ K ring[3][HY][HX];
  const int tx = threadIdx.x % BX, ty = threadIdx.x / BX;
  const int x0 = blockIdx.x * BX;
  const int y0 = DIM == 2 ? 0 : blockIdx.y * BY;
  const int S = DIM == 2 ? static_cast<int>(g.Y) : static_cast<int>(g.Z);  // streamed extent
  const int s0 = (DIM == 2 ? blockIdx.y : blockIdx.z) * chunk;
  const int s1 = min(s0 + chunk, S);
  // this thread's share of every halo plane: flat element ids, validity, base offset
  int64_t eoff[PL];
  bool evalid[PL];
#pragma unroll
  for (int j = 0; j < PL; ++j) {
    const int i = threadIdx.x + j * NT;
    const int hx = i % HX, hy = i / HX;
    const int x = x0 + hx - 1, y = DIM == 2 ? 0 : y0 + hy - 1;
    evalid[j] = i < HX * HY && x >= 0 && x < static_cast<int>(g.X) && y >= 0 &&
                y < static_cast<int>(g.Y);
    eoff[j] = evalid[j] ? static_cast<int64_t>(x) + static_cast<int64_t>(g.X) * y : 0;
  }
  const int64_t pstride = DIM == 2 ? static_cast<int64_t>(g.X) : static_cast<int64_t>(g.XY);
  // register pipeline: pre[u] holds a plane D steps ahead, so ~D planes of
  // loads are in flight per thread while the current plane is evaluated
  constexpr int D = 2;
  K pre[D][PL];
  auto fetch = [&](int sp, K* dst) {  // issue the loads of plane sp (no wait)
#pragma unroll
    for (int j = 0; j < PL; ++j)
      dst[j] = (evalid[j] && sp >= 0 && sp < S) ? okey(__ldg(vals + eoff[j] + pstride * sp)) : K(0);
  };
  auto commit = [&](int sp, const K* src) {
    const int slot = (sp + 3) % 3;
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      const int i = threadIdx.x + j * NT;
      if (i < HX * HY) (&ring[slot][0][0])[i] = src[j];
    }
  };
  fetch(s0 - 1, pre[0]);
  commit(s0 - 1, pre[0]);
  fetch(s0, pre[1]);
  commit(s0, pre[1]);
#pragma unroll
  for (int u = 0; u < D; ++u) fetch(s0 + 1 + u, pre[u]);
  const uint32_t x = x0 + tx;
  const uint32_t y = DIM == 2 ? 0 : y0 + ty;
  for (int sp0 = s0; sp0 < s1; sp0 += D) {
#pragma unroll
  for (int u = 0; u < D; ++u) {
    const int sp = sp0 + u;
    if (sp >= s1) break;
    commit(sp + 1, pre[u]);
    __syncthreads();
    fetch(sp + 1 + D, pre[u]);  // in flight while planes sp .. sp+D-1 are evaluated
    const uint32_t yy = DIM == 2 ? sp : y, zz = DIM == 2 ? 0 : sp;
    if (x < g.X && yy < g.Y) {
      uint32_t hc = kSelf, lc = kSelf;
      // Halo / out-of-grid cells hold key 0 (valid keys are >= 0x00800000...):
      // 0 never wins the ascending max, and key - 1 wraps to ~0 so it never
      // wins the descending min either -- no bounds tests per slot.
      const int row = (DIM == 2 ? 0 : ty + 1) * HX + tx + 1;
      const K* pl[3] = {&ring[(sp + 2) % 3][0][0] + row, &ring[sp % 3][0][0] + row,
                        &ring[(sp + 1) % 3][0][0] + row};
      K key[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int k = rank_slot<DIM>(r);
        int dx = 0, dy = 0, dz = 0;
        if (k != 15) stencil<DIM>(k, dx, dy, dz);
        const int ds = DIM == 2 ? dy : dz;
        key[r] = pl[ds + 1][(DIM == 2 ? 0 : dy * HX) + dx];
      }
      K hi = key[0], lo = key[0] - 1;
#pragma unroll
      for (int r = 1; r < NR; ++r) {
        hi = max(hi, key[r]);
        lo = min(lo, key[r] - 1);
      }
      // ties: ascending keeps the highest index (last in rank order),
      // descending the lowest index (first in rank order)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (key[r] == hi) hc = rank_slot<DIM>(r);
        if (key[NR - 1 - r] - 1 == lo) lc = rank_slot<DIM>(NR - 1 - r);
      }
      dir[static_cast<uint64_t>(x) + static_cast<uint64_t>(g.X) * yy +
          static_cast<uint64_t>(g.XY) * zz] = static_cast<uint8_t>(hc | (lc << 4));
    }
    __syncthreads();
  }
  }
}

// K1 (3D, block form).  The 3D Freudenthal link of (x,y,z) plus the vertex
// itself is exactly the union of four 2x2 cell blocks:
//   C(z-1) = {x-1,x} x {y-1,y} in plane z-1   slots 13, 9, 11, 5
//   C(z)   = {x-1,x} x {y-1,y} in plane z     slots  7, 3,  1, SELF
//   A(z)   = {x,x+1} x {y,y+1} in plane z     slots SELF, 0, 2, 6
//   A(z+1) = {x,x+1} x {y,y+1} in plane z+1   slots  4, 10, 8, 12
// whose vertex-index ranges are ordered C(z-1) < C(z) <= A(z) < A(z+1).  So each
// plane's 2x2 block extremes (with the SoS tie-break inside the block) are
// computed once per cell and every vertex combines four candidates in that
// order: >= for ascending (highest index wins ties), < for descending.
// Out-of-grid cells hold key 0 (and key-1 = ~0 for descending): they never win.
constexpr uint64_t kBlockSlot3 =  // nibble (candidate * 4 + position) -> stencil slot
    0xC8A4620FF1375B9Dull;

template <class K>
struct alignas(sizeof(K) == 4 ? 8 : 16) KeyPos {
  K key;
  uint32_t pos;
};

template <class T>
struct DirBlock3 {
  static constexpr int BX = 64, BY = sizeof(T) == 4 ? 8 : 4;
};

template <class T>
__global__ void __launch_bounds__(DirBlock3<T>::BX * DirBlock3<T>::BY)
    k_directions_block3(const T* __restrict__ vals, uint8_t* __restrict__ dir, Geom g, int chunk) {
  using K = typename KeyOf<T>::type;
  constexpr int BX = DirBlock3<T>::BX, BY = DirBlock3<T>::BY;
  constexpr int HX = BX + 2, HY = BY + 2;
  constexpr int BBX = BX + 1, NB = (BX + 1) * (BY + 1);
  constexpr int NT = BX * BY;
  constexpr int PL = (HX * HY + NT - 1) / NT;
  constexpr int D = 2;
  __shared__ K stage[HY * HX];
  __shared__ KeyPos<K> bmx[3][NB];
  __shared__ KeyPos<K> bmn[3][NB];
  const int tx = threadIdx.x % BX, ty = threadIdx.x / BX;
  const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
  const int S = static_cast<int>(g.Z);
  const int s0 = blockIdx.z * chunk;
  const int s1 = min(s0 + chunk, S);
  int64_t eoff[PL];
  bool evalid[PL];
#pragma unroll
  for (int j = 0; j < PL; ++j) {
    const int i = threadIdx.x + j * NT;
    const int hx = i % HX, hy = i / HX;
    const int x = x0 + hx - 1, y = y0 + hy - 1;
    evalid[j] = i < HX * HY && x >= 0 && x < static_cast<int>(g.X) && y >= 0 &&
                y < static_cast<int>(g.Y);
    eoff[j] = evalid[j] ? static_cast<int64_t>(x) + static_cast<int64_t>(g.X) * y : 0;
  }
  const int64_t pstride = static_cast<int64_t>(g.XY);
  K pre[D][PL];
  auto fetch = [&](int sp, K* dst) {
#pragma unroll
    for (int j = 0; j < PL; ++j)
      dst[j] = (evalid[j] && sp >= 0 && sp < S) ? okey(__ldg(vals + eoff[j] + pstride * sp)) : K(0);
  };
  auto commit = [&](const K* src) {
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      const int i = threadIdx.x + j * NT;
      if (i < HX * HY) stage[i] = src[j];
    }
  };
  // block extremes of the staged plane into ring slot `slot`
  auto build = [&](int slot) {
    for (int b = threadIdx.x; b < NB; b += NT) {
      const int bx = b % BBX, by = b / BBX;
      const K c0 = stage[by * HX + bx], c1 = stage[by * HX + bx + 1];
      const K c2 = stage[(by + 1) * HX + bx], c3 = stage[(by + 1) * HX + bx + 1];
      K hk = c0, lk = c0 - 1;
      uint32_t hp = 0, lp = 0;
      if (c1 >= hk) { hk = c1; hp = 1; }
      if (c2 >= hk) { hk = c2; hp = 2; }
      if (c3 >= hk) { hk = c3; hp = 3; }
      if (c1 - 1 < lk) { lk = c1 - 1; lp = 1; }
      if (c2 - 1 < lk) { lk = c2 - 1; lp = 2; }
      if (c3 - 1 < lk) { lk = c3 - 1; lp = 3; }
      bmx[slot][b] = KeyPos<K>{hk, hp};
      bmn[slot][b] = KeyPos<K>{lk, lp};
    }
  };
  fetch(s0 - 1, pre[0]);
  commit(pre[0]);
  __syncthreads();
  build((s0 + 2) % 3);
  __syncthreads();
  fetch(s0, pre[0]);
  commit(pre[0]);
  __syncthreads();
  build(s0 % 3);
#pragma unroll
  for (int u = 0; u < D; ++u) fetch(s0 + 1 + u, pre[u]);
  const uint32_t x = x0 + tx, y = y0 + ty;
  const int ci = ty * BBX + tx, ai = (ty + 1) * BBX + tx + 1;
  for (int sp0 = s0; sp0 < s1; sp0 += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int sp = sp0 + u;
      if (sp >= s1) break;
      __syncthreads();  // previous build / compute done before the stage is rewritten
      commit(pre[u]);
      __syncthreads();
      fetch(sp + 1 + D, pre[u]);
      build((sp + 1) % 3);
      __syncthreads();
      if (x < g.X && y < g.Y) {
        const int sm = (sp + 2) % 3, s0_ = sp % 3, sp1 = (sp + 1) % 3;
        const KeyPos<K> a0 = bmx[sm][ci], a1 = bmx[s0_][ci], a2 = bmx[s0_][ai], a3 = bmx[sp1][ai];
        const KeyPos<K> d0 = bmn[sm][ci], d1 = bmn[s0_][ci], d2 = bmn[s0_][ai], d3 = bmn[sp1][ai];
        K hk = a0.key, lk = d0.key;
        uint32_t hi = a0.pos, lo = d0.pos;
        if (a1.key >= hk) { hk = a1.key; hi = 4 + a1.pos; }
        if (a2.key >= hk) { hk = a2.key; hi = 8 + a2.pos; }
        if (a3.key >= hk) { hk = a3.key; hi = 12 + a3.pos; }
        if (d1.key < lk) { lk = d1.key; lo = 4 + d1.pos; }
        if (d2.key < lk) { lk = d2.key; lo = 8 + d2.pos; }
        if (d3.key < lk) { lk = d3.key; lo = 12 + d3.pos; }
        const uint32_t hc = static_cast<uint32_t>(kBlockSlot3 >> (4 * hi)) & 15u;
        const uint32_t lc = static_cast<uint32_t>(kBlockSlot3 >> (4 * lo)) & 15u;
        dir[static_cast<uint64_t>(x) + static_cast<uint64_t>(g.X) * y +
            static_cast<uint64_t>(g.XY) * sp] = static_cast<uint8_t>(hc | (lc << 4));
      }
    }
  }
}

// K1 (3D, f32, register-blocked).  Same decomposition as k_directions_block3,
// restructured so per-vertex work is a handful of compares:
//  * a warp owns one grid row of a 128-wide tile, each lane 4 consecutive x
//    (one 16-byte load and one 4-byte store per lane per plane); warps 1..H
//    are output rows, warp 0 the halo row above (cells only), warp H+1 the
//    halo row below (keys only);
//  * cell(x,y,z) = the 2x2 block {x,x+1} x {y,y+1} of plane z, extremes with
//    their position (SoS: >= keeps the later index for ascending, < the
//    earlier for descending);
//  * the A pair of vertex (x,y,z) is VA(x,y,z) = [cell(x,y,z), cell(x,y,z+1)];
//    its C pair [cell(x-1,y-1,z-1), cell(x-1,y-1,z)] is VA(x-1,y-1,z-1), so
//    each pair is reduced once by its own thread and read once by the vertex
//    at (x+1, y+1, z+1) through shared memory;
//  * one barrier per plane: keys of plane p+1 and VA of plane p-1 are
//    published while plane p-1's vertices read VA of plane p-2 (2 key slots,
//    3 VA slots).
// Keys: order-preserving u32 (x + 0.0f maps -0 to +0: SoS ties them); cells
// outside the grid hold key 0, which never wins ascending (key) nor
// descending (key - 1 wraps to ~0).
constexpr int kD3W = 128, kD3H = 14, kD3Warps = kD3H + 2, kD3P = 136;

__device__ __forceinline__ uint32_t fkey(float x) {
  const uint32_t b = __float_as_uint(x + 0.0f);
  return b ^ (static_cast<uint32_t>(static_cast<int32_t>(b) >> 31) | 0x80000000u);
}

// 2x2 cell extremes; corners in index order c0 (x,y) c1 (x+1,y) c2 (x,y+1) c3 (x+1,y+1).
// pos = ascending corner | descending corner << 2
__device__ __forceinline__ void cell_ext(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t& a,
                                         uint32_t& d, uint32_t& pos) {
  uint32_t hp = 0, lp = 0;
  a = c0;
  if (c1 >= a) { a = c1; hp = 1; }
  if (c2 >= a) { a = c2; hp = 2; }
  if (c3 >= a) { a = c3; hp = 3; }
  d = c0 - 1;
  if (c1 - 1 < d) { d = c1 - 1; lp = 1; }
  if (c2 - 1 < d) { d = c2 - 1; lp = 2; }
  if (c3 - 1 < d) { d = c3 - 1; lp = 3; }
  pos = hp | (lp << 2);
}

// pair [lower plane, upper plane] of cells: pos byte = asc (0..7) | desc (0..7) << 4
__device__ __forceinline__ void pair_ext(uint32_t a0, uint32_t d0, uint32_t p0, uint32_t a1, uint32_t d1,
                                         uint32_t p1, uint32_t& a, uint32_t& d, uint32_t& pos) {
  uint32_t hp = p0 & 3u, lp = p0 >> 2;
  a = a0;
  d = d0;
  if (a1 >= a) { a = a1; hp = 4 + (p1 & 3u); }
  if (d1 < d) { d = d1; lp = 4 + (p1 >> 2); }
  pos = hp | (lp << 4);
}

struct D3Smem {
  uint32_t skey[2][kD3Warps][kD3P];  // keys per row (column x at x - x0 + 4)
  uint32_t sva[2][kD3H + 1][kD3P];   // VA ascending keys per cell row
  uint32_t svd[2][kD3H + 1][kD3P];   // VA descending keys
  uint8_t svp[2][kD3H + 1][kD3P];    // VA positions
};

// per-thread constants of k_directions_reg3
struct D3Ctx {
  const float* vals;
  uint8_t* dir;
  int64_t XY, rowbase;
  int lane, w, x0, xl, c, X, Z, s1;
  bool row_in, cells, out;
};

// state carried from plane p-1 to plane p
struct D3State {
  uint4 k;                    // this row's keys of plane p
  uint32_t kh;                // halo key of plane p (lane 0: x0-1, lane 31: x0+128)
  uint32_t ca[5], cd[5], cp;  // cells of plane p-1 (own 4 + lane 0's x0-1), positions 4 bits each
};

template <bool kVec>
__device__ __forceinline__ void d3_load(const D3Ctx& t, int z, float4& v, float& h) {
  v = make_float4(0.f, 0.f, 0.f, 0.f);
  h = 0.f;
  if (!t.row_in || z < 0 || z >= t.Z) return;
  const float* base = t.vals + t.XY * z + t.rowbase;
  if (kVec) {
    if (t.xl < t.X) v = __ldg(reinterpret_cast<const float4*>(base + t.xl));
  } else {
    if (t.xl < t.X) v.x = __ldg(base + t.xl);
    if (t.xl + 1 < t.X) v.y = __ldg(base + t.xl + 1);
    if (t.xl + 2 < t.X) v.z = __ldg(base + t.xl + 2);
    if (t.xl + 3 < t.X) v.w = __ldg(base + t.xl + 3);
  }
  if (t.lane == 0 && t.x0 > 0) h = __ldg(base + t.x0 - 1);
  if (t.lane == 31 && t.x0 + kD3W < t.X) h = __ldg(base + t.x0 + kD3W);
}

__device__ __forceinline__ void d3_keys(const D3Ctx& t, int z, const float4& v, float h, uint4& k, uint32_t& kh) {
  const bool zin = t.row_in && z >= 0 && z < t.Z;
  k.x = (zin && t.xl < t.X) ? fkey(v.x) : 0u;
  k.y = (zin && t.xl + 1 < t.X) ? fkey(v.y) : 0u;
  k.z = (zin && t.xl + 2 < t.X) ? fkey(v.z) : 0u;
  k.w = (zin && t.xl + 3 < t.X) ? fkey(v.w) : 0u;
  const bool hin = zin && ((t.lane == 0 && t.x0 > 0) || (t.lane == 31 && t.x0 + kD3W < t.X));
  kh = hin ? fkey(h) : 0u;
}

__device__ __forceinline__ void d3_publish(const D3Ctx& t, uint32_t (*sk)[kD3P], const uint4& k, uint32_t kh) {
  *reinterpret_cast<uint4*>(&sk[t.w][t.c]) = k;
  if (t.lane == 0) sk[t.w][3] = kh;
  if (t.lane == 31) sk[t.w][kD3W + 4] = kh;
}

// One plane step (see k_directions_reg3).  PAR = parity of the step: keys of
// plane p sit in key slot PAR, VA(p-1) goes to VA slot PAR, VA(p-2) is read
// from slot PAR ^ 1.  pv/ph hold plane p+1's values on entry and receive
// plane p+3's on exit.
template <int PAR, bool kVec>
__device__ __forceinline__ void d3_step(const D3Ctx& t, D3Smem& S, int p, int s0, const D3State& in,
                                        D3State& o, float4& pv, float& ph) {
  // 1. keys of plane p+1 -> key slot PAR^1
  d3_keys(t, p + 1, pv, ph, o.k, o.kh);
  d3_publish(t, S.skey[PAR ^ 1], o.k, o.kh);
  d3_load<kVec>(t, p + 3, pv, ph);
  // 2. cells of plane p: rows y (in.k) and y+1 (smem)
  o.cp = 0;
  if (t.cells) {
    const uint32_t* below = S.skey[PAR][t.w + 1];
    const uint4 b = *reinterpret_cast<const uint4*>(below + t.c);
    const uint32_t b4 = below[t.c + 4];
    uint32_t a4 = __shfl_down_sync(0xffffffffu, in.k.x, 1);
    if (t.lane == 31) a4 = in.kh;
    uint32_t q;
    cell_ext(in.k.x, in.k.y, b.x, b.y, o.ca[0], o.cd[0], q);
    o.cp = q;
    cell_ext(in.k.y, in.k.z, b.y, b.z, o.ca[1], o.cd[1], q);
    o.cp |= q << 4;
    cell_ext(in.k.z, in.k.w, b.z, b.w, o.ca[2], o.cd[2], q);
    o.cp |= q << 8;
    cell_ext(in.k.w, a4, b.w, b4, o.ca[3], o.cd[3], q);
    o.cp |= q << 12;
    o.ca[4] = 0;
    o.cd[4] = ~0u;
    if (t.lane == 0) {
      cell_ext(in.kh, in.k.x, below[3], b.x, o.ca[4], o.cd[4], q);
      o.cp |= q << 16;
    }
  }
  if (p < s0 || !t.cells) return;
  // 3. VA(p-1) = [cell(p-1), cell(p)] -> VA slot PAR
  uint32_t va[4], vd[4], vpk = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t q;
    pair_ext(in.ca[i], in.cd[i], (in.cp >> (4 * i)) & 15u, o.ca[i], o.cd[i], (o.cp >> (4 * i)) & 15u, va[i],
             vd[i], q);
    vpk |= q << (8 * i);
  }
  *reinterpret_cast<uint4*>(&S.sva[PAR][t.w][t.c]) = make_uint4(va[0], va[1], va[2], va[3]);
  *reinterpret_cast<uint4*>(&S.svd[PAR][t.w][t.c]) = make_uint4(vd[0], vd[1], vd[2], vd[3]);
  *reinterpret_cast<uint32_t*>(&S.svp[PAR][t.w][t.c]) = vpk;
  if (t.lane == 0) {
    uint32_t ea, ed, ep;
    pair_ext(in.ca[4], in.cd[4], (in.cp >> 16) & 15u, o.ca[4], o.cd[4], (o.cp >> 16) & 15u, ea, ed, ep);
    S.sva[PAR][t.w][3] = ea;
    S.svd[PAR][t.w][3] = ed;
    S.svp[PAR][t.w][3] = static_cast<uint8_t>(ep);
  }
  // 4. vertices of plane p-1: C pair = VA(x-1, y-1, p-2) (slot PAR^1), A pair = own VA(p-1)
  if (p < s0 + 1 || p - 1 >= t.s1 || !t.out) return;
  const uint32_t* ra = S.sva[PAR ^ 1][t.w - 1];
  const uint32_t* rd = S.svd[PAR ^ 1][t.w - 1];
  const uint8_t* rp = S.svp[PAR ^ 1][t.w - 1];
  const uint4 qa = *reinterpret_cast<const uint4*>(ra + t.c);
  const uint4 qd = *reinterpret_cast<const uint4*>(rd + t.c);
  const uint32_t Cpk = (*reinterpret_cast<const uint32_t*>(rp + t.c) << 8) | rp[t.c - 1];
  const uint32_t Ca[4] = {ra[t.c - 1], qa.x, qa.y, qa.z};
  const uint32_t Cd[4] = {rd[t.c - 1], qd.x, qd.y, qd.z};
  uint32_t codes = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t cpi = (Cpk >> (8 * i)) & 0xFFu, vpi = (vpk >> (8 * i)) & 0xFFu;
    const uint32_t hi = va[i] >= Ca[i] ? 8 + (vpi & 15u) : (cpi & 15u);
    const uint32_t lo = vd[i] < Cd[i] ? 8 + (vpi >> 4) : (cpi >> 4);
    const uint32_t hc = static_cast<uint32_t>(kBlockSlot3 >> (4 * hi)) & 15u;
    const uint32_t lc = static_cast<uint32_t>(kBlockSlot3 >> (4 * lo)) & 15u;
    codes |= (hc | (lc << 4)) << (8 * i);
  }
  uint8_t* op = t.dir + t.XY * (p - 1) + t.rowbase + t.xl;
  if (kVec) {
    if (t.xl < t.X) *reinterpret_cast<uint32_t*>(op) = codes;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (t.xl + i < t.X) op[i] = static_cast<uint8_t>(codes >> (8 * i));
  }
}

template <bool kVec, int kMinBlocks>
__global__ void __launch_bounds__(kD3Warps * 32, kMinBlocks)
    k_directions_reg3(const float* __restrict__ vals, uint8_t* __restrict__ dir, Geom g, int chunk) {
  extern __shared__ __align__(16) unsigned char d3raw[];
  D3Smem& S = *reinterpret_cast<D3Smem*>(d3raw);
  D3Ctx t;
  t.vals = vals;
  t.dir = dir;
  t.lane = threadIdx.x & 31;
  t.w = threadIdx.x >> 5;
  t.x0 = blockIdx.x * kD3W;
  const int y0 = blockIdx.y * kD3H;
  const int y = y0 - 1 + t.w;
  t.xl = t.x0 + 4 * t.lane;
  t.c = 4 * t.lane + 4;
  t.X = static_cast<int>(g.X);
  t.Z = static_cast<int>(g.Z);
  t.XY = g.XY;
  t.rowbase = static_cast<int64_t>(y) * t.X;
  t.row_in = y >= 0 && y < static_cast<int>(g.Y);
  t.cells = t.w <= kD3H;
  t.out = t.w >= 1 && t.w <= kD3H && t.row_in;
  const int s0 = blockIdx.z * chunk;
  t.s1 = min(s0 + chunk, t.Z);
  D3State A, B;
  float4 pa, pb;  // values of planes p+1 (pa) and p+2 (pb) at an even step
  float ha, hb;
  {
    float4 v;
    float h;
    d3_load<kVec>(t, s0 - 1, v, h);
    d3_keys(t, s0 - 1, v, h, A.k, A.kh);
    d3_publish(t, S.skey[0], A.k, A.kh);
    d3_load<kVec>(t, s0, pa, ha);
    d3_load<kVec>(t, s0 + 1, pb, hb);
  }
  __syncthreads();
  // planes p = s0-1 .. s1 (the last step may run one past s1; it writes nothing)
  for (int p = s0 - 1; p <= t.s1; p += 2) {
    d3_step<0, kVec>(t, S, p, s0, A, B, pa, ha);
    __syncthreads();
    d3_step<1, kVec>(t, S, p + 1, s0, B, A, pb, hb);
    __syncthreads();
  }
}

// K1 (3D, f32, register columns) -- the default 3D f32 sweep since round 2.
// Same cube decomposition as the block forms above, rearranged so that no
// shared memory, no barrier and no packed position fields are involved:
//  * the up-cube of (x,y,z) is {x,x+1} x {y,y+1} x {z,z+1}; the link of a
//    vertex plus itself is up-cube(x,y,z) (VA) ∪ up-cube(x-1,y-1,z-1) (C),
//    with index ranges C <= self <= VA;
//  * a lane owns one column x (lanes 0..31 cover x0-1 .. x0+30; lanes 1..30
//    produce output) and a warp kK1R consecutive output rows, streaming z;
//  * every extreme is built separably: x-pairs (x, x+1) via one shuffle, cells
//    by joining the x-pairs of rows y and y+1 (registers of the same lane),
//    cubes by joining the cells of planes z and z+1 (the previous plane's
//    cells stay in registers), C by shuffling the previous plane's cube of row
//    y-1 up one lane;
//  * a level joins (lower, upper) halves whose indices are all ordered lower <
//    upper, so the SoS tie-break is ">= keeps upper" ascending and "< takes
//    upper" descending at every level, exactly the scan order of sos_greater /
//    sos_less (grid.hpp:53-63) over index-ranked slots;
//  * positions are cube corner ids pre-multiplied by 4 (x: 4, y: 8, z: 16), so
//    the final slot is one shift of a 32-bit half of kBlockSlot3.
// Out-of-grid vertices hold key 0 (key-1 = ~0 descending): they never win.
constexpr int kK1R = 8;      // output rows per warp
constexpr int kK1Warps = 8;  // warps per CTA, stacked in y
constexpr int kK1Cols = 30;  // output columns per warp (lanes 1..30)

struct K1Ext {
  uint32_t ak, ap;  // ascending: key, position * 4
  uint32_t dk, dp;  // descending: key - 1, position * 4
};

// join(lower, upper): `bit` is the upper half's position bit (pre-multiplied)
__device__ __forceinline__ K1Ext k1_join(const K1Ext& lo, const K1Ext& hi, uint32_t bit) {
  K1Ext r;
  const bool ta = hi.ak >= lo.ak;
  r.ak = ta ? hi.ak : lo.ak;
  r.ap = ta ? (hi.ap | bit) : lo.ap;
  const bool td = hi.dk < lo.dk;
  r.dk = td ? hi.dk : lo.dk;
  r.dp = td ? (hi.dp | bit) : lo.dp;
  return r;
}

__device__ __forceinline__ K1Ext k1_xpair(uint32_t k, uint32_t dk) {  // (x, x+1) of one row
  const uint32_t k1 = __shfl_down_sync(0xffffffffu, k, 1);
  const uint32_t dk1 = k1 - 1u;  // one shuffle: the shuffle pipe is shared with L1/shared
  K1Ext r;
  const bool ta = k1 >= k;
  r.ak = ta ? k1 : k;
  r.ap = ta ? 4u : 0u;
  const bool td = dk1 < dk;
  r.dk = td ? dk1 : dk;
  r.dp = td ? 4u : 0u;
  return r;
}

__device__ __forceinline__ uint32_t k1_code(const K1Ext& va, const K1Ext& c) {
  constexpr uint32_t kLoC = static_cast<uint32_t>(kBlockSlot3);         // C cube corners
  constexpr uint32_t kHiVA = static_cast<uint32_t>(kBlockSlot3 >> 32);  // VA cube corners
  const bool ta = va.ak >= c.ak;
  const uint32_t sa = (ta ? kHiVA : kLoC) >> (ta ? va.ap : c.ap);
  const bool td = va.dk < c.dk;
  const uint32_t sd = (td ? kHiVA : kLoC) >> (td ? va.dp : c.dp);
  return (sa & 15u) | ((sd & 15u) << 4);
}

// one plane step: keys of plane q (k, dk = k - 1) -> cells(q), cubes(q-1) from
// cells(q-1) (per thread and row in shared memory, `cell`) and cells(q), codes
// of plane q-1 when `emit`, then C <- cubes(q-1) of rows y-1 one lane to the left
// (shuffled: no shared-memory traffic)
__device__ __forceinline__ void k1_plane(const uint32_t (&k)[kK1R + 2], const uint32_t (&dk)[kK1R + 2],
                                         uint4* cell, K1Ext (&C)[kK1R], bool cubes, bool emit, uint8_t* out,
                                         uint32_t X, uint32_t rows_out) {
  constexpr int kStride = kK1Warps * 32;
  K1Ext xp = k1_xpair(k[0], dk[0]);
  K1Ext held;  // this plane's cube of row j-1 shifted up one lane, parked until row j-1's codes are out
#pragma unroll
  for (int j = 0; j <= kK1R; ++j) {
    const K1Ext xq = k1_xpair(k[j + 1], dk[j + 1]);
    const K1Ext nw = k1_join(xp, xq, 8u);
    xp = xq;
    uint4& slot = cell[j * kStride];
    if (cubes) {
      const uint4 p = slot;
      const K1Ext cube = k1_join(K1Ext{p.x, p.y, p.z, p.w}, nw, 16u);
      if (j >= 1) {
        // output row j-1: VA = cube row j, C = previous plane's cube row j-1 of lane - 1
        const uint32_t code = k1_code(cube, C[j - 1]);
        if (emit && static_cast<uint32_t>(j - 1) < rows_out) out[static_cast<uint64_t>(j - 1) * X] = static_cast<uint8_t>(code);
        C[j - 1] = held;
      }
      if (j < kK1R) {
        held.ak = __shfl_up_sync(0xffffffffu, cube.ak, 1);
        held.ap = __shfl_up_sync(0xffffffffu, cube.ap, 1);
        held.dk = __shfl_up_sync(0xffffffffu, cube.dk, 1);
        held.dp = __shfl_up_sync(0xffffffffu, cube.dp, 1);
      }
    }
    slot = make_uint4(nw.ak, nw.ap, nw.dk, nw.dp);
  }
}

constexpr size_t k1_smem_bytes() { return sizeof(uint4) * (kK1R + 1) * kK1Warps * 32; }

__global__ void __launch_bounds__(kK1Warps * 32, 2)
    k_directions_col3(const float* __restrict__ vals, uint8_t* __restrict__ dir, Geom g, int chunk) {
  constexpr int R = kK1R;
  // per [row][thread] 16-byte slots (conflict-free): the previous plane's cells (rows 0..R)
  extern __shared__ uint4 k1_smem[];  // k1_smem_bytes()
  uint4* scell = k1_smem;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x = static_cast<int>(blockIdx.x) * kK1Cols - 1 + lane;
  const int y0 = (static_cast<int>(blockIdx.y) * kK1Warps + w) * R;  // first output row
  const int X = static_cast<int>(g.X), Y = static_cast<int>(g.Y), Z = static_cast<int>(g.Z);
  const int s0 = static_cast<int>(blockIdx.z) * chunk, s1 = min(s0 + chunk, Z);
  if (y0 >= Y) return;  // warp-uniform; no block-wide barrier below
  const bool xok = x >= 0 && x < X;
  uint32_t rowok = 0;  // key rows y0-1 .. y0+R
#pragma unroll
  for (int r = 0; r < R + 2; ++r) rowok |= (y0 - 1 + r >= 0 && y0 - 1 + r < Y ? 1u : 0u) << r;
  if (!xok) rowok = 0;
  const bool out_lane = lane >= 1 && lane <= kK1Cols && xok;
  const uint32_t rows_out = out_lane ? static_cast<uint32_t>(min(R, Y - y0)) : 0u;
  uint4* cell = scell + threadIdx.x;
  // row r of plane q sits at q*XY + (y0-1+r)*X + x (u32: N < 2^32 per device)
  const uint32_t base = static_cast<uint32_t>(y0 - 1) * g.X + static_cast<uint32_t>(x);
  const uint32_t X1 = g.X;
  // out-of-grid rows load vertex 0 (their keys are forced to 0): no predicated
  // loads; warps whose rows and columns are all inside skip the per-row tests
  constexpr uint32_t kAll = (1u << (R + 2)) - 1;
  const bool inside = __all_sync(0xffffffffu, rowok == kAll);
  auto load = [&](int q, float (&v)[R + 2]) {
    const uint32_t pb = base + static_cast<uint32_t>(q) * g.XY;  // wraps for row y0-1 = -1
    if (inside && q >= 0 && q < Z) {
#pragma unroll
      for (int r = 0; r < R + 2; ++r) v[r] = __ldg(vals + (pb + r * X1));
    } else {
      const uint32_t ok = (q >= 0 && q < Z) ? rowok : 0u;
#pragma unroll
      for (int r = 0; r < R + 2; ++r) v[r] = __ldg(vals + (((ok >> r) & 1u) ? pb + r * X1 : 0u));
    }
  };
  auto keys = [&](int q, const float (&v)[R + 2], uint32_t (&k)[R + 2], uint32_t (&dk)[R + 2]) {
    if (inside && q >= 0 && q < Z) {
#pragma unroll
      for (int r = 0; r < R + 2; ++r) k[r] = fkey(v[r]);
    } else {
      const uint32_t ok = (q >= 0 && q < Z) ? rowok : 0u;
#pragma unroll
      for (int r = 0; r < R + 2; ++r) k[r] = ((ok >> r) & 1u) ? fkey(v[r]) : 0u;
    }
#pragma unroll
    for (int r = 0; r < R + 2; ++r) dk[r] = k[r] - 1u;
  };
  float v[R + 2];
  uint32_t k[R + 2], dk[R + 2];
  K1Ext C[R];
  load(s0 - 1, v);
  // q = s0-1: cells only; q = s0: cubes(s0-1); then one plane per trip
  keys(s0 - 1, v, k, dk);
  load(s0, v);
  k1_plane(k, dk, cell, C, false, false, nullptr, g.X, 0);
  keys(s0, v, k, dk);
  load(s0 + 1, v);
  k1_plane(k, dk, cell, C, true, false, nullptr, g.X, 0);
  uint8_t* out = dir + (base + g.X) + static_cast<uint64_t>(s0) * g.XY;  // row y0, plane s0
  for (int q = s0 + 1; q <= s1; ++q) {
    keys(q, v, k, dk);
    load(q + 1, v);
    k1_plane(k, dk, cell, C, true, true, out, g.X, rows_out);
    out += g.XY;
  }
}

// K1b (k_detect_kind, the full detect sweep) is defined with the subloop helpers below.

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
// Every helper takes (tid, stride) so it runs either grid-wide or inside one CTA.
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
  // z-slab windows: final f labels as u64 global ids (nullptr on a single device,
  // where fM / fm are the final labels)
  const uint64_t* fM64;
  const uint64_t* fm64;
  double xi;
  Ctl* ctl;
  uint8_t* tdirty;  // R-loop only: label tiles whose direction codes changed
  // z-slab sharding (shard.cuh): fixes lower only targets in [own_lo, own_lo + own_n),
  // frontier refreshes only vertices in [act_lo, act_lo + act_n) (owned planes plus
  // one halo plane per side).  Single device: both ranges are the whole grid.
  uint32_t own_lo, own_n, act_lo, act_n;
  uint32_t* cstamp;  // per 64-vertex chunk: mark id of the last batch that changed a code in it
};

// fmark value of a parked worklist item (never a batch mark: marks stay below
// 0xF0000000, Workspace::ensure)
constexpr uint32_t kParked = 0xFFFFFFFFu;

// list items per lane per step in fix_batch (1 or 2; MSSZ_FIX_PER_LANE at build)
#ifndef MSSZ_FIX_PER_LANE
#define MSSZ_FIX_PER_LANE 2
#endif
constexpr int kFixPerLane = MSSZ_FIX_PER_LANE;
#ifndef MSSZ_FIX_LIST_PER_LANE
#define MSSZ_FIX_LIST_PER_LANE 4
#endif

// claim (edit_engine.cpp:160-169) + lower_step (:75-86): the first claimant of
// t in this batch lowers it from the pre-batch value; exactly one winner per
// target, so Σ winners == the reference's applied count.
template <class T>
__device__ __forceinline__ bool claim_and_lower(const State<T>& s, uint32_t t, uint32_t batch) {
  if (atomicExch(&s.stamp[t], batch) == batch) return false;
  T nv;
  if (!lower_value<T>(__ldcg(s.g + t), __ldg(s.f + t), s.xi, nv)) return false;
  s.g[t] = nv;
  if (s.touched) s.touched[t] = 1;
  return true;
}

// retry (optional): list items whose target this item did not lower itself
// (claim lost, or target at its floor).  Every other item is a neighbour of
// (or is) a lowered target, hence in this batch's frontier, and is
// re-evaluated there; only retry items need the old-list membership test.
template <class T, int J = kFixPerLane>
__device__ __forceinline__ void fix_batch(const State<T>& s, const uint32_t* __restrict__ list,
                                          uint32_t n, int rule, uint32_t batch, uint32_t* s_count,
                                          uint64_t tid, uint64_t stride, uint32_t* retry = nullptr,
                                          uint32_t* retry_count = nullptr, uint32_t* park = nullptr,
                                          uint32_t* park_count = nullptr) {
  // J list items per lane per step: their loads and claims overlap
  const uint64_t step = J * stride;
  __shared__ uint32_t sstage[kStageWarps][kStageK * 32], rstage[kStageWarps][kStageK * 32];
  WarpBuffer<kStageK> sbuf(warp_stage(sstage)), rbuf(warp_stage(rstage));
  for (uint64_t wb = (tid & ~uint64_t(31)) * J; wb < n; wb += step) {
    uint32_t t[J], v[J], prev[J];
    bool live[J], ok[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint64_t i = wb + (threadIdx.x & 31) + 32 * j;
      live[j] = i < n;
      v[j] = live[j] ? __ldcg(list + i) : 0u;
      t[j] = 0;
      prev[j] = batch;
      ok[j] = false;
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (!live[j]) continue;
      if (rule == 0) t[j] = v[j];
      else if (rule == 1) t[j] = v[j] + s.geo.off[__ldcg(s.gdir + v[j]) & 15u];
      else t[j] = v[j] + s.geo.off[__ldg(s.fdir + v[j]) >> 4];
    }
#pragma unroll
    for (int j = 0; j < J; ++j)  // only the owner of a target lowers it (owner-computes)
      if (live[j] && t[j] - s.own_lo < s.own_n) prev[j] = atomicExch(&s.stamp[t[j]], batch);
    T gv[J], fv[J];
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (prev[j] != batch) {
        gv[j] = __ldcg(s.g + t[j]);
        fv[j] = __ldg(s.f + t[j]);
      }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      T nv;
      if (prev[j] != batch && lower_value<T>(gv[j], fv[j], s.xi, nv)) {
        s.g[t[j]] = nv;
        if (s.touched) s.touched[t[j]] = 1;  // single device: derived at compaction
        ok[j] = true;
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) sbuf.push(ok[j], t[j], s.S, s_count);
    if (park) {  // won the claim, target at its floor: park the item (see k_subloop)
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const bool pk = live[j] && prev[j] != batch && !ok[j];
        if (pk) s.fmark[v[j]] = kParked;
        rbuf.push(pk, v[j], park, park_count);
      }
    } else if (retry) {
#pragma unroll
      for (int j = 0; j < J; ++j) rbuf.push(live[j] && !ok[j], v[j], retry, retry_count);
    }
  }
  sbuf.flush(s.S, s_count);
  if (park) rbuf.flush(park, park_count);
  else if (retry) rbuf.flush(retry, retry_count);
}

// Stencil slot k -> (dx, dy, dz) without tables: slots come in (+d, -d) pairs
// (grid.cpp:8-16); pair j's components are bit j of a per-axis mask.
template <int DIM>
__device__ __forceinline__ void slot_delta(int k, int& dx, int& dy, int& dz) {
  const int j = k >> 1, sgn = (k & 1) ? -1 : 1;
  if (DIM == 2) {
    dx = ((0x5 >> j) & 1) * sgn;
    dy = ((0x6 >> j) & 1) * sgn;
    dz = 0;
  } else {
    dx = ((0x69 >> j) & 1) * sgn;
    dy = ((0x5A >> j) & 1) * sgn;
    dz = ((0x74 >> j) & 1) * sgn;
  }
}

// Re-evaluates gdir where a batch can have changed it, each vertex once (fmark
// dedupe), and collects the re-evaluated vertices in F.
// One lane per (edited vertex t, u in {t} ∪ N(t)): 16 lanes per edit in 3D,
// 8 in 2D.  A batch only LOWERS values, so for u (with all lowered values
// final):
//   * asc(u) = SoS-argmax over {u} ∪ N(u) can change only if asc(u) itself
//     was lowered (any other member only decreased);
//   * desc(u) can change only if some lowered t in {u} ∪ N(u) now beats the
//     current minimum desc(u) in SoS order.
// So lane (t, u) recomputes u only when asc(u) == t or t <_SoS desc(u): two
// loads decide, and every vertex whose code can change is recomputed by the
// lane of the edit that changed it.  Unchanged codes keep their class, so the
// old worklist's entries that were not recomputed stay valid (rebuild_retry).
// A stale gdir[u] read (another lane recomputing u concurrently) is harmless:
// the recompute reads final values, and a claim lost to it changes nothing.
// next (optional, C-loop): instead of collecting F, append every re-evaluated
// vertex that is of `kind` under its refreshed code straight to the next
// worklist (f_count then only counts them).
template <class T, int DIM>
__device__ __forceinline__ void frontier_update(const State<T>& s, uint32_t ns, uint32_t mark,
                                                uint32_t* f_count, uint64_t tid, uint64_t stride,
                                                int kind = -1, uint32_t* next = nullptr,
                                                uint32_t* next_count = nullptr) {
  constexpr int LPS = DIM == 2 ? 8 : 16;  // lanes per edited vertex
  constexpr int NS = StencilSize<DIM>::value;
  const uint64_t total = static_cast<uint64_t>(ns) * LPS;
  __shared__ uint32_t nstage[kStageWarps][kStageK * 32];
  WarpBuffer<kStageK> nbuf(warp_stage(nstage));
  uint32_t nmine = 0;
  // software pipeline over the dependent chain S -> gdir -> g -> fmark ->
  // recompute: a lane's edited vertex is loaded two iterations ahead and its
  // neighbour's code one iteration ahead
  constexpr uint32_t kNone = 0xFFFFFFFFu;
  auto load_sv = [&](uint64_t i) -> uint32_t {
    return (i < total && static_cast<int>(i % LPS) <= NS) ? __ldcg(s.S + i / LPS) : 0u;
  };
  auto locate = [&](uint64_t i, uint32_t sv) -> uint32_t {  // lane i's vertex u, or kNone
    if (i >= total) return kNone;
    const int k = static_cast<int>(i % LPS) - 1;  // -1 = the edited vertex itself
    if (k >= NS) return kNone;
    uint32_t x, y, z;
    coords(s.geo, sv, x, y, z);
    int dx = 0, dy = 0, dz = 0;
    if (k >= 0) slot_delta<DIM>(k, dx, dy, dz);
    const uint32_t ux = x + dx, uy = y + dy, uz = z + dz;
    if (!(ux < s.geo.X && uy < s.geo.Y && (DIM == 2 || uz < s.geo.Z))) return kNone;
    const uint32_t u = ux + s.geo.X * uy + s.geo.XY * uz;
    return u - s.act_lo < s.act_n ? u : kNone;
  };
  const uint64_t i0 = (tid & ~uint64_t(31)) + (threadIdx.x & 31);
  uint32_t sv_c = load_sv(i0), sv_n = load_sv(i0 + stride);
  uint32_t u_c = locate(i0, sv_c);
  uint32_t cu_c = u_c != kNone ? __ldcg(s.gdir + u_c) : 0u;
  for (uint64_t wb = tid & ~uint64_t(31); wb < total; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    const uint32_t sv_nn = load_sv(i + 2 * stride);
    const uint32_t u_n = locate(i + stride, sv_n);
    const uint32_t cu_n = u_n != kNone ? __ldcg(s.gdir + u_n) : 0u;
    bool mine = false, keep = false;
    const uint32_t u = u_c == kNone ? 0u : u_c;
    if (u_c != kNone) {
      const uint32_t sv = sv_c, cu = cu_c;
      const uint32_t ca = cu & 15u, cd = cu >> 4;
      const uint32_t um = cd == kSelf ? u : u + s.geo.off[cd];
      bool fire = (ca == kSelf ? u : u + s.geo.off[ca]) == sv;
      if (!fire && um != sv) {
        const auto kt = okey(__ldcg(s.g + sv)), km = okey(__ldcg(s.g + um));
        fire = kt < km || (kt == km && sv < um);
      }
      if (fire && __ldcg(s.fmark + u) != mark && atomicExch(&s.fmark[u], mark) != mark) {
        mine = true;
        uint32_t ux, uy, uz;
        coords(s.geo, u, ux, uy, uz);
        const uint8_t code =
            static_cast<uint8_t>(direction_code<T, DIM, true>(s.g, s.geo, u, ux, uy, uz));
        if (next) keep = kind_match(kind, __ldg(s.fdir + u), code);
        // cu is u's pre-batch code: only the fmark winner writes gdir[u]
        if (cu != code) {
          s.gdir[u] = code;
          // the chunk's change mark: incremental subloop detection
          // (k_detect_dirty) and the sparse R pass's incremental X
          // (k_cross_chunks) both read it
          if (s.cstamp && s.cstamp[u >> 6] != mark) s.cstamp[u >> 6] = mark;
          if (s.tdirty) s.tdirty[label_tile_of<DIM>(s.geo, ux, uy, uz)] = 1;
        }
      }
    }
    if (next) {
      nbuf.push(keep, u, next, next_count);
      nmine += mine ? 1u : 0u;
    } else {
      warp_append(mine, u, s.F, f_count);
    }
    sv_c = sv_n;
    sv_n = sv_nn;
    u_c = u_n;
    cu_c = cu_n;
  }
  if (next) {
    nbuf.flush(next, next_count);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nmine += __shfl_xor_sync(0xffffffffu, nmine, o);
    if ((threadIdx.x & 31) == 0 && nmine) atomicAdd(f_count, nmine);
  }
}

// New worklist = (old list minus re-evaluated) ∪ {u re-evaluated : kind(u)}.
// The second part is appended by frontier_update; here the old entries that
// were not re-evaluated are kept.  Exact: a vertex whose code did not change
// keeps its class.
__device__ __forceinline__ void rebuild_retry(const uint32_t* __restrict__ retry, uint32_t nr,
                                              const uint32_t* __restrict__ fmark, uint32_t mark,
                                              uint32_t* nxt, uint32_t* nxt_count, uint64_t tid,
                                              uint64_t stride) {
  for (uint64_t wb = tid & ~uint64_t(31); wb < nr; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    bool keep = false;
    uint32_t v = 0;
    if (i < nr) {
      v = __ldcg(retry + i);
      const uint32_t fm = __ldcg(fmark + v);
      keep = fm != mark && fm != kParked;
    }
    warp_append(keep, v, nxt, nxt_count);
  }
}

// SWAR helpers on 4 packed direction codes: 0x80 in every byte whose
// nibble is all ones (SELF), exact per byte.
__device__ __forceinline__ uint32_t zero_bytes(uint32_t u) {
  const uint32_t y = (u & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
  return ~(y | u | 0x7F7F7F7Fu);
}
__device__ __forceinline__ uint32_t kind_bytes(int kind, uint32_t f, uint32_t g) {
  switch (kind) {
    case 0: return zero_bytes(~g & 0x0F0F0F0Fu) & ~zero_bytes(~f & 0x0F0F0F0Fu);   // FPmax
    case 1: return zero_bytes(~g & 0xF0F0F0F0u) & ~zero_bytes(~f & 0xF0F0F0F0u);   // FPmin
    case 2: return zero_bytes(~f & 0x0F0F0F0Fu) & ~zero_bytes(~g & 0x0F0F0F0Fu);   // FNmax
    default: return zero_bytes(~f & 0xF0F0F0F0u) & ~zero_bytes(~g & 0xF0F0F0F0u);  // FNmin
  }
}
__device__ __forceinline__ uint32_t bytes_to_nibble(uint32_t x) {  // 0x80 flags -> 4-bit mask
  return (((x >> 7) & 0x01010101u) * 0x01020408u) >> 24 & 0xFu;
}

// detect_kind over 16 vertices per thread, warp-compacted (edit_engine.cpp:104-132).
template <bool kCoherent>
__device__ __forceinline__ void detect_chunks(const uint8_t* __restrict__ fdir,
                                              const uint8_t* __restrict__ gdir, uint32_t n,
                                              int kind, uint32_t* __restrict__ list,
                                              uint32_t* count, uint64_t tid, uint64_t stride) {
  const uint64_t nchunks = (static_cast<uint64_t>(n) + 15) / 16;
  // block-uniform trip count (block_reserve)
  for (uint64_t bb = tid - threadIdx.x; bb < nchunks; bb += stride) {
    const uint64_t c = bb + threadIdx.x;
    uint32_t mask = 0;
    if (c < nchunks) {
      const uint64_t v0 = c * 16;
      if (v0 + 16 <= n) {
        const uint4 f = __ldg(reinterpret_cast<const uint4*>(fdir + v0));
        const uint4 g = ld<kCoherent>(reinterpret_cast<const uint4*>(gdir + v0));
        mask = bytes_to_nibble(kind_bytes(kind, f.x, g.x)) |
               bytes_to_nibble(kind_bytes(kind, f.y, g.y)) << 4 |
               bytes_to_nibble(kind_bytes(kind, f.z, g.z)) << 8 |
               bytes_to_nibble(kind_bytes(kind, f.w, g.w)) << 12;
      } else {
        for (int j = 0; j < 16; ++j)
          if (v0 + j < n && kind_match(kind, fdir[v0 + j], ld<kCoherent>(gdir + v0 + j)))
            mask |= 1u << j;
      }
    }
    if (!__syncthreads_or(mask != 0)) continue;
    uint32_t pos = block_reserve(__popc(mask), count);
    while (mask) {
      const int j = __ffs(mask) - 1;
      mask &= mask - 1;
      list[pos++] = static_cast<uint32_t>(c * 16 + j);
    }
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_fix_list(State<T> s, const uint32_t* __restrict__ list,
                                                  uint32_t n, int rule, uint32_t batch) {
  // standalone list fix (R batches, huge C batches): four items per lane in flight
  fix_batch<T, MSSZ_FIX_LIST_PER_LANE>(s, list, n, rule, batch, &s.ctl->s_count,
            static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
            static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

__global__ void __launch_bounds__(256) k_detect_kind(const uint8_t* __restrict__ fdir,
                                                     const uint8_t* __restrict__ gdir,
                                                     uint32_t n, int kind,
                                                     uint32_t* __restrict__ list,
                                                     uint32_t* count) {
  detect_chunks<false>(fdir, gdir, n, kind, list, count,
                       static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                       static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

// detect_kind restricted to the 64-vertex chunks whose codes changed since
// mark `since` (cstamp[c] >= since).  At the end of a subloop its kind's list
// is empty, and a vertex can only change class when its g-direction changes,
// so at the kind's next subloop these chunks hold every item.
// [lo, hi): vertex range kept (z-slab sharding: the active range of a window)
__global__ void __launch_bounds__(256) k_detect_dirty(const uint8_t* __restrict__ fdir,
                                                      const uint8_t* __restrict__ gdir, uint32_t n,
                                                      const uint32_t* __restrict__ cstamp, uint32_t since,
                                                      int kind, uint32_t* __restrict__ list,
                                                      uint32_t* count, uint32_t lo, uint32_t hi) {
  // warp-centric: a warp ballots the stamps of 4 x 32 consecutive chunks (all
  // loads in flight at once), then scans its dirty chunks 8 at a time, four
  // lanes x 16 vertices per chunk
  const uint32_t nch = (n + 63) / 64;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c0 = gw * 128; c0 < nch; c0 += nw * 128) {
    uint32_t st[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint64_t c = c0 + g * 32 + lane;
      st[g] = c < nch ? __ldg(cstamp + c) : 0u;
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint32_t bits = __ballot_sync(0xffffffffu, st[g] >= since && c0 + g * 32 + lane < nch);
      const int nd = __popc(bits);
      for (int b0 = 0; b0 < nd; b0 += 8) {
        const int k = b0 + (lane >> 2);
        uint32_t mask = 0;
        uint64_t v0 = 0;
        if (k < nd) {
          const uint64_t c = c0 + g * 32 + __fns(bits, 0, k + 1);
          v0 = c * 64 + (lane & 3) * 16;
          if (v0 >= lo && v0 + 16 <= hi) {
            const uint4 f = __ldg(reinterpret_cast<const uint4*>(fdir + v0));
            const uint4 gg = __ldg(reinterpret_cast<const uint4*>(gdir + v0));
            mask = bytes_to_nibble(kind_bytes(kind, f.x, gg.x)) | bytes_to_nibble(kind_bytes(kind, f.y, gg.y)) << 4 |
                   bytes_to_nibble(kind_bytes(kind, f.z, gg.z)) << 8 |
                   bytes_to_nibble(kind_bytes(kind, f.w, gg.w)) << 12;
          } else {
            for (int j = 0; j < 16; ++j)
              if (v0 + j >= lo && v0 + j < hi && kind_match(kind, fdir[v0 + j], gdir[v0 + j])) mask |= 1u << j;
          }
        }
        uint32_t pos = warp_reserve(__popc(mask), count);
        while (mask) {
          const int j = __ffs(mask) - 1;
          mask &= mask - 1;
          list[pos++] = static_cast<uint32_t>(v0 + j);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent subloop (run_subloop, edit_engine.cpp:246-278): detect → fix →
// refresh until the kind's list is empty, entirely on the device, in one
// cooperative launch per subloop invocation.
//
// CTA 0 is the leader.  Batches with at most small_max worklist items run in
// the leader CTA alone, separated by __syncthreads (most batches touch < 64
// vertices); the other CTAs sleep on a command word.  Larger
// batches are broadcast (ctl->cmd_*) and run grid-wide between grid barriers.
// Worklists above huge_min return to the host (kStatusHuge), which runs that
// batch with streaming kernels: at that size one full direction sweep + one
// detect sweep (6 B/vertex) beats ~15 random read-modify-writes per edit.
// batch ids: batch_base + 2*it (+1 for the FPmin fallback); mark ids: mark_base + it.
constexpr int kSubThreads = 512;
enum : uint32_t { kCmdBatch = 1, kCmdExit = 2, kCmdMerge = 3, kCmdFallback = 4 };
constexpr uint32_t kNeedMerge = 0xFFFFFFFFu;  // BatchResult::applied: merge parked items first

struct BatchResult {
  uint32_t applied;
  uint32_t nf;
};

// Parked items (k_subloop).  An item that won its claim while its target sat at
// the floor fails every later batch until its own code is re-evaluated: the
// target (asc_g(v) or v itself) is fixed while gdir[v] is, and g only falls, so
// lower_step keeps failing, and it blocks nobody (no claimant can lower a target
// at its floor).  Such items leave the worklist for the parked list P
// (fmark[v] = kParked) instead of being re-fixed every batch; a frontier
// re-evaluation overwrites fmark[v] and re-adds v to the worklist if it is
// still of the kind, which drops its P entry.  P is merged back whenever the
// reference's batch would see a different outcome without it: before the
// FPmin fallback (the fallback runs over the whole list), when the worklist
// runs empty, and on every exit from the kernel.  Batch outcomes, ids and
// counts are exactly the reference's.
//
// merge: (optionally) clear the parked flag of the first nclear worklist items
// (parked in the batch being redone), then append every P entry still parked
// (atomicCAS dedupes repeated entries) to list[cur].
template <class T, bool kGrid>
__device__ void merge_parked(const State<T>& s, cg::grid_group& grid, uint32_t cur, uint32_t nclear,
                             uint64_t tid, uint64_t stride) {
  auto sync = [&] {
    if (kGrid) grid.sync();
    else __syncthreads();
  };
  Ctl* ctl = s.ctl;
  const uint32_t* list = s.list[cur];
  for (uint64_t i = tid; i < nclear; i += stride) {
    const uint32_t v = __ldcg(list + i);
    if (__ldcg(s.fmark + v) == kParked) s.fmark[v] = 0u;
  }
  sync();
  const uint32_t np = *reinterpret_cast<volatile uint32_t*>(&ctl->park_count);
  for (uint64_t wb = tid & ~uint64_t(31); wb < np; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    bool keep = false;
    uint32_t v = 0;
    if (i < np) {
      v = __ldcg(s.F + i);
      keep = __ldcg(s.fmark + v) == kParked && atomicCAS(&s.fmark[v], kParked, 0u) == kParked;
    }
    warp_append(keep, v, s.list[cur], &ctl->list_count[cur]);
  }
  sync();
  if (tid == 0) {
    ctl->park_count = 0;
    ++ctl->merges;
  }
  sync();
}

// One batch: fix (rule pass, or the FPmin fallback alone when fallback_only),
// frontier refresh, rebuild.  Parking is on in the rule pass only.
template <class T, int DIM>
__device__ BatchResult big_batch(const State<T>& s, cg::grid_group& grid, int kind, uint32_t n,
                                 uint32_t cur, uint32_t it, uint32_t batch_base,
                                 uint32_t mark_base, bool fallback_only) {
  Ctl* ctl = s.ctl;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const int rule = (kind == 0 || kind == 3) ? 0 : 1;
  const uint32_t batch = batch_base + 2 * it, mark = mark_base + it;
  uint64_t t0 = 0, t1 = 0, t2 = 0;
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t applied = 0;
  if (!fallback_only) {
    fix_batch(s, s.list[cur], n, rule, batch, &ctl->s_count, tid, stride, nullptr, nullptr, s.F,
              &ctl->park_count);
    grid.sync();
    applied = *reinterpret_cast<volatile uint32_t*>(&ctl->s_count);
    if (applied == 0 && kind == 1 && *reinterpret_cast<volatile uint32_t*>(&ctl->park_count))
      return {kNeedMerge, 0};
  }
  if (applied == 0 && kind == 1) {
    grid.sync();  // every thread has read applied == 0 before the fallback appends to S
    fix_batch(s, s.list[cur], n, 2, batch + 1, &ctl->s_count, tid, stride);
    grid.sync();
    applied = *reinterpret_cast<volatile uint32_t*>(&ctl->s_count);
  }
  if (applied == 0) return {0, 0};
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  // frontier size only feeds EditStats: count it per CTA in shared memory
  __shared__ uint32_t block_frontier;
  if (threadIdx.x == 0) block_frontier = 0;
  __syncthreads();
  frontier_update<T, DIM>(s, applied, mark, &block_frontier, tid, stride, kind, s.list[cur ^ 1],
                          &ctl->list_count[cur ^ 1]);
  __syncthreads();
  if (threadIdx.x == 0 && block_frontier) atomicAdd(&ctl->f_count, block_frontier);
  grid.sync();
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
  const uint32_t nf = *reinterpret_cast<volatile uint32_t*>(&ctl->f_count);
  rebuild_retry(s.list[cur], n, s.fmark, mark, s.list[cur ^ 1], &ctl->list_count[cur ^ 1], tid, stride);
  grid.sync();
  if (tid == 0) {
    uint64_t t3;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
    ctl->phase_ns[0] += t1 - t0;
    ctl->phase_ns[1] += t2 - t1;
    ctl->phase_ns[2] += t3 - t2;
    ctl->s_count = 0;
    ctl->f_count = 0;
    ctl->list_count[cur] = 0;
  }
  return {applied, nf};
}

template <class T, int DIM>
__device__ BatchResult small_batch(const State<T>& s, int kind, uint32_t n, uint32_t cur,
                                   uint32_t it, uint32_t batch_base, uint32_t mark_base,
                                   bool fallback_only, uint32_t* cnt /* smem [4] */) {
  const uint64_t tid = threadIdx.x, stride = blockDim.x;
  const int rule = (kind == 0 || kind == 3) ? 0 : 1;
  const uint32_t batch = batch_base + 2 * it, mark = mark_base + it;
  uint32_t applied = 0;
  if (!fallback_only) {
    fix_batch(s, s.list[cur], n, rule, batch, &cnt[0], tid, stride, nullptr, nullptr, s.F,
              &s.ctl->park_count);
    __syncthreads();
    applied = *reinterpret_cast<volatile uint32_t*>(&cnt[0]);
    if (applied == 0 && kind == 1 && *reinterpret_cast<volatile uint32_t*>(&s.ctl->park_count)) {
      __syncthreads();
      return {kNeedMerge, 0};
    }
  }
  if (applied == 0 && kind == 1) {
    __syncthreads();
    fix_batch(s, s.list[cur], n, 2, batch + 1, &cnt[0], tid, stride);
    __syncthreads();
    applied = *reinterpret_cast<volatile uint32_t*>(&cnt[0]);
  }
  if (applied == 0) return {0, 0};
  frontier_update<T, DIM>(s, applied, mark, &cnt[1], tid, stride, kind, s.list[cur ^ 1], &cnt[2]);
  __syncthreads();
  const uint32_t nf = *reinterpret_cast<volatile uint32_t*>(&cnt[1]);
  rebuild_retry(s.list[cur], n, s.fmark, mark, s.list[cur ^ 1], &cnt[2], tid, stride);
  __syncthreads();
  if (threadIdx.x == 0) {
    s.ctl->list_count[cur ^ 1] = cnt[2];
    s.ctl->list_count[cur] = 0;
    cnt[0] = cnt[1] = cnt[2] = cnt[3] = 0;
  }
  __syncthreads();
  return {applied, nf};
}

template <class T, int DIM>
// 3 CTAs per SM (40 registers, a few spills): the kernel is bound by random
// DRAM lines, and 75% occupancy keeps more of them in flight than 50% (C4:
// 226.5 -> 208.1 ms per step); at 4 CTAs (32 registers) the spills dominate
// (279.7 ms).
__global__ void __launch_bounds__(kSubThreads, 3)
    k_subloop(State<T> s, int kind, uint64_t cap, uint32_t batch_base, uint32_t mark_base,
              uint32_t max_batches, uint32_t small_max, uint32_t huge_min, uint32_t park_cap) {
  cg::grid_group grid = cg::this_grid();
  Ctl* ctl = s.ctl;
  __shared__ uint32_t cmd[4];
  __shared__ uint32_t cnt[4];
  if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
  __syncthreads();

  if (blockIdx.x != 0) {  // worker CTAs: join broadcast batches and merges
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint32_t seen = 0;
    for (;;) {
      if (threadIdx.x == 0) {
        volatile uint32_t* seq = &ctl->cmd_seq;
        while (*seq == seen) __nanosleep(100);
        __threadfence();
        cmd[0] = *reinterpret_cast<volatile uint32_t*>(&ctl->cmd_type);
        cmd[1] = *reinterpret_cast<volatile uint32_t*>(&ctl->cmd_n);
        cmd[2] = *reinterpret_cast<volatile uint32_t*>(&ctl->cmd_cur);
        cmd[3] = *reinterpret_cast<volatile uint32_t*>(&ctl->cmd_it);
      }
      __syncthreads();
      ++seen;
      const uint32_t type = cmd[0], n = cmd[1], cur = cmd[2], it = cmd[3];
      __syncthreads();
      if (type == kCmdExit) break;
      if (type == kCmdMerge)
        merge_parked<T, true>(s, grid, cur, n, tid, stride);
      else
        big_batch<T, DIM>(s, grid, kind, n, cur, it, batch_base, mark_base, type == kCmdFallback);
    }
    grid.sync();
    return;
  }

  uint32_t cur = *reinterpret_cast<volatile uint32_t*>(&ctl->cur);
  uint64_t attempted = *reinterpret_cast<volatile uint64_t*>(&ctl->attempted);
  // run statistics live in shared memory, kept by thread 0: as registers they
  // stayed live across the inlined batch bodies and forced spills there
  enum { kIters, kEdits, kFrontier, kBig, kItems, kSmallNs, kBigNs, kT0, kAcc };
  __shared__ unsigned long long acc[kAcc];
  if (threadIdx.x < kAcc) acc[threadIdx.x] = 0;
  __syncthreads();
  uint32_t status = kStatusOk, done = 0, seq = 0;
  auto post = [&](uint32_t type, uint32_t n, uint32_t it) {
    if (threadIdx.x == 0) {
      ctl->cmd_type = type;
      ctl->cmd_n = n;
      ctl->cmd_cur = cur;
      ctl->cmd_it = it;
      __threadfence();
      atomicExch(&ctl->cmd_seq, ++seq);
    }
  };
  // merge P into list[cur]: grid-wide when large, else in this CTA
  auto merge = [&](uint32_t nclear) {
    const uint32_t np = *reinterpret_cast<volatile uint32_t*>(&ctl->park_count);
    if (np + nclear > small_max) {
      post(kCmdMerge, nclear, 0);
      merge_parked<T, true>(s, grid, cur, nclear, threadIdx.x, static_cast<uint64_t>(gridDim.x) * blockDim.x);
    } else {
      merge_parked<T, false>(s, grid, cur, nclear, threadIdx.x, blockDim.x);
    }
  };
  for (;;) {
    uint32_t n = *reinterpret_cast<volatile uint32_t*>(&ctl->list_count[cur]);
    const uint32_t np = *reinterpret_cast<volatile uint32_t*>(&ctl->park_count);
    if (np && (n == 0 || n > huge_min || done >= max_batches || np + n > park_cap)) {
      merge(0);
      n = *reinterpret_cast<volatile uint32_t*>(&ctl->list_count[cur]);
    }
    if (n == 0 || done >= max_batches) break;
    if (n > huge_min) {
      status = kStatusHuge;
      break;
    }
    ++attempted;
    if (attempted > cap) {
      status = kStatusCap;
      break;
    }
    const uint32_t it = static_cast<uint32_t>(attempted);
    BatchResult r;
    if (threadIdx.x == 0) {
      uint64_t t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      acc[kT0] = t0;
    }
    bool fallback_only = false;
    for (;;) {  // at most twice: the rule pass, then (kNeedMerge) the fallback over list ∪ P
      if (n <= small_max) {
        r = small_batch<T, DIM>(s, kind, n, cur, it, batch_base, mark_base, fallback_only, cnt);
      } else {
        post(fallback_only ? kCmdFallback : kCmdBatch, n, it);
        r = big_batch<T, DIM>(s, grid, kind, n, cur, it, batch_base, mark_base, fallback_only);
        if (threadIdx.x == 0) ++acc[kBig];
        __syncthreads();
      }
      if (r.applied != kNeedMerge) break;
      merge(n);
      n = *reinterpret_cast<volatile uint32_t*>(&ctl->list_count[cur]);
      fallback_only = true;
    }
    if (threadIdx.x == 0) {
      uint64_t t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      acc[n <= small_max ? kSmallNs : kBigNs] += t1 - acc[kT0];
    }
    if (r.applied == 0) {
      status = kStatusStall;
      break;
    }
    if (threadIdx.x == 0) {
      ++acc[kIters];
      acc[kEdits] += r.applied;
      acc[kFrontier] += r.nf;
      acc[kItems] += n;
    }
    cur ^= 1;
    ++done;
  }
  // every exit leaves the complete worklist in list[cur] (huge batches, errors, on_batch)
  if (*reinterpret_cast<volatile uint32_t*>(&ctl->park_count)) merge(0);
  post(kCmdExit, 0, 0);
  grid.sync();
  if (threadIdx.x == 0) {
    ctl->cur = cur;
    ctl->attempted = attempted;
    ctl->iters += acc[kIters];
    ctl->edits += acc[kEdits];
    ctl->frontier += acc[kFrontier];
    ctl->big_batches += acc[kBig];
    ctl->items += acc[kItems];
    ctl->small_ns += acc[kSmallNs];
    ctl->big_ns += acc[kBigNs];
    ctl->status = status;
  }
}

// ---------------------------------------------------------------------------
// K3 (generic): u32 pointer jumping for arbitrary parent arrays (the exported
// compute_labels API, mss.cpp:51-97).  Asynchronous in-place doubling reaches
// the same unique fixpoint (the chain terminus) in no more rounds than the
// reference's round-synchronous version, so its round cap still applies.
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

// ---------------------------------------------------------------------------
// K3 (tiled): labels in three passes instead of ~log2(path) full-N rounds.
//  1. k_label_tile: one CTA per 8192-vertex tile resolves every chain inside
//     the tile by pointer jumping in shared memory.  A vertex's provisional
//     label is its chain's root (final) or the first vertex OUTSIDE the tile
//     (an "exit").  Each distinct exit is appended once to E (fmark dedupe).
//  2. k_label_exit_jump: pointer jumping over E only; an exit's provisional
//     label is itself a root or another exit, so E closes under lab[].
//  3. k_label_finish: one gather per vertex, lab[v] = lab[lab[v]].
// The fixpoint is the chain terminus, identical to the reference's
// round-synchronous doubling (mss.cpp:60-80).
constexpr int kLabelTileN = 8192;
constexpr int kLabelTileThreads = 512;
template <int DIM>
constexpr size_t label_tile_smem() {
  return kLabelTileN * 4 + kLabelTileN;  // 40 KB: four 512-thread CTAs per SM
}

// Per-tile label state kept across R-loop iterations (incremental labels).
struct TileStore {
  uint32_t* E;        // [ntiles][2][kSurface] distinct exits of the tile per family
  uint32_t* Ecnt;     // [ntiles][2]
  uint32_t* oldfin;   // [ntiles][2][kSurface] exit finals of the previous pass
  uint8_t* dirty;     // [ntiles] a direction code in the tile changed
  uint8_t* affected;  // [ntiles] an exit of the tile changed its final label
  uint32_t* mis_bits; // [ntiles][2][kLabelTileN / 32] divergent-and-mismatched bits
  uint32_t* mis_cnt;  // [ntiles]
  uint32_t ntiles;
  uint32_t surface;   // LabelTile<DIM>::kSurface
  // vertices outside [own_lo, own_hi) are labelled as extrema (z-slab windows:
  // chains stop at their first off-slab vertex); single device: the whole grid
  uint32_t own_lo, own_hi;
  uint32_t* err;  // set when in-tile doubling exceeds its round cap (a cycle)
};

// Phase 1.  Writes the provisional label (root, or first vertex outside the
// tile) to prov, fin[r] = r at roots, and the tile's distinct exits to the
// tile store.
// tile_list == nullptr: CTA i handles tile i.
template <int DIM>
__global__ void __launch_bounds__(kLabelTileThreads) k_label_tile(
    const uint8_t* __restrict__ dir, Geom g, uint32_t* __restrict__ M, uint32_t* __restrict__ m,
    uint32_t* __restrict__ finM, uint32_t* __restrict__ finm, const uint32_t* tile_list,
    TileStore ts, const __grid_constant__ CUtensorMap dmap, int use_tma, int seed_exits) {
  using TL = LabelTile<DIM>;
  constexpr int NS = StencilSize<DIM>::value;
  constexpr int PER = kLabelTileN / kLabelTileThreads;
  // dynamic shared memory (label_tile_smem<DIM>() bytes):
  //   ptr   u32[kLabelTileN]  (asc local parent) | (desc local parent) << 16
  //   sdir  u8[kLabelTileN]
  // (the tile's distinct exits go straight to its tile-store slots, ts.E)
  extern __shared__ __align__(128) uint8_t label_smem[];  // sdir at a 128-byte multiple: a TMA destination
  uint32_t* ptr = reinterpret_cast<uint32_t*>(label_smem);
  uint8_t* sdir = reinterpret_cast<uint8_t*>(ptr + kLabelTileN);
  __shared__ uint32_t sexit_n[2];
  // per-family bitmap over the tile's halo box: each distinct exit is listed once per tile
  constexpr int HBOX = (TL::TX + 2) * (TL::TY + 2) * (DIM == 2 ? 1 : TL::TZ + 2);
  __shared__ uint32_t seen[2][(HBOX + 31) / 32];
  for (int w = threadIdx.x; w < 2 * ((HBOX + 31) / 32); w += kLabelTileThreads)
    (&seen[0][0])[w] = 0u;
  if (threadIdx.x < 2) sexit_n[threadIdx.x] = 0;
  // per slot: global offset, faces of the tile it crosses
  // (bit 0 -x, 1 +x, 2 -y, 3 +y, 4 -z, 5 +z); SELF = slot 15: offset 0, no face
  __shared__ int32_t soff[16];
  __shared__ uint32_t sface[16];
  __shared__ int32_t shalo[16];  // offset in the tile's halo box (exit dedupe bitmap)
  if (threadIdx.x < 16) {
    int dx = 0, dy = 0, dz = 0;
#pragma unroll
    for (int k = 0; k < NS; ++k)
      if (k == static_cast<int>(threadIdx.x)) stencil<DIM>(k, dx, dy, dz);
    // = g.off[k] (mod 2^32), without a dynamically indexed kernel parameter
    soff[threadIdx.x] = static_cast<int32_t>(static_cast<uint32_t>(dx) + static_cast<uint32_t>(dy) * g.X +
                                             static_cast<uint32_t>(dz) * g.XY);
    sface[threadIdx.x] = (dx < 0 ? 1u : 0u) | (dx > 0 ? 2u : 0u) | (dy < 0 ? 4u : 0u) | (dy > 0 ? 8u : 0u) |
                         (dz < 0 ? 16u : 0u) | (dz > 0 ? 32u : 0u);
    shalo[threadIdx.x] = dx + (TL::TX + 2) * (dy + (TL::TY + 2) * dz);
  }
  // per direction byte (asc | desc << 4): both local parent offsets (int16 each)
  // and both face masks, so a local parent costs one shared load
  __shared__ uint2 scode[256];
  if (threadIdx.x < 256) {
    const int ca = threadIdx.x & 15, cd = threadIdx.x >> 4;
    int ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      if (k == ca) stencil<DIM>(k, ax, ay, az);
      if (k == cd) stencil<DIM>(k, bx, by, bz);
    }
    const int la = ax + (ay << TL::LX) + (az << (TL::LX + TL::LY));
    const int lb = bx + (by << TL::LX) + (bz << (TL::LX + TL::LY));
    auto faces = [](int x, int y, int z) {
      return (x < 0 ? 1u : 0u) | (x > 0 ? 2u : 0u) | (y < 0 ? 4u : 0u) | (y > 0 ? 8u : 0u) |
             (z < 0 ? 16u : 0u) | (z > 0 ? 32u : 0u);
    };
    scode[threadIdx.x] = make_uint2((static_cast<uint32_t>(la) & 0xFFFFu) | (static_cast<uint32_t>(lb) << 16),
                                    faces(ax, ay, az) | (faces(bx, by, bz) << 8));
  }
  const uint32_t ntx = (g.X + TL::TX - 1) / TL::TX;
  const uint32_t nty = (g.Y + TL::TY - 1) / TL::TY;
  const uint32_t b = tile_list ? tile_list[blockIdx.x] : blockIdx.x;
  const uint32_t tx = b % ntx, ty = (b / ntx) % nty, tz = b / (ntx * nty);
  const uint32_t x0 = tx * TL::TX, y0 = ty * TL::TY, z0 = tz * TL::TZ;
  const int ex = min(TL::TX, static_cast<int>(g.X - x0));
  const int ey = min(TL::TY, static_cast<int>(g.Y - y0));
  const int ez = DIM == 2 ? 1 : min(TL::TZ, static_cast<int>(g.Z - z0));
  const uint32_t base = x0 + g.X * y0 + g.XY * z0;
  const bool full = ex == TL::TX && ey == TL::TY && ez == TL::TZ;
  // dir tile of a whole 3D tile inside the owned range: one TMA box load
  // (cp.async.bulk.tensor.3d, 32x16x16 bytes in the tile's own element order)
  // completing on an mbarrier; otherwise 16-byte vector loads when rows are
  // 16-byte aligned and whole, else byte loads with out-of-range fill
  const bool tma = DIM == 3 && use_tma && full && base >= ts.own_lo &&
                   base + (TL::TX - 1) + g.X * (TL::TY - 1) + g.XY * (TL::TZ - 1) < ts.own_hi;
  if (tma) {
    __shared__ __align__(8) uint64_t tbar;
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&tbar));
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kLabelTileN)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              static_cast<uint32_t>(__cvta_generic_to_shared(sdir))),
          "l"(reinterpret_cast<uint64_t>(&dmap)), "r"(x0), "r"(y0), "r"(z0), "r"(bar)
          : "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    uint32_t done = 0;
    for (uint32_t it = 0; !done; ++it) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(bar)
          : "memory");
      if (it > (1u << 22)) __trap();  // a lost transfer fails the launch instead of hanging it
    }
  } else if (full && (g.X % 16) == 0) {
    constexpr int VPR = TL::TX / 16;  // uint4 per row
    for (int q = threadIdx.x; q < kLabelTileN / 16; q += kLabelTileThreads) {
      const int row = q / VPR, c = q % VPR;
      const int ly = row & (TL::TY - 1), lz = row / TL::TY;
      const uint32_t gv = base + g.X * ly + g.XY * lz + 16 * c;  // own bounds are plane (16 B) aligned here
      const uint4 w = (gv >= ts.own_lo && gv < ts.own_hi)
                          ? __ldg(reinterpret_cast<const uint4*>(dir + base + g.X * ly + g.XY * lz) + c)
                          : make_uint4(~0u, ~0u, ~0u, ~0u);
      reinterpret_cast<uint4*>(sdir)[q] = w;
    }
  } else {
#pragma unroll 4
    for (int i = threadIdx.x; i < kLabelTileN; i += kLabelTileThreads) {
      const int lx = i & (TL::TX - 1), ly = (i >> TL::LX) & (TL::TY - 1), lz = i >> (TL::LX + TL::LY);
      const uint32_t gv = base + lx + g.X * ly + g.XY * lz;
      const bool val = lx < ex && ly < ey && lz < ez && gv >= ts.own_lo && gv < ts.own_hi;
      sdir[i] = val ? __ldg(dir + gv) : 0xFF;
    }
  }
  __syncthreads();
  // local parents; a chain that leaves the tile stops at its last inside vertex.
  // Element i = tid + j*kLabelTileThreads: its column is a per-thread constant
  // (and in 3D its row too), so most of the face mask is computed once.
  uint32_t own[PER];
  const int lx0 = threadIdx.x & (TL::TX - 1);
  const uint32_t onx = (lx0 == 0 ? 1u : 0u) | (lx0 == ex - 1 ? 2u : 0u);
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * kLabelTileThreads;
    const int ly = (i >> TL::LX) & (TL::TY - 1), lz = i >> (TL::LX + TL::LY);
    const uint32_t code = sdir[i];
    // faces of the (partial) tile this element lies on; outside elements stay put
    const uint32_t ony = (ly == 0 ? 4u : 0u) | (ly == ey - 1 ? 8u : 0u);
    const uint32_t onz = (lz == 0 ? 16u : 0u) | (lz == ez - 1 ? 32u : 0u);
    const bool inside = lx0 < ex && ly < ey && lz < ez;
    const uint32_t on = inside ? (onx | ony | onz) : 63u;
    const uint2 e = scode[code];  // SELF: offset 0, no face
    const uint32_t pa = (e.y & on) ? i : i + static_cast<int32_t>(static_cast<int16_t>(e.x & 0xFFFFu));
    const uint32_t pd = ((e.y >> 8) & on) ? i : i + (static_cast<int32_t>(e.x) >> 16);
    own[j] = 4 * pa | ((4 * pd) << 16);  // byte offsets of the parents' words (< 2^15)
    ptr[i] = own[j];
  }
  __syncthreads();
  // in-place doubling on both families at once; a thread's own pointers live
  // in registers (only this thread writes them), the others are read from smem.
  // Chains inside a tile are shorter than kLabelTileN, so an acyclic field
  // settles within bit_width(kLabelTileN) + 1 rounds; a cyclic (corrupt)
  // direction field would never settle: capped, flagged, raised by the host
  // like the reference's round cap (mss.cpp:60-80).
  for (int round = 0;; ++round) {
    if (round > 2 * 14 + 4) {
      if (threadIdx.x == 0 && ts.err) atomicExch(ts.err, 1u);
      break;
    }
    bool changed = false;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * kLabelTileThreads;
      const uint32_t p = own[j];
      // the asc half of the word at byte offset p & 0xFFFF, the desc half of the one at p >> 16
      const uint32_t np = *reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(ptr) + (p & 0xFFFFu)) |
                          (static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(
                               reinterpret_cast<const uint8_t*>(ptr) + (p >> 16) + 2)) << 16);
      if (np != p) {
        own[j] = np;
        ptr[i] = np;
        changed = true;
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
  // provisional labels (root, or first vertex outside the tile) + the exits:
  // the chain's last inside vertex t is a root (code SELF) or steps out by
  // slot c, so the label is gid(t) + soff[c] (soff[SELF] = 0)
  // element j of this thread: gid = gi0 + j * jstride (its column, and in 3D
  // its row, are per-thread constants; a j step is RPJ rows)
  constexpr int RPJ = kLabelTileThreads / TL::TX;
  const uint32_t gi0 = base + lx0 + g.X * ((threadIdx.x >> TL::LX) & (TL::TY - 1)) +
                       g.XY * (threadIdx.x >> (TL::LX + TL::LY));
  const uint32_t jstride = DIM == 3 ? g.XY * (RPJ / TL::TY) : g.X * RPJ;
  // fin is only ever read at provisional-label values: roots and exits.  Roots
  // are written here.  Every exit is a surface element of the tile it lies in
  // (a chain leaves a tile by one stencil step), so with seed_exits (a pass
  // over every tile) surface elements also write fin = their provisional label
  // -- what k_exit_reset would copy there -- and that launch is skipped.
  auto label_one = [&](uint32_t p, uint32_t gi, bool surf) {
#pragma unroll
    for (int fam = 0; fam < 2; ++fam) {
      const int t = (fam ? (p >> 16) : (p & 0xFFFFu)) >> 2;
      const uint32_t c = (sdir[t] >> (4 * fam)) & 15u;
      const uint32_t res = base + (t & (TL::TX - 1)) + g.X * ((t >> TL::LX) & (TL::TY - 1)) +
                           g.XY * (t >> (TL::LX + TL::LY)) + soff[c];
      (fam ? m : M)[gi] = res;
      if (res == gi || surf) (fam ? finm : finM)[gi] = res;
    }
  };
  const bool sx = seed_exits && onx != 0;
  auto surface = [&](int ly, int lz) {
    return seed_exits && (sx || ly == 0 || ly == ey - 1 || lz == 0 || lz == ez - 1);
  };
  if (full) {
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * kLabelTileThreads;
      const int ly = (i >> TL::LX) & (TL::TY - 1), lz = i >> (TL::LX + TL::LY);
      label_one(own[j], gi0 + j * jstride, surface(ly, lz));
    }
  } else {
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * kLabelTileThreads;
      const int ly = (i >> TL::LX) & (TL::TY - 1), lz = i >> (TL::LX + TL::LY);
      if (lx0 < ex && ly < ey && lz < ez) label_one(own[j], gi0 + j * jstride, surface(ly, lz));
    }
  }
  // the tile's distinct exits: only surface elements can step out, so walk the
  // six faces (edges/corners repeat; the halo bitmap dedupes) with full warps
  {
    constexpr int NFX = TL::TY * TL::TZ, NFY = TL::TX * TL::TZ, NFZ = DIM == 2 ? 0 : TL::TX * TL::TY;
    constexpr int NF = 2 * (NFX + NFY + NFZ);
    for (int k = threadIdx.x; k < NF; k += kLabelTileThreads) {
      int lx, ly, lz, q = k;
      if (q < 2 * NFX) {
        lx = q < NFX ? 0 : ex - 1;
        q %= NFX;
        ly = q % TL::TY;
        lz = q / TL::TY;
      } else if ((q -= 2 * NFX) < 2 * NFY) {
        ly = q < NFY ? 0 : ey - 1;
        q %= NFY;
        lx = q % TL::TX;
        lz = q / TL::TX;
      } else {
        q -= 2 * NFY;
        lz = q < NFZ ? 0 : ez - 1;
        q %= NFZ;
        lx = q % TL::TX;
        ly = q / TL::TX;
      }
      if (lx >= ex || ly >= ey || lz >= ez) continue;
      const int i = lx + (ly << TL::LX) + (lz << (TL::LX + TL::LY));
      const uint32_t code = sdir[i];
      const uint32_t on = (lx == 0 ? 1u : 0u) | (lx == ex - 1 ? 2u : 0u) | (ly == 0 ? 4u : 0u) |
                          (ly == ey - 1 ? 8u : 0u) | (lz == 0 ? 16u : 0u) | (lz == ez - 1 ? 32u : 0u);
      const uint32_t gi = base + lx + g.X * ly + g.XY * lz;
      const int hb = (lx + 1) + (TL::TX + 2) * ((ly + 1) + (TL::TY + 2) * (DIM == 2 ? 0 : lz + 1));
#pragma unroll
      for (int fam = 0; fam < 2; ++fam) {
        const uint32_t c = (code >> (4 * fam)) & 15u;
        if (!(sface[c] & on)) continue;  // SELF or a step inside the tile
        const int h = hb + shalo[c];
        if (!(atomicOr(&seen[fam][h >> 5], 1u << (h & 31)) & (1u << (h & 31))))
          ts.E[(static_cast<size_t>(b) * 2 + fam) * LabelTile<DIM>::kSurface + atomicAdd(&sexit_n[fam], 1u)] =
              gi + soff[c];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 2) ts.Ecnt[b * 2 + threadIdx.x] = sexit_n[threadIdx.x];
}

// Phase 2a (all tiles): remember every exit's final label (k_exit_save), then
// restart it from the provisional one (k_exit_reset).  Two launches, so an exit
// listed by several tiles is saved before any tile resets it.  CTA per tile.
__global__ void __launch_bounds__(256) k_exit_save(TileStore ts, const uint32_t* __restrict__ finM,
                                                   const uint32_t* __restrict__ finm) {
  const uint32_t b = blockIdx.x;
#pragma unroll
  for (int fam = 0; fam < 2; ++fam) {
    const uint32_t n = ts.Ecnt[b * 2 + fam];
    const size_t o = (static_cast<size_t>(b) * 2 + fam) * ts.surface;
    const uint32_t* fin = fam ? finm : finM;
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) ts.oldfin[o + k] = fin[ts.E[o + k]];
  }
}

__global__ void __launch_bounds__(256) k_exit_reset(TileStore ts, const uint32_t* __restrict__ M,
                                                    const uint32_t* __restrict__ m,
                                                    uint32_t* __restrict__ finM,
                                                    uint32_t* __restrict__ finm) {
  const uint32_t b = blockIdx.x;
#pragma unroll
  for (int fam = 0; fam < 2; ++fam) {
    const uint32_t n = ts.Ecnt[b * 2 + fam];
    const size_t o = (static_cast<size_t>(b) * 2 + fam) * ts.surface;
    uint32_t* fin = fam ? finm : finM;
    const uint32_t* prov = fam ? m : M;
    // eight exits per thread per step: their loads and gathers overlap
    for (uint32_t k0 = threadIdx.x; k0 < n; k0 += 8 * blockDim.x) {
      uint32_t e[8], p[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t k = k0 + q * blockDim.x;
        e[q] = k < n ? ts.E[o + k] : kNoTarget;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) p[q] = e[q] != kNoTarget ? __ldg(prov + e[q]) : 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (e[q] != kNoTarget) fin[e[q]] = p[q];
    }
  }
}

// Phase 2b: first doubling round straight from the tile stores; unresolved
// exits go to the compact lists that k_label_exit_jump keeps halving.
__global__ void __launch_bounds__(256) k_exit_jump_tiles(TileStore ts, uint32_t* __restrict__ finM,
                                                         uint32_t* __restrict__ finm,
                                                         uint32_t* __restrict__ out_a,
                                                         uint32_t* __restrict__ out_d,
                                                         uint32_t* cnt_out) {
  const uint32_t b = blockIdx.x;
  for (int fam = 0; fam < 2; ++fam) {
    const uint32_t n = ts.Ecnt[b * 2 + fam];
    const size_t o = (static_cast<size_t>(b) * 2 + fam) * ts.surface;
    uint32_t* fin = fam ? finm : finM;
    // block-uniform trip count (block_reserve); four exits per thread per step
    // so the 3-deep gather chains overlap
    for (uint32_t kb = 0; kb < n; kb += 4 * blockDim.x) {
      uint32_t e[4], l[4], ll[4];
      bool live[4], keep[4] = {false, false, false, false};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t k = kb + threadIdx.x + q * blockDim.x;
        live[q] = k < n;
        e[q] = live[q] ? ts.E[o + k] : 0u;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) l[q] = live[q] ? fin[e[q]] : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) ll[q] = live[q] ? fin[l[q]] : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (live[q] && ll[q] != l[q]) {
          fin[e[q]] = ll[q];
          keep[q] = fin[ll[q]] != ll[q];
        }
      uint32_t nk = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) nk += keep[q] ? 1u : 0u;
      uint32_t pos = block_reserve(nk, cnt_out + fam);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (keep[q]) (fam ? out_d : out_a)[pos++] = e[q];
    }
  }
}

// Phase 2c: tiles whose exits changed their final label are "affected".
__global__ void __launch_bounds__(256) k_exit_changed(TileStore ts, const uint32_t* __restrict__ finM,
                                                      const uint32_t* __restrict__ finm) {
  const uint32_t b = blockIdx.x;
  bool changed = false;
  for (int fam = 0; fam < 2; ++fam) {
    const uint32_t n = ts.Ecnt[b * 2 + fam];
    const size_t o = (static_cast<size_t>(b) * 2 + fam) * ts.surface;
    const uint32_t* fin = fam ? finm : finM;
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x)
      changed |= fin[ts.E[o + k]] != ts.oldfin[o + k];
  }
  if (__syncthreads_or(changed) && threadIdx.x == 0) ts.affected[b] = 1;
}

// Tile selection: mode 0 dirty, 1 dirty|affected, 2 mis_cnt > 0.
__global__ void __launch_bounds__(256) k_select_tiles(TileStore ts, int mode, uint32_t* out,
                                                      uint32_t* count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t wb = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~uint64_t(31);
       wb < ts.ntiles; wb += stride) {
    const uint64_t t = wb + (threadIdx.x & 31);
    bool sel = false;
    if (t < ts.ntiles) {
      if (mode == 0) sel = ts.dirty[t];
      else if (mode == 1) sel = ts.dirty[t] || ts.affected[t];
      else sel = ts.mis_cnt[t] != 0;
    }
    warp_append(sel, static_cast<uint32_t>(t), out, count);
  }
}

// One doubling round over the unresolved exits: in[] -> out[] keeps only
// entries whose label is not yet a root (lab[lab[e]] != lab[e]).  cnt[0..1]
// are the (asc, desc) input sizes, cnt[2..3] the output sizes.  Exits may
// repeat (no dedupe); concurrent updates of one entry are benign because any
// value written is an ancestor on the same chain.
__global__ void __launch_bounds__(256) k_label_exit_jump(uint32_t* __restrict__ M,
                                                         uint32_t* __restrict__ m,
                                                         const uint32_t* __restrict__ in_a,
                                                         const uint32_t* __restrict__ in_d,
                                                         uint32_t* __restrict__ out_a,
                                                         uint32_t* __restrict__ out_d,
                                                         const uint32_t* cnt_in, uint32_t* cnt_out) {
  const uint32_t na = cnt_in[0], nd = cnt_in[1];
  const uint64_t total = static_cast<uint64_t>(na) + nd;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t wb = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~uint64_t(31);
       wb < total; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    bool keep_a = false, keep_d = false;
    uint32_t e = 0;
    if (i < total) {
      const bool asc = i < na;
      uint32_t* lab = asc ? M : m;
      e = asc ? in_a[i] : in_d[i - na];
      const uint32_t l = lab[e];
      const uint32_t ll = lab[l];
      if (ll != l) {
        lab[e] = ll;
        const uint32_t lll = lab[ll];
        if (lll != ll) (asc ? keep_a : keep_d) = true;
      }
    }
    warp_append(keep_a, e, out_a, cnt_out);
    warp_append(keep_d, e, out_d, cnt_out + 1);
  }
}

// Phase 3 (f labels only): final label of every vertex, lab[v] = fin[lab[v]].
// Phase 3, tile-ordered: one CTA per label tile, so the fin[] gathers of its
// vertices (their chain roots inside the tile, or exits next to it) stay in
// the tile's neighbourhood while it is resident in L2, instead of spreading
// over the 16 planes a tile spans when the field is walked in index order.
template <int DIM>
__global__ void __launch_bounds__(256) k_label_finish_tiles(uint32_t* __restrict__ M, uint32_t* __restrict__ m,
                                                            const uint32_t* __restrict__ finM,
                                                            const uint32_t* __restrict__ finm, Geom g) {
  using TL = LabelTile<DIM>;
  const uint32_t ntx = (g.X + TL::TX - 1) / TL::TX;
  const uint32_t nty = (g.Y + TL::TY - 1) / TL::TY;
  const uint32_t b = blockIdx.x;
  const uint32_t tx = b % ntx, ty = (b / ntx) % nty, tz = b / (ntx * nty);
  const uint32_t x0 = tx * TL::TX, y0 = ty * TL::TY, z0 = tz * TL::TZ;
  const int ex = min(TL::TX, static_cast<int>(g.X - x0));
  const int ey = min(TL::TY, static_cast<int>(g.Y - y0));
  const int ez = DIM == 2 ? 1 : min(TL::TZ, static_cast<int>(g.Z - z0));
  const uint32_t base = x0 + g.X * y0 + g.XY * z0;
  // four vertices per thread per step: their gathers overlap
  for (int i0 = threadIdx.x; i0 < kLabelTileN; i0 += 4 * blockDim.x) {
    uint32_t v[4], a[4], d[4];
    bool in[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q * blockDim.x;
      const int lx = i & (TL::TX - 1), ly = (i >> TL::LX) & (TL::TY - 1), lz = i >> (TL::LX + TL::LY);
      in[q] = lx < ex && ly < ey && lz < ez;
      v[q] = base + lx + g.X * ly + g.XY * lz;
      a[q] = in[q] ? M[v[q]] : 0u;
      d[q] = in[q] ? m[v[q]] : 0u;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!in[q]) continue;
      a[q] = __ldg(finM + a[q]);
      d[q] = __ldg(finm + d[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (in[q]) {
        M[v[q]] = a[q];
        m[v[q]] = d[q];
      }
  }
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
// stamps, then lower_step over the deduplicated targets).  k_rfix only lists
// the targets (a streaming pass with no atomics on its critical path);
// k_fix_list then claims and lowers them.
//
// The g labels arrive provisional (k_label_tile + exit jumping, no finish
// pass): lab[v] is a root or a resolved exit, so lab[lab[v]] is final.  Only
// divergent vertices need their label, so the full-N finish pass is skipped.
// ctl->mism counts divergent mismatched vertices: it is zero exactly when no
// vertex is mismatched (the walk argument above), which is the reference's
// collect_mismatched() == 0 test.
// Tile pass: for every vertex of the listed tiles, is it divergent AND
// mismatched (per family)?  One warp = 32 consecutive tile-local vertices =
// one bitmap word (ballot).  Final g labels are fin[prov[v]] (prov = gM/gm).
// Tiles not listed keep last iteration's bitmap: neither their directions
// (not dirty) nor the finals of the exits their chains leave through (not
// affected) changed, so their mismatch set is unchanged.
template <class T, int DIM>
__global__ void __launch_bounds__(256) k_rfix_tiles(State<T> s, const uint32_t* __restrict__ tiles,
                                                    TileStore ts, const uint32_t* __restrict__ finM,
                                                    const uint32_t* __restrict__ finm, SlabRes sr) {
  using TL = LabelTile<DIM>;
  const Geom& g = s.geo;
  const uint32_t ntx = (g.X + TL::TX - 1) / TL::TX;
  const uint32_t nty = (g.Y + TL::TY - 1) / TL::TY;
  const uint32_t b = tiles ? tiles[blockIdx.x] : blockIdx.x;
  const uint32_t tx = b % ntx, ty = (b / ntx) % nty, tz = b / (ntx * nty);
  const uint32_t x0 = tx * TL::TX, y0 = ty * TL::TY, z0 = tz * TL::TZ;
  const int ex = min(TL::TX, static_cast<int>(g.X - x0));
  const int ey = min(TL::TY, static_cast<int>(g.Y - y0));
  const int ez = DIM == 2 ? 1 : min(TL::TZ, static_cast<int>(g.Z - z0));
  const uint32_t base = x0 + g.X * y0 + g.XY * z0;
  uint32_t* bits = ts.mis_bits + static_cast<size_t>(b) * 2 * (kLabelTileN / 32);
  uint32_t cnt = 0, ndiv = 0;
  for (int i = threadIdx.x; i < kLabelTileN; i += blockDim.x) {
    const int lx = i & (TL::TX - 1), ly = (i >> TL::LX) & (TL::TY - 1), lz = i >> (TL::LX + TL::LY);
    bool ma = false, md = false;
    const uint32_t v = base + lx + g.X * ly + g.XY * lz;
    if (lx < ex && ly < ey && lz < ez && v - s.act_lo < s.act_n) {
      const uint32_t fc = __ldg(s.fdir + v), gc = __ldg(s.gdir + v);
      const bool wa = (gc & 15u) != (fc & 15u);  // ascending line diverges at v
      const bool wd = (gc >> 4) != (fc >> 4);    // descending line diverges at v
      uint32_t la = 0, ld = 0;
      uint64_t fa = 0, fd = 0;
      if (wa) {
        la = __ldg(s.gM + v);
        fa = s.fM64 ? __ldg(s.fM64 + v) : __ldg(s.fM + v);
      }
      if (wd) {
        ld = __ldg(s.gm + v);
        fd = s.fm64 ? __ldg(s.fm64 + v) : __ldg(s.fm + v);
      }
      ma = wa && resolve_label(sr, __ldg(finM + la), 0) != fa;
      md = wd && resolve_label(sr, __ldg(finm + ld), 1) != fd;
      ndiv += (wa ? 1u : 0u) + (wd ? 1u : 0u);
    }
    const uint32_t wa_bits = __ballot_sync(0xffffffffu, ma);
    const uint32_t wd_bits = __ballot_sync(0xffffffffu, md);
    if ((threadIdx.x & 31) == 0) {
      bits[i >> 5] = wa_bits;
      bits[kLabelTileN / 32 + (i >> 5)] = wd_bits;
      cnt += __popc(wa_bits) + __popc(wd_bits);
    }
  }
  __shared__ uint32_t scnt, sdiv;
  if (threadIdx.x == 0) scnt = sdiv = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&scnt, cnt);
  if (ndiv) atomicAdd(&sdiv, ndiv);
  __syncthreads();
  if (threadIdx.x == 0) {
    ts.mis_cnt[b] = scnt;
    if (sdiv) atomicAdd(reinterpret_cast<unsigned long long*>(&s.ctl->rfix_div), static_cast<unsigned long long>(sdiv));
  }
}

// Targets of the R batch from the mismatch bitmaps of the listed tiles
// (find_troublemaker's (v_i, v_t) for every falsely labelled vertex, see the
// argument above): ascending -> g's ascending neighbour, descending -> f's
// descending neighbour.  Also returns the total mismatch count in ctl->mism.
template <class T, int DIM>
__global__ void __launch_bounds__(256) k_expand_targets(State<T> s, const uint32_t* __restrict__ tiles,
                                                        TileStore ts, uint32_t* __restrict__ targets,
                                                        uint32_t* count) {
  using TL = LabelTile<DIM>;
  constexpr int NW = 2 * (kLabelTileN / 32);  // bitmap words per tile (both families)
  const Geom& g = s.geo;
  const uint32_t ntx = (g.X + TL::TX - 1) / TL::TX;
  const uint32_t nty = (g.Y + TL::TY - 1) / TL::TY;
  const uint32_t b = tiles[blockIdx.x];
  const uint32_t tx = b % ntx, ty = (b / ntx) % nty, tz = b / (ntx * nty);
  const uint32_t base = tx * TL::TX + g.X * (ty * TL::TY) + g.XY * (tz * TL::TZ);
  const uint32_t* bits = ts.mis_bits + static_cast<size_t>(b) * NW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int wpw = NW / nwarps;  // words per warp, contiguous
  // one reservation per tile: per-warp counts, scanned in shared memory
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t tbase;
  uint32_t c = 0;
  for (int k = lane; k < wpw; k += 32) c += __popc(__ldg(bits + warp * wpw + k));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) wsum[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < nwarps; ++w) {
      const uint32_t x = wsum[w];
      wsum[w] = t;
      t += x;
    }
    tbase = t ? atomicAdd(count, t) : 0u;
    if (t) atomicAdd(reinterpret_cast<unsigned long long*>(&s.ctl->mism), static_cast<unsigned long long>(t));
  }
  __syncthreads();
  uint32_t pos = tbase + wsum[warp];
  // lane j expands bit j of each of the warp's words, in word order
#pragma unroll 4
  for (int k = 0; k < wpw; ++k) {
    const int w = warp * wpw + k;
    const uint32_t word = __ldg(bits + w);
    if ((word >> lane) & 1u) {
      const int fam = w >= kLabelTileN / 32;
      const int i = ((w % (kLabelTileN / 32)) << 5) + lane;
      const int lx = i & (TL::TX - 1), ly = (i >> TL::LX) & (TL::TY - 1), lz = i >> (TL::LX + TL::LY);
      const uint32_t v = base + lx + g.X * ly + g.XY * lz;
      const uint32_t code = fam ? (__ldg(s.fdir + v) >> 4) : (__ldg(s.gdir + v) & 15u);
      const bool owned = v - s.own_lo < s.own_n;
      if (code == kSelf && owned) atomicExch(&s.ctl->status, kStatusTroubleMax);
      const uint32_t t = code == kSelf ? v : v + g.off[code];
      // owner-computes (z-slab windows): only targets this rank owns; on a
      // single device every target is owned.  A dropped slot keeps the list dense.
      targets[pos + __popc(word & ((1u << lane) - 1u))] = t - s.own_lo < s.own_n ? t : kNoTarget;
    }
    pos += __popc(word);
  }
}

// ---------------------------------------------------------------------------
// Sparse R iteration (late R-loop iterations, few mismatches).
//   X = { u : fL(step_g(u)) != fL(u) }: vertices whose g-step crosses an f-basin
//   boundary (L = M with ascending steps, m with descending).  If a vertex's
//   g-chain avoids X, fL is constant along it, so its g label equals its f
//   label: every mismatched vertex lies in Up(X), the g-forest upstream
//   closure of X.  At convergence X is empty.  So: list X, BFS backwards to
//   Up(X), resolve g labels by pointer jumping restricted to Up(X) (a chain
//   leaving Up(X) ends with the f label of its first outside vertex), and
//   emit the batch targets of divergent mismatched vertices -- the same target
//   set as the full pass.
// X built (from scratch: since = 0, no old lists) or maintained across any
// edits, both families at once.  Entries of the old lists outside dirty chunks
// are kept; every vertex of a dirty chunk is re-evaluated.  A chunk is dirty when a code in it changed since the old X:
// its change mark (cstamp, written by every frontier refresh) is >= `since`,
// the first mark issued after the old X (marks only grow; after a full
// direction sweep `since` is 0: every chunk is re-evaluated).  One warp per 32
// chunks; lanes cover a chunk's 64 vertices.
__global__ void __launch_bounds__(256) k_cross_chunks(
    const uint8_t* __restrict__ gdir, const uint32_t* __restrict__ fM,
    const uint32_t* __restrict__ fm, Geom g, const uint32_t* __restrict__ cstamp, uint32_t since,
    const uint32_t* __restrict__ Xa_old, uint32_t na_old, const uint32_t* __restrict__ Xd_old,
    uint32_t nd_old, uint32_t* __restrict__ Xa, uint32_t* __restrict__ Xd, uint32_t* counts,
    uint32_t cap) {
  const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const int lane = threadIdx.x & 31;
  // (a) surviving old entries
  const uint64_t nold = static_cast<uint64_t>(na_old) + nd_old;
  for (uint64_t wb = gtid & ~uint64_t(31); wb < nold; wb += stride) {
    const uint64_t i = wb + lane;
    bool ka = false, kd = false;
    uint32_t v = 0;
    if (i < nold) {
      v = i < na_old ? Xa_old[i] : Xd_old[i - na_old];
      const bool clean = __ldg(cstamp + (v >> 6)) < since;
      ka = clean && i < na_old;
      kd = clean && i >= na_old;
    }
    warp_append_cap(ka, v, Xa, counts + 0, cap);
    warp_append_cap(kd, v, Xd, counts + 1, cap);
  }
  // (b) re-evaluate dirty chunks: a warp ballots the change marks of 32
  // consecutive 64-vertex chunks
  const uint64_t nwords = (static_cast<uint64_t>(g.n) + 2047) / 2048;
  const uint64_t nch = (static_cast<uint64_t>(g.n) + 63) / 64;
  const uint64_t wstride = stride / 32;
  for (uint64_t w = gtid / 32; w < nwords; w += wstride) {
    const uint64_t c = w * 32 + lane;
    uint32_t bits = __ballot_sync(0xffffffffu, c < nch && __ldg(cstamp + c) >= since);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint64_t v = (w * 32 + b) * 64 + h * 32 + lane;
        bool ca = false, cd = false;
        if (v < g.n) {
          const uint32_t code = __ldg(gdir + v);
          const uint32_t a = code & 15u, d = code >> 4;
          if (a != kSelf) ca = __ldg(fM + v + g.off[a]) != __ldg(fM + v);
          if (d != kSelf) cd = __ldg(fm + v + g.off[d]) != __ldg(fm + v);
        }
        warp_append_cap(ca, static_cast<uint32_t>(v), Xa, counts + 0, cap);
        warp_append_cap(cd, static_cast<uint32_t>(v), Xd, counts + 1, cap);
      }
    }
  }
}

// Backward BFS over the g-forest of family fam from the frontier list in[]:
// u joins when its g-step points at a frontier vertex.  Persistent
// cooperative kernel, one grid barrier pair per level; every reached vertex is
// also appended to up[].  Aborts (ctl->sp_abort) when |Up| exceeds max_up.
template <int DIM>
__global__ void __launch_bounds__(512, 2)
    k_upstream(const uint8_t* __restrict__ gdir, Geom g, int fam, uint32_t* __restrict__ fmark,
               uint32_t mark, uint32_t* __restrict__ fa, uint32_t* __restrict__ fb,
               uint32_t* __restrict__ up, uint32_t max_up, uint32_t max_levels, Ctl* ctl) {
  cg::grid_group grid = cg::this_grid();
  constexpr int LPS = 16;
  constexpr int NS = StencilSize<DIM>::value;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t* cnt = ctl->sp_count;  // [1], [2]: frontier sizes; [3]: |Up|
  int cur = 0;
  uint32_t levels = 0;
  // Every exit decision must be identical in all threads (a thread that leaves
  // while others wait in grid.sync deadlocks the grid).  The frontier size and
  // the abort word are written only between the two grid barriers of a level,
  // so the reads at the top of the next level are stable; |Up| (cnt[3]) keeps
  // growing while fast warps already append the next level, so it is compared
  // with max_up by thread 0 between the barriers, never at the top.
  for (;;) {
    const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&cnt[1 + cur]);
    if (n == 0) break;
    if (*reinterpret_cast<volatile uint32_t*>(&ctl->sp_abort)) break;
    if (levels >= max_levels) {
      if (tid == 0) ctl->sp_abort = 1;
      break;
    }
    const uint32_t* in = cur ? fb : fa;
    uint32_t* out = cur ? fa : fb;
    const uint64_t total = static_cast<uint64_t>(n) * LPS;
    for (uint64_t wb = tid & ~uint64_t(31); wb < total; wb += stride) {
      const uint64_t i = wb + (threadIdx.x & 31);
      bool mine = false;
      uint32_t u = 0;
      if (i < total) {
        const int k = static_cast<int>(i % LPS);
        if (k < NS) {
          const uint32_t y = in[i / LPS];
          uint32_t x, yy, z;
          coords(g, y, x, yy, z);
          int dx, dy, dz;
          slot_delta<DIM>(k, dx, dy, dz);
          const uint32_t ux = x + dx, uy = yy + dy, uz = z + dz;
          if (ux < g.X && uy < g.Y && (DIM == 2 || uz < g.Z)) {
            u = ux + g.X * uy + g.XY * uz;
            const uint32_t c = (__ldg(gdir + u) >> (4 * fam)) & 15u;
            // u's step is the opposite slot of k (slots come in +d/-d pairs)
            if (c == static_cast<uint32_t>(k ^ 1) && __ldcg(fmark + u) != mark &&
                atomicExch(fmark + u, mark) != mark)
              mine = true;
          }
        }
      }
      warp_append_cap(mine, u, out, &cnt[2 - cur], max_up);
      warp_append_cap(mine, u, up, &cnt[3], max_up);
    }
    grid.sync();
    if (tid == 0) {
      cnt[1 + cur] = 0;
      if (*reinterpret_cast<volatile uint32_t*>(&cnt[3]) > max_up) ctl->sp_abort = 1;
    }
    cur ^= 1;
    ++levels;
    grid.sync();
  }
  if (tid == 0) ctl->sp_levels += levels;
}

__global__ void __launch_bounds__(256) k_up_seed(const uint32_t* __restrict__ X, uint32_t nx,
                                                 uint32_t* __restrict__ fmark, uint32_t mark,
                                                 uint32_t* __restrict__ up) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nx; i += stride) {
    fmark[X[i]] = mark;
    up[i] = X[i];
  }
}

// Restricted labels over Up, packed pv[i] = parent << 32 | value: parent is the
// Up index of i's g-step target when that target is in Up (fmark == mark);
// otherwise parent = ~0 and value = fL of the target (its chain avoids X).
// One 64-bit word per entry keeps in-place jumping race-free.
__global__ void __launch_bounds__(256) k_up_index(const uint32_t* __restrict__ up, uint32_t nup,
                                                  uint32_t* __restrict__ upidx) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nup; i += stride)
    upidx[up[i]] = static_cast<uint32_t>(i);
}

constexpr uint64_t kUpNone = 0xFFFFFFFF00000000ull;

__global__ void __launch_bounds__(256) k_up_parent(const uint32_t* __restrict__ up, uint32_t nup,
                                                   const uint8_t* __restrict__ gdir, Geom g, int fam,
                                                   const uint32_t* __restrict__ fmark, uint32_t mark,
                                                   const uint32_t* __restrict__ upidx,
                                                   const uint32_t* __restrict__ fL,
                                                   uint64_t* __restrict__ pv) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nup; i += stride) {
    const uint32_t v = up[i];
    const uint32_t c = (__ldg(gdir + v) >> (4 * fam)) & 15u;
    const uint32_t p = v + g.off[c];  // c != SELF: every Up vertex steps towards X
    pv[i] = __ldg(fmark + p) == mark ? (static_cast<uint64_t>(upidx[p]) << 32)
                                     : (kUpNone | __ldg(fL + p));
  }
}

__global__ void __launch_bounds__(256) k_up_jump(uint64_t* __restrict__ pv, uint32_t nup,
                                                 uint32_t* flag) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  bool changed = false;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nup; i += stride) {
    const uint64_t w = pv[i];
    if ((w >> 32) == 0xFFFFFFFFu) continue;
    const uint64_t wp = pv[w >> 32];
    // a resolved target passes its value on; otherwise skip to its parent
    pv[i] = (wp >> 32) == 0xFFFFFFFFu ? wp : (wp & 0xFFFFFFFF00000000ull);
    changed = true;
  }
  if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) *flag = 1;
}

template <class T>
__global__ void __launch_bounds__(256) k_up_targets(State<T> s, const uint32_t* __restrict__ up,
                                                    uint32_t nup, int fam,
                                                    const uint64_t* __restrict__ pv,
                                                    uint32_t* __restrict__ targets) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint32_t* fL = fam ? s.fm : s.fM;
  uint32_t mism = 0;
  for (uint64_t wb = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~uint64_t(31);
       wb < nup; wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    bool hit = false;
    uint32_t t = 0;
    if (i < nup) {
      const uint32_t v = up[i];
      const uint32_t fc = (__ldg(s.fdir + v) >> (4 * fam)) & 15u;
      const uint32_t gc = (__ldg(s.gdir + v) >> (4 * fam)) & 15u;
      if (gc != fc && static_cast<uint32_t>(pv[i]) != __ldg(fL + v)) {  // divergent, mismatched
        ++mism;
        const uint32_t c = fam ? fc : gc;  // desc lowers f's step, asc g's step
        if (c == kSelf) atomicExch(&s.ctl->status, kStatusTroubleMax);
        t = c == kSelf ? v : v + s.geo.off[c];
        hit = true;
      }
    }
    warp_append(hit, t, targets, &s.ctl->list_count[0]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mism += __shfl_xor_sync(0xffffffffu, mism, o);
  if ((threadIdx.x & 31) == 0 && mism)
    atomicAdd(reinterpret_cast<unsigned long long*>(&s.ctl->mism),
              static_cast<unsigned long long>(mism));
}

// Gate of the R-loop (detect_false_critical().empty(), edit_engine.cpp:338):
// a vertex is a false critical point of some kind iff its max flag or its min
// flag differs between f and g.  SWAR over 16 codes per thread.
__device__ __forceinline__ uint32_t false_cp_bytes(uint32_t f, uint32_t g) {
  const uint32_t fmx = zero_bytes(~f & 0x0F0F0F0Fu), gmx = zero_bytes(~g & 0x0F0F0F0Fu);
  const uint32_t fmn = zero_bytes(~f & 0xF0F0F0F0u), gmn = zero_bytes(~g & 0xF0F0F0F0u);
  return (fmx ^ gmx) | (fmn ^ gmn);
}

// Gate restricted to the vertices whose codes an R batch may have changed
// (the frontier list F of k_frontier): before the batch there were none.
__global__ void __launch_bounds__(256) k_count_false_list(const uint8_t* __restrict__ fdir,
                                                          const uint8_t* __restrict__ gdir,
                                                          const uint32_t* __restrict__ F,
                                                          const uint32_t* nF, uint64_t* total) {
  const uint32_t n = *nF;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t c = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t u = F[i];
    c += __popc(false_cp_bytes(fdir[u], gdir[u]) & 0xFFu);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c)
    atomicAdd(reinterpret_cast<unsigned long long*>(total), static_cast<unsigned long long>(c));
}

__global__ void __launch_bounds__(256) k_count_false(const uint8_t* __restrict__ fdir,
                                                     const uint8_t* __restrict__ gdir, uint32_t n,
                                                     uint64_t* total) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n16 = n / 16;
  uint32_t c = 0;
  for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n16;
       q += stride) {
    const uint4 f = __ldg(reinterpret_cast<const uint4*>(fdir) + q);
    const uint4 gg = __ldg(reinterpret_cast<const uint4*>(gdir) + q);
    c += __popc(false_cp_bytes(f.x, gg.x)) + __popc(false_cp_bytes(f.y, gg.y)) +
         __popc(false_cp_bytes(f.z, gg.z)) + __popc(false_cp_bytes(f.w, gg.w));
  }
  for (uint64_t v = n16 * 16 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       v < n; v += stride)
    c += __popc(false_cp_bytes(fdir[v], gdir[v]) & 0xFFu);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c)
    atomicAdd(reinterpret_cast<unsigned long long*>(total), static_cast<unsigned long long>(c));
}

// Non-persistent frontier refresh (after an R batch).
template <class T, int DIM>
__global__ void __launch_bounds__(256) k_frontier(State<T> s, uint32_t ns, uint32_t mark) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  frontier_update<T, DIM>(s, ns, mark, &s.ctl->f_count, tid, stride);
}

// ---------------------------------------------------------------------------
// Input validation (derive_edits, edit_engine.cpp:389-402): non-finite values
// and |f - fhat| > xi counted in double.
template <class T>
__global__ void __launch_bounds__(256) k_validate(const T* __restrict__ f,
                                                  const T* __restrict__ fh, uint64_t n, double xi,
                                                  Ctl* ctl) {
  uint32_t bad = 0, viol = 0;
  auto check = [&](T fa, T fb) {
    const double a = static_cast<double>(fa), b = static_cast<double>(fb);
    if (!isfinite(a) || !isfinite(b)) ++bad;
    else if (fabs(__dsub_rn(a, b)) > xi) ++viol;
  };
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t head = 0;
  if (sizeof(T) == 4 && ((reinterpret_cast<uintptr_t>(f) | reinterpret_cast<uintptr_t>(fh)) & 15u) == 0) {
    // f32, 16-byte aligned (slab windows may not be): two 16-byte loads per array in flight
    const uint64_t n4 = n / 4;
    const float4* f4 = reinterpret_cast<const float4*>(f);
    const float4* h4 = reinterpret_cast<const float4*>(fh);
    for (uint64_t i = t0; i < n4; i += 2 * stride) {
      const bool two = i + stride < n4;
      const float4 a0 = __ldg(f4 + i), b0 = __ldg(h4 + i);
      float4 a1 = a0, b1 = b0;
      if (two) {
        a1 = __ldg(f4 + i + stride);
        b1 = __ldg(h4 + i + stride);
      }
      check(a0.x, b0.x), check(a0.y, b0.y), check(a0.z, b0.z), check(a0.w, b0.w);
      if (two) check(a1.x, b1.x), check(a1.y, b1.y), check(a1.z, b1.z), check(a1.w, b1.w);
    }
    head = n4 * 4;
  }
  for (uint64_t i = head + t0; i < n; i += stride) check(__ldg(f + i), __ldg(fh + i));
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

// touched == (g != fhat) bitwise: every successful lower_step strictly lowers
// g (edit_engine.cpp:75-86), so the single-device engine keeps no touched
// array (one random line less per edit) and derives it here before K6.
template <class T>
__global__ void __launch_bounds__(256) k_flag_changed(const T* __restrict__ g, const T* __restrict__ fh,
                                                      uint64_t n, uint8_t* __restrict__ flag) {
  using B = typename KeyOf<T>::type;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n4 = n / 4;
  for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += stride) {
    uint32_t f4 = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const B a = reinterpret_cast<const B*>(g)[q * 4 + j], b = __ldg(reinterpret_cast<const B*>(fh) + q * 4 + j);
      f4 |= (a != b ? 1u : 0u) << (8 * j);
    }
    reinterpret_cast<uint32_t*>(flag)[q] = f4;
  }
  for (uint64_t v = n4 * 4 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    flag[v] = reinterpret_cast<const B*>(g)[v] != reinterpret_cast<const B*>(fh)[v] ? 1 : 0;
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
    T* __restrict__ val_out, uint64_t base) {
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
    idx_out[pos] = base + v0 + j;  // base: global id of the first slab vertex
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

__global__ void k_scatter_check(uint64_t count, const uint64_t* __restrict__ idx, uint64_t n,
                                uint32_t* flags) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    const uint64_t v = idx[i];
    if (v >= n) flags[0] = 1;
    if (i + 1 < count && idx[i + 1] < v) flags[1] = 1;
  }
}

// non-decreasing indices: the last element of each run of equal indices wins
template <class T>
__global__ void k_scatter(uint64_t count, const uint64_t* __restrict__ idx,
                          const T* __restrict__ vals, T* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    const uint64_t v = idx[i];
    if (i + 1 == count || idx[i + 1] != v) out[v] = vals[i];
  }
}

// unsorted indices: the largest position per vertex wins (in-order application)
__global__ void k_scatter_winner(uint64_t count, const uint64_t* __restrict__ idx,
                                 unsigned long long* __restrict__ win) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride)
    atomicMax(win + idx[i], static_cast<unsigned long long>(i + 1));
}

template <class T>
__global__ void k_scatter_won(uint64_t count, const uint64_t* __restrict__ idx,
                              const T* __restrict__ vals, const unsigned long long* __restrict__ win,
                              T* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride)
    if (win[idx[i]] == i + 1) out[idx[i]] = vals[i];
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
    // u32 wraparound: off holds the stencil offset mod 2^32 (make_geom)
    asc[v] = static_cast<uint32_t>(v) + static_cast<uint32_t>(off[c & 15u]);
    desc[v] = static_cast<uint32_t>(v) + static_cast<uint32_t>(off[c >> 4]);
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
