// Base-codec quantisation / reconstruction on the GPU:
// compress_base (base_codec.cpp:76-120) and decompress_base after its Huffman
// decode (base_codec.cpp:122-152), bit-exact.
//
// Order-1 Lorenzo (base_codec.cpp:26-49) predicts v from the reconstruction at
// (x-1 | y-1 | z-1) neighbours only, so every vertex with the same x+y+z is
// independent.  Block wavefront: the grid is cut into B^3 blocks (32^2 in 2D);
// blocks on one block-diagonal (i+j+k = const) run in parallel, one launch per
// diagonal.  A CTA stages its block's inputs and the reconstructed -x/-y/-z
// halo in shared memory; thread (y,z) owns a row and walks it along x, one
// internal hyperplane per step (barrier per step), so each vertex evaluates
// exactly the reference expression -- every double operation an explicit
// round-to-nearest intrinsic, the terms in the reference's order.
#pragma once

namespace mssz_b200 {
namespace {

constexpr int64_t kQuantRadius = 32766;  // base_codec.cpp:13

template <int DIM>
struct LorBlock;
template <>
struct LorBlock<3> {
  static constexpr int BX = 16, BY = 16, BZ = 16;
};
template <>
struct LorBlock<2> {
  static constexpr int BX = 32, BY = 32, BZ = 1;
};

__device__ __forceinline__ uint32_t zigzag32(int64_t q) {
  return static_cast<uint32_t>(q >= 0 ? 2 * q : -2 * q - 1);
}
__device__ __forceinline__ int64_t unzigzag32(uint32_t z) {
  return (z & 1) ? -static_cast<int64_t>((z + 1) / 2) : static_cast<int64_t>(z / 2);
}

// kCompress: vals -> (sym, recon), escapes counted; else (sym, recon preset at
// escapes) -> recon.  diag = block-diagonal index; CTA (j, k) takes block
// i = diag - j - k.
template <class T, int DIM, bool kCompress>
__global__ void __launch_bounds__(LorBlock<DIM>::BY * LorBlock<DIM>::BZ)
    k_lorenzo_block(const T* __restrict__ vals, uint32_t* __restrict__ sym, T* __restrict__ recon, Geom g,
                    double xi, int diag, unsigned long long* escapes) {
  using LB = LorBlock<DIM>;
  constexpr int BX = LB::BX, BY = LB::BY, BZ = LB::BZ;
  constexpr int HX = BX + 1, HY = BY + 1, HZ = DIM == 3 ? BZ + 1 : 1;
  const int nbx = (g.X + BX - 1) / BX;
  const int j = blockIdx.x, k = blockIdx.y;
  const int i = diag - j - k;
  if (i < 0 || i >= nbx) return;
  const int x0 = i * BX, y0 = j * BY, z0 = k * BZ;
  // s: reconstruction with a one-cell -x/-y/-z halo; in: the block's inputs
  // inputs are staged for f32 only (f64 reads them in place: static smem is 48 KB)
  constexpr bool kStage = sizeof(T) == 4;
  __shared__ T s[HZ][HY][HX];
  __shared__ uint32_t sin_[!kCompress && kStage ? BZ : 1][!kCompress && kStage ? BY : 1][!kCompress && kStage ? BX : 1];
  __shared__ T sval[kCompress && kStage ? BZ : 1][kCompress && kStage ? BY : 1][kCompress && kStage ? BX : 1];
  const int X = g.X, Y = g.Y, Z = DIM == 3 ? g.Z : 1;
  const int nt = BY * BZ;
  // stage the halo (reconstructed by earlier diagonals) and the block's inputs
  for (int c = threadIdx.x; c < HX * HY * HZ; c += nt) {
    const int hx = c % HX, hy = (c / HX) % HY, hz = c / (HX * HY);
    const int x = x0 + hx - 1, y = y0 + hy - 1, z = DIM == 3 ? z0 + hz - 1 : 0;
    const bool halo = hx == 0 || hy == 0 || (DIM == 3 && hz == 0);
    if (halo && x >= 0 && y >= 0 && z >= 0 && x < X && y < Y && z < Z)
      s[hz][hy][hx] = recon[static_cast<uint64_t>(x) + static_cast<uint64_t>(X) * y + g.XY * z];
  }
  for (int c = threadIdx.x; c < BX * BY * BZ; c += nt) {
    const int bx = c % BX, by = (c / BX) % BY, bz = c / (BX * BY);
    const int x = x0 + bx, y = y0 + by, z = z0 + bz;
    if (x < X && y < Y && z < Z) {
      const uint64_t v = static_cast<uint64_t>(x) + static_cast<uint64_t>(X) * y + g.XY * z;
      if (kCompress) {
        if (kStage) sval[bz][by][bx] = vals[v];
      } else {
        const uint32_t sy = sym[v];
        if (kStage) sin_[bz][by][bx] = sy;
        if (sy == 0) s[DIM == 3 ? bz + 1 : 0][by + 1][bx + 1] = recon[v];  // preset literal
      }
    }
  }
  __syncthreads();
  const int ty = threadIdx.x % BY, tz = threadIdx.x / BY;
  const int y = y0 + ty, z = z0 + tz;
  const bool row_in = y < Y && z < Z;
  const double two_xi = __dmul_rn(2.0, xi);
  const uint64_t XY = g.XY;
  unsigned long long esc = 0;
  const int hz = DIM == 3 ? tz + 1 : 0;
  for (int h = 0; h < BX + BY + BZ - 2; ++h) {
    const int bx = h - ty - tz;
    const int x = x0 + bx;
    if (row_in && bx >= 0 && bx < BX && x < X) {
      const bool hx = x > 0, hy = y > 0, hzz = DIM == 3 && z > 0;
      auto at = [&](int dx, int dy, int dz) {
        return static_cast<double>(s[hz - dz][ty + 1 - dy][bx + 1 - dx]);
      };
      // lorenzo_predict (base_codec.cpp:26-49), terms in the reference's order
      double p = 0.0;
      if (DIM == 2) {
        if (hx) p = __dadd_rn(p, at(1, 0, 0));
        if (hy) p = __dadd_rn(p, at(0, 1, 0));
        if (hx && hy) p = __dsub_rn(p, at(1, 1, 0));
      } else {
        if (hx) p = __dadd_rn(p, at(1, 0, 0));
        if (hy) p = __dadd_rn(p, at(0, 1, 0));
        if (hzz) p = __dadd_rn(p, at(0, 0, 1));
        if (hx && hy) p = __dsub_rn(p, at(1, 1, 0));
        if (hy && hzz) p = __dsub_rn(p, at(0, 1, 1));
        if (hx && hzz) p = __dsub_rn(p, at(1, 0, 1));
        if (hx && hy && hzz) p = __dadd_rn(p, at(1, 1, 1));
      }
      const uint64_t v = static_cast<uint64_t>(x) + static_cast<uint64_t>(X) * y + XY * z;
      if (kCompress) {
        // compress_base (base_codec.cpp:87-113)
        const T fv = kStage ? sval[tz][ty][bx] : vals[v];
        const double f = static_cast<double>(fv);
        const double rs = __ddiv_rn(__dsub_rn(f, p), two_xi);
        int64_t q = 0;
        bool escape = !(fabs(rs) <= static_cast<double>(kQuantRadius) + 1.0);
        if (!escape) {
          q = llround(rs);
          escape = (q < 0 ? -q : q) > kQuantRadius;
        }
        T r{};
        if (!escape) {
          r = narrow(__dadd_rn(p, __dmul_rn(two_xi, static_cast<double>(q))), T{});
          escape = !(fabs(__dsub_rn(f, static_cast<double>(r))) <= xi) || !isfinite(static_cast<double>(r));
        }
        s[hz][ty + 1][bx + 1] = escape ? fv : r;
        sym[v] = escape ? 0u : 1u + zigzag32(q);
        esc += escape ? 1 : 0;
      } else {
        // decompress_base (base_codec.cpp:138-148); escapes were preset
        const uint32_t sy = kStage ? sin_[tz][ty][bx] : sym[v];
        if (sy != 0)
          s[hz][ty + 1][bx + 1] =
              narrow(__dadd_rn(p, __dmul_rn(two_xi, static_cast<double>(unzigzag32(sy - 1)))), T{});
      }
    }
    __syncthreads();
  }
  for (int c = threadIdx.x; c < BX * BY * BZ; c += nt) {
    const int bx = c % BX, by = (c / BX) % BY, bz = c / (BX * BY);
    const int x = x0 + bx, yy = y0 + by, zz = z0 + bz;
    if (x < X && yy < Y && zz < Z)
      recon[static_cast<uint64_t>(x) + static_cast<uint64_t>(X) * yy + g.XY * zz] =
          s[DIM == 3 ? bz + 1 : 0][by + 1][bx + 1];
  }
  if (kCompress) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) esc += __shfl_xor_sync(0xffffffffu, esc, o);
    if ((threadIdx.x & 31) == 0 && esc) atomicAdd(escapes, esc);
  }
}

// literals (in index order, base_codec.cpp:140-144) -> recon at escape positions
template <class T>
__global__ void k_scatter_literals(const uint64_t* __restrict__ esc_idx, const T* __restrict__ lits, uint64_t nl,
                                   T* __restrict__ recon) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nl; k += stride)
    recon[esc_idx[k]] = lits[k];
}

__global__ void k_zero_flags(const uint32_t* __restrict__ sym, uint64_t n, uint8_t* __restrict__ flag) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    flag[v] = sym[v] == 0 ? 1 : 0;
}

template <class T>
void lorenzo_run(Workspace& ws, const Geom& geo, const T* vals, uint32_t* sym, T* recon, double xi, bool compress,
                 unsigned long long* d_esc) {
  auto launch = [&](auto dimc) {
    constexpr int DIM = decltype(dimc)::value;
    using LB = LorBlock<DIM>;
    const int nbx = (geo.X + LB::BX - 1) / LB::BX, nby = (geo.Y + LB::BY - 1) / LB::BY;
    const int nbz = DIM == 3 ? (geo.Z + LB::BZ - 1) / LB::BZ : 1;
    const dim3 grid(nby, nbz);
    for (int d = 0; d < nbx + nby + nbz - 2; ++d) {
      if (compress)
        k_lorenzo_block<T, DIM, true><<<grid, LB::BY * LB::BZ, 0, ws.stream>>>(vals, sym, recon, geo, xi, d, d_esc);
      else
        k_lorenzo_block<T, DIM, false><<<grid, LB::BY * LB::BZ, 0, ws.stream>>>(vals, sym, recon, geo, xi, d, d_esc);
    }
    CK_LAUNCH();
  };
  if (geo.ndims == 2) launch(std::integral_constant<int, 2>{});
  else launch(std::integral_constant<int, 3>{});
}

// Host entry: compress (values -> recon, symbols, escape count) or decompress
// (symbols + literals -> recon).  Timing of the device part in *ms.
template <class T>
void base_codec_entry(int ndims, const uint64_t* dims, const T* values, const uint32_t* sym_in, const T* literals,
                      uint64_t n_literals, double xi, T* recon_out, uint32_t* sym_out, uint64_t* escapes_out,
                      double* device_ms, bool compress) {
  const Geom geo = make_geom(ndims, dims);
  if (!(xi > 0.0)) fail(MSSZ_CU_ERR_USAGE, compress ? "compress_base requires xi > 0" : "decompress_base requires xi > 0");
  if (!recon_out || (compress && !values) || (!compress && !sym_in)) fail(MSSZ_CU_ERR_USAGE, "null pointer");
  if (!compress && n_literals && !literals) fail(MSSZ_CU_ERR_USAGE, "null literals");
  mssz_cu_options opt;
  mssz_cu_default_options(&opt);
  Workspace& ws = workspace(-1);
  std::lock_guard<std::mutex> lk(ws.mu);
  ws.ensure(geo.n, sizeof(T));
  const uint64_t n = geo.n;
  T* d_vals = ws.f.as<T>();
  T* d_rec = ws.g.as<T>();
  uint32_t* d_sym = ws.lists.as<uint32_t>();
  Engine<T> eng(ws, geo, opt);
  eng.reset_ctl();
  ws.push_ctl();
  cudaEvent_t t0, t1;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  if (compress) {
    CK(cudaMemcpyAsync(d_vals, values, sizeof(T) * n, cudaMemcpyHostToDevice, ws.stream));
    eng.pre(kProfValidate);
    k_validate<T><<<grid_for(n, 256, ws.sms, 8), 256, 0, ws.stream>>>(d_vals, d_vals, n, 0.0, ws.ctl);
    eng.launched(kProfValidate);
    ws.pull_ctl();
    if (ws.hctl->nonfinite) fail(MSSZ_CU_ERR_IO, "compress_base: non-finite value");
    CK(cudaEventRecord(t0, ws.stream));
    lorenzo_run<T>(ws, geo, d_vals, d_sym, d_rec, xi, true, reinterpret_cast<unsigned long long*>(&ws.ctl->counts[0]));
  } else {
    CK(cudaMemcpyAsync(d_sym, sym_in, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, ws.stream));
    // escapes in index order (the K6 compaction), literals scattered to them
    uint8_t* flag = ws.touched.as<uint8_t>();
    k_zero_flags<<<grid_for(n, 256, ws.sms, 8), 256, 0, ws.stream>>>(d_sym, n, flag);
    uint64_t* esc_idx = reinterpret_cast<uint64_t*>(ws.lab.p);  // 16 B/vertex scratch
    const uint64_t ne = eng.compact(flag, 1, static_cast<const T*>(nullptr), esc_idx, nullptr);
    if (ne != n_literals)
      fail(MSSZ_CU_ERR_CORRUPT_ARCHIVE, ne > n_literals ? "literal stream exhausted" : "unused literals in payload");
    T* d_lit = reinterpret_cast<T*>(ws.fin.p);
    if (ne) {
      if (sizeof(T) * ne > ws.fin.cap) fail(MSSZ_CU_ERR_INTERNAL, "literal scratch too small");
      CK(cudaMemcpyAsync(d_lit, literals, sizeof(T) * ne, cudaMemcpyHostToDevice, ws.stream));
      k_scatter_literals<T><<<grid_for(ne, 256, ws.sms, 8), 256, 0, ws.stream>>>(esc_idx, d_lit, ne, d_rec);
      CK_LAUNCH();
    }
    CK(cudaEventRecord(t0, ws.stream));
    lorenzo_run<T>(ws, geo, nullptr, d_sym, d_rec, xi, false, nullptr);
  }
  CK(cudaEventRecord(t1, ws.stream));
  CK(cudaMemcpyAsync(recon_out, d_rec, sizeof(T) * n, cudaMemcpyDeviceToHost, ws.stream));
  if (compress && sym_out) CK(cudaMemcpyAsync(sym_out, d_sym, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, ws.stream));
  ws.pull_ctl();
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, t0, t1));
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (device_ms) *device_ms = ms;
  if (compress && escapes_out) *escapes_out = ws.hctl->counts[0];
}

}  // namespace
}  // namespace mssz_b200

extern "C" {
#define MSSZ_CU_DEFINE_BASE(SUF, T)                                                                      \
  int mssz_cu_compress_base_##SUF(int ndims, const uint64_t* dims, const T* values, double xi,            \
                                  T* recon, uint32_t* symbols, uint64_t* escapes, double* device_ms) {    \
    return mssz_b200::guarded([&] {                                                                      \
      mssz_b200::base_codec_entry<T>(ndims, dims, values, nullptr, nullptr, 0, xi, recon, symbols,        \
                                     escapes, device_ms, true);                                          \
    });                                                                                                  \
  }                                                                                                      \
  int mssz_cu_decompress_base_##SUF(int ndims, const uint64_t* dims, const uint32_t* symbols,            \
                                    const T* literals, uint64_t n_literals, double xi, T* recon,         \
                                    double* device_ms) {                                                 \
    return mssz_b200::guarded([&] {                                                                      \
      mssz_b200::base_codec_entry<T>(ndims, dims, nullptr, symbols, literals, n_literals, xi, recon,      \
                                     nullptr, nullptr, device_ms, false);                                \
    });                                                                                                  \
  }
MSSZ_CU_DEFINE_BASE(f32, float)
MSSZ_CU_DEFINE_BASE(f64, double)
}  // extern "C"
