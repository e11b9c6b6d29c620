// Edit-set encoding: encode_edits<T> (edit_codec.cpp:188-222),
// byte-identical payload.
//
//   index stream = backend( huffman( rle( leb128( delta(indices) ) ) ) )
//   value stream = backend( raw little-endian value bytes )
//
// GPU: deltas + LEB128 lengths, a scan, the varint bytes; RLE per maximal run of
// equal bytes (the reference's greedy loop emits, for a run of R bytes of b,
// floor(R/65535) 4-byte records and then either a record or the raw bytes for
// the remainder, so every run's output is known independently; edit_codec.cpp:72-90);
// the byte histogram; MSB-first bit packing of the canonical codes
// (huffman.cpp:118-141, bitstream.hpp) at scanned bit offsets.
// Host: the 256-symbol code-length construction (huffman.cpp:92-116, deterministic
// (weight, creation order) ties) and the raw DEFLATE backend through the same zlib
// call as the reference (edit_codec.cpp:111-130).
#pragma once

#include <zlib.h>

#include <cub/device/device_scan.cuh>
#include <queue>

namespace mssz_b200 {
namespace {

constexpr uint8_t kRleMarker = 0xF5;   // edit_codec.cpp:15
constexpr uint32_t kRleMinRun = 4;     // edit_codec.cpp:16
constexpr uint32_t kRleMaxRun = 65535;
constexpr int kMaxCodeLength = 57;     // huffman.cpp:17

__global__ void k_delta_len(const uint64_t* __restrict__ idx, uint64_t n, uint64_t* __restrict__ delta,
                            uint64_t* __restrict__ len, uint32_t* bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
    const uint64_t a = idx[k];
    uint64_t d = a;
    if (k) {
      const uint64_t p = idx[k - 1];
      if (a <= p) atomicExch(bad, 1u);
      d = a - p;
    }
    delta[k] = d;
    len[k] = d ? (64 - __clzll(static_cast<long long>(d)) + 6) / 7 : 1;  // LEB128 bytes (edit_codec.cpp:41-51)
  }
}

__global__ void k_leb_write(const uint64_t* __restrict__ delta, const uint64_t* __restrict__ off, uint64_t n,
                            uint8_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
    uint64_t v = delta[k], o = off[k];
    while (v >= 0x80) {
      out[o++] = static_cast<uint8_t>(v) | 0x80;
      v >>= 7;
    }
    out[o] = static_cast<uint8_t>(v);
  }
}

// 1 where a maximal run of equal bytes starts
__global__ void k_run_starts(const uint8_t* __restrict__ b, uint64_t L, uint64_t* __restrict__ flag) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L; i += stride)
    flag[i] = (i == 0 || b[i] != b[i - 1]) ? 1 : 0;
}

// run index (exclusive scan of flags) -> start position of every run
__global__ void k_run_pos(const uint64_t* __restrict__ flag, const uint64_t* __restrict__ ridx, uint64_t L,
                          uint64_t* __restrict__ start) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L; i += stride)
    if (flag[i]) start[ridx[i]] = i;
}

__device__ __forceinline__ uint64_t rle_out_bytes(uint64_t R, uint8_t b) {
  const uint64_t full = R / kRleMaxRun, rem = R % kRleMaxRun;
  return 4 * full + (rem == 0 ? 0 : (rem >= kRleMinRun || b == kRleMarker ? 4 : rem));
}

__global__ void k_run_size(const uint8_t* __restrict__ b, const uint64_t* __restrict__ start, uint64_t nruns,
                           uint64_t L, uint64_t* __restrict__ sz) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < nruns; r += stride) {
    const uint64_t s = start[r], e = r + 1 < nruns ? start[r + 1] : L;
    sz[r] = rle_out_bytes(e - s, b[s]);
  }
}

__global__ void k_run_write(const uint8_t* __restrict__ b, const uint64_t* __restrict__ start,
                            const uint64_t* __restrict__ roff, uint64_t nruns, uint64_t L,
                            uint8_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < nruns; r += stride) {
    const uint64_t s = start[r], e = r + 1 < nruns ? start[r + 1] : L;
    const uint8_t v = b[s];
    uint64_t R = e - s, o = roff[r];
    while (R > 0) {
      const uint64_t run = R < kRleMaxRun ? R : kRleMaxRun;
      if (run >= kRleMinRun || v == kRleMarker) {
        out[o] = kRleMarker;
        out[o + 1] = v;
        out[o + 2] = static_cast<uint8_t>(run);
        out[o + 3] = static_cast<uint8_t>(run >> 8);
        o += 4;
      } else {
        for (uint64_t j = 0; j < run; ++j) out[o++] = v;
      }
      R -= run;
    }
  }
}

__global__ void k_byte_hist(const uint8_t* __restrict__ b, uint64_t L, unsigned long long* __restrict__ hist) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // the stream is dominated by a few byte values: one shared atomic per
  // distinct value per warp (__match_any_sync groups equal lanes)
  for (uint64_t wb = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~uint64_t(31); wb < L;
       wb += stride) {
    const uint64_t i = wb + (threadIdx.x & 31);
    const uint32_t v = i < L ? b[i] : 256u;
    const uint32_t same = __match_any_sync(0xffffffffu, v);
    if (v < 256 && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&h[v], static_cast<uint32_t>(__popc(same)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], static_cast<unsigned long long>(h[i]));
}

__global__ void k_code_len(const uint8_t* __restrict__ b, uint64_t L, const uint8_t* __restrict__ clen,
                           uint64_t* __restrict__ bits) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L; i += stride)
    bits[i] = clen[b[i]];
}

// MSB-first packing: bit p of the stream is bit (31 - p % 32) of word p / 32
// (big-endian words, byte-swapped when copied out).  A CTA packs a chunk of
// kPackChunk consecutive symbols into shared-memory words (shared atomics),
// then stores its interior words directly and ORs only its two edge words.
constexpr int kPackChunk = 2048;
constexpr int kPackWords = kPackChunk * kMaxCodeLength / 32 + 4;
__global__ void __launch_bounds__(256) k_bit_pack(const uint8_t* __restrict__ b, uint64_t L,
                                                  const uint64_t* __restrict__ code,
                                                  const uint8_t* __restrict__ clen,
                                                  const uint64_t* __restrict__ boff, uint32_t* __restrict__ words) {
  __shared__ uint32_t sw[kPackWords];
  __shared__ uint64_t sc[256];
  __shared__ uint8_t sl[256];
  for (int k = threadIdx.x; k < 256; k += blockDim.x) {
    sc[k] = code[k];
    sl[k] = clen[k];
  }
  __syncthreads();
  for (uint64_t c0 = static_cast<uint64_t>(blockIdx.x) * kPackChunk; c0 < L;
       c0 += static_cast<uint64_t>(gridDim.x) * kPackChunk) {
    const uint64_t c1 = min(c0 + kPackChunk, L);
    const uint64_t wbase = boff[c0] >> 5;
    const uint64_t wend = (boff[c1 - 1] + sl[b[c1 - 1]] + 31) >> 5;  // exclusive
    const int nw = static_cast<int>(wend - wbase);
    __syncthreads();  // the previous chunk's words are written out
    for (int k = threadIdx.x; k < nw + 4; k += blockDim.x) sw[k] = 0u;
    __syncthreads();
    for (uint64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
      const uint8_t s = b[i];
      const int l = sl[s];
      const uint64_t p = boff[i] - (wbase << 5);
      const uint64_t w0 = p >> 5;
      const int b0 = static_cast<int>(p & 31);
      const unsigned __int128 v = static_cast<unsigned __int128>(sc[s]) << (128 - l - b0);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint32_t part = static_cast<uint32_t>(v >> (96 - 32 * k));
        if (part) atomicOr(&sw[w0 + k], part);
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nw; k += blockDim.x) {
      if (k == 0 || k == nw - 1) atomicOr(&words[wbase + k], sw[k]);  // shared with neighbour chunks
      else words[wbase + k] = sw[k];
    }
  }
}

__global__ void k_bswap_words(const uint32_t* __restrict__ words, uint64_t nbytes, uint8_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nbytes; i += stride)
    out[i] = static_cast<uint8_t>(words[i >> 2] >> (24 - 8 * (i & 3)));
}

// ---- host side ----
void put_u16(std::vector<uint8_t>& o, uint16_t v) {
  o.push_back(static_cast<uint8_t>(v));
  o.push_back(static_cast<uint8_t>(v >> 8));
}
void put_u32(std::vector<uint8_t>& o, uint32_t v) {
  for (int s = 0; s < 32; s += 8) o.push_back(static_cast<uint8_t>(v >> s));
}
void put_u64(std::vector<uint8_t>& o, uint64_t v) {
  for (int s = 0; s < 64; s += 8) o.push_back(static_cast<uint8_t>(v >> s));
}

// huffman::build_code_lengths (huffman.cpp:92-116): min-heap on (weight,
// creation order), depths by DFS, a lone symbol gets length 1.
std::vector<uint8_t> code_lengths(const std::vector<uint64_t>& freqs) {
  struct Node {
    uint64_t weight, order;
    int32_t left, right, symbol;
  };
  std::vector<Node> nodes;
  std::vector<uint8_t> lengths(freqs.size(), 0);
  for (uint32_t s = 0; s < freqs.size(); ++s)
    if (freqs[s]) nodes.push_back({freqs[s], nodes.size(), -1, -1, static_cast<int32_t>(s)});
  if (nodes.empty()) return lengths;
  auto heavier = [&](int32_t a, int32_t b) {
    if (nodes[a].weight != nodes[b].weight) return nodes[a].weight > nodes[b].weight;
    return nodes[a].order > nodes[b].order;
  };
  std::priority_queue<int32_t, std::vector<int32_t>, decltype(heavier)> heap(heavier);
  const size_t leaves = nodes.size();
  for (size_t i = 0; i < leaves; ++i) heap.push(static_cast<int32_t>(i));
  while (heap.size() > 1) {
    const int32_t a = heap.top();
    heap.pop();
    const int32_t b = heap.top();
    heap.pop();
    nodes.push_back({nodes[a].weight + nodes[b].weight, nodes.size(), a, b, -1});
    heap.push(static_cast<int32_t>(nodes.size() - 1));
  }
  std::vector<std::pair<int32_t, int>> stack{{heap.top(), 0}};
  while (!stack.empty()) {
    const auto [id, depth] = stack.back();
    stack.pop_back();
    const Node& nd = nodes[id];
    if (nd.symbol >= 0) {
      if (depth > kMaxCodeLength) fail(MSSZ_CU_ERR_INTERNAL, "huffman code length out of range");
      lengths[nd.symbol] = static_cast<uint8_t>(std::max(depth, 1));
    } else {
      stack.emplace_back(nd.left, depth + 1);
      stack.emplace_back(nd.right, depth + 1);
    }
  }
  return lengths;
}

// raw DEFLATE exactly as backend_encode (edit_codec.cpp:111-130)
std::vector<uint8_t> backend(const uint8_t* data, size_t size, int codec) {
  if (codec == 0) return std::vector<uint8_t>(data, data + size);
  z_stream zs{};
  if (deflateInit2(&zs, Z_DEFAULT_COMPRESSION, Z_DEFLATED, -15, 8, Z_DEFAULT_STRATEGY) != Z_OK)
    fail(MSSZ_CU_ERR_INTERNAL, "deflateInit failed");
  std::vector<uint8_t> out(deflateBound(&zs, static_cast<uLong>(size)));
  zs.next_in = const_cast<Bytef*>(data);
  zs.avail_in = static_cast<uInt>(size);
  zs.next_out = out.data();
  zs.avail_out = static_cast<uInt>(out.size());
  const int rc = deflate(&zs, Z_FINISH);
  deflateEnd(&zs);
  if (rc != Z_STREAM_END) fail(MSSZ_CU_ERR_INTERNAL, "deflate failed");
  out.resize(zs.total_out);
  return out;
}

template <class V>
void exclusive_scan(const V* in, V* out, uint64_t n, cudaStream_t s) {
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  void* d_tmp = nullptr;
  CK(cudaMallocAsync(&d_tmp, tmp ? tmp : 16, s));
  CK(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, in, out, n, s));
  CK(cudaFreeAsync(d_tmp, s));
}

template <class U>
U* dalloc(size_t count, cudaStream_t s) {
  void* p = nullptr;
  CK(cudaMallocAsync(&p, sizeof(U) * (count ? count : 1), s));
  return static_cast<U*>(p);
}

template <class T>
void encode_edits_entry(const uint64_t* idx, const T* val, uint64_t n, int codec, uint8_t** out_p, uint64_t* out_len,
                        double* device_ms) {
  if (!out_p || !out_len || (n && (!idx || !val))) fail(MSSZ_CU_ERR_USAGE, "null pointer");
  if (codec < 0 || codec > 1) fail(MSSZ_CU_ERR_CORRUPT_ARCHIVE, "unsupported edit backend codec id");
  std::vector<uint8_t> payload;
  put_u64(payload, n);
  double ms_total = 0;
  if (n == 0) {
    put_u64(payload, 0);  // index-stream-len
  } else {
    if (n > 0xFFFFFFFFull) fail(MSSZ_CU_ERR_USAGE, "edit set too large for the u32 symbol count");
    Workspace& ws = workspace(-1);
    std::lock_guard<std::mutex> lk(ws.mu);
    cudaStream_t s = ws.stream;
    {  // keep freed temporaries in the stream-ordered pool across the syncs below
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, ws.device));
      uint64_t keep = ~uint64_t(0);
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    uint64_t* d_idx = dalloc<uint64_t>(n, s);
    uint64_t* d_delta = dalloc<uint64_t>(n, s);
    uint64_t* d_len = dalloc<uint64_t>(n + 1, s);
    uint64_t* d_off = dalloc<uint64_t>(n + 1, s);
    uint32_t* d_bad = dalloc<uint32_t>(1, s);
    CK(cudaMemcpyAsync(d_idx, idx, 8 * n, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(e0, s));
    CK(cudaMemsetAsync(d_bad, 0, 4, s));
    CK(cudaMemsetAsync(d_len + n, 0, 8, s));
    const uint32_t bl = grid_for(n, 256, ws.sms, 16);
    k_delta_len<<<bl, 256, 0, s>>>(d_idx, n, d_delta, d_len, d_bad);
    CK_LAUNCH();
    exclusive_scan(d_len, d_off, n + 1, s);
    uint32_t bad = 0;
    uint64_t L = 0;
    CK(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&L, d_off + n, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bad) fail(MSSZ_CU_ERR_USAGE, "edit indices must be strictly increasing");
    uint8_t* d_b = dalloc<uint8_t>(L, s);
    k_leb_write<<<bl, 256, 0, s>>>(d_delta, d_off, n, d_b);
    CK_LAUNCH();
    CK(cudaFreeAsync(d_idx, s));
    CK(cudaFreeAsync(d_delta, s));
    CK(cudaFreeAsync(d_len, s));
    CK(cudaFreeAsync(d_off, s));
    // RLE over the varint bytes
    uint64_t* d_flag = dalloc<uint64_t>(L + 1, s);
    uint64_t* d_ridx = dalloc<uint64_t>(L + 1, s);
    const uint32_t bL = grid_for(L, 256, ws.sms, 16);
    k_run_starts<<<bL, 256, 0, s>>>(d_b, L, d_flag);
    CK(cudaMemsetAsync(d_flag + L, 0, 8, s));
    exclusive_scan(d_flag, d_ridx, L + 1, s);
    uint64_t R = 0;
    CK(cudaMemcpyAsync(&R, d_ridx + L, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint64_t* d_start = dalloc<uint64_t>(R, s);
    k_run_pos<<<bL, 256, 0, s>>>(d_flag, d_ridx, L, d_start);
    CK(cudaFreeAsync(d_flag, s));
    CK(cudaFreeAsync(d_ridx, s));
    uint64_t* d_rsz = dalloc<uint64_t>(R + 1, s);
    uint64_t* d_roff = dalloc<uint64_t>(R + 1, s);
    const uint32_t bR = grid_for(R, 256, ws.sms, 16);
    k_run_size<<<bR, 256, 0, s>>>(d_b, d_start, R, L, d_rsz);
    CK(cudaMemsetAsync(d_rsz + R, 0, 8, s));
    exclusive_scan(d_rsz, d_roff, R + 1, s);
    uint64_t L2 = 0;
    CK(cudaMemcpyAsync(&L2, d_roff + R, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (L2 > 0xFFFFFFFFull) fail(MSSZ_CU_ERR_USAGE, "index stream too long for the u32 symbol count");
    uint8_t* d_c = dalloc<uint8_t>(L2, s);
    k_run_write<<<bR, 256, 0, s>>>(d_b, d_start, d_roff, R, L, d_c);
    CK_LAUNCH();
    CK(cudaFreeAsync(d_b, s));
    CK(cudaFreeAsync(d_start, s));
    CK(cudaFreeAsync(d_rsz, s));
    CK(cudaFreeAsync(d_roff, s));
    // Huffman (huffman::encode_stream, huffman.cpp:118-141)
    unsigned long long* d_hist = dalloc<unsigned long long>(256, s);
    CK(cudaMemsetAsync(d_hist, 0, 8 * 256, s));
    const uint32_t bL2 = grid_for(L2, 256, ws.sms, 8);
    k_byte_hist<<<bL2, 256, 0, s>>>(d_c, L2, d_hist);
    CK_LAUNCH();
    std::vector<uint64_t> hist(256);
    CK(cudaMemcpyAsync(hist.data(), d_hist, 8 * 256, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint32_t max_symbol = 0;
    for (uint32_t k = 0; k < 256; ++k)
      if (hist[k]) max_symbol = k;
    const uint32_t table_size = max_symbol + 1;  // L2 > 0 here
    std::vector<uint64_t> freqs(hist.begin(), hist.begin() + table_size);
    const std::vector<uint8_t> lengths = code_lengths(freqs);
    // canonical codes (huffman.cpp:60-90, :126-135): by (length, symbol)
    uint32_t count[kMaxCodeLength + 1] = {};
    uint64_t first[kMaxCodeLength + 1] = {};
    int maxlen = 0;
    for (uint32_t k = 0; k < table_size; ++k)
      if (lengths[k]) {
        ++count[lengths[k]];
        maxlen = std::max<int>(maxlen, lengths[k]);
      }
    uint64_t code = 0;
    for (int len = 1; len <= maxlen; ++len) {
      first[len] = code;
      code = (code + count[len]) << 1;
    }
    std::vector<uint64_t> codes(256, 0);
    std::vector<uint8_t> clen(256, 0);
    uint32_t rank[kMaxCodeLength + 1] = {};
    for (int len = 1; len <= maxlen; ++len)
      for (uint32_t k = 0; k < table_size; ++k)
        if (lengths[k] == len) {
          codes[k] = first[len] + rank[len]++;
          clen[k] = static_cast<uint8_t>(len);
        }
    uint64_t* d_code = dalloc<uint64_t>(256, s);
    uint8_t* d_clen = dalloc<uint8_t>(256, s);
    CK(cudaMemcpyAsync(d_code, codes.data(), 8 * 256, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_clen, clen.data(), 256, cudaMemcpyHostToDevice, s));
    uint64_t* d_bits = dalloc<uint64_t>(L2 + 1, s);
    uint64_t* d_boff = dalloc<uint64_t>(L2 + 1, s);
    k_code_len<<<bL2, 256, 0, s>>>(d_c, L2, d_clen, d_bits);
    CK(cudaMemsetAsync(d_bits + L2, 0, 8, s));
    exclusive_scan(d_bits, d_boff, L2 + 1, s);
    uint64_t nbits = 0;
    CK(cudaMemcpyAsync(&nbits, d_boff + L2, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t nwords = (nbits + 31) / 32 + 4, nbytes = (nbits + 7) / 8;
    uint32_t* d_words = dalloc<uint32_t>(nwords, s);
    CK(cudaMemsetAsync(d_words, 0, 4 * nwords, s));
    k_bit_pack<<<grid_for((L2 + kPackChunk - 1) / kPackChunk, 1, ws.sms, 8), 256, 0, s>>>(d_c, L2, d_code, d_clen,
                                                                                           d_boff, d_words);
    uint8_t* d_body = dalloc<uint8_t>(nbytes, s);
    k_bswap_words<<<grid_for(nbytes, 256, ws.sms, 8), 256, 0, s>>>(d_words, nbytes, d_body);
    CK_LAUNCH();
    CK(cudaEventRecord(e1, s));
    std::vector<uint8_t> huffed;
    huffed.reserve(6 + table_size + nbytes);
    put_u32(huffed, static_cast<uint32_t>(L2));
    put_u16(huffed, static_cast<uint16_t>(table_size));
    for (uint32_t k = 0; k < table_size; ++k) huffed.push_back(lengths[k]);
    const size_t hdr = huffed.size();
    huffed.resize(hdr + nbytes);
    CK(cudaMemcpyAsync(huffed.data() + hdr, d_body, nbytes, cudaMemcpyDeviceToHost, s));
    for (void* p : {static_cast<void*>(d_c), static_cast<void*>(d_hist), static_cast<void*>(d_code),
                    static_cast<void*>(d_clen), static_cast<void*>(d_bits), static_cast<void*>(d_boff),
                    static_cast<void*>(d_words), static_cast<void*>(d_body), static_cast<void*>(d_bad)})
      CK(cudaFreeAsync(p, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms_total = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const auto index_stream = backend(huffed.data(), huffed.size(), codec);
    // value bytes: little-endian bit patterns (x86 hosts store them that way)
    const auto value_stream = backend(reinterpret_cast<const uint8_t*>(val), sizeof(T) * n, codec);
    put_u64(payload, index_stream.size());
    payload.insert(payload.end(), index_stream.begin(), index_stream.end());
    payload.insert(payload.end(), value_stream.begin(), value_stream.end());
  }
  uint8_t* out = static_cast<uint8_t*>(std::malloc(payload.size()));
  if (!out) throw std::bad_alloc();
  std::memcpy(out, payload.data(), payload.size());
  *out_p = out;
  *out_len = payload.size();
  if (device_ms) *device_ms = ms_total;
}

}  // namespace
}  // namespace mssz_b200

extern "C" {
int mssz_cu_encode_edits_f32(const uint64_t* indices, const float* values, uint64_t count, int codec,
                             uint8_t** payload, uint64_t* payload_len, double* device_ms) {
  return mssz_b200::guarded([&] {
    mssz_b200::encode_edits_entry<float>(indices, values, count, codec, payload, payload_len, device_ms);
  });
}
int mssz_cu_encode_edits_f64(const uint64_t* indices, const double* values, uint64_t count, int codec,
                             uint8_t** payload, uint64_t* payload_len, double* device_ms) {
  return mssz_b200::guarded([&] {
    mssz_b200::encode_edits_entry<double>(indices, values, count, codec, payload, payload_len, device_ms);
  });
}
}  // extern "C"
