// Random-access DRAM ceiling of this B200: how many random cache-line reads (and
// read-modify-writes) per second HBM3e sustains when every access touches a new
// line, the access pattern of the persistent C-loop kernel (k_subloop: ~40
// scattered lines per applied edit).  The streaming roofline
// (MEASURED_PEAKS.json hbm_gbs) does not bound such a kernel; this does.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rgp tools/random_gather_peak.cu
//   /tmp/rgp [GiB=4]
// Prints one JSON line: DRAM bytes/s (ncu-consistent: lines x line size) for
//   gather32  : 4-byte loads, one per random 32-byte sector
//   gather64  : 4-byte loads, one per random 64-byte line
//   rmw       : 4-byte atomicExch per random line (claims, fmark)
//   gather4x  : 4 dependent-free loads per thread per step (memory-level parallelism)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

template <int STRIDE_WORDS, int ILP, bool RMW>
__global__ void __launch_bounds__(512) k_gather(uint32_t* __restrict__ a, uint64_t nlines, uint64_t iters,
                                                uint32_t* __restrict__ sink) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nt = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t it = 0; it < iters; ++it) {
    uint64_t idx[ILP];
#pragma unroll
    for (int q = 0; q < ILP; ++q) idx[q] = (mix(tid + nt * (it * ILP + q)) % nlines) * STRIDE_WORDS;
    if (RMW) {
#pragma unroll
      for (int q = 0; q < ILP; ++q) acc += atomicExch(a + idx[q], static_cast<uint32_t>(it));
    } else {
      uint32_t v[ILP];
#pragma unroll
      for (int q = 0; q < ILP; ++q) v[q] = __ldcg(a + idx[q]);
#pragma unroll
      for (int q = 0; q < ILP; ++q) acc += v[q];
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int STRIDE_WORDS, int ILP, bool RMW>
double run(uint32_t* a, uint64_t bytes, uint32_t* sink, int sms) {
  const uint64_t nlines = bytes / (STRIDE_WORDS * 4);
  const int blocks = sms * 4;
  const uint64_t iters = 64;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_gather<STRIDE_WORDS, ILP, RMW><<<blocks, 512>>>(a, nlines, 4, sink);  // warm
  cudaEventRecord(e0);
  k_gather<STRIDE_WORDS, ILP, RMW><<<blocks, 512>>>(a, nlines, iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double accesses = double(blocks) * 512 * iters * ILP;
  return accesses / (ms * 1e-3);  // accesses per second
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 4.0;
  const uint64_t bytes = static_cast<uint64_t>(gib * (1ull << 30));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *a, *sink;
  if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess) {
    fprintf(stderr, "allocation failed\n");
    return 1;
  }
  cudaMemset(a, 1, bytes);
  const double g32 = run<8, 4, false>(a, bytes, sink, sms);
  const double g64 = run<16, 4, false>(a, bytes, sink, sms);
  const double g64x1 = run<16, 1, false>(a, bytes, sink, sms);
  const double rmw = run<16, 4, true>(a, bytes, sink, sms);
  printf("{\"array_GiB\": %.1f, \"gather32_Gaccess_s\": %.3f, \"gather64_Gaccess_s\": %.3f, "
         "\"gather64_ilp1_Gaccess_s\": %.3f, \"rmw64_Gaccess_s\": %.3f, "
         "\"note\": \"random 4-byte accesses, one per 32/64-byte line; bytes/s at DRAM = accesses x the "
         "line granularity ncu reports (see profiles/r02_random_gather_peak.json)\"}\n",
         gib, g32 * 1e-9, g64 * 1e-9, g64x1 * 1e-9, rmw * 1e-9);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
