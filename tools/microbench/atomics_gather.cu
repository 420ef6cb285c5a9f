// Microbenchmarks that decide the histogram / partition design (SURVEY.md §7 "Hard parts" 2-3):
//   1. shared-memory atomic throughput for the "lane = feature, one row per warp instruction"
//      pattern (64-bit packed vs two 32-bit arrays), random vs structured codes;
//   2. global RED.64 flush throughput (per-CTA histogram flush into one node histogram);
//   3. HBM gather throughput of 32-byte code rows addressed through a row-index list
//      (identity, sorted subsets of several densities, random permutation).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics_gather atomics_gather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// mode 0: random codes; mode 1: structured (code constant over 128 consecutive rows)
template <int KIND>
__global__ void smem_atomic_kernel(int rows_per_warp, int mode, unsigned long long* sink) {
  extern __shared__ unsigned long long hist[];  // 256 bins x 32 features
  uint32_t* h32 = reinterpret_cast<uint32_t*>(hist);
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t row0 = warp * rows_per_warp;
  for (int r = 0; r < rows_per_warp; ++r) {
    uint32_t row = row0 + r;
    uint32_t code = mode == 0 ? (hash32(row * 32u + lane) & 255u) : (hash32((row >> 7) * 32u + lane) & 255u);
    uint32_t g = hash32(row) & 0x7fff;
    if (KIND == 0) {
      unsigned long long v = ((unsigned long long)g << 32) | (g & 0x3fff);
      atomicAdd(&hist[code * 32 + lane], v);
    } else if (KIND == 1) {
      atomicAdd(&h32[code * 32 + lane], g);
      atomicAdd(&h32[8192 + code * 32 + lane], g & 0x3fff);
    } else {
      atomicAdd(&h32[code * 32 + lane], g);
    }
  }
  __syncthreads();
  unsigned long long acc = 0;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) acc += hist[i];
  atomicAdd(sink, acc);
}

__global__ void red_flush_kernel(long long* ghist, int nbins, int distinct) {
  long long* dst = ghist + (distinct ? (size_t)blockIdx.x * nbins * 2 : 0);
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) {
    atomicAdd((unsigned long long*)&dst[2 * i], (unsigned long long)(i + blockIdx.x));
    atomicAdd((unsigned long long*)&dst[2 * i + 1], (unsigned long long)(i ^ blockIdx.x));
  }
}

// each warp gathers 32 rows (32 B each) per iteration: lane l loads 32 B of row ridx[base+l]
__global__ void gather_kernel(const uint4* __restrict__ codes, const uint32_t* __restrict__ ridx, int64_t n,
                              unsigned long long* sink) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = tid; i < n; i += stride) {
    uint32_t r = ridx[i];
    uint4 a = __ldg(&codes[2 * (size_t)r]);
    uint4 b = __ldg(&codes[2 * (size_t)r + 1]);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void stream_kernel(const uint4* __restrict__ src, int64_t n16, unsigned long long* sink) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = tid; i < n16; i += stride) { uint4 a = __ldg(&src[i]); acc ^= a.x ^ a.y ^ a.z ^ a.w; }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s SMs %d clock %d kHz smemPerSM %zu\n", prop.name, sms, prop.clockRate, prop.sharedMemPerMultiprocessor);
  unsigned long long* sink; CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // ---- 1. shared atomics
  const char* kn[3] = {"packed64 (1 ATOMS.64/row-feature)", "two u32 arrays (2 ATOMS.32)", "single u32 (1 ATOMS.32)"};
  for (int kind = 0; kind < 3; ++kind) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int threads : {256, 512}) {
        int smem = 65536;
        void* fn = kind == 0 ? (void*)smem_atomic_kernel<0> : kind == 1 ? (void*)smem_atomic_kernel<1> : (void*)smem_atomic_kernel<2>;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
        int blocks = sms * occ; int rpw = 4096;
        for (int it = 0; it < 2; ++it) {
          cudaEventRecord(e0);
          if (kind == 0) smem_atomic_kernel<0><<<blocks, threads, smem>>>(rpw, mode, sink);
          else if (kind == 1) smem_atomic_kernel<1><<<blocks, threads, smem>>>(rpw, mode, sink);
          else smem_atomic_kernel<2><<<blocks, threads, smem>>>(rpw, mode, sink);
          cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        }
        double updates = (double)blocks * (threads / 32) * rpw * 32;
        printf("smem %-36s %-10s threads %d occ %d: %.1f G row-feature updates/s (%.2f per SM-cycle)\n", kn[kind],
               mode ? "structured" : "random", threads, occ, updates / ms / 1e6,
               updates / (ms * 1e-3) / sms / (prop.clockRate * 1e3));
      }
    }
  }
  // ---- 2. global RED flush
  {
    int nbins = 8192; long long* gh; CK(cudaMalloc(&gh, (size_t)sms * 4 * nbins * 16));
    for (int distinct = 0; distinct < 2; ++distinct) for (int blocks : {sms * 2, sms * 4}) {
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(e0); red_flush_kernel<<<blocks, 512>>>(gh, nbins, distinct); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      }
      double ops = (double)blocks * nbins * 2;
      printf("global RED.64 flush %s blocks %d: %.1f us, %.1f G ops/s\n", distinct ? "distinct" : "same-node", blocks,
             ms * 1e3, ops / ms / 1e6);
    }
    cudaFree(gh);
  }
  // ---- 3. gather
  {
    int64_t n = 10000000; size_t bytes = (size_t)n * 32;
    uint4* codes; CK(cudaMalloc(&codes, bytes)); CK(cudaMemset(codes, 1, bytes));
    uint32_t* ridx; CK(cudaMalloc(&ridx, n * 4));
    std::vector<uint32_t> h(n);
    std::mt19937_64 rng(1);
    int blocks = sms * 8;
    for (int it = 0; it < 3; ++it) { cudaEventRecord(e0); stream_kernel<<<blocks, 256>>>(codes, bytes / 16, sink); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); }
    cudaEventElapsedTime(&ms, e0, e1); printf("stream read 320MB: %.1f GB/s\n", bytes / ms / 1e6);
    for (int dens : {1, 2, 8, 32, 128, 0}) {
      int64_t m = 0;
      if (dens > 0) { for (int64_t i = 0; i < n; ++i) if (dens == 1 || (rng() % dens) == 0) h[m++] = (uint32_t)i; }
      else { for (int64_t i = 0; i < n; ++i) h[i] = (uint32_t)i; std::shuffle(h.begin(), h.end(), rng); m = n; }
      CK(cudaMemcpy(ridx, h.data(), m * 4, cudaMemcpyHostToDevice));
      for (int it = 0; it < 3; ++it) { cudaEventRecord(e0); gather_kernel<<<blocks, 256>>>(codes, ridx, m, sink); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("gather 32B rows, %s: %lld rows, %.1f us, useful %.1f GB/s (incl ridx %.1f GB/s)\n",
             dens == 0 ? "random permutation" : dens == 1 ? "identity" : (std::string("sorted density 1/") + std::to_string(dens)).c_str(),
             (long long)m, ms * 1e3, m * 32.0 / ms / 1e6, m * 36.0 / ms / 1e6);
    }
  }
  return 0;
}
