// Sector-gather throughput of 32-byte rows addressed through a sorted row-index list, as a function
// of the list's density in the row space (the level histogram's access pattern: the rows of the
// built children are a sorted-by-block subset of the identity order).  Variants: two 16-byte loads
// per row (LDG.128 x2), one 32-byte load (LDG.256), each thread holding U rows in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_density gather_density.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U, bool W256>
__global__ void gather(const uint4* __restrict__ codes, const uint32_t* __restrict__ ridx, int64_t n, unsigned long long* sink) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i0 = tid; i0 < n; i0 += stride * U) {
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ridx[min(i0 + u * stride, n - 1)];
    uint32_t v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4* p = codes + 2 * (size_t)r[u];
      if (W256) {
        asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]), "=r"(v[u][4]), "=r"(v[u][5]),
                       "=r"(v[u][6]), "=r"(v[u][7]) : "l"(p));
      } else {
        uint4 a = __ldg(p), b = __ldg(p + 1);
        v[u][0] = a.x; v[u][1] = a.y; v[u][2] = a.z; v[u][3] = a.w; v[u][4] = b.x; v[u][5] = b.y; v[u][6] = b.z; v[u][7] = b.w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc ^= v[u][k];
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t space = 80000000;   // 2.56 GB of code rows
  uint4* codes; CK(cudaMalloc(&codes, (size_t)space * 32)); CK(cudaMemset(codes, 1, (size_t)space * 32));
  uint32_t* ridx; CK(cudaMalloc(&ridx, space * 4));
  unsigned long long* sink; CK(cudaMalloc(&sink, 8));
  std::vector<uint32_t> h(space);
  std::mt19937_64 rng(1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("device SMs %d; row space %lld rows (2.56 GB)\n", sms, (long long)space);
  for (int dens : {1, 2, 4, 8, 16, 32}) {
    int64_t m = 0;
    for (int64_t i = 0; i < space; ++i) if (dens == 1 || (int)(rng() % dens) == 0) h[m++] = (uint32_t)i;
    CK(cudaMemcpy(ridx, h.data(), m * 4, cudaMemcpyHostToDevice));
    auto run = [&](auto kern, const char* name) {
      float best = 1e30f;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0); kern<<<sms * 8, 256>>>(codes, ridx, m, sink); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (it) best = std::min(best, ms);
      }
      printf("density 1/%-3d rows %9lld  %-10s %8.1f us  useful %7.1f GB/s  (rows %6.1f G/s)\n", dens, (long long)m, name,
             best * 1e3, m * 32.0 / best / 1e6, m / best / 1e6);
    };
    run(gather<1, false>, "2xLDG128");
    run(gather<4, false>, "2xLDG128x4");
    run(gather<1, true>, "LDG256");
    run(gather<4, true>, "LDG256x4");
  }
  return 0;
}
