// wg.cu — the workload generator's request model and sampler (§III-B, P:L128-132;
// SURVEY.md §8(f) NEXT-3), on the device.
//
// Build:
//   per parameter p, bins = the fit's quantile cuts (binning.cu, O2) with 64 bins: one bin per
//   distinct value when a parameter has at most 64, else equal-frequency quantiles;
//   k_wg_keys: one pass over the traces — each row's bin per parameter (upper_bound over the cuts in
//   shared memory), its mixed-radix joint key sum_p code_p * stride_p, and each bin's min / max
//   (per-CTA shared-memory min/max on order-preserving integer images of the floats, one global
//   atomic per bin per CTA); centre = (min + max) / 2 in fp64;
//   sparse joint histogram = radix sort of the keys (only the key space's bits) + run-length
//   encoding (distinct keys, counts) + inclusive scan (cumulative counts).
// Sample: one thread per request: r = rng4(seed, 0x5747, s, 0), t = floor(r * n / 2^64)
//   (multiply-high), the first joint bin with cumulative count > t (binary search), its key decoded
//   into bin centres.  Counts are integers and the draw is an integer map, so the samples are
//   bit-exact against the CPU reference (tests/test_gpu_parity.py).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace llmp {

constexpr int WG_BINS = 64;
constexpr int WG_THREADS = 256;

// order-preserving map of a float to uint32 (-0 canonicalised to +0 first)
__device__ __forceinline__ uint32_t f2ord(float x) {
  if (x == 0.0f) x = 0.0f;
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

struct WgKeyArgs {
  const float* T;
  int64_t n;
  int P;
  const float* cuts;     // [32][255]
  const int32_t* ncuts;  // [32]
  uint64_t stride[kMaxF];
  uint64_t* keys;
  uint32_t* bmin;        // [P][64] order images
  uint32_t* bmax;
  int* flag;             // set on a non-finite value
};

__global__ void __launch_bounds__(WG_THREADS) k_wg_keys(const WgKeyArgs a) {
  __shared__ float s_cuts[kMaxF][WG_BINS];
  __shared__ int s_nc[kMaxF];
  __shared__ uint32_t s_min[kMaxF * WG_BINS], s_max[kMaxF * WG_BINS];
  for (int i = threadIdx.x; i < a.P * WG_BINS; i += WG_THREADS) {
    const int p = i / WG_BINS, b = i % WG_BINS;
    if (b < WG_BINS - 1) s_cuts[p][b] = a.cuts[p * (kBins - 1) + b];
    s_min[i] = 0xffffffffu;
    s_max[i] = 0u;
  }
  for (int p = threadIdx.x; p < a.P; p += WG_THREADS) s_nc[p] = a.ncuts[p];
  __syncthreads();
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * WG_THREADS + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * WG_THREADS) {
    uint64_t key = 0;
    for (int p = 0; p < a.P; ++p) {
      const float x = a.T[i * a.P + p];
      bad |= !isfinite(x);
      int lo = 0, hi = s_nc[p];   // upper_bound: number of cuts <= x (O2)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_cuts[p][mid] <= x) lo = mid + 1;
        else hi = mid;
      }
      key += (uint64_t)lo * a.stride[p];
      const uint32_t o = f2ord(x);
      atomicMin(&s_min[p * WG_BINS + lo], o);
      atomicMax(&s_max[p * WG_BINS + lo], o);
    }
    a.keys[i] = key;
  }
  if (bad) atomicExch(a.flag, 1);
  __syncthreads();
  for (int i = threadIdx.x; i < a.P * WG_BINS; i += WG_THREADS) {
    if (s_min[i] != 0xffffffffu) atomicMin(&a.bmin[i], s_min[i]);
    if (s_max[i] != 0u) atomicMax(&a.bmax[i], s_max[i]);
  }
}

__global__ void k_wg_centres(const uint32_t* bmin, const uint32_t* bmax, const int32_t* ncuts, int P, float* centres) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * WG_BINS) return;
  const int p = i / WG_BINS, b = i % WG_BINS;
  float c = 0.0f;
  if (b <= ncuts[p] && bmin[i] != 0xffffffffu)
    c = (float)__dmul_rn(__dadd_rn((double)ord2f(bmin[i]), (double)ord2f(bmax[i])), 0.5);
  centres[i] = c;
}

struct WgSampleArgs {
  const uint64_t* keys;
  const int64_t* cum;
  int64_t m, n;
  int P;
  const int32_t* nbins;
  const float* centres;   // [P][64]
  uint64_t seed;
  int64_t first, count;
  float* out;
};

__global__ void __launch_bounds__(WG_THREADS) k_wg_sample(const WgSampleArgs a) {
  __shared__ float s_c[kMaxF * WG_BINS];
  __shared__ uint32_t s_nb[kMaxF];
  for (int i = threadIdx.x; i < a.P * WG_BINS; i += WG_THREADS) s_c[i] = a.centres[i];
  for (int p = threadIdx.x; p < a.P; p += WG_THREADS) s_nb[p] = (uint32_t)a.nbins[p];
  __syncthreads();
  for (int64_t s = (int64_t)blockIdx.x * WG_THREADS + threadIdx.x; s < a.count; s += (int64_t)gridDim.x * WG_THREADS) {
    const uint64_t r = rng4(a.seed, 0x5747u, (uint64_t)(a.first + s), 0);
    const uint64_t t = __umul64hi(r, (uint64_t)a.n);   // floor(r * n / 2^64), in [0, n)
    int64_t lo = 0, hi = a.m - 1;                      // first j with cum[j] > t
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((uint64_t)__ldg(a.cum + mid) > t) hi = mid;
      else lo = mid + 1;
    }
    uint64_t key = __ldg(a.keys + lo);
    float* o = a.out + s * a.P;
    for (int p = 0; p < a.P; ++p) {
      const uint64_t nb = s_nb[p];
      const uint64_t q = key / nb;
      o[p] = s_c[p * WG_BINS + (int)(key - q * nb)];
      key = q;
    }
  }
}

void wg_build(Ctx* ctx, const float* T, int64_t n, int P, WgData& out) {
  LLMP_REQUIRE(n >= 1 && P >= 1 && P <= kMaxF, "workload generator: n must be >= 1 and P in [1, 32]");
  cudaStream_t s = ctx->stream;
  out.P = P;
  out.n = n;
  compute_cuts(ctx, T, n, P, 0, n, WG_BINS, out.cuts, false);   // local: no collective
  LLMP_CUDA(cudaStreamSynchronize(s));
  WgKeyArgs a{};
  double space = 1.0;
  uint64_t st = 1;
  out.nbins.assign(P, 0);
  for (int p = 0; p < P; ++p) {
    out.nbins[p] = out.cuts.h_ncuts[p] + 1;
    a.stride[p] = st;
    space *= (double)out.nbins[p];
    st *= (uint64_t)out.nbins[p];
  }
  LLMP_REQUIRE(space <= 9.2e18, "workload generator: joint key space exceeds 2^63");
  int end_bit = 1;
  while (end_bit < 64 && ((uint64_t)1 << end_bit) < st) ++end_bit;
  a.T = T;
  a.n = n;
  a.P = P;
  a.cuts = out.cuts.d_cuts.as<float>();
  a.ncuts = out.cuts.d_ncuts.as<int32_t>();
  DevBuf& d_keys = ctx->workspace("wg_keys", (size_t)n * 8);
  DevBuf& d_sorted = ctx->workspace("wg_sorted", (size_t)n * 8);
  DevBuf& d_mm = ctx->workspace("wg_minmax", (size_t)2 * kMaxF * WG_BINS * 4 + 16);
  a.keys = d_keys.as<uint64_t>();
  a.bmin = d_mm.as<uint32_t>();
  a.bmax = a.bmin + kMaxF * WG_BINS;
  a.flag = reinterpret_cast<int*>(a.bmax + kMaxF * WG_BINS);
  LLMP_CUDA(cudaMemsetAsync(a.bmin, 0xff, (size_t)kMaxF * WG_BINS * 4, s));
  LLMP_CUDA(cudaMemsetAsync(a.bmax, 0, (size_t)kMaxF * WG_BINS * 4 + 16, s));
  const int grid = (int)std::min<int64_t>((n + WG_THREADS - 1) / WG_THREADS, (int64_t)ctx->sms * 8);
  LLMP_LAUNCH(ctx, KC_WG, n, k_wg_keys, grid, WG_THREADS, 0, a);
  // sparse joint histogram: sort, run-length encode, cumulative counts
  DevBuf& d_unique = ctx->workspace("wg_unique", (size_t)n * 8);
  DevBuf& d_counts = ctx->workspace("wg_counts", (size_t)n * 8);
  DevBuf& d_nruns = ctx->workspace("wg_nruns", 8);
  size_t t1 = 0, t2 = 0, t3 = 0;
  LLMP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, d_keys.as<uint64_t>(), d_sorted.as<uint64_t>(), (int64_t)n, 0,
                                           end_bit, s));
  LLMP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, t2, d_sorted.as<uint64_t>(), d_unique.as<uint64_t>(),
                                               d_counts.as<int64_t>(), d_nruns.as<int64_t>(), (int64_t)n, s));
  LLMP_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t3, d_counts.as<int64_t>(), d_keys.as<int64_t>(), (int64_t)n, s));
  DevBuf& d_tmp = ctx->workspace("wg_cubtmp", std::max(t1, std::max(t2, t3)));
  size_t tb = d_tmp.bytes;
  LLMP_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp.p, tb, d_keys.as<uint64_t>(), d_sorted.as<uint64_t>(), (int64_t)n, 0,
                                           end_bit, s));
  tb = d_tmp.bytes;
  LLMP_CUDA(cub::DeviceRunLengthEncode::Encode(d_tmp.p, tb, d_sorted.as<uint64_t>(), d_unique.as<uint64_t>(),
                                               d_counts.as<int64_t>(), d_nruns.as<int64_t>(), (int64_t)n, s));
  int64_t m = 0;
  int flag = 0;
  LLMP_CUDA(cudaMemcpyAsync(&m, d_nruns.p, 8, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(&flag, a.flag, 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaStreamSynchronize(s));
  LLMP_REQUIRE(flag == 0, "workload generator: traces hold a non-finite value");
  out.m = m;
  // model buffers (stream-ordered, owned by the handle)
  out.d_keys.set_stream(s);
  out.d_cum.set_stream(s);
  out.d_centres.set_stream(s);
  out.d_nbins.set_stream(s);
  out.d_keys.ensure((size_t)m * 8);
  out.d_cum.ensure((size_t)m * 8);
  out.d_centres.ensure((size_t)kMaxF * WG_BINS * 4);
  out.d_nbins.ensure((size_t)kMaxF * 4);
  LLMP_CUDA(cudaMemcpyAsync(out.d_keys.p, d_unique.p, (size_t)m * 8, cudaMemcpyDeviceToDevice, s));
  tb = d_tmp.bytes;
  LLMP_CUDA(cub::DeviceScan::InclusiveSum(d_tmp.p, tb, d_counts.as<int64_t>(), out.d_cum.as<int64_t>(), m, s));
  LLMP_LAUNCH(ctx, KC_WG, 0, k_wg_centres, (P * WG_BINS + 255) / 256, 256, 0, a.bmin, a.bmax, a.ncuts, P,
              out.d_centres.as<float>());
  LLMP_CUDA(cudaMemcpyAsync(out.d_nbins.p, out.nbins.data(), (size_t)P * 4, cudaMemcpyHostToDevice, s));
  out.centres.assign((size_t)P * WG_BINS, 0.f);
  out.h_keys.resize(m);
  out.h_counts.resize(m);
  LLMP_CUDA(cudaMemcpyAsync(out.centres.data(), out.d_centres.p, (size_t)P * WG_BINS * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(out.h_keys.data(), d_unique.p, (size_t)m * 8, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(out.h_counts.data(), d_counts.p, (size_t)m * 8, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaStreamSynchronize(s));
}

void wg_sample(Ctx* ctx, const WgData& w, int64_t count, uint64_t seed, int64_t first, float* out) {
  LLMP_REQUIRE(count >= 0 && first >= 0, "workload generator: bad sample range");
  if (count == 0) return;
  WgSampleArgs a{};
  a.keys = w.d_keys.as<uint64_t>();
  a.cum = w.d_cum.as<int64_t>();
  a.m = w.m;
  a.n = w.n;
  a.P = w.P;
  a.nbins = w.d_nbins.as<int32_t>();
  a.centres = w.d_centres.as<float>();
  a.seed = seed;
  a.first = first;
  a.count = count;
  a.out = out;
  const int grid = (int)std::min<int64_t>((count + WG_THREADS - 1) / WG_THREADS, (int64_t)ctx->sms * 8);
  LLMP_LAUNCH(ctx, KC_WG, count, k_wg_sample, grid, WG_THREADS, 0, a);
}

}  // namespace llmp
