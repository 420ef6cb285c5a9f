// binning.cu — quantile cuts and bin codes ("number of bins for the histogram tree method",
// P:L209).
//
// cuts: per feature, from the rows whose GLOBAL index i == 0 (mod s), s = max(1, ceil(n_global /
// 2^20)); sorted (CUB segmented sort — the one library primitive on this path, used once per fit);
// k distinct values d_1<..<d_k: k <= B -> cuts = d_2..d_k, else c_j = v[floor(j m / B)],
// j = 1..B-1, dropping c_j == v[0] and duplicates.  codes: code(x) = #{c in cuts_f : c <= x}.
#include <cub/device/device_segmented_sort.cuh>

#include "internal.cuh"

namespace llmp {

// gather the strided sample, transposed to [F][m], -0 canonicalised to +0
__global__ void k_gather_sample(const float* X, int64_t n, int F, int64_t i0, int64_t s, int64_t m, int64_t ld,
                                float* keys) {
  const int64_t total = m * F;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / F;
    const int f = (int)(e % F);
    float x = X[(i0 + j * s) * F + f];
    if (x == 0.0f) x = 0.0f;
    keys[(int64_t)f * ld + j] = x;
  }
}

__global__ void k_offsets(int64_t* off, int F, int64_t m) {
  int i = threadIdx.x;
  if (i <= F) off[i] = (int64_t)i * m;
}

// one CTA per feature over its sorted sample
constexpr int CUT_THREADS = 1024;
__global__ void __launch_bounds__(CUT_THREADS) k_select_cuts(const float* sorted, int64_t m, int B, float* cuts,
                                                             int32_t* ncuts) {
  const int f = blockIdx.x;
  const float* v = sorted + (int64_t)f * m;
  float* cf = cuts + (int64_t)f * (kBins - 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int64_t s_w[CUT_THREADS / 32];
  __shared__ int64_t s_total;
  // contiguous chunk per thread: count "first occurrence" flags
  const int64_t c0 = m * tid / CUT_THREADS, c1 = m * (tid + 1) / CUT_THREADS;
  int64_t cnt = 0;
  for (int64_t i = c0; i < c1; ++i) cnt += (i == 0 || v[i] != v[i - 1]);
  int64_t inc = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    int64_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  int64_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += s_w[w];
  if (tid == CUT_THREADS - 1) s_total = woff + inc;
  __syncthreads();
  const int64_t k = s_total;
  if (k <= B) {
    // the r-th distinct value (0-based), r >= 1, is cut r-1
    int64_t r = woff + inc - cnt;
    for (int64_t i = c0; i < c1; ++i) {
      if (i == 0 || v[i] != v[i - 1]) {
        if (r >= 1) cf[r - 1] = v[i];
        ++r;
      }
    }
    if (tid == 0) ncuts[f] = (int32_t)(k - 1);
  } else if (tid == 0) {
    int nc = 0;
    for (int j = 1; j < B; ++j) {
      const float c = v[((int64_t)j * m) / B];
      if (c == v[0]) continue;
      if (nc > 0 && cf[nc - 1] == c) continue;
      cf[nc++] = c;
    }
    ncuts[f] = nc;
  }
}

void compute_cuts(Ctx* ctx, const float* X, int64_t n, int F, int64_t row_offset, int64_t n_global, int max_bin,
                  CutsData& out, bool sharded) {
  LLMP_REQUIRE(F >= 1 && F <= kMaxF, "n_features must be in [1, 32]");
  LLMP_REQUIRE(max_bin >= 2 && max_bin <= kBins, "max_bin must be in [2, 256]");
  LLMP_REQUIRE(n >= 1 && n_global >= n, "bad row counts");
  cudaStream_t s = ctx->stream;
  const int64_t cap = int64_t(1) << 20;
  int64_t stride = (n_global + cap - 1) / cap;
  if (stride < 1) stride = 1;
  // local rows i with (row_offset + i) % stride == 0
  const int64_t i0 = (stride - row_offset % stride) % stride;
  const int64_t m_local = (i0 < n) ? (n - 1 - i0) / stride + 1 : 0;
  // global sample size (every rank computes it identically)
  const int64_t m = (n_global - 1) / stride + 1;
  // grow-only context workspaces: no per-fit cudaMalloc/cudaFree (cudaFree synchronises the device,
  // and a large cudaMalloc occasionally stalls for hundreds of ms)
  DevBuf& keys = ctx->workspace("cut_keys", (size_t)std::max<int64_t>(m, 1) * F * 4);
  DevBuf& sorted = ctx->workspace("cut_sorted", (size_t)std::max<int64_t>(m, 1) * F * 4);
  LLMP_REQUIRE(!sharded || ctx->sharded(), "sharded cuts need a communicator");
  if (!sharded) {
    LLMP_REQUIRE(m_local == m, "sample size mismatch");
    if (m > 0)
      LLMP_LAUNCH(ctx, KC_CUTS, m, k_gather_sample, 1024, 256, 0, X, n, F, i0, stride, m, m, keys.as<float>());
  } else {
    // multi-GPU: ranks hold contiguous shards in rank order, so the global sample
    // is the concatenation of the per-rank samples.  All-gather (row_offset, n) to size them,
    // then all-gather fixed-size padded [F][m_pad] samples and re-pack into [F][m].
    const int R = ctx->nranks;
    DevBuf& meta = ctx->workspace("cut_meta", 2 * 8);
    DevBuf& metas = ctx->workspace("cut_metas", (size_t)R * 2 * 8);
    int64_t mine[2] = {row_offset, n};
    LLMP_CUDA(cudaMemcpyAsync(meta.p, mine, 16, cudaMemcpyHostToDevice, s));
    allgather_bytes(ctx, meta.p, metas.p, 16);
    std::vector<int64_t> hm((size_t)R * 2);
    LLMP_CUDA(cudaMemcpyAsync(hm.data(), metas.p, (size_t)R * 16, cudaMemcpyDeviceToHost, s));
    LLMP_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> mr(R), pref(R + 1, 0);
    int64_t m_pad = 1;
    for (int r = 0; r < R; ++r) {
      const int64_t off_r = hm[2 * r], n_r = hm[2 * r + 1];
      const int64_t i0r = (stride - off_r % stride) % stride;
      mr[r] = (i0r < n_r) ? (n_r - 1 - i0r) / stride + 1 : 0;
      pref[r + 1] = pref[r] + mr[r];
      m_pad = std::max(m_pad, mr[r]);
    }
    LLMP_REQUIRE(pref[R] == m, "shards do not tile the global row range");
    DevBuf& local = ctx->workspace("cut_local", (size_t)m_pad * F * 4);
    DevBuf& all = ctx->workspace("cut_all", (size_t)R * m_pad * F * 4);
    if (m_local > 0)
      LLMP_LAUNCH(ctx, KC_CUTS, m_local, k_gather_sample, 1024, 256, 0, X, n, F, i0, stride, m_local, m_pad,
                  local.as<float>());
    allgather_bytes(ctx, local.p, all.p, (size_t)m_pad * F * 4);
    for (int r = 0; r < R; ++r)
      if (mr[r] > 0)
        LLMP_CUDA(cudaMemcpy2DAsync(keys.as<float>() + pref[r], (size_t)m * 4, all.as<float>() + (size_t)r * m_pad * F,
                                    (size_t)m_pad * 4, (size_t)mr[r] * 4, F, cudaMemcpyDeviceToDevice, s));
  }
  DevBuf& off = ctx->workspace("cut_off", (F + 1) * 8);
  LLMP_LAUNCH(ctx, KC_CUTS, 0, k_offsets, 1, 64, 0, off.as<int64_t>(), F, m);
  size_t temp = 0;
  LLMP_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, temp, keys.as<float>(), sorted.as<float>(), m * F, F,
                                               off.as<int64_t>(), off.as<int64_t>() + 1, s));
  DevBuf& tmp = ctx->workspace("cut_sort_tmp", std::max<size_t>(temp, 1));
  LLMP_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.p, temp, keys.as<float>(), sorted.as<float>(), m * F, F,
                                               off.as<int64_t>(), off.as<int64_t>() + 1, s));
  ctx->launches[KC_CUTS] += 1;
  out.F = F;
  out.max_bin = max_bin;
  out.d_cuts.set_stream(ctx->stream);
  out.d_ncuts.set_stream(ctx->stream);
  out.d_cuts.ensure((size_t)kMaxF * (kBins - 1) * 4);
  out.d_ncuts.ensure((size_t)kMaxF * 4);
  LLMP_CUDA(cudaMemsetAsync(out.d_cuts.p, 0, out.d_cuts.bytes, s));
  LLMP_CUDA(cudaMemsetAsync(out.d_ncuts.p, 0, out.d_ncuts.bytes, s));
  LLMP_LAUNCH(ctx, KC_CUTS, m * F, k_select_cuts, F, CUT_THREADS, 0, sorted.as<float>(), m, max_bin,
              out.d_cuts.as<float>(), out.d_ncuts.as<int32_t>());
  out.h_cuts.assign((size_t)kMaxF * (kBins - 1), 0.f);
  out.h_ncuts.assign(kMaxF, 0);
  LLMP_CUDA(cudaMemcpyAsync(out.h_cuts.data(), out.d_cuts.p, out.h_cuts.size() * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(out.h_ncuts.data(), out.d_ncuts.p, kMaxF * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaStreamSynchronize(s));
}

// codes: CTA of 256 threads per 128-row tile; warp = row, lane = feature; cuts transposed in smem
// ([bin][feature]) so the 32 lanes' binary searches never share a bank.
constexpr int CODE_ROWS = 128;
__global__ void __launch_bounds__(256) k_codes(const float* __restrict__ X, int64_t n, int F,
                                               const float* __restrict__ cuts, const int32_t* __restrict__ ncuts,
                                               uint8_t* __restrict__ codes, uint8_t* __restrict__ codesT, int64_t ldT,
                                               int* flag) {
  __shared__ float s_cut[kBins][kMaxF];
  __shared__ int s_nc[kMaxF];
  __shared__ __align__(16) uint8_t s_tile[CODE_ROWS][kMaxF];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < (kBins - 1) * kMaxF; i += 256) {
    const int f = i / (kBins - 1), b = i % (kBins - 1);
    s_cut[b][f] = cuts[i];
  }
  if (tid < kMaxF) s_nc[tid] = ncuts[tid];
  __syncthreads();
  const int nc = s_nc[lane];
  for (int64_t r0 = (int64_t)blockIdx.x * CODE_ROWS; r0 < n; r0 += (int64_t)gridDim.x * CODE_ROWS) {
    const int rows = (int)min((int64_t)CODE_ROWS, n - r0);
    for (int r = warp; r < CODE_ROWS; r += 8) {
      uint8_t code = 0;
      if (r < rows && lane < F) {
        const float x = X[(r0 + r) * F + lane];
        if (flag && !isfinite(x)) atomicOr(flag, 1);
        int lo = 0, hi = nc;   // upper_bound over the feature's cuts
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_cut[mid][lane] <= x) lo = mid + 1;
          else hi = mid;
        }
        code = (uint8_t)lo;
      }
      s_tile[r][lane] = code;
    }
    __syncthreads();
    if (codes) {
      // row-major: rows * 32 contiguous bytes, 16 B per thread
      uint4* dst = reinterpret_cast<uint4*>(codes + r0 * kMaxF);
      const uint4* src = reinterpret_cast<const uint4*>(&s_tile[0][0]);
      for (int i = tid; i < rows * 2; i += 256) dst[i] = src[i];
    }
    if (codesT) {
      // column-major: feature f, rows r0..r0+rows; 4 rows per thread-word when aligned
      for (int i = tid; i < kMaxF * CODE_ROWS; i += 256) {
        const int f = i / CODE_ROWS, r = i % CODE_ROWS;
        if (r < rows) codesT[(int64_t)f * ldT + r0 + r] = s_tile[r][f];
      }
    }
    __syncthreads();
  }
}

void compute_codes(Ctx* ctx, const float* X, int64_t n, int F, const CutsData& cuts, uint8_t* codes, uint8_t* codesT,
                   int64_t ldT, int* flag) {
  int64_t tiles = (n + CODE_ROWS - 1) / CODE_ROWS;
  int grid = (int)std::min<int64_t>(tiles, (int64_t)ctx->sms * 8);
  if (grid < 1) grid = 1;
  LLMP_LAUNCH(ctx, KC_CODES, n, k_codes, grid, 256, 0, X, n, F, cuts.d_cuts.as<float>(), cuts.d_ncuts.as<int32_t>(),
              codes, codesT, ldT, flag);
}

}  // namespace llmp
