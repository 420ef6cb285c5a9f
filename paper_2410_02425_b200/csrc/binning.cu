// binning.cu — quantile cuts and bin codes ("number of bins for the histogram tree method",
// P:L209).
//
// cuts: per feature, from the rows whose GLOBAL index i == 0 (mod s), s = max(1, ceil(n_global /
// 2^20)); sorted (CUB segmented sort — the one library primitive on this path, used once per fit);
// k distinct values d_1<..<d_k: k <= B -> cuts = d_2..d_k, else c_j = v[floor(j m / B)],
// j = 1..B-1, dropping c_j == v[0] and duplicates.  codes: code(x) = #{c in cuts_f : c <= x}.
#include <cub/device/device_segmented_sort.cuh>

#include "bulk.cuh"
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
// B = 0: exact tree method (every distinct value its own bin; ncuts = -1 flags more distinct values
// than the cut stride holds); stride: cuts per feature row (255 for 8-bit codes, 1023 for 16-bit)
__global__ void __launch_bounds__(CUT_THREADS) k_select_cuts(const float* sorted, int64_t m, int B, int stride,
                                                             float* cuts, int32_t* ncuts) {
  const int f = blockIdx.x;
  const float* v = sorted + (int64_t)f * m;
  float* cf = cuts + (int64_t)f * stride;
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
  if (B == 0 && k - 1 > stride) {
    if (tid == 0) ncuts[f] = -1;
  } else if (B == 0 || k <= B) {
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
                  CutsData& out, bool sharded, bool wide) {
  LLMP_REQUIRE(F >= 1 && F <= kMaxF, "n_features must be in [1, 32]");
  const int cstride = wide ? kMaxCuts16 : kBins - 1;   // cuts per feature row
  LLMP_REQUIRE(max_bin == 0 || (max_bin >= 2 && max_bin <= cstride + 1),
               wide ? "max_bin must be in [2, 1024] (0: exact)"
                    : "max_bin must be in [2, 256] (0: exact); more bins (16-bit codes) are supported by the batched "
                      "small-fit path (cross-validation, n <= 8192 rows)");
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
  out.stride = cstride;
  out.d_cuts.set_stream(ctx->stream);
  out.d_ncuts.set_stream(ctx->stream);
  out.d_cuts.ensure((size_t)kMaxF * cstride * 4);
  out.d_ncuts.ensure((size_t)kMaxF * 4);
  LLMP_CUDA(cudaMemsetAsync(out.d_cuts.p, 0, out.d_cuts.bytes, s));
  LLMP_CUDA(cudaMemsetAsync(out.d_ncuts.p, 0, out.d_ncuts.bytes, s));
  LLMP_LAUNCH(ctx, KC_CUTS, m * F, k_select_cuts, F, CUT_THREADS, 0, sorted.as<float>(), m, max_bin,
              cstride, out.d_cuts.as<float>(), out.d_ncuts.as<int32_t>());
  out.h_cuts.assign((size_t)kMaxF * cstride, 0.f);
  out.h_ncuts.assign(kMaxF, 0);
  LLMP_CUDA(cudaMemcpyAsync(out.h_cuts.data(), out.d_cuts.p, out.h_cuts.size() * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(out.h_ncuts.data(), out.d_ncuts.p, kMaxF * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaStreamSynchronize(s));
  for (int f = 0; f < F; ++f)
    LLMP_REQUIRE(out.h_ncuts[f] >= 0, wide ? "exact tree method: a feature has more than 1024 distinct values"
                                            : "exact tree method: a feature has more than 256 distinct values (the "
                                              "8-bit code path); the small-fit path takes up to 1024");
}

// 16-bit codes with wide cuts (stride kMaxCuts16): one thread per (row, feature), binary search over
// the feature's cuts in global memory (the small-fit path's data are small: L2-resident)
__global__ void k_codes16(const float* __restrict__ X, int64_t n, int F, const float* __restrict__ cuts,
                          const int32_t* __restrict__ ncuts, uint16_t* __restrict__ codes) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * kMaxF; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / kMaxF;
    const int f = (int)(e % kMaxF);
    uint16_t code = 0;
    if (f < F) {
      const float x = X[i * F + f];
      const float* cf = cuts + (int64_t)f * kMaxCuts16;
      int lo = 0, hi = ncuts[f];
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cf[mid] <= x) lo = mid + 1;
        else hi = mid;
      }
      code = (uint16_t)lo;
    }
    codes[e] = code;
  }
}

void compute_codes16(Ctx* ctx, const float* X, int64_t n, int F, const CutsData& cuts, uint16_t* codes) {
  LLMP_REQUIRE(cuts.stride == kMaxCuts16, "16-bit codes need wide cuts");
  const int grid = (int)std::min<int64_t>(std::max<int64_t>((n * kMaxF + 255) / 256, 1), (int64_t)ctx->sms * 8);
  LLMP_LAUNCH(ctx, KC_CODES, n, k_codes16, grid, 256, 0, X, n, F, cuts.d_cuts.as<float>(), cuts.d_ncuts.as<int32_t>(),
              codes);
}

// codes: persistent CTAs of 256 threads over 128-row tiles, every transfer a bulk copy (TMA engine):
// the tile's X rows (128 x F floats, contiguous) land in a double-buffered shared-memory stage through
// cp.async.bulk + an mbarrier while the previous tile is binned; the codes leave as bulk stores — the
// row-major tile (128 x 32 B, contiguous) and, column-major, one 128-byte run per feature.  Binning:
// warp = row, lane = feature, binary search over the feature's cuts transposed in shared memory
// ([bin][feature]: the 32 lanes' searches never share a bank), 16 rows per warp in flight.
constexpr int CODE_ROWS = 128;
constexpr int CODE_THREADS = 256;
constexpr int CODE_TSTRIDE = CODE_ROWS + 16;   // column-major tile: 16-B aligned runs, 4-way (not 32-way) bank sharing
constexpr int CODE_SMEM = 2 * CODE_ROWS * kMaxF * 4 + CODE_ROWS * kMaxF + kMaxF * CODE_TSTRIDE;   // 40.5 KB
__global__ void __launch_bounds__(CODE_THREADS) k_codes(const float* __restrict__ X, int64_t n, int F,
                                                        const float* __restrict__ cuts,
                                                        const int32_t* __restrict__ ncuts, uint8_t* __restrict__ codes,
                                                        uint8_t* __restrict__ codesT, int64_t ldT, int* flag, int al) {
  __shared__ float s_cut[kBins][kMaxF];
  __shared__ int s_nc[kMaxF];
  extern __shared__ __align__(128) uint8_t code_smem[];
  float(*s_x)[CODE_ROWS * kMaxF] = reinterpret_cast<float(*)[CODE_ROWS * kMaxF]>(code_smem);       // [2] stages
  uint8_t(*s_tile)[kMaxF] = reinterpret_cast<uint8_t(*)[kMaxF]>(code_smem + 2 * CODE_ROWS * kMaxF * 4);  // row-major
  uint8_t(*s_tileT)[CODE_TSTRIDE] =
      reinterpret_cast<uint8_t(*)[CODE_TSTRIDE]>(code_smem + 2 * CODE_ROWS * kMaxF * 4 + CODE_ROWS * kMaxF);   // column-major
  __shared__ __align__(8) uint64_t s_bar[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n + CODE_ROWS - 1) / CODE_ROWS;
  // bulk path: whole tiles whose byte count is a multiple of 16 (the tail goes through plain loads)
  auto tile_rows = [&](int64_t t) { return (int)min((int64_t)CODE_ROWS, n - t * CODE_ROWS); };
  // al: bit 0 X, bit 1 codes, bit 2 codesT (with ldT) are 16-byte aligned (bulk copies need it)
  auto bulk_ok = [&](int64_t t) { return (al & 1) && ((size_t)tile_rows(t) * F * 4) % 16 == 0; };
  if (tid == 0) {
    mbar_init(smem_u32(&s_bar[0]), 1);
    mbar_init(smem_u32(&s_bar[1]), 1);
    mbar_fence_init();
  }
  if (tid < kMaxF) s_nc[tid] = ncuts[tid];
  __syncthreads();
  // cuts padded with NaN to 255 entries (no comparison with NaN holds): a fixed 8-step upper_bound
  for (int i = tid; i < (kBins - 1) * kMaxF; i += CODE_THREADS) {
    const int f = i / (kBins - 1), b = i % (kBins - 1);
    s_cut[b][f] = b < s_nc[f] ? cuts[i] : __int_as_float(0x7fffffff);   // NaN: never <= x
  }
  __syncthreads();
  auto issue = [&](int64_t t, int buf) {   // thread 0: tile t's X rows into stage buf
    if (t < ntiles && bulk_ok(t)) {
      const uint32_t bytes = (uint32_t)((size_t)tile_rows(t) * F * 4);
      mbar_arrive_expect_tx(smem_u32(&s_bar[buf]), bytes);
      bulk_g2s(smem_u32(&s_x[buf][0]), X + t * CODE_ROWS * F, bytes, smem_u32(&s_bar[buf]));
    }
  };
  if (tid == 0) issue(blockIdx.x, 0);
  uint32_t phase[2] = {0u, 0u};
  int k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int buf = k & 1;
    const int rows = tile_rows(t);
    const int64_t r0 = t * CODE_ROWS;
    const bool bulk = bulk_ok(t);
    if (tid == 0) {
      bulk_wait_read0();   // the previous tile's bulk stores have read s_tile / s_tileT
      issue(t + gridDim.x, buf ^ 1);   // next tile's stage was consumed in the previous iteration
    }
    if (bulk) {
      mbar_wait(smem_u32(&s_bar[buf]), phase[buf]);
      phase[buf] ^= 1u;
    }
    __syncthreads();   // (s_tile free again: thread 0's wait above is ordered before every write below)
    float xv[CODE_ROWS / 8];
#pragma unroll
    for (int j = 0; j < CODE_ROWS / 8; ++j) {
      const int r = warp + 8 * j;
      xv[j] = 0.f;
      if (r < rows && lane < F) xv[j] = bulk ? s_x[buf][r * F + lane] : X[(r0 + r) * F + lane];
    }
#pragma unroll
    for (int j = 0; j < CODE_ROWS / 8; ++j) {
      const int r = warp + 8 * j;
      uint8_t code = 0;
      if (r < rows && lane < F) {
        const float x = xv[j];
        if (flag && !isfinite(x)) atomicOr(flag, 1);
        int pos = 0;   // upper_bound: #{cuts <= x} over the 255 padded cuts
#pragma unroll
        for (int st = 128; st >= 1; st >>= 1)
          if (s_cut[pos + st - 1][lane] <= x) pos += st;
        code = (uint8_t)pos;
      }
      s_tile[r][lane] = code;
      s_tileT[lane][r] = code;
    }
    fence_proxy_async_smem();   // the code tiles are read by the bulk stores below
    __syncthreads();
    // one bulk store per destination run: thread 0 the row-major tile, the lanes of warp 1 the 32
    // column-major 128-byte runs (a tail tile or an unaligned destination: plain stores)
    const bool full = rows == CODE_ROWS;
    if (full && codes && (al & 2) && tid == 0) {
      bulk_s2g(codes + r0 * kMaxF, smem_u32(&s_tile[0][0]), CODE_ROWS * kMaxF);
      bulk_commit();
    }
    if (full && codesT && (al & 4) && warp == 1) {
      bulk_s2g(codesT + (int64_t)lane * ldT + r0, smem_u32(&s_tileT[lane][0]), CODE_ROWS);
      bulk_commit();
    }
    {
      if (codes && !(full && (al & 2))) {
        if (al & 2) {
          uint4* dst = reinterpret_cast<uint4*>(codes + r0 * kMaxF);
          const uint4* src = reinterpret_cast<const uint4*>(&s_tile[0][0]);
          for (int i = tid; i < rows * 2; i += CODE_THREADS) dst[i] = src[i];
        } else {
          for (int i = tid; i < rows * kMaxF; i += CODE_THREADS) codes[r0 * kMaxF + i] = (&s_tile[0][0])[i];
        }
      }
      if (codesT && !(full && (al & 4)))
        for (int i = tid; i < kMaxF * rows; i += CODE_THREADS) {
          const int f = i / rows, r = i % rows;
          codesT[(int64_t)f * ldT + r0 + r] = s_tileT[f][r];
        }
    }
    if (warp == 1) bulk_wait_read0();   // warp 1's column stores have read s_tileT
    __syncthreads();
  }
  if (tid == 0 || warp == 1) bulk_wait0();
}

void compute_codes(Ctx* ctx, const float* X, int64_t n, int F, const CutsData& cuts, uint8_t* codes, uint8_t* codesT,
                   int64_t ldT, int* flag) {
  LLMP_REQUIRE(cuts.stride == kBins - 1, "8-bit codes need at most 256 bins");
  int64_t tiles = (n + CODE_ROWS - 1) / CODE_ROWS;
  const int al = ((((uintptr_t)X & 15) == 0) ? 1 : 0) | ((((uintptr_t)codes & 15) == 0) ? 2 : 0) |
                 (((((uintptr_t)codesT | (uintptr_t)ldT) & 15) == 0) ? 4 : 0);
  ensure_smem_attr((const void*)k_codes, CODE_SMEM);
  int per_sm = 1;   // persistent CTAs: exactly the resident count (no partial second wave)
  LLMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_codes, CODE_THREADS, CODE_SMEM));
  int grid = (int)std::min<int64_t>(tiles, (int64_t)ctx->sms * std::max(1, per_sm));
  if (grid < 1) grid = 1;
  // (unaligned buffers, and tiles whose byte count is not a multiple of 16, take plain loads / stores)
  LLMP_LAUNCH(ctx, KC_CODES, n, k_codes, grid, CODE_THREADS, CODE_SMEM, X, n, F, cuts.d_cuts.as<float>(),
              cuts.d_ncuts.as<int32_t>(), codes, codesT, ldT, flag, al);
}

}  // namespace llmp
