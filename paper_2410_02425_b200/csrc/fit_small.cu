// fit_small.cu — one thread block per (fit, ensemble) for small training sets (n <= 8192 rows):
// the nested leave-one-LLM-out cross-validation of P:L207-209 / P:L271 fits hundreds to thousands
// of models of ~4.6K rows, each far too small to fill a B200 (SURVEY §7 hard part 4).  Every block
// runs one whole boosting fit (O3-O9) out of shared memory and L2, and predicts its held-out rows
// tree by tree (O10), so all the fits of a cross-validation run in one launch.
//
// The arithmetic is the one of the level-wise path in fit.cu (and of the oracle):
//   O3 base score from the quantised gradients at p = 0 (lambda = 0);
//   O4 per tree t: g = w (p - y), h = w (0 when the row is sampled out), exponents of the tree's
//      max |g|, max h, q = rint(v 2^(K - e)) as 16-bit halves of one word;
//   O5 integer histograms of every node of a level, built directly from its rows (no sibling
//      subtraction: a node's histogram equals its parent's minus its sibling's exactly, so both
//      constructions give the same integers);
//   O6 per (node, feature): prefix sums, fp64 weights and gains with the monotone veto, best (loss,
//      b); per node: best (loss desc, f asc, b asc), split iff loss > 1e-6; O7 child bounds;
//   O8 leaf v = (float)(eta W); O9 p += v; O10 held-out rows p = base + sum_t v_t in tree order.
// Shared-memory layout of a block: gradient pairs, training predictions, each row's node at the
// current level and its final leaf (12 B per row), a per-warp staging ring of code rows, the tree
// being grown, and the histograms of as many nodes of a level as fit (compact: only the bins each
// feature has, C = sum_f nbins_f cells; a level with more nodes takes several passes over the rows).
// The histogram pass walks the rows in identity order (the paper-ordered dataset's natural order)
// with the change-row scheme of k_hist3: a ballot of the rows whose node or any non-users code
// differs from the previous row; lanes = features flush their finished runs only at those rows.
#include <math.h>

#include <algorithm>

#include "internal.cuh"

namespace llmp {

constexpr int SF_MAX_N = 8192;
constexpr int SF_THREADS = 1024;
constexpr int SF_WARPS = SF_THREADS / 32;
constexpr int SF_MAX_D = 8;
constexpr int SF_MAX_NN = (1 << (SF_MAX_D + 1)) - 1;   // 511 tree nodes
constexpr int SF_MAX_LVL = 1 << (SF_MAX_D - 1);        // 128 nodes at the deepest split level
// CW: bytes per code (1: up to 256 bins; 2: 16-bit codes, up to 1024 bins — NEXT-4)
template <int CW> __host__ __device__ constexpr int sf_rowb() { return 32 * CW; }                    // staged code row
template <int CW> __host__ __device__ constexpr int sf_stage() { return 32 * sf_rowb<CW>() + 32 * 4; }   // per warp: 32 rows + 32 slots
constexpr int SF_RES = 32;                             // bytes per (node, feature) split result
constexpr int SF_SMEM_CAP = 227 * 1024 - 24 * 1024;    // dynamic budget (static tables take the rest)

struct SFRes {
  double loss;
  int32_t b, valid;
  int64_t GLq, HLq;
};
static_assert(sizeof(SFRes) == 32, "split result");

__device__ __forceinline__ double sf_exp2i(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }

__device__ __forceinline__ bool sf_sampled_out(uint64_t seed, int target, int t, int64_t gi, float subsample) {
  if (subsample >= 1.0f) return false;
  const uint64_t r = rng4(seed, (uint64_t)(2 * target), (uint64_t)t, (uint64_t)gi);
  const double u = (double)(r >> 11) * 0x1.0p-53;
  return u >= (double)subsample;
}

__device__ __forceinline__ float sf_wmax(float v) {   // warp max of non-negative floats
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int CW>
__global__ void __launch_bounds__(SF_THREADS, 1) k_fit_small(const SmallFitItem* items, const SmallFitHp* hps,
                                                             int smem_bytes) {
  constexpr int SF_ROWB = sf_rowb<CW>(), SF_STAGE = sf_stage<CW>(), NW = 8 * CW;   // NW: 32-bit words per row
  const SmallFitItem it = items[blockIdx.x];
  const SmallFitHp hp = hps[it.hp];
  const int n = it.n, tg = it.target, F = hp.F, D = hp.D, T = hp.T, K = hp.K;
  const int ucol = (hp.users_col >= 0 && hp.users_col < F) ? hp.users_col : -1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_gp = reinterpret_cast<uint32_t*>(smem);                       // [n]
  float* s_p = reinterpret_cast<float*>(smem + 4 * (size_t)it.n_cap);       // [n]
  int16_t* s_pos = reinterpret_cast<int16_t*>(smem + 8 * (size_t)it.n_cap); // [n] node at the level, -1 done
  int16_t* s_leaf = s_pos + it.n_cap;                                        // [n] final tree node
  uint8_t* s_stage = smem + 12 * (size_t)it.n_cap;                           // [warps][SF_STAGE]
  uint8_t* s_hist = s_stage + SF_WARPS * SF_STAGE;                           // histograms + results
  const int hist_bytes = smem_bytes - (int)(s_hist - smem);

  __shared__ int s_off[kMaxF + 1];          // compact cell offset of feature f (C = s_off[F])
  __shared__ int8_t s_pkw[kMaxF];           // split-evaluation feature packs (see below)
  __shared__ int8_t s_pkf[kMaxF][4];
  __shared__ int s_npk;
  __shared__ uint32_t s_inpk;
  __shared__ int s_nc[kMaxF];
  __shared__ int8_t s_tf[SF_MAX_NN];        // tree being grown: feature (-1 leaf, -2 absent)
  __shared__ uint16_t s_tb[SF_MAX_NN];
  __shared__ float s_tv[SF_MAX_NN];
  __shared__ double s_lo[2][SF_MAX_LVL * 2], s_hi[2][SF_MAX_LVL * 2];   // bounds by level parity
  __shared__ int16_t s_list[SF_MAX_LVL];    // existing nodes of the level
  __shared__ int16_t s_nlist[SF_MAX_LVL];
  __shared__ long long s_tot[SF_MAX_LVL][2];   // node totals (q_g, q_h) of the pass
  __shared__ int16_t s_slot[SF_MAX_LVL];    // node -> slot of the current pass (-1: not in it)
  __shared__ int8_t s_sf[SF_MAX_LVL];       // split feature of each node of the level (-1 none)
  __shared__ uint16_t s_sb[SF_MAX_LVL];
  __shared__ int s_ne, s_ne_next;
  __shared__ uint32_t s_colmask;
  __shared__ unsigned s_mg, s_mh;
  __shared__ long long s_sum[2];
  __shared__ float s_base;

  if (tid < kMaxF) s_nc[tid] = tid < F ? it.ncuts[tid] : 0;
  __syncthreads();
  if (tid == 0) {
    int o = 0;
    for (int f = 0; f < kMaxF; ++f) {
      s_off[f] = o;
      o += (f < F) ? s_nc[f] + 1 : 0;
    }
    s_off[kMaxF] = o;
    // feature packs for the split evaluation: features with <= 8 / <= 16 / <= 32 bins share a warp
    // four / two / one at a time (width = lanes per feature); > 32 bins: a warp of 8 bins per lane
    // (width 64 marks it); features with one bin have no threshold and are left out, except feature
    // 0, whose pass also yields the node totals
    int np_ = 0;
    uint32_t inpk = 0;
    for (int wdt = 8; wdt <= 64; wdt <<= 1) {
      const int per = wdt >= 32 ? 1 : 32 / wdt;
      int fill = per;
      for (int f = 0; f < F; ++f) {
        const int nb = s_nc[f] + 1;
        const int want = nb > 32 ? 64 : nb > 16 ? 32 : nb > 8 ? 16 : 8;
        if (want != wdt || (nb == 1 && f != 0)) continue;
        if (fill == per) {
          s_pkw[np_] = (int8_t)wdt;
          for (int q = 0; q < 4; ++q) s_pkf[np_][q] = -1;
          ++np_;
          fill = 0;
        }
        s_pkf[np_ - 1][fill++] = (int8_t)f;
        inpk |= 1u << f;
      }
    }
    s_npk = np_;
    s_inpk = inpk;
  }
  __syncthreads();
  const int C = s_off[kMaxF];
  const int node_bytes = 8 * C;
  const int per_pass = max(1, min(SF_MAX_LVL, hist_bytes / (node_bytes + 32 * SF_RES)));
  uint32_t* const hg = reinterpret_cast<uint32_t*>(s_hist);                          // [per_pass][2][C]
  SFRes* const res = reinterpret_cast<SFRes*>(s_hist + (size_t)per_pass * node_bytes);   // [per_pass][32]
  const float* __restrict__ yv = it.y;
  const float* __restrict__ wv = it.w;
  const uint8_t* __restrict__ codes = it.codes;

  // ---- O3 base score: quantised g = w (0 - y), h = w, lambda = 0
  auto block_max2 = [&](float a, float b) {   // -> s_mg, s_mh (float bits of non-negatives)
    a = sf_wmax(a);
    b = sf_wmax(b);
    if (lane == 0) {
      atomicMax(&s_mg, __float_as_uint(a));
      atomicMax(&s_mh, __float_as_uint(b));
    }
  };
  if (tid == 0) {
    s_mg = 0u;
    s_mh = 0u;
    s_sum[0] = 0;
    s_sum[1] = 0;
  }
  __syncthreads();
  {
    float mg = 0.f, mh = 0.f;
    for (int i = tid; i < n; i += SF_THREADS) {
      const float w = wv[i];
      mg = fmaxf(mg, fabsf(__fmul_rn(w, __fsub_rn(0.0f, yv[2 * i + tg]))));
      mh = fmaxf(mh, w);
    }
    block_max2(mg, mh);
  }
  __syncthreads();
  {
    const double sg = sf_exp2i(K - exp_of(__uint_as_float(s_mg))), sh = sf_exp2i(K - exp_of(__uint_as_float(s_mh)));
    long long gs = 0, hs = 0;
    for (int i = tid; i < n; i += SF_THREADS) {
      const float w = wv[i];
      gs += quantize(__fmul_rn(w, __fsub_rn(0.0f, yv[2 * i + tg])), sg);
      hs += quantize(w, sh);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gs += __shfl_xor_sync(0xffffffffu, gs, o);
      hs += __shfl_xor_sync(0xffffffffu, hs, o);
    }
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[0]), (unsigned long long)gs);
      atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[1]), (unsigned long long)hs);
    }
  }
  __syncthreads();
  if (tid == 0) {
    const double G = dequant(s_sum[0], sf_exp2i(exp_of(__uint_as_float(s_mg)) - K));
    const double H = dequant(s_sum[1], sf_exp2i(exp_of(__uint_as_float(s_mh)) - K));
    s_base = H > 0.0 ? (float)__ddiv_rn(-G, H) : 0.0f;
    s_mg = 0u;
    s_mh = 0u;
  }
  __syncthreads();
  const float base = s_base;
  for (int i = tid; i < it.m_test; i += SF_THREADS) it.pred_test[2 * i + tg] = base;
  // p = base; tree 0's gradient maxima
  {
    float mg = 0.f, mh = 0.f;
    for (int i = tid; i < n; i += SF_THREADS) {
      s_p[i] = base;
      if (T > 0) {
        const float w = wv[i];
        float g = __fmul_rn(w, __fsub_rn(base, yv[2 * i + tg]));
        float h = w;
        if (sf_sampled_out(hp.seed, tg, 0, i, hp.subsample)) {
          g = 0.f;
          h = 0.f;
        }
        mg = fmaxf(mg, fabsf(g));
        mh = fmaxf(mh, h);
      }
    }
    block_max2(mg, mh);
  }
  __syncthreads();

  const int nn = (1 << (D + 1)) - 1;
  const uint32_t sst = (uint32_t)__cvta_generic_to_shared(s_stage + warp * SF_STAGE);
  const uint32_t shg = (uint32_t)__cvta_generic_to_shared(hg);
  const int my_off = (lane < F) ? s_off[lane] : 0;
  const bool fact = lane < F && lane != ucol;   // feature side: lane = feature, run-length
  const int uoff = ucol >= 0 ? s_off[ucol] : 0;
  // rows of this warp in identity order
  const int w0 = (int)((int64_t)n * warp / SF_WARPS), w1 = (int)((int64_t)n * (warp + 1) / SF_WARPS);
  // the users code is masked out of the change test (its column goes row-parallel)
  const int uwrd = CW == 1 ? ucol >> 2 : ucol >> 1;
  const uint32_t umask = ucol < 0 ? 0xffffffffu
                                  : CW == 1 ? ~(0xffu << (8 * (ucol & 3))) : ~(0xffffu << (16 * (ucol & 1)));
  auto code_at = [&](const uint8_t* base, int64_t row, int f) -> uint32_t {   // code of (row, f) in global memory
    return CW == 1 ? (uint32_t)base[row * kMaxF + f] : (uint32_t)reinterpret_cast<const uint16_t*>(base)[row * kMaxF + f];
  };

  for (int t = 0; t < T; ++t) {
    // ---- O4: quantise tree t's pairs with its exponents; every row starts at the root
    const double sg = sf_exp2i(K - exp_of(__uint_as_float(s_mg))), sh = sf_exp2i(K - exp_of(__uint_as_float(s_mh)));
    const int eg = exp_of(__uint_as_float(s_mg)), eh = exp_of(__uint_as_float(s_mh));
    for (int i = tid; i < n; i += SF_THREADS) {
      const float w = wv[i];
      float g = __fmul_rn(w, __fsub_rn(s_p[i], yv[2 * i + tg]));
      float h = w;
      if (sf_sampled_out(hp.seed, tg, t, i, hp.subsample)) {
        g = 0.f;
        h = 0.f;
      }
      s_gp[i] = pack_gp(quantize(g, sg), quantize(h, sh));
      s_pos[i] = 0;
    }
    for (int k = tid; k < nn; k += SF_THREADS) {
      s_tf[k] = -2;
      s_tb[k] = 0;
      s_tv[k] = 0.f;
    }
    if (tid == 0) {
      s_ne = 1;
      s_list[0] = 0;
      s_lo[0][0] = -INFINITY;
      s_hi[0][0] = INFINITY;
      // O6 column sample of tree t: the ceil(colsample F) features with the smallest keys (ties by f)
      uint32_t m = 0;
      if (hp.colsample >= 1.0f) {
        m = F >= 32 ? 0xffffffffu : ((1u << F) - 1u);
      } else {
        int nkeep = (int)ceil((double)hp.colsample * (double)F);
        if (nkeep < 1) nkeep = 1;
        for (int f = 0; f < F; ++f) {
          const uint64_t kf = rng4(hp.seed, (uint64_t)(2 * tg + 1), (uint64_t)t, (uint64_t)f);
          int less = 0;
          for (int f2 = 0; f2 < F; ++f2) {
            const uint64_t k2 = rng4(hp.seed, (uint64_t)(2 * tg + 1), (uint64_t)t, (uint64_t)f2);
            less += (k2 < kf || (k2 == kf && f2 < f)) ? 1 : 0;
          }
          if (less < nkeep) m |= 1u << f;
        }
      }
      s_colmask = m;
    }
    __syncthreads();
    const double sgi = sf_exp2i(eg - K), shi = sf_exp2i(eh - K);
    for (int d = 0; d < D; ++d) {
      const int ne = s_ne;
      const int par = d & 1;
      for (int j0 = 0; j0 < ne; j0 += per_pass) {
        const int np = min(per_pass, ne - j0);
        // ---- O5: histograms of the pass's nodes, one walk over the rows in identity order
        for (int k = tid; k < (1 << d); k += SF_THREADS) s_slot[k] = -1;
        for (int i = tid; i < np * 2 * C; i += SF_THREADS) hg[i] = 0u;
        __syncthreads();
        for (int j = tid; j < np; j += SF_THREADS) s_slot[s_list[j0 + j]] = (int16_t)j;
        __syncthreads();
        int cur = -1;          // feature side: cell word index of the pending run (-1: none)
        int32_t acc_g = 0;
        uint32_t acc_h = 0;
        for (int b0 = w0; b0 < w1; b0 += 32) {
          const int i = b0 + lane;
          const bool valid = i < w1;
          uint4 cv[2 * CW];
#pragma unroll
          for (int q = 0; q < 2 * CW; ++q) cv[q] = make_uint4(0u, 0u, 0u, 0u);
          int slot = -1;
          uint32_t gp = 0u;
          if (valid) {
            const uint4* cr = reinterpret_cast<const uint4*>(codes + (size_t)i * SF_ROWB);
#pragma unroll
            for (int q = 0; q < 2 * CW; ++q) cv[q] = __ldg(cr + q);
            const int pk = s_pos[i];
            slot = pk >= 0 ? s_slot[pk] : -1;
            gp = slot >= 0 ? s_gp[i] : 0u;   // rows outside the pass add nothing
          }
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 2 * CW; ++q)
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sst + lane * SF_ROWB + 16 * q), "r"(cv[q].x),
                         "r"(cv[q].y), "r"(cv[q].z), "r"(cv[q].w) : "memory");
          asm volatile("st.shared.s32 [%0], %1;" ::"r"(sst + 32 * SF_ROWB + lane * 4), "r"(slot) : "memory");
          // change test against the previous row of the warp's range (row 0 of a batch: always flagged)
          uint32_t cw[NW];
#pragma unroll
          for (int q = 0; q < 2 * CW; ++q) {
            cw[4 * q] = cv[q].x;
            cw[4 * q + 1] = cv[q].y;
            cw[4 * q + 2] = cv[q].z;
            cw[4 * q + 3] = cv[q].w;
          }
          const int pslot = __shfl_up_sync(0xffffffffu, slot, 1);
          uint32_t dx = 0;
#pragma unroll
          for (int j = 0; j < NW; ++j) dx |= (cw[j] ^ __shfl_up_sync(0xffffffffu, cw[j], 1)) & (j == uwrd ? umask : 0xffffffffu);
          unsigned B = __ballot_sync(0xffffffffu, valid && (lane == 0 || dx != 0u || slot != pslot));
          const int32_t qg = gp_g(gp);
          const uint32_t qh = (uint32_t)gp_h(gp);
          if (ucol >= 0 && slot >= 0) {   // users column, row-parallel
            uint32_t wsel = 0;
#pragma unroll
            for (int j = 0; j < NW; ++j) wsel = j == uwrd ? cw[j] : wsel;
            const uint32_t cu = CW == 1 ? (wsel >> (8 * (ucol & 3))) & 0xffu : (wsel >> (16 * (ucol & 1))) & 0xffffu;
            const uint32_t a = shg + (uint32_t)((slot * 2 * C + uoff + (int)cu) * 4);
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(qg) : "memory");
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a + (uint32_t)C * 4u), "r"(qh) : "memory");
          }
          __syncwarp();
          int32_t bg = 0;
          uint32_t bh = 0;
          while (B) {
            const int r = __ffs(B) - 1;
            B &= B - 1u;
            int sl;
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(sl) : "r"(sst + 32 * SF_ROWB + r * 4));
            uint32_t c;
            if (CW == 1) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(c) : "r"(sst + r * SF_ROWB + lane));
            else asm volatile("ld.shared.u16 %0, [%1];" : "=r"(c) : "r"(sst + r * SF_ROWB + 2 * lane));
            const int32_t vg = (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)(lane < r ? qg : 0));
            const uint32_t vh = __reduce_add_sync(0xffffffffu, lane < r ? qh : 0u);
            const int na = sl >= 0 ? sl * 2 * C + my_off + (int)c : -1;
            if (fact && na != cur) {
              if (cur >= 0) {
                const uint32_t a = shg + (uint32_t)cur * 4u;
                asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(acc_g + (vg - bg)) : "memory");
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a + (uint32_t)C * 4u), "r"(acc_h + (vh - bh)) : "memory");
              }
              acc_g = 0;
              acc_h = 0;
              bg = vg;
              bh = vh;
              cur = na;
            }
          }
          acc_g += (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)qg) - bg;
          acc_h += __reduce_add_sync(0xffffffffu, qh) - bh;
        }
        if (fact && cur >= 0 && (acc_g | (int32_t)acc_h)) {
          const uint32_t a = shg + (uint32_t)cur * 4u;
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(acc_g) : "memory");
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a + (uint32_t)C * 4u), "r"(acc_h) : "memory");
        }
        __syncthreads();
        // ---- O6 per (node, feature pack): one warp evaluates up to four features of one node, lane
        // = bin within a segment of 8, 16 or 32 lanes (segmented scans and argmax); a feature with
        // more than 32 bins gets a warp, lane l owning ceil(nb/32) consecutive bins.  A node's sums fit 32
        // bits (|sum q| <= n 2^K <= 2^27), so prefix sums are 32-bit.
        for (int task = warp; task < np * s_npk; task += SF_WARPS) {
          const int sl = task / s_npk, pk = task % s_npk;
          const int W = s_pkw[pk];
          const bool wide = W > 32;
          const int Wl = wide ? 32 : W;
          const int seg = lane / Wl, bl_ = lane % Wl;
          const int f = s_pkf[pk][seg];
          const int nb = f >= 0 ? s_nc[f] + 1 : 0;
          const int nthr = nb - 1;
          const bool fin = f >= 0 && ((s_colmask >> f) & 1u);
          const int k = s_list[j0 + sl];
          const int32_t* Gs = reinterpret_cast<const int32_t*>(hg) + (size_t)sl * 2 * C + (f >= 0 ? s_off[f] : 0);
          const uint32_t* Hs = hg + (size_t)sl * 2 * C + C + (f >= 0 ? s_off[f] : 0);
          const double lo = s_lo[par][k], hi = s_hi[par][k];
          double bl = -INFINITY;
          int bb = 0x7fffffff;
          int32_t Gq, wGL;
          uint32_t Hq, wHL;
          // one threshold's loss (O6), or -inf when the candidate is invalid
          auto cand = [&](int32_t GLq, uint32_t HLq, double gainP) -> double {
            const double GL = dequant(GLq, sgi), HL = dequant(HLq, shi);
            const double GR = dequant(Gq - GLq, sgi), HR = dequant(Hq - HLq, shi);
            if (!(HL >= hp.mcw && HR >= hp.mcw)) return -INFINITY;
            const double wl = calc_weight(GL, HL, lo, hi, hp.lambda, hp.mcw);
            const double wr = calc_weight(GR, HR, lo, hi, hp.lambda, hp.mcw);
            if (hp.monotone && f == hp.users_col && wl > wr) return -INFINITY;
            return __dsub_rn(__dadd_rn(calc_gain(GL, HL, wl, hp.lambda), calc_gain(GR, HR, wr, hp.lambda)), gainP);
          };
          if (!wide) {   // lane = bin of its segment's feature
            int32_t ig = (bl_ < nb) ? Gs[bl_] : 0;
            uint32_t ih = (bl_ < nb) ? Hs[bl_] : 0u;
            for (int o = 1; o < Wl; o <<= 1) {
              const int32_t ug = __shfl_up_sync(0xffffffffu, ig, o, Wl);
              const uint32_t uh = __shfl_up_sync(0xffffffffu, ih, o, Wl);
              if (bl_ >= o) {
                ig += ug;
                ih += uh;
              }
            }
            Gq = __shfl_sync(0xffffffffu, ig, Wl - 1, Wl);
            Hq = __shfl_sync(0xffffffffu, ih, Wl - 1, Wl);
            // a feature with at most one non-empty bin has every candidate's loss exactly 0
            const int32_t pg = __shfl_up_sync(0xffffffffu, ig, 1, Wl);
            const uint32_t ph = __shfl_up_sync(0xffffffffu, ih, 1, Wl);
            const unsigned ne = __ballot_sync(0xffffffffu, bl_ < nb && (ig != (bl_ ? pg : 0) || ih != (bl_ ? ph : 0u)));
            const unsigned segm = (Wl == 32 ? 0xffffffffu : ((1u << Wl) - 1u)) << (seg * Wl);
            if (fin && bl_ < nthr && __popc(ne & segm) > 1) {
              const double G = dequant(Gq, sgi), H = dequant(Hq, shi);
              const double gainP = calc_gain(G, H, calc_weight(G, H, lo, hi, hp.lambda, hp.mcw), hp.lambda);
              bl = cand(ig, ih, gainP);
              if (bl > -INFINITY) bb = bl_;
            }
            for (int o = Wl >> 1; o > 0; o >>= 1) {
              const double ol = __shfl_down_sync(0xffffffffu, bl, o, Wl);
              const int ob = __shfl_down_sync(0xffffffffu, bb, o, Wl);
              if (ol > bl || (ol == bl && ob < bb)) {
                bl = ol;
                bb = ob;
              }
            }
            bb = __shfl_sync(0xffffffffu, bb, 0, Wl);
            bl = __shfl_sync(0xffffffffu, bl, 0, Wl);
            const int own = bb == 0x7fffffff ? 0 : bb;
            wGL = __shfl_sync(0xffffffffu, ig, own, Wl);
            wHL = __shfl_sync(0xffffffffu, ih, own, Wl);
          } else {          // one feature with nb > 32 bins: lane l owns bins [per l, per (l+1)), per = ceil(nb/32)
            const int per = (nb + 31) >> 5;   // <= 32 (16-bit codes: up to 1024 bins)
            int32_t lg = 0;
            uint32_t lh = 0;
            for (int q = 0; q < per; ++q) {
              const int bq = lane * per + q;
              if (bq < nb) {
                lg += Gs[bq];
                lh += Hs[bq];
              }
            }
            int32_t ig = lg;
            uint32_t ih = lh;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int32_t ug = __shfl_up_sync(0xffffffffu, ig, o);
              const uint32_t uh = __shfl_up_sync(0xffffffffu, ih, o);
              if (lane >= o) {
                ig += ug;
                ih += uh;
              }
            }
            Gq = __shfl_sync(0xffffffffu, ig, 31);
            Hq = __shfl_sync(0xffffffffu, ih, 31);
            int32_t myg = 0;
            uint32_t myh = 0;
            if (fin && lane * per < nthr) {
              const double G = dequant(Gq, sgi), H = dequant(Hq, shi);
              const double gainP = calc_gain(G, H, calc_weight(G, H, lo, hi, hp.lambda, hp.mcw), hp.lambda);
              int32_t rg = ig - lg;    // prefix before the lane's first bin
              uint32_t rh = ih - lh;
              for (int q = 0; q < per; ++q) {
                const int b = lane * per + q;
                if (b >= nthr) break;
                rg += Gs[b];
                rh += Hs[b];
                const double loss = cand(rg, rh, gainP);
                if (loss > bl) {   // b ascending within the lane: strict keeps the smaller b
                  bl = loss;
                  bb = b;
                  myg = rg;
                  myh = rh;
                }
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const double ol = __shfl_down_sync(0xffffffffu, bl, o);
              const int ob = __shfl_down_sync(0xffffffffu, bb, o);
              const int32_t og = __shfl_down_sync(0xffffffffu, myg, o);
              const uint32_t oh = __shfl_down_sync(0xffffffffu, myh, o);
              if (ol > bl || (ol == bl && ob < bb)) {
                bl = ol;
                bb = ob;
                myg = og;
                myh = oh;
              }
            }
            bb = __shfl_sync(0xffffffffu, bb, 0);
            bl = __shfl_sync(0xffffffffu, bl, 0);
            wGL = __shfl_sync(0xffffffffu, myg, 0);
            wHL = __shfl_sync(0xffffffffu, myh, 0);
          }
          if (bl_ == 0 && f >= 0 && (!wide || lane == 0)) {
            SFRes r;
            r.loss = bl;
            r.b = bb;
            r.valid = bl > -INFINITY ? 1 : 0;
            r.GLq = wGL;
            r.HLq = (int64_t)wHL;
            res[sl * kMaxF + f] = r;
            if (f == 0) {   // node totals (every feature's bins sum to them)
              s_tot[sl][0] = Gq;
              s_tot[sl][1] = (long long)Hq;
            }
          }
        }
        __syncthreads();
        // ---- node decisions of the pass: one warp per node, lane = feature (O6 argmax, O7, O8)
        for (int sl = warp; sl < np; sl += SF_WARPS) {
          const int k = s_list[j0 + sl];
          double ml = -INFINITY;
          int mf = lane, mb = 0x7fffffff;
          if (lane < F && ((s_inpk >> lane) & 1u)) {
            const SFRes r = res[sl * kMaxF + lane];
            if (r.valid) {
              ml = r.loss;
              mb = r.b;
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ol = __shfl_down_sync(0xffffffffu, ml, o);
            const int of = __shfl_down_sync(0xffffffffu, mf, o), ob = __shfl_down_sync(0xffffffffu, mb, o);
            if (ol > ml || (ol == ml && (of < mf || (of == mf && ob < mb)))) {
              ml = ol;
              mf = of;
              mb = ob;
            }
          }
          if (lane != 0) continue;
          const double lo = s_lo[par][k], hi = s_hi[par][k];
          const int64_t GqN = s_tot[sl][0], HqN = s_tot[sl][1];
          const double G = dequant(GqN, sgi), H = dequant(HqN, shi);
          const double wP = calc_weight(G, H, lo, hi, hp.lambda, hp.mcw);
          const int gk = (1 << d) - 1 + k;
          if (ml > 1e-6) {
            const int64_t GLs = res[sl * kMaxF + mf].GLq, HLs = res[sl * kMaxF + mf].HLq;
            const double GL = dequant(GLs, sgi), HL = dequant(HLs, shi);
            const double GR = dequant(GqN - GLs, sgi), HR = dequant(HqN - HLs, shi);
            const double wl = calc_weight(GL, HL, lo, hi, hp.lambda, hp.mcw);
            const double wr = calc_weight(GR, HR, lo, hi, hp.lambda, hp.mcw);
            double loL = lo, hiL = hi, loR = lo, hiR = hi;
            if (hp.monotone && mf == hp.users_col) {
              const double mid = __dmul_rn(__dadd_rn(wl, wr), 0.5);
              hiL = mid;
              loR = mid;
            }
            s_sf[k] = (int8_t)mf;
            s_sb[k] = (uint16_t)mb;
            s_tf[gk] = (int8_t)mf;
            s_tb[gk] = (uint16_t)mb;
            if (d + 1 < D) {
              s_lo[par ^ 1][2 * k] = loL;
              s_hi[par ^ 1][2 * k] = hiL;
              s_lo[par ^ 1][2 * k + 1] = loR;
              s_hi[par ^ 1][2 * k + 1] = hiR;
            } else {   // children at max depth are leaves
              s_tf[2 * gk + 1] = -1;
              s_tv[2 * gk + 1] = (float)__dmul_rn(hp.eta, calc_weight(GL, HL, loL, hiL, hp.lambda, hp.mcw));
              s_tf[2 * gk + 2] = -1;
              s_tv[2 * gk + 2] = (float)__dmul_rn(hp.eta, calc_weight(GR, HR, loR, hiR, hp.lambda, hp.mcw));
            }
          } else {
            s_sf[k] = -1;
            s_tf[gk] = -1;
            s_tv[gk] = (float)__dmul_rn(hp.eta, wP);
          }
        }
        __syncthreads();
      }
      // ---- every row of a split node moves to its child; rows of leaves record their leaf
      for (int i = tid; i < n; i += SF_THREADS) {
        const int pk = s_pos[i];
        if (pk < 0) continue;
        const int f = s_sf[pk];
        if (f >= 0) {
          const int child = 2 * pk + (code_at(codes, i, f) > s_sb[pk] ? 1 : 0);
          if (d + 1 == D) {
            s_leaf[i] = (int16_t)((1 << (d + 1)) - 1 + child);
            s_pos[i] = -1;
          } else {
            s_pos[i] = (int16_t)child;
          }
        } else {
          s_leaf[i] = (int16_t)((1 << d) - 1 + pk);
          s_pos[i] = -1;
        }
      }
      if (tid == 0) {   // next level's nodes (ascending)
        int m = 0;
        if (d + 1 < D)
          for (int j = 0; j < s_ne; ++j) {
            const int k = s_list[j];
            if (s_sf[k] >= 0) {
              s_nlist[m++] = (int16_t)(2 * k);
              s_nlist[m++] = (int16_t)(2 * k + 1);
            }
          }
        s_ne_next = m;
      }
      __syncthreads();
      if (tid == 0) s_ne = s_ne_next;
      for (int j = tid; j < s_ne_next; j += SF_THREADS) s_list[j] = s_nlist[j];
      __syncthreads();
      if (s_ne == 0) break;
    }
    // ---- O9: p += v of the row's leaf; tree t+1's gradient maxima.  O10 for the held-out rows.
    if (tid == 0) {
      s_mg = 0u;
      s_mh = 0u;
    }
    __syncthreads();
    {
      float mg = 0.f, mh = 0.f;
      const bool has_next = t + 1 < T;
      for (int i = tid; i < n; i += SF_THREADS) {
        const float pn = __fadd_rn(s_p[i], s_tv[s_leaf[i]]);
        s_p[i] = pn;
        if (has_next) {
          const float w = wv[i];
          float g = __fmul_rn(w, __fsub_rn(pn, yv[2 * i + tg]));
          float h = w;
          if (sf_sampled_out(hp.seed, tg, t + 1, i, hp.subsample)) {
            g = 0.f;
            h = 0.f;
          }
          mg = fmaxf(mg, fabsf(g));
          mh = fmaxf(mh, h);
        }
      }
      block_max2(mg, mh);
    }
    for (int i = tid; i < it.m_test; i += SF_THREADS) {
      int k = 0;
      for (int s2 = 0; s2 < D; ++s2) {
        const int f = s_tf[k];
        if (f >= 0) k = 2 * k + 1 + (code_at(it.codes_test, i, f) > s_tb[k] ? 1 : 0);
      }
      it.pred_test[2 * i + tg] = __fadd_rn(it.pred_test[2 * i + tg], s_tv[k]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
int fit_small_max_rows() { return SF_MAX_N; }

void fit_small_run(Ctx* ctx, const std::vector<SmallFitItem>& items, const std::vector<SmallFitHp>& hps) {
  if (items.empty()) return;
  int n_cap = 1;
  for (const auto& itm : items) {
    LLMP_REQUIRE(itm.n >= 1 && itm.n <= SF_MAX_N, "small fit: n must be in [1, 8192]");
    LLMP_REQUIRE(itm.hp >= 0 && itm.hp < (int)hps.size(), "small fit: bad hparams index");
    LLMP_REQUIRE(itm.cw == 1 || itm.cw == 2, "small fit: codes are 8- or 16-bit");
    n_cap = std::max(n_cap, itm.n);
  }
  for (const auto& h : hps) {
    LLMP_REQUIRE(h.D >= 1 && h.D <= SF_MAX_D, "small fit: max_depth must be in [1, 8]");
    LLMP_REQUIRE(h.F >= 1 && h.F <= kMaxF, "small fit: bad F");
  }
  n_cap = (n_cap + 7) & ~7;
  DevBuf& d_hps = ctx->workspace("sf_hps", hps.size() * sizeof(SmallFitHp));
  LLMP_CUDA(cudaMemcpyAsync(d_hps.p, hps.data(), hps.size() * sizeof(SmallFitHp), cudaMemcpyHostToDevice, ctx->stream));
  // one launch per code width (a template instantiation each)
  for (int cw = 1; cw <= 2; ++cw) {
    std::vector<SmallFitItem> its;
    for (const auto& itm : items)
      if (itm.cw == cw) {
        its.push_back(itm);
        its.back().n_cap = n_cap;
      }
    if (its.empty()) continue;
    const int fixed = 12 * n_cap + SF_WARPS * (cw == 1 ? sf_stage<1>() : sf_stage<2>());
    const int smem = SF_SMEM_CAP;
    LLMP_REQUIRE(fixed + 64 * 1024 <= smem, "small fit: too many rows for shared memory");
    const void* kf = cw == 1 ? (const void*)k_fit_small<1> : (const void*)k_fit_small<2>;
    ensure_smem_attr(kf, smem);
    DevBuf& d_items = ctx->workspace(cw == 1 ? "sf_items1" : "sf_items2", its.size() * sizeof(SmallFitItem));
    LLMP_CUDA(cudaMemcpyAsync(d_items.p, its.data(), its.size() * sizeof(SmallFitItem), cudaMemcpyHostToDevice,
                              ctx->stream));
    double rows = 0;
    for (const auto& itm : its) rows += (double)itm.n * hps[itm.hp].T;
    if (cw == 1)
      LLMP_LAUNCH(ctx, KC_FIT_SMALL, rows, k_fit_small<1>, (int)its.size(), SF_THREADS, smem,
                  d_items.as<SmallFitItem>(), d_hps.as<SmallFitHp>(), smem);
    else
      LLMP_LAUNCH(ctx, KC_FIT_SMALL, rows, k_fit_small<2>, (int)its.size(), SF_THREADS, smem,
                  d_items.as<SmallFitItem>(), d_hps.as<SmallFitHp>(), smem);
  }
}

}  // namespace llmp
