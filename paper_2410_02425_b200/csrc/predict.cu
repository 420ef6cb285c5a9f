// predict.cu — batched ensemble predictor and the cheapest-feasible argmin, Eq. (1)-(3)
// (P:L166-183).
//
// Predictor on bin codes: routing a row by `x_f < cuts_f[b]` is identical to `code_f(x) <= b`
// (O2/O10, R15), so rows are binned once with the model's cuts (32 code bytes per row)
// and the trees are walked on codes.  A CTA stages 1024 rows' codes in shared memory (36-byte
// stride: conflict-free) and streams the trees through shared memory in 32 KB chunks of compact
// fixed-depth routing tables (u16 node word f | b << 8, padded leaf subtrees route left on b = 255;
// then the 2^D leaf values at the leftmost-descendant slots), 4 rows per thread.  A row's prediction
// is base + the leaf values in tree order (one fp32 rounding per tree, identical to training).
// Recommendation rows [llm feats | profile feats | u] are assembled from the three small code tables
// of the LLM features, the profile features and the user levels, never materialised in HBM.
#include <math.h>

#include <algorithm>

#include "internal.cuh"

namespace llmp {

constexpr int PC_THREADS = 256;
constexpr int PC_RSTRIDE = 36;                     // bytes per staged row (9 words: distinct banks per lane)
constexpr int PC_TREE_SMEM = 32768;                // bytes of routing tables per chunk
// PC_R rows per thread (independent tree walks), PC_THREADS * PC_R rows per CTA pass
__host__ __device__ constexpr int pc_smem(int R) { return PC_THREADS * R * PC_RSTRIDE + PC_TREE_SMEM; }

__host__ __device__ inline int rtab_inner_bytes(int D) { return ((((1 << D) - 1) * 2) + 3) / 4 * 4; }
__host__ __device__ inline int rtab_bytes(int D) { return rtab_inner_bytes(D) + (4 << D); }

struct PredArgs {
  const uint8_t* rtab;  // [2][T] routing tables of rtab_bytes(D) each
  int T, D;
  float base0, base1;
  int64_t n;
  const uint8_t* codes;        // plain rows: n x 32 codes
  const uint8_t* llm_codes;    // assembled rows: n_llm x F_llm, n_prof x F_prof, n_levels codes
  const uint8_t* prof_codes;
  const uint8_t* level_codes;
  int F_llm, F_prof, n_prof, n_levels, users_col;
  float* out;  // n x 2
};

template <bool ASSEMBLE, int PC_R, int DC>   // DC: compile-time depth (0 = a.D)
__global__ void __launch_bounds__(PC_THREADS) k_predict(const PredArgs a) {
  constexpr int PC_ROWS = PC_THREADS * PC_R;
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* rows = smem;
  uint8_t* tabs = smem + PC_ROWS * PC_RSTRIDE;
  const int tid = threadIdx.x;
  const int tb = rtab_bytes(a.D), tin = rtab_inner_bytes(a.D);
  const int n_int = (1 << a.D) - 1;
  const int trees_per_chunk = max(1, PC_TREE_SMEM / tb);
  for (int64_t r0 = (int64_t)blockIdx.x * PC_ROWS; r0 < a.n; r0 += (int64_t)gridDim.x * PC_ROWS) {
    const int nr = (int)min((int64_t)PC_ROWS, a.n - r0);
    __syncthreads();   // previous pass done with the staged rows
    if (!ASSEMBLE) {   // 8 words per row, coalesced
      const uint32_t* src = reinterpret_cast<const uint32_t*>(a.codes + r0 * kMaxF);
      for (int e = tid; e < nr * 8; e += PC_THREADS)
        *reinterpret_cast<uint32_t*>(rows + (e >> 3) * PC_RSTRIDE + (e & 7) * 4) = __ldg(src + e);
    } else {
      const int64_t per_llm = (int64_t)a.n_prof * a.n_levels;
      for (int e = tid; e < nr * kMaxF; e += PC_THREADS) {
        const int r = e >> 5, f = e & 31;
        const int64_t row = r0 + r;
        const int64_t i = row / per_llm;
        const int g = (int)((row / a.n_levels) % a.n_prof);
        const int lv = (int)(row % a.n_levels);
        uint8_t c = 0;
        if (f < a.F_llm) c = a.llm_codes[i * a.F_llm + f];
        else if (f < a.F_llm + a.F_prof) c = a.prof_codes[(int64_t)g * a.F_prof + (f - a.F_llm)];
        else if (f == a.users_col) c = a.level_codes[lv];
        rows[r * PC_RSTRIDE + f] = c;
      }
    }
    for (int target = 0; target < 2; ++target) {
      float p[PC_R];
#pragma unroll
      for (int q = 0; q < PC_R; ++q) p[q] = target == 0 ? a.base0 : a.base1;
      const uint8_t* tt = a.rtab + (size_t)target * a.T * tb;
      for (int c0 = 0; c0 < a.T; c0 += trees_per_chunk) {
        const int nt = min(trees_per_chunk, a.T - c0);
        __syncthreads();
        const uint4* src = reinterpret_cast<const uint4*>(tt + (size_t)c0 * tb);   // tb is a multiple of 16 for D >= 2
        if ((tb & 15) == 0) {
          for (int e = tid; e < nt * tb / 16; e += PC_THREADS) reinterpret_cast<uint4*>(tabs)[e] = __ldg(src + e);
        } else {
          const uint32_t* s4 = reinterpret_cast<const uint32_t*>(tt + (size_t)c0 * tb);
          for (int e = tid; e < nt * tb / 4; e += PC_THREADS) reinterpret_cast<uint32_t*>(tabs)[e] = __ldg(s4 + e);
        }
        __syncthreads();
        for (int k = 0; k < nt; ++k) {
          const uint16_t* inode = reinterpret_cast<const uint16_t*>(tabs + k * tb);
          const float* lval = reinterpret_cast<const float*>(tabs + k * tb + tin);
          int node[PC_R];
#pragma unroll
          for (int q = 0; q < PC_R; ++q) node[q] = 0;
#pragma unroll
          for (int s = 0; s < (DC ? DC : a.D); ++s) {   // fixed depth; the PC_R walks are independent
#pragma unroll
            for (int q = 0; q < PC_R; ++q) {
              const uint32_t w = inode[node[q]];
              const uint32_t c = rows[(tid + q * PC_THREADS) * PC_RSTRIDE + (w & 0xffu)];
              node[q] = 2 * node[q] + 1 + (c > (w >> 8) ? 1 : 0);   // code <= b  <=>  x < cuts_f[b]: left
            }
          }
#pragma unroll
          for (int q = 0; q < PC_R; ++q) p[q] = __fadd_rn(p[q], lval[node[q] - n_int]);
        }
      }
#pragma unroll
      for (int q = 0; q < PC_R; ++q) {
        const int r = tid + q * PC_THREADS;
        if (r < nr) a.out[(r0 + r) * 2 + target] = p[q];
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Recommendation grid predictor: the rows of a sweep are the Cartesian product
// (LLM i) x (profile g) x (user level lv), and within one (i, g) pair only the users column varies.
// The user levels are strictly increasing (the API requires it), so their codes are non-decreasing
// and a split "users code <= b" sends exactly the levels lv < t_b left, t_b = #{lv : code_lv <= b}:
// the levels that reach any node form a contiguous range.  One thread per (pair, ensemble) walks
// each tree once per distinct leaf: starting from the lowest level not yet placed, lo, it descends
// with the range [lo, hi) (a split on another feature sends the whole range the pair's way; a users
// split narrows hi to t_b when lo < t_b and goes left, else goes right), adds the leaf value to
// levels lo .. hi-1 and continues from lo = hi.  Every row still gets base + its leaf values in tree
// order with one fp32 rounding per tree: the same bits as k_predict.
#ifndef LLMP_PG_THREADS
#define LLMP_PG_THREADS 128
#endif
#ifndef LLMP_PG_TREE_SMEM
#define LLMP_PG_TREE_SMEM 16384
#endif
constexpr int PG_THREADS = LLMP_PG_THREADS;
constexpr int PG_TREE_SMEM = LLMP_PG_TREE_SMEM;
__host__ __device__ constexpr int pg_smem(int nl) {
  return PG_THREADS * PC_RSTRIDE + 256 + nl * PG_THREADS * 4 + PG_TREE_SMEM;
}

template <int DC>
__global__ void __launch_bounds__(PG_THREADS) k_predict_grid(const PredArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* rows = smem;                                     // the pairs' codes
  uint8_t* lvt = smem + PG_THREADS * PC_RSTRIDE;            // [256] t_b = #{lv : code_lv <= b}
  float* acc = reinterpret_cast<float*>(lvt + 256);         // [n_levels][PG_THREADS]
  const int NL = a.n_levels;
  uint8_t* tabs = reinterpret_cast<uint8_t*>(acc + NL * PG_THREADS);
  const int tid = threadIdx.x, target = blockIdx.y;
  const int D = DC ? DC : a.D;
  const int tb = rtab_bytes(a.D), tin = rtab_inner_bytes(a.D);
  const int n_int = (1 << a.D) - 1;
  const int trees_per_chunk = max(1, PG_TREE_SMEM / tb);
  const int ucol = a.users_col;
  for (int b = tid; b < 256; b += PG_THREADS) {
    int t = 0;
    for (int lv = 0; lv < NL; ++lv) t += a.level_codes[lv] <= b ? 1 : 0;
    lvt[b] = (uint8_t)t;
  }
  const int64_t npairs = a.n / NL;
  const int FP = a.F_llm + a.F_prof;
  const float base = target ? a.base1 : a.base0;
  const uint8_t* tt = a.rtab + (size_t)target * a.T * tb;
  for (int64_t p0 = (int64_t)blockIdx.x * PG_THREADS; p0 < npairs; p0 += (int64_t)gridDim.x * PG_THREADS) {
    const int np = (int)min((int64_t)PG_THREADS, npairs - p0);
    __syncthreads();   // previous pass done with the staged pairs and the accumulators
    for (int e = tid; e < np * FP; e += PG_THREADS) {   // LLM features, then profile features
      const int r = e / FP, f = e - r * FP;
      const int64_t pr = p0 + r;
      const int64_t i = pr / a.n_prof;
      const int g = (int)(pr - i * a.n_prof);
      rows[r * PC_RSTRIDE + f] =
          f < a.F_llm ? a.llm_codes[i * a.F_llm + f] : a.prof_codes[(int64_t)g * a.F_prof + (f - a.F_llm)];
    }
    for (int lv = 0; lv < NL; ++lv) acc[lv * PG_THREADS + tid] = base;
    const uint8_t* myrow = rows + tid * PC_RSTRIDE;
    float* myacc = acc + tid;
    for (int c0 = 0; c0 < a.T; c0 += trees_per_chunk) {
      const int nt = min(trees_per_chunk, a.T - c0);
      __syncthreads();
      if ((tb & 15) == 0) {
        const uint4* src = reinterpret_cast<const uint4*>(tt + (size_t)c0 * tb);
        for (int e = tid; e < nt * tb / 16; e += PG_THREADS) reinterpret_cast<uint4*>(tabs)[e] = __ldg(src + e);
      } else {
        const uint32_t* s4 = reinterpret_cast<const uint32_t*>(tt + (size_t)c0 * tb);
        for (int e = tid; e < nt * tb / 4; e += PG_THREADS) reinterpret_cast<uint32_t*>(tabs)[e] = __ldg(s4 + e);
      }
      __syncthreads();
      if (tid < np) {
        for (int kk = 0; kk < nt; ++kk) {
          const uint16_t* inode = reinterpret_cast<const uint16_t*>(tabs + kk * tb);
          const float* lval = reinterpret_cast<const float*>(tabs + kk * tb + tin);
          int lo = 0;
          do {   // one descent per distinct leaf, levels in increasing order
            int hi = NL, k = 0;
#pragma unroll
            for (int s2 = 0; s2 < (DC ? DC : kMaxDepth); ++s2)
              if (DC || s2 < D) {
                // branch-free: every split is "levels below t go left" — t = t_b on the users column,
                // else NL (the pair's code <= b: the whole range left) or 0 (all right)
                const uint32_t w = inode[k];
                const uint32_t f = w & 0xffu, b = w >> 8;
                const int tu = lvt[b];
                const int tc = (uint32_t)myrow[f] <= b ? NL : 0;
                const int t = (int)f == ucol ? tu : tc;
                const bool right = lo >= t;
                hi = right ? hi : min(hi, t);
                k = 2 * k + 1 + (right ? 1 : 0);
              }
            const float v = lval[k - n_int];
            for (int lv = lo; lv < hi; ++lv) myacc[lv * PG_THREADS] = __fadd_rn(myacc[lv * PG_THREADS], v);
            lo = hi;
          } while (lo < NL);
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < np * NL; e += PG_THREADS) {   // row (p0 + r) * NL + lv, rows consecutive
      const int r = e / NL, lv = e - r * NL;
      a.out[((p0 + r) * NL + lv) * 2 + target] = acc[lv * PG_THREADS + r];
    }
  }
}

// Device routing tables (see the header comment): per tree the 2^D - 1 node words of the slots above
// depth D — a split {f, b}, or {0, 255} ("always left") for a leaf and everything below it — then
// the 2^D leaf values: a leaf k at depth d < D is reached at its leftmost depth-D descendant
// (k+1)·2^(D-d) - 1.  Same leaf, same value, same fp32 add as walking the tree on raw x.
void upload_model_nodes(Ctx* ctx, ModelData& m) {
  const int D = m.D, n_int = (1 << D) - 1;
  const size_t tb = (size_t)rtab_bytes(D), tin = (size_t)rtab_inner_bytes(D);
  const size_t ntrees = (size_t)2 * m.T;
  std::vector<uint8_t> h(std::max<size_t>(ntrees * tb, 16), 0);
  for (size_t tr = 0; tr < ntrees; ++tr) {
    uint16_t* inode = reinterpret_cast<uint16_t*>(h.data() + tr * tb);
    float* lval = reinterpret_cast<float*>(h.data() + tr * tb + tin);
    const size_t o = tr * m.nn;
    for (int k = 0; k < n_int; ++k) inode[k] = (uint16_t)(255u << 8);
    for (int k = 0; k < m.nn; ++k) {
      const int f = m.feat[o + k];
      if (f >= 0) {
        inode[k] = (uint16_t)((uint32_t)f | ((uint32_t)(m.bin[o + k] & 0xff) << 8));
      } else if (f == -1) {
        int dl = 0;
        while (((2 << dl) - 1) <= k) ++dl;   // depth of slot k
        lval[((k + 1) << (D - dl)) - 1 - n_int] = m.val[o + k];
      }
    }
  }
  m.d_nodes.set_stream(ctx->stream);
  m.d_base.set_stream(ctx->stream);
  m.d_nodes.ensure(h.size());
  LLMP_CUDA(cudaMemcpyAsync(m.d_nodes.p, h.data(), h.size(), cudaMemcpyHostToDevice, ctx->stream));
  m.d_base.ensure(8);
  LLMP_CUDA(cudaMemcpyAsync(m.d_base.p, m.base, 8, cudaMemcpyHostToDevice, ctx->stream));
  LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
}

template <int R, int DC>
static void launch_predict_r(Ctx* ctx, const PredArgs& a, bool assemble, int cls) {
  ensure_smem_attr((const void*)k_predict<false, R, DC>, pc_smem(R));
  ensure_smem_attr((const void*)k_predict<true, R, DC>, pc_smem(R));
  const int64_t rows = (int64_t)PC_THREADS * R;
  const int per_sm = std::max(1, (int)(220000 / (pc_smem(R) + 1024)));
  int grid = (int)std::min<int64_t>(std::max<int64_t>((a.n + rows - 1) / rows, 1), (int64_t)ctx->sms * per_sm);
  if (assemble) LLMP_LAUNCH(ctx, cls, a.n, (k_predict<true, R, DC>), grid, PC_THREADS, pc_smem(R), a);
  else LLMP_LAUNCH(ctx, cls, a.n, (k_predict<false, R, DC>), grid, PC_THREADS, pc_smem(R), a);
}
// 4 rows per thread: 188.6 M rows/s on the bench sweep vs 177.6 (2) and 145.8 (8; tools/ab_predict.py);
// compile-time depth for the configs' depths (6, 8)
static void launch_predict(Ctx* ctx, const PredArgs& a, bool assemble, int cls) {
  static const bool dct = !(getenv("LLMP_PRED_DC") && atoi(getenv("LLMP_PRED_DC")) == 0);
  if (dct && a.D == 8) launch_predict_r<4, 8>(ctx, a, assemble, cls);
  else if (dct && a.D == 6) launch_predict_r<4, 6>(ctx, a, assemble, cls);
  else launch_predict_r<4, 0>(ctx, a, assemble, cls);
}

template <int DC>
static void launch_predict_grid_d(Ctx* ctx, const PredArgs& a, int64_t npairs) {
  ensure_smem_attr((const void*)k_predict_grid<DC>, pg_smem(64));
  const int smem = pg_smem(a.n_levels);
  const int per_sm = std::max(1, (int)(220000 / (smem + 1024)));
  const int gx = (int)std::min<int64_t>(std::max<int64_t>((npairs + PG_THREADS - 1) / PG_THREADS, 1),
                                        (int64_t)ctx->sms * per_sm);
  LLMP_LAUNCH(ctx, KC_PREDICT, a.n, k_predict_grid<DC>, dim3(gx, 2), PG_THREADS, smem, a);
}
static void launch_predict_grid(Ctx* ctx, const PredArgs& a, int64_t npairs) {
  if (a.D == 8) launch_predict_grid_d<8>(ctx, a, npairs);
  else if (a.D == 6) launch_predict_grid_d<6>(ctx, a, npairs);
  else launch_predict_grid_d<0>(ctx, a, npairs);
}

// codes of a small table whose columns are the model's features col0 .. col0 + ncols - 1
__global__ void k_table_codes(const float* t, int64_t nrows, int ncols, int col0, const float* cuts,
                              const int32_t* ncuts, uint8_t* out, int* flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nrows * ncols; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % ncols), f = col0 + c;
    const float x = t[e];
    if (!isfinite(x)) atomicExch(flag, 1);
    const float* cf = cuts + (size_t)f * (kBins - 1);
    int lo = 0, hi = ncuts[f];   // number of cuts <= x
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cf[mid] <= x) lo = mid + 1;
      else hi = mid;
    }
    out[e] = (uint8_t)lo;
  }
}

static void check_flag(Ctx* ctx, DevBuf& flag, const char* what) {
  int h = 0;
  LLMP_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
  LLMP_REQUIRE(h == 0, what);
}

void predict_impl(Ctx* ctx, const ModelData& m, const float* X, int64_t n, float* out) {
  if (n == 0) return;
  DevBuf& codes = ctx->workspace("pred_codes", (size_t)n * kMaxF);
  DevBuf& flag = ctx->workspace("pred_flag", sizeof(int));
  LLMP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
  compute_codes(ctx, X, n, m.F, m.cuts, codes.as<uint8_t>(), nullptr, n, flag.as<int>());
  check_flag(ctx, flag, "X holds a non-finite value");
  PredArgs a{};
  a.rtab = m.d_nodes.as<uint8_t>();
  a.T = m.T;
  a.D = m.D;
  a.base0 = m.base[0];
  a.base1 = m.base[1];
  a.n = n;
  a.codes = codes.as<uint8_t>();
  a.out = out;
  launch_predict(ctx, a, false, KC_PREDICT);
}

// ---------------------------------------------------------------------------------------------
// Eq. (3): u_max = largest level whose whole prefix meets both constraints; Eq. (2): n =
// ceil(U / u_max); Eq. (1): argmin n * c(G), ties -> lowest profile index.  One thread per LLM.
__global__ void k_argmin(const float* pred, int n_llm, int n_prof, int n_levels, const int32_t* levels,
                         const double* cost, const uint8_t* allowed, float L1, float L2, int64_t U, int32_t* o_prof,
                         int64_t* o_npods, double* o_cost, int32_t* o_umax) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_llm) return;
  int best_g = -1;
  int64_t best_n = 0;
  double best_c = INFINITY;
  int best_u = 0;
  for (int g = 0; g < n_prof; ++g) {
    if (allowed && !allowed[(int64_t)i * n_prof + g]) continue;
    const float* pr = pred + ((int64_t)i * n_prof + g) * n_levels * 2;
    int um = 0;
    for (int k = 0; k < n_levels; ++k) {
      if (!(pr[2 * k] <= L1 && pr[2 * k + 1] <= L2)) break;
      um = levels[k];
    }
    if (um <= 0) continue;
    const int64_t npods = (U + um - 1) / um;
    const double c = __dmul_rn((double)npods, cost[g]);
    if (c < best_c) {
      best_g = g;
      best_n = npods;
      best_c = c;
      best_u = um;
    }
  }
  o_prof[i] = best_g;
  o_npods[i] = best_n;
  o_cost[i] = best_c;
  o_umax[i] = best_u;
}

void argmin_impl(Ctx* ctx, const float* pred, int n_llm, int n_prof, int n_levels, const int32_t* levels_host,
                 const double* cost_host, const uint8_t* allowed_host, float L1, float L2, int64_t U, RecOut& out) {
  cudaStream_t s = ctx->stream;
  DevBuf& d_lv = ctx->workspace("am_levels", (size_t)n_levels * 4);
  DevBuf& d_cost = ctx->workspace("am_cost", (size_t)n_prof * 8);
  DevBuf& d_al = ctx->workspace("am_allowed", allowed_host ? (size_t)n_llm * n_prof : 1);
  LLMP_CUDA(cudaMemcpyAsync(d_lv.p, levels_host, (size_t)n_levels * 4, cudaMemcpyHostToDevice, s));
  LLMP_CUDA(cudaMemcpyAsync(d_cost.p, cost_host, (size_t)n_prof * 8, cudaMemcpyHostToDevice, s));
  if (allowed_host)
    LLMP_CUDA(cudaMemcpyAsync(d_al.p, allowed_host, (size_t)n_llm * n_prof, cudaMemcpyHostToDevice, s));
  DevBuf& d_o = ctx->workspace("am_out", (size_t)n_llm * (4 + 8 + 8 + 4));
  int32_t* o_prof = d_o.as<int32_t>();
  int32_t* o_umax = o_prof + n_llm;
  int64_t* o_npods = reinterpret_cast<int64_t*>(d_o.as<uint8_t>() + (size_t)n_llm * 8);
  double* o_cost = reinterpret_cast<double*>(o_npods + n_llm);
  LLMP_LAUNCH(ctx, KC_RECOMMEND, n_llm, k_argmin, (n_llm + 127) / 128, 128, 0, pred, n_llm, n_prof, n_levels,
              d_lv.as<int32_t>(), d_cost.as<double>(), allowed_host ? d_al.as<uint8_t>() : nullptr, L1, L2, U, o_prof,
              o_npods, o_cost, o_umax);
  out.profile.resize(n_llm);
  out.u_max.resize(n_llm);
  out.n_pods.resize(n_llm);
  out.cost.resize(n_llm);
  LLMP_CUDA(cudaMemcpyAsync(out.profile.data(), o_prof, (size_t)n_llm * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(out.u_max.data(), o_umax, (size_t)n_llm * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(out.n_pods.data(), o_npods, (size_t)n_llm * 8, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(out.cost.data(), o_cost, (size_t)n_llm * 8, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaStreamSynchronize(s));
}

void recommend_impl(Ctx* ctx, const ModelData& m, const float* llm_feats, int n_llm, int F_llm,
                    const float* prof_feats, int n_prof, int F_prof, const double* cost, const uint8_t* allowed,
                    const int32_t* levels, int n_levels, float L1, float L2, int64_t U, RecOut& out,
                    float* pred_out_dev) {
  const int64_t n = (int64_t)n_llm * n_prof * n_levels;
  float* pred = pred_out_dev ? pred_out_dev
                             : ctx->workspace("rec_pred", (size_t)std::max<int64_t>(n, 1) * 8).as<float>();
  // codes of the three small tables (columns: LLM features, then profile features, then users)
  LLMP_REQUIRE(F_llm + F_prof + 1 == m.F && m.users_col == F_llm + F_prof, "feature layout does not match the model");
  DevBuf& c_llm = ctx->workspace("rec_c_llm", std::max<size_t>((size_t)n_llm * F_llm, 1));
  DevBuf& c_prof = ctx->workspace("rec_c_prof", std::max<size_t>((size_t)n_prof * F_prof, 1));
  DevBuf& c_lv = ctx->workspace("rec_c_lv", std::max<size_t>((size_t)n_levels, 1));
  DevBuf& d_lvf = ctx->workspace("rec_levels_f", (size_t)n_levels * 4);
  DevBuf& flag = ctx->workspace("pred_flag", sizeof(int));
  std::vector<float> lvf(levels, levels + n_levels);
  LLMP_CUDA(cudaMemcpyAsync(d_lvf.p, lvf.data(), (size_t)n_levels * 4, cudaMemcpyHostToDevice, ctx->stream));
  LLMP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
  const float* cuts = m.cuts.d_cuts.as<float>();
  const int32_t* ncuts = m.cuts.d_ncuts.as<int32_t>();
  if ((int64_t)n_llm * F_llm > 0)
    LLMP_LAUNCH(ctx, KC_RECOMMEND, 0, k_table_codes, 64, 256, 0, llm_feats, (int64_t)n_llm, F_llm, 0, cuts, ncuts,
                c_llm.as<uint8_t>(), flag.as<int>());
  if ((int64_t)n_prof * F_prof > 0)
    LLMP_LAUNCH(ctx, KC_RECOMMEND, 0, k_table_codes, 64, 256, 0, prof_feats, (int64_t)n_prof, F_prof, F_llm, cuts, ncuts,
                c_prof.as<uint8_t>(), flag.as<int>());
  LLMP_LAUNCH(ctx, KC_RECOMMEND, 0, k_table_codes, 1, 256, 0, d_lvf.as<float>(), (int64_t)n_levels, 1, m.users_col, cuts,
              ncuts, c_lv.as<uint8_t>(), flag.as<int>());
  // a caller's device pred_out must not be written on bad input: check before predicting; otherwise the
  // check rides on argmin's final synchronisation (one host round trip less; no output leaves on error)
  const bool early_check = pred_out_dev != nullptr;
  if (early_check) check_flag(ctx, flag, "feature tables hold a non-finite value");
  PredArgs a{};
  a.rtab = m.d_nodes.as<uint8_t>();
  a.T = m.T;
  a.D = m.D;
  a.base0 = m.base[0];
  a.base1 = m.base[1];
  a.n = n;
  a.llm_codes = c_llm.as<uint8_t>();
  a.prof_codes = c_prof.as<uint8_t>();
  a.level_codes = c_lv.as<uint8_t>();
  a.F_llm = F_llm;
  a.F_prof = F_prof;
  a.n_prof = n_prof;
  a.n_levels = n_levels;
  a.users_col = m.users_col;
  a.out = pred;
  // the grid predictor (tree walks per (LLM, profile) pair, one per distinct leaf) for up to 64 user
  // levels; LLMP_PRED_GRID=0 keeps the per-row walk
  static const bool grid_env = !(getenv("LLMP_PRED_GRID") && atoi(getenv("LLMP_PRED_GRID")) == 0);
  if (n > 0 && grid_env && n_levels <= 64) launch_predict_grid(ctx, a, (int64_t)n_llm * n_prof);
  else if (n > 0) launch_predict(ctx, a, true, KC_PREDICT);
  argmin_impl(ctx, pred, n_llm, n_prof, n_levels, levels, cost, allowed, L1, L2, U, out);
  if (!early_check) check_flag(ctx, flag, "feature tables hold a non-finite value");
}

}  // namespace llmp
