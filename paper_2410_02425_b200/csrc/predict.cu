// predict.cu — batched ensemble predictor and the cheapest-feasible argmin, Eq. (1)-(3)
// (P:L166-183).
//
// Predictor: trees are streamed through shared memory in chunks (node = {thr | leaf value, feat},
// 8 B) while each thread keeps R rows' features in shared memory; a row's prediction is
// base + sum of leaf values in tree order (one fp32 rounding per tree, identical to training).
// Recommendation rows [llm feats | profile feats | u] are assembled on the fly from the two small
// feature tables, never materialised in HBM.
#include <math.h>

#include <algorithm>

#include "internal.cuh"

namespace llmp {

constexpr int PRED_THREADS = 256;
constexpr int PRED_R = 2;                          // rows per thread
constexpr int PRED_ROWS = PRED_THREADS * PRED_R;   // rows per CTA pass
constexpr int XS_STRIDE = kMaxF + 1;               // floats per staged row
constexpr int TREE_SMEM = 32768;                   // bytes of tree nodes per chunk
constexpr int PRED_SMEM = PRED_ROWS * XS_STRIDE * 4 + TREE_SMEM;

struct PredArgs {
  const uint2* nodes;  // [2][T][nn]
  int T, D, nn, F;
  float base0, base1;
  int64_t n;
  // plain rows
  const float* X;
  // assembled rows (recommendation)
  const float* llm_feats;
  const float* prof_feats;
  const int32_t* levels;
  int F_llm, F_prof, n_prof, n_levels;
  float* out;  // n x 2
};

template <bool ASSEMBLE>
__global__ void __launch_bounds__(PRED_THREADS, 2) k_predict(const PredArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  float* xs = reinterpret_cast<float*>(smem);
  uint2* tn = reinterpret_cast<uint2*>(smem + PRED_ROWS * XS_STRIDE * 4);
  const int tid = threadIdx.x;
  const int trees_per_chunk = max(1, TREE_SMEM / (a.nn * 8));
  for (int64_t r0 = (int64_t)blockIdx.x * PRED_ROWS; r0 < a.n; r0 += (int64_t)gridDim.x * PRED_ROWS) {
    // stage rows (coalesced over the row block)
    const int rows = (int)min((int64_t)PRED_ROWS, a.n - r0);
    for (int e = tid; e < rows * a.F; e += PRED_THREADS) {
      const int r = e / a.F, f = e % a.F;
      const int64_t row = r0 + r;
      float x;
      if (!ASSEMBLE) {
        x = a.X[row * a.F + f];
      } else {
        const int64_t per_llm = (int64_t)a.n_prof * a.n_levels;
        const int64_t i = row / per_llm;
        const int g = (int)((row / a.n_levels) % a.n_prof);
        const int lv = (int)(row % a.n_levels);
        if (f < a.F_llm) x = a.llm_feats[i * a.F_llm + f];
        else if (f < a.F_llm + a.F_prof) x = a.prof_feats[(int64_t)g * a.F_prof + (f - a.F_llm)];
        else x = (float)a.levels[lv];
      }
      xs[r * XS_STRIDE + f] = x;
    }
    for (int target = 0; target < 2; ++target) {
      float p[PRED_R];
#pragma unroll
      for (int q = 0; q < PRED_R; ++q) p[q] = target == 0 ? a.base0 : a.base1;
      const uint2* tt = a.nodes + (size_t)target * a.T * a.nn;
      for (int c0 = 0; c0 < a.T; c0 += trees_per_chunk) {
        const int nt = min(trees_per_chunk, a.T - c0);
        __syncthreads();
        const uint2* src = tt + (size_t)c0 * a.nn;   // 8-byte aligned (T * nn may be odd)
        for (int e = tid; e < nt * a.nn; e += PRED_THREADS) tn[e] = __ldg(src + e);
        __syncthreads();
        for (int k = 0; k < nt; ++k) {
          const uint2* tree = tn + k * a.nn;
#pragma unroll
          for (int q = 0; q < PRED_R; ++q) {
            const float* x = xs + (tid + q * PRED_THREADS) * XS_STRIDE;
            int node = 0;
            for (int s = 0; s < a.D; ++s) {   // fixed depth (see upload_model_nodes)
              const uint2 nd = tree[node];
              node = 2 * node + 1 + (x[nd.y] < __uint_as_float(nd.x) ? 0 : 1);  // x < thr goes left
            }
            p[q] = __fadd_rn(p[q], __uint_as_float(tree[node].x));
          }
        }
      }
#pragma unroll
      for (int q = 0; q < PRED_R; ++q) {
        const int r = tid + q * PRED_THREADS;
        if (r < rows) a.out[(r0 + r) * 2 + target] = p[q];
      }
    }
    __syncthreads();
  }
}

// Device node table: every tree as a fixed-depth complete tree, so the predictor descends exactly D
// levels with no leaf test.  Slots above depth D: a split {thr, f}, or — for a leaf and everything
// below it — {+inf, 0}: x < +inf always holds (X is finite), so the row keeps going left.  A leaf k at
// depth d < D is therefore reached at its leftmost depth-D descendant (k+1)·2^(D-d) - 1, which holds
// k's value; a depth-D leaf holds its own.  Same leaf, same value, same fp32 add as the plain walk.
void upload_model_nodes(Ctx* ctx, ModelData& m) {
  const size_t tot = (size_t)2 * m.T * m.nn;
  const int n_int = (m.nn - 1) / 2;
  std::vector<uint2> h(std::max<size_t>(tot, 1));
  const float inf = INFINITY;
  uint32_t inf_bits;
  memcpy(&inf_bits, &inf, 4);
  for (size_t tr = 0; tr * m.nn < tot; ++tr) {
    const size_t o = tr * m.nn;
    for (int k = 0; k < m.nn; ++k) h[o + k] = make_uint2(k < n_int ? inf_bits : 0u, k < n_int ? 0u : 0xffffffffu);
    for (int k = 0; k < m.nn; ++k) {
      const int f = m.feat[o + k];
      if (f >= 0) {
        uint32_t bits;
        memcpy(&bits, &m.thr[o + k], 4);
        h[o + k] = make_uint2(bits, (uint32_t)f);
      } else if (f == -1) {
        int dl = 0;
        while (((2 << dl) - 1) <= k) ++dl;   // depth of slot k
        const int leaf = ((k + 1) << (m.D - dl)) - 1;
        uint32_t bits;
        memcpy(&bits, &m.val[o + k], 4);
        h[o + leaf] = make_uint2(bits, 0xffffffffu);
      }
    }
  }
  m.d_nodes.set_stream(ctx->stream);
  m.d_base.set_stream(ctx->stream);
  m.d_nodes.ensure(h.size() * 8);
  LLMP_CUDA(cudaMemcpyAsync(m.d_nodes.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  m.d_base.ensure(8);
  LLMP_CUDA(cudaMemcpyAsync(m.d_base.p, m.base, 8, cudaMemcpyHostToDevice, ctx->stream));
  LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
}

static void launch_predict(Ctx* ctx, const PredArgs& a, bool assemble, int cls) {
  static bool attr = false;
  if (!attr) {
    LLMP_CUDA(cudaFuncSetAttribute(k_predict<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, PRED_SMEM));
    LLMP_CUDA(cudaFuncSetAttribute(k_predict<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, PRED_SMEM));
    attr = true;
  }
  int64_t blocks = (a.n + PRED_ROWS - 1) / PRED_ROWS;
  int grid = (int)std::min<int64_t>(std::max<int64_t>(blocks, 1), (int64_t)ctx->sms * 2);
  if (assemble) LLMP_LAUNCH(ctx, cls, a.n, k_predict<true>, grid, PRED_THREADS, PRED_SMEM, a);
  else LLMP_LAUNCH(ctx, cls, a.n, k_predict<false>, grid, PRED_THREADS, PRED_SMEM, a);
}

void predict_impl(Ctx* ctx, const ModelData& m, const float* X, int64_t n, float* out) {
  if (n == 0) return;
  PredArgs a{};
  a.nodes = m.d_nodes.as<uint2>();
  a.T = m.T;
  a.D = m.D;
  a.nn = m.nn;
  a.F = m.F;
  a.base0 = m.base[0];
  a.base1 = m.base[1];
  a.n = n;
  a.X = X;
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
  DevBuf& d_lv = ctx->workspace("rec_levels", (size_t)n_levels * 4);
  LLMP_CUDA(cudaMemcpyAsync(d_lv.p, levels, (size_t)n_levels * 4, cudaMemcpyHostToDevice, ctx->stream));
  PredArgs a{};
  a.nodes = m.d_nodes.as<uint2>();
  a.T = m.T;
  a.D = m.D;
  a.nn = m.nn;
  a.F = m.F;
  a.base0 = m.base[0];
  a.base1 = m.base[1];
  a.n = n;
  a.llm_feats = llm_feats;
  a.prof_feats = prof_feats;
  a.levels = d_lv.as<int32_t>();
  a.F_llm = F_llm;
  a.F_prof = F_prof;
  a.n_prof = n_prof;
  a.n_levels = n_levels;
  a.out = pred;
  if (n > 0) launch_predict(ctx, a, true, KC_PREDICT);
  argmin_impl(ctx, pred, n_llm, n_prof, n_levels, levels, cost, allowed, L1, L2, U, out);
}

}  // namespace llmp
