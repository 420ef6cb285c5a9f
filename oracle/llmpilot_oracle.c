/* oracle/llmpilot_oracle.c — TEST INFRASTRUCTURE ONLY (see llmpilot_oracle.h).
 *
 * A plain, slow, single-threaded CPU implementation of what the LLM-Pilot hot path computes,
 * written step by step from SURVEY.md §8(c) O1-O12 and the paper (PAPER.md, "P:L<n>").
 * No blocking, fusion or reordering: every node histogram is built directly from its rows,
 * every split candidate is enumerated, every tree is grown level by level.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -msse2 -mfpmath=sse -fPIC -shared
 *        -o oracle/liboracle.so oracle/llmpilot_oracle.c -lm
 * (-ffp-contract=off: no FMA contraction, so every fp operation rounds once, as written.)
 */
#include "llmpilot_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* counter-based generator: splitmix64 finaliser            */
static uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t orc_rng4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return sm64(sm64(sm64(sm64(seed) ^ a) ^ b) ^ c);
}

/* ------------------------------------------------------------------------------------------ */
/* O1 — Eq. (4), P:L192-197:
 *   w_t(M,G,u) = 1 - |l_t(M,G,u) - L_t| / max_{v in U} |l_t(M,G,v) - L_t|,   t in {1,2}
 *   w = (w_1 + w_2) / 2   ("We combine both weights using arithmetic mean")
 * Group = (llm_id, profile_id).  Zero denominator => weight 1 (reading R6).      */
/* Poisson(1) by inversion (DESIGN R34): k = min{k : u < F(k)}, F(k) = sum_{j<=k} e^-1 / j!, with
 * the terms and the running sum in fp64 in exactly this order (p_0 = e^-1, p_k = p_{k-1} / k); capped
 * at 16 (F(16) rounds to 1 in fp64) */
int32_t orc_poisson1(uint64_t seed, int32_t t, int64_t i) {
  double u = (double)(orc_rng4(seed, 0x5246u, (uint64_t)t, (uint64_t)i) >> 11) * 0x1.0p-53;
  double p = 0x1.78b56362cef38p-2; /* e^-1 rounded to double */
  double F = p;
  int32_t k = 0;
  while (u >= F && k < 16) {
    ++k;
    p = p / (double)k;
    F = F + p;
  }
  return k;
}

void orc_weights(int64_t n, const float* y, const int32_t* llm_id, const int32_t* prof_id, int32_t n_llm,
                 int32_t n_prof, float L1, float L2, float* w_out) {
  int64_t ng = (int64_t)n_llm * n_prof;
  double* Dmax = (double*)calloc((size_t)(ng * 2), sizeof(double));
  double L[2] = {(double)L1, (double)L2};
  for (int64_t i = 0; i < n; ++i) {
    int64_t gidx = (int64_t)llm_id[i] * n_prof + prof_id[i];
    for (int t = 0; t < 2; ++t) {
      double d = fabs((double)y[i * 2 + t] - L[t]);
      if (d > Dmax[gidx * 2 + t]) Dmax[gidx * 2 + t] = d;
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    int64_t gidx = (int64_t)llm_id[i] * n_prof + prof_id[i];
    double wt[2];
    for (int t = 0; t < 2; ++t) {
      double d = fabs((double)y[i * 2 + t] - L[t]);
      double D = Dmax[gidx * 2 + t];
      wt[t] = D > 0.0 ? 1.0 - d / D : 1.0;
    }
    w_out[i] = (float)((wt[0] + wt[1]) * 0.5);
  }
  free(Dmax);
}

/* ------------------------------------------------------------------------------------------ */
/* O2 — cuts ("number of bins for the histogram tree method")          */
static int cmp_float(const void* a, const void* b) {
  float x = *(const float*)a, y = *(const float*)b;
  return (x > y) - (x < y);
}

int orc_cuts(const float* X, int64_t n, int32_t F, int64_t row_offset, int64_t n_global, int32_t max_bin,
             float* cuts, int32_t* ncuts) {
  if (F < 1 || F > ORC_MAX_F || !(max_bin == 0 || (max_bin >= 2 && max_bin <= ORC_MAX_BIN)) || n < 1) return 1;
  const int64_t cap = (int64_t)1 << 20;
  int64_t s = (n_global + cap - 1) / cap;
  if (s < 1) s = 1;
  /* sample rows: global index i == 0 (mod s) */
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if ((row_offset + i) % s == 0) ++m;
  float* v = (float*)malloc((size_t)(m > 0 ? m : 1) * sizeof(float));
  for (int32_t f = 0; f < F; ++f) {
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
      if ((row_offset + i) % s != 0) continue;
      float x = X[i * F + f];
      if (x == 0.0f) x = 0.0f; /* canonicalise -0 to +0 */
      v[k++] = x;
    }
    qsort(v, (size_t)m, sizeof(float), cmp_float);
    /* distinct values d_1 < ... < d_k */
    int64_t ndist = 0;
    for (int64_t i = 0; i < m; ++i)
      if (i == 0 || v[i] != v[i - 1]) ++ndist;
    int32_t nc = 0;
    float* cf = cuts + (int64_t)f * (ORC_MAX_BIN - 1);
    if (max_bin == 0 && ndist > ORC_MAX_BIN) { /* exact: more distinct values than codes */
      free(v);
      return 1;
    }
    if (max_bin == 0 || ndist <= max_bin) {
      /* cuts = [d_2 .. d_k] */
      for (int64_t i = 1; i < m; ++i)
        if (v[i] != v[i - 1]) cf[nc++] = v[i];
    } else {
      /* c_j = v[floor(j*|v|/B)], j = 1..B-1; drop c_j == v[0]; dedupe */
      for (int32_t j = 1; j < max_bin; ++j) {
        float c = v[((int64_t)j * m) / max_bin];
        if (c == v[0]) continue;
        if (nc > 0 && cf[nc - 1] == c) continue;
        cf[nc++] = c;
      }
    }
    ncuts[f] = nc;
  }
  free(v);
  return 0;
}

void orc_codes(const float* X, int64_t n, int32_t F, const float* cuts, const int32_t* ncuts, uint16_t* codes) {
  for (int64_t i = 0; i < n; ++i)
    for (int32_t f = 0; f < F; ++f) {
      const float* cf = cuts + (int64_t)f * (ORC_MAX_BIN - 1);
      float x = X[i * F + f];
      /* upper_bound: number of cuts <= x */
      int32_t lo = 0, hi = ncuts[f];
      while (lo < hi) {
        int32_t mid = (lo + hi) / 2;
        if (cf[mid] <= x) lo = mid + 1;
        else hi = mid;
      }
      codes[i * F + f] = (uint16_t)lo;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* O4 — q = (int32) rint(ldexpf(g, K - e)),  e = M == 0 ? 0 : ilogb(M) + 1,  M = max |g|      */
int32_t orc_quantize(int64_t n, const float* v, int32_t K, int32_t* q) {
  float M = 0.0f;
  for (int64_t i = 0; i < n; ++i)
    if (fabsf(v[i]) > M) M = fabsf(v[i]);
  int32_t e = M == 0.0f ? 0 : ilogbf(M) + 1;
  for (int64_t i = 0; i < n; ++i) q[i] = (int32_t)rintf(ldexpf(v[i], K - e));
  return e;
}

/* ------------------------------------------------------------------------------------------ */
/* O6 — XGBoost-convention weight and gain ("XGBoost regressor")        */
double orc_calc_weight(double G, double H, double lo, double hi, double lambda, double mcw) {
  double w = 0.0;
  if (!(H < mcw || H <= 0.0)) w = -G / (H + lambda);
  if (w < lo) w = lo;
  else if (w > hi) w = hi;
  return w;
}
double orc_calc_gain(double G, double H, double w, double lambda) {
  if (H <= 0.0) return 0.0;
  return -((2.0 * G) * w + (H + lambda) * (w * w));
}

/* O5 — Hg[f][b] = sum_{i in node, code_if = b} q_g,i ; likewise Hh */
void orc_node_hist(const uint16_t* codes, int32_t F, const int64_t* idx, int64_t m, const int32_t* qg,
                   const int32_t* qh, int64_t* Hg, int64_t* Hh) {
  memset(Hg, 0, sizeof(int64_t) * (size_t)F * ORC_MAX_BIN);
  memset(Hh, 0, sizeof(int64_t) * (size_t)F * ORC_MAX_BIN);
  for (int64_t j = 0; j < m; ++j) {
    int64_t i = idx[j];
    for (int32_t f = 0; f < F; ++f) {
      int32_t b = codes[i * F + f];
      Hg[f * ORC_MAX_BIN + b] += qg[i];
      Hh[f * ORC_MAX_BIN + b] += qh[i];
    }
  }
}

int orc_best_split(const int64_t* Hg, const int64_t* Hh, int32_t F, const int32_t* nbins, const uint8_t* fmask,
                   int32_t users_col, int32_t monotone_users, int32_t eg, int32_t eh, int32_t K, double lo,
                   double hi, double lambda, double mcw, orc_split* out) {
  /* node totals: every feature's histogram sums to them; read feature 0 */
  int64_t Gq = 0, Hq = 0;
  for (int32_t b = 0; b < ORC_MAX_BIN; ++b) {
    Gq += Hg[b];
    Hq += Hh[b];
  }
  double G = ldexp((double)Gq, eg - K), H = ldexp((double)Hq, eh - K);
  double wP = orc_calc_weight(G, H, lo, hi, lambda, mcw);
  double gainP = orc_calc_gain(G, H, wP, lambda);
  int found = 0;
  double best = -INFINITY;
  for (int32_t f = 0; f < F; ++f) {
    if (!fmask[f]) continue;
    int64_t GLq = 0, HLq = 0;
    for (int32_t b = 0; b + 1 < nbins[f]; ++b) {
      GLq += Hg[f * ORC_MAX_BIN + b];
      HLq += Hh[f * ORC_MAX_BIN + b];
      int64_t GRq = Gq - GLq, HRq = Hq - HLq;
      double GL = ldexp((double)GLq, eg - K), HL = ldexp((double)HLq, eh - K);
      double GR = ldexp((double)GRq, eg - K), HR = ldexp((double)HRq, eh - K);
      if (!(HL >= mcw && HR >= mcw)) continue;
      double wl = orc_calc_weight(GL, HL, lo, hi, lambda, mcw);
      double wr = orc_calc_weight(GR, HR, lo, hi, lambda, mcw);
      if (monotone_users && f == users_col && wl > wr) continue; /* l non-decreasing in u */
      double loss = (orc_calc_gain(GL, HL, wl, lambda) + orc_calc_gain(GR, HR, wr, lambda)) - gainP;
      if (loss > best) { /* strict: ties keep the smaller f, then the smaller b */
        best = loss;
        out->f = f;
        out->b = b;
        out->loss = loss;
        out->wl = wl;
        out->wr = wr;
        out->GLq = GLq;
        out->HLq = HLq;
        out->GRq = GRq;
        out->HRq = HRq;
        found = 1;
      }
    }
  }
  return found && best > 1e-6;
}

/* ------------------------------------------------------------------------------------------ */
/* O3-O9 — fit                                                                                 */
typedef struct {
  int32_t k;       /* complete-tree index */
  int64_t* rows;   /* row indices */
  int64_t m;
  double lo, hi;   /* monotone bounds */
} orc_node;

static int fit_one_target(const uint16_t* codes, const float* y, const float* w, int64_t n, int32_t F,
                          int32_t users_col, int64_t row_offset, const orc_hparams* hp, const float* cuts,
                          const int32_t* ncuts, int target, float* base_out, int32_t* feat, int32_t* bin,
                          float* thr, float* val, double* gain, float* p, int32_t n_trees_fit) {
  const int32_t K = hp->grad_bits, D = hp->max_depth;
  const int64_t n_nodes = ((int64_t)1 << (D + 1)) - 1;
  const double lambda = (double)hp->lambda, mcw = (double)hp->min_child_weight, eta = (double)hp->eta;
  float* g = (float*)malloc(sizeof(float) * (size_t)n);
  float* h = (float*)malloc(sizeof(float) * (size_t)n);
  int32_t* qg = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* qh = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int64_t* Hg = (int64_t*)malloc(sizeof(int64_t) * (size_t)F * ORC_MAX_BIN);
  int64_t* Hh = (int64_t*)malloc(sizeof(int64_t) * (size_t)F * ORC_MAX_BIN);
  int32_t nbins[ORC_MAX_F];
  for (int32_t f = 0; f < F; ++f) nbins[f] = ncuts[f] + 1;

  const int rf = hp->model == 1;
  /* O3 — base score: quantise g = w*(0 - y), h = w (no subsampling); base = -G/H (lambda = 0).
   * Random forest (R33): no intercept, base 0 (every tree predicts the mean of its bootstrap). */
  for (int64_t i = 0; i < n; ++i) {
    float d = 0.0f - y[i * 2 + target];
    g[i] = w[i] * d;
    h[i] = w[i];
  }
  int32_t eg = orc_quantize(n, g, K, qg), eh = orc_quantize(n, h, K, qh);
  int64_t Gq = 0, Hq = 0;
  for (int64_t i = 0; i < n; ++i) {
    Gq += qg[i];
    Hq += qh[i];
  }
  double G0 = ldexp((double)Gq, eg - K), H0 = ldexp((double)Hq, eh - K);
  float base = H0 > 0.0 ? (float)(-G0 / H0) : 0.0f;
  if (rf) base = 0.0f;
  *base_out = base;
  for (int64_t i = 0; i < n; ++i) p[i] = base;

  int64_t* all = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) all[i] = i;
  orc_node* cur = (orc_node*)malloc(sizeof(orc_node) * ((size_t)1 << D));
  orc_node* nxt = (orc_node*)malloc(sizeof(orc_node) * ((size_t)1 << D));
  int64_t* leaf_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);

  for (int32_t t = 0; t < n_trees_fit; ++t) {
    int32_t* tf = feat + (int64_t)t * n_nodes;
    int32_t* tb = bin + (int64_t)t * n_nodes;
    float* tt = thr + (int64_t)t * n_nodes;
    float* tv = val + (int64_t)t * n_nodes;
    double* tgn = gain ? gain + (int64_t)t * n_nodes : NULL;
    for (int64_t k = 0; k < n_nodes; ++k) {
      tf[k] = -2;
      tb[k] = 0;
      tt[k] = 0.0f;
      tv[k] = 0.0f;
      if (tgn) tgn[k] = 0.0;
    }
    /* O4 — gradients of weighted squared error, fp32; row subsampling.
     * Random forest (R33, R34): every tree fits y itself (p = 0 in the gradient, no boosting) with
     * the row's Poisson(1) bootstrap count as an integer weight: w_t = c_t,i * w (fp32). */
    for (int64_t i = 0; i < n; ++i) {
      if (rf) {
        const float c = hp->rf_bootstrap ? (float)orc_poisson1(hp->seed, t, row_offset + i) : 1.0f;
        const float wt = c * w[i];
        g[i] = wt * (0.0f - y[i * 2 + target]);
        h[i] = wt;
        continue;
      }
      float d = p[i] - y[i * 2 + target];
      g[i] = w[i] * d;
      h[i] = w[i];
      if (hp->subsample < 1.0f) {
        double r = (double)(orc_rng4(hp->seed, (uint64_t)(2 * target), (uint64_t)t, (uint64_t)(row_offset + i)) >> 11) *
                   0x1.0p-53;
        if (r >= (double)hp->subsample) {
          g[i] = 0.0f;
          h[i] = 0.0f;
        }
      }
    }
    eg = orc_quantize(n, g, K, qg);
    eh = orc_quantize(n, h, K, qh);
    /* O6.3 — column sample: keep ceil(colsample*F) features with the smallest keys (ties by f) */
    uint8_t fmask[ORC_MAX_F];
    int32_t nkeep = F;
    if (hp->colsample_bytree < 1.0f) {
      nkeep = (int32_t)ceil((double)hp->colsample_bytree * (double)F);
      if (nkeep < 1) nkeep = 1;
    }
    for (int32_t f = 0; f < F; ++f) {
      uint64_t kf = orc_rng4(hp->seed, (uint64_t)(2 * target + 1), (uint64_t)t, (uint64_t)f);
      int32_t rank = 0;
      for (int32_t f2 = 0; f2 < F; ++f2) {
        uint64_t k2 = orc_rng4(hp->seed, (uint64_t)(2 * target + 1), (uint64_t)t, (uint64_t)f2);
        if (k2 < kf || (k2 == kf && f2 < f)) ++rank;
      }
      fmask[f] = (uint8_t)(rank < nkeep);
    }
    /* grow level by level */
    int32_t ncur = 1;
    cur[0].k = 0;
    cur[0].rows = all;
    cur[0].m = n;
    cur[0].lo = -INFINITY;
    cur[0].hi = INFINITY;
    int64_t* scratch = (int64_t*)malloc(sizeof(int64_t) * (size_t)n * 2);
    int64_t* buf[2] = {scratch, scratch + n};
    int which = 0;
    for (int32_t d = 0; d <= D && ncur > 0; ++d) {
      int32_t nn = 0;
      int64_t pos = 0;
      int64_t* out = buf[which];
      for (int32_t j = 0; j < ncur; ++j) {
        orc_node* nd = &cur[j];
        int64_t Gn = 0, Hn = 0;
        for (int64_t r = 0; r < nd->m; ++r) {
          Gn += qg[nd->rows[r]];
          Hn += qh[nd->rows[r]];
        }
        orc_split sp;
        int split = 0;
        if (d < D) {
          if (rf) {
            /* R35 — random forest: the node's own feature sample, the ceil(max_features F) features
             * with the smallest keys rng4(seed, 2 target + 1, t, (k + 1) * 32 + f), ties by f */
            int32_t mk = (int32_t)ceil((double)hp->max_features * (double)F);
            if (mk < 1) mk = 1;
            for (int32_t f = 0; f < F; ++f) {
              uint64_t kf = orc_rng4(hp->seed, (uint64_t)(2 * target + 1), (uint64_t)t,
                                     (uint64_t)(nd->k + 1) * 32u + (uint64_t)f);
              int32_t rank = 0;
              for (int32_t f2 = 0; f2 < F; ++f2) {
                uint64_t k2 = orc_rng4(hp->seed, (uint64_t)(2 * target + 1), (uint64_t)t,
                                       (uint64_t)(nd->k + 1) * 32u + (uint64_t)f2);
                if (k2 < kf || (k2 == kf && f2 < f)) ++rank;
              }
              fmask[f] = (uint8_t)(rank < mk);
            }
          }
          orc_node_hist(codes, F, nd->rows, nd->m, qg, qh, Hg, Hh);
          split = orc_best_split(Hg, Hh, F, nbins, fmask, users_col, hp->monotone_users, eg, eh, K, nd->lo, nd->hi,
                                 lambda, mcw, &sp);
        }
        if (!split) {
          /* O8 — leaf value v = (float)(eta * W(G,H,lo,hi)); random forest (R36): (float)(W / T), so
           * the prediction base + sum_t v_t is the average of the trees */
          double Gd = ldexp((double)Gn, eg - K), Hd = ldexp((double)Hn, eh - K);
          double Wl = orc_calc_weight(Gd, Hd, nd->lo, nd->hi, lambda, mcw);
          float v = rf ? (float)(Wl / (double)hp->n_trees) : (float)(eta * Wl);
          tf[nd->k] = -1;
          tv[nd->k] = v;
          for (int64_t r = 0; r < nd->m; ++r) leaf_of[nd->rows[r]] = nd->k;
          continue;
        }
        tf[nd->k] = sp.f;
        tb[nd->k] = sp.b;
        if (tgn) tgn[nd->k] = sp.loss;   /* the split's loss reduction (O6), kept for MDI */
        tt[nd->k] = cuts[(int64_t)sp.f * (ORC_MAX_BIN - 1) + sp.b];
        /* O7 — children: code <= b goes left; monotone bounds on users splits */
        double lo_l = nd->lo, hi_l = nd->hi, lo_r = nd->lo, hi_r = nd->hi;
        if (hp->monotone_users && sp.f == users_col) {
          double mid = (sp.wl + sp.wr) * 0.5;
          hi_l = mid;
          lo_r = mid;
        }
        orc_node* L = &nxt[nn++];
        orc_node* R = &nxt[nn++];
        L->k = 2 * nd->k + 1;
        R->k = 2 * nd->k + 2;
        L->lo = lo_l;
        L->hi = hi_l;
        R->lo = lo_r;
        R->hi = hi_r;
        L->rows = out + pos;
        L->m = 0;
        for (int64_t r = 0; r < nd->m; ++r) {
          int64_t i = nd->rows[r];
          if (codes[i * F + sp.f] <= sp.b) out[pos++] = i, L->m++;
        }
        R->rows = out + pos;
        R->m = 0;
        for (int64_t r = 0; r < nd->m; ++r) {
          int64_t i = nd->rows[r];
          if (codes[i * F + sp.f] > sp.b) out[pos++] = i, R->m++;
        }
      }
      orc_node* tmp = cur;
      cur = nxt;
      nxt = tmp;
      ncur = nn;
      which ^= 1;
      /* note: the rows of the new level live in buf[which^1]; the next level writes buf[which] */
    }
    /* O9 — p_i = p_i + v_leaf(i), one fp32 rounding */
    for (int64_t i = 0; i < n; ++i) p[i] = p[i] + tv[leaf_of[i]];
    free(scratch);
  }
  free(g);
  free(h);
  free(qg);
  free(qh);
  free(Hg);
  free(Hh);
  free(all);
  free(cur);
  free(nxt);
  free(leaf_of);
  return 0;
}

int orc_fit(const float* X, const float* y, const float* w_in, const int32_t* llm_id, const int32_t* prof_id,
            int64_t n, int32_t F, int32_t users_col, int32_t n_llm, int32_t n_prof, int64_t row_offset,
            int64_t n_global, const orc_hparams* hp, float L1, float L2, float* cuts, int32_t* ncuts, float* base,
            int32_t* feat, int32_t* bin, float* thr, float* val, float* train_pred, int32_t n_trees_limit) {
  return orc_fit_gain(X, y, w_in, llm_id, prof_id, n, F, users_col, n_llm, n_prof, row_offset, n_global, hp, L1, L2,
                      cuts, ncuts, base, feat, bin, thr, val, NULL, train_pred, n_trees_limit);
}

int orc_fit_gain(const float* X, const float* y, const float* w_in, const int32_t* llm_id, const int32_t* prof_id,
                 int64_t n, int32_t F, int32_t users_col, int32_t n_llm, int32_t n_prof, int64_t row_offset,
                 int64_t n_global, const orc_hparams* hp, float L1, float L2, float* cuts, int32_t* ncuts,
                 float* base, int32_t* feat, int32_t* bin, float* thr, float* val, double* gain, float* train_pred,
                 int32_t n_trees_limit) {
  if (n < 1 || F < 1 || F > ORC_MAX_F || users_col < 0 || users_col >= F) return 1;
  if (hp->max_depth < 1 || hp->max_depth > 12 || hp->n_trees < 0 || hp->grad_bits < 2 || hp->grad_bits > 14) return 1;
  if (hp->tree_method != 0 && hp->tree_method != 1) return 1;
  if (hp->tree_method == 0 && (hp->max_bin < 2 || hp->max_bin > ORC_MAX_BIN)) return 1;
  if (hp->model != 0 && hp->model != 1) return 1;
  if (hp->model == 1 && (!(hp->max_features > 0.0f && hp->max_features <= 1.0f) || hp->subsample != 1.0f ||
                         hp->monotone_users != 0))
    return 1;
  for (int64_t i = 0; i < n * F; ++i)
    if (!isfinite(X[i])) return 1;
  for (int64_t i = 0; i < n * 2; ++i)
    if (!isfinite(y[i])) return 1;
  float* w = (float*)malloc(sizeof(float) * (size_t)n);
  if (hp->use_eq4_weights) {
    orc_weights(n, y, llm_id, prof_id, n_llm, n_prof, L1, L2, w);
  } else {
    for (int64_t i = 0; i < n; ++i) w[i] = w_in ? w_in[i] : 1.0f;
  }
  if (orc_cuts(X, n, F, row_offset, n_global, hp->tree_method == 1 ? 0 : hp->max_bin, cuts, ncuts)) {
    free(w);
    return 1;
  }
  uint16_t* codes = (uint16_t*)malloc((size_t)n * F * sizeof(uint16_t));
  orc_codes(X, n, F, cuts, ncuts, codes);
  const int64_t n_nodes = ((int64_t)1 << (hp->max_depth + 1)) - 1;
  int32_t nt = hp->n_trees;
  if (n_trees_limit > 0 && n_trees_limit < nt) nt = n_trees_limit;
  float* p = (float*)malloc(sizeof(float) * (size_t)n);
  for (int target = 0; target < 2; ++target) {
    int64_t off = (int64_t)target * hp->n_trees * n_nodes;
    fit_one_target(codes, y, w, n, F, users_col, row_offset, hp, cuts, ncuts, target, &base[target], feat + off,
                   bin + off, thr + off, val + off, gain ? gain + off : NULL, p, nt);
    if (train_pred)
      for (int64_t i = 0; i < n; ++i) train_pred[i * 2 + target] = p[i];
  }
  free(p);
  free(codes);
  free(w);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* MDI feature importance (§III-B P:L120 and §III-D P:L156-158 use
 * the Mean Decrease in Impurity [3]).  For weighted squared error the impurity decrease of a
 * split is SSE(parent) - SSE(left) - SSE(right) = GL^2/HL + GR^2/HR - G^2/H, i.e. the split loss
 * of O6 (with lambda = 0; the regularised loss otherwise).  raw[t][f] = sum over the trees in
 * order, and over each tree's nodes in index order, of the loss of every split on f (fp64);
 * normalised: raw / sum_f raw (all zeros stay zero). */
void orc_importance(int32_t n_trees, int32_t max_depth, int32_t F, const int32_t* feat, const double* gain,
                    int32_t normalize, double* out /* 2 x F */) {
  const int64_t n_nodes = ((int64_t)1 << (max_depth + 1)) - 1;
  for (int target = 0; target < 2; ++target) {
    double* o = out + (int64_t)target * F;
    for (int32_t f = 0; f < F; ++f) o[f] = 0.0;
    for (int32_t t = 0; t < n_trees; ++t) {
      const int64_t off = ((int64_t)target * n_trees + t) * n_nodes;
      for (int64_t k = 0; k < n_nodes; ++k)
        if (feat[off + k] >= 0) o[feat[off + k]] += gain[off + k];
    }
    if (normalize) {
      double tot = 0.0;
      for (int32_t f = 0; f < F; ++f) tot += o[f];
      if (tot > 0.0)
        for (int32_t f = 0; f < F; ++f) o[f] = o[f] / tot;
    }
  }
}

/* ------------------------------------------------------------------------------------------ */
/* O10 — predict                                                                               */
void orc_predict(const float* X, int64_t n, int32_t F, int32_t n_trees, int32_t max_depth, const float* base,
                 const int32_t* feat, const float* thr, const float* val, float* out) {
  const int64_t n_nodes = ((int64_t)1 << (max_depth + 1)) - 1;
  for (int target = 0; target < 2; ++target) {
    const int64_t off = (int64_t)target * n_trees * n_nodes;
    for (int64_t i = 0; i < n; ++i) {
      float p = base[target];
      for (int32_t t = 0; t < n_trees; ++t) {
        const int32_t* tf = feat + off + (int64_t)t * n_nodes;
        int64_t k = 0;
        while (tf[k] >= 0) k = X[i * F + tf[k]] < thr[off + (int64_t)t * n_nodes + k] ? 2 * k + 1 : 2 * k + 2;
        p = p + val[off + (int64_t)t * n_nodes + k];
      }
      out[i * 2 + target] = p;
    }
  }
}

/* ------------------------------------------------------------------------------------------ */
/* O11 — Eq. (3): u_max = max{u in U : l1(u') <= L1 and l2(u') <= L2 for all u' <= u}
 * (P:L174); 0 when the set is empty (reading R2).  Levels ascending.                       */
static int32_t umax_prefix(int32_t n_levels, const int32_t* levels, const float* p1, const float* p2, int stride,
                           float L1, float L2) {
  int32_t um = 0;
  for (int32_t k = 0; k < n_levels; ++k) {
    if (!(p1[k * stride] <= L1 && p2[k * stride] <= L2)) break;
    um = levels[k];
  }
  return um;
}

void orc_recommend(const float* pred, int32_t n_llm, int32_t n_prof, int32_t n_levels, const int32_t* user_levels,
                   const double* cost, const uint8_t* allowed, float L1, float L2, int64_t U, orc_rec* out) {
  for (int32_t i = 0; i < n_llm; ++i) {
    orc_rec best = {-1, 0, INFINITY, 0};
    for (int32_t gp = 0; gp < n_prof; ++gp) {
      if (allowed && !allowed[(int64_t)i * n_prof + gp]) continue;
      const float* pr = pred + (((int64_t)i * n_prof + gp) * n_levels) * 2;
      int32_t um = umax_prefix(n_levels, user_levels, pr, pr + 1, 2, L1, L2);
      if (um <= 0) continue;
      int64_t npods = (U + um - 1) / um;            /* Eq. (2), ceiling (reading R1) */
      double c = (double)npods * cost[gp];          /* Eq. (1) objective n * c(G) */
      if (c < best.cost) {                          /* ties -> lowest profile index (R4) */
        best.profile = gp;
        best.n_pods = npods;
        best.cost = c;
        best.u_max = um;
      }
    }
    out[i] = best;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* O12 — CV                                                                                    */
double orc_wmape(int64_t n, const float* pred, const float* y, const float* w, int target) {
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double yt = (double)y[i * 2 + target];
    num += (double)w[i] * (fabs((double)pred[i * 2 + target] - yt) / fabs(yt));
    den += (double)w[i];
  }
  return den > 0.0 ? num / den : 0.0;
}

double orc_so_score(double S, double O) {
  double inv = 1.0 - O;
  if (inv < 0.0) inv = 0.0;
  double den = S + inv;
  return den > 0.0 ? (2.0 * S * inv) / den : 0.0;
}

typedef struct {
  float *X, *y, *w;
  int32_t *llm, *prof;
  int64_t n;
} subset;

static subset make_subset(const float* X, const float* y, const float* w, const int32_t* llm, const int32_t* prof,
                          int64_t n, int32_t F, int32_t ex1, int32_t ex2, int keep_only) {
  subset s;
  s.n = 0;
  for (int64_t i = 0; i < n; ++i) {
    int in = keep_only ? (llm[i] == ex1) : (llm[i] != ex1 && llm[i] != ex2);
    if (in) s.n++;
  }
  s.X = (float*)malloc(sizeof(float) * (size_t)(s.n * F + 1));
  s.y = (float*)malloc(sizeof(float) * (size_t)(s.n * 2 + 1));
  s.w = (float*)malloc(sizeof(float) * (size_t)(s.n + 1));
  s.llm = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s.n + 1));
  s.prof = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s.n + 1));
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    int in = keep_only ? (llm[i] == ex1) : (llm[i] != ex1 && llm[i] != ex2);
    if (!in) continue;
    memcpy(s.X + k * F, X + i * F, sizeof(float) * (size_t)F);
    s.y[k * 2] = y[i * 2];
    s.y[k * 2 + 1] = y[i * 2 + 1];
    s.w[k] = w[i];
    s.llm[k] = llm[i];
    s.prof[k] = prof[i];
    ++k;
  }
  return s;
}
static void free_subset(subset* s) {
  free(s->X);
  free(s->y);
  free(s->w);
  free(s->llm);
  free(s->prof);
}

/* fit on `tr`, predict rows of `te` */
static int fit_predict(const subset* tr, const subset* te, int32_t F, int32_t users_col, int32_t n_llm,
                       int32_t n_prof, const orc_hparams* hp, float L1, float L2, float* pred) {
  const int64_t n_nodes = ((int64_t)1 << (hp->max_depth + 1)) - 1;
  size_t nn = (size_t)(2 * (int64_t)hp->n_trees * n_nodes + 1);
  float* cuts = (float*)malloc(sizeof(float) * ORC_MAX_F * (ORC_MAX_BIN - 1));
  int32_t ncuts[ORC_MAX_F];
  float base[2];
  int32_t* feat = (int32_t*)malloc(sizeof(int32_t) * nn);
  int32_t* bin = (int32_t*)malloc(sizeof(int32_t) * nn);
  float* thr = (float*)malloc(sizeof(float) * nn);
  float* val = (float*)malloc(sizeof(float) * nn);
  int rc = orc_fit(tr->X, tr->y, NULL, tr->llm, tr->prof, tr->n, F, users_col, n_llm, n_prof, 0, tr->n, hp, L1, L2,
                   cuts, ncuts, base, feat, bin, thr, val, NULL, 0);
  if (rc == 0) orc_predict(te->X, te->n, F, hp->n_trees, hp->max_depth, base, feat, thr, val, pred);
  free(cuts);
  free(feat);
  free(bin);
  free(thr);
  free(val);
  return rc;
}

/* recommendation from one LLM's rows (profile ids x user levels), on values v (pred or truth) */
static orc_rec rec_from_rows(const subset* te, int32_t F, int32_t users_col, int32_t n_prof, const float* v,
                             const double* cost, float L1, float L2, int64_t U, int32_t* umax_per_prof) {
  orc_rec best = {-1, 0, INFINITY, 0};
  int32_t* lv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(te->n + 1));
  float* p1 = (float*)malloc(sizeof(float) * (size_t)(te->n + 1));
  float* p2 = (float*)malloc(sizeof(float) * (size_t)(te->n + 1));
  for (int32_t gp = 0; gp < n_prof; ++gp) {
    /* rows of profile gp, sorted by users ascending (insertion sort, stable) */
    int32_t m = 0;
    for (int64_t i = 0; i < te->n; ++i) {
      if (te->prof[i] != gp) continue;
      int32_t u = (int32_t)te->X[i * F + users_col];
      int32_t j = m++;
      while (j > 0 && lv[j - 1] > u) {
        lv[j] = lv[j - 1];
        p1[j] = p1[j - 1];
        p2[j] = p2[j - 1];
        --j;
      }
      lv[j] = u;
      p1[j] = v[i * 2];
      p2[j] = v[i * 2 + 1];
    }
    if (umax_per_prof) umax_per_prof[gp] = 0;
    if (m == 0) continue; /* candidate set: profiles measured for this LLM (reading R5) */
    int32_t um = umax_prefix(m, lv, p1, p2, 1, L1, L2);
    if (umax_per_prof) umax_per_prof[gp] = um;
    if (um <= 0) continue;
    int64_t npods = (U + um - 1) / um;
    double c = (double)npods * cost[gp];
    if (c < best.cost) {
      best.profile = gp;
      best.n_pods = npods;
      best.cost = c;
      best.u_max = um;
    }
  }
  free(lv);
  free(p1);
  free(p2);
  return best;
}

int orc_cv(const float* X, const float* y, const int32_t* llm_id, const int32_t* prof_id, int64_t n, int32_t F,
           int32_t users_col, int32_t n_llm, int32_t n_prof, const orc_hparams* grid, int32_t n_grid, float L1,
           float L2, int64_t U, const double* prof_cost, orc_fold* folds, int32_t* n_folds, double* S, double* O,
           double* SO) {
  if (n_grid < 1) return 1;
  float* w = (float*)malloc(sizeof(float) * (size_t)n);
  orc_weights(n, y, llm_id, prof_id, n_llm, n_prof, L1, L2, w); /* per group: independent of folds */
  uint8_t* present = (uint8_t*)calloc((size_t)n_llm, 1);
  for (int64_t i = 0; i < n; ++i) present[llm_id[i]] = 1;
  int32_t nf = 0, n_feasible = 0, n_success = 0;
  double sumO = 0.0;
  int32_t* umax_truth = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_prof);
  for (int32_t M = 0; M < n_llm; ++M) {
    if (!present[M]) continue;
    subset trM = make_subset(X, y, w, llm_id, prof_id, n, F, M, -1, 0);
    subset teM = make_subset(X, y, w, llm_id, prof_id, n, F, M, -1, 1);
    int32_t best_hp = 0;
    if (n_grid > 1) {
      double best_err = INFINITY;
      for (int32_t hpi = 0; hpi < n_grid; ++hpi) {
        double err_sum = 0.0;
        int32_t nv = 0;
        for (int32_t V = 0; V < n_llm; ++V) {
          if (!present[V] || V == M) continue;
          subset trV = make_subset(X, y, w, llm_id, prof_id, n, F, M, V, 0);
          subset teV = make_subset(X, y, w, llm_id, prof_id, n, F, V, -1, 1);
          float* pv = (float*)malloc(sizeof(float) * (size_t)(teV.n * 2 + 1));
          fit_predict(&trV, &teV, F, users_col, n_llm, n_prof, &grid[hpi], L1, L2, pv);
          double e = 0.5 * (orc_wmape(teV.n, pv, teV.y, teV.w, 0) + orc_wmape(teV.n, pv, teV.y, teV.w, 1));
          err_sum += e;
          ++nv;
          free(pv);
          free_subset(&trV);
          free_subset(&teV);
        }
        double err = nv > 0 ? err_sum / nv : 0.0;
        if (err < best_err) {
          best_err = err;
          best_hp = hpi;
        }
      }
    }
    float* pm = (float*)malloc(sizeof(float) * (size_t)(teM.n * 2 + 1));
    fit_predict(&trM, &teM, F, users_col, n_llm, n_prof, &grid[best_hp], L1, L2, pm);
    orc_fold* fd = &folds[nf++];
    fd->llm = M;
    fd->hp_index = best_hp;
    fd->rec = rec_from_rows(&teM, F, users_col, n_prof, pm, prof_cost, L1, L2, U, NULL);
    fd->truth = rec_from_rows(&teM, F, users_col, n_prof, teM.y, prof_cost, L1, L2, U, umax_truth);
    fd->truth_feasible = fd->truth.profile >= 0;
    fd->success = 0;
    fd->overspend = 0.0;
    if (fd->truth_feasible) {
      ++n_feasible;
      int32_t g = fd->rec.profile;
      /* S_M = 1 iff n(M,G*) * u_max_true(M,G*) >= U */
      if (g >= 0 && umax_truth[g] > 0 && fd->rec.n_pods * (int64_t)umax_truth[g] >= U) {
        fd->success = 1;
        ++n_success;
        fd->overspend = (fd->rec.cost - fd->truth.cost) / fd->truth.cost; /* Eq. (6) */
        sumO += fd->overspend;
      }
    }
    free(pm);
    free_subset(&trM);
    free_subset(&teM);
  }
  *n_folds = nf;
  *S = n_feasible > 0 ? (double)n_success / n_feasible : 0.0;
  *O = n_success > 0 ? sumO / n_success : 0.0;
  *SO = orc_so_score(*S, *O); /* Eq. (7) */
  free(w);
  free(present);
  free(umax_truth);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Workload generator (§III-B).  Test infrastructure. */
/* Model: per parameter p, bins = O2's cuts with B = ORC_WG_BINS (64) — one bin per distinct value
 * when there are at most 64 ("unless the cardinality of the parameter is lower"), else
 * equal-frequency quantiles (exact on <= 2^20 rows, strided sample beyond); the centre of bin b is
 * (min + max) / 2 of the trace values in it (fp64, stored as float; -0 counts as +0).  Joint model
 * (P:L128-130): key(row) = sum_p code_p * stride_p (mixed radix, stride_0 = 1, stride_{p+1} =
 * stride_p * nbins_p); the non-empty keys in ascending order with their row counts.
 * Sampling: sample s of seed draws r = rng4(seed, 0x5747, s, 0), t = floor(r * n / 2^64)
 * in [0, n), picks the first key whose cumulative count exceeds t (probability count / n) and
 * emits every parameter's bin centre. */
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

int orc_wg_build(const float* T, int64_t n, int32_t P, int32_t* nbins, float* centres, uint64_t* keys,
                 int64_t* counts, int64_t* m_out) {
  if (n < 1 || P < 1 || P > ORC_MAX_F) return 1;
  for (int64_t i = 0; i < n * P; ++i)
    if (!isfinite(T[i])) return 1;
  float* cuts = (float*)malloc(sizeof(float) * ORC_MAX_F * (ORC_MAX_BIN - 1));
  int32_t ncuts[ORC_MAX_F];
  if (orc_cuts(T, n, P, 0, n, ORC_WG_BINS, cuts, ncuts)) {
    free(cuts);
    return 1;
  }
  /* mixed-radix strides; the key space must fit 63 bits */
  uint64_t stride[ORC_MAX_F];
  double space = 1.0;
  uint64_t st = 1;
  for (int32_t p = 0; p < P; ++p) {
    nbins[p] = ncuts[p] + 1;
    stride[p] = st;
    space *= (double)nbins[p];
    st *= (uint64_t)nbins[p];
  }
  if (space > 9.2e18) {
    free(cuts);
    return 1;
  }
  uint16_t* codes = (uint16_t*)malloc((size_t)n * P * sizeof(uint16_t));
  orc_codes(T, n, P, cuts, ncuts, codes);
  /* per-bin min / max -> centres */
  double* mn = (double*)malloc(sizeof(double) * P * ORC_WG_BINS);
  double* mx = (double*)malloc(sizeof(double) * P * ORC_WG_BINS);
  for (int64_t i = 0; i < (int64_t)P * ORC_WG_BINS; ++i) {
    mn[i] = INFINITY;
    mx[i] = -INFINITY;
    centres[i] = 0.0f;
  }
  uint64_t* k = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t key = 0;
    for (int32_t p = 0; p < P; ++p) {
      int32_t c = codes[i * P + p];
      double x = (double)T[i * P + p];
      if (x == 0.0) x = 0.0;
      if (x < mn[p * ORC_WG_BINS + c]) mn[p * ORC_WG_BINS + c] = x;
      if (x > mx[p * ORC_WG_BINS + c]) mx[p * ORC_WG_BINS + c] = x;
      key += (uint64_t)c * stride[p];
    }
    k[i] = key;
  }
  for (int32_t p = 0; p < P; ++p)
    for (int32_t b = 0; b < nbins[p]; ++b)
      centres[p * ORC_WG_BINS + b] = (float)((mn[p * ORC_WG_BINS + b] + mx[p * ORC_WG_BINS + b]) * 0.5);
  /* sparse joint histogram: sorted distinct keys with counts */
  qsort(k, (size_t)n, sizeof(uint64_t), cmp_u64);
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (i == 0 || k[i] != k[i - 1]) {
      keys[m] = k[i];
      counts[m] = 0;
      ++m;
    }
    counts[m - 1] += 1;
  }
  *m_out = m;
  free(k);
  free(mn);
  free(mx);
  free(codes);
  free(cuts);
  return 0;
}

void orc_wg_sample(const uint64_t* keys, const int64_t* counts, int64_t m, int32_t P, const int32_t* nbins,
                   const float* centres, uint64_t seed, int64_t first, int64_t n_samples, float* out) {
  int64_t n = 0;
  for (int64_t j = 0; j < m; ++j) n += counts[j];
  for (int64_t s = 0; s < n_samples; ++s) {
    uint64_t r = orc_rng4(seed, 0x5747u, (uint64_t)(first + s), 0);
    uint64_t t = (uint64_t)(((unsigned __int128)r * (unsigned __int128)(uint64_t)n) >> 64);
    /* first j with cumulative count > t (a linear walk: plain and obviously correct) */
    int64_t j = 0, cum = counts[0];
    while ((uint64_t)cum <= t) cum += counts[++j];
    uint64_t key = keys[j];
    for (int32_t p = 0; p < P; ++p) {
      uint64_t digit = key % (uint64_t)nbins[p];
      key /= (uint64_t)nbins[p];
      out[s * P + p] = centres[p * ORC_WG_BINS + digit];
    }
  }
}
