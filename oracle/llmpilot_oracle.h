/* oracle/llmpilot_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle of the LLM-Pilot GPU-recommendation hot path
 * (arxiv 2410.02425, /root/reference/PAPER.md, cited "P:L<n>").  Only tests/, the graft
 * entry's smoke() and bench.py's cpu_baseline / --impl reference leg may load it.  It shares
 * no code, header, table or constant with the CUDA library (paper_2410_02425_b200/csrc);
 * it follows SURVEY.md §8(c) O1-O12 step by step, in the paper's order and notation.
 *
 * Parity status per function: every function is pinned by tests/test_oracle_*.py except
 * the end-to-end paper outcome (S=80%, O<20%), which needs the real dataset:
 * "parity unpinned" for that number only.
 */
#ifndef LLMPILOT_ORACLE_H
#define LLMPILOT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_F 32
#define ORC_MAX_BIN 1024   /* bins per feature: codes are 16-bit */

typedef struct {
  int32_t n_trees, max_depth, max_bin, grad_bits;
  float eta, lambda, min_child_weight, subsample, colsample_bytree;
  uint64_t seed;
  int32_t use_eq4_weights, monotone_users;
  /* model = 1: random-forest regressor (DESIGN R33-R36):
   * trees fit independently on Poisson(1) bootstrap counts, max_features sampled per node, leaf =
   * weighted mean / n_trees, no boosting, base 0.  rf_bootstrap = 0 disables the bootstrap (c = 1). */
  int32_t model;
  float max_features;
  int32_t rf_bootstrap;
  /* tree building method: 0 = hist (O2 cuts with max_bin bins), 1 = exact (every distinct
   * value of the sample its own bin, i.e. hist with unbounded max_bin; at most ORC_MAX_BIN) */
  int32_t tree_method;
} orc_hparams;

/* RF bootstrap count of (tree t, global row i): Poisson(1) by inversion of u = top 53 bits of
 * rng4(seed, 0x5246, t, i) / 2^53 (DESIGN R34) */
int32_t orc_poisson1(uint64_t seed, int32_t t, int64_t i);

/* counter-based generator: sm64 finaliser chained over (seed, a, b, c) */
uint64_t orc_rng4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);

/* O1 — Eq. (4) sample weights.  y is n x 2 row-major (nTTFT, ITL). */
void orc_weights(int64_t n, const float* y, const int32_t* llm_id, const int32_t* prof_id,
                 int32_t n_llm, int32_t n_prof, float L1, float L2, float* w_out);

/* O2 — quantile cuts from the global-index strided sample; returns 0 on success.
 * cuts: F x (ORC_MAX_BIN - 1) (row f holds ncuts[f] strictly increasing values).  max_bin in
 * [2, ORC_MAX_BIN]; max_bin = 0: exact (every distinct sample value starts a bin; fails if a
 * feature has more than ORC_MAX_BIN distinct values). */
int orc_cuts(const float* X, int64_t n, int32_t F, int64_t row_offset, int64_t n_global,
             int32_t max_bin, float* cuts, int32_t* ncuts);
/* O2 — code(x) = #{c in cuts_f : c <= x}; codes n x F row-major (16-bit) */
void orc_codes(const float* X, int64_t n, int32_t F, const float* cuts, const int32_t* ncuts,
               uint16_t* codes);

/* O4 — quantisation of one gradient vector: returns e (exponent) and writes q = rint(ldexpf(v, K-e)) */
int32_t orc_quantize(int64_t n, const float* v, int32_t K, int32_t* q);

/* O6 primitives (fp64, no FMA, fixed operation order) */
double orc_calc_weight(double G, double H, double lo, double hi, double lambda, double mcw);
double orc_calc_gain(double G, double H, double w, double lambda);

/* O5 — node histogram (int64), rows listed in idx[0..m) */
void orc_node_hist(const uint16_t* codes, int32_t F, const int64_t* idx, int64_t m, const int32_t* qg,
                   const int32_t* qh, int64_t* Hg /* F x ORC_MAX_BIN */, int64_t* Hh /* F x ORC_MAX_BIN */);

/* O6 — split search on one node's histogram.  Returns 1 and fills (f,b,loss,wl,wr,...) if a split
 * with loss > 1e-6 exists among the features with fmask[f] != 0, else 0. */
typedef struct {
  int32_t f, b;
  double loss, wl, wr;
  int64_t GLq, HLq, GRq, HRq;
} orc_split;
int orc_best_split(const int64_t* Hg, const int64_t* Hh, int32_t F, const int32_t* nbins,
                   const uint8_t* fmask, int32_t users_col, int32_t monotone_users, int32_t eg, int32_t eh,
                   int32_t K, double lo, double hi, double lambda, double mcw, orc_split* out);

/* O3-O9 — fit two ensembles.  Trees use complete-binary indexing (children 2k+1, 2k+2),
 * n_nodes = 2^(max_depth+1)-1 per tree; arrays are [2][n_trees][n_nodes].
 * feat = -1 leaf, -2 unused slot; thr = cuts_f[bin]; val = leaf value (float).
 * w_in: explicit weights used when hp->use_eq4_weights == 0 (NULL => w = 1).
 * train_pred (n x 2, may be NULL) receives the internal training predictions p.
 * row_offset/n_global: this shard's global position (cut sample + row subsampling).
 * Returns 0 on success, non-zero on invalid input. */
int orc_fit(const float* X, const float* y, const float* w_in, const int32_t* llm_id, const int32_t* prof_id,
            int64_t n, int32_t F, int32_t users_col, int32_t n_llm, int32_t n_prof, int64_t row_offset,
            int64_t n_global, const orc_hparams* hp, float L1, float L2, float* cuts, int32_t* ncuts,
            float* base, int32_t* feat, int32_t* bin, float* thr, float* val, float* train_pred,
            int32_t n_trees_limit /* <=0: all; else fit only the first k trees of each target */);

/* orc_fit plus gain [2][n_trees][nodes] (may be NULL): the loss of every split node, 0 elsewhere */
int orc_fit_gain(const float* X, const float* y, const float* w_in, const int32_t* llm_id, const int32_t* prof_id,
                 int64_t n, int32_t F, int32_t users_col, int32_t n_llm, int32_t n_prof, int64_t row_offset,
                 int64_t n_global, const orc_hparams* hp, float L1, float L2, float* cuts, int32_t* ncuts,
                 float* base, int32_t* feat, int32_t* bin, float* thr, float* val, double* gain, float* train_pred,
                 int32_t n_trees_limit);

/* MDI feature importance: per target, the sum
 * of the split losses on each feature over trees (in order) and nodes (index order), fp64;
 * normalize != 0 divides by the target's total.  out: 2 x F. */
void orc_importance(int32_t n_trees, int32_t max_depth, int32_t F, const int32_t* feat, const double* gain,
                    int32_t normalize, double* out);

/* Workload generator (§III-B): bins = O2 cuts with 64 bins,
 * centres = (min + max)/2 of each bin's values, sparse joint histogram of mixed-radix keys.
 * nbins: P; centres: P x 64; keys, counts: capacity n (m_out distinct keys, ascending).
 * Returns non-zero for invalid input (non-finite values, P out of range, key space > 2^63). */
#define ORC_WG_BINS 64
int orc_wg_build(const float* T, int64_t n, int32_t P, int32_t* nbins, float* centres, uint64_t* keys,
                 int64_t* counts, int64_t* m_out);
/* samples first .. first + n_samples - 1 of `seed` -> out (n_samples x P) */
void orc_wg_sample(const uint64_t* keys, const int64_t* counts, int64_t m, int32_t P, const int32_t* nbins,
                   const float* centres, uint64_t seed, int64_t first, int64_t n_samples, float* out);

/* O10 — predict: p = base; p = p + v_t(x) in tree order; x_f < thr goes left */
void orc_predict(const float* X, int64_t n, int32_t F, int32_t n_trees, int32_t max_depth, const float* base,
                 const int32_t* feat, const float* thr, const float* val, float* out /* n x 2 */);

/* O11 — Eq. (1)-(3).  pred: [n_llm][n_prof][n_levels][2]; allowed NULL => all. */
typedef struct {
  int32_t profile;
  int64_t n_pods;
  double cost;
  int32_t u_max;
} orc_rec;
void orc_recommend(const float* pred, int32_t n_llm, int32_t n_prof, int32_t n_levels, const int32_t* user_levels,
                   const double* cost, const uint8_t* allowed, float L1, float L2, int64_t U, orc_rec* out);

/* O12 — nested leave-one-LLM-out CV, success S_M, overspend Eq. (6), S/O Eq. (7).
 * Folds are written for every LLM id present, ascending.  Returns 0 on success. */
typedef struct {
  int32_t llm, hp_index;
  orc_rec rec, truth;
  int32_t success;
  double overspend;
  int32_t truth_feasible;
} orc_fold;
int orc_cv(const float* X, const float* y, const int32_t* llm_id, const int32_t* prof_id, int64_t n, int32_t F,
           int32_t users_col, int32_t n_llm, int32_t n_prof, const orc_hparams* grid, int32_t n_grid, float L1,
           float L2, int64_t U, const double* prof_cost, orc_fold* folds, int32_t* n_folds, double* S, double* O,
           double* SO);

/* O12 pieces exposed for pinning */
double orc_wmape(int64_t n, const float* pred, const float* y, const float* w, int target);
double orc_so_score(double S, double O);

#ifdef __cplusplus
}
#endif
#endif
