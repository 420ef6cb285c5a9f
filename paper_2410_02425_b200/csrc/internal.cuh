// internal.cuh — interfaces between the library's translation units.
#pragma once
#include "common.cuh"

namespace llmp {

// cuts: device [32][255] floats + [32] int32 counts; host mirror for export / model
struct CutsData {
  int F = 0;
  int max_bin = 256;
  int stride = kBins - 1;   // cuts per feature row: 255 (8-bit codes) or kMaxCuts16 (16-bit codes)
  DevBuf d_cuts;    // float [32][255]
  DevBuf d_ncuts;   // int32 [32]
  std::vector<float> h_cuts;     // [32*255]
  std::vector<int32_t> h_ncuts;  // [32]
};

// a fitted model (two ensembles, complete-binary trees)
struct ModelData {
  int F = 0, users_col = 0, T = 0, D = 0, nn = 0;
  int64_t n_train = 0;
  int device = 0;
  float base[2] = {0.f, 0.f};
  std::vector<int32_t> feat, bin;  // [2][T][nn]
  std::vector<float> thr, val;
  std::vector<double> gain;        // [2][T][nn] split losses (0 at leaves / unused slots)
  CutsData cuts;
  DevBuf d_nodes;                  // [2][T] fixed-depth routing tables on bin codes (predict.cu)
  DevBuf d_base;                   // float [2]
  DevBuf d_train_pred;             // float [2][n_train] (planar) training predictions, on the device
};

// workload generator (wg.cu): per-parameter bins (64-bin quantile cuts) and centres, the sparse
// joint histogram (ascending mixed-radix keys, cumulative counts) — PAPER.md §III-B
struct WgData {
  int P = 0;
  int64_t n = 0, m = 0;               // trace rows, non-empty joint bins
  CutsData cuts;
  std::vector<int32_t> nbins;         // [P]
  std::vector<float> centres;         // [P][64]
  std::vector<uint64_t> h_keys;       // [m]
  std::vector<int64_t> h_counts;      // [m]
  DevBuf d_keys, d_cum, d_centres, d_nbins;
};
void wg_build(Ctx* ctx, const float* T, int64_t n, int P, WgData& out);
void wg_sample(Ctx* ctx, const WgData& w, int64_t count, uint64_t seed, int64_t first, float* out);

// binning.cu
// sharded = true: this rank holds rows [row_offset, row_offset + n) of n_global and the global sample is
// all-gathered over the context's communicator (every rank must call); false: X is the whole data
// max_bin = 0: exact tree method; wide: 16-bit codes (up to 1024 bins, cut stride kMaxCuts16)
void compute_cuts(Ctx* ctx, const float* X, int64_t n, int F, int64_t row_offset, int64_t n_global, int max_bin,
                  CutsData& out, bool sharded, bool wide = false);
void compute_codes16(Ctx* ctx, const float* X, int64_t n, int F, const CutsData& cuts, uint16_t* codes);
// codes: row-major n x 32 (may be null); codesT: column-major 32 x n (may be null).
// flag (device int, may be null) is set to 1 when X holds a non-finite value.
// codesT leading dimension ldT >= n (bytes between features; the fit pads it to a multiple of 32)
void compute_codes(Ctx* ctx, const float* X, int64_t n, int F, const CutsData& cuts, uint8_t* codes, uint8_t* codesT,
                   int64_t ldT, int* flag);

// fit.cu
struct DatasetDev {  // resolved device pointers
  int64_t n, row_offset, n_global;
  int F, users_col, n_llm, n_prof;
  const float* X;
  const float* y;
  const int32_t* llm;
  const int32_t* prof;
  const float* w;
};
void fit_impl(Ctx* ctx, const DatasetDev& ds, const llmpilot_hparams& hp, float L1, float L2, ModelData& out,
              bool keep_train_pred);
void validate_hparams(const llmpilot_hparams& hp);
void compute_weights(Ctx* ctx, const DatasetDev& ds, float L1, float L2, float* w);
void debug_histogram(Ctx* ctx, const uint8_t* codes, int64_t n, const int32_t* idx, int64_t m, const int32_t* qg,
                     const int32_t* qh, int64_t* Hg, int64_t* Hh);

// predict.cu
void upload_model_nodes(Ctx* ctx, ModelData& m);
void predict_impl(Ctx* ctx, const ModelData& m, const float* X, int64_t n, float* out);
struct RecOut {
  std::vector<int32_t> profile, u_max;
  std::vector<int64_t> n_pods;
  std::vector<double> cost;
};
// pred: device [n_llm][n_prof][n_levels][2]; argmin on the device (Eq. 1-3)
void argmin_impl(Ctx* ctx, const float* pred, int n_llm, int n_prof, int n_levels, const int32_t* levels_host,
                 const double* cost_host, const uint8_t* allowed_host, float L1, float L2, int64_t U, RecOut& out);
void recommend_impl(Ctx* ctx, const ModelData& m, const float* llm_feats, int n_llm, int F_llm,
                    const float* prof_feats, int n_prof, int F_prof, const double* cost, const uint8_t* allowed,
                    const int32_t* levels, int n_levels, float L1, float L2, int64_t U, RecOut& out,
                    float* pred_out_dev);

// fit_small.cu: one thread block per (fit, ensemble) for n <= fit_small_max_rows() rows (the CV's
// fits).  Each item fits one ensemble on its rows (codes with the fit's own cuts) and writes the
// predictions of its held-out rows (column `target` of pred_test, n_test x 2).
struct SmallFitHp {
  int T, D, K, F, users_col, monotone;
  double eta, lambda, mcw;
  float subsample, colsample;
  uint64_t seed;
};
struct SmallFitItem {
  int n, m_test, target, hp;
  int n_cap;                    // set by fit_small_run (shared-memory stride)
  int cw;                       // bytes per code: 1 (<= 256 bins) or 2 (16-bit codes, up to 1024 bins)
  const uint8_t* codes;         // n x 32 codes of cw bytes, row-major (the fit's cuts)
  const uint8_t* codes_test;    // m_test x 32 (the same cuts)
  const float* y;               // n x 2
  const float* w;               // n (Eq. 4 or explicit weights)
  const int32_t* ncuts;         // [32] cuts per feature of the fit
  float* pred_test;             // m_test x 2
};
int fit_small_max_rows();
void fit_small_run(Ctx* ctx, const std::vector<SmallFitItem>& items, const std::vector<SmallFitHp>& hps);

// cv.cu
struct CvFold {
  int llm, hp_index;
  llmpilot_rec rec, truth;
  int success;
  double overspend;
  int truth_feasible;
};
void cv_impl(Ctx* ctx, const DatasetDev& ds, const llmpilot_hparams* grid, int n_grid, float L1, float L2, int64_t U,
             const double* prof_cost, std::vector<CvFold>& folds, double& S, double& O, double& SO, int& n_scored);

}  // namespace llmp
