/* include/llmpilot.h — C-ABI of the B200-native LLM-Pilot hot path (arxiv 2410.02425).
 *
 * The library fits and evaluates LLM-Pilot's performance model (§IV-B):
 * two gradient-boosted regression-tree ensembles predicting nTTFT (l1) and ITL (l2) from
 * [LLM features | GPU-profile features | concurrent users], trained with the
 * constraint-distance sample weights of Eq. (4) and a monotone-in-users constraint
 * (P:L199-205); it then recommends the cheapest GPU profile and pod count meeting the latency
 * constraints, Eq. (1)-(3), and evaluates the whole tool with nested
 * leave-one-LLM-out cross-validation, success S_M, overspend Eq. (6) and S/O Eq. (7)
 * (P:L271-288).  Every step runs in hand-written sm_100a CUDA kernels; there is no CPU fallback.
 *
 * Conventions (all entry points):
 *  - Return an llmpilot_status; LLMP_OK == 0.  No C++ exception crosses the ABI.  On failure the
 *    call writes no partial output and llmpilot_last_error() describes the failure (thread-local).
 *  - "bulk" arrays (X, y, ids, weights, predictions) may be device pointers on the context's
 *    device OR host pointers (pageable or pinned); the library detects which with
 *    cudaPointerGetAttributes and copies host data on the context stream inside the call.
 *    Small tables (costs, user levels, hyper-parameter grids, recommendation outputs) are host.
 *  - The caller owns every input and output buffer; the library owns the opaque handles
 *    (llmpilot_ctx, llmpilot_cuts, llmpilot_model, llmpilot_cv_report) and frees them with
 *    the matching *_free / *_destroy call.
 *  - All work is enqueued on the context's CUDA stream; calls return after their outputs are
 *    complete (host outputs) or enqueued (device outputs; synchronise the stream before use).
 *  - Determinism: integer histograms and fixed-order fp64/fp32 arithmetic make every result
 *    bit-identical across runs, launch configurations and GPU counts.
 *  - Limits: 1 <= n_features <= 32, 2 <= max_bin <= 256, 1 <= max_depth <= 10,
 *    2 <= grad_bits <= 14, n_rows < 2^30 per rank.  Violations return LLMP_EINVAL.
 */
#ifndef LLMPILOT_H
#define LLMPILOT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LLMP_OK = 0,
  LLMP_EINVAL = 1,   /* bad argument: NaN/Inf in X or y, id out of range, limits above, ... */
  LLMP_ENOMEM = 2,   /* device or host allocation failed */
  LLMP_ECUDA = 3,    /* a CUDA runtime error (message has the CUDA error string) */
  LLMP_ENCCL = 4,    /* an NCCL error in a multi-GPU context */
  LLMP_EINTERNAL = 5 /* invariant violated inside the library */
} llmpilot_status;

/* Message for the last failure on the calling thread ("" if none). Valid until the next call. */
const char* llmpilot_last_error(void);
/* Library version string, e.g. "llmpilot-b200 0.1 sm_100a". */
const char* llmpilot_version(void);

typedef struct llmpilot_ctx llmpilot_ctx;
typedef struct llmpilot_cuts llmpilot_cuts;
typedef struct llmpilot_model llmpilot_model;

/* Create a context on `device` that enqueues on `cuda_stream` (a cudaStream_t; NULL = the
 * legacy default stream).  nccl_unique_id: NULL for one GPU, else a pointer to the 128-byte
 * ncclUniqueId shared by all `nranks` ranks (each rank passes its `rank`); the library then
 * row-shards fits across ranks and combines histograms with NCCL all-reduce. */
llmpilot_status llmpilot_ctx_create(int device, void* cuda_stream, const void* nccl_unique_id, int rank, int nranks,
                                    llmpilot_ctx** out);
void llmpilot_ctx_destroy(llmpilot_ctx* ctx);
/* Test / emulation communicator: nranks contexts on ONE device in one process (NCCL refuses two
 * ranks on one GPU), each with its own library-created stream.  Collectives go through device
 * memory with host barriers, so every rank must be driven by its own host thread, and all ranks
 * must issue the same sequence of calls (like NCCL).  Models are bit-identical to a one-context
 * fit of the whole data.  out: nranks handles, destroyed individually with llmpilot_ctx_destroy.
 * Errors: LLMP_EINVAL for nranks outside [1, 64]; LLMP_ECUDA if a context cannot be created. */
llmpilot_status llmpilot_ctx_create_local_group(int device, int nranks, llmpilot_ctx** out);

/* Write a fresh 128-byte ncclUniqueId into out (rank 0 calls it, then broadcasts the bytes to
 * the other ranks, e.g. over a torch.distributed process group).  LLMP_ENCCL if NCCL is absent. */
llmpilot_status llmpilot_nccl_unique_id(void* out);

/* Instrumentation (used by bench.py).  llmpilot_ctx_set_timing(ctx, every): every == 0 turns
 * timing off (fits then replay each tree from a CUDA graph); every >= 1 brackets every
 * every-th launch of each kernel class with CUDA events on the context stream (plain launches,
 * no graphs).  Stats report, per kernel class, the launches, the event-timed launches and their
 * summed milliseconds, and the rows (units) processed, since the last reset.  Class names are
 * listed by llmpilot_kernel_class_name(i) for i < LLMP_N_KERNEL_CLASSES. */
#define LLMP_N_KERNEL_CLASSES 16
typedef struct {
  uint64_t launches[LLMP_N_KERNEL_CLASSES];
  uint64_t timed[LLMP_N_KERNEL_CLASSES];  /* launches that were event-timed */
  double ms[LLMP_N_KERNEL_CLASSES];       /* summed duration of the timed launches */
  double rows[LLMP_N_KERNEL_CLASSES];     /* rows (units) each class processed (all launches) */
  uint64_t total_launches;
} llmpilot_stats;
llmpilot_status llmpilot_ctx_set_timing(llmpilot_ctx* ctx, int every);
llmpilot_status llmpilot_ctx_stats(llmpilot_ctx* ctx, llmpilot_stats* out); /* synchronises the stream */
llmpilot_status llmpilot_ctx_reset_stats(llmpilot_ctx* ctx);
const char* llmpilot_kernel_class_name(int i);

/* Characterization dataset, this rank's row shard.  Rows are
 * x = [LLM features | profile features | users]; y = (nTTFT, ITL) in the same
 * units as L1, L2.  Groups (llm_id, profile_id) define the Eq. (4)
 * normaliser; they must not straddle ranks. */
typedef struct {
  int64_t n_rows;          /* rows in this shard (>= 1) */
  int64_t row_offset;      /* global index of the first row (cut sample, row subsampling RNG) */
  int64_t n_rows_global;   /* rows over all ranks (== n_rows for one GPU) */
  int32_t n_features;      /* F, 1..32 */
  int32_t users_col;       /* column of the number of concurrent users u (monotone +1 feature) */
  int32_t n_llm;           /* llm_id in [0, n_llm) */
  int32_t n_prof;          /* profile_id in [0, n_prof) */
  const float* X;          /* n_rows x F, row-major, finite */
  const float* y;          /* n_rows x 2, row-major (nTTFT, ITL), finite */
  const int32_t* llm_id;   /* n_rows */
  const int32_t* profile_id; /* n_rows */
  const float* w;          /* optional n_rows explicit weights, used iff use_eq4_weights == 0 (NULL => 1) */
} llmpilot_dataset;

/* Hyper-parameters (number of trees, depth, learning rate, subsampling, tree method
 * = histogram, number of bins).  Defaults (llmpilot_hparams_default) follow XGBoost. */
typedef struct {
  int32_t n_trees;          /* >= 0 */
  int32_t max_depth;        /* 1..10 */
  int32_t max_bin;          /* 2..1024, number of histogram bins per feature (see tree_method) */
  int32_t grad_bits;        /* K: gradients quantised to K-bit integers per tree (2..14; default 14) */
  float eta;                /* learning rate */
  float lambda;             /* L2 regulariser on leaf weights */
  float min_child_weight;   /* minimum hessian sum per child */
  float subsample;          /* row subsampling rate per tree, (0, 1] */
  float colsample_bytree;   /* feature subsampling rate per tree, (0, 1] */
  uint64_t seed;            /* counter-based RNG seed for the two subsamplings */
  int32_t use_eq4_weights;  /* 1 = paper's Eq. (4) sample weights; 0 = dataset.w or 1 */
  int32_t monotone_users;   /* 1 = paper's monotone constraint on users */
  /* model = 1: random-forest regressor, the model of the paper's MDI importance studies ("a
   * RF regressor ... to predict the latency", "a RF regressor to predict the TTFT and ITL";
   * DESIGN R33-R36): every tree fits y itself on Poisson(1) bootstrap counts of the rows (integer
   * weights, counter-based per (tree, global row)), with ceil(max_features F) features sampled per
   * node; leaf = (float)(W / n_trees) (lambda as given, so the prediction base(0) + sum_t v_t is the
   * average of the trees); eta and colsample_bytree are ignored; requires subsample = 1 and
   * monotone_users = 0.  rf_bootstrap = 0 fits every tree on the plain weights. */
  int32_t model;            /* 0 = gradient-boosted trees (the paper's performance model), 1 = random forest */
  float max_features;       /* RF: fraction of the features sampled per node, (0, 1] */
  int32_t rf_bootstrap;     /* RF: 1 = Poisson(1) bootstrap (default), 0 = none */
  /* tree building method: 0 = hist (max_bin bins per feature), 1 = exact (every distinct
   * value of the cut sample its own bin = hist with unbounded max_bin).  More than 256 bins (16-bit
   * codes, up to 1024) are supported by the cross-validation's batched small-fit path (n <= 8192
   * rows, depth <= 8); llmpilot_fit keeps 8-bit codes and returns LLMP_EINVAL beyond 256 bins. */
  int32_t tree_method;
} llmpilot_hparams;
void llmpilot_hparams_default(llmpilot_hparams* hp); /* n_trees 100, depth 6, bins 256, K 14, eta .3,
                                                         lambda 1, mcw 1, subsample 1, colsample 1,
                                                         seed 0, eq4 1, monotone 1, model 0 (GBDT),
                                                         max_features 1, rf_bootstrap 1, tree_method 0 */

/* Quantile binning for the histogram tree method ("the number of bins for the histogram
 * tree method" is one of the tuned HPs; the exact method's cuts are every distinct value; DESIGN.md
 * R14, oracle O2): per-feature cuts from a deterministic strided sample of at
 * most 2^20 rows, then code(x) = #{cuts <= x}.  X: n x F (host or device).  cuts_in != NULL
 * reuses existing cuts; else cuts are computed from X and returned in *cuts_out (may be NULL).
 * codes_out: caller-owned DEVICE buffer of n x 32 bytes (row-major, features >= F padded with
 * code 0), may be NULL to compute cuts only. */
llmpilot_status llmpilot_bin(llmpilot_ctx* ctx, const float* X, int64_t n, int32_t F, int32_t max_bin,
                             const llmpilot_cuts* cuts_in, llmpilot_cuts** cuts_out, uint8_t* codes_out);
/* Copy cuts to host: cuts (F x 255 floats, row f holds ncuts[f] values), ncuts (F ints). */
llmpilot_status llmpilot_cuts_export(const llmpilot_cuts* cuts, int32_t* F, float* cuts_out, int32_t* ncuts_out);
void llmpilot_cuts_free(llmpilot_cuts* cuts);   /* stream-ordered release, as llmpilot_model_free */

/* Fit the two ensembles (nTTFT, ITL) on the dataset with constraints L1, L2 used by Eq. (4).
 * In a multi-GPU context every rank calls with its shard; the model is bit-identical on all. */
llmpilot_status llmpilot_fit(llmpilot_ctx* ctx, const llmpilot_dataset* ds, const llmpilot_hparams* hp, float L1,
                             float L2, llmpilot_model** out);
/* Model shape: F, n_trees, max_depth (nodes per tree = 2^(max_depth+1)-1). */
llmpilot_status llmpilot_model_info(const llmpilot_model* m, int32_t* F, int32_t* n_trees, int32_t* max_depth,
                                    int32_t* users_col);
/* Copy the model to host arrays: base[2]; feat/bin/thr/val each [2][n_trees][nodes] with
 * feat = split feature, -1 leaf, -2 unused slot; thr = cuts_f[bin] (x < thr goes left);
 * val = leaf value.  Any pointer may be NULL.  The training predictions (n_rows x 2) of the
 * last fit are returned by llmpilot_model_train_pred when train_pred != NULL. */
llmpilot_status llmpilot_model_export(const llmpilot_model* m, float* base, int32_t* feat, int32_t* bin, float* thr,
                                      float* val);
llmpilot_status llmpilot_model_train_pred(const llmpilot_model* m, float* train_pred /* host, n_rows x 2 */);
/* Split losses ((gain(L) + gain(R)) - gain(parent), fp64) of every split node,
 * [2][n_trees][nodes] host doubles, 0 at leaves and unused slots. */
llmpilot_status llmpilot_model_gains(const llmpilot_model* m, double* gain);
/* MDI feature importance (Mean Decrease in Impurity, §III-B P:L120 and §III-D
 * P:L156-158).  For weighted squared error a split's impurity decrease is its
 * loss G_L^2/(H_L+lambda) + G_R^2/(H_R+lambda) - G^2/(H+lambda) (the weighted SSE decrease when
 * lambda = 0).  out (host, 2 x F doubles, target-major): per target, the losses of the splits on
 * each feature summed over the trees in order and each tree's nodes in index order; if normalize
 * != 0, divided by the target's total (all zeros when the ensemble has no split).
 * Errors: LLMP_EINVAL for NULL arguments. */
llmpilot_status llmpilot_model_importance(const llmpilot_model* m, int32_t normalize, double* out);
/* Persist a model to a file and load it back (optional model save/load; the paper
 * persists only its dataset).  Little-endian binary: magic "LLMPMDL1", shape (F, users_col,
 * n_trees, max_depth), base[2], the cuts (F x 255 floats + F counts) and feat/bin/thr/val/gain
 * [2][n_trees][nodes].  A loaded model predicts, recommends and exports bit-identically to the
 * saved one; its device tables live on ctx's device.  Errors: LLMP_EINVAL for NULL arguments, an
 * unreadable or malformed file (bad magic, sizes out of range, short read). */
llmpilot_status llmpilot_model_save(const llmpilot_model* m, const char* path);
llmpilot_status llmpilot_model_load(llmpilot_ctx* ctx, const char* path, llmpilot_model** out);
/* Free a model.  Its device buffers are released stream-ordered (cudaFreeAsync into the
 * device's default memory pool, which keeps the memory cached) on the stream of the context
 * that fitted it: free a model before destroying that stream, and only after work that reads the
 * model on other streams has completed.  Never synchronises the device. */
void llmpilot_model_free(llmpilot_model* m);

/* Predict both targets: out[i] = (nTTFT, ITL) = base + sum over trees in order.
 * X: n x F (host or device), finite (the rows are binned with the model's cuts and routed on codes,
 * code <= b <=> x < cut: LLMP_EINVAL for NaN/Inf); out: n x 2 (host or device). */
llmpilot_status llmpilot_predict(llmpilot_ctx* ctx, const llmpilot_model* m, const float* X, int64_t n, float* out);

/* Recommendation (Eq. 1-3): for each unseen LLM i, rows [llm_feats[i] | prof_feats[g] | u]
 * for every profile g and level u are assembled on the device, predicted, and
 *   u_max(i,g) = largest u whose whole prefix u' <= u meets l1 <= L1 and l2 <= L2 (Eq. 3),
 *   n(i,g) = ceil(U / u_max) (Eq. 2), G* = argmin_g n * cost[g] (Eq. 1), ties -> lowest g.
 * llm_feats: n_llm x F_llm, prof_feats: n_prof x F_prof (host or device); F_llm + F_prof + 1
 * must equal the model's F with users at column F_llm + F_prof.  prof_cost: host, > 0.
 * allowed: host n_llm x n_prof mask or NULL.  user_levels: host, strictly increasing, > 0.
 * The feature tables must be finite (LLMP_EINVAL otherwise).
 * out: host n_llm records; infeasible => profile -1, n_pods 0, cost +inf, u_max 0.
 * pred_out (optional, host or device): n_llm x n_prof x n_levels x 2 predictions. */
typedef struct {
  int32_t profile;
  int64_t n_pods;
  double cost;
  int32_t u_max;
} llmpilot_rec;
llmpilot_status llmpilot_recommend(llmpilot_ctx* ctx, const llmpilot_model* m, const float* llm_feats, int32_t n_llm,
                                   int32_t F_llm, const float* prof_feats, int32_t n_prof, int32_t F_prof,
                                   const double* prof_cost, const uint8_t* allowed, const int32_t* user_levels,
                                   int32_t n_levels, float L1, float L2, int64_t U, llmpilot_rec* out,
                                   float* pred_out);

/* Nested leave-one-LLM-out cross-validation.  For each LLM M present
 * (ascending id): if n_grid > 1, each grid entry is scored by the mean over inner held-out
 * LLMs V != M of (wMAPE_1 + wMAPE_2)/2 with Eq. (4) weights, the argmin (first on ties) is
 * refit on all rows not of M; M's rows (its measured profiles x user levels, a regular grid)
 * are predicted and Eq. (1)-(3) give the recommendation; the same rule on M's measured latencies
 * gives the truth.  S = mean success over LLMs with a truly feasible profile, O = mean
 * overspend (Eq. 6) over successes, SO = Eq. (7).  prof_cost: host, n_prof entries. */
typedef struct {
  int32_t llm;
  int32_t hp_index;
  llmpilot_rec rec, truth;
  int32_t success;
  double overspend;
  int32_t truth_feasible;
} llmpilot_cv_fold;
typedef struct {
  double S, O, SO;
  int32_t n_folds, n_scored;
  llmpilot_cv_fold* folds; /* library-owned, n_folds entries */
} llmpilot_cv_report;
llmpilot_status llmpilot_cv_leave_one_llm_out(llmpilot_ctx* ctx, const llmpilot_dataset* ds,
                                              const llmpilot_hparams* grid, int32_t n_grid, float L1, float L2,
                                              int64_t U, const double* prof_cost, llmpilot_cv_report** out);
void llmpilot_cv_report_free(llmpilot_cv_report* r);

/* ---- Workload generator (§III-B "Workload generator").
 * Request model: for each of the P request parameters the values are divided into 64 bins of
 * approximately equal request counts — one bin per distinct value when the parameter has at most
 * 64 — using the same quantile rule as llmpilot_bin (exact on <= 2^20 rows, a global
 * strided sample beyond); each bin's centre is (min + max) / 2 of the trace values in it; the joint
 * model is the sparse histogram of the rows' bin tuples, keyed by the mixed-radix
 * key sum_p bin_p * prod_{q<p} nbins_q (must fit 63 bits, else LLMP_EINVAL).
 * traces: n x P floats, row-major, host or device, finite (LLMP_EINVAL otherwise); 1 <= n < 2^31,
 * 1 <= P <= 32.  The handle owns its device buffers (release with llmpilot_wg_free). */
typedef struct llmpilot_wg llmpilot_wg;
llmpilot_status llmpilot_wg_build(llmpilot_ctx* ctx, const float* traces, int64_t n, int32_t P, llmpilot_wg** out);
/* P, trace rows, number of non-empty joint bins (any pointer may be NULL). */
llmpilot_status llmpilot_wg_info(const llmpilot_wg* w, int32_t* P, int64_t* n_rows, int64_t* n_nonempty);
/* Host copies: nbins [P], centres [P][64] (bin b of parameter p at p*64+b), keys [n_nonempty]
 * ascending, counts [n_nonempty] (sum = n_rows).  Any pointer may be NULL. */
llmpilot_status llmpilot_wg_export(const llmpilot_wg* w, int32_t* nbins, float* centres, uint64_t* keys,
                                   int64_t* counts);
/* Sampling: request s (s = first .. first + n_samples - 1) draws r = rng4(seed, 0x5747, s, 0)
 * (splitmix64 chain, R21), t = floor(r * n_rows / 2^64), takes the first joint bin (key
 * order) whose cumulative count exceeds t — i.e. a bin with probability count / n_rows — and emits
 * each parameter's bin centre.  out: n_samples x P floats, host or device.  Samples are indexed
 * globally, so shards (first = rank * chunk) draw disjoint, reproducible requests. */
llmpilot_status llmpilot_wg_sample(llmpilot_ctx* ctx, const llmpilot_wg* w, int64_t n_samples, uint64_t seed,
                                   int64_t first, float* out);
void llmpilot_wg_free(llmpilot_wg* w);

/* Test hook (parity of the histogram kernel): int64 histograms
 * Hg, Hh [32][256] (host) of the rows listed in idx (device int32, m entries; NULL = all n rows
 * in order) over codes (device n x 32) with integer gradient pairs qg, qh (device int32,
 * |qg| <= 2^14, 0 <= qh <= 2^14) — computed by the same kernel the fit uses. */
llmpilot_status llmpilot_debug_histogram(llmpilot_ctx* ctx, const uint8_t* codes, int64_t n, const int32_t* idx,
                                         int64_t m, const int32_t* qg, const int32_t* qh, int64_t* Hg, int64_t* Hh);

#ifdef __cplusplus
}
#endif
#endif /* LLMPILOT_H */
