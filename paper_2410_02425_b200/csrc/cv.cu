// cv.cu — nested leave-one-LLM-out cross-validation of the GPU recommendation tool
// (P:L207-209 hyper-parameter tuning, P:L271 protocol, P:L273-288 metrics).
//
// Orchestration only: every fit, prediction, weight and recommendation runs in the library's
// kernels; the host keeps the fold loop and the fp64 fold metrics (wMAPE, S_M, O_M, S, O, SO).
#include <math.h>

#include <algorithm>
#include <map>

#include "internal.cuh"

namespace llmp {

__global__ void k_gather_rows(const int32_t* idx, int64_t m, int F, const float* X, const float* y, const int32_t* llm,
                              const int32_t* prof, float* Xo, float* yo, int32_t* llmo, int32_t* profo) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[e];
    for (int f = 0; f < F; ++f) Xo[e * F + f] = X[i * F + f];
    yo[2 * e] = y[2 * i];
    yo[2 * e + 1] = y[2 * i + 1];
    llmo[e] = llm[i];
    profo[e] = prof[i];
  }
}

namespace {
struct Subset {
  DevBuf X, y, llm, prof, idx;
  int64_t m = 0;
  DatasetDev ds{};
};

void make_subset(Ctx* ctx, const DatasetDev& full, const std::vector<int32_t>& rows, Subset& s) {
  s.m = (int64_t)rows.size();
  const int F = full.F;
  s.idx.ensure(std::max<size_t>(rows.size(), 1) * 4);
  s.X.ensure(std::max<size_t>(rows.size(), 1) * F * 4);
  s.y.ensure(std::max<size_t>(rows.size(), 1) * 8);
  s.llm.ensure(std::max<size_t>(rows.size(), 1) * 4);
  s.prof.ensure(std::max<size_t>(rows.size(), 1) * 4);
  if (s.m > 0) {
    LLMP_CUDA(cudaMemcpyAsync(s.idx.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    int grid = (int)std::min<int64_t>((s.m + 255) / 256, (int64_t)ctx->sms * 4);
    LLMP_LAUNCH(ctx, KC_MISC, s.m, k_gather_rows, grid, 256, 0, s.idx.as<int32_t>(), s.m, F, full.X, full.y, full.llm,
                full.prof, s.X.as<float>(), s.y.as<float>(), s.llm.as<int32_t>(), s.prof.as<int32_t>());
  }
  s.ds = full;
  s.ds.n = s.m;
  s.ds.n_global = s.m;
  s.ds.row_offset = 0;
  s.ds.X = s.X.as<float>();
  s.ds.y = s.y.as<float>();
  s.ds.llm = s.llm.as<int32_t>();
  s.ds.prof = s.prof.as<int32_t>();
  s.ds.w = nullptr;
}

// fit on `train`, predict the rows of `test`; predictions copied to host (m x 2)
void fit_predict(Ctx* ctx, const Subset& train, const Subset& test, const llmpilot_hparams& hp, float L1, float L2,
                 std::vector<float>& pred_host, DevBuf& pred_dev) {
  ModelData model;
  fit_impl(ctx, train.ds, hp, L1, L2, model, false);
  pred_dev.ensure(std::max<int64_t>(test.m, 1) * 8);
  predict_impl(ctx, model, test.ds.X, test.m, pred_dev.as<float>());
  pred_host.resize((size_t)test.m * 2);
  if (test.m > 0)
    LLMP_CUDA(cudaMemcpyAsync(pred_host.data(), pred_dev.p, (size_t)test.m * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
}

// weighted MAPE, fp64, rows in order ("MAPE weighted using the sample weights of Eq. (4)")
double wmape(const std::vector<float>& pred, const std::vector<int32_t>& rows, const std::vector<float>& y,
             const std::vector<float>& w, int t) {
  double num = 0.0, den = 0.0;
  for (size_t k = 0; k < rows.size(); ++k) {
    const int32_t i = rows[k];
    const double yt = (double)y[2 * (size_t)i + t];
    num += (double)w[i] * (fabs((double)pred[2 * k + t] - yt) / fabs(yt));
    den += (double)w[i];
  }
  return den > 0.0 ? num / den : 0.0;
}
// ---------------------------------------------------------------------------------------------
// Batched small fits (fit_small.cu): every fit of a CV stage in ONE launch, one thread block per
// (fit, ensemble).  A fit is (training rows, held-out rows, hparams); its cuts (O2) come from its
// own training rows, its codes are built with them for both row sets.
struct BatchFit {
  std::vector<int32_t> tr, te;   // row indices into the full dataset (ascending)
  int hp;                        // index into the grid
};

SmallFitHp small_hp(const llmpilot_hparams& h, const DatasetDev& ds) {
  SmallFitHp s{};
  s.T = h.n_trees;
  s.D = h.max_depth;
  s.K = h.grad_bits;
  s.F = ds.F;
  s.users_col = ds.users_col;
  s.monotone = h.monotone_users;
  s.eta = (double)h.eta;
  s.lambda = (double)h.lambda;
  s.mcw = (double)h.min_child_weight;
  s.subsample = h.subsample;
  s.colsample = h.colsample_bytree;
  s.seed = h.seed;
  return s;
}

bool small_path_ok(const DatasetDev& ds, const llmpilot_hparams* grid, int n_grid) {
  static const bool off = getenv("LLMP_CV_SMALL") && atoi(getenv("LLMP_CV_SMALL")) == 0;
  if (off || ds.n > (int64_t)fit_small_max_rows()) return false;
  for (int g = 0; g < n_grid; ++g)
    if (grid[g].max_depth > 8 || grid[g].model != 0) return false;   // (the small-fit kernel is GBDT only)
  return true;
}

// predictions (m x 2 per fit, host) of every fit, in order
void run_batch(Ctx* ctx, const DatasetDev& ds, const std::vector<float>& w_host, const llmpilot_hparams* grid,
               const std::vector<BatchFit>& fits, std::vector<std::vector<float>>& preds) {
  const int F = ds.F;
  cudaStream_t s = ctx->stream;
  std::vector<SmallFitHp> hps;
  for (size_t g = 0; g < (size_t)(std::max_element(fits.begin(), fits.end(), [](const BatchFit& a, const BatchFit& b) {
                                   return a.hp < b.hp; })->hp + 1); ++g)
    hps.push_back(small_hp(grid[g], ds));
  // arena: per fit codes (train + test), y, w, ncuts, predictions
  std::vector<size_t> o_ctr(fits.size()), o_cte(fits.size()), o_y(fits.size()), o_w(fits.size()), o_nc(fits.size()),
      o_pr(fits.size());
  size_t tot = 0;
  auto take = [&](size_t bytes) {
    const size_t o = tot;
    tot += (bytes + 255) & ~(size_t)255;
    return o;
  };
  size_t max_rows = 1;
  for (size_t i = 0; i < fits.size(); ++i) {
    const size_t n = fits[i].tr.size(), m = fits[i].te.size();
    o_ctr[i] = take(n * kMaxF * 2);   // (room for 16-bit codes)
    o_cte[i] = take(std::max<size_t>(m, 1) * kMaxF * 2);
    o_y[i] = take(n * 8);
    o_w[i] = take(n * 4);
    o_nc[i] = take(kMaxF * 4);
    o_pr[i] = take(std::max<size_t>(m, 1) * 8);
    max_rows = std::max(max_rows, n + m);
  }
  DevBuf& arena = ctx->workspace("cvb_arena", tot);
  uint8_t* A = arena.as<uint8_t>();
  DevBuf& d_idx = ctx->workspace("cvb_idx", max_rows * 4);
  DevBuf& d_X = ctx->workspace("cvb_X", max_rows * F * 4);
  DevBuf& d_y = ctx->workspace("cvb_y", max_rows * 8);
  DevBuf& d_l = ctx->workspace("cvb_l", max_rows * 4);
  DevBuf& d_p = ctx->workspace("cvb_p", max_rows * 4);
  std::vector<float> wsub;
  std::vector<int32_t> idx;
  std::vector<SmallFitItem> items;
  for (size_t i = 0; i < fits.size(); ++i) {
    const BatchFit& bf = fits[i];
    const int64_t n = (int64_t)bf.tr.size(), m = (int64_t)bf.te.size();
    idx.assign(bf.tr.begin(), bf.tr.end());
    idx.insert(idx.end(), bf.te.begin(), bf.te.end());
    LLMP_CUDA(cudaMemcpyAsync(d_idx.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, s));
    const int grid_g = (int)std::min<int64_t>((n + m + 255) / 256, (int64_t)ctx->sms * 4);
    LLMP_LAUNCH(ctx, KC_MISC, n + m, k_gather_rows, grid_g, 256, 0, d_idx.as<int32_t>(), n + m, F, ds.X, ds.y, ds.llm,
                ds.prof, d_X.as<float>(), d_y.as<float>(), d_l.as<int32_t>(), d_p.as<int32_t>());
    LLMP_CUDA(cudaMemcpyAsync(A + o_y[i], d_y.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    wsub.resize(n);
    // Eq. (4) weights are per (LLM, profile) group, so a subset's weights are the full set's (O1);
    // use_eq4_weights = 0: w = 1 (a CV subset carries no explicit weights)
    const bool eq4 = grid[bf.hp].use_eq4_weights != 0;
    for (int64_t k = 0; k < n; ++k) wsub[k] = eq4 ? w_host[bf.tr[k]] : 1.0f;
    LLMP_CUDA(cudaMemcpyAsync(A + o_w[i], wsub.data(), (size_t)n * 4, cudaMemcpyHostToDevice, s));
    // O2 on the fit's rows; more than 256 bins (or exact with more than 256 distinct values) take
    // 16-bit codes (NEXT-4)
    const llmpilot_hparams& hb = grid[bf.hp];
    const bool wide = hb.tree_method == 1 || hb.max_bin > kBins;
    CutsData cuts;
    compute_cuts(ctx, d_X.as<float>(), n, F, 0, n, hb.tree_method == 1 ? 0 : hb.max_bin, cuts, false, wide);
    const int cw = wide ? 2 : 1;
    if (cw == 1) {
      compute_codes(ctx, d_X.as<float>(), n, F, cuts, A + o_ctr[i], nullptr, 0, nullptr);
      if (m > 0) compute_codes(ctx, d_X.as<float>() + (size_t)n * F, m, F, cuts, A + o_cte[i], nullptr, 0, nullptr);
    } else {
      compute_codes16(ctx, d_X.as<float>(), n, F, cuts, reinterpret_cast<uint16_t*>(A + o_ctr[i]));
      if (m > 0)
        compute_codes16(ctx, d_X.as<float>() + (size_t)n * F, m, F, cuts, reinterpret_cast<uint16_t*>(A + o_cte[i]));
    }
    LLMP_CUDA(cudaMemcpyAsync(A + o_nc[i], cuts.d_ncuts.p, kMaxF * 4, cudaMemcpyDeviceToDevice, s));
    LLMP_CUDA(cudaStreamSynchronize(s));   // wsub / cuts are reused by the next fit
    for (int tg = 0; tg < 2; ++tg) {
      SmallFitItem itm{};
      itm.n = (int)n;
      itm.m_test = (int)m;
      itm.target = tg;
      itm.hp = bf.hp;
      itm.cw = cw;
      itm.codes = A + o_ctr[i];
      itm.codes_test = A + o_cte[i];
      itm.y = reinterpret_cast<const float*>(A + o_y[i]);
      itm.w = reinterpret_cast<const float*>(A + o_w[i]);
      itm.ncuts = reinterpret_cast<const int32_t*>(A + o_nc[i]);
      itm.pred_test = reinterpret_cast<float*>(A + o_pr[i]);
      items.push_back(itm);
    }
  }
  fit_small_run(ctx, items, hps);
  preds.assign(fits.size(), {});
  for (size_t i = 0; i < fits.size(); ++i) {
    preds[i].resize(fits[i].te.size() * 2);
    if (!fits[i].te.empty())
      LLMP_CUDA(cudaMemcpyAsync(preds[i].data(), A + o_pr[i], preds[i].size() * 4, cudaMemcpyDeviceToHost, s));
  }
  LLMP_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

void cv_impl(Ctx* ctx, const DatasetDev& ds, const llmpilot_hparams* grid, int n_grid, float L1, float L2, int64_t U,
             const double* prof_cost, std::vector<CvFold>& folds, double& S, double& O, double& SO, int& n_scored) {
  LLMP_REQUIRE(ctx->nranks == 1, "cross-validation runs on one GPU per process (shard folds across ranks)");
  LLMP_REQUIRE(n_grid >= 1 && grid, "the hyper-parameter grid must hold at least one entry");
  LLMP_REQUIRE(U >= 1, "U must be >= 1");
  LLMP_REQUIRE(L1 > 0.f && L2 > 0.f, "L1, L2 must be > 0");
  LLMP_REQUIRE(ds.llm && ds.prof, "cross-validation needs llm_id and profile_id");
  for (int g = 0; g < n_grid; ++g) validate_hparams(grid[g]);
  for (int g = 0; g < ds.n_prof; ++g) LLMP_REQUIRE(prof_cost[g] > 0.0 && isfinite(prof_cost[g]), "costs must be > 0");
  const int64_t n = ds.n;
  const int F = ds.F;
  cudaStream_t s = ctx->stream;
  // host copies of the grouping columns, users and latencies; Eq. (4) weights from the kernel
  std::vector<int32_t> llm(n), prof(n);
  std::vector<float> y((size_t)n * 2), X((size_t)n * F), w(n);
  LLMP_CUDA(cudaMemcpyAsync(llm.data(), ds.llm, n * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(prof.data(), ds.prof, n * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(y.data(), ds.y, n * 8, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaMemcpyAsync(X.data(), ds.X, (size_t)n * F * 4, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) {
    LLMP_REQUIRE(llm[i] >= 0 && llm[i] < ds.n_llm && prof[i] >= 0 && prof[i] < ds.n_prof, "id out of range");
    for (int f = 0; f < F; ++f) LLMP_REQUIRE(isfinite(X[(size_t)i * F + f]), "non-finite X");
    LLMP_REQUIRE(isfinite(y[2 * i]) && isfinite(y[2 * i + 1]), "non-finite y");
  }
  {
    DevBuf& d_w = ctx->workspace("cv_w", n * 4);
    compute_weights(ctx, ds, L1, L2, d_w.as<float>());
    LLMP_CUDA(cudaMemcpyAsync(w.data(), d_w.p, n * 4, cudaMemcpyDeviceToHost, s));
    LLMP_CUDA(cudaStreamSynchronize(s));
  }
  std::vector<char> present(ds.n_llm, 0);
  for (int64_t i = 0; i < n; ++i) present[llm[i]] = 1;

  folds.clear();
  int n_feasible = 0, n_success = 0;
  double sumO = 0.0;
  Subset tr, te, trV, teV;
  DevBuf pred_dev;
  std::vector<float> pred;
  // batched path (all fits of a stage in one launch, fit_small.cu) for small datasets
  const bool batched = small_path_ok(ds, grid, n_grid);
  std::vector<int> llms;
  for (int M = 0; M < ds.n_llm; ++M)
    if (present[M]) llms.push_back(M);
  std::vector<std::vector<int32_t>> rows_of(ds.n_llm);
  for (int64_t i = 0; i < n; ++i) rows_of[llm[i]].push_back((int32_t)i);
  std::vector<int> best_of(ds.n_llm, 0);
  std::vector<std::vector<float>> outer_pred;
  if (batched) {
    if (n_grid > 1) {   // inner stage: (M, V, hp) for every ordered pair of distinct LLMs
      std::vector<BatchFit> inner;
      for (int M : llms)
        for (int V : llms) {
          if (V == M) continue;
          BatchFit bf;
          for (int64_t i = 0; i < n; ++i)
            if (llm[i] != M && llm[i] != V) bf.tr.push_back((int32_t)i);
          if (bf.tr.empty()) continue;
          bf.te = rows_of[V];
          for (int h = 0; h < n_grid; ++h) {
            bf.hp = h;
            inner.push_back(bf);
          }
        }
      std::vector<std::vector<float>> ip;
      run_batch(ctx, ds, w, grid, inner, ip);
      // err(hp) = mean over V of (wMAPE_1 + wMAPE_2)/2, V ascending (O12), first minimum wins
      size_t q = 0;
      for (int M : llms) {
        std::vector<double> err_sum(n_grid, 0.0);
        std::vector<int> nv(n_grid, 0);
        for (int V : llms) {
          if (V == M) continue;
          if (q >= inner.size() || inner[q].te != rows_of[V]) continue;   // V skipped (no training rows)
          for (int h = 0; h < n_grid; ++h, ++q) {
            err_sum[h] += 0.5 * (wmape(ip[q], rows_of[V], y, w, 0) + wmape(ip[q], rows_of[V], y, w, 1));
            ++nv[h];
          }
        }
        double best_err = INFINITY;
        for (int h = 0; h < n_grid; ++h) {
          const double err = nv[h] > 0 ? err_sum[h] / nv[h] : 0.0;
          if (err < best_err) {
            best_err = err;
            best_of[M] = h;
          }
        }
      }
    }
    std::vector<BatchFit> outer;
    for (int M : llms) {
      BatchFit bf;
      for (int64_t i = 0; i < n; ++i)
        if (llm[i] != M) bf.tr.push_back((int32_t)i);
      LLMP_REQUIRE(!bf.tr.empty(), "leave-one-LLM-out needs at least two LLMs");
      bf.te = rows_of[M];
      bf.hp = best_of[M];
      outer.push_back(bf);
    }
    run_batch(ctx, ds, w, grid, outer, outer_pred);
  }
  size_t mi = 0;
  for (int M = 0; M < ds.n_llm; ++M) {
    if (!present[M]) continue;
    std::vector<int32_t> rows_tr, rows_M;
    for (int64_t i = 0; i < n; ++i) (llm[i] == M ? rows_M : rows_tr).push_back((int32_t)i);
    LLMP_REQUIRE(!rows_tr.empty(), "leave-one-LLM-out needs at least two LLMs");
    int best_hp = 0;
    if (batched) {
      best_hp = best_of[M];
      pred = outer_pred[mi++];
    } else {
      if (n_grid > 1) {
        double best_err = INFINITY;
        for (int h = 0; h < n_grid; ++h) {
          double err_sum = 0.0;
          int nv = 0;
          for (int V = 0; V < ds.n_llm; ++V) {
            if (!present[V] || V == M) continue;
            std::vector<int32_t> r_tr, r_v;
            for (int64_t i = 0; i < n; ++i) {
              if (llm[i] == V) r_v.push_back((int32_t)i);
              else if (llm[i] != M) r_tr.push_back((int32_t)i);
            }
            if (r_tr.empty()) continue;
            make_subset(ctx, ds, r_tr, trV);
            make_subset(ctx, ds, r_v, teV);
            fit_predict(ctx, trV, teV, grid[h], L1, L2, pred, pred_dev);
            err_sum += 0.5 * (wmape(pred, r_v, y, w, 0) + wmape(pred, r_v, y, w, 1));
            ++nv;
          }
          const double err = nv > 0 ? err_sum / nv : 0.0;
          if (err < best_err) {
            best_err = err;
            best_hp = h;
          }
        }
      }
      make_subset(ctx, ds, rows_tr, tr);
      make_subset(ctx, ds, rows_M, te);
      fit_predict(ctx, tr, te, grid[best_hp], L1, L2, pred, pred_dev);
    }
    // M's measured grid: profiles present x user levels (regular grid required)
    std::vector<int32_t> levels;
    for (int32_t i : rows_M) levels.push_back((int32_t)X[(size_t)i * F + ds.users_col]);
    std::sort(levels.begin(), levels.end());
    levels.erase(std::unique(levels.begin(), levels.end()), levels.end());
    const int nL = (int)levels.size(), nP = ds.n_prof;
    std::vector<float> gp((size_t)nP * nL * 2, 0.f), gt((size_t)nP * nL * 2, 0.f);
    std::vector<int> filled((size_t)nP * nL, 0);
    std::vector<uint8_t> allowed(nP, 0);
    for (size_t k = 0; k < rows_M.size(); ++k) {
      const int32_t i = rows_M[k];
      const int g = prof[i];
      const int lv = (int)(std::lower_bound(levels.begin(), levels.end(), (int32_t)X[(size_t)i * F + ds.users_col]) -
                           levels.begin());
      const size_t c = (size_t)g * nL + lv;
      LLMP_REQUIRE(!filled[c], "held-out LLM has two rows for one (profile, users) cell");
      filled[c] = 1;
      allowed[g] = 1;
      gp[2 * c] = pred[2 * k];
      gp[2 * c + 1] = pred[2 * k + 1];
      gt[2 * c] = y[2 * (size_t)i];
      gt[2 * c + 1] = y[2 * (size_t)i + 1];
    }
    for (int g = 0; g < nP; ++g)
      if (allowed[g])
        for (int lv = 0; lv < nL; ++lv)
          LLMP_REQUIRE(filled[(size_t)g * nL + lv], "held-out LLM's (profile x users) grid is irregular");
    DevBuf& d_grid = ctx->workspace("cv_grid", (size_t)nP * nL * 2 * 4 * 2);
    LLMP_CUDA(cudaMemcpyAsync(d_grid.p, gp.data(), gp.size() * 4, cudaMemcpyHostToDevice, s));
    LLMP_CUDA(cudaMemcpyAsync(d_grid.as<float>() + gp.size(), gt.data(), gt.size() * 4, cudaMemcpyHostToDevice, s));
    RecOut rp, rt;
    argmin_impl(ctx, d_grid.as<float>(), 1, nP, nL, levels.data(), prof_cost, allowed.data(), L1, L2, U, rp);
    argmin_impl(ctx, d_grid.as<float>() + gp.size(), 1, nP, nL, levels.data(), prof_cost, allowed.data(), L1, L2, U, rt);
    // truth u_max of every profile (single-profile masks)
    CvFold fd{};
    fd.llm = M;
    fd.hp_index = best_hp;
    fd.rec = llmpilot_rec{rp.profile[0], rp.n_pods[0], rp.cost[0], rp.u_max[0]};
    fd.truth = llmpilot_rec{rt.profile[0], rt.n_pods[0], rt.cost[0], rt.u_max[0]};
    fd.truth_feasible = fd.truth.profile >= 0;
    if (fd.truth_feasible) {
      ++n_feasible;
      const int g = fd.rec.profile;
      if (g >= 0) {
        // true u_max on the recommended profile (Eq. 3 on D_M)
        std::vector<uint8_t> only(nP, 0);
        only[g] = 1;
        RecOut rg;
        argmin_impl(ctx, d_grid.as<float>() + gp.size(), 1, nP, nL, levels.data(), prof_cost, only.data(), L1, L2, U,
                    rg);
        const int64_t um_true = rg.profile[0] == g ? rg.u_max[0] : 0;
        // S_M: n(M, G*) * u_max_true(M, G*) >= U
        if (um_true > 0 && fd.rec.n_pods * um_true >= U) {
          fd.success = 1;
          ++n_success;
          fd.overspend = (fd.rec.cost - fd.truth.cost) / fd.truth.cost;  // Eq. (6)
          sumO += fd.overspend;
        }
      }
    }
    folds.push_back(fd);
  }
  S = n_feasible > 0 ? (double)n_success / n_feasible : 0.0;
  O = n_success > 0 ? sumO / n_success : 0.0;
  const double inv = std::max(0.0, 1.0 - O);
  SO = (S + inv) > 0.0 ? (2.0 * S * inv) / (S + inv) : 0.0;  // Eq. (7)
  n_scored = n_feasible;
}

}  // namespace llmp
