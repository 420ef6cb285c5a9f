// api.cu — the extern "C" boundary (include/llmpilot.h).  Converts exceptions to status codes,
// resolves host/device pointers, and owns the opaque handles.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <new>

#include <stdio.h>

#include "internal.cuh"

struct llmpilot_ctx {
  llmp::Ctx c;
};
struct llmpilot_cuts {
  llmp::CutsData d;
};
struct llmpilot_model {
  llmp::ModelData m;
};
struct llmpilot_wg {
  llmp::WgData w;
};

namespace {
thread_local std::string g_err;

template <class Fn>
llmpilot_status guarded(Fn&& fn) {
  try {
    g_err.clear();
    fn();
    return LLMP_OK;
  } catch (const llmp::Error& e) {
    g_err = e.msg;
    return e.st;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return LLMP_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LLMP_EINTERNAL;
  } catch (...) {
    g_err = "unknown internal error";
    return LLMP_EINTERNAL;
  }
}

const char* kClassNames[LLMP_N_KERNEL_CLASSES] = {
    "validate", "weights", "cuts", "codes", "base_score", "hist_root", "partition", "hist_level",
    "split", "update", "predict", "recommend", "misc", "nccl", "wg", "fit_small"};

void set_device(llmp::Ctx* c) { LLMP_CUDA(cudaSetDevice(c->device)); }

// resolve a dataset's bulk arrays to device pointers (copies host arrays on the ctx stream)
struct ResolvedDataset {
  llmp::DevBuf X, y, llm, prof, w;
  llmp::DatasetDev d{};
};
void resolve(llmp::Ctx* ctx, const llmpilot_dataset* ds, ResolvedDataset& r) {
  LLMP_REQUIRE(ds != nullptr, "dataset is NULL");
  LLMP_REQUIRE(ds->n_rows >= 1, "n_rows must be >= 1");
  LLMP_REQUIRE(ds->n_features >= 1 && ds->n_features <= llmp::kMaxF, "n_features must be in [1, 32]");
  LLMP_REQUIRE(ds->X && ds->y, "X and y are required");
  LLMP_REQUIRE(ds->users_col >= 0 && ds->users_col < ds->n_features, "users_col out of range");
  LLMP_REQUIRE(ds->row_offset >= 0 && ds->n_rows_global >= ds->row_offset + ds->n_rows, "bad shard geometry");
  const size_t n = (size_t)ds->n_rows;
  r.d.n = ds->n_rows;
  r.d.row_offset = ds->row_offset;
  r.d.n_global = ds->n_rows_global;
  r.d.F = ds->n_features;
  r.d.users_col = ds->users_col;
  r.d.n_llm = ds->n_llm;
  r.d.n_prof = ds->n_prof;
  // host arrays land in grow-only context workspaces (no per-call cudaMalloc)
  r.d.X = (const float*)llmp::to_device(ctx, ds->X, n * ds->n_features * 4, ctx->ws["in_X"]);
  r.d.y = (const float*)llmp::to_device(ctx, ds->y, n * 8, ctx->ws["in_y"]);
  r.d.llm = (const int32_t*)llmp::to_device(ctx, ds->llm_id, n * 4, ctx->ws["in_llm"]);
  r.d.prof = (const int32_t*)llmp::to_device(ctx, ds->profile_id, n * 4, ctx->ws["in_prof"]);
  r.d.w = (const float*)llmp::to_device(ctx, ds->w, n * 4, ctx->ws["in_w"]);
}
}  // namespace

extern "C" {

const char* llmpilot_last_error(void) { return g_err.c_str(); }
const char* llmpilot_version(void) { return "llmpilot-b200 0.1 sm_100a"; }

llmpilot_status llmpilot_ctx_create(int device, void* cuda_stream, const void* nccl_unique_id, int rank, int nranks,
                                    llmpilot_ctx** out) {
  return guarded([&] {
    LLMP_REQUIRE(out != nullptr, "out is NULL");
    LLMP_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    LLMP_REQUIRE(nranks == 1 || nccl_unique_id != nullptr, "multi-rank contexts need an ncclUniqueId");
    int ndev = 0;
    LLMP_CUDA(cudaGetDeviceCount(&ndev));
    LLMP_REQUIRE(device >= 0 && device < ndev, "device out of range");
    auto* h = new llmpilot_ctx();
    h->c.device = device;
    h->c.stream = (cudaStream_t)cuda_stream;
    h->c.rank = rank;
    h->c.nranks = nranks;
    try {
      set_device(&h->c);
      cudaDeviceProp prop;
      LLMP_CUDA(cudaGetDeviceProperties(&prop, device));
      LLMP_REQUIRE(prop.major >= 10, "this library is built for sm_100a (B200); device is older");
      h->c.sms = prop.multiProcessorCount;
      {  // model/cuts buffers come from the default pool (stream-ordered): keep freed memory cached
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
          uint64_t thr = UINT64_MAX;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
      }
      LLMP_CUDA(cudaMalloc(&h->c.d_units, LLMP_N_KERNEL_CLASSES * 8));
      LLMP_CUDA(cudaMemset(h->c.d_units, 0, LLMP_N_KERNEL_CLASSES * 8));
      if (nccl_unique_id) llmp::nccl_init(&h->c, nccl_unique_id);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

llmpilot_status llmpilot_ctx_create_local_group(int device, int nranks, llmpilot_ctx** out) {
  return guarded([&] {
    LLMP_REQUIRE(out != nullptr, "out is NULL");
    LLMP_REQUIRE(nranks >= 1 && nranks <= 64, "nranks must be in [1, 64]");
    for (int r = 0; r < nranks; ++r) out[r] = nullptr;
    llmp::LocalGroup* g = llmp::local_group_create(nranks);
    int made = 0;
    try {
      for (int r = 0; r < nranks; ++r) {
        llmpilot_ctx* c = nullptr;
        const llmpilot_status st = llmpilot_ctx_create(device, nullptr, nullptr, 0, 1, &c);
        if (st != LLMP_OK) llmp::fail(st, g_err);
        c->c.rank = r;
        c->c.nranks = nranks;
        c->c.lgroup = g;
        LLMP_CUDA(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
        c->c.own_stream = true;
        out[r] = c;
        ++made;
      }
    } catch (...) {
      for (int r = 0; r < made; ++r) llmpilot_ctx_destroy(out[r]);   // each release drops one reference
      for (int r = made; r < nranks; ++r) llmp::local_group_release(g);
      throw;
    }
  });
}

llmpilot_status llmpilot_nccl_unique_id(void* out) {
  return guarded([&] {
    LLMP_REQUIRE(out != nullptr, "out is NULL");
    llmp::nccl_unique_id(out);
  });
}

void llmpilot_ctx_destroy(llmpilot_ctx* ctx) {
  if (!ctx) return;
  try {
    ctx->c.collect();
  } catch (...) {
  }
  for (auto e : ctx->c.free_events) cudaEventDestroy(e);
  llmp::nccl_destroy(&ctx->c);
  llmp::local_group_release(ctx->c.lgroup);
  if (ctx->c.own_stream && ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  if (ctx->c.d_units) cudaFree(ctx->c.d_units);
  for (auto st : ctx->c.cap_stream)
    if (st) cudaStreamDestroy(st);
  if (ctx->c.fork_event) cudaEventDestroy(ctx->c.fork_event);
  if (ctx->c.join_event) cudaEventDestroy(ctx->c.join_event);
  delete ctx;
}

llmpilot_status llmpilot_ctx_set_timing(llmpilot_ctx* ctx, int every) {
  return guarded([&] {
    LLMP_REQUIRE(ctx, "ctx is NULL");
    LLMP_REQUIRE(every >= 0, "every must be >= 0");
    ctx->c.collect();
    ctx->c.timing = every != 0;
    ctx->c.timing_every = every > 0 ? every : 1;
  });
}

llmpilot_status llmpilot_ctx_stats(llmpilot_ctx* ctx, llmpilot_stats* out) {
  return guarded([&] {
    LLMP_REQUIRE(ctx && out, "NULL argument");
    set_device(&ctx->c);
    ctx->c.collect();
    LLMP_CUDA(cudaStreamSynchronize(ctx->c.stream));
    memset(out, 0, sizeof(*out));
    unsigned long long units[LLMP_N_KERNEL_CLASSES];
    LLMP_CUDA(cudaMemcpy(units, ctx->c.d_units, sizeof(units), cudaMemcpyDeviceToHost));
    for (int i = 0; i < LLMP_N_KERNEL_CLASSES; ++i) {
      out->launches[i] = ctx->c.launches[i];
      out->timed[i] = ctx->c.timed[i];
      out->ms[i] = ctx->c.ms_done[i];
      const bool dev_counted = i == llmp::KC_HIST_ROOT || i == llmp::KC_HIST || i == llmp::KC_PARTITION;
      out->rows[i] = dev_counted ? (double)units[i] : ctx->c.rows[i];
      if (i != llmp::KC_NCCL) out->total_launches += ctx->c.launches[i];
    }
  });
}

llmpilot_status llmpilot_ctx_reset_stats(llmpilot_ctx* ctx) {
  return guarded([&] {
    LLMP_REQUIRE(ctx, "ctx is NULL");
    ctx->c.collect();
    for (int i = 0; i < LLMP_N_KERNEL_CLASSES; ++i) {
      ctx->c.launches[i] = 0;
      ctx->c.timed[i] = 0;
      ctx->c.ms_done[i] = 0;
      ctx->c.rows[i] = 0;
    }
    LLMP_CUDA(cudaMemsetAsync(ctx->c.d_units, 0, LLMP_N_KERNEL_CLASSES * 8, ctx->c.stream));
  });
}

const char* llmpilot_kernel_class_name(int i) {
  return (i >= 0 && i < LLMP_N_KERNEL_CLASSES) ? kClassNames[i] : "";
}

void llmpilot_hparams_default(llmpilot_hparams* hp) {
  if (!hp) return;
  hp->n_trees = 100;
  hp->max_depth = 6;
  hp->max_bin = 256;
  hp->grad_bits = 14;
  hp->eta = 0.3f;
  hp->lambda = 1.0f;
  hp->min_child_weight = 1.0f;
  hp->subsample = 1.0f;
  hp->colsample_bytree = 1.0f;
  hp->seed = 0;
  hp->use_eq4_weights = 1;
  hp->monotone_users = 1;
  hp->model = 0;
  hp->max_features = 1.0f;
  hp->rf_bootstrap = 1;
  hp->tree_method = 0;
}

llmpilot_status llmpilot_bin(llmpilot_ctx* ctx, const float* X, int64_t n, int32_t F, int32_t max_bin,
                             const llmpilot_cuts* cuts_in, llmpilot_cuts** cuts_out, uint8_t* codes_out) {
  return guarded([&] {
    llmp::NvtxRange nvtx_("llmpilot_bin");
    LLMP_REQUIRE(ctx && X, "NULL argument");
    LLMP_REQUIRE(n >= 1 && F >= 1 && F <= llmp::kMaxF, "bad sizes");
    LLMP_REQUIRE(!codes_out || llmp::is_device_ptr(codes_out), "codes_out must be a device buffer");
    set_device(&ctx->c);
    llmp::DevBuf tmp;
    const float* Xd = (const float*)llmp::to_device(&ctx->c, X, (size_t)n * F * 4, tmp);
    llmpilot_cuts* made = nullptr;
    const llmp::CutsData* cuts = nullptr;
    if (cuts_in) {
      LLMP_REQUIRE(cuts_in->d.F == F, "cuts were made for a different number of features");
      cuts = &cuts_in->d;
    } else {
      made = new llmpilot_cuts();
      try {
        llmp::compute_cuts(&ctx->c, Xd, n, F, 0, n, max_bin, made->d, false);   // this rank's X only
      } catch (...) {
        delete made;
        throw;
      }
      cuts = &made->d;
    }
    try {
      if (codes_out) {
        llmp::DevBuf flag(sizeof(int));
        LLMP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->c.stream));
        llmp::compute_codes(&ctx->c, Xd, n, F, *cuts, codes_out, nullptr, n, flag.as<int>());
        int hf = 0;
        LLMP_CUDA(cudaMemcpyAsync(&hf, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->c.stream));
        LLMP_CUDA(cudaStreamSynchronize(ctx->c.stream));
        LLMP_REQUIRE(hf == 0, "X holds a non-finite value");
      }
    } catch (...) {
      delete made;
      throw;
    }
    if (made) {
      if (cuts_out) *cuts_out = made;
      else delete made;
    }
  });
}

llmpilot_status llmpilot_cuts_export(const llmpilot_cuts* cuts, int32_t* F, float* cuts_out, int32_t* ncuts_out) {
  return guarded([&] {
    LLMP_REQUIRE(cuts, "cuts is NULL");
    const int f = cuts->d.F;
    if (F) *F = f;
    for (int i = 0; i < f; ++i) {
      if (ncuts_out) ncuts_out[i] = cuts->d.h_ncuts[i];
      if (cuts_out) memcpy(cuts_out + (size_t)i * 255, cuts->d.h_cuts.data() + (size_t)i * 255, 255 * 4);
    }
  });
}

void llmpilot_cuts_free(llmpilot_cuts* cuts) { delete cuts; }

llmpilot_status llmpilot_fit(llmpilot_ctx* ctx, const llmpilot_dataset* ds, const llmpilot_hparams* hp, float L1,
                             float L2, llmpilot_model** out) {
  return guarded([&] {
    llmp::NvtxRange nvtx_("llmpilot_fit");
    LLMP_REQUIRE(ctx && ds && hp && out, "NULL argument");
    set_device(&ctx->c);
    ResolvedDataset r;
    resolve(&ctx->c, ds, r);
    auto* m = new llmpilot_model();
    try {
      llmp::fit_impl(&ctx->c, r.d, *hp, L1, L2, m->m, true);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

llmpilot_status llmpilot_model_info(const llmpilot_model* m, int32_t* F, int32_t* n_trees, int32_t* max_depth,
                                    int32_t* users_col) {
  return guarded([&] {
    LLMP_REQUIRE(m, "model is NULL");
    if (F) *F = m->m.F;
    if (n_trees) *n_trees = m->m.T;
    if (max_depth) *max_depth = m->m.D;
    if (users_col) *users_col = m->m.users_col;
  });
}

llmpilot_status llmpilot_model_export(const llmpilot_model* m, float* base, int32_t* feat, int32_t* bin, float* thr,
                                      float* val) {
  return guarded([&] {
    LLMP_REQUIRE(m, "model is NULL");
    const size_t tot = m->m.feat.size();
    if (base) memcpy(base, m->m.base, 8);
    if (feat) memcpy(feat, m->m.feat.data(), tot * 4);
    if (bin) memcpy(bin, m->m.bin.data(), tot * 4);
    if (thr) memcpy(thr, m->m.thr.data(), tot * 4);
    if (val) memcpy(val, m->m.val.data(), tot * 4);
  });
}

llmpilot_status llmpilot_model_gains(const llmpilot_model* m, double* gain) {
  return guarded([&] {
    LLMP_REQUIRE(m && gain, "NULL argument");
    memcpy(gain, m->m.gain.data(), m->m.gain.size() * 8);
  });
}

// MDI: per target, split losses summed by feature over trees in order
// and nodes in index order (fp64, the order the oracle uses), optionally divided by the total
llmpilot_status llmpilot_model_importance(const llmpilot_model* m, int32_t normalize, double* out) {
  return guarded([&] {
    LLMP_REQUIRE(m && out, "NULL argument");
    const llmp::ModelData& md = m->m;
    const int F = md.F;
    for (int tg = 0; tg < 2; ++tg) {
      double* o = out + (size_t)tg * F;
      for (int f = 0; f < F; ++f) o[f] = 0.0;
      for (int t = 0; t < md.T; ++t) {
        const size_t off = ((size_t)tg * md.T + t) * md.nn;
        for (int k = 0; k < md.nn; ++k)
          if (md.feat[off + k] >= 0) o[md.feat[off + k]] += md.gain[off + k];
      }
      if (normalize) {
        double tot = 0.0;
        for (int f = 0; f < F; ++f) tot += o[f];
        if (tot > 0.0)
          for (int f = 0; f < F; ++f) o[f] = o[f] / tot;
      }
    }
  });
}

llmpilot_status llmpilot_model_train_pred(const llmpilot_model* m, float* train_pred) {
  return guarded([&] {
    LLMP_REQUIRE(m && train_pred, "NULL argument");
    LLMP_REQUIRE(m->m.d_train_pred.p != nullptr, "no training predictions kept");
    const int64_t n = m->m.n_train;
    std::vector<float> planar((size_t)n * 2);
    LLMP_CUDA(cudaSetDevice(m->m.device));
    LLMP_CUDA(cudaMemcpy(planar.data(), m->m.d_train_pred.p, (size_t)n * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) {
      train_pred[2 * i] = planar[i];
      train_pred[2 * i + 1] = planar[n + i];
    }
  });
}

void llmpilot_model_free(llmpilot_model* m) { delete m; }

namespace {
constexpr char kModelMagic[8] = {'L', 'L', 'M', 'P', 'M', 'D', 'L', '1'};
}

llmpilot_status llmpilot_model_save(const llmpilot_model* m, const char* path) {
  return guarded([&] {
    LLMP_REQUIRE(m && path, "NULL argument");
    const llmp::ModelData& d = m->m;
    LLMP_REQUIRE(d.cuts.stride == llmp::kBins - 1, "only 8-bit-code models are persisted");
    FILE* fp = fopen(path, "wb");
    LLMP_REQUIRE(fp != nullptr, std::string("cannot open ") + path + " for writing");
    const int32_t hdr[4] = {d.F, d.users_col, d.T, d.D};
    const size_t tot = (size_t)2 * d.T * d.nn;
    bool ok = fwrite(kModelMagic, 1, 8, fp) == 8 && fwrite(hdr, 4, 4, fp) == 4 && fwrite(d.base, 4, 2, fp) == 2 &&
              fwrite(d.cuts.h_cuts.data(), 4, (size_t)d.F * 255, fp) == (size_t)d.F * 255 &&
              fwrite(d.cuts.h_ncuts.data(), 4, (size_t)d.F, fp) == (size_t)d.F;
    ok = ok && fwrite(d.feat.data(), 4, tot, fp) == tot && fwrite(d.bin.data(), 4, tot, fp) == tot &&
         fwrite(d.thr.data(), 4, tot, fp) == tot && fwrite(d.val.data(), 4, tot, fp) == tot &&
         fwrite(d.gain.data(), 8, tot, fp) == tot;
    ok = (fclose(fp) == 0) && ok;
    LLMP_REQUIRE(ok, std::string("write failed: ") + path);
  });
}

llmpilot_status llmpilot_model_load(llmpilot_ctx* ctx, const char* path, llmpilot_model** out) {
  return guarded([&] {
    llmp::NvtxRange nvtx_("llmpilot_model_load");
    LLMP_REQUIRE(ctx && path && out, "NULL argument");
    FILE* fp = fopen(path, "rb");
    LLMP_REQUIRE(fp != nullptr, std::string("cannot open ") + path);
    auto* mo = new llmpilot_model();
    try {
      char mg[8];
      int32_t hdr[4];
      bool ok = fread(mg, 1, 8, fp) == 8 && memcmp(mg, kModelMagic, 8) == 0 && fread(hdr, 4, 4, fp) == 4;
      LLMP_REQUIRE(ok, "not an llmpilot model file");
      llmp::ModelData& d = mo->m;
      d.F = hdr[0];
      d.users_col = hdr[1];
      d.T = hdr[2];
      d.D = hdr[3];
      LLMP_REQUIRE(d.F >= 1 && d.F <= llmp::kMaxF && d.users_col >= 0 && d.users_col < d.F && d.T >= 0 &&
                       d.T <= (1 << 24) && d.D >= 1 && d.D <= llmp::kMaxDepth,
                   "model file: shape out of range");
      d.nn = (1 << (d.D + 1)) - 1;
      const size_t tot = (size_t)2 * d.T * d.nn;
      d.cuts.F = d.F;
      d.cuts.stride = llmp::kBins - 1;
      d.cuts.h_cuts.assign((size_t)llmp::kMaxF * 255, 0.f);
      d.cuts.h_ncuts.assign(llmp::kMaxF, 0);
      d.feat.resize(tot);
      d.bin.resize(tot);
      d.thr.resize(tot);
      d.val.resize(tot);
      d.gain.resize(tot);
      ok = fread(d.base, 4, 2, fp) == 2 && fread(d.cuts.h_cuts.data(), 4, (size_t)d.F * 255, fp) == (size_t)d.F * 255 &&
           fread(d.cuts.h_ncuts.data(), 4, (size_t)d.F, fp) == (size_t)d.F && fread(d.feat.data(), 4, tot, fp) == tot &&
           fread(d.bin.data(), 4, tot, fp) == tot && fread(d.thr.data(), 4, tot, fp) == tot &&
           fread(d.val.data(), 4, tot, fp) == tot && fread(d.gain.data(), 8, tot, fp) == tot;
      LLMP_REQUIRE(ok, "model file: short read");
      for (int f = 0; f < d.F; ++f) LLMP_REQUIRE(d.cuts.h_ncuts[f] >= 0 && d.cuts.h_ncuts[f] <= 255, "model file: bad cuts");
      for (size_t i = 0; i < tot; ++i)
        LLMP_REQUIRE(d.feat[i] >= -2 && d.feat[i] < d.F && d.bin[i] >= 0 && d.bin[i] <= 255, "model file: bad node");
      fclose(fp);
      fp = nullptr;
      set_device(&ctx->c);
      d.device = ctx->c.device;
      d.cuts.d_cuts.set_stream(ctx->c.stream);
      d.cuts.d_ncuts.set_stream(ctx->c.stream);
      d.cuts.d_cuts.ensure((size_t)llmp::kMaxF * 255 * 4);
      d.cuts.d_ncuts.ensure((size_t)llmp::kMaxF * 4);
      LLMP_CUDA(cudaMemcpyAsync(d.cuts.d_cuts.p, d.cuts.h_cuts.data(), (size_t)llmp::kMaxF * 255 * 4,
                                cudaMemcpyHostToDevice, ctx->c.stream));
      LLMP_CUDA(cudaMemcpyAsync(d.cuts.d_ncuts.p, d.cuts.h_ncuts.data(), (size_t)llmp::kMaxF * 4, cudaMemcpyHostToDevice,
                                ctx->c.stream));
      llmp::upload_model_nodes(&ctx->c, d);   // (synchronises the stream)
      *out = mo;
    } catch (...) {
      if (fp) fclose(fp);
      delete mo;
      throw;
    }
  });
}

// ---- workload generator (§III-B)
llmpilot_status llmpilot_wg_build(llmpilot_ctx* ctx, const float* traces, int64_t n, int32_t P, llmpilot_wg** out) {
  return guarded([&] {
    LLMP_REQUIRE(ctx && traces && out, "NULL argument");
    LLMP_REQUIRE(n >= 1 && n < (int64_t(1) << 31) && P >= 1 && P <= llmp::kMaxF, "bad sizes (n in [1, 2^31), P in [1, 32])");
    set_device(&ctx->c);
    llmp::DevBuf tmp;
    const float* Td = (const float*)llmp::to_device(&ctx->c, traces, (size_t)n * P * 4, tmp);
    llmpilot_wg* w = new llmpilot_wg();
    try {
      llmp::wg_build(&ctx->c, Td, n, P, w->w);
    } catch (...) {
      delete w;
      throw;
    }
    *out = w;
  });
}

llmpilot_status llmpilot_wg_info(const llmpilot_wg* w, int32_t* P, int64_t* n_rows, int64_t* n_nonempty) {
  return guarded([&] {
    LLMP_REQUIRE(w, "NULL argument");
    if (P) *P = w->w.P;
    if (n_rows) *n_rows = w->w.n;
    if (n_nonempty) *n_nonempty = w->w.m;
  });
}

llmpilot_status llmpilot_wg_export(const llmpilot_wg* w, int32_t* nbins, float* centres, uint64_t* keys,
                                   int64_t* counts) {
  return guarded([&] {
    LLMP_REQUIRE(w, "NULL argument");
    const llmp::WgData& d = w->w;
    if (nbins) memcpy(nbins, d.nbins.data(), (size_t)d.P * 4);
    if (centres) memcpy(centres, d.centres.data(), (size_t)d.P * 64 * 4);
    if (keys) memcpy(keys, d.h_keys.data(), (size_t)d.m * 8);
    if (counts) memcpy(counts, d.h_counts.data(), (size_t)d.m * 8);
  });
}

llmpilot_status llmpilot_wg_sample(llmpilot_ctx* ctx, const llmpilot_wg* w, int64_t n_samples, uint64_t seed,
                                   int64_t first, float* out) {
  return guarded([&] {
    LLMP_REQUIRE(ctx && w && (out || n_samples == 0), "NULL argument");
    set_device(&ctx->c);
    const size_t bytes = (size_t)n_samples * w->w.P * 4;
    if (llmp::is_device_ptr(out)) {
      llmp::wg_sample(&ctx->c, w->w, n_samples, seed, first, out);
    } else {
      llmp::DevBuf& d = ctx->c.workspace("wg_out", std::max<size_t>(bytes, 4));
      llmp::wg_sample(&ctx->c, w->w, n_samples, seed, first, d.as<float>());
      LLMP_CUDA(cudaMemcpyAsync(out, d.p, bytes, cudaMemcpyDeviceToHost, ctx->c.stream));
      LLMP_CUDA(cudaStreamSynchronize(ctx->c.stream));
    }
  });
}

void llmpilot_wg_free(llmpilot_wg* w) { delete w; }

llmpilot_status llmpilot_predict(llmpilot_ctx* ctx, const llmpilot_model* m, const float* X, int64_t n, float* out) {
  return guarded([&] {
    llmp::NvtxRange nvtx_("llmpilot_predict");
    LLMP_REQUIRE(ctx && m && X && out, "NULL argument");
    LLMP_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return;
    set_device(&ctx->c);
    const float* Xd = (const float*)llmp::to_device(&ctx->c, X, (size_t)n * m->m.F * 4, ctx->c.ws["pred_X"]);
    const bool out_dev = llmp::is_device_ptr(out);
    float* od = out;
    if (!out_dev) od = ctx->c.workspace("pred_out", (size_t)n * 8).as<float>();
    llmp::predict_impl(&ctx->c, m->m, Xd, n, od);
    if (!out_dev) {
      LLMP_CUDA(cudaMemcpyAsync(out, od, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
      LLMP_CUDA(cudaStreamSynchronize(ctx->c.stream));
    }
  });
}

llmpilot_status llmpilot_recommend(llmpilot_ctx* ctx, const llmpilot_model* m, const float* llm_feats, int32_t n_llm,
                                   int32_t F_llm, const float* prof_feats, int32_t n_prof, int32_t F_prof,
                                   const double* prof_cost, const uint8_t* allowed, const int32_t* user_levels,
                                   int32_t n_levels, float L1, float L2, int64_t U, llmpilot_rec* out,
                                   float* pred_out) {
  return guarded([&] {
    llmp::NvtxRange nvtx_("llmpilot_recommend");
    LLMP_REQUIRE(ctx && m && out && prof_cost && user_levels, "NULL argument");
    LLMP_REQUIRE(n_llm >= 0 && n_prof >= 1 && n_levels >= 1, "bad sizes");
    LLMP_REQUIRE(F_llm >= 0 && F_prof >= 0 && F_llm + F_prof + 1 == m->m.F, "F_llm + F_prof + 1 must equal the model's F");
    LLMP_REQUIRE(m->m.users_col == F_llm + F_prof, "the model's users column must be the last column");
    LLMP_REQUIRE(U >= 1, "U must be >= 1");
    LLMP_REQUIRE(L1 > 0.f && L2 > 0.f && isfinite(L1) && isfinite(L2), "L1, L2 must be positive and finite");
    for (int k = 0; k < n_levels; ++k) {
      LLMP_REQUIRE(user_levels[k] > 0, "user levels must be > 0");
      LLMP_REQUIRE(k == 0 || user_levels[k] > user_levels[k - 1], "user levels must be strictly increasing");
    }
    for (int g = 0; g < n_prof; ++g) LLMP_REQUIRE(prof_cost[g] > 0.0 && isfinite(prof_cost[g]), "costs must be > 0");
    if (n_llm == 0) return;
    LLMP_REQUIRE((F_llm == 0 || llm_feats) && (F_prof == 0 || prof_feats), "feature tables are required");
    set_device(&ctx->c);
    llmp::DevBuf tpred;
    const float* lf =
        (const float*)llmp::to_device(&ctx->c, llm_feats, (size_t)n_llm * F_llm * 4, ctx->c.ws["rec_llm"]);
    const float* pf =
        (const float*)llmp::to_device(&ctx->c, prof_feats, (size_t)n_prof * F_prof * 4, ctx->c.ws["rec_prof"]);
    const int64_t nrows = (int64_t)n_llm * n_prof * n_levels;
    // predictions requested on the host: one pass into a device buffer, then one copy
    const bool pred_is_dev = pred_out && llmp::is_device_ptr(pred_out);
    if (pred_out && !pred_is_dev) tpred.ensure((size_t)nrows * 8);
    float* pred_dev = pred_is_dev ? pred_out : (pred_out ? tpred.as<float>() : nullptr);
    llmp::RecOut r;
    llmp::recommend_impl(&ctx->c, m->m, lf, n_llm, F_llm, pf, n_prof, F_prof, prof_cost, allowed, user_levels, n_levels,
                         L1, L2, U, r, pred_dev);
    if (pred_out && !pred_is_dev) {
      LLMP_CUDA(cudaMemcpyAsync(pred_out, tpred.p, (size_t)nrows * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
      LLMP_CUDA(cudaStreamSynchronize(ctx->c.stream));
    }
    for (int i = 0; i < n_llm; ++i) out[i] = llmpilot_rec{r.profile[i], r.n_pods[i], r.cost[i], r.u_max[i]};
  });
}

llmpilot_status llmpilot_cv_leave_one_llm_out(llmpilot_ctx* ctx, const llmpilot_dataset* ds,
                                              const llmpilot_hparams* grid, int32_t n_grid, float L1, float L2,
                                              int64_t U, const double* prof_cost, llmpilot_cv_report** out) {
  return guarded([&] {
    llmp::NvtxRange nvtx_("llmpilot_cv_leave_one_llm_out");
    LLMP_REQUIRE(ctx && ds && grid && prof_cost && out, "NULL argument");
    LLMP_REQUIRE(ds->n_llm >= 2 && ds->n_prof >= 1, "need n_llm >= 2 and n_prof >= 1");
    LLMP_REQUIRE(ds->llm_id && ds->profile_id, "llm_id and profile_id are required");
    set_device(&ctx->c);
    ResolvedDataset r;
    resolve(&ctx->c, ds, r);
    std::vector<llmp::CvFold> folds;
    double S = 0, O = 0, SO = 0;
    int scored = 0;
    llmp::cv_impl(&ctx->c, r.d, grid, n_grid, L1, L2, U, prof_cost, folds, S, O, SO, scored);
    auto* rep = new llmpilot_cv_report();
    rep->S = S;
    rep->O = O;
    rep->SO = SO;
    rep->n_folds = (int32_t)folds.size();
    rep->n_scored = scored;
    rep->folds = new llmpilot_cv_fold[std::max<size_t>(folds.size(), 1)];
    for (size_t i = 0; i < folds.size(); ++i) {
      const auto& f = folds[i];
      rep->folds[i] = llmpilot_cv_fold{f.llm, f.hp_index, f.rec, f.truth, f.success, f.overspend, f.truth_feasible};
    }
    *out = rep;
  });
}

void llmpilot_cv_report_free(llmpilot_cv_report* r) {
  if (!r) return;
  delete[] r->folds;
  delete r;
}

llmpilot_status llmpilot_debug_histogram(llmpilot_ctx* ctx, const uint8_t* codes, int64_t n, const int32_t* idx,
                                         int64_t m, const int32_t* qg, const int32_t* qh, int64_t* Hg, int64_t* Hh) {
  return guarded([&] {
    LLMP_REQUIRE(ctx && codes && qg && qh && Hg && Hh, "NULL argument");
    LLMP_REQUIRE(llmp::is_device_ptr(codes) && llmp::is_device_ptr(qg) && llmp::is_device_ptr(qh),
                 "codes, qg, qh must be device buffers");
    LLMP_REQUIRE(!idx || llmp::is_device_ptr(idx), "idx must be a device buffer");
    set_device(&ctx->c);
    llmp::debug_histogram(&ctx->c, codes, n, idx, m, qg, qh, Hg, Hh);
  });
}

}  // extern "C"
