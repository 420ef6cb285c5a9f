// fit.cu — LLM-Pilot performance-model training on B200 (§IV-B).
//
// Two gradient-boosted regression-tree ensembles (nTTFT, ITL) with Eq. (4) sample weights and
// a monotone constraint on users, grown level-wise with quantised integer gradients so every
// histogram is an exact, order-free integer sum:
//
//   per tree t:   k_hist<ROOT>   root histogram over all rows (identity order), fused with the
//                                gradient computation + quantisation (writes gp_root)
//                 k_split3(0)
//                 for d = 1..D-1:
//                   k_part(d)       partition of the split parents' row indices into children
//                                   (2048-row tiles, one atomic reservation per child per tile);
//                                   zeroes the built-child histograms
//                   k_hist<LEVEL>   histogram of the smaller child of each split parent (codes
//                                   and packed gradient pairs gathered by row index)
//                   k_split3(d)     sibling = parent - built; prefix scan; fp64 gains; argmax
//                 k_hist<UPDROOT>(t)  route every row to its leaf, p += v, and build tree t+1's
//                                   root histogram (k_update when unfused)
//
// No host synchronisation happens inside the tree loop; all decisions live on the device.
#include <float.h>
#include <math.h>

#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <memory>

#include "bulk.cuh"
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace llmp {

// ---------------------------------------------------------------------------------------------
constexpr int HIST_THREADS = 512;
constexpr int HIST_WARPS = HIST_THREADS / 32;
constexpr int HIST_CHUNK = 65536;          // rows per CTA between flushes: |sum q_g| < 2^30 in int32
constexpr int ROWBUF_STRIDE = 48;          // bytes per staged code row (conflict-free 16B stores)
constexpr int MAX_PIECES = 512;            // built children per level (2^(kMaxDepth-1))
// shared histogram: [257 bin rows][32 features] int32 for q_g, then the same for q_h; bin row 256 is
// a dummy cell row (the users lane's run target, see k_hist)
constexpr int HH_OFF = (kBins + 1) * kMaxF * 4;   // byte offset of the q_h half (32,896)
constexpr int U_OFF = 2 * HH_OFF + HIST_WARPS * 32 * ROWBUF_STRIDE;     // users column: [256] q_g, [256] q_h
constexpr int GS_OFF = U_OFF + 2 * kBins * 4;                                // per warp: 8 four-row group sums (uint2)
constexpr int HIST_SMEM = GS_OFF + HIST_WARPS * 8 * 8;                       // 64.3 KB + 24 KB + 2 KB + 1 KB

constexpr int SLOT = 2 * kHistBins;        // int64 per histogram slot (g then h)
constexpr int FQ_INTS = 2 + 2 * MAX_PIECES; // fold-in queue: head, tail, one slot per piece of a launch


__device__ __forceinline__ double exp2i(int e) {  // exact 2^e for e in [-1022, 1023]
  return __longlong_as_double((long long)(e + 1023) << 52);
}

struct LevelView {
  int64_t* start;    // [2^d] segment start in the row-index buffer (a child lies inside its parent's range)
  int64_t* cnt;      // [2^d] local rows
  int64_t* gcnt;     // [2^d] (unused: kept for the table layout)
  double* lo;        // [2^d] monotone bounds
  double* hi;
  int32_t* split_f;  // [2^d] -1 = leaf / absent
  int32_t* split_b;
  int32_t* built;    // [2^(d-1)] which child of parent j was histogrammed (0 left, 1 right)
  int32_t* done;     // [2^d] per-node count of finished split warps (self-resetting; plain k_split3)
};

// best split of one (node, feature), published by the split kernel for the node's final reduction
struct FeatBest {
  double loss;
  int32_t b, valid;
  int64_t GLq, HLq, Gq, Hq;
};

struct FitArgs {
  int64_t n, row_offset;
  int F, users_col, D, K, T, target;
  const uint8_t* codes;
  const uint8_t* codesT;
  int64_t ldT;       // codesT leading dimension: n rounded up to 32 (aligned 32-row vectors)
  const float* y;
  const float* w;
  float* p;
  uint32_t* gp_root;
  uint32_t* sr[2];   // row-index ping-pong buffers, n each (level d's segments in sr[d & 1])
  int64_t* H[2];
  LevelView lv[kMaxDepth + 1];
  const int* d_tree; // device-side index of the tree being grown (advanced by k_next_tree)
  uint32_t* maxg;    // [T+1] float bits of max |g| per tree (slot T: base score)
  uint32_t* maxh;
  const float* cuts;     // [32][255]
  const int32_t* ncuts;  // [32]
  int32_t* tfeat;        // [T][nn] this target's trees
  int32_t* tbin;
  float* tthr;
  float* tval;
  double* tgain;         // [T][nn] split losses (MDI importance), 0 elsewhere
  double eta, lambda, mcw;
  float subsample, colsample;
  uint64_t seed;
  int monotone;
  int fused_root;     // 1: k_hist<UPDROOT> builds the next root speculatively (root_needed)
  int urow;           // 1: the histogram kernels take the users column row-parallel
  int hist_swar;      // 1: k_hist's four-row fast path (group sums when no run changes)
  int built_by_h;     // 1 (sharded): the split kernel picks the built child by hessian sum
  int rf, rf_boot;    // random forest (DESIGN R33-R36): bootstrap weights, per-node features, leaf W / T
  float max_features;
  const float* w_base;  // RF: the rows' weights before the bootstrap (w then holds the current tree's)
  int* fq;              // fold-in work queue of the level histogram (k_hist3): [0] head, [1] tail, slots
  const uint32_t* cmask;  // [n/32 batches][32 lanes] precomputed change masks (k_cmask), or null
  int64_t* hroot;         // h_fixed: the root's q_h histogram (tree-invariant), saved at tree 0
  int nn;
  FeatBest* fbest;            // [2^(D-1)][32] per-(node, feature) best split of the current level
  unsigned long long* units;  // device counters of rows processed per kernel class (instrumentation)
};

// both ensembles' arguments: every tree-loop kernel runs the two (independent) targets as
// blockIdx.y = 0, 1 of one launch — one stream, one launch per step for both trees
struct FitPair {
  FitArgs t[2];
};

// debug-mode inputs of the histogram kernel
struct DbgArgs {
  const int32_t* idx;
  const int32_t* qg;
  const int32_t* qh;
  int64_t m;
  int64_t* out;  // one slot
};

// row sampling decision: keep iff u < subsample, u = top 53 bits / 2^53
__device__ __forceinline__ bool row_sampled_out(uint64_t seed, int target, int t, int64_t gi, float subsample) {
  if (subsample >= 1.0f) return false;
  uint64_t r = rng4(seed, (uint64_t)(2 * target), (uint64_t)t, (uint64_t)gi);
  double u = (double)(r >> 11) * 0x1.0p-53;
  return u >= (double)subsample;
}

// RF bootstrap count of (tree t, global row gi) (DESIGN R34): Poisson(1) by inversion of the top 53
// bits of rng4(seed, 0x5246, t, gi), the terms and the running sum in fp64 in the oracle's order
__device__ __forceinline__ int poisson1(uint64_t seed, int t, int64_t gi) {
  const double u = (double)(rng4(seed, 0x5246u, (uint64_t)t, (uint64_t)gi) >> 11) * 0x1.0p-53;
  double p = 0x1.78b56362cef38p-2;   // e^-1 rounded to double
  double F = p;
  int k = 0;
  while (u >= F && k < 16) {
    ++k;
    p = __ddiv_rn(p, (double)k);
    F = __dadd_rn(F, p);
  }
  return k;
}

// O4 gradient pair of global row gi for tree t: weighted squared error g = w (p - y), h = w, zeroed
// when the row is sampled out.  Random forest (R33, R34): every tree fits y itself (p = 0), and `w`
// is then the tree's bootstrap weight c_t,i w (a.w points at the per-tree buffer k_rf_weights fills),
// so the hot kernels carry no bootstrap arithmetic
__device__ __forceinline__ void grad_pair(const FitArgs& a, int t, int64_t gi, float y, float w, float p, float& g,
                                          float& h) {
  g = __fmul_rn(w, __fsub_rn(a.rf ? 0.0f : p, y));
  h = w;
  if (row_sampled_out(a.seed, a.target, t, gi, a.subsample)) {
    g = 0.f;
    h = 0.f;
  }
}

// O8 leaf value: (float)(eta W); random forest (R36): (float)(W / T), the trees' average
__device__ __forceinline__ float leaf_value(const FitArgs& a, double W) {
  return a.rf ? (float)__ddiv_rn(W, (double)a.T) : (float)__dmul_rn(a.eta, W);
}

// slot of node k at level d inside H[d&1]: built child of parent j -> j, sibling -> 2^(d-1)+j
__device__ __forceinline__ int node_slot(const FitArgs& a, int d, int k) {
  if (d == 0) return 0;
  int j = k >> 1;
  int side = a.lv[d].built[j];
  return ((k & 1) == side) ? j : (1 << (d - 1)) + j;
}

// ---------------------------------------------------------------------------------------------
// histogram kernel: lane = feature, one row per warp step, run-length aggregation of equal
// consecutive codes in registers, 32-bit shared atomics on change, zero-skipping int64 flush
enum { HM_ROOT = 0, HM_LEVEL = 1, HM_DEBUG = 2, HM_UPDROOT = 3 };

// Fused update + next root (HM_UPDROOT): the update pass of tree t also builds tree
// t+1's root histogram, quantising tree t+1's gradients with tree t's exponents e (O4) — the
// speculation that max|g| and max h keep their binary exponent from one tree to the next (true for
// ~99% of trees: the maxima shrink slowly).  Tree t+1's own maxima are computed in the same pass;
// when an exponent did change, the speculative histogram and packed pairs are discarded: k_root_fix
// zeroes the root slot and k_hist<ROOT> rebuilds both with the right scale.  Every histogram is
// therefore exactly the one O4-O6 define, whichever way it was built.
__device__ __forceinline__ bool root_needed(const FitArgs& a, int t) {
  if (!a.fused_root || t == 0) return true;
  return exp_of(__uint_as_float(a.maxg[t])) != exp_of(__uint_as_float(a.maxg[t - 1])) ||
         exp_of(__uint_as_float(a.maxh[t])) != exp_of(__uint_as_float(a.maxh[t - 1]));
}
// one tree in shared memory after the histogram kernels' dynamic smem, sized for the fit's depth
// (nnp = nn + 1 = 2^(D+1)): k_hist: s_feat (int8, nnp), s_bin (u8, nnp), s_val (f32, nnp);
// k_hist2: the fixed-depth routing table (s_rt: u16 x 2^D node words, s_lv: f32 x 2^D).
// Depth 8 adds 3 KB (two CTAs per SM); depth 10 adds 12 KB.
__host__ __device__ constexpr int updroot_tree_smem(int D) { return 6 << (D + 1); }

// One row of a lane's run-length aggregation: if the row's cell address `ca` differs from the
// current run's `pa`, flush the run (two 32-bit shared reductions) and start a new one; then add
// the row's (q_g, q_h), stored unpacked so one 64-bit shared load fetches both.  The common
// no-change path is compare, branch, two adds.
constexpr uint32_t kNoRun = 0xffffffffu;
__device__ __forceinline__ void run_flush(uint32_t pa, int32_t ag, uint32_t ah) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(pa), "r"(ag) : "memory");
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(pa), "r"(ah), "n"(HH_OFF) : "memory");
}
// The run is tracked by its code byte; the cell address sbase + code * cstride is formed only when a run
// is flushed (the users lane reads a never-written padding byte, so its run never changes).
__device__ __forceinline__ void run_step(uint32_t& pc, int32_t& ag, uint32_t& ah, uint32_t c, uint2 gh,
                                         uint32_t sbase, uint32_t cstride) {
  if (c != pc) {
    run_flush(sbase + pc * cstride, ag, ah);
    ag = 0;
    ah = 0;
    pc = c;
  }
  ag += (int32_t)gh.x;
  ah += gh.y;
}

template <int MODE>
__global__ void __launch_bounds__(HIST_THREADS, 2) k_hist(const FitPair fp, const int d, const int t_in, const DbgArgs dbg) {
  pdl_wait();
  const FitArgs& a = fp.t[blockIdx.y];
  const int t = (MODE == HM_ROOT || MODE == HM_UPDROOT) ? *a.d_tree : t_in;   // graph replays: tree index from the device
  if (MODE == HM_ROOT && !root_needed(a, t)) return;   // built speculatively by the previous update pass
  const bool has_next = (MODE == HM_UPDROOT) ? (t + 1 < a.T) : true;
  const int ucol = (a.urow && a.users_col >= 0 && a.users_col < kMaxF) ? a.users_col : -1;   // row-parallel column
  extern __shared__ __align__(16) uint8_t smem[];
  int32_t* sg = reinterpret_cast<int32_t*>(smem);                 // [256 bins][32 features]
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem + HH_OFF);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* rowbuf = smem + 2 * HH_OFF + warp * 32 * ROWBUF_STRIDE;
  uint2* gsum = reinterpret_cast<uint2*>(smem + GS_OFF) + warp * 8;

  __shared__ int64_t s_vstart[MAX_PIECES + 1];
  __shared__ int64_t s_pstart[MAX_PIECES];
  __shared__ int32_t s_slot[MAX_PIECES];
  __shared__ int s_np;

  int32_t* sug = reinterpret_cast<int32_t*>(smem + U_OFF);   // users column (row-parallel), bank = bin
  uint32_t* suh = reinterpret_cast<uint32_t*>(smem + U_OFF + kBins * 4);
  for (int i = tid; i < kHistBins; i += HIST_THREADS) {
    sg[i] = 0;
    sh[i] = 0;
  }
  for (int i = tid; i < kBins; i += HIST_THREADS) {
    sug[i] = 0;
    suh[i] = 0;
  }
  // staged-row padding bytes 40..47 are never written afterwards: zero them once (the users lane
  // compares byte 40 of every row, which must therefore never change)
  for (int i = tid; i < HIST_WARPS * 32; i += HIST_THREADS)
    *reinterpret_cast<uint2*>(smem + 2 * HH_OFF + i * ROWBUF_STRIDE + 40) = make_uint2(0u, 0u);
  // fused mode: tree t (the one just grown) in shared memory for routing
  int8_t* s_feat = reinterpret_cast<int8_t*>(smem + HIST_SMEM);
  uint8_t* s_bin = smem + HIST_SMEM + (a.nn + 1);
  float* s_val = reinterpret_cast<float*>(smem + HIST_SMEM + 2 * (a.nn + 1));
  if (MODE == HM_UPDROOT) {
    const size_t to = (size_t)t * a.nn;
    for (int i = tid; i < a.nn; i += HIST_THREADS) {
      const int f = a.tfeat[to + i];
      s_feat[i] = (int8_t)(f < 0 ? -1 : f);
      s_bin[i] = (uint8_t)a.tbin[to + i];
      s_val[i] = a.tval[to + i];
    }
  }
  // ---- piece list (virtual concatenation of the rows to histogram)
  if (MODE == HM_LEVEL) {
    const int NP = 1 << (d - 1);
    const LevelView& P = a.lv[d - 1];
    const LevelView& C = a.lv[d];
    // one parent per thread (NP <= 512 <= HIST_THREADS)
    int64_t len = 0, pst = 0;
    int side = 0;
    bool sp = false;
    if (tid < NP) {
      sp = P.split_f[tid] >= 0;
      if (sp) {
        const int64_t nL = C.cnt[2 * tid], nR = C.cnt[2 * tid + 1];
        side = a.built_by_h ? C.built[tid] : (nL <= nR) ? 0 : 1;   // the smaller child (rows; hessian when sharded)
        len = C.cnt[2 * tid + side];
        // k_part: left child at the parent's start, right child after it
        const int64_t ps = (d == 1) ? 0 : P.start[tid], cl = C.cnt[2 * tid];
        pst = side ? ps + cl : ps;
        if (blockIdx.x == 0) {
          C.built[tid] = side;
          C.start[2 * tid] = ps;
          C.start[2 * tid + 1] = ps + cl;
        }
      }
    }
    // block exclusive scan of len over 512 threads
    __shared__ int64_t s_wsum[HIST_WARPS];
    int64_t v = len;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) s_wsum[warp] = v;
    __syncthreads();
    int64_t woff = 0;
    for (int w2 = 0; w2 < warp; ++w2) woff += s_wsum[w2];
    if (tid < NP) {
      s_vstart[tid] = woff + v - len;
      s_pstart[tid] = pst;
      s_slot[tid] = tid;
    }
    if (tid == NP - 1) s_vstart[NP] = woff + v;
    if (tid == 0) s_np = NP;
  } else {
    if (tid == 0) {
      s_np = 1;
      s_vstart[0] = 0;
      s_vstart[1] = (MODE == HM_ROOT || MODE == HM_UPDROOT) ? a.n : dbg.m;
      s_pstart[0] = 0;
      s_slot[0] = 0;
    }
  }
  __syncthreads();
  const int np = s_np;
  const int64_t S = s_vstart[np];
  const int64_t v0 = S * blockIdx.x / gridDim.x, v1 = S * (blockIdx.x + 1) / gridDim.x;
  if (v0 >= v1) return;
  if (tid == 0 && MODE != HM_DEBUG && a.units)
    atomicAdd(&a.units[MODE == HM_ROOT ? KC_HIST_ROOT : MODE == HM_UPDROOT ? KC_UPDATE : KC_HIST], (unsigned long long)(v1 - v0));

  // quantisation scales for ROOT (tree t): q = rint(v * 2^(K-e))
  // (HM_UPDROOT: tree t+1's pairs with tree t's exponents — the speculation described above)
  double scale_g = 0.0, scale_h = 0.0;
  if (MODE == HM_ROOT || MODE == HM_UPDROOT) {
    scale_g = exp2i(a.K - exp_of(__uint_as_float(a.maxg[t])));
    scale_h = exp2i(a.K - exp_of(__uint_as_float(a.maxh[t])));
  }
  float mg = 0.f, mh = 0.f;   // HM_UPDROOT: tree t+1's max |g|, max h
  int64_t* Hbase = (MODE == HM_DEBUG) ? dbg.out : a.H[d & 1];
  const uint32_t* sr_in = (MODE == HM_LEVEL) ? a.sr[d & 1] : nullptr;

  // first piece overlapping [v0, v1)
  int pc = 0;
  while (pc + 1 < np && s_vstart[pc + 1] <= v0) ++pc;
  for (; pc < np && s_vstart[pc] < v1; ++pc) {
    int64_t s0 = max(v0, s_vstart[pc]), s1 = min(v1, s_vstart[pc + 1]);
    if (s0 >= s1) continue;
    int64_t* Hg = Hbase + (size_t)s_slot[pc] * SLOT;
    int64_t* Hh = Hg + kHistBins;
    for (int64_t c0 = s0; c0 < s1; c0 += HIST_CHUNK) {
      const int64_t c1 = min(s1, c0 + HIST_CHUNK);
      const int64_t clen = c1 - c0;
      // contiguous sub-range per warp; rows staged 32 at a time in the warp's smem buffer
      // (bytes 0..31 = the row's codes, bytes 32..35 = its packed gradient pair)
      const int64_t w0 = c0 + clen * warp / HIST_WARPS, w1 = c0 + clen * (warp + 1) / HIST_WARPS;

      // The users column changes on nearly every row of paper-ordered data, so run-length
      // aggregation cannot help it and its flushes would make the whole warp take the flush branch
      // on every row: it is histogrammed row-parallel by the loader lanes instead (two shared
      // reductions per 32-row batch), and its lane's runs target the dummy bin row (never read).
      const uint32_t sg0 = (uint32_t)__cvta_generic_to_shared(sg);
      const uint32_t su0 = (uint32_t)__cvta_generic_to_shared(sug);
      const bool ulane = lane == ucol;
      const uint32_t sbase = ulane ? sg0 + (uint32_t)(kBins * 128) + (uint32_t)lane * 4u : sg0 + (uint32_t)lane * 4u;
      const uint32_t cstride = ulane ? 0u : 128u;
      const int ccol = ulane ? 40 : lane;   // staged byte this lane compares (40: row padding, never written)
      uint32_t rc = kNoRun;       // code of the current run's (bin, feature) cell
      int32_t ag = 0;             // run sums
      uint32_t ah = 0;
      // register prefetch of the first batch
      uint4 nc0 = make_uint4(0, 0, 0, 0), nc1 = nc0;
      uint32_t ngp = 0;
      float ny = 0.f, nw = 0.f, np_ = 0.f;
      // HM_LEVEL: row indices run two batches ahead of the gathers (one exposed round trip per batch)
      uint32_t nri = 0;
      auto load_ridx = [&](int64_t base) {
        const int64_t vi = base + lane;
        if (MODE == HM_LEVEL && vi < w1) nri = sr_in[s_pstart[pc] + (vi - s_vstart[pc])];
      };
      auto load_batch = [&](int64_t base) {
        const int64_t vi = base + lane;
        if (vi < w1) {
          const int64_t pi = s_pstart[pc] + (vi - s_vstart[pc]);  // physical position
          int64_t ridx;
          if (MODE == HM_ROOT || MODE == HM_UPDROOT) {
            ridx = pi;
            ny = a.y[ridx];
            nw = a.w[ridx];
            np_ = a.p[ridx];
          } else if (MODE == HM_LEVEL) {
            ridx = nri;              // loaded by load_ridx(base)
            ngp = a.gp_root[ridx];   // gathered by row index (written by this tree's root pass)
          } else {
            ridx = dbg.idx ? dbg.idx[pi] : pi;
            ngp = pack_gp(dbg.qg[ridx], dbg.qh[ridx]);
          }
          const uint4* crow = reinterpret_cast<const uint4*>(a.codes + (size_t)ridx * kMaxF);
          nc0 = __ldg(crow);
          nc1 = __ldg(crow + 1);
        }
      };
      if (w0 < w1) {
        load_ridx(w0);
        load_batch(w0);
        load_ridx(w0 + 32);
      }
      for (int64_t base = w0; base < w1; base += 32) {
        const int cnt = (int)min((int64_t)32, w1 - base);
        uint32_t gp = ngp;
        if (MODE == HM_ROOT && lane < cnt) {
          const int64_t ridx = base + lane + (s_pstart[pc] - s_vstart[pc]);
          float g, h;
          grad_pair(a, t, a.row_offset + ridx, ny, nw, np_, g, h);
          gp = pack_gp(quantize(g, scale_g), quantize(h, scale_h));
          a.gp_root[ridx] = gp;
        }
        __syncwarp();   // previous batch fully consumed
        *reinterpret_cast<uint4*>(rowbuf + lane * ROWBUF_STRIDE) = nc0;
        *reinterpret_cast<uint4*>(rowbuf + lane * ROWBUF_STRIDE + 16) = nc1;
        if (MODE == HM_UPDROOT && lane < cnt) {
          // O9 for tree t (route the lane's own staged row, p += v), then O4 for tree t+1
          const int64_t ridx = base + lane + (s_pstart[pc] - s_vstart[pc]);
          int k = 0;
          for (int s2 = 0; s2 < a.D; ++s2) {
            const int f = s_feat[k];
            if (f >= 0) k = 2 * k + 1 + (rowbuf[lane * ROWBUF_STRIDE + f] > s_bin[k] ? 1 : 0);
          }
          const float pn = __fadd_rn(np_, s_val[k]);   // one fp32 rounding, tree order
          a.p[ridx] = pn;
          if (has_next) {
            float g, h;
            grad_pair(a, t + 1, a.row_offset + ridx, ny, nw, pn, g, h);
            mg = fmaxf(mg, fabsf(g));
            mh = fmaxf(mh, h);
            gp = pack_gp(quantize(g, scale_g), quantize(h, scale_h));
            a.gp_root[ridx] = gp;
          }
        }
        *reinterpret_cast<uint2*>(rowbuf + lane * ROWBUF_STRIDE + 32) = make_uint2((uint32_t)gp_g(gp), (uint32_t)gp_h(gp));
        if (a.hist_swar) {   // (q_g, q_h) sums of the batch's four-row groups (lane = row)
          int32_t gx = lane < cnt ? gp_g(gp) : 0;
          uint32_t hx = lane < cnt ? (uint32_t)gp_h(gp) : 0u;
          gx += __shfl_xor_sync(0xffffffffu, gx, 1);
          hx += __shfl_xor_sync(0xffffffffu, hx, 1);
          gx += __shfl_xor_sync(0xffffffffu, gx, 2);
          hx += __shfl_xor_sync(0xffffffffu, hx, 2);
          if ((lane & 3) == 0) gsum[lane >> 2] = make_uint2((uint32_t)gx, hx);
        }
        __syncwarp();
        if (base + 32 < w1) {   // prefetch the next batch (and the row indices of the one after)
          load_batch(base + 32);
          load_ridx(base + 64);
        }
        if (MODE == HM_UPDROOT && !has_next) continue;   // last tree: update only
        if (ucol >= 0 && lane < cnt) {   // users column, row-parallel (lane = row)
          const uint32_t cu = rowbuf[lane * ROWBUF_STRIDE + ucol];
          const uint2 ghu = *reinterpret_cast<const uint2*>(rowbuf + lane * ROWBUF_STRIDE + 32);
          const uint32_t ua = su0 + cu * 4u;   // dense per-bin cells: distinct bins, distinct banks
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(ua), "r"((int32_t)ghu.x) : "memory");
          asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(ua), "r"(ghu.y), "n"(kBins * 4) : "memory");
        }
        if (rc == kNoRun) rc = rowbuf[ccol];
        int r = 0;
        for (; r + 4 <= cnt; r += 4) {   // the group's shared loads first, then 4 branch-free steps
          uint32_t ca[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) ca[q] = rowbuf[(r + q) * ROWBUF_STRIDE + ccol];
          // four-row fast path: when no lane's run changes inside the group (most groups of the
          // child lists), every lane adds the group's precomputed sums in one step
          if (a.hist_swar &&
              __all_sync(0xffffffffu, (ca[0] == rc) & (ca[1] == rc) & (ca[2] == rc) & (ca[3] == rc))) {
            const uint2 gs = gsum[r >> 2];
            ag += (int32_t)gs.x;
            ah += gs.y;
            continue;
          }
          uint2 gh[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) gh[q] = *reinterpret_cast<const uint2*>(rowbuf + (r + q) * ROWBUF_STRIDE + 32);
#pragma unroll
          for (int q = 0; q < 4; ++q) run_step(rc, ag, ah, ca[q], gh[q], sbase, cstride);
        }
        for (; r < cnt; ++r)
          run_step(rc, ag, ah, rowbuf[r * ROWBUF_STRIDE + ccol], *reinterpret_cast<const uint2*>(rowbuf + r * ROWBUF_STRIDE + 32),
                   sbase, cstride);
      }
      if (rc != kNoRun) run_flush(sbase + rc * cstride, ag, ah);
      __syncthreads();
      if (ucol >= 0) {   // the users column's cells (left zero by its lane) from the dense histogram
        for (int b = tid; b < kBins; b += HIST_THREADS) {
          sg[b * 32 + ucol] = sug[b];
          sh[b * 32 + ucol] = suh[b];
          sug[b] = 0;
          suh[b] = 0;
        }
        __syncthreads();
      }
      // flush: zero-skipping int64 atomics into the node histogram ([f][b] layout)
      for (int i = tid; i < kHistBins; i += HIST_THREADS) {
        const int32_t g = sg[i];
        const uint32_t h = sh[i];
        if (g != 0 || h != 0) {
          const int b = i >> 5, f = i & 31;
          atomicAdd(reinterpret_cast<unsigned long long*>(&Hg[f * kBins + b]), (unsigned long long)(long long)g);
          atomicAdd(reinterpret_cast<unsigned long long*>(&Hh[f * kBins + b]), (unsigned long long)h);
          sg[i] = 0;
          sh[i] = 0;
        }
      }
      __syncthreads();
    }
  }
  if (MODE == HM_UPDROOT && has_next) {   // tree t+1's maxima (float bits of non-negatives order as uints)
    for (int o = 16; o > 0; o >>= 1) {
      mg = fmaxf(mg, __shfl_xor_sync(0xffffffffu, mg, o));
      mh = fmaxf(mh, __shfl_xor_sync(0xffffffffu, mh, o));
    }
    if (lane == 0) {
      atomicMax(&a.maxg[t + 1], __float_as_uint(mg));
      atomicMax(&a.maxh[t + 1], __float_as_uint(mh));
    }
  }
}

// ---------------------------------------------------------------------------------------------
// k_hist2: change-mask histogram.  Same modes, piece list, chunking and flush as
// k_hist; a different inner loop, built so that equal codes in consecutive rows cost no per-row
// work.  Per warp batch of 32 staged rows:
//   lane r (row side)  XORs its row's 32 code bytes with the previous row's (8 words, SWAR) into a
//                      32-bit mask of the features whose code changes at row r; the warp transposes
//                      the 32 masks (5 shuffle stages), after which lane L holds, for feature
//                      f = h2_feat(L), the rows of the batch where its code changes; the warp's
//                      inclusive prefix sums of (q_g, q_h) give every run's sums as differences;
//   lane L (feature side) flushes each finished run of its feature with one pair of 32-bit shared
//                      reductions ("light" features, <= H2_HEAVY changes in the batch); "heavy"
//                      features (random codes, deep levels) go row-parallel instead (lane = row, a
//                      pair of reductions per row at (code, f)); the bank-padded [bin][33] layout
//                      keeps both access patterns conflict-light.
// The users column (a change on every row of paper-ordered data) stays row-parallel into the dense
// per-bin histogram (bank = bin).
constexpr int H2_THREADS = 512;
constexpr int H2_WARPS = H2_THREADS / 32;
constexpr int H2_PAD = 33;
constexpr int H2_CELLS = kBins * H2_PAD;                 // words per channel
constexpr int H2_HH = H2_CELLS * 4;                      // byte offset of the q_h channel
constexpr int H2_ROWB = 48;                              // bytes per staged row (conflict-free 16-B stores)
constexpr int H2_WBUF = 33 * H2_ROWB;                    // per warp: slots 1..32 = the batch's rows
constexpr int H2_U_OFF = 2 * H2_HH + H2_WARPS * H2_WBUF;
constexpr int H2_SMEM = H2_U_OFF + 2 * kBins * 4;        // 66 KB + 24.8 KB + 2 KB
constexpr int H2_HEAVY = 3;

// bit 8j+7-q of a row's change mask is feature 4q+j, so after the transpose lane L holds feature
__device__ __forceinline__ int h2_feat(int L) { return 4 * (7 - (L & 7)) + (L >> 3); }
// bit 8j+7 set iff byte j of x is non-zero
__device__ __forceinline__ uint32_t byte_ne_hi(uint32_t x) {
  return (x | ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu)) & 0x80808080u;
}
// 32x32 bit transpose across the warp: afterwards bit r of lane L = bit L of lane r's input
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m = s == 16 ? 0x0000ffffu : s == 8 ? 0x00ff00ffu : s == 4 ? 0x0f0f0f0fu : s == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y << s) & ~m));
  }
  return x;
}
__device__ __forceinline__ void red2(uint32_t addr, int32_t g, uint32_t h) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(g) : "memory");
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(addr), "r"(h), "n"(H2_HH) : "memory");
}

// DC: compile-time tree depth of the fused update's routing (0 = a.D); HF (fused update only): the
// root's q_h channel is tree-invariant and copied from a.hroot, so only q_g is histogrammed.
// DUAL (fused update only, with the q_h channel tree-invariant): BOTH ensembles in one pass over the rows —
// each row's code row, change-mask word and weight are loaded and staged once, the row is routed through
// both ensembles' trees t, and the histogram's second channel holds ensemble 1's q_g instead of
// ensemble 0's q_h (the run walk over the shared change mask serves both), flushed into ensemble 1's
// root slot
template <int MODE, int DC = 0, bool HF = false, bool DUAL = false>
__global__ void __launch_bounds__(H2_THREADS, 2) k_hist2(const FitPair fp, const int d, const int t_in, const DbgArgs dbg) {
  static_assert(!DUAL || (MODE == HM_UPDROOT && !HF), "DUAL: fused update, two q_g channels");
  pdl_wait();
  const FitArgs& a = fp.t[DUAL ? 0 : blockIdx.y];
  const FitArgs& a1 = fp.t[1];   // DUAL: ensemble 1
  const int t = (MODE == HM_ROOT || MODE == HM_UPDROOT) ? *a.d_tree : t_in;   // graph replays: tree index from the device
  if (MODE == HM_ROOT && !root_needed(a, t)) return;   // built speculatively by the previous update pass
  const bool has_next = (MODE == HM_UPDROOT) ? (t + 1 < a.T) : true;
  const int ucol = (a.users_col >= 0 && a.users_col < kMaxF) ? a.users_col : -1;   // row-parallel column
  extern __shared__ __align__(16) uint8_t smem[];
  int32_t* sg = reinterpret_cast<int32_t*>(smem);                 // [256 bins][33] (column 32 unused)
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem + H2_HH);
  int32_t* sug = reinterpret_cast<int32_t*>(smem + H2_U_OFF);     // users column (row-parallel), bank = bin
  uint32_t* suh = reinterpret_cast<uint32_t*>(smem + H2_U_OFF + kBins * 4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* wb = smem + 2 * H2_HH + warp * H2_WBUF;                // staged row r at wb + (r+1)*48

  __shared__ int64_t s_vstart[MAX_PIECES + 1];
  __shared__ int64_t s_pstart[MAX_PIECES];
  __shared__ int32_t s_slot[MAX_PIECES];
  __shared__ int s_np;

  for (int i = tid; i < 2 * H2_CELLS; i += H2_THREADS) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  for (int i = tid; i < 2 * kBins; i += H2_THREADS) reinterpret_cast<uint32_t*>(sug)[i] = 0u;
  // fused mode: tree t (the one just grown) in shared memory as a fixed-depth routing table: every
  // row descends exactly D levels.  Internal node k (depth < D): s_rt[k] = its split (f | b << 8); a leaf
  // above depth D and everything below it get (0, 255), i.e. "always left" (no code exceeds 255), so
  // a row reaching leaf k at depth d ends at k's leftmost depth-D descendant (k+1)·2^(D-d) - 1,
  // whose slot in s_lv holds k's value.  No per-level leaf test.
  // one u16 word per internal node: feature | bin << 8 (a single shared load per level)
  uint16_t* s_rt = reinterpret_cast<uint16_t*>(smem + H2_SMEM);
  float* s_lv = reinterpret_cast<float*>(smem + H2_SMEM + (a.nn + 1));   // 2^D depth-D slots
  const int n_int = (a.nn - 1) / 2;   // 2^D - 1 slots above depth D
  // DUAL: ensemble 1's table right after ensemble 0's (6 * 2^D bytes each)
  uint16_t* s_rt1 = reinterpret_cast<uint16_t*>(smem + H2_SMEM + 3 * (a.nn + 1));
  float* s_lv1 = reinterpret_cast<float*>(smem + H2_SMEM + 4 * (a.nn + 1));
  if (MODE == HM_UPDROOT) {
    for (int q = 0; q < (DUAL ? 2 : 1); ++q) {
      const FitArgs& aq = q ? a1 : a;
      uint16_t* rt = q ? s_rt1 : s_rt;
      float* lv = q ? s_lv1 : s_lv;
      const size_t to = (size_t)t * aq.nn;
      for (int i = tid; i < aq.nn; i += H2_THREADS) {
        const int f = aq.tfeat[to + i];
        if (i < n_int) {
          rt[i] = (uint16_t)(f >= 0 ? ((uint32_t)f | ((uint32_t)(aq.tbin[to + i] & 0xff) << 8)) : (255u << 8));
        }
        if (f == -1) {   // leaf at depth d = floor(log2(i + 1))
          const int dl = 31 - __clz(i + 1);
          lv[((i + 1) << (aq.D - dl)) - 1 - n_int] = aq.tval[to + i];
        }
      }
    }
  }
  // ---- piece list (virtual concatenation of the rows to histogram)
  if (MODE == HM_LEVEL) {
    const int NP = 1 << (d - 1);
    const LevelView& P = a.lv[d - 1];
    const LevelView& C = a.lv[d];
    int64_t len = 0, pst = 0;
    int side = 0;
    if (tid < NP && P.split_f[tid] >= 0) {
      const int64_t nL = C.cnt[2 * tid], nR = C.cnt[2 * tid + 1];
      side = a.built_by_h ? C.built[tid] : (nL <= nR) ? 0 : 1;   // the smaller child (rows; hessian when sharded)
      len = C.cnt[2 * tid + side];
      // k_part: left child at the parent's start, right child after it
      const int64_t ps = (d == 1) ? 0 : P.start[tid], cl = C.cnt[2 * tid];
      pst = side ? ps + cl : ps;
      if (blockIdx.x == 0) {
        C.built[tid] = side;
        C.start[2 * tid] = ps;
        C.start[2 * tid + 1] = ps + cl;
      }
    }
    __shared__ int64_t s_wsum[H2_WARPS];
    int64_t v = len;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) s_wsum[warp] = v;
    __syncthreads();
    int64_t woff = 0;
    for (int w2 = 0; w2 < warp; ++w2) woff += s_wsum[w2];
    if (tid < NP) {
      s_vstart[tid] = woff + v - len;
      s_pstart[tid] = pst;
      s_slot[tid] = tid;
    }
    if (tid == NP - 1) s_vstart[NP] = woff + v;
    if (tid == 0) s_np = NP;
  } else if (tid == 0) {
    s_np = 1;
    s_vstart[0] = 0;
    s_vstart[1] = (MODE == HM_ROOT || MODE == HM_UPDROOT) ? a.n : dbg.m;
    s_pstart[0] = 0;
    s_slot[0] = 0;
  }
  __syncthreads();
  const int np = s_np;
  const int64_t S = s_vstart[np];
  // identity-order modes with precomputed change masks: CTA, chunk and warp ranges start on 32-row
  // batch boundaries, so every staged batch is one precomputed mask batch
  constexpr bool IDN = (MODE == HM_ROOT || MODE == HM_UPDROOT);
  constexpr bool pre = IDN;   // identity order always uses the fit's precomputed masks (k_cmask)
  const int64_t am = pre ? ~(int64_t)31 : ~(int64_t)0;
  const int64_t v0 = (S * blockIdx.x / gridDim.x) & am;
  const int64_t v1 = (blockIdx.x + 1 == gridDim.x) ? S : ((S * (blockIdx.x + 1) / gridDim.x) & am);
  if (v0 >= v1) return;
  if (tid == 0 && MODE != HM_DEBUG && a.units)
    atomicAdd(&a.units[MODE == HM_ROOT ? KC_HIST_ROOT : MODE == HM_UPDROOT ? KC_UPDATE : KC_HIST],
              (unsigned long long)(v1 - v0) * (DUAL ? 2 : 1));

  // quantisation scales for ROOT (tree t): q = rint(v * 2^(K-e))
  // (HM_UPDROOT: tree t+1's pairs with tree t's exponents — the speculation described at k_hist)
  double scale_g = 0.0, scale_h = 0.0, scale_g1 = 0.0, scale_h1 = 0.0;
  if (MODE == HM_ROOT || MODE == HM_UPDROOT) {
    scale_g = exp2i(a.K - exp_of(__uint_as_float(a.maxg[t])));
    scale_h = exp2i(a.K - exp_of(__uint_as_float(a.maxh[t])));
  }
  if (DUAL) {
    scale_g1 = exp2i(a1.K - exp_of(__uint_as_float(a1.maxg[t])));
    scale_h1 = exp2i(a1.K - exp_of(__uint_as_float(a1.maxh[t])));
  }
  float mg = 0.f, mh = 0.f;   // HM_UPDROOT: tree t+1's max |g|, max h
  float mg1 = 0.f, mh1 = 0.f;   // DUAL: ensemble 1's
  int64_t* Hbase = (MODE == HM_DEBUG) ? dbg.out : a.H[d & 1];
  const uint32_t* sr_in = (MODE == HM_LEVEL) ? a.sr[d & 1] : nullptr;
  const uint32_t sgb = (uint32_t)__cvta_generic_to_shared(sg);
  const uint32_t sub = (uint32_t)__cvta_generic_to_shared(sug);
  const int myf = h2_feat(lane);
  const bool active = myf < a.F && myf != ucol;
  const bool hist_on = !(MODE == HM_UPDROOT && !has_next);   // last tree: update only

  int pc = 0;
  while (pc + 1 < np && s_vstart[pc + 1] <= v0) ++pc;
  for (; pc < np && s_vstart[pc] < v1; ++pc) {
    int64_t s0 = max(v0, s_vstart[pc]), s1 = min(v1, s_vstart[pc + 1]);
    if (s0 >= s1) continue;
    int64_t* Hg = Hbase + (size_t)s_slot[pc] * SLOT;
    int64_t* Hh = DUAL ? a1.H[0] : Hg + kHistBins;   // DUAL: second channel = ensemble 1's root q_g
    const int64_t poff = s_pstart[pc] - s_vstart[pc];   // physical position = virtual + poff
    for (int64_t c0 = s0; c0 < s1; c0 += HIST_CHUNK) {
      const int64_t c1 = min(s1, c0 + HIST_CHUNK);
      const int64_t clen = c1 - c0;
      const int64_t w0 = c0 + ((clen * warp / H2_WARPS) & am);
      const int64_t w1 = (warp + 1 == H2_WARPS) ? c1 : c0 + ((clen * (warp + 1) / H2_WARPS) & am);
      uint32_t cur = 0;           // pending run of feature myf: byte offset of its (bin, f) cell
      int32_t acc_g = 0;          // its sums from earlier batches
      uint32_t acc_h = 0;
      bool fresh = true;          // no previous row yet
      uint4 nc0 = make_uint4(0, 0, 0, 0), nc1 = nc0;
      uint32_t ngp = 0, nri = 0, nmask = 0;
      float ny = 0.f, nw = 0.f, np_ = 0.f;
      float ny1 = 0.f, np1 = 0.f;   // DUAL: ensemble 1's target and prediction
      auto load_ridx = [&](int64_t vb) {
        const int64_t vi = vb + lane;
        if (MODE == HM_LEVEL && vi < w1) nri = sr_in[vi + poff];
      };
      auto load_batch = [&](int64_t vb) {
        const int64_t vi = vb + lane;
        if (vi < w1) {
          const int64_t pi = vi + poff;
          int64_t ridx;
          if (MODE == HM_ROOT || MODE == HM_UPDROOT) {
            ridx = pi;
            ny = a.y[ridx];
            nw = a.w[ridx];
            np_ = a.p[ridx];
            if (DUAL) {
              ny1 = a1.y[ridx];
              np1 = a1.p[ridx];
            }
          } else if (MODE == HM_LEVEL) {
            ridx = nri;
            ngp = a.gp_root[ridx];
          } else {
            ridx = dbg.idx ? dbg.idx[pi] : pi;
            ngp = pack_gp(dbg.qg[ridx], dbg.qh[ridx]);
          }
          const uint4* crow = reinterpret_cast<const uint4*>(a.codes + (size_t)ridx * kMaxF);
          nc0 = __ldg(crow);
          nc1 = __ldg(crow + 1);
        }
        if (pre) nmask = __ldg(a.cmask + ((vb + poff) >> 5) * 32 + lane);   // the batch's mask word of this lane
      };
      if (w0 < w1) {
        load_ridx(w0);
        load_batch(w0);
        load_ridx(w0 + 32);
      }
      for (int64_t base = w0; base < w1; base += 32) {
        const int cnt = (int)min((int64_t)32, w1 - base);
        const bool valid = lane < cnt;
        uint32_t gp = ngp;
        uint32_t gp1 = 0;   // DUAL: ensemble 1's packed pair
        if (MODE == HM_ROOT && valid) {
          const int64_t ridx = base + lane + poff;
          float g, h;
          grad_pair(a, t, a.row_offset + ridx, ny, nw, np_, g, h);
          gp = pack_gp(quantize(g, scale_g), quantize(h, scale_h));
          a.gp_root[ridx] = gp;
        }
        const uint32_t bmask = nmask;       // this batch's precomputed mask word (pre)
        // previous row of lane 0: the last staged row of the previous batch (read before it is overwritten)
        uint4 pv0 = nc0, pv1 = nc1;
        if (!pre && lane == 0 && !fresh) {
          pv0 = *reinterpret_cast<const uint4*>(wb + 32 * H2_ROWB);
          pv1 = *reinterpret_cast<const uint4*>(wb + 32 * H2_ROWB + 16);
        }
        __syncwarp();   // previous batch fully consumed
        uint8_t* myrow = wb + (lane + 1) * H2_ROWB;
        *reinterpret_cast<uint4*>(myrow) = nc0;
        *reinterpret_cast<uint4*>(myrow + 16) = nc1;
        if (MODE == HM_UPDROOT && valid) {
          // O9 for tree t (route the lane's own staged row, p += v), then O4 for tree t+1
          const int64_t ridx = base + lane + poff;
          // both children's node words are loaded together with the row's code byte, so each level
          // costs one shared-memory round trip (a leaf keeps k; its child indices stay < nn)
          int k = 0;
          const int D = DC ? DC : a.D;
#pragma unroll
          for (int s2 = 0; s2 < (DC ? DC : kMaxDepth); ++s2)
            if (DC || s2 < D) {
              const uint32_t w = s_rt[k];
              k = 2 * k + 1 + ((uint32_t)myrow[w & 0xffu] > (w >> 8) ? 1 : 0);
            }
          const float pn = __fadd_rn(np_, s_lv[k - n_int]);   // one fp32 rounding, tree order
          a.p[ridx] = pn;
          if (has_next) {
            float g, h;
            grad_pair(a, t + 1, a.row_offset + ridx, ny, nw, pn, g, h);
            mg = fmaxf(mg, fabsf(g));
            mh = fmaxf(mh, h);
            gp = pack_gp(quantize(g, scale_g), quantize(h, scale_h));
            a.gp_root[ridx] = gp;
          }
          if (DUAL) {   // the same row through ensemble 1's tree t
            int k1 = 0;
#pragma unroll
            for (int s2 = 0; s2 < (DC ? DC : kMaxDepth); ++s2)
              if (DC || s2 < D) {
                const uint32_t w = s_rt1[k1];
                k1 = 2 * k1 + 1 + ((uint32_t)myrow[w & 0xffu] > (w >> 8) ? 1 : 0);
              }
            const float pn1 = __fadd_rn(np1, s_lv1[k1 - n_int]);
            a1.p[ridx] = pn1;
            if (has_next) {
              float g, h;
              grad_pair(a1, t + 1, a1.row_offset + ridx, ny1, nw, pn1, g, h);
              mg1 = fmaxf(mg1, fabsf(g));
              mh1 = fmaxf(mh1, h);
              gp1 = pack_gp(quantize(g, scale_g1), quantize(h, scale_h1));
              a1.gp_root[ridx] = gp1;
            }
          }
        }
        __syncwarp();
        const uint4 cc0 = nc0, cc1 = nc1;   // this batch's row (the prefetch below overwrites nc*)
        if (!pre && lane > 0) {
          pv0 = *reinterpret_cast<const uint4*>(myrow - H2_ROWB);
          pv1 = *reinterpret_cast<const uint4*>(myrow - H2_ROWB + 16);
        }
        if (base + 32 < w1) {   // prefetch the next batch (and the row indices of the one after)
          load_batch(base + 32);
          load_ridx(base + 64);
        }
        if (!hist_on) continue;
        // ---- row side: change mask of this lane's row (bit 8j+7-q = feature 4q+j)
        uint32_t m = 0;
        if (!pre && valid) {
          m = byte_ne_hi(cc0.x ^ pv0.x) | (byte_ne_hi(cc0.y ^ pv0.y) >> 1) | (byte_ne_hi(cc0.z ^ pv0.z) >> 2) |
              (byte_ne_hi(cc0.w ^ pv0.w) >> 3) | (byte_ne_hi(cc1.x ^ pv1.x) >> 4) | (byte_ne_hi(cc1.y ^ pv1.y) >> 5) |
              (byte_ne_hi(cc1.z ^ pv1.z) >> 6) | (byte_ne_hi(cc1.w ^ pv1.w) >> 7);
        }
        const int32_t qg = valid ? gp_g(gp) : 0;
        const uint32_t qh = valid ? (DUAL ? (uint32_t)gp_g(gp1) : (uint32_t)gp_h(gp)) : 0u;
        if (ucol >= 0 && valid) {   // users column, row-parallel into the dense per-bin histogram
          const uint32_t ua = sub + (uint32_t)myrow[ucol] * 4u;
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(ua), "r"(qg) : "memory");
          if (!HF) asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(ua), "r"(qh), "n"(kBins * 4) : "memory");
        }
        // inclusive prefix sums of the pairs over the batch's rows
        int32_t pg = qg;
        uint32_t ph = HF ? 0u : qh;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t ug = __shfl_up_sync(0xffffffffu, pg, o);
          const uint32_t uh = HF ? 0u : __shfl_up_sync(0xffffffffu, ph, o);
          if (lane >= o) {
            pg += ug;
            ph += uh;
          }
        }
        const int32_t tot_g = __shfl_sync(0xffffffffu, pg, 31);
        const uint32_t tot_h = HF ? 0u : __shfl_sync(0xffffffffu, ph, 31);
        // ---- feature side
        uint32_t M = pre ? (fresh ? bmask & ~1u : bmask) : warp_transpose32(m, lane);
        if (fresh) {
          if (active) cur = (uint32_t)(wb[H2_ROWB + myf] * H2_PAD + myf) * 4u;   // run starts at row 0
          fresh = false;
        }
        if (!active) M = 0;
        const bool heavy = __popc(M) > H2_HEAVY;
        uint32_t Ml = heavy ? 0u : M;
        int32_t bg = 0;      // prefix before the current run's first row in this batch
        uint32_t bh = 0;
        while (__any_sync(0xffffffffu, Ml != 0u)) {
          const int r = __ffs(Ml) - 1;
          const int32_t pgr = __shfl_sync(0xffffffffu, pg, (r - 1) & 31);
          const uint32_t phr = HF ? 0u : __shfl_sync(0xffffffffu, ph, (r - 1) & 31);
          if (Ml) {
            const int32_t vg = r ? pgr : 0;
            const uint32_t vh = r ? phr : 0u;
            if (HF) asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(sgb + cur), "r"(acc_g + (vg - bg)) : "memory");
            else red2(sgb + cur, acc_g + (vg - bg), acc_h + (vh - bh));
            acc_g = 0;
            acc_h = 0;
            bg = vg;
            bh = vh;
            cur = (uint32_t)(wb[(r + 1) * H2_ROWB + myf] * H2_PAD + myf) * 4u;
            Ml &= Ml - 1u;
          }
        }
        if (!heavy) {
          acc_g += tot_g - bg;
          acc_h += tot_h - bh;
        }
        // heavy features: row-parallel, one feature at a time, unrolled over the lanes so every
        // feature index is a constant and each row's code byte comes from its own registers
        const unsigned hm = __ballot_sync(0xffffffffu, heavy);
        if (hm) {
          if (heavy) {   // flush the pending run of earlier batches; the run continues from the last row
            if (acc_g | (int32_t)acc_h) red2(sgb + cur, acc_g, acc_h);
            acc_g = 0;
            acc_h = 0;
            cur = (uint32_t)(wb[cnt * H2_ROWB + myf] * H2_PAD + myf) * 4u;
          }
          const uint32_t cw[8] = {cc0.x, cc0.y, cc0.z, cc0.w, cc1.x, cc1.y, cc1.z, cc1.w};
#pragma unroll
          for (int q = 0; q < 8; ++q) {   // lanes 7-q, 15-q, 23-q, 31-q hold features 4q .. 4q+3
            if (hm & (0x01010101u << (7 - q))) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int hl = 8 * j + 7 - q, hf = 4 * q + j;
                if ((hm & (1u << hl)) && valid)
                  red2(sgb + (((cw[q] >> (8 * j)) & 0xffu) * H2_PAD + (uint32_t)hf) * 4u, qg, HF ? 0u : qh);
              }
            }
          }
        }
      }
      if (active && !fresh && (acc_g | (int32_t)acc_h)) red2(sgb + cur, acc_g, acc_h);
      __syncthreads();
      if (ucol >= 0) {   // the users column's cells (untouched by its lane) from the dense histogram
        for (int b = tid; b < kBins; b += H2_THREADS) {
          sg[b * H2_PAD + ucol] = sug[b];
          sh[b * H2_PAD + ucol] = suh[b];
          sug[b] = 0;
          suh[b] = 0;
        }
        __syncthreads();
      }
      // flush: zero-skipping int64 atomics into the node histogram ([f][b] layout)
      for (int i = tid; i < kHistBins; i += H2_THREADS) {
        const int b = i >> 5, f = i & 31;
        const int32_t g = sg[b * H2_PAD + f];
        const uint32_t h = sh[b * H2_PAD + f];
        if (g != 0 || h != 0) {
          atomicAdd(reinterpret_cast<unsigned long long*>(&Hg[f * kBins + b]), (unsigned long long)(long long)g);
          if (DUAL)   // ensemble 1's q_g: signed
            atomicAdd(reinterpret_cast<unsigned long long*>(&Hh[f * kBins + b]),
                      (unsigned long long)(long long)(int32_t)h);
          else if (!HF)
            atomicAdd(reinterpret_cast<unsigned long long*>(&Hh[f * kBins + b]), (unsigned long long)h);
          sg[b * H2_PAD + f] = 0;
          sh[b * H2_PAD + f] = 0;
        }
      }
      __syncthreads();
    }
  }
  if (MODE == HM_UPDROOT && has_next) {   // tree t+1's maxima (float bits of non-negatives order as uints)
    for (int o = 16; o > 0; o >>= 1) {
      mg = fmaxf(mg, __shfl_xor_sync(0xffffffffu, mg, o));
      mh = fmaxf(mh, __shfl_xor_sync(0xffffffffu, mh, o));
    }
    if (lane == 0) {
      atomicMax(&a.maxg[t + 1], __float_as_uint(mg));
      atomicMax(&a.maxh[t + 1], __float_as_uint(mh));
    }
    if (DUAL) {
      for (int o = 16; o > 0; o >>= 1) {
        mg1 = fmaxf(mg1, __shfl_xor_sync(0xffffffffu, mg1, o));
        mh1 = fmaxf(mh1, __shfl_xor_sync(0xffffffffu, mh1, o));
      }
      if (lane == 0) {
        atomicMax(&a1.maxg[t + 1], __float_as_uint(mg1));
        atomicMax(&a1.maxh[t + 1], __float_as_uint(mh1));
      }
    }
  }
}

// Change masks of the identity row order, once per fit (the codes never change during a fit): word
// L of batch B (rows 32B .. 32B+31) has bit r set iff feature h2_feat(L)'s code at row 32B+r differs
// from the one at row 32B+r-1 (bit 0 of batch 0: 0; rows >= n: 0) — exactly the transposed mask
// k_hist2 would build per batch, so the identity-order passes (root, fused update) load one word
// per lane instead of recomputing it every tree (4 B per row read, ~80 instructions per batch saved)
__global__ void __launch_bounds__(256) k_cmask(const uint8_t* codes, int64_t n, uint32_t* cmask) {
  const int lane = threadIdx.x & 31;
  const int64_t nb = (n + 31) / 32;
  for (int64_t B = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5; B < nb; B += ((int64_t)gridDim.x * 256) >> 5) {
    const int64_t r = B * 32 + lane;
    uint32_t m = 0;
    if (r < n && r > 0) {
      const uint4* c = reinterpret_cast<const uint4*>(codes + (size_t)r * kMaxF);
      const uint4 c0 = __ldg(c), c1 = __ldg(c + 1), p0 = __ldg(c - 2), p1 = __ldg(c - 1);
      m = byte_ne_hi(c0.x ^ p0.x) | (byte_ne_hi(c0.y ^ p0.y) >> 1) | (byte_ne_hi(c0.z ^ p0.z) >> 2) |
          (byte_ne_hi(c0.w ^ p0.w) >> 3) | (byte_ne_hi(c1.x ^ p1.x) >> 4) | (byte_ne_hi(c1.y ^ p1.y) >> 5) |
          (byte_ne_hi(c1.z ^ p1.z) >> 6) | (byte_ne_hi(c1.w ^ p1.w) >> 7);
    }
    cmask[B * 32 + lane] = warp_transpose32(m, lane);
  }
}

// the fused update kernel for a depth: compile-time routing depth for the configs' depths (6, 8)
using Hist2Kernel = void (*)(const FitPair, const int, const int, const DbgArgs);
static Hist2Kernel updroot2_kernel(int D, bool hf, bool dual = false) {
  if (dual) {
    if (D == 8) return k_hist2<HM_UPDROOT, 8, false, true>;
    if (D == 6) return k_hist2<HM_UPDROOT, 6, false, true>;
    return k_hist2<HM_UPDROOT, 0, false, true>;
  }
  if (hf) {
    if (D == 8) return k_hist2<HM_UPDROOT, 8, true>;
    if (D == 6) return k_hist2<HM_UPDROOT, 6, true>;
    return k_hist2<HM_UPDROOT, 0, true>;
  }
  if (D == 8) return k_hist2<HM_UPDROOT, 8>;
  if (D == 6) return k_hist2<HM_UPDROOT, 6>;
  return k_hist2<HM_UPDROOT, 0>;
}

// histogram inner loop per mode: change-mask k_hist2 or run-length k_hist.  LLMP_HIST2 is a bit mask
// of the modes that use k_hist2 (1 root, 2 level, 4 fused update + root); default 5 = the measured
// winners (root and update on k_hist2, level histograms on k_hist)
static int hist1_mask() {
  static const int v = 7 & ~(getenv("LLMP_HIST2") ? atoi(getenv("LLMP_HIST2")) : 5);
  return v;
}
// level-histogram kernel: LLMP_LEVEL = 3 (default) change-row k_hist3; 1 run-length k_hist; 2 change-mask
// k_hist2.  The test hook (llmpilot_debug_histogram) follows the same choice.
static int level_kernel() {
  static const int v = getenv("LLMP_LEVEL") ? atoi(getenv("LLMP_LEVEL")) : 3;
  return (v == 1 || v == 2) ? v : 3;
}

// zero the root histogram slot when k_hist<ROOT> is going to (re)build it (see root_needed)
__global__ void k_root_fix(const FitPair fp) {
  pdl_wait();
  const FitArgs& a = fp.t[blockIdx.y];
  if (!root_needed(a, *a.d_tree)) return;
  int64_t* H = a.H[0];
  for (int i = threadIdx.x; i < SLOT; i += blockDim.x) H[i] = 0;
}

// ---------------------------------------------------------------------------------------------
// Root histogram, hybrid run/row-parallel form (HM_ROOT only; rows in identity order).
// Per warp batch of 32 rows:
//   lane r   computes row r's gradient pair (weighted squared error, sampling, quantisation),
//            writes it to gp_root and takes part in a warp prefix scan of (q_g, q_h);
//   lane f   loads feature f's 32 codes as two aligned 16-byte vectors from the column-major
//            codes, builds the 32-bit mask of rows where its code changes, and
//            - "light" lanes (<= 3 changes): flush each finished run with one pair of 32-bit shared
//              reductions, the run sum being a difference of the batch prefix sums;
//            - "heavy" lanes (> 3 changes, e.g. the users column of paper-ordered rows, or random
//              codes): processed row-parallel — for each heavy feature the 32 lanes add their own
//              row's pair at (code, feature) in a bank-padded [bin][33] histogram.
// Equal codes in consecutive rows therefore cost no per-row work at all.
constexpr int R2_THREADS = 512;
constexpr int R2_WARPS = R2_THREADS / 32;
constexpr int R2_PAD = 33;                                   // [bin][33] words: both access patterns conflict-light
constexpr int R2_HIST_WORDS = kBins * R2_PAD;                // per channel
constexpr int R2_FSTRIDE = 36;                               // bytes per feature row of a batch in smem
constexpr int R2_SMEM = 2 * R2_HIST_WORDS * 4 + R2_WARPS * (32 * R2_FSTRIDE + 2 * 32 * 4);
constexpr int R2_HEAVY = 3;

__device__ __forceinline__ uint32_t change_nibble(uint32_t cur, uint32_t prevw) {
  // bit i (i < 4) set iff byte i of cur differs from byte i of (cur << 8 | prevw >> 24)
  const uint32_t x = cur ^ __funnelshift_l(prevw, cur, 8);
  const uint32_t t = (x | ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu)) & 0x80808080u;
  return (t * 0x00204081u) >> 28;
}

__global__ void __launch_bounds__(R2_THREADS, 2) k_hist_root2(const FitPair fp) {
  const FitArgs& a = fp.t[blockIdx.y];
  const int t = *a.d_tree;
  extern __shared__ __align__(16) uint8_t smem[];
  int32_t* hg = reinterpret_cast<int32_t*>(smem);                       // [256][33]
  uint32_t* hh = reinterpret_cast<uint32_t*>(smem + R2_HIST_WORDS * 4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* fbuf = smem + 2 * R2_HIST_WORDS * 4 + warp * (32 * R2_FSTRIDE + 2 * 32 * 4);
  int32_t* pbg = reinterpret_cast<int32_t*>(fbuf + 32 * R2_FSTRIDE);  // batch prefix of q_g
  uint32_t* pbh = reinterpret_cast<uint32_t*>(pbg + 32);              // batch prefix of q_h
  for (int i = tid; i < 2 * R2_HIST_WORDS; i += R2_THREADS) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  __syncthreads();
  const int64_t n = a.n;
  // 32-row aligned contiguous range per CTA
  const int64_t nb = (n + 31) / 32;
  const int64_t v0 = (nb * blockIdx.x / gridDim.x) * 32, v1 = min(n, (nb * (blockIdx.x + 1) / gridDim.x) * 32);
  if (v0 >= v1) return;
  if (tid == 0 && a.units) atomicAdd(&a.units[KC_HIST_ROOT], (unsigned long long)(v1 - v0));
  const double scale_g = exp2i(a.K - exp_of(__uint_as_float(a.maxg[t])));
  const double scale_h = exp2i(a.K - exp_of(__uint_as_float(a.maxh[t])));
  const bool fin = lane < a.F;
  const uint32_t sb_g = (uint32_t)__cvta_generic_to_shared(hg), sb_h = (uint32_t)__cvta_generic_to_shared(hh);
  for (int64_t c0 = v0; c0 < v1; c0 += HIST_CHUNK) {        // flush at least every 65,536 rows
    const int64_t c1 = min(v1, c0 + HIST_CHUNK);
    const int64_t nbc = (c1 - c0 + 31) / 32;
    const int64_t w0 = c0 + (nbc * warp / R2_WARPS) * 32, w1 = min(c1, c0 + (nbc * (warp + 1) / R2_WARPS) * 32);
    int cur = -1;            // code of the pending run of this lane's feature
    int32_t acc_g = 0;       // pending run sums
    uint32_t acc_h = 0;
    // register prefetch of the next batch (y, w, p of lane r's row; lane f's 32 codes)
    float ny = 0.f, nw = 0.f, np_ = 0.f;
    uint4 na = make_uint4(0, 0, 0, 0), nb2 = na;
    auto load_batch = [&](int64_t b) {
      if (b + lane < w1) {
        ny = a.y[b + lane];
        nw = a.w[b + lane];
        np_ = a.p[b + lane];
      }
      const uint4* cp = reinterpret_cast<const uint4*>(a.codesT + (size_t)lane * a.ldT + b);
      na = __ldg(cp);
      nb2 = __ldg(cp + 1);
    };
    if (w0 < w1) load_batch(w0);
    for (int64_t base = w0; base < w1; base += 32) {
      const int cnt = (int)min((int64_t)32, w1 - base);
      const float yv = ny, wv = nw, pv = np_;
      const uint4 ca = na, cb = nb2;
      if (base + 32 < w1) load_batch(base + 32);
      // ---- row-side: gradient pair of row base + lane
      int32_t qg = 0, qh = 0;
      if (lane < cnt) {
        const int64_t i = base + lane;
        float g, h;
        grad_pair(a, t, a.row_offset + i, yv, wv, pv, g, h);
        qg = quantize(g, scale_g);
        qh = quantize(h, scale_h);
        a.gp_root[i] = pack_gp(qg, qh);
      }
      // ---- feature-side: 32 codes of this lane's feature (aligned vectors; padding rows are 0)
      uint32_t cw[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
      // inclusive warp prefix of the pairs
      int32_t pg = qg;
      uint32_t ph = (uint32_t)qh;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t ug = __shfl_up_sync(0xffffffffu, pg, o);
        const uint32_t uh = __shfl_up_sync(0xffffffffu, ph, o);
        if (lane >= o) {
          pg += ug;
          ph += uh;
        }
      }
      __syncwarp();
      pbg[lane] = pg;
      pbh[lane] = ph;
#pragma unroll
      for (int q = 0; q < 8; ++q) *reinterpret_cast<uint32_t*>(fbuf + lane * R2_FSTRIDE + 4 * q) = cw[q];
      const int32_t tot_g = __shfl_sync(0xffffffffu, pg, 31);
      const uint32_t tot_h = __shfl_sync(0xffffffffu, ph, 31);
      __syncwarp();
      // change mask over rows 0..cnt-1 (row 0 compares with the pending run's code)
      if (cur < 0) cur = (int)(cw[0] & 0xffu);
      uint32_t M = 0;
      uint32_t prevw = (uint32_t)cur << 24;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        M |= change_nibble(cw[q], prevw) << (4 * q);
        prevw = cw[q];
      }
      if (cnt < 32) M &= (1u << cnt) - 1u;
      if (!fin) M = 0;
      const int nch = __popc(M);
      const bool heavy = fin && nch > R2_HEAVY;
      // ---- light lanes: flush finished runs with prefix differences
      {
        uint32_t Ml = heavy ? 0u : M;
        const int iters = __reduce_max_sync(0xffffffffu, heavy ? 0 : nch);
        int32_t base_g = 0;   // prefix before the current run's first row
        uint32_t base_h = 0;
        for (int it = 0; it < iters; ++it) {
          if (Ml) {
            const int r = __ffs(Ml) - 1;
            Ml &= Ml - 1;
            const int32_t pgr = r ? pbg[r - 1] : 0;
            const uint32_t phr = r ? pbh[r - 1] : 0u;
            const int32_t rg = acc_g + (pgr - base_g);
            const uint32_t rh = acc_h + (phr - base_h);
            const uint32_t ad = (uint32_t)(cur * R2_PAD + lane) * 4u;
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(sb_g + ad), "r"(rg) : "memory");
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sb_h + ad), "r"(rh) : "memory");
            acc_g = 0;
            acc_h = 0;
            base_g = pgr;
            base_h = phr;
            cur = fbuf[lane * R2_FSTRIDE + r];
          }
        }
        if (!heavy && fin) {
          acc_g += tot_g - base_g;
          acc_h += tot_h - base_h;
        }
      }
      // ---- heavy lanes: row-parallel, one feature at a time
      unsigned hm = __ballot_sync(0xffffffffu, heavy);
      while (hm) {
        const int hf = __ffs(hm) - 1;
        hm &= hm - 1;
        if (lane == hf && (acc_g | (int32_t)acc_h)) {   // pending run of earlier batches
          const uint32_t ad = (uint32_t)(cur * R2_PAD + lane) * 4u;
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(sb_g + ad), "r"(acc_g) : "memory");
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sb_h + ad), "r"(acc_h) : "memory");
        }
        if (lane < cnt) {
          const int code = fbuf[hf * R2_FSTRIDE + lane];
          const uint32_t ad = (uint32_t)(code * R2_PAD + hf) * 4u;
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(sb_g + ad), "r"(qg) : "memory");
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sb_h + ad), "r"((uint32_t)qh) : "memory");
        }
        if (lane == hf) {
          acc_g = 0;
          acc_h = 0;
          cur = fbuf[hf * R2_FSTRIDE + cnt - 1];
        }
      }
      __syncwarp();
    }
    if (fin && cur >= 0 && (acc_g | (int32_t)acc_h)) {
      atomicAdd(&hg[cur * R2_PAD + lane], acc_g);
      atomicAdd(&hh[cur * R2_PAD + lane], acc_h);
    }
    __syncthreads();
    // zero-skipping int64 flush into the root histogram ([f][b] layout)
    int64_t* Hg = a.H[0];
    int64_t* Hh = Hg + kHistBins;
    for (int i = tid; i < kHistBins; i += R2_THREADS) {
      const int b = i >> 5, f = i & 31;
      const int32_t g = hg[b * R2_PAD + f];
      const uint32_t h = hh[b * R2_PAD + f];
      if (g != 0 || h != 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&Hg[f * kBins + b]), (unsigned long long)(long long)g);
        atomicAdd(reinterpret_cast<unsigned long long*>(&Hh[f * kBins + b]), (unsigned long long)h);
        hg[b * R2_PAD + f] = 0;
        hh[b * R2_PAD + f] = 0;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// Row partition of the split parents (level d-1) into their children (level d): see k_part.
constexpr int PT_THREADS = 128;
constexpr int PT_ITEMS = 16;
constexpr int PT_TILE = PT_THREADS * PT_ITEMS;   // 2048 rows
constexpr int PT_WORDS = PT_TILE / 32;           // bitmask words per tile
constexpr int PT_WPL = PT_WORDS / 32;            // words per lane in the group-prefix warp
constexpr int PT_PPT = MAX_PIECES / PT_THREADS;  // parents per thread in parent_prefixes
static_assert(PT_WORDS % 32 == 0 && MAX_PIECES % PT_THREADS == 0, "partition tile shape");

// tile and row prefixes over the level's split parents (computed by each CTA; NP <= 512); also
// caches every parent's split, start and count in shared memory (s_pp), so the per-tile lookups
// are shared-memory loads instead of a chain of dependent global loads
struct PartParent {
  int64_t start, cnt;
  int32_t f, b;
};
__device__ __forceinline__ void parent_prefixes(const FitArgs& a, int d, int* s_tile_pref, int64_t* s_seq_pref,
                                                int* s_w, int64_t* s_w64, PartParent* s_pp) {
  const int NP = 1 << (d - 1);
  const LevelView& P = a.lv[d - 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int tl[PT_PPT];
  int64_t rl[PT_PPT];
  int tv = 0;
  int64_t rv = 0;
#pragma unroll
  for (int q = 0; q < PT_PPT; ++q) {
    const int j = tid * PT_PPT + q;
    tl[q] = 0;
    rl[q] = 0;
    if (j < NP) {
      // every load unconditional (one round trip; the entries of parents that did not split are
      // in bounds and ignored)
      const int f = P.split_f[j];
      const int sb = P.split_b[j];
      const int64_t st = (d == 1) ? 0 : P.start[j];
      const int64_t ct = (d == 1) ? a.n : P.cnt[j];
      PartParent pp;
      pp.f = f;
      pp.b = f >= 0 ? sb : 0;
      pp.start = st;
      pp.cnt = (f < 0) ? 0 : ct;
      s_pp[j] = pp;
      if (f >= 0) {
        rl[q] = pp.cnt;
        tl[q] = (int)((rl[q] + PT_TILE - 1) / PT_TILE);
      }
    }
    tv += tl[q];
    rv += rl[q];
  }
  int tinc = tv;
  int64_t rinc = rv;
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, tinc, o);
    const int64_t u64 = __shfl_up_sync(0xffffffffu, rinc, o);
    if (lane >= o) {
      tinc += u;
      rinc += u64;
    }
  }
  if (lane == 31) {
    s_w[warp] = tinc;
    s_w64[warp] = rinc;
  }
  __syncthreads();
  int toff = 0;
  int64_t roff = 0;
  for (int w2 = 0; w2 < warp; ++w2) {
    toff += s_w[w2];
    roff += s_w64[w2];
  }
  int te = toff + tinc - tv;
  int64_t re = roff + rinc - rv;
#pragma unroll
  for (int q = 0; q < PT_PPT; ++q) {
    const int j = tid * PT_PPT + q;
    if (j < NP) {
      s_tile_pref[j] = te;
      s_seq_pref[j] = re;
    }
    te += tl[q];
    re += rl[q];
  }
  if (tid == (int)blockDim.x - 1) {
    s_tile_pref[NP] = te;
    s_seq_pref[NP] = re;
  }
  __syncthreads();
}

// parent j of tile t: largest j with tile_pref[j] <= t
__device__ __forceinline__ int parent_of_tile(const int* s_tile_pref, int NP, int t) {
  int lo = 0, hi = NP - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_tile_pref[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------------------------------------
// Single-pass partition.  Every histogram is an integer sum, so the order of the rows inside a
// child segment cannot change any result — only which CTA processes which rows.  Each 2048-row
// tile of a split parent j therefore reserves its block of each child with one global atomic per
// child instead of waiting for a prefix over all tiles: the left child fills the parent's own range
// [s_j, s_j + n_j) of the other ping-pong buffer from the bottom (cursor C.cnt[2j]), the right child
// from the top (cursor C.cnt[2j+1]); inside a block the rows keep their order (ballot + per-group
// prefix table), so the children are block-wise permutations of runs of the parent's order.  Row
// indices are read once; the next tile's row indices are loaded while this tile waits for its
// reservation.  The cursors start at 0 (zeroed by the split kernel of level d-1); the children's
// starts follow from the counts (s_j and s_j + n_L; written by the level histogram kernel).
constexpr int PT_CTAS_PER_SM = 8;
__global__ void __launch_bounds__(PT_THREADS, PT_CTAS_PER_SM) k_part(const FitPair fp, const int d) {
  pdl_wait();
  const FitArgs& a = fp.t[blockIdx.y];
  __shared__ int s_tile_pref[MAX_PIECES + 1];
  __shared__ int64_t s_seq_pref[MAX_PIECES + 1];
  __shared__ int s_w[PT_THREADS / 32];
  __shared__ int64_t s_w64[PT_THREADS / 32];
  __shared__ __align__(16) uint32_t s_bits[2][PT_WORDS];   // the tile's ballot words, group = (q, warp); by tile parity
  __shared__ __align__(16) int s_pre[PT_WORDS];         // exclusive left prefix of each group
  __shared__ int64_t s_lb, s_rb;                        // the tile's block offsets (left from the bottom, right from the top)
  __shared__ PartParent s_pp[MAX_PIECES];
  const int NP = 1 << (d - 1);
  const LevelView& P = a.lv[d - 1];
  const LevelView& C = a.lv[d];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.fq && blockIdx.x == 0)   // the level histogram's fold-in work queue (head, tail, slots)
    for (int i = tid; i < FQ_INTS; i += PT_THREADS) a.fq[i] = 0;
  {   // zero the built-child histogram slots [0, NP) of this level for split parents
    int4* Hz = reinterpret_cast<int4*>(a.H[d & 1]);
    const size_t per_slot = SLOT / 2;  // int4 per slot
    const size_t total = (size_t)NP * per_slot;
    for (size_t e = (size_t)blockIdx.x * PT_THREADS + tid; e < total; e += (size_t)gridDim.x * PT_THREADS) {
      const int j = (int)(e / per_slot);
      if (P.split_f[j] >= 0) Hz[e] = make_int4(0, 0, 0, 0);
    }
  }
  parent_prefixes(a, d, s_tile_pref, s_seq_pref, s_w, s_w64, s_pp);
  const int ntiles = s_tile_pref[NP];
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t* const rin_all = a.sr[(d - 1) & 1];
  uint32_t* const rout = a.sr[d & 1];
  // row indices of tile t (the parent's segment in the input buffer; identity at d = 1)
  // the parent of each tile is found once (when its row indices are loaded) and carried along
  auto load_rows = [&](int t, uint32_t (&r)[PT_ITEMS], int& jt) {
    if (t >= ntiles) return;
    const int j = parent_of_tile(s_tile_pref, NP, t);
    jt = j;
    const int64_t cnt_j = s_pp[j].cnt;
    const int64_t o = (int64_t)(t - s_tile_pref[j]) * PT_TILE;
    const int len = (int)min((int64_t)PT_TILE, cnt_j - o);
    const uint32_t* rin = rin_all + s_pp[j].start + o;
    if (d == 1) {
#pragma unroll
      for (int q = 0; q < PT_ITEMS; ++q) {   // identity (a tail's rows past the parent read row 0)
        const int k = q * PT_THREADS + tid;
        r[q] = k < len ? (uint32_t)(o + k) : 0u;
      }
    } else if (len == PT_TILE) {
#pragma unroll
      for (int q = 0; q < PT_ITEMS; ++q) r[q] = rin[q * PT_THREADS + tid];
    } else {
#pragma unroll
      for (int q = 0; q < PT_ITEMS; ++q) {
        const int k = q * PT_THREADS + tid;
        r[q] = k < len ? rin[k] : 0u;
      }
    }
  };
  uint32_t ridx[PT_ITEMS], nridx[PT_ITEMS];
  int jcur = 0, jnext = 0;
  load_rows(blockIdx.x, ridx, jcur);
  int par = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, par ^= 1) {
    uint32_t* const bits = s_bits[par];
    const int j = jcur;
    const PartParent pp = s_pp[j];
    const int64_t cnt_j = pp.cnt;
    const int64_t start_j = pp.start;
    const int64_t o = (int64_t)(t - s_tile_pref[j]) * PT_TILE;
    const int len = (int)min((int64_t)PT_TILE, cnt_j - o);
    const int f = pp.f, b = pp.b;
    const uint8_t* col = a.codesT + (size_t)f * a.ldT;
    const bool full = len == PT_TILE;   // every tile but a parent's last: no row predicates
    uint32_t code[PT_ITEMS];
#pragma unroll
    for (int q = 0; q < PT_ITEMS; ++q) code[q] = __ldg(col + ridx[q]);
    if (full) {
#pragma unroll
      for (int q = 0; q < PT_ITEMS; ++q) {
        const unsigned mw = __ballot_sync(0xffffffffu, code[q] <= (uint32_t)b);
        if (lane == 0) bits[q * (PT_THREADS / 32) + warp] = mw;
      }
    } else {
#pragma unroll
      for (int q = 0; q < PT_ITEMS; ++q) {
        const int k = q * PT_THREADS + tid;
        const unsigned mw = __ballot_sync(0xffffffffu, k < len && code[q] <= (uint32_t)b);
        if (lane == 0) bits[q * (PT_THREADS / 32) + warp] = mw;
      }
    }
    load_rows(t + gridDim.x, nridx, jnext);   // in flight across the reservation below
    __syncthreads();
    if (warp == 0) {   // group prefixes: lane L takes words PT_WPL*L ..; one atomic per child
      int c[PT_WPL];
      int lsum = 0;
#pragma unroll
      for (int w2 = 0; w2 < PT_WPL; ++w2) {
        c[w2] = __popc(bits[PT_WPL * lane + w2]);
        lsum += c[w2];
      }
      int inc = lsum;
      for (int off = 1; off < 32; off <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += u;
      }
      int ex = inc - lsum;
#pragma unroll
      for (int w2 = 0; w2 < PT_WPL; ++w2) {
        s_pre[PT_WPL * lane + w2] = ex;
        ex += c[w2];
      }
      if (lane == 31) {
        const int L = inc, R = len - inc;
        s_lb = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(&C.cnt[2 * j]), (unsigned long long)L);
        s_rb = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(&C.cnt[2 * j + 1]), (unsigned long long)R) + R;
        if (a.units) atomicAdd(&a.units[KC_PARTITION], (unsigned long long)len);
      }
    }
    __syncthreads();
    const int64_t lbase = start_j + s_lb;                // left rows: lbase + (lefts before the row)
    const int64_t rtop = start_j + cnt_j - s_rb;         // right rows: rtop + (rights before the row)
    if (full) {
      uint32_t* const lp = rout + lbase;
      uint32_t* const rp = rout + rtop;
#pragma unroll
      for (int q = 0; q < PT_ITEMS; ++q) {
        const int k = q * PT_THREADS + tid;
        const uint32_t mw = bits[q * (PT_THREADS / 32) + warp];
        const int pre = s_pre[q * (PT_THREADS / 32) + warp] + __popc(mw & lt);   // lefts before row k
        *(((mw >> lane) & 1u) ? lp + pre : rp + (k - pre)) = ridx[q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < PT_ITEMS; ++q) {
        const int k = q * PT_THREADS + tid;
        if (k < len) {
          const uint32_t mw = bits[q * (PT_THREADS / 32) + warp];
          const int pre = s_pre[q * (PT_THREADS / 32) + warp] + __popc(mw & lt);   // lefts before row k
          const bool left = (mw >> lane) & 1u;
          rout[left ? lbase + pre : rtop + (k - pre)] = ridx[q];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < PT_ITEMS; ++q) ridx[q] = nridx[q];
    jcur = jnext;
    // (no barrier: s_bits is double-buffered; the next writes of s_pre / s_lb follow the next
    // tile's first barrier)
  }
}

// ---------------------------------------------------------------------------------------------
// split evaluation: one thread-block CLUSTER of 8 CTAs per node of level d, one WARP per
// (node, feature f) — 4 warps per CTA.  Lane l owns bins 8l .. 8l+7; the warp forms the feature's
// histogram (sibling = parent - built, exact int64, written back for the next level),
// prefix-scans it, evaluates every threshold in fp64 (monotone veto on users) and reduces
// (loss desc, b asc) into its CTA's shared memory.  After a cluster barrier, warp 0 of the
// cluster's first CTA reads the 32 per-feature results through distributed shared memory,
// reduces them (loss desc, f asc, b asc) and writes the tree; a second barrier keeps the other
// CTAs' shared memory alive until then.  Every index and scalar the kernel needs is loaded at
// entry (one round trip).
constexpr int SP3_WARPS = 4;
constexpr int SP3_CLUSTER = 32 / SP3_WARPS;   // 8 CTAs = the node's 32 features
// O6 for feature f of node k of level d, by one warp (lane l owns bins 8l .. 8l+7): the feature's
// histogram (sibling = parent - built, exact int64, written back for the next level), prefix scan,
// fp64 gains with the monotone veto, best (loss desc, b asc).  Lane 0 receives the result in r.
// Returns false when the node does not exist (its parent did not split).
// the node's scalars split_feature loaded, reused by the node's decision (split_node): one fewer
// dependent round trip to global memory in the last-arriving warp
struct NodeScalars {
  double lo, hi;
  int t;
  uint32_t mgb, mhb;
};
__device__ __forceinline__ bool split_feature(const FitArgs& a, const int d, const int k, const int f, const int lane,
                                              FeatBest& r, const int side_in = -1, NodeScalars* ns = nullptr) {
  const LevelView& V = a.lv[d];
  const int j = k >> 1;                                     // parent (level d-1)
  // ---- independent loads, all issued up front
  const int t = *a.d_tree;
  const int pf = (d == 0) ? 0 : a.lv[d - 1].split_f[j];
  // (the level histogram's fold-in passes the built side it computed: V.built may not be visible yet)
  const int side = (d == 0) ? 0 : side_in >= 0 ? side_in : V.built[j];
  const int pside = (d >= 2) ? a.lv[d - 1].built[j >> 1] : 0;
  const double lo = (d == 0) ? -INFINITY : V.lo[k], hi = (d == 0) ? INFINITY : V.hi[k];
  const int nthr = a.ncuts[f];   // thresholds b = 0 .. nbins_f - 2
  if (d > 0 && pf < 0) {         // node absent (uniform over the node's warps)
    if (f == 0 && lane == 0) V.split_f[k] = -1;
    return false;
  }
  const uint32_t mgb = a.maxg[t], mhb = a.maxh[t];
  if (ns) *ns = NodeScalars{lo, hi, t, mgb, mhb};
  int64_t* Hself;
  int64_t g8[8], h8[8];
  if (d == 0) {
    Hself = a.H[0];
  } else {
    const bool is_built = (k & 1) == side;
    Hself = a.H[d & 1] + (size_t)(is_built ? j : (1 << (d - 1)) + j) * SLOT;
    if (!is_built) {
      // parent's slot at level d-1 (node_slot without the dependent load)
      const int pslot = (d == 1) ? 0 : (((j & 1) == pside) ? (j >> 1) : (1 << (d - 2)) + (j >> 1));
      const longlong2* Hp = reinterpret_cast<const longlong2*>(a.H[(d - 1) & 1] + (size_t)pslot * SLOT);
      const longlong2* Hb = reinterpret_cast<const longlong2*>(a.H[d & 1] + (size_t)j * SLOT);
      longlong2* Hs = reinterpret_cast<longlong2*>(Hself);
      const int eg0 = (f * kBins + lane * 8) / 2, eh0 = (kHistBins + f * kBins + lane * 8) / 2;
      longlong2 pg[4], bg2[4], ph[4], bh2[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {   // (L2 loads: the built histogram may come from other CTAs' atomics)
        pg[q] = __ldcg(Hp + eg0 + q);
        bg2[q] = __ldcg(Hb + eg0 + q);
        ph[q] = __ldcg(Hp + eh0 + q);
        bh2[q] = __ldcg(Hb + eh0 + q);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        g8[2 * q] = pg[q].x - bg2[q].x;
        g8[2 * q + 1] = pg[q].y - bg2[q].y;
        h8[2 * q] = ph[q].x - bh2[q].x;
        h8[2 * q + 1] = ph[q].y - bh2[q].y;
        if (d + 1 < a.D) {   // (kept for the next level's sibling subtraction; the last level's is not)
          Hs[eg0 + q] = make_longlong2(g8[2 * q], g8[2 * q + 1]);
          Hs[eh0 + q] = make_longlong2(h8[2 * q], h8[2 * q + 1]);
        }
      }
    }
  }
  if (d == 0 || (k & 1) == side) {
    const longlong2* G2 = reinterpret_cast<const longlong2*>(Hself + f * kBins + lane * 8);
    const longlong2* H2 = reinterpret_cast<const longlong2*>(Hself + kHistBins + f * kBins + lane * 8);
    longlong2 gv[4], hv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      gv[q] = __ldcg(G2 + q);
      hv[q] = __ldcg(H2 + q);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      g8[2 * q] = gv[q].x;
      g8[2 * q + 1] = gv[q].y;
      h8[2 * q] = hv[q].x;
      h8[2 * q + 1] = hv[q].y;
    }
  }
  if (d == 0 && a.hroot && t == 0) {   // h_fixed: keep tree 0's root q_h histogram
    longlong2* hs = reinterpret_cast<longlong2*>(a.hroot + f * kBins + lane * 8);
#pragma unroll
    for (int q = 0; q < 4; ++q) hs[q] = make_longlong2(h8[2 * q], h8[2 * q + 1]);
  }
#pragma unroll
  for (int q = 1; q < 8; ++q) {
    g8[q] += g8[q - 1];
    h8[q] += h8[q - 1];
  }
  int64_t ig = g8[7], ih = h8[7];
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t ug = __shfl_up_sync(0xffffffffu, ig, o), uh = __shfl_up_sync(0xffffffffu, ih, o);
    if (lane >= o) {
      ig += ug;
      ih += uh;
    }
  }
  const int64_t bgp = ig - g8[7], bhp = ih - h8[7];
  const int64_t Gq = __shfl_sync(0xffffffffu, ig, 31), Hq = __shfl_sync(0xffffffffu, ih, 31);
  bool fin = f < a.F;
  if (fin && (a.rf ? a.max_features < 1.0f : a.colsample < 1.0f)) {
    // GBDT: the tree's column sample (O6.3); random forest (R35): the node's own sample, keys
    // rng4(seed, 2 target + 1, t, (k + 1) 32 + f) with k the node's complete-tree index
    const int F = a.F;
    int nkeep = (int)ceil((double)(a.rf ? a.max_features : a.colsample) * (double)F);
    if (nkeep < 1) nkeep = 1;
    const uint64_t c0 = a.rf ? (uint64_t)((1 << d) + k) * 32u : 0u;   // (1 << d) - 1 + k + 1
    const uint64_t kf = rng4(a.seed, (uint64_t)(2 * a.target + 1), (uint64_t)t, c0 + (uint64_t)f);
    const uint64_t kl = lane < F ? rng4(a.seed, (uint64_t)(2 * a.target + 1), (uint64_t)t, c0 + (uint64_t)lane) : ~0ull;
    const unsigned less = __ballot_sync(0xffffffffu, lane < F && (kl < kf || (kl == kf && lane < f)));
    fin = __popc(less) < nkeep;
  }
  const int eg = exp_of(__uint_as_float(mgb)), eh = exp_of(__uint_as_float(mhb));
  const double sgi = exp2i(eg - a.K), shi = exp2i(eh - a.K);
  const double lambda = a.lambda, mcw = a.mcw;
  double bl = -INFINITY;
  int bb = 0x7fffffff;
  int64_t bGL = 0, bHL = 0;
  if (fin) {
    if (lane * 8 < nthr) {
      const double G = dequant(Gq, sgi), H = dequant(Hq, shi);
      const double gainP = calc_gain(G, H, calc_weight(G, H, lo, hi, lambda, mcw), lambda);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int b = lane * 8 + q;
        if (b < nthr) {
          const int64_t GLq = bgp + g8[q], HLq = bhp + h8[q];
          const double GL = dequant(GLq, sgi), HL = dequant(HLq, shi);
          const double GR = dequant(Gq - GLq, sgi), HR = dequant(Hq - HLq, shi);
          if (HL >= mcw && HR >= mcw) {
            const double wl = calc_weight(GL, HL, lo, hi, lambda, mcw);
            const double wr = calc_weight(GR, HR, lo, hi, lambda, mcw);
            if (!(a.monotone && f == a.users_col && wl > wr)) {
              const double loss =
                  __dsub_rn(__dadd_rn(calc_gain(GL, HL, wl, lambda), calc_gain(GR, HR, wr, lambda)), gainP);
              if (loss > bl) {   // b ascending within the lane: strict keeps the smaller b
                bl = loss;
                bb = b;
                bGL = GLq;
                bHL = HLq;
              }
            }
          }
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ol = __shfl_down_sync(0xffffffffu, bl, o);
    const int ob = __shfl_down_sync(0xffffffffu, bb, o);
    const int64_t oG = __shfl_down_sync(0xffffffffu, bGL, o), oH = __shfl_down_sync(0xffffffffu, bHL, o);
    if (ol > bl || (ol == bl && ob < bb)) {
      bl = ol;
      bb = ob;
      bGL = oG;
      bHL = oH;
    }
  }
  if (lane == 0) {
    r.loss = bl;
    r.b = bb;
    r.valid = (bl > -INFINITY) ? 1 : 0;
    r.GLq = bGL;
    r.HLq = bHL;
    r.Gq = Gq;
    r.Hq = Hq;
  }
  return true;
}

// the node's decision (O6 argmax over features, O7 children, O8 leaves), by one warp: lane l holds
// feature l's result
__device__ __forceinline__ void split_node(const FitArgs& a, const int d, const int k, const int lane, int rvalid,
                                           int rb, double rloss, int64_t rGL, int64_t rHL, int64_t rG, int64_t rH,
                                           const NodeScalars* ns = nullptr) {
  const LevelView& V = a.lv[d];
  const int t = ns ? ns->t : *a.d_tree;
  const double lo = ns ? ns->lo : (d == 0) ? -INFINITY : V.lo[k], hi = ns ? ns->hi : (d == 0) ? INFINITY : V.hi[k];
  const int eg = exp_of(__uint_as_float(ns ? ns->mgb : a.maxg[t])), eh = exp_of(__uint_as_float(ns ? ns->mhb : a.maxh[t]));
  const double sgi = exp2i(eg - a.K), shi = exp2i(eh - a.K);
  const double lambda = a.lambda, mcw = a.mcw;
  double ml = rvalid ? rloss : -INFINITY;
  int mf = lane, mb = rb;
  for (int o = 16; o > 0; o >>= 1) {
    const double ol = __shfl_down_sync(0xffffffffu, ml, o);
    const int of = __shfl_down_sync(0xffffffffu, mf, o), ob = __shfl_down_sync(0xffffffffu, mb, o);
    if (ol > ml || (ol == ml && (of < mf || (of == mf && ob < mb)))) {
      ml = ol;
      mf = of;
      mb = ob;
    }
  }
  ml = __shfl_sync(0xffffffffu, ml, 0);
  mf = __shfl_sync(0xffffffffu, mf, 0);
  mb = __shfl_sync(0xffffffffu, mb, 0);
  const int64_t GLs = __shfl_sync(0xffffffffu, rGL, mf), HLs = __shfl_sync(0xffffffffu, rHL, mf);
  // node totals from feature 0 (always < F): the histogram kernels leave features >= F empty
  const int64_t GqN = __shfl_sync(0xffffffffu, rG, 0), HqN = __shfl_sync(0xffffffffu, rH, 0);
  if (lane != 0) return;
  int32_t* const tfeat = a.tfeat + (size_t)t * a.nn;
  int32_t* const tbin = a.tbin + (size_t)t * a.nn;
  float* const tthr = a.tthr + (size_t)t * a.nn;
  float* const tval = a.tval + (size_t)t * a.nn;
  double* const tgain = a.tgain + (size_t)t * a.nn;
  const double G = dequant(GqN, sgi), H = dequant(HqN, shi);
  const double wP = calc_weight(G, H, lo, hi, lambda, mcw);
  const int gk = (1 << d) - 1 + k;
  if (ml > 1e-6) {
    const int fs = mf, bs = mb;
    const double GL = dequant(GLs, sgi), HL = dequant(HLs, shi);
    const double GR = dequant(GqN - GLs, sgi), HR = dequant(HqN - HLs, shi);
    const double wl = calc_weight(GL, HL, lo, hi, lambda, mcw);
    const double wr = calc_weight(GR, HR, lo, hi, lambda, mcw);
    double loL = lo, hiL = hi, loR = lo, hiR = hi;
    if (a.monotone && fs == a.users_col) {
      const double mid = __dmul_rn(__dadd_rn(wl, wr), 0.5);
      hiL = mid;
      loR = mid;
    }
    V.split_f[k] = fs;
    V.split_b[k] = bs;
    tfeat[gk] = fs;
    tbin[gk] = bs;
    tthr[gk] = a.cuts[fs * (kBins - 1) + bs];   // (8-bit code path: cut stride 255)
    tval[gk] = 0.0f;
    tgain[gk] = ml;   // the split's loss reduction (MDI)
    if (d + 1 < a.D) {
      const LevelView& N = a.lv[d + 1];
      // sharded fits build the child with the smaller hessian sum (an exact global integer, so every
      // rank makes the same choice without exchanging child counts); unsharded ones the smaller
      // row count (decided by the level histogram kernel) — either way sibling = parent - built
      if (a.built_by_h) N.built[k] = (HLs <= HqN - HLs) ? 0 : 1;
      N.cnt[2 * k] = 0;   // k_part's child cursors
      N.cnt[2 * k + 1] = 0;
      N.lo[2 * k] = loL;
      N.hi[2 * k] = hiL;
      N.lo[2 * k + 1] = loR;
      N.hi[2 * k + 1] = hiR;
    } else {
      // children at max depth are leaves: v = (float)(eta * W(G, H, lo, hi))
      tfeat[2 * gk + 1] = -1;
      tval[2 * gk + 1] = leaf_value(a, calc_weight(GL, HL, loL, hiL, lambda, mcw));
      tfeat[2 * gk + 2] = -1;
      tval[2 * gk + 2] = leaf_value(a, calc_weight(GR, HR, loR, hiR, lambda, mcw));
    }
  } else {
    V.split_f[k] = -1;
    tfeat[gk] = -1;
    tval[gk] = leaf_value(a, wP);
  }
}

template <bool CL>
__global__ void __launch_bounds__(SP3_WARPS * 32) k_split3(const FitPair fp, const int d) {
  pdl_wait();
  const FitArgs& a = fp.t[blockIdx.y];
  __shared__ FeatBest s_fb[SP3_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = blockIdx.x / SP3_CLUSTER;                  // node of level d
  const int f = (blockIdx.x % SP3_CLUSTER) * SP3_WARPS + warp;
  const LevelView& V = a.lv[d];
  FeatBest r;
  NodeScalars ns;
  if (!split_feature(a, d, k, f, lane, r, -1, &ns)) return;
  if (lane == 0) {
    if (CL) s_fb[warp] = r;
    else a.fbest[(size_t)k * 32 + f] = r;
  }
  // ---- the node's reduction, by one warp: lane l takes feature l's result
  int rvalid, rb;
  double rloss;
  int64_t rGL, rHL, rG, rH;
  if constexpr (CL) {   // cluster launch: results exchanged through distributed shared memory
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (blockIdx.x % SP3_CLUSTER != 0 || warp != 0) {
      cluster.sync();   // keep this CTA's s_fb readable until the reduction warp has read it
      return;
    }
    const FeatBest* rf = cluster.map_shared_rank(&s_fb[0], lane / SP3_WARPS) + (lane % SP3_WARPS);
    rvalid = rf->valid;
    rb = rf->b;
    rloss = rf->loss;
    rGL = rf->GLq;
    rHL = rf->HLq;
    rG = rf->Gq;
    rH = rf->Hq;
    cluster.sync();
  } else {              // plain launch: the node's last-arriving warp (global ticket) reduces
    int last = 0;
    if (lane == 0) {
      __threadfence();
      last = atomicAdd(&V.done[k], 1) == 31;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
    const volatile FeatBest* rf = a.fbest + (size_t)k * 32 + lane;
    rvalid = rf->valid;
    rb = rf->b;
    rloss = rf->loss;
    rGL = rf->GLq;
    rHL = rf->HLq;
    rG = rf->Gq;
    rH = rf->Hq;
    if (lane == 0) V.done[k] = 0;
  }
  split_node(a, d, k, lane, rvalid, rb, rloss, rGL, rHL, rG, rH, &ns);
}


#include "hist3.cuh"

using Upd3Kernel = void (*)(const FitPair);
static Upd3Kernel upd3_kernel(int D) {
  if (D == 8) return k_upd3<8>;
  if (D == 6) return k_upd3<6>;
  return k_upd3<0>;
}
// fused update kernel: LLMP_UPD = 2 (default) change-mask k_hist2 with the precomputed masks; 3 the
// bulk-staged change-row k_upd3 (measured slower: 385 vs 311 us per paired launch on C3 — the pass is
// issue-bound, and the precomputed masks cost less than per-batch change tests)
static int upd_kernel() {
  static const int v = getenv("LLMP_UPD") ? atoi(getenv("LLMP_UPD")) : 2;
  return v == 3 ? 3 : 2;
}
// ---------------------------------------------------------------------------------------------
// leaf routing + prediction update + next tree's gradient maxima
constexpr int UPD_THREADS = 256;
constexpr int MAX_NODES = (1 << (kMaxDepth + 1)) - 1;

__device__ __forceinline__ void block_max2(float& a, float& b, float* s_a, float* s_b) {
  for (int o = 16; o > 0; o >>= 1) {
    a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_a[warp] = a;
    s_b[warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w2 = 1; w2 < (int)(blockDim.x >> 5); ++w2) {
      a = fmaxf(a, s_a[w2]);
      b = fmaxf(b, s_b[w2]);
    }
  }
}

constexpr int UPD_R = 4;   // rows per thread per iteration (independent traversals for ILP)
__global__ void __launch_bounds__(UPD_THREADS) k_update(const FitPair fp) {
  const FitArgs& a = fp.t[blockIdx.y];
  const int t = *a.d_tree;
  const int32_t* const tfeat = a.tfeat + (size_t)t * a.nn;
  const int32_t* const tbin = a.tbin + (size_t)t * a.nn;
  const float* const tval = a.tval + (size_t)t * a.nn;
  __shared__ int8_t s_feat[MAX_NODES];
  __shared__ uint8_t s_bin[MAX_NODES];
  __shared__ float s_val[MAX_NODES];
  __shared__ __align__(16) uint8_t s_row[UPD_R][UPD_THREADS * 32];
  __shared__ float s_ma[UPD_THREADS / 32], s_mb[UPD_THREADS / 32];
  const int tid = threadIdx.x;
  for (int i = tid; i < a.nn; i += UPD_THREADS) {   // a.tfeat/tbin/tval point at tree t
    const int f = tfeat[i];
    s_feat[i] = (int8_t)(f < 0 ? -1 : f);
    s_bin[i] = (uint8_t)tbin[i];
    s_val[i] = tval[i];
  }
  __syncthreads();
  const bool has_next = t + 1 < a.T;
  float mg = 0.f, mh = 0.f;
  const int64_t stride = (int64_t)gridDim.x * UPD_THREADS;
  for (int64_t i0 = (int64_t)blockIdx.x * UPD_THREADS + tid; i0 < a.n; i0 += stride * UPD_R) {
    float pv[UPD_R], yv[UPD_R], wv[UPD_R];
    uint4 cv0[UPD_R], cv1[UPD_R];
    // all loads first (clamped index, no branches), then the shared-memory stores
#pragma unroll
    for (int q = 0; q < UPD_R; ++q) {
      const int64_t i = min(i0 + q * stride, a.n - 1);
      const uint4* crow = reinterpret_cast<const uint4*>(a.codes + (size_t)i * kMaxF);
      cv0[q] = __ldg(crow);
      cv1[q] = __ldg(crow + 1);
      pv[q] = a.p[i];
      yv[q] = a.y[i];
      wv[q] = a.w[i];
    }
#pragma unroll
    for (int q = 0; q < UPD_R; ++q) {
      *reinterpret_cast<uint4*>(&s_row[q][tid * 32]) = cv0[q];
      *reinterpret_cast<uint4*>(&s_row[q][tid * 32 + 16]) = cv1[q];
    }
    int k[UPD_R];
#pragma unroll
    for (int q = 0; q < UPD_R; ++q) k[q] = 0;
    // fixed-trip traversal (a leaf stays put), the UPD_R rows interleaved
    for (int s = 0; s < a.D; ++s) {
#pragma unroll
      for (int q = 0; q < UPD_R; ++q) {
        const int f = s_feat[k[q]];
        if (f >= 0) k[q] = 2 * k[q] + 1 + (s_row[q][tid * 32 + f] > s_bin[k[q]] ? 1 : 0);
      }
    }
#pragma unroll
    for (int q = 0; q < UPD_R; ++q) {
      const int64_t i = i0 + q * stride;
      if (i < a.n) {
        const float pn = __fadd_rn(pv[q], s_val[k[q]]);  // O9: one fp32 rounding
        a.p[i] = pn;
        if (has_next) {
          float g, h;
          grad_pair(a, t + 1, a.row_offset + i, yv[q], wv[q], pn, g, h);
          mg = fmaxf(mg, fabsf(g));
          mh = fmaxf(mh, h);
        }
      }
    }
  }
  if (!has_next) return;
  block_max2(mg, mh, s_ma, s_mb);
  if (tid == 0) {
    atomicMax(&a.maxg[t + 1], __float_as_uint(mg));
    atomicMax(&a.maxh[t + 1], __float_as_uint(mh));
  }
}

// ---------------------------------------------------------------------------------------------
// base score (O3): quantise g = w*(0 - y), h = w over all rows; base = -G/H (lambda = 0)
constexpr int BASE_THREADS = 256;

__global__ void __launch_bounds__(BASE_THREADS) k_base_max(const FitArgs a) {
  __shared__ float s_a[BASE_THREADS / 32], s_b[BASE_THREADS / 32];
  float mg = 0.f, mh = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * BASE_THREADS + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * BASE_THREADS) {
    const float wv = a.w[i];
    const float g = __fmul_rn(wv, __fsub_rn(0.0f, a.y[i]));
    mg = fmaxf(mg, fabsf(g));
    mh = fmaxf(mh, wv);
  }
  block_max2(mg, mh, s_a, s_b);
  if (threadIdx.x == 0) {
    atomicMax(&a.maxg[a.T], __float_as_uint(mg));
    atomicMax(&a.maxh[a.T], __float_as_uint(mh));
  }
}

__global__ void __launch_bounds__(BASE_THREADS) k_base_sum(const FitArgs a, int64_t* sums) {
  const double sg = exp2i(a.K - exp_of(__uint_as_float(a.maxg[a.T])));
  const double sh = exp2i(a.K - exp_of(__uint_as_float(a.maxh[a.T])));
  int64_t gs = 0, hs = 0;
  for (int64_t i = (int64_t)blockIdx.x * BASE_THREADS + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * BASE_THREADS) {
    const float wv = a.w[i];
    gs += quantize(__fmul_rn(wv, __fsub_rn(0.0f, a.y[i])), sg);
    hs += quantize(wv, sh);
  }
  for (int o = 16; o > 0; o >>= 1) {
    gs += __shfl_xor_sync(0xffffffffu, gs, o);
    hs += __shfl_xor_sync(0xffffffffu, hs, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&sums[0]), (unsigned long long)gs);
    atomicAdd(reinterpret_cast<unsigned long long*>(&sums[1]), (unsigned long long)hs);
  }
}

// p = base for all rows; tree 0's gradient maxima
__global__ void __launch_bounds__(BASE_THREADS) k_base_init(const FitArgs a, const int64_t* sums, float* base_out) {
  __shared__ float s_a[BASE_THREADS / 32], s_b[BASE_THREADS / 32];
  const double G = dequant(sums[0], exp2i(exp_of(__uint_as_float(a.maxg[a.T])) - a.K));
  const double H = dequant(sums[1], exp2i(exp_of(__uint_as_float(a.maxh[a.T])) - a.K));
  // random forest (R33): no intercept — every tree predicts the mean of its bootstrap
  const float base = a.rf ? 0.0f : H > 0.0 ? (float)__ddiv_rn(-G, H) : 0.0f;
  if (blockIdx.x == 0 && threadIdx.x == 0) *base_out = base;
  float mg = 0.f, mh = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * BASE_THREADS + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * BASE_THREADS) {
    a.p[i] = base;
    if (a.T > 0) {
      const float wv = a.w[i];
      float g, h;
      grad_pair(a, 0, a.row_offset + i, a.y[i], wv, base, g, h);
      mg = fmaxf(mg, fabsf(g));
      mh = fmaxf(mh, h);
    }
  }
  block_max2(mg, mh, s_a, s_b);
  if (threadIdx.x == 0 && a.T > 0) {
    atomicMax(&a.maxg[0], __float_as_uint(mg));
    atomicMax(&a.maxh[0], __float_as_uint(mh));
  }
}

// RF (R34): this target's bootstrap weights of tree t = *d_tree + ahead: w_t,i = c_t,i w_i (fp32)
__global__ void k_rf_weights(const FitPair fp, int ahead) {
  pdl_wait();
  const FitArgs& a = fp.t[blockIdx.y];
  const int t = *a.d_tree + ahead;
  if (t >= a.T) return;
  float* wt = const_cast<float*>(a.w);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
    wt[i] = a.rf_boot ? __fmul_rn((float)poisson1(a.seed, t, a.row_offset + i), a.w_base[i]) : a.w_base[i];
}

__global__ void k_next_tree(int* d_tree) {
  pdl_wait();
  *d_tree += 1;
}
__global__ void k_stamp(unsigned long long* stamps) {
  unsigned long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  stamps[0] = ns;
}
// graph form: advance the tree index and keep the device-side while loop running while t < T
__global__ void k_next_tree_cond(int* d_tree, int T, cudaGraphConditionalHandle h, unsigned long long* stamps) {
  pdl_wait();
  const int t = *d_tree + 1;
  *d_tree = t;
  cudaGraphSetConditional(h, t < T ? 1u : 0u);
  if (stamps) {   // diagnostics (LLMP_ROUND_TIMES=1): device time at the end of each round
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    stamps[t] = ns;
  }
}

__global__ void k_fill_trees(int32_t* feat, int32_t* bin, float* thr, float* val, size_t count) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    feat[i] = -2;
    bin[i] = 0;
    thr[i] = 0.f;
    val[i] = 0.f;
  }
}

// ---------------------------------------------------------------------------------------------
// Eq. (4) weights and input validation
__global__ void k_validate(const float* X, const float* y, const int32_t* llm, const int32_t* prof, const float* w,
                           int64_t n, int F, int n_llm, int n_prof, int* flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool bad = !isfinite(y[2 * i]) || !isfinite(y[2 * i + 1]);
    if (w && !(isfinite(w[i]) && w[i] >= 0.0f)) bad = true;   // explicit weights: finite and >= 0
    if (llm && (llm[i] < 0 || llm[i] >= n_llm)) bad = true;
    if (prof && (prof[i] < 0 || prof[i] >= n_prof)) bad = true;
    if (bad) atomicOr(flag, 1);
  }
  // X as one flat array of n * F floats, coalesced 16-byte loads (X is cudaMalloc'ed or a torch
  // tensor: 16-byte aligned when its base is; a scalar head and tail otherwise)
  const int64_t m = n * (int64_t)F;
  const int64_t head = (int64_t)((16 - (reinterpret_cast<uintptr_t>(X) & 15)) & 15) / 4;
  const int64_t h = min(head, m);
  const int64_t nv = (m - h) / 4;
  const float4* X4 = reinterpret_cast<const float4*>(X + h);
  bool badx = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nv; e += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(X4 + e);
    badx |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
  }
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gt < h && !isfinite(X[gt])) badx = true;                    // unaligned head
  if (gt < m - h - 4 * nv && !isfinite(X[h + 4 * nv + gt])) badx = true;   // tail
  if (badx) atomicOr(flag, 1);
}

__global__ void k_weights_max(const float* y, const int32_t* llm, const int32_t* prof, int64_t n, int n_prof, double L1,
                              double L2, unsigned long long* Dmax) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = (int64_t)llm[i] * n_prof + prof[i];
    const double d1 = fabs(__dsub_rn((double)y[2 * i], L1));
    const double d2 = fabs(__dsub_rn((double)y[2 * i + 1], L2));
    atomicMax(&Dmax[2 * g], (unsigned long long)__double_as_longlong(d1));      // d >= 0: bit order = value order
    atomicMax(&Dmax[2 * g + 1], (unsigned long long)__double_as_longlong(d2));
  }
}

__global__ void k_weights_apply(const float* y, const int32_t* llm, const int32_t* prof, int64_t n, int n_prof,
                                double L1, double L2, const unsigned long long* Dmax, float* w, float* y0, float* y1) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = (int64_t)llm[i] * n_prof + prof[i];
    const float ya = y[2 * i], yb = y[2 * i + 1];
    const double d1 = fabs(__dsub_rn((double)ya, L1)), d2 = fabs(__dsub_rn((double)yb, L2));
    const double D1 = __longlong_as_double((long long)Dmax[2 * g]), D2 = __longlong_as_double((long long)Dmax[2 * g + 1]);
    const double w1 = D1 > 0.0 ? __dsub_rn(1.0, __ddiv_rn(d1, D1)) : 1.0;
    const double w2 = D2 > 0.0 ? __dsub_rn(1.0, __ddiv_rn(d2, D2)) : 1.0;
    w[i] = (float)__dmul_rn(__dadd_rn(w1, w2), 0.5);
    y0[i] = ya;
    y1[i] = yb;
  }
}

__global__ void k_weights_given(const float* y, const float* win, int64_t n, float* w, float* y0, float* y1) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    w[i] = win ? win[i] : 1.0f;
    y0[i] = y[2 * i];
    y1[i] = y[2 * i + 1];
  }
}

// Eq. (4) weights of a whole dataset (used by the CV's weighted MAPE)
void compute_weights(Ctx* ctx, const DatasetDev& ds, float L1, float L2, float* w) {
  const int64_t n = ds.n;
  DevBuf& d_y0 = ctx->workspace("cw_y0", n * 4);
  DevBuf& d_y1 = ctx->workspace("cw_y1", n * 4);
  const size_t ng = (size_t)ds.n_llm * ds.n_prof;
  DevBuf& d_D = ctx->workspace("cw_groupmax", ng * 2 * 8);
  LLMP_CUDA(cudaMemsetAsync(d_D.p, 0, d_D.bytes, ctx->stream));
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sms * 8);
  LLMP_LAUNCH(ctx, KC_WEIGHTS, n, k_weights_max, grid, 256, 0, ds.y, ds.llm, ds.prof, n, ds.n_prof, (double)L1,
              (double)L2, d_D.as<unsigned long long>());
  allreduce_max_u64(ctx, d_D.as<uint64_t>(), ng * 2);
  LLMP_LAUNCH(ctx, KC_WEIGHTS, n, k_weights_apply, grid, 256, 0, ds.y, ds.llm, ds.prof, n, ds.n_prof, (double)L1,
              (double)L2, d_D.as<unsigned long long>(), w, d_y0.as<float>(), d_y1.as<float>());
}

static bool split_cluster_env() {
  static const bool v = getenv("LLMP_SPLIT_CLUSTER") && atoi(getenv("LLMP_SPLIT_CLUSTER")) != 0;
  return v;
}

// ---------------------------------------------------------------------------------------------
void validate_hparams(const llmpilot_hparams& hp) {
  LLMP_REQUIRE(hp.n_trees >= 0, "n_trees must be >= 0");
  LLMP_REQUIRE(hp.max_depth >= 1 && hp.max_depth <= kMaxDepth, "max_depth must be in [1, 10]");
  LLMP_REQUIRE(hp.tree_method == 0 || hp.tree_method == 1, "tree_method must be 0 (hist) or 1 (exact)");
  LLMP_REQUIRE(hp.tree_method == 1 || (hp.max_bin >= 2 && hp.max_bin <= kMaxCuts16 + 1),
               "max_bin must be in [2, 1024]");
  LLMP_REQUIRE(hp.grad_bits >= 2 && hp.grad_bits <= kMaxGradBits, "grad_bits must be in [2, 14]");
  LLMP_REQUIRE(hp.subsample > 0.0f && hp.subsample <= 1.0f, "subsample must be in (0, 1]");
  LLMP_REQUIRE(hp.colsample_bytree > 0.0f && hp.colsample_bytree <= 1.0f, "colsample_bytree must be in (0, 1]");
  LLMP_REQUIRE(hp.lambda >= 0.0f && isfinite(hp.lambda), "lambda must be >= 0");
  LLMP_REQUIRE(hp.min_child_weight >= 0.0f && isfinite(hp.min_child_weight), "min_child_weight must be >= 0");
  LLMP_REQUIRE(isfinite(hp.eta), "eta must be finite");
  LLMP_REQUIRE(hp.model == 0 || hp.model == 1, "model must be 0 (GBDT) or 1 (random forest)");
  if (hp.model == 1) {
    LLMP_REQUIRE(hp.max_features > 0.0f && hp.max_features <= 1.0f, "max_features must be in (0, 1]");
    LLMP_REQUIRE(hp.subsample == 1.0f, "random forest: subsample must be 1 (the bootstrap samples the rows)");
    LLMP_REQUIRE(hp.monotone_users == 0, "random forest: monotone_users must be 0");
  }
}

static int grid_for(Ctx* ctx, int64_t n, int threads, int per_sm) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)ctx->sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

void fit_impl(Ctx* ctx, const DatasetDev& ds, const llmpilot_hparams& hp, float L1, float L2, ModelData& out,
              bool keep_train_pred) {
  validate_hparams(hp);
  const int64_t n = ds.n;
  const int F = ds.F, D = hp.max_depth, T = hp.n_trees;
  LLMP_REQUIRE(n >= 1 && n < (int64_t(1) << 30), "n_rows must be in [1, 2^30)");
  LLMP_REQUIRE(F >= 1 && F <= kMaxF, "n_features must be in [1, 32]");
  LLMP_REQUIRE(ds.users_col >= 0 && ds.users_col < F, "users_col out of range");
  LLMP_REQUIRE(isfinite(L1) && isfinite(L2) && L1 > 0.f && L2 > 0.f, "L1, L2 must be positive and finite");
  const bool eq4 = hp.use_eq4_weights != 0;
  LLMP_REQUIRE(!eq4 || (ds.llm && ds.prof && ds.n_llm >= 1 && ds.n_prof >= 1),
               "Eq. (4) weights need llm_id/profile_id and n_llm, n_prof >= 1");
  cudaStream_t s = ctx->stream;

  // diagnostics (LLMP_FIT_PHASES=1): host-synchronised phase times on stderr
  static const bool phases = getenv("LLMP_FIT_PHASES") && atoi(getenv("LLMP_FIT_PHASES")) != 0;
  auto ph_t0 = std::chrono::steady_clock::now();
  std::unique_ptr<NvtxRange> ph_range(new NvtxRange("validate"));
  auto phase = [&](const char* name) {
    ph_range.reset();
    static const char* const next_of[][2] = {{"validate", "weights"}, {"weights", "cuts+codes"}, {"cuts+codes", "state"},
                                             {"state", "base"}, {"base", "tree loop"}, {"loop", "to_host"},
                                             {"to_host", "upload"}};
    for (const auto& nx : next_of)
      if (!strcmp(nx[0], name)) ph_range.reset(new NvtxRange(nx[1]));
    if (!phases) return;
    LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[llmp] phase %-10s %9.3f ms\n", name, std::chrono::duration<double, std::milli>(t1 - ph_t0).count());
    ph_t0 = t1;
  };
  // ---- validation (NaN/Inf, id ranges) — one host sync per fit
  DevBuf& d_flag = ctx->workspace("flag", sizeof(int));
  LLMP_CUDA(cudaMemsetAsync(d_flag.p, 0, sizeof(int), s));
  LLMP_LAUNCH(ctx, KC_VALIDATE, n, k_validate, grid_for(ctx, n, 256, 8), 256, 0, ds.X, ds.y, eq4 ? ds.llm : nullptr,
              eq4 ? ds.prof : nullptr, eq4 ? nullptr : ds.w, n, F, ds.n_llm, ds.n_prof, d_flag.as<int>());
  // sharded: every rank must take the same decision, or the others would block in the next collective
  allreduce_max_u32(ctx, reinterpret_cast<uint32_t*>(d_flag.p), 1);
  int h_flag = 0;
  LLMP_CUDA(cudaMemcpyAsync(&h_flag, d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaStreamSynchronize(s));
  LLMP_REQUIRE(h_flag == 0, "dataset holds a non-finite X or y value, a negative or non-finite weight or an id out of range (on some rank)");

  phase("validate");
  // ---- weights (Eq. 4) + de-interleaved targets
  DevBuf& d_w = ctx->workspace("w", n * 4);
  DevBuf& d_y0 = ctx->workspace("y0", n * 4);
  DevBuf& d_y1 = ctx->workspace("y1", n * 4);
  if (eq4) {
    const size_t ng = (size_t)ds.n_llm * ds.n_prof;
    DevBuf& d_D = ctx->workspace("groupmax", ng * 2 * 8);
    LLMP_CUDA(cudaMemsetAsync(d_D.p, 0, ng * 2 * 8, s));
    LLMP_LAUNCH(ctx, KC_WEIGHTS, n, k_weights_max, grid_for(ctx, n, 256, 8), 256, 0, ds.y, ds.llm, ds.prof, n,
                ds.n_prof, (double)L1, (double)L2, d_D.as<unsigned long long>());
    allreduce_max_u64(ctx, d_D.as<uint64_t>(), ng * 2);
    LLMP_LAUNCH(ctx, KC_WEIGHTS, n, k_weights_apply, grid_for(ctx, n, 256, 8), 256, 0, ds.y, ds.llm, ds.prof, n,
                ds.n_prof, (double)L1, (double)L2, d_D.as<unsigned long long>(), d_w.as<float>(), d_y0.as<float>(),
                d_y1.as<float>());
  } else {
    LLMP_LAUNCH(ctx, KC_WEIGHTS, n, k_weights_given, grid_for(ctx, n, 256, 8), 256, 0, ds.y, ds.w, n, d_w.as<float>(),
                d_y0.as<float>(), d_y1.as<float>());
  }

  phase("weights");
  // ---- cuts + codes (row-major for histograms/routing, column-major for partitions)
  // this path keeps 8-bit codes (one 32-byte sector per row): at most 256 bins (exact: 256 distinct values)
  LLMP_REQUIRE(hp.tree_method == 1 || hp.max_bin <= kBins,
               "max_bin > 256 (16-bit codes) is supported by the batched small-fit path (cross-validation, n <= 8192 "
               "rows, depth <= 8); this fit path takes at most 256 bins");
  compute_cuts(ctx, ds.X, n, F, ds.row_offset, ds.n_global, hp.tree_method == 1 ? 0 : hp.max_bin, out.cuts,
               ctx->sharded());
  DevBuf& d_codes = ctx->workspace("codes", (size_t)n * kMaxF);
  const int64_t ldT = (n + 31) / 32 * 32;
  DevBuf& d_codesT = ctx->workspace("codesT", (size_t)ldT * kMaxF);
  LLMP_CUDA(cudaMemsetAsync(d_codesT.p, 0, (size_t)ldT * kMaxF, s));   // zero the padding rows
  compute_codes(ctx, ds.X, n, F, out.cuts, d_codes.as<uint8_t>(), d_codesT.as<uint8_t>(), ldT, nullptr);

  phase("cuts+codes");
  // ---- training state
  const int nn = (1 << (D + 1)) - 1;
  const int half_max = 1 << (D - 1);        // slots per histogram parity buffer
  // p of both targets: kept by the model (llmpilot_model_train_pred) or a reused workspace
  if (keep_train_pred) {
    out.d_train_pred.set_stream(s);
    out.d_train_pred.ensure((size_t)n * 4 * 2);
  }
  DevBuf& d_p = keep_train_pred ? out.d_train_pred : ctx->workspace("p", (size_t)n * 4 * 2);
  out.device = ctx->device;
  DevBuf& d_trees = ctx->workspace("trees", (size_t)2 * std::max(T, 1) * nn * 16);
  DevBuf& d_gain = ctx->workspace("gains", (size_t)2 * std::max(T, 1) * nn * 8);
  LLMP_CUDA(cudaMemsetAsync(d_gain.p, 0, d_gain.bytes, s));
  DevBuf& d_max = ctx->workspace("gradmax", (size_t)2 * 2 * (T + 1) * 4);
  DevBuf& d_sums = ctx->workspace("basesums", 2 * 2 * 8);
  DevBuf& d_base = ctx->workspace("base", 2 * 4);
  int32_t* feat_all = d_trees.as<int32_t>();
  int32_t* bin_all = feat_all + (size_t)2 * T * nn;
  float* thr_all = reinterpret_cast<float*>(bin_all + (size_t)2 * T * nn);
  float* val_all = thr_all + (size_t)2 * T * nn;
  if (T > 0)
    LLMP_LAUNCH(ctx, KC_MISC, 0, k_fill_trees, 256, 256, 0, feat_all, bin_all, thr_all, val_all, (size_t)2 * T * nn);
  LLMP_CUDA(cudaMemsetAsync(d_max.p, 0, d_max.bytes, s));
  LLMP_CUDA(cudaMemsetAsync(d_sums.p, 0, d_sums.bytes, s));
  int* d_tree = ctx->workspace("tree_idx", sizeof(int)).as<int>();

  // the two ensembles are independent: every tree-loop kernel grows both (blockIdx.y = target)
  // sharded (a communicator is attached): plain launches — the NCCL calls are never captured, in
  // particular not into the body of a conditional graph node.  A 1-rank communicator runs this same
  // sharded path (trivial collectives), which is how the GPU tests cover it on one device.
  const bool sharded = ctx->sharded();
  // NCCL-sharded fits replay each round as a captured graph with the collectives inside (host-side
  // replay: no conditional node around NCCL kernels); the in-process local group's collectives are
  // host barriers and cannot be captured
  const bool nccl_mode = ctx->nccl != nullptr;
  const bool graphs = T > 0 && !ctx->timing && ctx->use_graphs && (!sharded || nccl_mode);
  size_t lvl_nodes = 0;
  for (int d = 0; d <= D; ++d) lvl_nodes += (size_t)1 << d;
  const size_t tab_bytes = lvl_nodes * (8 /*start*/ + 8 /*cnt*/ + 8 /*gcnt*/ + 8 + 8 /*lo,hi*/ + 4 + 4 /*split*/ +
                                        4 /*built*/ + 4 /*done*/);
  // root histogram variant: run-length lane-per-feature (default) or the hybrid run/row-parallel
  // kernel (LLMP_ROOT2=1; faster on random codes, slower on paper-ordered rows).  The default
  // fuses each tree's update with the next tree's root histogram (LLMP_NOFUSE=1 disables).
  static const bool use_root2 = getenv("LLMP_ROOT2") && atoi(getenv("LLMP_ROOT2")) != 0;
  static const bool fused = !use_root2 && !(getenv("LLMP_NOFUSE") && atoi(getenv("LLMP_NOFUSE")) != 0);
  static const bool urow = !(getenv("LLMP_NO_UROW") && atoi(getenv("LLMP_NO_UROW")) != 0);
  static const bool pdl_env = !(getenv("LLMP_PDL") && atoi(getenv("LLMP_PDL")) == 0);
  // (every tree-loop kernel waits on griddepcontrol.wait before touching memory, so a kernel following
  // an NCCL kernel starts only once the collective is complete; the local group's host barriers are
  // outside any stream dependency and stay unlaunched-ahead)
  ctx->pdl = pdl_env && ctx->lgroup == nullptr;
  static const bool hist_swar = !(getenv("LLMP_HIST_SWAR") && atoi(getenv("LLMP_HIST_SWAR")) == 0);
  DevBuf& d_cm = ctx->workspace("cmask", (size_t)((n + 31) / 32) * 32 * 4);
  LLMP_LAUNCH(ctx, KC_MISC, n, k_cmask, grid_for(ctx, n, 256, 8), 256, 0, d_codes.as<uint8_t>(), n,
              d_cm.as<uint32_t>());
  const uint32_t* cmask = d_cm.as<uint32_t>();
  static const int hist1 = hist1_mask();
  // with h = w on every row of every tree (no row subsampling, not a random forest) the root's
  // q_h histogram is the same for every tree; the fused update then builds only the q_g channel and
  // the round copies q_h from tree 0's.  Sharded: the root slot is summed across ranks after the
  // update, and tree 0's saved q_h channel is already the global one, so rank 0 contributes it and the
  // other ranks zeros (an exact integer sum either way)
  static const bool hfix_env = !(getenv("LLMP_HFIX") && atoi(getenv("LLMP_HFIX")) == 0);
  const bool hfix = hfix_env && fused && hp.subsample >= 1.0f && hp.model == 0 && !(hist1 & 4) && upd_kernel() == 2;
  const int lvk = level_kernel();
  // split evaluation folded into k_hist3 (LLMP_FOLD=1; unsharded only: no all-reduce between the
  // histogram and the split).  Measured slower than the separate k_split3 launch (107 vs 55 + 14 us per
  // paired level on C3): one CTA evaluates a node's 64 (child, feature) tasks in four serial rounds
  // (~12 us), and the last-completed pieces put that on the kernel's tail, where k_split3 spreads
  // every node over 8 CTAs of the whole GPU
  static const bool fold_env = getenv("LLMP_FOLD") && atoi(getenv("LLMP_FOLD")) != 0;
  const bool fold = fold_env && lvk == 3 && !sharded && !split_cluster_env();
  FitArgs A[2];
  for (int tg = 0; tg < 2; ++tg) {
    // per-target workspaces: the fused update pass leaves the next tree's root histogram and
    // packed pairs in them, so the two ensembles never share one (also when they run in sequence)
    const std::string sx = (tg == 1) ? "_1" : "_0";
    FitArgs& a = A[tg];
    a = FitArgs{};
    a.n = n;
    a.row_offset = ds.row_offset;
    a.F = F;
    a.users_col = ds.users_col;
    a.D = D;
    a.K = hp.grad_bits;
    a.T = T;
    a.target = tg;
    a.codes = d_codes.as<uint8_t>();
    a.codesT = d_codesT.as<uint8_t>();
    a.ldT = ldT;
    a.w = d_w.as<float>();
    a.y = (tg == 0) ? d_y0.as<float>() : d_y1.as<float>();
    a.p = d_p.as<float>() + (size_t)tg * n;
    a.gp_root = ctx->workspace("gp_root" + sx, (size_t)n * 4).as<uint32_t>();
    a.sr[0] = ctx->workspace("ridx0" + sx, (size_t)n * 4).as<uint32_t>();
    a.sr[1] = ctx->workspace("ridx1" + sx, (size_t)n * 4).as<uint32_t>();
    a.H[0] = ctx->workspace("hist0" + sx, (size_t)half_max * SLOT * 8).as<int64_t>();
    a.H[1] = ctx->workspace("hist1" + sx, (size_t)half_max * SLOT * 8).as<int64_t>();
    a.cuts = out.cuts.d_cuts.as<float>();
    a.ncuts = out.cuts.d_ncuts.as<int32_t>();
    a.eta = (double)hp.eta;
    a.lambda = (double)hp.lambda;
    a.mcw = (double)hp.min_child_weight;
    a.subsample = hp.subsample;
    a.colsample = hp.colsample_bytree;
    a.seed = hp.seed;
    a.monotone = hp.monotone_users;
    a.fused_root = fused ? 1 : 0;
    a.urow = urow ? 1 : 0;
    a.hist_swar = hist_swar ? 1 : 0;
    a.built_by_h = sharded ? 1 : 0;
    a.rf = hp.model == 1 ? 1 : 0;
    a.rf_boot = hp.rf_bootstrap ? 1 : 0;
    a.max_features = hp.max_features;
    a.w_base = a.w;
    a.fq = ctx->workspace("fold_q" + sx, (size_t)FQ_INTS * 4).as<int>();
    if (a.rf) a.w = ctx->workspace("rf_w" + sx, (size_t)n * 4).as<float>();   // per-tree bootstrap weights
    a.cmask = cmask;
    a.hroot = hfix ? ctx->workspace("hroot" + sx, (size_t)kHistBins * 8).as<int64_t>() : nullptr;
    a.nn = nn;
    a.units = ctx->d_units;
    a.fbest = reinterpret_cast<FeatBest*>(ctx->workspace("featbest" + sx, (size_t)half_max * 32 * 48).p);
    a.d_tree = d_tree;
    a.maxg = d_max.as<uint32_t>() + (size_t)tg * 2 * (T + 1);
    a.maxh = a.maxg + (T + 1);
    a.tfeat = feat_all + (size_t)tg * T * nn;
    a.tbin = bin_all + (size_t)tg * T * nn;
    a.tthr = thr_all + (size_t)tg * T * nn;
    a.tval = val_all + (size_t)tg * T * nn;
    a.tgain = d_gain.as<double>() + (size_t)tg * T * nn;
    DevBuf& d_tab = ctx->workspace("tab" + sx, tab_bytes);
    uint8_t* tb = d_tab.as<uint8_t>();
    int64_t* start = reinterpret_cast<int64_t*>(tb);
    int64_t* cnt = start + lvl_nodes;
    int64_t* gcnt = cnt + lvl_nodes;
    double* lo = reinterpret_cast<double*>(gcnt + lvl_nodes);
    double* hi = lo + lvl_nodes;
    int32_t* sf = reinterpret_cast<int32_t*>(hi + lvl_nodes);
    int32_t* sb = sf + lvl_nodes;
    int32_t* bu = sb + lvl_nodes;
    int32_t* dn = bu + lvl_nodes;
    size_t off = 0;
    for (int d = 0; d <= D; ++d) {
      LevelView& L = a.lv[d];
      L.start = start + off;
      L.cnt = cnt + off;
      L.gcnt = gcnt + off;
      L.lo = lo + off;
      L.hi = hi + off;
      L.split_f = sf + off;
      L.split_b = sb + off;
      L.built = bu + off;
      L.done = dn + off;
      off += (size_t)1 << d;
    }
    LLMP_CUDA(cudaMemsetAsync(d_tab.p, 0, d_tab.bytes, s));
  }

  const int upd_grid = grid_for(ctx, n, UPD_THREADS, 8);
  const int base_grid = grid_for(ctx, n, BASE_THREADS, 8);
  ensure_smem_attr((const void*)k_hist_root2, R2_SMEM);
  ensure_smem_attr((const void*)k_hist<HM_ROOT>, HIST_SMEM);
  ensure_smem_attr((const void*)k_hist<HM_LEVEL>, HIST_SMEM);
  ensure_smem_attr((const void*)k_hist2<HM_ROOT>, H2_SMEM);
  ensure_smem_attr((const void*)k_hist2<HM_LEVEL>, H2_SMEM);
  ensure_smem_attr((const void*)k_hist3<HM_LEVEL, false>, H3_SMEM);
  ensure_smem_attr((const void*)k_hist3<HM_LEVEL, true>, H3_SMEM);
  // the fused update kernels' dynamic shared memory depends on the depth (the tree they route)
  ensure_smem_attr((const void*)k_hist<HM_UPDROOT>, HIST_SMEM + updroot_tree_smem(D));
  const Hist2Kernel k_upd2 = updroot2_kernel(D, hfix);
  ensure_smem_attr((const void*)k_upd2, H2_SMEM + updroot_tree_smem(D));
  // both ensembles' fused update in one pass (LLMP_DUAL=0 keeps one pass per ensemble):
  // needs the tree-invariant q_h channel, one weight vector and the k_hist2 update kernel
  static const bool dual_env = !(getenv("LLMP_DUAL") && atoi(getenv("LLMP_DUAL")) == 0);
  const bool dual = dual_env && hfix && A[0].w == A[1].w && upd_kernel() == 2;
  const Hist2Kernel k_upd2d = updroot2_kernel(D, false, true);
  ensure_smem_attr((const void*)k_upd2d, H2_SMEM + updroot_tree_smem(D));
  const Upd3Kernel k_up3 = upd3_kernel(D);
  ensure_smem_attr((const void*)k_up3, U3_SMEM + updroot_tree_smem(D));
  const int updk = upd_kernel();
  const DbgArgs nodbg{};

  phase("state");
  const bool rf = hp.model == 1;
  const int rfw_grid = grid_for(ctx, n, 256, 8);
  LLMP_CUDA(cudaMemsetAsync(d_tree, 0, sizeof(int), s));
  // ---- base scores (O3) and tree 0's gradient maxima
  for (int tg = 0; tg < 2; ++tg) {
    const FitArgs& a = A[tg];
    int64_t* sums = d_sums.as<int64_t>() + 2 * tg;
    if (rf) {   // tree 0's bootstrap weights (R34)
      FitPair f1;
      f1.t[0] = a;
      LLMP_LAUNCH(ctx, KC_MISC, n, k_rf_weights, dim3(rfw_grid, 1), 256, 0, f1, 0);
    }
    LLMP_LAUNCH(ctx, KC_BASE, n, k_base_max, base_grid, BASE_THREADS, 0, a);
    allreduce_max_u32(ctx, a.maxg + T, 1);
    allreduce_max_u32(ctx, a.maxh + T, 1);
    LLMP_LAUNCH(ctx, KC_BASE, n, k_base_sum, base_grid, BASE_THREADS, 0, a, sums);
    allreduce_sum_i64(ctx, sums, 2);
    LLMP_LAUNCH(ctx, KC_BASE, n, k_base_init, base_grid, BASE_THREADS, 0, a, sums, d_base.as<float>() + tg);
    if (T > 0) {
      allreduce_max_u32(ctx, a.maxg, 1);
      allreduce_max_u32(ctx, a.maxh, 1);
    }
  }

  // one tree of each target = a fixed sequence of launches (blockIdx.y = target) that reads the
  // tree index from the device; one "round" (tree t of both ensembles + the index advance) is
  // captured once into a CUDA graph and replayed T times (plain launches when timing is on)
  // split kernel: plain launch with a global ticket per node (default) or one thread-block cluster
  // per node exchanging results through distributed shared memory (LLMP_SPLIT_CLUSTER=1)
  phase("base");
  FitPair FP;
  FP.t[0] = A[0];
  FP.t[1] = A[1];
  static const bool split_cluster = split_cluster_env();
  // diagnostic (LLMP_SPLIT_TWICE=1): every split launch is issued twice — result-neutral (the second
  // launch recomputes the same decisions from the same histograms), so the step-time difference is the
  // marginal cost of the split launches inside the graph
  static const bool split_twice = getenv("LLMP_SPLIT_TWICE") && atoi(getenv("LLMP_SPLIT_TWICE")) != 0;
  auto split = [&](const FitPair& fp, int ny, int d) {
    const dim3 grid((1 << d) * SP3_CLUSTER, ny);
    if (!split_cluster) {
      LLMP_LAUNCH_PDL(ctx, KC_SPLIT, ny << d, k_split3<false>, grid, SP3_WARPS * 32, 0, fp, d);
      if (split_twice) LLMP_LAUNCH_PDL(ctx, KC_SPLIT, ny << d, k_split3<false>, grid, SP3_WARPS * 32, 0, fp, d);
      return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(SP3_WARPS * 32);
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = SP3_CLUSTER;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t ev = nullptr;
    ctx->before(KC_SPLIT, &ev);
    LLMP_CUDA(cudaLaunchKernelEx(&cfg, k_split3<true>, fp, d));
    ctx->after(KC_SPLIT, ev, (double)(ny << d));
  };
  static const bool round_times = getenv("LLMP_ROUND_TIMES") && atoi(getenv("LLMP_ROUND_TIMES")) != 0;
  unsigned long long* stamps = nullptr;
  if (round_times && T > 0) {
    stamps = ctx->workspace("round_stamps", (size_t)(T + 1) * 8).as<unsigned long long>();
  }
  // one tree of the targets in `fp` (ny = 2: both as blockIdx.y = 0, 1; ny = 1: fp.t[0] only)
  auto trees = [&](const FitPair& fp, int ny) {
    const cudaStream_t st = ctx->stream;
    // histogram kernels: 2 CTAs per SM in total, but no more CTAs than 2048-row slices of the data
    // (small fits would otherwise launch hundreds of CTAs that only zero their shared histograms)
    const dim3 hg((unsigned)std::min<int64_t>(ctx->sms * 2 / ny, std::max<int64_t>(1, (n + 2047) / 2048)), ny);
    // k_upd3: one CTA per SM and ensemble
    const dim3 hu3((unsigned)std::min<int64_t>(std::max(1, ctx->sms / ny), std::max<int64_t>(1, (n + 2047) / 2048)), ny);
    // k_hist3: one CTA per SM; one launch covers the built children of every ensemble in fp
    const dim3 hg3((unsigned)std::min<int64_t>(ctx->sms, std::max<int64_t>(1, (n * ny + 2047) / 2048)));
    // fused: the previous round's update pass built this root already unless root_needed
    if (fused) {
      LLMP_LAUNCH_PDL(ctx, KC_MISC, 0, k_root_fix, dim3(1, ny), 1024, 0, fp);
    } else {
      for (int q = 0; q < ny; ++q) LLMP_CUDA(cudaMemsetAsync(fp.t[q].H[0], 0, (size_t)SLOT * 8, st));
    }
    if (use_root2) LLMP_LAUNCH(ctx, KC_HIST_ROOT, ny * n, k_hist_root2, hg, R2_THREADS, R2_SMEM, fp);
    else if (hist1 & 1) LLMP_LAUNCH(ctx, KC_HIST_ROOT, ny * n, k_hist<HM_ROOT>, hg, HIST_THREADS, HIST_SMEM, fp, 0, 0, nodbg);
    else LLMP_LAUNCH_PDL(ctx, KC_HIST_ROOT, ny * n, k_hist2<HM_ROOT>, hg, H2_THREADS, H2_SMEM, fp, 0, 0, nodbg);
    nccl_group_start(ctx);
    for (int q = 0; q < ny; ++q) allreduce_sum_i64(ctx, fp.t[q].H[0], SLOT);
    nccl_group_end(ctx);
    split(fp, ny, 0);
    static const char* const level_name[] = {"level 0", "level 1", "level 2", "level 3", "level 4",
                                             "level 5", "level 6", "level 7", "level 8", "level 9"};
    for (int d = 1; d < D; ++d) {
      NvtxRange lr(level_name[d]);
      const int tiles_d = (int)((n + PT_TILE - 1) / PT_TILE) + (1 << (d - 1));
      // persistent tile loop (upper bound of the level's tile count: one partial tile per parent)
      LLMP_LAUNCH_PDL(ctx, KC_PARTITION, ny * n, k_part, dim3(std::min(tiles_d, PT_CTAS_PER_SM / ny * ctx->sms), ny),
                  PT_THREADS, 0, fp, d);
      if (lvk == 3 && fold) LLMP_LAUNCH_PDL(ctx, KC_HIST, 0, (k_hist3<HM_LEVEL, true>), hg3, H3_THREADS, H3_SMEM, fp, ny, d, nodbg);
      else if (lvk == 3) LLMP_LAUNCH_PDL(ctx, KC_HIST, 0, (k_hist3<HM_LEVEL, false>), hg3, H3_THREADS, H3_SMEM, fp, ny, d, nodbg);
      else if (lvk == 1) LLMP_LAUNCH_PDL(ctx, KC_HIST, 0, k_hist<HM_LEVEL>, hg, HIST_THREADS, HIST_SMEM, fp, d, 0, nodbg);
      else LLMP_LAUNCH(ctx, KC_HIST, 0, k_hist2<HM_LEVEL>, hg, H2_THREADS, H2_SMEM, fp, d, 0, nodbg);
      nccl_group_start(ctx);   // both targets' built-child histograms in one NCCL launch
      for (int q = 0; q < ny; ++q) allreduce_sum_i64(ctx, fp.t[q].H[d & 1], (size_t)SLOT << (d - 1));
      nccl_group_end(ctx);
      if (!fold) split(fp, ny, d);
    }
    if (dual) {
      // the dual update (after the join) accumulates tree t+1's root q_g into the root slot: reset it
      // here, at the end of this ensemble's own branch (its last split has consumed the level-0 slot),
      // so the reset overlaps the other branch instead of sitting between the join and the update.
      // q_g channel zeroed, q_h channel = tree 0's (rank 0; zeros on the other ranks)
      for (int q = 0; q < ny; ++q) {
        if (!sharded || ctx->rank == 0) {
          LLMP_CUDA(cudaMemsetAsync(fp.t[q].H[0], 0, (size_t)kHistBins * 8, st));
          LLMP_CUDA(cudaMemcpyAsync(fp.t[q].H[0] + kHistBins, fp.t[q].hroot, (size_t)kHistBins * 8,
                                    cudaMemcpyDeviceToDevice, st));
        } else {
          LLMP_CUDA(cudaMemsetAsync(fp.t[q].H[0], 0, (size_t)SLOT * 8, st));
        }
      }
    }
    // RF: tree t+1's bootstrap weights, read by the update's gradients (and the next root rebuild)
    if (rf) LLMP_LAUNCH_PDL(ctx, KC_MISC, ny * n, k_rf_weights, dim3(rfw_grid, ny), 256, 0, fp, 1);
    if (fused && !dual) {   // update tree t + root histogram of tree t+1 (into the now free root slot)
      for (int q = 0; q < ny; ++q) {
        if (hfix && (!sharded || ctx->rank == 0)) {   // q_g channel zeroed, q_h channel = tree 0's
          LLMP_CUDA(cudaMemsetAsync(fp.t[q].H[0], 0, (size_t)kHistBins * 8, st));
          LLMP_CUDA(cudaMemcpyAsync(fp.t[q].H[0] + kHistBins, fp.t[q].hroot, (size_t)kHistBins * 8,
                                    cudaMemcpyDeviceToDevice, st));
        } else {
          LLMP_CUDA(cudaMemsetAsync(fp.t[q].H[0], 0, (size_t)SLOT * 8, st));
        }
      }
      if (hist1 & 4)
        LLMP_LAUNCH(ctx, KC_UPDATE, ny * n, k_hist<HM_UPDROOT>, hg, HIST_THREADS, HIST_SMEM + updroot_tree_smem(D), fp,
                    0, 0, nodbg);
      else if (updk == 3)
        LLMP_LAUNCH_PDL(ctx, KC_UPDATE, ny * n, k_up3, hu3, U3_THREADS, U3_SMEM + updroot_tree_smem(D), fp);
      else
        LLMP_LAUNCH_PDL(ctx, KC_UPDATE, ny * n, k_upd2, hg, H2_THREADS, H2_SMEM + updroot_tree_smem(D), fp, 0, 0, nodbg);
    } else if (!fused) {
      LLMP_LAUNCH(ctx, KC_UPDATE, ny * n, k_update, dim3(std::max(1, upd_grid * ny / 2), ny), UPD_THREADS, 0, fp);
    }
  };
  // dual: the update of tree t + root histograms of trees t+1 of BOTH ensembles, one pass over the rows
  // (after both ensembles' levels: the branches have joined)
  auto dual_update = [&]() {   // (the root slots were reset at the end of each branch)
    const dim3 hg1((unsigned)std::min<int64_t>(ctx->sms * 2, std::max<int64_t>(1, (n + 2047) / 2048)), 1);
    LLMP_LAUNCH_PDL(ctx, KC_UPDATE, 2 * n, k_upd2d, hg1, H2_THREADS, H2_SMEM + updroot_tree_smem(D), FP, 0, 0, nodbg);
  };
  // both ensembles' trees t: two concurrent graph branches (default on one GPU: one ensemble's
  // latency-bound split / partition kernels overlap the other's streaming kernels; 592 vs 652 ms
  // per 500-tree fit), or one paired launch sequence (LLMP_PAIRED=1, and always with NCCL:
  // collectives must be issued in one order on every rank)
  static const bool branches_env = !(getenv("LLMP_PAIRED") && atoi(getenv("LLMP_PAIRED")) != 0);
  FitPair FPa, FPb;
  FPa.t[0] = A[0];
  FPb.t[0] = A[1];
  auto round = [&](const cudaGraphConditionalHandle* loop) {
    // sharded: the second branch issues its collectives on the second communicator (ctx->nccl2)
    const bool branches = branches_env && graphs && (!sharded || ctx->nccl2 != nullptr);
    if (branches) {
      const cudaStream_t sa = ctx->stream, sb = ctx->capture_stream(1);
      LLMP_CUDA(cudaEventRecord(ctx->fork_event, sa));
      LLMP_CUDA(cudaStreamWaitEvent(sb, ctx->fork_event, 0));
      trees(FPa, 1);
      ctx->stream = sb;
      ctx->comm_sel = 1;
      trees(FPb, 1);
      ctx->comm_sel = 0;
      LLMP_CUDA(cudaEventRecord(ctx->join_event, sb));
      ctx->stream = sa;
      LLMP_CUDA(cudaStreamWaitEvent(sa, ctx->join_event, 0));
    } else {
      trees(FP, 2);
    }
    if (dual) dual_update();
    // next tree's gradient maxima of both targets (contiguous; past slots are already equal on
    // every rank, future ones 0)
    allreduce_max_u32(ctx, A[0].maxg, (size_t)4 * (T + 1));
    if (loop) LLMP_LAUNCH_PDL(ctx, KC_MISC, 0, k_next_tree_cond, 1, 1, 0, d_tree, T, *loop, stamps);
    else LLMP_LAUNCH(ctx, KC_MISC, 0, k_next_tree, 1, 1, 0, d_tree);
  };
  LLMP_CUDA(cudaMemsetAsync(d_tree, 0, sizeof(int), s));
  // graphs: the whole tree loop is ONE graph launch — a device-side while loop (conditional graph
  // node) around the captured round, so no host thread sits between the T rounds (host jitter
  // cannot starve the GPU).  LLMP_GRAPH_REPLAY=1 replays the round graph T times from the host.
  static const bool replay_env = getenv("LLMP_GRAPH_REPLAY") && atoi(getenv("LLMP_GRAPH_REPLAY")) != 0;
  const bool replay = replay_env || sharded;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  if (graphs) {
    const cudaStream_t user = ctx->stream;
    const cudaStream_t sa = ctx->capture_stream(0);
    uint64_t l0[LLMP_N_KERNEL_CLASSES];
    double r0[LLMP_N_KERNEL_CLASSES];
    memcpy(l0, ctx->launches, sizeof(l0));
    memcpy(r0, ctx->rows, sizeof(r0));
    cudaGraphConditionalHandle loop = 0;
    if (!replay) {
      LLMP_CUDA(cudaGraphCreate(&g, 0));
      LLMP_CUDA(cudaGraphConditionalHandleCreate(&loop, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = loop;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t cn;
      LLMP_CUDA(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
      ctx->stream = sa;
      LLMP_CUDA(cudaStreamBeginCaptureToGraph(sa, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                              cudaStreamCaptureModeThreadLocal));
    } else {
      ctx->stream = sa;
      LLMP_CUDA(cudaStreamBeginCapture(sa, cudaStreamCaptureModeThreadLocal));
    }
    bool ok = true;
    try {
      round(replay ? nullptr : &loop);
    } catch (...) {
      ctx->comm_sel = 0;
      ctx->stream = sa;
      cudaGraph_t gc = nullptr;
      cudaStreamEndCapture(sa, &gc);
      if (replay && gc) cudaGraphDestroy(gc);
      if (g) cudaGraphDestroy(g);
      g = nullptr;
      ctx->stream = user;
      cudaGetLastError();
      if (!sharded) throw;
      ok = false;   // sharded: NCCL collectives that could not be captured -> plain launches below
    }
    if (ok) {
      cudaGraph_t gc = nullptr;
      LLMP_CUDA(cudaStreamEndCapture(sa, &gc));
      if (replay) g = gc;
      ctx->stream = user;
      const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
      if (e != cudaSuccess) {
        cudaGetLastError();
        cudaGraphDestroy(g);
        g = nullptr;
        ge = nullptr;
        if (!sharded) check_cuda(e, "cudaGraphInstantiate", __FILE__, __LINE__);
        ok = false;
      }
    }
    if (ok) {   // launch counters: the captured round runs T times
      for (int c = 0; c < LLMP_N_KERNEL_CLASSES; ++c) {
        ctx->launches[c] += (ctx->launches[c] - l0[c]) * (uint64_t)(T - 1);
        ctx->rows[c] += (ctx->rows[c] - r0[c]) * (double)(T - 1);
      }
      if (stamps) k_stamp<<<1, 1, 0, s>>>(stamps);
      if (replay) {
        for (int t = 0; t < T; ++t) LLMP_CUDA(cudaGraphLaunch(ge, s));
      } else {
        LLMP_CUDA(cudaGraphLaunch(ge, s));
      }
      LLMP_CUDA(cudaGraphExecDestroy(ge));
      LLMP_CUDA(cudaGraphDestroy(g));
    } else {    // the same rounds as plain launches
      memcpy(ctx->launches, l0, sizeof(l0));
      memcpy(ctx->rows, r0, sizeof(r0));
      nccl_health(ctx);
      ctx->pdl = false;
      for (int t = 0; t < T; ++t) {
        NvtxRange tr("tree");
        round(nullptr);
      }
    }
  } else {
    for (int t = 0; t < T; ++t) {
      NvtxRange tr("tree");
      round(nullptr);
    }
  }

  if (stamps) {   // diagnostics: per-round device durations
    std::vector<unsigned long long> h(T + 1);
    LLMP_CUDA(cudaMemcpyAsync(h.data(), stamps, (T + 1) * 8, cudaMemcpyDeviceToHost, s));
    LLMP_CUDA(cudaStreamSynchronize(s));
    std::vector<double> du(T);
    for (int t = 0; t < T; ++t) du[t] = (h[t + 1] - h[t]) * 1e-3;
    std::vector<double> so(du);
    std::sort(so.begin(), so.end());
    double tot = 0;
    for (double x : du) tot += x;
    fprintf(stderr, "[llmp] rounds: total %.1f ms  min %.1f  p10 %.1f  med %.1f  p90 %.1f  max %.1f us; slowest:", tot * 1e-3,
            so[0], so[T / 10], so[T / 2], so[(9 * T) / 10], so[T - 1]);
    for (int k = 0; k < 6 && k < T; ++k) {
      int am = 0;
      for (int t = 1; t < T; ++t)
        if (du[t] > du[am]) am = t;
      fprintf(stderr, " t%d=%.0f", am, du[am]);
      du[am] = -1;
    }
    fprintf(stderr, "\n");
  }
  phase("loop");
  nccl_health(ctx);   // an asynchronous NCCL failure surfaces here (LLMP_ENCCL), not as a hang
  // ---- model to host
  out.F = F;
  out.users_col = ds.users_col;
  out.T = T;
  out.D = D;
  out.nn = nn;
  out.n_train = n;
  const size_t tot = (size_t)2 * T * nn;
  out.feat.resize(tot);
  out.bin.resize(tot);
  out.thr.resize(tot);
  out.val.resize(tot);
  out.gain.resize(tot);
  if (tot) {
    LLMP_CUDA(cudaMemcpyAsync(out.gain.data(), d_gain.p, tot * 8, cudaMemcpyDeviceToHost, s));
    LLMP_CUDA(cudaMemcpyAsync(out.feat.data(), feat_all, tot * 4, cudaMemcpyDeviceToHost, s));
    LLMP_CUDA(cudaMemcpyAsync(out.bin.data(), bin_all, tot * 4, cudaMemcpyDeviceToHost, s));
    LLMP_CUDA(cudaMemcpyAsync(out.thr.data(), thr_all, tot * 4, cudaMemcpyDeviceToHost, s));
    LLMP_CUDA(cudaMemcpyAsync(out.val.data(), val_all, tot * 4, cudaMemcpyDeviceToHost, s));
  }
  LLMP_CUDA(cudaMemcpyAsync(out.base, d_base.p, 8, cudaMemcpyDeviceToHost, s));
  LLMP_CUDA(cudaStreamSynchronize(s));
  phase("to_host");
  upload_model_nodes(ctx, out);
  phase("upload");
}

// ---------------------------------------------------------------------------------------------
void debug_histogram(Ctx* ctx, const uint8_t* codes, int64_t n, const int32_t* idx, int64_t m, const int32_t* qg,
                     const int32_t* qh, int64_t* Hg, int64_t* Hh) {
  LLMP_REQUIRE(n >= 1 && m >= 0, "bad sizes");
  FitArgs a{};
  a.urow = 1;   // users_col = 0: lane 0 takes the row-parallel path (both paths covered by the tests)
  a.codes = codes;
  a.n = n;
  a.F = kMaxF;
  DevBuf& d_out = ctx->workspace("dbg_hist", (size_t)SLOT * 8);
  LLMP_CUDA(cudaMemsetAsync(d_out.p, 0, d_out.bytes, ctx->stream));
  DbgArgs dbg{idx, qg, qh, idx ? m : n, d_out.as<int64_t>()};
  ensure_smem_attr((const void*)k_hist<HM_DEBUG>, HIST_SMEM);
  ensure_smem_attr((const void*)k_hist2<HM_DEBUG>, H2_SMEM);
  ensure_smem_attr((const void*)k_hist3<HM_DEBUG, false>, H3_SMEM);
  FitPair fp;
  fp.t[0] = a;
  if (level_kernel() == 3)
    LLMP_LAUNCH(ctx, KC_HIST, dbg.m, (k_hist3<HM_DEBUG, false>), ctx->sms, H3_THREADS, H3_SMEM, fp, 1, 0, dbg);
  else if (level_kernel() == 1)
    LLMP_LAUNCH(ctx, KC_HIST, dbg.m, k_hist<HM_DEBUG>, 2 * ctx->sms, HIST_THREADS, HIST_SMEM, fp, 0, 0, dbg);
  else
    LLMP_LAUNCH(ctx, KC_HIST, dbg.m, k_hist2<HM_DEBUG>, 2 * ctx->sms, H2_THREADS, H2_SMEM, fp, 0, 0, dbg);
  LLMP_CUDA(cudaMemcpyAsync(Hg, d_out.p, kHistBins * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LLMP_CUDA(cudaMemcpyAsync(Hh, d_out.as<int64_t>() + kHistBins, kHistBins * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace llmp
