// hist3.cuh — level histogram of the built children, "change-row" form (included by fit.cu inside
// namespace llmp, after FitArgs / FitPair / DbgArgs).  DESIGN.md §6, k_hist3.
//
// Computes the same integer histograms as k_hist (O5): for every built child of the
// level, Hg[f][b] = sum of q_g and Hh[f][b] = sum of q_h over the child's rows whose feature-f code
// is b.  Integer sums, so any order and any grouping give the same bits.
//
// Layout of the work: one CTA per SM (512 threads, 16 warps); the CTA's slice of the virtual
// concatenation of the built children is split per (child, 65,536-row chunk) into 16 contiguous
// warp ranges.  Per warp, rows move through a 6-stage cp.async ring in shared memory (row indices
// loaded ten batches ahead, 32-byte code-row and packed-pair gathers issued four batches ahead of
// their use), so the gather latency is hidden without registers.  Per 32-row batch:
//   row side (lane = row r)   compares its code row with row r-1's (XOR of the 8 words, users byte
//                             masked) -> one ballot gives the rows where ANY feature's code changes;
//                             warp reductions of (q_g, q_h) over the rows before a flagged row give
//                             every run's sum as a difference;
//                             the users column (a new code on nearly every row of paper-ordered data)
//                             goes row-parallel into a dense per-bin histogram (bank = bin);
//   feature side (lane = f)   walks only the flagged rows (warp-uniform loop): at each, a lane whose
//                             code changed flushes its finished run with one pair of 32-bit shared
//                             reductions into the bin-major [256][32] histogram (bank = feature:
//                             conflict-free); unchanged lanes do nothing.
// Rows whose codes all equal the previous row's cost no feature-side work at all, so a batch costs
// ~65 warp-instructions plus ~17 per flagged row (k_hist: ~390 per batch).  Zero-skipping int64
// atomics flush the shared histogram into the node slot after each chunk.
#ifndef LLMP_H3_THREADS
#define LLMP_H3_THREADS 512
#endif
#ifndef LLMP_H3_AHEAD
#define LLMP_H3_AHEAD 4
#endif
constexpr int H3_THREADS = LLMP_H3_THREADS;
constexpr int H3_WARPS = H3_THREADS / 32;
constexpr int H3_AHEAD = LLMP_H3_AHEAD;                          // gathers issued this many batches ahead of their use
constexpr int H3_STAGES = H3_AHEAD + 2;               // ring: b+AHEAD issued while b is processed, b-1 kept
constexpr int H3_GP = 32 * 32;                        // stage offset of the 32 packed pairs
constexpr int H3_STAGE = H3_GP + 32 * 4;              // 32 code rows (32 B, halves swizzled) + pairs
constexpr int H3_HH = kBins * kMaxF * 4;              // byte offset of the q_h channel (32 KB)
constexpr int H3_U_OFF = 2 * H3_HH;                   // users column: [256] q_g, [256] q_h
constexpr int H3_RING_OFF = H3_U_OFF + 2 * kBins * 4;
constexpr int H3_SMEM = H3_RING_OFF + H3_WARPS * H3_STAGES * H3_STAGE;   // 64 + 2 + 108 KB

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red2_h3(uint32_t addr, int32_t g, uint32_t h) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(g) : "memory");
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(addr), "r"(h), "n"(H3_HH) : "memory");
}
// byte offset of row r's half h (0: codes 0..15, 1: codes 16..31) in a stage: the halves of rows with
// (r >> 2) & 1 are swapped, so the 8 lanes of one phase of a 16-byte load hit 8 distinct bank quads
__device__ __forceinline__ uint32_t h3_half(int r, int h) { return (uint32_t)(r * 32) + ((uint32_t)(h ^ ((r >> 2) & 1)) << 4); }

// ---------------------------------------------------------------------------------------------
// Split evaluation folded into the level histogram (unsharded fits): the CTA that
// completes the last contribution to parent j's built child evaluates both children of j — the 64
// (child, feature) warps of k_split3 over the CTA's 16 warps, then one warp per child for the node
// decision — so a level costs one launch instead of two and the split's dependent-load chain
// overlaps the other CTAs' histogram work.
__device__ __forceinline__ void fold_split(const FitPair& fp, int tg, int d, int j, int side) {
  const FitArgs& a = fp.t[tg];
  __shared__ FeatBest s_fb2[2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool split = a.lv[d - 1].split_f[j] >= 0;   // else split_feature marks both children absent
  for (int task = warp; task < 64; task += H3_WARPS) {
    const int c = task >> 5, f = task & 31;
    FeatBest r;
    const bool ok = split_feature(a, d, 2 * j + c, f, lane, r, side);
    if (ok && lane == 0) s_fb2[c][f] = r;
  }
  __syncthreads();
  if (split && warp < 2) {
    const FeatBest q = s_fb2[warp][lane];
    split_node(a, d, 2 * j + warp, lane, q.valid, q.b, q.loss, q.GLq, q.HLq, q.Gq, q.Hq);
  }
  __syncthreads();
}

template <int MODE, bool FOLD = false>
__global__ void __launch_bounds__(H3_THREADS, 1) k_hist3(const FitPair fp, const int ny, const int d, const DbgArgs dbg) {
  constexpr bool fold = FOLD;
  pdl_wait();
  const FitArgs& a0 = fp.t[0];   // F, users_col, codes: the same for both ensembles
  const int ucol = (a0.users_col >= 0 && a0.users_col < kMaxF) ? a0.users_col : -1;
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // pieces: the built children of ensemble 0, then those of ensemble 1 (ny = 2: one launch covers
  // both, and the CTAs split the rows of both evenly whatever their balance between the ensembles)
  __shared__ int64_t s_vstart[2 * MAX_PIECES + 1];
  __shared__ int64_t s_pstart[2 * MAX_PIECES];
  __shared__ int16_t s_slot[2 * MAX_PIECES];
  __shared__ int8_t s_tg[2 * MAX_PIECES];
  __shared__ int8_t s_side[2 * MAX_PIECES];   // built child of the piece's parent (fold-in)
  __shared__ int s_np, s_last;

  {   // zero both histogram channels and the users column
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (int i = tid; i < H3_RING_OFF / 16; i += H3_THREADS) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  // ---- piece list (virtual concatenation of the rows to histogram)
  if (MODE == HM_LEVEL) {
    // both ensembles' parents at once (entry e = tg * NP + j; thread tid takes entries 2 tid and
    // 2 tid + 1, E = ny * NP <= 2 * 512): every load is issued unconditionally, so the list costs one
    // round trip to global memory and one block scan
    const int NP = 1 << (d - 1);
    const int E = ny * NP;
    __shared__ int64_t s_wsum[H3_WARPS];
    int64_t len2[2], pst2[2];
    int side2[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int e = 2 * tid + q;
      len2[q] = 0;
      pst2[q] = 0;
      side2[q] = 0;
      if (e < E) {
        const int tg = e >= NP ? 1 : 0, j = e - tg * NP;
        const FitArgs& a = fp.t[tg];
        const LevelView& P = a.lv[d - 1];
        const LevelView& C = a.lv[d];
        const int pf = P.split_f[j];
        const int64_t nL = C.cnt[2 * j], nR = C.cnt[2 * j + 1];
        const int bh = a.built_by_h ? C.built[j] : 0;
        const int64_t ps = (d == 1) ? 0 : P.start[j];
        if (pf >= 0) {
          const int side = a.built_by_h ? bh : (nL <= nR) ? 0 : 1;   // smaller child (rows; hessian when sharded)
          side2[q] = side;
          len2[q] = side ? nR : nL;
          pst2[q] = side ? ps + nL : ps;   // k_part: left child first
          if (blockIdx.x == 0) {
            C.built[j] = side;
            C.start[2 * j] = ps;
            C.start[2 * j + 1] = ps + nL;
          }
        }
      }
    }
    const int64_t mine = len2[0] + len2[1];
    int64_t v = mine;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) s_wsum[warp] = v;
    __syncthreads();
    int64_t woff = 0, tot = 0;
    for (int w2 = 0; w2 < H3_WARPS; ++w2) {
      if (w2 < warp) woff += s_wsum[w2];
      tot += s_wsum[w2];
    }
    int64_t ex = woff + v - mine;   // rows of the entries before 2 tid
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int e = 2 * tid + q;
      if (e < E) {
        const int tg = e >= NP ? 1 : 0;
        s_vstart[e] = ex;
        s_pstart[e] = pst2[q];
        s_slot[e] = (int16_t)(e - tg * NP);
        s_tg[e] = (int8_t)tg;
        s_side[e] = (int8_t)side2[q];
      }
      ex += len2[q];
    }
    if (tid == 0) {
      s_vstart[E] = tot;
      s_np = E;
    }
  } else if (tid == 0) {
    s_np = 1;
    s_vstart[0] = 0;
    s_vstart[1] = dbg.m;
    s_pstart[0] = 0;
    s_slot[0] = 0;
    s_tg[0] = 0;
  }
  __syncthreads();
  const int np = s_np;
  const int64_t S = s_vstart[np];
  const int64_t v0 = S * blockIdx.x / gridDim.x, v1 = S * (blockIdx.x + 1) / gridDim.x;
  if (MODE == HM_LEVEL && fold) {
    // fold-in: pieces without rows (a parent that did not split, or an empty built child) are
    // evaluated by CTA p mod G up front (nothing to wait for: the built slot was zeroed by k_part)
    for (int pp = blockIdx.x; pp < np; pp += gridDim.x)
      if (s_vstart[pp + 1] == s_vstart[pp]) fold_split(fp, s_tg[pp], d, s_slot[pp], s_side[pp]);
  }
  if (v0 >= v1 && !(MODE == HM_LEVEL && fold)) return;   // (fold-in: an idle CTA still evaluates queued pieces)
  if (v0 < v1 && tid == 0 && MODE == HM_LEVEL && a0.units) atomicAdd(&a0.units[KC_HIST], (unsigned long long)(v1 - v0));

  const uint32_t sgb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sub = sgb + H3_U_OFF;
  const uint32_t ring = sgb + H3_RING_OFF + (uint32_t)(warp * H3_STAGES * H3_STAGE);
  const bool active = lane < a0.F && lane != ucol;   // feature side: lane = feature f
  const uint32_t foff0 = (uint32_t)lane, foff1 = (uint32_t)(lane ^ 16);   // feature byte in an unswapped / swapped row
  // row side: the users byte is masked out of the change test (its column goes row-parallel)
  uint32_t um[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) um[j] = (ucol >= 0 && (ucol >> 2) == j) ? ~(0xffu << (8 * (ucol & 3))) : 0xffffffffu;
  const uint32_t uoff = ucol >= 0 ? h3_half(lane, ucol >> 4) + (uint32_t)(ucol & 15) : 0u;   // own row's users byte

  int pc = 0;   // first piece ending after v0 (binary search: deep levels have up to 2 x 512 pieces)
  {
    int hi = np - 1;
    while (pc < hi) {
      const int mid = (pc + hi) >> 1;
      if (s_vstart[mid + 1] <= v0) pc = mid + 1;
      else hi = mid;
    }
  }
  // The CTA's work is a sequence of segments (piece, <= HIST_CHUNK-row chunk), each split evenly over
  // the warps and flushed between two barriers.  A warp's gather pipeline does not drain at a segment
  // boundary: once its rows of segment s are processed it issues the row-index loads and the first
  // H3_AHEAD gathers of its rows of segment s+1 into the (now free) ring, and only then waits at the
  // barrier that precedes segment s's flush — so the next segment's first gathers overlap the wait for
  // the slowest warp and the flush (deep levels: several short segments per CTA).
  struct Seg {
    int pc;              // piece
    int64_t c0, c1;      // virtual range of the chunk
    int64_t rbase;       // physical position of the warp's first row
    int nb, rem;         // the warp's batches; batch b holds this lane's row iff 32 b < rem
    const uint32_t* sr;  // the piece's row indices (level d's segments) and packed pairs
    const uint32_t* gpr;
  };
  auto seg_make = [&](int p_, int64_t c0_) {
    Seg g;
    g.pc = p_;
    const int64_t s1_ = min(v1, s_vstart[p_ + 1]);
    g.c0 = c0_;
    g.c1 = min(s1_, c0_ + HIST_CHUNK);
    const int64_t clen = g.c1 - g.c0;
    const int64_t w0 = g.c0 + clen * warp / H3_WARPS, w1 = g.c0 + clen * (warp + 1) / H3_WARPS;
    g.nb = (int)((w1 - w0 + 31) >> 5);
    g.rem = (int)(w1 - w0) - lane;
    g.rbase = w0 + (s_pstart[p_] - s_vstart[p_]);   // physical position = virtual + (pstart - vstart)
    const FitArgs& ag = fp.t[s_tg[p_]];
    g.sr = (MODE == HM_LEVEL) ? ag.sr[d & 1] : nullptr;
    g.gpr = ag.gp_root;
    return g;
  };
  // the segment after g (pc = -1: none)
  auto seg_next = [&](const Seg& g) {
    const int64_t s1_ = min(v1, s_vstart[g.pc + 1]);
    if (g.c1 < s1_) return seg_make(g.pc, g.c1);
    for (int p_ = g.pc + 1; p_ < np && s_vstart[p_] < v1; ++p_) {
      const int64_t a0_ = max(v0, s_vstart[p_]), a1_ = min(v1, s_vstart[p_ + 1]);
      if (a0_ < a1_) return seg_make(p_, a0_);
    }
    Seg none;
    none.pc = -1;
    none.c0 = none.c1 = 0;
    none.rbase = 0;
    none.nb = 0;
    none.rem = 0;
    none.sr = nullptr;
    none.gpr = nullptr;
    return none;
  };
  // row-index loads are never predicated (a predicated load feeds a select that would wait for it):
  // rows past the range read the warp range's first row index instead (unused)
  auto ridx_of = [&](const Seg& g, int b) -> uint32_t {
    const int64_t pi = g.rbase + ((32 * b < g.rem) ? 32 * b + lane : 0);
    if (MODE == HM_LEVEL) return g.sr[pi];
    return dbg.idx ? (uint32_t)dbg.idx[pi] : (uint32_t)pi;
  };
  auto issue = [&](const Seg& g, int b, int stage, uint32_t ri) {   // gathers of batch b into `stage` (one commit group)
    if (32 * b < g.rem) {
      const uint32_t st = ring + (uint32_t)(stage * H3_STAGE);
      const uint8_t* src = a0.codes + (size_t)ri * kMaxF;
      cp_async16(st + h3_half(lane, 0), src);
      cp_async16(st + h3_half(lane, 1), src + 16);
      if (MODE == HM_LEVEL) cp_async4(st + H3_GP + lane * 4, g.gpr + ri);
      else sts32(st + H3_GP + lane * 4, pack_gp(dbg.qg[ri], dbg.qh[ri]));
    }
    cp_async_commit();
  };
  // gathers run H3_AHEAD batches ahead of their use, row indices H3_STAGES batches ahead of their
  // gathers (a register ring; the loop is unrolled by H3_STAGES, so every stage and ring index is a
  // compile-time constant and no copy waits on a load)
  uint32_t R[H3_STAGES];
  auto prologue = [&](const Seg& g) {
    if (g.nb > 0) {
#pragma unroll
      for (int k = 0; k < H3_AHEAD; ++k) issue(g, k, k, ridx_of(g, k));
#pragma unroll
      for (int k = 0; k < H3_STAGES; ++k) R[k] = ridx_of(g, H3_AHEAD + k);
    }
  };
  Seg cs;
  cs.pc = -1;
  if (pc < np && s_vstart[pc] < v1) {
    const int64_t a0_ = max(v0, s_vstart[pc]);
    if (a0_ < min(v1, s_vstart[pc + 1])) cs = seg_make(pc, a0_);
    else {
      Seg t0;
      t0.pc = pc;
      t0.c1 = min(v1, s_vstart[pc + 1]);
      cs = seg_next(t0);
    }
  }
  if (v0 < v1 && cs.pc >= 0) prologue(cs);
  while (cs.pc >= 0) {
    const int pc = cs.pc;
    const FitArgs& a = fp.t[s_tg[pc]];
    int64_t* Hg = ((MODE == HM_DEBUG) ? dbg.out : a.H[d & 1]) + (size_t)s_slot[pc] * SLOT;
    int64_t* Hh = Hg + kHistBins;
    const int nb = cs.nb;
    const int rem = cs.rem;
    uint32_t cur = 0;          // feature side: byte offset of the pending run's (bin, f) cell
    int32_t acc_g = 0;         // its sums from earlier batches
    uint32_t acc_h = 0;
    bool fresh = true;
    if (nb > 0) {
      for (int bb = 0; bb < nb; bb += H3_STAGES) {
#pragma unroll
        for (int k = 0; k < H3_STAGES; ++k) {
          const int b = bb + k;
          if (b >= nb) break;
          __syncwarp();            // the stage being refilled (batch b-2's) is fully consumed
          issue(cs, b + H3_AHEAD, (k + H3_AHEAD) % H3_STAGES, R[k]);
          R[k] = ridx_of(cs, b + H3_AHEAD + H3_STAGES);
          cp_async_wait<H3_AHEAD>();   // batch b has landed (b+1 .. b+AHEAD may be in flight)
          __syncwarp();
          const uint32_t st = ring + (uint32_t)(k * H3_STAGE);
          const bool valid = 32 * b < rem;
          // ---- row side: does row `lane` differ from its predecessor in any (non-users) feature?
          const uint4 c0v = lds128(st + h3_half(lane, 0)), c1v = lds128(st + h3_half(lane, 1));
          const uint32_t pst = lane ? st : ring + (uint32_t)(((k + H3_STAGES - 1) % H3_STAGES) * H3_STAGE);
          const int pr = lane ? lane - 1 : 31;
          const uint4 p0 = lds128(pst + h3_half(pr, 0)), p1 = lds128(pst + h3_half(pr, 1));
          const uint32_t dx = ((c0v.x ^ p0.x) & um[0]) | ((c0v.y ^ p0.y) & um[1]) | ((c0v.z ^ p0.z) & um[2]) |
                              ((c0v.w ^ p0.w) & um[3]) | ((c1v.x ^ p1.x) & um[4]) | ((c1v.y ^ p1.y) & um[5]) |
                              ((c1v.z ^ p1.z) & um[6]) | ((c1v.w ^ p1.w) & um[7]);
          unsigned B = __ballot_sync(0xffffffffu, valid && (dx != 0u || (fresh && lane == 0)));
          const uint32_t gp = valid ? lds32(st + H3_GP + lane * 4) : 0u;
          const int32_t qg = gp_g(gp);
          const uint32_t qh = (uint32_t)gp_h(gp);
          if (ucol >= 0 && valid) {   // users column, row-parallel into the dense per-bin histogram
            const uint32_t ua = sub + lds8(st + uoff) * 4u;
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(ua), "r"(qg) : "memory");
            asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(ua), "r"(qh), "n"(kBins * 4) : "memory");
          }
          // ---- feature side: walk the flagged rows only; the sum of the batch's rows before a
          // flagged row r (lanes < r) is one warp reduction per channel
          if (fresh) {   // the first row starts every lane's run
            cur = (lds8(st + foff0) * 32u + (uint32_t)lane) * 4u;
            fresh = false;
            B &= ~1u;
          }
          int32_t bg = 0;          // sum of the batch's rows before the pending run's first row
          uint32_t bh = 0;
          // two flagged rows per step: both rows' code loads and prefix reductions are issued
          // before either update (the updates are a short dependent chain per lane)
          while (B) {
            const int r1 = __ffs(B) - 1;
            B &= B - 1u;
            const bool two = B != 0u;
            const int r2 = two ? __ffs(B) - 1 : r1;
            B &= B - 1u;
            const uint32_t c1 = lds8(st + (uint32_t)(r1 * 32) + (((r1 >> 2) & 1) ? foff1 : foff0));
            const uint32_t c2 = lds8(st + (uint32_t)(r2 * 32) + (((r2 >> 2) & 1) ? foff1 : foff0));
            const int32_t vg1 = (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)(lane < r1 ? qg : 0));
            const uint32_t vh1 = __reduce_add_sync(0xffffffffu, lane < r1 ? qh : 0u);
            const int32_t vg2 = (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)(lane < r2 ? qg : 0));
            const uint32_t vh2 = __reduce_add_sync(0xffffffffu, lane < r2 ? qh : 0u);
            const uint32_t na1 = (c1 * 32u + (uint32_t)lane) * 4u;
            if (active && na1 != cur) {
              red2_h3(sgb + cur, acc_g + (vg1 - bg), acc_h + (vh1 - bh));
              acc_g = 0;
              acc_h = 0;
              bg = vg1;
              bh = vh1;
              cur = na1;
            }
            const uint32_t na2 = (c2 * 32u + (uint32_t)lane) * 4u;
            if (two && active && na2 != cur) {
              red2_h3(sgb + cur, acc_g + (vg2 - bg), acc_h + (vh2 - bh));
              acc_g = 0;
              acc_h = 0;
              bg = vg2;
              bh = vh2;
              cur = na2;
            }
          }
          acc_g += (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)qg) - bg;
          acc_h += __reduce_add_sync(0xffffffffu, qh) - bh;
        }
      }
    }
    if (active && !fresh && (acc_g | (int32_t)acc_h)) red2_h3(sgb + cur, acc_g, acc_h);
    // the next segment's first gathers go out before the barrier (the ring is free once every lane
    // has read its last batch)
    const Seg ns = seg_next(cs);
    __syncwarp();
    if (ns.pc >= 0) prologue(ns);
    else cp_async_wait<0>();
    __syncthreads();
    int32_t* sg = reinterpret_cast<int32_t*>(smem);
    uint32_t* sh = reinterpret_cast<uint32_t*>(smem + H3_HH);
    int32_t* sug = reinterpret_cast<int32_t*>(smem + H3_U_OFF);
    uint32_t* suh = reinterpret_cast<uint32_t*>(smem + H3_U_OFF + kBins * 4);
    if (ucol >= 0) {   // the users column's cells (never written by its lane) from the dense histogram
      for (int b = tid; b < kBins; b += H3_THREADS) {
        sg[b * 32 + ucol] = sug[b];
        sh[b * 32 + ucol] = suh[b];
        sug[b] = 0;
        suh[b] = 0;
      }
      __syncthreads();
    }
    // flush: zero-skipping int64 atomics into the node histogram ([f][b] layout)
    for (int i = tid; i < kHistBins; i += H3_THREADS) {
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
    if (MODE == HM_LEVEL && fold && ns.pc != pc) {
      // this CTA's contribution to the piece is flushed: the CTA completing the count of CTAs that
      // cover the piece evaluates the split of the piece's parent
      const FitArgs& ap = fp.t[s_tg[pc]];
      int* ticket = &ap.lv[d].done[2 * s_slot[pc]];
      if (tid == 0) {
        const int64_t G = gridDim.x;
        auto cta_of = [&](int64_t v) {   // largest b with floor(S b / G) <= v: the CTA holding v
          int lo = 0, hi = (int)G - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (S * mid / G <= v) lo = mid;
            else hi = mid - 1;
          }
          return lo;
        };
        const int ncta = cta_of(s_vstart[pc + 1] - 1) - cta_of(s_vstart[pc]) + 1;
        __threadfence();
        const int prev = atomicAdd(ticket, 1);
        s_last = prev + 1 == ncta;
        if (s_last) {
          *ticket = 0;   // self-resetting for the next tree
          __threadfence();
        }
      }
      __syncthreads();
      // the piece is complete: queue its split evaluation (any CTA whose histogram work is done
      // takes it — a CTA covering many small pieces would otherwise evaluate them all in series)
      if (s_last && tid == 0) {
        int* fq = fp.t[0].fq;
        const int slot = atomicAdd(&fq[1], 1);
        atomicExch(&fq[2 + slot], pc + 1);
      }
    }
    cs = ns;
  }
  if (MODE == HM_LEVEL && fold) {
    // this CTA's histogram work is done: evaluate queued pieces until every non-empty piece is taken
    int* fq = fp.t[0].fq;
    int n_ne = 0;
    for (int pp = 0; pp < np; ++pp) n_ne += s_vstart[pp + 1] > s_vstart[pp];
    while (true) {
      if (tid == 0) {
        const int h = atomicAdd(&fq[0], 1);
        int pc = -1;
        if (h < n_ne) {
          volatile int* slot = &fq[2 + h];
          while ((pc = *slot) == 0) __nanosleep(200);   // produced by a CTA still flushing
          __threadfence();
          --pc;
        }
        s_last = pc;
      }
      __syncthreads();
      const int pc = s_last;
      if (pc < 0) break;
      fold_split(fp, s_tg[pc], d, s_slot[pc], s_side[pc]);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// k_upd3: fused update of tree t + root histogram of tree t+1 (HM_UPDROOT semantics, see k_hist2:
// O9 p += v for every row, then O4 for tree t+1 quantised with tree t's exponents — the speculation
// that k_root_fix / k_hist2<ROOT> undo when an exponent changed — and O5 over all rows), rows in
// identity order.  Every input moves by bulk copy (TMA engine): per warp (32 per CTA, one CTA per
// SM) a 3-stage ring, one stage =
// one 32-row batch = its code rows (1 KB, contiguous) and its y, w, p (128 B each), issued by lane 0
// with cp.async.bulk on the stage's mbarrier two batches ahead of use.  Per batch, lane = row routes
// its row through tree t (fixed-depth table), updates p, computes and quantises tree t+1's pair;
// then the root histogram takes the change-row form of k_hist3 (a ballot of the rows whose codes
// differ from the previous row, lanes = features flushing runs only there; users row-parallel).
constexpr int U3_THREADS = 1024;
constexpr int U3_WARPS = U3_THREADS / 32;
constexpr int U3_STAGES = 3;
constexpr int U3_AHEAD = 2;                              // batches in flight ahead of the one in use
                                                         // (lane 0's previous row is kept in registers)
constexpr int U3_Y = 32 * 32, U3_W = U3_Y + 128, U3_P = U3_W + 128;
constexpr int U3_STAGE = U3_P + 128;                     // 1,408 B
constexpr int U3_RING_OFF = H3_RING_OFF;                 // histogram channels + users column first
constexpr int U3_SMEM = U3_RING_OFF + U3_WARPS * U3_STAGES * U3_STAGE;   // 66 + 132 KB (+ the tree)

template <int DC>
__global__ void __launch_bounds__(U3_THREADS, 1) k_upd3(const FitPair fp) {
  pdl_wait();
  const FitArgs& a = fp.t[blockIdx.y];
  const int t = *a.d_tree;
  const bool has_next = t + 1 < a.T;
  const int ucol = (a.users_col >= 0 && a.users_col < kMaxF) ? a.users_col : -1;
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ __align__(8) uint64_t s_bar[U3_WARPS][U3_STAGES];
  {   // zero both histogram channels and the users column
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (int i = tid; i < H3_RING_OFF / 16; i += U3_THREADS) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (lane == 0) {
    for (int s = 0; s < U3_STAGES; ++s) mbar_init(smem_u32(&s_bar[warp][s]), 1);
    mbar_fence_init();
  }
  // tree t as a fixed-depth routing table (as in k_hist2): internal slots above depth D hold their
  // split, leaves and everything below them "always left" (0, 255); 2^D leaf values
  uint8_t* s_rf = smem + U3_SMEM;
  uint8_t* s_rb = s_rf + (a.nn + 1) / 2;
  float* s_lv = reinterpret_cast<float*>(smem + U3_SMEM + (a.nn + 1));
  const int n_int = (a.nn - 1) / 2;
  {
    const size_t to = (size_t)t * a.nn;
    for (int i = tid; i < a.nn; i += U3_THREADS) {
      const int f = a.tfeat[to + i];
      if (i < n_int) {
        s_rf[i] = (uint8_t)(f >= 0 ? f : 0);
        s_rb[i] = (uint8_t)(f >= 0 ? a.tbin[to + i] : 255);
      }
      if (f == -1) {
        const int dl = 31 - __clz(i + 1);
        s_lv[((i + 1) << (a.D - dl)) - 1 - n_int] = a.tval[to + i];
      }
    }
  }
  __syncthreads();
  const int64_t n = a.n;
  const int64_t nb_all = (n + 31) / 32;
  const int64_t v0 = (nb_all * blockIdx.x / gridDim.x) * 32, v1 = min(n, (nb_all * (blockIdx.x + 1) / gridDim.x) * 32);
  if (v0 >= v1) return;
  if (tid == 0 && a.units) atomicAdd(&a.units[KC_UPDATE], (unsigned long long)(v1 - v0));
  const double scale_g = exp2i(a.K - exp_of(__uint_as_float(a.maxg[t])));
  const double scale_h = exp2i(a.K - exp_of(__uint_as_float(a.maxh[t])));
  float mg = 0.f, mh = 0.f;
  const uint32_t sgb = smem_u32(smem);
  const uint32_t sub = sgb + H3_U_OFF;
  const uint32_t ring = sgb + U3_RING_OFF + (uint32_t)(warp * U3_STAGES * U3_STAGE);
  const bool active = lane < a.F && lane != ucol;
  uint32_t um[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) um[j] = (ucol >= 0 && (ucol >> 2) == j) ? ~(0xffu << (8 * (ucol & 3))) : 0xffffffffu;
  uint32_t phase = 0;   // bit s: parity of stage s's barrier
  for (int64_t c0 = v0; c0 < v1; c0 += HIST_CHUNK) {
    const int64_t c1 = min(v1, c0 + HIST_CHUNK);
    const int64_t nbc = (c1 - c0 + 31) / 32;
    const int64_t w0 = c0 + (nbc * warp / U3_WARPS) * 32, w1 = min(c1, c0 + (nbc * (warp + 1) / U3_WARPS) * 32);
    const int nb = (int)((w1 - w0 + 31) >> 5);
    auto rows_of = [&](int b) { return (int)min((int64_t)32, w1 - (w0 + 32 * (int64_t)b)); };
    // lane 0: batch b into its stage (full batches by bulk copy; a partial last batch of the data
    // — its byte counts need not be multiples of 16 — by the whole warp with plain loads)
    auto issue = [&](int b) {
      if (b >= nb) return;
      const int cnt = rows_of(b);
      const int s = b % U3_STAGES;
      const uint32_t st = ring + (uint32_t)(s * U3_STAGE);
      const int64_t r0 = w0 + 32 * (int64_t)b;
      // bulk copies need 16-byte aligned sources (p of the second ensemble starts at p + n)
      const bool al = ((((uintptr_t)(a.y + r0)) | ((uintptr_t)(a.w + r0)) | ((uintptr_t)(a.p + r0))) & 15) == 0;
      if (cnt == 32 && al) {
        if (lane == 0) {
          const uint32_t bar = smem_u32(&s_bar[warp][s]);
          mbar_arrive_expect_tx(bar, 32 * 32 + 3 * 128);
          bulk_g2s(st, a.codes + r0 * kMaxF, 32 * 32, bar);
          bulk_g2s(st + U3_Y, a.y + r0, 128, bar);
          bulk_g2s(st + U3_W, a.w + r0, 128, bar);
          bulk_g2s(st + U3_P, a.p + r0, 128, bar);
        }
      } else {
        if (lane < cnt) {
          const uint4* cr = reinterpret_cast<const uint4*>(a.codes + (r0 + lane) * kMaxF);
          const uint4 q0 = cr[0], q1 = cr[1];
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(st + lane * 32), "r"(q0.x), "r"(q0.y), "r"(q0.z),
                       "r"(q0.w) : "memory");
          asm volatile("st.shared.v4.u32 [%0+16], {%1, %2, %3, %4};" ::"r"(st + lane * 32), "r"(q1.x), "r"(q1.y),
                       "r"(q1.z), "r"(q1.w) : "memory");
          sts32(st + U3_Y + lane * 4, __float_as_uint(a.y[r0 + lane]));
          sts32(st + U3_W + lane * 4, __float_as_uint(a.w[r0 + lane]));
          sts32(st + U3_P + lane * 4, __float_as_uint(a.p[r0 + lane]));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(smem_u32(&s_bar[warp][s]), 0);   // completes the phase
      }
    };
#pragma unroll
    for (int k = 0; k < U3_AHEAD; ++k) issue(k);
    uint32_t cur = 0;
    int32_t acc_g = 0;
    uint32_t acc_h = 0;
    bool fresh = true;
    uint32_t prv[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};   // row 31 of the previous batch
    for (int b = 0; b < nb; ++b) {
      __syncwarp();   // the stage being refilled (batch b-1's) is consumed by every lane
      issue(b + U3_AHEAD);
      const int s = b % U3_STAGES;
      const uint32_t st = ring + (uint32_t)(s * U3_STAGE);
      mbar_wait(smem_u32(&s_bar[warp][s]), (phase >> s) & 1u);
      phase ^= 1u << s;
      const int cnt = rows_of(b);
      const bool valid = lane < cnt;
      const int64_t ridx = w0 + 32 * (int64_t)b + lane;
      // ---- O9 for tree t: route the lane's row (fixed depth), p += v (one fp32 rounding)
      const uint32_t myrow = st + (uint32_t)(lane * 32);
      int k = 0;
      const int D = DC ? DC : a.D;
#pragma unroll
      for (int s2 = 0; s2 < (DC ? DC : kMaxDepth); ++s2)
        if (DC || s2 < D) k = 2 * k + 1 + (lds8(myrow + s_rf[k]) > s_rb[k] ? 1 : 0);
      const float pv = __uint_as_float(lds32(st + U3_P + lane * 4));
      const float yv = __uint_as_float(lds32(st + U3_Y + lane * 4));
      const float wv = __uint_as_float(lds32(st + U3_W + lane * 4));
      const float pn = __fadd_rn(pv, s_lv[k - n_int]);
      uint32_t gp = 0u;
      if (valid) {
        a.p[ridx] = pn;
        if (has_next) {   // O4 for tree t+1 with tree t's exponents (speculation)
          float g, h;
          grad_pair(a, t + 1, a.row_offset + ridx, yv, wv, pn, g, h);
          mg = fmaxf(mg, fabsf(g));
          mh = fmaxf(mh, h);
          gp = pack_gp(quantize(g, scale_g), quantize(h, scale_h));
          a.gp_root[ridx] = gp;
        }
      }
      if (!has_next) continue;   // last tree: update only
      // ---- O5 root histogram of tree t+1: change-row form
      const uint4 c0v = lds128(myrow), c1v = lds128(myrow + 16);
      uint4 p0 = lds128(st + (uint32_t)((lane ? lane - 1 : 0) * 32)), p1 = lds128(st + (uint32_t)((lane ? lane - 1 : 0) * 32 + 16));
      if (lane == 0) {   // the previous batch's last row (its stage may already be refilled)
        p0 = make_uint4(prv[0], prv[1], prv[2], prv[3]);
        p1 = make_uint4(prv[4], prv[5], prv[6], prv[7]);
      }
      {
        const uint32_t cw[8] = {c0v.x, c0v.y, c0v.z, c0v.w, c1v.x, c1v.y, c1v.z, c1v.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) prv[j] = __shfl_sync(0xffffffffu, cw[j], 31);
      }
      const uint32_t dx = ((c0v.x ^ p0.x) & um[0]) | ((c0v.y ^ p0.y) & um[1]) | ((c0v.z ^ p0.z) & um[2]) |
                          ((c0v.w ^ p0.w) & um[3]) | ((c1v.x ^ p1.x) & um[4]) | ((c1v.y ^ p1.y) & um[5]) |
                          ((c1v.z ^ p1.z) & um[6]) | ((c1v.w ^ p1.w) & um[7]);
      unsigned B = __ballot_sync(0xffffffffu, valid && (dx != 0u || (fresh && lane == 0)));
      const int32_t qg = valid ? gp_g(gp) : 0;
      const uint32_t qh = valid ? (uint32_t)gp_h(gp) : 0u;
      if (ucol >= 0 && valid) {
        const uint32_t ua = sub + lds8(myrow + ucol) * 4u;
        asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(ua), "r"(qg) : "memory");
        asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(ua), "r"(qh), "n"(kBins * 4) : "memory");
      }
      if (fresh) {
        cur = (lds8(st + lane) * 32u + (uint32_t)lane) * 4u;
        fresh = false;
        B &= ~1u;
      }
      int32_t bg = 0;
      uint32_t bh = 0;
      while (B) {
        const int r1 = __ffs(B) - 1;
        B &= B - 1u;
        const bool two = B != 0u;
        const int r2 = two ? __ffs(B) - 1 : r1;
        B &= B - 1u;
        const uint32_t cc1 = lds8(st + (uint32_t)(r1 * 32 + lane));
        const uint32_t cc2 = lds8(st + (uint32_t)(r2 * 32 + lane));
        const int32_t vg1 = (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)(lane < r1 ? qg : 0));
        const uint32_t vh1 = __reduce_add_sync(0xffffffffu, lane < r1 ? qh : 0u);
        const int32_t vg2 = (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)(lane < r2 ? qg : 0));
        const uint32_t vh2 = __reduce_add_sync(0xffffffffu, lane < r2 ? qh : 0u);
        const uint32_t na1 = (cc1 * 32u + (uint32_t)lane) * 4u;
        if (active && na1 != cur) {
          red2_h3(sgb + cur, acc_g + (vg1 - bg), acc_h + (vh1 - bh));
          acc_g = 0;
          acc_h = 0;
          bg = vg1;
          bh = vh1;
          cur = na1;
        }
        const uint32_t na2 = (cc2 * 32u + (uint32_t)lane) * 4u;
        if (two && active && na2 != cur) {
          red2_h3(sgb + cur, acc_g + (vg2 - bg), acc_h + (vh2 - bh));
          acc_g = 0;
          acc_h = 0;
          bg = vg2;
          bh = vh2;
          cur = na2;
        }
      }
      acc_g += (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)qg) - bg;
      acc_h += __reduce_add_sync(0xffffffffu, qh) - bh;
    }
    if (!has_next) continue;
    if (active && !fresh && (acc_g | (int32_t)acc_h)) red2_h3(sgb + cur, acc_g, acc_h);
    __syncthreads();
    int32_t* sg = reinterpret_cast<int32_t*>(smem);
    uint32_t* sh = reinterpret_cast<uint32_t*>(smem + H3_HH);
    int32_t* sug = reinterpret_cast<int32_t*>(smem + H3_U_OFF);
    uint32_t* suh = reinterpret_cast<uint32_t*>(smem + H3_U_OFF + kBins * 4);
    if (ucol >= 0) {
      for (int bb = tid; bb < kBins; bb += U3_THREADS) {
        sg[bb * 32 + ucol] = sug[bb];
        sh[bb * 32 + ucol] = suh[bb];
        sug[bb] = 0;
        suh[bb] = 0;
      }
      __syncthreads();
    }
    int64_t* Hg = a.H[0];
    int64_t* Hh = Hg + kHistBins;
    for (int i = tid; i < kHistBins; i += U3_THREADS) {
      const int32_t g = sg[i];
      const uint32_t h = sh[i];
      if (g != 0 || h != 0) {
        const int bb = i >> 5, f = i & 31;
        atomicAdd(reinterpret_cast<unsigned long long*>(&Hg[f * kBins + bb]), (unsigned long long)(long long)g);
        atomicAdd(reinterpret_cast<unsigned long long*>(&Hh[f * kBins + bb]), (unsigned long long)h);
        sg[i] = 0;
        sh[i] = 0;
      }
    }
    __syncthreads();
  }
  if (has_next) {
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
