// hist3.cuh — level histogram of the built children, "change-row" form (included by fit.cu inside
// namespace llmp, after FitArgs / FitPair / DbgArgs).  DESIGN.md §6, k_hist3.
//
// Computes the same integer histograms as k_hist (O5): for every built child of the
// level, Hg[f][b] = sum of q_g and Hh[f][b] = sum of q_h over the child's rows whose feature-f code
// is b.  Integer sums, so any order and any grouping give the same bits.
//
// Layout of the work: one CTA per SM (512 threads, 16 warps); the CTA's slice of the virtual
// concatenation of the built children is split per (child, 65,536-row chunk) into 16 contiguous
// warp ranges.  Per warp, rows move through a 4-stage cp.async ring in shared memory (row indices
// loaded two batches ahead of their 32-byte code-row gathers, gathers issued two batches ahead of
// their use), so the gather latency is hidden without registers.  Per 32-row batch:
//   row side (lane = row r)   compares its code row with row r-1's (XOR of the 8 words, users byte
//                             masked) -> one ballot gives the rows where ANY feature's code changes;
//                             a warp prefix scan of (q_g, q_h) gives every run's sum as a difference;
//                             the users column (a new code on nearly every row of paper-ordered data)
//                             goes row-parallel into a dense per-bin histogram (bank = bin);
//   feature side (lane = f)   walks only the flagged rows (warp-uniform loop): at each, a lane whose
//                             code changed flushes its finished run with one pair of 32-bit shared
//                             reductions into the bin-major [256][32] histogram (bank = feature:
//                             conflict-free); unchanged lanes do nothing.
// Rows whose codes all equal the previous row's cost no feature-side work at all, so a batch costs
// ~65 warp-instructions plus ~17 per flagged row (k_hist: ~390 per batch).  Zero-skipping int64
// atomics flush the shared histogram into the node slot after each chunk.
constexpr int H3_THREADS = 512;
constexpr int H3_WARPS = H3_THREADS / 32;
constexpr int H3_STAGES = 4;                          // ring: b+2 issued while b is processed, b-1 kept
constexpr int H3_GP = 32 * 32;                        // stage offset of the 32 packed pairs
constexpr int H3_STAGE = H3_GP + 32 * 4;              // 32 code rows (32 B, halves swizzled) + pairs
constexpr int H3_HH = kBins * kMaxF * 4;              // byte offset of the q_h channel (32 KB)
constexpr int H3_U_OFF = 2 * H3_HH;                   // users column: [256] q_g, [256] q_h
constexpr int H3_RING_OFF = H3_U_OFF + 2 * kBins * 4;
constexpr int H3_SMEM = H3_RING_OFF + H3_WARPS * H3_STAGES * H3_STAGE;   // 64 + 2 + 72 KB

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

template <int MODE>
__global__ void __launch_bounds__(H3_THREADS, 1) k_hist3(const FitPair fp, const int d, const DbgArgs dbg) {
  pdl_wait();
  const FitArgs& a = fp.t[blockIdx.y];
  const int ucol = (a.users_col >= 0 && a.users_col < kMaxF) ? a.users_col : -1;
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  __shared__ int64_t s_vstart[MAX_PIECES + 1];
  __shared__ int64_t s_pstart[MAX_PIECES];
  __shared__ int32_t s_slot[MAX_PIECES];
  __shared__ int s_np;

  {   // zero both histogram channels and the users column
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (int i = tid; i < H3_RING_OFF / 16; i += H3_THREADS) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  // ---- piece list (virtual concatenation of the rows to histogram), as in k_hist
  if (MODE == HM_LEVEL) {
    const int NP = 1 << (d - 1);
    const LevelView& P = a.lv[d - 1];
    const LevelView& C = a.lv[d];
    int64_t len = 0, pst = 0;
    if (tid < NP && P.split_f[tid] >= 0) {
      const int64_t nL = C.cnt[2 * tid], nR = C.cnt[2 * tid + 1];
      const int side = a.built_by_h ? C.built[tid] : (nL <= nR) ? 0 : 1;   // smaller child (rows; hessian when sharded)
      len = C.cnt[2 * tid + side];
      const int64_t ps = (d == 1) ? 0 : P.start[tid], cl = C.cnt[2 * tid];   // k_part: left child first
      pst = side ? ps + cl : ps;
      if (blockIdx.x == 0) {
        C.built[tid] = side;
        C.start[2 * tid] = ps;
        C.start[2 * tid + 1] = ps + cl;
      }
    }
    __shared__ int64_t s_wsum[H3_WARPS];
    int64_t v = len;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
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
    s_vstart[1] = dbg.m;
    s_pstart[0] = 0;
    s_slot[0] = 0;
  }
  __syncthreads();
  const int np = s_np;
  const int64_t S = s_vstart[np];
  const int64_t v0 = S * blockIdx.x / gridDim.x, v1 = S * (blockIdx.x + 1) / gridDim.x;
  if (v0 >= v1) return;
  if (tid == 0 && MODE == HM_LEVEL && a.units) atomicAdd(&a.units[KC_HIST], (unsigned long long)(v1 - v0));

  int64_t* Hbase = (MODE == HM_DEBUG) ? dbg.out : a.H[d & 1];
  const uint32_t* sr_in = (MODE == HM_LEVEL) ? a.sr[d & 1] : nullptr;
  const uint32_t sgb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sub = sgb + H3_U_OFF;
  const uint32_t ring = sgb + H3_RING_OFF + (uint32_t)(warp * H3_STAGES * H3_STAGE);
  const bool active = lane < a.F && lane != ucol;   // feature side: lane = feature f
  const uint32_t foff0 = (uint32_t)lane, foff1 = (uint32_t)(lane ^ 16);   // feature byte in an unswapped / swapped row
  // row side: the users byte is masked out of the change test (its column goes row-parallel)
  uint32_t um[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) um[j] = (ucol >= 0 && (ucol >> 2) == j) ? ~(0xffu << (8 * (ucol & 3))) : 0xffffffffu;
  const uint32_t uoff = ucol >= 0 ? h3_half(lane, ucol >> 4) + (uint32_t)(ucol & 15) : 0u;   // own row's users byte

  int pc = 0;
  while (pc + 1 < np && s_vstart[pc + 1] <= v0) ++pc;
  for (; pc < np && s_vstart[pc] < v1; ++pc) {
    const int64_t s0 = max(v0, s_vstart[pc]), s1 = min(v1, s_vstart[pc + 1]);
    if (s0 >= s1) continue;
    int64_t* Hg = Hbase + (size_t)s_slot[pc] * SLOT;
    int64_t* Hh = Hg + kHistBins;
    const int64_t poff = s_pstart[pc] - s_vstart[pc];   // physical position = virtual + poff
    for (int64_t c0 = s0; c0 < s1; c0 += HIST_CHUNK) {
      const int64_t c1 = min(s1, c0 + HIST_CHUNK);
      const int64_t clen = c1 - c0;
      const int64_t w0 = c0 + clen * warp / H3_WARPS, w1 = c0 + clen * (warp + 1) / H3_WARPS;
      const int nb = (int)((w1 - w0 + 31) >> 5);
      auto ridx_of = [&](int b) -> uint32_t {   // this lane's row index in batch b (0 past the range)
        const int64_t vi = w0 + 32 * (int64_t)b + lane;
        if (vi >= w1) return 0u;
        if (MODE == HM_LEVEL) return sr_in[vi + poff];
        return dbg.idx ? (uint32_t)dbg.idx[vi + poff] : (uint32_t)(vi + poff);
      };
      auto issue = [&](int b, uint32_t ri) {   // gathers of batch b into its stage (one commit group)
        if (b < nb && w0 + 32 * (int64_t)b + lane < w1) {
          const uint32_t st = ring + (uint32_t)((b % H3_STAGES) * H3_STAGE);
          const uint8_t* src = a.codes + (size_t)ri * kMaxF;
          cp_async16(st + h3_half(lane, 0), src);
          cp_async16(st + h3_half(lane, 1), src + 16);
          if (MODE == HM_LEVEL) cp_async4(st + H3_GP + lane * 4, a.gp_root + ri);
          else sts32(st + H3_GP + lane * 4, pack_gp(dbg.qg[ri], dbg.qh[ri]));
        }
        cp_async_commit();
      };
      uint32_t ri_a = ridx_of(2), ri_b = ridx_of(3);
      issue(0, ridx_of(0));
      issue(1, ridx_of(1));
      uint32_t cur = 0;          // feature side: byte offset of the pending run's (bin, f) cell
      int32_t acc_g = 0;         // its sums from earlier batches
      uint32_t acc_h = 0;
      bool fresh = true;
      for (int b = 0; b < nb; ++b) {
        __syncwarp();            // batch b-2's stage (and b-3's) fully consumed by every lane
        issue(b + 2, ri_a);
        ri_a = ri_b;
        ri_b = ridx_of(b + 4);
        cp_async_wait<2>();      // batch b has landed (b+1, b+2 may be in flight)
        __syncwarp();
        const uint32_t st = ring + (uint32_t)((b % H3_STAGES) * H3_STAGE);
        const int cnt = (int)min((int64_t)32, w1 - (w0 + 32 * (int64_t)b));
        const bool valid = lane < cnt;
        // ---- row side: does row `lane` differ from its predecessor in any (non-users) feature?
        const uint4 c0v = lds128(st + h3_half(lane, 0)), c1v = lds128(st + h3_half(lane, 1));
        const uint32_t pst = lane ? st : ring + (uint32_t)(((b + H3_STAGES - 1) % H3_STAGES) * H3_STAGE);
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
        int32_t pg = qg;          // inclusive prefix sums of the pairs over the batch's rows
        uint32_t ph = qh;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t ug = __shfl_up_sync(0xffffffffu, pg, o);
          const uint32_t uh = __shfl_up_sync(0xffffffffu, ph, o);
          if (lane >= o) {
            pg += ug;
            ph += uh;
          }
        }
        const int32_t tot_g = __shfl_sync(0xffffffffu, pg, 31);
        const uint32_t tot_h = __shfl_sync(0xffffffffu, ph, 31);
        // ---- feature side: walk the flagged rows only
        if (fresh) {   // the first row starts every lane's run
          cur = (lds8(st + foff0) * 32u + (uint32_t)lane) * 4u;
          fresh = false;
          B &= ~1u;
        }
        int32_t bg = 0;          // prefix before the pending run's first row in this batch
        uint32_t bh = 0;
        while (B) {
          const int r = __ffs(B) - 1;
          B &= B - 1u;
          const uint32_t c = lds8(st + (uint32_t)(r * 32) + (((r >> 2) & 1) ? foff1 : foff0));
          const int32_t vg0 = __shfl_sync(0xffffffffu, pg, (r - 1) & 31);
          const uint32_t vh0 = __shfl_sync(0xffffffffu, ph, (r - 1) & 31);
          const int32_t vg = r ? vg0 : 0;
          const uint32_t vh = r ? vh0 : 0u;
          const uint32_t na = (c * 32u + (uint32_t)lane) * 4u;
          if (active && na != cur) {
            red2_h3(sgb + cur, acc_g + (vg - bg), acc_h + (vh - bh));
            acc_g = 0;
            acc_h = 0;
            bg = vg;
            bh = vh;
            cur = na;
          }
        }
        acc_g += tot_g - bg;
        acc_h += tot_h - bh;
      }
      if (active && !fresh && (acc_g | (int32_t)acc_h)) red2_h3(sgb + cur, acc_g, acc_h);
      cp_async_wait<0>();
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
    }
  }
}
