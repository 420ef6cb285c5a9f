// common.cuh — shared internals of the llmpilot CUDA library (sm_100a).
// Nothing here is shared with oracle/: the oracle is an independent C program.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string.h>

#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/llmpilot.h"

namespace llmp {

// NVTX range (header-only NVTX3: a no-op unless a tool such as nsys or ncu --nvtx attaches): every
// C-ABI entry point, the fit phases, and per tree / level when the tree loop runs as plain launches
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kMaxF = 32;        // features per row (codes padded to 32 bytes = one DRAM sector)
constexpr int kBins = 256;       // histogram bins per feature (u8 codes)
constexpr int kHistBins = kMaxF * kBins;  // 8192 (feature, bin) cells per node
constexpr int kMaxDepth = 10;
constexpr int kMaxCuts16 = 1023; // 16-bit codes (small-fit path): up to 1024 bins per feature
constexpr int kMaxGradBits = 14; // |q_g| <= 2^14 fits int16; q_h <= 2^14 fits uint16 => 32-bit pair

// kernel classes for instrumentation (llmpilot_kernel_class_name)
enum KernelClass {
  KC_VALIDATE = 0, KC_WEIGHTS, KC_CUTS, KC_CODES, KC_BASE, KC_HIST_ROOT, KC_PARTITION, KC_HIST, KC_SPLIT,
  KC_UPDATE, KC_PREDICT, KC_RECOMMEND, KC_MISC, KC_NCCL, KC_WG, KC_FIT_SMALL, KC_COUNT
};

// ---------------------------------------------------------------------------------------------
// error handling: every failure becomes an exception inside the library, converted to a status
// at the C-ABI boundary (api.cu).
struct Error {
  llmpilot_status st;
  std::string msg;
};
[[noreturn]] void fail(llmpilot_status st, const std::string& msg);
void check_cuda(cudaError_t e, const char* what, const char* file, int line);
#define LLMP_CUDA(x) ::llmp::check_cuda((x), #x, __FILE__, __LINE__)
#define LLMP_REQUIRE(cond, msg) \
  do {                          \
    if (!(cond)) ::llmp::fail(LLMP_EINVAL, msg); \
  } while (0)

// ---------------------------------------------------------------------------------------------
// device buffer (RAII)
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  // stream-ordered buffers (model and cuts handles returned to the caller): allocated with
  // cudaMallocAsync and released with cudaFreeAsync on `ord` from the device's default pool, so a
  // fit/free cycle neither synchronises the device nor returns memory to the driver
  cudaStream_t ord = nullptr;
  bool stream_ordered = false;
  DevBuf() = default;
  explicit DevBuf(size_t b) { alloc(b); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), ord(o.ord), stream_ordered(o.stream_ordered) {
    o.p = nullptr; o.bytes = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p; bytes = o.bytes; ord = o.ord; stream_ordered = o.stream_ordered; o.p = nullptr; o.bytes = 0;
    return *this;
  }
  void set_stream(cudaStream_t s) { ord = s; stream_ordered = true; }
  ~DevBuf() { release(); }
  void alloc(size_t b);
  void ensure(size_t b) { if (b > bytes) { release(); alloc(b); } }
  void release();
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// ---------------------------------------------------------------------------------------------
// context
struct EventPair { cudaEvent_t a, b; int cls; };

struct LocalGroup;   // runtime.cu: N ranks on one device in one process (test/emulation communicator)
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, nranks = 1;
  void* nccl = nullptr;   // ncclComm_t (dlopen'ed NCCL), null for one GPU
  void* nccl2 = nullptr;  // a second communicator over the same ranks (the second ensemble's graph branch)
  int comm_sel = 0;       // 1: collectives being issued go to nccl2
  LocalGroup* lgroup = nullptr;   // set instead of nccl by llmpilot_ctx_create_local_group
  bool own_stream = false;        // the stream was created by the library (local groups)
  bool sharded() const { return nccl != nullptr || lgroup != nullptr; }
  int sms = 148;
  unsigned long long* d_units = nullptr;  // [LLMP_N_KERNEL_CLASSES] device-side unit counters
  bool timing = false;
  int timing_every = 1;                    // time every k-th launch of each class
  uint64_t timed[LLMP_N_KERNEL_CLASSES] = {};
  bool use_graphs = true;                  // replay each tree from a CUDA graph (off while timing)
  bool pdl = false;                        // programmatic dependent launch inside the tree loop
  cudaStream_t cap_stream[2] = {nullptr, nullptr};   // private streams used only for graph capture
  cudaEvent_t fork_event = nullptr, join_event = nullptr;
  cudaStream_t capture_stream(int i) {
    if (!cap_stream[i]) {
      check_cuda(cudaStreamCreateWithFlags(&cap_stream[i], cudaStreamNonBlocking), "capture stream", __FILE__,
                 __LINE__);
      if (!fork_event) {
        check_cuda(cudaEventCreateWithFlags(&fork_event, cudaEventDisableTiming), "event", __FILE__, __LINE__);
        check_cuda(cudaEventCreateWithFlags(&join_event, cudaEventDisableTiming), "event", __FILE__, __LINE__);
      }
    }
    return cap_stream[i];
  }
  uint64_t launches[LLMP_N_KERNEL_CLASSES] = {};
  double rows[LLMP_N_KERNEL_CLASSES] = {};
  double ms_done[LLMP_N_KERNEL_CLASSES] = {};
  std::vector<EventPair> pending;
  std::vector<cudaEvent_t> free_events;
  // named device workspaces reused across calls (grow-only): repeated fits on one context do
  // no cudaMalloc/cudaFree (cudaFree synchronises the device).  A context is not thread-safe.
  std::map<std::string, DevBuf> ws;
  DevBuf& workspace(const std::string& name, size_t bytes) {
    DevBuf& b = ws[name];
    b.ensure(bytes);
    return b;
  }
  cudaEvent_t get_event();
  void before(int cls, cudaEvent_t* ev);
  void after(int cls, cudaEvent_t ev, double nrows);
  void collect();   // sync + fold pending event pairs into ms_done
};

// launch helper: instrumentation + error check
#define LLMP_LAUNCH(ctx, cls, nrows, kernel, grid, block, smem, ...)                \
  do {                                                                            \
    cudaEvent_t _ev = nullptr;                                                    \
    (ctx)->before((cls), &_ev);                                                   \
    kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);              \
    LLMP_CUDA(cudaGetLastError());                                                \
    (ctx)->after((cls), _ev, (double)(nrows));                                    \
  } while (0)

// Programmatic dependent launch (LLMP_PDL): the kernel may be scheduled while its predecessor in the
// stream finishes; every kernel launched this way calls pdl_wait() (griddepcontrol.wait) before it
// touches memory, so only the launch latency overlaps.  Without the attribute the wait is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define LLMP_LAUNCH_PDL(ctx, cls, nrows, kernel, grid, block, smem, ...)                         \
  do {                                                                                           \
    if (!(ctx)->pdl) {                                                                           \
      LLMP_LAUNCH(ctx, cls, nrows, kernel, grid, block, smem, __VA_ARGS__);                      \
      break;                                                                                     \
    }                                                                                            \
    cudaEvent_t _ev = nullptr;                                                                   \
    (ctx)->before((cls), &_ev);                                                                  \
    cudaLaunchConfig_t _cfg = {};                                                                \
    _cfg.gridDim = dim3(grid);                                                                   \
    _cfg.blockDim = dim3(block);                                                                 \
    _cfg.dynamicSmemBytes = (smem);                                                              \
    _cfg.stream = (ctx)->stream;                                                                 \
    cudaLaunchAttribute _at[1];                                                                  \
    _at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                              \
    _at[0].val.programmaticStreamSerializationAllowed = 1;                                       \
    _cfg.attrs = _at;                                                                            \
    _cfg.numAttrs = 1;                                                                           \
    LLMP_CUDA(cudaLaunchKernelEx(&_cfg, kernel, __VA_ARGS__));                                   \
    (ctx)->after((cls), _ev, (double)(nrows));                                                   \
  } while (0)

// copy a bulk array to the device if it is a host pointer; returns a device pointer (either the
// original or `tmp`'s storage)
bool is_device_ptr(const void* p);
// per-device, thread-safe opt-in to `bytes` of dynamic shared memory for a kernel (only grows)
void ensure_smem_attr(const void* func, int bytes);
const void* to_device(Ctx* ctx, const void* p, size_t bytes, DevBuf& tmp);

// multi-GPU collectives (nccl.cu); no-ops for one rank
void allreduce_sum_i64(Ctx* ctx, int64_t* buf, size_t count);
void nccl_group_start(Ctx* ctx);
void nccl_group_end(Ctx* ctx);
void allreduce_max_u32(Ctx* ctx, uint32_t* buf, size_t count);
void allreduce_max_u64(Ctx* ctx, uint64_t* buf, size_t count);
void allgather_bytes(Ctx* ctx, const void* send, void* recv, size_t bytes_per_rank);
LocalGroup* local_group_create(int nranks);
void local_group_release(LocalGroup* g);   // the last rank's release deletes it
void nccl_init(Ctx* ctx, const void* unique_id);
void nccl_unique_id(void* out);
void nccl_destroy(Ctx* ctx);
void nccl_health(Ctx* ctx);   // ncclCommGetAsyncError; abort + LLMP_ENCCL on an error

// ---------------------------------------------------------------------------------------------
// device helpers
__host__ __device__ inline uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// counter-based generator shared by GPU kernels: chained splitmix64 finaliser
__host__ __device__ inline uint64_t rng4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return sm64(sm64(sm64(sm64(seed) ^ a) ^ b) ^ c);
}

// e with M = m * 2^e, m in [0.5, 1) (0 for M == 0); M >= 0 finite, from the IEEE bits
__host__ __device__ inline int exp_of(float M) {
  uint32_t b;
#ifdef __CUDA_ARCH__
  b = __float_as_uint(M);
#else
  memcpy(&b, &M, 4);
#endif
  int ex = (int)((b >> 23) & 0xffu);
  if (ex != 0) return ex - 126;
  uint32_t mant = b & 0x7fffffu;
  if (mant == 0) return 0;
  int p = 31;
  while (!(mant >> p)) --p;
  return p - 148;
}

// q = rint(v * 2^(K-e)) evaluated exactly in fp64 (v * 2^s is exact in double for any float v)
__device__ __forceinline__ int32_t quantize(float v, double scale) {
  return __double2int_rn(__dmul_rn((double)v, scale));
}

// packed gradient pair: high 16 bits = q_g (int16), low 16 bits = q_h (uint16)
__device__ __forceinline__ uint32_t pack_gp(int32_t qg, int32_t qh) {
  return ((uint32_t)(qg & 0xffff) << 16) | (uint32_t)(qh & 0xffff);
}
__device__ __forceinline__ int32_t gp_g(uint32_t gp) { return (int32_t)gp >> 16; }
__device__ __forceinline__ int32_t gp_h(uint32_t gp) { return (int32_t)(gp & 0xffffu); }

// XGBoost-convention leaf weight and gain (fp64, explicit rounding intrinsics, no FMA)
__device__ __forceinline__ double calc_weight(double G, double H, double lo, double hi, double lambda, double mcw) {
  double w = 0.0;
  if (!(H < mcw || H <= 0.0)) w = __ddiv_rn(-G, __dadd_rn(H, lambda));
  if (w < lo) w = lo;
  else if (w > hi) w = hi;
  return w;
}
__device__ __forceinline__ double calc_gain(double G, double H, double w, double lambda) {
  if (H <= 0.0) return 0.0;
  return -__dadd_rn(__dmul_rn(__dmul_rn(2.0, G), w), __dmul_rn(__dadd_rn(H, lambda), __dmul_rn(w, w)));
}
// ldexp((double)q, s) exactly: multiply by the exact power of two
__device__ __forceinline__ double dequant(int64_t q, double scale_inv) { return __dmul_rn((double)q, scale_inv); }

inline int ceil_div_i(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace llmp
