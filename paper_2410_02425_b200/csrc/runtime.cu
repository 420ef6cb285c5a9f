// runtime.cu — context, error plumbing, instrumentation, host/device pointer handling and the
// NCCL collectives (NCCL is dlopen'ed so a one-GPU process needs no NCCL at all).
#include <dlfcn.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <map>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "common.cuh"

namespace llmp {

[[noreturn]] void fail(llmpilot_status st, const std::string& msg) { throw Error{st, msg}; }

void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  llmpilot_status st = (e == cudaErrorMemoryAllocation) ? LLMP_ENOMEM : LLMP_ECUDA;
  cudaGetLastError();  // clear sticky-free errors
  fail(st, std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" + std::to_string(line) + ")");
}

void DevBuf::alloc(size_t b) {
  bytes = b;
  if (b == 0) { p = nullptr; return; }
  cudaError_t e = stream_ordered ? cudaMallocAsync(&p, b, ord) : cudaMalloc(&p, b);
  if (e != cudaSuccess) {
    p = nullptr;
    bytes = 0;
    cudaGetLastError();
    fail(LLMP_ENOMEM, "cudaMalloc(" + std::to_string(b) + " bytes) failed: " + cudaGetErrorString(e));
  }
}
void DevBuf::release() {
  if (p && stream_ordered) {
    if (cudaFreeAsync(p, ord) != cudaSuccess) {   // e.g. the stream is gone: synchronous fallback
      cudaGetLastError();
      cudaDeviceSynchronize();
      cudaFree(p);
    }
  } else if (p) {
    cudaFree(p);
  }
  p = nullptr;
  bytes = 0;
}

cudaEvent_t Ctx::get_event() {
  if (!free_events.empty()) {
    cudaEvent_t e = free_events.back();
    free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  LLMP_CUDA(cudaEventCreate(&e));
  return e;
}
void Ctx::before(int cls, cudaEvent_t* ev) {
  if (!timing || (launches[cls] % (uint64_t)timing_every) != 0) return;
  timed[cls] += 1;
  *ev = get_event();
  LLMP_CUDA(cudaEventRecord(*ev, stream));
}
void Ctx::after(int cls, cudaEvent_t ev, double nrows) {
  launches[cls] += 1;
  rows[cls] += nrows;
  if (!timing || !ev) return;
  cudaEvent_t b = get_event();
  LLMP_CUDA(cudaEventRecord(b, stream));
  pending.push_back(EventPair{ev, b, cls});
  if (pending.size() > 200000) collect();
}
void Ctx::collect() {
  if (pending.empty()) return;
  LLMP_CUDA(cudaStreamSynchronize(stream));
  for (auto& e : pending) {
    float ms = 0.f;
    LLMP_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
    ms_done[e.cls] += ms;
    free_events.push_back(e.a);
    free_events.push_back(e.b);
  }
  pending.clear();
}

// Max dynamic shared memory opt-in, per (device, kernel): cudaFuncSetAttribute applies to the
// current device only, and contexts on several devices (or several host threads) may launch the same
// kernel, so the record is keyed by device and guarded by a lock.  Only grows.
void ensure_smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice", __FILE__, __LINE__);
  std::lock_guard<std::mutex> lk(mu);
  int& cur = done[std::make_pair(dev, func)];
  if (cur >= bytes) return;
  check_cuda(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
             "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)", __FILE__, __LINE__);
  cur = bytes;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

const void* to_device(Ctx* ctx, const void* p, size_t bytes, DevBuf& tmp) {
  if (!p || is_device_ptr(p)) return p;
  tmp.ensure(bytes);
  LLMP_CUDA(cudaMemcpyAsync(tmp.p, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return tmp.p;
}

// ---------------------------------------------------------------------------------------------
// NCCL through dlopen (the torch-bundled libnccl.so.2 is already loaded in a torch process)
namespace {
typedef int ncclResult_t;
typedef void* ncclComm_t;
struct NcclUniqueId { char internal[128]; };
enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclUint32 = 3, ncclInt64 = 4, ncclUint64 = 5 };
enum { ncclSum = 0, ncclProd = 1, ncclMax = 2, ncclMin = 3 };
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*getUniqueId)(NcclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
  ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;
void load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);   // contexts may be created from several host threads
  if (g_nccl.loaded) return;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) fail(LLMP_ENCCL, std::string("cannot dlopen libnccl.so.2: ") + dlerror());
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
  g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
  g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.groupStart = (decltype(g_nccl.groupStart))dlsym(h, "ncclGroupStart");
  g_nccl.groupEnd = (decltype(g_nccl.groupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.commSplit = (decltype(g_nccl.commSplit))dlsym(h, "ncclCommSplit");
  g_nccl.commGetAsyncError = (decltype(g_nccl.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
  g_nccl.commAbort = (decltype(g_nccl.commAbort))dlsym(h, "ncclCommAbort");
  if (!g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.allGather || !g_nccl.commDestroy || !g_nccl.groupStart ||
      !g_nccl.groupEnd)
    fail(LLMP_ENCCL, "libnccl.so.2 lacks the needed symbols");
  g_nccl.loaded = true;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r == 0) return;
  fail(LLMP_ENCCL, std::string(what) + ": " + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "nccl error"));
}
}  // namespace

void nccl_init(Ctx* ctx, const void* unique_id) {
  load_nccl();
  NcclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  nccl_check(g_nccl.commInitRank(&comm, ctx->nranks, id, ctx->rank), "ncclCommInitRank");
  ctx->nccl = comm;
  // a second communicator over the same ranks for the second ensemble's collectives: the two
  // ensembles' trees then grow as concurrent graph branches, each branch ordering its own
  // communicator's collectives identically on every rank (one communicator shared by two concurrent
  // branches could interleave its collectives differently on different ranks)
  if (g_nccl.commSplit) {
    ncclComm_t c2 = nullptr;
    if (g_nccl.commSplit(comm, 0, ctx->rank, &c2, nullptr) == 0) ctx->nccl2 = c2;
  }
}
// ncclCommGetAsyncError on both communicators; on an error, abort them and fail (LLMP_ENCCL) instead
// of letting the next collective hang
void nccl_health(Ctx* ctx) {
  if (!ctx->nccl || !g_nccl.commGetAsyncError) return;
  for (void* c : {ctx->nccl, ctx->nccl2}) {
    if (!c) continue;
    ncclResult_t r = 0;
    g_nccl.commGetAsyncError((ncclComm_t)c, &r);
    if (r != 0 && r != 7 /* ncclInProgress */) {
      const std::string msg = std::string("NCCL asynchronous error: ") + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?");
      if (g_nccl.commAbort) {
        if (ctx->nccl2) g_nccl.commAbort((ncclComm_t)ctx->nccl2);
        g_nccl.commAbort((ncclComm_t)ctx->nccl);
      }
      ctx->nccl = ctx->nccl2 = nullptr;
      fail(LLMP_ENCCL, msg);
    }
  }
}
void nccl_unique_id(void* out) {
  load_nccl();
  LLMP_REQUIRE(g_nccl.getUniqueId != nullptr, "ncclGetUniqueId missing");
  NcclUniqueId id;
  nccl_check(g_nccl.getUniqueId(&id), "ncclGetUniqueId");
  memcpy(out, &id, sizeof(id));
}
void nccl_destroy(Ctx* ctx) {
  if (ctx->nccl2 && g_nccl.commDestroy) g_nccl.commDestroy((ncclComm_t)ctx->nccl2);
  if (ctx->nccl && g_nccl.commDestroy) g_nccl.commDestroy((ncclComm_t)ctx->nccl);
  ctx->nccl = ctx->nccl2 = nullptr;
}
// the communicator of the collectives being issued (ctx->comm_sel: the graph branch)
static ncclComm_t comm_of(Ctx* ctx) {
  return (ncclComm_t)((ctx->comm_sel == 1 && ctx->nccl2) ? ctx->nccl2 : ctx->nccl);
}
static void coll_before(Ctx* ctx, cudaEvent_t* ev) { ctx->before(KC_NCCL, ev); }

// ---------------------------------------------------------------------------------------------
// Local group: N ranks (contexts) on ONE device in one process, each driven by its own host thread.
// NCCL refuses two ranks on one GPU, so this is how the multi-rank fit path (shard geometry, the
// all-gathered cut sample, hessian-chosen built children, summed partial histograms) is exercised
// on one B200.  A collective: every rank synchronises its stream and publishes its buffer; rank 0
// reduces the others' buffers into its own on the device; the rest copy the result back; host
// barriers separate the phases.  Slow by design (host round trips), exact like NCCL's integer sums.
struct LocalGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0, refs = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
LocalGroup* local_group_create(int nranks) {
  auto* g = new LocalGroup();
  g->n = nranks;
  g->refs = nranks;
  g->ptr.assign(nranks, nullptr);
  return g;
}
void local_group_release(LocalGroup* g) {
  if (!g) return;
  bool last;
  {
    std::lock_guard<std::mutex> lk(g->m);
    last = --g->refs == 0;
  }
  if (last) delete g;
}
enum { LG_SUM_I64 = 0, LG_MAX_U32 = 1, LG_MAX_U64 = 2 };
__global__ void k_lg_reduce(void* dst, const void* src, size_t n, int op) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    if (op == LG_SUM_I64) static_cast<int64_t*>(dst)[i] += static_cast<const int64_t*>(src)[i];
    else if (op == LG_MAX_U32)
      static_cast<uint32_t*>(dst)[i] = max(static_cast<uint32_t*>(dst)[i], static_cast<const uint32_t*>(src)[i]);
    else static_cast<uint64_t*>(dst)[i] = max(static_cast<uint64_t*>(dst)[i], static_cast<const uint64_t*>(src)[i]);
  }
}
static void lg_allreduce(Ctx* ctx, void* buf, size_t count, size_t esize, int op) {
  LocalGroup* g = ctx->lgroup;
  LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
  g->ptr[ctx->rank] = buf;
  g->barrier();
  if (ctx->rank == 0) {
    for (int r = 1; r < g->n; ++r)
      k_lg_reduce<<<(int)std::min<size_t>((count + 255) / 256, 1024), 256, 0, ctx->stream>>>(buf, g->ptr[r], count, op);
    LLMP_CUDA(cudaGetLastError());
    LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  g->barrier();
  if (ctx->rank != 0) {
    LLMP_CUDA(cudaMemcpyAsync(buf, g->ptr[0], count * esize, cudaMemcpyDeviceToDevice, ctx->stream));
    LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  g->barrier();   // rank 0's buffer stays untouched until every rank has its copy
}
static void lg_allgather(Ctx* ctx, const void* send, void* recv, size_t bytes) {
  LocalGroup* g = ctx->lgroup;
  LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
  g->ptr[ctx->rank] = send;
  g->barrier();
  for (int r = 0; r < g->n; ++r)
    LLMP_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + (size_t)r * bytes, g->ptr[r], bytes,
                              cudaMemcpyDeviceToDevice, ctx->stream));
  LLMP_CUDA(cudaStreamSynchronize(ctx->stream));
  g->barrier();
}
// several collectives issued between these become one NCCL launch (no-ops without a communicator,
// and while per-launch event timing is on, so every collective keeps its own events)
void nccl_group_start(Ctx* ctx) {
  if (ctx->nccl && !ctx->timing) nccl_check(g_nccl.groupStart(), "ncclGroupStart");
}
void nccl_group_end(Ctx* ctx) {
  if (ctx->nccl && !ctx->timing) nccl_check(g_nccl.groupEnd(), "ncclGroupEnd");
}
void allreduce_sum_i64(Ctx* ctx, int64_t* buf, size_t count) {
  if (count == 0) return;
  if (ctx->lgroup) return lg_allreduce(ctx, buf, count, 8, LG_SUM_I64);
  if (!ctx->nccl) return;
  cudaEvent_t ev = nullptr;
  coll_before(ctx, &ev);
  nccl_check(g_nccl.allReduce(buf, buf, count, ncclInt64, ncclSum, comm_of(ctx), ctx->stream), "ncclAllReduce");
  ctx->after(KC_NCCL, ev, (double)count * 8);
}
void allreduce_max_u32(Ctx* ctx, uint32_t* buf, size_t count) {
  if (count == 0) return;
  if (ctx->lgroup) return lg_allreduce(ctx, buf, count, 4, LG_MAX_U32);
  if (!ctx->nccl) return;
  cudaEvent_t ev = nullptr;
  coll_before(ctx, &ev);
  nccl_check(g_nccl.allReduce(buf, buf, count, ncclUint32, ncclMax, comm_of(ctx), ctx->stream), "ncclAllReduce");
  ctx->after(KC_NCCL, ev, (double)count * 4);
}
void allreduce_max_u64(Ctx* ctx, uint64_t* buf, size_t count) {
  if (count == 0) return;
  if (ctx->lgroup) return lg_allreduce(ctx, buf, count, 8, LG_MAX_U64);
  if (!ctx->nccl) return;
  cudaEvent_t ev = nullptr;
  coll_before(ctx, &ev);
  nccl_check(g_nccl.allReduce(buf, buf, count, ncclUint64, ncclMax, comm_of(ctx), ctx->stream), "ncclAllReduce");
  ctx->after(KC_NCCL, ev, (double)count * 8);
}
void allgather_bytes(Ctx* ctx, const void* send, void* recv, size_t bytes_per_rank) {
  if (ctx->lgroup) return lg_allgather(ctx, send, recv, bytes_per_rank);
  if (!ctx->nccl) {
    if (send != recv) LLMP_CUDA(cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  cudaEvent_t ev = nullptr;
  coll_before(ctx, &ev);
  nccl_check(g_nccl.allGather(send, recv, bytes_per_rank, ncclUint8, comm_of(ctx), ctx->stream), "ncclAllGather");
  ctx->after(KC_NCCL, ev, (double)bytes_per_rank * ctx->nranks);
}

}  // namespace llmp
