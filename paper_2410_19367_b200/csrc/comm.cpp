// Runtime context of libbitpipe_b200.so (include/bitpipe_comm.h): NCCL
// communicators, message-slot slabs, events and CUDA-graph capture for a
// host that drives the pipeline through the C ABI.  NCCL is resolved with
// dlopen at first use, so the library has no link-time NCCL dependency and
// shares the copy torch already loaded (same soname) when there is one.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/bitpipe_comm.h"

namespace bp {
void set_error(const char* fmt, ...);
}

struct bp_ctx {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  std::vector<void*> slabs;
};

namespace {

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
};

// Resolve the NCCL entry points from a library handle (false if incomplete).
bool resolve(Nccl& n, void* h) {
#define BP_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
  BP_SYM(GetUniqueId, "ncclGetUniqueId");
  BP_SYM(CommInitRank, "ncclCommInitRank");
  BP_SYM(CommSplit, "ncclCommSplit");
  BP_SYM(CommDestroy, "ncclCommDestroy");
  BP_SYM(Send, "ncclSend");
  BP_SYM(Recv, "ncclRecv");
  BP_SYM(AllReduce, "ncclAllReduce");
  BP_SYM(GroupStart, "ncclGroupStart");
  BP_SYM(GroupEnd, "ncclGroupEnd");
  BP_SYM(GetErrorString, "ncclGetErrorString");
  BP_SYM(CommCount, "ncclCommCount");
  BP_SYM(CommUserRank, "ncclCommUserRank");
#undef BP_SYM
  return n.GetUniqueId && n.CommInitRank && n.CommSplit && n.CommDestroy && n.Send && n.Recv && n.AllReduce &&
         n.GroupStart && n.GroupEnd && n.GetErrorString && n.CommCount && n.CommUserRank;
}

void* loaded_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_NOLOAD);
  return h;
}

// The process's NCCL.  Prefer the copy already loaded (torch's).  With
// `allow_load`, load libnccl.so.2 when none is: that copy stays in the
// process, and a later torch import resolves its own libnccl.so.2 dependency
// to it by soname (RTLD_LOCAL only limits symbol scope), so a host mixing
// torch and this ABI must import torch first.  A failed lookup is never
// cached: the next call retries (e.g. after torch has loaded NCCL).
Nccl& nccl(bool allow_load = true) {
  static Nccl n;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (n.ok) return n;
  void* h = loaded_nccl();
  if (!h && allow_load) {
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  }
  if (h) {
    Nccl t;
    if (resolve(t, h)) {
      t.ok = true;
      n = t;
    }
  }
  return n;
}

int need_nccl() {
  if (nccl().ok) return BP_OK;
  bp::set_error("NCCL library (libnccl.so.2) not found or incomplete");
  return BP_ERR_COMM;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return BP_OK;
  bp::set_error("%s: %s", what, nccl().GetErrorString(r));
  return BP_ERR_COMM;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return BP_OK;
  bp::set_error("%s: %s", what, cudaGetErrorString(e));
  return BP_ERR_CUDA;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int bp_comm_available(void) {
  if (loaded_nccl()) return nccl(false).ok ? 1 : 0;
  // not in the process yet: probe whether one can be loaded, without keeping it
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  if (!h) return 0;
  Nccl t;
  const bool ok = resolve(t, h);
  dlclose(h);
  return ok ? 2 : 0;
}

int bp_nccl_unique_id(void* id_out) {
  if (int rc = need_nccl()) return rc;
  if (!id_out) {
    bp::set_error("bp_nccl_unique_id: NULL output");
    return BP_ERR_INVALID;
  }
  ncclUniqueId id;
  if (int rc = nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId")) return rc;
  static_assert(sizeof(ncclUniqueId) == BP_NCCL_ID_BYTES, "NCCL unique id size");
  memcpy(id_out, &id, sizeof(id));
  return BP_OK;
}

int bp_init(int rank, int world, const void* nccl_id, int device, bp_ctx** ctx_out) {
  if (int rc = need_nccl()) return rc;
  if (!nccl_id || !ctx_out || world < 1 || rank < 0 || rank >= world) {
    bp::set_error("bp_init: invalid arguments (rank %d, world %d)", rank, world);
    return BP_ERR_INVALID;
  }
  if (int rc = cuda_check(cudaSetDevice(device), "cudaSetDevice")) return rc;
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  auto* c = new bp_ctx;
  c->rank = rank;
  c->world = world;
  c->device = device;
  if (int rc = nccl_check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank")) {
    delete c;
    return rc;
  }
  *ctx_out = c;
  return BP_OK;
}

int bp_comm_split(bp_ctx* ctx, int color, int key, bp_ctx** ctx_out) {
  if (int rc = need_nccl()) return rc;
  if (!ctx || !ctx_out) {
    bp::set_error("bp_comm_split: NULL context");
    return BP_ERR_INVALID;
  }
  ncclComm_t sub = nullptr;
  if (int rc = nccl_check(nccl().CommSplit(ctx->comm, color < 0 ? NCCL_SPLIT_NOCOLOR : color, key, &sub, nullptr),
                          "ncclCommSplit"))
    return rc;
  if (!sub) {
    *ctx_out = nullptr;
    return BP_OK;
  }
  auto* c = new bp_ctx;
  c->comm = sub;
  c->device = ctx->device;
  // rank / size inside the sub-communicator (ranks of one color ordered by key)
  int n = -1, r = -1;
  if (nccl().CommCount(sub, &n) != ncclSuccess || nccl().CommUserRank(sub, &r) != ncclSuccess || n < 1 || r < 0) {
    bp::set_error("bp_comm_split: cannot determine rank / size of the sub-communicator");
    nccl().CommDestroy(sub);
    delete c;
    return BP_ERR_COMM;
  }
  c->world = n;
  c->rank = r;
  *ctx_out = c;
  return BP_OK;
}

int bp_comm_rank(const bp_ctx* ctx) { return ctx ? ctx->rank : -1; }
int bp_comm_size(const bp_ctx* ctx) { return ctx ? ctx->world : -1; }

size_t bp_slot_stride(size_t bytes) { return (bytes + 255) & ~size_t(255); }

int bp_slots_alloc(bp_ctx* ctx, size_t bytes, int count, void** base_out) {
  if (!ctx || !base_out || count < 1 || bytes == 0) {
    bp::set_error("bp_slots_alloc: invalid arguments");
    return BP_ERR_INVALID;
  }
  void* p = nullptr;
  if (int rc = cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice")) return rc;
  if (int rc = cuda_check(cudaMalloc(&p, bp_slot_stride(bytes) * (size_t)count), "cudaMalloc(slots)")) return rc;
  ctx->slabs.push_back(p);
  *base_out = p;
  return BP_OK;
}

int bp_send(bp_ctx* ctx, int peer, const void* ptr, size_t bytes, void* stream) {
  if (int rc = need_nccl()) return rc;
  if (!ctx || (!ptr && bytes)) {
    bp::set_error("bp_send: invalid arguments");
    return BP_ERR_INVALID;
  }
  return nccl_check(nccl().Send(ptr, bytes, ncclUint8, peer, ctx->comm, S(stream)), "ncclSend");
}

int bp_recv(bp_ctx* ctx, int peer, void* ptr, size_t bytes, void* stream) {
  if (int rc = need_nccl()) return rc;
  if (!ctx || (!ptr && bytes)) {
    bp::set_error("bp_recv: invalid arguments");
    return BP_ERR_INVALID;
  }
  return nccl_check(nccl().Recv(ptr, bytes, ncclUint8, peer, ctx->comm, S(stream)), "ncclRecv");
}

int bp_group_start(void) {
  if (int rc = need_nccl()) return rc;
  return nccl_check(nccl().GroupStart(), "ncclGroupStart");
}

int bp_group_end(void) {
  if (int rc = need_nccl()) return rc;
  return nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}

int bp_allreduce_mean(bp_ctx* ctx, void* ptr, size_t n, int dtype, void* stream) {
  if (int rc = need_nccl()) return rc;
  if (!ctx || (!ptr && n) || (dtype != BP_F32 && dtype != BP_BF16)) {
    bp::set_error("bp_allreduce_mean: invalid arguments");
    return BP_ERR_INVALID;
  }
  const ncclDataType_t dt = dtype == BP_F32 ? ncclFloat32 : ncclBfloat16;
  return nccl_check(nccl().AllReduce(ptr, ptr, n, dt, ncclAvg, ctx->comm, S(stream)), "ncclAllReduce(avg)");
}

int bp_destroy(bp_ctx* ctx) {
  if (!ctx) return BP_OK;
  int rc = BP_OK;
  for (void* p : ctx->slabs) {
    const int r = cuda_check(cudaFree(p), "cudaFree(slots)");
    if (r && !rc) rc = r;
  }
  if (ctx->comm && nccl().ok) {
    const int r = nccl_check(nccl().CommDestroy(ctx->comm), "ncclCommDestroy");
    if (r && !rc) rc = r;
  }
  delete ctx;
  return rc;
}

int bp_event_create(void** ev_out) {
  if (!ev_out) {
    bp::set_error("bp_event_create: NULL output");
    return BP_ERR_INVALID;
  }
  cudaEvent_t e;
  if (int rc = cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate")) return rc;
  *ev_out = e;
  return BP_OK;
}

int bp_event_record(void* ev, void* stream) {
  return cuda_check(cudaEventRecord(static_cast<cudaEvent_t>(ev), S(stream)), "cudaEventRecord");
}

int bp_stream_wait_event(void* stream, void* ev) {
  return cuda_check(cudaStreamWaitEvent(S(stream), static_cast<cudaEvent_t>(ev), 0), "cudaStreamWaitEvent");
}

int bp_event_destroy(void* ev) { return cuda_check(cudaEventDestroy(static_cast<cudaEvent_t>(ev)), "cudaEventDestroy"); }

int bp_graph_begin(void* stream) {
  return cuda_check(cudaStreamBeginCapture(S(stream), cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
}

int bp_graph_end(void* stream, void** graph_exec_out) {
  if (!graph_exec_out) {
    bp::set_error("bp_graph_end: NULL output");
    return BP_ERR_INVALID;
  }
  cudaGraph_t g = nullptr;
  if (int rc = cuda_check(cudaStreamEndCapture(S(stream), &g), "cudaStreamEndCapture")) return rc;
  cudaGraphExec_t x = nullptr;
  const int rc = cuda_check(cudaGraphInstantiate(&x, g, 0), "cudaGraphInstantiate");
  cudaGraphDestroy(g);
  if (rc) return rc;
  *graph_exec_out = x;
  return BP_OK;
}

int bp_graph_launch(void* graph_exec, void* stream) {
  return cuda_check(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), S(stream)), "cudaGraphLaunch");
}

int bp_graph_destroy(void* graph_exec) {
  return cuda_check(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec)), "cudaGraphExecDestroy");
}

}  // extern "C"
