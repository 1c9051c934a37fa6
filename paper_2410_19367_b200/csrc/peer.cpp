// Peer-memory transport of libbitpipe_b200.so (include/bitpipe_comm.h,
// "peer memory" section): CUDA IPC export / import of device buffers, copy-
// engine copies into a peer's buffer, and stream-ordered 32-bit flags
// (cuStreamWriteValue32 / cuStreamWaitValue32) that gate a consumer stream on
// a producer in another process without the host and without an SM.
//
// This is the B200 realisation of "CUDA-event-gated P2P activation and
// gradient send/recv over NVLink" (BASELINE north star): the sender's stream
// copies a message straight into the receiver's tag-addressed slot (NVLink
// through NVSwitch when the receiver is another GPU, HBM when it is another
// process on the same GPU) and then bumps the slot's flag in the receiver's
// mailbox; the receiver's stream waits on that flag.  The same flags gate the
// fused peer-read replica-mean AdamW (bp_adam reading the partner's gradient
// through its imported pointer).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/bitpipe_comm.h"

namespace bp {
void set_error(const char* fmt, ...);
void count_launch();
}

namespace {

typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

struct Driver {
  bool ok = false;
  WaitFn wait = nullptr;
  WriteFn write = nullptr;
  RangeFn range = nullptr;
};

// The driver entry points come through the runtime (no link dependency on
// libcuda); a failed lookup is retried on the next call, never cached.
Driver& driver() {
  static Driver d;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (d.ok) return d;
  void* w = nullptr;
  void* x = nullptr;
  void* r = nullptr;
  cudaDriverEntryPointQueryResult q1, q2, q3;
  if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &w, 12000, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &x, 12000, cudaEnableDefault, &q2) != cudaSuccess ||
      cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &r, 12000, cudaEnableDefault, &q3) != cudaSuccess ||
      q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || q3 != cudaDriverEntryPointSuccess) {
    return d;
  }
  d.wait = reinterpret_cast<WaitFn>(w);
  d.write = reinterpret_cast<WriteFn>(x);
  d.range = reinterpret_cast<RangeFn>(r);
  d.ok = true;
  return d;
}

int need_driver() {
  if (driver().ok) return BP_OK;
  bp::set_error("CUDA driver entry points for stream memory operations are unavailable");
  return BP_ERR_CUDA;
}

int cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return BP_OK;
  bp::set_error("%s: CUDA driver error %d", what, (int)r);
  return BP_ERR_CUDA;
}

int rt_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return BP_OK;
  bp::set_error("%s: %s", what, cudaGetErrorString(e));
  return BP_ERR_CUDA;
}

// Imported allocations, one mapping per (device, handle) with a reference
// count: a process may import the same peer buffer for several purposes.
struct Import {
  void* base;
  int refs;
};
std::mutex g_ipc_mu;
std::map<std::string, Import> g_by_handle;
std::map<void*, std::string> g_by_base;

}  // namespace

extern "C" {

int bp_ipc_export(const void* ptr, void* handle_out, size_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) {
    bp::set_error("bp_ipc_export: NULL argument");
    return BP_ERR_INVALID;
  }
  if (int rc = need_driver()) return rc;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (int rc = cu_check(driver().range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)), "cuMemGetAddressRange"))
    return rc;
  cudaIpcMemHandle_t h;
  if (int rc = rt_check(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle")) return rc;
  static_assert(sizeof(h) == BP_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uintptr_t>(ptr) - static_cast<uintptr_t>(base);
  return BP_OK;
}

int bp_ipc_open(const void* handle, void** base_out) {
  if (!handle || !base_out) {
    bp::set_error("bp_ipc_open: NULL argument");
    return BP_ERR_INVALID;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  std::string key(static_cast<const char*>(handle), BP_IPC_HANDLE_BYTES);
  key += std::to_string(dev);
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  auto it = g_by_handle.find(key);
  if (it != g_by_handle.end()) {
    ++it->second.refs;
    *base_out = it->second.base;
    return BP_OK;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  if (int rc = rt_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle"))
    return rc;
  g_by_handle[key] = Import{p, 1};
  g_by_base[p] = key;
  *base_out = p;
  return BP_OK;
}

int bp_ipc_close(void* base) {
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  auto it = g_by_base.find(base);
  if (it == g_by_base.end()) {
    bp::set_error("bp_ipc_close: %p was not opened by bp_ipc_open", base);
    return BP_ERR_INVALID;
  }
  Import& imp = g_by_handle[it->second];
  if (--imp.refs > 0) return BP_OK;
  g_by_handle.erase(it->second);
  g_by_base.erase(it);
  return rt_check(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle");
}

int bp_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if ((!dst || !src) && bytes) {
    bp::set_error("bp_memcpy_async: NULL pointer");
    return BP_ERR_INVALID;
  }
  if (!bytes) return BP_OK;
  return rt_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)),
                  "cudaMemcpyAsync(peer)");
}

int bp_flag_set(void* stream, void* addr, uint32_t value) {
  if (!addr || (reinterpret_cast<uintptr_t>(addr) & 3)) {
    bp::set_error("bp_flag_set: flag address must be 4-byte aligned device memory");
    return BP_ERR_INVALID;
  }
  if (int rc = need_driver()) return rc;
  // default flags: a stream-scoped release fence precedes the write, so the
  // consumer that observes the value also observes every write (copies,
  // kernels) issued on this stream before it
  return cu_check(driver().write(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value,
                                 CU_STREAM_WRITE_VALUE_DEFAULT),
                  "cuStreamWriteValue32");
}

int bp_flag_wait(void* stream, const void* addr, uint32_t value) {
  if (!addr || (reinterpret_cast<uintptr_t>(addr) & 3)) {
    bp::set_error("bp_flag_wait: flag address must be 4-byte aligned device memory");
    return BP_ERR_INVALID;
  }
  if (int rc = need_driver()) return rc;
  // GEQ is the wrap-around-safe signed comparison (int32)(*addr - value) >= 0
  return cu_check(driver().wait(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value,
                                CU_STREAM_WAIT_VALUE_GEQ),
                  "cuStreamWaitValue32");
}

}  // extern "C"
