// Kernel-side flag wait of the peer transport (include/bitpipe_comm.h):
// one thread polls a 32-bit flag with acquire loads (system scope: the flag
// lives in another process's / GPU's memory) and nanosleep back-off until
// (int32)(*addr - value) >= 0.  Used instead of the stream-memory-operation
// wait (cuStreamWaitValue32, bp_flag_wait) when several ranks share ONE GPU
// (tests): a channel blocked in a semaphore acquire is not time-sliced out,
// so a waiting rank's context can starve the rank that would raise the
// flag; a spinning kernel is preemptible.  One GPU per rank uses bp_flag_wait.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/bitpipe_comm.h"

namespace bp {
void set_error(const char* fmt, ...);
void count_launch();
}

namespace {
__global__ void flag_wait_kernel(const uint32_t* addr, uint32_t value) {
  uint32_t ns = 32;
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(addr) : "memory");
    if ((int32_t)(v - value) >= 0) break;
    __nanosleep(ns);
    if (ns < 4096) ns <<= 1;
  }
}
}  // namespace

extern "C" int bp_flag_wait_spin(void* stream, const void* addr, uint32_t value) {
  if (!addr || (reinterpret_cast<uintptr_t>(addr) & 3)) {
    bp::set_error("bp_flag_wait_spin: flag address must be 4-byte aligned device memory");
    return BP_ERR_INVALID;
  }
  flag_wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint32_t*>(addr), value);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    bp::set_error("bp_flag_wait_spin: %s", cudaGetErrorString(e));
    return BP_ERR_CUDA;
  }
  bp::count_launch();
  return BP_OK;
}
