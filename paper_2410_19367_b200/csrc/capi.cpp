// Library-wide state of libbitpipe_b200.so: thread-local error text, the
// kernel launch counter, cached device properties and testing switches.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "../../include/bitpipe.h"

namespace bp {

static thread_local char g_err[1024] = "";
static std::atomic<unsigned long long> g_launches{0};
static std::atomic<int> g_opt_attn_exact{0}, g_opt_gemm_simt{0}, g_opt_gemm_mode{0}, g_opt_stream_k{2}, g_opt_gemm_wide{0}, g_opt_gemm_debug{0}, g_opt_gemm_tma_store{1}, g_opt_ln_unfused{0}, g_opt_ln_cps{1}, g_opt_ln_bwd_mode{0}, g_opt_attn_fwd_mode{0}, g_opt_gemm_occ{0}, g_opt_gemm_grid{0}, g_opt_gemm_bn{0}, g_opt_attn_bwd_mode{0}, g_opt_gemm_ew{0}, g_opt_attn_fwd_exf{0}, g_opt_gemm_l2{1}, g_opt_gemm_pick{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
  return BP_ERR_CUDA;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int num_sms() {
  static thread_local int cached_dev = -1, cached = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cached;
  if (dev != cached_dev) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0) cached = n;
    cached_dev = dev;
  }
  return cached;
}

bool opt_attn_exact() { return g_opt_attn_exact.load() == 1; }
bool opt_attn_no_tc() { return g_opt_attn_exact.load() != 0; }
bool opt_gemm_simt() { return g_opt_gemm_simt.load() != 0; }
int gemm_mode() { return g_opt_gemm_mode.load(); }
int stream_k_mode() { return g_opt_stream_k.load(); }
int gemm_wide_mode() { return g_opt_gemm_wide.load(); }
int gemm_debug_nostore() { return g_opt_gemm_debug.load() == 1; }
int gemm_tma_store_mode() { return g_opt_gemm_tma_store.load(); }
bool ln_bwd_unfused() { return g_opt_ln_unfused.load() != 0; }
int ln_ctas_per_sm() { return g_opt_ln_cps.load(); }
int ln_bwd_mode() { return g_opt_ln_bwd_mode.load(); }
int attn_fwd_mode() { return g_opt_attn_fwd_mode.load(); }
int gemm_occ_mode() { return g_opt_gemm_occ.load(); }
int gemm_grid_mode() { return g_opt_gemm_grid.load(); }
int gemm_force_bn() { return g_opt_gemm_bn.load(); }
int attn_bwd_mode() { return g_opt_attn_bwd_mode.load(); }
int gemm_epi_warps_mode() { return g_opt_gemm_ew.load(); }
int attn_fwd_exf() { return g_opt_attn_fwd_exf.load(); }
int gemm_l2_hints() { return g_opt_gemm_l2.load(); }
int gemm_pick_mode() { return g_opt_gemm_pick.load(); }

}  // namespace bp

extern "C" {

int bp_abi_version(void) { return BP_ABI_VERSION; }

const char* bp_last_error(void) { return bp::g_err; }

int bp_sm_count(int device) {
  int n = 0;
  cudaError_t e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return -bp::cuda_status(e, "cudaDeviceGetAttribute");
  return n;
}

int bp_tc_available(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}

unsigned long long bp_launch_count(void) { return bp::g_launches.load(); }

int bp_set_option(int option, int value) {
  switch (option) {
    case BP_OPT_ATTN_EXACT: bp::g_opt_attn_exact.store(value); return BP_OK;
    case BP_OPT_GEMM_SIMT: bp::g_opt_gemm_simt.store(value); return BP_OK;
    case BP_OPT_GEMM_MODE: bp::g_opt_gemm_mode.store(value); return BP_OK;
    case BP_OPT_STREAM_K: bp::g_opt_stream_k.store(value); return BP_OK;
    case BP_OPT_GEMM_WIDE: bp::g_opt_gemm_wide.store(value); return BP_OK;
    case BP_OPT_GEMM_DEBUG: bp::g_opt_gemm_debug.store(value); return BP_OK;
    case BP_OPT_GEMM_TMA_STORE: bp::g_opt_gemm_tma_store.store(value); return BP_OK;
    case BP_OPT_LN_UNFUSED: bp::g_opt_ln_unfused.store(value); return BP_OK;
    case BP_OPT_LN_CTAS_PER_SM:
      if (value < 1 || value > 8) return BP_ERR_INVALID;
      bp::g_opt_ln_cps.store(value);
      return BP_OK;
    case BP_OPT_LN_BWD_MODE: bp::g_opt_ln_bwd_mode.store(value); return BP_OK;
    case BP_OPT_ATTN_FWD_MODE: bp::g_opt_attn_fwd_mode.store(value); return BP_OK;
    case BP_OPT_GEMM_OCC: bp::g_opt_gemm_occ.store(value); return BP_OK;
    case BP_OPT_GEMM_GRID: bp::g_opt_gemm_grid.store(value); return BP_OK;
    case BP_OPT_ATTN_BWD_MODE: bp::g_opt_attn_bwd_mode.store(value); return BP_OK;
    case BP_OPT_ATTN_FWD_EXF:
      if (value != 0 && (value < 2 || value > 8)) {
        bp::set_error("bp_set_option: attention forward FMA-pipe exponential mode must be 0 (default) or 2..8");
        return BP_ERR_INVALID;
      }
      bp::g_opt_attn_fwd_exf.store(value);
      return BP_OK;
    case BP_OPT_GEMM_L2_HINTS: bp::g_opt_gemm_l2.store(value); return BP_OK;
    case BP_OPT_GEMM_PICK: bp::g_opt_gemm_pick.store(value); return BP_OK;
    case BP_OPT_GEMM_EPI_WARPS:
      if (value != 0 && value != 4 && value != 8) {
        bp::set_error("bp_set_option: GEMM epilogue warps must be 0 (auto), 4 or 8");
        return BP_ERR_INVALID;
      }
      bp::g_opt_gemm_ew.store(value);
      return BP_OK;
    case BP_OPT_GEMM_BN:
      if (value != 0 && value != 128 && value != 192 && value != 224 && value != 256 && value != 512) {
        bp::set_error("bp_set_option: GEMM pair-tile width must be 0, 128, 192, 224, 256 or 512");
        return BP_ERR_INVALID;
      }
      bp::g_opt_gemm_bn.store(value);
      return BP_OK;
    default: bp::set_error("bp_set_option: unknown option %d", option); return BP_ERR_INVALID;
  }
}

}  // extern "C"
