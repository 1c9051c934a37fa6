// Multi-head attention forward / backward.
//
// Two implementations behind bp_attn_fwd / bp_attn_bwd:
//   * flash path (bf16, Dh in {64,128}): FlashAttention-2 style tiles with
//     online softmax, tensor-core mma.sync m16n8k16 (see attention_flash.cuh);
//   * exact path (fp32 check mode, or any shape): one warp per query row,
//     online softmax in fp32, fp32 atomics for dK/dV.  Used for the 1e-4
//     parity mode and as the cross-check of the flash path in tests.
// Layout: qkv [B*S, 3*H*Dh] (q heads | k heads | v heads), o [B*S, H*Dh],
// lse [B*H*S] (natural-log logsumexp of the scaled scores).
#include "common.cuh"

namespace bp {
void count_launch();
int num_sms();
int attn_flash_fwd(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, void* o, float* lse,
                   cudaStream_t st);
int attn_flash_bwd(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, const void* o,
                   const void* dout, const float* lse, void* dqkv, float* ws, cudaStream_t st);
bool attn_flash_supported(int dtype, int S, int Dh);
bool attn_tc_supported(int dtype, int S, int Dh);
int attn_tc_fwd(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, void* o, float* lse,
                cudaStream_t st);
int attn_tc_bwd(int B, int S, int H, int Dh, int causal, float scale, float* dbias, const void* qkv, const void* o,
                const void* dout, const float* lse, void* dqkv, float* ws, cudaStream_t st);

constexpr int kMaxDhPerLane = 4;  // Dh <= 128

template <typename T>
__global__ void attn_fwd_exact(int B, int S, int H, int Dh, int causal, float scale, const T* __restrict__ qkv,
                               T* __restrict__ o, float* __restrict__ lse) {
  const int warp_global = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (warp_global >= B * H * S) return;
  const int i = warp_global % S;
  const int h = (warp_global / S) % H;
  const int b = warp_global / (S * H);
  const int64_t ld = 3LL * H * Dh;
  const T* qrow = qkv + ((int64_t)b * S + i) * ld + h * Dh;
  float q[kMaxDhPerLane], acc[kMaxDhPerLane];
  const int per = (Dh + 31) / 32;
  for (int t = 0; t < per; ++t) {
    const int d = lane + 32 * t;
    q[t] = d < Dh ? to_f<T>(qrow[d]) * scale : 0.f;
    acc[t] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const int jend = causal ? i + 1 : S;
  for (int j = 0; j < jend; ++j) {
    const T* krow = qkv + ((int64_t)b * S + j) * ld + (int64_t)H * Dh + h * Dh;
    const T* vrow = krow + (int64_t)H * Dh;
    float s = 0.f;
    for (int t = 0; t < per; ++t) {
      const int d = lane + 32 * t;
      if (d < Dh) s += q[t] * to_f<T>(krow[d]);
    }
    s = warp_sum(s);
    const float mn = fmaxf(m, s);
    const float corr = __expf(m - mn);
    const float p = __expf(s - mn);
    l = l * corr + p;
    for (int t = 0; t < per; ++t) {
      const int d = lane + 32 * t;
      acc[t] = acc[t] * corr + (d < Dh ? p * to_f<T>(vrow[d]) : 0.f);
    }
    m = mn;
  }
  T* orow = o + ((int64_t)b * S + i) * H * Dh + h * Dh;
  for (int t = 0; t < per; ++t) {
    const int d = lane + 32 * t;
    if (d < Dh) orow[d] = from_f<T>(acc[t] / l);
  }
  if (lane == 0) lse[((int64_t)b * H + h) * S + i] = m + logf(l);
}

// delta[b,h,i] = sum_d dO[i,d] * O[i,d]
template <typename T>
__global__ void attn_delta(int B, int S, int H, int Dh, const T* __restrict__ o, const T* __restrict__ dout,
                           float* __restrict__ delta) {
  const int warp_global = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (warp_global >= B * H * S) return;
  const int i = warp_global % S, h = (warp_global / S) % H, b = warp_global / (S * H);
  const int64_t off = ((int64_t)b * S + i) * H * Dh + h * Dh;
  float s = 0.f;
  for (int d = lane; d < Dh; d += 32) s += to_f<T>(o[off + d]) * to_f<T>(dout[off + d]);
  s = warp_sum(s);
  if (lane == 0) delta[((int64_t)b * H + h) * S + i] = s;
}

// One warp per query row i: dQ_i directly, dK_j / dV_j via fp32 atomics into
// ws_dk / ws_dv ([B*S, H*Dh] fp32 each).
template <typename T>
__global__ void attn_bwd_exact(int B, int S, int H, int Dh, int causal, float scale, const T* __restrict__ qkv,
                               const T* __restrict__ dout, const float* __restrict__ lse,
                               const float* __restrict__ delta, T* __restrict__ dqkv, float* __restrict__ ws_dk,
                               float* __restrict__ ws_dv) {
  const int warp_global = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (warp_global >= B * H * S) return;
  const int i = warp_global % S, h = (warp_global / S) % H, b = warp_global / (S * H);
  const int64_t ld = 3LL * H * Dh;
  const int64_t hd = (int64_t)H * Dh;
  const T* qrow = qkv + ((int64_t)b * S + i) * ld + h * Dh;
  const T* dorow = dout + ((int64_t)b * S + i) * hd + h * Dh;
  const int per = (Dh + 31) / 32;
  float q[kMaxDhPerLane], dO[kMaxDhPerLane], dq[kMaxDhPerLane];
  for (int t = 0; t < per; ++t) {
    const int d = lane + 32 * t;
    q[t] = d < Dh ? to_f<T>(qrow[d]) : 0.f;
    dO[t] = d < Dh ? to_f<T>(dorow[d]) : 0.f;
    dq[t] = 0.f;
  }
  const float L = lse[((int64_t)b * H + h) * S + i];
  const float dl = delta[((int64_t)b * H + h) * S + i];
  const int jend = causal ? i + 1 : S;
  for (int j = 0; j < jend; ++j) {
    const T* krow = qkv + ((int64_t)b * S + j) * ld + hd + h * Dh;
    const T* vrow = krow + hd;
    float s = 0.f, dp = 0.f;
    for (int t = 0; t < per; ++t) {
      const int d = lane + 32 * t;
      if (d < Dh) {
        s += q[t] * to_f<T>(krow[d]);
        dp += dO[t] * to_f<T>(vrow[d]);
      }
    }
    s = warp_sum(s) * scale;
    dp = warp_sum(dp);
    const float p = __expf(s - L);
    const float ds = p * (dp - dl);
    float* dkrow = ws_dk + ((int64_t)b * S + j) * hd + h * Dh;
    float* dvrow = ws_dv + ((int64_t)b * S + j) * hd + h * Dh;
    for (int t = 0; t < per; ++t) {
      const int d = lane + 32 * t;
      if (d < Dh) {
        dq[t] += ds * to_f<T>(krow[d]);
        atomicAdd(&dkrow[d], ds * q[t] * scale);
        atomicAdd(&dvrow[d], p * dO[t]);
      }
    }
  }
  T* dqrow = dqkv + ((int64_t)b * S + i) * ld + h * Dh;
  for (int t = 0; t < per; ++t) {
    const int d = lane + 32 * t;
    if (d < Dh) dqrow[d] = from_f<T>(dq[t] * scale);
  }
}

// dqkv[:, H*Dh + c] = ws_dk ; dqkv[:, 2*H*Dh + c] = ws_dv
template <typename T>
__global__ void attn_scatter_kv(int rows, int hd, const float* __restrict__ dk, const float* __restrict__ dv,
                                T* __restrict__ dqkv) {
  const int64_t n = (int64_t)rows * hd;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / hd, c = e % hd;
    dqkv[r * 3 * hd + hd + c] = from_f<T>(dk[e]);
    dqkv[r * 3 * hd + 2 * hd + c] = from_f<T>(dv[e]);
  }
}

template <typename T>
static int fwd_exact(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, void* o, float* lse,
                     cudaStream_t st) {
  const int warps = B * H * S;
  attn_fwd_exact<T><<<(warps + 7) / 8, 256, 0, st>>>(B, S, H, Dh, causal, scale, (const T*)qkv, (T*)o, lse);
  count_launch();
  BP_CHECK_LAUNCH("attn_fwd_exact");
  return BP_OK;
}

template <typename T>
static int bwd_exact(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, const void* o,
                     const void* dout, const float* lse, void* dqkv, float* ws, cudaStream_t st) {
  const int warps = B * H * S;
  const int64_t hd = (int64_t)H * Dh;
  float* delta = ws;
  float* dk = ws + (int64_t)B * H * S;
  float* dv = dk + (int64_t)B * S * hd;
  BP_CUDA(cudaMemsetAsync(dk, 0, sizeof(float) * 2 * (size_t)B * S * hd, st));
  attn_delta<T><<<(warps + 7) / 8, 256, 0, st>>>(B, S, H, Dh, (const T*)o, (const T*)dout, delta);
  attn_bwd_exact<T><<<(warps + 7) / 8, 256, 0, st>>>(B, S, H, Dh, causal, scale, (const T*)qkv, (const T*)dout, lse,
                                                     delta, (T*)dqkv, dk, dv);
  attn_scatter_kv<T><<<num_sms() * 4, 256, 0, st>>>(B * S, (int)hd, dk, dv, (T*)dqkv);
  count_launch();
  count_launch();
  count_launch();
  BP_CHECK_LAUNCH("attn_bwd_exact");
  return BP_OK;
}

}  // namespace bp

using namespace bp;

namespace bp {
// tcgen05 backward: dS^T (bf16 [B H][S][S]) after delta, 256-byte aligned
int64_t attn_ds_offset_floats(int B, int S, int H) { return ((int64_t)B * H * S + 63) / 64 * 64; }
}

extern "C" int64_t bp_attn_workspace_bytes(int B, int S, int H, int Dh) {
  // delta [B*H*S] + three fp32 [B*S, H*Dh] accumulators (dq/dk/dv, exact
  // path), or delta + the bf16 dS^T matrix of the tcgen05 path
  const int64_t exact = (int64_t)sizeof(float) * ((int64_t)B * H * S + 3LL * B * S * H * Dh);
  const int64_t tc = (int64_t)sizeof(float) * attn_ds_offset_floats(B, S, H) + 2LL * B * H * S * S;
  return exact > tc ? exact : tc;
}

static int attn_check(int B, int S, int H, int Dh) {
  if (B <= 0 || S <= 0 || H <= 0 || Dh <= 0 || Dh > 32 * kMaxDhPerLane) {
    set_error("attention: unsupported shape B=%d S=%d H=%d Dh=%d", B, S, H, Dh);
    return BP_ERR_UNSUPPORTED;
  }
  return BP_OK;
}

extern "C" int bp_attn_fwd(int dtype, int B, int S, int H, int Dh, int causal, float scale, const void* qkv, void* o,
                           float* lse, void* stream) {
  if (int rc = attn_check(B, S, H, Dh)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (attn_tc_supported(dtype, S, Dh)) return attn_tc_fwd(B, S, H, Dh, causal, scale, qkv, o, lse, st);
  if (attn_flash_supported(dtype, S, Dh)) return attn_flash_fwd(B, S, H, Dh, causal, scale, qkv, o, lse, st);
  return dtype == BP_F32 ? fwd_exact<float>(B, S, H, Dh, causal, scale, qkv, o, lse, st)
                         : fwd_exact<__nv_bfloat16>(B, S, H, Dh, causal, scale, qkv, o, lse, st);
}

extern "C" int bp_attn_bwd_ex(int dtype, int B, int S, int H, int Dh, int causal, float scale, const void* qkv,
                              const void* o, const void* dout, const float* lse, void* dqkv, float* workspace,
                              float* dbias, void* stream) {
  if (int rc = attn_check(B, S, H, Dh)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  // tcgen05 path: the QKV bias gradient is reduced in the dK/dV and dQ
  // kernels' epilogues; other paths take a column-reduction launch
  if (attn_tc_supported(dtype, S, Dh))
    return attn_tc_bwd(B, S, H, Dh, causal, scale, dbias, qkv, o, dout, lse, dqkv, workspace, st);
  int rc;
  if (attn_flash_supported(dtype, S, Dh))
    rc = attn_flash_bwd(B, S, H, Dh, causal, scale, qkv, o, dout, lse, dqkv, workspace, st);
  else
    rc = dtype == BP_F32 ? bwd_exact<float>(B, S, H, Dh, causal, scale, qkv, o, dout, lse, dqkv, workspace, st)
                         : bwd_exact<__nv_bfloat16>(B, S, H, Dh, causal, scale, qkv, o, dout, lse, dqkv, workspace, st);
  if (rc || !dbias) return rc;
  return bp_colsum_acc(dtype, B * S, 3 * H * Dh, dqkv, 3LL * H * Dh, dbias, stream);
}

extern "C" int bp_attn_bwd(int dtype, int B, int S, int H, int Dh, int causal, float scale, const void* qkv,
                           const void* o, const void* dout, const float* lse, void* dqkv, float* workspace,
                           void* stream) {
  return bp_attn_bwd_ex(dtype, B, S, H, Dh, causal, scale, qkv, o, dout, lse, dqkv, workspace, nullptr, stream);
}
