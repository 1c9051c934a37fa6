// LayerNorm forward/backward -- HBM-bound.
//
// Fast path (bf16 or fp32, cols % (32*VEC) == 0, cols <= 4096): one warp per
// row, the row held in registers as packed 16-byte vectors, two-pass mean /
// variance from registers, warp-shuffle reductions.  dgamma/dbeta are
// column sums over rows: a coalesced column kernel (thread per column,
// row chunks spread over the GPU, one fp32 atomicAdd per chunk).
// Generic path (any shape): block per row.
#include "common.cuh"

namespace bp {
void count_launch();
int num_sms();
bool ln_bwd_unfused();
int ln_ctas_per_sm();
int ln_bwd_mode();
template <typename T, int MODE>
int launch_colred(int rows, int cols, const void* a, int64_t lda, const void* x, const float* mean, const float* rstd,
                  float* out0, float* out1, cudaStream_t st);

template <typename T>
struct Vec;  // 16-byte vector of T
template <>
struct Vec<float> {
  static constexpr int N = 4;
  using U = float4;
  BP_DEV static void unpack(const U& u, float* f) { f[0] = u.x; f[1] = u.y; f[2] = u.z; f[3] = u.w; }
  BP_DEV static U pack(const float* f) { return make_float4(f[0], f[1], f[2], f[3]); }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  using U = uint4;
  BP_DEV static void unpack(const U& u, float* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 t = __bfloat1622float2(h[j]);
      f[2 * j] = t.x;
      f[2 * j + 1] = t.y;
    }
  }
  BP_DEV static U pack(const float* f) {
    U u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
    return u;
  }
};

// ------------------------------------------------------------ fast path --
template <typename T, int NV>  // NV vectors per lane; cols = 32 * NV * Vec::N
__global__ void __launch_bounds__(256) ln_fwd_warp(int rows, const T* __restrict__ x, const T* __restrict__ g,
                                                   const T* __restrict__ b, float eps, T* __restrict__ y,
                                                   float* __restrict__ mean, float* __restrict__ rstd) {
  using V = Vec<T>;
  constexpr int E = V::N;
  constexpr int cols = 32 * NV * E;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const typename V::U* xr = reinterpret_cast<const typename V::U*>(x + (int64_t)row * cols);
  const typename V::U* gr = reinterpret_cast<const typename V::U*>(g);
  const typename V::U* br = reinterpret_cast<const typename V::U*>(b);
  // gamma / beta are requested together with the row so their latency hides
  // behind the reductions; E independent partial sums per lane instead of
  // one 64-long dependent add chain
  typename V::U pv[NV], pg[NV], pb[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) pv[i] = xr[i * 32 + lane];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    pg[i] = gr[i * 32 + lane];
    pb[i] = br[i * 32 + lane];
  }
  float sp[E] = {};
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float t[E];
    V::unpack(pv[i], t);
#pragma unroll
    for (int j = 0; j < E; ++j) sp[j] += t[j];
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < E; ++j) s += sp[j];
  const float mu = warp_sum(s) * (1.f / cols);
#pragma unroll
  for (int j = 0; j < E; ++j) sp[j] = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float t[E];
    V::unpack(pv[i], t);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const float d = t[j] - mu;
      sp[j] = fmaf(d, d, sp[j]);
    }
  }
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < E; ++j) q += sp[j];
  const float rs = rsqrtf(warp_sum(q) * (1.f / cols) + eps);
  typename V::U* yr = reinterpret_cast<typename V::U*>(y + (int64_t)row * cols);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float gg[E], bb[E], o[E], t[E];
    V::unpack(pv[i], t);
    V::unpack(pg[i], gg);
    V::unpack(pb[i], bb);
#pragma unroll
    for (int j = 0; j < E; ++j) o[j] = (t[j] - mu) * rs * gg[j] + bb[j];
    yr[i * 32 + lane] = V::pack(o);
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

template <typename T, int NV>
__global__ void __launch_bounds__(256) ln_bwd_warp(int rows, const T* __restrict__ dy, const T* __restrict__ x,
                                                   const T* __restrict__ g, const float* __restrict__ mean,
                                                   const float* __restrict__ rstd, const T* __restrict__ dres,
                                                   T* __restrict__ dx) {
  // dx only; dgamma/dbeta come from the coalesced column kernel below.
  using V = Vec<T>;
  using U = typename V::U;
  constexpr int E = V::N;
  constexpr int cols = 32 * NV * E;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const U* dyr = reinterpret_cast<const U*>(dy + (int64_t)row * cols);
  const U* xr = reinterpret_cast<const U*>(x + (int64_t)row * cols);
  const U* gr = reinterpret_cast<const U*>(g);
  const float mu = mean[row], rs = rstd[row];
  U pa[NV], pd[NV], pg[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    pa[i] = xr[i * 32 + lane];
    pd[i] = dyr[i * 32 + lane];
    pg[i] = gr[i * 32 + lane];
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float a[E], d[E], gg[E];
    V::unpack(pa[i], a);
    V::unpack(pd[i], d);
    V::unpack(pg[i], gg);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const float dh = d[j] * gg[j];
      s1 += dh;
      s2 += dh * (a[j] - mu) * rs;
    }
  }
  s1 = warp_sum(s1) * (1.f / cols);
  s2 = warp_sum(s2) * (1.f / cols);
  U* dxr = reinterpret_cast<U*>(dx + (int64_t)row * cols);
  const U* rr = dres ? reinterpret_cast<const U*>(dres + (int64_t)row * cols) : nullptr;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float a[E], d[E], gg[E], r[E], o[E];
    V::unpack(pa[i], a);
    V::unpack(pd[i], d);
    V::unpack(pg[i], gg);
    if (rr) V::unpack(rr[i * 32 + lane], r);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const float xh = (a[j] - mu) * rs;
      o[j] = rs * (d[j] * gg[j] - s1 - xh * s2) + (rr ? r[j] : 0.f);
    }
    dxr[i * 32 + lane] = V::pack(o);
  }
}

// Fused backward: dx, dgamma, dbeta and (optionally) the column sum of dx
// in one launch.  A CTA owns a contiguous run of rows and all columns.
// Phase 1 (warp per row): the two row reductions (mean of dy*g and of
// dy*g*xhat) into shared memory.  Phase 2 (thread per 16-byte column
// vector): walk the rows, write dx and accumulate the column sums in
// registers; one fp32 atomicAdd per column and output at the end.  The
// phase-2 re-read of dy / x hits L2 (the CTA's rows were just read).
// The column sum of dx is the bias gradient of the preceding half-block's
// output projection (its output gradient IS this dx), taken over the
// values as stored.
// RG row groups of 32*NV threads: phase 2 runs RG rows at a time, so a
// CTA of rows finishes in ~2 memory round trips instead of rows_per.
template <typename T, int NV, int RG>
__global__ void __launch_bounds__(32 * NV * RG) ln_bwd_fused(int rows, int rows_per, const T* __restrict__ dy,
                                                             const T* __restrict__ x, const T* __restrict__ g,
                                                             const float* __restrict__ mean,
                                                             const float* __restrict__ rstd,
                                                             const T* __restrict__ dres, T* __restrict__ dx,
                                                             float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                             float* __restrict__ dxsum) {
  using V = Vec<T>;
  using U = typename V::U;
  constexpr int E = V::N;
  constexpr int nvec = 32 * NV;  // 16-byte vectors per row
  constexpr int cols = nvec * E;
  constexpr int NW = NV * RG;    // warps per CTA
  extern __shared__ float sstat[];  // [rows_per][4]: s1, s2, mu, rs; then [RG-1][3][cols] partials
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * rows_per, r1 = min(rows, r0 + rows_per);
  const U* DY = reinterpret_cast<const U*>(dy);
  const U* X = reinterpret_cast<const U*>(x);
  const U* G = reinterpret_cast<const U*>(g);
  for (int r = r0 + warp; r < r1; r += NW) {
    const float mu = mean[r], rs = rstd[r];
    constexpr int CH = NV < 8 ? NV : 8;  // vectors in flight per lane
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i0 = 0; i0 < NV; i0 += CH) {
      U pa[CH], pd[CH], pg[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        pa[i] = X[(int64_t)r * nvec + (i0 + i) * 32 + lane];
        pd[i] = DY[(int64_t)r * nvec + (i0 + i) * 32 + lane];
        pg[i] = G[(i0 + i) * 32 + lane];
      }
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        float a[E], d[E], gg[E];
        V::unpack(pa[i], a);
        V::unpack(pd[i], d);
        V::unpack(pg[i], gg);
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const float dh = d[j] * gg[j];
          s1 += dh;
          s2 += dh * (a[j] - mu) * rs;
        }
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      float* q = sstat + 4 * (r - r0);
      q[0] = s1 * (1.f / cols);
      q[1] = s2 * (1.f / cols);
      q[2] = mu;
      q[3] = rs;
    }
  }
  __syncthreads();
  const int t = threadIdx.x % nvec, rg = threadIdx.x / nvec;
  float gg[E], sg[E] = {}, sb[E] = {}, sx[E] = {};
  V::unpack(G[t], gg);
  const U* R = reinterpret_cast<const U*>(dres);
  U* DX = reinterpret_cast<U*>(dx);
  constexpr int UR = 4;  // rows in flight per thread
  for (int rb = r0 + rg; rb < r1; rb += UR * RG) {
    U pd[UR], pa[UR], pr[UR];
#pragma unroll
    for (int k = 0; k < UR; ++k) {
      const int r = rb + k * RG;
      if (r < r1) {
        pd[k] = DY[(int64_t)r * nvec + t];
        pa[k] = X[(int64_t)r * nvec + t];
        if (R) pr[k] = R[(int64_t)r * nvec + t];
      }
    }
#pragma unroll
    for (int k = 0; k < UR; ++k) {
      const int r = rb + k * RG;
      if (r >= r1) break;
      const float* q = sstat + 4 * (r - r0);
      const float s1 = q[0], s2 = q[1], mu = q[2], rs = q[3];
      float a[E], d[E], rr[E], o[E];
      V::unpack(pa[k], a);
      V::unpack(pd[k], d);
      if (R) V::unpack(pr[k], rr);
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const float xh = (a[j] - mu) * rs;
        o[j] = rs * (d[j] * gg[j] - s1 - xh * s2) + (R ? rr[j] : 0.f);
        sg[j] += d[j] * xh;
        sb[j] += d[j];
      }
      const U packed = V::pack(o);
      DX[(int64_t)r * nvec + t] = packed;
      if (dxsum) {
        V::unpack(packed, o);  // as stored
#pragma unroll
        for (int j = 0; j < E; ++j) sx[j] += o[j];
      }
    }
  }
  if (r0 >= r1) return;
  // row groups 1..RG-1 hand their partials to group 0 through shared memory
  if (RG > 1) {
    float* part = sstat + 4 * rows_per;
    if (rg > 0) {
      float* my = part + (rg - 1) * 3 * cols;
#pragma unroll
      for (int j = 0; j < E; ++j) {
        my[t * E + j] = sg[j];
        my[cols + t * E + j] = sb[j];
        my[2 * cols + t * E + j] = sx[j];
      }
    }
    __syncthreads();
    if (rg > 0) return;
#pragma unroll
    for (int o = 0; o < RG - 1; ++o) {
      const float* pp = part + o * 3 * cols;
#pragma unroll
      for (int j = 0; j < E; ++j) {
        sg[j] += pp[t * E + j];
        sb[j] += pp[cols + t * E + j];
        sx[j] += pp[2 * cols + t * E + j];
      }
    }
  }
  // one 16-byte vector reduction per 4 columns and output
#pragma unroll
  for (int j = 0; j < E; j += 4) {
    const int c = t * E + j;
    if (dgamma) red_add_v4(dgamma + c, sg[j], sg[j + 1], sg[j + 2], sg[j + 3]);
    if (dbeta) red_add_v4(dbeta + c, sb[j], sb[j + 1], sb[j + 2], sb[j + 3]);
    if (dxsum) red_add_v4(dxsum + c, sx[j], sx[j + 1], sx[j + 2], sx[j + 3]);
  }
}

// Single-pass bf16 backward.  One CTA per SM owns a contiguous block of
// rows; thread 0 brings the block's x, dy and dres rows into shared memory
// with three 1-D bulk (TMA) copies issued at once, so the whole block is in
// flight from the first cycle.  Thread t then owns the 16-byte column vector
// t of every row: the two per-row dot products of all rows are reduced in one
// multi-value warp butterfly (31 shuffles for up to 16 rows) plus one
// cross-warp pass, dx is written straight from registers, and the dgamma /
// dbeta / dx column sums stay in registers and leave as one 16-byte vector
// reduction per 4 columns.  HBM traffic = read dy, x, dres + write dx.
template <int NT>
__global__ void __launch_bounds__(NT, 1) ln_bwd_tma(int rows, int rows_per, int rmax,
                                                   const __nv_bfloat16* __restrict__ dy,
                                                   const __nv_bfloat16* __restrict__ x,
                                                   const __nv_bfloat16* __restrict__ g,
                                                   const float* __restrict__ mean, const float* __restrict__ rstd,
                                                   const __nv_bfloat16* __restrict__ dres,
                                                   __nv_bfloat16* __restrict__ dx, float* __restrict__ dgamma,
                                                   float* __restrict__ dbeta, float* __restrict__ dxsum) {
  using V = Vec<__nv_bfloat16>;
  using U = uint4;
  constexpr int cols = NT * 8, NW = NT / 32;
  extern __shared__ __align__(128) uint8_t ln_smem[];  // [3][rmax][cols] bf16: x, dy, dres
  __shared__ __align__(8) uint64_t bar;
  __shared__ float red[NW][32];
  __shared__ float fin[32];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int r0 = blockIdx.x * rows_per, r1 = min(rows, r0 + rows_per);
  if (r0 >= r1) return;
  const U* SX = reinterpret_cast<const U*>(ln_smem);
  const U* SD = SX + (size_t)rmax * NT;
  const U* SR = SD + (size_t)rmax * NT;
  U* DX = reinterpret_cast<U*>(dx);
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  float gg[8];
  V::unpack(reinterpret_cast<const U*>(g)[t], gg);
  float sg[8] = {}, sb[8] = {}, sx[8] = {};
  uint32_t phase = 0;
  for (int rb = r0; rb < r1; rb += rmax) {
    const int nr = min(rmax, r1 - rb);
    if (t == 0) {
      if (rb != r0) fence_proxy_async_smem();  // generic reads of the last batch before async overwrite
      const uint32_t bytes = (uint32_t)nr * cols * 2;
      mbar_expect_tx(&bar, (dres ? 3u : 2u) * bytes);
      bulk_g2s((void*)SX, x + (int64_t)rb * cols, bytes, &bar);
      bulk_g2s((void*)SD, dy + (int64_t)rb * cols, bytes, &bar);
      if (dres) bulk_g2s((void*)SR, dres + (int64_t)rb * cols, bytes, &bar);
    }
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    float mu[16], rs[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      mu[k] = k < nr ? mean[rb + k] : 0.f;
      rs[k] = k < nr ? rstd[rb + k] : 0.f;
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < nr) {
        float a[8], d[8];
        V::unpack(SX[k * NT + t], a);
        V::unpack(SD[k * NT + t], d);
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float dh = d[j] * gg[j];
          s1 += dh;
          s2 += dh * (a[j] - mu[k]);
        }
        v[2 * k] = s1;
        v[2 * k + 1] = s2 * rs[k];
      }
    }
    // butterfly reduce-scatter: afterwards lane l holds the warp sum of value l
#pragma unroll
    for (int stage = 16; stage >= 1; stage >>= 1) {
      const bool up = (lane & stage) != 0;
#pragma unroll
      for (int i = 0; i < stage; ++i) {
        const float send = up ? v[i] : v[i + stage];
        const float keep = up ? v[i + stage] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, stage);
      }
    }
    red[warp][lane] = v[0];
    __syncthreads();
    if (t < 32) {
      float a = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) a += red[w][t];
      fin[t] = a * (1.f / cols);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < nr) {
        const float s1 = fin[2 * k], s2 = fin[2 * k + 1];
        float a[8], d[8], rr[8], o[8];
        V::unpack(SX[k * NT + t], a);
        V::unpack(SD[k * NT + t], d);
        if (dres) V::unpack(SR[k * NT + t], rr);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (a[j] - mu[k]) * rs[k];
          o[j] = rs[k] * (d[j] * gg[j] - s1 - xh * s2) + (dres ? rr[j] : 0.f);
          sg[j] += d[j] * xh;
          sb[j] += d[j];
        }
        const U packed = V::pack(o);
        DX[(int64_t)(rb + k) * NT + t] = packed;
        if (dxsum) {
          V::unpack(packed, o);  // as stored
#pragma unroll
          for (int j = 0; j < 8; ++j) sx[j] += o[j];
        }
      }
    }
    __syncthreads();  // shared rows / red / fin are reused by the next row batch
  }
#pragma unroll
  for (int j = 0; j < 8; j += 4) {
    const int c = t * 8 + j;
    if (dgamma) red_add_v4(dgamma + c, sg[j], sg[j + 1], sg[j + 2], sg[j + 3]);
    if (dbeta) red_add_v4(dbeta + c, sb[j], sb[j + 1], sb[j + 2], sb[j + 3]);
    if (dxsum) red_add_v4(dxsum + c, sx[j], sx[j + 1], sx[j + 2], sx[j + 3]);
  }
}

template <int NT>
static int launch_ln_bwd_tma(int rows, const void* dy, const void* x, const void* g, const float* mean,
                             const float* rstd, const void* dres, void* dx, float* dgamma, float* dbeta, float* dxsum,
                             cudaStream_t st) {
  constexpr int cols = NT * 8;
  int rmax = 196608 / (6 * cols);
  if (rmax > 16) rmax = 16;
  const int rows_per = (rows + num_sms() - 1) / num_sms();
  const int grid = (rows + rows_per - 1) / rows_per;
  const size_t smem = (size_t)3 * rmax * cols * 2;
  static bool attr = false;
  if (!attr) {
    BP_CUDA(cudaFuncSetAttribute(ln_bwd_tma<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  ln_bwd_tma<NT><<<grid, NT, smem, st>>>(rows, rows_per, rmax, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x,
                                         (const __nv_bfloat16*)g, mean, rstd, (const __nv_bfloat16*)dres,
                                         (__nv_bfloat16*)dx, dgamma, dbeta, dxsum);
  count_launch();
  BP_CHECK_LAUNCH("ln_bwd_tma");
  return BP_OK;
}

// ---------------------------------------------------------- generic path --
template <typename T>
__global__ void ln_fwd_generic(int cols, const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b,
                               float eps, T* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd) {
  const int row = blockIdx.x;
  const T* xr = x + (int64_t)row * cols;
  __shared__ float sh[32];
  __shared__ float stat;
  float s = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) s += to_f<T>(xr[c]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    stat = t / cols;
  }
  __syncthreads();
  const float mu = stat;
  float q = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    float d = to_f<T>(xr[c]) - mu;
    q += d * d;
  }
  q = warp_sum(q);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    stat = rsqrtf(t / cols + eps);
    mean[row] = mu;
    rstd[row] = stat;
  }
  __syncthreads();
  const float rs = stat;
  for (int c = threadIdx.x; c < cols; c += blockDim.x)
    y[(int64_t)row * cols + c] = from_f<T>((to_f<T>(xr[c]) - mu) * rs * to_f<T>(g[c]) + to_f<T>(b[c]));
}

template <typename T>
__global__ void ln_bwd_generic_dx(int cols, const T* __restrict__ dy, const T* __restrict__ x,
                                  const T* __restrict__ g, const float* __restrict__ mean,
                                  const float* __restrict__ rstd, const T* __restrict__ dres, T* __restrict__ dx) {
  const int row = blockIdx.x;
  const float mu = mean[row], rs = rstd[row];
  const T* xr = x + (int64_t)row * cols;
  const T* dr = dy + (int64_t)row * cols;
  __shared__ float sh1[32], sh2[32];
  __shared__ float m1, m2;
  float s1 = 0.f, s2 = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    float xh = (to_f<T>(xr[c]) - mu) * rs;
    float dh = to_f<T>(dr[c]) * to_f<T>(g[c]);
    s1 += dh;
    s2 += dh * xh;
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if ((threadIdx.x & 31) == 0) {
    sh1[threadIdx.x >> 5] = s1;
    sh2[threadIdx.x >> 5] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += sh1[w];
      b += sh2[w];
    }
    m1 = a / cols;
    m2 = b / cols;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    float xh = (to_f<T>(xr[c]) - mu) * rs;
    float dh = to_f<T>(dr[c]) * to_f<T>(g[c]);
    float o = rs * (dh - m1 - xh * m2);
    if (dres) o += to_f<T>(dres[(int64_t)row * cols + c]);
    dx[(int64_t)row * cols + c] = from_f<T>(o);
  }
}

// dgamma[c] += sum_r dy*xhat ; dbeta[c] += sum_r dy.  grid.x over columns,
// grid.y over row chunks.
template <typename T>
__global__ void ln_bwd_generic_params(int rows, int cols, int rows_per, const T* __restrict__ dy,
                                      const T* __restrict__ x, const float* __restrict__ mean,
                                      const float* __restrict__ rstd, float* __restrict__ dgamma,
                                      float* __restrict__ dbeta) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int r0 = blockIdx.y * rows_per, r1 = min(rows, r0 + rows_per);
  float a = 0.f, b = 0.f;
  for (int r = r0; r < r1; ++r) {
    float d = to_f<T>(dy[(int64_t)r * cols + c]);
    a += d * (to_f<T>(x[(int64_t)r * cols + c]) - mean[r]) * rstd[r];
    b += d;
  }
  atomicAdd(&dgamma[c], a);
  atomicAdd(&dbeta[c], b);
}

template <typename T>
static int ln_fwd_t(int rows, int cols, const void* x, const void* g, const void* b, float eps, void* y, float* mean,
                    float* rstd, cudaStream_t st) {
  constexpr int E = Vec<T>::N;
  const int nv = cols % (32 * E) == 0 ? cols / (32 * E) : 0;
  const dim3 grid((rows + 7) / 8);
  const T *X = (const T*)x, *G = (const T*)g, *Bb = (const T*)b;
  T* Y = (T*)y;
  switch (nv) {
#define BP_LNF(n) \
  case n: ln_fwd_warp<T, n><<<grid, 256, 0, st>>>(rows, X, G, Bb, eps, Y, mean, rstd); break;
    BP_LNF(1) BP_LNF(2) BP_LNF(3) BP_LNF(4) BP_LNF(5) BP_LNF(6) BP_LNF(8) BP_LNF(12) BP_LNF(16)
#undef BP_LNF
    default: ln_fwd_generic<T><<<rows, 256, 0, st>>>(cols, X, G, Bb, eps, Y, mean, rstd);
  }
  count_launch();
  BP_CHECK_LAUNCH("ln_fwd");
  return BP_OK;
}

template <typename T>
static int ln_bwd_t(int rows, int cols, const void* dy, const void* x, const void* g, const float* mean,
                    const float* rstd, const void* dres, void* dx, float* dgamma, float* dbeta, float* dxsum,
                    cudaStream_t st) {
  constexpr int E = Vec<T>::N;
  const bool al = ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) |
                    reinterpret_cast<uintptr_t>(dres) | reinterpret_cast<uintptr_t>(dx) |
                    reinterpret_cast<uintptr_t>(dgamma) | reinterpret_cast<uintptr_t>(dbeta) |
                    reinterpret_cast<uintptr_t>(dxsum)) & 15) == 0;
  if (sizeof(T) == 2 && al && !ln_bwd_unfused() && ln_bwd_mode() == 1) {
    switch (cols) {
      case 1024: return launch_ln_bwd_tma<128>(rows, dy, x, g, mean, rstd, dres, dx, dgamma, dbeta, dxsum, st);
      case 2048: return launch_ln_bwd_tma<256>(rows, dy, x, g, mean, rstd, dres, dx, dgamma, dbeta, dxsum, st);
      case 4096: return launch_ln_bwd_tma<512>(rows, dy, x, g, mean, rstd, dres, dx, dgamma, dbeta, dxsum, st);
      default: break;
    }
  }
  const int nvf = cols % (32 * E) == 0 ? cols / (32 * E) : 0;
  if (al && (nvf == 1 || nvf == 2 || nvf == 4 || nvf == 8 || nvf == 16) && !ln_bwd_unfused()) {
    // one CTA of rows per SM; fewer CTAs = fewer column reductions at the end
    const int cps = ln_ctas_per_sm();
    int rows_per = (rows + cps * num_sms() - 1) / (cps * num_sms());
    if (rows_per < 4) rows_per = 4;
    const int grid = (rows + rows_per - 1) / rows_per;
    const T *DYp = (const T*)dy, *Xp = (const T*)x, *Gp = (const T*)g, *Rp = (const T*)dres;
    T* DXp = (T*)dx;
    switch (nvf) {
#define BP_LNBF(n, rg)                                                                                    \
  case n: {                                                                                               \
    const size_t smem = 16 * (size_t)rows_per + 12 * (size_t)cols * (rg - 1);                            \
    if (smem > 48 * 1024)                                                                                 \
      BP_CUDA(cudaFuncSetAttribute(ln_bwd_fused<T, n, rg>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                   (int)smem));                                                           \
    ln_bwd_fused<T, n, rg><<<grid, 32 * n * rg, smem, st>>>(rows, rows_per, DYp, Xp, Gp, mean, rstd, Rp, \
                                                            DXp, dgamma, dbeta, dxsum);                   \
    break;                                                                                                \
  }
      BP_LNBF(1, 4) BP_LNBF(2, 4) BP_LNBF(4, 4) BP_LNBF(8, 2) BP_LNBF(16, 1)
#undef BP_LNBF
    }
    count_launch();
    BP_CHECK_LAUNCH("ln_bwd_fused");
    return BP_OK;
  }
  const int nv = cols % (32 * E) == 0 ? cols / (32 * E) : 0;
  const T *DY = (const T*)dy, *X = (const T*)x, *G = (const T*)g, *R = (const T*)dres;
  T* DX = (T*)dx;
  switch (nv) {
#define BP_LNB(n)                                                                                       \
  case n:                                                                                               \
    ln_bwd_warp<T, n><<<(rows + 7) / 8, 256, 0, st>>>(rows, DY, X, G, mean, rstd, R, DX);             \
    break;
    BP_LNB(1) BP_LNB(2) BP_LNB(3) BP_LNB(4) BP_LNB(5) BP_LNB(6) BP_LNB(8) BP_LNB(12) BP_LNB(16)
#undef BP_LNB
    default:
      ln_bwd_generic_dx<T><<<rows, 256, 0, st>>>(cols, DY, X, G, mean, rstd, R, DX);
  }
  count_launch();
  BP_CHECK_LAUNCH("ln_bwd_dx");
  if (int rc = launch_colred<T, 1>(rows, cols, dy, cols, x, mean, rstd, dgamma, dbeta, st)) return rc;
  if (dxsum) return launch_colred<T, 0>(rows, cols, dx, cols, nullptr, nullptr, nullptr, dxsum, nullptr, st);
  return BP_OK;
}

}  // namespace bp

using namespace bp;

extern "C" int bp_layernorm_fwd(int dtype, int rows, int cols, const void* x, const void* gamma, const void* beta,
                                float eps, void* y, float* mean, float* rstd, void* stream) {
  if (rows <= 0 || cols <= 0) {
    set_error("layernorm_fwd: bad shape");
    return BP_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == BP_F32 ? ln_fwd_t<float>(rows, cols, x, gamma, beta, eps, y, mean, rstd, st)
                         : ln_fwd_t<__nv_bfloat16>(rows, cols, x, gamma, beta, eps, y, mean, rstd, st);
}

extern "C" int bp_layernorm_bwd_ex(int dtype, int rows, int cols, const void* dy, const void* x, const void* gamma,
                                   const float* mean, const float* rstd, const void* dres, void* dx, float* dgamma,
                                   float* dbeta, float* dx_colsum, void* stream) {
  if (rows <= 0 || cols <= 0) {
    set_error("layernorm_bwd: bad shape");
    return BP_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == BP_F32
             ? ln_bwd_t<float>(rows, cols, dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, dx_colsum, st)
             : ln_bwd_t<__nv_bfloat16>(rows, cols, dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, dx_colsum, st);
}

extern "C" int bp_layernorm_bwd(int dtype, int rows, int cols, const void* dy, const void* x, const void* gamma,
                                const float* mean, const float* rstd, const void* dres, void* dx, float* dgamma,
                                float* dbeta, void* stream) {
  return bp_layernorm_bwd_ex(dtype, rows, cols, dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, nullptr, stream);
}
