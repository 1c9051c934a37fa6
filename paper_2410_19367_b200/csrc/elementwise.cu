// Bandwidth kernels of the per-stage passes:
// bias-gradient column sums, embedding fwd/bwd, fused softmax
// cross-entropy fwd+bwd, dtype cast, fused replica-mean AdamW.
#include "common.cuh"

namespace bp {
void count_launch();
int num_sms();

// ------------------------------------------------------- column sums ----
// Column reductions over token rows, vectorised: a block is 32 x 8 threads;
// each thread owns 8 consecutive columns (one 16-byte bf16 vector / two
// fp32 vectors) and walks rows ty, ty+8, ... of the block's row chunk; the
// 8 row-groups are reduced in shared memory and each column gets one fp32
// atomicAdd per block.
//   MODE 0: out0[c] += sum_r x[r,c]
//   MODE 1: (LayerNorm parameters) out0[c] += sum_r dy*(x-mean_r)*rstd_r,
//                                  out1[c] += sum_r dy
template <typename T, int MODE>
__global__ void __launch_bounds__(256) colred_kernel(int rows, int cols, int rows_per, int vec, const T* __restrict__ a,
                                                     int64_t lda, const T* __restrict__ x, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, float* __restrict__ out0,
                                                     float* __restrict__ out1) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c0 = (blockIdx.x * 32 + tx) * 8;
  const int r0 = blockIdx.y * rows_per, r1 = min(rows, r0 + rows_per);
  float s0[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, s1[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const bool full = vec && c0 + 8 <= cols;
  auto load8 = [&](const T* p, float (&v)[8]) {
    if (full && sizeof(T) == 2) {
      const uint4 u = *reinterpret_cast<const uint4*>(p);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        v[2 * j] = f.x;
        v[2 * j + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (c0 + j < cols) ? to_f<T>(p[j]) : 0.f;
    }
  };
  if (c0 < cols) {
    // UR independent rows (8 apart) per iteration keep UR loads in flight
    constexpr int UR = 4;
    for (int rb = r0 + ty; rb < r1; rb += 8 * UR) {
      float v[UR][8], w[UR][8];
#pragma unroll
      for (int k = 0; k < UR; ++k) {
        const int r = rb + 8 * k;
        if (r < r1) {
          load8(a + (int64_t)r * lda + c0, v[k]);
          if (MODE == 1) load8(x + (int64_t)r * cols + c0, w[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < UR; ++k) {
        const int r = rb + 8 * k;
        if (r >= r1) continue;
        if (MODE == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j) s0[j] += v[k][j];
        } else {
          const float mu = mean[r], rs = rstd[r];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            s0[j] += v[k][j] * (w[k][j] - mu) * rs;
            s1[j] += v[k][j];
          }
        }
      }
    }
  }
  __shared__ float red[2][8][32 * 8 + 1];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    red[0][ty][tx * 8 + j] = s0[j];
    if (MODE == 1) red[1][ty][tx * 8 + j] = s1[j];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256 * (MODE + 1); i += 256) {
    const int which = i / 256, cc = i % 256;
    float t = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += red[which][y][cc];
    const int col = blockIdx.x * 256 + cc;
    if (col < cols) atomicAdd(which == 0 ? &out0[col] : &out1[col], t);
  }
}

template <typename T, int MODE>
int launch_colred(int rows, int cols, const void* a, int64_t lda, const void* x, const float* mean, const float* rstd,
                  float* out0, float* out1, cudaStream_t st) {
  const int cblocks = (cols + 255) / 256;
  int chunks = (2 * num_sms() + cblocks - 1) / cblocks;
  int rows_per = (rows + chunks - 1) / chunks;
  if (rows_per < 32) rows_per = 32;
  dim3 grid(cblocks, (rows + rows_per - 1) / rows_per);
  const int vec = (reinterpret_cast<uintptr_t>(a) % 16 == 0) && (lda % 8 == 0) &&
                  (!x || (reinterpret_cast<uintptr_t>(x) % 16 == 0 && cols % 8 == 0));
  colred_kernel<T, MODE><<<grid, 256, 0, st>>>(rows, cols, rows_per, vec, (const T*)a, lda, (const T*)x, mean, rstd,
                                               out0, out1);
  count_launch();
  BP_CHECK_LAUNCH("colred");
  return BP_OK;
}
template int launch_colred<float, 1>(int, int, const void*, int64_t, const void*, const float*, const float*,
                                     float*, float*, cudaStream_t);
template int launch_colred<float, 0>(int, int, const void*, int64_t, const void*, const float*, const float*,
                                     float*, float*, cudaStream_t);
template int launch_colred<__nv_bfloat16, 0>(int, int, const void*, int64_t, const void*, const float*,
                                             const float*, float*, float*, cudaStream_t);
template int launch_colred<__nv_bfloat16, 1>(int, int, const void*, int64_t, const void*, const float*,
                                             const float*, float*, float*, cudaStream_t);

// ------------------------------------------------------------- embed ----
template <typename T>
__global__ void embed_fwd_kernel(int B, int S, int H, const int32_t* __restrict__ tok, const T* __restrict__ wte,
                                 const T* __restrict__ wpe, T* __restrict__ out) {
  const int r = blockIdx.x;  // token row b*S + s
  const int s = r % S;
  const int64_t t = tok[r];
  for (int c = threadIdx.x; c < H; c += blockDim.x)
    out[(int64_t)r * H + c] = from_f<T>(to_f<T>(wte[t * H + c]) + to_f<T>(wpe[(int64_t)s * H + c]));
}

template <typename T>
__global__ void embed_bwd_tok_kernel(int H, const int32_t* __restrict__ tok, const T* __restrict__ dout,
                                     float* __restrict__ dwte) {
  const int r = blockIdx.x;
  const int64_t t = tok[r];
  for (int c = threadIdx.x; c < H; c += blockDim.x) atomicAdd(&dwte[t * H + c], to_f<T>(dout[(int64_t)r * H + c]));
}

template <typename T>
__global__ void embed_bwd_pos_kernel(int B, int S, int H, const T* __restrict__ dout, float* __restrict__ dwpe) {
  const int s = blockIdx.x;
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    float a = 0.f;
    for (int b = 0; b < B; ++b) a += to_f<T>(dout[((int64_t)b * S + s) * H + c]);
    dwpe[(int64_t)s * H + c] += a;
  }
}

// 16-byte vector variants (bf16, H % 8 == 0): thread = 8 columns of a row.
BP_DEV void unpack8(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}

__global__ void embed_fwd_vec(int S, int H8, const int32_t* __restrict__ tok, const uint4* __restrict__ wte,
                              const uint4* __restrict__ wpe, uint4* __restrict__ out) {
  const int r = blockIdx.x, s = r % S;
  const int64_t t = tok[r];
  for (int c = threadIdx.x; c < H8; c += blockDim.x) {
    float a[8], b[8];
    unpack8(wte[t * H8 + c], a);
    unpack8(wpe[(int64_t)s * H8 + c], b);
    uint4 o;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(a[2 * j] + b[2 * j], a[2 * j + 1] + b[2 * j + 1]);
    out[(int64_t)r * H8 + c] = o;
  }
}

__global__ void embed_bwd_tok_vec(int H8, const int32_t* __restrict__ tok, const uint4* __restrict__ dout,
                                  float* __restrict__ dwte) {
  const int r = blockIdx.x;
  const int64_t t = tok[r];
  for (int c = threadIdx.x; c < H8; c += blockDim.x) {
    float d[8];
    unpack8(dout[(int64_t)r * H8 + c], d);
    float* dst = dwte + (t * H8 + c) * 8;
    red_add_v4(dst, d[0], d[1], d[2], d[3]);
    red_add_v4(dst + 4, d[4], d[5], d[6], d[7]);
  }
}

__global__ void embed_bwd_pos_vec(int B, int S, int H8, const uint4* __restrict__ dout, float4* __restrict__ dwpe) {
  const int s = blockIdx.x;
  for (int c = threadIdx.x; c < H8; c += blockDim.x) {
    float acc[8] = {};
    for (int b = 0; b < B; ++b) {
      float d[8];
      unpack8(dout[((int64_t)b * S + s) * H8 + c], d);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += d[j];
    }
    float4* dst = dwpe + ((int64_t)s * H8 + c) * 2;
    float4 lo = dst[0], hi = dst[1];
    lo.x += acc[0]; lo.y += acc[1]; lo.z += acc[2]; lo.w += acc[3];
    hi.x += acc[4]; hi.y += acc[5]; hi.z += acc[6]; hi.w += acc[7];
    dst[0] = lo;
    dst[1] = hi;
  }
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// --------------------------------------------------------------- xent ----
// Block per row.  Pass 1: online max / sum-exp over 16-byte vectors.
// Pass 2: re-read (L2-resident), write the scaled gradient in place.
// Loss uses logsumexp - logit[target].
BP_DEV void lse_combine(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
  m = mm;
}

template <typename T>
__global__ void __launch_bounds__(512) xent_kernel(int V, T* __restrict__ logits, int64_t ld,
                                                   const int32_t* __restrict__ tgt, float grad_scale,
                                                   float loss_scale, float* __restrict__ loss, int vec) {
  const int r = blockIdx.x;
  T* row = logits + (int64_t)r * ld;
  constexpr int E = 16 / sizeof(T);
  const int nv = vec ? V / E : 0;
  float m = -INFINITY, s = 0.f;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const uint4 u = reinterpret_cast<const uint4*>(row)[i];
    const T* e = reinterpret_cast<const T*>(&u);
    float x[E], mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      x[j] = to_f<T>(e[j]);
      mx = fmaxf(mx, x[j]);
    }
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < E; ++j) t += __expf(x[j] - mx);
    lse_combine(m, s, mx, t);
  }
  for (int c = nv * E + threadIdx.x; c < V; c += blockDim.x) lse_combine(m, s, to_f<T>(row[c]), 1.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_combine(m, s, m2, s2);
  }
  __shared__ float sm[32], ss[32];
  __shared__ float g_lse;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[w] = m;
    ss[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY, S = 0.f;
    const int nw = blockDim.x >> 5;
    for (int i = 0; i < nw; ++i) lse_combine(M, S, sm[i], ss[i]);
    g_lse = M + logf(S);
    atomicAdd(loss, loss_scale * (g_lse - to_f<T>(row[tgt[r]])));
  }
  __syncthreads();
  const float lse = g_lse;
  const int t = tgt[r];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    uint4 u = reinterpret_cast<const uint4*>(row)[i];
    T* e = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int c = i * E + j;
      e[j] = from_f<T>((__expf(to_f<T>(e[j]) - lse) - (c == t ? 1.f : 0.f)) * grad_scale);
    }
    reinterpret_cast<uint4*>(row)[i] = u;
  }
  for (int c = nv * E + threadIdx.x; c < V; c += blockDim.x) {
    const float p = __expf(to_f<T>(row[c]) - lse);
    row[c] = from_f<T>((p - (c == t ? 1.f : 0.f)) * grad_scale);
  }
}

// --------------------------------------------------------------- cast ----
template <typename S, typename D>
__global__ void cast_kernel(int64_t n, const S* __restrict__ src, D* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = from_f<D>(to_f<S>(src[i]));
}

// --------------------------------------------------------------- adam ----
template <typename P>
__global__ void adam_kernel(int64_t n, float* __restrict__ master, const float* __restrict__ ga,
                            const float* __restrict__ gb, float* __restrict__ m, float* __restrict__ v,
                            P* __restrict__ pa, P* __restrict__ pb, float lr, float b1, float b2, float eps, float wd,
                            float bc1, float bc2, float gscale, const int* __restrict__ step_dev) {
  if (step_dev) {  // step counter in device memory (CUDA-graph replays advance it on the device)
    const float t = (float)*step_dev;
    bc1 = 1.f - powf(b1, t);
    bc2 = 1.f - powf(b2, t);
  }
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 g = reinterpret_cast<const float4*>(ga)[i];
    if (gb) {
      const float4 h = reinterpret_cast<const float4*>(gb)[i];
      g.x = (g.x + h.x) * 0.5f; g.y = (g.y + h.y) * 0.5f; g.z = (g.z + h.z) * 0.5f; g.w = (g.w + h.w) * 0.5f;
    }
    float4 w = reinterpret_cast<float4*>(master)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float gg[4] = {g.x, g.y, g.z, g.w}, ww[4] = {w.x, w.y, w.z, w.w};
    float m4[4] = {mm.x, mm.y, mm.z, mm.w}, v4[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float gj = gg[j] * gscale;
      m4[j] = b1 * m4[j] + (1.f - b1) * gj;
      v4[j] = b2 * v4[j] + (1.f - b2) * gj * gj;
      const float upd = (m4[j] / bc1) / (sqrtf(v4[j] / bc2) + eps) + wd * ww[j];
      ww[j] -= lr * upd;
    }
    reinterpret_cast<float4*>(master)[i] = make_float4(ww[0], ww[1], ww[2], ww[3]);
    reinterpret_cast<float4*>(m)[i] = make_float4(m4[0], m4[1], m4[2], m4[3]);
    reinterpret_cast<float4*>(v)[i] = make_float4(v4[0], v4[1], v4[2], v4[3]);
    if (sizeof(P) == 2) {  // 4 bf16 working-copy values = one 8-byte store per replica
      uint2 u;
      *reinterpret_cast<__nv_bfloat162*>(&u.x) = __floats2bfloat162_rn(ww[0], ww[1]);
      *reinterpret_cast<__nv_bfloat162*>(&u.y) = __floats2bfloat162_rn(ww[2], ww[3]);
      if (pa) reinterpret_cast<uint2*>(pa)[i] = u;
      if (pb) reinterpret_cast<uint2*>(pb)[i] = u;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (pa) pa[4 * i + j] = from_f<P>(ww[j]);
        if (pb) pb[4 * i + j] = from_f<P>(ww[j]);
      }
    }
  }
  // tail
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float g = ga[i];
    if (gb) g = (g + gb[i]) * 0.5f;
    g *= gscale;
    m[i] = b1 * m[i] + (1.f - b1) * g;
    v[i] = b2 * v[i] + (1.f - b2) * g * g;
    const float w = master[i] - lr * ((m[i] / bc1) / (sqrtf(v[i] / bc2) + eps) + wd * master[i]);
    master[i] = w;
    if (pa) pa[i] = from_f<P>(w);
    if (pb) pb[i] = from_f<P>(w);
  }
}

static int grid_for(int64_t n, int per_block) {
  int64_t g = (n + per_block - 1) / per_block;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace bp

using namespace bp;

extern "C" int bp_colsum_acc(int dtype, int rows, int cols, const void* x, int64_t ldx, float* out, void* stream) {
  if (rows <= 0 || cols <= 0) {
    set_error("colsum: bad shape");
    return BP_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == BP_F32
             ? launch_colred<float, 0>(rows, cols, x, ldx, nullptr, nullptr, nullptr, out, nullptr, st)
             : launch_colred<__nv_bfloat16, 0>(rows, cols, x, ldx, nullptr, nullptr, nullptr, out, nullptr, st);
}

extern "C" int bp_embed_fwd(int dtype, int B, int S, int H, const int32_t* tokens, const void* wte, const void* wpe,
                            void* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = H >= 256 ? 256 : 64;
  if (dtype == BP_BF16 && H % 8 == 0 && al16(wte) && al16(wpe) && al16(out)) {
    embed_fwd_vec<<<B * S, H / 8 >= 256 ? 256 : 64, 0, st>>>(S, H / 8, tokens, (const uint4*)wte, (const uint4*)wpe,
                                                              (uint4*)out);
  } else if (dtype == BP_F32)
    embed_fwd_kernel<float><<<B * S, threads, 0, st>>>(B, S, H, tokens, (const float*)wte, (const float*)wpe,
                                                        (float*)out);
  else
    embed_fwd_kernel<__nv_bfloat16><<<B * S, threads, 0, st>>>(B, S, H, tokens, (const __nv_bfloat16*)wte,
                                                                (const __nv_bfloat16*)wpe, (__nv_bfloat16*)out);
  count_launch();
  BP_CHECK_LAUNCH("embed_fwd");
  return BP_OK;
}

extern "C" int bp_embed_bwd(int dtype, int B, int S, int H, const int32_t* tokens, const void* dout, float* dwte,
                            float* dwpe, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = H >= 256 ? 256 : 64;
  if (dtype == BP_BF16 && H % 8 == 0 && al16(dout) && al16(dwte) && al16(dwpe)) {
    const int t8 = H / 8 >= 256 ? 256 : 64;
    embed_bwd_tok_vec<<<B * S, t8, 0, st>>>(H / 8, tokens, (const uint4*)dout, dwte);
    embed_bwd_pos_vec<<<S, t8, 0, st>>>(B, S, H / 8, (const uint4*)dout, (float4*)dwpe);
  } else if (dtype == BP_F32) {
    embed_bwd_tok_kernel<float><<<B * S, threads, 0, st>>>(H, tokens, (const float*)dout, dwte);
    embed_bwd_pos_kernel<float><<<S, threads, 0, st>>>(B, S, H, (const float*)dout, dwpe);
  } else {
    embed_bwd_tok_kernel<__nv_bfloat16><<<B * S, threads, 0, st>>>(H, tokens, (const __nv_bfloat16*)dout, dwte);
    embed_bwd_pos_kernel<__nv_bfloat16><<<S, threads, 0, st>>>(B, S, H, (const __nv_bfloat16*)dout, dwpe);
  }
  count_launch();
  count_launch();
  BP_CHECK_LAUNCH("embed_bwd");
  return BP_OK;
}

extern "C" int bp_xent_fwd_bwd(int dtype, int rows, int V, void* logits, int64_t ld, const int32_t* targets,
                               float grad_scale, float loss_scale, float* loss_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = V >= 4096 ? 512 : 128;
  const int esz = dtype == BP_F32 ? 4 : 2;
  const int vec = (reinterpret_cast<uintptr_t>(logits) % 16 == 0) && ((ld * esz) % 16 == 0);
  if (dtype == BP_F32)
    xent_kernel<float><<<rows, threads, 0, st>>>(V, (float*)logits, ld, targets, grad_scale, loss_scale, loss_out,
                                                 vec);
  else
    xent_kernel<__nv_bfloat16><<<rows, threads, 0, st>>>(V, (__nv_bfloat16*)logits, ld, targets, grad_scale,
                                                          loss_scale, loss_out, vec);
  count_launch();
  BP_CHECK_LAUNCH("xent");
  return BP_OK;
}

extern "C" int bp_cast(int sd, int dd, int64_t n, const void* src, void* dst, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(n, 256 * 4);
  if (sd == BP_F32 && dd == BP_BF16)
    cast_kernel<float, __nv_bfloat16><<<g, 256, 0, st>>>(n, (const float*)src, (__nv_bfloat16*)dst);
  else if (sd == BP_BF16 && dd == BP_F32)
    cast_kernel<__nv_bfloat16, float><<<g, 256, 0, st>>>(n, (const __nv_bfloat16*)src, (float*)dst);
  else if (sd == BP_F32 && dd == BP_F32)
    cast_kernel<float, float><<<g, 256, 0, st>>>(n, (const float*)src, (float*)dst);
  else
    cast_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>(n, (const __nv_bfloat16*)src, (__nv_bfloat16*)dst);
  count_launch();
  BP_CHECK_LAUNCH("cast");
  return BP_OK;
}

extern "C" int bp_adam_dev(int64_t n, int param_dtype, float* master, const float* grad_a, const float* grad_b,
                           float* m, float* v, void* param_a, void* param_b, float lr, float beta1, float beta2,
                           float eps, float weight_decay, int step, const int* step_dev, float grad_scale,
                           void* stream);

extern "C" int bp_adam(int64_t n, int param_dtype, float* master, const float* grad_a, const float* grad_b, float* m,
                       float* v, void* param_a, void* param_b, float lr, float beta1, float beta2, float eps,
                       float weight_decay, int step, float grad_scale, void* stream) {
  return bp_adam_dev(n, param_dtype, master, grad_a, grad_b, m, v, param_a, param_b, lr, beta1, beta2, eps,
                     weight_decay, step, nullptr, grad_scale, stream);
}

extern "C" int bp_adam_dev(int64_t n, int param_dtype, float* master, const float* grad_a, const float* grad_b,
                           float* m, float* v, void* param_a, void* param_b, float lr, float beta1, float beta2,
                           float eps, float weight_decay, int step, const int* step_dev, float grad_scale,
                           void* stream) {
  if (n <= 0 || (step < 1 && !step_dev)) {
    set_error("adam: bad n/step");
    return BP_ERR_INVALID;
  }
  if ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(grad_a) |
       reinterpret_cast<uintptr_t>(grad_b) | reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) {
    set_error("adam: fp32 buffers must be 16-byte aligned");
    return BP_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const float bc1 = 1.f - powf(beta1, (float)(step < 1 ? 1 : step)), bc2 = 1.f - powf(beta2, (float)(step < 1 ? 1 : step));
  const int g = grid_for(n / 4 + 1, 256);
  if (param_dtype == BP_F32)
    adam_kernel<float><<<g, 256, 0, st>>>(n, master, grad_a, grad_b, m, v, (float*)param_a, (float*)param_b, lr, beta1,
                                          beta2, eps, weight_decay, bc1, bc2, grad_scale, step_dev);
  else
    adam_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(n, master, grad_a, grad_b, m, v, (__nv_bfloat16*)param_a,
                                                  (__nv_bfloat16*)param_b, lr, beta1, beta2, eps, weight_decay, bc1,
                                                  bc2, grad_scale, step_dev);
  count_launch();
  BP_CHECK_LAUNCH("adam");
  return BP_OK;
}
