// Flash attention forward / backward for bf16, head_dim 64 or 128
// (SURVEY §8(a) K5).  FlashAttention-2 tiling on the warp-level tensor-core
// path (mma.sync m16n8k16 bf16 -> fp32):
//
//   forward : CTA = 64 query rows (4 warps x 16 rows) of one (batch, head);
//             K/V tiles of 64 keys stream through a cp.async double buffer;
//             online softmax in the exp2 domain; causal tiles above the
//             diagonal are skipped.  Writes O (bf16) and the natural-log
//             LSE per row.
//   backward: CTA = 64 keys (4 warps x 16 keys) of one (batch, head); loops
//             over the query tiles at/after the diagonal, recomputes P from
//             the saved LSE, accumulates dK, dV in registers, and adds dQ
//             partials into an fp32 workspace with vector atomics; a final
//             pass scales dQ and packs it into dqkv.
//
// Shared-memory tiles are [rows][Dh] bf16 with a 16-byte-chunk XOR swizzle
// (chunk ^ (row & 7)) so every ldmatrix phase is bank-conflict free.
#include "common.cuh"

namespace bp {
void count_launch();
int num_sms();
bool opt_attn_exact();

namespace fa {

constexpr int BR = 64, BC = 64, NT = 128;

BP_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

BP_DEV void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
BP_DEV void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

BP_DEV void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

BP_DEV void cp_async16(uint32_t saddr, const void* g, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(n) : "memory");
}
BP_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
BP_DEV void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// byte offset of (row, chunk) inside a swizzled [rows][CH chunks] tile
template <int CH>
BP_DEV uint32_t sw(int row, int chunk) {
  return (uint32_t)(row * CH * 16 + ((chunk ^ (row & 7)) << 4));
}

// Load a [64 rows][Dh] tile from global rows r0.. (row pitch ld elements).
template <int Dh>
BP_DEV void load_tile(uint32_t sbase, const __nv_bfloat16* g, int64_t ld, int r0, int rows_valid) {
  constexpr int CH = Dh / 8;
  for (int i = threadIdx.x; i < 64 * CH; i += NT) {
    const int r = i / CH, c = i % CH;
    const bool ok = (r0 + r) < rows_valid;
    const __nv_bfloat16* src = g + (int64_t)(ok ? r0 + r : 0) * ld + c * 8;
    cp_async16(sbase + sw<CH>(r, c), src, ok);
  }
}

// ------------------------------------------------------------- forward --
template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(NT) fwd_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ o,
                                                 float* __restrict__ lse, int S, int H, float scale_log2) {
  constexpr int CH = Dh / 8, KK = Dh / 16, DT = Dh / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK0 = sQ + 64 * Dh * 2;
  const uint32_t sV0 = sK0 + 2 * 64 * Dh * 2;
  // heaviest (last, for causal) query tiles first; heads vary fastest
  const int qt = gridDim.y - 1 - blockIdx.y, bh = blockIdx.x, b = bh / H, h = bh % H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ld = 3LL * H * Dh;
  const __nv_bfloat16* qg = qkv + (int64_t)b * S * ld + h * Dh;
  const __nv_bfloat16* kg = qg + H * Dh;
  const __nv_bfloat16* vg = qg + 2 * H * Dh;
  const int n_tiles = CAUSAL ? min(qt + 1, (S + BC - 1) / BC) : (S + BC - 1) / BC;

  load_tile<Dh>(sQ, qg, ld, qt * BR, S);
  load_tile<Dh>(sK0, kg, ld, 0, S);
  load_tile<Dh>(sV0, vg, ld, 0, S);
  cp_commit();

  float acc[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  uint32_t qf[KK][4];
  const int g = lane >> 2, tq = lane & 3;
  const int qrow0 = qt * BR + warp * 16 + g;  // query index for c0/c1; +8 for c2/c3

  for (int j = 0; j < n_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_tiles) {
      load_tile<Dh>(sK0 + (buf ^ 1) * 64 * Dh * 2, kg, ld, (j + 1) * BC, S);
      load_tile<Dh>(sV0 + (buf ^ 1) * 64 * Dh * 2, vg, ld, (j + 1) * BC, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < KK; ++kk)
        ldsm_x4(sQ + sw<CH>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), qf[kk]);
    }
    const uint32_t sK = sK0 + buf * 64 * Dh * 2, sV = sV0 + buf * 64 * Dh * 2;
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bfr[4];
        ldsm_x4(sK + sw<CH>(np * 16 + (lane >> 4) * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)), bfr);
        mma16816(s[2 * np], qf[kk], bfr[0], bfr[1]);
        mma16816(s[2 * np + 1], qf[kk], bfr[2], bfr[3]);
      }
    }
    // scale into the log2 domain, mask, online softmax
    const bool diag = CAUSAL && (j == qt);
    const bool ragged = (j + 1) * BC > S;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[nt][e] * scale_log2;
        const int key = j * BC + nt * 8 + 2 * tq + (e & 1);
        const int qi = qrow0 + (e >> 1) * 8;
        if ((diag && key > qi) || (ragged && key >= S)) v = -INFINITY;
        s[nt][e] = v;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float mx = m_r[r];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mx = fmaxf(mx, fmaxf(s[nt][2 * r], s[nt][2 * r + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float corr = (m_r[r] == -INFINITY) ? 0.f : exp2f(m_r[r] - mx);
      m_r[r] = mx;
      l_r[r] *= corr;
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        acc[dt][2 * r] *= corr;
        acc[dt][2 * r + 1] *= corr;
      }
      const float msafe = (mx == -INFINITY) ? 0.f : mx;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float p0 = exp2f(s[nt][2 * r] - msafe), p1 = exp2f(s[nt][2 * r + 1] - msafe);
        s[nt][2 * r] = p0;
        s[nt][2 * r + 1] = p1;
        l_r[r] += p0 + p1;
      }
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4] = {pack_bf16(s[2 * kk][0], s[2 * kk][1]), pack_bf16(s[2 * kk][2], s[2 * kk][3]),
                       pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int dp = 0; dp < DT / 2; ++dp) {
        uint32_t bfr[4];
        ldsm_x4_t(sV + sw<CH>(kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, dp * 2 + (lane >> 4)), bfr);
        mma16816(acc[2 * dp], a, bfr[0], bfr[1]);
        mma16816(acc[2 * dp + 1], a, bfr[2], bfr[3]);
      }
    }
    __syncthreads();
  }
  // finalize
  const int64_t ldo = (int64_t)H * Dh;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    float l = l_r[r];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int qi = qrow0 + r * 8;
    if (qi < S) {
      __nv_bfloat16* orow = o + ((int64_t)b * S + qi) * ldo + h * Dh;
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        const int d = dt * 8 + 2 * tq;
        *reinterpret_cast<__nv_bfloat162*>(orow + d) =
            __floats2bfloat162_rn(acc[dt][2 * r] * inv, acc[dt][2 * r + 1] * inv);
      }
      if (tq == 0) lse[((int64_t)b * H + h) * S + qi] = (m_r[r] + log2f(l)) * 0.6931471805599453f;
    }
  }
}

// ------------------------------------------------------------ backward --
template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(NT) bwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                 const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                                                 const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv,
                                                 float* __restrict__ dq_acc, int S, int H, float scale,
                                                 float scale_log2) {
  constexpr int CH = Dh / 8, KK = Dh / 16, DT = Dh / 8;
  constexpr uint32_t TILE = 64 * Dh * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sK = smem_u32(smem);
  const uint32_t sV = sK + TILE;
  const uint32_t sQ0 = sV + TILE;            // 2 buffers
  const uint32_t sO0 = sQ0 + 2 * TILE;       // dO, 2 buffers
  const uint32_t sdS = sO0 + 2 * TILE;       // [64 keys][64 q] bf16
  float* s_lse = reinterpret_cast<float*>(smem + 6 * TILE + 64 * 64 * 2);  // [2][64]
  float* s_del = s_lse + 128;                                            // [2][64]

  // heaviest (first, for causal) key tiles first; heads vary fastest
  const int kt = blockIdx.y, bh = blockIdx.x, b = bh / H, h = bh % H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t ld = 3LL * H * Dh, ldo = (int64_t)H * Dh;
  const __nv_bfloat16* qg = qkv + (int64_t)b * S * ld + h * Dh;
  const __nv_bfloat16* kg = qg + H * Dh;
  const __nv_bfloat16* vg = qg + 2 * H * Dh;
  const __nv_bfloat16* og = dout + (int64_t)b * S * ldo + h * Dh;
  const float* lse_g = lse + ((int64_t)b * H + h) * S;
  const float* del_g = delta + ((int64_t)b * H + h) * S;
  const int n_q = (S + BR - 1) / BR;
  const int q_begin = CAUSAL ? kt : 0;

  load_tile<Dh>(sK, kg, ld, kt * BC, S);
  load_tile<Dh>(sV, vg, ld, kt * BC, S);
  auto load_q = [&](int qi, int buf) {
    load_tile<Dh>(sQ0 + buf * TILE, qg, ld, qi * BR, S);
    load_tile<Dh>(sO0 + buf * TILE, og, ldo, qi * BR, S);
    for (int i = threadIdx.x; i < 64; i += NT) {
      const int q = qi * BR + i;
      s_lse[buf * 64 + i] = q < S ? lse_g[q] * 1.4426950408889634f : 0.f;
      s_del[buf * 64 + i] = q < S ? del_g[q] : 0.f;
    }
  };
  if (q_begin < n_q) load_q(q_begin, 0);
  cp_commit();

  float dk[DT][4], dv[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;

  for (int qi = q_begin; qi < n_q; ++qi) {
    const int buf = (qi - q_begin) & 1;
    if (qi + 1 < n_q) load_q(qi + 1, buf ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const uint32_t sQ = sQ0 + buf * TILE, sO = sO0 + buf * TILE;
    const float* lq = s_lse + buf * 64;
    const float* dq_ = s_del + buf * 64;

    // S^T = K_w Q^T   (16 keys x 64 queries)
    float st[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) st[nt][0] = st[nt][1] = st[nt][2] = st[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      uint32_t a[4];
      ldsm_x4(sK + sw<CH>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), a);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bfr[4];
        ldsm_x4(sQ + sw<CH>(np * 16 + (lane >> 4) * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)), bfr);
        mma16816(st[2 * np], a, bfr[0], bfr[1]);
        mma16816(st[2 * np + 1], a, bfr[2], bfr[3]);
      }
    }
    // P^T
    const bool diag = CAUSAL && (qi == kt);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + 2 * tq + (e & 1);
        const int q = qi * BR + ql;
        const int key = kt * BC + warp * 16 + g + (e >> 1) * 8;
        float p = exp2f(st[nt][e] * scale_log2 - lq[ql]);
        if ((diag && key > q) || q >= S || key >= S) p = 0.f;
        st[nt][e] = p;
      }
    // dV += P^T dO
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4] = {pack_bf16(st[2 * kk][0], st[2 * kk][1]), pack_bf16(st[2 * kk][2], st[2 * kk][3]),
                       pack_bf16(st[2 * kk + 1][0], st[2 * kk + 1][1]), pack_bf16(st[2 * kk + 1][2], st[2 * kk + 1][3])};
#pragma unroll
      for (int dp = 0; dp < DT / 2; ++dp) {
        uint32_t bfr[4];
        ldsm_x4_t(sO + sw<CH>(kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, dp * 2 + (lane >> 4)), bfr);
        mma16816(dv[2 * dp], a, bfr[0], bfr[1]);
        mma16816(dv[2 * dp + 1], a, bfr[2], bfr[3]);
      }
    }
    // dP^T = V_w dO^T
    float dpt[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) dpt[nt][0] = dpt[nt][1] = dpt[nt][2] = dpt[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      uint32_t a[4];
      ldsm_x4(sV + sw<CH>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), a);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bfr[4];
        ldsm_x4(sO + sw<CH>(np * 16 + (lane >> 4) * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)), bfr);
        mma16816(dpt[2 * np], a, bfr[0], bfr[1]);
        mma16816(dpt[2 * np + 1], a, bfr[2], bfr[3]);
      }
    }
    // dS^T = P^T * (dP^T - delta)   (into st), and stage it to smem as [key][q]
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + 2 * tq + (e & 1);
        st[nt][e] = st[nt][e] * (dpt[nt][e] - dq_[ql]);
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int krow = warp * 16 + g + r * 8;
        const int col = nt * 8 + 2 * tq;
        const uint32_t addr = sdS + sw<8>(krow, col >> 3) + (col & 7) * 2;
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(pack_bf16(st[nt][2 * r], st[nt][2 * r + 1])));
      }
    }
    // dK += dS^T Q
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4] = {pack_bf16(st[2 * kk][0], st[2 * kk][1]), pack_bf16(st[2 * kk][2], st[2 * kk][3]),
                       pack_bf16(st[2 * kk + 1][0], st[2 * kk + 1][1]), pack_bf16(st[2 * kk + 1][2], st[2 * kk + 1][3])};
#pragma unroll
      for (int dp = 0; dp < DT / 2; ++dp) {
        uint32_t bfr[4];
        ldsm_x4_t(sQ + sw<CH>(kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, dp * 2 + (lane >> 4)), bfr);
        mma16816(dk[2 * dp], a, bfr[0], bfr[1]);
        mma16816(dk[2 * dp + 1], a, bfr[2], bfr[3]);
      }
    }
    __syncthreads();
    // dQ (64 q x Dh) partial = dS (q x 64 keys) K ; warp w -> queries w*16..
    {
      float dqa[DT][4];
#pragma unroll
      for (int i = 0; i < DT; ++i) dqa[i][0] = dqa[i][1] = dqa[i][2] = dqa[i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // 64 keys / 16
        uint32_t a[4];
        ldsm_x4_t(sdS + sw<8>(kk * 16 + (lane & 7) + (lane >> 4) * 8, warp * 2 + ((lane >> 3) & 1)), a);
#pragma unroll
        for (int dp = 0; dp < DT / 2; ++dp) {
          uint32_t bfr[4];
          ldsm_x4_t(sK + sw<CH>(kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, dp * 2 + (lane >> 4)), bfr);
          mma16816(dqa[2 * dp], a, bfr[0], bfr[1]);
          mma16816(dqa[2 * dp + 1], a, bfr[2], bfr[3]);
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = qi * BR + warp * 16 + g + r * 8;
        if (q < S) {
          float* dst = dq_acc + ((int64_t)b * S + q) * ldo + h * Dh;
#pragma unroll
          for (int dt = 0; dt < DT; ++dt)
            atomicAdd(reinterpret_cast<float2*>(dst + dt * 8 + 2 * tq),
                      make_float2(dqa[dt][2 * r], dqa[dt][2 * r + 1]));
        }
      }
    }
    __syncthreads();
  }
  // write dK (scaled) and dV
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = kt * BC + warp * 16 + g + r * 8;
    if (key < S) {
      __nv_bfloat16* dkr = dqkv + ((int64_t)b * S + key) * ld + (int64_t)H * Dh + h * Dh;
      __nv_bfloat16* dvr = dkr + (int64_t)H * Dh;
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        const int d = dt * 8 + 2 * tq;
        *reinterpret_cast<__nv_bfloat162*>(dkr + d) =
            __floats2bfloat162_rn(dk[dt][2 * r] * scale, dk[dt][2 * r + 1] * scale);
        *reinterpret_cast<__nv_bfloat162*>(dvr + d) = __floats2bfloat162_rn(dv[dt][2 * r], dv[dt][2 * r + 1]);
      }
    }
  }
}

// delta[b,h,i] = sum_d dO*O  (bf16 inputs; one warp per row, 16-byte loads)
template <int Dh>
__global__ void delta_kernel(int rows_bhs, int S, int H, const __nv_bfloat16* __restrict__ o,
                             const __nv_bfloat16* __restrict__ dout, float* __restrict__ delta) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= rows_bhs) return;
  const int i = w % S, h = (w / S) % H, b = w / (S * H);
  const int64_t off = ((int64_t)b * S + i) * H * Dh + h * Dh;
  float s = 0.f;
  for (int d = lane * 2; d < Dh; d += 64) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + off + d));
    const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dout + off + d));
    s += a.x * c.x + a.y * c.y;
  }
  s = warp_sum(s);
  if (lane == 0) delta[((int64_t)b * H + h) * S + i] = s;
}

// dqkv[:, q part] = dq_acc * scale
__global__ void dq_pack_kernel(int64_t rows, int hd, const float* __restrict__ dq, float scale,
                               __nv_bfloat16* __restrict__ dqkv) {
  const int64_t n = rows * hd / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (2 * e) / hd, c = (2 * e) % hd;
    const float2 v = *reinterpret_cast<const float2*>(dq + 2 * e);
    *reinterpret_cast<__nv_bfloat162*>(dqkv + r * 3 * hd + c) = __floats2bfloat162_rn(v.x * scale, v.y * scale);
  }
}

template <int Dh>
constexpr size_t fwd_smem() { return (size_t)5 * 64 * Dh * 2; }
template <int Dh>
constexpr size_t bwd_smem() { return (size_t)6 * 64 * Dh * 2 + 64 * 64 * 2 + 4 * 64 * 4; }

template <int Dh, bool C>
static int launch_fwd(int B, int S, int H, float scale, const void* qkv, void* o, float* lse, cudaStream_t st) {
  auto k = fwd_kernel<Dh, C>;
  static bool set = false;
  if (!set) {
    BP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem<Dh>()));
    set = true;
  }
  dim3 grid(B * H, (S + BR - 1) / BR);
  k<<<grid, NT, fwd_smem<Dh>(), st>>>((const __nv_bfloat16*)qkv, (__nv_bfloat16*)o, lse, S, H,
                                       scale * 1.4426950408889634f);
  count_launch();
  BP_CHECK_LAUNCH("fa_fwd");
  return BP_OK;
}

template <int Dh, bool C>
static int launch_bwd(int B, int S, int H, float scale, const void* qkv, const void* o, const void* dout,
                      const float* lse, void* dqkv, float* ws, cudaStream_t st) {
  float* delta = ws;
  float* dq = ws + (int64_t)B * H * S;
  const int64_t hd = (int64_t)H * Dh;
  BP_CUDA(cudaMemsetAsync(dq, 0, sizeof(float) * (size_t)B * S * hd, st));
  const int rows = B * H * S;
  delta_kernel<Dh><<<(rows + 7) / 8, 256, 0, st>>>(rows, S, H, (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout,
                                                    delta);
  count_launch();
  auto k = bwd_kernel<Dh, C>;
  static bool set = false;
  if (!set) {
    BP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd_smem<Dh>()));
    set = true;
  }
  dim3 grid(B * H, (S + BC - 1) / BC);
  k<<<grid, NT, bwd_smem<Dh>(), st>>>((const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dout, lse, delta,
                                       (__nv_bfloat16*)dqkv, dq, S, H, scale, scale * 1.4426950408889634f);
  count_launch();
  dq_pack_kernel<<<num_sms() * 4, 256, 0, st>>>((int64_t)B * S, (int)hd, dq, scale, (__nv_bfloat16*)dqkv);
  count_launch();
  BP_CHECK_LAUNCH("fa_bwd");
  return BP_OK;
}

}  // namespace fa

bool attn_flash_supported(int dtype, int S, int Dh) {
  return dtype == BP_BF16 && (Dh == 64 || Dh == 128) && S >= 1 && !opt_attn_exact();
}

int attn_flash_fwd(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, void* o, float* lse,
                   cudaStream_t st) {
  if (Dh == 128) return causal ? fa::launch_fwd<128, true>(B, S, H, scale, qkv, o, lse, st)
                               : fa::launch_fwd<128, false>(B, S, H, scale, qkv, o, lse, st);
  return causal ? fa::launch_fwd<64, true>(B, S, H, scale, qkv, o, lse, st)
                : fa::launch_fwd<64, false>(B, S, H, scale, qkv, o, lse, st);
}

int attn_flash_bwd(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, const void* o,
                   const void* dout, const float* lse, void* dqkv, float* ws, cudaStream_t st) {
  if (Dh == 128) return causal ? fa::launch_bwd<128, true>(B, S, H, scale, qkv, o, dout, lse, dqkv, ws, st)
                               : fa::launch_bwd<128, false>(B, S, H, scale, qkv, o, dout, lse, dqkv, ws, st);
  return causal ? fa::launch_bwd<64, true>(B, S, H, scale, qkv, o, dout, lse, dqkv, ws, st)
                : fa::launch_bwd<64, false>(B, S, H, scale, qkv, o, dout, lse, dqkv, ws, st);
}

}  // namespace bp
