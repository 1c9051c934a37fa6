// Flash attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// bf16, head_dim 64/128, sequence length a multiple of 128
// (north star: "QKV, attention, MLP ... are tcgen05/TMEM
// tiles fed by TMA").
//
// Forward (one CTA = 128 query rows of one (batch, head), 256 threads):
//   warp 0  : TMA producer -- Q once, then K/V tiles of 128 keys through a
//             2-stage ring (one TMA box shape serves K as the K-major B
//             operand of S = Q K^T and V as the MN-major B operand of O += P V)
//   warp 1  : MMA issuer -- S(j) = Q K(j)^T into one of two TMEM S buffers,
//             then O += P(j-1) V(j-1); S(j+1) overlaps the softmax of S(j)
//   warps 4-7: softmax -- thread t owns query row t (= TMEM lane t): the
//             whole score row is in its registers, so max / sum need no
//             shuffles.  exp2 domain; the running max used for exponents is
//             only moved (and O in TMEM rescaled) when it grows by > 8, so
//             P <= 256.  P is written as bf16 to a SW128 K-major smem tile
//             (the A operand of the P V MMA).
// Backward = two kernels, no atomics:
//   dkdv : CTA = 128 keys; loops over 64-query tiles: S^T = K Q^T and
//          dP^T = V dO^T into TMEM, thread = key row computes P^T and
//          dS^T = P^T (dP^T - delta), then dV += P^T dO, dK += dS^T Q
//          (Q / dO tiles double as MN-major B operands).
//   dq   : CTA = 128 queries; loops over 64-key tiles: S, dP into TMEM,
//          dS = P (dP - delta), dQ += dS K (K tile as MN-major B).
#include "common.cuh"

namespace bp {
void count_launch();
int num_sms();
bool opt_attn_no_tc();
int make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, int64_t ld, uint32_t box_inner,
             uint32_t box_outer);

namespace fat {

#ifdef BP_ATTN_TRACE
__device__ long long g_trace[64][8];
#define TRACE(it, k) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 128 && (it) < 64) g_trace[(it)][(k)] = clock64();
#else
#define TRACE(it, k)
#endif

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// byte offset of 16-byte unit `u` (8 bf16) in row `r` of a K-major SW128
// tile whose K extent is split into 64-element atoms of `rows` x 128 B.
BP_DEV uint32_t kmaj_off(int r, int u, int rows) {
  return (uint32_t)((u >> 3) * rows * 128 + r * 128 + (((u & 7) ^ (r & 7)) << 4));
}

// 2^x in one MUFU op (flush-to-zero; inputs here are <= ~8 or -inf).
BP_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
BP_DEV float lds(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

BP_DEV uint4 pack8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
  return u;
}

BP_DEV void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// 1-D bulk copy global -> shared (bytes % 16 == 0), completion on `bar`.
BP_DEV void bulk_load(void* smem_dst, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(g), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// K-major SW128 descriptor for k-step `ks` (16 elements) of a tile with
// 64-element K atoms of `rows` rows.
BP_DEV uint64_t kdesc(uint32_t base, int ks, int rows) {
  return umma_desc_sw128(base + (ks >> 2) * rows * 128 + (ks & 3) * 32, 0, 1024);
}
// MN-major SW128 descriptor for k-step `ks` (16 K-rows) of a tile stored as
// [MN-chunk of 64][K rows][128 B] with `krows` K rows per chunk.
BP_DEV uint64_t mndesc(uint32_t base, int ks, int krows) {
  return umma_desc_sw128(base + ks * 2048, krows * 128, 1024);
}

// ============================================================ forward ====
template <int Dh>
struct Fwd {
  static constexpr int DC = Dh / 64;
  static constexpr uint32_t TILE = 128 * Dh * 2;
  static constexpr uint32_t PB = 128 * 128 * 2;
  static constexpr size_t SMEM = 1024 + TILE + 4 * TILE + PB + 512;
};

template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(256, 1)
fwd_tc(const __grid_constant__ CUtensorMap map_qkv, __nv_bfloat16* __restrict__ o, float* __restrict__ lse, int S,
       int H, float scale_log2) {
  using C = Fwd<Dh>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK[2] = {smem + C::TILE, smem + 3 * C::TILE};
  uint8_t* sV[2] = {smem + 2 * C::TILE, smem + 4 * C::TILE};
  uint8_t* sP = smem + 5 * C::TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::PB);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_free = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* pv_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x, qt = gridDim.y - 1 - blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int n_kv = CAUSAL ? qt + 1 : S / 128;
  const int HD = H * Dh;

  if (warp == 0 && lane == 0) tma_prefetch_desc(&map_qkv);
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------ producer
      const int qrow = b * S + qt * 128;
#pragma unroll
      for (int c = 0; c < C::DC; ++c) tma_load_2d(sQ + c * 16384, &map_qkv, h * Dh + c * 64, qrow, q_full);
      mbar_expect_tx(q_full, C::TILE);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        const int krow = b * S + j * 128;
#pragma unroll
        for (int c = 0; c < C::DC; ++c) {
          tma_load_2d(sK[st] + c * 16384, &map_qkv, HD + h * Dh + c * 64, krow, &kv_full[st]);
          tma_load_2d(sV[st] + c * 16384, &map_qkv, 2 * HD + h * Dh + c * 64, krow, &kv_full[st]);
        }
        mbar_expect_tx(&kv_full[st], 2 * C::TILE);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, Dh, false, true);
      const uint32_t aQ = smem_u32(sQ), aP = smem_u32(sP);
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j <= n_kv; ++j) {
        if (j < n_kv) {
          const int st = j & 1;
          mbar_wait(&kv_full[st], (j >> 1) & 1);
          mbar_wait(&s_free[st], ((j >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t aK = smem_u32(sK[st]);
#pragma unroll
          for (int ks = 0; ks < Dh / 16; ++ks)
            tc_mma_f16(tmem + st * 128, kdesc(aQ, ks, 128), kdesc(aK, ks, 128), idesc_s, ks > 0);
          tc_commit(&s_full[st]);
        }
        if (j >= 1) {
          const int jj = j - 1, st = jj & 1;
          mbar_wait(p_full, jj & 1);
          tc_fence_after();
          const uint32_t aV = smem_u32(sV[st]);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc_mma_f16(tmem + 256, kdesc(aP, ks, 128), mndesc(aV, ks, 128), idesc_o, (jj > 0 || ks > 0));
          tc_commit(pv_done);
          tc_commit(&kv_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {  // ---------------------------------- softmax
    const int r = (warp - 4) * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)((warp - 4) * 32) << 16);
    const uint32_t aP = smem_u32(sP);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tl + st * 128 + c * 32, *reinterpret_cast<float(*)[32]>(s + 32 * c));
      tc_fence_before();
      mbar_arrive(&s_free[st]);
      float mx = -INFINITY;
      const bool diag = CAUSAL && (j == qt);
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        float v = s[i] * scale_log2;
        if (diag && i > r) v = -INFINITY;
        s[i] = v;
        mx = fmaxf(mx, v);
      }
      bool waited = (j == 0);
      if (mx > m_used + 8.f) {
        if (j > 0) {
          mbar_wait(pv_done, (j - 1) & 1);
          waited = true;
          tc_fence_after();
          const float f = ex2(m_used - mx);
#pragma unroll 1
          for (int c = 0; c < Dh / 32; ++c) {
            float ov[32];
            tmem_ld_32x32b_x32(tl + 256 + c * 32, ov);
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] *= f;
            tmem_st_32x32b_x32(tl + 256 + c * 32, ov);
          }
          l *= f;
        }
        m_used = mx;
      }
      float lsum = 0.f;
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        s[i] = ex2(s[i] - m_used);
        lsum += s[i];
      }
      l += lsum;
      if (!waited) mbar_wait(pv_done, (j - 1) & 1);
#pragma unroll
      for (int u = 0; u < 16; ++u) st_shared_v4(aP + kmaj_off(r, u, 128), pack8(s + 8 * u));
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: O / l
    mbar_wait(pv_done, (n_kv - 1) & 1);
    tc_fence_after();
    const int q = qt * 128 + r;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = o + ((int64_t)b * S + q) * HD + h * Dh;
#pragma unroll 1
    for (int c = 0; c < Dh / 32; ++c) {
      float ov[32];
      tmem_ld_32x32b_x32(tl + 256 + c * 32, ov);
#pragma unroll
      for (int i = 0; i < 32; ++i) ov[i] *= inv;
#pragma unroll
      for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(orow + c * 32 + 8 * u) = pack8(ov + 8 * u);
    }
    lse[((int64_t)b * H + h) * S + q] = (m_used + log2f(l)) * kLn2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// =================================================== backward: dK, dV ====
template <int Dh>
struct Dkdv {
  static constexpr int DC = Dh / 64;
  static constexpr uint32_t KT = 128 * Dh * 2;  // K / V tile (128 keys)
  static constexpr uint32_t QT = 64 * Dh * 2;   // Q / dO tile (64 queries)
  static constexpr uint32_t PB = 128 * 64 * 2;  // P^T / dS^T tile
  static constexpr size_t SMEM = 1024 + 2 * KT + 4 * QT + 2 * PB + 2 * 512 + 512;
};

template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(256, 1)
dkdv_tc(const __grid_constant__ CUtensorMap map_kv, const __grid_constant__ CUtensorMap map_q,
        const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse, const float* __restrict__ delta,
        __nv_bfloat16* __restrict__ dqkv, int S, int H, float scale, float scale_log2) {
  using C = Dkdv<Dh>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::KT;
  uint8_t* sQ[2] = {smem + 2 * C::KT, smem + 2 * C::KT + 2 * C::QT};
  uint8_t* sO[2] = {smem + 2 * C::KT + C::QT, smem + 2 * C::KT + 3 * C::QT};
  uint8_t* sP = smem + 2 * C::KT + 4 * C::QT;
  uint8_t* sD = sP + C::PB;
  float* sL[2] = {reinterpret_cast<float*>(sD + C::PB), reinterpret_cast<float*>(sD + C::PB + 512)};
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + C::PB + 1024);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;   // [2]
  uint64_t* q_empty = bars + 3;  // [2]
  uint64_t* sdp_full = bars + 5;
  uint64_t* sdp_free = bars + 6;
  uint64_t* p_full = bars + 7;
  uint64_t* mm_done = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  // TMEM columns: S^T [0,64), dP^T [64,128), dV [128,128+Dh), dK [128+Dh, 128+2Dh)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x, kt = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int nq = S / 64;
  const int q0 = CAUSAL ? 2 * kt : 0;  // first 64-query tile that can see these keys
  const int n_it = nq - q0;
  const int HD = H * Dh;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_kv);
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_do);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(sdp_free, 128);
    mbar_init(p_full, 128);
    mbar_init(mm_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------ producer
      const int krow = b * S + kt * 128;
#pragma unroll
      for (int c = 0; c < C::DC; ++c) {
        tma_load_2d(sK + c * 16384, &map_kv, HD + h * Dh + c * 64, krow, kv_full);
        tma_load_2d(sV + c * 16384, &map_kv, 2 * HD + h * Dh + c * 64, krow, kv_full);
      }
      mbar_expect_tx(kv_full, 2 * C::KT);
      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1, qi = q0 + it;
        mbar_wait(&q_empty[st], ((it >> 1) & 1) ^ 1);
        const int qrow = b * S + qi * 64;
#pragma unroll
        for (int c = 0; c < C::DC; ++c) {
          tma_load_2d(sQ[st] + c * 8192, &map_q, h * Dh + c * 64, qrow, &q_full[st]);
          tma_load_2d(sO[st] + c * 8192, &map_do, h * Dh + c * 64, qrow, &q_full[st]);
        }
        const int64_t lrow = ((int64_t)b * H + h) * S + qi * 64;
        bulk_load(sL[st], lse + lrow, 256, &q_full[st]);
        bulk_load(sL[st] + 64, delta + lrow, 256, &q_full[st]);
        mbar_expect_tx(&q_full[st], 2 * C::QT + 512);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 64, false, false);  // S^T, dP^T: M=keys, N=64 q
      constexpr uint32_t idesc_g = umma_idesc_bf16(128, Dh, false, true);   // dV, dK: B MN-major
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aP = smem_u32(sP), aD = smem_u32(sD);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      for (int it = 0; it <= n_it; ++it) {
        if (it < n_it) {
          const int st = it & 1;
          mbar_wait(&q_full[st], (it >> 1) & 1);
          mbar_wait(sdp_free, (it & 1) ^ 1);
          tc_fence_after();
          const uint32_t aQ = smem_u32(sQ[st]), aO = smem_u32(sO[st]);
#pragma unroll
          for (int ks = 0; ks < Dh / 16; ++ks) {
            tc_mma_f16(tmem + 0, kdesc(aK, ks, 128), kdesc(aQ, ks, 64), idesc_s, ks > 0);
            tc_mma_f16(tmem + 64, kdesc(aV, ks, 128), kdesc(aO, ks, 64), idesc_s, ks > 0);
          }
          tc_commit(sdp_full);
        }
        if (it >= 1) {
          const int jj = it - 1, st = jj & 1;
          mbar_wait(p_full, jj & 1);
          tc_fence_after();
          const uint32_t aQ = smem_u32(sQ[st]), aO = smem_u32(sO[st]);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {  // 64 queries / 16
            tc_mma_f16(tmem + 128, kdesc(aP, ks, 128), mndesc(aO, ks, 64), idesc_g, (jj > 0 || ks > 0));
            tc_mma_f16(tmem + 128 + Dh, kdesc(aD, ks, 128), mndesc(aQ, ks, 64), idesc_g, (jj > 0 || ks > 0));
          }
          tc_commit(mm_done);
          tc_commit(&q_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {  // -------------------------- P^T / dS^T rows
    const int r = (warp - 4) * 32 + lane;  // key row in the tile
    const int key = kt * 128 + r;
    const uint32_t tl = tmem + ((uint32_t)((warp - 4) * 32) << 16);
    const uint32_t aP = smem_u32(sP), aD = smem_u32(sD);
    for (int it = 0; it < n_it; ++it) {
      const int st = it & 1, qi = q0 + it;
      TRACE(it, 0);
      mbar_wait(&q_full[st], (it >> 1) & 1);  // lse / delta of this tile are in smem
      TRACE(it, 1);
      mbar_wait(sdp_full, it & 1);
      TRACE(it, 2);
      tc_fence_after();
      float sv[64], dp[64];
      tmem_ld_32x32b_x32(tl + 0, *reinterpret_cast<float(*)[32]>(sv));
      tmem_ld_32x32b_x32(tl + 32, *reinterpret_cast<float(*)[32]>(sv + 32));
      tmem_ld_32x32b_x32(tl + 64, *reinterpret_cast<float(*)[32]>(dp));
      tmem_ld_32x32b_x32(tl + 96, *reinterpret_cast<float(*)[32]>(dp + 32));
      TRACE(it, 3);
      tc_fence_before();
      mbar_arrive(sdp_free);
      const uint32_t aL = smem_u32(sL[st]);
      const bool diag = CAUSAL && qi * 64 < key;  // some query of this tile precedes the key
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const int q = qi * 64 + i;
        float p = ex2(fmaf(sv[i], scale_log2, -lds(aL + 4 * i) * kLog2e));
        if (diag && q < key) p = 0.f;
        sv[i] = p;
        dp[i] = p * (dp[i] - lds(aL + 256 + 4 * i));
      }
      TRACE(it, 4);
      if (it > 0) mbar_wait(mm_done, (it - 1) & 1);
      TRACE(it, 5);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        st_shared_v4(aP + kmaj_off(r, u, 128), pack8(sv + 8 * u));
        st_shared_v4(aD + kmaj_off(r, u, 128), pack8(dp + 8 * u));
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
      TRACE(it, 6);
    }
    // epilogue: dV, dK (scaled) -> dqkv
    if (n_it > 0) mbar_wait(mm_done, (n_it - 1) & 1);
    tc_fence_after();
    __nv_bfloat16* dkrow = dqkv + ((int64_t)b * S + key) * 3 * HD + HD + h * Dh;
    __nv_bfloat16* dvrow = dkrow + HD;
#pragma unroll 1
    for (int c = 0; c < Dh / 32; ++c) {
      float v[32];
      if (n_it > 0) {
        tmem_ld_32x32b_x32(tl + 128 + c * 32, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(dvrow + c * 32 + 8 * u) = pack8(v + 8 * u);
      if (n_it > 0) tmem_ld_32x32b_x32(tl + 128 + Dh + c * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= scale;
#pragma unroll
      for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(dkrow + c * 32 + 8 * u) = pack8(v + 8 * u);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ========================================================= backward: dQ ====
template <int Dh>
struct Dq {
  static constexpr int DC = Dh / 64;
  static constexpr uint32_t QT = 128 * Dh * 2;  // Q / dO tile (128 queries)
  static constexpr uint32_t KT = 64 * Dh * 2;   // K / V tile (64 keys)
  static constexpr uint32_t DB = 128 * 64 * 2;  // dS tile
  static constexpr size_t SMEM = 1024 + 2 * QT + 4 * KT + DB + 512;
};

template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(256, 1)
dq_tc(const __grid_constant__ CUtensorMap map_q128, const __grid_constant__ CUtensorMap map_kv64,
      const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse, const float* __restrict__ delta,
      __nv_bfloat16* __restrict__ dqkv, int S, int H, float scale, float scale_log2) {
  using C = Dq<Dh>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sO = smem + C::QT;
  uint8_t* sK[2] = {smem + 2 * C::QT, smem + 2 * C::QT + 2 * C::KT};
  uint8_t* sV[2] = {smem + 2 * C::QT + C::KT, smem + 2 * C::QT + 3 * C::KT};
  uint8_t* sD = smem + 2 * C::QT + 4 * C::KT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + C::DB);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* sdp_full = bars + 5;
  uint64_t* sdp_free = bars + 6;
  uint64_t* p_full = bars + 7;
  uint64_t* mm_done = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  // TMEM: S [0,64), dP [64,128), dQ [128, 128+Dh)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x, qt = gridDim.y - 1 - blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int n_it = CAUSAL ? 2 * qt + 2 : S / 64;
  const int HD = H * Dh;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_q128);
    tma_prefetch_desc(&map_kv64);
    tma_prefetch_desc(&map_do);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(sdp_free, 128);
    mbar_init(p_full, 128);
    mbar_init(mm_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const int qrow = b * S + qt * 128;
#pragma unroll
      for (int c = 0; c < C::DC; ++c) {
        tma_load_2d(sQ + c * 16384, &map_q128, h * Dh + c * 64, qrow, q_full);
        tma_load_2d(sO + c * 16384, &map_do, h * Dh + c * 64, qrow, q_full);
      }
      mbar_expect_tx(q_full, 2 * C::QT);
      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1;
        mbar_wait(&kv_empty[st], ((it >> 1) & 1) ^ 1);
        const int krow = b * S + it * 64;
#pragma unroll
        for (int c = 0; c < C::DC; ++c) {
          tma_load_2d(sK[st] + c * 8192, &map_kv64, HD + h * Dh + c * 64, krow, &kv_full[st]);
          tma_load_2d(sV[st] + c * 8192, &map_kv64, 2 * HD + h * Dh + c * 64, krow, &kv_full[st]);
        }
        mbar_expect_tx(&kv_full[st], 2 * C::KT);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_q = umma_idesc_bf16(128, Dh, false, true);
      const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO), aD = smem_u32(sD);
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int it = 0; it <= n_it; ++it) {
        if (it < n_it) {
          const int st = it & 1;
          mbar_wait(&kv_full[st], (it >> 1) & 1);
          mbar_wait(sdp_free, (it & 1) ^ 1);
          tc_fence_after();
          const uint32_t aK = smem_u32(sK[st]), aV = smem_u32(sV[st]);
#pragma unroll
          for (int ks = 0; ks < Dh / 16; ++ks) {
            tc_mma_f16(tmem + 0, kdesc(aQ, ks, 128), kdesc(aK, ks, 64), idesc_s, ks > 0);
            tc_mma_f16(tmem + 64, kdesc(aO, ks, 128), kdesc(aV, ks, 64), idesc_s, ks > 0);
          }
          tc_commit(sdp_full);
        }
        if (it >= 1) {
          const int jj = it - 1, st = jj & 1;
          mbar_wait(p_full, jj & 1);
          tc_fence_after();
          const uint32_t aK = smem_u32(sK[st]);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc_mma_f16(tmem + 128, kdesc(aD, ks, 128), mndesc(aK, ks, 64), idesc_q, (jj > 0 || ks > 0));
          tc_commit(mm_done);
          tc_commit(&kv_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;
    const int q = qt * 128 + r;
    const uint32_t tl = tmem + ((uint32_t)((warp - 4) * 32) << 16);
    const uint32_t aD = smem_u32(sD);
    const int64_t li = ((int64_t)b * H + h) * S + q;
    const float lse2 = lse[li] * kLog2e, dl = delta[li];
    for (int it = 0; it < n_it; ++it) {
      mbar_wait(sdp_full, it & 1);
      tc_fence_after();
      float sv[64], dp[64];
      tmem_ld_32x32b_x32(tl + 0, *reinterpret_cast<float(*)[32]>(sv));
      tmem_ld_32x32b_x32(tl + 32, *reinterpret_cast<float(*)[32]>(sv + 32));
      tmem_ld_32x32b_x32(tl + 64, *reinterpret_cast<float(*)[32]>(dp));
      tmem_ld_32x32b_x32(tl + 96, *reinterpret_cast<float(*)[32]>(dp + 32));
      tc_fence_before();
      mbar_arrive(sdp_free);
      const bool diag = CAUSAL && (it * 64 + 63 > q);
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        float p = ex2(fmaf(sv[i], scale_log2, -lse2));
        if (diag && it * 64 + i > q) p = 0.f;
        dp[i] = p * (dp[i] - dl);
      }
      if (it > 0) mbar_wait(mm_done, (it - 1) & 1);
#pragma unroll
      for (int u = 0; u < 8; ++u) st_shared_v4(aD + kmaj_off(r, u, 128), pack8(dp + 8 * u));
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(mm_done, (n_it - 1) & 1);
    tc_fence_after();
    __nv_bfloat16* dqrow = dqkv + ((int64_t)b * S + q) * 3 * HD + h * Dh;
#pragma unroll 1
    for (int c = 0; c < Dh / 32; ++c) {
      float v[32];
      tmem_ld_32x32b_x32(tl + 128 + c * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= scale;
#pragma unroll
      for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(dqrow + c * 32 + 8 * u) = pack8(v + 8 * u);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<256>(tmem);
}

template <int Dh>
__global__ void delta_tc_kernel(int rows_bhs, int S, int H, const __nv_bfloat16* __restrict__ o,
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

template <typename K>
static int set_smem(K kern, size_t bytes) {
  BP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return BP_OK;
}

template <int Dh, bool CAUSAL>
static int fwd(int B, int S, int H, float scale, const void* qkv, void* o, float* lse, cudaStream_t st) {
  CUtensorMap m;
  if (int rc = make_map(&m, qkv, 3ull * H * Dh, (uint64_t)B * S, 3LL * H * Dh, 64, 128)) return rc;
  auto k = fwd_tc<Dh, CAUSAL>;
  static bool once = false;
  if (!once) {
    if (int rc = set_smem(k, Fwd<Dh>::SMEM)) return rc;
    once = true;
  }
  k<<<dim3(B * H, S / 128), 256, Fwd<Dh>::SMEM, st>>>(m, (__nv_bfloat16*)o, lse, S, H, scale * kLog2e);
  count_launch();
  BP_CHECK_LAUNCH("attn_fwd_tc");
  return BP_OK;
}

template <int Dh, bool CAUSAL>
static int bwd(int B, int S, int H, float scale, const void* qkv, const void* o, const void* dout, const float* lse,
               void* dqkv, float* ws, cudaStream_t st) {
  float* delta = ws;
  const int rows = B * H * S;
  delta_tc_kernel<Dh><<<(rows + 7) / 8, 256, 0, st>>>(rows, S, H, (const __nv_bfloat16*)o,
                                                       (const __nv_bfloat16*)dout, delta);
  count_launch();
  CUtensorMap kv128, q64, do64, q128, kv64, do128;
  const uint64_t W = 3ull * H * Dh, R = (uint64_t)B * S;
  if (int rc = make_map(&kv128, qkv, W, R, (int64_t)W, 64, 128)) return rc;
  if (int rc = make_map(&q64, qkv, W, R, (int64_t)W, 64, 64)) return rc;
  if (int rc = make_map(&do64, dout, (uint64_t)H * Dh, R, (int64_t)H * Dh, 64, 64)) return rc;
  if (int rc = make_map(&q128, qkv, W, R, (int64_t)W, 64, 128)) return rc;
  if (int rc = make_map(&kv64, qkv, W, R, (int64_t)W, 64, 64)) return rc;
  if (int rc = make_map(&do128, dout, (uint64_t)H * Dh, R, (int64_t)H * Dh, 64, 128)) return rc;
  auto k1 = dkdv_tc<Dh, CAUSAL>;
  auto k2 = dq_tc<Dh, CAUSAL>;
  static bool once = false;
  if (!once) {
    if (int rc = set_smem(k1, Dkdv<Dh>::SMEM)) return rc;
    if (int rc = set_smem(k2, Dq<Dh>::SMEM)) return rc;
    once = true;
  }
  const float sl2 = scale * kLog2e;
  k1<<<dim3(B * H, S / 128), 256, Dkdv<Dh>::SMEM, st>>>(kv128, q64, do64, lse, delta, (__nv_bfloat16*)dqkv, S, H,
                                                         scale, sl2);
  count_launch();
  k2<<<dim3(B * H, S / 128), 256, Dq<Dh>::SMEM, st>>>(q128, kv64, do128, lse, delta, (__nv_bfloat16*)dqkv, S, H,
                                                       scale, sl2);
  count_launch();
  BP_CHECK_LAUNCH("attn_bwd_tc");
  return BP_OK;
}

}  // namespace fat

// Debug aid (BP_ATTN_TRACE builds): copy the dK/dV softmax-warp timestamps.
extern "C" int bp_attn_trace_dump(long long* host, int n) {
#ifdef BP_ATTN_TRACE
  return cudaMemcpyFromSymbol(host, fat::g_trace, sizeof(long long) * (n < 512 ? n : 512)) == cudaSuccess ? 0 : 2;
#else
  (void)host; (void)n;
  return 3;
#endif
}

bool attn_tc_supported(int dtype, int S, int Dh) {
  return dtype == BP_BF16 && (Dh == 64 || Dh == 128) && S >= 128 && S % 128 == 0 && !opt_attn_no_tc();
}

int attn_tc_fwd(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, void* o, float* lse,
                cudaStream_t st) {
  if (Dh == 128)
    return causal ? fat::fwd<128, true>(B, S, H, scale, qkv, o, lse, st)
                  : fat::fwd<128, false>(B, S, H, scale, qkv, o, lse, st);
  return causal ? fat::fwd<64, true>(B, S, H, scale, qkv, o, lse, st)
                : fat::fwd<64, false>(B, S, H, scale, qkv, o, lse, st);
}

int attn_tc_bwd(int B, int S, int H, int Dh, int causal, float scale, const void* qkv, const void* o,
                const void* dout, const float* lse, void* dqkv, float* ws, cudaStream_t st) {
  if (Dh == 128)
    return causal ? fat::bwd<128, true>(B, S, H, scale, qkv, o, dout, lse, dqkv, ws, st)
                  : fat::bwd<128, false>(B, S, H, scale, qkv, o, dout, lse, dqkv, ws, st);
  return causal ? fat::bwd<64, true>(B, S, H, scale, qkv, o, dout, lse, dqkv, ws, st)
                : fat::bwd<64, false>(B, S, H, scale, qkv, o, dout, lse, dqkv, ws, st);
}

}  // namespace bp
