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
int attn_fwd_mode();
int attn_fwd_exf();
int attn_bwd_mode();
int64_t attn_ds_offset_floats(int B, int S, int H);
int make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, int64_t ld, uint32_t box_inner,
             uint32_t box_outer);

namespace fat {

#ifdef BP_ATTN_TRACE
__device__ long long g_trace[64][16];
#define TRACE(it, k) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 128 && (it) < 64) g_trace[(it)][(k)] = clock64();
#define TRACE_MMA(it, k) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && (it) < 64) g_trace[(it)][(k)] = clock64();
#else
#define TRACE(it, k)
#define TRACE_MMA(it, k)
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
// 2^x on the FMA pipe (x <= ~126): round-to-nearest split x = n + f through
// the 1.5 * 2^23 magic constant, 2^f (|f| <= 1/2) by a cubic (max relative
// error 7.6e-5, below the bf16 rounding of P), exponent added as integer
// bits.  Offloads part of the softmax exponentials from the MUFU, the limit
// of the forward softmax.  Inputs of -inf / below -126 give 0.
BP_DEV float ex2_fma(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.05517025f, 0.24260790f);
  p = fmaf(f, p, 0.69326093f);
  p = fmaf(f, p, 0.99992828f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// Packed fp32 pairs (sm_100: FFMA2 / FADD2 -- one issue slot for two
// lanes' worth of work) and the 3-input max (FMNMX3): the forward softmax is
// issue-bound (tools/attn_fwd_trace.py), so these cut its instruction count
// without changing a single rounding (same .rn ops per element).
BP_DEV uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
BP_DEV void f2unpack(uint64_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
BP_DEV uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
BP_DEV uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
BP_DEV uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// P^T = 2^(s scale - lse log2 e) and dS^T = P^T (dP^T - delta) for a pair of
// queries (FMUL2 / FFMA2 / FADD2 / FMUL2: the roundings of the scalar form)
BP_DEV void pds2(float& s0, float& s1, float& d0, float& d1, float l0, float l1, float dl0, float dl1,
                 uint64_t sc2) {
  const uint64_t nl = fmul2(f2pack(l0, l1), f2pack(-kLog2e, -kLog2e));
  float x0, x1;
  f2unpack(ffma2(f2pack(s0, s1), sc2, nl), x0, x1);
  s0 = ex2(x0);
  s1 = ex2(x1);
  f2unpack(fmul2(f2pack(s0, s1), fadd2(f2pack(d0, d1), f2pack(-dl0, -dl1))), d0, d1);
}

BP_DEV float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// ex2_fma on a packed pair (same split and cubic, FFMA2 / FADD2)
BP_DEV uint64_t ex2_fma2(float x0, float x1) {
  const uint64_t x = f2pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t mg = f2pack(12582912.f, 12582912.f), nmg = f2pack(-12582912.f, -12582912.f);
  const uint64_t t = fadd2(x, mg);
  float t0, t1, u0, u1;
  f2unpack(fadd2(t, nmg), u0, u1);
  const uint64_t f = fadd2(x, f2pack(-u0, -u1));
  uint64_t p = ffma2(f, f2pack(0.05517025f, 0.05517025f), f2pack(0.24260790f, 0.24260790f));
  p = ffma2(f, p, f2pack(0.69326093f, 0.69326093f));
  p = ffma2(f, p, f2pack(0.99992828f, 0.99992828f));
  float p0, p1;
  f2unpack(p, p0, p1);
  f2unpack(t, t0, t1);
  return f2pack(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
                __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
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

// 32 consecutive bf16 (64 B, 32-byte aligned) from 32 floats as two 256-bit
// stores: whole 32-byte sectors (a thread's row segment; the rows of a warp
// are strided, so 128-bit stores left every sector half written)
BP_DEV void st_row32_bf16(__nv_bfloat16* dst, const float* v) {
  const uint4 a = pack8(v), b = pack8(v + 8), c = pack8(v + 16), d = pack8(v + 24);
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 16), "r"(c.x), "r"(c.y), "r"(c.z),
               "r"(c.w), "r"(d.x), "r"(d.y), "r"(d.z), "r"(d.w)
               : "memory");
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
// 384 threads: warp 0 TMA, warp 1 MMA, warp 2 TMEM allocator, warps 4-11
// softmax.  Softmax warp w owns TMEM lane quarter (w & 3) -- 32 query rows --
// and column half hh = (w - 4) >> 2 of every 128-key score tile, so each
// thread handles 64 scores per tile; the two halves of a row exchange their
// partial maxima through shared memory (named barrier per lane quarter) and
// each half rescales / stores its own half of the O columns.
template <int Dh>
struct Fwd {
  static constexpr int DC = Dh / 64;
  static constexpr int KS = 3;  // K ring depth (a K slot frees when S is done, a V slot only after P V)
  static constexpr uint32_t TILE = 128 * Dh * 2;
  static constexpr size_t SMEM = 1024 + TILE + KS * TILE + 2 * TILE + 2048 + 512;
};

// EXF of every 8 exponentials run on the FMA pipe (ex2_fma), the rest on
// the MUFU (16 lanes / clk / SM: the softmax's exponential phase is
// MUFU-bound at EXF = 2, tools/attn_fwd_trace.py)
template <int EXF>
BP_DEV bool exp_on_fma(int i) {
  const int k = i & 7;
  if (EXF <= 0 || EXF >= 6) return false;
  if (EXF == 2) return k == 3 || k == 7;
  if (EXF == 3) return k == 2 || k == 5 || k == 7;
  if (EXF == 4) return (k & 1) == 1;
  if (EXF == 5) return (k & 1) == 1 || k == 4;
  return k == 3 || k == 7;
}
// EXF >= 6: whole pairs on the FMA pipe (packed ex2_fma2): EXF - 4 of the 8
// pairs of every 16 exponentials
template <int EXF>
BP_DEV bool pair_on_fma(int i) {
  const int k = (i >> 1) & 7;
  if (EXF == 6) return k == 3 || k == 7;
  if (EXF == 7) return k == 2 || k == 5 || k == 7;
  if (EXF == 8) return (k & 1) == 1;
  return false;
}

template <int Dh, bool CAUSAL, int EXF = 2>
__global__ void __launch_bounds__(384, 1)
fwd_tc(const __grid_constant__ CUtensorMap map_qkv, __nv_bfloat16* __restrict__ o, float* __restrict__ lse, int S,
       int H, float scale_log2) {
  using C = Fwd<Dh>;
  constexpr int KS = C::KS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK0 = smem + C::TILE;              // K slot s at sK0 + s TILE
  uint8_t* sV0 = sK0 + KS * C::TILE;          // V slot s at sV0 + s TILE
  float* sX = reinterpret_cast<float*>(sV0 + 2 * C::TILE);  // [2 parity][2 halves][128 rows] partial maxima
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV0 + 2 * C::TILE + 2048);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;        // [KS]
  uint64_t* k_empty = bars + 1 + KS;  // [KS]
  uint64_t* v_full = bars + 1 + 2 * KS;   // [2]
  uint64_t* v_empty = v_full + 2;         // [2]
  uint64_t* s_full = v_full + 4;          // [3]
  uint64_t* s_free = v_full + 7;          // [3]
  // P(j) ready: one barrier per j mod 4.  S(j+2) is issued right after P V(j),
  // so a softmax warp can run up to three tiles ahead of a slower one (S(j+3)
  // only waits for every warp to have READ S(j)); with fewer barriers its
  // arrival for a later tile would complete tile j's phase early
  uint64_t* p_full = v_full + 10;  // [4]
  uint64_t* pv_done = v_full + 14;
  uint64_t* o_done = v_full + 15;  // single phase: every P V of the CTA complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_full + 16);
  // TMEM: three S buffers [0,128), [128,256), [256,384) -- S(j+2) is computed
  // while the softmax of tile j runs, so the softmax of tile j+1 never waits
  // for its scores (with two buffers S(j+1) could only be issued after
  // P V(j-1), ~300 cycles of every 2,200-cycle tile spent waiting) -- P of
  // tile j written back as bf16 over the first 64 columns of its S buffer
  // (the TMEM A operand of O += P V); O [384, 384+Dh)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x, qt = gridDim.y - 1 - blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int n_kv = CAUSAL ? qt + 1 : S / 128;
  const int HD = H * Dh;

  if (warp == 0 && lane == 0) tma_prefetch_desc(&map_qkv);
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 256);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&p_full[i], 256);
    mbar_init(pv_done, 1);
    mbar_init(o_done, 1);
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
      // K runs up to KS tiles ahead, V two; interleave so that neither waits
      // behind the other's (later) free slot
      int jk = 0, jv = 0;
      while (jv < n_kv) {
        if (jk < n_kv && jk < jv + KS) {
          const int st = jk % KS;
          mbar_wait(&k_empty[st], ((jk / KS) & 1) ^ 1);
          TRACE_MMA(32 + jk, 10);
#pragma unroll
          for (int c = 0; c < C::DC; ++c)
            tma_load_2d(sK0 + st * C::TILE + c * 16384, &map_qkv, HD + h * Dh + c * 64, b * S + jk * 128, &k_full[st]);
          mbar_expect_tx(&k_full[st], C::TILE);
          ++jk;
        }
        if (jv < jk - 1 || jk == n_kv) {
          const int st = jv & 1;
          mbar_wait(&v_empty[st], ((jv >> 1) & 1) ^ 1);
#pragma unroll
          for (int c = 0; c < C::DC; ++c)
            tma_load_2d(sV0 + st * C::TILE + c * 16384, &map_qkv, 2 * HD + h * Dh + c * 64, b * S + jv * 128,
                        &v_full[st]);
          mbar_expect_tx(&v_full[st], C::TILE);
          ++jv;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, Dh, false, true);
      const uint32_t aQ = smem_u32(sQ);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int j) {   // S(j) into buffer j % 3
        const int sb = j % 3, ks_ = j % KS;
        TRACE_MMA(32 + j, 11);
        mbar_wait(&k_full[ks_], (j / KS) & 1);
        TRACE_MMA(32 + j, 12);
        mbar_wait(&s_free[sb], ((j / 3) & 1) ^ 1);   // every softmax thread has read S(j - 3)
        TRACE_MMA(32 + j, 8);
        tc_fence_after();
        const uint32_t aK = smem_u32(sK0 + ks_ * C::TILE);
#pragma unroll
        for (int ks = 0; ks < Dh / 16; ++ks)
          tc_mma_f16(tmem + sb * 128, kdesc(aQ, ks, 128), kdesc(aK, ks, 128), idesc_s, ks > 0);
        tc_commit(&s_full[sb]);
        tc_commit(&k_empty[ks_]);
      };
      issue_s(0);
      if (n_kv > 1) issue_s(1);
      for (int jj = 0; jj < n_kv; ++jj) {
        const int vs = jj & 1;
        TRACE_MMA(32 + jj, 13);
        mbar_wait(&p_full[jj & 3], (jj >> 2) & 1);
        TRACE_MMA(32 + jj, 14);
        mbar_wait(&v_full[vs], (jj >> 1) & 1);
        TRACE_MMA(32 + jj, 9);
        tc_fence_after();
        const uint32_t aV = smem_u32(sV0 + vs * C::TILE);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc_mma_f16_ts(tmem + 384, tmem + (jj % 3) * 128 + 8 * ks, mndesc(aV, ks, 128), idesc_o, (jj > 0 || ks > 0));
        TRACE_MMA(32 + jj, 15);
        tc_commit(pv_done);
        tc_commit(&v_empty[vs]);
        if (jj == n_kv - 1) tc_commit(o_done);
        // after P V(jj) in the in-order tensor pipe: S(jj + 2) overwrites the
        // buffer of P(jj - 1), which P V(jj - 1) has consumed
        if (jj + 2 < n_kv) issue_s(jj + 2);
      }
    }
  } else if (warp >= 4) {  // ---------------------------------- softmax
    const int wq = warp & 3, hh = (warp - 4) >> 2;
    const int r = wq * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(wq * 32) << 16);
    constexpr int OC = Dh / 64;  // 32-column O chunks per half
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int st = j % 3;
      TRACE(32 + j, 0);
      mbar_wait(&s_full[st], (j / 3) & 1);
      TRACE(32 + j, 1);
      tc_fence_after();
      float s[64];
      tmem_ld_32x32b_x64(tl + st * 128 + hh * 64, s);
      tc_fence_before();
      mbar_arrive(&s_free[st]);
      TRACE(32 + j, 2);
      const bool diag = CAUSAL && (j == qt);
      // max over the raw scores (scale > 0), the scale folds into the exponent FMA
      if (diag) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (hh * 64 + i > r) s[i] = -INFINITY;
      }
      float m4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) m4[e] = fmaxf(s[2 * e], s[2 * e + 1]);
#pragma unroll
      for (int i = 8; i < 64; i += 2) m4[(i >> 1) & 3] = fmax3(m4[(i >> 1) & 3], s[i], s[i + 1]);
      float mx = scale_log2 * fmax3(fmaxf(m4[0], m4[1]), m4[2], m4[3]);
      float* xs = sX + (j & 1) * 256;
      xs[hh * 128 + r] = mx;
      named_bar_sync(1 + wq, 64);
      mx = fmaxf(mx, xs[(hh ^ 1) * 128 + r]);
      TRACE(32 + j, 3);
      // lazy rescale (only when a row max grew by > 2^8).  The decision is
      // per row but tcgen05.ld / st are .sync.aligned warp collectives: the
      // whole warp rescales when any of its rows needs it (f = 1 for the
      // others) -- a partial-warp tcgen05.ld hangs the CTA
      const bool up = mx > m_used + 8.f;
      if (j > 0 && __any_sync(0xffffffffu, up)) {  // rescale O: needs P V of tile j-1 complete
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
        const float f = up ? ex2(m_used - mx) : 1.f;
#pragma unroll 1
        for (int c = 0; c < OC; ++c) {
          float ov[32];
          const uint32_t ta = tl + 384 + (hh * OC + c) * 32;
          tmem_ld_32x32b_x32(ta, ov);
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] *= f;
          tmem_st_32x32b_x32(ta, ov);
        }
        l *= f;
      }
      if (up) m_used = mx;
      TRACE(32 + j, 4);
      // x = s scale - m and the row-sum partials on packed pairs: l2[k] holds
      // the partial sums of elements i = 8n + 2k, 8n + 2k + 1
      const uint64_t sc2 = f2pack(scale_log2, scale_log2), nm2 = f2pack(-m_used, -m_used);
      uint64_t l2[4];
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        float x0, x1;
        f2unpack(ffma2(f2pack(s[i], s[i + 1]), sc2, nm2), x0, x1);
        uint64_t e2;
        if (EXF >= 6 && pair_on_fma<EXF>(i)) {
          e2 = ex2_fma2(x0, x1);
          f2unpack(e2, s[i], s[i + 1]);
        } else {
          s[i] = exp_on_fma<EXF>(i) ? ex2_fma(x0) : ex2(x0);  // EXF / 8 on the FMA pipe
          s[i + 1] = exp_on_fma<EXF>(i + 1) ? ex2_fma(x1) : ex2(x1);
          e2 = f2pack(s[i], s[i + 1]);
        }
        l2[(i >> 1) & 3] = i < 8 ? e2 : fadd2(l2[(i >> 1) & 3], e2);
      }
      float l8[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) f2unpack(l2[e], l8[2 * e], l8[2 * e + 1]);
      l += ((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7]));
      TRACE(32 + j, 5);
      // P (bf16 pairs) over this half's 32 of the S buffer's first 64 columns
      // (already read by both halves: s_free); P V of tile j-2 that read this
      // buffer completed before S(j) (in-order tensor pipe)
      float pk[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) pk[i] = __uint_as_float(pack_bf16x2(s[2 * i], s[2 * i + 1]));
      TRACE(32 + j, 6);
      tmem_st_32x32b_x32(tl + st * 128 + hh * 32, pk);
      tc_fence_before();
      mbar_arrive(&p_full[j & 3]);
      TRACE(32 + j, 7);
    }
    // epilogue: O / l (l = sum of both halves' partial sums)
    float* xs = sX + (n_kv & 1) * 256;
    xs[hh * 128 + r] = l;
    named_bar_sync(1 + wq, 64);
    l += xs[(hh ^ 1) * 128 + r];
    // not a parity wait on pv_done: that is ambiguous while P V(n_kv-2) may
    // still be in flight (the last S commit only covers P V(n_kv-3))
    mbar_wait(o_done, 0);
    tc_fence_after();
    const int q = qt * 128 + r;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = o + ((int64_t)b * S + q) * HD + h * Dh;
#pragma unroll 1
    for (int c = hh * OC; c < (hh + 1) * OC; ++c) {
      float ov[32];
      tmem_ld_32x32b_x32(tl + 384 + c * 32, ov);
#pragma unroll
      for (int i = 0; i < 32; ++i) ov[i] *= inv;
      st_row32_bf16(orow + c * 32, ov);
    }
    if (hh == 0) lse[((int64_t)b * H + h) * S + q] = (m_used + log2f(l)) * kLn2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ================================================ forward, two Q tiles ====
// CTA = two 128-row query tiles A = 2t, B = 2t + 1 of one (batch, head),
// 352 threads: warp 0 TMA, warp 1 TMEM allocator + MMA issuer of tile A,
// warp 2 MMA issuer of tile B, warps 3-6 softmax of A, warps 7-10 softmax of
// B (warp w owns TMEM lane quarter w & 3 = 32 query rows, whole 128-key score
// rows per thread).  K / V tiles are loaded once for both query tiles, on
// separate K and V rings (a K slot frees when both S MMAs are done, a V slot
// when both P V MMAs are).  The two tiles are independent pipelines, so
// while group A exponentiates S_A(j) the tensor pipe runs tile B's MMAs.  P
// is written back as bf16 over the S columns it came from and is the TMEM A
// operand of O += P V; shared memory only holds Q / K / V.  TMEM: S_A
// [0,128), S_B [128,256), O_A [256, 256+Dh), O_B [256+Dh, 256+2Dh).
template <int Dh>
struct Fwd2 {
  static constexpr int DC = Dh / 64;
  static constexpr uint32_t TILE = 128 * Dh * 2;
  static constexpr size_t SMEM = 1024 + 2 * TILE + 4 * TILE + 512;  // Q_A, Q_B, 2 x (K, V)
};

template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(352, 1)
fwd2_tc(const __grid_constant__ CUtensorMap map_qkv, __nv_bfloat16* __restrict__ o, float* __restrict__ lse, int S,
        int H, float scale_log2) {
  using C = Fwd2<Dh>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;  // tile X at sQ + X * TILE
  uint8_t* sKV = smem + 2 * C::TILE;  // stage s: K at sKV + 2 s TILE, V right after
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * C::TILE);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;    // [2] ring slots
  uint64_t* k_empty = bars + 3;   // [2]
  uint64_t* v_full = bars + 5;    // [2]
  uint64_t* v_empty = bars + 7;   // [2]
  uint64_t* s_full = bars + 9;    // [2] per query tile
  uint64_t* p_full = bars + 11;   // [2]
  uint64_t* o_done = bars + 13;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x, t = gridDim.y - 1 - blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int n_all = S / 128;
  const int nA = CAUSAL ? 2 * t + 1 : n_all, nB = CAUSAL ? 2 * t + 2 : n_all;
  const int HD = H * Dh;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_qkv);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 2);  // one commit per query tile
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 2);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------ producer
#pragma unroll
      for (int X = 0; X < 2; ++X) {
        const int qrow = b * S + (2 * t + X) * 128;
#pragma unroll
        for (int c = 0; c < C::DC; ++c)
          tma_load_2d(sQ + X * C::TILE + c * 16384, &map_qkv, h * Dh + c * 64, qrow, q_full);
      }
      mbar_expect_tx(q_full, 2 * C::TILE);
      for (int j = 0; j < nB; ++j) {
        const int st = j & 1, ph = ((j >> 1) & 1) ^ 1;
        const int krow = b * S + j * 128;
        uint8_t* sk = sKV + st * 2 * C::TILE;
        mbar_wait(&k_empty[st], ph);
        TRACE_MMA(32 + j, 13);
#pragma unroll
        for (int c = 0; c < C::DC; ++c) tma_load_2d(sk + c * 16384, &map_qkv, HD + h * Dh + c * 64, krow, &k_full[st]);
        mbar_expect_tx(&k_full[st], C::TILE);
        mbar_wait(&v_empty[st], ph);
        TRACE_MMA(32 + j, 14);
#pragma unroll
        for (int c = 0; c < C::DC; ++c)
          tma_load_2d(sk + C::TILE + c * 16384, &map_qkv, 2 * HD + h * Dh + c * 64, krow, &v_full[st]);
        mbar_expect_tx(&v_full[st], C::TILE);
      }
    }
  } else if (warp <= 2) {
    if (lane == 0) {  // ------------------------ MMA issuer of query tile X
      const int X = warp - 1, n = X ? nB : nA;
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, Dh, false, true);
      const uint32_t aQ = smem_u32(sQ + X * C::TILE);
      const uint32_t tS = tmem + X * 128, tO = tmem + 256 + X * Dh;
      mbar_wait(q_full, 0);
      // tile B starts half a period behind tile A, so one group exponentiates
      // while the other's MMAs run (in lock-step both would contend for the
      // MUFU and then leave the tensor pipe idle together)
      if (X == 1 && n > 1) mbar_wait(&p_full[0], 0);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        TRACE_MMA(32 + j, X ? 12 : 10);
        tc_fence_after();
        const uint32_t aK = smem_u32(sKV + st * 2 * C::TILE);
#pragma unroll
        for (int ks = 0; ks < Dh / 16; ++ks) tc_mma_f16(tS, kdesc(aQ, ks, 128), kdesc(aK, ks, 128), idesc_s, ks > 0);
        tc_commit(&s_full[X]);
        tc_commit(&k_empty[st]);
      };
      issue_s(0);
      for (int j = 0; j < n; ++j) {
        const int st = j & 1;
        mbar_wait(&p_full[X], j & 1);
        TRACE_MMA(32 + j, X ? 11 : 8);
        mbar_wait(&v_full[st], (j >> 1) & 1);
        if (!X) TRACE_MMA(32 + j, 9);
        tc_fence_after();
        const uint32_t aV = smem_u32(sKV + st * 2 * C::TILE + C::TILE);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)  // 128 keys / 16
          tc_mma_f16_ts(tO, tS + 8 * ks, mndesc(aV, ks, 128), idesc_o, (j > 0 || ks > 0));
        tc_commit(&v_empty[st]);
        if (j + 1 < n)
          issue_s(j + 1);
        else
          tc_commit(&o_done[X]);
      }
    }
  } else {  // -------------------------------------------- softmax (warps 3-10)
    const int X = (warp - 3) >> 2, wq = warp & 3;
    const int r = wq * 32 + lane;  // query row within the tile
    const int qt = 2 * t + X, n = X ? nB : nA;
    const uint32_t tl = tmem + ((uint32_t)(wq * 32) << 16);
    const uint32_t tS = tl + X * 128, tO = tl + 256 + X * Dh;
    float m_used = -INFINITY, l = 0.f;  // m_used in the scaled (log2) domain
    for (int j = 0; j < n; ++j) {
      if (threadIdx.x == 96) TRACE_MMA(32 + j, 0);
      mbar_wait(&s_full[X], j & 1);
      if (threadIdx.x == 96) TRACE_MMA(32 + j, 1);
      tc_fence_after();
      // registers hold half a score row at a time (the group's 10 warps
      // allocate as 12, so 168 registers per thread): pass 1 takes the row
      // max over two 64-column loads, pass 2 reloads, exponentiates and
      // writes P back over the first 64 columns
      const bool diag = CAUSAL && j == qt;
      // 8 independent max / sum accumulators: a single running fmaxf / fadd
      // is a 128-long dependency chain (~4 cycles per link)
      // (3-input maxima: 4 accumulators, two scores per FMNMX3)
      float m4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) m4[e] = -INFINITY;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float s[64];
        tmem_ld_32x32b_x32_pair(tS + 64 * hf, tS + 64 * hf + 32, *reinterpret_cast<float(*)[32]>(s),
                                *reinterpret_cast<float(*)[32]>(s + 32));
        if (diag) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (64 * hf + i > r) s[i] = -INFINITY;
        }
#pragma unroll
        for (int i = 0; i < 64; i += 2) m4[(i >> 1) & 3] = fmax3(m4[(i >> 1) & 3], s[i], s[i + 1]);
      }
      const float mx = fmax3(fmaxf(m4[0], m4[1]), m4[2], m4[3]);
      if (threadIdx.x == 96) TRACE_MMA(32 + j, 2);
      const float mxs = mx * scale_log2;
      const bool up = mxs > m_used + 8.f;  // warp-uniform rescale (see fwd_tc)
      if (j > 0 && __any_sync(0xffffffffu, up)) {  // O_X holds PV(j-1) complete: S_X(j) was issued after it
        const float f = up ? ex2(m_used - mxs) : 1.f;
#pragma unroll 1
        for (int c = 0; c < Dh / 32; ++c) {
          float ov[32];
          tmem_ld_32x32b_x32(tO + c * 32, ov);
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] *= f;
          tmem_st_32x32b_x32(tO + c * 32, ov);
        }
        l *= f;
      }
      if (up) m_used = mxs;
      if (threadIdx.x == 96) TRACE_MMA(32 + j, 3);
      // x = s scale - m and the row-sum partials on packed pairs (FFMA2 /
      // FADD2; l2[k] = the partial sums of elements 8n + 2k, 8n + 2k + 1)
      const uint64_t sc2 = f2pack(scale_log2, scale_log2), nm2 = f2pack(-m_used, -m_used);
      uint64_t l2[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) l2[e] = 0;  // +0.0f pairs
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float s[64];
        tmem_ld_32x32b_x32_pair(tS + 64 * hf, tS + 64 * hf + 32, *reinterpret_cast<float(*)[32]>(s),
                                *reinterpret_cast<float(*)[32]>(s + 32));
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          float x0, x1;
          f2unpack(ffma2(f2pack(s[i], s[i + 1]), sc2, nm2), x0, x1);
          s[i] = diag && 64 * hf + i > r ? 0.f : ex2(x0);
          s[i + 1] = diag && 64 * hf + i + 1 > r ? 0.f : ex2(x1);
          l2[(i >> 1) & 3] = fadd2(l2[(i >> 1) & 3], f2pack(s[i], s[i + 1]));
        }
        float pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = __uint_as_float(pack_bf16x2(s[2 * i], s[2 * i + 1]));
        // P columns [32 hf, 32 hf + 32) overwrite S columns already read
        tmem_st_32x32b_x32(tS + 32 * hf, pk);
      }
      float l8[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) f2unpack(l2[e], l8[2 * e], l8[2 * e + 1]);
      l += ((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7]));
      if (threadIdx.x == 96) TRACE_MMA(32 + j, 4);
      tc_fence_before();
      mbar_arrive(&p_full[X]);
      if (threadIdx.x == 96) TRACE_MMA(32 + j, 5);
    }
    mbar_wait(&o_done[X], 0);
    tc_fence_after();
    const int q = qt * 128 + r;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = o + ((int64_t)b * S + q) * HD + h * Dh;
#pragma unroll 1
    for (int c = 0; c < Dh / 32; ++c) {
      float ov[32];
      tmem_ld_32x32b_x32(tO + c * 32, ov);
#pragma unroll
      for (int i = 0; i < 32; ++i) ov[i] *= inv;
      st_row32_bf16(orow + c * 32, ov);
    }
    lse[((int64_t)b * H + h) * S + q] = (m_used + log2f(l)) * kLn2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// =================================================== backward: dK, dV ====
// CTA = 128 keys, 384 threads.  Two compute warpgroups ping-pong over the
// 64-query tiles (warps 4-7 take even tiles, warps 8-11 odd ones), so one
// group's exp / dS math overlaps the other's and the tensor pipe always has
// the next S^T / dP^T pair queued (double-buffered in TMEM).  P^T and dS^T
// are written back as bf16 into the TMEM columns their S^T / dP^T came from
// and feed dV += P^T dO and dK += dS^T Q as tensor-memory A operands, so the
// shared-memory port (the bound of this kernel) only serves the Q / dO / K /
// V operand reads.  Q / dO / LSE / delta stream through a QST-deep TMA ring.
template <int Dh>
struct Dkdv {
  static constexpr int DC = Dh / 64;
  static constexpr int QST = 4;
  static constexpr uint32_t KT = 128 * Dh * 2;  // K / V tile (128 keys)
  static constexpr uint32_t QT = 64 * Dh * 2;   // Q / dO tile (64 queries)
  static constexpr size_t SMEM = 1024 + 2 * KT + QST * 2 * QT + QST * 512 + 512;
};

BP_DEV float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(384, 1)
dkdv_tc(const __grid_constant__ CUtensorMap map_kv, const __grid_constant__ CUtensorMap map_q,
        const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse, const float* __restrict__ delta,
        __nv_bfloat16* __restrict__ dqkv, float* __restrict__ dbias, int S, int H, float scale, float scale_log2,
        __nv_bfloat16* __restrict__ ds_t) {
  using C = Dkdv<Dh>;
  constexpr int QST = C::QST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::KT;
  uint8_t* sQ0 = smem + 2 * C::KT;  // stage s: Q at sQ0 + 2 s QT, dO right after
  float* sL0 = reinterpret_cast<float*>(sQ0 + QST * 2 * C::QT);  // stage s: 64 lse then 64 delta
  uint64_t* bars = reinterpret_cast<uint64_t*>(sQ0 + QST * 2 * C::QT + QST * 512);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;          // [QST]
  uint64_t* q_empty = bars + 1 + QST;   // [QST]
  uint64_t* sdp_full = bars + 1 + 2 * QST;  // [2]
  uint64_t* sdp_free = sdp_full + 2;        // [2]
  uint64_t* p_full = sdp_full + 4;          // [2]
  uint64_t* all_done = sdp_full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sdp_full + 9);
  // TMEM columns: buffer g: S^T [128g, 128g+64) -> P^T bf16 in [128g, 128g+32),
  //               dP^T [128g+64, 128g+128) -> dS^T bf16 in [128g+64, 128g+96);
  //               dV [256, 256+Dh), dK [256+Dh, 256+2Dh)
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
    for (int i = 0; i < QST; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&sdp_full[g], 1);
      mbar_init(&sdp_free[g], 128);
      mbar_init(&p_full[g], 128);
    }
    mbar_init(all_done, 1);
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
        const int st = it % QST, qi = q0 + it;
        mbar_wait(&q_empty[st], ((it / QST) & 1) ^ 1);
        TRACE_MMA(it, 12);
        const int qrow = b * S + qi * 64;
        uint8_t* sq = sQ0 + st * 2 * C::QT;
#pragma unroll
        for (int c = 0; c < C::DC; ++c) {
          tma_load_2d(sq + c * 8192, &map_q, h * Dh + c * 64, qrow, &q_full[st]);
          tma_load_2d(sq + C::QT + c * 8192, &map_do, h * Dh + c * 64, qrow, &q_full[st]);
        }
        const int64_t lrow = ((int64_t)b * H + h) * S + qi * 64;
        bulk_load(sL0 + st * 128, lse + lrow, 256, &q_full[st]);
        bulk_load(sL0 + st * 128 + 64, delta + lrow, 256, &q_full[st]);
        mbar_expect_tx(&q_full[st], 2 * C::QT + 512);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 64, false, false);  // S^T, dP^T: M=keys, N=64 q
      constexpr uint32_t idesc_g = umma_idesc_bf16(128, Dh, false, true);   // dV, dK: B MN-major
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      auto issue_sdp = [&](int it) {
        const int st = it % QST, g = it & 1;
        TRACE_MMA(it, 8);
        mbar_wait(&q_full[st], (it / QST) & 1);
        TRACE_MMA(it, 9);
        mbar_wait(&sdp_free[g], ((it >> 1) & 1) ^ 1);
        TRACE_MMA(it, 10);
        tc_fence_after();
        const uint32_t aQ = smem_u32(sQ0 + st * 2 * C::QT), aO = aQ + C::QT;
#pragma unroll
        for (int ks = 0; ks < Dh / 16; ++ks) {
          tc_mma_f16(tmem + g * 128, kdesc(aK, ks, 128), kdesc(aQ, ks, 64), idesc_s, ks > 0);
          tc_mma_f16(tmem + g * 128 + 64, kdesc(aV, ks, 128), kdesc(aO, ks, 64), idesc_s, ks > 0);
        }
        tc_commit(&sdp_full[g]);
      };
      issue_sdp(0);
      if (n_it > 1) issue_sdp(1);
      for (int it = 0; it < n_it; ++it) {
        const int st = it % QST, g = it & 1;
        mbar_wait(&p_full[g], (it >> 1) & 1);
        TRACE_MMA(it, 11);
        tc_fence_after();
        const uint32_t aQ = smem_u32(sQ0 + st * 2 * C::QT), aO = aQ + C::QT;
        const uint32_t tP = tmem + g * 128, tD = tP + 64;  // P^T / dS^T as TMEM A operands
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {  // 64 queries / 16
          tc_mma_f16_ts(tmem + 256, tP + 8 * ks, mndesc(aO, ks, 64), idesc_g, (it > 0 || ks > 0));
          tc_mma_f16_ts(tmem + 256 + Dh, tD + 8 * ks, mndesc(aQ, ks, 64), idesc_g, (it > 0 || ks > 0));
        }
        tc_commit(&q_empty[st]);
        if (it + 2 < n_it) issue_sdp(it + 2);
      }
      tc_commit(all_done);
    }
  } else if (warp >= 4) {  // -------------------------- P^T / dS^T rows
    const int wq = warp & 3, g = (warp - 4) >> 2;
    const int r = wq * 32 + lane;  // key row in the tile
    const int key = kt * 128 + r;
    const uint32_t tl = tmem + ((uint32_t)(wq * 32) << 16) + g * 128;
    const uint64_t ds_pol = l2_policy_evict_last();
    for (int it = g; it < n_it; it += 2) {
      const int st = it % QST, qi = q0 + it, u = it >> 1;
      TRACE(it, 0);
      mbar_wait(&q_full[st], (it / QST) & 1);  // lse / delta of this tile are in smem
      TRACE(it, 1);
      mbar_wait(&sdp_full[g], u & 1);
      TRACE(it, 2);
      tc_fence_after();
      const uint32_t aL = smem_u32(sL0 + st * 128);
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        float sv[32], dp[32];
        tmem_ld_32x32b_x32_pair(tl + hf * 32, tl + 64 + hf * 32, sv, dp);
        if (hf == 1) {
          tc_fence_before();
          mbar_arrive(&sdp_free[g]);
        }
        TRACE(it, 3);
        const int qb = qi * 64 + hf * 32;
        if (CAUSAL && qb < key) {  // some query of this half precedes the key
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 l4 = lds4(aL + 4 * (hf * 32 + 4 * k)), d4 = lds4(aL + 256 + 4 * (hf * 32 + 4 * k));
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dl[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = 4 * k + e;
              float p = ex2(fmaf(sv[i], scale_log2, -lv[e] * kLog2e));
              p = qb + i < key ? 0.f : p;
              sv[i] = p;
              dp[i] = p * (dp[i] - dl[e]);
            }
          }
        } else {
          const uint64_t sc2 = f2pack(scale_log2, scale_log2);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 l4 = lds4(aL + 4 * (hf * 32 + 4 * k)), d4 = lds4(aL + 256 + 4 * (hf * 32 + 4 * k));
            const int i = 4 * k;
            pds2(sv[i], sv[i + 1], dp[i], dp[i + 1], l4.x, l4.y, d4.x, d4.y, sc2);
            pds2(sv[i + 2], sv[i + 3], dp[i + 2], dp[i + 3], l4.z, l4.w, d4.z, d4.w, sc2);
          }
        }
        TRACE(it, 4);
        // P^T / dS^T (bf16 pairs) over the S^T / dP^T columns just read; the
        // dV/dK MMAs of tile it - 2 that read this buffer completed before
        // this tile's S^T / dP^T MMAs (in-order tensor pipe)
        uint32_t pk[16], dk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          pk[i] = pack_bf16x2(sv[2 * i], sv[2 * i + 1]);
          dk[i] = pack_bf16x2(dp[2 * i], dp[2 * i + 1]);
        }
        tmem_st_32x32b_x16(tl + hf * 16, pk);
        tmem_st_32x32b_x16(tl + 64 + hf * 16, dk);
        if (ds_t) {  // dS^T row of this key, 32 queries (64 B), for the dQ GEMM: two
                     // 256-bit stores, each a whole 32-byte sector (no partial-sector writes),
                     // evict_last in L2: the dQ GEMM reads them right after this kernel
          uint32_t* dst = reinterpret_cast<uint32_t*>(ds_t + ((int64_t)bh * S + key) * S + qi * 64 + hf * 32);
#pragma unroll
          for (int u = 0; u < 2; ++u)
            asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(dst + 8 * u),
                         "r"(dk[8 * u]), "r"(dk[8 * u + 1]), "r"(dk[8 * u + 2]), "r"(dk[8 * u + 3]),
                         "r"(dk[8 * u + 4]), "r"(dk[8 * u + 5]), "r"(dk[8 * u + 6]), "r"(dk[8 * u + 7]),
                         "l"(ds_pol)
                         : "memory");
        }
        TRACE(it, 5);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[g]);
      TRACE(it, 6);
    }
    // epilogue: dV, dK (scaled) -> dqkv; group g writes 32-column chunks g, g+2, ...
    mbar_wait(all_done, 0);
    tc_fence_after();
    const uint32_t te = tmem + ((uint32_t)(wq * 32) << 16) + 256;
    __nv_bfloat16* dkrow = dqkv + ((int64_t)b * S + key) * 3 * HD + HD + h * Dh;
    __nv_bfloat16* dvrow = dkrow + HD;
#pragma unroll 1
    for (int c = g; c < Dh / 32; c += 2) {
      float v[32];
      tmem_ld_32x32b_x32(te + c * 32, v);
      st_row32_bf16(dvrow + c * 32, v);
      if (dbias) {  // V-bias gradient: column sums of this warp's 32 keys, as stored
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = bf16_round(v[i]);
        atomicAdd(dbias + 2 * HD + h * Dh + c * 32 + lane, warp_colsum32(v, lane));
      }
      tmem_ld_32x32b_x32(te + Dh + c * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= scale;
      st_row32_bf16(dkrow + c * 32, v);
      if (dbias) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = bf16_round(v[i]);
        atomicAdd(dbias + HD + h * Dh + c * 32 + lane, warp_colsum32(v, lane));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ========================================================= backward: dQ ====
// CTA = 128 queries, 384 threads; two compute warpgroups ping-pong over the
// 64-key tiles exactly as in dkdv_tc (S / dP double-buffered in TMEM; dS is
// written back as bf16 over its dP columns and is the TMEM A operand of
// dQ += dS K); K / V stream through a KST-deep ring.
template <int Dh>
struct Dq {
  static constexpr int DC = Dh / 64;
  static constexpr int KST = 4;
  static constexpr uint32_t QT = 128 * Dh * 2;  // Q / dO tile (128 queries)
  static constexpr uint32_t KT = 64 * Dh * 2;   // K / V tile (64 keys)
  static constexpr size_t SMEM = 1024 + 2 * QT + KST * 2 * KT + 512;
};

template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(384, 1)
dq_tc(const __grid_constant__ CUtensorMap map_q128, const __grid_constant__ CUtensorMap map_kv64,
      const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse, const float* __restrict__ delta,
      __nv_bfloat16* __restrict__ dqkv, float* __restrict__ dbias, int S, int H, float scale, float scale_log2) {
  using C = Dq<Dh>;
  constexpr int KST = C::KST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sO = smem + C::QT;
  uint8_t* sK0 = smem + 2 * C::QT;  // stage s: K at sK0 + 2 s KT, V right after
  uint64_t* bars = reinterpret_cast<uint64_t*>(sK0 + KST * 2 * C::KT);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;          // [KST]
  uint64_t* kv_empty = bars + 1 + KST;   // [KST]
  uint64_t* sdp_full = bars + 1 + 2 * KST;  // [2]
  uint64_t* sdp_free = sdp_full + 2;        // [2]
  uint64_t* p_full = sdp_full + 4;          // [2]
  uint64_t* all_done = sdp_full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sdp_full + 9);
  // TMEM: buffer g: S [128g, 128g+64), dP [128g+64, 128g+128) -> dS bf16 in
  //       [128g+64, 128g+96); dQ [256, 256+Dh)
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
    for (int i = 0; i < KST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&sdp_full[g], 1);
      mbar_init(&sdp_free[g], 128);
      mbar_init(&p_full[g], 128);
    }
    mbar_init(all_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
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
        const int st = it % KST;
        mbar_wait(&kv_empty[st], ((it / KST) & 1) ^ 1);
        const int krow = b * S + it * 64;
        uint8_t* sk = sK0 + st * 2 * C::KT;
#pragma unroll
        for (int c = 0; c < C::DC; ++c) {
          tma_load_2d(sk + c * 8192, &map_kv64, HD + h * Dh + c * 64, krow, &kv_full[st]);
          tma_load_2d(sk + C::KT + c * 8192, &map_kv64, 2 * HD + h * Dh + c * 64, krow, &kv_full[st]);
        }
        mbar_expect_tx(&kv_full[st], 2 * C::KT);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_q = umma_idesc_bf16(128, Dh, false, true);
      const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_sdp = [&](int it) {
        const int st = it % KST, g = it & 1;
        mbar_wait(&kv_full[st], (it / KST) & 1);
        mbar_wait(&sdp_free[g], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t aK = smem_u32(sK0 + st * 2 * C::KT), aV = aK + C::KT;
#pragma unroll
        for (int ks = 0; ks < Dh / 16; ++ks) {
          tc_mma_f16(tmem + g * 128, kdesc(aQ, ks, 128), kdesc(aK, ks, 64), idesc_s, ks > 0);
          tc_mma_f16(tmem + g * 128 + 64, kdesc(aO, ks, 128), kdesc(aV, ks, 64), idesc_s, ks > 0);
        }
        tc_commit(&sdp_full[g]);
      };
      issue_sdp(0);
      if (n_it > 1) issue_sdp(1);
      for (int it = 0; it < n_it; ++it) {
        const int st = it % KST, g = it & 1;
        mbar_wait(&p_full[g], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t aK = smem_u32(sK0 + st * 2 * C::KT), tD = tmem + g * 128 + 64;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          tc_mma_f16_ts(tmem + 256, tD + 8 * ks, mndesc(aK, ks, 64), idesc_q, (it > 0 || ks > 0));
        tc_commit(&kv_empty[st]);
        if (it + 2 < n_it) issue_sdp(it + 2);
      }
      tc_commit(all_done);
    }
  } else if (warp >= 4) {
    const int wq = warp & 3, g = (warp - 4) >> 2;
    const int r = wq * 32 + lane;
    const int q = qt * 128 + r;
    const uint32_t tl = tmem + ((uint32_t)(wq * 32) << 16) + g * 128;
    const int64_t li = ((int64_t)b * H + h) * S + q;
    const float lse2 = lse[li] * kLog2e, dl = delta[li];
    for (int it = g; it < n_it; it += 2) {
      mbar_wait(&sdp_full[g], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float sv[32], dp[32];
        tmem_ld_32x32b_x32_pair(tl + hf * 32, tl + 64 + hf * 32, sv, dp);
        if (hf == 1) {
          tc_fence_before();
          mbar_arrive(&sdp_free[g]);
        }
        const int kb = it * 64 + hf * 32;
        if (CAUSAL && kb + 31 > q) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float p = ex2(fmaf(sv[i], scale_log2, -lse2));
            p = kb + i > q ? 0.f : p;
            dp[i] = p * (dp[i] - dl);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float p = ex2(fmaf(sv[i], scale_log2, -lse2));
            dp[i] = p * (dp[i] - dl);
          }
        }
        uint32_t dk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) dk[i] = pack_bf16x2(dp[2 * i], dp[2 * i + 1]);
        tmem_st_32x32b_x16(tl + 64 + hf * 16, dk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[g]);
    }
    mbar_wait(all_done, 0);
    tc_fence_after();
    const uint32_t te = tmem + ((uint32_t)(wq * 32) << 16) + 256;
    __nv_bfloat16* dqrow = dqkv + ((int64_t)b * S + q) * 3 * HD + h * Dh;
#pragma unroll 1
    for (int c = g; c < Dh / 32; c += 2) {
      float v[32];
      tmem_ld_32x32b_x32(te + c * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= scale;
      st_row32_bf16(dqrow + c * 32, v);
      if (dbias) {  // Q-bias gradient
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = bf16_round(v[i]);
        atomicAdd(dbias + h * Dh + c * 32 + lane, warp_colsum32(v, lane));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}


// ===================================================== backward: dQ from dS ====
// dQ = scale dS K as a plain tcgen05 GEMM over the dS^T tiles the dK/dV
// kernel stored (bf16 [B H][S keys][S queries], exactly the values it used
// for dK): no recomputation of S = Q K^T and dP = dO V^T (7 -> 5 attention
// GEMMs).  CTA = 128 queries of one (batch, head); warp 0 TMA producer, warp
// 1 MMA issuer, warp 2 TMEM allocator, warps 4-7 epilogue.  Per 64-key tile:
// A = dS (M = 128 queries, K = 64 keys; the dS^T tile is its MN-major
// storage), B = K (K = 64 keys, N = Dh; MN-major), D = dQ in TMEM.
template <int Dh>
struct DqDs {
  static constexpr int DC = Dh / 64;
  static constexpr int ST = 6;
  static constexpr uint32_t AT = 64 * 128 * 2;   // dS^T tile: 64 keys x 128 queries
  static constexpr uint32_t BT = 64 * Dh * 2;    // K tile: 64 keys x Dh
  static constexpr size_t SMEM = 1024 + ST * (AT + BT) + 256;
};

template <int Dh, bool CAUSAL>
__global__ void __launch_bounds__(256, 1)
dq_ds_tc(const __grid_constant__ CUtensorMap map_ds, const __grid_constant__ CUtensorMap map_kv64,
         __nv_bfloat16* __restrict__ dqkv, float* __restrict__ dbias, int S, int H, float scale) {
  using C = DqDs<Dh>;
  constexpr int ST = C::ST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA0 = smem;                      // stage s: dS^T at sA0 + s AT
  uint8_t* sB0 = smem + ST * C::AT;         // stage s: K at sB0 + s BT
  uint64_t* full = reinterpret_cast<uint64_t*>(sB0 + ST * C::BT);
  uint64_t* empty = full + ST;
  uint64_t* done = empty + ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x, qt = gridDim.y - 1 - blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int n_it = CAUSAL ? 2 * qt + 2 : S / 64;
  const int HD = H * Dh;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_ds);
    tma_prefetch_desc(&map_kv64);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<Dh>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------ producer
      const uint64_t ds_pol = l2_policy_evict_first();  // the last read of dS^T
      for (int it = 0; it < n_it; ++it) {
        const int st = it % ST;
        mbar_wait(&empty[st], ((it / ST) & 1) ^ 1);
        const int kr = it * 64;
        // dS^T rows (bh S + keys), query columns in two 64-wide boxes
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tma_load_2d_hint(sA0 + st * C::AT + c * 8192, &map_ds, qt * 128 + c * 64, bh * S + kr, &full[st], ds_pol);
#pragma unroll
        for (int c = 0; c < C::DC; ++c)
          tma_load_2d(sB0 + st * C::BT + c * 8192, &map_kv64, HD + h * Dh + c * 64, b * S + kr, &full[st]);
        mbar_expect_tx(&full[st], C::AT + C::BT);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------ MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(128, Dh, true, true);
      for (int it = 0; it < n_it; ++it) {
        const int st = it % ST;
        mbar_wait(&full[st], (it / ST) & 1);
        tc_fence_after();
        const uint32_t aA = smem_u32(sA0 + st * C::AT), aB = smem_u32(sB0 + st * C::BT);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)  // 64 keys / 16
          tc_mma_f16(tmem, mndesc(aA, ks, 64), mndesc(aB, ks, 64), idesc, (it > 0 || ks > 0));
        tc_commit(&empty[st]);
      }
      tc_commit(done);
    }
  } else if (warp >= 4) {  // ---------------------------------- epilogue
    const int wq = warp & 3;
    const int q = qt * 128 + wq * 32 + lane;
    mbar_wait(done, 0);
    tc_fence_after();
    const uint32_t te = tmem + ((uint32_t)(wq * 32) << 16);
    __nv_bfloat16* dqrow = dqkv + ((int64_t)b * S + q) * 3 * HD + h * Dh;
#pragma unroll 1
    for (int c = 0; c < Dh / 32; ++c) {
      float v[32];
      tmem_ld_32x32b_x32(te + c * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= scale;
      st_row32_bf16(dqrow + c * 32, v);
      if (dbias) {  // Q-bias gradient: column sums of this warp's 32 queries, as stored
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = bf16_round(v[i]);
        atomicAdd(dbias + h * Dh + c * 32 + lane, warp_colsum32(v, lane));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<Dh>(tmem);
}

// delta[b,h,i] = <O[b,i,h,:], dO[b,i,h,:]>: Dh/8 lanes per (token, head)
// row, one 16-byte load of O and dO per lane, rows in memory order.
template <int Dh>
__global__ void __launch_bounds__(256) delta_tc_kernel(int rows, int S, int H, const __nv_bfloat16* __restrict__ o,
                                                       const __nv_bfloat16* __restrict__ dout,
                                                       float* __restrict__ delta) {
  constexpr int LPR = Dh / 8;
  const int gt = blockIdx.x * 256 + threadIdx.x;
  const int row = gt / LPR, sub = gt % LPR;  // row = (b * S + i) * H + h
  const bool ok = row < rows;
  float s = 0.f;
  if (ok) {
    const int64_t off = (int64_t)row * Dh + sub * 8;
    const uint4 a = *reinterpret_cast<const uint4*>(o + off), c = *reinterpret_cast<const uint4*>(dout + off);
    const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* hc = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 fa = __bfloat1622float2(ha[j]), fc = __bfloat1622float2(hc[j]);
      s = fmaf(fa.x, fc.x, fmaf(fa.y, fc.y, s));
    }
  }
#pragma unroll
  for (int m = LPR / 2; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  if (ok && sub == 0) {
    const int h = row % H, bi = row / H, i = bi % S, b = bi / S;
    delta[((int64_t)b * H + h) * S + i] = s;
  }
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
  // two query tiles per CTA for non-causal attention (BERT shape 17.1 -> 15.2
  // us); causal: one-tile CTAs, heaviest first, are faster at every measured
  // shape (S=2048: H=16 31.6 vs 54.6 us, H=32 58.3 vs 60.4, B=2 57.2 vs 60.1)
  const bool two = S % 256 == 0 && !CAUSAL;
  const int mode = attn_fwd_mode();
  if (mode == 2 || (mode == 0 && two && S % 256 == 0)) {
    auto k2 = fwd2_tc<Dh, CAUSAL>;
    static bool once2 = false;
    if (!once2) {
      if (int rc = set_smem(k2, Fwd2<Dh>::SMEM)) return rc;
      once2 = true;
    }
    k2<<<dim3(B * H, S / 256), 352, Fwd2<Dh>::SMEM, st>>>(m, (__nv_bfloat16*)o, lse, S, H, scale * kLog2e);
    count_launch();
    BP_CHECK_LAUNCH("attn_fwd2_tc");
    return BP_OK;
  }
  const int exf = attn_fwd_exf();  // BP_OPT_ATTN_FWD_EXF (0: default)
  auto k = exf == 3 ? fwd_tc<Dh, CAUSAL, 3> : exf == 4 ? fwd_tc<Dh, CAUSAL, 4> : exf == 5 ? fwd_tc<Dh, CAUSAL, 5>
          : exf == 6 ? fwd_tc<Dh, CAUSAL, 6> : exf == 7 ? fwd_tc<Dh, CAUSAL, 7> : exf == 8 ? fwd_tc<Dh, CAUSAL, 8>
                                                                             : fwd_tc<Dh, CAUSAL, 2>;
  static bool once[7] = {false, false, false, false, false, false, false};
  const int oi = exf >= 3 && exf <= 8 ? exf - 2 : 0;
  if (!once[oi]) {
    if (int rc = set_smem(k, Fwd<Dh>::SMEM)) return rc;
    once[oi] = true;
  }
  k<<<dim3(B * H, S / 128), 384, Fwd<Dh>::SMEM, st>>>(m, (__nv_bfloat16*)o, lse, S, H, scale * kLog2e);
  count_launch();
  BP_CHECK_LAUNCH("attn_fwd_tc");
  return BP_OK;
}

template <int Dh, bool CAUSAL>
static int bwd(int B, int S, int H, float scale, float* dbias, const void* qkv, const void* o, const void* dout,
               const float* lse, void* dqkv, float* ws, cudaStream_t st) {
  float* delta = ws;
  const int rows = B * H * S;
  delta_tc_kernel<Dh><<<(int)(((int64_t)rows * (Dh / 8) + 255) / 256), 256, 0, st>>>(rows, S, H, (const __nv_bfloat16*)o,
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
  auto k3 = dq_ds_tc<Dh, CAUSAL>;
  static bool once = false;
  if (!once) {
    if (int rc = set_smem(k1, Dkdv<Dh>::SMEM)) return rc;
    if (int rc = set_smem(k2, Dq<Dh>::SMEM)) return rc;
    if (int rc = set_smem(k3, DqDs<Dh>::SMEM)) return rc;
    once = true;
  }
  const float sl2 = scale * kLog2e;
  // mode 0 (default): dK/dV stores dS^T, dQ = dS K as a GEMM over it; mode 1:
  // the dQ kernel recomputes S and dP
  const bool via_ds = attn_bwd_mode() == 0;
  __nv_bfloat16* ds_t = via_ds ? reinterpret_cast<__nv_bfloat16*>(ws + attn_ds_offset_floats(B, S, H)) : nullptr;
  k1<<<dim3(B * H, S / 128), 384, Dkdv<Dh>::SMEM, st>>>(kv128, q64, do64, lse, delta, (__nv_bfloat16*)dqkv, dbias, S, H,
                                                         scale, sl2, ds_t);
  count_launch();
  if (via_ds) {
    CUtensorMap mds;
    if (int rc = make_map(&mds, ds_t, (uint64_t)S, (uint64_t)B * H * S, (int64_t)S, 64, 64)) return rc;
    k3<<<dim3(B * H, S / 128), 256, DqDs<Dh>::SMEM, st>>>(mds, kv64, (__nv_bfloat16*)dqkv, dbias, S, H, scale);
  } else {
    k2<<<dim3(B * H, S / 128), 384, Dq<Dh>::SMEM, st>>>(q128, kv64, do128, lse, delta, (__nv_bfloat16*)dqkv, dbias, S,
                                                         H, scale, sl2);
  }
  count_launch();
  BP_CHECK_LAUNCH("attn_bwd_tc");
  return BP_OK;
}

}  // namespace fat

// Debug aid (BP_ATTN_TRACE builds): copy the dK/dV softmax-warp timestamps.
extern "C" __attribute__((visibility("default"))) int bp_attn_trace_dump(long long* host, int n) {
#ifdef BP_ATTN_TRACE
  return cudaMemcpyFromSymbol(host, fat::g_trace, sizeof(long long) * (n < 1024 ? n : 1024)) == cudaSuccess ? 0 : 2;
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

int attn_tc_bwd(int B, int S, int H, int Dh, int causal, float scale, float* dbias, const void* qkv, const void* o,
                const void* dout, const float* lse, void* dqkv, float* ws, cudaStream_t st) {
  if (Dh == 128)
    return causal ? fat::bwd<128, true>(B, S, H, scale, dbias, qkv, o, dout, lse, dqkv, ws, st)
                  : fat::bwd<128, false>(B, S, H, scale, dbias, qkv, o, dout, lse, dqkv, ws, st);
  return causal ? fat::bwd<64, true>(B, S, H, scale, dbias, qkv, o, dout, lse, dqkv, ws, st)
                : fat::bwd<64, false>(B, S, H, scale, dbias, qkv, o, dout, lse, dqkv, ws, st);
}

}  // namespace bp
