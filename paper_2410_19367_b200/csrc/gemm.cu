// GEMM for the per-virtual-stage transformer passes.
//
// bf16: persistent warp-specialised tcgen05 kernel.
//   * 128 x BN x 64 tiles (BN = 256 or 128), 4-6 stage TMA -> smem ring
//     (SWIZZLE_128B), fp32 accumulators in TMEM, double-buffered so the
//     epilogue of tile i overlaps the MMAs of tile i+1.
//   * warp 0: TMA producer (one elected lane), warp 1: MMA issuer (one
//     lane issues tcgen05.mma, tcgen05.commit frees smem slots / signals
//     the epilogue), warp 2: TMEM allocator, warps 4-7: epilogue
//     (tcgen05.ld 32x32b -> registers -> fused bias / GELU / dGELU /
//     residual / fp32-accumulate -> global); the CTA-pair kernel runs
//     warps 4-11 (two per TMEM lane quarter, half the columns each) when a
//     launch has one tile per pair and its epilogue cannot hide behind a
//     next tile's MMAs.
//   * A and B may each be K-major or MN-major; the smem descriptors and
//     the instruction descriptor's transpose bits absorb the layout, so
//     fprop (X W^T), dgrad (dY W) and wgrad (dY^T X) run without any
//     explicit transpose.
// fp32: exact-fp32 SIMT kernel (check mode; no TF32) with the same epilogue.
#include "common.cuh"

#include <mutex>
#include <unordered_map>

namespace bp {

struct Epi {
  int M, N;
  void* C;
  int64_t ldc;
  int c_dtype;
  float alpha;
  int accumulate;
  const void* bias;
  int bias_dtype;
  const void* residual;
  int64_t ldr;
  void* aux;
  int64_t ldaux;
  int epilogue;
  int vec_ok;
  int nostore;  // debug: drain TMEM but skip the global epilogue (BP_OPT_GEMM_DEBUG)
  int tma_store;  // 2-SM kernel: stage 32-column chunks in smem, TMA-store them
  float* colsum;  // optional: colsum[n] += sum over rows of C as stored (TMA epilogue only)
  int aux_evict_first;  // GELU pre-activation (read only by the backward, much later): streamed past L2
};

BP_DEV float ld_any(const void* p, int dtype, int64_t i) {
  return dtype == BP_F32 ? static_cast<const float*>(p)[i]
                         : __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}
BP_DEV void st_any(void* p, int dtype, int64_t i, float v) {
  if (dtype == BP_F32)
    static_cast<float*>(p)[i] = v;
  else
    static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
}

// Scalar epilogue for one element (used by the SIMT kernel and ragged tiles).
BP_DEV void epi_one(const Epi& ep, int r, int c, float acc) {
  float v = acc * ep.alpha;
  if (ep.bias) v += ld_any(ep.bias, ep.bias_dtype, c);
  if (ep.epilogue == BP_EPI_GELU) {
    st_any(ep.aux, ep.c_dtype, (int64_t)r * ep.ldaux + c, v);
    // GELU is applied to the value as stored (rounded) so fwd/bwd agree.
    v = gelu_f(ld_any(ep.aux, ep.c_dtype, (int64_t)r * ep.ldaux + c));
  } else if (ep.epilogue == BP_EPI_DGELU) {
    v *= gelu_grad_f(ld_any(ep.aux, ep.c_dtype, (int64_t)r * ep.ldaux + c));
  }
  if (ep.residual) v += ld_any(ep.residual, ep.c_dtype, (int64_t)r * ep.ldr + c);
  int64_t o = (int64_t)r * ep.ldc + c;
  if (ep.accumulate) v += static_cast<const float*>(ep.C)[o];
  st_any(ep.C, ep.c_dtype, o, v);
}

// 32 consecutive columns of one row, vectorised (16-byte accesses).
BP_DEV void load32(const void* p, int dtype, int64_t off, float (&x)[32]) {
  if (dtype == BP_F32) {
    const float4* q = reinterpret_cast<const float4*>(static_cast<const float*>(p) + off);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 t = q[i];
      x[4 * i] = t.x; x[4 * i + 1] = t.y; x[4 * i + 2] = t.z; x[4 * i + 3] = t.w;
    }
  } else {
    const uint4* q = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p) + off);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 t = q[i];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        x[8 * i + 2 * j] = f.x;
        x[8 * i + 2 * j + 1] = f.y;
      }
    }
  }
}
BP_DEV void store32(void* p, int dtype, int64_t off, const float (&x)[32]) {
  if (dtype == BP_F32) {
    float4* q = reinterpret_cast<float4*>(static_cast<float*>(p) + off);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]);
  } else {
    uint4* q = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p) + off);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 t;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(x[8 * i + 2 * j], x[8 * i + 2 * j + 1]);
      q[i] = t;
    }
  }
}

BP_DEV void epi_row32(const Epi& ep, int r, int c0, float (&v)[32]) {
  if (r >= ep.M || ep.nostore) return;
  if (!ep.vec_ok || c0 + 32 > ep.N) {
    for (int i = 0; i < 32 && c0 + i < ep.N; ++i) epi_one(ep, r, c0 + i, v[i]);
    return;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] *= ep.alpha;
  float t[32];
  if (ep.bias) {
    load32(ep.bias, ep.bias_dtype, c0, t);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += t[i];
  }
  if (ep.epilogue == BP_EPI_GELU) {
    const int64_t ao = (int64_t)r * ep.ldaux + c0;
    store32(ep.aux, ep.c_dtype, ao, v);
    if (ep.c_dtype == BP_BF16) {  // gelu of the rounded pre-activation
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = gelu_fast(__bfloat162float(__float2bfloat16_rn(v[i])));
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = gelu_f(v[i]);
    }
  } else if (ep.epilogue == BP_EPI_DGELU) {
    load32(ep.aux, ep.c_dtype, (int64_t)r * ep.ldaux + c0, t);
    if (ep.c_dtype == BP_BF16) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_fast(t[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_f(t[i]);
    }
  }
  if (ep.residual) {
    load32(ep.residual, ep.c_dtype, (int64_t)r * ep.ldr + c0, t);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += t[i];
  }
  const int64_t o = (int64_t)r * ep.ldc + c0;
  if (ep.accumulate) {
    load32(ep.C, BP_F32, o, t);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += t[i];
  }
  store32(ep.C, ep.c_dtype, o, v);
}

// Epilogue of one accumulator tile slice: 32 TMEM lanes (rows) x ncols
// columns for the calling warp.  The extra global input of the epilogue
// (fp32 C for accumulation, the residual, or the saved pre-activation for
// dGELU) of chunk c+1 is loaded while chunk c is finished, so the DRAM
// latency of the read-modify-write is not serialised across chunks.
template <int NCHUNK>
BP_DEV void epi_tile(const Epi& ep, uint32_t tmem_addr, int row, int n0) {
  if (ep.nostore) {
#pragma unroll 1
    for (int c = 0; c < NCHUNK; ++c) {
      float v[32];
      tmem_ld_32x32b_x32(tmem_addr + c * 32, v);
      if (v[0] == 12345.f) static_cast<float*>(ep.C)[0] = v[1];  // keep the load live
    }
    return;
  }
  const void* xin = nullptr;
  int xdt = ep.c_dtype;
  int64_t xld = 0;
  if (ep.accumulate) {
    xin = ep.C; xdt = BP_F32; xld = ep.ldc;
  } else if (ep.residual) {
    xin = ep.residual; xld = ep.ldr;
  } else if (ep.epilogue == BP_EPI_DGELU) {
    xin = ep.aux; xld = ep.ldaux;
  }
  // must be warp-uniform: tcgen05.ld below is a .sync.aligned warp collective
  const bool fast = __all_sync(0xffffffffu, ep.vec_ok && row < ep.M && n0 + NCHUNK * 32 <= ep.N &&
                                                xin != nullptr &&
                                                !(ep.residual && (ep.accumulate || ep.epilogue == BP_EPI_DGELU)));
  if (!fast) {
#pragma unroll 1
    for (int c = 0; c < NCHUNK; ++c) {
      float v[32];
      tmem_ld_32x32b_x32(tmem_addr + c * 32, v);
      if (n0 + c * 32 < ep.N) epi_row32(ep, row, n0 + c * 32, v);
    }
    return;
  }
  const int64_t xrow = (int64_t)row * xld + n0;
  float nxt[32];
  load32(xin, xdt, xrow, nxt);
#pragma unroll 1
  for (int c = 0; c < NCHUNK; ++c) {
    float cur[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) cur[i] = nxt[i];
    if (c + 1 < NCHUNK) load32(xin, xdt, xrow + (c + 1) * 32, nxt);
    float v[32];
    tmem_ld_32x32b_x32(tmem_addr + c * 32, v);
    const int c0 = n0 + c * 32;
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= ep.alpha;
    if (ep.bias) {
      float t[32];
      load32(ep.bias, ep.bias_dtype, c0, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += t[i];
    }
    if (ep.epilogue == BP_EPI_DGELU) {
      if (ep.c_dtype == BP_BF16) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_fast(cur[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_f(cur[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += cur[i];
    }
    store32(ep.C, ep.c_dtype, (int64_t)row * ep.ldc + c0, v);
  }
}

// TMA-store epilogue of one accumulator slice (warp = 32 TMEM lanes = 32
// rows, NCHUNK x 32 columns).  Each 32-column chunk is finished in
// registers, written to a per-warp shared staging unit in the TMA swizzle
// (bf16: 64-byte rows, SWIZZLE_64B; fp32: 128-byte rows, SWIZZLE_128B --
// conflict-free 16-byte stores), and sent with one bulk tensor store (a
// bulk reduce-add for fp32 accumulation: C += tile happens at L2, C is
// never read into the SM).  Replaces 32 rows x 16-byte scattered stores
// per warp instruction with full-line bulk writes.  Two staging units per
// warp alternate; `ubuf` carries the unit parity across tiles.  Rows past
// M / columns past N are clipped by the TMA unit.
BP_DEV void stage_row32(uint8_t* unit, int lane, int dtype, const float (&v)[32]) {
  if (dtype == BP_F32) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t off = lane * 128 + ((j ^ (lane & 7)) << 4);
      *reinterpret_cast<float4*>(unit + off) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 t;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
      for (int q = 0; q < 4; ++q) h[q] = __floats2bfloat162_rn(v[8 * j + 2 * q], v[8 * j + 2 * q + 1]);
      const uint32_t off = lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
      *reinterpret_cast<uint4*>(unit + off) = t;
    }
  }
}

// bf16 row of a SWIZZLE_64B staging unit -> 32 floats
BP_DEV void unstage_row32_bf16(const uint8_t* unit, int lane, float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 t = *reinterpret_cast<const uint4*>(unit + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(h[q]);
      x[8 * j + 2 * q] = f.x;
      x[8 * j + 2 * q + 1] = f.y;
    }
  }
}

// Phase timestamps of every CTA of the last traced 2-SM GEMM launch
// (BP_GEMM_TRACE builds only, tools/gemm_trace.py): clock64 at entry, after
// the prologue, first operand stage landed, last MMA issued, accumulator
// ready in the epilogue, epilogue issued, stores drained, exit; then the
// global timer at entry and the CTA's tile count.
#ifdef BP_GEMM_TRACE
__device__ long long g_gemm_trace[2 * 160][10];
__device__ long long g_gemm_etrace[2 * 160][8][5];  // first tile, epilogue warp 0: per-chunk stamps
#define GTRACE(k) (g_gemm_trace[blockIdx.x][k] = clock64())
#define ETRACE(c, k) \
  do {                                                                                         \
    if (etr && lane == 0 && (c) < 8) g_gemm_etrace[blockIdx.x][c][k] = clock64();            \
  } while (0)
#else
#define GTRACE(k) ((void)0)
#define ETRACE(c, k) ((void)0)
#endif

// Per-warp state of the TMA epilogue, carried across tiles.
struct EpiTma {
  uint8_t* stage;    // U units x 4 KB: [0, 2K) output / [2K, 4K) aux-out or input
  uint64_t* bar;     // U mbarriers (input tile landed in unit u)
  int ubuf;          // next unit
  uint32_t phase;    // bit u = parity of bar[u]
};

// The extra epilogue input (residual, or the saved pre-activation for
// dGELU) arrives by TMA too: chunk c+1's 32 x 32 tile is requested while
// chunk c is finished, into the upper half of the other unit.
BP_DEV void epi_tma_prefetch_input(const CUtensorMap* mx, EpiTma& es, int u, int c0, int row0,
                                   bool last_use = false) {
  uint8_t* dst = es.stage + u * 4096 + 2048;
  fence_proxy_async_smem();  // earlier generic reads of this half precede the async write
  mbar_expect_tx(&es.bar[u], 2048);
  if (last_use)  // the dGELU pre-activation: its last read, leave L2 first
    tma_load_2d_hint(dst, mx, c0, row0, &es.bar[u], l2_policy_evict_first());
  else
    tma_load_2d(dst, mx, c0, row0, &es.bar[u]);
}

// U staging units per epilogue warp: up to U - 1 TMA stores of earlier
// chunks may still be reading shared memory while chunk c is staged.
template <int NCHUNK, int U = 2>
BP_DEV void epi_tile_tma(const Epi& ep, const CUtensorMap* mc, const CUtensorMap* mx, uint32_t tmem_addr,
                         int row0, int lane, int n0, EpiTma& es, bool input_issued, bool etr = false,
                         const float* sbias = nullptr, int nlim = 0x7fffffff) {
  if (nlim > ep.N) nlim = ep.N;  // columns past the tile (split epilogue) or the matrix are not this warp's
  const bool gelu = ep.epilogue == BP_EPI_GELU;
  const bool has_in = ep.residual != nullptr || ep.epilogue == BP_EPI_DGELU;
  if (has_in && !input_issued && lane == 0) epi_tma_prefetch_input(mx, es, es.ubuf, n0, row0, ep.aux_evict_first && ep.epilogue == BP_EPI_DGELU);
#pragma unroll 1
  for (int c = 0; c < NCHUNK; ++c) {
    const int c0 = n0 + c * 32;
    if (c0 >= nlim) break;  // warp-uniform
    const int u = es.ubuf;
    uint8_t* unit = es.stage + u * 4096;
    if (has_in && lane == 0 && c + 1 < NCHUNK && c0 + 32 < nlim)
      epi_tma_prefetch_input(mx, es, (u + 1) % U, c0 + 32, row0, ep.aux_evict_first && ep.epilogue == BP_EPI_DGELU);
    ETRACE(c, 0);
    float v[32];
    tmem_ld_32x32b_x32(tmem_addr + c * 32, v);
    ETRACE(c, 1);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= ep.alpha;
    if (sbias) {  // the tile's bias, staged in shared memory (broadcast reads)
      const float4* q = reinterpret_cast<const float4*>(sbias + c * 32);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 t = q[i];
        v[4 * i] += t.x; v[4 * i + 1] += t.y; v[4 * i + 2] += t.z; v[4 * i + 3] += t.w;
      }
    } else if (ep.bias) {
      float t[32];
      load32(ep.bias, ep.bias_dtype, c0, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += t[i];
    }
    if (has_in) {
      float cur[32];
      mbar_wait(&es.bar[u], (es.phase >> u) & 1);
      ETRACE(c, 2);
      es.phase ^= 1u << u;
      unstage_row32_bf16(unit + 2048, lane, cur);
      if (ep.epilogue == BP_EPI_DGELU) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_fast(cur[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += cur[i];
      }
    }
    if (lane == 0) bulk_wait_read<U - 1>();  // this unit's previous store has read it
    __syncwarp();
    ETRACE(c, 3);
    if (gelu) {
      stage_row32(unit + 2048, lane, ep.c_dtype, v);  // pre-activation -> aux
      if (ep.c_dtype == BP_BF16) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = gelu_fast(__bfloat162float(__float2bfloat16_rn(v[i])));
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = gelu_f(v[i]);
      }
    }
    stage_row32(unit, lane, ep.c_dtype, v);
    if (ep.colsum) {  // bias gradient: column sums of this warp's 32 rows, as stored
      float t[32];
      const bool row_ok = row0 + lane < ep.M;
#pragma unroll
      for (int i = 0; i < 32; ++i) t[i] = row_ok ? (ep.c_dtype == BP_BF16 ? bf16_round(v[i]) : v[i]) : 0.f;
      atomicAdd(ep.colsum + c0 + lane, warp_colsum32(t, lane));
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (ep.accumulate)
        tma_reduce_add_2d(mc, unit, c0, row0);
      else
        tma_store_2d(mc, unit, c0, row0);
      if (gelu) {
        if (ep.aux_evict_first)
          tma_store_2d_hint(mx, unit + 2048, c0, row0, l2_policy_evict_first());
        else
          tma_store_2d(mx, unit + 2048, c0, row0);
      }
      bulk_commit();
    }
    ETRACE(c, 4);
    es.ubuf = (es.ubuf + 1) % U;
  }
}

// ===================================================== tcgen05 kernel ====
template <int BN>
struct TcCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN;  // two fp32 accumulators
  static constexpr size_t SMEM = 1024 + STAGES * (size_t)STAGE_BYTES + 256;
};

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               int M, int N, int K, Epi ep) {
  using C = TcCfg<BN>;
  constexpr int BM = C::BM, BK = C::BK, STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int kblocks = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile % tiles_m) * BM, n0 = (tile / tiles_m) * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d(a, &map_a, k0, m0, &full[stage]);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) tma_load_2d(a + c * (BK * 128), &map_a, m0 + 64 * c, k0, &full[stage]);
          }
          if (!B_MN) {
            tma_load_2d(b, &map_b, k0, n0, &full[stage]);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) tma_load_2d(b + c * (BK * 128), &map_b, n0 + 64 * c, k0, &full[stage]);
          }
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------- MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(a_addr + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(a_addr + k * 32, 0, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(b_addr + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(b_addr + k * 32, 0, 1024);
            tc_mma_f16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // ------------------------------ epilogue
    const int ew = warp - 4;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (tile % tiles_m) * BM, n0 = (tile / tiles_m) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + ew * 32 + lane;
      const uint32_t t0 = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
      epi_tile<BN / 32>(ep, t0, row, n0);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}


// ============================================ stream-K work schedule ====
// Tiles 0..dp-1 are handed out round-robin as whole tiles ("data
// parallel"); the remaining tiles' k-blocks are split evenly over the P CTA
// pairs ("stream-K"), so every pair gets the same number of k-blocks and
// the last wave is no longer quantised to whole tiles.  A pair's stream-K
// range covers at most one partial tile head (a "contributor" segment,
// k-blocks [kb0, kb1) with kb1 < KB: its raw fp32 accumulator goes to the
// pair's workspace slot and a flag is raised) and at most one partial tile
// tail (an "owner" segment, kb1 == KB, kb0 > 0: it waits for the
// contributors' flags and adds their partials before the epilogue).
// Contributor segments run FIRST and owner segments LAST, so no pair ever
// waits on a pair that is itself waiting.
struct Seg {
  int tile, kb0, kb1, role;  // role: 0 whole tile, 1 owner, 2 contributor
};

struct SkSched {
  int T, KB, P, p, dp;
  long U, lo, hi;
  int nsk;
  Seg sk[4];
  int first_contrib;  // 1 if sk[0] is this pair's contributor segment (run first)

  BP_DEV void init(int T_, int KB_, int P_, int p_, int enable) {
    T = T_; KB = KB_; P = P_; p = p_;
    dp = (!enable || T % P == 0) ? T : (T / P >= 1 ? (T / P - 1) * P : 0);
    U = (long)(T - dp) * KB;
    lo = U * p / P;
    hi = U * (p + 1) / P;
    nsk = 0;
    Seg tmp[4];
    int n = 0;
    for (long u = lo; u < hi && n < 4;) {
      const int rel = (int)(u / KB), kb0 = (int)(u % KB);
      const long take = (hi - u) < (long)(KB - kb0) ? (hi - u) : (long)(KB - kb0);
      const int kb1 = kb0 + (int)take;
      const int role = (kb0 == 0 && kb1 == KB) ? 0 : (kb1 == KB ? 1 : 2);
      tmp[n++] = Seg{dp + rel, kb0, kb1, role};
      u += take;
    }
    first_contrib = (n > 0 && tmp[n - 1].role == 2) ? 1 : 0;
    if (first_contrib) sk[nsk++] = tmp[n - 1];
    for (int i = 0; i < n - first_contrib; ++i) sk[nsk++] = tmp[i];
  }
  BP_DEV int n_dp() const { return dp > p ? (dp - p + P - 1) / P : 0; }
  BP_DEV int count() const { return n_dp() + nsk; }
  // execution order: [contributor] [dp tiles] [owner / whole sk tiles]
  BP_DEV Seg get(int i) const {
    if (first_contrib) {
      if (i == 0) return sk[0];
      --i;
      if (i < n_dp()) return Seg{p + i * P, 0, KB, 0};
      return sk[1 + (i - n_dp())];
    }
    if (i < n_dp()) return Seg{p + i * P, 0, KB, 0};
    return sk[i - n_dp()];
  }
  // pairs whose contributor segment belongs to SK tile `tile`: q in
  // [q_lo, p) with hi_q strictly inside the tile's unit range
  BP_DEV int contrib_lo(int tile) const {
    const long ts = (long)(tile - dp) * KB;
    int q = p;
    while (q > 0 && U * q / P > ts) --q;  // hi_{q-1} = U*q/P
    return q;
  }
};

struct SkWs {
  float* part;      // [P][2 CTAs][128][BN] fp32 partial accumulators
  unsigned* flag;   // [P][2]
  unsigned epoch;
  int enable;
};

BP_DEV void flag_release(unsigned* f, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
BP_DEV unsigned flag_acquire(const unsigned* f) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}
template <int EW = 4>
BP_DEV void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory"); }

// ============================================ tcgen05 2-SM (CTA pair) ====
// Pair tile 256 x 256: each CTA of the cluster holds 128 rows of A and 128
// rows (N-half) of B per stage; the leader issues tcgen05.mma.cta_group::2
// (M=256, N=256) reading both CTAs' smem, each CTA's TMEM receives its own
// 128 x 256 accumulator.  Halves the per-SM operand traffic of the 1-SM
// kernel (L2 -> SM bandwidth is the bound there).
// OCC = 2: the co-resident variant -- one TMEM accumulator (<= 256
// columns) and a shared-memory budget of half an SM, so TWO CTA pairs (of
// different kernels: the co-resident executor runs one stream per logical
// device) share each SM pair.  A single-wave GEMM (one tile per pair: most
// M = 2048 per-micro-batch shapes) then has its pipeline fill and epilogue
// overlapped by the other pair's MMAs instead of leaving the tensor pipe
// idle; no stream-K paths (its owner CTAs spin).
// EW = epilogue warps: 4 (one per TMEM lane quarter, each drains its 32
// rows x all BN columns) or 8 (two per lane quarter, each drains half the
// columns: half the serial chunk chain of a tile's epilogue, which is
// exposed when a launch has one tile per CTA pair).
template <int BN_, bool B_MN_, int OCC_ = 1, int EW_ = 4>
struct Tc2Cfg {
  // BN = pair-tile width; wider than 256 is issued as NSUB MMAs of N = 256
  // per k-step into adjacent TMEM columns (one accumulator buffer then).
  static constexpr int BM = 128, BN = BN_, BNH = BN_ / 2, BK = 64;
  static constexpr int NSUB = BN_ > 256 ? BN_ / 256 : 1;
  static constexpr int MMA_N = BN_ / NSUB;
  static constexpr int SUBH = MMA_N / 2;        // B rows per CTA per sub-MMA
  static constexpr int BCH = (SUBH + 63) / 64;  // 64-wide chunks of an MN-major B sub-half
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t SUB_BYTES = B_MN_ ? BCH * 64 * BK * 2 : SUBH * BK * 2;
  static constexpr uint32_t B_BYTES = NSUB * SUB_BYTES;
  static constexpr int OCC = OCC_;
  static constexpr int EW = EW_;
  static constexpr int THREADS = 128 + 32 * EW;
  static_assert(EW == 4 || (EW == 8 && OCC == 1), "8 epilogue warps: the one-pair-per-SM-pair variant");
  // TMA-store staging units per epilogue warp (up to EPI_UNITS - 1 earlier
  // chunks' stores in flight).  Measured with 4: single-tile epilogues no
  // faster (proj fprop 27.7 us either way) and the stage lost to the extra
  // 32 KB slows the long-K launches (fc2 fprop 58.4 -> 60.4 us)
  static constexpr int EPI_UNITS = 2;
  static constexpr uint32_t EPI_BYTES = EW * EPI_UNITS * 4096;
  static constexpr uint32_t BIAS_BYTES = 4 * BN_;       // the tile's bias columns (fp32)
  static_assert(OCC == 1 || (OCC == 2 && BN_ <= 256), "co-resident variant: one <= 256-column accumulator");
  // per-CTA budget: the SM's 232448 B (OCC = 1), or half of it less the
  // 1 KB the hardware reserves per resident CTA (OCC = 2)
  static constexpr int SM_BUDGET = OCC == 1 ? 232448 : 232448 / 2 - 1024;
  static constexpr int STAGE_BUDGET = SM_BUDGET - 1024 - 512 - (int)EPI_BYTES - (int)BIAS_BYTES;
  static constexpr int STAGES = STAGE_BUDGET / (A_BYTES + B_BYTES) > 8 ? 8 : STAGE_BUDGET / (A_BYTES + B_BYTES);
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int ACC = (OCC == 1 && 2 * BN_ <= 512) ? 2 : 1;  // TMEM accumulator buffers
  static constexpr uint32_t TMEM_COLS = ACC * BN_ <= 256 ? 256 : 512;  // power of two
  static constexpr size_t SMEM = 1024 + STAGES * (size_t)STAGE_BYTES + EPI_BYTES + BIAS_BYTES + 512;  // 512 B barriers
  static_assert((2 * STAGES + 4 + EW * EPI_UNITS) * 8 + 4 <= 512, "barrier region");
};

template <int BN, bool A_MN, bool B_MN, int OCC, int EW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + 32 * EW, OCC)
gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_aux,
                int M, int N, int K, Epi ep, SkWs ws) {
  using C = Tc2Cfg<BN, B_MN, OCC, EW>;
  constexpr int BK = C::BK, STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sEpi = sB + STAGES * C::B_BYTES;
  float* sBias = reinterpret_cast<float*>(sEpi + C::EPI_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + C::EPI_BYTES + C::BIAS_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ebar = tempty + 2;  // EW epilogue warps x EPI_UNITS input-tile barriers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + EW * C::EPI_UNITS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int tiles_m = (M + 255) / 256, tiles_n = (N + C::BN - 1) / C::BN;
  const int num_tiles = tiles_m * tiles_n;
  const int kblocks = (K + BK - 1) / BK;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  SkSched sch;
  sch.init(num_tiles, kblocks, ncl, cid, OCC == 1 ? ws.enable : 0);
  const int nseg = sch.count();
#ifdef BP_GEMM_TRACE
  if (threadIdx.x == 0) {
    GTRACE(0);
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    g_gemm_trace[blockIdx.x][8] = (long long)gt;
    g_gemm_trace[blockIdx.x][9] = nseg;
  }
#endif

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * 32 * EW);  // every epilogue thread of both CTAs
    }
    for (int e = 0; e < EW * C::EPI_UNITS; ++e) mbar_init(&ebar[e], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) GTRACE(1);

  if (warp == 0) {
    if (lane == 0) {  // -------------------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int si = 0; si < nseg; ++si) {
        const Seg sg = sch.get(si);
        const int tile = sg.tile;
        const int m0 = (tile % tiles_m) * 256 + rank * 128;
        const int n0 = (tile / tiles_m) * C::BN + rank * C::SUBH;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_2sm(a, &map_a, k0, m0, &full[stage]);
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) tma_load_2d_2sm(a + c * (BK * 128), &map_a, m0 + 64 * c, k0, &full[stage]);
          }
#pragma unroll
          for (int j = 0; j < C::NSUB; ++j) {
            const int nj = n0 + j * C::MMA_N;
            uint8_t* bj = b + j * C::SUB_BYTES;
            if (!B_MN) {
              tma_load_2d_2sm(bj, &map_b, k0, nj, &full[stage]);
            } else {
#pragma unroll
              for (int c = 0; c < C::BCH; ++c)
                tma_load_2d_2sm(bj + c * (BK * 128), &map_b, nj + 64 * c, k0, &full[stage]);
            }
          }
          if (leader)
            mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          else
            mbar_arrive_remote(&full[stage], 0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader only)
      constexpr uint32_t idesc = umma_idesc_bf16(256, C::MMA_N, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int si = 0; si < nseg; ++si, ++it) {
        const Seg sg = sch.get(si);
        const int acc = C::ACC == 2 ? (it & 1) : 0;
        const uint32_t acc_phase = C::ACC == 2 ? ((it >> 1) & 1) : (it & 1);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::BN;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          if (si == 0 && kb == sg.kb0) GTRACE(2);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(a_addr + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(a_addr + k * 32, 0, 1024);
#pragma unroll
            for (int j = 0; j < C::NSUB; ++j) {
              const uint32_t bj = b_addr + j * C::SUB_BYTES;
              const uint64_t bd = B_MN ? umma_desc_sw128(bj + k * 2048, BK * 128, 1024)
                                       : umma_desc_sw128(bj + k * 32, 0, 1024);
              tc_mma_f16_2sm(d_tmem + j * C::MMA_N, ad, bd, idesc, (kb > sg.kb0) || (k != 0));
            }
          }
          tc_commit_2sm_mc(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit_2sm_mc(&tfull[acc]);
      }
      GTRACE(3);
    }
  } else if (warp >= 4) {  // ---------------------- epilogue (both CTAs)
    const int ew = warp - 4;
    const int q = ew & 3;  // TMEM lane quarter (warp % 4) = rows q*32 .. q*32+31
    constexpr int HCH = EW == 8 ? (C::BN / 32 + 1) / 2 : C::BN / 32;  // 32-column chunks per warp
    const int cofs = EW == 8 ? (ew >> 2) * HCH * 32 : 0;             // this warp's first column in the tile
    int it = 0;
    EpiTma es{sEpi + ew * C::EPI_UNITS * 4096, ebar + C::EPI_UNITS * ew, 0, 0u};
    const bool tma_in = ep.tma_store && (ep.residual != nullptr || ep.epilogue == BP_EPI_DGELU);
    if (ep.tma_store && lane == 0) {
      tma_prefetch_desc(&map_c);
      if (ep.epilogue != BP_EPI_NONE || ep.residual) tma_prefetch_desc(&map_aux);
    }
    for (int si = 0; si < nseg; ++si, ++it) {
      const Seg sg = sch.get(si);
      const int tile = sg.tile;
      const int acc = C::ACC == 2 ? (it & 1) : 0;
      const uint32_t acc_phase = C::ACC == 2 ? ((it >> 1) & 1) : (it & 1);
      const int m0 = (tile % tiles_m) * 256 + rank * 128;
      const int n0 = (tile / tiles_m) * C::BN;
      // the first input tile is requested before waiting for the accumulator
      if (tma_in && sg.role == 0 && lane == 0 && cofs < C::BN && n0 + cofs < N)
        epi_tma_prefetch_input(&map_aux, es, es.ubuf, n0 + cofs, m0 + q * 32,
                               ep.aux_evict_first && ep.epilogue == BP_EPI_DGELU);
      // the tile's bias columns into shared memory, also before the wait: a
      // per-chunk bias load put an L2 round trip on every 32-column chunk
      // (~4 k cycles of a single-tile epilogue, tools/gemm_trace.py)
      const bool sbias = ep.tma_store && ep.bias && sg.role == 0;
      if (sbias) {
        epi_bar<EW>();  // every epilogue warp is done with the previous tile's bias
        for (int j = ew * 32 + lane; j < C::BN; j += 32 * EW)
          sBias[j] = n0 + j < N ? ld_any(ep.bias, ep.bias_dtype, n0 + j) : 0.f;
        epi_bar<EW>();
      }
      mbar_wait(&tfull[acc], acc_phase);
      if (si == 0 && ew == 0 && lane == 0) GTRACE(4);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const int lrow = q * 32 + lane;  // row within this CTA's half tile
      const uint32_t t0 = tmem_base + ((uint32_t)(q * 32) << 16) + acc * C::BN;
      // stream-K roles and the per-thread epilogue: 4 epilogue warps only (launcher)
      if (EW == 4 && OCC == 1 && sg.role == 2) {
        // contributor: raw fp32 partial -> workspace slot, then publish
        float* dst = ws.part + (((size_t)cid * 2 + rank) * 128 + lrow) * C::BN;
#pragma unroll 1
        for (int c = 0; c < C::BN / 32; ++c) {
          float v[32];
          tmem_ld_32x32b_x32(t0 + c * 32, v);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(dst + c * 32)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        __threadfence();
        epi_bar<EW>();
        if (ew == 0 && lane == 0) flag_release(&ws.flag[cid * 2 + rank], ws.epoch);
      } else if (EW == 4 && OCC == 1 && sg.role == 1) {
        // owner: wait for every contributor of this tile, add partials
        const int qlo = sch.contrib_lo(tile);
        for (int q = qlo; q < cid; ++q)
          while (flag_acquire(&ws.flag[q * 2 + rank]) != ws.epoch) {
          }
        // partial sum of all contributors for chunk c, one chunk of lookahead
        auto load_part = [&](int c, float (&acc)[32]) {
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] = 0.f;
          for (int q = qlo; q < cid; ++q) {
            const float4* src =
                reinterpret_cast<const float4*>(ws.part + (((size_t)q * 2 + rank) * 128 + lrow) * C::BN + c * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 t = __ldcg(src + i);
              acc[4 * i] += t.x; acc[4 * i + 1] += t.y; acc[4 * i + 2] += t.z; acc[4 * i + 3] += t.w;
            }
          }
        };
        float nxt[32];
        load_part(0, nxt);
#pragma unroll 1
        for (int c = 0; c < C::BN / 32; ++c) {
          float v[32], cur[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) cur[i] = nxt[i];
          if (c + 1 < C::BN / 32) load_part(c + 1, nxt);
          tmem_ld_32x32b_x32(t0 + c * 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += cur[i];
          if (n0 + c * 32 < N) epi_row32(ep, row, n0 + c * 32, v);
        }
      } else if (EW == 8 || ep.tma_store) {
        if (cofs < C::BN)
          epi_tile_tma<HCH, C::EPI_UNITS>(ep, &map_c, &map_aux, t0 + cofs, m0 + q * 32, lane, n0 + cofs, es, tma_in,
                                          si == 0 && ew == 0, sbias ? sBias + cofs : nullptr, n0 + C::BN);
      } else {
        epi_tile<C::BN / 32>(ep, t0, row, n0);
      }
      tc_fence_before();
      if (leader)
        mbar_arrive(&tempty[acc]);
      else
        mbar_arrive_remote(&tempty[acc], 0);
    }
    if (ew == 0 && lane == 0) GTRACE(5);
    if (ep.tma_store && lane == 0) bulk_wait<0>();  // stores complete before the CTA retires
    if (ew == 0 && lane == 0) GTRACE(6);
  }
  __syncthreads();
  cluster_sync();
  if (warp == 2) tmem_dealloc_2sm<C::TMEM_COLS>(tmem_base);
  if (threadIdx.x == 0) GTRACE(7);
}

// ======================================================== SIMT kernel ====
// 64x64 tile, 256 threads x (4x4) outputs, fp32 FFMA accumulate.
template <typename T>
__global__ void __launch_bounds__(256)
gemm_simt_kernel(int M, int N, int K, const T* __restrict__ A, int64_t lda, int a_kmajor,
                 const T* __restrict__ B, int64_t ldb, int b_kmajor, Epi ep) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      int kk, mm;
      if (a_kmajor) { kk = i % 16; mm = i / 16; } else { mm = i % 64; kk = i / 64; }
      const int gm = m0 + mm, gk = k0 + kk;
      float va = 0.f;
      if (gm < M && gk < K) va = to_f<T>(a_kmajor ? A[(int64_t)gm * lda + gk] : A[(int64_t)gk * lda + gm]);
      As[kk][mm] = va;
      int nn;
      if (b_kmajor) { kk = i % 16; nn = i / 16; } else { nn = i % 64; kk = i / 64; }
      const int gn = n0 + nn;
      const int gk2 = k0 + kk;
      float vb = 0.f;
      if (gn < N && gk2 < K) vb = to_f<T>(b_kmajor ? B[(int64_t)gn * ldb + gk2] : B[(int64_t)gk2 * ldb + gn]);
      Bs[kk][nn] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = m0 + ty * 4 + i, c = n0 + tx * 4 + j;
      if (r < M && c < N) epi_one(ep, r, c, acc[i][j]);
    }
}

// ============================================================== host ======
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// bf16 2-D map over a row-major matrix with `inner` contiguous elements per
// row (row pitch `ld` elements) and `outer` rows; box = box_inner x box_outer.
int make_map_dt(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, int64_t ld,
                uint32_t box_inner, uint32_t box_outer, int dtype, int swizzle_bytes) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BP_ERR_CUDA;
  }
  const int esz = dtype == BP_F32 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(map, dtype == BP_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu ld=%lld box=%ux%u", (int)r,
              (unsigned long long)inner, (unsigned long long)outer, (long long)ld, box_inner, box_outer);
    return BP_ERR_INVALID;
  }
  return BP_OK;
}

int make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, int64_t ld, uint32_t box_inner,
             uint32_t box_outer) {
  return make_map_dt(map, ptr, inner, outer, ld, box_inner, box_outer, BP_BF16, 128);
}

void count_launch();
int num_sms();
bool opt_gemm_simt();
int gemm_mode();

template <int BN, bool A_MN, bool B_MN>
static int launch_tc(const bp_gemm_args& g, const Epi& ep, cudaStream_t st) {
  using C = TcCfg<BN>;
  CUtensorMap ma, mb;
  int rc;
  if (!A_MN)
    rc = make_map(&ma, g.A, g.K, g.M, g.lda, 64, 128);
  else
    rc = make_map(&ma, g.A, g.M, g.K, g.lda, 64, 64);
  if (rc) return rc;
  if (!B_MN)
    rc = make_map(&mb, g.B, g.K, g.N, g.ldb, 64, BN);
  else
    rc = make_map(&mb, g.B, g.N, g.K, g.ldb, 64, 64);
  if (rc) return rc;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    BP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr_set = true;
  }
  const int tiles = ((g.M + 127) / 128) * ((g.N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  kern<<<grid, 256, C::SMEM, st>>>(ma, mb, g.M, g.N, g.K, ep);
  count_launch();
  BP_CHECK_LAUNCH("gemm_tc");
  return BP_OK;
}

template <int BN>
static int dispatch_tc(const bp_gemm_args& g, const Epi& ep, cudaStream_t st) {
  const bool amn = !g.a_kmajor, bmn = !g.b_kmajor;
  if (!amn && !bmn) return launch_tc<BN, false, false>(g, ep, st);
  if (!amn && bmn) return launch_tc<BN, false, true>(g, ep, st);
  if (amn && !bmn) return launch_tc<BN, true, false>(g, ep, st);
  return launch_tc<BN, true, true>(g, ep, st);
}



// Per-stream stream-K workspace (partials + flags).  Concurrent GEMMs on
// different streams never share a slot; the epoch makes flags self-resetting.
struct SkWsState {
  float* part = nullptr;
  size_t part_floats = 0;
  unsigned* flag = nullptr;
  int nflag = 0;
  unsigned epoch = 0;
};
static std::mutex g_sk_mu;
static std::unordered_map<uint64_t, SkWsState> g_sk;

int stream_k_mode();
int gemm_debug_nostore();
int gemm_tma_store_mode();

static int sk_workspace(cudaStream_t st, size_t floats, int nflag, SkWs* out) {
  int dev = 0;
  BP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_sk_mu);
  SkWsState& w = g_sk[(reinterpret_cast<uint64_t>(st) << 4) ^ (uint64_t)dev];
  if (w.part_floats < floats) {
    if (w.part) BP_CUDA(cudaFree(w.part));
    BP_CUDA(cudaMalloc(&w.part, floats * sizeof(float)));
    w.part_floats = floats;
  }
  if (w.nflag < nflag) {
    if (w.flag) BP_CUDA(cudaFree(w.flag));
    BP_CUDA(cudaMalloc(&w.flag, nflag * sizeof(unsigned)));
    BP_CUDA(cudaMemset(w.flag, 0, nflag * sizeof(unsigned)));
    w.nflag = nflag;
  }
  ++w.epoch;
  if (w.epoch == 0) w.epoch = 1;
  out->part = w.part;
  out->flag = w.flag;
  out->epoch = w.epoch;
  return BP_OK;
}

int gemm_grid_mode();

template <int BN, bool A_MN, bool B_MN, int OCC, int EW = 4>
static int launch_tc2(const bp_gemm_args& g, const Epi& ep, cudaStream_t st) {
  using C = Tc2Cfg<BN, B_MN, OCC, EW>;
  CUtensorMap ma, mb;
  int rc;
  if (!A_MN)
    rc = make_map(&ma, g.A, g.K, g.M, g.lda, 64, 128);
  else
    rc = make_map(&ma, g.A, g.M, g.K, g.lda, 64, 64);
  if (rc) return rc;
  if (!B_MN)
    rc = make_map(&mb, g.B, g.K, g.N, g.ldb, 64, C::SUBH);
  else
    rc = make_map(&mb, g.B, g.N, g.K, g.ldb, 64, 64);
  if (rc) return rc;
  // epilogue staging unit = 32 rows x 32 columns (bf16: 64 B rows, fp32: 128 B rows)
  CUtensorMap mc, maux;
  memset(&mc, 0, sizeof(mc));
  memset(&maux, 0, sizeof(maux));
  if (ep.tma_store) {
    const int sw = g.c_dtype == BP_F32 ? 128 : 64;
    if ((rc = make_map_dt(&mc, g.C, g.N, g.M, g.ldc, 32, 32, g.c_dtype, sw))) return rc;
    // aux map: GELU pre-activation output, dGELU input, or the residual input
    if (g.epilogue != BP_EPI_NONE) {
      if ((rc = make_map_dt(&maux, g.aux, g.N, g.M, g.ldaux, 32, 32, g.c_dtype, sw))) return rc;
    } else if (g.residual) {
      if ((rc = make_map_dt(&maux, g.residual, g.N, g.M, g.ldr, 32, 32, g.c_dtype, sw))) return rc;
    }
  }
  auto kern = gemm_tc2_kernel<BN, A_MN, B_MN, OCC, EW>;
  static bool attr_set = false;
  if (!attr_set) {
    BP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr_set = true;
  }
  const int tiles = ((g.M + 255) / 256) * ((g.N + C::BN - 1) / C::BN);
  const int pairs = num_sms() / 2;
  int npairs = tiles < pairs ? tiles : pairs;
  if (gemm_grid_mode() == 1 && tiles >= 4) {
    // throughput grid (co-resident executor): at least two tiles per CTA
    // pair and equal rounds, so every pair overlaps one tile's epilogue with
    // the next tile's MMAs; the SMs left over run other streams' kernels.
    // Less SM-time per GEMM than one exposed-epilogue tile per pair.
    int rounds = (tiles + pairs - 1) / pairs;
    if (rounds < 2) rounds = 2;
    npairs = (tiles + rounds - 1) / rounds;
  }
  SkWs ws{};
  // stream-K: mode 1 = wherever the last wave is ragged; mode 0 (auto) =
  // only sub-wave GEMMs with a long K (>= 64 k-blocks, e.g. the K = 8192
  // MLP-down / LM-head dgrad shapes), which then use all pairs.
  const int skm = stream_k_mode();
  const int kb = (g.K + 63) / 64;
  const bool sk_sub = OCC == 1 && skm != 2 && tiles < pairs && kb >= 64 && tiles * 2 > pairs;
  if (sk_sub) npairs = pairs;
  ws.enable = OCC == 1 && (sk_sub || (skm == 1 && tiles > npairs && tiles % npairs != 0)) ? 1 : 0;
  if (EW == 8 && (ws.enable || !ep.tma_store)) {
    set_error("bp_gemm: 8 epilogue warps need the TMA-store epilogue and no stream-K");
    return BP_ERR_INVALID;
  }
  if (ws.enable) {
    if (int rc = sk_workspace(st, (size_t)npairs * 2 * 128 * C::BN, npairs * 2, &ws)) return rc;
  }
  kern<<<2 * npairs, C::THREADS, C::SMEM, st>>>(ma, mb, mc, maux, g.M, g.N, g.K, ep, ws);
  count_launch();
  BP_CHECK_LAUNCH("gemm_tc2");
  return BP_OK;
}

template <int BN, int OCC = 1, int EW = 4>
static int dispatch_tc2_bn(const bp_gemm_args& g, const Epi& ep, cudaStream_t st) {
  const bool amn = !g.a_kmajor, bmn = !g.b_kmajor;
  if (!amn && !bmn) return launch_tc2<BN, false, false, OCC, EW>(g, ep, st);
  if (!amn && bmn) return launch_tc2<BN, false, true, OCC, EW>(g, ep, st);
  if (amn && !bmn) return launch_tc2<BN, true, false, OCC, EW>(g, ep, st);
  return launch_tc2<BN, true, true, OCC, EW>(g, ep, st);
}

// Pair-tile width BN in {256, 224, 192, 128}.  Per k-block a CTA streams
// 16 KB of A plus BN/2 x 128 B of B from L2, so narrower tiles move more
// bytes per FLOP (measured: BN=128 runs 30% slower per FLOP than 256).
// Model the time of a launch as rounds(BN) * (128 + BN/2) -- the wave
// quantisation over 74 CTA pairs times the per-tile operand traffic -- and
// pick the minimum (N = 8192 at M = 2048: 224 gives exactly 4 waves).
int gemm_wide_mode();

int gemm_force_bn();
int gemm_pick_mode();

int pick_tc2_bn(int M, int N, int pairs, bool b_mn_major) {
  if (const int f = gemm_force_bn()) return f;   // measurement aid (BP_OPT_GEMM_BN)
  // throughput pick (BP_OPT_GEMM_PICK = 1, set by the co-resident executor):
  // several logical devices' streams share the GPU, so CTA pairs a launch
  // leaves idle are taken by other streams' kernels and what counts is each
  // tile's efficiency, not the launch's wave quantisation: 256-wide tiles,
  // the fewest operand bytes per FLOP (BERT-large D=4 N=8: 282 k -> 311 k
  // tok/s for its N = 1024 / 3072 GEMMs, which the model gives 128 / 192;
  // GPT-1.3B's fc1 forward 224 -> 256 with 8 epilogue warps: +0.6 %)
  if (gemm_pick_mode() == 1 && N >= 256 && M >= 256) return 256;
  static const int cand[5] = {256, 512, 224, 192, 128};
  const int tm = (M + 255) / 256;
  int best = 256;
  long best_score = -1;
  const int wide = gemm_wide_mode();
  for (int i = 0; i < 5; ++i) {
    const int bn = cand[i];
    if (bn == 512 && wide != 1) continue;  // measured slower than 256 on every shape: opt-in only
    if (wide == 1 && bn != 512 && N >= 512) continue;  // testing aid: force 512
    // an MN-major B half of 112 / 96 columns still loads two full 64-wide
    // TMA boxes; measured slower than 256, so only K-major B narrows
    if (b_mn_major && (bn == 224 || bn == 192)) continue;
    const long tiles = (long)tm * ((N + bn - 1) / bn);
    const long rounds = (tiles + pairs - 1) / pairs;
    // 512-wide tiles have a single TMEM accumulator: the epilogue is not
    // hidden behind the next tile's MMAs (~12% of a K = 2048 tile)
    const long score = rounds * (128 + bn / 2) * (bn == 512 ? 112 : 100) / 100;
    if (best_score < 0 || score < best_score) {
      best_score = score;
      best = bn;
    }
  }
  return best;
}

int gemm_occ_mode();
int gemm_grid_mode();
int gemm_epi_warps_mode();
int gemm_l2_hints();

static int dispatch_tc2(const bp_gemm_args& g, const Epi& ep, cudaStream_t st) {
  const int pairs = num_sms() / 2;
  const int bn = pick_tc2_bn(g.M, g.N, pairs, !g.b_kmajor);
  // co-resident variant (BP_OPT_GEMM_OCC: 0 never -- the default; 1
  // single-wave launches; 2 always; 3 short-K launches, K <= 1024).
  // Measured: GPT-1.3B step 103.4 k (mode 1) vs 106.7 k tok/s (0) -- two
  // 32 KB stages per CTA do not cover the operand latency of K >= 2048 main
  // loops; BERT-large (K = 1024 GEMMs, epilogue-dominated) 290.0 k (mode 2),
  // 286.3 k (3) vs 278.3 k (0), but a BERT-large stress run with mode 3 hung
  // after 1,747 steps (a CTA pair of this variant at its first cluster
  // barrier, one CTA never through its TMEM allocation): not the default
  const int occm = gemm_occ_mode();
  const long tiles = (long)((g.M + 255) / 256) * ((g.N + bn - 1) / bn);
  const bool occ = occm == 2 || (occm == 1 && tiles <= pairs) || (occm == 3 && g.K <= 1024);
  if (bn <= 256 && occ) {
    switch (bn) {
      case 224: return dispatch_tc2_bn<224, 2>(g, ep, st);
      case 192: return dispatch_tc2_bn<192, 2>(g, ep, st);
      case 128: return dispatch_tc2_bn<128, 2>(g, ep, st);
      default: return dispatch_tc2_bn<256, 2>(g, ep, st);
    }
  }
  // 8 epilogue warps (two per TMEM lane quarter) where a CTA pair has ONE
  // tile: its epilogue is then not hidden behind a next tile's MMAs, and
  // halving each warp's chunk chain shortens the exposed part
  // (BP_OPT_GEMM_EPI_WARPS: 0 auto = single-wave launches, or every launch
  // under the throughput pick; 4 never, 8 always)
  const int ewm = gemm_epi_warps_mode();
  const int kb = (g.K + 63) / 64;
  const bool sk_possible = stream_k_mode() != 2 && tiles < pairs && kb >= 64 && tiles * 2 > pairs;
  const bool ew8_ok = ep.tma_store && bn <= 256 && !sk_possible && stream_k_mode() != 1;
  // Under the co-resident executor (throughput pick) 8 warps on every
  // launch: BERT-large D=4 N=8 313 k -> 330 k tok/s, GPT-1.3B +1.5 % (same
  // boxes), although standalone multi-tile launches gain nothing from it
  if (ew8_ok && (ewm == 8 || (ewm == 0 && (tiles <= pairs || gemm_pick_mode() == 1)))) {
    switch (bn) {
      case 224: return dispatch_tc2_bn<224, 1, 8>(g, ep, st);
      case 192: return dispatch_tc2_bn<192, 1, 8>(g, ep, st);
      case 128: return dispatch_tc2_bn<128, 1, 8>(g, ep, st);
      default: return dispatch_tc2_bn<256, 1, 8>(g, ep, st);
    }
  }
  switch (bn) {
    case 512: return dispatch_tc2_bn<512>(g, ep, st);
    case 224: return dispatch_tc2_bn<224>(g, ep, st);
    case 192: return dispatch_tc2_bn<192>(g, ep, st);
    case 128: return dispatch_tc2_bn<128>(g, ep, st);
    default: return dispatch_tc2_bn<256>(g, ep, st);
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename T, int MODE>
int launch_colred(int rows, int cols, const void* a, int64_t lda, const void* x, const float* mean, const float* rstd,
                  float* out0, float* out1, cudaStream_t st);

// Unfused bias gradient: a column-reduction launch over C after the GEMM.
static int gemm_colsum_after(const bp_gemm_args& g, cudaStream_t st) {
  if (!g.colsum) return BP_OK;
  return g.c_dtype == BP_F32
             ? launch_colred<float, 0>(g.M, g.N, g.C, g.ldc, nullptr, nullptr, nullptr, g.colsum, nullptr, st)
             : launch_colred<__nv_bfloat16, 0>(g.M, g.N, g.C, g.ldc, nullptr, nullptr, nullptr, g.colsum, nullptr, st);
}

}  // namespace bp

using namespace bp;

extern "C" int bp_gemm(const bp_gemm_args* gp, void* stream) {
  if (!gp) {
    set_error("bp_gemm: null args");
    return BP_ERR_INVALID;
  }
  const bp_gemm_args& g = *gp;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) {
    set_error("bp_gemm: bad shape M=%d N=%d K=%d", g.M, g.N, g.K);
    return BP_ERR_INVALID;
  }
  if (g.beta != 0.f && (g.beta != 1.f || g.c_dtype != BP_F32)) {
    set_error("bp_gemm: beta must be 0, or 1 with an fp32 C");
    return BP_ERR_INVALID;
  }
  if ((g.epilogue == BP_EPI_GELU || g.epilogue == BP_EPI_DGELU) && !g.aux) {
    set_error("bp_gemm: GELU epilogues need aux");
    return BP_ERR_INVALID;
  }
  Epi ep;
  ep.M = g.M; ep.N = g.N; ep.C = g.C; ep.ldc = g.ldc; ep.c_dtype = g.c_dtype; ep.alpha = g.alpha;
  ep.accumulate = g.beta != 0.f; ep.bias = g.bias; ep.bias_dtype = g.in_dtype;
  ep.residual = g.residual; ep.ldr = g.ldr; ep.aux = g.aux; ep.ldaux = g.ldaux; ep.epilogue = g.epilogue;
  ep.aux_evict_first = gemm_l2_hints();
  ep.nostore = gemm_debug_nostore();
  ep.tma_store = 0;
  ep.colsum = nullptr;
  const int esz = g.c_dtype == BP_F32 ? 4 : 2;
  ep.vec_ok = aligned16(g.C) && (g.ldc * esz) % 16 == 0 && (!g.bias || aligned16(g.bias)) &&
              (!g.residual || (aligned16(g.residual) && (g.ldr * esz) % 16 == 0)) &&
              (!g.aux || (aligned16(g.aux) && (g.ldaux * esz) % 16 == 0));
  // TMA needs 16-byte aligned bases and row pitches; other bf16 operands
  // (e.g. a vocabulary that is not a multiple of 8) take the SIMT kernel.
  const bool tma_ok = aligned16(g.A) && aligned16(g.B) && (g.lda % 8) == 0 && (g.ldb % 8) == 0;
  if (g.in_dtype == BP_BF16 && !g.force_simt && !opt_gemm_simt() && tma_ok) {
    const int mode = gemm_mode();
    if (mode == 2 || (mode == 0 && g.M >= 256 && g.N >= 256)) {
      // TMA-store epilogue: whole 32-column chunks, 16-byte aligned
      // pitches, at most one extra epilogue input besides bias.
      ep.tma_store = gemm_tma_store_mode() && ep.vec_ok && g.N % 32 == 0 &&
                     (!ep.accumulate || g.c_dtype == BP_F32) &&
                     // TMA-loaded inputs are staged as bf16
                     ((!g.residual && g.epilogue != BP_EPI_DGELU) || g.c_dtype == BP_BF16) &&
                     !(g.residual && (ep.accumulate || g.epilogue != BP_EPI_NONE)) &&
                     !(ep.accumulate && g.epilogue != BP_EPI_NONE);
      if (g.colsum && ep.tma_store && !ep.accumulate) {
        ep.colsum = g.colsum;
        return dispatch_tc2(g, ep, st);
      }
      if (int rc = dispatch_tc2(g, ep, st)) return rc;
      return gemm_colsum_after(g, st);
    }
    const int tiles256 = ((g.M + 127) / 128) * ((g.N + 255) / 256);
    const int rc = (g.N > 128 && tiles256 >= num_sms()) ? dispatch_tc<256>(g, ep, st) : dispatch_tc<128>(g, ep, st);
    return rc ? rc : gemm_colsum_after(g, st);
  }
  dim3 grid((g.N + 63) / 64, (g.M + 63) / 64);
  if (g.in_dtype == BP_F32)
    gemm_simt_kernel<float><<<grid, 256, 0, st>>>(g.M, g.N, g.K, static_cast<const float*>(g.A), g.lda, g.a_kmajor,
                                                   static_cast<const float*>(g.B), g.ldb, g.b_kmajor, ep);
  else
    gemm_simt_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        g.M, g.N, g.K, static_cast<const __nv_bfloat16*>(g.A), g.lda, g.a_kmajor,
        static_cast<const __nv_bfloat16*>(g.B), g.ldb, g.b_kmajor, ep);
  count_launch();
  BP_CHECK_LAUNCH("gemm_simt");
  return gemm_colsum_after(g, st);
}

// Debug aid (BP_GEMM_TRACE builds): copy the per-CTA phase stamps of the
// last 2-SM GEMM launch ([2 * 160][10] long long).
extern "C" __attribute__((visibility("default"))) int bp_gemm_trace_dump(long long* host, int n) {
#ifdef BP_GEMM_TRACE
  const int cap = 2 * 160 * 10, ecap = 2 * 160 * 8 * 5;
  if (cudaMemcpyFromSymbol(host, bp::g_gemm_trace, sizeof(long long) * (n < cap ? n : cap)) != cudaSuccess) return 2;
  if (n >= cap + ecap &&
      cudaMemcpyFromSymbol(host + cap, bp::g_gemm_etrace, sizeof(long long) * ecap) != cudaSuccess)
    return 2;
  return 0;
#else
  (void)host; (void)n;
  return 3;
#endif
}
