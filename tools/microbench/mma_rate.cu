// tcgen05.mma issue rate in isolation (one CTA per SM, one thread issuing
// back-to-back MMAs into one TMEM accumulator, no other traffic): cycles per
// MMA for the shapes the attention kernels use.  Operand contents are
// whatever shared / tensor memory holds (rate only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_19367_b200/csrc \
//        -I include tools/microbench/mma_rate.cu -o tools/microbench/mma_rate && tools/microbench/mma_rate
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace bp;

// mode 0: SS  M128 N128 (K-major A, K-major B)      -- attention S = Q K^T
// mode 1: TS  M128 N128 (A in TMEM, MN-major B)     -- attention O += P V
// mode 2: SS  M128 N256 (K-major A, K-major B)
// mode 3: SS  M128 N64  (K-major A, K-major B)      -- dK/dV S^T = K Q^T (64 queries)
// mode 4: SS  M128 N128 (K-major A, MN-major B)
// mode 5: the attention forward's MMA-warp sequence without its waits:
//         8 SS MMAs into S buffer (r % 3) (first one overwrites), two
//         commits, 8 TS MMAs into O, two commits
// mode 6: mode 5 with one commit per group
// BG (background work by warps 4..7 while the MMAs run): 0 none, 1 tcgen05.ld
// of 32 columns in a loop (TMEM reads, as the softmax's score loads), 2
// shared-memory 16-byte stores in a loop (as TMA tile writes / P stores),
// 3 shared-memory 16-byte loads in a loop
template <int MODE, int BG = 0>
__global__ void __launch_bounds__(256, 1) mma_rate(int rounds, long long* out, volatile int* stop,
                                                   const uint8_t* gsrc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar[4];
  __shared__ uint64_t bgbar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bgbar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp >= 4 && BG != 0) {  // background traffic until the MMA thread is done
    const int w4 = warp - 4;
    // BG 6: all three at once (warp 4 ld, warp 5 st, warps 6-7 bulk copies), as in the forward
    const int bg = BG != 6 ? BG : (w4 == 0 ? 1 : w4 == 1 ? 4 : 5);
    float acc = 0.f;
    uint4* region = reinterpret_cast<uint4*>(smem + 131072);  // 16 KB per warp... past the operands
    long long n = 0;
    while (*stop == 0) {
      if (bg == 1) {
        float v[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)(w4 * 32) << 16) + 384, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += v[i];
      } else if (bg == 4) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = acc + i;
        tmem_st_32x32b_x32(tmem + ((uint32_t)(w4 * 32) << 16) + 448, v);
        tmem_wait_st();
      } else if (bg == 5) {
        // bulk async copies global -> shared, 16 KB per warp per round (TMA-like tile writes)
        if (lane == 0) {
          uint64_t* b = &bgbar[w4];
          mbar_expect_tx(b, 16384);
          bulk_g2s(smem + 131072 + w4 * 16384, gsrc + w4 * 16384, 16384, b);
          mbar_wait(b, n & 1);
        }
        __syncwarp();
      } else if (bg == 2) {
#pragma unroll
        for (int i = 0; i < 8; ++i) region[(w4 * 8 + i) * 32 + lane] = make_uint4(n, i, lane, w4);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint4 t = region[(w4 * 8 + i) * 32 + lane];
          acc += t.x;
        }
      }
      ++n;
    }
    if (acc == 12345.f) out[1023] = n;
  }
  if (warp == 1 && lane == 0) {
    constexpr int N = MODE == 2 ? 256 : MODE == 3 ? 64 : 128;
    constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, MODE == 1 || MODE == 4);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t ad = umma_desc_sw128(a + (ks >> 2) * 128 * 128 + (ks & 3) * 32, 0, 1024);
        const uint64_t bd = (MODE == 1 || MODE == 4) ? umma_desc_sw128(b + ks * 2048, 128 * 128, 1024)
                                                     : umma_desc_sw128(b + (ks >> 2) * N * 128 + (ks & 3) * 32, 0, 1024);
        if (MODE == 5 || MODE == 6) {
          tc_mma_f16(tmem + (r % 3) * 128, ad, umma_desc_sw128(b + (ks >> 2) * N * 128 + (ks & 3) * 32, 0, 1024),
                     umma_idesc_bf16(128, 128, false, false), ks > 0);
        } else if (MODE == 1)
          tc_mma_f16_ts(tmem, tmem + 256 + 8 * ks, bd, idesc, 1);
        else
          tc_mma_f16(tmem, ad, bd, idesc, 1);
      }
      if (MODE == 5 || MODE == 6) {
        tc_commit(&cbar[0]);
        if (MODE == 5) tc_commit(&cbar[1]);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc_mma_f16_ts(tmem + 384, tmem + (r % 3) * 128 + 8 * ks, umma_desc_sw128(b + ks * 2048, 128 * 128, 1024),
                        umma_idesc_bf16(128, 128, false, true), 1);
        tc_commit(&cbar[2]);
        if (MODE == 5) tc_commit(&cbar[3]);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    if (BG != 0) *stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE, int BG = 0>
static void run(const char* name, int ctas) {
  long long* d;
  int* stop;
  cudaMalloc(&d, 1024 * sizeof(long long));
  cudaMalloc(&stop, sizeof(int));
  const int smem = 1024 + 65536 + 65536 + 65536;
  cudaFuncSetAttribute(mma_rate<MODE, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 2000;
  // one CTA per SM and one flag per launch: the first CTA to finish stops
  // every CTA's background warps (the rate is taken while all were running)
  uint8_t* g;
  cudaMalloc(&g, 1 << 20);
  cudaMemset(stop, 0, sizeof(int));
  mma_rate<MODE, BG><<<ctas, 256, smem>>>(10, d, stop, g);
  cudaMemset(stop, 0, sizeof(int));
  mma_rate<MODE, BG><<<ctas, 256, smem>>>(rounds, d, stop, g);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d, ctas * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  double avg = 0;
  for (int i = 0; i < ctas; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    avg += h[i];
  }
  avg /= ctas;
  const double per = (MODE == 5 || MODE == 6) ? rounds * 16.0 : rounds * 8.0;
  printf("%-44s %3d CTAs: %6.1f cycles / MMA (avg), %6.1f (max CTA)  [%s]\n", name, ctas, avg / per, mx / per,
         cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(stop);
  cudaFree(g);
}

int main() {
  for (int ctas : {1, 148}) {
    run<0>("SS M128 N128 K16 (S = Q K^T)", ctas);
    run<1>("TS M128 N128 K16 (A in TMEM, B MN-major: P V)", ctas);
    run<4>("SS M128 N128 K16 (B MN-major)", ctas);
    run<2>("SS M128 N256 K16", ctas);
    run<3>("SS M128 N64 K16 (dK/dV S^T)", ctas);
  }
  run<5>("attention fwd MMA sequence, 2 commits/group", 148);
  run<6>("attention fwd MMA sequence, 1 commit/group", 148);
  run<5, 1>("attention fwd MMA sequence + tcgen05.ld loop", 148);
  run<5, 4>("attention fwd MMA sequence + tcgen05.st loop", 148);
  run<5, 5>("attention fwd MMA sequence + bulk g2s loop", 148);
  run<5, 6>("attention fwd MMA sequence + ld + st + bulk g2s", 148);
  run<0, 5>("SS N128 + bulk g2s loop", 148);
  run<0, 1>("SS N128 + 4 warps tcgen05.ld loop", 148);
  run<1, 1>("TS N128 + 4 warps tcgen05.ld loop", 148);
  run<0, 2>("SS N128 + 4 warps st.shared.v4 loop", 148);
  run<1, 2>("TS N128 + 4 warps st.shared.v4 loop", 148);
  run<0, 3>("SS N128 + 4 warps ld.shared.v4 loop", 148);
  run<1, 3>("TS N128 + 4 warps ld.shared.v4 loop", 148);
  return 0;
}
