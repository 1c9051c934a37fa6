/*
 * bitpipe.h -- C ABI of libbitpipe_b200.so, the sm_100a compute library of
 * the B200-native BitPipe train step.
 *
 * The reference (pipesched, pure Python) has NO native interface: its
 * train step exists only as the SPEC's `run_schedule_numeric(schedule,
 * model, batch, seed)` (reference SPEC.md:426-434) and its per-task
 * semantics ("each worker executes its task list in order;
 * activations/gradients flow along schedule edges; gradients accumulate
 * over micro-batches; ... replica gradients are averaged (allreduce) before
 * the single weight update").  Each entry point below is one piece of that
 * per-task work; INTEGRATION.md maps them onto the reference's call sites
 * and shows the ctypes binding the Python host driver uses.
 *
 * Conventions
 *   - All pointers are DEVICE pointers owned by the caller (the library
 *     never allocates or frees caller memory).  `stream` is a cudaStream_t
 *     passed as void*.  Every call is asynchronous on that stream.
 *   - Matrices are row-major with an explicit leading dimension in
 *     ELEMENTS.  Token-major activations are [rows = B*S, cols = hidden].
 *   - Return value: BP_OK (0) or an error code; bp_last_error() gives a
 *     thread-local message.  Errors are never swallowed and there is no
 *     CPU fallback: a missing GPU or unsupported shape is an error.
 */
#ifndef BITPIPE_B200_H
#define BITPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_ABI_VERSION 2

#if defined(__GNUC__)
#define BP_API __attribute__((visibility("default")))
#else
#define BP_API
#endif

enum bp_status { BP_OK = 0, BP_ERR_INVALID = 1, BP_ERR_CUDA = 2, BP_ERR_UNSUPPORTED = 3 };
enum bp_dtype { BP_F32 = 0, BP_BF16 = 1 };
enum bp_epilogue {
  BP_EPI_NONE = 0,  /* C = alpha*acc (+bias) (+residual) (+C if beta) */
  BP_EPI_GELU = 1,  /* aux = alpha*acc + bias ; C = gelu(aux)            */
  BP_EPI_DGELU = 2  /* C = alpha*acc * gelu'(aux)   (aux = saved pre-act)  */
};

/* ---------------------------------------------------------------- misc -- */
BP_API int bp_abi_version(void);
BP_API const char* bp_last_error(void);
/* Number of SMs of `device` (sizing persistent grids); <0 on error. */
BP_API int bp_sm_count(int device);
/* 1 if the tcgen05 GEMM path is usable on the current device. */
BP_API int bp_tc_available(void);
/* Count of kernels this library launched since load (per process). */
BP_API unsigned long long bp_launch_count(void);
/* Process-wide switches (testing aids): route attention to the exact
 * kernel / GEMMs to the SIMT kernel even when the fast path applies. */
enum bp_option {
  BP_OPT_ATTN_EXACT = 1, /* attention impl: 0 auto (tcgen05 > mma.sync flash
                            > exact), 1 exact kernel, 2 mma.sync flash       */
  BP_OPT_GEMM_SIMT = 2,  /* 1: SIMT GEMM for bf16 too                          */
  BP_OPT_GEMM_MODE = 3,  /* tcgen05 tiling: 0 auto, 1 single-SM, 2 CTA pair    */
  BP_OPT_STREAM_K = 4,   /* stream-K GEMM scheduling: 0 auto (sub-wave, K >= 4096
                            only), 1 every ragged last wave, 2 off (default:
                            measured slower on the GPT-1.3B shapes).  Testing
                            aid for a GEMM running ALONE on the GPU: its
                            owner CTAs spin on contributor CTAs of the same
                            launch, which can deadlock when kernels of other
                            streams hold SMs (the co-resident executor)     */
  BP_OPT_GEMM_WIDE = 5,  /* 256 x 512 pair tiles: 1 force (default 0: never,
                            measured slower than 256 x 256)                  */
  BP_OPT_GEMM_DEBUG = 6,  /* 1: skip the GEMM epilogue stores (profiling only) */
  BP_OPT_GEMM_TMA_STORE = 7, /* 1 (default): 2-SM GEMM epilogue writes through
                                smem + TMA bulk stores; 0: per-thread stores */
  BP_OPT_LN_UNFUSED = 8,     /* 1: LayerNorm bwd as dx kernel + column kernels
                                (default 0: one fused launch)                */
  BP_OPT_LN_CTAS_PER_SM = 9, /* fused LayerNorm bwd: row blocks per SM (1..8) */
  BP_OPT_LN_BWD_MODE = 10,   /* bf16 LayerNorm bwd at h in {1024,2048,4096}:
                                0 (default) two-pass fused kernel, 1 single-
                                pass TMA-staged kernel (measured 6% slower
                                cold in the train step, equal L2-warm)      */
  BP_OPT_ATTN_FWD_MODE = 11,  /* tcgen05 attention fwd: 0 (default) auto
                                (two query tiles per CTA for non-causal
                                attention at S % 256 == 0, else one), 1 one
                                tile per CTA, 2 two tiles                   */
  BP_OPT_GEMM_OCC = 12,       /* 2-SM GEMM co-resident variant (two CTA pairs
                                per SM pair, one accumulator, 2 stages):
                                0 (default) never; 1 single-wave launches;
                                2 always (tiles <= 256 wide); 3 short-K
                                launches (K <= 1024: BERT-large +3 %).  Off
                                by default: a BERT-large stress run hung
                                after 1,747 steps with a pair of it stuck
                                at its first cluster barrier (one CTA never
                                completed its TMEM allocation)              */
  BP_OPT_GEMM_GRID = 13,      /* 2-SM GEMM grid: 0 (default) one pair per tile
                                up to all pairs; 1 >= 2 tiles per pair in
                                equal rounds, leaving SMs to other streams
                                (measured: GPT-1.3B step 109.0 k vs 109.1 k,
                                BERT-large +2 %: no default change)          */
  BP_OPT_GEMM_BN = 14,        /* 2-SM GEMM pair-tile width: 0 (default) the
                                wave x operand-traffic model, else forced
                                128 / 192 / 224 / 256 / 512 (measurements)  */
  BP_OPT_ATTN_BWD_MODE = 15,  /* tcgen05 attention backward: 0 (default) the
                                dK/dV kernel stores dS^T (bf16, in the
                                workspace) and dQ = dS K runs as a GEMM over
                                it; 1 the dQ kernel recomputes S and dP     */
  BP_OPT_GEMM_EPI_WARPS = 16, /* 2-SM GEMM epilogue warps: 0 (default) 8 on
                                launches with one tile per CTA pair (the
                                epilogue is exposed there) and on every
                                launch under BP_OPT_GEMM_PICK = 1, else 4;
                                4 / 8 force (TMA-store epilogues, no
                                stream-K)                                    */
  BP_OPT_ATTN_FWD_EXF = 17,   /* tcgen05 attention fwd (one query tile per
                                CTA): exponentials per 8 computed on the FMA
                                pipe instead of the MUFU, 2..5 (0: default) */
  BP_OPT_GEMM_L2_HINTS = 18,  /* 1 (default): the GELU GEMM's saved pre-
                                activation is stored L2 evict_first (only
                                the backward reads it) and read evict_first
                                by the dGELU epilogue (its last use); 0:
                                default policy                               */
  BP_OPT_GEMM_PICK = 19,      /* 2-SM GEMM tile width: 0 (default) the wave x
                                operand-traffic model (a GEMM running alone);
                                1 throughput pick -- 256-wide tiles wherever
                                N >= 256 (several streams share the GPU, so
                                idle CTA pairs are filled by other kernels;
                                set by the co-resident executor)             */
};
BP_API int bp_set_option(int option, int value);

/* ---------------------------------------------------------------- GEMM --
 * C[M,N] = epilogue( alpha * op(A)[M,K] . op(B)[K,N] )
 *   a_kmajor = 1 : A stored [M,K] (row-major, lda >= K)
 *   a_kmajor = 0 : A stored [K,M] (row-major, lda >= M)
 *   b_kmajor = 1 : B stored [N,K] (row-major, ldb >= K)   ("x W^T")
 *   b_kmajor = 0 : B stored [K,N] (row-major, ldb >= N)
 * in_dtype BP_BF16 runs the tcgen05/TMEM/TMA tensor-core kernel (fp32
 * accumulate) whenever A/B have 16-byte aligned bases and row pitches
 * (else the SIMT kernel); BP_F32 runs an exact-fp32 SIMT kernel (check
 * mode, no TF32).
 * beta must be 0 or 1; beta = 1 accumulates into C (C must be fp32).
 * bias: [N] in in_dtype or NULL.  residual: [M,N] in c_dtype or NULL.
 * aux : [M,N] in c_dtype (GELU pre-activation) for BP_EPI_GELU/DGELU.
 */
typedef struct bp_gemm_args {
  int M, N, K;
  int in_dtype;
  int a_kmajor, b_kmajor;
  const void* A; int64_t lda;
  const void* B; int64_t ldb;
  void* C; int64_t ldc; int c_dtype;
  float alpha, beta;
  const void* bias;
  const void* residual; int64_t ldr;
  void* aux; int64_t ldaux;
  int epilogue;
  int force_simt; /* testing aid: run the SIMT kernel even for bf16 */
  float* colsum;  /* optional (ABI 2): colsum[n] += sum_m C[m, n] over the
                     values as stored -- the bias gradient when C is a layer's
                     output gradient; fused into the 2-SM epilogue, else a
                     column-reduction launch after the GEMM                 */
} bp_gemm_args;
BP_API int bp_gemm(const bp_gemm_args* args, void* stream);

/* ----------------------------------------------------------- LayerNorm --
 * y = (x - mean) * rstd * gamma + beta over `cols`; mean/rstd saved (fp32).
 * bwd: dx = dres + dLN(dy)   (dres may be NULL); dgamma/dbeta += (fp32).
 */
BP_API int bp_layernorm_fwd(int dtype, int rows, int cols, const void* x, const void* gamma,
                     const void* beta, float eps, void* y, float* mean, float* rstd,
                     void* stream);
BP_API int bp_layernorm_bwd(int dtype, int rows, int cols, const void* dy, const void* x,
                     const void* gamma, const float* mean, const float* rstd,
                     const void* dres, void* dx, float* dgamma, float* dbeta, void* stream);
/* as bp_layernorm_bwd, and dx_colsum[c] += sum_r dx[r, c] (the values as
 * stored) when dx_colsum is non-NULL: the bias gradient of the preceding
 * half-block's output projection, fused into the same launch.           */
BP_API int bp_layernorm_bwd_ex(int dtype, int rows, int cols, const void* dy, const void* x,
                     const void* gamma, const float* mean, const float* rstd,
                     const void* dres, void* dx, float* dgamma, float* dbeta,
                     float* dx_colsum, void* stream);

/* ------------------------------------------------------- elementwise --- */
/* out[r, :] += sum over rows of x (fp32 accumulate into out[cols]). */
BP_API int bp_colsum_acc(int dtype, int rows, int cols, const void* x, int64_t ldx, float* out,
                  void* stream);
/* out[b*S+s, :] = wte[tok[b*S+s], :] + wpe[s, :] */
BP_API int bp_embed_fwd(int dtype, int B, int S, int H, const int32_t* tokens, const void* wte,
                 const void* wpe, void* out, void* stream);
/* dwte[tok] += dout ; dwpe[s] += sum_b dout  (fp32 grads) */
BP_API int bp_embed_bwd(int dtype, int B, int S, int H, const int32_t* tokens, const void* dout,
                 float* dwte, float* dwpe, void* stream);
/* Fused softmax cross-entropy over V columns, in place:
 * logits[r,:] <- (softmax(logits[r,:]) - onehot(target[r])) * grad_scale ;
 * loss_out[0] += loss_scale * sum_r (logsumexp - logit[target]). */
BP_API int bp_xent_fwd_bwd(int dtype, int rows, int V, void* logits, int64_t ld, const int32_t* targets,
                    float grad_scale, float loss_scale, float* loss_out, void* stream);
/* y = x (elementwise cast / copy), n elements */
BP_API int bp_cast(int src_dtype, int dst_dtype, int64_t n, const void* src, void* dst, void* stream);

/* ----------------------------------------------------------- attention --
 * Multi-head attention over a packed QKV activation [B*S, 3*H*Dh]
 * (columns: q heads | k heads | v heads, head-major within each).
 * o: [B*S, H*Dh].  lse: [B*H*S] fp32 (saved for backward).
 * bwd writes dqkv [B*S, 3*H*Dh]; workspace: bp_attn_workspace_bytes().
 */
BP_API int64_t bp_attn_workspace_bytes(int B, int S, int H, int Dh);
BP_API int bp_attn_fwd(int dtype, int B, int S, int H, int Dh, int causal, float scale,
                const void* qkv, void* o, float* lse, void* stream);
BP_API int bp_attn_bwd(int dtype, int B, int S, int H, int Dh, int causal, float scale,
                const void* qkv, const void* o, const void* dout, const float* lse,
                void* dqkv, float* workspace, void* stream);
/* as bp_attn_bwd, and dbias[c] += sum_r dqkv[r, c] (fp32, the values as
 * stored; c < 3*H*Dh) when dbias is non-NULL: the QKV bias gradient, fused
 * into the tcgen05 kernels' epilogues (ABI 2).                           */
BP_API int bp_attn_bwd_ex(int dtype, int B, int S, int H, int Dh, int causal, float scale,
                   const void* qkv, const void* o, const void* dout, const float* lse,
                   void* dqkv, float* workspace, float* dbias, void* stream);

/* -------------------------------------------------------------- Adam ----
 * Fused replica-mean + AdamW on a flat parameter buffer of n elements.
 *   g = (grad_a + grad_b) * 0.5   (grad_b may be NULL: g = grad_a)
 *   g *= grad_scale
 *   m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2
 *   master -= lr * ( mhat / (sqrt(vhat) + eps) + wd * master )
 *   param_a, param_b (optional, param dtype) <- master
 * The order of the replica sum is fixed (a then b) so every replica that
 * performs the update computes bit-identical weights.
 */
BP_API int bp_adam(int64_t n, int param_dtype, float* master, const float* grad_a, const float* grad_b,
            float* m, float* v, void* param_a, void* param_b, float lr, float beta1, float beta2,
            float eps, float weight_decay, int step, float grad_scale, void* stream);
/* as bp_adam with the step counter read on the device from *step_dev when
 * step_dev is non-NULL (ABI 2; CUDA-graph replays of a train step advance it
 * on the device). */
BP_API int bp_adam_dev(int64_t n, int param_dtype, float* master, const float* grad_a, const float* grad_b,
            float* m, float* v, void* param_a, void* param_b, float lr, float beta1, float beta2,
            float eps, float weight_decay, int step, const int* step_dev, float grad_scale, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BITPIPE_B200_H */
