/*
 * nautilus_b200.h -- C ABI of the B200-native MA-tile executor.
 *
 * This is the drop-in boundary that replaces the reference's CPU tile
 * executor.  The reference seam is the Python function
 *
 *   interpret_ma(module, inputs, device, precision) -> (buffers, CostReport)
 *     /root/reference/pkg/src/tilecc/ma/interp.py:102-148
 *   (wrapped by run_pipeline, tilecc/pipeline.py:62-64, and called by the
 *    tuner's score, tilecc/tuner/tuner.py:139, and the CLI gates,
 *    tilecc/cli.py:185,193,288)
 *
 * The host package paper_2604_14825_b200 recognises each MA kernel
 * (tilecc/ma/ir.py:46-62) as one of the kernel families below and calls the
 * matching entry point through ctypes.  All pointers are DEVICE pointers
 * owned by the caller; `stream` is a cudaStream_t (NULL = legacy default
 * stream).  Every entry point is asynchronous on `stream` and returns
 * NT_OK or an error code; nt_last_error() gives a thread-local message.
 * No torch types cross this boundary.
 */
#ifndef NAUTILUS_B200_H_
#define NAUTILUS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2: workspace_bytes in the decode / gemm / chain argument structs (the library
 *    rejects a workspace smaller than the launch needs instead of writing past it) */
#define NT_ABI_VERSION 4

/* status codes (mapped by the host onto tilecc.errors CompilerError subclasses) */
#define NT_OK 0
#define NT_ERR_INVALID 1     /* bad arguments (shape/stride/alignment)            */
#define NT_ERR_UNSUPPORTED 2 /* no sm_100a realisation for this configuration    */
#define NT_ERR_CUDA 3        /* CUDA runtime / driver error                        */

#define NT_MASK_NONE 0
#define NT_MASK_CAUSAL 1 /* Mask[i, j] = 0 if j <= i + causal_offset else -inf */
#define NT_MASK_TENSOR 2 /* explicit fp32 Mask[seq_q, seq_kv] added to S*c    */
#define NT_MASK_BITS 3   /* a 0 / -inf Mask as visibility bits (nt_mask_to_bits):
                          * `mask` = uint32 rows, bit j % 32 of word j / 32 set = key j
                          * visible; mask_stride_row in words (multiple of 4, >=
                          * ceil(seq_kv / 128) * 4); rows 16-byte aligned */

#define NT_DTYPE_BF16 0
#define NT_DTYPE_F32 1
#define NT_DTYPE_E4M3 2 /* fp8 e4m3 (attention inputs, with per-tensor descales) */

/* Rank-4 view [batch, heads, seq, dim]; dim is contiguous; strides in elements. */
typedef struct nt_tensor4 {
  void* ptr;
  int64_t stride_b, stride_h, stride_s;
} nt_tensor4;

/*
 * K1 fused attention forward -- realises the MA kernel the auto-scheduler
 * discovers for softmax(Q (K c)^T [+ Mask]) V (SURVEY.md B.2 / Appendix C
 * V0-V4), i.e. what interpret_ma executes over the block grid i0 with the
 * sequential KV loop j0 (tilecc/ma/interp.py:121-127, 174-211).
 * q/k/v are bf16; o is bf16 or fp32 (out_dtype).  GQA: head hq reads kv head
 * hq / (heads_q / heads_kv).  The batch x head grid is the runtime outer grid.
 */
typedef struct nt_attn_args {
  nt_tensor4 q, k, v, o;
  int32_t batch, heads_q, heads_kv, seq_q, seq_kv, head_dim; /* head_dim 64 or 128 */
  float scale;            /* c in S = Q (K c)^T (1.0 for the unscaled program) */
  int32_t mask_kind;      /* NT_MASK_* */
  int32_t causal_offset;  /* NT_MASK_CAUSAL: 0 = top-left (the MA fixture) */
  const float* mask;      /* NT_MASK_TENSOR: fp32 [seq_q, seq_kv] */
  int64_t mask_stride_row;
  int32_t out_dtype; /* NT_DTYPE_BF16 | NT_DTYPE_F32 */
  int32_t* err_flag; /* device int32 or NULL: bit0 = zero softmax denominator */
  /* device int32[2], zero before the first launch, or NULL.  The kernel is
   * persistent (one CTA per SM); with a counter the CTAs draw work items
   * greedily in LPT order and the last CTA resets it, so one counter serves
   * every launch ordered on one stream.  NULL = static round-robin items. */
  int32_t* work_counter;
  /* the MA kernel's `stages` tunable (0 = the scheduler default 2): K/V tiles
   * kept in flight -- 1 -> one K/V pair (D=128) / two (D=64), >= 2 -> two / four */
  int32_t kv_stages;
  /* q/k/v element type: NT_DTYPE_BF16 (0) or NT_DTYPE_E4M3 (head_dim 128, no or
   * causal mask; tcgen05 kind::f8f6f4 with P rounded to e4m3 -- the paper's FP8
   * regime).  Descales (0 reads as 1): S = (Q K^T) q_descale
   * k_descale c, O = v_descale P V / l. */
  int32_t in_dtype;
  float q_descale, k_descale, v_descale;
  /* split KV for few, long work items (e.g. one kv-group per GPU): device memory
   * of nt_attn_workspace_bytes(args) bytes (0 = never split; NULL or smaller =
   * run unsplit).  The kernel then writes fp32 partials and a merge kernel follows. */
  void* workspace;
  int64_t workspace_bytes;
  /* query rows per work item (ABI 3): 0 = library choice, 256 = two 128-row
   * tiles per CTA (one CTA per SM), 128 = one tile per CTA, two CTAs per SM
   * (bf16 only).  The MA's t0_i tunable realised on the GPU (tuner.py). */
  int32_t item_rows;
} nt_attn_args;
int nt_attn_fwd(const nt_attn_args* args, void* stream);
int64_t nt_attn_workspace_bytes(const nt_attn_args* args);
/* Everything nt_attn_fwd does except the launch: validation, tensor-map encoding,
 * split plan, kernel choice and the per-device shared-memory attribute (which
 * loads the lazily loaded kernel image).  Call once per plan so the first
 * launch costs what every later one does.  No device work is enqueued. */
int nt_attn_prepare(const nt_attn_args* args);
/* CTAs of the kernel `args` selects that are resident per SM (the persistent
 * grid is this x #SMs); a negative NT_ERR_* on invalid arguments. */
int nt_attn_resident_ctas(const nt_attn_args* args);
/* Attention plans: everything of nt_attn_fwd that depends only on the arguments
 * (validation, the five tensor maps, split plan, instantiation choice, kernel
 * load) done once; nt_attn_plan_launch is then one kernel launch (plus the
 * split-KV merge).  The plan keeps the pointers of `args`; the caller keeps the
 * buffers alive.  Not tied to a stream (launches on one stream are ordered), but to
 * the device current at creation: launching with another device current is
 * NT_ERR_INVALID. */
typedef struct nt_attn_plan nt_attn_plan;
int nt_attn_plan_create(const nt_attn_args* args, nt_attn_plan** plan);
int nt_attn_plan_launch(const nt_attn_plan* plan, void* stream);
void nt_attn_plan_destroy(nt_attn_plan* plan);

/*
 * K2 split-KV decode attention + combine (flash-decoding) for short query
 * blocks (seq_q <= 16 rows per (batch, kv-head) group): the reference runs one
 * block with a sequential KV loop; here the KV range is split
 * over CTAs and partial (m, l, O) are merged with the repair law
 * exp2(m_i - m) (tilecc/schedule/repair.py:80-88).  q/k/v bf16, o fp32/bf16.
 * `workspace` must hold nt_decode_workspace_bytes(...) bytes of device memory.
 */
typedef struct nt_decode_args {
  nt_tensor4 q, k, v, o;
  int32_t batch, heads_q, heads_kv, seq_q, seq_kv, head_dim;
  float scale;
  int32_t num_splits; /* >= 1 (see nt_decode_num_splits) */
  int32_t out_dtype;
  void* workspace;
  int32_t* err_flag;
  int64_t workspace_bytes; /* size of `workspace`; < nt_decode_workspace_bytes(...) -> NT_ERR_INVALID */
  /* q/k/v element type (ABI 4): NT_DTYPE_BF16 (0) or NT_DTYPE_E4M3 -- an FP8 KV
   * cache; q is e4m3 too (one kind::f8f6f4 MMA for S and for PV, P in e4m3).
   * Descales (0 reads as 1): S = (q k^T) q_descale k_descale scale, O = v_descale P V / l. */
  int32_t in_dtype;
  float q_descale, k_descale, v_descale;
} nt_decode_args;
/* rows_per_group = (heads_q / heads_kv) * seq_q; workspace = fp32 (O, m, l) per split */
int64_t nt_decode_workspace_bytes(int32_t batch, int32_t heads_kv, int32_t rows_per_group, int32_t head_dim,
                                  int32_t num_splits);
/* split count the library would choose (requested > 0 is clamped to the key count) */
int nt_decode_num_splits(int32_t batch, int32_t heads_kv, int32_t seq_kv, int32_t requested);
int nt_attn_decode(const nt_decode_args* args, void* stream);

/*
 * K2 over a PAGED KV cache: the same split-KV decode,
 * with K/V gathered by TMA page by page from page pools through a block table
 * -- the serving layout of the decode MA's K/V buffers (vLLM/FlashInfer-style
 * "NHD" pools [num_pages, page_size, heads_kv, 128] or "HND" pools
 * [num_pages, heads_kv, page_size, 128]; any element strides with head_dim
 * contiguous).  Sequence b attends to its first seq_lens[b] keys;
 * block_table[b * block_table_stride + i] is the physical page of its
 * logical page i.  page_size: 8, 16, 32, 64 or a multiple of 64.
 * Workspace: nt_decode_workspace_bytes(batch, heads_kv, rows, 128, num_splits),
 * splits from nt_decode_num_splits(batch, heads_kv, max_seq_kv, requested).
 */
typedef struct nt_decode_paged_args {
  nt_tensor4 q, o;                /* [batch, heads_q, seq_q, 128] */
  const void* k_pages;            /* bf16 (or e4m3, in_dtype) page pools */
  const void* v_pages;
  int64_t page_stride, token_stride, head_stride; /* element strides, same for K and V */
  int32_t num_pages, page_size;
  const int32_t* block_table;     /* device int32 [batch, block_table_stride] */
  int32_t block_table_stride;
  const int32_t* seq_lens;        /* device int32 [batch] */
  int32_t batch, heads_q, heads_kv, seq_q, max_seq_kv, head_dim;
  float scale;
  int32_t num_splits;
  int32_t out_dtype;
  void* workspace;
  int32_t* err_flag;
  int64_t workspace_bytes; /* size of `workspace`; too small -> NT_ERR_INVALID */
  /* ABI 4: e4m3 page pools + q (NT_DTYPE_E4M3; page_size dividing or a multiple of
   * 128), descales as in nt_decode_args */
  int32_t in_dtype;
  float q_descale, k_descale, v_descale;
} nt_decode_paged_args;
int nt_attn_decode_paged(const nt_decode_paged_args* args, void* stream);

/*
 * K3 GEMM (tcgen05, fp32 accumulate): C[M,N] = A[M,K] . B[K,N] with bf16 A, B
 * (row-major, unit inner stride) and bf16 or fp32 C
 * (the MA's zero-initialised `acc=Y[...]` accumulation is the GEMM's own K loop).
 * Used twice for the GEMM chain (X.W1).W2 when the Y accumulator does not fit
 * TMEM, and fused (nt_gemm_chain) when E <= 256.
 */
typedef struct nt_gemm_args {
  const void* a; int64_t lda;   /* bf16 [M, K] */
  const void* b; int64_t ldb;   /* bf16 [K, N] */
  void* c; int64_t ldc;         /* out */
  int32_t m, n, k;
  int32_t out_dtype;            /* NT_DTYPE_BF16 | NT_DTYPE_F32 */
  /* split K over CTAs (N <= 128 shapes with few output tiles): fp32 partials in
   * `workspace` (nt_gemm_workspace_bytes), then one reduce launch.  1 / NULL = off. */
  int32_t k_splits;
  void* workspace;
  int64_t workspace_bytes; /* size of `workspace`; k_splits is clamped to what it holds */
} nt_gemm_args;
int nt_gemm(const nt_gemm_args* args, void* stream);
int32_t nt_gemm_k_splits(int32_t m, int32_t n, int32_t k);
int64_t nt_gemm_workspace_bytes(int32_t m, int32_t n, int32_t k);

/* Fused chain Y = (X . W1) . W2 with the T tile kept on chip (E <= 256).
 * F is split over CTAs; fp32 partials go to `workspace`
 * (nt_gemm_chain_workspace_bytes(n, f, e) bytes, may be 0 -> NULL allowed). */
typedef struct nt_chain_args {
  const void* x; int64_t ldx;   /* bf16 [N, K] */
  const void* w1; int64_t ldw1; /* bf16 [K, F] */
  const void* w2; int64_t ldw2; /* bf16 [F, E] */
  void* y; int64_t ldy;         /* out [N, E] */
  int32_t n, k, f, e;
  int32_t out_dtype;
  void* workspace;
  int64_t workspace_bytes; /* size of `workspace`; too small -> NT_ERR_INVALID */
} nt_chain_args;
int64_t nt_gemm_chain_workspace_bytes(int32_t n, int32_t f, int32_t e);
int nt_gemm_chain(const nt_chain_args* args, void* stream);

/*
 * Generic MA programs: MA kernels with no tcgen05
 * family above (element-wise chains, reductions, small matmuls, fp64
 * programs, ...) are lowered by paper_2604_14825_b200/simt.py to CUDA C that
 * mirrors interpret_ma statement by statement (tilecc/ma/interp.py:174-280),
 * compiled by nvcc to an sm_100a cubin (cached by content hash) and run
 * through these entry points -- the load / launch / unload surface of
 * SURVEY.md 8(b).  `image` is a cubin; `fn` is a CUfunction handle; `params`
 * is the cuLaunchKernel parameter array.  Launches are 1-D.
 */
typedef struct nt_module nt_module;
int nt_module_load(const void* image, size_t nbytes, nt_module** out);
int nt_module_function(nt_module* module, const char* entry, void** fn);
int nt_launch(void* fn, uint32_t grid_x, uint32_t block_x, uint32_t smem_bytes, void** params, void* stream);
int nt_module_unload(nt_module* module);

/* dtype conversion helpers (device buffers) */
/* Pack a 0 / -inf fp32 Mask[seq_q, seq_kv] (row stride in elements) into
 * NT_MASK_BITS rows of words_per_row uint32 (>= ceil(seq_kv / 128) * 4; words past
 * seq_kv are written 0).  Sets *flag bit 0 (device int32, may be NULL) if any value
 * is neither 0 nor -inf.  Stream-ordered; seq_q <= 65535. */
int nt_mask_to_bits(const float* mask, int64_t seq_q, int64_t seq_kv, int64_t row_stride, uint32_t* bits,
                    int64_t words_per_row, int32_t* flag, void* stream);
int nt_cast_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream);
int nt_cast_bf16_to_f32(const void* src, float* dst, int64_t n, void* stream);

/* strided host<->device block copy (cudaMemcpy2DAsync, any direction): `height`
 * rows of `width` bytes, row pitches in bytes.  Used by the streamed execution
 * path to move (batch x head) x rows slices of [B, H, S, D] tensors in one call. */
int nt_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                      void* stream);

/* introspection */
int nt_abi_version(void);
const char* nt_last_error(void);
/* number of kernel launches issued by this library since load (for gpu_launches accounting) */
int64_t nt_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* NAUTILUS_B200_H_ */
