/*
 * cachecraft_b200.h — C ABI of the B200-native Cache-Craft fix-up prefill path.
 *
 * The reference (cachecraft 0.1.0, pure Python/numpy) has no FFI: its drop-in
 * boundary is the Python API re-exported from cachecraft/__init__.py:5-94.
 * This header is the native layer UNDER that API: every tensor op the
 * reference performs with numpy on the hot path has one entry point here, and
 * the Python package `paper_2502_15734_b200` binds them with ctypes (see
 * INTEGRATION.md).  Each entry point cites the reference code it replaces
 * (paths relative to /root/reference/pkg/src/cachecraft/).
 *
 * Conventions
 *   - Plain device pointers, element counts and strides; no framework types.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - All calls are asynchronous on `stream` and return CC_OK (0) or a
 *     negative CC_E* code; cc_last_error() returns the thread's last message.
 *   - dtype codes: CC_F64 (parity mode), CC_F32 (parity mode), CC_BF16
 *     (performance mode: bf16 storage, fp32 accumulation).
 *   - "hidden" (the residual stream) is f64 in CC_F64 mode, f32 otherwise.
 *   - Weights are stored [out, in] (K-major, "N x K"): y = x @ W^T.
 *   - The chunk pool is position-free K/V in 16-token blocks laid out
 *     [layer][block][K|V][16][kv_width] (store.py:18 BLOCK_SIZE = 16).
 */
#ifndef CACHECRAFT_B200_H
#define CACHECRAFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CC_ABI_VERSION 1

#if defined(__GNUC__)
#define CC_API __attribute__((visibility("default")))
#else
#define CC_API
#endif

enum cc_dtype { CC_F64 = 0, CC_F32 = 1, CC_BF16 = 2 };

enum cc_status {
  CC_OK = 0,
  CC_E_ARG = -1,     /* invalid argument (maps to ArgumentError / ShapeError) */
  CC_E_CUDA = -2,    /* CUDA runtime / launch failure */
  CC_E_UNSUP = -3,   /* shape or dtype combination not supported by a kernel */
};

/* GEMM epilogues (model.py:399-419) */
enum cc_epilogue {
  CC_EPI_STORE = 0,      /* C = A B^T, stored in C's dtype                    */
  CC_EPI_RESID_ADD = 1,  /* H += A B^T  (H is the f32/f64 residual stream)    */
  CC_EPI_SWIGLU = 2,     /* C[:, j] = silu(g_j) * u_j over 64-col gate|up groups */
  CC_EPI_GELU = 3,       /* C = gelu_tanh(A B^T)  (model.py:125-126)          */
};

/* gather item: one 16-row pool block copied into request slots */
typedef struct {
  int32_t src_block;  /* pool block index                                   */
  int32_t dst_slot;   /* first request slot the block lands on              */
  int32_t n_rows;     /* rows of the block that belong to the request (<=16) */
  int32_t _pad;
} cc_gather_item;

CC_API int cc_abi_version(void);
CC_API const char* cc_last_error(void);
CC_API int cc_sm_count(int device);
/* Number of SIMT (non-tensor-core) GEMM / attention / segment-mass kernel
 * launches made with CC_BF16 data since load.  Only an explicit impl == 2
 * test call reaches them in bf16: the bench and smoke assert it stays 0. */
CC_API long long cc_bf16_simt_launches(void);

/* RoPE cos/sin table [max_pos][half] of (cos, sin) pairs in the engine
 * dtype's float type (double2 for CC_F64, float2 otherwise), angles built in
 * fp64 from inv_freq[half] = base^(-2j/d_head)  (rpe.py:34-36). */
CC_API int cc_rope_table(void* table, const double* inv_freq_dev, int max_pos, int half, int dtype, void* stream);

/* apply_rpe / remove_rpe (rpe.py:47-59): y[n][width] = rotate(x, pos, sign)
 * per d_head slice; float64 in/out (the reference's own precision). */
CC_API int cc_rope_apply_f64(const double* x, double* y, const int64_t* positions, int n, int width,
                      int d_head, const double* inv_freq_dev, int sign, void* stream);

/* K1 — cache -> request K/V assembly fused with key RoPE (model.py:387-393,
 * :404; rpe.py:34-44).  For each item and each layer l in [l0, l1): copy the
 * block's K and V rows into kv_k / kv_v (position-free, returned KV) and write
 * the rotated key into k_rot, skipping slots active at layer l
 * (active_until[slot] > l: the QKV epilogue writes those rows).
 * Request buffers are [layer][n_slots][kv_width]. */
CC_API int cc_gather_rope_kv(const void* pool, int64_t pool_layer_stride, int64_t pool_block_stride,
                      const cc_gather_item* items, int n_items, int l0, int l1,
                      const int32_t* slot_pos, const int32_t* active_until, const void* rope_table,
                      void* kv_k, void* kv_v, void* k_rot, int64_t req_layer_stride,
                      int kv_width, int d_head, int dtype, void* stream);

/* Active-row Q/K/V post-processing after the fused QKV GEMM (model.py:399-404):
 * q_rot[r] = RoPE(q, pos[r]); kv_k[slot] = k; k_rot[slot] = RoPE(k, pos);
 * kv_v[slot] = v.  qkv rows are [q | k | v]. */
CC_API int cc_rope_scatter_qkv(const void* qkv, int64_t ld_qkv, int n_rows, const int32_t* row_slot,
                        const int32_t* row_pos, const void* rope_table, void* q_rot, void* kv_k,
                        void* kv_v, void* k_rot, int n_heads, int n_kv_heads, int d_head, int dtype,
                        void* stream);

/* hidden[r] = embed[token[r]] (model.py:373-374); embed [vocab][d] in dtype. */
CC_API int cc_embed_rows(const void* embed, const int32_t* tokens, void* hidden, int n_rows, int d,
                  int dtype, void* stream);

/* y = x / sqrt(mean(x^2) + eps) * w (model.py:121-122; w may be NULL). */
CC_API int cc_rmsnorm(const void* hidden, void* out, const float* weight, int n_rows, int d, double eps,
               int dtype, void* stream);

/* C = A[M,K] B[N,K]^T with an epilogue (model.py:399-401, :417-419).  A is
 * the normed activations in dtype; B the weight in dtype; for
 * CC_EPI_RESID_ADD, C is the residual stream (f32/f64).  In CC_BF16 mode the
 * tcgen05/TMEM tensor-core kernels run, tiling chosen per shape (1-CTA tiles,
 * swap-AB, or CTA-pair units; impl 0 = product path: bf16 runs the M <= 4
 * GEMV route or the tcgen05 kernel and returns CC_E_UNSUP for a shape neither
 * supports (no silent fallback), fp32/fp64 parity modes run SIMT;
 * 1 = force tcgen05, 2 = force SIMT reference kernel used by tests,
 * 4 = tcgen05 without K splits: a row's result independent of M). */
CC_API int cc_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M,
            int N, int K, int epilogue, int dtype, int impl, void* stream);

/* QKV projection with RoPE and the K/V scatter fused (K3, model.py:399-404;
 * replaces cc_gemm(CC_EPI_STORE) + cc_rope_scatter_qkv): qkv = x W_qkv^T,
 * q_rot[r] = RoPE(q, pos[r]); kv_k[slot[r]] = k; k_rot[slot[r]] = RoPE(k);
 * kv_v[slot[r]] = v.  bf16, d_head 128, (Hq + 2 Hkv) 128 % 256 == 0 and
 * 64 <= n_rows <= 8192: one tcgen05 CTA-pair kernel (epilogue does the
 * rotation and scatter).  Other shapes / dtypes: the GEMM into qkv_scratch
 * ([n_rows][(Hq + 2 Hkv) d_head], may be NULL when the fused kernel applies)
 * followed by cc_rope_scatter_qkv -- bit-identical results in bf16. */
CC_API int cc_gemm_qkv_rope(const void* x, int64_t ldx, const void* w_qkv, int64_t ldw, int n_rows, int d,
                     const int32_t* row_slot, const int32_t* row_pos, const void* rope_table, void* q_rot,
                     void* kv_k, void* kv_v, void* k_rot, void* qkv_scratch, int n_heads, int n_kv_heads,
                     int d_head, int dtype, void* stream);

/* K4 — causal attention of scattered query rows over all request keys
 * (model.py:406-416).  q [n_q][Hq][dh] rotated; k_rot/v [n_keys][Hkv][dh];
 * query row r sees keys j <= q_slot[r] with key_pad[j] == 0.  Writes
 * ctx [n_q][Hq*dh] and lse [n_q][Hq] (natural log of the softmax
 * denominator incl. the running max, scale applied; double in CC_F64 mode,
 * float otherwise). impl: 0 product path (bf16: the tcgen05 kernel only,
 * CC_E_UNSUP for d_head not in {64, 128} or a GQA group not dividing 128;
 * fp32/fp64: SIMT), 1 force tensor-core kernel, 2 force SIMT (tests). */
CC_API int cc_attention(const void* q, const void* k_rot, const void* v, const int32_t* q_slot,
                 const uint8_t* key_pad, void* ctx, void* lse, int n_q, int n_keys, int n_heads,
                 int n_kv_heads, int d_head, int dtype, int impl, void* stream);

/* Materialise softmax weights for AttentionRecord (model.py:320-335, :420):
 * probs [Hq][n_q][n_keys] (double for CC_F64, float otherwise). Debug/test. */
CC_API int cc_attention_probs(const void* q, const void* k_rot, const int32_t* q_slot,
                       const uint8_t* key_pad, const void* lse, void* probs, int n_q, int n_keys,
                       int n_heads, int n_kv_heads, int d_head, int dtype, void* stream);

/* K8a — head-mean attention mass of selected query rows onto key segments
 * (stats.py:68-106 without materialising weights): for each stats row s
 * (query row index rows[s]) mass[s][seg] = (1/Hq) sum_h sum_{j in seg} p_h,
 * mass[s][n_seg] = head-mean diagonal mass (key slot == query slot).
 * Segment seg covers key slots [seg_lo[seg], seg_hi[seg]).  Deterministic
 * (fixed-shape reductions, no atomics). lse as produced by cc_attention. */
CC_API int cc_segment_mass(const void* q, const void* k_rot, const int32_t* q_slot, const uint8_t* key_pad,
                    const void* lse, const int32_t* seg_lo, const int32_t* seg_hi, int n_seg,
                    const int32_t* rows, int n_rows, double* mass, int n_keys, int n_heads,
                    int n_kv_heads, int d_head, int dtype, void* stream);

/* K8b — creation-time chunk statistics (harness.py:331-354, stats.py:68-106)
 * from per-layer masses mass[L][n_rows][n_seg+1] of the rows of chunk
 * spans.  For chunk c (rows [row0[c], row0[c]+len[c]) of the stats rows,
 * segment id seg_of[c]): inter[c][l][j] = sum_rows mass[l][r][j] (j < seg),
 * intra[c][l] = sum_rows (mass[l][r][seg] - mass[l][r][n_seg]),
 * token[c][t] = sum_l sum_{j<seg} mass[l][r][j]. Outputs are packed:
 * inter [n_chunks][L][n_seg], intra [n_chunks][L], token [sum len]. */
CC_API int cc_chunk_stats(const double* mass, int L, int n_rows, int n_seg, const int32_t* row0,
                   const int32_t* len, const int32_t* seg_of, const int32_t* token_off, int n_chunks,
                   double* inter, double* intra, double* token, void* stream);

/* K9 — per-chunk top-count selection (planner.py:17-34): order by
 * (score desc, index asc), keep the first count[c], emit ascending indices
 * into out[off_out[c] ...].  Scores are float64; bit-exact vs the reference.
 * No length limit: chunks up to 8192 tokens sort in shared memory (bitonic),
 * longer ones use an exact radix select over global memory. */
CC_API int cc_topk_select(const double* scores, const int32_t* off, const int32_t* count,
                   const int32_t* off_out, int32_t* out, int n_chunks, int max_len, void* stream);

/* K7 — logits = rmsnorm(h) @ unembed (model.py:94-95) for m rows and the
 * greedy argmax (model.py:455, first maximum wins).  unembed [vocab][d]. */
CC_API int cc_logits_argmax(const void* hidden_rows, const float* norm_w, double eps, const void* unembed,
                     void* logits, int32_t* argmax, int m, int d, int vocab, int dtype, void* stream);

/* K10 — copy request rows [start, start+n_rows) of kv_k/kv_v for all layers
 * into fresh pool blocks (extract_chunk_cache model.py:487-492 +
 * pad_to_blocks store.py:30-53): rows beyond n_rows in the last block are
 * zero.  Never targets blocks of a live (HIT) variant. */
CC_API int cc_extract_to_pool(const void* kv_k, const void* kv_v, int64_t req_layer_stride, int L,
                       int start, int n_rows, const int32_t* blocks, int n_blocks, void* pool,
                       int64_t pool_layer_stride, int64_t pool_block_stride, int kv_width, int dtype,
                       void* stream);

/* ---- tensor parallel: o_proj / down_proj all-reduce over peer memory ---- */

/* Symmetric buffers of every TP rank (device pointers valid in the calling
 * process: same-process, P2P or CUDA-IPC mapped).  Rank r owns columns
 * [r*slice, (r+1)*slice) of the d-wide partial outputs. */
typedef struct {
  float* recv[8];     /* rank r: [world][m_cap][slice] f32 partials pushed to r   */
  int32_t* flags[8];  /* rank r: [world][tiles of r's slice] arrival stamps       */
  float* sum[8];      /* rank r: [m_cap][d] f32 reduced sums                      */
  int32_t* done[8];   /* rank r: monotonic count of reduced tiles written to sum  */
  int32_t rank, world, slice, m_cap, epoch;
} cc_tp_peers;

/* C_partial = A[M,K] B[N=d,K]^T of this rank with the reduce-scatter fused
 * into the tcgen05 GEMM epilogue: each 128xBN fp32 tile is stored straight
 * into its column owner's recv slab (NVLink P2P stores) and stamped with
 * tab->epoch as soon as it is produced (model.py:417, :419 reductions). */
CC_API int cc_tp_push_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
                           const cc_tp_peers* tab, void* stream);
/* Owner side: wait for every rank's stamp of each owned tile, sum the world
 * partials in rank order (deterministic, identical on all ranks) and store
 * the sum into every rank's `sum` (the all-gather), then bump their `done`. */
CC_API int cc_tp_reduce(const cc_tp_peers* tab, int M, int N, void* stream);
/* Stream-ordered wait until this rank's `done` counter reaches `target`. */
CC_API int cc_tp_wait(const cc_tp_peers* tab, int64_t target, void* stream);
/* CUDA IPC: 64-byte handle of the allocation dev_ptr lies in, plus dev_ptr's
 * byte offset from that allocation's base (caching allocators sub-allocate);
 * map a peer's handle (returns the allocation base: add the offset). */
CC_API int cc_ipc_get_handle(const void* dev_ptr, void* handle64, int64_t* offset);
CC_API int cc_ipc_open_handle(const void* handle64, void** dev_ptr);

/* dst[i] += src[i] over n f32 elements (the residual add after a tensor-
 * parallel all-reduce of the o_proj / down_proj partial outputs). */
CC_API int cc_add_f32(float* dst, const float* src, int64_t n, void* stream);

/* ---- decode continuation (model.py:445-484) ---------------------------- */

/* Launch the decode-chain kernels (cc_gemv*, cc_decode_attention*,
 * cc_rope_scatter_qkv, cc_embed_rows, cc_logits_argmax, cc_decode_advance)
 * with programmatic dependent launch: each kernel's independent prologue
 * overlaps its predecessor.  Process-wide; returns the previous setting. */
CC_API int cc_set_pdl(int on);
/* Stream-K GEMM tails on (1, default) / off (0); returns the previous
 * setting.  A stream-K fold spins on its sibling CTAs: with requests in
 * flight on several streams, two such GEMMs could each hold SMs while
 * waiting for CTAs that no SM is free to run, so concurrent (serving) mode
 * turns them off and keeps every GEMM free of cross-CTA waits. */
CC_API int cc_set_stream_k(int on);

/* Weight-streaming projection for 1..4 rows (the per-token QKV / o / MLP
 * products of decode, model.py:461-476): C[M,N] (+)= epi(A[M,K] W[N,K]^T),
 * bf16 A/W, same epilogues and C types as cc_gemm (which routes bf16 M <= 4
 * here when impl == 0).  CC_E_UNSUP unless K % 8 == 0, 16-byte aligned rows
 * and M*K*2 <= 96 KiB. */
CC_API int cc_gemv(const void* A, int64_t lda, const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N,
                   int K, int epilogue, void* stream);

/* cc_gemv with the weighted RMSNorm of the f32 residual rows fused into the
 * prologue (model.py:121-122, eps as cc_rmsnorm, norm_w may be NULL):
 * C = epi(bf16(rmsnorm(hidden)) W^T).  Decode: replaces rmsnorm + gemv. */
CC_API int cc_gemv_rmsnorm(const float* hidden, int64_t ld_hidden, const float* norm_w, double eps, const void* W,
                           int64_t ldw, void* C, int64_t ldc, int M, int N, int K, int epilogue, void* stream);

/* Attention of ONE new query row over all n_keys keys (model.py:467-474: the
 * decode token sees every valid key incl. its own), bf16, d_head 128,
 * split-KV over 128-key chunks with a fixed-order combine (deterministic).
 * q [Hq*dh] rotated; k_rot/v [n_keys][Hkv*dh]; key_pad[j] != 0 masks key j
 * (kv.valid false).  Writes ctx [Hq*dh] and lse [Hq] (as cc_attention). */
CC_API int cc_decode_attention(const void* q, const void* k_rot, const void* v, const uint8_t* key_pad, void* ctx,
                               float* lse, int n_keys, int n_heads, int n_kv_heads, int d_head, void* stream);

/* cc_decode_attention with the key count read from device memory
 * (*n_keys_dev <= max_keys) so one captured CUDA graph replays every decode
 * step; the grid is sized for max_keys and idle chunks exit. */
CC_API int cc_decode_attention_dev(const void* q, const void* k_rot, const void* v, const uint8_t* key_pad,
                                   void* ctx, float* lse, const int32_t* n_keys_dev, int max_keys, int n_heads,
                                   int n_kv_heads, int d_head, void* stream);

/* One decode layer's attention step in ONE launch (model.py:455-474): RoPE of
 * the new row's q and k heads at *pos (rope table as cc_rope_scatter_qkv),
 * the append of k (position-free), rotated k and v at row *slot of the
 * layer's kv_k / k_rot / kv_v [max_keys][Hkv*dh], then the split-KV attention
 * of q over keys 0 .. n_keys-1 (the new key included, key_pad[j] != 0 masks
 * key j) with the chunk combine done by the last CTA of each kv head (fixed
 * chunk order, deterministic).  qkv = the raw projection row [q | k | v].
 * n_keys_dev != NULL: the key count is read on the device (graph replay) and
 * n_keys is ignored; the grid is sized for max_keys (<= 131072).  bf16,
 * d_head 128, GQA group 1/2/4/8.  Same appended bits as cc_rope_scatter_qkv. */
CC_API int cc_decode_attention_qkv(const void* qkv, const int32_t* slot, const int32_t* pos, const void* rope_table,
                                   void* kv_k, void* kv_v, void* k_rot, const uint8_t* key_pad, void* ctx, float* lse,
                                   int n_keys, const int32_t* n_keys_dev, int max_keys, int n_heads, int n_kv_heads,
                                   int d_head, void* stream);

/* Decode step bookkeeping on the device (model.py:455-483 loop state):
 * tokens[state[0]] = *cur_token, then state[0..3] (count, slot, position,
 * live keys) += 1. */
CC_API int cc_decode_advance(int32_t* state, const int32_t* cur_token, int32_t* tokens, void* stream);

/* y[r] = RoPE(x[r], positions[r % n]) for n_rows rows of `width` (= heads x
 * d_head) (rpe.py:19-44 apply_rpe; decode rotates the stored position-free
 * keys at their positions, model.py:467-468).  x == y allowed. */
CC_API int cc_rope_rows(const void* x, void* y, int64_t n_rows, int n, int width, const int32_t* positions,
                        const void* rope_table, int d_head, int dtype, void* stream);

/* Pull a read-only device range (the next projection's weights) into L2 on a
 * side stream while the SMs run other work (engine: o_proj weights during
 * attention). */
CC_API int cc_prefetch_l2(const void* p, size_t bytes, void* stream);

/* L2 flush helper for benchmarks: writes `bytes` of scratch. */
CC_API int cc_flush_l2(void* scratch, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CACHECRAFT_B200_H */
