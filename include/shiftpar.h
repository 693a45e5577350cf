/*
 * shiftpar.h — C-ABI of the B200 (sm_100a) Shift-Parallel forward path.
 *
 * The drop-in boundary between the Python engine (paper_2507_11830_b200,
 * mirroring the reference `shiftsim` Engine API) and the hand-written CUDA
 * kernels in libshiftpar.so.  Conventions:
 *   - plain pointers to caller-owned DEVICE memory, sizes in elements,
 *     row strides ("ld") in elements; no torch types;
 *   - every call is stream-ordered on `stream` (a cudaStream_t, passed as
 *     void*), never synchronises, never allocates device memory;
 *   - return 0 on success, a nonzero sp_status otherwise; sp_last_error()
 *     returns the message of the last failure on the calling thread.
 *     The Python wrapper maps nonzero codes to ContractViolation
 *     (reference errors.py:4-13) BEFORE any further work is enqueued.
 *
 * Each entry cites the reference interface it replaces
 * (/root/reference/pkg/src/shiftsim/<file>:<line>).
 */
#ifndef SHIFTPAR_H_
#define SHIFTPAR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int sp_status;
#define SP_OK 0
#define SP_ERR_INVALID 1     /* argument outside the contract (-> ContractViolation) */
#define SP_ERR_CUDA 2        /* CUDA runtime/launch error */
#define SP_ERR_UNSUPPORTED 3 /* shape/arch the kernels do not cover */

/* GEMM epilogues (sp_gemm_bf16 `epilogue`) */
#define SP_EPI_STORE_BF16 0 /* D(bf16)  = acc */
#define SP_EPI_STORE_F32 1  /* D(f32)   = acc */
#define SP_EPI_ADD_F32 2    /* D(f32)  += acc (residual stream, in place) */
#define SP_EPI_SWIGLU 3     /* D(bf16)  = silu(acc[:, gate]) * acc[:, up]; B rows interleaved
                               in 128-row chunks [gate 128 | up 128], D width N/2 */
#define SP_EPI_GELU 4       /* D(bf16)  = gelu_tanh(acc) (reference-compat MLP) */
#define SP_EPI_PARTIAL_F32 5 /* D(f32) = n raw K-split partial sums [n][M][N] (ldd = N),
                                n = sp_gemm_partials(M, N, K); the consumer sums them in
                                ascending order (sp_add_rmsnorm n_add) — the split-K
                                reduction fused into the next kernel */
/* Flag OR-ed into `epilogue`: ordered regime — every D element is ONE
 * ascending-K chain of 16-deep MMA steps (never the split-K decode regime),
 * so column/row splits of an operand recombine bit-exactly at any M
 * (the matmul contract of tensor_core.py:1-28; used by the operator-level
 * drop-in paper_2507_11830_b200.tensor_core). */
#define SP_GEMM_ORDERED 0x100

/* -------------------------------------------------------------- runtime */
const char* sp_last_error(void);
int sp_abi_version(void);
/* Kernels this library has launched so far in the process (all entries). */
int64_t sp_kernel_launches(void);
/* 0 when the current device is sm_100 (B200) and the kernels can run. */
sp_status sp_device_check(int* sm_count);
/* Debug builds (-DSTEP_TRACE) only: bind a device buffer of `cap` 32-byte
 * records {tag, t_entry, t_wait, t_exit} and a uint32 record counter; every
 * CTA of every kernel then appends its globaltimer stamps (tools/step_trace.py).
 * Returns SP_UNSUPPORTED (3) in production builds.  No reference counterpart:
 * instrumentation of the B200 kernel chain. */
sp_status sp_step_trace_bind(void* buf, void* counter, int cap);

/* --------------------------------------------------------------- GEMM
 * Replaces tensor_core.matmul (tensor_core.py:75-102) for every projection:
 * QKV (parallel_engine.py:359-361 / :479-481), O (:369 / :515), MLP
 * (:374-377 / :516-517) and the LM head (:394 / :534).
 *
 *   D[m, n] = epi( sum_k A[m, k] * B[n, k] )        (bf16 in, f32 accumulate)
 *
 * A: logical [M, K] bf16.  If a_kchunk > 0, K is stored as K/a_kchunk
 *    chunks: element (m, k) lives at A + (k / a_kchunk) * a_chunk_stride
 *    + m * lda + (k % a_kchunk)  (the per-peer layout an all-to-all receive
 *    leaves behind — SP head->seq unpack fused into the operand load).
 * B: [N, K] bf16 (nn.Linear layout, K contiguous), row stride ldb; a TP shard
 *    is a row range or a K-column window of the resident replica (zero copy).
 * D: row stride ldd.  If peer_width > 0, column n is written to
 *    D + (n / peer_width) * peer_stride + m * ldd + (n % peer_width)
 *    (the per-peer contiguous send layout of the SP seq->head all-to-all,
 *    i.e. the pack fused into the epilogue).
 * Fixed tiling: outside the decode regime each D element is one
 * ascending-K reduction independent of M, of the N window and of the tile
 * shape chosen (2-CTA 256x256 pairs or 1-CTA 128x{256,128,64,32}, picked by a
 * wave model) -> row/column splits are bit-exact (the property of
 * tensor_core.py:1-28 the SP path relies on).  Decode regime (M <= 256 and
 * fewer 256-row weight super tiles than SMs): the weight is streamed swap-AB
 * over 256-row super tiles (tokens padded to 32/64/128/256) with K split just
 * enough to cover the SMs; split partials are summed in ascending split order
 * (deterministic within the regime; SP_GEMM_NO_SPLITK=1 disables it).
 */
sp_status sp_gemm_bf16(const void* A, int64_t lda, int64_t a_kchunk, int64_t a_chunk_stride,
                       const void* B, int64_t ldb, void* D, int64_t ldd, int M, int N, int K,
                       int epilogue, int64_t peer_width, int64_t peer_stride, void* stream);
/* Device workspace for the small-M (decode) regime: split-K partials are
 * written here and reduced in ascending split order (deterministic) before
 * the epilogue.  NULL disables split-K.  Results are identical within a
 * regime; across regimes they differ at f32 rounding level. */
sp_status sp_gemm_set_workspace(void* ws, int64_t bytes);
/* QKV projection with RoPE and the paged KV write fused into the epilogue
 * (parallel_engine.py:359-361 QKV matmul + kv_cache.py:99-122 append, with the
 * build's rotary embedding): the [M, (q_heads + 2 kv_heads) * 128] product of
 * A [M, K] and B [N, K] is never stored; q heads are rotated into q_out
 * (row stride ldq), k heads rotated and v heads copied into the pools at
 * slot[m] (slot < 0: skipped) exactly as sp_rope_kv_write lays them out.
 * head_dim 128; rope_table NULL = no rotation.  Bit-identical to
 * sp_gemm_bf16(SP_EPI_STORE_BF16) followed by sp_rope_kv_write. */
sp_status sp_gemm_bf16_qkv_rope(const void* A, int64_t lda, const void* B, int64_t ldb, int M,
                                int K, const int32_t* pos, const int32_t* slot,
                                const float* rope_table, void* q_out, int64_t ldq, void* k_pool,
                                void* v_pool, int q_heads, int kv_heads, int block_size,
                                void* stream);
/* Kernel sp_gemm_bf16 runs for a shape on a GPU with `sms` SMs (host only,
 * split-K workspace assumed): 0 = swap-AB decode kernel, 1 = 2-CTA 256x256
 * pairs, 256/128/64/32 = 1-CTA 128xBN tiles (wave-model choice); -1 = bad
 * arguments.  For diagnostics and tests. */
int sp_gemm_plan(int M, int N, int K, int epilogue, int sms);
/* Number of f32 [M][N] partial slabs SP_EPI_PARTIAL_F32 writes for this shape
 * (1 outside the split-K regime).  Host-only, deterministic. */
int sp_gemm_partials(int M, int N, int K);

/* ------------------------------------------------ fused decode layer
 * One persistent kernel (one CTA per SM) for the projections of a TP (P = 1)
 * decode pass between two attention calls — the layer loop body of
 * _forward_tp (parallel_engine.py:359-379) minus the attention itself:
 *   [leading RMSNorm]  lead_out = norm(x) * lead_gain              (:354)
 *   proj[i]  (in order)  acc = x_in[rows][k] . w[n][k]^T, then by kind:
 *     SP_DL_RES_NORM : x += acc (residual, :369/:377); out = norm(x) * gain
 *                      (:372, or the next layer's :354 / final :390);
 *                      out == NULL: residual add only
 *     SP_DL_SWIGLU   : out[:, c] = silu(acc[gate c]) * acc[up c], w rows
 *                      interleaved [gate 128 | up 128] as SP_EPI_SWIGLU (:376)
 *     SP_DL_ROPE_KV  : the QKV projection (:359-361): q rotated -> q_out,
 *                      k rotated / v -> k_pool / v_pool at slot[r] exactly as
 *                      sp_rope_kv_write lays them out (head_dim 128)
 * Later projections read rows the earlier ones write (proj[i].x may alias an
 * earlier out); the kernel orders them with grid barriers on `sync` (2
 * zero-initialised uint32 per stream; re-armed by the kernel itself, so CUDA
 * graph replays are safe).  rows <= 64; each output is a fixed ascending-k
 * sum of stream-K segment partials: deterministic run to run, equal to the
 * unfused path within f32 summation-order rounding (different K split).
 * Workspace: sp_decode_layer_ws_bytes(args) bytes of f32 partial slabs. */
#define SP_DL_RES_NORM 0
#define SP_DL_SWIGLU 1
#define SP_DL_ROPE_KV 2
typedef struct {
  const void* w;   /* bf16 weight rows [n][k] (K-major), row stride ldw */
  int64_t ldw;
  const void* x;   /* bf16 input rows [rows][k], row stride ldx */
  int64_t ldx;
  int n, k, kind, pad_;
  const float* gain; /* RES_NORM: gain of the normed output */
  void* out;         /* RES_NORM: bf16 [rows][n]; SWIGLU: bf16 [rows][n / 2] */
  int64_t ldo;
} sp_dl_proj;
typedef struct {
  int rows, hidden;     /* decode rows (tokens) <= 64, model width (% 256, <= 8192) */
  float* x;             /* f32 residual stream [rows][ldx], updated in place */
  int64_t ldx;
  float eps;
  int n_proj;           /* 0..4 */
  sp_dl_proj proj[4];
  const float* lead_gain; /* optional leading RMSNorm of x -> lead_out (bf16, ld_lead) */
  void* lead_out;
  int64_t ld_lead;
  const int32_t* pos;   /* ROPE_KV: positions [rows], cache slots [rows] (< 0: skip) */
  const int32_t* slot;
  const float* rope;    /* [pos][64] (cos, sin) pairs; NULL = no rotation */
  void* q_out;          /* bf16 [rows][ldq] */
  int64_t ldq;
  void* k_pool;
  void* v_pool;
  int q_heads, kv_heads, block_size, head_dim;
  void* ws;             /* f32 partial slabs */
  int64_t ws_bytes;
  uint32_t* sync;
} sp_decode_layer_args;
sp_status sp_decode_layer(const sp_decode_layer_args* args, void* stream);
/* Workspace bytes sp_decode_layer needs for these projections (host only; -1 = bad args). */
int64_t sp_decode_layer_ws_bytes(const sp_decode_layer_args* args);

/* ------------------------------------------------ embedding / norms
 * Embedding gather (parallel_engine.py:339-346 TP, :462-469 SP): out[r, :] =
 * f32(table[ids[r], :]) (+ pos_table[pos[r], :] when pos_table != NULL, the
 * reference's additive sinusoidal rows, tensor_core.py:184-206).
 */
sp_status sp_embed(const int32_t* ids, const void* table_bf16, const int32_t* pos,
                   const float* pos_table, float* out_f32, int rows, int hidden, void* stream);

/* Fused residual-add + RMSNorm (tensor_core.py:115-123 at parallel_engine.py
 * :354,:372,:390,:477,:516,:533):
 *   if add != NULL: x[r] += sum_{s < n_add} add[s][r]   (ascending s; written
 *                   back — the TP all-reduce result, or the K-split partials
 *                   of a SP_EPI_PARTIAL_F32 projection: [n_add][rows][hidden])
 *   out[r] = bf16( gain * x[r] / sqrt(mean(x[r]^2) + eps) )
 * If row_idx != NULL, input row r is x[row_idx[r]] (final norm on end rows).
 */
sp_status sp_add_rmsnorm(float* x, int64_t ldx, const float* add, int n_add, const float* gain,
                         float eps, const int32_t* row_idx, void* out_bf16, int64_t ldo, int rows,
                         int hidden, void* stream);

/* ----------------------------------------------- RoPE + paged KV write
 * Replaces KvCache.append (kv_cache.py:99-122) plus positions: for each
 * token r of qkv ([rows, q_heads+2*kv_heads, head_dim] at row stride ldqkv,
 * layout [q | k | v]) apply rotate-half RoPE (table [max_pos, d/2, 2] f32;
 * NULL = no rotation) at pos[r] to q and k, write rotated q to q_out
 * (NULL or q_heads == 0 -> skipped) and k/v to the head-sharded paged pool
 * ([num_blocks][kv_heads][block_size][head_dim], this layer's slice) at
 * slot[r] (block = slot / block_size); slot < 0 skips the row.
 */
sp_status sp_rope_kv_write(const void* qkv, int64_t ldqkv, const int32_t* pos,
                           const int32_t* slot, const float* rope_table, void* q_out,
                           int64_t ldq, void* k_pool, void* v_pool, int rows, int q_heads,
                           int kv_heads, int head_dim, int block_size, void* stream);
/* Same, reading the QKV projection as n_parts f32 K-split partials
 * [n_parts][rows][ldqkv] (SP_EPI_PARTIAL_F32) summed in ascending order and
 * rounded to bf16 first — the split-K reduction fused into this kernel. */
sp_status sp_rope_kv_write_partials(const float* parts, int n_parts, int64_t ldqkv,
                                    const int32_t* pos, const int32_t* slot,
                                    const float* rope_table, void* q_out, int64_t ldq,
                                    void* k_pool, void* v_pool, int rows, int q_heads,
                                    int kv_heads, int head_dim, int block_size, void* stream);

/* ----------------------------------------------------- paged attention
 * Replaces attend_cached (tensor_core.py:135-176) looped per (item, head)
 * at parallel_engine.py:362-368 (TP) / :494-500 (SP) / tails :423-429,
 * :603-611.  Item i owns q rows [cu_q[i], cu_q[i+1]); its first query sits
 * at absolute position first_pos[i] and may attend keys j <= first_pos[i]+t
 * of a window of kv_len[i] keys read through block_tables row i.
 * GQA: q head h reads kv head h / (q_heads / kv_heads).
 * work: int32 pairs (item, first q row of a tile) — host-built schedule;
 * pass n_work = 0 to let the call build the decode schedule (1 row/item).
 * ws: f32 workspace of sp_attn_workspace_bytes() bytes (split-KV partials).
 * q_rows: rows of the q buffer; pool_blocks: blocks of the (per-layer) pool.
 */
sp_status sp_attention(const void* q, int64_t ldq, int64_t q_rows, const void* k_pool,
                       const void* v_pool, int64_t pool_blocks, const int32_t* block_tables,
                       int64_t bt_stride, const int32_t* cu_q,
                       const int32_t* first_pos, const int32_t* kv_len, int n_items,
                       const int32_t* work, int n_work, int max_q_len, int max_kv_len,
                       void* out, int64_t ldo, int q_heads, int kv_heads, int head_dim,
                       int block_size, void* ws, int64_t ws_bytes, void* stream);
/* Split-KV variant of the tcgen05 prefill (head_dim 128) for passes with few
 * work tiles (e.g. one long request under SP=8: 128 CTAs, causal rows up to
 * 64x longer than others).  Entry w of `work` (item, t0) comes with
 * split[w] = (first key tile, end key tile, slot, 0): slot < 0 -> the entry
 * covers all of its keys and stores the output; slot >= 0 -> unnormalised
 * partial O and (max, sum) go to workspace slot `slot * kv_heads + kv_head`
 * ([slots][256][128] f32 then [slots][256][2] f32, slots = ws_bytes /
 * (256*130*4)), and combine entry (item, t0, first slot, n slots) merges them
 * in ascending key order (deterministic). */
sp_status sp_attention_prefill_split(const void* q, int64_t ldq, int64_t q_rows,
                                     const void* k_pool, const void* v_pool, int64_t pool_blocks,
                                     const int32_t* block_tables, int64_t bt_stride,
                                     const int32_t* cu_q, const int32_t* first_pos,
                                     const int32_t* kv_len, const int32_t* work,
                                     const int32_t* split, int n_work, const int32_t* combine,
                                     int n_combine, void* out, int64_t ldo, int q_heads,
                                     int kv_heads, int head_dim, int block_size, void* ws,
                                     int64_t ws_bytes, void* stream);
int64_t sp_attn_workspace_bytes(int n_items, int q_heads, int head_dim, int max_kv_len);
/* Decode attention (one query row per item, cu_q[item] = its row) fed by the
 * QKV projection's K-split partials instead of a rotated Q: replaces the pair
 * kv_cache.append (kv_cache.py:99-122, with RoPE) + attend_cached
 * (tensor_core.py:135-176) of one decode layer (parallel_engine.py:359-368).
 * parts: [n_parts][parts_rows][ld_qkv] f32, ld_qkv = (q_heads + 2 kv_heads)
 * * 128, columns [q heads | k heads | v heads].  The kernel sums the partials
 * in ascending order, rounds to bf16, rotates q and k (rope_table as in
 * sp_rope_kv_write; NULL = none), writes the row's K/V into the pools at
 * slot[row] and attends with its Q — bit-identical to
 * sp_rope_kv_write_partials followed by sp_attention.  head_dim 128,
 * block_size % 64 == 0; ws as for sp_attention. */
sp_status sp_attention_decode_qkv(const float* parts, int n_parts, int64_t ld_qkv, int parts_rows,
                                  const int32_t* pos, const int32_t* slot, const float* rope_table,
                                  void* k_pool, void* v_pool, int64_t pool_blocks,
                                  const int32_t* block_tables, int64_t bt_stride,
                                  const int32_t* cu_q, const int32_t* kv_len, int n_items,
                                  int max_kv_len, void* out, int64_t ldo, int q_heads,
                                  int kv_heads, int block_size, void* ws, int64_t ws_bytes,
                                  void* stream);
/* Tokens per prefill work tile (host schedule).  head_dim 128 with pages of a
 * multiple of 64 keys selects the tcgen05/TMEM kernel (2 x 128 packed rows
 * per CTA); other shapes use the mma.sync kernel (64 packed rows). */
int sp_attn_tile_tokens(int q_heads, int kv_heads, int head_dim, int block_size);

/* ------------------------------------------- all-to-all pack / unpack
 * The reference re-shards with np.ascontiguousarray(tensor[:, lo:hi, :])
 * per peer (parallel_engine.py:539-542) and np.concatenate(..., axis=1)
 * on receive (:514).  pack: src [rows, P*w] -> dst [P][rows][w];
 * unpack: src [P][rows][w] -> dst [rows, P*w]  (bf16, w % 8 == 0).
 */
sp_status sp_a2a_pack(const void* src, int64_t lds, void* dst, int rows, int peers, int width,
                      void* stream);
sp_status sp_a2a_unpack(const void* src, void* dst, int64_t ldd, int rows, int peers,
                        int width, void* stream);

/* ---------------------------------- fused all-to-all over peer memory
 * The SP re-shards without a collective library on the data path:
 *  - seq->head (parallel_engine.py:485-487): the QKV GEMM stores column block
 *    b = n / peer_width of row m straight into peer b's receive buffer,
 *    peer_ptrs[b] + (row_off + m) * ldd + (n % peer_width)  (device array of
 *    P peer pointers — NVLink addresses via symmetric memory, or in-process
 *    buffers for loopback ranks);
 *  - head->seq (:503-509): row t of src [rows_total, width] goes to its owner
 *    s's buffer dst_ptrs[s] at row my_rank * rows_s + (t - lo_s), i.e. the
 *    [P][rows_s][width] layout the O-projection reads through a chunked-K map;
 *  - completion: sp_peer_signal sets flag slot [my_rank] in every peer's flag
 *    array (system-scope release after the stores), sp_peer_wait acquires all
 *    P local flags and resets them.
 */
/* peer_ptrs_host (may be NULL): the same P pointers in host memory.  With them
 * and a bf16 epilogue in the 2-CTA (prefill) regime, each epilogue warp stages
 * 32 rows x 64 columns in shared memory and a TMA store
 * (cp.async.bulk.tensor, one map per peer) writes whole 128-B lines of the
 * peer's rows; otherwise the epilogue stores directly.  SP_PEER_TMA=0 forces
 * the direct stores.  Bit-identical either way. */
sp_status sp_gemm_bf16_to_peers(const void* A, int64_t lda, int64_t a_kchunk,
                                int64_t a_chunk_stride, const void* B, int64_t ldb,
                                const unsigned long long* peer_ptrs,
                                const unsigned long long* peer_ptrs_host, int64_t row_off,
                                int64_t ldd, int M, int N, int K, int epilogue,
                                int64_t peer_width, void* stream);
sp_status sp_peer_scatter_rows(const void* src, int64_t lds, int rows_total, int width, int peers,
                               int my_rank, const unsigned long long* dst_ptrs, void* stream);
sp_status sp_peer_signal(const unsigned long long* flag_ptrs, int peers, int my_rank, void* stream);
sp_status sp_peer_wait(int* flags, int peers, void* stream);
/* TP all-reduce fused into the residual add + RMSNorm (parallel_engine.py
 * :371-372, :379 + :354): x[r] += sum_s part_s[r] (ascending rank s; rank s's
 * partial is its `slabs` K-split slabs [slabs][rows][hidden] f32 at
 * part_ptrs[s], summed in ascending order first); if out != NULL also writes
 * the bf16 RMSNorm of the updated row. */
sp_status sp_peer_allreduce_add_rmsnorm(const unsigned long long* part_ptrs, int peers, int slabs,
                                        float* x, int64_t ldx, const float* gain, float eps,
                                        void* out_bf16, int64_t ldo, int rows, int hidden,
                                        void* stream);
/* Two-shot variant for prefill-size passes (TP all-reduce, fabric.py:117-143,
 * at parallel_engine.py:371/379 followed by the next rms_norm): rank my_rank
 * owns rows [lo, hi) of the contiguous split of `rows` (remainder to low
 * ranks); for each it sums the P f32 partials part_ptrs[s] ([rows][hidden],
 * ascending s), adds them into its residual row x, and stores bf16(gain * x /
 * sqrt(mean(x^2) + eps)) into EVERY rank's xn_ptrs[s] row (row stride ldo).
 * Bit-identical to the one-shot kernel per row; reads (P-1)/P of the bytes. */
sp_status sp_peer_reduce_scatter_rmsnorm(const unsigned long long* part_ptrs, int peers,
                                         int my_rank, float* x, int64_t ldx, const float* gain,
                                         float eps, const unsigned long long* xn_ptrs,
                                         int64_t ldo, int rows, int hidden, void* stream);

/* ---------------------------------------------- reductions and heads
 * In-process (loopback) all-reduce: dst = a + b, f32, ascending order as in
 * DeviceGroup.all_reduce_sum (fabric.py:117-143).
 */
/* Cross-process peer buffers (CUDA IPC) for the fused exchanges when ranks are
 * separate processes: export the allocation holding `ptr` as a 64-byte handle
 * plus the offset of `ptr` inside it; import a peer's handle (mapped over
 * NVLink P2P when the peer is another GPU). */
sp_status sp_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out);
sp_status sp_ipc_import(const void* handle, int64_t offset, void** ptr_out);

sp_status sp_add_f32(const float* a, const float* b, float* dst, int64_t n, void* stream);
/* f64 variant for callers that hand the reference-shaped DeviceGroup f64
 * shards (paper_2507_11830_b200.collectives, fabric.py:117-143). */
sp_status sp_add_f64(const double* a, const double* b, double* dst, int64_t n, void* stream);

/* ------------------------------------- operator-level drop-in primitives
 * The reference's primitive API beyond matmul/attend_cached, f32 in and out
 * (paper_2507_11830_b200.tensor_core binds them):
 *   sp_rms_norm_f32      rms_norm(x, gain, eps)   tensor_core.py:115-123
 *                        out = gain * (x / sqrt(mean(x^2) + eps)) per row
 *   sp_gelu_f32          gelu(x)                  tensor_core.py:126-132 (tanh form)
 *   sp_softmax_rows_f32  softmax_rows(x)          tensor_core.py:105-112
 *                        shift by row max; -inf entries give 0 */
sp_status sp_rms_norm_f32(const float* x, int64_t ldx, const float* gain, float eps, float* out,
                          int64_t ldo, int rows, int hidden, void* stream);
sp_status sp_gelu_f32(const float* x, float* out, int64_t n, void* stream);
sp_status sp_softmax_rows_f32(const float* x, int64_t ldx, float* out, int64_t ldo, int rows,
                              int width, void* stream);
/* greedy_token (model.py:303-307): per row argmax, lowest index wins ties. */
sp_status sp_argmax(const float* logits, int64_t ld, int rows, int vocab, int32_t* idx,
                    float* val, void* stream);
/* dst[r, :] = src[idx[r], :] for f32 rows (end-row / tail selection). */
sp_status sp_gather_rows_f32(const float* src, int64_t lds, const int32_t* idx, float* dst,
                             int64_t ldd, int rows, int width, void* stream);
/* The same for bf16 rows (end rows of a pushed final-norm buffer). */
sp_status sp_gather_rows_bf16(const void* src, int64_t lds, const int32_t* idx, void* dst,
                              int64_t ldd, int rows, int width, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SHIFTPAR_H_ */
