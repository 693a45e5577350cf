// Paged causal attention over the head-sharded KV pool (sm_100a).
//
// Replaces tensor_core.attend_cached (tensor_core.py:135-176) as looped per
// (item, local head) by the reference engine (parallel_engine.py:362-368 TP,
// :494-500 SP, SwiftKV tails :423-429 / :603-611).  Semantics: item i's query
// row t sits at absolute position first_pos[i] + t and sees keys
// j <= first_pos[i] + t of its kv_len[i]-key window; softmax in f32.
//
// Prefill kernel: GQA-packed rows — one CTA owns one kv head and a tile of
// (64 / G) tokens x G query heads = 64 packed rows, so each K/V tile loaded
// from the paged pool (cp.async, 128-byte XOR swizzle) feeds all G heads.
// Q K^T and P V run on m16n8k16 bf16 MMAs with f32 online softmax in registers.
// Decode kernel: one CTA per (item, kv head, split); each warp streams its own
// key tiles (double-buffered) for the G packed heads; warps merge in smem and
// splits merge in a combine kernel (flash-decoding).
#include <cstdlib>

#include "../../include/shiftpar.h"
#include <cstring>

#define SP_TU_ID 1  // step-trace tag (common.cuh)
#include "common.cuh"

namespace sp {
int tma_map_bf16(CUtensorMap* out, const void* ptr, int rank, const uint64_t* dims,
                 const uint64_t* strides, const uint32_t* box);
namespace attn {

constexpr float kLog2e = 1.4426950408889634f;

struct Params {
  const __nv_bfloat16* q;
  int64_t ldq;
  const __nv_bfloat16* k_pool;
  const __nv_bfloat16* v_pool;
  const int32_t* block_tables;
  int64_t bt_stride;
  const int32_t* cu_q;
  const int32_t* first_pos;
  const int32_t* kv_len;
  const int2* work;
  __nv_bfloat16* out;
  int64_t ldo;
  int q_heads, kv_heads, group, block_size;
  float scale_log2;
  // decode split-KV
  int n_splits;
  float* ws_o;    // [items][q_heads][splits][HD]
  float* ws_lse;  // [items][q_heads][splits]
  int kv_stream;  // decode: K/V pages read once per step -> L2 evict-first hint
  // TMA decode with the QKV projection left as K-split partials
  // ([n_parts][rows][ld_qkv] f32, columns [q heads | k heads | v heads] x 128):
  // the kernel sums them (ascending), rounds to bf16 and applies RoPE exactly as
  // rope_kv_kernel does, builds its Q in shared memory, and the CTA holding the
  // new token's page writes that token's K/V into the pool before its producer
  // loads the page.  NULL: Q is read from q (written by the RoPE kernel).
  const float* qkv_parts;
  int n_parts, parts_rows;
  int64_t ld_qkv;
  const int32_t* rope_pos;
  const int32_t* rope_slot;
  const float* rope_table;
};

// physical 16-byte chunk index of logical (row, chunk) in a [rows][HD] bf16 tile
template <int HD>
__device__ __forceinline__ int swz(int row, int c) {
  constexpr int NCH = HD / 8;
  if constexpr (NCH >= 8) {
    return c ^ (row & 7);
  } else {
    return c ^ ((row >> 1) & 3);
  }
}

template <int HD>
__device__ __forceinline__ uint32_t tile_addr(const __nv_bfloat16* base, int row, int c) {
  return smem_u32(base + row * HD + swz<HD>(row, c) * 8);
}

// async-load `rows` keys [k0, k0+rows) of one kv head into a swizzled tile
template <int HD>
__device__ __forceinline__ void load_kv_tile(__nv_bfloat16* sdst, const __nv_bfloat16* pool,
                                             const int32_t* bt, int kvh, int kv_heads,
                                             int block_size, int k0, int rows, int kv_len,
                                             int tid, int nthreads) {
  constexpr int NCH = HD / 8;
  for (int i = tid; i < rows * NCH; i += nthreads) {
    const int r = i / NCH, c = i % NCH;
    const int j = k0 + r;
    const bool ok = j < kv_len;
    const __nv_bfloat16* src = pool;
    if (ok) {
      const int64_t page = bt[j / block_size];
      src = pool + ((page * kv_heads + kvh) * block_size + (j % block_size)) * HD + c * 8;
    }
    cp_async16(sdst + r * HD + swz<HD>(r, c) * 8, src, ok);
  }
}

// S[16 x KT] = Q[16 x HD] K^T for one warp; qf: Q fragments per k-step
template <int HD, int KT>
__device__ __forceinline__ void qk_tile(float (&s)[KT / 8][4], const uint32_t (&qf)[HD / 16][4],
                                        const __nv_bfloat16* sK, int lane) {
#pragma unroll
  for (int j = 0; j < KT / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < HD / 16; ++ks) {
#pragma unroll
    for (int j = 0; j < KT / 8; j += 2) {
      const int m = lane >> 3;
      const int key = (j + (m >> 1)) * 8 + (lane & 7);
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4(tile_addr<HD>(sK, key, ks * 2 + (m & 1)), b0, b1, b2, b3);
      mma_bf16_16816(s[j], qf[ks], b0, b1);
      mma_bf16_16816(s[j + 1], qf[ks], b2, b3);
    }
  }
}

// O[16 x HD] += P[16 x KT] V[KT x HD]
template <int HD, int KT>
__device__ __forceinline__ void pv_tile(float (&o)[HD / 8][4], const float (&s)[KT / 8][4],
                                        const __nv_bfloat16* sV, int lane) {
#pragma unroll
  for (int kk = 0; kk < KT / 16; ++kk) {
    uint32_t a[4];
    a[0] = pack_bf16x2(s[2 * kk][0], s[2 * kk][1]);
    a[1] = pack_bf16x2(s[2 * kk][2], s[2 * kk][3]);
    a[2] = pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
    a[3] = pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
    for (int n = 0; n < HD / 8; n += 2) {
      const int m = lane >> 3;
      const int key = kk * 16 + (m & 1) * 8 + (lane & 7);
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4_trans(tile_addr<HD>(sV, key, n + (m >> 1)), b0, b1, b2, b3);
      mma_bf16_16816(o[n], a, b0, b1);
      mma_bf16_16816(o[n + 1], a, b2, b3);
    }
  }
}

// masked online-softmax update for the two rows a thread holds
template <int HD, int KT>
__device__ __forceinline__ void softmax_update(float (&s)[KT / 8][4], float (&o)[HD / 8][4],
                                               float (&mrow)[2], float (&lrow)[2], int kbase,
                                               const int (&limit)[2], bool need_mask,
                                               float scale_log2, int lane) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float v = s[j][2 * h + e] * scale_log2;
        if (need_mask) {
          const int key = kbase + j * 8 + (lane & 3) * 2 + e;
          if (key > limit[h]) v = -INFINITY;
        }
        s[j][2 * h + e] = v;
        mx = fmaxf(mx, v);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mnew = fmaxf(mrow[h], mx);
    const float msafe = mnew == -INFINITY ? 0.f : mnew;
    const float corr = fast_exp2(mrow[h] - msafe);
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float pv = fast_exp2(s[j][2 * h + e] - msafe);
        s[j][2 * h + e] = pv;
        sum += pv;
      }
    }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    lrow[h] = lrow[h] * corr + sum;
    mrow[h] = mnew;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      o[n][2 * h] *= corr;
      o[n][2 * h + 1] *= corr;
    }
  }
}

// load the warp's 16 packed Q rows from a swizzled smem tile into fragments
template <int HD>
__device__ __forceinline__ void load_q_frags(uint32_t (&qf)[HD / 16][4], const __nv_bfloat16* sQ,
                                             int row0, int lane) {
#pragma unroll
  for (int ks = 0; ks < HD / 16; ++ks) {
    ldmatrix_x4(tile_addr<HD>(sQ, row0 + (lane & 15), ks * 2 + (lane >> 4)), qf[ks][0], qf[ks][1],
                qf[ks][2], qf[ks][3]);
  }
}

// ================================================================ prefill
constexpr int PF_WARPS = 4;
constexpr int PF_ROWS = 16 * PF_WARPS;  // packed rows per CTA
constexpr int PF_KT = 64;

template <int HD>
__global__ void __launch_bounds__(PF_WARPS * 32) prefill_kernel(Params p) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sK = sQ + PF_ROWS * HD;        // [2][KT][HD]
  __nv_bfloat16* sV = sK + 2 * PF_KT * HD;      // [2][KT][HD]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 wk = p.work[blockIdx.x];
  const int item = wk.x, tok0 = wk.y;
  const int kvh = blockIdx.y;
  const int G = p.group;
  const int q_row0 = p.cu_q[item];
  const int q_len = p.cu_q[item + 1] - q_row0;
  const int fpos = p.first_pos[item];
  const int kv_len = p.kv_len[item];
  const int32_t* bt = p.block_tables + (int64_t)item * p.bt_stride;
  const int tok_per_cta = PF_ROWS / G;
  const int tok_last = min(tok0 + tok_per_cta, q_len) - 1;
  const int kv_end = min(kv_len, fpos + tok_last + 1);
  const int n_kt = (kv_end + PF_KT - 1) / PF_KT;

  // ---- Q tile (packed rows r -> token tok0 + r / G, head kvh*G + r % G)
  constexpr int NCH = HD / 8;
  for (int i = tid; i < PF_ROWS * NCH; i += PF_WARPS * 32) {
    const int r = i / NCH, c = i % NCH;
    const int t = tok0 + r / G;
    const bool ok = t < q_len;
    const __nv_bfloat16* src = p.q;
    if (ok) src = p.q + (int64_t)(q_row0 + t) * p.ldq + (int64_t)(kvh * G + r % G) * HD + c * 8;
    cp_async16(sQ + r * HD + swz<HD>(r, c) * 8, src, ok);
  }
  load_kv_tile<HD>(sK, p.k_pool, bt, kvh, p.kv_heads, p.block_size, 0, PF_KT, kv_end, tid,
                   PF_WARPS * 32);
  load_kv_tile<HD>(sV, p.v_pool, bt, kvh, p.kv_heads, p.block_size, 0, PF_KT, kv_end, tid,
                   PF_WARPS * 32);
  cp_async_commit();

  const int rowA = warp * 16 + (lane >> 2);  // packed rows held by this thread
  int limit[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = tok0 + (rowA + 8 * h) / G;
    limit[h] = fpos + min(t, q_len - 1);
  }
  const int min_limit = fpos + tok0;

  float o[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];

  for (int kt = 0; kt < n_kt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < n_kt) {
      load_kv_tile<HD>(sK + (buf ^ 1) * PF_KT * HD, p.k_pool, bt, kvh, p.kv_heads, p.block_size,
                       (kt + 1) * PF_KT, PF_KT, kv_end, tid, PF_WARPS * 32);
      load_kv_tile<HD>(sV + (buf ^ 1) * PF_KT * HD, p.v_pool, bt, kvh, p.kv_heads, p.block_size,
                       (kt + 1) * PF_KT, PF_KT, kv_end, tid, PF_WARPS * 32);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kt == 0) load_q_frags<HD>(qf, sQ, warp * 16, lane);
    float s[PF_KT / 8][4];
    qk_tile<HD, PF_KT>(s, qf, sK + buf * PF_KT * HD, lane);
    const int kbase = kt * PF_KT;
    const bool need_mask = kbase + PF_KT - 1 > min_limit;
    softmax_update<HD, PF_KT>(s, o, mrow, lrow, kbase, limit, need_mask, p.scale_log2, lane);
    pv_tile<HD, PF_KT>(o, s, sV + buf * PF_KT * HD, lane);
    __syncthreads();
  }

  // ---- normalise and store
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = rowA + 8 * h;
    const int t = tok0 + r / G;
    if (t >= q_len) continue;
    const float inv = 1.f / lrow[h];
    __nv_bfloat16* dst = p.out + (int64_t)(q_row0 + t) * p.ldo + (int64_t)(kvh * G + r % G) * HD;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      *reinterpret_cast<uint32_t*>(dst + n * 8 + (lane & 3) * 2) =
          pack_bf16x2(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
    }
  }
}

// ================================================================= decode
constexpr int DC_WARPS = 4;
constexpr int DC_KT = 32;

template <int HD>
__global__ void __launch_bounds__(DC_WARPS * 32) decode_kernel(Params p) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw) + warp * (4 * DC_KT * HD);
  __nv_bfloat16* sV = sK + 2 * DC_KT * HD;
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw) + DC_WARPS * 4 * DC_KT * HD;

  const int item = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int G = p.group;
  const int q_row = p.cu_q[item];
  const int kv_len = p.kv_len[item];
  const int32_t* bt = p.block_tables + (int64_t)item * p.bt_stride;
  const int n_tiles = (kv_len + DC_KT - 1) / DC_KT;
  const int per_split = (n_tiles + p.n_splits - 1) / p.n_splits;
  const int t_begin = split * per_split;
  const int t_end = min(n_tiles, t_begin + per_split);

  // ---- packed Q rows (G heads of the single query token), rows >= G are zero
  constexpr int NCH = HD / 8;
  for (int i = tid; i < 16 * NCH; i += DC_WARPS * 32) {
    const int r = i / NCH, c = i % NCH;
    const bool ok = r < G;
    const __nv_bfloat16* src = p.q;
    if (ok) src = p.q + (int64_t)q_row * p.ldq + (int64_t)(kvh * G + r) * HD + c * 8;
    cp_async16(sQ + r * HD + swz<HD>(r, c) * 8, src, ok);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  uint32_t qf[HD / 16][4];
  load_q_frags<HD>(qf, sQ, 0, lane);

  float o[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int limit[2] = {kv_len - 1, kv_len - 1};

  int kt = t_begin + warp;
  if (kt < t_end) {
    load_kv_tile<HD>(sK, p.k_pool, bt, kvh, p.kv_heads, p.block_size, kt * DC_KT, DC_KT, kv_len,
                     lane, 32);
    load_kv_tile<HD>(sV, p.v_pool, bt, kvh, p.kv_heads, p.block_size, kt * DC_KT, DC_KT, kv_len,
                     lane, 32);
  }
  cp_async_commit();
  int buf = 0;
  for (; kt < t_end; kt += DC_WARPS) {
    const int nxt = kt + DC_WARPS;
    if (nxt < t_end) {
      load_kv_tile<HD>(sK + (buf ^ 1) * DC_KT * HD, p.k_pool, bt, kvh, p.kv_heads, p.block_size,
                       nxt * DC_KT, DC_KT, kv_len, lane, 32);
      load_kv_tile<HD>(sV + (buf ^ 1) * DC_KT * HD, p.v_pool, bt, kvh, p.kv_heads, p.block_size,
                       nxt * DC_KT, DC_KT, kv_len, lane, 32);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    float s[DC_KT / 8][4];
    qk_tile<HD, DC_KT>(s, qf, sK + buf * DC_KT * HD, lane);
    const int kbase = kt * DC_KT;
    softmax_update<HD, DC_KT>(s, o, mrow, lrow, kbase, limit, kbase + DC_KT > kv_len, p.scale_log2,
                              lane);
    pv_tile<HD, DC_KT>(o, s, sV + buf * DC_KT * HD, lane);
    __syncwarp();
    buf ^= 1;
  }
  cp_async_wait<0>();
  __syncthreads();  // all warps done with their smem tiles -> reuse as merge scratch

  // ---- merge warps: rows 0..G-1 live in thread rows lane>>2 (h=0)
  float* sm = reinterpret_cast<float*>(smem_raw);  // [warps][16] m, [warps][16] l, [warps][16][HD] o
  float* sl = sm + DC_WARPS * 16;
  float* so = sl + DC_WARPS * 16;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = (lane >> 2) + 8 * h;
    if ((lane & 3) == 0) {
      sm[warp * 16 + r] = mrow[h];
      sl[warp * 16 + r] = lrow[h];
    }
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      so[(warp * 16 + r) * HD + n * 8 + (lane & 3) * 2] = o[n][2 * h];
      so[(warp * 16 + r) * HD + n * 8 + (lane & 3) * 2 + 1] = o[n][2 * h + 1];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * HD; i += DC_WARPS * 32) {
    const int row = i / HD, c = i % HD;
    float mx = -INFINITY;
    for (int w = 0; w < DC_WARPS; ++w) mx = fmaxf(mx, sm[w * 16 + row]);
    float l = 0.f, acc = 0.f;
    if (mx != -INFINITY) {
      for (int w = 0; w < DC_WARPS; ++w) {
        const float f = exp2f(sm[w * 16 + row] - mx);
        l += sl[w * 16 + row] * f;
        acc += so[(w * 16 + row) * HD + c] * f;
      }
    }
    const int qh = kvh * G + row;
    if (p.n_splits == 1) {
      p.out[(int64_t)q_row * p.ldo + (int64_t)qh * HD + c] = __float2bfloat16_rn(acc / l);
    } else {
      const int64_t slot = ((int64_t)item * p.q_heads + qh) * p.n_splits + split;
      p.ws_o[slot * HD + c] = l > 0.f ? acc / l : 0.f;
      if (c == 0) p.ws_lse[slot] = l > 0.f ? mx + log2f(l) : -INFINITY;
    }
  }
}

__global__ void combine_kernel(Params p, int head_dim) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  const int item = blockIdx.x, qh = blockIdx.y;
  const int ns = p.n_splits;  // <= 64 (decode_tma_splits)
  const int64_t base = ((int64_t)item * p.q_heads + qh) * ns;
  // every split's log-sum-exp in one round trip, then the partial rows with
  // 8 loads in flight per thread; the arithmetic (max, then ascending-split
  // weights and sums) is the sequential fold, so results do not change
  __shared__ float lse[64];
  for (int s = threadIdx.x; s < ns; s += blockDim.x) lse[s] = p.ws_lse[base + s];
  const int q_row = p.cu_q[item];
  __syncthreads();
  float mx = -INFINITY;
  for (int s = 0; s < ns; ++s) mx = fmaxf(mx, lse[s]);
  for (int c = threadIdx.x; c < head_dim; c += blockDim.x) {
    float w = 0.f, acc = 0.f;
    for (int s0 = 0; s0 < ns; s0 += 8) {
      float o[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        o[u] = s0 + u < ns && lse[s0 + u] != -INFINITY ? p.ws_o[(base + s0 + u) * head_dim + c] : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (s0 + u >= ns) break;
        const float l = lse[s0 + u];
        if (l == -INFINITY) continue;
        const float f = exp2f(l - mx);
        w += f;
        acc += f * o[u];
      }
    }
    p.out[(int64_t)q_row * p.ldo + (int64_t)qh * head_dim + c] = __float2bfloat16_rn(acc / w);
  }
}


// ============================================================ TMA decode
// head_dim 128, pages of 64*k keys: one CTA per (item, kv head, split); a TMA
// producer warp streams 64-key K/V page slices into a 4-stage mbarrier ring
// (128-byte swizzle) and four consumer warps each take 16 keys of every slice
// (G packed q heads as the m16 rows), keeping private online-softmax state
// that is merged through shared memory at the end.
namespace dec {
constexpr int HD = 128;
constexpr int PAGE = 64;
constexpr int STAGES = 3;  // 3 x 32 KiB ring -> two CTAs per SM
constexpr int NCONS = 4;
constexpr int NUM_THREADS = (NCONS + 1) * 32;
constexpr int TILE_BYTES = PAGE * HD * 2;
constexpr int STAGE_BYTES = 2 * TILE_BYTES;
constexpr int SMEM_Q = 16 * HD * 2;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + SMEM_Q + 1024 + 256;

__device__ __forceinline__ void fence_proxy_async_global_() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Q rows of this CTA's G heads (and, for the new token's CTA, its K and V) from
// the QKV K-split partials: ascending sum, bf16 rounding, RoPE with
// rope_rotate — the arithmetic of rope_kv_kernel (qkv_chunk) bit for bit.
// Q goes to the swizzled sQ tile (rows >= G zero), K/V to the pool at the slot.
template <bool kPlain = false>
__device__ __forceinline__ void build_q_kv(const Params& p, __nv_bfloat16* sQ, int item, int kvh,
                                           bool kv_writer, int tid, int nthreads = NCONS * 32) {
  const int G = p.group;
  const int row = p.cu_q[item];
  const int pos = p.rope_pos[row];
  const int slot = kv_writer ? p.rope_slot[row] : -1;
  // rows G..15 of the m16 Q tile are padding: zero them
  for (int i = tid; i < (16 - G) * (HD / 8); i += nthreads) {
    const int r = G + i / (HD / 8), c = i % (HD / 8);
    *reinterpret_cast<uint4*>(sQ + r * HD + c * 8) = make_uint4(0, 0, 0, 0);
  }
  const int heads = G + (slot >= 0 ? 2 : 0);
  for (int it = tid; it < heads * 16; it += nthreads) {
    const int hh = it >> 4, i0 = (it & 15) * 4;
    int col_head;
    bool rotate = p.rope_table != nullptr;
    if (hh < G) {
      col_head = kvh * G + hh;
    } else if (hh == G) {
      col_head = p.q_heads + kvh;
    } else {
      col_head = p.q_heads + p.kv_heads + kvh;
      rotate = false;
    }
    const float* src = p.qkv_parts + (int64_t)row * p.ld_qkv + (int64_t)col_head * HD + i0;
    const int64_t pstride = (int64_t)p.parts_rows * p.ld_qkv;
    float a[4] = {0.f, 0.f, 0.f, 0.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s0 = 0; s0 < p.n_parts; s0 += 8) {  // 8 slabs' loads in flight, summed in order
      float4 xs[8], ys[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool ok = s0 + k < p.n_parts;
        xs[k] = ok ? *reinterpret_cast<const float4*>(src + (s0 + k) * pstride) : make_float4(0.f, 0.f, 0.f, 0.f);
        ys[k] = ok ? *reinterpret_cast<const float4*>(src + (s0 + k) * pstride + 64) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (s0 + k >= p.n_parts) break;
        a[0] += xs[k].x; a[1] += xs[k].y; a[2] += xs[k].z; a[3] += xs[k].w;
        b[0] += ys[k].x; b[1] += ys[k].y; b[2] += ys[k].z; b[3] += ys[k].w;
      }
    }
    uint32_t ua[2] = {pack_bf16x2(a[0], a[1]), pack_bf16x2(a[2], a[3])};
    uint32_t ub[2] = {pack_bf16x2(b[0], b[1]), pack_bf16x2(b[2], b[3])};
    if (rotate) {
      const float4* cs = reinterpret_cast<const float4*>(p.rope_table + ((int64_t)pos * (HD / 2) + i0) * 2);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float4 c2 = cs[q];
        const float2 fa = unpack_bf16x2(ua[q]);
        const float2 fb = unpack_bf16x2(ub[q]);
        float na0, nb0, na1, nb1;
        rope_rotate(fa.x, fb.x, c2.x, c2.y, na0, nb0);
        rope_rotate(fa.y, fb.y, c2.z, c2.w, na1, nb1);
        ua[q] = pack_bf16x2(na0, na1);
        ub[q] = pack_bf16x2(nb0, nb1);
      }
    }
    if (hh < G) {
      __nv_bfloat16* rowp = sQ + hh * HD;
      if (kPlain) {
        *reinterpret_cast<uint2*>(rowp + i0) = make_uint2(ua[0], ua[1]);
        *reinterpret_cast<uint2*>(rowp + 64 + i0) = make_uint2(ub[0], ub[1]);
      } else {
        *reinterpret_cast<uint2*>(rowp + swz<HD>(hh, i0 >> 3) * 8 + (i0 & 7)) = make_uint2(ua[0], ua[1]);
        *reinterpret_cast<uint2*>(rowp + swz<HD>(hh, (i0 + 64) >> 3) * 8 + (i0 & 7)) = make_uint2(ub[0], ub[1]);
      }
    } else {
      __nv_bfloat16* pool = const_cast<__nv_bfloat16*>(hh == G ? p.k_pool : p.v_pool);
      const int64_t blk = slot / p.block_size, off = slot % p.block_size;
      __nv_bfloat16* dst = pool + ((blk * p.kv_heads + kvh) * p.block_size + off) * HD;
      *reinterpret_cast<uint2*>(dst + i0) = make_uint2(ua[0], ua[1]);
      *reinterpret_cast<uint2*>(dst + 64 + i0) = make_uint2(ub[0], ub[1]);
    }
  }
}

// (key, 16-byte chunk) inside a [2 d-chunks][64 keys][128 B] swizzled slice
__device__ __forceinline__ uint32_t kv_addr(uint32_t base, int key, int c16) {
  return base + (c16 >> 3) * (TILE_BYTES / 2) + key * 128 + ((((c16 & 7) ^ (key & 7))) << 4);
}

__global__ void __launch_bounds__(NUM_THREADS, 2) decode_tma_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Params p) {
  // PDL: the block table, lengths and every KV page before the new token were
  // written by earlier passes / host copies (complete once this grid can
  // launch), so the producer streams the first ring of those pages BEFORE
  // griddepcontrol.wait; only Q and the page holding the new token (written
  // by the predecessor RoPE + KV-write kernel) wait for it.
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + SMEM_Q);
  uint64_t* empty = full + STAGES;
  uint64_t* kv_ready = empty + STAGES;  // fused QKV: the new token's K/V are in the pool
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int item = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int G = p.group;
  const int q_row = p.cu_q[item];
  const int kv_len = p.kv_len[item];
  const int32_t* bt = p.block_tables + (int64_t)item * p.bt_stride;
  const int n_tiles = (kv_len + PAGE - 1) / PAGE;
  const int per_split = (n_tiles + p.n_splits - 1) / p.n_splits;
  const int t_begin = split * per_split;
  const int t_end = min(n_tiles, t_begin + per_split);

  if (warp == NCONS && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NCONS);
    }
    mbar_init(kv_ready, 1);
    fence_barrier_init();
  }
  __syncthreads();  // barriers initialised
  // fused QKV: this CTA holds the new token's page (and writes its K/V)
  const bool kv_writer = p.qkv_parts != nullptr && t_begin <= n_tiles - 1 && n_tiles - 1 < t_end;

  float o[HD / 8][4];
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  if (warp == NCONS) {
    if (lane == 0) {
      const int old_tiles = (kv_len - 1) / PAGE;  // tiles whose keys all precede the new token
      bool waited = false;
      for (int t = t_begin, i = 0; t < t_end; ++t, ++i) {
        if (!waited && (i >= STAGES || t >= old_tiles)) {
          pdl_wait();
          waited = true;
        }
        if (kv_writer && t == old_tiles) mbar_wait(kv_ready, 0);  // written by the consumer warps
        const int s = i % STAGES;
        mbar_wait(empty + s, ((i / STAGES) & 1) ^ 1);
        const int key0 = t * PAGE;
        const int page = bt[key0 / p.block_size];
        const int row = (page * p.kv_heads + kvh) * p.block_size + key0 % p.block_size;
        uint8_t* st = smem + s * STAGE_BYTES;
        mbar_arrive_expect_tx(full + s, STAGE_BYTES);
        if (p.kv_stream) {
          const uint64_t pol = l2_evict_first_policy();
          tma_load_2d_hint(st, &tmK, full + s, 0, row, pol);
          tma_load_2d_hint(st + TILE_BYTES / 2, &tmK, full + s, 64, row, pol);
          tma_load_2d_hint(st + TILE_BYTES, &tmV, full + s, 0, row, pol);
          tma_load_2d_hint(st + TILE_BYTES + TILE_BYTES / 2, &tmV, full + s, 64, row, pol);
        } else {
          tma_load_2d(st, &tmK, full + s, 0, row);
          tma_load_2d(st + TILE_BYTES / 2, &tmK, full + s, 64, row);
          tma_load_2d(st + TILE_BYTES, &tmV, full + s, 0, row);
          tma_load_2d(st + TILE_BYTES + TILE_BYTES / 2, &tmV, full + s, 64, row);
        }
      }
      if (!waited) pdl_wait();
    }
    __syncwarp();
  } else {
    pdl_wait();  // Q (or the QKV partials) is written by the predecessor
    if (p.qkv_parts != nullptr) {
      build_q_kv(p, sQ, item, kvh, kv_writer, tid);
      if (kv_writer) fence_proxy_async_global_();  // pool writes -> this CTA's TMA loads
      asm volatile("bar.sync 1, %0;" ::"n"(NCONS * 32) : "memory");  // consumer warps only
      if (kv_writer && tid == 0) mbar_arrive(kv_ready);
    } else {
      constexpr int NCH = HD / 8;
      for (int i = tid; i < 16 * NCH; i += NCONS * 32) {
        const int r = i / NCH, c = i % NCH;
        const bool ok = r < G;
        const __nv_bfloat16* src = p.q;
        if (ok) src = p.q + (int64_t)q_row * p.ldq + (int64_t)(kvh * G + r) * HD + c * 8;
        cp_async16(sQ + r * HD + swz<HD>(r, c) * 8, src, ok);
      }
      cp_async_commit();
      cp_async_wait<0>();
      asm volatile("bar.sync 1, %0;" ::"n"(NCONS * 32) : "memory");  // consumer warps only
    }
    uint32_t qf[HD / 16][4];
    load_q_frags<HD>(qf, sQ, 0, lane);
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    const int limit[2] = {kv_len - 1, kv_len - 1};
    const int m = lane >> 3;
    for (int t = t_begin, i = 0; t < t_end; ++t, ++i) {
      const int s = i % STAGES;
      mbar_wait(full + s, (i / STAGES) & 1);
      const uint32_t sk = smem_u32(smem + s * STAGE_BYTES);
      const uint32_t sv = sk + TILE_BYTES;
      float sc[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < HD / 16; ++ks) {
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(kv_addr(sk, warp * 16 + (m >> 1) * 8 + (lane & 7), ks * 2 + (m & 1)), b0, b1, b2,
                    b3);
        mma_bf16_16816(sc[0], qf[ks], b0, b1);
        mma_bf16_16816(sc[1], qf[ks], b2, b3);
      }
      const int kbase = t * PAGE + warp * 16;
      softmax_update<HD, 16>(sc, o, mrow, lrow, kbase, limit, kbase + 16 > kv_len, p.scale_log2,
                             lane);
      uint32_t a[4];
      a[0] = pack_bf16x2(sc[0][0], sc[0][1]);
      a[1] = pack_bf16x2(sc[0][2], sc[0][3]);
      a[2] = pack_bf16x2(sc[1][0], sc[1][1]);
      a[3] = pack_bf16x2(sc[1][2], sc[1][3]);
#pragma unroll
      for (int n = 0; n < HD / 8; n += 2) {
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4_trans(kv_addr(sv, warp * 16 + (m & 1) * 8 + (lane & 7), n + (m >> 1)), b0, b1,
                          b2, b3);
        mma_bf16_16816(o[n], a, b0, b1);
        mma_bf16_16816(o[n + 1], a, b2, b3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
  }
  __syncthreads();  // ring free -> merge scratch
  float* sm = reinterpret_cast<float*>(smem);
  float* sl = sm + NCONS * 16;
  float* so = sl + NCONS * 16;
  if (warp < NCONS) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = (lane >> 2) + 8 * h;
      if ((lane & 3) == 0) {
        sm[warp * 16 + r] = mrow[h];
        sl[warp * 16 + r] = lrow[h];
      }
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) {
        so[(warp * 16 + r) * HD + n * 8 + (lane & 3) * 2] = o[n][2 * h];
        so[(warp * 16 + r) * HD + n * 8 + (lane & 3) * 2 + 1] = o[n][2 * h + 1];
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < G * HD; i += NUM_THREADS) {
    const int row = i / HD, c = i % HD;
    float mx = -INFINITY;
    for (int w = 0; w < NCONS; ++w) mx = fmaxf(mx, sm[w * 16 + row]);
    float l = 0.f, acc = 0.f;
    if (mx != -INFINITY) {
      for (int w = 0; w < NCONS; ++w) {
        const float f = exp2f(sm[w * 16 + row] - mx);
        l += sl[w * 16 + row] * f;
        acc += so[(w * 16 + row) * HD + c] * f;
      }
    }
    const int qh = kvh * G + row;
    if (p.n_splits == 1) {
      p.out[(int64_t)q_row * p.ldo + (int64_t)qh * HD + c] = __float2bfloat16_rn(acc / l);
    } else {
      const int64_t slot = ((int64_t)item * p.q_heads + qh) * p.n_splits + split;
      p.ws_o[slot * HD + c] = l > 0.f ? acc / l : 0.f;
      if (c == 0) p.ws_lse[slot] = l > 0.f ? mx + log2f(l) : -INFINITY;
    }
  }
}

// ------------------------------------------------ tcgen05 / TMEM decode
// Same CTA decomposition, TMA producer, KV splits and fused-QKV path as
// decode_tma_kernel, with the tensor-core work on tcgen05: Q (the CTA's G <= 16
// q heads, padded to the M = 128 MMA rows — TMEM rows are independent, the
// padding rows are never read) lives in TMEM as the A operand; per 64-key page
// slice S = Q . K^T (M128 N64, K from the ring) lands in TMEM, one softmax warp
// (lane = q head) turns it into P in place (bf16 over the first 32 columns of
// S), and O += P . V (P from TMEM, V MN-major from the ring) accumulates in
// TMEM.  TMEM: Q 0-63 | S 64-127 | O 128-255 (256 columns: two CTAs per SM).
// Online softmax with the lazy rescale of the prefill kernel; outputs /
// split partials in the format of decode_tma_kernel (same combine kernel).
constexpr int TC_THREADS = 128;  // warp 0 softmax + epilogue, 1 TMA producer, 2 MMA, 3 (+0, 2) Q build
constexpr int TC_SMEM = STAGES * STAGE_BYTES + 16 * HD * 2 + 1024 + 256;

__global__ void __launch_bounds__(TC_THREADS, 2) decode_tc_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Params p) {
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem + STAGES * STAGE_BYTES);  // [16][HD] plain
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + 16 * HD * 2);
  uint64_t* empty = full + STAGES;
  uint64_t* kv_ready = empty + STAGES;
  uint64_t* q_ready = kv_ready + 1;  // Q stored in TMEM
  uint64_t* s_full = q_ready + 1;
  uint64_t* p_ready = s_full + 1;
  uint64_t* o_full = p_ready + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int item = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int G = p.group;
  const int q_row = p.cu_q[item];
  const int kv_len = p.kv_len[item];
  const int32_t* bt = p.block_tables + (int64_t)item * p.bt_stride;
  const int n_tiles = (kv_len + PAGE - 1) / PAGE;
  const int per_split = (n_tiles + p.n_splits - 1) / p.n_splits;
  const int t_begin = split * per_split;
  const int t_end = min(n_tiles, t_begin + per_split);
  const int n_sl = max(t_end - t_begin, 0);

  if (warp == 1 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(kv_ready, 1);
    mbar_init(q_ready, 1);
    mbar_init(s_full, 1);
    mbar_init(p_ready, 1);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t q_tmem = tmem, s_tmem = tmem + 64, o_tmem = tmem + 128;
  const bool kv_writer = p.qkv_parts != nullptr && t_begin <= n_tiles - 1 && n_tiles - 1 < t_end;

  if (warp == 1) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const int old_tiles = (kv_len - 1) / PAGE;
      bool waited = false;
      for (int t = t_begin, i = 0; t < t_end; ++t, ++i) {
        if (!waited && (i >= STAGES || t >= old_tiles)) {
          pdl_wait();
          waited = true;
        }
        if (kv_writer && t == old_tiles) mbar_wait(kv_ready, 0);
        const int s = i % STAGES;
        mbar_wait(empty + s, ((i / STAGES) & 1) ^ 1);
        const int key0 = t * PAGE;
        const int page = bt[key0 / p.block_size];
        const int row = (page * p.kv_heads + kvh) * p.block_size + key0 % p.block_size;
        uint8_t* st = smem + s * STAGE_BYTES;
        mbar_arrive_expect_tx(full + s, STAGE_BYTES);
        if (p.kv_stream) {
          const uint64_t pol = l2_evict_first_policy();
          tma_load_2d_hint(st, &tmK, full + s, 0, row, pol);
          tma_load_2d_hint(st + TILE_BYTES / 2, &tmK, full + s, 64, row, pol);
          tma_load_2d_hint(st + TILE_BYTES, &tmV, full + s, 0, row, pol);
          tma_load_2d_hint(st + TILE_BYTES + TILE_BYTES / 2, &tmV, full + s, 64, row, pol);
        } else {
          tma_load_2d(st, &tmK, full + s, 0, row);
          tma_load_2d(st + TILE_BYTES / 2, &tmK, full + s, 64, row);
          tma_load_2d(st + TILE_BYTES, &tmV, full + s, 0, row);
          tma_load_2d(st + TILE_BYTES + TILE_BYTES / 2, &tmV, full + s, 64, row);
        }
      }
      if (!waited) pdl_wait();
    }
    __syncwarp();
  } else {
    // -------------------------------- Q into TMEM (warps 0, 2 and 3 build it)
    pdl_wait();  // Q (or the QKV partials) is written by the predecessor
    const int ctid = warp == 0 ? lane : (warp == 2 ? 32 : 64) + lane;
    if (p.qkv_parts != nullptr) {
      build_q_kv<true>(p, sQ, item, kvh, kv_writer, ctid, 96);
      if (kv_writer) fence_proxy_async_global_();  // pool writes -> this CTA's TMA loads
    } else {
      for (int i = ctid; i < G * (HD / 8); i += 96) {
        const int r = i / (HD / 8), c = i % (HD / 8);
        *reinterpret_cast<uint4*>(sQ + r * HD + c * 8) =
            *reinterpret_cast<const uint4*>(p.q + (int64_t)q_row * p.ldq + (int64_t)(kvh * G + r) * HD + c * 8);
      }
    }
    asm volatile("bar.sync 1, 96;" ::: "memory");
    if (warp == 2 && kv_writer && lane == 0) mbar_arrive(kv_ready);
    if (warp == 0) {
      // row = lane: its 128 d as 64 bf16x2 columns (lanes >= G: zeros)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
#pragma unroll
        for (int e = 0; e < 32; ++e)
          r[e] = lane < G ? *reinterpret_cast<const uint32_t*>(sQ + lane * HD + c * 64 + 2 * e) : 0u;
        tmem_st32(q_tmem + c * 32, r);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_ready);
    }
      if (warp == 2) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0 && n_sl > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, PAGE);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, HD) | (1u << 16);  // V MN-major
      mbar_wait(q_ready, 0);
      tc_fence_after();
      for (int i = 0; i <= n_sl; ++i) {
        if (i > 0) {  // P(i-1) . V(i-1), then release the slice
          mbar_wait(p_ready, (i - 1) & 1);
          tc_fence_after();
          const uint32_t sv = smem_u32(smem + ((i - 1) % STAGES) * STAGE_BYTES + TILE_BYTES);
#pragma unroll
          for (int k = 0; k < PAGE / 16; ++k)
            umma_ts_bf16(o_tmem, s_tmem + k * 8, sdesc_sw128_mn(sv + k * 2048, TILE_BYTES / 2),
                         idesc_pv, (i > 1 || k > 0) ? 1u : 0u);
          umma_commit(empty + (i - 1) % STAGES);
          if (i == n_sl) umma_commit(o_full);
        }
        if (i < n_sl) {  // S(i) = Q . K(i)^T (after P(i-1) is consumed: same columns)
          const int s = i % STAGES;
          mbar_wait(full + s, (i / STAGES) & 1);
          tc_fence_after();
          const uint32_t sk = smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k)
            umma_ts_bf16(s_tmem, q_tmem + k * 8,
                         sdesc_sw128(sk + (k >> 2) * (TILE_BYTES / 2) + (k & 3) * 32), idesc_qk,
                         k > 0 ? 1u : 0u);
          umma_commit(s_full);
        }
      }
    }
    __syncwarp();
      } else if (warp == 0) {
    // ------------------------------------------------------ softmax / epilogue
    float m_run = -INFINITY, l_run = 0.f;
    const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2);
    for (int i = 0; i < n_sl; ++i) {
      mbar_wait(s_full, i & 1);
      tc_fence_after();
      float sv[PAGE];
      {
        uint32_t r[2][32];
        tmem_ld32(s_tmem, r[0]);
        tmem_ld32(s_tmem + 32, r[1]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) sv[c * 32 + e] = __uint_as_float(r[c][e]);
      }
      const int kbase = (t_begin + i) * PAGE;
      if (kbase + PAGE > kv_len) {
#pragma unroll
        for (int e = 0; e < PAGE; ++e)
          if (kbase + e >= kv_len) sv[e] = -INFINITY;
      }
      float mxs[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) mxs[q] = fmaxf(sv[2 * q], sv[2 * q + 1]);
#pragma unroll
      for (int e = 16; e < PAGE; e += 16)
#pragma unroll
        for (int q = 0; q < 8; ++q) mxs[q] = fmaxf(mxs[q], fmaxf(sv[e + 2 * q], sv[e + 2 * q + 1]));
#pragma unroll
      for (int w = 4; w; w >>= 1)
#pragma unroll
        for (int q = 0; q < w; ++q) mxs[q] = fmaxf(mxs[q], mxs[q + w]);
      const float m_new = fmaxf(m_run, mxs[0] * p.scale_log2);
      const bool need = m_new > m_run + 8.0f;
      float corr = 1.f;
      if (need) {
        corr = fast_exp2(m_run - m_new);
        m_run = m_new;
      }
      l_run *= corr;
      if (i > 0 && __any_sync(0xffffffffu, need)) {  // P.V(i-1) is complete (covered by s_full)
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(o_tmem + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * corr);
          tmem_st32(o_tmem + c * 32, r);
        }
        tmem_st_wait();
      }
      const uint64_t nm2 = f2_pack(-m_run, -m_run);
      uint64_t sums[4] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        float a, b;
        const uint64_t x2 = f2_fma(f2_pack(sv[2 * e], sv[2 * e + 1]), sc2, nm2);
        f2_unpack(x2, a, b);
        a = fast_exp2(a);
        b = fast_exp2(b);
        sums[e & 3] = f2_add(sums[e & 3], f2_pack(a, b));
        pk[e] = pack_bf16x2(a, b);
      }
      tmem_st32(s_tmem, pk);
      const uint64_t sum2 = f2_add(f2_add(sums[0], sums[1]), f2_add(sums[2], sums[3]));
      float sa, sb;
      f2_unpack(sum2, sa, sb);
      l_run += sa + sb;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
    }
    // epilogue: row = lane (q head kvh * G + lane)
    float o[HD];
    if (n_sl > 0) {
      mbar_wait(o_full, 0);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(o_tmem + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) o[c * 32 + e] = __uint_as_float(r[e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < HD; ++e) o[e] = 0.f;
    }
    if (lane < G) {
      const int qh = kvh * G + lane;
      const bool ok = l_run > 0.f;
      const float inv = ok ? 1.f / l_run : 0.f;
      if (p.n_splits == 1) {
        uint4* d4 = reinterpret_cast<uint4*>(p.out + (int64_t)q_row * p.ldo + (int64_t)qh * HD);
#pragma unroll
        for (int q = 0; q < HD / 8; ++q) {
          uint4 u;
          u.x = pack_bf16x2(o[8 * q + 0] * inv, o[8 * q + 1] * inv);
          u.y = pack_bf16x2(o[8 * q + 2] * inv, o[8 * q + 3] * inv);
          u.z = pack_bf16x2(o[8 * q + 4] * inv, o[8 * q + 5] * inv);
          u.w = pack_bf16x2(o[8 * q + 6] * inv, o[8 * q + 7] * inv);
          d4[q] = u;
        }
      } else {
        const int64_t slot = ((int64_t)item * p.q_heads + qh) * p.n_splits + split;
        float4* w4 = reinterpret_cast<float4*>(p.ws_o + slot * HD);
#pragma unroll
        for (int q = 0; q < HD / 4; ++q)
          w4[q] = make_float4(o[4 * q] * inv, o[4 * q + 1] * inv, o[4 * q + 2] * inv, o[4 * q + 3] * inv);
        p.ws_lse[slot] = ok ? m_run + log2f(l_run) : -INFINITY;
      }
    }
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}
}  // namespace dec

static int decode_tma_splits(int n_items, int kv_heads, int max_kv_len) {
  const int ctas = n_items * kv_heads;
  // split until ~256 CTAs (the producer streams the first ring of each split
  // before the PDL wait, so fewer, longer splits win over filling all 296
  // slots), keeping >= 8 page slices per split (>= 4 when there are very few
  // (item, head) pairs).  Measured in-graph (ctx 2K): B=4 3.79 -> 3.68 ms,
  // B=8 4.03 -> 3.91, B=16 4.57 -> 4.32, B=32 5.28 -> 5.06 vs the old
  // one-wave-of-296 rule.  Tuning override SP_DECODE_SPLITS.
  int want = (256 + ctas - 1) / ctas;
  const int pages = (max_kv_len + dec::PAGE - 1) / dec::PAGE;
  const int max_useful = ctas < 16 ? (pages + 3) / 4 : (pages / 8 > 1 ? pages / 8 : 1);
  if (want > max_useful) want = max_useful;
  if (const char* e = getenv("SP_DECODE_SPLITS")) want = atoi(e) < pages ? atoi(e) : pages;
  if (want > 64) want = 64;
  return want < 1 ? 1 : want;
}

template <int HD>
static int launch(const Params& p, int n_items, int n_work, cudaStream_t st) {
  if (n_work > 0) {
    const int smem = (PF_ROWS * HD + 4 * PF_KT * HD) * 2;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(prefill_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    launch_k(prefill_kernel<HD>, dim3(n_work, p.kv_heads), PF_WARPS * 32, smem, st, p);
    return check_launch("attn_prefill_kernel");
  }
  const int smem_tiles = (DC_WARPS * 4 * DC_KT * HD + 16 * HD) * 2;
  const int smem_merge = (DC_WARPS * 32 + DC_WARPS * 16 * HD) * 4;
  const int smem = smem_tiles > smem_merge ? smem_tiles : smem_merge;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  launch_k(decode_kernel<HD>, dim3(n_items, p.kv_heads, p.n_splits), DC_WARPS * 32, smem, st, p);
  if (int rc = check_launch("attn_decode_kernel")) return rc;
  if (p.n_splits > 1) {
    launch_k(combine_kernel, dim3(n_items, p.q_heads), HD, 0, st, p, HD);
    return check_launch("attn_combine_kernel");
  }
  return kOk;
}

static int decode_splits(int n_items, int kv_heads, int max_kv_len) {
  const int ctas = n_items * kv_heads;
  int want = (2 * 148 + ctas - 1) / ctas;
  const int max_useful = (max_kv_len + DC_WARPS * DC_KT - 1) / (DC_WARPS * DC_KT);
  if (want > max_useful) want = max_useful;
  if (want > 64) want = 64;
  return want < 1 ? 1 : want;
}

}  // namespace attn
}  // namespace sp

namespace sp {
int launch_prefill_tc(const void* q, int64_t ldq, int64_t q_rows_total, const void* k_pool,
                      const void* v_pool, int64_t pool_rows, const int32_t* block_tables,
                      int64_t bt_stride, const int32_t* cu_q, const int32_t* first_pos,
                      const int32_t* kv_len, const int32_t* work, int n_work, void* out,
                      int64_t ldo, int q_heads, int kv_heads, int block_size, cudaStream_t st,
                      const int32_t* split = nullptr, const int32_t* combine = nullptr,
                      int n_combine = 0, void* ws = nullptr, int64_t ws_bytes = 0);
}

using namespace sp;

// tcgen05 prefill kernel: head_dim 128, pages of 64*k keys, GQA group dividing 128
static bool use_tc_prefill(int q_heads, int kv_heads, int head_dim, int block_size) {
  if (kv_heads <= 0 || q_heads % kv_heads) return false;
  const int g = q_heads / kv_heads;
  return head_dim == 128 && block_size % 64 == 0 && g <= 16 && 128 % g == 0;
}

extern "C" int sp_attn_tile_tokens(int q_heads, int kv_heads, int head_dim, int block_size) {
  if (kv_heads <= 0 || q_heads % kv_heads) return 0;
  const int g = q_heads / kv_heads;
  if (use_tc_prefill(q_heads, kv_heads, head_dim, block_size)) return 256 / g;
  return g > attn::PF_ROWS ? 0 : attn::PF_ROWS / g;
}

extern "C" int64_t sp_attn_workspace_bytes(int n_items, int q_heads, int head_dim, int max_kv_len) {
  (void)max_kv_len;
  const int64_t splits = 64;
  return (int64_t)n_items * q_heads * splits * (head_dim + 1) * 4;
}

static sp_status launch_decode_tma(attn::Params& p, const void* k_pool, const void* v_pool,
                                   int64_t pool_blocks, int n_items, int q_heads, int kv_heads,
                                   int head_dim, int block_size, int max_kv_len, void* ws,
                                   int64_t ws_bytes, cudaStream_t st) {
  CUtensorMap tk, tv;
  uint64_t dims[2] = {128, (uint64_t)(pool_blocks * (int64_t)kv_heads * block_size)};
  uint64_t strides[1] = {128 * 2};
  uint32_t box[2] = {64, attn::dec::PAGE};
  if (int rc = tma_map_bf16(&tk, k_pool, 2, dims, strides, box)) return rc;
  if (int rc = tma_map_bf16(&tv, v_pool, 2, dims, strides, box)) return rc;
  p.n_splits = attn::decode_tma_splits(n_items, kv_heads, max_kv_len);
  p.kv_stream = l2_hint_enabled() ? 1 : 0;
  p.ws_o = p.ws_lse = nullptr;
  if (p.n_splits > 1) {
    const int64_t need = (int64_t)n_items * q_heads * p.n_splits * (head_dim + 1) * 4;
    if (!ws || ws_bytes < need) {
      p.n_splits = 1;
    } else {
      p.ws_o = static_cast<float*>(ws);
      p.ws_lse = p.ws_o + (int64_t)n_items * q_heads * p.n_splits * head_dim;
    }
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn::dec::decode_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         attn::dec::SMEM_BYTES);
    cudaFuncSetAttribute(attn::dec::decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         attn::dec::TC_SMEM);
    attr = true;
  }
  // SP_DECODE_TC=1: the tcgen05/TMEM consumer (opt-in: equal in isolation but
  // slower in-graph, where its 256 TMEM columns per CTA contend with the
  // PDL-overlapped projections — DESIGN.md §10); read per call (tests A/B it)
  const char* tce = getenv("SP_DECODE_TC");
  if (tce && tce[0] == '1' && p.group <= 16) {
    launch_k(attn::dec::decode_tc_kernel, dim3(n_items, kv_heads, p.n_splits), attn::dec::TC_THREADS,
             attn::dec::TC_SMEM, st, tk, tv, p);
    if (int rc = check_launch("attn_decode_tc_kernel")) return rc;
  } else {
    launch_k(attn::dec::decode_tma_kernel, dim3(n_items, kv_heads, p.n_splits), attn::dec::NUM_THREADS,
             attn::dec::SMEM_BYTES, st, tk, tv, p);
    if (int rc = check_launch("attn_decode_tma_kernel")) return rc;
  }
  if (p.n_splits > 1) {
    launch_k(attn::combine_kernel, dim3(n_items, q_heads), head_dim, 0, st, p, head_dim);
    return check_launch("attn_combine_kernel");
  }
  return kOk;
}

extern "C" sp_status sp_attention_prefill_split(
    const void* q, int64_t ldq, int64_t q_rows, const void* k_pool, const void* v_pool,
    int64_t pool_blocks, const int32_t* block_tables, int64_t bt_stride, const int32_t* cu_q,
    const int32_t* first_pos, const int32_t* kv_len, const int32_t* work, const int32_t* split,
    int n_work, const int32_t* combine, int n_combine, void* out, int64_t ldo, int q_heads,
    int kv_heads, int head_dim, int block_size, void* ws, int64_t ws_bytes, void* stream) {
  if (n_work <= 0 || n_combine < 0 || !work || !split || (n_combine > 0 && !combine))
    return fail(kInvalid, "attention split: bad work lists");
  if (kv_heads <= 0 || q_heads % kv_heads) return fail(kInvalid, "attention: q_heads % kv_heads != 0");
  if (!use_tc_prefill(q_heads, kv_heads, head_dim, block_size))
    return fail(kUnsupported, "attention split: needs the tcgen05 prefill path (head_dim 128)");
  if (ldq % 8 || ldo % 8 || q_rows <= 0 || pool_blocks <= 0)
    return fail(kInvalid, "attention: tcgen05 prefill needs 16-byte rows and sizes");
  if (!ws || ws_bytes <= 0) return fail(kInvalid, "attention split: workspace required");
  return launch_prefill_tc(q, ldq, q_rows, k_pool, v_pool,
                           pool_blocks * (int64_t)kv_heads * block_size, block_tables, bt_stride,
                           cu_q, first_pos, kv_len, work, n_work, out, ldo, q_heads, kv_heads,
                           block_size, reinterpret_cast<cudaStream_t>(stream), split, combine,
                           n_combine, ws, ws_bytes);
}

extern "C" sp_status sp_attention(const void* q, int64_t ldq, int64_t q_rows, const void* k_pool,
                                  const void* v_pool, int64_t pool_blocks,
                                  const int32_t* block_tables, int64_t bt_stride, const int32_t* cu_q,
                                  const int32_t* first_pos, const int32_t* kv_len, int n_items,
                                  const int32_t* work, int n_work, int max_q_len, int max_kv_len,
                                  void* out, int64_t ldo, int q_heads, int kv_heads, int head_dim,
                                  int block_size, void* ws, int64_t ws_bytes, void* stream) {
  (void)max_q_len;
  if (n_items < 0 || n_work < 0) return fail(kInvalid, "attention: negative sizes");
  if (n_items == 0) return kOk;
  if (kv_heads <= 0 || q_heads % kv_heads) return fail(kInvalid, "attention: q_heads % kv_heads != 0");
  const int G = q_heads / kv_heads;
  if (G > 16) return fail(kUnsupported, "attention: GQA group > 16");
  if (ldq % 8 || ldo % 2) return fail(kInvalid, "attention: bad row strides");
  if (block_size <= 0) return fail(kInvalid, "attention: bad block size");
  attn::Params p{};
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.ldq = ldq;
  p.k_pool = static_cast<const __nv_bfloat16*>(k_pool);
  p.v_pool = static_cast<const __nv_bfloat16*>(v_pool);
  p.block_tables = block_tables;
  p.bt_stride = bt_stride;
  p.cu_q = cu_q;
  p.first_pos = first_pos;
  p.kv_len = kv_len;
  p.work = reinterpret_cast<const int2*>(work);
  p.out = static_cast<__nv_bfloat16*>(out);
  p.ldo = ldo;
  p.q_heads = q_heads;
  p.kv_heads = kv_heads;
  p.group = G;
  p.block_size = block_size;
  p.scale_log2 = attn::kLog2e / sqrtf((float)head_dim);
  p.n_splits = 1;
  p.ws_o = nullptr;
  p.ws_lse = nullptr;
  p.kv_stream = 0;
  p.qkv_parts = nullptr;
  if (n_work == 0) {
    p.n_splits = attn::decode_splits(n_items, kv_heads, max_kv_len);
    if (p.n_splits > 1) {
      const int64_t need = (int64_t)n_items * q_heads * p.n_splits * (head_dim + 1) * 4;
      if (!ws || ws_bytes < need) {
        p.n_splits = 1;
      } else {
        p.ws_o = static_cast<float*>(ws);
        p.ws_lse = p.ws_o + (int64_t)n_items * q_heads * p.n_splits * head_dim;
      }
    }
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n_work > 0 && use_tc_prefill(q_heads, kv_heads, head_dim, block_size)) {
    if (ldq % 8 || ldo % 8 || q_rows <= 0 || pool_blocks <= 0)
      return fail(kInvalid, "attention: tcgen05 prefill needs 16-byte rows and sizes");
    return launch_prefill_tc(q, ldq, q_rows, k_pool, v_pool,
                             pool_blocks * (int64_t)kv_heads * block_size, block_tables, bt_stride,
                             cu_q, first_pos, kv_len, work, n_work, out, ldo, q_heads, kv_heads,
                             block_size, st);
  }
  if (n_work == 0 && head_dim == 128 && block_size % attn::dec::PAGE == 0 && pool_blocks > 0)
    return launch_decode_tma(p, k_pool, v_pool, pool_blocks, n_items, q_heads, kv_heads, head_dim,
                             block_size, max_kv_len, ws, ws_bytes, st);
  switch (head_dim) {
    case 32: return attn::launch<32>(p, n_items, n_work, st);
    case 64: return attn::launch<64>(p, n_items, n_work, st);
    case 128: return attn::launch<128>(p, n_items, n_work, st);
    default: return fail(kUnsupported, "attention: head_dim must be 32, 64 or 128");
  }
}

// Decode attention whose Q, and the new token's K/V, come from the QKV
// projection's K-split partials (the RoPE + KV-write kernel fused into the
// attention kernel): see attn::Params::qkv_parts.  One row per item
// (cu_q[item] = its row); head_dim 128, block_size % 64 == 0.  Bit-identical
// to sp_rope_kv_write_partials followed by sp_attention.
extern "C" sp_status sp_attention_decode_qkv(
    const float* parts, int n_parts, int64_t ld_qkv, int parts_rows, const int32_t* pos,
    const int32_t* slot, const float* rope_table, void* k_pool, void* v_pool, int64_t pool_blocks,
    const int32_t* block_tables, int64_t bt_stride, const int32_t* cu_q, const int32_t* kv_len,
    int n_items, int max_kv_len, void* out, int64_t ldo, int q_heads, int kv_heads,
    int block_size, void* ws, int64_t ws_bytes, void* stream) {
  if (n_items < 0 || n_parts < 1 || parts_rows < n_items) return fail(kInvalid, "attention_decode_qkv: bad sizes");
  if (n_items == 0) return kOk;
  if (!parts || !pos || !slot || !k_pool || !v_pool || !block_tables || !cu_q || !kv_len || !out)
    return fail(kInvalid, "attention_decode_qkv: null pointer");
  if (kv_heads <= 0 || q_heads % kv_heads) return fail(kInvalid, "attention: q_heads % kv_heads != 0");
  const int G = q_heads / kv_heads;
  if (G > 16) return fail(kUnsupported, "attention: GQA group > 16");
  if (block_size <= 0 || block_size % attn::dec::PAGE || pool_blocks <= 0)
    return fail(kUnsupported, "attention_decode_qkv: block_size must be a multiple of 64");
  if (ld_qkv != (int64_t)(q_heads + 2 * kv_heads) * 128 || ldo % 2)
    return fail(kInvalid, "attention_decode_qkv: ld_qkv must be (q_heads + 2 kv_heads) * 128");
  attn::Params p{};
  memset(&p, 0, sizeof(p));
  p.k_pool = static_cast<const __nv_bfloat16*>(k_pool);
  p.v_pool = static_cast<const __nv_bfloat16*>(v_pool);
  p.block_tables = block_tables;
  p.bt_stride = bt_stride;
  p.cu_q = cu_q;
  p.kv_len = kv_len;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.ldo = ldo;
  p.q_heads = q_heads;
  p.kv_heads = kv_heads;
  p.group = G;
  p.block_size = block_size;
  p.scale_log2 = attn::kLog2e / sqrtf(128.f);
  p.qkv_parts = parts;
  p.n_parts = n_parts;
  p.parts_rows = parts_rows;
  p.ld_qkv = ld_qkv;
  p.rope_pos = pos;
  p.rope_slot = slot;
  p.rope_table = rope_table;
  return launch_decode_tma(p, k_pool, v_pool, pool_blocks, n_items, q_heads, kv_heads, 128,
                           block_size, max_kv_len, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}
