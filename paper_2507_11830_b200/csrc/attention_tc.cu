// tcgen05 / TMEM / TMA paged causal prefill attention for sm_100a (head_dim 128).
//
// Same contract as the mma.sync prefill kernel in attention.cu (reference
// tensor_core.attend_cached, tensor_core.py:135-176), selected by sp_attention
// when head_dim == 128 and the pool's block_size is a multiple of 64.
//
// One CTA = one kv head x two 128-row query tiles of GQA-packed rows
// (row = token * G + head-in-group, so one K/V tile feeds all G heads):
//   warps 0-3  softmax warpgroup for Q tile 0 (one TMEM lane = one row per thread)
//   warps 4-7  softmax warpgroup for Q tile 1
//   warp 8     TMA producer: Q tiles once (3-D map over [tokens][G][d]), then
//              128-key K/V tiles page by page from the paged pool (2-stage ring)
//   warp 9     TMEM allocator + single-thread MMA issuer (warps 10-11 idle);
//              setmaxnreg moves registers from this warpgroup to the softmax ones
// TMEM (512 cols): S0 | S1 (128 f32 cols each; P_i is written back as bf16 over
// the first 64 columns of S_i and consumed as the TMEM A-operand of P·V) |
// O0 | O1 (128 f32 cols each).  MMA issue order per key tile j:
//   PV0_j, QK0_{j+1}, PV1_j, QK1_{j+1}  — softmax i works on S_i(j+1) while the
// tensor core runs the other tile's PV/QK.  O is rescaled lazily by the softmax
// warps (only when a row max grows by > 2^8), safe because the commit that
// signals S_i(j+1) also covers PV_i(j).
#include <cudaTypedefs.h>

#include "../../include/shiftpar.h"
#define SP_TU_ID 2  // step-trace tag (common.cuh)
#include "common.cuh"

namespace sp {
namespace attn_tc {

constexpr int HD = 128;
constexpr int QROWS = 128;       // rows per Q tile
constexpr int KT = 128;          // keys per tile
// Softmax exponential variants (tools/kbench.py attn, 8K causal): with the K/V
// release split alone, 4 of every 32 pairs through the FMA-pipe polynomial
// (ATTN_POLY_PAIRS=4) was best (1190 vs 1140 TFLOP/s all-MUFU); once P·V
// starts per half of P the SFU is off the critical path and all-MUFU is as
// fast or faster (1210 vs 1195), so the default is 0.  One MUFU.EX2.bf16x2
// per pair (ATTN_EXP_BF16X2=1) was slower (1077).
#ifndef ATTN_EXP_BF16X2
#define ATTN_EXP_BF16X2 0
#endif
#ifndef ATTN_POLY_PAIRS
#define ATTN_POLY_PAIRS 0
#endif
constexpr int kPolyPairs = ATTN_POLY_PAIRS;  // of 32 pairs per 64 columns (tools/kbench.py attn)

// 2^x, x <= 0, for a PAIR of lanes on the FMA/ALU pipes: round-to-nearest
// split x = n + r (magic-number add, |r| <= 1/2), cubic 2^r (rel err 1.8e-4,
// far below the bf16 rounding of P), exponent n added into the bits.  x is
// clamped at -126 (2^-126 ~ 0 next to the row max's 1).
__device__ __forceinline__ void exp2_poly2(uint64_t x2, float& a, float& b) {
  float xa, xb;
  f2_unpack(x2, xa, xb);
  x2 = f2_pack(fmaxf(xa, -126.f), fmaxf(xb, -126.f));
  const uint64_t magic = f2_pack(12582912.f, 12582912.f);  // 1.5 * 2^23
  const uint64_t y = f2_add(x2, magic);                   // n in the low mantissa bits
  const uint64_t n = f2_add(y, f2_pack(-12582912.f, -12582912.f));
  const uint64_t r = f2_fma(n, f2_pack(-1.f, -1.f), x2);  // x - n
  uint64_t p = f2_fma(f2_pack(0.0546027f, 0.0546027f), r, f2_pack(0.24192398f, 0.24192398f));
  p = f2_fma(p, r, f2_pack(0.69331645f, 0.69331645f));
  p = f2_fma(p, r, f2_pack(1.f, 1.f));
  float pa, pb, ya, yb;
  f2_unpack(p, pa, pb);
  f2_unpack(y, ya, yb);
  // bits(y) << 23 == n << 23 (mod 2^32): the magic's own bits shift out
  a = __int_as_float(__float_as_int(pa) + (__float_as_int(ya) << 23));
  b = __int_as_float(__float_as_int(pb) + (__float_as_int(yb) << 23));
}

constexpr int NUM_THREADS = 384;  // 3 warpgroups: softmax 0, softmax 1, producer/MMA
constexpr int Q_TILE_BYTES = QROWS * HD * 2;      // 32 KiB (two 64-wide d chunks)
constexpr int KV_TILE_BYTES = KT * HD * 2;        // 32 KiB
constexpr int SMEM_Q = 2 * Q_TILE_BYTES;
// K ring 2 slots, V ring V_STAGES slots (3 measured no faster than 2: the MMA
// issuer's V wait shrank from ~400 to ~65 cycles but the period did not move —
// the tensor core itself, at ~68% of its peak rate, sets it; tools/attn_trace.py)
#ifndef ATTN_V_STAGES
#define ATTN_V_STAGES 2
#endif
constexpr int K_STAGES = 2, V_STAGES = ATTN_V_STAGES;
constexpr int SMEM_KV = (K_STAGES + V_STAGES) * KV_TILE_BYTES;
constexpr int SMEM_BYTES = SMEM_Q + SMEM_KV + 1024 + 256;
constexpr float kRescaleThreshold = 8.0f;         // log2 units

struct Params {
  const int32_t* block_tables;
  int64_t bt_stride;
  const int32_t* cu_q;
  const int32_t* first_pos;
  const int32_t* kv_len;
  const int2* work;
  __nv_bfloat16* out;
  int64_t ldo;
  int kv_heads, group, block_size;
  float scale_log2;
  // split-KV prefill (few CTAs, long causal rows): work entry w covers key
  // tiles [split[w].x, split[w].y); split[w].z >= 0 -> unnormalised partial
  // (O, m, l) into slot split[w].z * kv_heads + kvh, merged by
  // prefill_combine_kernel.  NULL -> every entry covers all its key tiles.
  const int4* split;
  float* ws_o;   // [slots][256 rows][HD]
  float* ws_ml;  // [slots][256 rows][2]
};

#ifdef ATTN_TRACE
// instrumented build (-DATTN_TRACE): clock64 stamps of CTA (0,0), iterations
// 0..31: [role][it][event], role 0 = MMA issuer, 1/2 = softmax warpgroup 0/1
__device__ unsigned long long g_attn_trace[3 * 32 * 8];
#define TR(role, it, ev)                                                              \
  do {                                                                                \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (it) < 32)                              \
      g_attn_trace[((role) * 32 + (it)) * 8 + (ev)] = clock64();                      \
  } while (0)
#else
#define TR(role, it, ev) \
  do {                   \
  } while (0)
#endif

__global__ void __launch_bounds__(NUM_THREADS, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const Params p) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                 // [tile][dchunk][128 rows][128 B]
  uint8_t* sKs = smem + SMEM_Q;                            // [K slot][dchunk][128 keys][128 B]
  uint8_t* sVs = sKs + K_STAGES * KV_TILE_BYTES;           // [V slot][dchunk][128 keys][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_Q + SMEM_KV);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [K_STAGES]
  uint64_t* k_empty = bars + 3;  // [K_STAGES] K slot free (both tiles' QK done)
  uint64_t* s_full = bars + 5;   // [2] per Q tile
  uint64_t* p_full = bars + 7;   // [2] per Q tile
  uint64_t* o_full = bars + 9;   // [2] per Q tile
  uint64_t* p_half = bars + 11;  // [2] per Q tile: P of keys 0-63 stored (PV may start)
  uint64_t* v_full = bars + 13;  // [V_STAGES]
  uint64_t* v_empty = bars + 16; // [V_STAGES] V slot free (both tiles' PV done)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 19);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 wk = p.work[blockIdx.x];
  const int item = wk.x, tok0 = wk.y;
  const int kvh = blockIdx.y;
  const int G = p.group;
  const int q_row0 = p.cu_q[item];
  const int q_len = p.cu_q[item + 1] - q_row0;
  const int fpos = p.first_pos[item];
  const int kv_len = p.kv_len[item];
  const int toks_per_tile = QROWS / G;
  const int tok_last = min(tok0 + 2 * toks_per_tile, q_len) - 1;
  const int kv_end = min(kv_len, fpos + tok_last + 1);
  int j_begin = 0, n_kt = (kv_end + KT - 1) / KT, slot = -1;
  if (p.split != nullptr) {
    const int4 sp = p.split[blockIdx.x];
    j_begin = sp.x;
    n_kt = min(n_kt, sp.y);
    slot = sp.z < 0 ? -1 : sp.z * p.kv_heads + kvh;
  }
  const int n_it = max(n_kt - j_begin, 0);  // iterations of this CTA (key tiles j_begin..n_kt-1)
  const int n_pages = (kv_len + p.block_size - 1) / p.block_size;

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < V_STAGES; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
      mbar_init(s_full + s, 1);
      mbar_init(p_full + s, 4);  // one arrival per softmax warp
      mbar_init(p_half + s, 4);
      mbar_init(o_full + s, 1);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, SMEM_Q);
      for (int t = 0; t < 2; ++t)
        for (int c = 0; c < 2; ++c)
          tma_load_3d(sQ + t * Q_TILE_BYTES + c * (Q_TILE_BYTES / 2), &tmQ, q_full, c * 64,
                      kvh * G, q_row0 + tok0 + t * toks_per_tile);
      const int32_t* bt = p.block_tables + (int64_t)item * p.bt_stride;
      for (int it = 0; it < n_it; ++it) {
        const int j = j_begin + it, s = it & 1, vs = it % V_STAGES;
        uint8_t* sK = sKs + s * KV_TILE_BYTES;
        uint8_t* sV = sVs + vs * KV_TILE_BYTES;
        int rows[2];
        for (int h = 0; h < 2; ++h) {
          const int key0 = j * KT + h * 64;
          const int pg_i = key0 / p.block_size;
          const int page = pg_i < n_pages ? bt[pg_i] : 0;
          rows[h] = (page * p.kv_heads + kvh) * p.block_size + key0 % p.block_size;
        }
        // K and V slots are released separately: K(j) frees once both tiles'
        // QK(j) are done (an iteration before V(j) frees), so K(j+2) is in
        // flight a full iteration before QK(j+2) needs it
        mbar_wait(k_empty + s, ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(k_full + s, KV_TILE_BYTES);
        for (int c = 0; c < 2; ++c)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sK + c * (KV_TILE_BYTES / 2) + h * 8192, &tmK, k_full + s, c * 64, rows[h]);
        mbar_wait(v_empty + vs, ((it / V_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(v_full + vs, KV_TILE_BYTES);
        for (int c = 0; c < 2; ++c)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sV + c * (KV_TILE_BYTES / 2) + h * 8192, &tmV, v_full + vs, c * 64, rows[h]);
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, KT);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, HD) | (1u << 16);  // B (V) MN-major
      const uint32_t sq = smem_u32(sQ);
      mbar_wait(q_full, 0);
      auto issue_qk = [&](int t, int it) {  // S_t of this CTA's it-th key tile
        const int s = it & 1;
        const uint32_t sk = smem_u32(sKs + s * KV_TILE_BYTES);
        const uint32_t qa = sq + t * Q_TILE_BYTES;
        const uint32_t d_tmem = tmem + t * 128;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * (Q_TILE_BYTES / 2) + (k & 3) * 32;
          const uint32_t koff = (k >> 2) * (KV_TILE_BYTES / 2) + (k & 3) * 32;
          umma_bf16(d_tmem, sdesc_sw128(qa + off), sdesc_sw128(sk + koff), idesc_qk, k > 0 ? 1u : 0u);
        }
        umma_commit(s_full + t);
      };
      mbar_wait(k_full + 0, 0);
      tc_fence_after();
      issue_qk(0, 0);
      issue_qk(1, 0);
      umma_commit(k_empty + 0);
      for (int it = 0; it < n_it; ++it) {
        const int s = it & 1, vs = it % V_STAGES;
        TR(0, it, 0);
        mbar_wait(v_full + vs, (it / V_STAGES) & 1);
        TR(0, it, 1);
        const uint32_t sv = smem_u32(sVs + vs * KV_TILE_BYTES);
        const bool more = it + 1 < n_it;
        if (more) mbar_wait(k_full + (s ^ 1), ((it + 1) >> 1) & 1);
        for (int t = 0; t < 2; ++t) {
          const uint32_t p_tmem = tmem + t * 128;
          const uint32_t o_tmem = tmem + 256 + t * 128;
          // P·V in two halves: keys 0-63 start while the softmax finishes 64-127
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            mbar_wait((h == 0 ? p_half : p_full) + t, it & 1);
            TR(0, it, 2 + 2 * t + h);
            tc_fence_after();
#pragma unroll
            for (int k = h * (KT / 32); k < (h + 1) * (KT / 32); ++k) {
              umma_ts_bf16(o_tmem, p_tmem + k * 8, sdesc_sw128_mn(sv + k * 2048, KV_TILE_BYTES / 2),
                           idesc_pv, (it | k) != 0 ? 1u : 0u);
            }
          }
          if (more)
            issue_qk(t, it + 1);
          else
            umma_commit(o_full + t);
          TR(0, it, 6 + t);
        }
        umma_commit(v_empty + vs);
        if (more) umma_commit(k_empty + (s ^ 1));
      }
    }
    __syncwarp();
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    // ----------------------------------------------------- softmax warpgroups
    const int t = warp >> 2;            // Q tile
    const int quarter = warp & 3;       // TMEM lane quarter
    const int row = quarter * 32 + lane;
    const int prow = t * QROWS + row;   // packed row in the CTA
    const int tok = tok0 + prow / G;
    const int head = kvh * G + prow % G;
    const int limit = fpos + min(tok, q_len - 1);
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_tmem = tmem + lane_base + t * 128;
    const uint32_t o_tmem = tmem + lane_base + 256 + t * 128;
    float m_run = -INFINITY, l_run = 0.f;
    for (int it = 0; it < n_it; ++it) {
      const int j = j_begin + it;
      if (quarter == 0 && lane == 0) TR(1 + t, it, 0);
      mbar_wait(s_full + t, it & 1);
      if (quarter == 0 && lane == 0) TR(1 + t, it, 1);
      tc_fence_after();
      float s[KT];  // raw scores; the softmax scale is folded into one FFMA below
      {
        // all four 32-column loads in flight, one wait (not a TMEM round trip each)
        uint32_t r[KT / 32][32];
#pragma unroll
        for (int c = 0; c < KT / 32; ++c) tmem_ld32(s_tmem + c * 32, r[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < KT / 32; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(r[c][e]);
      }
      const int kbase = j * KT;
      if (kbase + KT - 1 > limit) {
#pragma unroll
        for (int e = 0; e < KT; ++e)
          if (kbase + e > limit) s[e] = -INFINITY;
      }
      // row max as 8 independent FMNMX3 chains (depth 8 + 3) instead of one
      // 64-deep dependent chain
      float mxs[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mxs[i] = fmaxf(s[2 * i], s[2 * i + 1]);
#pragma unroll
      for (int e = 16; e < KT; e += 16)
#pragma unroll
        for (int i = 0; i < 8; ++i) mxs[i] = fmaxf(mxs[i], fmaxf(s[e + 2 * i], s[e + 2 * i + 1]));
#pragma unroll
      for (int w = 4; w; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) mxs[i] = fmaxf(mxs[i], mxs[i + w]);
      const float mx = mxs[0];
      if (quarter == 0 && lane == 0) TR(1 + t, it, 2);
      const float m_new = fmaxf(m_run, mx * p.scale_log2);
      const bool need = m_new > m_run + kRescaleThreshold;
      float corr = 1.f;
      if (need) {
        corr = fast_exp2(m_run - m_new);
        m_run = m_new;
      }
      l_run *= corr;
      if (it > 0 && __any_sync(0xffffffffu, need)) {
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
      // p = 2^(raw * scale - m_run): FFMA2 + 2 x MUFU.EX2 (or the FMA-pipe
      // polynomial for the last kPolyPairs pairs of each 64 columns, so the
      // SFU is not the co-bottleneck with the tensor core) + FADD2 per pair
      const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2);
      const uint64_t nm2 = f2_pack(-m_run, -m_run);
      // row sum in 4 independent FADD2 chains (summed at the end)
      uint64_t sums[4] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
#pragma unroll
      for (int c = 0; c < KT / 64; ++c) {
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float a, b;
          const uint64_t x2 = f2_fma(f2_pack(s[c * 64 + 2 * e], s[c * 64 + 2 * e + 1]), sc2, nm2);
#if ATTN_EXP_BF16X2
          if (true) {  // one MUFU.EX2 per PAIR: exponent rounded to bf16, P produced as bf16x2
            f2_unpack(x2, a, b);
            uint32_t pb;
            asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(pb) : "r"(pack_bf16x2(a, b)));
            const float2 pf = unpack_bf16x2(pb);
            sums[e & 3] = f2_add(sums[e & 3], f2_pack(pf.x, pf.y));
            pk[e] = pb;
            continue;
          }
#endif
          if (e >= 32 - kPolyPairs) {
            exp2_poly2(x2, a, b);
          } else {
            f2_unpack(x2, a, b);
            a = fast_exp2(a);
            b = fast_exp2(b);
          }
          sums[e & 3] = f2_add(sums[e & 3], f2_pack(a, b));
          pk[e] = pack_bf16x2(a, b);
        }
        tmem_st32(s_tmem + c * 32, pk);
        if (c == 0) {  // first half of P ready: let P·V start on keys 0-63
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_half + t);
          if (quarter == 0 && lane == 0) TR(1 + t, it, 3);
        }
      }
      const uint64_t sum2 = f2_add(f2_add(sums[0], sums[1]), f2_add(sums[2], sums[3]));
      float sa, sb;
      f2_unpack(sum2, sa, sb);
      l_run += sa + sb;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();  // every lane's P stores complete before the warp's single arrival
      if (lane == 0) mbar_arrive(p_full + t);
      if (quarter == 0 && lane == 0) TR(1 + t, it, 4);
    }
    // ------------------------------------------------------------- epilogue
    mbar_wait(o_full + t, 0);
    tc_fence_after();
    if (slot >= 0) {  // split-KV: unnormalised partial O and (m, l), merged later
      float* po = p.ws_o + ((int64_t)slot * 2 * QROWS + prow) * HD;
#pragma unroll 1
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(o_tmem + c * 32, r);
        tmem_ld_wait();
        float4* d4 = reinterpret_cast<float4*>(po + c * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          d4[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                              __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
      }
      float* pml = p.ws_ml + ((int64_t)slot * 2 * QROWS + prow) * 2;
      pml[0] = m_run;
      pml[1] = l_run;
    } else {
    const float inv = 1.f / l_run;
    const bool store = tok < q_len;
    __nv_bfloat16* dst = p.out + (int64_t)(q_row0 + tok) * p.ldo + (int64_t)head * HD;
#pragma unroll 1
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(o_tmem + c * 32, r);
      tmem_ld_wait();
      if (store) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_bf16x2(__uint_as_float(r[8 * q + 0]) * inv, __uint_as_float(r[8 * q + 1]) * inv);
          u.y = pack_bf16x2(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv);
          u.z = pack_bf16x2(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv);
          u.w = pack_bf16x2(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv);
          d4[q] = u;
        }
      }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Merge the split-KV partials of one (work tile, kv head): block = 32 packed
// rows x 128 d (thread: one row, 16 d); entries of `combine` are (item, t0,
// first split, n splits).  Splits are merged in ascending key order.
__global__ void prefill_combine_kernel(const int4* __restrict__ combine, const Params p) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  const int4 cb = combine[blockIdx.x];
  const int kvh = blockIdx.y;
  const int prow = blockIdx.z * 32 + (threadIdx.x >> 3);
  const int c0 = (threadIdx.x & 7) * 16;
  const int G = p.group;
  const int q_row0 = p.cu_q[cb.x];
  const int q_len = p.cu_q[cb.x + 1] - q_row0;
  const int t = prow / QROWS;
  const int tok = cb.y + t * (QROWS / G) + (prow % QROWS) / G;
  if (tok >= q_len) return;
  const int head = kvh * G + (prow % QROWS) % G;
  float mx = -INFINITY;
  for (int k = 0; k < cb.w; ++k) {
    const int64_t slot = (int64_t)(cb.z + k) * p.kv_heads + kvh;
    mx = fmaxf(mx, p.ws_ml[(slot * 2 * QROWS + prow) * 2]);
  }
  float l = 0.f, acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.f;
  for (int k = 0; k < cb.w; ++k) {
    const int64_t slot = (int64_t)(cb.z + k) * p.kv_heads + kvh;
    const float* ml = p.ws_ml + (slot * 2 * QROWS + prow) * 2;
    if (ml[0] == -INFINITY) continue;
    const float f = exp2f(ml[0] - mx);
    l += ml[1] * f;
    const float4* o4 = reinterpret_cast<const float4*>(p.ws_o + (slot * 2 * QROWS + prow) * HD + c0);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 v = o4[e];
      acc[4 * e] += v.x * f;
      acc[4 * e + 1] += v.y * f;
      acc[4 * e + 2] += v.z * f;
      acc[4 * e + 3] += v.w * f;
    }
  }
  const float inv = 1.f / l;
  uint4* dst = reinterpret_cast<uint4*>(p.out + (int64_t)(q_row0 + tok) * p.ldo + (int64_t)head * HD + c0);
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    uint4 u;
    u.x = pack_bf16x2(acc[8 * e] * inv, acc[8 * e + 1] * inv);
    u.y = pack_bf16x2(acc[8 * e + 2] * inv, acc[8 * e + 3] * inv);
    u.z = pack_bf16x2(acc[8 * e + 4] * inv, acc[8 * e + 5] * inv);
    u.w = pack_bf16x2(acc[8 * e + 6] * inv, acc[8 * e + 7] * inv);
    dst[e] = u;
  }
}

}  // namespace attn_tc

// host launcher, called from sp_attention (attention.cu)
int launch_prefill_tc(const void* q, int64_t ldq, int64_t q_rows_total, const void* k_pool,
                      const void* v_pool, int64_t pool_rows, const int32_t* block_tables,
                      int64_t bt_stride, const int32_t* cu_q, const int32_t* first_pos,
                      const int32_t* kv_len, const int32_t* work, int n_work, void* out,
                      int64_t ldo, int q_heads, int kv_heads, int block_size, cudaStream_t st,
                      const int32_t* split, const int32_t* combine, int n_combine, void* ws,
                      int64_t ws_bytes);

// tensor maps (shared cache with the GEMM)
int tma_map_bf16(CUtensorMap* out, const void* ptr, int rank, const uint64_t* dims,
                 const uint64_t* strides, const uint32_t* box);

int launch_prefill_tc(const void* q, int64_t ldq, int64_t q_rows_total, const void* k_pool,
                      const void* v_pool, int64_t pool_rows, const int32_t* block_tables,
                      int64_t bt_stride, const int32_t* cu_q, const int32_t* first_pos,
                      const int32_t* kv_len, const int32_t* work, int n_work, void* out,
                      int64_t ldo, int q_heads, int kv_heads, int block_size, cudaStream_t st,
                      const int32_t* split, const int32_t* combine, int n_combine, void* ws,
                      int64_t ws_bytes) {
  using namespace attn_tc;
  const int G = q_heads / kv_heads;
  CUtensorMap tq, tk, tv;
  {
    // Q viewed as [tokens][q_heads][d]; the box {64, G, 128/G} at head
    // coordinate kvh*G picks the G heads of one kv group = 128 packed rows.
    uint64_t dims[3] = {(uint64_t)HD, (uint64_t)q_heads, (uint64_t)q_rows_total};
    uint64_t strides[2] = {(uint64_t)HD * 2, (uint64_t)ldq * 2};
    uint32_t box[3] = {64, (uint32_t)G, (uint32_t)(QROWS / G)};
    if (int rc = tma_map_bf16(&tq, q, 3, dims, strides, box)) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)HD, (uint64_t)pool_rows};
    uint64_t strides[1] = {(uint64_t)HD * 2};
    uint32_t box[2] = {64, 64};
    if (int rc = tma_map_bf16(&tk, k_pool, 2, dims, strides, box)) return rc;
    if (int rc = tma_map_bf16(&tv, v_pool, 2, dims, strides, box)) return rc;
  }
  Params p;
  p.block_tables = block_tables;
  p.bt_stride = bt_stride;
  p.cu_q = cu_q;
  p.first_pos = first_pos;
  p.kv_len = kv_len;
  p.work = reinterpret_cast<const int2*>(work);
  p.out = static_cast<__nv_bfloat16*>(out);
  p.ldo = ldo;
  p.kv_heads = kv_heads;
  p.group = G;
  p.block_size = block_size;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  p.split = reinterpret_cast<const int4*>(split);
  p.ws_o = p.ws_ml = nullptr;
  if (split != nullptr) {
    if (!ws) return fail(kInvalid, "attention split: workspace required");
    p.ws_o = static_cast<float*>(ws);
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  if (split != nullptr) {  // ws = [slots][256][HD] O partials, then [slots][256][2] (m, l)
    const int64_t slots = ws_bytes / ((int64_t)2 * QROWS * (HD + 2) * 4);
    p.ws_ml = p.ws_o + slots * 2 * QROWS * HD;
  }
  launch_k(prefill_tc_kernel, dim3(n_work, kv_heads), NUM_THREADS, SMEM_BYTES, st, tq, tk, tv, p);
  if (int rc = check_launch("attn_prefill_tc_kernel")) return rc;
  if (split != nullptr && n_combine > 0) {
    launch_k(prefill_combine_kernel, dim3(n_combine, kv_heads, 2 * QROWS / 32), 256, 0, st,
             reinterpret_cast<const int4*>(combine), p);
    return check_launch("attn_prefill_combine_kernel");
  }
  return kOk;
}

}  // namespace sp

#ifdef ATTN_TRACE
extern "C" int sp_attn_trace_copy(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, sp::attn_tc::g_attn_trace,
                                   sizeof(unsigned long long) * (n < 768 ? n : 768));
}
#endif
