// tcgen05 / TMEM / TMA bf16 GEMM for sm_100a — every projection of the
// Shift-Parallel forward (QKV, O, gate/up, down, LM head).
//
//   D[m, n] = epi( sum_k A[m, k] * B[n, k] )     A, B bf16 K-major; f32 accumulate in TMEM
//
// Design (one CTA per SM, persistent, warp-specialised):
//   warp 0   : TMA producer — 128x64 A tile (3-D map: the per-peer chunked K of an
//              all-to-all receive is addressed directly) + 256x64 B tile per stage,
//              4-stage mbarrier ring, 128-byte swizzle.
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer, M=128 N=256 K=16,
//              accumulators double-buffered in TMEM (2 x 256 f32 columns).
//   warps 2-5: epilogue — tcgen05.ld 32 rows x 32 cols per warp, fused epilogue
//              (bf16/f32 store, residual add, SwiGLU, GeLU, per-peer send layout),
//              overlapped with the next tile's main loop.
// Fixed tiles, no split-K: each output is one ascending-K chain independent of M
// and of the N window, so row/column shards are bit-identical to the full GEMM.
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>
#include <cstdio>

#include "../../include/shiftpar.h"
#define SP_TU_ID 4  // step-trace tag (common.cuh)
#include "common.cuh"

namespace sp {
namespace gemm {

// per-call peer target of sp_gemm_bf16_to_peers (host thread-local)
static thread_local const unsigned long long* t_peer_ptrs = nullptr;
static thread_local int64_t t_peer_row_off = 0;

constexpr int BM = 128, BK = 64, ACC_STAGES = 2;
constexpr int A_BYTES = BM * BK * 2;
constexpr int NUM_THREADS = 192;

// N-tile variants: 256 for large GEMMs (1 CTA/SM), 128/64/32 so that small-M
// (decode) GEMMs still spread the weight stream over every SM (2 CTAs/SM).
// The K loop and MMA K-step are identical for every width, so a given output
// element is bit-identical whichever variant computes it.
template <int BN_>
struct Tile {
  static constexpr int BN = BN_;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN >= 256 ? 4 : (BN >= 128 ? 6 : 4);
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int MIN_BLOCKS = BN >= 128 ? 1 : 2;
};

struct Params {
  int M, N, K;
  int num_m, num_n, num_tiles, k_blocks;
  int epi;
  int a_kchunk;
  void* D;
  int64_t ldd;
  int64_t peer_width, peer_stride;
  // split-K (small-M regime): tile t covers k-blocks of split t % ksplit and
  // stores raw f32 partials to ws[split][M][N]; splitk_reduce applies the epilogue
  int ksplit, kb_per_split;
  float* ws;
  int group_m;  // m-tiles per raster group (A rows of a group stay L2-resident)
  int group_n;  // > 0: n-tiles per raster group instead (B rows stay L2-resident)
  int w_stream;  // swap-AB: weights are streamed once -> L2 evict-first hint
  // fused all-to-all: column block b = n / peer_width goes to peer b's buffer
  // peer_ptrs[b] at row (m + peer_row_off) — stores cross NVLink directly
  const unsigned long long* peer_ptrs;
  int64_t peer_row_off;
  // EPI_QKV_ROPE (sp_gemm_bf16_qkv_rope): columns are [q heads | k heads | v
  // heads] x 128; q rotated -> q_out, k rotated -> k_pool, v -> v_pool at the
  // row's cache slot (the work of rope_kv_kernel, fused into the epilogue)
  struct Rope {
    const float* table;  // [pos][64] (cos, sin) pairs
    const int32_t* pos;
    const int32_t* slot;
    __nv_bfloat16* q_out;
    int64_t ldq;
    __nv_bfloat16* k_pool;
    __nv_bfloat16* v_pool;
    int q_heads, kv_heads, block_size;
  } rope;
};

constexpr int EPI_QKV_ROPE = 100;  // internal: only via sp_gemm_bf16_qkv_rope
static thread_local Params::Rope t_rope = {};

// Per-peer TMA store maps of the fused seq->head exchange (pair kernel):
// m[b] = 2-D bf16 map over peer b's receive rows [row_off + M][peer_width]
// (rows past the pass are clipped by the map), box 64 cols x 32 rows, 128-B
// swizzle.  n == 0: the epilogue stores directly (row-strided 16-B stores).
constexpr int kMaxPeerMaps = 8;
struct PeerMaps {
  CUtensorMap m[kMaxPeerMaps];
  int n;
  // EPI_ADD_F32 through TMA (pair kernel): m[0] is an f32 map of D, box 32 x
  // 32 with 128-B swizzle; each epilogue warp TMA-loads its rows' old residual
  // box, adds the accumulator in shared memory and TMA-stores it back — whole
  // 128-B lines per instruction instead of 32 row-strided lines per warp access
  int add_tma;
  // bf16 outputs (STORE_BF16 / GELU / SWIGLU) through TMA: m[0] is a bf16 map
  // of D, box 64 x 32 with 128-B swizzle; each warp packs 32 rows x 64 columns
  // into a staging box (two per warp, alternating) and one TMA store writes it
  int store_tma;
};
static thread_local const unsigned long long* t_peer_ptrs_host = nullptr;

static bool add_tma_enabled() {  // SP_ADD_TMA=0: direct residual-add stores (A/B runs)
  const char* e = getenv("SP_ADD_TMA");
  return !(e && e[0] == '0');
}

static bool store_tma_enabled() {  // SP_STORE_TMA=0: direct bf16 epilogue stores (A/B runs)
  const char* e = getenv("SP_STORE_TMA");
  return !(e && e[0] == '0');
}

static bool peer_tma_enabled() {  // SP_PEER_TMA=0: direct epilogue stores (A/B runs)
  const char* e = getenv("SP_PEER_TMA");
  return !(e && e[0] == '0');
}

// destination element (m, n) of D honouring the per-peer layouts
template <typename T>
__device__ __forceinline__ T* out_ptr(const Params& p, int m, int64_t n) {
  T* base = reinterpret_cast<T*>(p.D);
  int64_t col = n, row = m, off = 0;
  if (p.peer_width > 0) {
    const int64_t peer = n / p.peer_width;
    col = n - peer * p.peer_width;
    if (p.peer_ptrs != nullptr) {
      base = reinterpret_cast<T*>(p.peer_ptrs[peer]);
      row = m + p.peer_row_off;
    } else {
      off = peer * p.peer_stride;
    }
  }
  return base + off + row * p.ldd + col;
}

// EPI_QKV_ROPE for one accumulator row (token m) over the 256 columns
// [n0, n0 + 256) = two 128-wide heads.  Values are rounded to bf16 first and
// rotated with rope_rotate, exactly what rope_kv_kernel does with the bf16
// qkv the plain epilogue would have stored.  tcgen05.ld is warp-collective:
// every lane loads, only valid rows store.
__device__ __forceinline__ void qkv_rope_row(const Params& p, int m, int n0, uint32_t tb) {
  const Params::Rope& R = p.rope;
  const bool valid = m < p.M;
  int pos = 0, slot = -1;
  if (valid) {
    pos = R.pos[m];
    slot = R.slot ? R.slot[m] : -1;
  }
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    const int h = (n0 >> 7) + hh;
    __nv_bfloat16* dst = nullptr;
    bool rotate = false;
    if (h < R.q_heads) {
      dst = R.q_out ? R.q_out + (int64_t)m * R.ldq + (int64_t)h * 128 : nullptr;
      rotate = R.table != nullptr;
    } else if (slot >= 0 && h < R.q_heads + 2 * R.kv_heads) {
      const int kv = h - R.q_heads;
      const int kvh = kv % R.kv_heads;
      __nv_bfloat16* pool = kv < R.kv_heads ? R.k_pool : R.v_pool;
      const int64_t blk = slot / R.block_size, off = slot % R.block_size;
      dst = pool + ((blk * R.kv_heads + kvh) * R.block_size + off) * 128;
      rotate = R.table != nullptr && kv < R.kv_heads;
    }
#pragma unroll 1
    for (int c = 0; c < 64; c += 32) {
      uint32_t ra[32], rb[32];
      tmem_ld32(tb + hh * 128 + c, ra);
      tmem_ld32(tb + hh * 128 + 64 + c, rb);
      tmem_ld_wait();
      if (!valid || dst == nullptr) continue;
      uint32_t oa[16], ob[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        // the bf16 rounding the plain epilogue applies before rope_kv_kernel reads it
        const float2 a = unpack_bf16x2(pack_bf16x2(__uint_as_float(ra[j]), __uint_as_float(ra[j + 1])));
        const float2 b = unpack_bf16x2(pack_bf16x2(__uint_as_float(rb[j]), __uint_as_float(rb[j + 1])));
        if (rotate) {
          const float4 cs = *reinterpret_cast<const float4*>(R.table + ((int64_t)pos * 64 + c + j) * 2);
          float na0, nb0, na1, nb1;
          rope_rotate(a.x, b.x, cs.x, cs.y, na0, nb0);
          rope_rotate(a.y, b.y, cs.z, cs.w, na1, nb1);
          oa[j / 2] = pack_bf16x2(na0, na1);
          ob[j / 2] = pack_bf16x2(nb0, nb1);
        } else {
          oa[j / 2] = pack_bf16x2(a.x, a.y);
          ob[j / 2] = pack_bf16x2(b.x, b.y);
        }
      }
      uint4* da = reinterpret_cast<uint4*>(dst + c);
      uint4* db = reinterpret_cast<uint4*>(dst + 64 + c);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        da[q] = make_uint4(oa[4 * q], oa[4 * q + 1], oa[4 * q + 2], oa[4 * q + 3]);
        db[q] = make_uint4(ob[4 * q], ob[4 * q + 1], ob[4 * q + 2], ob[4 * q + 3]);
      }
    }
  }
}

// EPI_QKV_ROPE for a tile of two query heads through TMA: the warp's 32 rows
// of each head are rotated exactly as qkv_rope_row does, packed into two
// 128-B-swizzled boxes (head columns [0, 64) and [64, 128)) and TMA-stored
// into q_out with the map `qmap` (rows past M are clipped by the map)
__device__ __forceinline__ void qkv_rope_q_tma(const Params& p, const CUtensorMap* qmap, int m,
                                               int n0, uint32_t tb, uint8_t* stage, int lane,
                                               int mrow0) {
  const Params::Rope& R = p.rope;
  const int pos = m < p.M ? R.pos[m] : 0;
  const bool rotate = R.table != nullptr;
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    const int h = (n0 >> 7) + hh;
    if (lane == 0) bulk_wait_read0();  // both boxes of the previous head have left smem
    __syncwarp();
#pragma unroll 1
    for (int c = 0; c < 64; c += 32) {
      uint32_t ra[32], rb[32];
      tmem_ld32(tb + hh * 128 + c, ra);
      tmem_ld32(tb + hh * 128 + 64 + c, rb);
      tmem_ld_wait();
      uint32_t oa[16], ob[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 a = unpack_bf16x2(pack_bf16x2(__uint_as_float(ra[j]), __uint_as_float(ra[j + 1])));
        const float2 b = unpack_bf16x2(pack_bf16x2(__uint_as_float(rb[j]), __uint_as_float(rb[j + 1])));
        if (rotate) {
          const float4 cs = *reinterpret_cast<const float4*>(R.table + ((int64_t)pos * 64 + c + j) * 2);
          float na0, nb0, na1, nb1;
          rope_rotate(a.x, b.x, cs.x, cs.y, na0, nb0);
          rope_rotate(a.y, b.y, cs.z, cs.w, na1, nb1);
          oa[j / 2] = pack_bf16x2(na0, na1);
          ob[j / 2] = pack_bf16x2(nb0, nb1);
        } else {
          oa[j / 2] = pack_bf16x2(a.x, a.y);
          ob[j / 2] = pack_bf16x2(b.x, b.y);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = (c >> 3) + q;  // 16-B chunk index inside the 128-B box row
        const uint32_t off = lane * 128 + ((j ^ (lane & 7)) << 4);
        *reinterpret_cast<uint4*>(stage + off) = make_uint4(oa[4 * q], oa[4 * q + 1], oa[4 * q + 2], oa[4 * q + 3]);
        *reinterpret_cast<uint4*>(stage + 4096 + off) =
            make_uint4(ob[4 * q], ob[4 * q + 1], ob[4 * q + 2], ob[4 * q + 3]);
      }
    }
    fence_async_shared();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(qmap, stage, h * 128, mrow0);
      tma_store_2d(qmap, stage + 4096, h * 128 + 64, mrow0);
      bulk_commit();
    }
  }
}

__device__ __forceinline__ void tile_coords(int t, const Params& p, int& mb, int& nb) {
  if (p.group_n > 0) {  // B-resident raster: a group of N tiles sweeps every M tile
    const int per_group = p.group_n * p.num_m;
    const int g = t / per_group;
    const int first_n = g * p.group_n;
    const int gn = min(p.num_n - first_n, p.group_n);
    const int r = t - g * per_group;
    nb = first_n + r % gn;
    mb = r / gn;
    return;
  }
  const int per_group = p.group_m * p.num_n;
  const int g = t / per_group;
  const int first_m = g * p.group_m;
  const int gm = min(p.num_m - first_m, p.group_m);
  const int r = t - g * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

__device__ __forceinline__ void split_coords(int t, const Params& p, int& mb, int& nb, int& kb0,
                                             int& kb1, int& ks) {
  ks = t % p.ksplit;
  tile_coords(t / p.ksplit, p, mb, nb);
  kb0 = ks * p.kb_per_split;
  kb1 = min(p.k_blocks, kb0 + p.kb_per_split);
}


__device__ __forceinline__ float gelu_tanh(float x) {
  const float c = 0.7978845608028654f, k = 0.044715f;
  return 0.5f * x * (1.f + tanhf(c * (x + k * x * x * x)));
}

// x * sigmoid(x) with SFU ex2 + rcp (no IEEE division sequence)
__device__ __forceinline__ float silu(float x) {
  float e = fast_exp2(-1.4426950408889634f * x), r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + e));
  return x * r;
}

// one thread: 32 consecutive columns [n0, n0+32) of row m
__device__ __forceinline__ void store_chunk(const Params& p, int m, int n0, const float (&v)[32],
                                            int epi, int N) {
  if (m >= p.M || n0 >= N) return;
  const int ncols = min(32, N - n0);
  if (epi == SP_EPI_STORE_BF16 || epi == SP_EPI_GELU) {
    __nv_bfloat16* dst = out_ptr<__nv_bfloat16>(p, m, n0);
    if (ncols == 32) {
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 u;
        u.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
        u.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
        u.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
        u.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
        d4[j] = u;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < ncols) dst[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* dst = out_ptr<float>(p, m, n0);
    if (ncols == 32) {
      float4* d4 = reinterpret_cast<float4*>(dst);
      if (epi == SP_EPI_ADD_F32) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o = d4[j];
          o.x += v[4 * j + 0];
          o.y += v[4 * j + 1];
          o.z += v[4 * j + 2];
          o.w += v[4 * j + 3];
          d4[j] = o;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          d4[j] = make_float4(v[4 * j + 0], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < ncols) {
          if (epi == SP_EPI_ADD_F32)
            dst[j] += v[j];
          else
            dst[j] = v[j];
        }
      }
    }
  }
}

template <int BN_>
__global__ void __launch_bounds__(NUM_THREADS, Tile<BN_>::MIN_BLOCKS)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const Params p) {
  using T = Tile<BN_>;
  constexpr int BN = T::BN, STAGES = T::STAGES, STAGE_BYTES = T::STAGE_BYTES;
  constexpr int TMEM_COLS = T::TMEM_COLS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC_STAGES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < ACC_STAGES; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------- TMA producer
      // PDL: the first ring of weight (B) tiles is fetched before pdl_wait();
      // the activation (A) loads of those stages are issued after it.
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t evict_first = l2_evict_first_policy();
      int n_def = 0;
      int def_stage[STAGES], def_kc[STAGES], def_m[STAGES], def_ko[STAGES];
      bool waited = false;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb, kb0, kb1, ks;
        split_coords(t, p, mb, nb, kb0, kb1, ks);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(full + stage, STAGE_BYTES);
          const int k = kb * BK;
          int ko = 0, kc = k;
          if (p.a_kchunk > 0) {
            ko = k / p.a_kchunk;
            kc = k - ko * p.a_kchunk;
          }
          tma_load_2d(sa + A_BYTES, &tmB, full + stage, k, nb * BN);
          if (waited) {
            tma_load_3d(sa, &tmA, full + stage, kc, mb * BM, ko);
          } else {
            def_stage[n_def] = stage;
            def_kc[n_def] = kc;
            def_m[n_def] = mb * BM;
            def_ko[n_def] = ko;
            if (++n_def == STAGES) {
              pdl_wait();
              waited = true;
              for (int i = 0; i < n_def; ++i)
                tma_load_3d(smem + def_stage[i] * STAGE_BYTES, &tmA, full + def_stage[i], def_kc[i],
                            def_m[i], def_ko[i]);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (!waited) {
        pdl_wait();
        for (int i = 0; i < n_def; ++i)
          tma_load_3d(smem + def_stage[i] * STAGE_BYTES, &tmA, full + def_stage[i], def_kc[i],
                      def_m[i], def_ko[i]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb, kb0, kb1, ks;
        split_coords(t, p, mb, nb, kb0, kb1, ks);
        mbar_wait(tempty + acc, aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            umma_bf16(d_tmem, sdesc_sw128(a_addr + k * 32), sdesc_sw128(b_addr + k * 32), idesc,
                      (kb != kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit(empty + stage);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull + acc);
        if (++acc == ACC_STAGES) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    // ----------------------------------------------------------- epilogue
    pdl_wait();  // D (e.g. the residual stream) belongs to the predecessor until it completes
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int mb, nb, kb0, kb1, ks;
      split_coords(t, p, mb, nb, kb0, kb1, ks);
      mbar_wait(tfull + acc, aphase);
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      const int m = mb * BM + row;
      if (p.ws != nullptr) {
        // split-K partial: raw f32 into ws[ks][M][N]
        Params q = p;
        q.D = p.ws + (int64_t)ks * p.M * p.N;
        q.ldd = p.N;
        q.peer_width = 0;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(tb + c, r);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          store_chunk(q, m, nb * BN + c, v, SP_EPI_STORE_F32, p.N);
        }
      } else if (BN == 256 && p.epi == EPI_QKV_ROPE) {
        qkv_rope_row(p, m, nb * 256, tb);
      } else if (p.epi == SP_EPI_SWIGLU) {
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(tb + c, g);
          tmem_ld32(tb + BN / 2 + c, u);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = silu(__uint_as_float(g[j])) * __uint_as_float(u[j]);
          store_chunk(p, m, nb * (BN / 2) + c, v, SP_EPI_STORE_BF16, p.N / 2);
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(tb + c, r);
          tmem_ld_wait();
          float v[32];
          if (p.epi == SP_EPI_GELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(__uint_as_float(r[j]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          }
          store_chunk(p, m, nb * BN + c, v, p.epi, p.N);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (++acc == ACC_STAGES) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------ swap-AB (decode-size M)
// D^T = W · X^T: the 128-row MMA operand is a weight tile, the token rows (M <=
// 128, padded to NT) are the N operand, so every staged byte is a weight byte.
//
// Work item = (super tile, K split).  A super tile is 2 x 128 weight rows —
// for SwiGLU exactly one gate|up pair, so the activation is applied in place
// when K is not split.  K is split only as far as needed to put enough CTAs
// on the weight stream (one round of items, no tail); split items store raw
// f32 partials to ws[split][M][N] and splitk_reduce_kernel sums them in
// ascending split order (deterministic) and applies the epilogue.
namespace swp {
constexpr int WT = 2;                 // weight tiles per super tile
constexpr int W_TILE = 128 * BK * 2;  // 16 KiB
}  // namespace swp

template <int NT>
struct SwapTile {
  static constexpr int W_BYTES = swp::WT * swp::W_TILE;
  static constexpr int X_BYTES = NT * BK * 2;
  static constexpr int STAGE_BYTES = W_BYTES + X_BYTES;
  // M <= 32 (latency-bound decode): two CTAs per SM, so a successor's CTAs can
  // start streaming weights (PDL) while this one drains; larger M: one CTA per
  // SM with a ~200 KB ring.
#ifndef SWAP_CPS_MAX_NT
#define SWAP_CPS_MAX_NT 32
#endif
  static constexpr int CTAS_PER_SM = NT <= SWAP_CPS_MAX_NT ? 2 : 1;
  static constexpr int RING = (CTAS_PER_SM == 2 ? 108 : 200) * 1024;
  static constexpr int STAGES = RING / STAGE_BYTES > 10 ? 10 : RING / STAGE_BYTES;
  static constexpr int ACC_COLS = swp::WT * NT;  // one accumulator stage
  // NT = 256 (M in (128, 256]): both 128-row halves x 256 tokens fill all 512
  // TMEM columns, so a single accumulator stage (one item per CTA anyway)
  static constexpr int ACC_STAGES = NT >= 256 ? 1 : 2;
  static constexpr int TMEM_COLS = ACC_STAGES * ACC_COLS < 32 ? 32 : ACC_STAGES * ACC_COLS;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
};

// Outputs of super tile t for weight row nl of each 128-row half, rows
// [m0, m0 + R) (those < m_end): v[0] = row t*256 + nl, v[1] = row t*256 + 128 + nl
// (gate and up for SwiGLU).  Residual reads are issued together before any
// store so their latencies overlap.
template <int R>
__device__ __forceinline__ void swap_store_rows(const Params& p, int m0, int m_end, int t, int nl,
                                                const float (&v)[swp::WT][R]) {
  if (p.epi == SP_EPI_SWIGLU && p.ws == nullptr) {
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (m0 + j < m_end)
        *out_ptr<__nv_bfloat16>(p, m0 + j, t * 128 + nl) = __float2bfloat16_rn(silu(v[0][j]) * v[1][j]);
    return;
  }
#pragma unroll
  for (int w = 0; w < swp::WT; ++w) {
    const int n = t * swp::WT * 128 + w * 128 + nl;
    if (n >= p.N) continue;
    if (p.ws != nullptr) {  // raw partial of split ks (set by the caller in p.D)
      float* dst = reinterpret_cast<float*>(p.D) + n;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (m0 + j < m_end) dst[(int64_t)(m0 + j) * p.N] = v[w][j];
    } else if (p.epi == SP_EPI_ADD_F32) {
      float old[R];
#pragma unroll
      for (int j = 0; j < R; ++j) old[j] = m0 + j < m_end ? *out_ptr<float>(p, m0 + j, n) : 0.f;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (m0 + j < m_end) *out_ptr<float>(p, m0 + j, n) = old[j] + v[w][j];
    } else if (p.epi == SP_EPI_STORE_F32) {
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (m0 + j < m_end) *out_ptr<float>(p, m0 + j, n) = v[w][j];
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (m0 + j >= m_end) continue;
        float x = v[w][j];
        if (p.epi == SP_EPI_GELU) x = gelu_tanh(x);
        *out_ptr<__nv_bfloat16>(p, m0 + j, n) = __float2bfloat16_rn(x);
      }
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NUM_THREADS, SwapTile<NT>::CTAS_PER_SM)
    gemm_swap_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                     const Params p) {
  using T = SwapTile<NT>;
  using namespace swp;
  constexpr int STAGES = T::STAGES, STAGE_BYTES = T::STAGE_BYTES, TMEM_COLS = T::TMEM_COLS;
  constexpr int ACC_STAGES = T::ACC_STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC_STAGES);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < ACC_STAGES; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t evict_first = l2_evict_first_policy();
      int n_def = 0;
      int def_stage[STAGES], def_kc[STAGES], def_ko[STAGES];
      bool waited = false;
      for (int it = blockIdx.x; it < p.num_tiles; it += gridDim.x) {
        const int ks = it % p.ksplit, t = it / p.ksplit;
        const int kb0 = ks * p.kb_per_split, kb1 = min(p.k_blocks, kb0 + p.kb_per_split);
        const int row0 = t * WT * 128;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sw = smem + stage * STAGE_BYTES;
          // one 256-row box = both 128-row weight tiles (rows past N zero-filled)
          mbar_arrive_expect_tx(full + stage, WT * W_TILE + T::X_BYTES);
          const int k = kb * BK;
          int ko = 0, kc = k;
          if (p.a_kchunk > 0) {
            ko = k / p.a_kchunk;
            kc = k - ko * p.a_kchunk;
          }
          // weights: no dependency on the predecessor; streamed exactly once per
          // decode step, so evicted first from L2 (keeps activations, partial
          // sums and code resident between the step's kernels)
          if (p.w_stream)
            tma_load_2d_hint(sw, &tmW, full + stage, k, row0, evict_first);
          else
            tma_load_2d(sw, &tmW, full + stage, k, row0);
          if (waited) {
            tma_load_3d(sw + T::W_BYTES, &tmX, full + stage, kc, 0, ko);
          } else {
            def_stage[n_def] = stage;
            def_kc[n_def] = kc;
            def_ko[n_def] = ko;
            if (++n_def == STAGES) {
              pdl_wait();
              waited = true;
              for (int i = 0; i < n_def; ++i)
                tma_load_3d(smem + def_stage[i] * STAGE_BYTES + T::W_BYTES, &tmX, full + def_stage[i],
                            def_kc[i], 0, def_ko[i]);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (!waited) {
        pdl_wait();
        for (int i = 0; i < n_def; ++i)
          tma_load_3d(smem + def_stage[i] * STAGE_BYTES + T::W_BYTES, &tmX, full + def_stage[i],
                      def_kc[i], 0, def_ko[i]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, NT);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int it = blockIdx.x; it < p.num_tiles; it += gridDim.x) {
        const int ks = it % p.ksplit, t = it / p.ksplit;
        const int kb0 = ks * p.kb_per_split, kb1 = min(p.k_blocks, kb0 + p.kb_per_split);
        const int wv = min(WT, (p.N - t * WT * 128 + 127) / 128);
        mbar_wait(tempty + acc, aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * T::ACC_COLS;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t w_addr = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t x_addr = w_addr + T::W_BYTES;
          for (int w = 0; w < wv; ++w) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16(d_tmem + w * NT, sdesc_sw128(w_addr + w * W_TILE + k * 32),
                        sdesc_sw128(x_addr + k * 32), idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit(empty + stage);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull + acc);
        if (++acc == ACC_STAGES) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    pdl_wait();
    const int quarter = warp & 3;
    const int nl = quarter * 32 + lane;  // this thread's weight row inside a 128-row tile
    int acc = 0;
    uint32_t aphase = 0;
    for (int it = blockIdx.x; it < p.num_tiles; it += gridDim.x) {
      const int ks = it % p.ksplit, t = it / p.ksplit;
      Params q = p;  // split items write raw partials to ws[ks][M][N]
      if (p.ws != nullptr) q.D = p.ws + (int64_t)ks * p.M * p.N;
      mbar_wait(tfull + acc, aphase);
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * T::ACC_COLS;
      // 8 token rows per step, rolled: the epilogue runs once per item, so
      // compact code matters more than unrolling (a fully unrolled version
      // stalled on instruction fetch)
#pragma unroll 1
      for (int c0 = 0; c0 < p.M; c0 += 8) {
        float v[WT][8];
#pragma unroll
        for (int w = 0; w < WT; ++w) {
          uint32_t r[8];
          tmem_ld8(tb + w * NT + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j) v[w][j] = __uint_as_float(r[j]);
        }
        swap_store_rows<8>(q, c0, p.M, t, nl, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (++acc == ACC_STAGES) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------ 2-CTA (cta_group::2) kernel
// A CTA pair on one TPC computes a 256x256 tile: CTA r holds A rows
// [m0 + 128 r, +128) and B rows [n0 + 128 r, +128) in its own shared memory;
// the leader (rank 0) issues tcgen05.mma.cta_group::2 M=256 N=256, which reads
// both CTAs' operands and writes each CTA's 128 accumulator rows into its own
// TMEM.  Per SM this halves the B bytes staged per FLOP vs the 1-CTA kernel.
namespace pair {
#ifndef PAIR_STAGES
#define PAIR_STAGES 6
#endif
constexpr int STAGES = PAIR_STAGES;
constexpr int A_BYTES = 128 * BK * 2;
constexpr int B_BYTES = 128 * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
// TMA-epilogue variants: per-epilogue-warp staging boxes — peer exchange: one
// 4 KiB box [32 rows][64 bf16] at quarter * 4096; residual add: two 4 KiB
// boxes [32 rows][32 f32] at quarter * 8192 (double-buffered loads)
constexpr int OUT_OFF = STAGES * STAGE_BYTES + 1024;  // past the barriers, 1024-aligned
constexpr int OUT_BYTES = 8 * 4096;
constexpr int OUT_BAR_OFF = OUT_OFF + OUT_BYTES;      // 8 box-load barriers (residual add)
#ifdef STEP_TRACE  // the trace slot's static shared word (1 KiB-aligned) leaves less dynamic room
constexpr int SMEM_BYTES_TMA = OUT_BAR_OFF + 64 + 896;
#else
constexpr int SMEM_BYTES_TMA = OUT_BAR_OFF + 64 + 1024;
#endif
static_assert(SMEM_BYTES_TMA <= 232448, "pair TMA-epilogue smem over the 227 KiB limit");

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA whose completion bytes land on the LEADER's barrier (peer bit cleared)
__device__ __forceinline__ void tma2_load_2d(void* dst, const void* desc, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(desc), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma2_load_3d(void* dst, const void* desc, uint64_t* bar, int c0, int c1,
                                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(desc), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void umma2_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
}  // namespace pair

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const Params p, const __grid_constant__ PeerMaps pm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + pair::STAGES * pair::STAGE_BYTES);
  uint64_t* empty = full + pair::STAGES;
  uint64_t* tfull = empty + pair::STAGES;
  uint64_t* tempty = tfull + ACC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC_STAGES);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = pair::cta_rank();
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  pdl_trigger();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < pair::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < ACC_STAGES; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);  // 4 epilogue warps x 2 CTAs (leader's barrier is used)
    }
    if (pm.add_tma) {
      tma_prefetch_desc(&pm.m[0]);
      for (int i = 0; i < 8; ++i) mbar_init(reinterpret_cast<uint64_t*>(smem + pair::OUT_BAR_OFF) + i, 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  pair::cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t evict_first = l2_evict_first_policy();
      int n_def = 0;
      int def_stage[pair::STAGES], def_kc[pair::STAGES], def_m[pair::STAGES], def_ko[pair::STAGES];
      bool waited = false;
      for (int t = cluster; t < p.num_tiles; t += n_clusters) {
        int mb, nb;
        tile_coords(t, p, mb, nb);
        const int m0 = mb * 256 + rank * 128;
        const int n0 = nb * 256 + rank * 128;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * pair::STAGE_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(full + stage, 2 * pair::STAGE_BYTES);
          const int k = kb * BK;
          int ko = 0, kc = k;
          if (p.a_kchunk > 0) {
            ko = k / p.a_kchunk;
            kc = k - ko * p.a_kchunk;
          }
          pair::tma2_load_2d(sa + pair::A_BYTES, &tmB, full + stage, k, n0);
          if (waited) {
            pair::tma2_load_3d(sa, &tmA, full + stage, kc, m0, ko);
          } else {
            def_stage[n_def] = stage;
            def_kc[n_def] = kc;
            def_m[n_def] = m0;
            def_ko[n_def] = ko;
            if (++n_def == pair::STAGES) {
              pdl_wait();
              waited = true;
              for (int i = 0; i < n_def; ++i)
                pair::tma2_load_3d(smem + def_stage[i] * pair::STAGE_BYTES, &tmA, full + def_stage[i], def_kc[i],
                             def_m[i], def_ko[i]);
            }
          }
          if (++stage == pair::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (!waited) {
        pdl_wait();
        for (int i = 0; i < n_def; ++i)
          pair::tma2_load_3d(smem + def_stage[i] * pair::STAGE_BYTES, &tmA, full + def_stage[i], def_kc[i],
                       def_m[i], def_ko[i]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, 256);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int t = cluster; t < p.num_tiles; t += n_clusters) {
        mbar_wait(tempty + acc, aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * pair::STAGE_BYTES);
          const uint32_t b_addr = a_addr + pair::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            pair::umma2_bf16(d_tmem, sdesc_sw128(a_addr + k * 32), sdesc_sw128(b_addr + k * 32), idesc,
                       (kb | k) != 0 ? 1u : 0u);
          pair::umma2_commit_both(empty + stage);
          if (++stage == pair::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        pair::umma2_commit_both(tfull + acc);
        if (++acc == ACC_STAGES) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    pdl_wait();
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t leader_tempty = pair::map_to_rank(smem_u32(tempty), 0);
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = cluster; t < p.num_tiles; t += n_clusters) {
      int mb, nb;
      tile_coords(t, p, mb, nb);
      mbar_wait(tfull + acc, aphase);
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * 256;
      const int m = mb * 256 + rank * 128 + row;
      if (p.epi == EPI_QKV_ROPE) {
        if (pm.store_tma && nb * 2 + 1 < p.rope.q_heads)
          qkv_rope_q_tma(p, &pm.m[0], m, nb * 256, tb, smem + pair::OUT_OFF + quarter * 8192, lane,
                         mb * 256 + rank * 128 + quarter * 32);
        else
          qkv_rope_row(p, m, nb * 256, tb);
      } else if (pm.store_tma) {
        uint8_t* stage = smem + pair::OUT_OFF + quarter * 8192;
        const int mrow0 = mb * 256 + rank * 128 + quarter * 32;
        const bool swiglu = p.epi == SP_EPI_SWIGLU;
        const int out_cols = swiglu ? 128 : 256;
#pragma unroll 1
        for (int c = 0; c < out_cols; c += 64) {
          uint32_t r0[32], r1[32];
          float v[64];
          if (swiglu) {
            uint32_t u0[32], u1[32];
            tmem_ld32(tb + c, r0);
            tmem_ld32(tb + c + 32, r1);
            tmem_ld32(tb + 128 + c, u0);
            tmem_ld32(tb + 128 + c + 32, u1);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              v[j] = silu(__uint_as_float(r0[j])) * __uint_as_float(u0[j]);
              v[32 + j] = silu(__uint_as_float(r1[j])) * __uint_as_float(u1[j]);
            }
          } else {
            tmem_ld32(tb + c, r0);
            tmem_ld32(tb + c + 32, r1);
            tmem_ld_wait();
            const bool gelu = p.epi == SP_EPI_GELU;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float x0 = __uint_as_float(r0[j]), x1 = __uint_as_float(r1[j]);
              v[j] = gelu ? gelu_tanh(x0) : x0;
              v[32 + j] = gelu ? gelu_tanh(x1) : x1;
            }
          }
          uint8_t* box = stage + ((c >> 6) & 1) * 4096;
          if (lane == 0) bulk_wait_read1();  // this buffer's store two boxes back has left smem
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint4 u;
            u.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
            u.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
            u.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
            u.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
            *reinterpret_cast<uint4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) = u;
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&pm.m[0], box, nb * out_cols + c, mrow0);
            bulk_commit();
          }
        }
      } else if (p.epi == SP_EPI_SWIGLU) {
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(tb + c, g);
          tmem_ld32(tb + 128 + c, u);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = silu(__uint_as_float(g[j])) * __uint_as_float(u[j]);
          store_chunk(p, m, nb * 128 + c, v, SP_EPI_STORE_BF16, p.N / 2);
        }
      } else if (pm.add_tma) {
        // residual add through TMA: per 32-column chunk the warp's old x box
        // [32 rows][32 f32] (128-B swizzled) is TMA-loaded one chunk ahead,
        // each lane adds its row's accumulator (old + acc, the order of
        // store_chunk) in shared memory, and one TMA store writes it back
        uint8_t* stage = smem + pair::OUT_OFF + quarter * 8192;
        uint64_t* lbar = reinterpret_cast<uint64_t*>(smem + pair::OUT_BAR_OFF) + quarter * 2;
        const int mrow0 = mb * 256 + rank * 128 + quarter * 32;
        const int ncol0 = nb * 256;
        if (lane == 0) {
          bulk_wait_read1();  // buffer 0's last store (two chunks back) has left smem
          mbar_arrive_expect_tx(lbar, 4096);
          tma_load_2d(stage, &pm.m[0], lbar, ncol0, mrow0);
        }
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
          uint8_t* box = stage + (k & 1) * 4096;
          if (k + 1 < 8 && lane == 0) {
            bulk_wait_read0();  // the store of chunk k-1 (the other buffer) has left smem
            mbar_arrive_expect_tx(lbar + ((k + 1) & 1), 4096);
            tma_load_2d(stage + ((k + 1) & 1) * 4096, &pm.m[0], lbar + ((k + 1) & 1),
                        ncol0 + (k + 1) * 32, mrow0);
          }
          uint32_t r[32];
          tmem_ld32(tb + k * 32, r);
          tmem_ld_wait();
          mbar_wait(lbar + (k & 1), (uint32_t)(k >> 1) & 1);  // 4 uses per buffer per tile
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4* q = reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4));
            float4 o = *q;
            o.x += __uint_as_float(r[4 * j + 0]);
            o.y += __uint_as_float(r[4 * j + 1]);
            o.z += __uint_as_float(r[4 * j + 2]);
            o.w += __uint_as_float(r[4 * j + 3]);
            *q = o;
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&pm.m[0], box, ncol0 + k * 32, mrow0);
            bulk_commit();
          }
        }
      } else if (pm.n > 0) {
        // fused seq->head exchange (bf16): each warp stages its 32 rows x 64
        // columns in a 128-B-swizzled box and one TMA store writes it into the
        // owning peer's receive rows — whole 128-B lines over NVLink instead of
        // 32 row-strided 16-B stores per warp instruction
        uint8_t* stage = smem + pair::OUT_OFF + quarter * 4096;
        const int mrow0 = mb * 256 + rank * 128 + quarter * 32;
#pragma unroll 1
        for (int c = 0; c < 256; c += 64) {
          uint32_t r0[32], r1[32];
          tmem_ld32(tb + c, r0);
          tmem_ld32(tb + c + 32, r1);
          tmem_ld_wait();
          if (lane == 0) bulk_wait_read0();  // the previous box has left `stage`
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t* r = j < 4 ? r0 : r1;
            const int e = (j & 3) * 8;
            uint4 u;
            u.x = pack_bf16x2(__uint_as_float(r[e + 0]), __uint_as_float(r[e + 1]));
            u.y = pack_bf16x2(__uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
            u.z = pack_bf16x2(__uint_as_float(r[e + 4]), __uint_as_float(r[e + 5]));
            u.w = pack_bf16x2(__uint_as_float(r[e + 6]), __uint_as_float(r[e + 7]));
            *reinterpret_cast<uint4*>(stage + lane * 128 + ((j ^ (lane & 7)) << 4)) = u;
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            const int n = nb * 256 + c;
            const int b = (int)(n / p.peer_width);
            tma_store_2d(&pm.m[b], stage, (int)(n - b * p.peer_width),
                         (int)(mrow0 + p.peer_row_off));
            bulk_commit();
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < 256; c += 32) {
          uint32_t r[32];
          tmem_ld32(tb + c, r);
          tmem_ld_wait();
          float v[32];
          if (p.epi == SP_EPI_GELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(__uint_as_float(r[j]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          }
          store_chunk(p, m, nb * 256 + c, v, p.epi, p.N);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) pair::arrive_remote(pair::map_to_rank(smem_u32(tempty + acc), 0));
      (void)leader_tempty;
      if (++acc == ACC_STAGES) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  if ((pm.n > 0 || pm.add_tma || pm.store_tma) && warp >= 2 && (threadIdx.x & 31) == 0)
    bulk_wait0();  // stores landed
  tc_fence_before();
  pair::cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// split-K reduction: v = sum_s ws[s] in ascending s (deterministic), then the
// epilogue; one thread = 8 consecutive output columns of one row.
__global__ void splitk_reduce_kernel(const Params p) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  const int n_out = p.epi == SP_EPI_SWIGLU ? p.N / 2 : p.N;
  const int64_t per_row = n_out / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.M * per_row) return;
  const int m = (int)(idx / per_row);
  const int c = (int)(idx % per_row) * 8;
  const int64_t split_stride = (int64_t)p.M * p.N;
  float v[8];
  if (p.epi == SP_EPI_SWIGLU) {
    const int g0 = (c / 128) * 256 + c % 128;
    float g[8], u[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = u[j] = 0.f;
    for (int s = 0; s < p.ksplit; ++s) {
      const float* row = p.ws + s * split_stride + (int64_t)m * p.N;
      const float4 a0 = *reinterpret_cast<const float4*>(row + g0);
      const float4 a1 = *reinterpret_cast<const float4*>(row + g0 + 4);
      const float4 b0 = *reinterpret_cast<const float4*>(row + g0 + 128);
      const float4 b1 = *reinterpret_cast<const float4*>(row + g0 + 132);
      g[0] += a0.x; g[1] += a0.y; g[2] += a0.z; g[3] += a0.w;
      g[4] += a1.x; g[5] += a1.y; g[6] += a1.z; g[7] += a1.w;
      u[0] += b0.x; u[1] += b0.y; u[2] += b0.z; u[3] += b0.w;
      u[4] += b1.x; u[5] += b1.y; u[6] += b1.z; u[7] += b1.w;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = silu(g[j]) * u[j];
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.f;
    for (int s = 0; s < p.ksplit; ++s) {
      const float* row = p.ws + s * split_stride + (int64_t)m * p.N + c;
      const float4 a0 = *reinterpret_cast<const float4*>(row);
      const float4 a1 = *reinterpret_cast<const float4*>(row + 4);
      v[0] += a0.x; v[1] += a0.y; v[2] += a0.z; v[3] += a0.w;
      v[4] += a1.x; v[5] += a1.y; v[6] += a1.z; v[7] += a1.w;
    }
    if (p.epi == SP_EPI_GELU) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = gelu_tanh(v[j]);
    }
  }
  if (p.epi == SP_EPI_STORE_F32 || p.epi == SP_EPI_ADD_F32) {
    float4* d4 = reinterpret_cast<float4*>(out_ptr<float>(p, m, c));
    if (p.epi == SP_EPI_ADD_F32) {
      float4 x0 = d4[0], x1 = d4[1];
      d4[0] = make_float4(x0.x + v[0], x0.y + v[1], x0.z + v[2], x0.w + v[3]);
      d4[1] = make_float4(x1.x + v[4], x1.y + v[5], x1.z + v[6], x1.w + v[7]);
    } else {
      d4[0] = make_float4(v[0], v[1], v[2], v[3]);
      d4[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  } else {
    __nv_bfloat16* dst = out_ptr<__nv_bfloat16>(p, m, c);
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]);
    u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]);
    u.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4*>(dst) = u;
  }
}

// ------------------------------------------------------------------ host side
// Raster choice: keep a group of A tiles (B streamed once per group) or of B
// tiles (A streamed once per group) L2-resident, whichever moves fewer DRAM
// bytes; SP_GEMM_L2_MB overrides the resident budget (default 40 MB of the
// 126 MB L2: measured best — larger resident groups thrash).
static void choose_raster(Params& p, int64_t tm, int64_t tn, int64_t K, int64_t M, int64_t N) {
  int64_t budget = 40ll << 20;
  if (const char* e = getenv("SP_GEMM_L2_MB")) budget = (int64_t)atoi(e) << 20;
  const int64_t a_tile = tm * K * 2, b_tile = tn * K * 2;
  const int64_t gm = std::max<int64_t>(1, std::min<int64_t>(budget / std::max<int64_t>(a_tile, 1), p.num_m));
  const int64_t gn = std::max<int64_t>(1, std::min<int64_t>(budget / std::max<int64_t>(b_tile, 1), p.num_n));
  const int64_t a_bytes = M * K * 2, b_bytes = N * K * 2;
  const int64_t traffic_m = a_bytes + b_bytes * ((p.num_m + gm - 1) / gm);
  const int64_t traffic_n = b_bytes + a_bytes * ((p.num_n + gn - 1) / gn);
  p.group_m = (int)gm;
  p.group_n = traffic_n < traffic_m ? (int)gn : 0;
  if (const char* e = getenv("SP_GEMM_RASTER")) p.group_n = e[0] == 'n' ? (int)gn : 0;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::mutex g_mu;
static std::map<std::array<uint64_t, 12>, CUtensorMap> g_maps;

static int encoder() {
  if (g_encode) return kOk;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return fail(kCuda, "cuTensorMapEncodeTiled entry point unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return kOk;
}

// tiled map with 128-byte swizzle (bf16 unless f32); dims/strides innermost first
int get_map(CUtensorMap* out, const void* ptr, int rank, const uint64_t* dims,
                   const uint64_t* strides, const uint32_t* box, bool f32 = false) {
  std::array<uint64_t, 12> key{};
  key[11] = f32 ? 1 : 0;
  key[0] = reinterpret_cast<uint64_t>(ptr);
  key[1] = rank;
  for (int i = 0; i < rank; ++i) key[2 + i] = dims[i];
  for (int i = 0; i < rank - 1; ++i) key[5 + i] = strides[i];
  for (int i = 0; i < rank; ++i) key[7 + i] = box[i];
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_maps.find(key);
  if (it != g_maps.end()) {
    *out = it->second;
    return kOk;
  }
  if (int rc = encoder()) return rc;
  uint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(out, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr),
                        dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(kInvalid, "cuTensorMapEncodeTiled failed (code " +
                                                   std::to_string((int)r) + ")");
  if (g_maps.size() > 8192) g_maps.clear();
  g_maps.emplace(key, *out);
  return kOk;
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace gemm

int tma_map_bf16(CUtensorMap* out, const void* ptr, int rank, const uint64_t* dims,
                 const uint64_t* strides, const uint32_t* box) {
  return gemm::get_map(out, ptr, rank, dims, strides, box);
}

}  // namespace sp

using namespace sp;

template <int BN>
static int launch(const void* A, int64_t lda, int64_t a_kchunk, int64_t a_chunk_stride,
                  const void* B, int64_t ldb, void* D, int64_t ldd, int M, int N, int K,
                  int epilogue, int64_t peer_width, int64_t peer_stride, void* stream,
                  float* ws = nullptr, int ksplit = 1) {
  using namespace sp::gemm;
  using T = Tile<BN>;
  CUtensorMap ta, tb;
  {
    const uint64_t kin = a_kchunk > 0 ? (uint64_t)a_kchunk : (uint64_t)K;
    const uint64_t kout = a_kchunk > 0 ? (uint64_t)(K / a_kchunk) : 1;
    const uint64_t cstride = a_kchunk > 0 ? (uint64_t)a_chunk_stride * 2
                                          : (uint64_t)lda * 2 * (uint64_t)M;
    uint64_t dims[3] = {kin, (uint64_t)M, kout};
    uint64_t strides[2] = {(uint64_t)lda * 2, cstride};
    uint32_t box[3] = {BK, BM, 1};
    if (int rc = get_map(&ta, A, 3, dims, strides, box)) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
    uint64_t strides[1] = {(uint64_t)ldb * 2};
    uint32_t box[2] = {BK, (uint32_t)BN};
    if (int rc = get_map(&tb, B, 2, dims, strides, box)) return rc;
  }
  Params p;
  p.peer_ptrs = t_peer_ptrs;
  p.peer_row_off = t_peer_row_off;
  p.rope = t_rope;
  p.M = M;
  p.N = N;
  p.K = K;
  p.num_m = (int)cdiv(M, BM);
  p.num_n = (int)cdiv(N, BN);
  p.num_tiles = p.num_m * p.num_n;
  p.k_blocks = (int)cdiv(K, BK);
  p.epi = epilogue;
  p.a_kchunk = (int)(a_kchunk > 0 ? a_kchunk : 0);
  p.D = D;
  p.ldd = ldd;
  p.peer_width = peer_width;
  p.peer_stride = peer_stride;
  // raster: walk all N tiles of a group of m-tiles whose A rows fit ~40 MB of L2,
  // so every B (weight) tile is streamed from HBM once per group
  choose_raster(p, BM, BN, K, M, N);
  p.ws = ws;
  p.ksplit = ws ? ksplit : 1;
  p.kb_per_split = (int)cdiv(p.k_blocks, p.ksplit);
  p.num_tiles *= p.ksplit;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         T::SMEM_BYTES);
    attr = true;
  }
  const int grid = std::min(p.num_tiles, sm_count() * T::MIN_BLOCKS);
  launch_k(gemm_kernel<BN>, grid, NUM_THREADS, T::SMEM_BYTES, reinterpret_cast<cudaStream_t>(stream), ta, tb, p);
  if (int rc = check_launch("gemm_kernel")) return rc;
  if (ws) {
    const int n_out = epilogue == SP_EPI_SWIGLU ? N / 2 : N;
    const int64_t threads = (int64_t)M * (n_out / 8);
    launch_k(splitk_reduce_kernel, (unsigned)cdiv(threads, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream), p);
    return check_launch("splitk_reduce_kernel");
  }
  return kOk;
}

// K splits of the swap-AB regime: split only until ~4/5 of the SMs stream
// weights (all SMs when two CTAs share one), in ONE round of items — a CTA
// with ~200 KB in flight streams well above its 1/148 share of HBM, so
// partial SM coverage still saturates HBM, while a second round would leave a
// tail.  Tuning override: SP_SWAP_MIN_CTAS.
template <int NT>
static int64_t swap_splits(int N, int K, int sms) {
  using namespace sp::gemm;
  using T = SwapTile<NT>;
  const int64_t k_blocks = cdiv(K, BK);
  const int64_t n_super = cdiv(N, swp::WT * 128);
  const int64_t slots = (int64_t)sms * T::CTAS_PER_SM;
  // measured best in-graph: ~1.3x the SMs at two CTAs per SM (M <= 32,
  // tools/gpu_swap_ab.sh: 192 CTAs on 148 SMs beat 148 by 1.0/1.3/0.8% TPOT at
  // B=1/8/32 — more streams in flight, while the N=4096 projections' K splits
  // stay <= 12, the partial count the consuming norm loads in one batch); at
  // one CTA per SM 3/4 of the SMs for NT=64 (tools/gpu_swap64_ab.sh: the
  // N=4096 projections split 7 ways instead of 8, B=48/64 -0.4/-1.0%) and 4/5
  // for NT >= 128 (B=128 best at 118-133)
  int64_t min_ctas = T::CTAS_PER_SM == 2 ? (13 * sms) / 10 : NT <= 64 ? (3 * sms) / 4 : (4 * sms) / 5;
  if (const char* e = getenv("SP_SWAP_MIN_CTAS")) min_ctas = atoi(e);
  int64_t ks = 1;
  while (n_super * ks < min_ctas && ks * 2 <= k_blocks) ++ks;
  while (ks > 1 && n_super * ks > slots) --ks;
  const int64_t per = cdiv(k_blocks, ks);
  return cdiv(k_blocks, per);
}

// the swap-AB (decode) regime applies: one 128-row M tile that cannot cover the SMs.
// Wide projections (more 256-row weight tiles than a quarter of the SMs) only up
// to 64 tokens: there the 1-CTA 128x256 tiles stream faster than the swap-AB
// variants for 65..256 tokens (tools/swap_probe.py, graph-replayed, gate/up
// N = 28672 K = 4096 at M = 96 / 128 / 256: 42.2 / 42.6 / 55.2 us tiled vs
// 46.6 / 48.6 / 62.8 swap-AB; at M <= 64 swap-AB wins, 40.3-41.1 vs 43.0-43.3).
// Projections with at least one 256-row weight tile per SM (the LM head, 70B
// gate/up) stay swap-AB only up to 32 tokens, where its two streaming CTAs per
// SM beat the tiled kernel (graph-replayed, tools/swap_probe.py: 8B LM head
// M = 1/8/32 182/181/173 -> 157/156/159 us; 70B gate/up M = 1/16 184/151 ->
// 141/142 us; at M = 64 neutral or worse).
static bool swap_regime(int M, int N, int sms) {
  using namespace sp::gemm;
  const int64_t n_super = cdiv(N, 256);
  if (getenv("SP_GEMM_NO_SPLITK") != nullptr || N % 32 != 0) return false;
  if (n_super >= sms) return M <= 32;
  return M <= 256 && (M <= 64 || n_super <= sms / 4);
}

template <int NT>
static int launch_swap(const void* A, int64_t lda, int64_t a_kchunk, int64_t a_chunk_stride,
                       const void* B, int64_t ldb, void* D, int64_t ldd, int M, int N, int K,
                       int epilogue, int64_t peer_width, int64_t peer_stride, void* stream,
                       float* ws, int64_t ws_bytes) {
  using namespace sp::gemm;
  using T = SwapTile<NT>;
  const int sms = sm_count();
  const int64_t k_blocks = cdiv(K, BK);
  const int64_t n_super = cdiv(N, swp::WT * 128);
  const int64_t slots = (int64_t)sms * T::CTAS_PER_SM;
  const int64_t ks = swap_splits<NT>(N, K, sms);
  const int64_t per = cdiv(k_blocks, ks);
  const bool partial = epilogue == SP_EPI_PARTIAL_F32;
  if (partial) {  // raw split partials go to the caller's D ([ks][M][N]); no reduce here
    if (ks > 1) {
      ws = static_cast<float*>(D);
      ws_bytes = ks * (int64_t)M * N * 4;
    } else {
      epilogue = SP_EPI_STORE_F32;
    }
  }
  if (ks > 1 && (!ws || ks * (int64_t)M * N * 4 > ws_bytes)) return -1;  // caller falls back
  CUtensorMap tx, tw;
  {
    const uint64_t kin = a_kchunk > 0 ? (uint64_t)a_kchunk : (uint64_t)K;
    const uint64_t kout = a_kchunk > 0 ? (uint64_t)(K / a_kchunk) : 1;
    const uint64_t cstride = a_kchunk > 0 ? (uint64_t)a_chunk_stride * 2
                                          : (uint64_t)lda * 2 * (uint64_t)M;
    uint64_t dims[3] = {kin, (uint64_t)M, kout};
    uint64_t strides[2] = {(uint64_t)lda * 2, cstride};
    uint32_t box[3] = {BK, (uint32_t)NT, 1};
    if (int rc = get_map(&tx, A, 3, dims, strides, box)) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
    uint64_t strides[1] = {(uint64_t)ldb * 2};
    uint32_t box[2] = {BK, (uint32_t)(swp::WT * 128)};
    if (int rc = get_map(&tw, B, 2, dims, strides, box)) return rc;
  }
  Params p;
  p.peer_ptrs = t_peer_ptrs;
  p.peer_row_off = t_peer_row_off;
  p.rope = t_rope;
  p.M = M;
  p.N = N;
  p.K = K;
  p.num_m = 1;
  p.num_n = (int)n_super;
  p.k_blocks = (int)k_blocks;
  p.epi = epilogue;
  p.a_kchunk = (int)(a_kchunk > 0 ? a_kchunk : 0);
  p.D = D;
  p.ldd = ldd;
  p.peer_width = peer_width;
  p.peer_stride = peer_stride;
  p.group_m = 1;
  p.group_n = 0;
  p.w_stream = l2_hint_enabled() ? 1 : 0;
  p.ws = ks > 1 ? ws : nullptr;
  p.ksplit = (int)ks;
  p.kb_per_split = (int)per;
  p.num_tiles = (int)(n_super * ks);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_swap_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         T::SMEM_BYTES);
    attr = true;
  }
  const int grid = (int)std::min<int64_t>(p.num_tiles, slots);
  launch_k(gemm_swap_kernel<NT>, grid, NUM_THREADS, T::SMEM_BYTES, reinterpret_cast<cudaStream_t>(stream), tx, tw, p);
  if (int rc = check_launch("gemm_swap_kernel")) return rc;
  if (ks > 1 && !partial) {
    const int n_out = epilogue == SP_EPI_SWIGLU ? N / 2 : N;
    const int64_t threads = (int64_t)M * (n_out / 8);
    launch_k(splitk_reduce_kernel, (unsigned)cdiv(threads, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream), p);
    return check_launch("splitk_reduce_kernel");
  }
  return kOk;
}


static int launch_pair(const void* A, int64_t lda, int64_t a_kchunk, int64_t a_chunk_stride,
                       const void* B, int64_t ldb, void* D, int64_t ldd, int M, int N, int K,
                       int epilogue, int64_t peer_width, int64_t peer_stride, void* stream) {
  using namespace sp::gemm;
  CUtensorMap ta, tb;
  {
    const uint64_t kin = a_kchunk > 0 ? (uint64_t)a_kchunk : (uint64_t)K;
    const uint64_t kout = a_kchunk > 0 ? (uint64_t)(K / a_kchunk) : 1;
    const uint64_t cstride = a_kchunk > 0 ? (uint64_t)a_chunk_stride * 2
                                          : (uint64_t)lda * 2 * (uint64_t)M;
    uint64_t dims[3] = {kin, (uint64_t)M, kout};
    uint64_t strides[2] = {(uint64_t)lda * 2, cstride};
    uint32_t box[3] = {BK, 128, 1};
    if (int rc = get_map(&ta, A, 3, dims, strides, box)) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
    uint64_t strides[1] = {(uint64_t)ldb * 2};
    uint32_t box[2] = {BK, 128};
    if (int rc = get_map(&tb, B, 2, dims, strides, box)) return rc;
  }
  Params p;
  p.peer_ptrs = t_peer_ptrs;
  p.peer_row_off = t_peer_row_off;
  p.rope = t_rope;
  p.M = M;
  p.N = N;
  p.K = K;
  p.num_m = (int)cdiv(M, 256);
  p.num_n = (int)cdiv(N, 256);
  p.num_tiles = p.num_m * p.num_n;
  p.k_blocks = (int)cdiv(K, BK);
  p.epi = epilogue;
  p.a_kchunk = (int)(a_kchunk > 0 ? a_kchunk : 0);
  p.D = D;
  p.ldd = ldd;
  p.peer_width = peer_width;
  p.peer_stride = peer_stride;
  p.ws = nullptr;
  p.ksplit = 1;
  p.kb_per_split = p.k_blocks;
  choose_raster(p, 256, 256, K, M, N);
  PeerMaps pm;
  pm.n = 0;
  pm.add_tma = 0;
  pm.store_tma = 0;
  if (epilogue == SP_EPI_ADD_F32 && peer_width == 0 && add_tma_enabled() && ldd % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(D) & 15) == 0) {
    uint64_t dims[2] = {(uint64_t)N, (uint64_t)M};
    uint64_t strides[1] = {(uint64_t)ldd * 4};
    uint32_t box[2] = {32, 32};
    if (int rc = get_map(&pm.m[0], D, 2, dims, strides, box, true)) return rc;
    pm.add_tma = 1;
  }
  if ((epilogue == SP_EPI_STORE_BF16 || epilogue == SP_EPI_GELU || epilogue == SP_EPI_SWIGLU) &&
      peer_width == 0 && store_tma_enabled() && ldd % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(D) & 15) == 0) {
    const int out_cols = epilogue == SP_EPI_SWIGLU ? N / 2 : N;
    uint64_t dims[2] = {(uint64_t)out_cols, (uint64_t)M};
    uint64_t strides[1] = {(uint64_t)ldd * 2};
    uint32_t box[2] = {64, 32};
    if (int rc = get_map(&pm.m[0], D, 2, dims, strides, box)) return rc;
    pm.store_tma = 1;
  }
  if (epilogue == EPI_QKV_ROPE && p.rope.q_out != nullptr && store_tma_enabled() &&
      p.rope.ldq % 8 == 0 && (reinterpret_cast<uintptr_t>(p.rope.q_out) & 15) == 0) {
    uint64_t dims[2] = {(uint64_t)p.rope.q_heads * 128, (uint64_t)M};
    uint64_t strides[1] = {(uint64_t)p.rope.ldq * 2};
    uint32_t box[2] = {64, 32};
    if (int rc = get_map(&pm.m[0], p.rope.q_out, 2, dims, strides, box)) return rc;
    pm.store_tma = 1;
  }
  if (t_peer_ptrs_host != nullptr && p.peer_ptrs != nullptr && epilogue == SP_EPI_STORE_BF16 &&
      peer_width % 64 == 0 && N / peer_width <= kMaxPeerMaps && peer_tma_enabled()) {
    // one store map per peer over the rows this pass owns in it
    const int np = (int)(N / peer_width);
    for (int b = 0; b < np; ++b) {
      uint64_t dims[2] = {(uint64_t)peer_width, (uint64_t)(p.peer_row_off + M)};
      uint64_t strides[1] = {(uint64_t)ldd * 2};
      uint32_t box[2] = {64, 32};
      if (int rc = get_map(&pm.m[b], reinterpret_cast<const void*>(t_peer_ptrs_host[b]), 2, dims,
                           strides, box))
        return rc;
    }
    pm.n = np;
  }
  const int smem = (pm.n > 0 || pm.add_tma || pm.store_tma) ? pair::SMEM_BYTES_TMA : pair::SMEM_BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         pair::SMEM_BYTES_TMA);
    attr = true;
  }
  const int clusters = std::min(p.num_tiles, sm_count() / 2);
  launch_k(gemm_pair_kernel, 2 * clusters, NUM_THREADS, smem,
           reinterpret_cast<cudaStream_t>(stream), ta, tb, p, pm);
  return check_launch("gemm_pair_kernel");
}

// split-K workspace per device (registered by the host, never allocated in
// the hot path; the host keeps every registered buffer alive because captured
// CUDA graphs hold its address)
static constexpr int kMaxDevices = 64;
static float* g_ws[kMaxDevices] = {};
static int64_t g_ws_bytes[kMaxDevices] = {};

static int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDevices ? 0 : d;
}

extern "C" sp_status sp_gemm_set_workspace(void* ws, int64_t bytes) {
  if (bytes < 0 || (ws == nullptr && bytes > 0)) return fail(kInvalid, "gemm workspace: bad args");
  if (reinterpret_cast<uintptr_t>(ws) & 15) return fail(kInvalid, "gemm workspace must be 16B aligned");
  const int d = cur_device();
  g_ws[d] = static_cast<float*>(ws);
  g_ws_bytes[d] = bytes;
  return kOk;
}

static int64_t swap_splits_for(int M, int N, int K, int sms) {
  if (M <= 32) return swap_splits<32>(N, K, sms);
  if (M <= 64) return swap_splits<64>(N, K, sms);
  if (M <= 128) return swap_splits<128>(N, K, sms);
  return swap_splits<256>(N, K, sms);
}

extern "C" int sp_gemm_partials(int M, int N, int K) {
  using namespace sp::gemm;
  if (M <= 0 || N <= 0 || K <= 0) return 1;
  const int sms = sm_count();
  if (!swap_regime(M, N, sms)) return 1;
  return (int)swap_splits_for(M, N, K, sms);
}

// Tile of the non-decode regime: 256 (2-CTA pairs unless *no_pair) or a
// narrower 1-CTA width.
static int plan_tile(int M, int N, int epilogue, int sms, bool* no_pair) {
  using namespace sp::gemm;
  const int64_t m_tiles = cdiv(M, BM);
  int bn = 256;
  *no_pair = false;
  if (m_tiles * cdiv(N, 256) < sms && epilogue != SP_EPI_SWIGLU) {
    // fewer 128x256 tiles than SMs: pick the tile by a wave model — cost =
    // waves x per-SM tile work (relative to half a 256x256 pair tile) x the
    // measured per-SM efficiency loss of 1-CTA tiles vs 2-CTA pairs
    // (tools/gemm_sweep.py: ~1.3 for 128x256, ~1.4 for 128x128, ~1.7 for 128x64,
    // ~2.5 for 128x32).  All candidates share the K loop: bit-identical.
    const bool pair_ok = M >= 256 && N % 256 == 0;
    double best = pair_ok ? (double)cdiv(cdiv(M, 256) * cdiv(N, 256), sms / 2) : 1e30;
    bn = 256;
    bool use_pair = pair_ok;
    const struct { int bn; double f; } cands[] = {{256, 1.3}, {128, 1.4}, {64, 1.7}, {32, 2.5}};
    for (const auto& c : cands) {
      const double cost = (double)cdiv(m_tiles * cdiv(N, c.bn), sms) * (c.bn / 256.0) * c.f;
      if (cost < best) {
        best = cost;
        bn = c.bn;
        use_pair = false;
      }
    }
    *no_pair = !use_pair;
  }
  return bn;
}

// THE dispatch decision of sp_gemm_bf16 (and what sp_gemm_plan reports):
// 0 = swap-AB decode kernel, 1 = 2-CTA 256x256 pairs, 256/128/64/32 = 1-CTA
// 128xBN tiles.  Env overrides apply in one order: SP_GEMM_NO_SPLITK (inside
// swap_regime), SP_GEMM_FORCE_BN, SP_GEMM_2CTA.  The swap-AB regime needs the
// device's split-K workspace when it splits K (except for raw partials).
static int gemm_plan(int M, int N, int K, int epilogue, int sms, const float* ws,
                     int64_t ws_bytes, bool ordered = false) {
  if (!ordered && swap_regime(M, N, sms)) {
    const int64_t ks = swap_splits_for(M, N, K, sms);
    if (ks == 1 || epilogue == SP_EPI_PARTIAL_F32 ||
        (ws && ks * (int64_t)M * N * 4 <= ws_bytes))
      return 0;
  }
  if (epilogue == SP_EPI_PARTIAL_F32) epilogue = SP_EPI_STORE_F32;
  bool no_pair = false;
  int bn = plan_tile(M, N, epilogue, sms, &no_pair);
  if (const char* f = getenv("SP_GEMM_FORCE_BN")) {
    const int fb = atoi(f);
    if ((fb == 32 || fb == 64 || fb == 128 || fb == 256) && epilogue != SP_EPI_SWIGLU) {
      bn = fb;
      no_pair = false;
    }
  }
  const char* e = getenv("SP_GEMM_2CTA");
  if (bn == 256 && M >= 256 && N % 256 == 0 && !no_pair && !(e && e[0] == '0')) return 1;
  return bn;
}

extern "C" int sp_gemm_plan(int M, int N, int K, int epilogue, int sms) {
  if (M <= 0 || N <= 0 || K <= 0 || sms <= 0) return -1;
  const int d = cur_device();
  return gemm_plan(M, N, K, epilogue & ~SP_GEMM_ORDERED, sms, g_ws[d], g_ws_bytes[d],
                   (epilogue & SP_GEMM_ORDERED) != 0);
}

extern "C" sp_status sp_gemm_bf16(const void* A, int64_t lda, int64_t a_kchunk,
                                  int64_t a_chunk_stride, const void* B, int64_t ldb, void* D,
                                  int64_t ldd, int M, int N, int K, int epilogue,
                                  int64_t peer_width, int64_t peer_stride, void* stream) {
  using namespace sp::gemm;
  const bool ordered = (epilogue & SP_GEMM_ORDERED) != 0;
  epilogue &= ~SP_GEMM_ORDERED;
  if (M < 0 || N <= 0 || K <= 0) return fail(kInvalid, "gemm: bad M/N/K");
  if (M == 0) return kOk;
  if (!A || !B || !D) return fail(kInvalid, "gemm: null pointer");
  if (epilogue < SP_EPI_STORE_BF16 || epilogue > SP_EPI_PARTIAL_F32)
    return fail(kInvalid, "gemm: unknown epilogue");
  if (epilogue == SP_EPI_PARTIAL_F32 && (peer_width > 0 || ldd != N))
    return fail(kInvalid, "gemm: partial epilogue needs a dense [n][M][N] D (ldd == N)");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15)
    return fail(kInvalid, "gemm: A/B must be 16-byte aligned");
  if (lda % 8 || ldb % 8 || ldd % 8) return fail(kInvalid, "gemm: leading dims must be multiples of 8");
  if (a_kchunk > 0 && (a_kchunk % BK || K % a_kchunk || a_chunk_stride % 8))
    return fail(kUnsupported, "gemm: chunked-K A needs chunk % 64 == 0 and K % chunk == 0");
  if (epilogue == SP_EPI_SWIGLU && N % 256)
    return fail(kUnsupported, "gemm: SwiGLU epilogue needs N % 256 == 0");
  if (peer_width > 0 && (peer_width % 32 || peer_stride % 8))
    return fail(kUnsupported, "gemm: peer layout needs width % 32 == 0");
  if (reinterpret_cast<uintptr_t>(D) & 15) return fail(kInvalid, "gemm: D must be 16-byte aligned");

  // Regime selection (numerics are identical within a regime):
  //  * decode-size M (<= 256) with fewer 256-row weight super tiles than SMs
  //                                                  -> swap-AB weight streaming over
  //    256-row super tiles (tokens padded to NT = 32/64/128/256), K split just
  //    enough to cover the SMs in one round; split partials summed in ascending
  //    split order (splitk_reduce_kernel, or the consumer for EPI_PARTIAL_F32)
  //  * enough 128x256 tiles to cover the SMs        -> BN=256 (2-CTA pairs)
  //  * otherwise                                     -> narrower N tiles (128/64/32),
  //    bit-identical to BN=256 (same K loop)
  const int sms = sm_count();
  const int dev = cur_device();
  const int plan = gemm_plan(M, N, K, epilogue, sms, g_ws[dev], g_ws_bytes[dev], ordered);
  if (plan == 0) {
    float* ws = g_ws[dev];
    const int64_t wsb = g_ws_bytes[dev];
    if (M <= 32)
      return launch_swap<32>(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue,
                             peer_width, peer_stride, stream, ws, wsb);
    if (M <= 64)
      return launch_swap<64>(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue,
                             peer_width, peer_stride, stream, ws, wsb);
    if (M <= 128)
      return launch_swap<128>(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue,
                              peer_width, peer_stride, stream, ws, wsb);
    return launch_swap<256>(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue,
                            peer_width, peer_stride, stream, ws, wsb);
  }
  if (epilogue == SP_EPI_PARTIAL_F32) epilogue = SP_EPI_STORE_F32;  // one "partial" = the result
  if (plan == 1)
    return launch_pair(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue,
                       peer_width, peer_stride, stream);
  switch (plan) {
    case 256: return launch<256>(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue, peer_width, peer_stride, stream);
    case 128: return launch<128>(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue, peer_width, peer_stride, stream);
    case 64: return launch<64>(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue, peer_width, peer_stride, stream);
    default: return launch<32>(A, lda, a_kchunk, a_chunk_stride, B, ldb, D, ldd, M, N, K, epilogue, peer_width, peer_stride, stream);
  }
}

// QKV projection with RoPE + paged KV write fused into the epilogue
// (prefill-size M): 256-column tiles = two whole heads, so every rotation
// pair (i, i + 64) sits in one thread's accumulator row.  Bit-identical to
// sp_gemm_bf16(EPI_STORE_BF16) followed by sp_rope_kv_write.
extern "C" sp_status sp_gemm_bf16_qkv_rope(const void* A, int64_t lda, const void* B, int64_t ldb,
                                           int M, int K, const int32_t* pos, const int32_t* slot,
                                           const float* rope_table, void* q_out, int64_t ldq,
                                           void* k_pool, void* v_pool, int q_heads, int kv_heads,
                                           int block_size, void* stream) {
  using namespace sp::gemm;
  const int N = (q_heads + 2 * kv_heads) * 128;
  if (M < 0 || K <= 0 || q_heads <= 0 || kv_heads < 0 || block_size <= 0)
    return fail(kInvalid, "gemm_qkv_rope: bad shape");
  if (M == 0) return kOk;
  if (!A || !B || !pos || (kv_heads > 0 && (!k_pool || !v_pool || !slot)))
    return fail(kInvalid, "gemm_qkv_rope: null pointer");
  if (N % 256) return fail(kUnsupported, "gemm_qkv_rope: q_heads + 2 kv_heads must be even");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15 || lda % 8 || ldb % 8 ||
      ldq % 8)
    return fail(kInvalid, "gemm_qkv_rope: 16-byte aligned operands and rows required");
  t_rope = Params::Rope{rope_table, pos, slot, static_cast<__nv_bfloat16*>(q_out), ldq,
                        static_cast<__nv_bfloat16*>(k_pool), static_cast<__nv_bfloat16*>(v_pool),
                        q_heads, kv_heads, block_size};
  int rc;
  const char* e = getenv("SP_GEMM_2CTA");
  if (M >= 256 && !(e && e[0] == '0'))
    rc = launch_pair(A, lda, 0, 0, B, ldb, q_out, ldq, M, N, K, EPI_QKV_ROPE, 0, 0, stream);
  else
    rc = launch<256>(A, lda, 0, 0, B, ldb, q_out, ldq, M, N, K, EPI_QKV_ROPE, 0, 0, stream);
  t_rope = Params::Rope{};
  return rc;
}

extern "C" sp_status sp_gemm_bf16_to_peers(const void* A, int64_t lda, int64_t a_kchunk,
                                           int64_t a_chunk_stride, const void* B, int64_t ldb,
                                           const unsigned long long* peer_ptrs,
                                           const unsigned long long* peer_ptrs_host,
                                           int64_t row_off, int64_t ldd, int M, int N, int K,
                                           int epilogue, int64_t peer_width, void* stream) {
  using namespace sp::gemm;
  if (!peer_ptrs || peer_width <= 0 || N % peer_width)
    return fail(kInvalid, "gemm_to_peers: need peer pointers and N % peer_width == 0");
  if (epilogue != SP_EPI_STORE_BF16 && epilogue != SP_EPI_STORE_F32)
    return fail(kUnsupported, "gemm_to_peers: store epilogues only");
  t_peer_ptrs = peer_ptrs;
  t_peer_ptrs_host = peer_ptrs_host;
  t_peer_row_off = row_off;
  // D is never dereferenced in peer mode; pass an aligned placeholder for validation
  const int rc = sp_gemm_bf16(A, lda, a_kchunk, a_chunk_stride, B, ldb,
                              reinterpret_cast<void*>(const_cast<unsigned long long*>(peer_ptrs)),
                              ldd, M, N, K, epilogue, peer_width, 0, stream);
  t_peer_ptrs = nullptr;
  t_peer_ptrs_host = nullptr;
  t_peer_row_off = 0;
  return rc;
}
