// Fused decode layer: ONE persistent kernel per transformer layer of a TP
// (P = 1) decode pass — O projection + residual + RMSNorm, gate/up + SwiGLU,
// down + residual + RMSNorm, and the next layer's QKV + RoPE + paged KV
// write — replacing the 9-11 kernels per layer of the unfused path
// (reference: the layer loop of _forward_tp, parallel_engine.py:359-379, at a
// decode step).
//
// Why: at decode every projection streams its weights from HBM once
// (8B: 436 MB per layer) while its activation operand is a few KB.  Weight
// tiles never depend on the previous op, so one CTA per SM runs a TMA
// producer that streams the weight tiles of ALL the layer's projections back
// to back through one shared-memory ring; only the tiny activation box of each
// stage waits for its producer op.  The dependencies between ops become
// grid-wide counter barriers inside the kernel instead of kernel boundaries,
// so the weight stream does not drain and refill at every op.
//
// Per CTA (192 threads):
//   warp 0   : TMA producer — per stage one 256-row x 64-k weight box (both
//              128-row MMA tiles) + one NT-row x 64-k activation box; the
//              activation load of a stage is deferred until its op's input is
//              published (grid barrier counter, acquire + async-proxy fence),
//              while weight loads keep filling the ring.
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer (swap-AB:
//              weights are the M=128 operand, the <= 64 tokens the N operand),
//              accumulators double-buffered in TMEM.
//   warps 2-5: epilogue — f32 partial sums of each stream-K segment to an L2
//              slab; then, between grid barriers, the op's reduction fused with
//              its consumer: residual add + RMSNorm, SwiGLU, or RoPE + KV write.
//
// Work split (stream-K): projection p has U = tiles x k-blocks units of one
// 256x64 weight box; CTA c owns units [U c / G, U (c+1) / G), i.e. every SM
// streams the same number of weight bytes per op.  A run of units inside one
// 256-row tile is a segment; its f32 partial goes to slab (tile, c - first
// owner of the tile) and the reduction sums a tile's segments in ascending
// k order — deterministic for a given (shape, grid).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>

#include "../../include/shiftpar.h"
#define SP_TU_ID 3  // step-trace tag (common.cuh)
#include "common.cuh"

namespace sp {
int tma_map_bf16(CUtensorMap* out, const void* ptr, int rank, const uint64_t* dims,
                 const uint64_t* strides, const uint32_t* box);

namespace dl {

constexpr int BK = 64;
constexpr int W_TILE = 128 * BK * 2;  // one 128-row MMA tile of a stage: 16 KiB
constexpr int W_BYTES = 2 * W_TILE;   // the 256-row weight box
constexpr int NUM_THREADS = 192;
constexpr int EPI_THREADS = 128;
constexpr int MAX_PROJ = 4;
constexpr int MAX_VEC = 16;  // hidden <= 8192 (4 floats x 128 threads x 16)

struct Proj {
  CUtensorMap tw;  // weights [n][k], box {64, 256}
  CUtensorMap tx;  // input rows [rows][k], box {64, NT}
  int n, k, kb, tiles, units, maxseg, kind;
  int need;        // grid barriers before this projection's input rows are published
  float* slab;     // [tiles][maxseg][rows][256] f32
  const float* gain;
  __nv_bfloat16* out;
  int64_t ldo;
};

struct Args {
  Proj proj[MAX_PROJ];
  int n_proj, rows, hidden, grid;
  float* x;
  int64_t ldx;
  float eps;
  const float* lead_gain;
  __nv_bfloat16* lead_out;
  int64_t ld_lead;
  const int32_t* pos;
  const int32_t* slot;
  const float* rope;
  __nv_bfloat16* q_out;
  int64_t ldq;
  __nv_bfloat16* k_pool;
  __nv_bfloat16* v_pool;
  int q_heads, kv_heads, block_size;
  unsigned* sync;  // [0] barrier arrivals (monotonic within a launch), [1] exits
};

// Timeline instrumentation (debug builds, SP_NVCC_EXTRA=-DDL_TRACE): per CTA,
// globaltimer stamps of the producer / MMA / epilogue milestones of the LAST
// launch, read back with sp_decode_layer_trace (tools/dl_trace.py).
constexpr int TR_SLOTS = 64;
#ifdef DL_TRACE
__device__ unsigned long long g_trace[160 * TR_SLOTS];
__device__ __forceinline__ void tr(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (slot < TR_SLOTS) g_trace[blockIdx.x * TR_SLOTS + slot] = t;
}
// per launch (index = launches completed so far): earliest CTA start, latest CTA end
__device__ unsigned long long g_kt[512][2];
__device__ unsigned g_kcount;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
__device__ __forceinline__ void tr(int) {}
#endif
// slots: 0 epilogue start, 1 first weight box, 2 predecessor wait returned,
// 3+p input of projection p ready, 7+p first MMA of p, 11+p last MMA of p,
// 15+p last partial of p written, 20+2k / 21+2k grid barrier k+1 arrive / pass

template <int NT>
struct Cfg {
  static constexpr int X_BYTES = NT * BK * 2;
  static constexpr int STAGE_BYTES = W_BYTES + X_BYTES;
  static constexpr int STAGES = (216 * 1024) / STAGE_BYTES > 8 ? 8 : (216 * 1024) / STAGE_BYTES;
  static constexpr int ACC_COLS = 2 * NT;  // both 128-row tiles of a segment
  static constexpr int TMEM_COLS = 2 * ACC_COLS < 32 ? 32 : 2 * ACC_COLS;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 512;
};

// ------------------------------------------------------------ work split
// (32-bit: units * grid < 2^32 is checked on the host)
__host__ __device__ __forceinline__ int range_start(int units, int grid, int c) {
  return (int)(((unsigned)units * (unsigned)c) / (unsigned)grid);
}
// the CTA whose unit range holds unit u
__host__ __device__ __forceinline__ int owner(int units, int grid, int u) {
  return (int)((((unsigned)u + 1u) * (unsigned)grid - 1u) / (unsigned)units);
}

// ---------------------------------------------------------- sync helpers
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void epi_sync() {  // the 128 epilogue threads only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Grid barrier of the epilogue warps: every CTA's 128 epilogue threads
// arrive; returns once all `grid` CTAs have arrived `k` times in total.  Their
// prior global writes are visible to every thread past the barrier (bar.sync
// + gpu-scope release/acquire, cumulative) and, through the async-proxy
// fences, to TMA loads.  Thread 0 then publishes the count to this CTA's
// producer in shared memory (release/acquire at CTA scope), so the producer
// never polls global memory.
__device__ __forceinline__ void st_release_cta(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_cta(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned k, unsigned grid, int etid,
                                             unsigned* smem_done) {
  fence_proxy_async_global();
  epi_sync();
  if (etid == 0) {
    red_release_add(ctr, 1u);
    while (ld_acquire(ctr) < k * grid) __nanosleep(20);
    fence_proxy_async_global();
    st_release_cta(smem_done, k);
  }
  epi_sync();
}

__device__ __forceinline__ float silu(float x) {  // as the split-K reduce kernel's SwiGLU
  float e = fast_exp2(-1.4426950408889634f * x), r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + e));
  return x * r;
}

__device__ __forceinline__ float4 ldcg4(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void add4(float4& a, float4 b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// Segment sums of IB items x R column offsets: item i = tile t[i], token
// j[i]; output rows t*256 + r[i][q].  acc = ascending-k sum of the tile's
// segment partials (slab (t, s), s < the tile's segment count; a CTA whose unit
// range is empty — only when units < grid — contributes +0).  All loads of a
// batch of 4 segments x IB x R are issued before any is summed.
template <int IB, int R>
__device__ __forceinline__ void seg_sums(const Proj& P, int grid, int rows, const int (&t)[IB],
                                         const int (&j)[IB], const int (&r)[IB][R],
                                         const bool (&valid)[IB], float4 (&acc)[IB][R]) {
  const bool dense = P.units >= grid;
  const int64_t stride = (int64_t)rows * 256;
  int first[IB], n[IB], nmax = 0;
  const float* base[IB];
#pragma unroll
  for (int i = 0; i < IB; ++i) {
    const int u0 = t[i] * P.kb;
    first[i] = owner(P.units, grid, u0);
    n[i] = valid[i] ? owner(P.units, grid, u0 + P.kb - 1) - first[i] + 1 : 0;
    nmax = max(nmax, n[i]);
    base[i] = P.slab + ((int64_t)t[i] * P.maxseg * rows + j[i]) * 256;
#pragma unroll
    for (int q = 0; q < R; ++q) acc[i][q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int s0 = 0; s0 < nmax; s0 += 4) {
    float4 v[IB][R][4];
#pragma unroll
    for (int i = 0; i < IB; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int sg = s0 + k;
        bool ok = sg < n[i];
        if (ok && !dense) {
          const int c = first[i] + sg, u0 = t[i] * P.kb;
          ok = max(range_start(P.units, grid, c), u0) <
               min(range_start(P.units, grid, c + 1), u0 + P.kb);
        }
#pragma unroll
        for (int q = 0; q < R; ++q)
          v[i][q][k] = ok ? ldcg4(base[i] + sg * stride + r[i][q]) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int i = 0; i < IB; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (s0 + k < n[i])
#pragma unroll
          for (int q = 0; q < R; ++q) add4(acc[i][q], v[i][q][k]);
  }
}

// Row-sum of squares over float4 chunks q = i * 128 + etid (chunk-ordered tree
// of rms_chunk_sum in common.cuh, on the epilogue warps' named barrier) —
// bit-identical to the standalone norm kernels for the same row.
__device__ __forceinline__ float epi_chunk_sum(const float (&ssq)[MAX_VEC], int vec, int hidden,
                                               float* red, int etid) {
  const int w = etid >> 5, lane = etid & 31;
  const int n_groups = (hidden / 4 + 31) / 32;
#pragma unroll
  for (int i = 0; i < MAX_VEC; ++i) {
    if (i >= vec) break;
    float s = ssq[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int grp = i * 4 + w;
    if (lane == 0 && grp < n_groups) red[grp] = s;
  }
  epi_sync();
  if (etid < 32) {
    float s = 0.f;
    for (int g = lane; g < n_groups; g += 32) s += red[g];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (etid == 0) red[n_groups] = s;
  }
  epi_sync();
  const float r = red[n_groups];
  epi_sync();  // red is reused by the next row
  return r;
}

// out[j] = bf16(gain * x[j] / rms(x[j])), one CTA per row (the chunk tree of
// the standalone norm kernels: bit-identical for the same x).
__device__ void norm_rows(const Args& a, const float* gain, __nv_bfloat16* out, int64_t ldo,
                          float* red, int etid) {
  const int vec = (a.hidden / 4 + EPI_THREADS - 1) / EPI_THREADS;
  for (int j = blockIdx.x; j < a.rows; j += a.grid) {
    if (etid == 0) tr(40);
    const float* xr = a.x + (int64_t)j * a.ldx;
    float4 v[MAX_VEC];
    float ssq[MAX_VEC];
    float4 g[MAX_VEC];
#pragma unroll
    for (int i = 0; i < MAX_VEC; ++i) {
      const int col = (i * EPI_THREADS + etid) * 4;
      const bool ok = i < vec && col < a.hidden;
      v[i] = ok ? ldcg4(xr + col) : make_float4(0.f, 0.f, 0.f, 0.f);
      g[i] = ok ? *reinterpret_cast<const float4*>(gain + col) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < MAX_VEC; ++i) ssq[i] = norm_sq4(v[i]);
    if (etid == 0) tr(41);
    const float ss = epi_chunk_sum(ssq, vec, a.hidden, red, etid);
    const float den = norm_den(ss, a.hidden, a.eps);
    if (etid == 0) tr(42);
#pragma unroll
    for (int i = 0; i < MAX_VEC; ++i) {
      if (i >= vec) continue;
      const int col = (i * EPI_THREADS + etid) * 4;
      if (col >= a.hidden) continue;
      *reinterpret_cast<uint2*>(out + (int64_t)j * ldo + col) =
          norm_pack4(g[i], v[i].x, v[i].y, v[i].z, v[i].w, den);
    }
    if (etid == 0) tr(43);
  }
}

// Grid-stride items of a reduction step, IB per round: idx = k-th item of this
// thread (k = 0, 1, ...), valid while < total.
#define DL_ITEMS(IB, total)                                                          \
  for (int base_ = blockIdx.x * EPI_THREADS + etid, step_ = a.grid * EPI_THREADS;    \
       base_ < (total); base_ += (IB) * step_)

// x[j][t*256 + r] += segment sums (residual add of a hidden-wide projection),
// all CTAs, 4 columns per item
__device__ void res_rows(const Args& a, const Proj& P, int etid) {
  constexpr int IB = 4;
  const int per_row = P.tiles * 64;
  const int total = a.rows * per_row;
  DL_ITEMS(IB, total) {
    int t[IB], j[IB], r[IB][1];
    bool ok[IB];
    float4 xv[IB], s4[IB][1];
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      const int idx = base_ + i * step_;
      ok[i] = idx < total;
      const int jj = ok[i] ? idx / per_row : 0, rem = ok[i] ? idx - jj * per_row : 0;
      j[i] = jj;
      t[i] = rem >> 6;
      r[i][0] = (rem & 63) * 4;
      xv[i] = ok[i] ? ldcg4(a.x + (int64_t)jj * a.ldx + t[i] * 256 + r[i][0])
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    seg_sums<IB, 1>(P, a.grid, a.rows, t, j, r, ok, s4);
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      if (!ok[i]) continue;
      add4(xv[i], s4[i][0]);
      __stcg(reinterpret_cast<float4*>(a.x + (int64_t)j[i] * a.ldx + t[i] * 256 + r[i][0]), xv[i]);
    }
  }
}

// act[j][t*128 + r] = bf16(silu(gate) * up); gate/up = rows r / 128 + r of tile t
__device__ void swiglu_rows(const Args& a, const Proj& P, int etid) {
  constexpr int IB = 2;
  const int per_row = P.tiles * 32;
  const int total = a.rows * per_row;
  DL_ITEMS(IB, total) {
    int t[IB], j[IB], r[IB][2];
    bool ok[IB];
    float4 s4[IB][2];
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      const int idx = base_ + i * step_;
      ok[i] = idx < total;
      const int jj = ok[i] ? idx / per_row : 0, rem = ok[i] ? idx - jj * per_row : 0;
      j[i] = jj;
      t[i] = rem >> 5;
      r[i][0] = (rem & 31) * 4;
      r[i][1] = 128 + r[i][0];
    }
    seg_sums<IB, 2>(P, a.grid, a.rows, t, j, r, ok, s4);
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      if (!ok[i]) continue;
      const float4 g = s4[i][0], u = s4[i][1];
      uint2 o;
      o.x = pack_bf16x2(silu(g.x) * u.x, silu(g.y) * u.y);
      o.y = pack_bf16x2(silu(g.z) * u.z, silu(g.w) * u.w);
      *reinterpret_cast<uint2*>(P.out + (int64_t)j[i] * P.ldo + t[i] * 128 + r[i][0]) = o;
    }
  }
}

// QKV rows [q heads | k heads | v heads] x 128: bf16-rounded sums, RoPE on q
// and k (rope_rotate: the rounding of rope_kv_kernel), q -> q_out, k/v -> the
// paged pool at the token's slot.  One item = 4 rotation pairs (i, i + 64).
__device__ void rope_rows(const Args& a, const Proj& P, int etid) {
  constexpr int IB = 2;
  const int heads = a.q_heads + 2 * a.kv_heads;
  const int per_row = heads * 16;
  const int total = a.rows * per_row;
  DL_ITEMS(IB, total) {
    int t[IB], j[IB], r[IB][2], h[IB];
    bool ok[IB];
    float4 s4[IB][2];
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      const int idx = base_ + i * step_;
      ok[i] = idx < total;
      const int jj = ok[i] ? idx / per_row : 0, rem = ok[i] ? idx - jj * per_row : 0;
      j[i] = jj;
      h[i] = rem >> 4;
      t[i] = h[i] >> 1;
      r[i][0] = (h[i] & 1) * 128 + (rem & 15) * 4;
      r[i][1] = r[i][0] + 64;
    }
    seg_sums<IB, 2>(P, a.grid, a.rows, t, j, r, ok, s4);
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      if (!ok[i]) continue;
      const int hh = h[i], jj = j[i], ii = r[i][0] & 127;
      __nv_bfloat16* dst;
      bool rotate = a.rope != nullptr;
      if (hh < a.q_heads) {
        dst = a.q_out + (int64_t)jj * a.ldq + (int64_t)hh * 128;
      } else {
        const int sl = a.slot[jj];
        if (sl < 0) continue;
        const int kv = hh - a.q_heads;
        const int kvh = kv % a.kv_heads;
        __nv_bfloat16* pool = kv < a.kv_heads ? a.k_pool : a.v_pool;
        rotate = rotate && kv < a.kv_heads;
        const int64_t blk = sl / a.block_size, off = sl % a.block_size;
        dst = pool + ((blk * a.kv_heads + kvh) * a.block_size + off) * 128;
      }
      const float4 sa = s4[i][0], sb = s4[i][1];
      // the bf16 rounding of the stored projection, as rope_kv_kernel reads it
      float2 a01 = unpack_bf16x2(pack_bf16x2(sa.x, sa.y)), a23 = unpack_bf16x2(pack_bf16x2(sa.z, sa.w));
      float2 b01 = unpack_bf16x2(pack_bf16x2(sb.x, sb.y)), b23 = unpack_bf16x2(pack_bf16x2(sb.z, sb.w));
      if (rotate) {
        const float4* cs = reinterpret_cast<const float4*>(a.rope + ((int64_t)a.pos[jj] * 64 + ii) * 2);
        const float4 c0 = cs[0], c1 = cs[1];
        float na, nb, nc, nd;
        rope_rotate(a01.x, b01.x, c0.x, c0.y, na, nb);
        rope_rotate(a01.y, b01.y, c0.z, c0.w, nc, nd);
        a01 = make_float2(na, nc);
        b01 = make_float2(nb, nd);
        rope_rotate(a23.x, b23.x, c1.x, c1.y, na, nb);
        rope_rotate(a23.y, b23.y, c1.z, c1.w, nc, nd);
        a23 = make_float2(na, nc);
        b23 = make_float2(nb, nd);
      }
      *reinterpret_cast<uint2*>(dst + ii) =
          make_uint2(pack_bf16x2(a01.x, a01.y), pack_bf16x2(a23.x, a23.y));
      *reinterpret_cast<uint2*>(dst + 64 + ii) =
          make_uint2(pack_bf16x2(b01.x, b01.y), pack_bf16x2(b23.x, b23.y));
    }
  }
}

// L2 prefetch, at kernel start, of what the reduction steps will read from
// HBM (the weight stream keeps HBM saturated, so a cold load there waits
// several microseconds): the norm gains (CTAs that normalise a row), the
// rotary rows and the pos / slot of the rows.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ void prefetch_inputs(const Args& a, int etid) {
  if (blockIdx.x < a.rows) {
    const int lines = a.hidden / 32;  // 128-B lines of one f32 gain vector
    for (int p = -1; p < a.n_proj; ++p) {
      const float* g = p < 0 ? (a.lead_out ? a.lead_gain : nullptr)
                             : (a.proj[p].kind == SP_DL_RES_NORM && a.proj[p].out ? a.proj[p].gain : nullptr);
      if (!g) continue;
      for (int l = etid; l < lines; l += EPI_THREADS) prefetch_l2(g + l * 32);
    }
    if (a.rope != nullptr && a.pos != nullptr && etid < 4)
      prefetch_l2(a.rope + (int64_t)a.pos[blockIdx.x] * 128 + etid * 32);
  }
  if (blockIdx.x == 0 && etid < 2 && a.pos != nullptr)
    prefetch_l2(etid == 0 ? (const void*)a.pos : (const void*)a.slot);
}

template <int NT>
__global__ void __launch_bounds__(NUM_THREADS, 1) decode_layer_kernel(const __grid_constant__ Args a) {
  using C = Cfg<NT>;
  constexpr int STAGES = C::STAGES, STAGE_BYTES = C::STAGE_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // >= hidden / 128 + 1 floats
  unsigned* bars_done = reinterpret_cast<unsigned*>(red + 72);  // grid barriers passed (epilogue -> producer)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.grid, c = blockIdx.x;
  const bool lead = a.lead_out != nullptr;
#ifdef DL_TRACE
  unsigned launch_idx = 0;
  if (threadIdx.x == 0) {
    launch_idx = *(volatile unsigned*)&g_kcount;
    if (launch_idx < 512) atomicMin(&g_kt[launch_idx][0], gtime());
  }
#endif

  if (warp == 0 && lane == 0) {
    for (int p = 0; p < a.n_proj; ++p) {
      tma_prefetch_desc(&a.proj[p].tw);
      tma_prefetch_desc(&a.proj[p].tx);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull + s, 1);
      mbar_init(tempty + s, 4);
    }
    *bars_done = 0;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t evict_first = l2_evict_first_policy();
      int dq_stage[STAGES], dq_proj[STAGES], dq_k[STAGES];
      int dq_head = 0, dq_n = 0;
      int ready_upto = -1;  // projections whose input rows are known published
      // projection p's input rows: written by the predecessor kernel (need == 0:
      // griddepcontrol.wait, only once the ring is full of weight boxes) or by
      // this kernel's epilogue warps before grid barrier `need`
      auto ready = [&](int p, bool block) -> bool {
        if (p <= ready_upto) return true;
        const int need = a.proj[p].need;
        if (need == 0) {
          if (!block) return false;
          pdl_wait_impl();
          tr(2);
        } else {
          if (ld_acquire_cta(bars_done) < (unsigned)need) return false;
          fence_proxy_async_global();
        }
        ready_upto = p;
        tr(3 + p);
        return true;
      };
      auto service = [&](bool block) {
        while (dq_n > 0) {
          const int s = dq_stage[dq_head], p = dq_proj[dq_head];
          if (!ready(p, block)) return;
          tma_load_2d(smem + s * STAGE_BYTES + W_BYTES, &a.proj[p].tx, full + s, dq_k[dq_head], 0);
          dq_head = dq_head + 1 == STAGES ? 0 : dq_head + 1;
          --dq_n;
        }
      };
      for (int p = 0; p < a.n_proj; ++p) {
        const Proj& P = a.proj[p];
        const int u1 = range_start(P.units, G, c + 1);
        for (int u = range_start(P.units, G, c); u < u1; ++u) {
          const int t = u / P.kb, kb = u - t * P.kb;
          while (!mbar_try(empty + stage, phase ^ 1)) service(true);
          mbar_arrive_expect_tx(full + stage, STAGE_BYTES);
          tma_load_2d_hint(smem + stage * STAGE_BYTES, &P.tw, full + stage, kb * BK, t * 256,
                           evict_first);
          if (p == 0 && u == range_start(P.units, G, c)) tr(1);
          const int tail = dq_head + dq_n >= STAGES ? dq_head + dq_n - STAGES : dq_head + dq_n;
          dq_stage[tail] = stage;
          dq_proj[tail] = p;
          dq_k[tail] = kb * BK;
          ++dq_n;
          service(false);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      while (dq_n > 0) service(true);
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(128, NT);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int p = 0; p < a.n_proj; ++p) {
        const Proj& P = a.proj[p];
        const int u1 = range_start(P.units, G, c + 1);
        int u = range_start(P.units, G, c);
        while (u < u1) {
          const int t = u / P.kb;
          const int seg_end = min(u1, (t + 1) * P.kb);
          const int wv = min(2, (P.n - t * 256 + 127) / 128);
          mbar_wait(tempty + acc, aphase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
          for (int uu = u; uu < seg_end; ++uu) {
            mbar_wait(full + stage, phase);
            tc_fence_after();
            if (uu == range_start(P.units, G, c)) tr(7 + p);
            const uint32_t w_addr = smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t x_addr = w_addr + W_BYTES;
            for (int w = 0; w < wv; ++w) {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                umma_bf16(d_tmem + w * NT, sdesc_sw128(w_addr + w * W_TILE + k * 32),
                          sdesc_sw128(x_addr + k * 32), idesc, (uu != u || k != 0) ? 1u : 0u);
            }
            umma_commit(empty + stage);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(tfull + acc);
          acc ^= 1;
          if (acc == 0) aphase ^= 1;
          u = seg_end;
        }
        tr(11 + p);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int etid = threadIdx.x - 64;
    const int quarter = warp & 3;  // TMEM lanes this warp may read
    const int nl = quarter * 32 + lane;
    pdl_wait_impl();  // x, the input rows and the pool are written by predecessors
    unsigned bars = 0;
    int acc = 0;
    uint32_t aphase = 0;
    bool triggered = false;
    if (etid == 0) tr(0);
    prefetch_inputs(a, etid);
    auto barrier = [&]() {
      ++bars;
      if (etid == 0) tr(18 + 2 * (int)bars);
      grid_barrier(a.sync, bars, (unsigned)G, etid, bars_done);
      if (etid == 0) tr(19 + 2 * (int)bars);
      if (!triggered) {  // every CTA is resident now: successors may launch
        pdl_trigger_impl();
        triggered = true;
      }
    };
    if (lead) {
      norm_rows(a, a.lead_gain, a.lead_out, a.ld_lead, red, etid);
      barrier();
    }
    for (int p = 0; p < a.n_proj; ++p) {
      const Proj& P = a.proj[p];
      const int u1 = range_start(P.units, G, c + 1);
      int u = range_start(P.units, G, c);
      while (u < u1) {
        const int t = u / P.kb;
        const int seg_end = min(u1, (t + 1) * P.kb);
        const int seg = c - owner(P.units, G, t * P.kb);
        mbar_wait(tfull + acc, aphase);
        tc_fence_after();
        const uint32_t tb = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * C::ACC_COLS;
        float* dst = P.slab + ((int64_t)t * P.maxseg + seg) * a.rows * 256;
#pragma unroll 1
        for (int c0 = 0; c0 < a.rows; c0 += 8) {
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            uint32_t r[8];
            tmem_ld8(tb + w * NT + c0, r);
            tmem_ld_wait();
            const int row = w * 128 + nl;
            if (t * 256 + row < P.n) {
#pragma unroll
              for (int jj = 0; jj < 8; ++jj)
                if (c0 + jj < a.rows) __stcg(dst + (int64_t)(c0 + jj) * 256 + row, __uint_as_float(r[jj]));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + acc);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
        u = seg_end;
      }
      if (etid == 0) tr(15 + p);
      barrier();  // every partial of projection p is in its slab
      if (P.kind == SP_DL_RES_NORM) {
        res_rows(a, P, etid);
        if (P.out != nullptr) {
          barrier();  // whole residual rows are in x
          norm_rows(a, P.gain, P.out, P.ldo, red, etid);
        }
      } else if (P.kind == SP_DL_SWIGLU) {
        swiglu_rows(a, P, etid);
      } else {
        rope_rows(a, P, etid);
      }
      if (p + 1 < a.n_proj) barrier();  // the next projection's input rows are out
    }
    if (!triggered) pdl_trigger_impl();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  if (threadIdx.x == 0) {  // the last CTA out re-arms the counters (graph replays)
#ifdef DL_TRACE
    if (launch_idx < 512) atomicMax(&g_kt[launch_idx][1], gtime());
#endif
    __threadfence();
    const unsigned prev = atomicAdd(a.sync + 1, 1u);
    if (prev == (unsigned)G - 1) {
#ifdef DL_TRACE
      atomicAdd(&g_kcount, 1u);
#endif
      atomicExch(a.sync, 0u);
      atomicExch(a.sync + 1, 0u);
    }
  }
}

// ------------------------------------------------------------------ host side
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

static int max_segs(int units, int grid, int kb, int tiles) {
  int m = 1;
  for (int t = 0; t < tiles; ++t) {
    const int s = owner(units, grid, t * kb + kb - 1) - owner(units, grid, t * kb) + 1;
    if (s > m) m = s;
  }
  return m;
}

static int64_t slab_floats(const sp_dl_proj& p, int rows, int grid) {
  const int kb = (int)cdiv(p.k, BK), tiles = (int)cdiv(p.n, 256);
  return (int64_t)tiles * max_segs(tiles * kb, grid, kb, tiles) * rows * 256;
}

static int64_t ws_bytes(const sp_decode_layer_args* a, int grid) {
  int64_t f = 0;
  for (int p = 0; p < a->n_proj; ++p) f += (slab_floats(a->proj[p], a->rows, grid) + 63) / 64 * 64;
  return f * 4;
}

template <int NT>
static int launch(Args& A, cudaStream_t st) {
  using C = Cfg<NT>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_layer_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::SMEM_BYTES);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_layer_kernel<NT>, NUM_THREADS,
                                                  C::SMEM_BYTES);
    if (per_sm < 1) return fail(kCuda, "decode_layer: kernel does not fit on an SM");
    attr = true;
  }
  launch_k(decode_layer_kernel<NT>, A.grid, NUM_THREADS, C::SMEM_BYTES, st, A);
  return check_launch("decode_layer_kernel");
}

}  // namespace dl
}  // namespace sp

using namespace sp;

// debug: per-launch [start, end] globaltimer pairs since the last reset (DL_TRACE builds)
extern "C" int sp_decode_layer_ktrace(unsigned long long* host, int reset) {
#ifdef DL_TRACE
  cudaDeviceSynchronize();
  unsigned n = 0;
  cudaMemcpyFromSymbol(&n, dl::g_kcount, sizeof(n));
  if (host) cudaMemcpyFromSymbol(host, dl::g_kt, sizeof(unsigned long long) * 1024);
  if (reset) {
    static unsigned long long init[512][2];
    for (int i = 0; i < 512; ++i) { init[i][0] = ~0ull; init[i][1] = 0; }
    cudaMemcpyToSymbol(dl::g_kt, init, sizeof(init));
    unsigned z = 0;
    cudaMemcpyToSymbol(dl::g_kcount, &z, sizeof(z));
  }
  return (int)n;
#else
  (void)host;
  (void)reset;
  return 0;
#endif
}

// debug: copy the trace of the last launch (DL_TRACE builds; else returns 0)
extern "C" int sp_decode_layer_trace(unsigned long long* host, int n) {
#ifdef DL_TRACE
  const int m = n < 160 * dl::TR_SLOTS ? n : 160 * dl::TR_SLOTS;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, dl::g_trace, m * sizeof(unsigned long long));
  return m;
#else
  (void)host;
  (void)n;
  return 0;
#endif
}

extern "C" int64_t sp_decode_layer_ws_bytes(const sp_decode_layer_args* a) {
  if (!a || a->n_proj < 0 || a->n_proj > dl::MAX_PROJ || a->rows <= 0) return -1;
  return dl::ws_bytes(a, dl::sm_count());
}

extern "C" sp_status sp_decode_layer(const sp_decode_layer_args* a, void* stream) {
  using namespace sp::dl;
  if (!a) return fail(kInvalid, "decode_layer: null args");
  if (a->n_proj < 0 || a->n_proj > MAX_PROJ) return fail(kInvalid, "decode_layer: n_proj out of range");
  if (a->rows <= 0 || a->rows > 64) return fail(kUnsupported, "decode_layer: rows must be in [1, 64]");
  if (a->hidden <= 0 || a->hidden % 256 || a->hidden > 4 * EPI_THREADS * MAX_VEC)
    return fail(kUnsupported, "decode_layer: hidden must be a multiple of 256, <= 8192");
  if (!a->x || a->ldx % 4 || !a->sync) return fail(kInvalid, "decode_layer: x / sync");
  if (a->n_proj == 0 && !a->lead_out) return kOk;
  if (a->lead_out && (!a->lead_gain || a->ld_lead % 4))
    return fail(kInvalid, "decode_layer: leading norm needs a gain and a 4-aligned row stride");
  const int grid = sm_count();
  if (!a->ws || a->ws_bytes < ws_bytes(a, grid)) return fail(kInvalid, "decode_layer: workspace too small");
  const int nt = a->rows <= 16 ? 16 : (a->rows <= 32 ? 32 : 64);
  Args A;
  memset(&A, 0, sizeof(A));
  A.n_proj = a->n_proj;
  A.rows = a->rows;
  A.hidden = a->hidden;
  A.grid = grid;
  A.x = a->x;
  A.ldx = a->ldx;
  A.eps = a->eps;
  A.lead_gain = a->lead_gain;
  A.lead_out = static_cast<__nv_bfloat16*>(a->lead_out);
  A.ld_lead = a->ld_lead;
  A.pos = a->pos;
  A.slot = a->slot;
  A.rope = a->rope;
  A.q_out = static_cast<__nv_bfloat16*>(a->q_out);
  A.ldq = a->ldq;
  A.k_pool = static_cast<__nv_bfloat16*>(a->k_pool);
  A.v_pool = static_cast<__nv_bfloat16*>(a->v_pool);
  A.q_heads = a->q_heads;
  A.kv_heads = a->kv_heads;
  A.block_size = a->block_size;
  A.sync = a->sync;
  float* ws = static_cast<float*>(a->ws);
  int need = a->lead_out ? 1 : 0;  // grid barriers before each projection's input is out
  for (int p = 0; p < a->n_proj; ++p) {
    const sp_dl_proj& s = a->proj[p];
    Proj& P = A.proj[p];
    if (!s.w || !s.x || s.n <= 0 || s.k <= 0 || s.k % BK || s.ldw % 8 || s.ldx % 8)
      return fail(kInvalid, "decode_layer: projection needs k % 64 == 0 and 16-byte rows");
    if ((reinterpret_cast<uintptr_t>(s.w) | reinterpret_cast<uintptr_t>(s.x)) & 15)
      return fail(kInvalid, "decode_layer: projection operands must be 16-byte aligned");
    P.n = s.n;
    P.k = s.k;
    P.kb = s.k / BK;
    P.tiles = (int)cdiv(s.n, 256);
    P.units = P.tiles * P.kb;
    if ((int64_t)P.units * (grid + 1) >= (1ll << 32))
      return fail(kUnsupported, "decode_layer: projection too large for the 32-bit work split");
    P.maxseg = max_segs(P.units, grid, P.kb, P.tiles);
    P.kind = s.kind;
    P.need = need;
    need += 2 + (s.kind == SP_DL_RES_NORM && s.out ? 1 : 0);
    P.slab = ws;
    ws += (slab_floats(s, a->rows, grid) + 63) / 64 * 64;
    P.gain = s.gain;
    P.out = static_cast<__nv_bfloat16*>(s.out);
    P.ldo = s.ldo;
    if (s.kind == SP_DL_RES_NORM) {
      if (s.n != a->hidden) return fail(kInvalid, "decode_layer: RES_NORM projection must be hidden wide");
      if (s.out && (!s.gain || s.ldo % 4)) return fail(kInvalid, "decode_layer: RES_NORM output needs a gain");
    } else if (s.kind == SP_DL_SWIGLU) {
      if (s.n % 256 || !s.out || s.ldo % 4) return fail(kInvalid, "decode_layer: SWIGLU needs n % 256 == 0 and an output");
    } else if (s.kind == SP_DL_ROPE_KV) {
      if (a->head_dim != 128) return fail(kUnsupported, "decode_layer: RoPE/KV write needs head_dim 128");
      if (s.n != (a->q_heads + 2 * a->kv_heads) * 128 || !a->q_out || a->ldq % 4 || !a->pos ||
          (a->kv_heads > 0 && (!a->slot || !a->k_pool || !a->v_pool)) || a->block_size <= 0)
        return fail(kInvalid, "decode_layer: RoPE/KV write geometry");
    } else {
      return fail(kInvalid, "decode_layer: unknown projection kind");
    }
    {
      uint64_t dims[2] = {(uint64_t)s.k, (uint64_t)s.n};
      uint64_t strides[1] = {(uint64_t)s.ldw * 2};
      uint32_t box[2] = {BK, 256};
      if (int rc = tma_map_bf16(&P.tw, s.w, 2, dims, strides, box)) return rc;
    }
    {
      uint64_t dims[2] = {(uint64_t)s.k, (uint64_t)a->rows};
      uint64_t strides[1] = {(uint64_t)s.ldx * 2};
      uint32_t box[2] = {BK, (uint32_t)nt};
      if (int rc = tma_map_bf16(&P.tx, s.x, 2, dims, strides, box)) return rc;
    }
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (nt == 16) return launch<16>(A, st);
  if (nt == 32) return launch<32>(A, st);
  return launch<64>(A, st);
}
