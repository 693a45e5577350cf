// Shared device/host helpers for the sm_100a kernels of the Shift-Parallel path.
// Inline-PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor), tcgen05
// (alloc / mma / commit / ld) and the legacy ldmatrix/mma.sync used by the
// attention kernels.  Written for sm_100a only.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

namespace sp {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

enum Status : int {
  kOk = 0,
  kInvalid = 1,
  kCuda = 2,
  kUnsupported = 3,
};

// ------------------------------------------- programmatic dependent launch
// Every kernel is launched with programmatic stream serialization: it may start
// while its predecessor drains, so it must (a) touch only immutable data (the
// weights) before pdl_wait(), and (b) call pdl_trigger() so its own successor
// can launch early.  Disabled with SP_PDL=0.
bool pdl_enabled();

__device__ __forceinline__ void pdl_wait_impl() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger_impl() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------ step timeline (debug builds)
// Built with -DSTEP_TRACE (tools/step_trace.py): every CTA of every kernel
// records the call site of its entry pdl_trigger() (translation unit, line),
// its block, and globaltimer stamps at entry, at griddepcontrol.wait release
// and at exit into a device buffer the host binds with sp_step_trace_bind.
// The production build compiles none of it.
struct StepTraceRec {
  unsigned long long tag;  // [63:32] linear block index, [31:16] TU id, [15:0] line
  unsigned long long t_entry, t_wait, t_exit;
};
void step_trace_register(void (*bind)(void* buf, void* counter, int cap));

#ifndef SP_TU_ID
#define SP_TU_ID 0
#endif

#ifdef STEP_TRACE
__device__ __forceinline__ unsigned long long sp_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
static __device__ StepTraceRec* g_st_buf = nullptr;
static __device__ unsigned int* g_st_n = nullptr;
static __device__ int g_st_cap = 0;
static __shared__ unsigned int sp_st_slot;

struct StepTraceScope {
  __device__ explicit StepTraceScope(unsigned tag) {
    if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0) {
      unsigned s = ~0u;
      if (g_st_buf != nullptr) s = atomicAdd(g_st_n, 1u);
      sp_st_slot = s;
      if (s < (unsigned)g_st_cap) {
        const unsigned long long blk = blockIdx.x + (unsigned long long)blockIdx.y * gridDim.x +
                                       (unsigned long long)blockIdx.z * gridDim.x * gridDim.y;
        g_st_buf[s].tag = (blk << 32) | tag;
        g_st_buf[s].t_wait = 0;
        g_st_buf[s].t_entry = sp_gtime();
      }
    }
    __syncwarp();
  }
  __device__ ~StepTraceScope() {
    if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0) {
      const unsigned s = sp_st_slot;
      if (s < (unsigned)g_st_cap) g_st_buf[s].t_exit = sp_gtime();
    }
  }
};
__device__ __forceinline__ void sp_trace_wait() {
  if ((threadIdx.x & 31) == 0 && g_st_buf != nullptr) {
    const unsigned s = sp_st_slot;
    if (s < (unsigned)g_st_cap) atomicCAS(&g_st_buf[s].t_wait, 0ull, sp_gtime());
  }
}
#define pdl_trigger()                                                                \
  ::sp::StepTraceScope sp_step_trace_scope_((SP_TU_ID << 16) | (__LINE__ & 0xffff)); \
  ::sp::pdl_trigger_impl()
#define pdl_wait() (::sp::pdl_wait_impl(), ::sp::sp_trace_wait())
// binds this translation unit's trace pointers (registered at load time)
static void step_trace_bind_local(void* buf, void* counter, int cap) {
  cudaMemcpyToSymbol(g_st_buf, &buf, sizeof(buf));
  cudaMemcpyToSymbol(g_st_n, &counter, sizeof(counter));
  cudaMemcpyToSymbol(g_st_cap, &cap, sizeof(cap));
}
static const bool sp_step_trace_registered_ = (step_trace_register(step_trace_bind_local), true);
#else
#define pdl_trigger() ::sp::pdl_trigger_impl()
#define pdl_wait() ::sp::pdl_wait_impl()
#endif

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// RoPE rotation of one (x_i, x_{i+d/2}) pair, rounding explicit (no FMA
// contraction) so the standalone RoPE kernel and the GEMM epilogue that fuses
// it produce identical bits: (a cos - b sin, b cos + a sin).
__device__ __forceinline__ void rope_rotate(float a, float b, float c, float s, float& na,
                                            float& nb) {
  na = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s));
  nb = __fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s));
}

// ------------------------------------------------------------ small utils
__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float2 unpack_bf16x2(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}

// -------------------------------------------------------------- fast math
// 2^x on the SFU (ex2.approx.ftz: no denormal-range fix-up instructions);
// inputs here are softmax exponents <= 0 (or -inf -> +0).
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Blackwell paired f32 ops (FFMA2 / FADD2): two lanes of work per instruction
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// --------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// -------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* desc, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* desc, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// L2 cache policy for data streamed exactly once (decode weights: 15 GB per
// step through a 126 MB L2) — evicted first, so it does not push the kernels'
// code, activations and partial sums out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// SP_L2_HINT=0 turns the evict-first hint of the decode streams off (A/B runs)
bool l2_hint_enabled();

__device__ __forceinline__ void tma_load_2d_hint(void* smem_dst, const void* desc, uint64_t* bar,
                                                 int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// TMA store (smem box -> global tile, bulk-group completion): used for the
// fused exchange epilogues, whose destination rows live in a peer's buffer
__device__ __forceinline__ void tma_store_2d(const void* desc, const void* smem_src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(desc),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, f32 accumulate)
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// arrive on an mbarrier once all previously issued tcgen05 ops of this thread finish
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Shared-memory matrix descriptor: K-major operand, 128-byte swizzle, rows of
// 128 B, 8-row swizzle atoms 1024 B apart (SBO), LBO unused (=16 B), version 1.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor for kind::f16: bf16 A/B, f32 D, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// 32 lanes x 32 consecutive f32 columns (one row per thread)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}

// 32 lanes x 8 consecutive f32 columns
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// TMEM stores, the TMEM-A-operand MMA and the MN-major shared-memory
// descriptor (attention: P, or Q, from TMEM; V as an MN-major B operand)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]   (A = P, bf16 packed two per 32-bit column)
__device__ __forceinline__ void umma_ts_bf16(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// MN-major (N contiguous) 128-byte-swizzle descriptor: 64-element rows of
// 128 B along N, 8-row atoms SBO = 1024 B apart along K, next 64-wide N
// chunk LBO bytes away.
__device__ __forceinline__ uint64_t sdesc_sw128_mn(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// ----------------------------------------------------- RMSNorm reduction
// Sum of squares of a row in an order defined on float4 CHUNKS, not threads
// (chunk q = i * blockDim + tid; ssq[i] = that chunk's x*x sum): butterfly
// inside each group of 32 consecutive chunks, then the group sums in ascending
// stride-32 order and a final butterfly.  Identical bits for any block size
// (a multiple of 32), so launchers may size blocks by row count; every norm
// kernel uses it so fused and unfused paths agree bit-for-bit.  `red` is a
// shared array of >= hidden/128 floats.  Returns the row sum to every thread.
template <int VEC>
__device__ __forceinline__ float rms_chunk_sum(const float (&ssq)[VEC], int hidden, float* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_groups = (hidden / 4 + 31) / 32;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    float s = ssq[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int grp = i * (blockDim.x >> 5) + warp;
    if (lane == 0 && grp < n_groups) red[grp] = s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    float s = 0.f;
    for (int g = lane; g < n_groups; g += 32) s += red[g];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

// Row-norm arithmetic shared by every RMSNorm kernel (add_rmsnorm and the
// fused TP all-reduce variants), with the rounding pinned — no FMA
// contraction, which nvcc applies per call site — so the fused kernels are
// bit-identical to the plain one by construction.
__device__ __forceinline__ float norm_sq4(float4 t) {
  return __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(t.x, t.x), __fmul_rn(t.y, t.y)),
                             __fmul_rn(t.z, t.z)),
                   __fmul_rn(t.w, t.w));
}

__device__ __forceinline__ float norm_den(float ss, int hidden, float eps) {
  return sqrtf(__fadd_rn(__fdiv_rn(ss, (float)hidden), eps));
}

// bf16x4 of gain * (v / den)
__device__ __forceinline__ uint2 norm_pack4(float4 g, float v0, float v1, float v2, float v3,
                                            float den) {
  uint2 u;
  u.x = pack_bf16x2(__fmul_rn(g.x, __fdiv_rn(v0, den)), __fmul_rn(g.y, __fdiv_rn(v1, den)));
  u.y = pack_bf16x2(__fmul_rn(g.z, __fdiv_rn(v2, den)), __fmul_rn(g.w, __fdiv_rn(v3, den)));
  return u;
}

// Block size of the norm kernels: one float4 per thread (up to 1024 threads)
// for few rows (decode: one CTA per row, loads spread wide), 256-thread
// blocks for many rows (prefill) — measured: 1024 costs ~2.5% of an 8K
// prefill, 256 costs ~5% of a B=64 decode.  Results do not depend on it.
inline int norm_block_threads(int rows, int hidden) {
  const int wide = hidden / 4 >= 1024 ? 1024 : ((hidden / 4 + 31) / 32) * 32;
  const int w = wide < 32 ? 32 : wide;
  if (rows <= 2 * 148) return w;
  int narrow = ((hidden / 32 + 31) / 32) * 32;
  if (narrow < 256) narrow = 256;
  return narrow < w ? narrow : w;
}

// ------------------------------------------------- legacy tensor-core helpers
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, bool pred) {
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                            uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                                  uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D = A(16x16 bf16) * B(16x8 bf16) + C, f32 accumulate
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

}  // namespace sp
