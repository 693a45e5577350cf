#include <algorithm>
// Error plumbing, device check and the small HBM-bound kernels of the path:
// embedding gather, fused residual-add + RMSNorm, RoPE + paged KV write,
// all-to-all pack/unpack, loopback add, argmax and row gather.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/shiftpar.h"
#define SP_TU_ID 6  // step-trace tag (common.cuh)
#include "common.cuh"

namespace sp {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

static std::atomic<long long> g_launches{0};

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SP_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

static std::vector<void (*)(void*, void*, int)>& step_trace_registry() {
  static std::vector<void (*)(void*, void*, int)> v;
  return v;
}

void step_trace_register(void (*bind)(void* buf, void* counter, int cap)) {
  step_trace_registry().push_back(bind);
}

bool l2_hint_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SP_L2_HINT");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
  return kOk;
}

// ----------------------------------------------------------------- embedding
__global__ void embed_kernel(const int32_t* __restrict__ ids, const __nv_bfloat16* __restrict__ table,
                             const int32_t* __restrict__ pos, const float* __restrict__ pos_table,
                             float* __restrict__ out, int hidden) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  const int r = blockIdx.x;
  const int64_t tok = ids[r];
  const __nv_bfloat16* src = table + tok * hidden;
  float* dst = out + (int64_t)r * hidden;
  const float* pt = pos_table ? pos_table + (int64_t)pos[r] * hidden : nullptr;
  for (int c = threadIdx.x * 8; c < hidden; c += blockDim.x * 8) {
    uint4 u = *reinterpret_cast<const uint4*>(src + c);
    float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y), e = unpack_bf16x2(u.z),
           f = unpack_bf16x2(u.w);
    float v[8] = {a.x, a.y, b.x, b.y, e.x, e.y, f.x, f.y};
    if (pt) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += pt[c + j];
    }
    reinterpret_cast<float4*>(dst + c)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(dst + c)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// ------------------------------------------------------- add + rmsnorm
template <int VEC>
__global__ void add_rmsnorm_kernel(float* __restrict__ x, int64_t ldx, const float* __restrict__ add,
                                   int n_add, int64_t add_stride, const float* __restrict__ gain,
                                   float eps,
                                   const int32_t* __restrict__ row_idx,
                                   __nv_bfloat16* __restrict__ out, int64_t ldo, int hidden) {
  // the gain is a weight (never written by a predecessor): fetched before the wait
  float4 g[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    g[i] = out && c < hidden ? *reinterpret_cast<const float4*>(gain + c)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  constexpr int BATCH = VEC == 1 ? 12 : 4;  // partial loads in flight together
  const int r = blockIdx.x;
  const int64_t src_row = row_idx ? row_idx[r] : r;
  float* xr = x + src_row * ldx;
  const float* ar = add ? add + (int64_t)r * hidden : nullptr;
  float v[VEC * 4];
  float ssq[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < hidden) {
      t = *reinterpret_cast<const float4*>(xr + c);
      if (ar) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s0 = 0; s0 < n_add; s0 += BATCH) {  // ascending: the split-K / all-reduce order
          float4 b[BATCH];
#pragma unroll
          for (int u = 0; u < BATCH; ++u)
            b[u] = s0 + u < n_add ? *reinterpret_cast<const float4*>(ar + (s0 + u) * add_stride + c)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < BATCH; ++u) {
            if (s0 + u < n_add) {
              a.x += b[u].x;
              a.y += b[u].y;
              a.z += b[u].z;
              a.w += b[u].w;
            }
          }
        }
        t.x += a.x;
        t.y += a.y;
        t.z += a.z;
        t.w += a.w;
        *reinterpret_cast<float4*>(xr + c) = t;
      }
    }
    v[4 * i + 0] = t.x;
    v[4 * i + 1] = t.y;
    v[4 * i + 2] = t.z;
    v[4 * i + 3] = t.w;
    ssq[i] = norm_sq4(t);
  }
  __shared__ float red[256];
  const float ss = rms_chunk_sum<VEC>(ssq, hidden, red);
  const float den = norm_den(ss, hidden, eps);
  __nv_bfloat16* orow = out + (int64_t)r * ldo;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    if (c < hidden) {
      const uint2 u = norm_pack4(g[i], v[4 * i + 0], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3], den);
      *reinterpret_cast<uint2*>(orow + c) = u;
    }
  }
}

// RMSNorm without a residual add (the prefill norms: the projection epilogue
// already added the residual), register-lean so that 6+ CTAs per SM keep
// enough row bytes in flight (the general kernel's 76 registers allowed 3 and
// reached half the HBM bandwidth): the gains are loaded only for the store
// (L2-resident), not held across the reduction.  Same block size and chunk
// order -> bit-identical to add_rmsnorm_kernel.
template <int VEC, int MINB>
__global__ void __launch_bounds__(256, MINB)
    rmsnorm_lean_kernel(const float* __restrict__ x, int64_t ldx, const float* __restrict__ gain,
                        float eps, __nv_bfloat16* __restrict__ out, int64_t ldo, int hidden) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // x is written by the predecessor
  const int64_t r = blockIdx.x;
  const float* xr = x + r * ldx;
  float4 v[VEC];
  float ssq[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    v[i] = c < hidden ? __ldcs(reinterpret_cast<const float4*>(xr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < VEC; ++i) ssq[i] = norm_sq4(v[i]);
  __shared__ float red[256];
  const float ss = rms_chunk_sum<VEC>(ssq, hidden, red);
  const float den = norm_den(ss, hidden, eps);
  __nv_bfloat16* orow = out + r * ldo;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    if (c < hidden) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c));
      *reinterpret_cast<uint2*>(orow + c) = norm_pack4(g, v[i].x, v[i].y, v[i].z, v[i].w, den);
    }
  }
}

// ------------------------------------------------- RoPE + paged KV write
// 8 threads per (token, head): thread j owns rotation pairs [8j, 8j+8) of a
// 128-dim head (16-byte loads of both halves, one float4x2 of cos/sin each);
// generic head_dim falls back to one pair per lane.
// 8 consecutive values at column c of row r: the bf16 qkv row, or (parts !=
// NULL) the ascending sum of n_parts f32 K-split partials [n][rows][ldqkv]
// rounded to bf16 — the split-K reduction of the QKV projection fused here,
// bit-identical to reducing first (same order, same final rounding).
__device__ __forceinline__ uint4 qkv_chunk(const __nv_bfloat16* qkv, const float* parts, int n_parts,
                                           int64_t ldqkv, int rows, int r, int64_t c) {
  if (parts == nullptr) return *reinterpret_cast<const uint4*>(qkv + (int64_t)r * ldqkv + c);
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = 0.f;
  for (int s = 0; s < n_parts; ++s) {
    const float* src = parts + ((int64_t)s * rows + r) * ldqkv + c;
    const float4 a = *reinterpret_cast<const float4*>(src);
    const float4 b = *reinterpret_cast<const float4*>(src + 4);
    v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
    v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
  }
  uint4 u;
  u.x = pack_bf16x2(v[0], v[1]);
  u.y = pack_bf16x2(v[2], v[3]);
  u.z = pack_bf16x2(v[4], v[5]);
  u.w = pack_bf16x2(v[6], v[7]);
  return u;
}

__global__ void rope_kv_kernel(const __nv_bfloat16* __restrict__ qkv, const float* __restrict__ parts,
                               int n_parts, int64_t ldqkv,
                               const int32_t* __restrict__ pos, const int32_t* __restrict__ slot,
                               const float* __restrict__ rope, __nv_bfloat16* __restrict__ q_out,
                               int64_t ldq, __nv_bfloat16* __restrict__ k_pool,
                               __nv_bfloat16* __restrict__ v_pool, int rows, int q_heads,
                               int kv_heads, int head_dim, int block_size) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  const int heads = q_heads + 2 * kv_heads;
  const int half = head_dim >> 1;
  const int tpg = half / 8;  // threads per (token, head) when vectorised
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t item = gid / tpg;
  if (item >= (int64_t)rows * heads) return;
  const int j = (int)(gid % tpg);
  const int r = (int)(item / heads);
  const int h = (int)(item % heads);
  const int64_t col = (int64_t)h * head_dim;
  __nv_bfloat16* dst;
  if (h < q_heads) {
    if (!q_out) return;
    dst = q_out + (int64_t)r * ldq + (int64_t)h * head_dim;
  } else {
    const int s = slot[r];
    if (s < 0) return;
    const int kvh = (h - q_heads) % kv_heads;
    __nv_bfloat16* pool = (h - q_heads) < kv_heads ? k_pool : v_pool;
    const int64_t blk = s / block_size, off = s % block_size;
    dst = pool + ((blk * kv_heads + kvh) * block_size + off) * head_dim;
  }
  const bool rotate = rope != nullptr && h < q_heads + kv_heads;
  const int i0 = j * 8;
  uint4 ua = qkv_chunk(qkv, parts, n_parts, ldqkv, rows, r, col + i0);
  uint4 ub = qkv_chunk(qkv, parts, n_parts, ldqkv, rows, r, col + half + i0);
  if (rotate) {
    const float4* cs = reinterpret_cast<const float4*>(rope + ((int64_t)pos[r] * half + i0) * 2);
    uint32_t* pa = reinterpret_cast<uint32_t*>(&ua);
    uint32_t* pb = reinterpret_cast<uint32_t*>(&ub);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 c2 = cs[q];  // (cos, sin) of pairs i0+2q and i0+2q+1
      const float2 a = unpack_bf16x2(pa[q]);
      const float2 b = unpack_bf16x2(pb[q]);
      float na0, nb0, na1, nb1;
      rope_rotate(a.x, b.x, c2.x, c2.y, na0, nb0);
      rope_rotate(a.y, b.y, c2.z, c2.w, na1, nb1);
      pa[q] = pack_bf16x2(na0, na1);
      pb[q] = pack_bf16x2(nb0, nb1);
    }
  }
  *reinterpret_cast<uint4*>(dst + i0) = ua;
  *reinterpret_cast<uint4*>(dst + half + i0) = ub;
}

// ------------------------------------------------------ a2a pack/unpack
__global__ void pack_kernel(const uint4* __restrict__ src, int64_t lds_v, uint4* __restrict__ dst,
                            int rows, int peers, int width_v) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  const int64_t total = (int64_t)rows * peers * width_v;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % width_v;
    const int64_t r = (i / width_v) % rows;
    const int64_t p = i / ((int64_t)width_v * rows);
    dst[i] = src[r * lds_v + p * width_v + c];
  }
}

__global__ void unpack_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t ldd_v,
                              int rows, int peers, int width_v) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  const int64_t total = (int64_t)rows * peers * width_v;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % width_v;
    const int64_t p = (i / width_v) % peers;
    const int64_t r = i / ((int64_t)width_v * peers);
    dst[r * ldd_v + p * width_v + c] = src[(p * rows + r) * width_v + c];
  }
}

// ------------------------------------------------------------ small ops
__global__ void add_f32_kernel(const float4* __restrict__ a, const float4* __restrict__ b,
                               float4* __restrict__ d, int64_t n4) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 x = a[i], y = b[i];
    d[i] = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
  }
}

__global__ void add_f32_tail_kernel(const float* a, const float* b, float* d, int64_t lo, int64_t n) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  int64_t i = lo + threadIdx.x;
  if (i < n) d[i] = a[i] + b[i];
}

__global__ void argmax_kernel(const float* __restrict__ logits, int64_t ld, int vocab,
                              int32_t* __restrict__ idx, float* __restrict__ val) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  const float* row = logits + (int64_t)blockIdx.x * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
    float x = row[i];
    if (x > best || (x == best && i < bi)) {
      best = x;
      bi = i;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    best = threadIdx.x < nw ? sv[threadIdx.x] : -INFINITY;
    bi = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (threadIdx.x == 0) {
      idx[blockIdx.x] = bi;
      if (val) val[blockIdx.x] = best;
    }
  }
}

__global__ void gather_rows_kernel(const float* __restrict__ src, int64_t lds,
                                   const int32_t* __restrict__ idx, float* __restrict__ dst,
                                   int64_t ldd, int width) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();  // inputs of this kernel are written by its predecessor
  const float* s = src + (int64_t)idx[blockIdx.x] * lds;
  float* d = dst + (int64_t)blockIdx.x * ldd;
  for (int c = threadIdx.x; c < width; c += blockDim.x) d[c] = s[c];
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace sp

using namespace sp;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" const char* sp_last_error(void) { return sp::g_err.c_str(); }

extern "C" int sp_abi_version(void) { return 1; }

extern "C" int64_t sp_kernel_launches(void) { return (int64_t)sp::g_launches.load(); }

extern "C" sp_status sp_device_check(int* sm_count) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(kCuda, std::string("no CUDA device: ") + cudaGetErrorString(e));
  int major = 0, minor = 0, sms = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sm_count) *sm_count = sms;
  if (major != 10 || minor != 0)
    return fail(kUnsupported, "libshiftpar is built for sm_100a (B200); device is sm_" +
                                  std::to_string(major) + std::to_string(minor));
  return kOk;
}

extern "C" sp_status sp_embed(const int32_t* ids, const void* table_bf16, const int32_t* pos,
                              const float* pos_table, float* out_f32, int rows, int hidden,
                              void* stream) {
  if (rows < 0 || hidden <= 0 || hidden % 8) return fail(kInvalid, "embed: hidden % 8 != 0");
  if (rows == 0) return kOk;
  if (pos_table && !pos) return fail(kInvalid, "embed: pos_table without positions");
  launch_k(embed_kernel, rows, 128, 0, S(stream), ids, static_cast<const __nv_bfloat16*>(table_bf16), pos,
                                            pos_table, out_f32, hidden);
  return check_launch("embed_kernel");
}

extern "C" sp_status sp_add_rmsnorm(float* x, int64_t ldx, const float* add, int n_add,
                                    const float* gain, float eps, const int32_t* row_idx,
                                    void* out_bf16, int64_t ldo, int rows, int hidden,
                                    void* stream) {
  if (add && n_add < 1) return fail(kInvalid, "add_rmsnorm: n_add must be >= 1");
  const int64_t add_stride = (int64_t)rows * hidden;
  if (rows < 0 || hidden <= 0 || hidden % 4 || ldx % 4 || ldo % 4)
    return fail(kInvalid, "add_rmsnorm: hidden and strides must be multiples of 4");
  if (rows == 0) return kOk;
  if (add && row_idx) return fail(kInvalid, "add_rmsnorm: add with row_idx unsupported");
  int threads = norm_block_threads(rows, hidden);
  if (const char* e = getenv("SP_NORM_THREADS")) threads = atoi(e);
  const int per = (hidden + threads * 4 - 1) / (threads * 4);
  auto out = static_cast<__nv_bfloat16*>(out_bf16);
  // many rows, no residual add, no gather: the register-lean kernel (SP_NORM_LEAN=0: general)
  const char* lean = getenv("SP_NORM_LEAN");
  if (!add && !row_idx && out && rows > 2 * 148 && threads == 256 && per == 4 &&
      !(lean && lean[0] == '0')) {
    launch_k(rmsnorm_lean_kernel<4, 6>, rows, threads, 0, S(stream), x, ldx, gain, eps, out, ldo, hidden);
    return check_launch("rmsnorm_lean_kernel");
  }
  switch (per) {
    case 1: launch_k(add_rmsnorm_kernel<1>, rows, threads, 0, S(stream), x, ldx, add, n_add, add_stride, gain, eps, row_idx, out, ldo, hidden); break;
    case 2: launch_k(add_rmsnorm_kernel<2>, rows, threads, 0, S(stream), x, ldx, add, n_add, add_stride, gain, eps, row_idx, out, ldo, hidden); break;
    case 3: launch_k(add_rmsnorm_kernel<3>, rows, threads, 0, S(stream), x, ldx, add, n_add, add_stride, gain, eps, row_idx, out, ldo, hidden); break;
    case 4: launch_k(add_rmsnorm_kernel<4>, rows, threads, 0, S(stream), x, ldx, add, n_add, add_stride, gain, eps, row_idx, out, ldo, hidden); break;
    case 5: case 6: case 7: case 8:
      launch_k(add_rmsnorm_kernel<8>, rows, threads, 0, S(stream), x, ldx, add, n_add, add_stride, gain, eps, row_idx, out, ldo, hidden); break;
    default: return fail(kUnsupported, "add_rmsnorm: hidden > 32768");
  }
  return check_launch("add_rmsnorm_kernel");
}

static sp_status rope_kv_launch(const void* qkv, const float* parts, int n_parts, int64_t ldqkv,
                                const int32_t* pos, const int32_t* slot, const float* rope_table,
                                void* q_out, int64_t ldq, void* k_pool, void* v_pool, int rows,
                                int q_heads, int kv_heads, int head_dim, int block_size,
                                void* stream);

extern "C" sp_status sp_rope_kv_write(const void* qkv, int64_t ldqkv, const int32_t* pos,
                                      const int32_t* slot, const float* rope_table, void* q_out,
                                      int64_t ldq, void* k_pool, void* v_pool, int rows,
                                      int q_heads, int kv_heads, int head_dim, int block_size,
                                      void* stream) {
  return rope_kv_launch(qkv, nullptr, 0, ldqkv, pos, slot, rope_table, q_out, ldq, k_pool, v_pool,
                        rows, q_heads, kv_heads, head_dim, block_size, stream);
}

extern "C" sp_status sp_rope_kv_write_partials(const float* parts, int n_parts, int64_t ldqkv,
                                               const int32_t* pos, const int32_t* slot,
                                               const float* rope_table, void* q_out, int64_t ldq,
                                               void* k_pool, void* v_pool, int rows, int q_heads,
                                               int kv_heads, int head_dim, int block_size,
                                               void* stream) {
  if (!parts || n_parts < 1) return fail(kInvalid, "rope_kv_write_partials: need >= 1 partial");
  return rope_kv_launch(nullptr, parts, n_parts, ldqkv, pos, slot, rope_table, q_out, ldq, k_pool,
                        v_pool, rows, q_heads, kv_heads, head_dim, block_size, stream);
}

static sp_status rope_kv_launch(const void* qkv, const float* parts, int n_parts, int64_t ldqkv,
                                const int32_t* pos, const int32_t* slot, const float* rope_table,
                                void* q_out, int64_t ldq, void* k_pool, void* v_pool, int rows,
                                int q_heads, int kv_heads, int head_dim, int block_size,
                                void* stream) {
  if (rows < 0 || q_heads < 0 || kv_heads < 0 || head_dim <= 0 || head_dim % 2 || block_size <= 0)
    return fail(kInvalid, "rope_kv_write: bad geometry");
  if (rows == 0 || q_heads + kv_heads == 0) return kOk;
  if (kv_heads > 0 && (!k_pool || !v_pool || !slot)) return fail(kInvalid, "rope_kv_write: null pool/slot");
  if (head_dim % 16) return fail(kUnsupported, "rope_kv_write: head_dim must be a multiple of 16");
  if (ldqkv % 8 || (q_out && ldq % 8)) return fail(kInvalid, "rope_kv_write: rows must be 16-byte aligned");
  const int heads = q_heads + 2 * kv_heads;
  const int64_t threads = (int64_t)rows * heads * (head_dim / 16);
  launch_k(rope_kv_kernel, (unsigned)((threads + 255) / 256), 256, 0, S(stream),
           static_cast<const __nv_bfloat16*>(qkv), parts, n_parts, ldqkv, pos, slot, rope_table,
           static_cast<__nv_bfloat16*>(q_out), ldq, static_cast<__nv_bfloat16*>(k_pool),
           static_cast<__nv_bfloat16*>(v_pool), rows, q_heads, kv_heads, head_dim, block_size);
  return check_launch("rope_kv_kernel");
}

extern "C" sp_status sp_a2a_pack(const void* src, int64_t lds, void* dst, int rows, int peers,
                                 int width, void* stream) {
  if (rows < 0 || peers <= 0 || width <= 0 || width % 8 || lds % 8)
    return fail(kInvalid, "a2a_pack: width and stride must be multiples of 8");
  if (rows == 0) return kOk;
  const int64_t n = (int64_t)rows * peers * (width / 8);
  launch_k(pack_kernel, grid_for(n, 256), 256, 0, S(stream), static_cast<const uint4*>(src), lds / 8,
                                                      static_cast<uint4*>(dst), rows, peers, width / 8);
  return check_launch("pack_kernel");
}

extern "C" sp_status sp_a2a_unpack(const void* src, void* dst, int64_t ldd, int rows, int peers,
                                   int width, void* stream) {
  if (rows < 0 || peers <= 0 || width <= 0 || width % 8 || ldd % 8)
    return fail(kInvalid, "a2a_unpack: width and stride must be multiples of 8");
  if (rows == 0) return kOk;
  const int64_t n = (int64_t)rows * peers * (width / 8);
  launch_k(unpack_kernel, grid_for(n, 256), 256, 0, S(stream), static_cast<const uint4*>(src),
                                                        static_cast<uint4*>(dst), ldd / 8, rows,
                                                        peers, width / 8);
  return check_launch("unpack_kernel");
}

extern "C" sp_status sp_add_f32(const float* a, const float* b, float* dst, int64_t n, void* stream) {
  if (n < 0) return fail(kInvalid, "add_f32: n < 0");
  if (n == 0) return kOk;
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
       reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(kInvalid, "add_f32: pointers must be 16-byte aligned");
  const int64_t n4 = n / 4;
  if (n4) launch_k(add_f32_kernel, grid_for(n4, 256), 256, 0, S(stream), reinterpret_cast<const float4*>(a), reinterpret_cast<const float4*>(b),
      reinterpret_cast<float4*>(dst), n4);
  if (n % 4) launch_k(add_f32_tail_kernel, 1, 32, 0, S(stream), a, b, dst, n4 * 4, n);
  return check_launch("add_f32_kernel");
}

extern "C" sp_status sp_argmax(const float* logits, int64_t ld, int rows, int vocab, int32_t* idx,
                               float* val, void* stream) {
  if (rows < 0 || vocab <= 0) return fail(kInvalid, "argmax: bad shape");
  if (rows == 0) return kOk;
  launch_k(argmax_kernel, rows, 1024, 0, S(stream), logits, ld, vocab, idx, val);
  return check_launch("argmax_kernel");
}

extern "C" sp_status sp_gather_rows_f32(const float* src, int64_t lds, const int32_t* idx, float* dst,
                                        int64_t ldd, int rows, int width, void* stream) {
  if (rows < 0 || width <= 0) return fail(kInvalid, "gather_rows: bad shape");
  if (rows == 0) return kOk;
  launch_k(gather_rows_kernel, rows, 256, 0, S(stream), src, lds, idx, dst, ldd, width);
  return check_launch("gather_rows_kernel");
}

// ------------------------------------------ operator-level drop-in kernels
// The reference's primitive API (tensor_core.py:105-132) as device kernels for
// paper_2507_11830_b200.tensor_core: f32 in, f32 out, one row per block.
__global__ void rms_norm_f32_kernel(const float* __restrict__ x, int64_t ldx,
                                    const float* __restrict__ gain, float eps,
                                    float* __restrict__ out, int64_t ldo, int hidden) {
  __shared__ float red[32];
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  const float* row = x + (int64_t)blockIdx.x * ldx;
  float s = 0.f;
  for (int c = threadIdx.x; c < hidden; c += blockDim.x) s += row[c] * row[c];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float den = sqrtf(red[0] / (float)hidden + eps);  // gain * (x / sqrt(mean + eps))
  float* o = out + (int64_t)blockIdx.x * ldo;
  for (int c = threadIdx.x; c < hidden; c += blockDim.x) o[c] = gain[c] * (row[c] / den);
}

__global__ void gelu_f32_kernel(const float* __restrict__ x, float* __restrict__ out, int64_t n) {
  const float c = 0.7978845608028654f, k = 0.044715f;  // sqrt(2/pi), tanh-form GeLU
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    out[i] = 0.5f * v * (1.f + tanhf(c * (v + k * v * v * v)));
  }
}

__global__ void softmax_rows_f32_kernel(const float* __restrict__ x, int64_t ldx,
                                        float* __restrict__ out, int64_t ldo, int width) {
  __shared__ float red[32];
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  const float* row = x + (int64_t)blockIdx.x * ldx;
  float* o = out + (int64_t)blockIdx.x * ldo;
  const int w = blockDim.x >> 5, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float m = -INFINITY;
  for (int c = threadIdx.x; c < width; c += blockDim.x) m = fmaxf(m, row[c]);
#pragma unroll
  for (int s = 16; s; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = -INFINITY;
  for (int i = 0; i < w; ++i) m = fmaxf(m, red[i]);
  __syncthreads();
  float sum = 0.f;
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    const float e = expf(row[c] - m);  // -inf entries (masked keys) -> 0
    o[c] = e;
    sum += e;
  }
#pragma unroll
  for (int s = 16; s; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  sum = 0.f;
  for (int i = 0; i < w; ++i) sum += red[i];
  for (int c = threadIdx.x; c < width; c += blockDim.x) o[c] = o[c] / sum;
}

extern "C" sp_status sp_rms_norm_f32(const float* x, int64_t ldx, const float* gain, float eps,
                                     float* out, int64_t ldo, int rows, int hidden, void* stream) {
  if (rows < 0 || hidden <= 0 || ldx < hidden || ldo < hidden)
    return fail(kInvalid, "rms_norm_f32: bad shape");
  if (rows == 0) return kOk;
  if (!x || !gain || !out) return fail(kInvalid, "rms_norm_f32: null pointer");
  launch_k(rms_norm_f32_kernel, rows, 256, 0, S(stream), x, ldx, gain, eps, out, ldo, hidden);
  return check_launch("rms_norm_f32_kernel");
}

extern "C" sp_status sp_gelu_f32(const float* x, float* out, int64_t n, void* stream) {
  if (n < 0) return fail(kInvalid, "gelu_f32: n < 0");
  if (n == 0) return kOk;
  if (!x || !out) return fail(kInvalid, "gelu_f32: null pointer");
  launch_k(gelu_f32_kernel, grid_for(n, 256), 256, 0, S(stream), x, out, n);
  return check_launch("gelu_f32_kernel");
}

extern "C" sp_status sp_softmax_rows_f32(const float* x, int64_t ldx, float* out, int64_t ldo,
                                         int rows, int width, void* stream) {
  if (rows < 0 || width <= 0 || ldx < width || ldo < width)
    return fail(kInvalid, "softmax_rows_f32: bad shape");
  if (rows == 0) return kOk;
  if (!x || !out) return fail(kInvalid, "softmax_rows_f32: null pointer");
  launch_k(softmax_rows_f32_kernel, rows, 256, 0, S(stream), x, ldx, out, ldo, width);
  return check_launch("softmax_rows_f32_kernel");
}

__global__ void add_f64_kernel(const double* __restrict__ a, const double* __restrict__ b,
                               double* __restrict__ d, int64_t n) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = a[i] + b[i];
}

extern "C" sp_status sp_add_f64(const double* a, const double* b, double* dst, int64_t n,
                                void* stream) {
  if (n < 0) return fail(kInvalid, "add_f64: n < 0");
  if (n == 0) return kOk;
  if (!a || !b || !dst) return fail(kInvalid, "add_f64: null pointer");
  launch_k(add_f64_kernel, grid_for(n, 256), 256, 0, S(stream), a, b, dst, n);
  return check_launch("add_f64_kernel");
}

__global__ void gather_rows_u16_kernel(const uint16_t* __restrict__ src, int64_t lds,
                                       const int32_t* __restrict__ idx, uint16_t* __restrict__ dst,
                                       int64_t ldd, int width) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  const uint16_t* s = src + (int64_t)idx[blockIdx.x] * lds;
  uint16_t* d = dst + (int64_t)blockIdx.x * ldd;
  for (int c = threadIdx.x; c < width; c += blockDim.x) d[c] = s[c];
}

extern "C" sp_status sp_gather_rows_bf16(const void* src, int64_t lds, const int32_t* idx,
                                         void* dst, int64_t ldd, int rows, int width,
                                         void* stream) {
  if (rows < 0 || width <= 0) return fail(kInvalid, "gather_rows_bf16: bad shape");
  if (rows == 0) return kOk;
  launch_k(gather_rows_u16_kernel, rows, 256, 0, S(stream), static_cast<const uint16_t*>(src), lds,
           idx, static_cast<uint16_t*>(dst), ldd, width);
  return check_launch("gather_rows_u16_kernel");
}

// Step timeline (debug builds only, see common.cuh): bind the record buffer
// (StepTraceRec[cap], 32 B each) and its 32-bit record counter in every
// translation unit; cap 0 / NULL buffer unbinds.
extern "C" sp_status sp_step_trace_bind(void* buf, void* counter, int cap) {
#ifdef STEP_TRACE
  if (cap < 0 || (cap > 0 && (buf == nullptr || counter == nullptr)))
    return sp::fail(sp::kInvalid, "step_trace_bind: buffer, counter and cap >= 0 required");
  for (auto f : sp::step_trace_registry()) f(cap > 0 ? buf : nullptr, counter, cap);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return sp::fail(sp::kCuda, std::string("step_trace_bind: ") + cudaGetErrorString(e));
  return sp::kOk;
#else
  (void)buf;
  (void)counter;
  (void)cap;
  return sp::fail(sp::kUnsupported, "step_trace_bind: library built without -DSTEP_TRACE");
#endif
}
