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

#include <array>
#include <map>
#include <mutex>

#include "../../include/shiftpar.h"
#include "common.cuh"

namespace sp {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, ACC_STAGES = 2;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;
constexpr int NUM_THREADS = 192;
constexpr int GROUP_M = 16;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;

struct Params {
  int M, N, K;
  int num_m, num_n, num_tiles, k_blocks;
  int epi;
  int a_kchunk;
  void* D;
  int64_t ldd;
  int64_t peer_width, peer_stride;
};

__device__ __forceinline__ void tile_coords(int t, const Params& p, int& mb, int& nb) {
  const int per_group = GROUP_M * p.num_n;
  const int g = t / per_group;
  const int first_m = g * GROUP_M;
  const int gm = min(p.num_m - first_m, GROUP_M);
  const int r = t - g * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

__device__ __forceinline__ float gelu_tanh(float x) {
  const float c = 0.7978845608028654f, k = 0.044715f;
  return 0.5f * x * (1.f + tanhf(c * (x + k * x * x * x)));
}

__device__ __forceinline__ float silu(float x) { return x / (1.f + __expf(-x)); }

// one thread: 32 consecutive columns [n0, n0+32) of row m
__device__ __forceinline__ void store_chunk(const Params& p, int m, int n0, const float (&v)[32],
                                            int epi, int N) {
  if (m >= p.M || n0 >= N) return;
  const int ncols = min(32, N - n0);
  int64_t col = n0;
  int64_t base = 0;
  if (p.peer_width > 0) {
    const int64_t peer = n0 / p.peer_width;
    col = n0 - peer * p.peer_width;
    base = peer * p.peer_stride;
  }
  if (epi == SP_EPI_STORE_BF16 || epi == SP_EPI_GELU) {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.D) + base + (int64_t)m * p.ldd + col;
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
    float* dst = reinterpret_cast<float*>(p.D) + base + (int64_t)m * p.ldd + col;
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

__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const Params p) {
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
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, p, mb, nb);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(full + stage, STAGE_BYTES);
          const int k = kb * BK;
          int ko = 0, kc = k;
          if (p.a_kchunk > 0) {
            ko = k / p.a_kchunk;
            kc = k - ko * p.a_kchunk;
          }
          tma_load_3d(sa, &tmA, full + stage, kc, mb * BM, ko);
          tma_load_2d(sa + A_BYTES, &tmB, full + stage, k, nb * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
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
        mbar_wait(tempty + acc, aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            umma_bf16(d_tmem, sdesc_sw128(a_addr + k * 32), sdesc_sw128(b_addr + k * 32), idesc,
                      (kb | k) != 0 ? 1u : 0u);
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
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, p, mb, nb);
      mbar_wait(tfull + acc, aphase);
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      const int m = mb * BM + row;
      if (p.epi == SP_EPI_SWIGLU) {
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

// ------------------------------------------------------------------ host side
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

// bf16 tiled map with 128-byte swizzle; dims/strides innermost first
int get_map(CUtensorMap* out, const void* ptr, int rank, const uint64_t* dims,
                   const uint64_t* strides, const uint32_t* box) {
  std::array<uint64_t, 12> key{};
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
  CUresult r = g_encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr),
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

extern "C" sp_status sp_gemm_bf16(const void* A, int64_t lda, int64_t a_kchunk,
                                  int64_t a_chunk_stride, const void* B, int64_t ldb, void* D,
                                  int64_t ldd, int M, int N, int K, int epilogue,
                                  int64_t peer_width, int64_t peer_stride, void* stream) {
  using namespace sp::gemm;
  if (M < 0 || N <= 0 || K <= 0) return fail(kInvalid, "gemm: bad M/N/K");
  if (M == 0) return kOk;
  if (!A || !B || !D) return fail(kInvalid, "gemm: null pointer");
  if (epilogue < SP_EPI_STORE_BF16 || epilogue > SP_EPI_GELU)
    return fail(kInvalid, "gemm: unknown epilogue");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15)
    return fail(kInvalid, "gemm: A/B must be 16-byte aligned");
  if (lda % 8 || ldb % 8 || ldd % 8) return fail(kInvalid, "gemm: leading dims must be multiples of 8");
  if (a_kchunk > 0 && (a_kchunk % BK || K % a_kchunk || a_chunk_stride % 8))
    return fail(kUnsupported, "gemm: chunked-K A needs chunk % 64 == 0 and K % chunk == 0");
  if (epilogue == SP_EPI_SWIGLU && N % BN)
    return fail(kUnsupported, "gemm: SwiGLU epilogue needs N % 256 == 0");
  if (peer_width > 0 && (peer_width % 32 || peer_stride % 8))
    return fail(kUnsupported, "gemm: peer layout needs width % 32 == 0");
  if (reinterpret_cast<uintptr_t>(D) & 15) return fail(kInvalid, "gemm: D must be 16-byte aligned");

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
    uint32_t box[2] = {BK, BN};
    if (int rc = get_map(&tb, B, 2, dims, strides, box)) return rc;
  }
  Params p;
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

  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  const int grid = std::min(p.num_tiles, sm_count());
  gemm_kernel<<<grid, NUM_THREADS, SMEM_BYTES, reinterpret_cast<cudaStream_t>(stream)>>>(ta, tb, p);
  return check_launch("gemm_kernel");
}
