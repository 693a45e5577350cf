// Fused SP all-to-all over peer memory (NVLink P2P stores, no NCCL on the data
// path).  The seq->head exchange is fused into the QKV GEMM epilogue
// (sp_gemm_bf16_to_peers); the head->seq exchange is a vectorised scatter of
// attention rows straight into each owner's receive buffer.  Completion uses
// one flag per (receiver, sender): the sender's signal kernel publishes with a
// system-scope release after its stores, the receiver's wait kernel acquires
// all P flags and resets them (reset-on-consume keeps the protocol valid under
// CUDA-graph replay; the SP data dependences order the next signal after the
// reset).  In-process (loopback) ranks use the same kernels on one GPU.
#include <cuda.h>
#include <cstring>
#include <string>

#include "../../include/shiftpar.h"
#define SP_TU_ID 5  // step-trace tag (common.cuh)
#include "common.cuh"

namespace sp {

__global__ void peer_scatter_kernel(const uint4* __restrict__ src, int64_t lds_v, int rows_total,
                                    int peers, int my_rank, int width_v,
                                    const unsigned long long* __restrict__ dst_ptrs) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  const int base = rows_total / peers, rem = rows_total % peers;
  const int64_t n = (int64_t)rows_total * width_v;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / width_v);
    const int c = (int)(i % width_v);
    // owner of global row t under the contiguous split (remainder to low ranks)
    const int edge = rem * (base + 1);
    int s, lo, rows;
    if (t < edge) {
      s = t / (base + 1);
      lo = s * (base + 1);
      rows = base + 1;
    } else {
      s = rem + (t - edge) / base;
      lo = edge + (s - rem) * base;
      rows = base;
    }
    uint4* dst = reinterpret_cast<uint4*>(dst_ptrs[s]);
    dst[((int64_t)my_rank * rows + (t - lo)) * width_v + c] = src[(int64_t)t * lds_v + c];
  }
}

__global__ void peer_signal_kernel(const unsigned long long* __restrict__ flag_ptrs, int peers,
                                   int my_rank) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  if (threadIdx.x < (unsigned)peers) {
    int* f = reinterpret_cast<int*>(flag_ptrs[threadIdx.x]) + my_rank;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(1) : "memory");
  }
}

__global__ void peer_wait_kernel(int* flags, int peers) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  if (threadIdx.x < (unsigned)peers) {
    int v = 0;
    do {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + threadIdx.x) : "memory");
    } while (v == 0);
    flags[threadIdx.x] = 0;
  }
  __syncthreads();
}

// One-shot TP all-reduce fused with the residual add and RMSNorm: every rank's
// O/down GEMM wrote its f32 partial into its own peer-visible buffer; this
// kernel sums the P partials of its row in ascending rank order (the order of
// DeviceGroup.all_reduce_sum, fabric.py:117-143), adds them to the residual x
// and (if out != NULL) writes bf16( gain * x / sqrt(mean(x^2) + eps) ).
template <int VEC>
__global__ void peer_allreduce_norm_kernel(const unsigned long long* __restrict__ part_ptrs,
                                           int peers, int slabs, int64_t slab_stride,
                                           float* __restrict__ x, int64_t ldx,
                                           const float* __restrict__ gain, float eps,
                                           __nv_bfloat16* __restrict__ out, int64_t ldo,
                                           int hidden) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  const int r = blockIdx.x;
  float* xr = x + (int64_t)r * ldx;
  float v[VEC * 4];
  float ssq[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < hidden) {
      // rank partial = its K-split slabs summed in ascending order (what the
      // GEMM's own split-K reduce would have written); ranks in ascending order
      float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < peers; ++s) {
        const float* base = reinterpret_cast<const float*>(part_ptrs[s]) + (int64_t)r * hidden + c;
        float4 q = *reinterpret_cast<const float4*>(base);
        for (int k = 1; k < slabs; ++k) {
          const float4 b = *reinterpret_cast<const float4*>(base + k * slab_stride);
          q.x += b.x;
          q.y += b.y;
          q.z += b.z;
          q.w += b.w;
        }
        if (s == 0) {
          sum = q;
        } else {
          sum.x += q.x;
          sum.y += q.y;
          sum.z += q.z;
          sum.w += q.w;
        }
      }
      t = *reinterpret_cast<const float4*>(xr + c);
      t.x += sum.x;
      t.y += sum.y;
      t.z += sum.z;
      t.w += sum.w;
      *reinterpret_cast<float4*>(xr + c) = t;
    }
    v[4 * i + 0] = t.x;
    v[4 * i + 1] = t.y;
    v[4 * i + 2] = t.z;
    v[4 * i + 3] = t.w;
    ssq[i] = norm_sq4(t);
  }
  if (out == nullptr) return;
  __shared__ float red[256];
  const float den = norm_den(rms_chunk_sum<VEC>(ssq, hidden, red), hidden, eps);
  __nv_bfloat16* orow = out + (int64_t)r * ldo;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    if (c < hidden) {
      const float4 g = *reinterpret_cast<const float4*>(gain + c);
      const uint2 u = norm_pack4(g, v[4 * i + 0], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3], den);
      *reinterpret_cast<uint2*>(orow + c) = u;
    }
  }
}

// Two-shot TP all-reduce for prefill-size passes (reduce-scatter + all-gather
// over the same peer buffers): rank r owns rows [lo, hi) of the contiguous
// split (remainder to low ranks, flops.py:68-80); for each owned row it sums
// the P partials in ascending rank order (exactly the one-shot sum), adds them
// into its residual row, normalises, and PUSHES the bf16 normed row into every
// rank's xn buffer (NVLink stores).  Per rank: reads (P-1)/P*M*h*4 bytes of
// peer partials and writes (P-1)/P*M*h*2, vs (P-1)*M*h*4 reads one-shot.  The
// residual stays row-sharded between reductions (only the owner reads a row
// again), so no f32 all-gather is needed; the final reduction pushes the
// final-normed rows the LM head needs.
template <int VEC>
__global__ void peer_reduce_scatter_norm_kernel(const unsigned long long* __restrict__ part_ptrs,
                                                int peers, int row_lo, float* __restrict__ x,
                                                int64_t ldx, const float* __restrict__ gain,
                                                float eps,
                                                const unsigned long long* __restrict__ xn_ptrs,
                                                int64_t ldo, int hidden) {
  pdl_trigger();  // successors may launch now: they wait for this grid before reading its outputs
  pdl_wait();
  const int r = row_lo + blockIdx.x;
  float* xr = x + (int64_t)r * ldx;
  float v[VEC * 4];
  float ssq[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < hidden) {
      float4 sum = *reinterpret_cast<const float4*>(
          reinterpret_cast<const float*>(part_ptrs[0]) + (int64_t)r * hidden + c);
      for (int s = 1; s < peers; ++s) {
        const float4 q = *reinterpret_cast<const float4*>(
            reinterpret_cast<const float*>(part_ptrs[s]) + (int64_t)r * hidden + c);
        sum.x += q.x;
        sum.y += q.y;
        sum.z += q.z;
        sum.w += q.w;
      }
      t = *reinterpret_cast<const float4*>(xr + c);
      t.x += sum.x;
      t.y += sum.y;
      t.z += sum.z;
      t.w += sum.w;
      *reinterpret_cast<float4*>(xr + c) = t;
    }
    v[4 * i + 0] = t.x;
    v[4 * i + 1] = t.y;
    v[4 * i + 2] = t.z;
    v[4 * i + 3] = t.w;
    ssq[i] = norm_sq4(t);
  }
  __shared__ float red[256];
  const float den = norm_den(rms_chunk_sum<VEC>(ssq, hidden, red), hidden, eps);
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    if (c < hidden) {
      const float4 g = *reinterpret_cast<const float4*>(gain + c);
      const uint2 u = norm_pack4(g, v[4 * i + 0], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3], den);
      for (int s = 0; s < peers; ++s)
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(xn_ptrs[s]) +
                                  (int64_t)r * ldo + c) = u;
    }
  }
}

}  // namespace sp

using namespace sp;

extern "C" sp_status sp_peer_reduce_scatter_rmsnorm(const unsigned long long* part_ptrs, int peers,
                                                    int my_rank, float* x, int64_t ldx,
                                                    const float* gain, float eps,
                                                    const unsigned long long* xn_ptrs,
                                                    int64_t ldo, int rows, int hidden,
                                                    void* stream) {
  if (!part_ptrs || !xn_ptrs || !gain || peers < 1 || my_rank < 0 || my_rank >= peers ||
      rows < 0 || hidden <= 0 || hidden % 4 || ldx % 4 || ldo % 4)
    return fail(kInvalid, "peer_reduce_scatter_rmsnorm: bad arguments");
  const int base = rows / peers, rem = rows % peers;
  const int lo = my_rank * base + (my_rank < rem ? my_rank : rem);
  const int mine = base + (my_rank < rem ? 1 : 0);
  if (mine == 0) return kOk;
  const int threads = norm_block_threads(mine, hidden);
  const int per = (hidden + threads * 4 - 1) / (threads * 4);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (per) {
    case 1: launch_k(peer_reduce_scatter_norm_kernel<1>, mine, threads, 0, st, part_ptrs, peers, lo, x, ldx, gain, eps, xn_ptrs, ldo, hidden); break;
    case 2: launch_k(peer_reduce_scatter_norm_kernel<2>, mine, threads, 0, st, part_ptrs, peers, lo, x, ldx, gain, eps, xn_ptrs, ldo, hidden); break;
    case 3: case 4: launch_k(peer_reduce_scatter_norm_kernel<4>, mine, threads, 0, st, part_ptrs, peers, lo, x, ldx, gain, eps, xn_ptrs, ldo, hidden); break;
    case 5: case 6: case 7: case 8: launch_k(peer_reduce_scatter_norm_kernel<8>, mine, threads, 0, st, part_ptrs, peers, lo, x, ldx, gain, eps, xn_ptrs, ldo, hidden); break;
    default: return fail(kUnsupported, "peer_reduce_scatter_rmsnorm: hidden > 8192");
  }
  return check_launch("peer_reduce_scatter_norm_kernel");
}

extern "C" sp_status sp_peer_allreduce_add_rmsnorm(const unsigned long long* part_ptrs, int peers,
                                                   int slabs, float* x, int64_t ldx,
                                                   const float* gain, float eps, void* out_bf16,
                                                   int64_t ldo, int rows, int hidden,
                                                   void* stream) {
  if (!part_ptrs || peers < 1 || slabs < 1 || rows < 0 || hidden <= 0 || hidden % 4 || ldx % 4 ||
      ldo % 4)
    return fail(kInvalid, "peer_allreduce_add_rmsnorm: bad arguments");
  if (out_bf16 && !gain) return fail(kInvalid, "peer_allreduce_add_rmsnorm: gain needed with out");
  if (rows == 0) return kOk;
  const int64_t slab_stride = (int64_t)rows * hidden;
  const int threads = norm_block_threads(rows, hidden);
  const int per = (hidden + threads * 4 - 1) / (threads * 4);
  auto out = static_cast<__nv_bfloat16*>(out_bf16);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (per) {
    case 1: launch_k(peer_allreduce_norm_kernel<1>, rows, threads, 0, st, part_ptrs, peers, slabs, slab_stride, x, ldx, gain, eps, out, ldo, hidden); break;
    case 2: launch_k(peer_allreduce_norm_kernel<2>, rows, threads, 0, st, part_ptrs, peers, slabs, slab_stride, x, ldx, gain, eps, out, ldo, hidden); break;
    case 3: case 4: launch_k(peer_allreduce_norm_kernel<4>, rows, threads, 0, st, part_ptrs, peers, slabs, slab_stride, x, ldx, gain, eps, out, ldo, hidden); break;
    case 5: case 6: case 7: case 8: launch_k(peer_allreduce_norm_kernel<8>, rows, threads, 0, st, part_ptrs, peers, slabs, slab_stride, x, ldx, gain, eps, out, ldo, hidden); break;
    default: return fail(kUnsupported, "peer_allreduce_add_rmsnorm: hidden > 8192");
  }
  return check_launch("peer_allreduce_norm_kernel");
}

extern "C" sp_status sp_peer_scatter_rows(const void* src, int64_t lds, int rows_total, int width,
                                          int peers, int my_rank,
                                          const unsigned long long* dst_ptrs, void* stream) {
  if (rows_total < 0 || width <= 0 || width % 8 || lds % 8 || peers < 1 || my_rank < 0 ||
      my_rank >= peers || !dst_ptrs)
    return fail(kInvalid, "peer_scatter_rows: bad arguments");
  if (rows_total == 0) return kOk;
  const int64_t n = (int64_t)rows_total * (width / 8);
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  launch_k(peer_scatter_kernel, (unsigned)g, 256, 0, reinterpret_cast<cudaStream_t>(stream),
           static_cast<const uint4*>(src), lds / 8, rows_total, peers, my_rank, width / 8, dst_ptrs);
  return check_launch("peer_scatter_kernel");
}

extern "C" sp_status sp_peer_signal(const unsigned long long* flag_ptrs, int peers, int my_rank,
                                    void* stream) {
  if (!flag_ptrs || peers < 1 || peers > 1024 || my_rank < 0 || my_rank >= peers)
    return fail(kInvalid, "peer_signal: bad arguments");
  launch_k(peer_signal_kernel, 1, 32 * ((peers + 31) / 32), 0, reinterpret_cast<cudaStream_t>(stream),
           flag_ptrs, peers, my_rank);
  return check_launch("peer_signal_kernel");
}

extern "C" sp_status sp_peer_wait(int* flags, int peers, void* stream) {
  if (!flags || peers < 1 || peers > 1024) return fail(kInvalid, "peer_wait: bad arguments");
  launch_k(peer_wait_kernel, 1, 32 * ((peers + 31) / 32), 0, reinterpret_cast<cudaStream_t>(stream),
           flags, peers);
  return check_launch("peer_wait_kernel");
}

// ------------------------------------------------------------------ CUDA IPC
// Cross-process peer buffers (one process per GPU under torchrun): export the
// allocation holding `ptr` (offset kept separately, since the caching
// allocator hands out interior pointers), import a peer's, close an import.
typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

extern "C" sp_status sp_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return fail(kInvalid, "ipc_export: null argument");
  static PFN_memGetAddressRange range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        !fn)
      return fail(kCuda, "cuMemGetAddressRange entry point unavailable");
    range = reinterpret_cast<PFN_memGetAddressRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(kCuda, "ipc_export: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(kCuda, std::string("ipc_export: ") + cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uintptr_t>(ptr) - static_cast<uintptr_t>(base);
  return kOk;
}

extern "C" sp_status sp_ipc_import(const void* handle, int64_t offset, void** ptr_out) {
  if (!handle || !ptr_out || offset < 0) return fail(kInvalid, "ipc_import: bad argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(kCuda, std::string("ipc_import: ") + cudaGetErrorString(e));
  *ptr_out = static_cast<uint8_t*>(base) + offset;
  return kOk;
}
