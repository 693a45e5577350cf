// Fused SP all-to-all over peer memory (NVLink P2P stores, no NCCL on the data
// path).  The seq->head exchange is fused into the QKV GEMM epilogue
// (sp_gemm_bf16_to_peers); the head->seq exchange is a vectorised scatter of
// attention rows straight into each owner's receive buffer.  Completion uses
// one flag per (receiver, sender): the sender's signal kernel publishes with a
// system-scope release after its stores, the receiver's wait kernel acquires
// all P flags and resets them (reset-on-consume keeps the protocol valid under
// CUDA-graph replay; the SP data dependences order the next signal after the
// reset).  In-process (loopback) ranks use the same kernels on one GPU.
#include "../../include/shiftpar.h"
#include "common.cuh"

namespace sp {

__global__ void peer_scatter_kernel(const uint4* __restrict__ src, int64_t lds_v, int rows_total,
                                    int peers, int my_rank, int width_v,
                                    const unsigned long long* __restrict__ dst_ptrs) {
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x < (unsigned)peers) {
    int* f = reinterpret_cast<int*>(flag_ptrs[threadIdx.x]) + my_rank;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(1) : "memory");
  }
}

__global__ void peer_wait_kernel(int* flags, int peers) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x < (unsigned)peers) {
    int v = 0;
    do {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + threadIdx.x) : "memory");
    } while (v == 0);
    flags[threadIdx.x] = 0;
  }
  __syncthreads();
}

}  // namespace sp

using namespace sp;

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
