// Microbenchmark: the HBM read ceiling for the decode weight streams.
// Each CTA streams a contiguous slice of a 2 GiB buffer (> L2) into a shared-
// memory ring with 1-D bulk copies (cp.async.bulk, mbarrier completion), the
// way the swap-AB decode GEMM's producer streams weight boxes, optionally with
// the L2 evict-first hint; the consumer thread only re-arms the stage.  Also
// an LDG.128 read kernel (all threads, sum folded into one store).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu -lcuda && ./read_bw
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <bool HINT>
__global__ void bulk_read(const uint8_t* src, size_t bytes_per_cta, int stage_bytes, int stages,
                          unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint8_t* base = src + (size_t)blockIdx.x * bytes_per_cta;
  const size_t n = bytes_per_cta / stage_bytes;
  uint32_t phase[32] = {0};
  unsigned long long acc = 0;
  auto issue = [&](size_t i) {
    const int s = (int)(i % stages);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)),
                 "r"(stage_bytes));
    if (HINT)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              su32(smem + (size_t)s * stage_bytes)),
          "l"(base + i * stage_bytes), "r"(stage_bytes), "r"(su32(full + s)), "l"(pol)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su32(smem + (size_t)s * stage_bytes)),
          "l"(base + i * stage_bytes), "r"(stage_bytes), "r"(su32(full + s))
          : "memory");
  };
  for (size_t i = 0; i < (size_t)stages && i < n; ++i) issue(i);
  for (size_t i = 0; i < n; ++i) {
    const int s = (int)(i % stages);
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(su32(full + s)), "r"(phase[s]));
    phase[s] ^= 1;
    acc += smem[(size_t)s * stage_bytes];
    if (i + stages < n) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// The decode attention's pattern: per 64-key page slice, four 2-D tensor-map
// boxes of [64 rows][64 bf16] (128-B swizzle): K columns 0-63 / 64-127 and the
// same for V, from a paged pool [blocks][kv_heads][64][128] bf16 where one
// CTA walks its (item, head)'s pages (pages of a sequence are consecutive
// blocks, so one head's pages sit kv_heads * 16 KB apart).
__global__ void tmap_read(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                          int pages_per_cta, int kv_heads, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int seq = blockIdx.x / kv_heads, head = blockIdx.x % kv_heads;
  uint32_t phase[32] = {0};
  unsigned long long acc = 0;
  auto issue = [&](int i) {
    const int s = i % stages;
    const int row = ((seq * pages_per_cta + i) * kv_heads + head) * 64;
    uint8_t* st = smem + (size_t)s * stage_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(stage_bytes));
    const CUtensorMap* maps[2] = {&tk, &tv};
    for (int kv = 0; kv < 2; ++kv)
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(su32(st + kv * 16384 + h * 8192)),
            "l"(maps[kv]), "r"(su32(full + s)), "r"(h * 64), "r"(row), "l"(pol)
            : "memory");
  };
  for (int i = 0; i < stages && i < pages_per_cta; ++i) issue(i);
  for (int i = 0; i < pages_per_cta; ++i) {
    const int s = i % stages;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(su32(full + s)), "r"(phase[s]));
    phase[s] ^= 1;
    acc += smem[(size_t)s * stage_bytes];
    if (i + stages < pages_per_cta) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

__global__ void ldg_read(const uint4* src, size_t n16, unsigned long long* sink) {
  uint32_t a = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src + i));
    a ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (a == 0xdeadbeef) *sink = a;
}

int main() {
  const size_t total = (size_t)2 << 30;
  uint8_t* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, total);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int cps, stage, stages; bool hint; };
  const Cfg cfgs[] = {{1, 32768, 6, false}, {1, 32768, 6, true},  {2, 32768, 3, true},
                      {2, 36864, 3, true},  {1, 16384, 12, true}, {2, 16384, 6, true},
                      {3, 32768, 2, true},  {4, 16384, 3, true},  {1, 65536, 3, true},
                      {2, 65536, 1, true},  {4, 32768, 1, true},  {8, 16384, 1, true}};
  for (const Cfg& c : cfgs) {
    const int ctas = sms * c.cps;
    size_t per = total / ctas / c.stage * c.stage;
    const int smem = c.stage * c.stages + 64 * 8;
    auto k = c.hint ? bulk_read<true> : bulk_read<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      k<<<ctas, 32, smem>>>(buf, per, c.stage, c.stages, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("bulk  ctas/SM %d stage %6d B x %2d (%3d KB in flight/SM) hint %d: %7.1f GB/s %s\n", c.cps,
           c.stage, c.stages, c.cps * c.stage * c.stages / 1024, (int)c.hint,
           (double)per * ctas / (best * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  // decode-GEMM-sized streams: 235 MB (8B gate/up weights) per launch,
  // rotating over 8 such slices of the buffer (nothing L2-resident), as
  // C CTAs with equal bytes each
  {
    const size_t slice = (size_t)28672 * 4096 * 2;
    struct Sh { int ctas, stage, stages; };
    const Sh shs[] = {{224, 36864, 3}, {296, 36864, 3}, {148, 36864, 6}, {296, 32768, 3},
                      {592, 16384, 3}, {444, 24576, 3}};
    for (const Sh& c : shs) {
      size_t per = slice / c.ctas / c.stage * c.stage;
      const int smem = c.stage * c.stages + 64 * 8;
      cudaFuncSetAttribute(bulk_read<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int w = 0; w < 8; ++w)
        bulk_read<true><<<c.ctas, 32, smem>>>(buf + (size_t)w * slice, per, c.stage, c.stages, sink);
      cudaEventRecord(e0);
      const int reps = 64;
      for (int r = 0; r < reps; ++r)
        bulk_read<true><<<c.ctas, 32, smem>>>(buf + (size_t)(r % 8) * slice, per, c.stage, c.stages, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      printf("235MB %3d CTAs x %6zu B (ring %d x %d): %6.1f us/launch  %7.1f GB/s\n", c.ctas, per,
             c.stages, c.stage, us, (double)per * c.ctas / (us * 1e-6) / 1e9);
    }
  }
  // decode-attention-sized streams: B=64 x 8 kv heads x ctx 2048 = 512 (item,
  // head) pairs of 1 MiB K+V each (537 MB per launch), rotating over 3 slices
  {
    const size_t slice = (size_t)512 << 20;
    struct Sh { int ctas, stage, stages, smem_pad; };
    const Sh shs[] = {{512, 32768, 3, 0}, {512, 32768, 3, 100000}, {512, 16384, 3, 0},
                      {1024, 32768, 3, 0}, {296, 32768, 3, 0}, {592, 32768, 3, 0}};
    for (const Sh& c : shs) {
      size_t per = slice / c.ctas / c.stage * c.stage;
      const int smem = c.stage * c.stages + 64 * 8 + c.smem_pad;
      cudaFuncSetAttribute(bulk_read<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int w = 0; w < 3; ++w)
        bulk_read<true><<<c.ctas, 32, smem>>>(buf + (size_t)w * slice, per, c.stage, c.stages, sink);
      cudaEventRecord(e0);
      const int reps = 30;
      for (int r = 0; r < reps; ++r)
        bulk_read<true><<<c.ctas, 32, smem>>>(buf + (size_t)(r % 3) * slice, per, c.stage, c.stages, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      printf("512MB %4d CTAs x %7zu B (ring %d x %d, smem %d): %6.1f us/launch  %7.1f GB/s\n", c.ctas, per,
             c.stages, c.stage, smem, us, (double)per * c.ctas / (us * 1e-6) / 1e9);
    }
  }
  // the decode attention's access pattern (tensor maps over a paged pool)
  {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    const int kv_heads = 8, seqs = 64, pages = 32;  // B=64, ctx 2048, 8 kv heads
    const uint64_t rows = (uint64_t)seqs * pages * kv_heads * 64;  // pool rows of 256 B
    const size_t pool_bytes = rows * 256;  // 268 MB each for K and V
    uint8_t* kbuf = buf;
    uint8_t* vbuf = buf + pool_bytes;
    CUtensorMap tk, tv;
    uint64_t dims[2] = {128, rows};
    uint64_t strides[1] = {256};
    uint32_t box[2] = {64, 64};
    uint32_t es[2] = {1, 1};
    enc(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kbuf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, vbuf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int stages : {3, 2}) {
      const int smem = stages * 32768 + 1024 + 256;
      cudaFuncSetAttribute(tmap_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int w = 0; w < 3; ++w) tmap_read<<<seqs * kv_heads, 32, smem>>>(tk, tv, pages, kv_heads, stages, sink);
      cudaEventRecord(e0);
      const int reps = 20;
      for (int r = 0; r < reps; ++r) tmap_read<<<seqs * kv_heads, 32, smem>>>(tk, tv, pages, kv_heads, stages, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      cudaError_t err = cudaGetLastError();
      printf("paged tmap 512 CTAs x 32 pages x 32 KB (ring %d): %6.1f us/launch  %7.1f GB/s %s\n", stages, us,
             2.0 * pool_bytes / (us * 1e-6) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
  }
  for (int tpb : {256, 512, 1024}) {
    for (int bps : {1, 2, 4, 8}) {
      if (tpb * bps > 2048) continue;
      float best = 1e30f;
      for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        ldg_read<<<sms * bps, tpb>>>(reinterpret_cast<const uint4*>(buf), total / 16, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("ldg   %4d thr x %d blocks/SM: %7.1f GB/s\n", tpb, bps, (double)total / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
