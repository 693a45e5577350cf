// Microbenchmark: how much earlier does a consumer kernel see its producer's
// data through a release counter than through griddepcontrol.wait?
// Producer: G CTAs, each stores, fences and increments a counter, then exits.
// Consumer (PDL-launched): either waits griddepcontrol.wait, or polls the
// counter (acquire) until G arrivals.  globaltimer stamps: each producer CTA's
// last store, the consumer's release.  nvcc -arch=sm_100a -o pdl_vs_flag pdl_vs_flag.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long g_last_store;
__device__ unsigned long long g_release;
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
__global__ void producer(float* buf, unsigned* ctr, int work) {
  asm volatile("griddepcontrol.launch_dependents;");
  float v = blockIdx.x;
  for (int i = 0; i < work; ++i) v = v * 1.0001f + 0.5f;   // some busy work
  buf[blockIdx.x * blockDim.x + threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    atomicMax(&g_last_store, gt());
  }
}
__global__ void consumer(const float* buf, unsigned* ctr, int G, int mode, float* out) {
  if (mode == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  } else {
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < (unsigned)G);
  }
  if (threadIdx.x == 0) g_release = gt();
  out[threadIdx.x] = buf[threadIdx.x];
}
int main() {
  const int G = 148, T = 256;
  float *buf, *out; unsigned* ctr;
  cudaMalloc(&buf, G * T * 4); cudaMalloc(&out, 4096); cudaMalloc(&ctr, 4);
  cudaStream_t st; cudaStreamCreate(&st);
  for (int mode = 0; mode < 2; ++mode) {
    double acc = 0; int n = 0;
    for (int it = 0; it < 50; ++it) {
      cudaMemsetAsync(ctr, 0, 4, st);
      unsigned long long z = 0;
      cudaMemcpyToSymbolAsync(g_last_store, &z, 8, 0, cudaMemcpyHostToDevice, st);
      producer<<<G, T, 0, st>>>(buf, ctr, 20000);
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = 1; cfg.blockDim = 256; cfg.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, consumer, (const float*)buf, ctr, G, mode, out);
      cudaStreamSynchronize(st);
      unsigned long long a, b;
      cudaMemcpyFromSymbol(&a, g_last_store, 8); cudaMemcpyFromSymbol(&b, g_release, 8);
      if (it >= 10) { acc += (double)(b - a); ++n; }
    }
    printf("%s: release - last producer store = %.0f ns (mean of %d)\n",
           mode ? "flag poll" : "griddepcontrol.wait", acc / n, n);
  }
  return 0;
}
