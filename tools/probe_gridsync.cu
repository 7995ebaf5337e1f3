// Probe: cost of a software grid barrier with 148 persistent CTAs (variants).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/probe_gridsync tools/probe_gridsync.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int V>
__global__ void k_sync(unsigned* bar, int iters, float* sink) {
  unsigned gen = 0;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x * 0.001f;
    __syncthreads();
    if (threadIdx.x == 0) {
      ++gen;
      if (V == 0) {  // fence + atomicAdd + nanosleep spin + fence
        __threadfence();
        const unsigned arrived = atomicAdd(&bar[0], 1u) + 1;
        if (arrived == gen * gridDim.x) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen) : "memory");
        else while (ld_acquire(&bar[1]) < gen) __nanosleep(32);
        __threadfence();
      } else if (V == 1) {  // atom.add.release, tight acquire spin
        unsigned arrived;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
        if (arrived + 1 == gen * gridDim.x) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen) : "memory");
        else while (ld_acquire(&bar[1]) < gen) {}
      } else if (V == 2) {  // every CTA spins on the arrival counter itself (no release store)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_acquire(&bar[0]) < gen * gridDim.x) {}
      } else {  // two-level: groups of 16 arrive on their own counter (128-B apart), last of a group
                // arrives on the top counter; everyone polls the top counter with relaxed loads
        const unsigned grp = blockIdx.x / 16, ngrp = (gridDim.x + 15) / 16;
        const unsigned gsz = min(16u, gridDim.x - grp * 16);
        unsigned prev;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar + 32 + grp * 32) : "memory");
        if (prev + 1 == gen * gsz) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned seen;
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
        } while (seen < gen * ngrp);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  if (acc == 12345.f) sink[0] = acc;
}

template <int V>
float run(unsigned* bar, float* sink, int G) {
  cudaMemset(bar, 0, 4096 * 4);
  k_sync<V><<<G, 256>>>(bar, 10, sink);
  cudaMemset(bar, 0, 4096 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_sync<V><<<G, 256>>>(bar, 2000, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / 2000.f;
}

int main() {
  unsigned* bar;
  float* sink;
  cudaMalloc(&bar, 4096 * 4);
  cudaMalloc(&sink, 4);
  int G;
  cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
  printf("grid %d: v0 fence+atomic+nanosleep %.2f us, v1 atom.release+spin %.2f us, v2 counter spin %.2f us, "
         "v3 two-level %.2f us\n", G, run<0>(bar, sink, G), run<1>(bar, sink, G), run<2>(bar, sink, G),
         run<3>(bar, sink, G));
  return 0;
}
