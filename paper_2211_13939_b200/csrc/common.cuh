// Shared helpers for the incrtts_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#define ITTS_API extern "C" __attribute__((visibility("default")))

// Status codes (ITTS_OK / ITTS_E*) come from the public header: 0 = success,
// a positive cudaError_t for CUDA failures, ITTS_E* for argument errors
// detected before any launch (so nothing is enqueued on failure).
#include "incrtts_b200.h"

// bilstm_tc.cu: the encoder BiLSTM on the tensor cores (bf16-exact W_hh tiles), see itts_r_bilstm_tc.
int bilstm_tc_launch(const float* PRE, const int64_t* plan, int32_t n, const void* Wt, void* stream);

// tier_r.cu: several row maps (as itts_r_rowmap) in one launch (vocoder call setup, voc_run.cu).
int itts_r_rowmaps(int32_t count, const int64_t* const* plans, int32_t* const* outs, const int64_t* spans, int32_t n,
                   void* stream);

// tier_r.cu: itts_r_mrf_combine that also re-zeroes the halo rows of the NEXT stage's operand buffer
// (itts_r_zero_halo(zplan, zn, zhalo, zX, zC)) in the same launch (vocoder call, voc_run.cu).
int mrf_combine_zero_halo(const void* y0, const void* y1, const void* y2, int64_t n, float slope, void* out,
                          const int64_t* zplan, int32_t zn, int64_t zhalo, void* zX, int32_t zC, void* stream);

// tc_conv.cu: itts_conv1d_tc with a choice of act_out activation: 0 leaky ReLU (slope), 1 tanh
// (PostNet), 2 GELU tanh form (BERT frontend).
int conv1d_tc_impl(const void* x, int64_t rows, int32_t c_in, int64_t x_ld, const void* w, int32_t n_total,
                   int32_t n_taps, const int32_t* host_tap_off, const float* bias, int32_t c_out,
                   const int32_t* row_out, const void* res_in, float res_slope, float* f32_out, int32_t ksplit,
                   void* acc, int32_t acc_mode, void* act_out, float slope, int32_t zero_halo, int32_t bn,
                   int32_t act, void* stream);

#define ITTS_RETURN_LAUNCH()                        \
  do {                                              \
    cudaError_t _e = cudaGetLastError();            \
    return _e == cudaSuccess ? ITTS_OK : (int)_e;   \
  } while (0)

namespace itts {

// Bit of the calling thread's current device: one-time per-device setup (cudaFuncSetAttribute
// applies to the current device only) is tracked in a 64-bit mask per call site.
inline uint64_t device_bit() {
  int d = 0;
  cudaGetDevice(&d);
  return 1ull << (d & 63);
}

// Programmatic dependent launch (PDL): kernels of the vocoder / encoder chains can be launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's prologue (barrier init, TMEM
// allocation, tensor-map prefetch, weight loads) overlaps the tail of the kernel before it.
// Every kernel calls pdl_trigger() on entry (dependents may launch once all its CTAs started) and
// pdl_wait() before its first access to data a previous kernel produced or still reads.
// OFF by default: tools/race_check.py (deterministic serving replay) shows corrupted chunks when
// the ResBlock and conv kernels both run with PDL on one stream, which no single kernel class
// reproduces alone -- not yet understood.  ITTS_PDL_MASK=<classes> turns it on for A/B and for
// that investigation; ITTS_NO_PDL=1 forces it off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// kernel classes for ITTS_PDL_MASK (debug bisection): 1 ResBlock, 2 tc_conv, 4 small vocoder /
// encoder kernels, 8 BiLSTM, 16 BERT
enum PdlClass { PDL_RESBLOCK = 1, PDL_CONV = 2, PDL_SMALL = 4, PDL_BILSTM = 8, PDL_BERT = 16 };

inline bool pdl_enabled(int cls = 0xff) {
  static int mask = -1;
  if (mask < 0) {
    const char* e = getenv("ITTS_NO_PDL");
    const char* m = getenv("ITTS_PDL_MASK");
    mask = (e && e[0] == '1') ? 0 : (m ? atoi(m) : 0);
  }
  return (mask & cls) != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cls(int cls, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(cls) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  return launch_pdl_cls(PDL_SMALL, kernel, grid, block, smem, st, std::forward<Args>(args)...);
}


template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reduction; `scratch` holds >= 32 T.  Result broadcast to all.
template <typename T, bool IsMax>
__device__ __forceinline__ T block_reduce(T v, T* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = IsMax ? warp_max(v) : warp_sum(v);
  __syncthreads();  // scratch reuse guard
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    T x = lane < nw ? scratch[lane] : (IsMax ? -INFINITY : T(0));
    x = IsMax ? warp_max(x) : warp_sum(x);
    if (lane == 0) scratch[0] = x;
  }
  __syncthreads();
  return scratch[0];
}

}  // namespace itts
