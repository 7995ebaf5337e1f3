// K1: slot gather / scatter -- packs per-request state rows that live
// anywhere in the ragged state arena into contiguous batch rows (and back).
//
// Reference semantics: the batch gather/scatter of run_iteration
// (pkg/src/incrtts/scheduler.py:452-468 gather (dec_state, enc) in pool
// order; :467 / :485 scatter the new states back to the items).  Batch row
// i is the i-th item of the module call, i.e. IterationReport.decoder_ids
// order, and a request's rows are read from its current state buffer and
// written to its next one, so the batch is always dense ("compacted")
// whatever subset of the pool is live.
//
// Rows move as 128-bit vectors (ld.global.nc.v4 / st.global.v4); row_bytes
// and every pointer must be 16-byte aligned.

#include "common.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint4 ld_nc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// dst rows are contiguous (row i at dst + i*row_vec); src rows at src_ptr[i].
__global__ void __launch_bounds__(kThreads) k_gather(uint4* __restrict__ dst,
                                                     const int64_t* __restrict__ src_ptr,
                                                     int64_t row_vec) {
  const uint4* src = reinterpret_cast<const uint4*>(src_ptr[blockIdx.y]);
  uint4* out = dst + (int64_t)blockIdx.y * row_vec;
  for (int64_t v = (int64_t)blockIdx.x * kThreads + threadIdx.x; v < row_vec;
       v += (int64_t)gridDim.x * kThreads)
    out[v] = ld_nc(src + v);
}

__global__ void __launch_bounds__(kThreads) k_scatter(const int64_t* __restrict__ dst_ptr,
                                                      const uint4* __restrict__ src,
                                                      int64_t row_vec) {
  uint4* out = reinterpret_cast<uint4*>(dst_ptr[blockIdx.y]);
  const uint4* in = src + (int64_t)blockIdx.y * row_vec;
  for (int64_t v = (int64_t)blockIdx.x * kThreads + threadIdx.x; v < row_vec;
       v += (int64_t)gridDim.x * kThreads)
    out[v] = ld_nc(in + v);
}

int grid_x(int64_t row_vec) {
  int64_t g = (row_vec + kThreads - 1) / kThreads;
  return (int)(g < 64 ? g : 64);
}

}  // namespace

ITTS_API int itts_gather_rows(void* dst, const int64_t* src_ptrs, int32_t n_rows, int64_t row_bytes,
                              void* stream) {
  if (n_rows <= 0) return n_rows == 0 ? ITTS_OK : ITTS_EINVAL;
  if (!dst || !src_ptrs || row_bytes <= 0) return ITTS_EINVAL;
  if ((row_bytes & 15) || ((uintptr_t)dst & 15)) return ITTS_EALIGN;
  const int64_t row_vec = row_bytes / 16;
  dim3 grid(grid_x(row_vec), (unsigned)n_rows);
  k_gather<<<grid, kThreads, 0, (cudaStream_t)stream>>>((uint4*)dst, src_ptrs, row_vec);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_scatter_rows(const int64_t* dst_ptrs, const void* src, int32_t n_rows,
                               int64_t row_bytes, void* stream) {
  if (n_rows <= 0) return n_rows == 0 ? ITTS_OK : ITTS_EINVAL;
  if (!src || !dst_ptrs || row_bytes <= 0) return ITTS_EINVAL;
  if ((row_bytes & 15) || ((uintptr_t)src & 15)) return ITTS_EALIGN;
  const int64_t row_vec = row_bytes / 16;
  dim3 grid(grid_x(row_vec), (unsigned)n_rows);
  k_scatter<<<grid, kThreads, 0, (cudaStream_t)stream>>>(dst_ptrs, (const uint4*)src, row_vec);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_version(void) { return 1; }
