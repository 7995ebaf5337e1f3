// K7 core: implicit-GEMM 1-D convolution on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// out[r, n] = epilogue( sum_j sum_ci X[r + off_j, ci] * Wt[j, n, ci] + bias[n % C_out] )
//
//   X   : bf16 activations, channels-last [R][C_in] (a packed batch of items,
//         each with a zero halo of >= max|off_j| rows on both sides, so the
//         shifted taps read zeros at every item edge = 'same' zero padding).
//   Wt  : bf16 weights [taps][N][C_in] (K-major B operand).
//   taps: regular conv -> off_j = dil*(j - (k-1)/2); ConvTranspose(stride u,
//         kernel 2u) -> 3 taps {-1,0,+1} over N = u*C_out phase-major
//         columns (see hifigan.py: the transpose conv is a 3-tap conv whose
//         output row q of width u*C_out is u consecutive output rows).
//
// Persistent kernel, one CTA per SM, static round-robin over output tiles
// 128 x BN (x K-split).  fp32 accumulators in TMEM, double-buffered (2 x BN
// columns) so the epilogue of tile i overlaps the MMAs of tile i+1 and the
// TMA ring runs ahead across tile boundaries.  Warp roles (192 threads):
//   warp 0   TMA producer (one lane): A box {KT,128} at row m0+off_j, B box
//            {KT,BN}; STAGES-deep smem ring (mbarrier full/empty).
//   warp 1   TMEM allocator + MMA issuer (one lane): KT/16 x
//            tcgen05.mma.cta_group::1.kind::f16 per stage; tcgen05.commit frees
//            the stage / publishes the accumulator (tmem_full[b]).
//   warps 2-5 epilogue: tcgen05.ld 32x32b.x32 -> +bias -> residual (bf16,
//            stored as lrelu(y) and inverted on load) / MRF accumulate (bf16) /
//            leaky-ReLU -> bf16 act, or raw fp32 (GEMM outputs, K-split
//            partials); then tmem_empty[b].
//
// Used by the HiFi-GAN V1 chunk vocoder (MRF resblock convs, the transposed
// upsampling convs, conv_pre) and the Tacotron2 encoder conv stack.

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "tcgen05.cuh"

namespace {

using namespace tcg;

constexpr int kBlockM = 128;
constexpr int kEpiWarps = 8;                 // 2 warps per TMEM lane quarter, each half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;  // producer warp + MMA warp + epilogue
constexpr int kMaxTaps = 16;

struct Taps {
  int n;
  int off[kMaxTaps];
};

struct Epi {
  const float* bias;          // [C_out] (added by split 0 only)
  const int32_t* row_out;     // [rows]: output row for input row r (phase p -> +p), -1 = halo
  const __nv_bfloat16* res_in;  // bf16 [out_rows][C_out] residual y stored as lrelu(y, res_slope), or null
  float res_slope;            // inverse leaky-ReLU applied to res_in (1.0 = stored raw)
  float* f32_out;             // fp32 [out_rows][C_out] raw output (per K-split slice), or null
  int64_t f32_split_stride;   // elements between K-split slices of f32_out
  __nv_bfloat16* acc;         // bf16 MRF accumulator [out_rows][C_out] (raw), or null
  __nv_bfloat16* act_out;     // bf16 [out_rows][C_out] = lrelu(y, slope), or null
  int64_t rows;               // input rows R
  int c_out;                  // output row width; N = phases * c_out
  int acc_mode;               // 0 none, 1 store, 2 add, 3 finalize: y = (acc + y) / 3
  float slope;                // leaky-ReLU slope for act_out (1.0 = identity, 0.0 = ReLU)
  int zero_halo;              // write zeros into act_out for halo rows (CONV mode only)
  int act;                    // act_out activation: 0 leaky ReLU (slope), 1 tanh (PostNet), 2 GELU (tanh form, BERT)
};

struct TileSched {
  int n_tiles, ksplit, iters_per_split;
  __device__ __forceinline__ void decode(int t, int& mt, int& nt, int& z) const {
    z = t % ksplit;
    const int mn = t / ksplit;
    nt = mn % n_tiles;
    mt = mn / n_tiles;
  }
};

template <int BN, int SWZ, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, Taps taps,
              int kchunks, int n_total, int num_tiles, TileSched sched, Epi epi) {
  constexpr int KT = SWZ / 2;                   // bf16 channels per smem row
  constexpr uint32_t A_BYTES = kBlockM * SWZ;
  constexpr uint32_t B_BYTES = BN * SWZ;
  constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int iters = sched.iters_per_split;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 32 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  itts::pdl_trigger();

  if (warp == 0) {
    itts::pdl_wait();  // A rows come from the previous kernel
    if (lane == 0) {
      uint32_t g = 0;  // running stage counter across tiles
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mt, nt, z;
        sched.decode(t, mt, nt, z);
        const int m0 = mt * kBlockM, n0 = nt * BN;
        for (int it = z * iters; it < (z + 1) * iters; ++it, ++g) {
          const uint32_t s = g % STAGES, ph = (g / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          const int j = it / kchunks, kc = it - j * kchunks;
          mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
          tma_load_2d(sA + s * A_BYTES, &mapA, &full[s], kc * KT, m0 + taps.off[j]);
          tma_load_2d(sB + s * B_BYTES, &mapB, &full[s], kc * KT, j * n_total + n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc<BN>();
      uint32_t g = 0, lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        const uint32_t b = lt & 1, tph = (lt >> 1) & 1;
        mbar_wait(&tempty[b], tph ^ 1);  // epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + b * BN;
        for (int it = 0; it < iters; ++it, ++g) {
          const uint32_t s = g % STAGES, ph = (g / STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = make_desc<SWZ>(smem_u32(sA + s * A_BYTES));
          const uint64_t db = make_desc<SWZ>(smem_u32(sB + s * B_BYTES));
#pragma unroll
          for (int kk = 0; kk < KT / 16; ++kk)  // +32 bytes per K=16 step inside the swizzle row
            umma_bf16(d, da + 2 * kk, db + 2 * kk, idesc, (it | kk) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[b]);
      }
    }
  } else {
    // Epilogue: 8 warps; warp w owns TMEM lanes [32*(w%4), +32) (tile rows) and one
    // half of the tile's columns.  Residual / accumulator loads for a chunk are
    // issued before its tcgen05.ld so their latency overlaps the TMEM read.
    constexpr int CW = BN >= 64 ? 32 : 16;   // columns per chunk
    const int ew = warp - 2;
    itts::pdl_wait();  // row map, residual, accumulator and output buffers
    const int quarter = warp & 3, half = ew >> 2;
    const int C = epi.c_out;
    const float inv_res = 1.0f / epi.res_slope;
    uint32_t lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      int mt, nt, z;
      sched.decode(t, mt, nt, z);
      const uint32_t b = lt & 1, tph = (lt >> 1) & 1;
      const int64_t r = (int64_t)mt * kBlockM + quarter * 32 + lane;
      const bool in_range = r < epi.rows;
      const int out_row = in_range ? __ldcg(epi.row_out + r) : -1;
      mbar_wait(&tfull[b], tph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += CW) {
        const int n = nt * BN + c0;   // first global column of this chunk
        const int phase = n / C, co = n - phase * C;
        const bool live = in_range && out_row >= 0;
        const int64_t o = live ? ((int64_t)out_row + phase) * C + co : 0;
        uint4 ru[CW / 8], au[CW / 8];
        if (live && epi.res_in) ld_bf16_raw<CW>(epi.res_in + o, ru);
        if (live && epi.acc_mode >= 2) ld_bf16_raw<CW>(epi.acc + o, au);
        float v[CW];
        tmem_ld<CW>(tmem + b * BN + ((uint32_t)(quarter * 32) << 16) + c0, v);
        if (!in_range) continue;
        if (out_row < 0) {
          if (epi.zero_halo && epi.act_out) {
            uint4* dst = reinterpret_cast<uint4*>(epi.act_out + r * C + co);
#pragma unroll
            for (int q = 0; q < CW / 8; ++q) dst[q] = make_uint4(0, 0, 0, 0);
          }
          continue;
        }
        if (z == 0) {
#pragma unroll
          for (int i = 0; i < CW; ++i) v[i] += __ldg(epi.bias + co + i);
        }
        if (epi.f32_out) {
          float4* dst = reinterpret_cast<float4*>(epi.f32_out + z * epi.f32_split_stride + o);
#pragma unroll
          for (int q = 0; q < CW / 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        if (epi.res_in) {
          float y[CW];
          unpack_bf16<CW>(ru, y);
#pragma unroll
          for (int i = 0; i < CW; ++i) v[i] += inv_lrelu(y[i], inv_res);
        }
        if (epi.acc_mode == 1) {
          store_bf16<CW>(epi.acc + o, v, 1.0f);
        } else if (epi.acc_mode >= 2) {
          float a[CW];
          unpack_bf16<CW>(au, a);
#pragma unroll
          for (int i = 0; i < CW; ++i) a[i] += v[i];
          if (epi.acc_mode == 2) {
            store_bf16<CW>(epi.acc + o, a, 1.0f);
          } else {  // finalize: x = (rb0 + rb1 + rb2) / 3
#pragma unroll
            for (int i = 0; i < CW; ++i) v[i] = a[i] * (1.0f / 3.0f);
          }
        }
        if (epi.act_out) {
          if (epi.act == 1) {
#pragma unroll
            for (int i = 0; i < CW; ++i) v[i] = tanhf(v[i]);
          } else if (epi.act == 2) {
#pragma unroll
            for (int i = 0; i < CW; ++i)
              v[i] = 0.5f * v[i] * (1.0f + tanhf(0.7978845608f * (v[i] + 0.044715f * v[i] * v[i] * v[i])));
          }
          store_bf16<CW>(epi.act_out + o, v, epi.act ? 1.0f : epi.slope);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[b]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

template <int BN, int SWZ, int STAGES>
int launch(const void* x, int64_t rows, int c_in, int64_t x_ld, const void* w, int n_total, const Taps& taps,
           int ksplit, const Epi& epi, cudaStream_t st) {
  constexpr int KT = SWZ / 2;
  CUtensorMap ma, mb;
  if (!encode_2d(&ma, x, (uint64_t)c_in, (uint64_t)rows, (uint64_t)x_ld, KT, kBlockM, SWZ)) return ITTS_EINVAL;
  if (!encode_2d(&mb, w, (uint64_t)c_in, (uint64_t)taps.n * n_total, (uint64_t)c_in, KT, BN, SWZ))
    return ITTS_EINVAL;
  const int kchunks = c_in / KT;
  const int total_iters = taps.n * kchunks;
  if (ksplit < 1 || total_iters % ksplit) return ITTS_EINVAL;
  const size_t smem = 1024 + STAGES * (kBlockM + BN) * SWZ + (2 * STAGES + 4) * 8 + 16;
  static uint64_t attr_set = 0;
  if (!(attr_set & itts::device_bit())) {
    cudaFuncSetAttribute(k_conv_tc<BN, SWZ, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set |= itts::device_bit();
  }
  TileSched sched{n_total / BN, ksplit, total_iters / ksplit};
  const int m_tiles = (int)((rows + kBlockM - 1) / kBlockM);
  const int tiles = m_tiles * sched.n_tiles * ksplit;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  const cudaError_t e = itts::launch_pdl_cls(itts::PDL_CONV, k_conv_tc<BN, SWZ, STAGES>, dim3(grid), dim3(kThreads), smem, st, ma, mb,
                                         taps, kchunks, n_total, tiles, sched, epi);
  return e == cudaSuccess ? ITTS_OK : (int)e;
}

}  // namespace

int conv1d_tc_impl(const void* x, int64_t rows, int32_t c_in, int64_t x_ld, const void* w, int32_t n_total,
                   int32_t n_taps, const int32_t* host_tap_off, const float* bias, int32_t c_out,
                   const int32_t* row_out, const void* res_in, float res_slope, float* f32_out, int32_t ksplit,
                   void* acc, int32_t acc_mode, void* act_out, float slope, int32_t zero_halo, int32_t bn,
                   int32_t act, void* stream) {
  if (!x || !w || !bias || !row_out || !host_tap_off || rows <= 0) return ITTS_EINVAL;
  if (n_taps < 1 || n_taps > kMaxTaps || c_out <= 0 || n_total % c_out) return ITTS_EINVAL;
  if (c_out % 32 || (acc_mode && !acc) || acc_mode < 0 || acc_mode > 3) return ITTS_EINVAL;
  if (x_ld < c_in || (x_ld * 2) % 16 || res_slope <= 0.f || res_slope > 1.f) return ITTS_EINVAL;
  if (!(slope >= 0.f && slope <= 1.f)) return ITTS_EINVAL;  // lrelu as max(x, slope * x)
  if (ksplit > 1 && (!f32_out || res_in || acc_mode || act_out)) return ITTS_EINVAL;  // partials are raw fp32
  if (((uintptr_t)x | (uintptr_t)w) & 15) return ITTS_EALIGN;
  Taps taps{};
  taps.n = n_taps;
  for (int i = 0; i < n_taps; ++i) taps.off[i] = host_tap_off[i];
  Epi epi{bias, row_out, (const __nv_bfloat16*)res_in, res_slope, f32_out, rows * (int64_t)c_out,
          (__nv_bfloat16*)acc, (__nv_bfloat16*)act_out, rows, c_out, acc_mode, slope, zero_halo, act};
  if (ksplit < 1) ksplit = 1;
  cudaStream_t st = (cudaStream_t)stream;
  const int swz = (c_in % 64 == 0) ? 128 : (c_in % 32 == 0 ? 64 : 0);
  if (!swz) return ITTS_EUNSUPPORTED;
  if (bn == 0) bn = n_total % 128 == 0 ? 128 : n_total % 64 == 0 ? 64 : 32;
  if (n_total % bn) return ITTS_EINVAL;
  if (swz == 128) {
    switch (bn) {
      case 256: return launch<256, 128, 4>(x, rows, c_in, x_ld, w, n_total, taps, ksplit, epi, st);
      case 128: return launch<128, 128, 6>(x, rows, c_in, x_ld, w, n_total, taps, ksplit, epi, st);
      case 64: return launch<64, 128, 8>(x, rows, c_in, x_ld, w, n_total, taps, ksplit, epi, st);
      case 32: return launch<32, 128, 8>(x, rows, c_in, x_ld, w, n_total, taps, ksplit, epi, st);
    }
  } else {
    switch (bn) {
      case 64: return launch<64, 64, 8>(x, rows, c_in, x_ld, w, n_total, taps, ksplit, epi, st);
      case 32: return launch<32, 64, 8>(x, rows, c_in, x_ld, w, n_total, taps, ksplit, epi, st);
    }
  }
  return ITTS_EUNSUPPORTED;
}

ITTS_API int itts_conv1d_tc(const void* x, int64_t rows, int32_t c_in, int64_t x_ld, const void* w,
                            int32_t n_total, int32_t n_taps, const int32_t* host_tap_off, const float* bias,
                            int32_t c_out, const int32_t* row_out, const void* res_in, float res_slope,
                            float* f32_out, int32_t ksplit, void* acc, int32_t acc_mode, void* act_out,
                            float slope, int32_t zero_halo, int32_t bn, void* stream) {
  return conv1d_tc_impl(x, rows, c_in, x_ld, w, n_total, n_taps, host_tap_off, bias, c_out, row_out, res_in,
                        res_slope, f32_out, ksplit, acc, acc_mode, act_out, slope, zero_halo, bn, 0, stream);
}
