// K7 MRF core: one HiFi-GAN ResBlock1 layer fused into a single tcgen05 kernel.
//
//   y   = x + c2( lrelu( c1( lrelu(x) ), 0.1 ) )        (c1: k taps, dilation d; c2: k taps, dilation 1)
//   out = epilogue(y): lrelu(y, 0.1) -> next layer, or the MRF accumulator
//         (store / add / finalize (acc + y) / 3 -> lrelu(., slope) for the next stage)
//
// Activations are bf16 channels-last [R][C] holding lrelu(x, 0.1) (the residual
// x is recovered by inverting the leaky ReLU on load); items are packed with
// zero halos of >= 25 rows, so a conv tap that crosses an item edge reads the
// 'same' zero padding.  Unlike the per-conv kernel (tc_conv.cu), the c1 output
// never leaves the SM:
//
//   X tile   rows [r0-h2-h1, r0+M+h2+h1) of the input, TMA-loaded ONCE per tile
//            (h1 = d(k-1)/2, h2 = (k-1)/2).  Every c1 tap is the same smem tile
//            read through a row-shifted UMMA descriptor (start + s*SWZ bytes),
//            so the A operand is not re-fetched per tap.
//   TMEM     acc1 = c1 over NB x 128 intermediate rows (NB*C columns), acc2 = c2
//            over the NB x 128 output rows (the last k-1 are discarded); NB*C = 256,
//            so the two accumulators fill the 512 TMEM columns.
//   T tile   epilogue 1: acc1 + b1 -> lrelu -> zero at halo rows (c2's padding)
//            -> bf16, written into smem in the UMMA 128B/64B-swizzled K-major
//            layout, one 64-channel panel at a time; c2's MMAs on a panel start
//            as soon as that panel is published (mbarrier per panel).
//   c2       row-shifted descriptors over the T tile (taps j = 0..k-1).
//   epilogue 2: acc2 + b2 + residual -> accumulator / leaky ReLU -> bf16 output tile,
//            staged in the T region (dead once c2 finished: the residual rows are TMA'd
//            there first, each thread overwrites its chunk in place) and written back
//            with TMA tensor stores; halo rows of the output are written as zeros.
//
// Tile of M = NB*128 - (k-1) output rows, persistent CTAs (one per SM).  Warp
// roles (352 threads): warp 0 weight producer (TMA ring of [C_out][KT] panels),
// warp 1 TMEM owner + MMA issuer, warp 2 X-tile producer, warps 3-10 epilogue.
// The X tile of tile i+1 loads while c2 of tile i runs; the epilogue-2 of tile i
// overlaps c1 of tile i+1.
//
// Replaces the reference model's vocoder step (a stand-in, src/vocoder.py:52-60)
// with HiFi-GAN V1's MRF as required by BASELINE config C3.

#include "tcgen05.cuh"

namespace {

using namespace tcg;

constexpr int kMaxK = 11;

struct RbArgs {
  const float* b1;
  const float* b2;
  const int32_t* row_out;        // [R] >= 0 valid row, < 0 halo
  const __nv_bfloat16* x;        // [R][C] layer input = lrelu(x, 0.1) (residual source)
  __nv_bfloat16* acc;            // [R][C] MRF accumulator (raw bf16) or null
  __nv_bfloat16* act_out;        // [R][C] lrelu(y, slope) or null
  int64_t rows;
  int taps, dil;
  int m_out;                     // output rows per tile
  int num_tiles;
  int nbox, box_rows;            // X tile = nbox TMA boxes of box_rows rows per panel
  int acc_mode;                  // 0 none, 1 store, 2 add, 3 finalize (acc + y) / 3
  float slope;
  unsigned long long* trace;     // debug: per-CTA [16] cycle counters (wait / work breakdown) or null
};

// Debug timing (itts_resblock_debug_trace): cycles a role spends waiting on each barrier.
struct Tw {
  unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph, int slot) {
    const long long t = clock64();
    tcg::mbar_wait(bar, ph);
    c[slot] += clock64() - t;
  }
  __device__ __forceinline__ void flush(unsigned long long* dst) {
    if (dst)
      for (int i = 0; i < 8; ++i) dst[i] = c[i];
  }
};

template <int SWZ>
__device__ __forceinline__ int swz_chunk(int row, int c) {
  return SWZ == 128 ? (c ^ (row & 7)) : (c ^ ((row >> 1) & 3));
}

// C >= 128: one CTA per SM, 8 epilogue warps, acc1 + acc2 fill the 512 TMEM columns.
// C <= 64: half-size tiles and 4 epilogue warps so TWO CTAs share an SM: while one waits on its
// epilogue (the c1 -> c2 dependency of a tile) the other one's MMAs run.
template <int C>
struct Cfg {
  static constexpr int SWZ = C >= 64 ? 128 : 64;
  static constexpr int KT = SWZ / 2;            // channels per panel
  static constexpr int NKC = C / KT;            // panels
  static constexpr int CPS = C >= 128 ? 1 : 2;  // CTAs per SM
  static constexpr int EW = C >= 128 ? 8 : 4;   // epilogue warps
  static constexpr int HP = EW / 4;             // epilogue warps per TMEM lane quarter
  static constexpr int THREADS = 32 * (3 + EW);
  static constexpr int NB = 256 / (C * CPS);    // 128-row M blocks per tile
  static constexpr uint32_t TMEM_COLS = 2 * NB * C;
  static constexpr int XR_MAX = NB * 128 + 5 * (kMaxK - 1);
  static constexpr int NBOX_MAX = (XR_MAX + 255) / 256;
  static constexpr int BOXR_MAX = ((XR_MAX + NBOX_MAX - 1) / NBOX_MAX + 7) / 8 * 8;
  static constexpr int XR = NBOX_MAX * BOXR_MAX;  // allocated X rows per panel
  static constexpr int TR = NB * 128;             // T rows per panel (taps past the end read the next panel:
                                                  // only discarded output rows see them)
  static constexpr int STAGES = C == 256 ? 2 : C == 128 ? 4 : C == 64 ? 4 : 16;
  static constexpr uint32_t X_BYTES = (uint32_t)NKC * XR * SWZ;
  static constexpr uint32_t T_BYTES = (uint32_t)NKC * TR * SWZ;
  static constexpr uint32_t W_BYTES = (uint32_t)C * SWZ;  // one (tap, panel) weight stage
  static constexpr uint32_t TAIL = 16 * SWZ;              // slack after T for over-reading taps (k-1 <= 10 rows)
  static constexpr size_t SMEM = 1024 + X_BYTES + T_BYTES + TAIL + STAGES * W_BYTES + 8 * (2 * STAGES + 16);
};

template <int C>
__global__ void __launch_bounds__(Cfg<C>::THREADS, Cfg<C>::CPS)
    k_resblock_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW1,
                  const __grid_constant__ CUtensorMap mapW2, const __grid_constant__ CUtensorMap mapR,
                  const __grid_constant__ CUtensorMap mapO, const __grid_constant__ CUtensorMap mapO2, RbArgs a) {
  using K = Cfg<C>;
  constexpr int SWZ = K::SWZ, KT = K::KT, NKC = K::NKC, NB = K::NB, STAGES = K::STAGES;
  constexpr int kEpiWarps = K::EW, HP = K::HP;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sX = smem;
  uint8_t* sT = sX + K::X_BYTES;
  uint8_t* sW = sT + K::T_BYTES + K::TAIL;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + STAGES * K::W_BYTES);
  uint64_t* w_full = bars;
  uint64_t* w_empty = w_full + STAGES;
  uint64_t* x_full = w_empty + STAGES;
  uint64_t* x_empty = x_full + 1;
  uint64_t* a1_full = x_empty + 1;
  uint64_t* a1_empty = a1_full + 1;
  uint64_t* a2_full = a1_empty + 1;
  uint64_t* a2_empty = a2_full + 1;
  uint64_t* t_empty = a2_empty + 1;
  uint64_t* r_full = t_empty + 1;
  uint64_t* t_ready = r_full + 1;  // [NKC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_ready + NKC);
  __shared__ __align__(16) float sB1[C], sB2[C];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = a.taps, d = a.dil, h1 = d * (k - 1) / 2, h2 = (k - 1) / 2;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    mbar_init(x_full, 1);
    mbar_init(x_empty, 1);
    mbar_init(a1_full, 1);
    mbar_init(a1_empty, kEpiWarps);
    mbar_init(a2_full, 1);
    mbar_init(a2_empty, kEpiWarps);
    mbar_init(t_empty, 1);
    mbar_init(r_full, 1);
    for (int p = 0; p < NKC; ++p) mbar_init(&t_ready[p], kEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapX)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapW1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapW2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapR)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapO)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapO2)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(K::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  itts::pdl_trigger();  // the weight producer and the MMA warp touch no data of earlier kernels

  if (warp == 0) {
    // ---------------- weight producer: c1 in (tap, panel) order, c2 in (panel, tap) order
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = blockIdx.x; t < a.num_tiles; t += gridDim.x) {
        for (int it = 0; it < 2 * k * NKC; ++it, ++g) {
          const uint32_t s = g % STAGES, ph = (g / STAGES) & 1;
          mbar_wait(&w_empty[s], ph ^ 1);
          mbar_expect_tx(&w_full[s], K::W_BYTES);
          if (it < k * NKC) {
            const int j = it / NKC, kc = it - j * NKC;
            tma_load_2d(sW + s * K::W_BYTES, &mapW1, &w_full[s], kc * KT, j * C);
          } else {
            const int i2 = it - k * NKC, kc = i2 / k, j = i2 - kc * k;
            tma_load_2d(sW + s * K::W_BYTES, &mapW2, &w_full[s], kc * KT, j * C);
          }
        }
      }
    }
  } else if (warp == 2) {
    // ---------------- X-tile producer; also loads each tile's residual rows into the T region
    // once c2 has consumed it (epilogue 2 then reads x from shared memory, not global).
    itts::pdl_wait();
    if (lane == 0) {
      uint32_t lt = 0;
      const uint32_t bytes = (uint32_t)NKC * a.nbox * a.box_rows * SWZ;
      auto residual = [&](int tp, uint32_t lp) {
        mbar_wait(t_empty, lp & 1);
        mbar_expect_tx(r_full, (uint32_t)NKC * NB * 128 * SWZ);
        for (int kc = 0; kc < NKC; ++kc)
          for (int b = 0; b < NB; ++b)
            tma_load_2d(sT + (size_t)kc * K::TR * SWZ + (size_t)b * 128 * SWZ, &mapR, r_full, kc * KT,
                        tp * a.m_out + b * 128);
      };
      int prev = -1;
      for (int t = blockIdx.x; t < a.num_tiles; t += gridDim.x, ++lt) {
        mbar_wait(x_empty, (lt & 1) ^ 1);
        mbar_expect_tx(x_full, bytes);
        const int y0 = t * a.m_out - h2 - h1;
        for (int kc = 0; kc < NKC; ++kc)
          for (int bx = 0; bx < a.nbox; ++bx)
            tma_load_2d(sX + (size_t)kc * K::XR * SWZ + (size_t)bx * a.box_rows * SWZ, &mapX, x_full, kc * KT,
                        y0 + bx * a.box_rows);
        if (prev >= 0) residual(prev, lt - 1);
        prev = t;
      }
      if (prev >= 0) residual(prev, lt - 1);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc<C>();
      const uint32_t acc1 = tmem, acc2 = tmem + NB * C;
      uint32_t g = 0, lt = 0;
      Tw tw;
      const long long t_start = clock64();
      for (int t = blockIdx.x; t < a.num_tiles; t += gridDim.x, ++lt) {
        const uint32_t ph = lt & 1;
        tw.wait(x_full, ph, 0);
        tw.wait(a1_empty, ph ^ 1, 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int it = 0; it < k * NKC; ++it, ++g) {
          const int j = it / NKC, kc = it - j * NKC;
          const uint32_t s = g % STAGES, sph = (g / STAGES) & 1;
          tw.wait(&w_full[s], sph, 2);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t db = make_desc<SWZ>(smem_u32(sW + s * K::W_BYTES));
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const uint64_t da = make_desc<SWZ>(smem_u32(sX + (size_t)kc * K::XR * SWZ + (size_t)(b * 128 + d * j) * SWZ));
#pragma unroll
            for (int kk = 0; kk < KT / 16; ++kk)
              umma_bf16(acc1 + b * C, da + 2 * kk, db + 2 * kk, idesc, (it | kk) != 0);
          }
          umma_commit(&w_empty[s]);
        }
        umma_commit(x_empty);
        umma_commit(a1_full);
        // c2 over the T tile, panel by panel as epilogue 1 publishes them
        tw.wait(a2_empty, ph ^ 1, 3);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kc = 0; kc < NKC; ++kc) {
          tw.wait(&t_ready[kc], ph, 4);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int j = 0; j < k; ++j, ++g) {
            const uint32_t s = g % STAGES, sph = (g / STAGES) & 1;
            tw.wait(&w_full[s], sph, 5);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t db = make_desc<SWZ>(smem_u32(sW + s * K::W_BYTES));
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              const uint64_t da = make_desc<SWZ>(smem_u32(sT + (size_t)kc * K::TR * SWZ + (size_t)(b * 128 + j) * SWZ));
#pragma unroll
              for (int kk = 0; kk < KT / 16; ++kk)
                umma_bf16(acc2 + b * C, da + 2 * kk, db + 2 * kk, idesc, (kc | j | kk) != 0);
            }
            umma_commit(&w_empty[s]);
          }
        }
        umma_commit(t_empty);
        umma_commit(a2_full);
      }
      tw.c[7] = clock64() - t_start;
      if (a.trace) tw.flush(a.trace + blockIdx.x * 16);
    }
  } else {
    // ---------------- epilogue warps 3..10: TMEM lane quarter q = warp % 4, pair index h.
    // Each warp owns 4 (block, 32-column) items per phase.  Row validity for the whole tile is
    // loaded into bit masks before the accumulators are ready; residual / accumulator rows of
    // item n+1 are in flight while item n is processed.
    constexpr int NIT = NB * (C / 32) / HP;  // items per warp per phase
    constexpr int CPP = KT / 32;             // 32-column chunks per panel
    const int q = warp & 3, h = (warp - 3) >> 2;  // h < HP
    const int et = threadIdx.x - 96;
    itts::pdl_wait();  // row map, output buffers
    for (int i = et; i < C; i += 32 * kEpiWarps) {
      sB1[i] = a.b1[i];
      sB2[i] = a.b2[i];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
    uint32_t lt = 0;
    Tw tw;
    long long tp = 0;
    for (int t = blockIdx.x; t < a.num_tiles; t += gridDim.x, ++lt) {
      const uint32_t ph = lt & 1;
      const int64_t r0 = (int64_t)t * a.m_out;
      uint32_t vT = 0, vO = 0;   // bit b: T row / output row of block b is a valid (non-halo) row
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int i = b * 128 + q * 32 + lane;
        const int64_t gt = r0 - h2 + i, go = r0 + i;
        if (gt >= 0 && gt < a.rows && __ldcg(a.row_out + gt) >= 0) vT |= 1u << b;
        if (i < a.m_out && go < a.rows && __ldcg(a.row_out + go) >= 0) vO |= 1u << b;
      }
      // ---- epilogue 1: acc1 -> T tile (bf16, swizzled), panel-major
      tw.wait(a1_full, ph, 0);
      tw.wait(t_empty, ph ^ 1, 1);
      tp = clock64();
      if (lt > 0) {  // the previous tile's output store must have read the T region
        if (warp == 3 && lane == 0) bulk_wait_read0();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kc = 0; kc < NKC; ++kc) {
#pragma unroll
        for (int n = 0; n < (NB * CPP) / HP; ++n) {
          const int item = HP * n + h;
          const int b = item / CPP, cw = item - b * CPP;
          const int i = b * 128 + q * 32 + lane;
          const bool valid = (vT >> b) & 1;
          const int col = kc * KT + cw * 32;
          float v[32];
          tmem_ld32(tmem + b * C + ((uint32_t)(q * 32) << 16) + col, v);
          float bb[32];
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) *reinterpret_cast<float4*>(&bb[4 * e4]) = reinterpret_cast<const float4*>(sB1 + col)[e4];
          uint32_t w[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x0 = lrelu(v[2 * e] + bb[2 * e], 0.1f);
            float x1 = lrelu(v[2 * e + 1] + bb[2 * e + 1], 0.1f);
            if (!valid) x0 = x1 = 0.f;
            __nv_bfloat162 b2 = __floats2bfloat162_rn(x0, x1);
            w[e] = *reinterpret_cast<uint32_t*>(&b2);
          }
          uint8_t* rowp = sT + (size_t)kc * K::TR * SWZ + (size_t)i * SWZ;
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int chunk = cw * 4 + c4;
            *reinterpret_cast<uint4*>(rowp + swz_chunk<SWZ>(i, chunk) * 16) =
                make_uint4(w[4 * c4], w[4 * c4 + 1], w[4 * c4 + 2], w[4 * c4 + 3]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_ready[kc]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(a1_empty);
      tw.c[2] += clock64() - tp;
      // ---- epilogue 2: acc2 + b2 + residual -> bf16 output tile.  The residual rows were TMA'd
      // into the (dead) T region; each thread overwrites its residual chunk with its output chunk
      // in place and one thread TMA-stores the tile (rows [0, m_out)), so global writes are
      // bulk and coalesced.  Accumulator rows of item n+1 are in flight while item n is processed.
      const bool to_acc = a.acc_mode == 1 || a.acc_mode == 2;
      const float oslope = to_acc ? 1.0f : a.slope;
      uint4 au[2][4];
      auto issue = [&](int n, int slot) {
        const int item = HP * n + h;
        const int b = item / (C / 32), c0 = (item - b * (C / 32)) * 32;
        const int64_t off = (r0 + b * 128 + q * 32 + lane) * C + c0;
        if (a.acc_mode >= 2 && ((vO >> b) & 1)) ld_bf16_raw<32>(a.acc + off, au[slot]);
      };
      issue(0, 0);
      tw.wait(a2_full, ph, 3);
      tw.wait(r_full, ph, 4);
      tp = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int n = 0; n < NIT; ++n) {
        if (n + 1 < NIT) issue(n + 1, (n + 1) & 1);
        const int item = HP * n + h;
        const int b = item / (C / 32), c0 = (item - b * (C / 32)) * 32;
        const int o = b * 128 + q * 32 + lane;
        const bool valid = (vO >> b) & 1;
        float v[32];
        tmem_ld32(tmem + NB * C + b * C + ((uint32_t)(q * 32) << 16) + c0, v);
        const int kc = c0 / KT, cw = (c0 - kc * KT) / 32;
        uint8_t* rowp = sT + (size_t)kc * K::TR * SWZ + (size_t)o * SWZ;
        uint4 ru[4];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) ru[c4] = *reinterpret_cast<const uint4*>(rowp + swz_chunk<SWZ>(o, cw * 4 + c4) * 16);
        float y[32], bb[32];
        unpack_bf16<32>(ru, y);
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) *reinterpret_cast<float4*>(&bb[4 * e4]) = reinterpret_cast<const float4*>(sB2 + c0)[e4];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] += bb[e] + inv_lrelu(y[e], 10.0f);
        if (a.acc_mode >= 2) {
          float sacc[32];
          unpack_bf16<32>(au[n & 1], sacc);
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] += sacc[e];
          if (a.acc_mode == 3) {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] *= (1.0f / 3.0f);
          }
        }
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(lrelu(v[2 * e], oslope), lrelu(v[2 * e + 1], oslope));
          w[e] = valid ? *reinterpret_cast<uint32_t*>(&b2) : 0u;
        }
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4)
          *reinterpret_cast<uint4*>(rowp + swz_chunk<SWZ>(o, cw * 4 + c4) * 16) =
              make_uint4(w[4 * c4], w[4 * c4 + 1], w[4 * c4 + 2], w[4 * c4 + 3]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(a2_empty);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tw.c[5] += clock64() - tp;
      tp = clock64();
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      tw.c[6] += clock64() - tp;
      if (warp == 3 && lane == 0) {
        const int last = (a.m_out - 1) / 128;   // block holding the tile's last output row
#pragma unroll 1
        for (int kc = 0; kc < NKC; ++kc)
          for (int b = 0; b <= last; ++b)
            tma_store_2d(b < last ? &mapO : &mapO2, sT + (size_t)kc * K::TR * SWZ + (size_t)b * 128 * SWZ, kc * KT,
                         (int)(r0 + b * 128));
        bulk_commit();
      }
    }
    if (warp == 3 && lane == 0) bulk_wait0();
    if (a.trace && warp == 3 && lane == 0) tw.flush(a.trace + blockIdx.x * 16 + 8);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(K::TMEM_COLS));
  }
}

unsigned long long* g_trace = nullptr;

template <int C>
int launch(const void* x, int64_t rows, const void* w1, const void* w2, int taps, RbArgs a, cudaStream_t st) {
  using K = Cfg<C>;
  const int xr = 128 * K::NB + a.dil * (taps - 1);
  a.nbox = (xr + 255) / 256;
  a.box_rows = ((xr + a.nbox - 1) / a.nbox + 7) / 8 * 8;
  if (a.nbox * a.box_rows > K::XR) return ITTS_EUNSUPPORTED;
  CUtensorMap mx, m1, m2, mr;
  if (!encode_2d(&mx, x, C, (uint64_t)rows, C, K::KT, a.box_rows, K::SWZ)) return ITTS_EINVAL;
  if (!encode_2d(&mr, x, C, (uint64_t)rows, C, K::KT, 128, K::SWZ)) return ITTS_EINVAL;
  if (!encode_2d(&m1, w1, C, (uint64_t)taps * C, C, K::KT, C, K::SWZ)) return ITTS_EINVAL;
  if (!encode_2d(&m2, w2, C, (uint64_t)taps * C, C, K::KT, C, K::SWZ)) return ITTS_EINVAL;
  static uint64_t attr_set = 0;
  if (!(attr_set & itts::device_bit())) {
    cudaError_t e = cudaFuncSetAttribute(k_resblock_tc<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set |= itts::device_bit();
  }
  a.m_out = 128 * K::NB - (taps - 1);
  void* out = (a.acc_mode == 1 || a.acc_mode == 2) ? (void*)a.acc : (void*)a.act_out;
  CUtensorMap mo, mo2;
  if (!encode_2d(&mo, out, C, (uint64_t)rows, C, K::KT, 128, K::SWZ)) return ITTS_EINVAL;
  if (!encode_2d(&mo2, out, C, (uint64_t)rows, C, K::KT, a.m_out - 128 * ((a.m_out - 1) / 128), K::SWZ))
    return ITTS_EINVAL;
  a.num_tiles = (int)((rows + a.m_out - 1) / a.m_out);
  const int slots = num_sms() * K::CPS;
  const int grid = a.num_tiles < slots ? a.num_tiles : slots;
  const cudaError_t e = itts::launch_pdl_cls(itts::PDL_RESBLOCK, k_resblock_tc<C>, dim3(grid), dim3(K::THREADS), K::SMEM, st, mx, m1, m2,
                                         mr, mo, mo2, a);
  return e == cudaSuccess ? ITTS_OK : (int)e;
}

}  // namespace

// Debug: subsequent itts_resblock_tc launches write per-CTA cycle counters to buf
// ([grid][16] u64: MMA-thread waits x_full, a1_empty, w_full(c1), a2_empty, t_ready, w_full(c2), -, total;
// epilogue warp 3: waits a1_full, t_empty, epi-1 work, a2_full, r_full, epi-2 work, bar, -).  null = off.
ITTS_API int itts_resblock_debug_trace(void* buf) {
  g_trace = static_cast<unsigned long long*>(buf);
  return ITTS_OK;
}

ITTS_API int itts_resblock_tc(const void* x, int64_t rows, int32_t c, const void* w1, const void* w2, const float* b1,
                              const float* b2, int32_t taps, int32_t dil, const int32_t* row_out, void* acc,
                              int32_t acc_mode, void* act_out, float slope, void* stream) {
  if (!x || !w1 || !w2 || !b1 || !b2 || !row_out || rows <= 0) return ITTS_EINVAL;
  if (taps < 1 || taps > kMaxK || taps % 2 == 0 || dil < 1 || dil > 5) return ITTS_EINVAL;
  if (acc_mode < 0 || acc_mode > 3 || (acc_mode && !acc)) return ITTS_EINVAL;
  if (!(slope >= 0.f && slope <= 1.f)) return ITTS_EINVAL;  // lrelu as max(y, slope * y)
  // exactly one output: act_out for modes 0 / 3, the accumulator for modes 1 / 2
  if ((acc_mode == 0 || acc_mode == 3) != (act_out != nullptr)) return ITTS_EINVAL;
  if ((act_out && act_out == x) || (acc && acc == x)) return ITTS_EINVAL;  // neighbouring tiles still read x
  if (((uintptr_t)x | (uintptr_t)w1 | (uintptr_t)w2 | (uintptr_t)acc | (uintptr_t)act_out) & 15) return ITTS_EALIGN;
  RbArgs a{b1, b2, row_out, (const __nv_bfloat16*)x, (__nv_bfloat16*)acc, (__nv_bfloat16*)act_out, rows, taps, dil,
           0, 0, 0, 0, acc_mode, slope, g_trace};
  cudaStream_t st = (cudaStream_t)stream;
  switch (c) {
    case 256: return launch<256>(x, rows, w1, w2, taps, a, st);
    case 128: return launch<128>(x, rows, w1, w2, taps, a, st);
    case 64: return launch<64>(x, rows, w1, w2, taps, a, st);
    case 32: return launch<32>(x, rows, w1, w2, taps, a, st);
  }
  return ITTS_EUNSUPPORTED;
}

static_assert(Cfg<256>::SMEM + 8 * 256 <= 232448 && Cfg<128>::SMEM + 8 * 128 <= 232448 &&
                  2 * (Cfg<64>::SMEM + 8 * 64 + 1024) <= 233472 && 2 * (Cfg<32>::SMEM + 8 * 32 + 1024) <= 233472,
              "resblock tile exceeds the 227 KB dynamic shared memory limit");
