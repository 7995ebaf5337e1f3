// K6P: the whole Tacotron2 decoder chunk (up to 32 autoregressive steps) as ONE persistent kernel.
//
// Replaces the per-step chain of ~10 launches (tier_r.cu k_gemv / k_lstm_cell / k_attention +
// two tc_conv gate GEMMs) for decode_chunk_batch (reference acoustic.py:191-219, :234-238;
// Tacotron2 decoder step = paper Eq. 2).  One CTA per SM; everything that is
// constant across steps stays on chip.  The five phases of a step are separated by grid-wide
// barriers for pooled batches > 96; up to 96 rows only the decoder-gate phase ends in one (and
// PRE above 40 rows), the other hand-offs are monotonic counters in global memory (PRE tasks,
// query partials per K-split, attention chunks per item, combined contexts):
//
//   PRE    mel(s-1) = bp + the 33 projection partials (fixed order) -> mel / gate outputs,
//          last_frame; H1 = relu(W0 . last_frame) (in shared memory); p = relu(W1 . H1)
//          (8-item x 32-column tasks)
//   ATT    gates = [p|ctx|att_h] . Wa^T on the tensor cores (tcgen05, weights as M), 4-way
//          K-split per 32-unit group; the LSTM cell is the fixup epilogue, which also emits the
//          group's query partial q_g = Wq[:, group] . att_h[group]  (no separate query phase)
//   ATT-A  per (item, 32-position chunk), two chunks at a time per CTA (half-CTA streams): q = sum
//          of the 32 group partials, location features as one tcgen05 MMA chain, energies,
//          chunk max, exp, chunk sum, unnormalised context partial
//   ATT-B  per item: combine chunks (max / rescale / sum, chunk order) -> context, W, W_acc
//   DEC    gates = [ctx|att_h|dec_h] . Wd^T + cell (as ATT); the fixup emits the group's
//          mel/gate projection partial of dec_h while the CTAs without a gate group project the
//          context (the 33rd partial), so the projection is summed by the next PRE
//
// The bf16 operand mirror keeps two banks of att_h / dec_h (step parity) so a GEMM phase never
// reads the h it is overwriting.  All reductions run in a fixed order: results do not depend
// on the batch composition or on the number of SMs.

#include <cuda_bf16.h>

#include "tcgen05.cuh"

// Gate weights resident in TMEM as the MMA A operand (pooled batches <= 128, weights exact in bf16
// or bf16 products): DEC_WRES = 1 the decoder gates (10 K-chunks x [128 rows][64] bf16 = 160 KB
// per gate CTA, TMEM columns [192, 512)), 2 the attention gates (7 K-chunks, 112 KB, [192, 416)),
// 0 off.  Written once per launch; that phase then streams only the operand tiles
// (tools/probe_tmem_a.cu: TMEM-A products are bit-identical to smem-A products).  Measured (same box,
// B = 1..128): no gain for either phase -- their MMAs wait on the prenet / combined-context operand
// chunks (PRE and ATT-B chains on other CTAs), not on the weight stream -- hence off by default.
#ifndef DEC_WRES
#define DEC_WRES 0
#endif
constexpr uint32_t WRES_COL = 192;
// Pooled batches up to DEC_MERGE_B: the chunk combine (ATT-B) runs at the start of the
// decoder-gate phase on the CTAs that do not own the context columns of that GEMM; the owners
// start with their att_h columns and wait for the combined contexts on a counter (one grid
// barrier fewer per step; same-box A/B: B=1 -4.4%, B=24 -2.7%, B=128 +2.5%, hence the cut-off).
// Larger batches: separate ATT-B phase.
#ifndef DEC_MERGE_B
#define DEC_MERGE_B 96
#endif
// Merged schedule: no grid barrier between ATT-A and the decoder-gate phase.  Every ATT-A task
// releases its item's chunk counter (bar + ITEM_CNT + b) after its U / AP stores; a combiner waits
// for that item's chunks only, and the gate CTAs go from their own attention tasks straight into
// the decoder-gate GEMM (its context chunks already wait on the combined-context counter).
#ifndef DEC_ITEM_CNT
#define DEC_ITEM_CNT 1
#endif
constexpr int ITEM_CNT = 64;     // bar[64 + b]: ATT-A chunks of item b done (monotonic over the launch)
// With DEC_ITEM_CNT, also no grid barrier between the attention-gate phase and ATT-A: every gate CTA
// releases bar[QCNT + ks] once per step after its query partials (items b = ks mod 4), and an
// attention task loads an item's q once the 32 unit groups of that split have released.
constexpr int QCNT = 36;
#ifndef DEC_H1_UNROLL
#define DEC_H1_UNROLL 5
#endif
#ifndef DEC_SPREAD
#define DEC_SPREAD 1   // context / prenet K-chunks spread over the four K-splits (chunk_of)
#endif
#ifndef DEC_WFENCE
#define DEC_WFENCE 0
#endif
// generic-proxy stores to the bf16 operand mirror are read by bulk copies (async proxy) of other
// CTAs: with DEC_WFENCE every writing thread fences its stores to the async proxy before the
// release that publishes them
#if DEC_WFENCE
#define WFENCE() asm volatile("fence.proxy.async.global;" ::: "memory")
#else
#define WFENCE() ((void)0)
#endif

namespace {

constexpr int NMEL = 80, EMB = 512, HID = 1024, PRE = 256, ATT = 128, KLOC = 31;
constexpr int P_OFF = 0, CTX_OFF = 256, ATTH_OFF = 768, DECH_OFF = 1792, ATTC_OFF = 2816, DECC_OFF = 3840,
              LAST_OFF = 4864, ROW = 4944;
constexpr int XB2 = 4864;        // bf16 mirror row: [p | ctx | att_h b0 | dec_h b0 | att_h b1 | dec_h b1]
constexpr int NCC = XB2 / 64;    // 64-column chunks of the mirror

// The bf16 operand mirror is kept in the UMMA-ready layout: per (128-item block, 64-column chunk)
// one [128 rows][128 B] tile with the 128B swizzle applied, so the A operand of a gate-GEMM
// stage is ONE contiguous bulk copy (no per-row TMA requests).
__device__ __forceinline__ int64_t xb_off(int r, int col) {
  const int cc = col >> 6, j = (col >> 3) & 7, e = col & 7;
  return ((int64_t)((r >> 7) * NCC + cc) * 128 + (r & 127)) * 64 + ((j ^ (r & 7)) << 3) + e;
}

struct DecArgs;
__device__ __forceinline__ void xb_store(const DecArgs& a, int b, int col, float v);

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tcg::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tcg::smem_u32(bar))
               : "memory");
}
// L2 residency: the decoder's weights are re-read every step (evict_last) while the attention's
// memory / processed-memory rows stream once per step (evict_first), so at large pooled batches the
// rows (B x L x 2.5 KB per step) do not push the 37 MB of gate weights out of L2
#ifndef DEC_L2_HINTS
#define DEC_L2_HINTS 1
#endif
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t p;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, bool keep) {
#if DEC_L2_HINTS
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          tcg::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tcg::smem_u32(bar)), "l"(l2_policy(keep))
      : "memory");
#else
  bulk_g2s(dst, src, bytes, bar);
#endif
}
constexpr int DPLAN = 8;
constexpr int NT = 256, NW = 8;  // threads / warps per CTA
constexpr int NGRP = HID / 32;   // 32-unit gate groups: query partials, projection partials (+1 ctx)
constexpr int GEMM_CTAS = HID / 8;  // 128 CTAs x 8 hidden units
constexpr int KA = 1792, KD = 2560;
constexpr int MAXCH = 256;       // max position chunks per item
constexpr int MAXB = 512;        // max pooled rows (two 256-column MMA N tiles)
constexpr int ACH = 64;          // max positions per attention chunk (pm + memory rows staged in smem)
// Staging: a chunk of n positions is [n pm rows][n memory rows].  One round of tasks (every CTA
// at most one chunk): chunks up to 64 positions in one 160 KB buffer.  Several rounds: 32-position
// chunks double-buffered (the next chunk streams in while this one computes).
constexpr uint32_t ASTAGE = 32 * (ATT + EMB) * 4;
constexpr int HALO = (KLOC - 1) / 2;

__device__ __forceinline__ int att_off(int bank) { return 768 + bank * 2048; }
__device__ __forceinline__ int dec_off(int bank) { return 1792 + bank * 2048; }
// LSTM cell nonlinearities with one ex2 + one fast reciprocal each (relative error ~1e-7, the fp32
// rounding level; the accurate expf / tanhf / IEEE division cost ~5x the instructions)
__device__ __forceinline__ float sigm_fast(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
// tanh via one exp2 and one reciprocal: absolute error ~1e-7 (the energies only sum it)
__device__ __forceinline__ float tanh_fast(float x) { return 1.0f - __fdividef(2.0f, 1.0f + __expf(2.0f * x)); }

struct DecArgs {
  int B, nsteps, step0;            // rows, steps in this launch, global index of the first step
  const int64_t* plan;             // [B][8]
  float* work;                     // [B][ROW]
  __nv_bfloat16* xb;               // [ceil(B/128)][NCC][128][64] swizzled tiles (see xb_off)
  __nv_bfloat16* xbl;              // split mode: the low bf16 parts v - bf16(v) of the mirror, same layout
  const float* W0T;                // [80][256]
  const float* W1T;                // [256][256]
  const __nv_bfloat16* Wa;         // [128 CTAs][28 chunks][32 rows][64] swizzled tiles, unit-interleaved rows
  const float* ba;                 // [128][32]
  const __nv_bfloat16* Wd;         // [128][40][32][64]
  const __nv_bfloat16* Wal;        // split mode: low bf16 parts of Wa / Wd (null: plain bf16 products)
  const __nv_bfloat16* Wdl;
  int split;                       // 0: bf16 products; 1: gates = Wh.Xh + Wh.Xl + Wl.Xh (fp32-level products,
                                   // fp32 accumulation); 2: weights exact in bf16 (Wl = 0): Wh.Xh + Wh.Xl
  const float* bd;                 // [128][32]
  const float* WqT;                // [1024][128]
  const float* WlocD;              // [2][31][128] = location conv composed with the location dense layer
  const float* v;                  // [128]
  const float* WpT;                // [1536][81]
  const float* bp;                 // [81]
  float* Gp;                       // [4 splits][32 groups][B16][128] gate GEMM K-split partials
  float* H1;                       // [B][256]
  float* Qp;                       // [NGRP][B][128] query partials per unit group
  float* Pp;                       // [NGRP + 1][B][81] projection partials (groups of dec_h, then ctx)
  float* U;                        // [B][u_ld] unnormalised attention numerators
  int64_t u_ld;
  float* AP;                       // [B][MAXCH][2 + 512] chunk max, sum, context partial
  unsigned* bar;                   // [2 + 32 + 1] grid barrier, gate-group counters, combined-context
                                   // counter (zeroed before launch)
  unsigned long long* trace;       // debug: [16] ns per phase summed over steps (CTA 0), or null
};

unsigned long long* g_dec_trace = nullptr;

// One value of the operand mirror: bf16(v), and in split mode also the remainder bf16(v - bf16(v))
// (together ~16 significant bits; the gate products then match fp32 GEMV to ~1e-5 relative).
__device__ __forceinline__ void xb_store(const DecArgs& a, int b, int col, float v) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const int64_t o = xb_off(b, col);
  a.xb[o] = hi;
  if (a.split) a.xbl[o] = __float2bfloat16_rn(v - __bfloat162float(hi));
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ grid barrier
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {  // arrive (release) on one counter, spin (acquire) until all CTAs arrived
    ++gen;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned seen;
    do {  // relaxed polling (an acquire load per poll would invalidate L1 every iteration)
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
    } while (seen < gen * gridDim.x);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

// Spin until a monotonic global counter reaches `target` (relaxed polls, then acquire).
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
  unsigned seen;
  do {
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p) : "memory");
  } while (seen < target);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// L2-coherent loads for data produced inside this kernel by other CTAs (never cached in L1).
__device__ __forceinline__ float ldf(const float* p) { return __ldcg(p); }

// per-item L and step counts, cached in shared memory at kernel start (B <= MAXB)
struct PlanCache {
  int L[MAXB], steps[MAXB];
};
__device__ __forceinline__ bool active(const PlanCache& pc, int b, int s) { return s < pc.steps[b]; }

// ------------------------------------------------------------------ small batched GEMV task
// Y[b][n] (n in [n0, n0+32)) for items [b0, b0+8): sum over k in [k0, k1) of X[b][k] W^T[k][n].
// x(b, k) is supplied by the caller; the 8 warps split the K range, partials reduced in warp order.
template <int KWM, bool STAGED = false, typename XF, typename OUT>
__device__ __forceinline__ void gemv_task(int b0, int nb, int n0, int N, int k0, int k1, const float* __restrict__ wT,
                                          float* sx, float* spart, XF xf, OUT out) {
  // STAGED: sx already holds X[8][k1 - k0] (written and synchronised by the caller)
  // KWM >= rows per warp: every weight load of the warp's K-slice is issued before the first FMA
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int KL = k1 - k0;
  const int kw = (KL + NW - 1) / NW, ka = warp * kw, kb = min(KL, ka + kw);
  const int n = n0 + lane;
  float w[KWM];
#pragma unroll
  for (int u = 0; u < KWM; ++u) w[u] = (ka + u < kb && n < N) ? __ldg(wT + (int64_t)(k0 + ka + u) * N + n) : 0.f;
  if (!STAGED) {
    for (int i = tid; i < 8 * KL; i += NT) {
      const int it = i / KL, k = k0 + i % KL;
      sx[i] = it < nb ? xf(b0 + it, k) : 0.f;
    }
    __syncthreads();
  }
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll
  for (int u = 0; u < KWM; ++u)
    if (ka + u < kb)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(w[u], sx[i * KL + ka + u], acc[i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) spart[(warp * 8 + i) * 32 + lane] = acc[i];
  __syncthreads();
  {
    const int it = tid >> 5, c = tid & 31;
    if (it < nb && n0 + c < N) {
      float vsum = spart[it * 32 + c];
#pragma unroll
      for (int w2 = 1; w2 < NW; ++w2) vsum += spart[(w2 * 8 + it) * 32 + c];
      out(b0 + it, n0 + c, vsum);
    }
  }
  __syncthreads();
}

// gemv_task over NCB column blocks in one pass (X staged in sx[8][KL], K range [0, KL)): every weight
// load of the NCB blocks is in flight together; each output keeps gemv_task's summation order
// (the warp's K slice in k order, then the warps in order), so the values are the same.
template <int KWM, int NCB, typename OUT>
__device__ __forceinline__ void gemv_staged_blocks(int b0, int nb, int n0, int N, int KL, const float* __restrict__ wT,
                                                   const float* sx, float* spart, OUT out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kw = (KL + NW - 1) / NW, ka = warp * kw, kb = min(KL, ka + kw);
  float w[NCB][KWM];
#pragma unroll
  for (int j = 0; j < NCB; ++j)
#pragma unroll
    for (int u = 0; u < KWM; ++u) {
      const int n = n0 + 32 * j + lane;
      w[j][u] = (ka + u < kb && n < N) ? __ldg(wT + (int64_t)(ka + u) * N + n) : 0.f;
    }
  float acc[NCB][8];
#pragma unroll
  for (int j = 0; j < NCB; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[j][i] = 0.f;
#pragma unroll
  for (int u = 0; u < KWM; ++u)
    if (ka + u < kb)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float x = sx[i * KL + ka + u];
#pragma unroll
        for (int j = 0; j < NCB; ++j) acc[j][i] = fmaf(w[j][u], x, acc[j][i]);
      }
#pragma unroll
  for (int j = 0; j < NCB; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) spart[((warp * 8 + i) * NCB + j) * 32 + lane] = acc[j][i];
  __syncthreads();
  for (int e = tid; e < 8 * 32 * NCB; e += NT) {
    const int it = e / (32 * NCB), j = (e / 32) % NCB, cc = e % 32, n = n0 + 32 * j + cc;
    if (it < nb && n < N) {
      float vsum = spart[(it * NCB + j) * 32 + cc];
#pragma unroll
      for (int w2 = 1; w2 < NW; ++w2) vsum += spart[((w2 * 8 + it) * NCB + j) * 32 + cc];
      out(b0 + it, n, vsum);
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ tensor-core gate GEMM + LSTM cell
// tcgen05: D[128 rows = items][32 gate columns] in TMEM; A (the bf16 operand mirror, 64-column
// boxes of up to 128 item rows) and this CTA's 32 weight rows stream through a TMA ring; the
// epilogue warps apply the LSTM cell straight from TMEM.
constexpr uint32_t RING_BYTES = 160 * 1024;   // gate bulk-copy ring / attention staging area
constexpr int MAXGS = 10;                      // ring stages (W tile 16 KB + X tile items x 128 B)

struct GateSync {
  uint64_t full[MAXGS], empty[MAXGS], accf, acce, abar[2], amma[2];
  uint32_t tmem;
};
static_assert(2 * ASTAGE <= RING_BYTES && ACH * (ATT + EMB) * 4 <= RING_BYTES, "attention staging exceeds the ring");

// Gate GEMM with the WEIGHTS as the MMA's M operand: CTA c owns unit group ug = c / 4 (32 hidden
// units = 128 gate rows, ordered [unit][gate]) and K split ks = c % 4.  D[128 gate rows][items] =
// W[rows][K/4] . X[items][K/4]^T accumulates in TMEM (N = items padded to 16), so a tiny pooled
// batch costs a tiny N instead of a 128-row M tile, and each CTA issues 7 / 10 K-chunks of 4 MMAs.
// The 4 K-split partials of a group are written to global, the group syncs on a counter, and each
// CTA then sums the partials in split order (deterministic) for 8 of the 32 units and applies the
// LSTM cell.
// MODE 0: attention LSTM (X = [p | ctx | att_h(old bank)], K = 1792)
// MODE 1: decoder LSTM   (X = [ctx | att_h(new bank) | dec_h(old bank)], K = 2560)
constexpr int KSPLIT = 4;
constexpr uint32_t GW_TILE = 128 * 128;  // weight stage: 128 rows x 64 bf16

// tcgen05.mma kind::f16 with A (M = 128 rows, K = 16: 8 TMEM columns of bf16 pairs, low half = even
// k, lane = row) read from TMEM and B from shared memory
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

// K-chunk (64 columns) taken i-th by K-split ks.  X columns: attention gates [p 0..3 | ctx 4..11 |
// att_h 12..27], decoder gates [ctx 0..7 | att_h 8..23 | dec_h 24..39].  The chunks that depend on
// this step's prenet / context go last; the map is fixed, so the fp32 accumulation order (and the
// bits) do not depend on the pooled batch.
template <int MODE>
__device__ __forceinline__ int chunk_of(int ks, int i) {
#if DEC_SPREAD
  if (MODE == 0) return i < 6 ? 4 + ks * 6 + i : ks;                  // 6 others, then prenet chunk ks
  return i < 8 ? 8 + ks * 8 + i : 2 * ks + (i - 8);                   // 8 others, then context 2ks, 2ks+1
#else
  if (MODE == 0) return ks * 7 + (ks == 0 ? (i + 4) % 7 : i);
  return ks * 10 + (ks == 0 ? (i + 8) % 10 : i);
#endif
}

template <int MODE>
__device__ void gate_phase(const DecArgs& a, int s, uint8_t* ring, GateSync& gsy, uint32_t x_stage_bytes, int nst,
                           uint32_t& ring_par, uint32_t& lt_tile, const PlanCache& pc, unsigned& grp_gen, float* hs,
                           bool wres_cta, bool merged = false, unsigned ctx_target = 0, unsigned p_target = 0,
                           bool q_release = false) {
  // p_target (attention gates, PRE overlapped with this phase): split 0 loads its prenet chunks
  // once that many PRE tasks have been counted in
  constexpr int K = MODE == 0 ? KA : KD;
  constexpr int NKC = K / 64;
  constexpr int KCS = NKC / KSPLIT;
  const int c = blockIdx.x, ug = c >> 2, ks = c & 3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int oldb = s & 1, newb = oldb ^ 1;
  const int n16 = (a.B + 15) / 16 * 16;
  const bool tr = a.trace && c == 0 && lane == 0;
  const unsigned long long t_in = tr ? gtimer() : 0;
  auto mark = [&](int slot) {
    if (tr) a.trace[16 + MODE * 8 + slot] += gtimer() - t_in;
  };
  const bool comb = a.split && n16 <= 128;   // combined split stages (see k_dec_persist)
  const int nw = a.split == 1 ? 2 : 1;       // weight tiles per combined stage (Wh [, Wl])
  // decoder gates with the weights resident in TMEM (see DEC_WRES): a stage is the operand tile
  // only ([Xh | Xl] in the x2 split mode, [Xh] for bf16 products), so up to MAXGS stages are in flight
  const bool wres = MODE == DEC_WRES - 1 && wres_cta;
  const uint32_t xres_bytes = (a.split ? 2u : 1u) * (uint32_t)n16 * 128;
  const uint32_t sbytes = wres ? xres_bytes : nw * GW_TILE + 2 * (uint32_t)n16 * 128;
  if (wres) nst = min(MAXGS, (int)(RING_BYTES / xres_bytes));
  // stage st: the weight tile and the operand tile (combined split stages: Wh, [Wl,] Xh, Xl)
  auto sW = [&](uint32_t st) { return comb ? ring + st * sbytes : ring + st * GW_TILE; };
  auto sX = [&](uint32_t st) {
    return wres ? ring + st * sbytes
                : comb ? ring + st * sbytes + nw * GW_TILE : ring + nst * GW_TILE + st * x_stage_bytes;
  };
  // virtual stages per K-chunk when the split products do not share one stage: (Wh, Xh), (Wh, Xl)
  // [, (Wl, Xh)] -- the same product order as a combined stage
  const int nsub = (a.split && !comb) ? (a.split == 1 ? 3 : 2) : 1;
  // Ring slots: use v of this phase takes slot v % nst; the mbarrier parity of every slot is
  // tracked in the bit mask `ring_par` (flipped once per use), so phases may use different nst.
  // Producer lanes: use v goes to lane v % np; np <= nst keeps the empty-barrier parity unambiguous
  const int np = min(3, nst);
  const int nv = KCS * nsub;
  ++grp_gen;
  // Loads that do not depend on this phase's GEMM, issued now so their latency hides behind the
  // GEMM and the group sync: the group's slice of the next linear layer (query / projection)
  // and, for the first fixup round, the gate biases and cell states.
  constexpr int NP = MODE == 0 ? ATT : NMEL + 1;
  const int pn = threadIdx.x & 127;
  float wq[32];
  const int nmine = (a.B - ks + KSPLIT - 1) / KSPLIT;
  const int c_off = MODE == 0 ? ATTC_OFF : DECC_OFF;
  const float* bias = (MODE == 0 ? a.ba : a.bd) + ug * 128;
  float4 pre_b[4];
  float pre_c[4];
  auto prefetch = [&]() {  // issued by each warp after its GEMM-critical work
#pragma unroll
    for (int u = 0; u < 32; ++u)
      wq[u] = pn < NP ? __ldg((MODE == 0 ? a.WqT : a.WpT) + ((int64_t)ug * 32 + u) * NP + pn) : 0.f;
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const int e = threadIdx.x + z * NT, b = ks + KSPLIT * (e >> 5), ul = e & 31;
      const bool live = e < 32 * nmine && active(pc, b, s);
      pre_b[z] = live ? __ldg(reinterpret_cast<const float4*>(bias + ul * 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
      pre_c[z] = live ? ldf(a.work + (int64_t)b * ROW + c_off + ug * 32 + ul) : 0.f;
    }
  };
  if (warp == 0 || warp == 2 || warp == 3) {
    if (lane == 0) {
      const uint32_t pi = warp == 0 ? 0 : warp - 1;
      asm volatile("fence.proxy.async.global;" ::: "memory");  // xb tiles written by generic stores
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the ring doubles as PRE scratch
      uint32_t par = ring_par;
      // decoder gates, split 0: the context columns (chunks 0..7) go last -- in the merged-combine
      // schedule after the combined contexts of every live item are counted in.  The order is the
      // same in both schedules, so the fp32 accumulation (and the result bits) do not depend on
      // which schedule the batch size selects.
#if DEC_SPREAD
      // the chunks that wait on another CTA's output (context / prenet) are spread over the four
      // splits (2 context / 1 prenet chunk each, taken last), so after the wait each split loads
      // and multiplies 1-2 stages instead of split 0 alone loading 8 / 4
      const bool ctx_last = MODE == 1, p_last = MODE == 0;
#else
      const bool ctx_last = MODE == 1 && ks == 0;
      // attention gates, split 0: the prenet columns (chunks 0..3) go last, in both schedules
      // (PRE before this phase or overlapped with it), so the accumulation order is the same
      const bool p_last = MODE == 0 && ks == 0;
#endif
      bool ctx_ready = !(ctx_last && merged);
      bool p_ready = !(p_last && p_target);
      for (int v = 0; v < nv; ++v) {
        const uint32_t st = v % nst, ph = (par >> st) & 1;
        par ^= 1u << st;
        if (v % np != (int)pi) continue;
        const int i = v / nsub, sub = v - i * nsub;
        tcg::mbar_wait(&gsy.empty[st], ph ^ 1);
        const int kc = chunk_of<MODE>(ks, i), k0 = kc * 64;
        if (!ctx_ready && k0 < EMB) {
          wait_count(a.bar + 2 + NGRP, ctx_target);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // contexts written by generic stores
          ctx_ready = true;
        }
        if (!p_ready && k0 < PRE) {
          wait_count(a.bar + 3 + NGRP, p_target);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // prenet outputs written by generic stores
          p_ready = true;
        }
        int col;
        if (MODE == 0) col = k0 < 768 ? k0 : att_off(oldb) + (k0 - 768);
        else col = k0 < 512 ? CTX_OFF + k0 : (k0 < 1536 ? att_off(newb) + (k0 - 512) : dec_off(oldb) + (k0 - 1536));
        const int64_t wofs = ((int64_t)ug * NKC + kc) * 128 * 64, xofs = (int64_t)(col >> 6) * 128 * 64;
        if (wres) {   // [Xh | Xl] or [Xh]: the weights are in TMEM
          tcg::mbar_expect_tx(&gsy.full[st], sbytes);
          bulk_g2s(sX(st), a.xb + xofs, n16 * 128, &gsy.full[st]);
          if (a.split) bulk_g2s(sX(st) + n16 * 128, a.xbl + xofs, n16 * 128, &gsy.full[st]);
          continue;
        }
        if (comb) {   // [Wh | Wl | Xh | Xl]  (split 2: [Wh | Xh | Xl])
          tcg::mbar_expect_tx(&gsy.full[st], sbytes);
          bulk_g2s_hint(sW(st), (MODE == 0 ? a.Wa : a.Wd) + wofs, GW_TILE, &gsy.full[st], true);
          if (nw == 2) bulk_g2s_hint(sW(st) + GW_TILE, (MODE == 0 ? a.Wal : a.Wdl) + wofs, GW_TILE, &gsy.full[st], true);
          bulk_g2s(sX(st), a.xb + xofs, n16 * 128, &gsy.full[st]);
          bulk_g2s(sX(st) + n16 * 128, a.xbl + xofs, n16 * 128, &gsy.full[st]);
          continue;
        }
        const __nv_bfloat16* wsrc = sub == 2 ? (MODE == 0 ? a.Wal : a.Wdl) : (MODE == 0 ? a.Wa : a.Wd);
        const __nv_bfloat16* xsrc = sub == 1 ? a.xbl : a.xb;
        tcg::mbar_expect_tx(&gsy.full[st], GW_TILE + n16 * 128);
        bulk_g2s_hint(sW(st), wsrc + wofs, GW_TILE, &gsy.full[st], true);
        for (int blk = 0; blk * 128 < n16; ++blk)  // items 128 blk.. live in 128-row block blk of the mirror
          bulk_g2s(sX(st) + blk * 128 * 128, xsrc + xofs + (int64_t)blk * NCC * 128 * 64,
                   min(128, n16 - 128 * blk) * 128, &gsy.full[st]);
      }
      if (pi == 0) mark(0);
    }
    prefetch();
  } else if (warp == 1) {
    if (lane == 0) {
      // N = pooled rows padded to 16; above 256 rows two MMAs per K-step, rows 256.. into TMEM
      // columns 256.. (the accumulator columns stay item-indexed)
      const int nA = min(n16, 256), nB = n16 - nA;
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nA >> 3) << 17) | ((128u >> 4) << 24);
      const uint32_t idescB = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nB >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t XB_OFF = 256 * 128;  // bytes to the second N tile of an operand tile
      uint32_t par = ring_par;
      tcg::mbar_wait(&gsy.acce, (lt_tile & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int i = 0; i < nv; ++i) {
        const uint32_t st = i % nst, ph = (par >> st) & 1;
        par ^= 1u << st;
        tcg::mbar_wait(&gsy.full[st], ph);
        if (i == 0) mark(1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t dx = tcg::make_desc<128>(tcg::smem_u32(sX(st)));
        if (wres) {   // A = this K-chunk's weight rows in TMEM (same product order as the smem path)
          const uint32_t wa = gsy.tmem + WRES_COL + 32 * i;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_ts(gsy.tmem, wa + 8 * kk, dx + 2 * kk, idesc, (i | kk) != 0);
          if (a.split) {
            const uint64_t dxl = tcg::make_desc<128>(tcg::smem_u32(sX(st) + n16 * 128));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) umma_ts(gsy.tmem, wa + 8 * kk, dxl + 2 * kk, idesc, 1);
          }
          tcg::umma_commit(&gsy.empty[st]);
          continue;
        }
        const uint64_t dw = tcg::make_desc<128>(tcg::smem_u32(sW(st)));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tcg::umma_bf16(gsy.tmem, dw + 2 * kk, dx + 2 * kk, idesc, (i | kk) != 0);
        if (nB) {  // no combined stages above 128 rows: every product has its own (W, X) stage
          const uint64_t dx2 = tcg::make_desc<128>(tcg::smem_u32(sX(st) + XB_OFF));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) tcg::umma_bf16(gsy.tmem + 256, dw + 2 * kk, dx2 + 2 * kk, idescB, (i | kk) != 0);
        }
        if (comb) {   // + Wh.Xl [+ Wl.Xh] from the same stage
          const uint64_t dxl = tcg::make_desc<128>(tcg::smem_u32(sX(st) + n16 * 128));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) tcg::umma_bf16(gsy.tmem, dw + 2 * kk, dxl + 2 * kk, idesc, 1);
          if (nw == 2) {
            const uint64_t dwl = tcg::make_desc<128>(tcg::smem_u32(sW(st) + GW_TILE));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) tcg::umma_bf16(gsy.tmem, dwl + 2 * kk, dx + 2 * kk, idesc, 1);
          }
        }
        tcg::umma_commit(&gsy.empty[st]);
      }
      tcg::umma_commit(&gsy.accf);
      mark(2);
    }
    prefetch();
  } else {
    prefetch();
    // epilogue warps 4..7: TMEM lanes 32q.. = gate rows; columns = items -> K-split partial
    const int q = warp & 3, r = q * 32 + lane;
    float* part = a.Gp + ((int64_t)ks * GEMM_CTAS / KSPLIT + ug) * n16 * 128;  // [ks][ug][item][row]
    tcg::mbar_wait(&gsy.accf, lt_tile & 1);
    if (q == 0) mark(3);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < n16; c0 += 16) {
      float v[16];
      tcg::tmem_ld16(gsy.tmem + ((uint32_t)(q * 32) << 16) + c0, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) __stcg(part + (int64_t)(c0 + i) * 128 + r, v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) tcg::mbar_arrive(&gsy.acce);
    // group sync: the 4 K-split CTAs of this unit group have written their partials
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (warp == 4 && lane == 0) {  // release: the partials of the 4 epilogue warps (ordered by bar.sync)
      unsigned* cnt = a.bar + 2 + ug;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned seen;
      do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
      } while (seen < KSPLIT * grp_gen);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (q == 0) mark(4);
  }
  __syncthreads();
  {
    // fixup (all 256 threads): this CTA finishes all 32 units of the group for items b = ks + 4i;
    // 4 cells per thread in flight (partials + c state loaded before any arithmetic)
    const int h_off = MODE == 0 ? ATTH_OFF : DECH_OFF;
    const int hb_off = MODE == 0 ? att_off(newb) : dec_off(newb);
    for (int e0 = threadIdx.x; e0 < 32 * nmine; e0 += 4 * NT) {
      float4 gs4[4];
      float cold[4];
      bool live[4];
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        const int e = e0 + z * NT, b = ks + KSPLIT * (e >> 5), ul = e & 31, j = ug * 32 + ul;
        live[z] = e < 32 * nmine && active(pc, b, s);
        gs4[z] = make_float4(0.f, 0.f, 0.f, 0.f);
        cold[z] = 0.f;
        if (!live[z]) continue;
        const bool first = e0 == (int)threadIdx.x;  // prefetched before the GEMM
        gs4[z] = first ? pre_b[z] : __ldg(reinterpret_cast<const float4*>(bias + ul * 4));
#pragma unroll
        for (int k2 = 0; k2 < KSPLIT; ++k2) {
          const float4 pv = __ldcg(reinterpret_cast<const float4*>(
              a.Gp + (((int64_t)k2 * GEMM_CTAS / KSPLIT + ug) * n16 + b) * 128 + ul * 4));
          gs4[z].x += pv.x;
          gs4[z].y += pv.y;
          gs4[z].z += pv.z;
          gs4[z].w += pv.w;
        }
        cold[z] = first ? pre_c[z] : ldf(a.work + (int64_t)b * ROW + c_off + j);
      }
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        const int e = e0 + z * NT;
        if (e >= 32 * nmine) continue;
        const int b = ks + KSPLIT * (e >> 5), ul = e & 31, j = ug * 32 + ul;
        float hn = 0.f;
        if (live[z]) {
          const float cn = sigm_fast(gs4[z].y) * cold[z] + sigm_fast(gs4[z].x) * tanh_fast(gs4[z].z);
          hn = sigm_fast(gs4[z].w) * tanh_fast(cn);
          float* st = a.work + (int64_t)b * ROW;
          st[c_off + j] = cn;
          st[h_off + j] = hn;
          xb_store(a, b, hb_off + j, hn);
        }
        hs[e] = hn;
      }
    }
    WFENCE();
    __syncthreads();
    if (threadIdx.x == 0) mark(6);
    // this group's share of the next linear layer: query (MODE 0, 128 outputs) or the mel/gate
    // projection of dec_h (MODE 1, 81 outputs); 32-term dot products in unit order
    constexpr int N = NP;
    const int n = pn, half = threadIdx.x >> 7;
    if (n < N) {
      float* out = (MODE == 0 ? a.Qp : a.Pp) + (int64_t)ug * a.B * N + n;
      const float* w = wq;
      // 4 items per pass (independent FMA chains; each item's sum stays in unit order)
      for (int i0 = half; i0 < nmine; i0 += 8) {
        const float4* h4[4];
        float acc[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          h4[j] = reinterpret_cast<const float4*>(hs + min(i0 + 2 * j, nmine - 1) * 32);
          acc[j] = 0.f;
        }
#pragma unroll
        for (int u4 = 0; u4 < 8; ++u4)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 h = h4[j][u4];
            acc[j] = fmaf(w[4 * u4], h.x, acc[j]);
            acc[j] = fmaf(w[4 * u4 + 1], h.y, acc[j]);
            acc[j] = fmaf(w[4 * u4 + 2], h.z, acc[j]);
            acc[j] = fmaf(w[4 * u4 + 3], h.w, acc[j]);
          }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + 2 * j, b = ks + KSPLIT * i;
          if (i < nmine && active(pc, b, s)) out[(int64_t)b * N] = acc[j];
        }
      }
    }
    __syncthreads();
    if (MODE == 0 && q_release && threadIdx.x == 0)   // the query partials above (ordered by the barrier)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar + QCNT + ks) : "memory");
    if (threadIdx.x == 0) mark(5);
  }
  for (int v = 0; v < nv; ++v) ring_par ^= 1u << (v % nst);
  lt_tile += 1;
}

// ------------------------------------------------------------------ attention
struct AttSmem {
  // location features on the tensor cores: loc[a][t] = sum_k WL[a][k] . WIN[t][k], k = 32 c + tap
  // (tap 31 = 0), WL = the location conv composed with the location dense layer; both operands as
  // bf16 high / low parts in the UMMA 128B-swizzled K-major layout (A: 128 rows x 128 B, B: 32 x 128 B)
  __align__(1024) uint8_t wl[2][ATT * 128];
  __align__(1024) uint8_t win[2][2][32 * 128];   // [half-CTA][hi / lo]
  float q[2][ATT], sv[ATT];
  float red[32];
  float ered[2][4][32];        // [half][warp][position] partials of the energies (ATT-A)
  float scale[MAXCH];
  int tstart[MAXB + 1];        // prefix sum of chunks per item (ATT-A task list)
  float wp[2][ACH + 2 * HALO + 2], wa[2][ACH + 2 * HALO + 2], e[2][32];
};
// Generic scratch in the ring (free outside the gate pipeline / attention staging): the gate fixup's
// h values [32 x B/4] and PRE's last frame [8][80] + H1 [8][256] + gemv partials [8 warps][8][32]
constexpr int SCRATCH_F = 8 * NMEL + 8 * PRE + NW * 8 * 32 * 2;   // (gemv partials of 2 column blocks)
static_assert(SCRATCH_F * 4 <= RING_BYTES && 32 * (MAXB / 4) * 4 <= RING_BYTES, "ring scratch");


__device__ __forceinline__ float block_max(float v, float* red) {
  v = itts::warp_max(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) r = fmaxf(r, red[w]);
  return r;
}
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = itts::warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) r += red[w];
  return r;
}

// ATT-A for one (item b, chunk [ta, tb)).
// Thread 0: the chunk's processed-memory and memory rows (contiguous) -> a staging buffer.
__device__ __forceinline__ void att_prefetch(const DecArgs& a, int b, int ta, int tb, uint8_t* stage, uint64_t* bar) {
  const int64_t* p = a.plan + b * DPLAN;
  const int n = tb - ta;
  float* sPm = reinterpret_cast<float*>(stage);
  float* sMem = sPm + n * ATT;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tcg::mbar_expect_tx(bar, (uint32_t)n * (ATT + EMB) * 4);
  bulk_g2s_hint(sPm, reinterpret_cast<const float*>(p[1]) + (int64_t)ta * ATT, n * ATT * 4, bar, false);
  bulk_g2s_hint(sMem, reinterpret_cast<const float*>(p[0]) + (int64_t)ta * EMB, n * EMB * 4, bar, false);
}

// 128B-swizzled K-major UMMA tile element (row r, k < 64) of a [rows][64] bf16 tile
__device__ __forceinline__ int swz128(int r, int k) { return r * 64 + ((((k >> 3) ^ (r & 7))) << 3) + (k & 7); }

// ATT-A: the CTA's contiguous run of (item, 32-position chunk) tasks is dealt alternately to its
// two half-CTAs (4 warps each, own named barrier, ring buffer, mbarriers, TMEM columns and
// operand tiles), so the latency chains of two chunks -- row / q / window loads, the MMA round
// trip, the reductions -- overlap.  One task on half h:
//   rows    the chunk's pm / memory rows -> ring half h (bulk copies, issued first);
//   load    q (new item: the 32 unit-group partials, group order) and the location window;
//   mma     WIN (rows t < 32: [wp[t .. t+30], 0, wa[t .. t+30], 0], bf16 hi / lo) built from the
//           window; the location term D[128 dims][32 pos] = WL . WIN^T as one tcgen05 chain (x3
//           hi/lo products, fp32) into TMEM columns [32 h, 32 h + 32);
//   energy  thread (dim a): v_a tanh(q_a + D[a][t] + pm[t][a]) for the 32 positions, summed over
//           the warp's 32 dims by a shuffle reduce-scatter (lane t keeps position t) and over the
//           half's 4 warps in warp order;
//   softmax chunk max / exp / sum on the half's first warp (lane = position);
//   context thread d: dims d + 128 j summed over the chunk's positions in order.
// Every reduction order depends only on the chunk (batch transparency).
__device__ __forceinline__ void half_sync(int h) { asm volatile("bar.sync %0, 128;" ::"r"(3 + h) : "memory"); }

__device__ __forceinline__ void att_task(const DecArgs& a, AttSmem& sm, GateSync& gsy, uint8_t* ring, int s, int h,
                                         int b, int L, int ch, bool load_q, uint32_t& aph, uint32_t& mph,
                                         unsigned long long* tr_t, unsigned* item_cnt, unsigned q_target) {
  const int tid = threadIdx.x & 127, lane = tid & 31, qd = tid >> 5;
  const int ta = ch * 32, n = min(L, ta + 32) - ta;
  auto mark = [&](int slot) {
    if (tr_t) {
      const unsigned long long t2 = gtimer();
      a.trace[slot] += t2 - *tr_t;
      *tr_t = t2;
    }
  };
  uint8_t* stage = ring + h * ASTAGE;
  if (tid == 0) att_prefetch(a, b, ta, ta + n, stage, &gsy.abar[h]);
  if (load_q && q_target) {  // no barrier after the attention gates: the 32 groups' partials of b
    if (tid == 0) wait_count(a.bar + QCNT + (b & 3), q_target);
    half_sync(h);
  }
  if (load_q) {  // q = sum of the 32 unit-group partials, group order (kept for the item's next chunk)
    float qv[NGRP];
#pragma unroll
    for (int z = 0; z < NGRP; ++z) qv[z] = ldf(a.Qp + ((int64_t)z * a.B + b) * ATT + tid);
    float qa = qv[0];
#pragma unroll
    for (int z = 1; z < NGRP; ++z) qa += qv[z];
    sm.q[h][tid] = qa;
  }
  if (tid < ACH + 2 * HALO + 2) {  // window w_c[ta - 15 + i]: zero outside [0, L) and past the chunk's taps
    const int64_t* p = a.plan + b * DPLAN;
    const float* wsrc = reinterpret_cast<const float*>(a.step0 + s == 0 ? p[3] : p[4]);
    const int t = ta - HALO + tid;
    const bool in = tid < n + 2 * HALO && t >= 0 && t < L;
    sm.wp[h][tid] = in ? ldf(wsrc + t) : 0.f;
    sm.wa[h][tid] = in ? ldf(wsrc + L + t) : 0.f;
  }
  half_sync(h);
  mark(8);
#pragma unroll
  for (int r2 = 0; r2 < 2; ++r2) {  // WIN: thread -> (row t, 8-column group j), two per thread
    const int idx = tid + 128 * r2, t = idx >> 3, j = idx & 7, cch = j >> 2;
    const float* wv = cch ? sm.wa[h] : sm.wp[h];
    alignas(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int tap = (j & 3) * 8 + e;
      const float x = (t < n && tap < KLOC) ? wv[t + tap] : 0.f;
      hi[e] = __float2bfloat16_rn(x);
      lo[e] = __float2bfloat16_rn(x - __bfloat162float(hi[e]));
    }
    const int o = swz128(t, 8 * j);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(sm.win[h][0]) + o) = *reinterpret_cast<const uint4*>(hi);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(sm.win[h][1]) + o) = *reinterpret_cast<const uint4*>(lo);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  half_sync(h);
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t dwh = tcg::make_desc<128>(tcg::smem_u32(sm.wl[0])), dwl = tcg::make_desc<128>(tcg::smem_u32(sm.wl[1]));
    const uint64_t dxh = tcg::make_desc<128>(tcg::smem_u32(sm.win[h][0]));
    const uint64_t dxl = tcg::make_desc<128>(tcg::smem_u32(sm.win[h][1]));
    const uint32_t d = gsy.tmem + 32 * h;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) tcg::umma_bf16(d, dwh + 2 * kk, dxh + 2 * kk, idesc, kk != 0);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) tcg::umma_bf16(d, dwh + 2 * kk, dxl + 2 * kk, idesc, 1);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) tcg::umma_bf16(d, dwl + 2 * kk, dxh + 2 * kk, idesc, 1);
    tcg::umma_commit(&gsy.amma[h]);
  }
  const float* sPm = reinterpret_cast<const float*>(stage);
  tcg::mbar_wait(&gsy.abar[h], aph);   // the chunk's pm / memory rows
  aph ^= 1;
  mark(9);
  {
    const int ad = qd * 32 + lane;
    tcg::mbar_wait(&gsy.amma[h], mph);
    mph ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float x[32];
    tcg::tmem_ld32(gsy.tmem + ((uint32_t)(qd * 32) << 16) + 32 * h, x);
    const float qa = sm.q[h][ad], va = sm.sv[ad];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = i < n ? va * tanh_fast((qa + x[i]) + sPm[i * ATT + ad]) : 0.f;
#pragma unroll
    for (int st = 16; st >= 1; st >>= 1) {  // reduce-scatter: lane t ends with position t
      const bool up = lane & st;
#pragma unroll
      for (int i = 0; i < st; ++i) {
        const float send = up ? x[i] : x[i + st], keep = up ? x[i + st] : x[i];
        x[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
      }
    }
    sm.ered[h][qd][lane] = x[0];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  half_sync(h);
  mark(10);
  if (qd == 0) {  // chunk softmax statistics: lane = position
    const float e = ((sm.ered[h][0][lane] + sm.ered[h][1][lane]) + sm.ered[h][2][lane]) + sm.ered[h][3][lane];
    const float M = itts::warp_max(lane < n ? e : -INFINITY);
    const float xv = lane < n ? expf(e - M) : 0.f;
    const float Ssum = itts::warp_sum(xv);
    sm.e[h][lane] = xv;
    if (lane < n) a.U[(int64_t)b * a.u_ld + ta + lane] = xv;
    if (lane == 0) {
      float* ap = a.AP + ((int64_t)b * MAXCH + ch) * (2 + EMB);
      ap[0] = M;
      ap[1] = Ssum;
    }
  }
  half_sync(h);
  mark(11);
  {  // unnormalised context partial: thread -> dims tid + 128 j, positions in order
    const float* sMem = sPm + n * ATT;
    float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
    for (int t = 0; t < n; ++t) {   // (unrolled: the shared-memory loads of 8 positions issue together)
      const float w = sm.e[h][t];
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] = fmaf(w, sMem[t * EMB + tid + 128 * j], c[j]);
    }
    float* ap = a.AP + ((int64_t)b * MAXCH + ch) * (2 + EMB);
#pragma unroll
    for (int j = 0; j < 4; ++j) ap[2 + tid + 128 * j] = c[j];
  }
  half_sync(h);   // ring half / e / q reuse
  if (item_cnt && tid == 0)  // this chunk's U / AP stores (ordered by the half barrier) are visible
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(item_cnt) : "memory");
  mark(12);
  if (tr_t) a.trace[13] += 1;
}

// ATT-B for item b: combine the chunks (max, sum, context partial; chunk order) -> context, W, W_acc.
// Part `part` of `nparts`: context dims [part, part + 1) x 512 / nparts and attention positions
// [part, part + 1) x ceil(L / nparts) (the chunk statistics are recomputed by every part); every
// value is computed the same way for any nparts.
__device__ void att_combine(const DecArgs& a, AttSmem& sm, int s, int b, int chunk, int part = 0, int nparts = 1) {
  const int tid = threadIdx.x;
  const int64_t* p = a.plan + b * DPLAN;
  const int L = (int)p[2];
  const int nch = (L + chunk - 1) / chunk;
  const float* wsrc = reinterpret_cast<const float*>(a.step0 + s == 0 ? p[3] : p[4]);
  float* wdst = reinterpret_cast<float*>(p[4]);
  const float* ap = a.AP + (int64_t)b * MAXCH * (2 + EMB);
  float* scale = sm.scale;  // [MAXCH]
  const float mc = tid < nch ? ldf(ap + tid * (2 + EMB)) : -INFINITY;
  const float sc = tid < nch ? ldf(ap + tid * (2 + EMB) + 1) : 0.f;
  const float M = block_max(mc, sm.red);
  const float ec = tid < nch ? expf(mc - M) : 0.f;
  const float Z = block_sum(sc * ec, sm.red);  // chunk order within a warp, then warp order
  if (tid < nch) scale[tid] = ec / Z;
  __syncthreads();
  float* st = a.work + (int64_t)b * ROW;
  const int d0 = part * (EMB / nparts), d1 = d0 + EMB / nparts;
  // both context dims of this thread at once, 8 chunk partials each in flight per round, every dim
  // summed in chunk order
  constexpr int ND = EMB / NT, CR = 8;
  float c[ND];
#pragma unroll
  for (int r = 0; r < ND; ++r) c[r] = 0.f;
  for (int k = 0; k < nch; k += CR) {
    float v[ND][CR];
#pragma unroll
    for (int r = 0; r < ND; ++r)
#pragma unroll
      for (int j = 0; j < CR; ++j) {
        const int d = d0 + tid + r * NT;
        v[r][j] = (d < d1 && k + j < nch) ? ldf(ap + (k + j) * (2 + EMB) + 2 + d) : 0.f;
      }
#pragma unroll
    for (int r = 0; r < ND; ++r)
#pragma unroll
      for (int j = 0; j < CR; ++j)
        if (k + j < nch) c[r] = fmaf(scale[k + j], v[r][j], c[r]);
  }
#pragma unroll
  for (int r = 0; r < ND; ++r) {
    const int d = d0 + tid + r * NT;
    if (d >= d1) continue;
    st[CTX_OFF + d] = c[r];
    xb_store(a, b, CTX_OFF + d, c[r]);
  }
  WFENCE();
  const int lp = (L + nparts - 1) / nparts, t1 = min(L, (part + 1) * lp);
  for (int t = part * lp + tid; t < t1; t += NT) {
    const float w = ldf(a.U + (int64_t)b * a.u_ld + t) * scale[t / chunk];
    const float acc = ldf(wsrc + L + t);
    wdst[t] = w;
    wdst[L + t] = acc + w;
  }
  __syncthreads();
}

// att_combine for the merged schedule (the decoder-gate CTAs wait for these contexts): the chunk
// statistics, the first CPF context partials and the first attention positions are loaded together
// (one L2 round trip before the reductions), and `ctx_cnt` is released as soon as the context is
// stored, before W / W_acc, which only the next step's attention reads.  Same arithmetic and order
// as att_combine.  (Kept separate: the same early loads in the separate ATT-B phase of larger
// batches, or one templated body for both, measured 1.5-2 % slower decoder chunks at B >= 128.)
#ifndef DEC_CPF
#define DEC_CPF 16
#endif
constexpr int CPF = DEC_CPF;   // chunk partials per context dim loaded with the statistics
constexpr int CPR = 8;         // then CPR partial loads in flight per round
__device__ void att_combine_early(const DecArgs& a, AttSmem& sm, int s, int b, int chunk, int part, int nparts,
                                  unsigned* ctx_cnt, unsigned chunks_target) {
  const int tid = threadIdx.x;
  const int64_t* p = a.plan + b * DPLAN;
  const int L = (int)p[2];
  const int nch = (L + chunk - 1) / chunk;
  if (chunks_target) {  // no barrier after ATT-A: wait for this item's chunk tasks of step s
    if (tid == 0) wait_count(a.bar + ITEM_CNT + b, chunks_target);
    __syncthreads();
  }
  const float* wsrc = reinterpret_cast<const float*>(a.step0 + s == 0 ? p[3] : p[4]);
  float* wdst = reinterpret_cast<float*>(p[4]);
  const float* ap = a.AP + (int64_t)b * MAXCH * (2 + EMB);
  float* scale = sm.scale;  // [MAXCH]
  const int d0 = part * (EMB / nparts), d1 = d0 + EMB / nparts;
  const int lp = (L + nparts - 1) / nparts, t1 = min(L, (part + 1) * lp);
  const float mc = tid < nch ? ldf(ap + tid * (2 + EMB)) : -INFINITY;
  const float sc = tid < nch ? ldf(ap + tid * (2 + EMB) + 1) : 0.f;
  float pv[EMB / NT][CPF];
#pragma unroll
  for (int r = 0; r < EMB / NT; ++r)
#pragma unroll
    for (int k = 0; k < CPF; ++k) {
      const int d = d0 + tid + r * NT;
      pv[r][k] = (d < d1 && k < nch) ? ldf(ap + k * (2 + EMB) + 2 + d) : 0.f;
    }
  const int tw = part * lp + tid;
  const float u0 = tw < t1 ? ldf(a.U + (int64_t)b * a.u_ld + tw) : 0.f;
  const float acc0 = tw < t1 ? ldf(wsrc + L + tw) : 0.f;
  const float M = block_max(mc, sm.red);
  const float ec = tid < nch ? expf(mc - M) : 0.f;
  const float Z = block_sum(sc * ec, sm.red);  // chunk order within a warp, then warp order
  if (tid < nch) scale[tid] = ec / Z;
  __syncthreads();
  float* st = a.work + (int64_t)b * ROW;
#pragma unroll
  for (int r = 0; r < EMB / NT; ++r) {
    const int d = d0 + tid + r * NT;
    if (d >= d1) continue;
    float c = 0.f;
#pragma unroll
    for (int k = 0; k < CPF; ++k)
      if (k < nch) c = fmaf(scale[k], pv[r][k], c);
    int k = CPF;
    for (; k < nch; k += CPR) {  // CPR partial loads in flight, summed in chunk order
      float v[CPR];
#pragma unroll
      for (int jj = 0; jj < CPR; ++jj) v[jj] = k + jj < nch ? ldf(ap + (k + jj) * (2 + EMB) + 2 + d) : 0.f;
#pragma unroll
      for (int jj = 0; jj < CPR; ++jj)
        if (k + jj < nch) c = fmaf(scale[k + jj], v[jj], c);
    }
    st[CTX_OFF + d] = c;
    xb_store(a, b, CTX_OFF + d, c);
  }
  WFENCE();
  __syncthreads();
  if (tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctx_cnt) : "memory");
  if (tw < t1) {
    const float w = u0 * scale[tw / chunk];
    wdst[tw] = w;
    wdst[L + tw] = acc0 + w;
  }
  for (int t = tw + NT; t < t1; t += NT) {
    const float w = ldf(a.U + (int64_t)b * a.u_ld + t) * scale[t / chunk];
    const float acc = ldf(wsrc + L + t);
    wdst[t] = w;
    wdst[L + t] = acc + w;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(NT, 1)
    k_dec_persist(DecArgs a, uint32_t a_box_bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = tcg::align_smem_1024(smem_raw);
  AttSmem& sm = *reinterpret_cast<AttSmem*>(ring + RING_BYTES);  // ring = gate pipeline / attention staging
  // Split mode with <= 128 pooled rows: one ring stage holds [Wh | Wl | Xh | Xl] and feeds all three
  // products (no tile loaded twice); larger batches use three (W, X) stages per K-chunk.
  const bool comb = a.split && a_box_bytes <= 128u * 128u;
  const uint32_t comb_bytes = (a.split == 1 ? 2 : 1) * GW_TILE + 2 * a_box_bytes;
  const int nst = min(MAXGS, (int)(RING_BYTES / (comb ? comb_bytes : GW_TILE + a_box_bytes)));
  __shared__ GateSync gsy;
  __shared__ PlanCache pc;
  const int tid = threadIdx.x, G = gridDim.x, c = blockIdx.x;
  const bool gemm_cta = c < GEMM_CTAS;
  unsigned gen = 0;
  uint32_t ring_par = 0, lt_tile = 0, aphase[2] = {0, 0}, mphase[2] = {0, 0};
  unsigned grp_gen = 0;

  if (tid == 0) {
    for (int i = 0; i < MAXGS; ++i) {
      tcg::mbar_init(&gsy.full[i], 1);
      tcg::mbar_init(&gsy.empty[i], 1);
    }
    tcg::mbar_init(&gsy.accf, 1);
    tcg::mbar_init(&gsy.acce, 4);
    tcg::mbar_init(&gsy.abar[0], 1);
    tcg::mbar_init(&gsy.abar[1], 1);
    tcg::mbar_init(&gsy.amma[0], 1);
    tcg::mbar_init(&gsy.amma[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // gate CTAs: accumulator columns = rows (2 N tiles above 256); every CTA: ATT-A location features
  // in columns [0, 64) (two pipeline buffers; free between gate phases)
  // gate CTAs with the decoder-gate weights resident: columns [WRES_COL, 512) hold them (n16 <= 128)
  const bool wres = DEC_WRES && gemm_cta && a.split != 1 && a_box_bytes <= 128u * 128u;
  const uint32_t tcols = !gemm_cta ? 64u : (wres || a_box_bytes > 256u * 128u) ? 512u : 256u;
  if ((tid >> 5) == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tcg::smem_u32(&gsy.tmem)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if constexpr (DEC_WRES > 0) if (wres) {
    // this CTA's resident gate-weight rows (unit group c / 4, K-split c % 4, chunks in chunk_of
    // order) -> TMEM: warps w and w + 4 own lane quarter w % 4 (row r = lane of the quarter) and
    // take alternate chunks; the swizzled 16-byte pieces of a row are read in k order
    constexpr int WM = DEC_WRES - 1, NKC = (WM == 0 ? KA : KD) / 64, KCS = NKC / KSPLIT;
    const int q = (tid >> 5) & 3, r = q * 32 + (tid & 31);
    for (int i = tid >> 7; i < KCS; i += 2) {
      const __nv_bfloat16* src = (WM == 0 ? a.Wa : a.Wd) + (((int64_t)(c >> 2) * NKC + chunk_of<WM>(c & 3, i)) * 128 + r) * 64;
      uint32_t w[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(src) + (j ^ (r & 7)));
        w[4 * j] = u.x, w[4 * j + 1] = u.y, w[4 * j + 2] = u.z, w[4 * j + 3] = u.w;
      }
      tmem_st32(gsy.tmem + ((uint32_t)(q * 32) << 16) + WRES_COL + 32 * i, w);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  for (int b = tid; b < a.B; b += NT) {
    pc.L[b] = (int)a.plan[b * DPLAN + 2];
    pc.steps[b] = (int)a.plan[b * DPLAN + 5];
  }
  // attention constants (resident for the whole chunk): WL[a][32 c + tap] as bf16 hi / lo UMMA tiles
  for (int i = tid; i < ATT * 64; i += NT) {
    const int ad = i >> 6, k = i & 63, cch = k >> 5, tap = k & 31;
    const float x = tap < KLOC ? __ldg(a.WlocD + (cch * KLOC + tap) * ATT + ad) : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    reinterpret_cast<__nv_bfloat16*>(sm.wl[0])[swz128(ad, k)] = hi;
    reinterpret_cast<__nv_bfloat16*>(sm.wl[1])[swz128(ad, k)] = __float2bfloat16_rn(x - __bfloat162float(hi));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid < ATT) sm.sv[tid] = __ldg(a.v + tid);
  __syncthreads();
  // bf16 operand mirror, bank 0, from the gathered fp32 state rows
  for (int b = c; b < a.B; b += G) {
    const float* st = a.work + (int64_t)b * ROW;
    for (int i = tid; i < ATTC_OFF; i += NT) xb_store(a, b, i, ldf(st + i));
  }
  WFENCE();
  grid_sync(a.bar, gen);

  // Fixed 32-position attention chunks: an item's softmax / context reduction order then depends on
  // its own L only, so a request decodes to the same bits in any pooled batch (batch transparency,
  // reference SPEC.md:232); one chunk = the N of one location-term MMA chain.
  constexpr int chunk = 32;
  const int nb8 = (a.B + 7) / 8;
  // Small batches: PRE runs on the CTAs without a gate group, overlapped with the attention-gate
  // phase (splits 1..3 need no prenet columns; split 0 takes its prenet chunks last and waits on a
  // counter) -- one grid barrier and one latency-bound phase fewer per step
  const int n_aux = G - GEMM_CTAS;
  const bool prem = n_aux > 0 && nb8 * 4 <= n_aux;
  // PRE tasks: column blocks per task minimising rounds x (mel + H1 + cpt x p-block) (~5 + 3 cpt us);
  // the arithmetic of every value is the same for any choice
  int pre_cpt = 1;
  if (prem) {
    pre_cpt = nb8 * 8 <= n_aux ? 1 : 2;
  } else {
    int best = 1 << 30;
    for (int cpt = 1; cpt <= 8; cpt *= 2) {
      const int cost = ((nb8 * (8 / cpt) + G - 1) / G) * (5 + 3 * cpt);
      if (cost < best) best = cost, pre_cpt = cpt;
    }
  }
  const bool merged = a.B <= DEC_MERGE_B;  // ATT-B folded into the decoder-gate phase
  const bool icnt = DEC_ITEM_CNT && merged;  // per-item chunk counters instead of the ATT-A barrier

  unsigned long long tph = gtimer(), tacc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  int ph_i = 0;
  unsigned long long t_sync = 0;   // trace: when this CTA left its last grid barrier
  auto phase_end = [&]() {
    grid_sync(a.bar, gen);
    if (a.trace && tid == 0) t_sync = gtimer();
    if (a.trace && c == 0 && tid == 0) {
      const unsigned long long now = gtimer();
      tacc[ph_i] += now - tph;
      tph = now;
    }
    ph_i = ph_i == (merged ? 3 : 4) - (prem ? 1 : 0) - (icnt ? 2 : 0) ? 0 : ph_i + 1;
  };
  // mel / gate value k of item b for the step whose projection partials are in Pp (group order, ctx last)
  auto mel_value = [&](int b, int k) {
    float pv[NGRP + 1];
#pragma unroll
    for (int z = 0; z <= NGRP; ++z) pv[z] = ldf(a.Pp + ((int64_t)z * a.B + b) * 81 + k);
    float m = __ldg(a.bp + k);
#pragma unroll
    for (int z = 0; z <= NGRP; ++z) m += pv[z];
    return m;
  };
  float* ringf = reinterpret_cast<float*>(ring);  // generic scratch outside the gate / staging uses
  unsigned ctx_target = 0;                         // combined contexts so far (merged ATT-B)
  unsigned pre_target = 0;                         // PRE tasks so far (overlapped schedule)
  for (int s = 0; s < a.nsteps; ++s) {
    const int gs = a.step0 + s;
    // ---- PRE: finish mel(s-1); H1 = relu(W0 . last) for the task's 8 items; p = relu(W1 . H1)
    // task = (8 items, pre_cpt blocks of 32 prenet columns): mel and H1 are computed once per task
    const int n_pre = nb8 * (8 / pre_cpt);
    unsigned pre_done = 0;
    for (int task = prem ? c - GEMM_CTAS : c; task < n_pre; task += prem ? n_aux : G) {
      if (task < 0) break;   // gate CTAs in the overlapped schedule
      ++pre_done;
      const int b0 = (task / (8 / pre_cpt)) * 8, cb0 = (task % (8 / pre_cpt)) * pre_cpt, nb = min(8, a.B - b0);
      const int n0 = cb0 * 32;
      const bool trp = a.trace && c == (prem ? GEMM_CTAS : 0) && tid == 0;   // first PRE CTA
      unsigned long long tp0 = trp ? gtimer() : 0;
      if (trp && s > 0) a.trace[15] += tp0 - t_sync;
      auto pmark = [&](int slot) {
        if (trp) {
          const unsigned long long t1 = gtimer();
          a.trace[slot] += t1 - tp0;
          tp0 = t1;
        }
      };
      float* sx = ringf;                 // [8][80]
      float* sh = sx + 8 * NMEL;         // [8][256]
      float* gsc = sh + 8 * PRE;         // gemv partials

      {  // warp w: item b0 + w; lane l: mel / gate values k = l, l + 32, l + 64 (< 81), all 3 x 34
         // partial loads in flight before the sums
        const int it = tid >> 5, lane = tid & 31, b = b0 + it;
        const bool was = it < nb && s > 0 && active(pc, b, gs - 1);
        float m[3] = {0.f, 0.f, 0.f};
        if (was) {
          float pv[3][NGRP + 1];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int k = lane + 32 * j;
#pragma unroll
            for (int z = 0; z <= NGRP; ++z) pv[j][z] = k < 81 ? ldf(a.Pp + ((int64_t)z * a.B + b) * 81 + k) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int k = lane + 32 * j;
            m[j] = k < 81 ? __ldg(a.bp + k) : 0.f;
#pragma unroll
            for (int z = 0; z <= NGRP; ++z) m[j] += pv[j][z];
          }
        }
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int k = lane + 32 * j;
          if (k >= 81) continue;
          if (k < NMEL)
            sx[it * NMEL + k] = it >= nb ? 0.f : was ? m[j] : ldf(a.work + (int64_t)b * ROW + LAST_OFF + k);
          if (n0 == 0 && was) {
            const int64_t* p = a.plan + b * DPLAN;
            if (k < NMEL) {
              reinterpret_cast<float*>(p[6])[(gs - 1) * NMEL + k] = m[j];
              a.work[(int64_t)b * ROW + LAST_OFF + k] = m[j];
            } else {
              reinterpret_cast<float*>(p[7])[gs - 1] = m[j];
            }
          }
        }
      }
      __syncthreads();
      pmark(5);
      {  // thread n: unit n of H1 for the 8 items (k order)
        static_assert(NT == PRE, "one thread per prenet unit");
        float acc[8];
#pragma unroll
        for (int it = 0; it < 8; ++it) acc[it] = 0.f;
        const float4* sx4 = reinterpret_cast<const float4*>(sx);
        constexpr int H1U = DEC_H1_UNROLL;   // k4 iterations (4 W0 loads each) unrolled together
#pragma unroll H1U
        for (int k4 = 0; k4 < NMEL / 4; ++k4) {
          float w[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) w[j] = __ldg(a.W0T + (4 * k4 + j) * PRE + tid);
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const float4 x = sx4[it * (NMEL / 4) + k4];
            acc[it] = fmaf(w[0], x.x, acc[it]);
            acc[it] = fmaf(w[1], x.y, acc[it]);
            acc[it] = fmaf(w[2], x.z, acc[it]);
            acc[it] = fmaf(w[3], x.w, acc[it]);
          }
        }
#pragma unroll
        for (int it = 0; it < 8; ++it) sh[it * PRE + tid] = fmaxf(acc[it], 0.f);
      }
      __syncthreads();
      pmark(6);
      auto p_out = [&](int b, int n, float y) {
        if (!active(pc, b, gs)) return;
        y = fmaxf(y, 0.f);
        a.work[(int64_t)b * ROW + P_OFF + n] = y;
        xb_store(a, b, P_OFF + n, y);
      };
      if (pre_cpt == 2)   // both column blocks' weight loads in flight together
        gemv_staged_blocks<32, 2>(b0, nb, n0, PRE, PRE, a.W1T, sh, gsc, p_out);
      else
        for (int cb = cb0; cb < cb0 + pre_cpt; ++cb)
          gemv_task<32, true>(b0, nb, cb * 32, PRE, 0, PRE, a.W1T, sh, gsc, [&](int b, int k) { return 0.f; }, p_out);
      WFENCE();
      pmark(7);
    }
    if (prem) {   // ---- overlapped: count the finished PRE tasks in, run the attention gates
      pre_target += (unsigned)n_pre;
      if (tid == 0 && pre_done)
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.bar + 3 + NGRP), "r"(pre_done) : "memory");
      if (a.trace && c == GEMM_CTAS && tid == 0 && s > 0) a.trace[14] += gtimer() - t_sync;
      if (gemm_cta) gate_phase<0>(a, gs, ring, gsy, a_box_bytes, nst, ring_par, lt_tile, pc, grp_gen, ringf, wres, false, 0,
                                  pre_target, icnt);
    } else {
      phase_end();
      // ---- ATT gates + cell + query partials
      if (gemm_cta) gate_phase<0>(a, gs, ring, gsy, a_box_bytes, nst, ring_par, lt_tile, pc, grp_gen, ringf, wres, false, 0,
                                  0, icnt);
    }
    if (icnt) __syncthreads();   // this CTA's gate / PRE work (TMEM columns, ring scratch) is done
    else phase_end();
    // ---- ATT-A: the non-empty (item, chunk) tasks of the live items, dealt round-robin
    if (tid < 32) {  // task prefix over items: 16 items per lane, then a warp scan
      constexpr int PL = MAXB / 32;
      auto cnt = [&](int b) { return (b < a.B && active(pc, b, gs)) ? (pc.L[b] + chunk - 1) / chunk : 0; };
      int loc = 0;
      for (int i = 0; i < PL; ++i) loc += cnt(tid * PL + i);
      int incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += y;
      }
      int run = incl - loc;
      for (int i = 0; i < PL; ++i) {
        const int b = tid * PL + i;
        if (b <= a.B) sm.tstart[b] = run;
        run += cnt(b);
      }
      if (tid == 31) sm.tstart[a.B] = run;  // the total (also for B == MAXB)
    }
    __syncthreads();
    {
      const int ntask = sm.tstart[a.B];
      // CTA c takes a contiguous run of tasks (consecutive chunks of one item share its q), dealt
      // alternately to its two half-CTAs
      const int t0 = (int)((int64_t)c * ntask / G), t1 = (int)((int64_t)(c + 1) * ntask / G);
      const int h = tid >> 7;
      unsigned long long tq = (a.trace && c == 0 && tid == 0) ? gtimer() : 0;
      int bi = 0, bprev = -1;
      for (int task = t0 + h; task < t1; task += 2) {
        while (sm.tstart[bi + 1] <= task) ++bi;
        att_task(a, sm, gsy, ring, gs, h, bi, pc.L[bi], task - sm.tstart[bi], bi != bprev, aphase[h], mphase[h],
                 (a.trace && c == 0 && tid == 0) ? &tq : nullptr, icnt ? a.bar + ITEM_CNT + bi : nullptr,
                 icnt ? (unsigned)(NGRP * (s + 1)) : 0u);
        bprev = bi;
      }
    }
    if (icnt) __syncthreads();   // this CTA's attention work (TMEM columns, ring) is done
    else phase_end();
    // ---- ATT-B: combine the chunks of every live item -> context, W, W_acc
    if (!merged) {
      for (int b = c; b < a.B; b += G)
        if (active(pc, b, gs)) att_combine(a, sm, gs, b, chunk);
      phase_end();
    } else {
      // At most n_aux items: on the CTAs without a gate group only, so every gate CTA starts its
      // GEMM at once (the context chunks are the last two of each split).  Otherwise on every CTA
      // but split 0 of each gate group, before their GEMM.  Small batches split each item's
      // combine into up to 4 parts so more CTAs share it (the values do not depend on the split).
      const bool aux_only = n_aux > 0 && a.B <= n_aux;
      const int ncomb = aux_only ? n_aux : 3 * (GEMM_CTAS / 4) + n_aux;
      const int nparts = a.B * 4 <= ncomb ? 4 : a.B * 2 <= ncomb ? 2 : 1;
      for (int b = 0; b < a.B; ++b) ctx_target += active(pc, b, gs) ? (unsigned)nparts : 0u;
      const bool combiner = aux_only ? !gemm_cta : !(gemm_cta && (c & 3) == 0);
      if (combiner) {
        const int ci = !gemm_cta ? (aux_only ? 0 : 3 * (GEMM_CTAS / 4)) + (c - GEMM_CTAS) : (c >> 2) * 3 + (c & 3) - 1;
        for (int task = ci; task < a.B * nparts; task += ncomb) {
          const int b = task / nparts;
          if (active(pc, b, gs))   // releases one count on the context counter, ends with __syncthreads
            att_combine_early(a, sm, gs, b, chunk, task % nparts, nparts, a.bar + 2 + NGRP,
                              icnt ? (unsigned)(((pc.L[b] + chunk - 1) / chunk) * (s + 1)) : 0u);
        }
      }
    }
    // ---- DEC gates + cell + projection partials of dec_h; the other CTAs project the context
    if (gemm_cta) gate_phase<1>(a, gs, ring, gsy, a_box_bytes, nst, ring_par, lt_tile, pc, grp_gen, ringf, wres,
                                merged, ctx_target);
    {
      const int c0 = G > GEMM_CTAS ? GEMM_CTAS : 0, nsp = G - c0;
      if (merged && c >= c0 && c - c0 < nb8 * 3) {  // the contexts of all live items
        if (tid == 0) wait_count(a.bar + 2 + NGRP, ctx_target);
        __syncthreads();
      }
      if (c >= c0)
        for (int task = c - c0; task < nb8 * 3; task += nsp) {
          const int b0 = (task / 3) * 8, n0 = (task % 3) * 32, nb = min(8, a.B - b0);
          gemv_task<EMB / NW>(b0, nb, n0, NMEL + 1, HID, HID + EMB, a.WpT, ringf, ringf + 8 * EMB,
                              [&](int b, int k) { return ldf(a.work + (int64_t)b * ROW + CTX_OFF + k - HID); },
                              [&](int b, int n, float y) {
                                if (active(pc, b, gs)) a.Pp[((int64_t)NGRP * a.B + b) * 81 + n] = y;
                              });
        }
    }
    phase_end();
  }
  // ---- finish mel of the last step
  {
    const int gs = a.step0 + a.nsteps;
    for (int i = c * NT + tid; i < a.B * 81; i += G * NT) {
      const int b = i / 81, k = i % 81;
      if (!active(pc, b, gs - 1)) continue;
      const float m = mel_value(b, k);
      const int64_t* p = a.plan + b * DPLAN;
      if (k < NMEL) {
        reinterpret_cast<float*>(p[6])[(gs - 1) * NMEL + k] = m;
        a.work[(int64_t)b * ROW + LAST_OFF + k] = m;
      } else {
        reinterpret_cast<float*>(p[7])[gs - 1] = m;
      }
    }
  }
  if (a.trace && c == 0 && tid == 0)
    for (int i = 0; i < 5; ++i) a.trace[i] = tacc[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if ((tid >> 5) == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(gsy.tmem), "r"(tcols));
  }
}

}  // namespace

// Debug: later itts_r_decode_persistent launches add per-phase wall time (ns, CTA 0, summed over
// the steps) to buf[0..4]: PRE, ATT gates (+query), ATT-A, ATT-B, DEC gates (+projection).  null = off.
ITTS_API int itts_r_decode_debug_trace(void* buf) {
  g_dec_trace = static_cast<unsigned long long*>(buf);
  return ITTS_OK;
}

// Runs `nsteps` decoder steps for B gathered rows (see DecArgs).  Scratch buffers are owned by
// the caller; `bar` (2 + 32 u32) is zeroed here on the stream.  grid = min(#SMs, 148) CTAs.
ITTS_API int itts_r_decode_persistent(int32_t B, int32_t nsteps, const int64_t* plan, float* work, void* xb,
                                      const float* W0T, const float* W1T, const void* Wa, const float* ba,
                                      const void* Wd, const float* bd, const float* WqT, const float* WlocD,
                                      const float* v, const float* WpT, const float* bp,
                                      float* Gp, float* H1, float* Qp, float* Pp, float* U, int64_t u_ld,
                                      float* AP, unsigned* bar, const void* Wa_lo, const void* Wd_lo,
                                      int32_t split_x, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  if (B > MAXB) return ITTS_EUNSUPPORTED;  // plan cache / attention task table in shared memory
  if (nsteps <= 0 || !plan || !work || !xb || !Wa || !Wd || !bar) return ITTS_EINVAL;
  if (tcg::num_sms() < GEMM_CTAS) return ITTS_EUNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  if ((Wa_lo == nullptr) != (Wd_lo == nullptr)) return ITTS_EINVAL;
  // 1: split weights and operands (x3 products); 2: bf16-exact weights, split operands (x2)
  const int split = Wa_lo != nullptr ? 1 : (split_x ? 2 : 0);
  // split mode: the mirror buffer holds the high parts, then the low parts (same tile layout)
  __nv_bfloat16* xbh = (__nv_bfloat16*)xb;
  __nv_bfloat16* xbl = split ? xbh + (int64_t)((B + 127) / 128) * NCC * 128 * 64 : nullptr;
  DecArgs a{B, nsteps, 0, plan, work, xbh, xbl, W0T, W1T, (const __nv_bfloat16*)Wa, ba,
            (const __nv_bfloat16*)Wd, (const __nv_bfloat16*)Wa_lo, (const __nv_bfloat16*)Wd_lo, split, bd,
            WqT, WlocD, v, WpT, bp, Gp, H1, Qp, Pp, U, u_ld, AP, bar, g_dec_trace};
  const size_t smem = 1024 + RING_BYTES + sizeof(AttSmem);
  const int b16 = (B + 15) / 16 * 16;
  uint32_t a_box_bytes = (uint32_t)b16 * 128;  // X stage: all items x 64 columns
  static uint64_t configured = 0;
  if (!(configured & itts::device_bit())) {
    cudaError_t e = cudaFuncSetAttribute(k_dec_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    configured |= itts::device_bit();
  }
  static_assert(QCNT >= 2 + NGRP + 2 && ITEM_CNT >= QCNT + 4, "counter ranges overlap");
  cudaError_t e = cudaMemsetAsync(bar, 0, (ITEM_CNT + B) * sizeof(unsigned), st);
  if (e != cudaSuccess) return (int)e;
  const int G = tcg::num_sms();
  void* args[] = {&a, &a_box_bytes};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelExC(&cfg, (const void*)k_dec_persist, args);
  return e == cudaSuccess ? ITTS_OK : (int)e;
}
