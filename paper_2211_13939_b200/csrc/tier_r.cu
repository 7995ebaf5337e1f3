// Tier R: Tacotron2 encoder / decoder-step chain and the HiFi-GAN chunk helpers.
//
// Reference boundary: the same three module calls as Tier S
// (encode_batch / decode_chunk_batch / vocode_batch, pkg/src/incrtts/
// acoustic.py:222-238, vocoder.py:139-143) with the stand-in arithmetic
// replaced by Tacotron2 + HiFi-GAN V1 (paper Eq. 1-3).
// The GEMM-shaped parts (encoder convs, BiLSTM input projection, the two
// decoder LSTM gate GEMMs, every HiFi-GAN conv) run on tcgen05 through
// tc_conv.cu; this file holds everything else:
//
//   K5  k_enc_embed      paper Eq. 1: sum of the 4 embedding rows -> bf16 conv input
//       k_bilstm         bidirectional LSTM recurrence, one 8-CTA cluster per
//                        (item, direction); W_hh slice resident in smem, h
//                        broadcast through distributed shared memory
//       k_pmem           processed memory = memory . W_mem^T
//   K6  k_dec_prepare    bf16 operand mirror of the gathered state rows
//       k_prenet         2 x (linear + ReLU), dropout off
//       k_lstm_cell      gates -> (h, c) for the attention / decoder LSTMCell
//       k_query          attention query q = Wq . att_h (item-tiled)
//       k_attention      location-sensitive attention: location conv,
//                        energies, masked softmax, context, W_acc += W
//       k_proj           mel / gate projection, writes the chunk's frame
//   K7  k_mel_assemble   [mel_tail; mel] -> zero-haloed bf16 conv_pre input
//       k_rowmap         per-stage row maps (halo / transpose-conv phase rows)
//       k_zero_halo      re-zero halo rows of a bf16 operand buffer
//       k_post_splice    conv_post + tanh + Eq.-3 cross-fade / hold-back
//
// Decoder state row (fp32, gathered per call by K1, slots.cu):
//   [p 256 | ctx 512 | att_h 1024 | dec_h 1024 | att_c 1024 | dec_c 1024 | last 80]
// so the two gate GEMM operands are contiguous column slices of one bf16
// mirror: X_att = [p|ctx|att_h] (K=1792), X_dec = [ctx|att_h|dec_h] (K=2560).

#include <algorithm>
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int NMEL = 80, EMB = 512, HID = 1024, PRE = 256, ATT = 128, NF = 32, KLOC = 31, EH = 256;
constexpr int P_OFF = 0, CTX_OFF = 256, ATTH_OFF = 768, DECH_OFF = 1792, ATTC_OFF = 2816, DECC_OFF = 3840,
              LAST_OFF = 4864, ROW = 4944, XB_ROW = 2816;
constexpr int DPLAN = 8;  // decoder plan width

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

// ----------------------------------------------------------------- decoder
// plan[b] = {mem_ptr, pm_ptr, L, w_src_ptr, w_dst_ptr, steps, mel_ptr, gate_ptr}

__global__ void k_dec_prepare(const float* __restrict__ state, __nv_bfloat16* __restrict__ xb) {
  const float* s = state + (int64_t)blockIdx.x * ROW;
  __nv_bfloat16* x = xb + (int64_t)blockIdx.x * XB_ROW;
  for (int i = threadIdx.x; i < XB_ROW; i += blockDim.x) x[i] = __float2bfloat16_rn(s[i]);
}

// Small batched GEMVs (prenet, attention query, mel/gate projection):
// Y[b][n] = sum_k X[b][k] W^T[k][n].  A CTA serves IT items (weights read
// once per IT items) with its 8 warps splitting K (each warp streams a
// contiguous K slice, lanes cover N with NPL outputs each, several weight
// loads in flight per iteration); partials are reduced across warps in a
// fixed order, so results do not depend on the batch composition.
constexpr int IT = 8;
constexpr int GW = 8;  // warps per CTA
constexpr int QKS = 8;  // K slices of the attention query GEMV (partials summed by k_attention)

struct GemvIO {
  const float* x;   // rows of the input, x_ld floats apart
  int x_ld, off0, len0, off1, len1;  // up to two input segments (K = len0 + len1)
  const float* wT;  // [K][N]
  int N;
  // epilogue targets
  float* y; int y_ld, y_off;          // fp32 output rows (may alias the state rows)
  __nv_bfloat16* yb; int yb_ld;       // optional bf16 mirror (same column offset)
  const float* bias;                  // optional
  int relu;
  const int64_t* plan; int step;      // proj mode: plan rows + step (mel / gate outputs)
};

// Epilogue of one output element (generic: bias, ReLU, fp32 + optional bf16 mirror;
// projection mode: state.last_frame + the chunk's mel / gate outputs).
template <int MODE>
__device__ __forceinline__ void gemv_store(const GemvIO& io, int b, int n, float v) {
  if (io.bias) v += io.bias[n];
  if (MODE == 0) {
    if (io.plan && io.step >= io.plan[b * DPLAN + 5]) return;
    if (io.relu) v = fmaxf(v, 0.f);
    io.y[(int64_t)b * io.y_ld + io.y_off + n] = v;
    if (io.yb) io.yb[(int64_t)b * io.yb_ld + io.y_off + n] = __float2bfloat16_rn(v);
  } else {
    const int64_t* p = io.plan + b * DPLAN;
    if (io.step >= p[5]) return;
    if (n < NMEL) {
      io.y[(int64_t)b * io.y_ld + LAST_OFF + n] = v;
      reinterpret_cast<float*>(p[6])[io.step * NMEL + n] = v;
    } else {
      reinterpret_cast<float*>(p[7])[io.step] = v;
    }
  }
}

// Grid (item tiles of IT, column tiles of 32*NPL, K slices).  The CTA's 8 warps split its
// K slice; warp partials are reduced in a fixed order.  With one K slice the epilogue is
// applied here; otherwise partials go to `part_out` [KS][B][N] and k_gemv_finish (or the
// consumer) sums them in slice order.
template <int NPL, int MODE>
__global__ void __launch_bounds__(GW * 32) k_gemv(GemvIO io, int B, float* __restrict__ part_out) {
  const int b0 = blockIdx.x * IT, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = min(IT, B - b0);
  const int n0 = blockIdx.y * 32 * NPL;
  const int K = io.len0 + io.len1, KS = gridDim.z;
  const int ks0 = (int)((int64_t)K * blockIdx.z / KS), ks1 = (int)((int64_t)K * (blockIdx.z + 1) / KS);
  const int KL = ks1 - ks0;
  extern __shared__ float sm[];
  float* xs = sm;                       // [IT][KL]
  float* part = sm + IT * KL;           // [GW][IT][32*NPL]
  for (int i = tid; i < IT * KL; i += GW * 32) {
    const int it = i / KL, k = ks0 + i % KL;
    float v = 0.f;
    if (it < nb) {
      const float* row = io.x + (int64_t)(b0 + it) * io.x_ld;
      v = k < io.len0 ? row[io.off0 + k] : row[io.off1 + k - io.len0];
    }
    xs[i] = v;
  }
  __syncthreads();
  const int kw = (KL + GW - 1) / GW, k0 = warp * kw, k1 = min(KL, k0 + kw);
  float acc[IT][NPL];
#pragma unroll
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int j = 0; j < NPL; ++j) acc[i][j] = 0.f;
  int k = k0;
  for (; k + 4 <= k1; k += 4) {  // 4*NPL independent weight loads in flight per iteration
    float w[4][NPL];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        const int n = n0 + lane + 32 * j;
        w[u][j] = n < io.N ? __ldg(io.wT + (int64_t)(ks0 + k + u) * io.N + n) : 0.f;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        const float xv = xs[i * KL + k + u];
#pragma unroll
        for (int j = 0; j < NPL; ++j) acc[i][j] = fmaf(w[u][j], xv, acc[i][j]);
      }
  }
  for (; k < k1; ++k) {
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int n = n0 + lane + 32 * j;
      const float w = n < io.N ? __ldg(io.wT + (int64_t)(ks0 + k) * io.N + n) : 0.f;
#pragma unroll
      for (int i = 0; i < IT; ++i) acc[i][j] = fmaf(w, xs[i * KL + k], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int j = 0; j < NPL; ++j) part[(warp * IT + i) * (NPL * 32) + lane + 32 * j] = acc[i][j];
  __syncthreads();
  for (int e = tid; e < nb * NPL * 32; e += GW * 32) {
    const int it = e / (NPL * 32), c = e % (NPL * 32), n = n0 + c, b = b0 + it;
    if (n >= io.N) continue;
    float v = part[it * (NPL * 32) + c];
#pragma unroll
    for (int w = 1; w < GW; ++w) v += part[(w * IT + it) * (NPL * 32) + c];
    if (KS == 1) gemv_store<MODE>(io, b, n, v);
    else part_out[((int64_t)blockIdx.z * B + b) * io.N + n] = v;
  }
}

template <int MODE>
__global__ void k_gemv_finish(GemvIO io, int B, int KS, const float* __restrict__ part) {
  const int e = blockIdx.x * 256 + threadIdx.x;
  if (e >= B * io.N) return;
  const int b = e / io.N, n = e % io.N;
  float v = part[e];
  for (int z = 1; z < KS; ++z) v += part[(int64_t)z * B * io.N + e];
  gemv_store<MODE>(io, b, n, v);
}

// part: scratch of KS*B*N floats (only when KS > 1).  finish=false leaves the partials
// for the consumer (the attention kernel sums query slices itself).
template <int NPL, int MODE>
int launch_gemv(const GemvIO& io, int B, int KS, float* part, bool finish, cudaStream_t st) {
  const int K = io.len0 + io.len1;
  const int KL = (K + KS - 1) / KS + 1;
  const size_t smem = (size_t)(IT * KL + GW * IT * NPL * 32) * 4;
  static uint64_t configured = 0;
  if (!(configured & itts::device_bit())) {
    cudaFuncSetAttribute(k_gemv<NPL, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured |= itts::device_bit();
  }
  dim3 grid((B + IT - 1) / IT, (io.N + 32 * NPL - 1) / (32 * NPL), KS);
  k_gemv<NPL, MODE><<<grid, GW * 32, smem, st>>>(io, B, part);
  if (KS > 1 && finish) k_gemv_finish<MODE><<<(B * io.N + 255) / 256, 256, 0, st>>>(io, B, KS, part);
  ITTS_RETURN_LAUNCH();
}

// G = nsplit K-split partial slices [nsplit][B][4096], summed in fixed order (+ bias).
__global__ void __launch_bounds__(256) k_lstm_cell(const float* __restrict__ G, int nsplit,
                                                   const float* __restrict__ bias, float* __restrict__ state,
                                                   __nv_bfloat16* __restrict__ xb, int h_off, int c_off,
                                                   const int64_t* __restrict__ plan, int step, int B) {
  const int idx = blockIdx.x * 256 + threadIdx.x;
  const int b = idx / HID, j = idx % HID;
  if (b >= B || step >= plan[b * DPLAN + 5]) return;
  float gate[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float a = G[(int64_t)b * 4 * HID + q * HID + j];
    for (int z = 1; z < nsplit; ++z) a += G[((int64_t)z * B + b) * 4 * HID + q * HID + j];
    gate[q] = a + bias[q * HID + j];
  }
  float* s = state + (int64_t)b * ROW;
  const float c = sigm(gate[1]) * s[c_off + j] + sigm(gate[0]) * tanhf(gate[2]);
  const float h = sigm(gate[3]) * tanhf(c);
  s[c_off + j] = c;
  s[h_off + j] = h;
  xb[(int64_t)b * XB_ROW + h_off + j] = __float2bfloat16_rn(h);
}

// One CL-CTA cluster per item (8 warps each; CL = 8 for small pooled batches, 4 otherwise):
// CTA r owns text positions [r*L/CL, (r+1)*L/CL) for the location features, energies,
// softmax numerators and the partial context; the softmax max / sum and the context are
// reduced across the cluster through distributed shared memory in rank order
// (deterministic, independent of the batch).
// Q = query K-slice partials [QKS][B][128], Wloc [32][2][31], WdT [32][128], v [128].
//
// Latency structure: every global load of a phase is issued before the first use (weights
// staged with float4 loads, pm rows for 4 positions per warp in flight while the location
// features are contracted), so a step costs a handful of memory round trips.
constexpr int AT_WARPS = 8;
constexpr int LT = 128;  // positions per location-feature tile

template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(AT_WARPS * 32, 3)
    k_attention(float* __restrict__ state, __nv_bfloat16* __restrict__ xb, const int64_t* __restrict__ plan,
                const float* __restrict__ Q, const float* __restrict__ Wloc, const float* __restrict__ WdT,
                const float* __restrict__ v, int step) {
  constexpr int NT = AT_WARPS * 32, HALO = (KLOC - 1) / 2;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CL, B = gridDim.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t* p = plan + b * DPLAN;
  if (step >= p[5]) return;  // the whole cluster returns together
  const float* mem = reinterpret_cast<const float*>(p[0]);
  const float* pm = reinterpret_cast<const float*>(p[1]);
  const int L = (int)p[2];
  const float* wsrc = reinterpret_cast<const float*>(step == 0 ? p[3] : p[4]);
  float* wdst = reinterpret_cast<float*>(p[4]);
  const int t_lo = (int)((int64_t)L * rank / CL), t_hi = (int)((int64_t)L * (rank + 1) / CL);
  const int Ls = t_hi - t_lo, Lh = Ls + 2 * HALO;

  extern __shared__ float dyn[];
  float* w_prev = dyn;             // [Lh] positions t_lo-HALO .. t_hi+HALO (zero outside [0, L))
  float* w_acc = dyn + Lh;         // [Lh]
  float* e = dyn + 2 * Lh;         // [Ls]
  float* locf = dyn + ((2 * Lh + Ls + 3) & ~3);  // [LT][33]; later the context partials
  __shared__ __align__(16) float q[ATT], sv[ATT], sWd[NF * ATT], sWlT[2 * KLOC * NF];  // sWlT[c][k][f]
  __shared__ float red[32];
  __shared__ float cl_max[CL], cl_sum[CL];
  __shared__ __align__(16) float ctx_local[EMB];

  // ---- prologue: all loads in flight, then the shared-memory stores
  {
    constexpr int NWL = NF * 2 * KLOC / 4, NWD = NF * ATT / 4;  // float4 counts (496, 1024)
    float4 wl[(NWL + NT - 1) / NT], wd[NWD / NT];
    const float4* wl4 = reinterpret_cast<const float4*>(Wloc);
    const float4* wd4 = reinterpret_cast<const float4*>(WdT);
#pragma unroll
    for (int r = 0; r < (NWL + NT - 1) / NT; ++r)
      if (tid + r * NT < NWL) wl[r] = __ldg(wl4 + tid + r * NT);
#pragma unroll
    for (int r = 0; r < NWD / NT; ++r) wd[r] = __ldg(wd4 + tid + r * NT);
    float qz[QKS];
    if (tid < ATT) {
#pragma unroll
      for (int z = 0; z < QKS; ++z) qz[z] = Q[((int64_t)z * B + b) * ATT + tid];
    }
    float wp[2], wa[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = tid + r * NT, t = t_lo - HALO + i;
      const bool in = i < Lh && t >= 0 && t < L;
      wp[r] = in ? wsrc[t] : 0.f;
      wa[r] = in ? wsrc[L + t] : 0.f;
    }
    for (int i = tid + 2 * NT; i < Lh; i += NT) {  // long texts only
      const int t = t_lo - HALO + i;
      const bool in = t >= 0 && t < L;
      w_prev[i] = in ? wsrc[t] : 0.f;
      w_acc[i] = in ? wsrc[L + t] : 0.f;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (tid + r * NT < Lh) {
        w_prev[tid + r * NT] = wp[r];
        w_acc[tid + r * NT] = wa[r];
      }
#pragma unroll
    for (int r = 0; r < (NWL + NT - 1) / NT; ++r) {
      const int i4 = tid + r * NT;
      if (i4 < NWL) {
        const float w4[4] = {wl[r].x, wl[r].y, wl[r].z, wl[r].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // source [f][c][k] -> [c][k][f]
          const int src = 4 * i4 + u, f = src / (2 * KLOC), ck = src - f * 2 * KLOC;
          sWlT[ck * NF + f] = w4[u];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < NWD / NT; ++r) reinterpret_cast<float4*>(sWd)[tid + r * NT] = wd[r];
    if (tid < ATT) {
      float qa = qz[0];
#pragma unroll
      for (int z = 1; z < QKS; ++z) qa += qz[z];  // query K-slices, fixed order
      q[tid] = qa;
      sv[tid] = v[tid];
    }
  }
  __syncthreads();

  // ---- location features + energies, LT positions at a time.  Energies: 8 lanes per position
  // (lane sl holds dims 4sl..4sl+3 of each 32-dim quarter), 4 positions per warp in flight.
  const int sub = lane >> 3, sl = lane & 7;
  for (int t0 = 0; t0 < Ls; t0 += LT) {
    const int nt = min(LT, Ls - t0);
    for (int i = tid; i < nt * NF; i += NT) {
      const int tl = t0 + i / NF, f = i % NF;  // local position; halo index = tl + k
      float c = 0.f;
#pragma unroll
      for (int k = 0; k < KLOC; ++k)
        c = fmaf(sWlT[k * NF + f], w_prev[tl + k], fmaf(sWlT[(KLOC + k) * NF + f], w_acc[tl + k], c));
      locf[(i / NF) * (NF + 1) + f] = c;
    }
    __syncthreads();
    for (int tt = warp * 4 + sub; tt - sub < nt; tt += AT_WARPS * 4) {
      const bool live = tt < nt;
      float4 pv[4];
      const float4* prow = reinterpret_cast<const float4*>(pm + (int64_t)(t_lo + t0 + (live ? tt : 0)) * ATT);
#pragma unroll
      for (int j = 0; j < 4; ++j) pv[j] = prow[8 * j + sl];
      float loc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) loc[i] = 0.f;
      const float* lf = locf + (live ? tt : 0) * (NF + 1);
#pragma unroll 8
      for (int f = 0; f < NF; ++f) {
        const float cf = lf[f];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 w4 = reinterpret_cast<const float4*>(sWd + f * ATT)[8 * j + sl];
          loc[4 * j] = fmaf(w4.x, cf, loc[4 * j]);
          loc[4 * j + 1] = fmaf(w4.y, cf, loc[4 * j + 1]);
          loc[4 * j + 2] = fmaf(w4.z, cf, loc[4 * j + 2]);
          loc[4 * j + 3] = fmaf(w4.w, cf, loc[4 * j + 3]);
        }
      }
      float en = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int a0 = 32 * j + 4 * sl;
        const float pa[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) en = fmaf(sv[a0 + u], tanhf((q[a0 + u] + loc[4 * j + u]) + pa[u]), en);
      }
      en += __shfl_xor_sync(0xffffffffu, en, 4);
      en += __shfl_xor_sync(0xffffffffu, en, 2);
      en += __shfl_xor_sync(0xffffffffu, en, 1);
      if (live && sl == 0) e[t0 + tt] = en;
    }
    __syncthreads();
  }
  // softmax over the whole text: cluster max, then cluster sum (rank order)
  float lmax = -INFINITY;
  for (int t = tid; t < Ls; t += NT) lmax = fmaxf(lmax, e[t]);
  lmax = itts::block_reduce<float, true>(lmax, red);
  if (tid < CL) *cluster.map_shared_rank(&cl_max[rank], tid) = lmax;
  cluster.sync();
  float M = cl_max[0];
#pragma unroll
  for (int r = 1; r < CL; ++r) M = fmaxf(M, cl_max[r]);
  float lsum = 0.f;
  for (int t = tid; t < Ls; t += NT) {
    const float x = expf(e[t] - M);
    e[t] = x;
    lsum += x;
  }
  lsum = itts::block_reduce<float, false>(lsum, red);
  if (tid < CL) *cluster.map_shared_rank(&cl_sum[rank], tid) = lsum;
  cluster.sync();
  float Z = cl_sum[0];
#pragma unroll
  for (int r = 1; r < CL; ++r) Z += cl_sum[r];
  const float iz = 1.0f / Z;
  for (int t = tid; t < Ls; t += NT) {
    const float a = e[t] * iz;
    e[t] = a;
    wdst[t_lo + t] = a;
    wdst[L + t_lo + t] = w_acc[HALO + t] + a;
  }
  __syncthreads();
  // partial context over this CTA's positions: warp w takes rows t = w (mod 8), lane 16 dims
  float4 acc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* mem4 = reinterpret_cast<const float4*>(mem);
#pragma unroll 4
  for (int t = warp; t < Ls; t += AT_WARPS) {
    const float a = e[t];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 m4 = mem4[(int64_t)(t_lo + t) * (EMB / 4) + lane + 32 * j];
      acc[j].x = fmaf(a, m4.x, acc[j].x);
      acc[j].y = fmaf(a, m4.y, acc[j].y);
      acc[j].z = fmaf(a, m4.z, acc[j].z);
      acc[j].w = fmaf(a, m4.w, acc[j].w);
    }
  }
  float4 (*cpart)[EMB / 4] = reinterpret_cast<float4 (*)[EMB / 4]>(locf);  // [AT_WARPS][128]
#pragma unroll
  for (int j = 0; j < 4; ++j) cpart[warp][lane + 32 * j] = acc[j];
  __syncthreads();
  const float* cp = reinterpret_cast<const float*>(cpart);
  for (int d = tid; d < EMB; d += NT) {
    float c = cp[d];
#pragma unroll
    for (int w = 1; w < AT_WARPS; ++w) c += cp[w * EMB + d];
    ctx_local[d] = c;
  }
  cluster.sync();
  if (rank == 0) {
    float* s = state + (int64_t)b * ROW;
    for (int d = tid; d < EMB; d += NT) {
      float c = ctx_local[d];
#pragma unroll
      for (int r = 1; r < CL; ++r) c += cluster.map_shared_rank(ctx_local, r)[d];
      s[CTX_OFF + d] = c;
      xb[(int64_t)b * XB_ROW + CTX_OFF + d] = __float2bfloat16_rn(c);
    }
  }
  cluster.sync();  // keep every CTA's shared memory alive until rank 0 has read it
}

// ----------------------------------------------------------------- encoder
// plan[i] = {tok_off, L, row_base (first valid row), mem_ptr, pm_ptr, 0}
constexpr int EPLAN = 6;
#ifndef BILSTM_TC_MIN
#define BILSTM_TC_MIN 96   // pooled encoder batches from which the tensor-core BiLSTM wins (measured crossover)
#endif

template <typename OutT>
__global__ void k_enc_embed(const int32_t* __restrict__ tok4, int64_t total, const int64_t* __restrict__ plan,
                            const float* __restrict__ Eph, const float* __restrict__ Epw,
                            const float* __restrict__ Epph, const float* __restrict__ Eiph,
                            OutT* __restrict__ X) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int64_t* p = plan + blockIdx.y * EPLAN;
  const int64_t L = p[1];
  const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (g >= L * EMB) return;
  const int64_t t = g / EMB;
  const int c = (int)(g % EMB);
  const int64_t idx = p[0] + t;
  const float v = ((Eph[(int64_t)tok4[idx] * EMB + c] + Epw[(int64_t)tok4[total + idx] * EMB + c]) +
                   Epph[(int64_t)tok4[2 * total + idx] * EMB + c]) + Eiph[(int64_t)tok4[3 * total + idx] * EMB + c];
  if constexpr (sizeof(OutT) == 4) X[(p[2] + t) * EMB + c] = v;
  else X[(p[2] + t) * EMB + c] = __float2bfloat16_rn(v);
}

// Split-bf16 parity encoder: fp32 activations [rows][512] (valid rows of each item) -> the bf16
// operand [rows][1536] = [hi | lo | hi] (hi = bf16(v), lo = bf16(v - hi)), so one tensor-core conv
// against weights [Wh | Wh | Wl] computes Wh.Xh + Wh.Xl + Wl.Xh (fp32-level products, fp32
// accumulation).  relu: apply max(v, 0) first.  Halo rows are never written (zero from a memset).
__global__ void k_split3(const float* __restrict__ src, const int64_t* __restrict__ plan, int relu,
                         __nv_bfloat16* __restrict__ dst) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int64_t* p = plan + blockIdx.y * EPLAN;
  const int64_t L = p[1];
  const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (g >= L * EMB) return;
  const int64_t row = p[2] + g / EMB;
  const int c = (int)(g % EMB);
  float v = src[row * EMB + c];
  if (relu) v = fmaxf(v, 0.f);
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
  __nv_bfloat16* d = dst + row * (3 * EMB) + c;
  d[0] = hi;
  d[EMB] = lo;
  d[2 * EMB] = hi;
}

// One 8-CTA cluster per (item, direction).  CTA r owns hidden units
// [32r, 32r+32): gate rows {g*256 + 32r + u}.  WhhT [2][256 k][1024 rows].
// PRE [rows][2048] = x . W_ih^T + b_ih + b_hh for both directions.
// Thread (row r, K half) keeps its 128 recurrent weights in registers.  The 32 new h values of a
// CTA go to every CTA of the cluster with st.async, which completes bytes on the receiver's
// mbarrier: a step waits only for the 1 KB of h it needs (double-buffered), no cluster barrier.
constexpr int BL_CLUSTER = 8, BL_UNITS = EH / BL_CLUSTER, BL_ROWS = 4 * BL_UNITS;

__device__ __forceinline__ uint32_t cl_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cl_map(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(bar), "r"(parity) : "memory");
}

__global__ void __cluster_dims__(BL_CLUSTER, 1, 1) __launch_bounds__(256, 1)
    k_bilstm(const float* __restrict__ PRE, const int64_t* __restrict__ plan, const float* __restrict__ WhhT) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int pair = blockIdx.x / BL_CLUSTER;
  const int item = pair >> 1, dir = pair & 1;
  const int tid = threadIdx.x;
  itts::pdl_trigger();

  __shared__ __align__(16) float hbuf[2][EH];
  __shared__ float gpart[2][BL_ROWS];
  __shared__ float cst[BL_UNITS];
  __shared__ __align__(8) uint64_t hbar[2];
  const float* Wd = WhhT + (int64_t)dir * EH * 4 * EH;  // this direction's [256 k][1024 rows]
  const int r = tid % BL_ROWS, half = tid / BL_ROWS;    // 2 K-halves of 128
  const int grow = (r / BL_UNITS) * EH + rank * BL_UNITS + (r % BL_UNITS);
  float w[128];
#pragma unroll
  for (int k = 0; k < 128; ++k) w[k] = __ldg(Wd + (int64_t)(half * 128 + k) * (4 * EH) + grow);
  itts::pdl_wait();  // the input projection PRE comes from the previous kernel
  const int64_t* p = plan + item * EPLAN;
  const int64_t L = p[1], row0 = p[2];
  float* mem = reinterpret_cast<float*>(p[3]);
  for (int i = tid; i < EH; i += 256) hbuf[0][i] = 0.f;
  if (tid < BL_UNITS) cst[tid] = 0.f;
  const uint32_t bar0 = cl_smem_u32(&hbar[0]);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();
  auto expect = [&](int b) {  // this CTA's next phase of hbar[b] receives 8 x 32 h values
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar0 + 8 * b), "r"(EH * 4)
                 : "memory");
  };
  if (tid == 0 && L > 1) expect(1);  // h_1

  // the input projection of step s+1 does not depend on h: load it while step s computes
  float4 pre_n = make_float4(0.f, 0.f, 0.f, 0.f);
  auto load_pre = [&](int64_t s) {
    if (tid < BL_UNITS && s < L) {
      const int64_t t = dir ? L - 1 - s : s;
      const float* pre = PRE + (row0 + t) * (8 * EH) + dir * 4 * EH;
      const int j = rank * BL_UNITS + tid;
      pre_n = make_float4(pre[j], pre[EH + j], pre[2 * EH + j], pre[3 * EH + j]);
    }
  };
  load_pre(0);
  for (int64_t s = 0; s < L; ++s) {
    const int64_t t = dir ? L - 1 - s : s;
    const int cur = (int)(s & 1);
    if (s > 0) {
      cl_mbar_wait(bar0 + 8 * cur, (uint32_t)((s - 1) >> 1) & 1u);
      if (tid == 0 && s + 2 < L) expect(cur);  // h_{s+2} lands in this buffer next
    } else if (tid == 0 && L > 2) {
      expect(0);  // h_2
    }
    const float4* h4 = reinterpret_cast<const float4*>(hbuf[cur] + half * 128);
    const float4 pre_c = pre_n;
    load_pre(s + 1);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;  // four independent FMA chains
#pragma unroll
    for (int k4 = 0; k4 < 32; ++k4) {
      const float4 h = h4[k4];
      a0 = fmaf(w[4 * k4], h.x, a0);
      a1 = fmaf(w[4 * k4 + 1], h.y, a1);
      a2 = fmaf(w[4 * k4 + 2], h.z, a2);
      a3 = fmaf(w[4 * k4 + 3], h.w, a3);
    }
    gpart[half][r] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (tid < BL_UNITS) {
      const int u = tid, j = rank * BL_UNITS + u;
      float gi = pre_c.x + (gpart[0][u] + gpart[1][u]);
      float gf = pre_c.y + (gpart[0][BL_UNITS + u] + gpart[1][BL_UNITS + u]);
      float gg = pre_c.z + (gpart[0][2 * BL_UNITS + u] + gpart[1][2 * BL_UNITS + u]);
      float go = pre_c.w + (gpart[0][3 * BL_UNITS + u] + gpart[1][3 * BL_UNITS + u]);
      const float c = sigm(gf) * cst[u] + sigm(gi) * tanhf(gg);
      const float hn = sigm(go) * tanhf(c);
      cst[u] = c;
      mem[t * EMB + dir * EH + j] = hn;
      if (s + 1 < L) {
        const uint32_t dst = cl_smem_u32(&hbuf[cur ^ 1][j]), bar = bar0 + 8 * (cur ^ 1);
#pragma unroll
        for (int q = 0; q < BL_CLUSTER; ++q)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                           cl_map(dst, q)),
                       "r"(__float_as_uint(hn)), "r"(cl_map(bar, q))
                       : "memory");
      }
    }
    __syncthreads();  // gpart / cst reuse
  }
  cluster.sync();  // no CTA leaves while a peer may still address its shared memory
}

// pm[t][a] = sum_k mem[t][k] WmT[k][a]; 16 rows per block.
__global__ void __launch_bounds__(256) k_pmem(const int64_t* __restrict__ plan, const float* __restrict__ WmT) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int64_t* p = plan + blockIdx.y * EPLAN;
  const int64_t L = p[1];
  const float* mem = reinterpret_cast<const float*>(p[3]);
  float* pm = reinterpret_cast<float*>(p[4]);
  const int64_t t0 = (int64_t)blockIdx.x * 16;
  if (t0 >= L) return;
  __shared__ float rows[16][EMB];
  const int nr = (int)min((int64_t)16, L - t0);
  for (int i = threadIdx.x; i < nr * EMB; i += 256) rows[i / EMB][i % EMB] = mem[(t0 + i / EMB) * EMB + i % EMB];
  __syncthreads();
  const int a = threadIdx.x & (ATT - 1), rh = threadIdx.x >> 7;  // 2 row groups of 8
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < EMB; ++k) {
    const float w = WmT[k * ATT + a];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fmaf(rows[rh * 8 + i][k], w, acc[i]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (rh * 8 + i < nr) pm[(t0 + rh * 8 + i) * ATT + a] = acc[i];
}

// ----------------------------------------------------------------- vocoder helpers
// mel plan[i] = {tail_ptr (fp32 [O][80]) or 0, mel_ptr (fp32 [m][80]), m, n_tail, row_base (first valid row)}
constexpr int MPLAN = 5;

__global__ void k_mel_assemble(const int64_t* __restrict__ plan, __nv_bfloat16* __restrict__ X0, int ld) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int64_t* p = plan + blockIdx.y * MPLAN;
  const int64_t m = p[2], nt = p[3];
  const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (g >= (nt + m) * ld) return;
  const int64_t t = g / ld;
  const int c = (int)(g % ld);
  float v = 0.f;
  if (c < NMEL) {
    const float* src = t < nt ? reinterpret_cast<const float*>(p[0]) + t * NMEL
                              : reinterpret_cast<const float*>(p[1]) + (t - nt) * NMEL;
    v = src[c];
  }
  X0[(p[4] + t) * ld + c] = __float2bfloat16_rn(v);
}

// rowmap plan[i] = {in_base, in_rows (valid), in_halo, out_first (first valid output row), up}
// row_out[in_base + r] = (valid ? out_first + up * (r - in_halo) : -1) for r in [0, 2*halo + rows).
__global__ void k_rowmap(const int64_t* __restrict__ plan, int32_t* __restrict__ row_out) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int64_t* p = plan + blockIdx.y * 5;
  const int64_t span = 2 * p[2] + p[1];
  const int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (r >= span) return;
  const int64_t q = r - p[2];
  row_out[p[0] + r] = (q >= 0 && q < p[1]) ? (int32_t)(p[3] + p[4] * q) : -1;
}

// Up to 9 row maps of one vocoder call in one launch (blockIdx.z = map); map k as k_rowmap with
// its own plan rows, output buffer and span.
struct RowMaps {
  const int64_t* plan[9];
  int32_t* out[9];
  int64_t span[9];
};
__global__ void k_rowmaps(const __grid_constant__ RowMaps m) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int k = blockIdx.z;
  const int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (r >= m.span[k]) return;
  const int64_t* p = m.plan[k] + blockIdx.y * 5;
  if (r >= 2 * p[2] + p[1]) return;
  const int64_t q = r - p[2];
  m.out[k][p[0] + r] = (q >= 0 && q < p[1]) ? (int32_t)(p[3] + p[4] * q) : -1;
}

// zero plan[i] = {base, rows, halo}: zero [base, base+halo) and [base+halo+rows, base+2halo+rows).
__global__ void k_zero_halo(const int64_t* __restrict__ plan, __nv_bfloat16* __restrict__ X, int C) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int64_t* p = plan + blockIdx.y * 3;
  const int64_t halo = p[2];
  const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (g >= 2 * halo * C) return;
  int64_t r = g / C;
  const int c = (int)(g % C);
  r = r < halo ? p[0] + r : p[0] + p[1] + r;
  X[r * C + c] = __float2bfloat16_rn(0.f);
}

// post plan[i] = {row_first (first valid stage-4 row), G, flags (1 tail, 2 last),
//                 held_src_ptr, vs_dst_ptr, out_off, mel_ptr, m}
// Vocoder state region (fp32): mel tail [O][80] then held [S].
constexpr int PPLAN = 8;

// conv_post weights [32][7] in constant memory: every FMA below takes its weight as a
// constant-bank operand (copied on the stream before each launch)
__constant__ float c_wpost[32 * 7];

__global__ void __launch_bounds__(256) k_post_splice(const __nv_bfloat16* __restrict__ X4,
                                                     const int64_t* __restrict__ plan,
                                                     const float* __restrict__ wpost,  // [32][7]
                                                     float bpost, const float* __restrict__ fade, int O, int S,
                                                     float* __restrict__ audio, int16_t* __restrict__ pcm,
                                                     int32_t* __restrict__ nonfinite) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int64_t* p = plan + blockIdx.y * PPLAN;
  const int64_t G = p[1];
  const bool has_tail = p[2] & 1, is_last = p[2] & 2;
  const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
  float* dst = reinterpret_cast<float*>(p[4]);
  if (!is_last && g < (int64_t)O * NMEL) {  // new mel tail = last O frames of this chunk
    const float* mel = reinterpret_cast<const float*>(p[6]);
    dst[g] = mel[(p[7] - O) * NMEL + g];
  }
  // stage the block's 256 + 6 halo rows of the 32-channel stage-4 activation (coalesced 16-byte
  // loads; rows padded to 80 bytes so the per-sample 16-byte reads below are conflict-free)
  __shared__ uint4 xs[(256 + 6) * 5];
  const int64_t g0 = (int64_t)blockIdx.x * 256;
  if (g0 >= G) return;  // the whole block is past this item's samples
  const uint4* src = reinterpret_cast<const uint4*>(X4 + (p[0] + g0 - 3) * 32);
  const int64_t rows_avail = G + 6 - g0;  // valid staged rows (the stage buffer has a zero halo of 25)
  for (int i = threadIdx.x; i < (256 + 6) * 4; i += 256) {
    const int r = i >> 2, c = i & 3;
    xs[r * 5 + c] = r < rows_avail ? src[i] : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  if (g >= G) return;
  float acc4[4] = {bpost, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < 7; ++j) {
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) {
      const uint4 u = xs[(threadIdx.x + j) * 5 + c4];
      const uint32_t wds[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wds[e]));
        const int c = c4 * 4 + e;
        acc4[e] = fmaf(c_wpost[(2 * c) * 7 + j], f.x, fmaf(c_wpost[(2 * c + 1) * 7 + j], f.y, acc4[e]));
      }
    }
  }
  const float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
  float v = tanhf(acc);
  const int64_t count = is_last ? G : G - S;
  if (g < count) {
    if (has_tail && g < S) v = fade[g] * v + fade[S + g] * reinterpret_cast<const float*>(p[3])[g];
    audio[p[5] + g] = v;
    if (nonfinite && !isfinite(v)) atomicAdd(nonfinite + blockIdx.y, 1);  // per-item guard (host reads n ints)
    if (pcm)  // f1: 16-bit PCM as pcm16_encode (src/vocoder.py:146-149): clamp, x 32767, round half to even
      pcm[p[5] + g] = (int16_t)__double2int_rn(fmin(fmax((double)v, -1.0), 1.0) * 32767.0);
  } else {
    dst[(int64_t)O * NMEL + (g - count)] = v;  // held tail for the next seam
  }
}

// f1 wire format: base64 of each chunk's little-endian PCM16 bytes (the reference server's
// encode_samples, src/server.py:78-79 + pcm16_encode, src/vocoder.py:146-149).  plan[i] =
// {first sample, sample count, first output char}; thread = one 3-byte group -> 4 ASCII chars,
// '=' padding at the chunk's end.
__global__ void k_pcm16_b64(const int16_t* __restrict__ pcm, const int64_t* __restrict__ plan, char* __restrict__ out) {
  const int64_t* p = plan + blockIdx.y * 3;
  const int64_t nbytes = 2 * p[1];
  const int64_t grp = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (3 * grp >= nbytes) return;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(pcm + p[0]);
  const int64_t b = 3 * grp;
  const int nb = (int)min((int64_t)3, nbytes - b);
  const uint32_t v = ((uint32_t)src[b] << 16) | (nb > 1 ? (uint32_t)src[b + 1] << 8 : 0u) | (nb > 2 ? src[b + 2] : 0u);
  const char* tab = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";
  char* o = out + p[2] + 4 * grp;
  o[0] = tab[(v >> 18) & 63];
  o[1] = tab[(v >> 12) & 63];
  o[2] = nb > 1 ? tab[(v >> 6) & 63] : '=';
  o[3] = nb > 2 ? tab[v & 63] : '=';
}

dim3 grid2(int64_t work, int n) { return dim3((unsigned)((work + 255) / 256), (unsigned)n); }

}  // namespace

// ----------------------------------------------------------------- C ABI
ITTS_API int itts_r_dec_prepare(const float* state, void* xb, int32_t B, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  k_dec_prepare<<<B, 256, 0, (cudaStream_t)stream>>>(state, (__nv_bfloat16*)xb);
  ITTS_RETURN_LAUNCH();
}

// Prenet: H1 = relu(last . W0^T) ; p = relu(H1 . W1^T) -> state p + bf16 mirror.  H1 = fp32 [B][256] scratch.
ITTS_API int itts_r_prenet(float* state, void* xb, const float* W0T, const float* W1T, const int64_t* plan,
                           float* H1, int32_t B, int32_t step, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  GemvIO a{state, ROW, LAST_OFF, NMEL, 0, 0, W0T, PRE, H1, PRE, 0, nullptr, 0, nullptr, 1, nullptr, step};
  int r = launch_gemv<1, 0>(a, B, 1, nullptr, false, st);
  if (r) return r;
  GemvIO c{H1, PRE, 0, PRE, 0, 0, W1T, PRE, state, ROW, P_OFF, (__nv_bfloat16*)xb, XB_ROW, nullptr, 1, plan, step};
  return launch_gemv<1, 0>(c, B, 1, nullptr, false, st);
}

// Query q = Wq . att_h as QKS K-slice partials Qp [QKS][B][128] (summed by k_attention).
ITTS_API int itts_r_query(const float* state, const float* WqT, float* Qp, int32_t B, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  GemvIO io{state, ROW, ATTH_OFF, HID, 0, 0, WqT, ATT, nullptr, ATT, 0, nullptr, 0, nullptr, 0, nullptr, 0};
  return launch_gemv<1, 0>(io, B, QKS, Qp, false, (cudaStream_t)stream);
}

ITTS_API int itts_r_lstm_cell(const float* G, int32_t nsplit, const float* bias, float* state, void* xb,
                              int32_t h_off, int32_t c_off, const int64_t* plan, int32_t B, int32_t step,
                              void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  if (nsplit < 1 || !bias) return ITTS_EINVAL;
  k_lstm_cell<<<(B * HID + 255) / 256, 256, 0, (cudaStream_t)stream>>>(G, nsplit, bias, state, (__nv_bfloat16*)xb,
                                                                       h_off, c_off, plan, step, B);
  ITTS_RETURN_LAUNCH();
}

template <int CL>
int launch_attention(float* state, void* xb, const int64_t* plan, int32_t B, int32_t max_len, const float* Q,
                     const float* Wloc, const float* WdT, const float* v, int32_t step, cudaStream_t st) {
  const int ls = (max_len + CL - 1) / CL + 1, lh = ls + KLOC;
  const size_t smem = ((size_t)(2 * lh + ls + 4) + (size_t)LT * (NF + 1)) * sizeof(float);
  static_assert(LT * (NF + 1) >= AT_WARPS * EMB, "context partials alias the location tile");
  if (smem > 150 * 1024) return ITTS_EUNSUPPORTED;
  static uint64_t configured = 0;
  if (!(configured & itts::device_bit())) {
    cudaFuncSetAttribute(k_attention<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    configured |= itts::device_bit();
  }
  k_attention<CL><<<B * CL, AT_WARPS * 32, smem, st>>>(state, (__nv_bfloat16*)xb, plan, Q, Wloc, WdT, v, step);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_attention(float* state, void* xb, const int64_t* plan, int32_t B, int32_t max_len,
                              const float* Q, const float* Wloc, const float* WdT, const float* v,
                              int32_t step, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  // small pooled batches spread each item over 8 SMs, large ones over 4 (one wave either way)
  if (B <= 48) return launch_attention<8>(state, xb, plan, B, max_len, Q, Wloc, WdT, v, step, (cudaStream_t)stream);
  return launch_attention<4>(state, xb, plan, B, max_len, Q, Wloc, WdT, v, step, (cudaStream_t)stream);
}

// Mel/gate projection; Pp = scratch [PKS][B][81].
constexpr int PKS = 8;
ITTS_API int itts_r_proj(float* state, const int64_t* plan, int32_t B, const float* WpT, const float* bp,
                         float* Pp, int32_t step, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  GemvIO io{state, ROW, DECH_OFF, HID, CTX_OFF, EMB, WpT, NMEL + 1, state, ROW, 0, nullptr, 0, bp, 0, plan, step};
  return launch_gemv<1, 1>(io, B, PKS, Pp, true, (cudaStream_t)stream);
}

ITTS_API int itts_r_enc_embed(const int32_t* tok4, int64_t total, const int64_t* plan, int32_t n,
                              int64_t max_len, const float* Eph, const float* Epw, const float* Epph,
                              const float* Eiph, void* X, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const cudaError_t le_ = itts::launch_pdl(k_enc_embed<__nv_bfloat16>, dim3(grid2(max_len * EMB, n)), dim3(256), 0,
                                           (cudaStream_t)stream, tok4, total, plan, Eph, Epw, Epph, Eiph,
                                           (__nv_bfloat16*)X);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_bilstm(const float* PRE, const int64_t* plan, int32_t n, const float* WhhT, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const cudaError_t e = itts::launch_pdl_cls(itts::PDL_BILSTM, k_bilstm, dim3(n * 2 * BL_CLUSTER), dim3(256), 0, (cudaStream_t)stream, PRE,
                                         plan, WhhT);
  return e == cudaSuccess ? ITTS_OK : (int)e;
}

ITTS_API int itts_r_pmem(const int64_t* plan, int32_t n, int64_t max_len, const float* WmT, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  dim3 grid((unsigned)((max_len + 15) / 16), (unsigned)n);
  const cudaError_t le_ = itts::launch_pdl(k_pmem, dim3(grid), dim3(256), 0, (cudaStream_t)stream, plan, WmT);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

// Zero n spans of fp32 (the fresh decoder-state rows of newly encoded requests): span i =
// {ptr, count}; one launch instead of one memset per request.
__global__ void k_zero_spans(const int64_t* __restrict__ spans) {
  itts::pdl_trigger();
  itts::pdl_wait();
  float* p = reinterpret_cast<float*>(spans[2 * blockIdx.y]);
  const int64_t cnt = spans[2 * blockIdx.y + 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.f;
}

// The whole Tier-R encoder launch sequence of one pooled encoder call (reference encode_batch,
// acoustic.py:146-160, behind encoder_batch src/modules.py:60-66), issued from C++: embedding
// sum -> 3 x (conv k5 + ReLU; BN folded) -> BiLSTM input projection (fp32) -> recurrence ->
// processed memory -> zeroed decoder-state rows.  `pack` holds, after the int32 tokens
// [4][total] padded to 8 bytes, the item plan [n][6], the row-map plan [n][5] and the state
// spans [n][2].  weights: Eph, Epw, Epph, Eiph, (conv w, conv b) x 3, Wih, b_ih, WhhT, WmT.
ITTS_API int itts_r_encode(const void* pack, int64_t total, int32_t n, int64_t max_len, int64_t rows,
                           int64_t max_span, const int64_t* weights, int32_t conv_taps, void* xa, void* xb,
                           float* pre, int32_t* rowmap, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  if (conv_taps < 1 || conv_taps > 15 || !pack || !weights || !xa || !xb || !pre || !rowmap) return ITTS_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t* tok4 = static_cast<const int32_t*>(pack);
  const int64_t* plan = static_cast<const int64_t*>(pack) + (4 * total + 1) / 2;
  const int64_t* rm_plan = plan + 6 * (int64_t)n;
  const int64_t* spans = rm_plan + 5 * (int64_t)n;
  auto W = [&](int i) { return reinterpret_cast<const void*>(weights[i]); };
  cudaError_t e = cudaMemsetAsync(xa, 0, (size_t)rows * EMB * 2, st);
  if (e != cudaSuccess) return (int)e;
  int r = itts_r_enc_embed(tok4, total, plan, n, max_len, (const float*)W(0), (const float*)W(1), (const float*)W(2),
                           (const float*)W(3), xa, stream);
  if (r) return r;
  if ((r = itts_r_rowmap(rm_plan, n, max_span, rowmap, stream))) return r;
  int32_t offs[16];
  for (int j = 0; j < conv_taps; ++j) offs[j] = j - (conv_taps - 1) / 2;
  void* bufs[2] = {xa, xb};
  for (int i = 0; i < 3; ++i)
    if ((r = itts_conv1d_tc(bufs[i & 1], rows, EMB, EMB, W(4 + 2 * i), EMB, conv_taps, offs, (const float*)W(5 + 2 * i),
                            EMB, rowmap, nullptr, 1.0f, nullptr, 1, nullptr, 0, bufs[(i + 1) & 1], 0.0f, 1, 0, stream)))
      return r;
  const int32_t off0 = 0;
  if ((r = itts_conv1d_tc(xb, rows, EMB, EMB, W(10), 8 * EH, 1, &off0, (const float*)W(11), 8 * EH, rowmap, nullptr,
                          1.0f, pre, 1, nullptr, 0, nullptr, 1.0f, 1, 128, stream)))
    return r;
  // BiLSTM: one SIMT cluster per (item, direction) (k_bilstm, ~0.85 us per step); pooled batches
  // of >= BILSTM_TC_MIN items (more than ~10 waves of clusters) run the tensor-core recurrence
  // instead when the weight table carries W_hh tiles (entry 14, bf16-exact weights): ~2-5 us per
  // step but 32 items per cluster
  if ((r = (W(14) && n >= BILSTM_TC_MIN) ? bilstm_tc_launch(pre, plan, n, W(14), stream)
                                         : itts_r_bilstm(pre, plan, n, (const float*)W(12), stream)))
    return r;
  if ((r = itts_r_pmem(plan, n, max_len, (const float*)W(13), stream))) return r;
  const cudaError_t le_ = itts::launch_pdl(k_zero_spans, dim3(dim3(8, n)), dim3(256), 0, st, spans);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

// The encoder of the split-bf16 parity mode: the same launch sequence as itts_r_encode with every
// tensor-core product (3 convs, the BiLSTM input projection) on [hi | lo | hi] operands against
// [Wh | Wh | Wl] weights (weights3: the itts_r_encode weight table with the conv / input-projection
// entries replaced by those [.][C_out][3 x 512] tensors); activations stay fp32 between layers
// (f32 [rows][512]), x3 = bf16 [rows][1536] operand buffer.
ITTS_API int itts_r_encode_split(const void* pack, int64_t total, int32_t n, int64_t max_len, int64_t rows,
                                 int64_t max_span, const int64_t* weights3, int32_t conv_taps, void* x3, float* f32,
                                 float* pre, int32_t* rowmap, int32_t parts, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  if (parts != 2 && parts != 3) return ITTS_EINVAL;
  const int32_t kin = parts * EMB;   // [hi | lo (| hi)] columns of the [rows][1536] operand
  if (conv_taps < 1 || conv_taps > 15 || !pack || !weights3 || !x3 || !f32 || !pre || !rowmap) return ITTS_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t* tok4 = static_cast<const int32_t*>(pack);
  const int64_t* plan = static_cast<const int64_t*>(pack) + (4 * total + 1) / 2;
  const int64_t* rm_plan = plan + 6 * (int64_t)n;
  const int64_t* spans = rm_plan + 5 * (int64_t)n;
  auto W = [&](int i) { return reinterpret_cast<const void*>(weights3[i]); };
  cudaError_t e = cudaMemsetAsync(x3, 0, (size_t)rows * 3 * EMB * 2, st);
  if (e != cudaSuccess) return (int)e;
  const dim3 g2 = grid2(max_len * EMB, n);
  if ((e = itts::launch_pdl(k_enc_embed<float>, g2, dim3(256), 0, st, tok4, total, plan, (const float*)W(0),
                            (const float*)W(1), (const float*)W(2), (const float*)W(3), f32)) != cudaSuccess)
    return (int)e;
  if ((e = itts::launch_pdl(k_split3, g2, dim3(256), 0, st, (const float*)f32, plan, 0, (__nv_bfloat16*)x3)) !=
      cudaSuccess)
    return (int)e;
  int r;
  if ((r = itts_r_rowmap(rm_plan, n, max_span, rowmap, stream))) return r;
  int32_t offs[16];
  for (int j = 0; j < conv_taps; ++j) offs[j] = j - (conv_taps - 1) / 2;
  for (int i = 0; i < 3; ++i) {
    if ((r = itts_conv1d_tc(x3, rows, kin, 3 * EMB, W(4 + 2 * i), EMB, conv_taps, offs, (const float*)W(5 + 2 * i),
                            EMB, rowmap, nullptr, 1.0f, f32, 1, nullptr, 0, nullptr, 0.0f, 0, 0, stream)))
      return r;
    if ((e = itts::launch_pdl(k_split3, g2, dim3(256), 0, st, (const float*)f32, plan, 1, (__nv_bfloat16*)x3)) !=
        cudaSuccess)
      return (int)e;
  }
  const int32_t off0 = 0;
  if ((r = itts_conv1d_tc(x3, rows, kin, 3 * EMB, W(10), 8 * EH, 1, &off0, (const float*)W(11), 8 * EH, rowmap,
                          nullptr, 1.0f, pre, 1, nullptr, 0, nullptr, 1.0f, 1, 128, stream)))
    return r;
  // BiLSTM: one SIMT cluster per (item, direction) (k_bilstm, ~0.85 us per step); pooled batches
  // of >= BILSTM_TC_MIN items (more than ~10 waves of clusters) run the tensor-core recurrence
  // instead when the weight table carries W_hh tiles (entry 14, bf16-exact weights): ~2-5 us per
  // step but 32 items per cluster
  if ((r = (W(14) && n >= BILSTM_TC_MIN) ? bilstm_tc_launch(pre, plan, n, W(14), stream)
                                         : itts_r_bilstm(pre, plan, n, (const float*)W(12), stream)))
    return r;
  if ((r = itts_r_pmem(plan, n, max_len, (const float*)W(13), stream))) return r;
  const cudaError_t le_ = itts::launch_pdl(k_zero_spans, dim3(dim3(8, n)), dim3(256), 0, st, spans);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

// PostNet residual: out[t][c] = mel[t][c] + post[first + t][c] (c < 80) per item; plan[i] =
// {mel_ptr, out_ptr, m, first_row}.
__global__ void k_postnet_add(const int64_t* __restrict__ plan, const float* __restrict__ post, int32_t ld) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int64_t* p = plan + 4 * blockIdx.y;
  const float* mel = reinterpret_cast<const float*>(p[0]);
  float* out = reinterpret_cast<float*>(p[1]);
  const int64_t m = p[2], first = p[3];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m * NMEL; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / NMEL, c = i - t * NMEL;
    out[i] = mel[i] + post[(first + t) * ld + c];
  }
}

// Tacotron2 PostNet over the chunks of one decoder call (the paper's decoder
// "contains ... a PostNet", absorbed as a no-op by the reference): 5 x conv k5
// (80 -> 512 -> 512 -> 512 -> 512 -> 80, batch norm folded, tanh after the first four), mel_out =
// mel + PostNet(mel), each chunk zero-padded at its edges (no look-ahead: chunk-local, so it adds
// no latency; the decoder's fed-back last frame stays the pre-PostNet frame).  Items are packed
// with 2-row zero halos like the vocoder stages.  pack = mel-assembly plan [n][5], row-map plan
// [n][5], residual plan [n][4]; weights = (w, b) x 5 in tc_conv layout (c_in / c_out of the mel
// ends padded to 96); x0 bf16 [rows][96], ya / yb bf16 [rows][512], post fp32 [rows][96].
ITTS_API int itts_r_postnet(const int64_t* pack, int32_t n, int64_t max_m, int64_t rows, int64_t max_span,
                            const int64_t* weights, void* x0, void* ya, void* yb, float* post, int32_t* rowmap,
                            void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  if (!pack || !weights || !x0 || !ya || !yb || !post || !rowmap || max_m < 1) return ITTS_EINVAL;
  constexpr int CP = 96, CH = 512, TAPS = 5;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t* mplan = pack;
  const int64_t* rm_plan = pack + 5 * (int64_t)n;
  const int64_t* aplan = rm_plan + 5 * (int64_t)n;
  auto W = [&](int i) { return reinterpret_cast<const void*>(weights[i]); };
  cudaError_t e = cudaMemsetAsync(x0, 0, (size_t)rows * CP * 2, st);
  if (e != cudaSuccess) return (int)e;
  int r = itts_r_mel_assemble(mplan, n, max_m, x0, CP, stream);
  if (r) return r;
  if ((r = itts_r_rowmap(rm_plan, n, max_span, rowmap, stream))) return r;
  int32_t offs[TAPS];
  for (int j = 0; j < TAPS; ++j) offs[j] = j - (TAPS - 1) / 2;
  const void* src = x0;
  int c_in = CP;
  void* bufs[2] = {ya, yb};
  for (int l = 0; l < 4; ++l) {  // conv + tanh; zero halos keep the chunk-edge padding
    const int bn = c_in % 64 ? 64 : 0;  // the 96-wide input uses the 64B-swizzle path (N tile <= 64)
    if ((r = conv1d_tc_impl(src, rows, c_in, c_in, W(2 * l), CH, TAPS, offs, (const float*)W(2 * l + 1), CH, rowmap,
                            nullptr, 1.0f, nullptr, 1, nullptr, 0, bufs[l & 1], 1.0f, 1, bn, 1, stream)))
      return r;
    src = bufs[l & 1];
    c_in = CH;
  }
  if ((r = conv1d_tc_impl(src, rows, CH, CH, W(8), CP, TAPS, offs, (const float*)W(9), CP, rowmap, nullptr, 1.0f,
                          post, 1, nullptr, 0, nullptr, 1.0f, 1, 0, 0, stream)))
    return r;
  const cudaError_t le = itts::launch_pdl(k_postnet_add, dim3((unsigned)((max_m * NMEL + 255) / 256), n), dim3(256), 0,
                                          st, aplan, (const float*)post, CP);
  return le == cudaSuccess ? ITTS_OK : (int)le;
}

ITTS_API int itts_r_mel_assemble(const int64_t* plan, int32_t n, int64_t max_rows, void* X0, int32_t ld,
                                 void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const cudaError_t le_ = itts::launch_pdl(k_mel_assemble, dim3(grid2(max_rows * ld, n)), dim3(256), 0, (cudaStream_t)stream,
                                           plan, (__nv_bfloat16*)X0, ld);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

// `count` (<= 9) row maps in one launch: plans[k] (n items x 5, as itts_r_rowmap), outs[k], spans[k].
int itts_r_rowmaps(int32_t count, const int64_t* const* plans, int32_t* const* outs, const int64_t* spans, int32_t n,
                   void* stream) {
  if (n <= 0 || count <= 0) return (n == 0 || count == 0) ? ITTS_OK : ITTS_EINVAL;
  if (count > 9) return ITTS_EINVAL;
  RowMaps m{};
  int64_t max_span = 1;
  for (int k = 0; k < count; ++k) {
    m.plan[k] = plans[k];
    m.out[k] = outs[k];
    m.span[k] = spans[k];
    max_span = max(max_span, spans[k]);
  }
  const dim3 grid((unsigned)((max_span + 255) / 256), (unsigned)n, (unsigned)count);
  const cudaError_t le_ = itts::launch_pdl(k_rowmaps, grid, dim3(256), 0, (cudaStream_t)stream, m);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_rowmap(const int64_t* plan, int32_t n, int64_t max_span, int32_t* row_out, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const cudaError_t le_ = itts::launch_pdl(k_rowmap, dim3(grid2(max_span, n)), dim3(256), 0, (cudaStream_t)stream,
                                           plan, row_out);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

// MRF branch merge: out = bf16(lrelu((y0 + y1 + y2) / 3, slope)), 8 bf16 per thread (16-byte
// accesses).  The three branches' last ResBlock1 layers write their y independently, so they can
// run concurrently; halo rows are zero in every input and stay zero.
// Optionally (zplan != null) the same launch zeroes the halo rows of the next stage's operand
// buffer zX (k_zero_halo's plan format, zn items of zhalo rows each side): that buffer's previous
// contents were last read by this stage's first ResBlock layers, which all finished before this
// kernel, and the next transposed conv writes only valid rows.
__global__ void __launch_bounds__(256) k_mrf_combine(const uint4* __restrict__ y0, const uint4* __restrict__ y1,
                                                     const uint4* __restrict__ y2, int64_t n8, float slope,
                                                     uint4* __restrict__ out, const int64_t* __restrict__ zplan,
                                                     int zn, int64_t zhalo, __nv_bfloat16* __restrict__ zX, int zC) {
  itts::pdl_trigger();
  itts::pdl_wait();
  if (zplan) {
    const int64_t per = 2 * zhalo * zC, tot = per * zn;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < tot; g += (int64_t)gridDim.x * blockDim.x) {
      const int64_t* p = zplan + (g / per) * 3;
      const int64_t e = g % per, r0 = e / zC, halo = p[2];
      if (r0 >= 2 * halo) continue;
      const int64_t r = r0 < halo ? p[0] + r0 : p[0] + p[1] + r0;
      zX[r * zC + e % zC] = __float2bfloat16_rn(0.f);
    }
  }
  const float third = 1.0f / 3.0f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 a = __ldcs(y0 + i), b = __ldcs(y1 + i), c = __ldcs(y2 + i);
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
    const __nv_bfloat162* pc = reinterpret_cast<const __nv_bfloat162*>(&c);
    uint4 o;
    __nv_bfloat162* po = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 fa = __bfloat1622float2(pa[j]), fb = __bfloat1622float2(pb[j]), fc = __bfloat1622float2(pc[j]);
      float vx = ((fa.x + fb.x) + fc.x) * third, vy = ((fa.y + fb.y) + fc.y) * third;
      vx = vx > 0.f ? vx : vx * slope;
      vy = vy > 0.f ? vy : vy * slope;
      po[j] = __floats2bfloat162_rn(vx, vy);
    }
    out[i] = o;
  }
}

int mrf_combine_zero_halo(const void* y0, const void* y1, const void* y2, int64_t n, float slope, void* out,
                          const int64_t* zplan, int32_t zn, int64_t zhalo, void* zX, int32_t zC, void* stream) {
  if (n < 0 || n % 8) return ITTS_EINVAL;
  if (zplan && (zn <= 0 || zhalo < 0 || zC <= 0 || !zX)) return ITTS_EINVAL;
  if (n == 0 && !zplan) return ITTS_OK;
  const int64_t n8 = n / 8, work = std::max<int64_t>(n8, zplan ? 2 * zhalo * zC * zn : 0);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 8));
  const cudaError_t le_ = itts::launch_pdl(k_mrf_combine, dim3(blocks), dim3(256), 0, (cudaStream_t)stream,
                                           (const uint4*)y0, (const uint4*)y1, (const uint4*)y2, n8,
                                           slope, (uint4*)out, zplan, (int)zn, zhalo, (__nv_bfloat16*)zX, (int)zC);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_mrf_combine(const void* y0, const void* y1, const void* y2, int64_t n, float slope, void* out,
                                void* stream) {
  return mrf_combine_zero_halo(y0, y1, y2, n, slope, out, nullptr, 0, 0, nullptr, 0, stream);
}

ITTS_API int itts_r_zero_halo(const int64_t* plan, int32_t n, int64_t max_halo, void* X, int32_t C,
                              void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const cudaError_t le_ = itts::launch_pdl(k_zero_halo, dim3(grid2(2 * max_halo * C, n)), dim3(256), 0, (cudaStream_t)stream,
                                           plan, (__nv_bfloat16*)X, C);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_pcm16_b64(const void* pcm16, const int64_t* plan, int32_t n, int64_t max_samples, void* out,
                              void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  if (!pcm16 || !plan || !out) return ITTS_EINVAL;
  const int64_t groups = (2 * max_samples + 2) / 3;
  k_pcm16_b64<<<grid2(max(groups, (int64_t)1), n), 256, 0, (cudaStream_t)stream>>>((const int16_t*)pcm16, plan,
                                                                                  (char*)out);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_post_splice(const void* X4, const int64_t* plan, int32_t n, int64_t max_g,
                                const float* wpost, float bpost, const float* fade, int32_t overlap_frames,
                                int32_t overlap_samples, float* audio, void* pcm16, int32_t* nonfinite,
                                void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const int64_t work = max(max_g, (int64_t)overlap_frames * NMEL);
  cudaError_t e = cudaMemcpyToSymbolAsync(c_wpost, wpost, sizeof(float) * 32 * 7, 0, cudaMemcpyDeviceToDevice,
                                          (cudaStream_t)stream);
  if (e != cudaSuccess) return (int)e;
  if (nonfinite && (e = cudaMemsetAsync(nonfinite, 0, sizeof(int32_t) * n, (cudaStream_t)stream)) != cudaSuccess)
    return (int)e;
  const cudaError_t le_ = itts::launch_pdl(k_post_splice, dim3(grid2(work, n)), dim3(256), 0, (cudaStream_t)stream,
                                           (const __nv_bfloat16*)X4, plan, wpost, bpost,
                                                                  fade, overlap_frames, overlap_samples, audio,
                                                                  (int16_t*)pcm16, nonfinite);
  if (le_ != cudaSuccess) return (int)le_;
  ITTS_RETURN_LAUNCH();
}
