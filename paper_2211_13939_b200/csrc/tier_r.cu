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

// Item-tiled small GEMVs: each CTA serves IT items so every weight matrix is
// read once per IT items instead of once per item (per-SM L2 bandwidth, not
// FLOPs, bounds these at large pooled batch).
constexpr int IT = 8;

// W0T [80][256], W1T [256][256] (input-major so threads read coalesced).
__global__ void __launch_bounds__(256) k_prenet(float* __restrict__ state, __nv_bfloat16* __restrict__ xb,
                                                const float* __restrict__ W0T, const float* __restrict__ W1T,
                                                const int64_t* __restrict__ plan, int step, int B) {
  const int b0 = blockIdx.x * IT, j = threadIdx.x;
  const int nb = min(IT, B - b0);
  __shared__ float x[IT][NMEL], h1[IT][PRE];
  for (int i = j; i < nb * NMEL; i += 256) x[i / NMEL][i % NMEL] = state[(int64_t)(b0 + i / NMEL) * ROW + LAST_OFF + i % NMEL];
  __syncthreads();
  float a[IT];
#pragma unroll
  for (int i = 0; i < IT; ++i) a[i] = 0.f;
  for (int k = 0; k < NMEL; ++k) {
    const float w = W0T[k * PRE + j];
#pragma unroll
    for (int i = 0; i < IT; ++i) a[i] = fmaf(w, x[i][k], a[i]);
  }
#pragma unroll
  for (int i = 0; i < IT; ++i) h1[i][j] = fmaxf(a[i], 0.f);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IT; ++i) a[i] = 0.f;
  for (int k = 0; k < PRE; ++k) {
    const float w = W1T[k * PRE + j];
#pragma unroll
    for (int i = 0; i < IT; ++i) a[i] = fmaf(w, h1[i][k], a[i]);
  }
  for (int i = 0; i < nb; ++i) {
    const int b = b0 + i;
    if (step >= plan[b * DPLAN + 5]) continue;
    const float v = fmaxf(a[i], 0.f);
    state[(int64_t)b * ROW + P_OFF + j] = v;
    xb[(int64_t)b * XB_ROW + P_OFF + j] = __float2bfloat16_rn(v);
  }
}

// q[b] = Wq . att_h[b] for IT items per CTA; WqT [1024][128].  256 threads:
// thread = (output a, item half).
__global__ void __launch_bounds__(256) k_query(const float* __restrict__ state, const float* __restrict__ WqT,
                                               float* __restrict__ Q, int B) {
  const int b0 = blockIdx.x * IT, tid = threadIdx.x;
  const int nb = min(IT, B - b0);
  extern __shared__ float hs[];  // [IT][1024]
  for (int i = tid; i < nb * HID; i += 256) hs[i] = state[(int64_t)(b0 + i / HID) * ROW + ATTH_OFF + i % HID];
  __syncthreads();
  const int a = tid & (ATT - 1), ih = tid >> 7;  // items ih*4 .. ih*4+3
  float acc[IT / 2] = {0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < HID; ++k) {
    const float w = WqT[k * ATT + a];
#pragma unroll
    for (int i = 0; i < IT / 2; ++i) acc[i] = fmaf(w, hs[(ih * (IT / 2) + i) * HID + k], acc[i]);
  }
#pragma unroll
  for (int i = 0; i < IT / 2; ++i) {
    const int it = ih * (IT / 2) + i;
    if (it < nb) Q[(int64_t)(b0 + it) * ATT + a] = acc[i];
  }
}

// G [B][4096] gate pre-activations (bias included), PyTorch order i, f, g, o.
__global__ void __launch_bounds__(256) k_lstm_cell(const float* __restrict__ G, float* __restrict__ state,
                                                   __nv_bfloat16* __restrict__ xb, int h_off, int c_off,
                                                   const int64_t* __restrict__ plan, int step, int B) {
  const int idx = blockIdx.x * 256 + threadIdx.x;
  const int b = idx / HID, j = idx % HID;
  if (b >= B || step >= plan[b * DPLAN + 5]) return;
  const float* g = G + (int64_t)b * 4 * HID;
  float* s = state + (int64_t)b * ROW;
  const float c = sigm(g[HID + j]) * s[c_off + j] + sigm(g[j]) * tanhf(g[2 * HID + j]);
  const float h = sigm(g[3 * HID + j]) * tanhf(c);
  s[c_off + j] = c;
  s[h_off + j] = h;
  xb[(int64_t)b * XB_ROW + h_off + j] = __float2bfloat16_rn(h);
}

// One CTA per item.  WqT [1024][128], Wloc [32][2][31], WdT [32][128], v [128].
// Dynamic smem: 3*L floats (W_prev, W_acc, energies).
__global__ void __launch_bounds__(256) k_attention(float* __restrict__ state, __nv_bfloat16* __restrict__ xb,
                                                   const int64_t* __restrict__ plan,
                                                   const float* __restrict__ Q, const float* __restrict__ Wloc,
                                                   const float* __restrict__ WdT, const float* __restrict__ v,
                                                   int step) {
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t* p = plan + b * DPLAN;
  if (step >= p[5]) return;
  const float* mem = reinterpret_cast<const float*>(p[0]);
  const float* pm = reinterpret_cast<const float*>(p[1]);
  const int L = (int)p[2];
  const float* wsrc = reinterpret_cast<const float*>(step == 0 ? p[3] : p[4]);
  float* wdst = reinterpret_cast<float*>(p[4]);
  float* s = state + (int64_t)b * ROW;

  extern __shared__ float dyn[];
  float* w_prev = dyn;
  float* w_acc = dyn + L;
  float* e = dyn + 2 * L;
  __shared__ float q[ATT], sWloc[NF * 2 * KLOC], sWd[NF * ATT], sv[ATT], red[32];
  __shared__ float4 cpart[8][EMB / 4];

  for (int i = tid; i < L; i += 256) {
    w_prev[i] = wsrc[i];
    w_acc[i] = wsrc[L + i];
  }
  if (tid < ATT) q[tid] = Q[(int64_t)b * ATT + tid];
  for (int i = tid; i < NF * 2 * KLOC; i += 256) sWloc[i] = Wloc[i];
  for (int i = tid; i < NF * ATT; i += 256) sWd[i] = WdT[i];
  if (tid < ATT) sv[tid] = v[tid];
  __syncthreads();

  // energies: one warp per text position; lane = location filter, then 4 attention dims per lane
  for (int t = warp; t < L; t += 8) {
    float conv = 0.f;
    const float* wf = sWloc + lane * 2 * KLOC;
#pragma unroll
    for (int k = 0; k < KLOC; ++k) {
      const int u = t + k - (KLOC - 1) / 2;
      if (u >= 0 && u < L) conv = fmaf(wf[k], w_prev[u], fmaf(wf[KLOC + k], w_acc[u], conv));
    }
    float loc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
    for (int f = 0; f < NF; ++f) {
      const float cf = __shfl_sync(0xffffffffu, conv, f);
#pragma unroll
      for (int i = 0; i < 4; ++i) loc[i] = fmaf(sWd[f * ATT + lane + 32 * i], cf, loc[i]);
    }
    float en = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int a = lane + 32 * i;
      en = fmaf(sv[a], tanhf((q[a] + loc[i]) + pm[(int64_t)t * ATT + a]), en);
    }
    en = itts::warp_sum(en);
    if (lane == 0) e[t] = en;
  }
  __syncthreads();
  float lmax = -INFINITY;
  for (int t = tid; t < L; t += 256) lmax = fmaxf(lmax, e[t]);
  const float M = itts::block_reduce<float, true>(lmax, red);
  float lsum = 0.f;
  for (int t = tid; t < L; t += 256) {
    const float x = expf(e[t] - M);
    e[t] = x;
    lsum += x;
  }
  const float Z = itts::block_reduce<float, false>(lsum, red);
  for (int t = tid; t < L; t += 256) {
    const float a = e[t] / Z;
    e[t] = a;
    wdst[t] = a;
    wdst[L + t] = w_acc[t] + a;
  }
  __syncthreads();
  // context = sum_t a_t * memory[t]: warp w takes rows t = w (mod 8), lane holds 16 dims as
  // 4 float4 (coalesced 512 B per row per j), then a cross-warp reduction through smem.
  float4 acc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* mem4 = reinterpret_cast<const float4*>(mem);
#pragma unroll 2
  for (int t = warp; t < L; t += 8) {
    const float a = e[t];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 m4 = mem4[(int64_t)t * (EMB / 4) + lane + 32 * j];
      acc[j].x = fmaf(a, m4.x, acc[j].x);
      acc[j].y = fmaf(a, m4.y, acc[j].y);
      acc[j].z = fmaf(a, m4.z, acc[j].z);
      acc[j].w = fmaf(a, m4.w, acc[j].w);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) cpart[warp][lane + 32 * j] = acc[j];
  __syncthreads();
  const float* cp = reinterpret_cast<const float*>(cpart);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int d = tid + 256 * r;
    float c = cp[d];
#pragma unroll
    for (int w = 1; w < 8; ++w) c += cp[w * EMB + d];
    s[CTX_OFF + d] = c;
    xb[(int64_t)b * XB_ROW + CTX_OFF + d] = __float2bfloat16_rn(c);
  }
}

// WpT [1536][81] (80 mel rows + gate row), bp [81].  hc = [dec_h, ctx]; IT items per CTA.
__global__ void __launch_bounds__(256) k_proj(float* __restrict__ state, const int64_t* __restrict__ plan,
                                              const float* __restrict__ WpT, const float* __restrict__ bp,
                                              int step, int B) {
  const int b0 = blockIdx.x * IT, tid = threadIdx.x;
  const int nb = min(IT, B - b0);
  extern __shared__ float hcs[];  // [IT][1536] then part [3][IT][81]
  float* part = hcs + IT * 1536;
  for (int i = tid; i < nb * 1536; i += 256) {
    const int it = i / 1536, k = i % 1536;
    const float* s = state + (int64_t)(b0 + it) * ROW;
    hcs[i] = k < HID ? s[DECH_OFF + k] : s[CTX_OFF + k - HID];
  }
  for (int i = nb * 1536 + tid; i < IT * 1536; i += 256) hcs[i] = 0.f;
  __syncthreads();
  const int g = tid / 81, n = tid % 81;
  if (g < 3) {
    float a[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) a[i] = 0.f;
    for (int k = g * 512; k < g * 512 + 512; ++k) {
      const float w = WpT[k * 81 + n];
#pragma unroll
      for (int i = 0; i < IT; ++i) a[i] = fmaf(w, hcs[i * 1536 + k], a[i]);
    }
#pragma unroll
    for (int i = 0; i < IT; ++i) part[(g * IT + i) * 81 + n] = a[i];
  }
  __syncthreads();
  for (int i = tid; i < nb * 81; i += 256) {
    const int it = i / 81, o = i % 81, b = b0 + it;
    const int64_t* p = plan + b * DPLAN;
    if (step >= p[5]) continue;
    const float out = bp[o] + ((part[(0 * IT + it) * 81 + o] + part[(1 * IT + it) * 81 + o]) + part[(2 * IT + it) * 81 + o]);
    if (o < NMEL) {
      state[(int64_t)b * ROW + LAST_OFF + o] = out;
      reinterpret_cast<float*>(p[6])[step * NMEL + o] = out;
    } else {
      reinterpret_cast<float*>(p[7])[step] = out;
    }
  }
}

// ----------------------------------------------------------------- encoder
// plan[i] = {tok_off, L, row_base (first valid row), mem_ptr, pm_ptr, 0}
constexpr int EPLAN = 6;

__global__ void k_enc_embed(const int32_t* __restrict__ tok4, int64_t total, const int64_t* __restrict__ plan,
                            const float* __restrict__ Eph, const float* __restrict__ Epw,
                            const float* __restrict__ Epph, const float* __restrict__ Eiph,
                            __nv_bfloat16* __restrict__ X) {
  const int64_t* p = plan + blockIdx.y * EPLAN;
  const int64_t L = p[1];
  const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (g >= L * EMB) return;
  const int64_t t = g / EMB;
  const int c = (int)(g % EMB);
  const int64_t idx = p[0] + t;
  const float v = ((Eph[(int64_t)tok4[idx] * EMB + c] + Epw[(int64_t)tok4[total + idx] * EMB + c]) +
                   Epph[(int64_t)tok4[2 * total + idx] * EMB + c]) + Eiph[(int64_t)tok4[3 * total + idx] * EMB + c];
  X[(p[2] + t) * EMB + c] = __float2bfloat16_rn(v);
}

// One 8-CTA cluster per (item, direction).  CTA r owns hidden units
// [32r, 32r+32): gate rows {g*256 + 32r + u}.  WhhT [2][256 k][1024 rows].
// PRE [rows][2048] = x . W_ih^T + b_ih + b_hh for both directions.
constexpr int BL_CLUSTER = 8, BL_UNITS = EH / BL_CLUSTER, BL_ROWS = 4 * BL_UNITS;

__global__ void __cluster_dims__(BL_CLUSTER, 1, 1) __launch_bounds__(256, 1)
    k_bilstm(const float* __restrict__ PRE, const int64_t* __restrict__ plan, const float* __restrict__ WhhT) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int pair = blockIdx.x / BL_CLUSTER;
  const int item = pair >> 1, dir = pair & 1;
  const int64_t* p = plan + item * EPLAN;
  const int64_t L = p[1], row0 = p[2];
  float* mem = reinterpret_cast<float*>(p[3]);
  const int tid = threadIdx.x;

  extern __shared__ float wsm[];               // [256 k][128 rows] for this CTA's gate rows
  __shared__ float hbuf[2][EH];
  __shared__ float gpart[2][BL_ROWS];
  __shared__ float cst[BL_UNITS];
  const float* Wd = WhhT + (int64_t)dir * EH * 4 * EH;  // this direction's [256 k][1024 rows]
  for (int i = tid; i < EH * BL_ROWS; i += 256) {
    const int k = i / BL_ROWS, r = i % BL_ROWS;
    const int grow = (r / BL_UNITS) * EH + rank * BL_UNITS + (r % BL_UNITS);
    wsm[i] = Wd[(int64_t)k * (4 * EH) + grow];
  }
  for (int i = tid; i < EH; i += 256) hbuf[0][i] = 0.f;
  if (tid < BL_UNITS) cst[tid] = 0.f;
  cluster.sync();

  const int r = tid % BL_ROWS, half = tid / BL_ROWS;  // 2 K-halves of 128
  const int grow = (r / BL_UNITS) * EH + rank * BL_UNITS + (r % BL_UNITS);
  for (int64_t s = 0; s < L; ++s) {
    const int64_t t = dir ? L - 1 - s : s;
    const float* h = hbuf[s & 1];
    float a = 0.f;
#pragma unroll 8
    for (int k = half * 128; k < half * 128 + 128; ++k) a = fmaf(wsm[k * BL_ROWS + r], h[k], a);
    gpart[half][r] = a;
    __syncthreads();
    if (tid < BL_UNITS) {
      const float* pre = PRE + (row0 + t) * (8 * EH) + dir * 4 * EH;
      const int u = tid, j = rank * BL_UNITS + u;
      float gi = pre[j] + (gpart[0][u] + gpart[1][u]);
      float gf = pre[EH + j] + (gpart[0][BL_UNITS + u] + gpart[1][BL_UNITS + u]);
      float gg = pre[2 * EH + j] + (gpart[0][2 * BL_UNITS + u] + gpart[1][2 * BL_UNITS + u]);
      float go = pre[3 * EH + j] + (gpart[0][3 * BL_UNITS + u] + gpart[1][3 * BL_UNITS + u]);
      const float c = sigm(gf) * cst[u] + sigm(gi) * tanhf(gg);
      const float hn = sigm(go) * tanhf(c);
      cst[u] = c;
      mem[t * EMB + dir * EH + j] = hn;
      float* nxt = hbuf[(s + 1) & 1];
#pragma unroll
      for (int q = 0; q < BL_CLUSTER; ++q) cluster.map_shared_rank(nxt, q)[j] = hn;
    }
    cluster.sync();
    (void)grow;
  }
}

// pm[t][a] = sum_k mem[t][k] WmT[k][a]; 16 rows per block.
__global__ void __launch_bounds__(256) k_pmem(const int64_t* __restrict__ plan, const float* __restrict__ WmT) {
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
  const int64_t* p = plan + blockIdx.y * 5;
  const int64_t span = 2 * p[2] + p[1];
  const int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (r >= span) return;
  const int64_t q = r - p[2];
  row_out[p[0] + r] = (q >= 0 && q < p[1]) ? (int32_t)(p[3] + p[4] * q) : -1;
}

// zero plan[i] = {base, rows, halo}: zero [base, base+halo) and [base+halo+rows, base+2halo+rows).
__global__ void k_zero_halo(const int64_t* __restrict__ plan, __nv_bfloat16* __restrict__ X, int C) {
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

__global__ void __launch_bounds__(256) k_post_splice(const __nv_bfloat16* __restrict__ X4,
                                                     const int64_t* __restrict__ plan,
                                                     const float* __restrict__ wpost,  // [32][7]
                                                     float bpost, const float* __restrict__ fade, int O, int S,
                                                     float* __restrict__ audio) {
  const int64_t* p = plan + blockIdx.y * PPLAN;
  const int64_t G = p[1];
  const bool has_tail = p[2] & 1, is_last = p[2] & 2;
  const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
  __shared__ float w[32 * 7];
  if (threadIdx.x < 32 * 7) w[threadIdx.x] = wpost[threadIdx.x];
  __syncthreads();
  float* dst = reinterpret_cast<float*>(p[4]);
  if (!is_last && g < (int64_t)O * NMEL) {  // new mel tail = last O frames of this chunk
    const float* mel = reinterpret_cast<const float*>(p[6]);
    dst[g] = mel[(p[7] - O) * NMEL + g];
  }
  if (g >= G) return;
  const __nv_bfloat16* x = X4 + (p[0] + g - 3) * 32;
  float acc = bpost;
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    const __nv_bfloat162* row = reinterpret_cast<const __nv_bfloat162*>(x + j * 32);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float2 f = __bfloat1622float2(row[c]);
      acc = fmaf(w[(2 * c) * 7 + j], f.x, fmaf(w[(2 * c + 1) * 7 + j], f.y, acc));
    }
  }
  float v = tanhf(acc);
  const int64_t count = is_last ? G : G - S;
  if (g < count) {
    if (has_tail && g < S) v = fade[g] * v + fade[S + g] * reinterpret_cast<const float*>(p[3])[g];
    audio[p[5] + g] = v;
  } else {
    dst[(int64_t)O * NMEL + (g - count)] = v;  // held tail for the next seam
  }
}

dim3 grid2(int64_t work, int n) { return dim3((unsigned)((work + 255) / 256), (unsigned)n); }

}  // namespace

// ----------------------------------------------------------------- C ABI
ITTS_API int itts_r_dec_prepare(const float* state, void* xb, int32_t B, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  k_dec_prepare<<<B, 256, 0, (cudaStream_t)stream>>>(state, (__nv_bfloat16*)xb);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_prenet(float* state, void* xb, const float* W0T, const float* W1T, const int64_t* plan,
                           int32_t B, int32_t step, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  k_prenet<<<(B + IT - 1) / IT, 256, 0, (cudaStream_t)stream>>>(state, (__nv_bfloat16*)xb, W0T, W1T, plan, step, B);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_query(const float* state, const float* WqT, float* Q, int32_t B, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_query, cudaFuncAttributeMaxDynamicSharedMemorySize, IT * HID * 4);
    configured = true;
  }
  k_query<<<(B + IT - 1) / IT, 256, IT * HID * 4, (cudaStream_t)stream>>>(state, WqT, Q, B);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_lstm_cell(const float* G, float* state, void* xb, int32_t h_off, int32_t c_off,
                              const int64_t* plan, int32_t B, int32_t step, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  k_lstm_cell<<<(B * HID + 255) / 256, 256, 0, (cudaStream_t)stream>>>(G, state, (__nv_bfloat16*)xb, h_off,
                                                                       c_off, plan, step, B);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_attention(float* state, void* xb, const int64_t* plan, int32_t B, int32_t max_len,
                              const float* Q, const float* Wloc, const float* WdT, const float* v,
                              int32_t step, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  const size_t smem = (size_t)3 * max_len * sizeof(float);
  if (smem > 160 * 1024) return ITTS_EUNSUPPORTED;  // L <= 13653 phonemes
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    configured = true;
  }
  k_attention<<<B, 256, smem, (cudaStream_t)stream>>>(state, (__nv_bfloat16*)xb, plan, Q, Wloc, WdT, v, step);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_proj(float* state, const int64_t* plan, int32_t B, const float* WpT, const float* bp,
                         int32_t step, void* stream) {
  if (B <= 0) return B == 0 ? ITTS_OK : ITTS_EINVAL;
  constexpr int smem = (IT * 1536 + 3 * IT * 81) * 4;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_proj, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  k_proj<<<(B + IT - 1) / IT, 256, smem, (cudaStream_t)stream>>>(state, plan, WpT, bp, step, B);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_enc_embed(const int32_t* tok4, int64_t total, const int64_t* plan, int32_t n,
                              int64_t max_len, const float* Eph, const float* Epw, const float* Epph,
                              const float* Eiph, void* X, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  k_enc_embed<<<grid2(max_len * EMB, n), 256, 0, (cudaStream_t)stream>>>(tok4, total, plan, Eph, Epw, Epph, Eiph,
                                                                        (__nv_bfloat16*)X);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_bilstm(const float* PRE, const int64_t* plan, int32_t n, const float* WhhT, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const size_t smem = (size_t)EH * BL_ROWS * sizeof(float);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_bilstm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  k_bilstm<<<n * 2 * BL_CLUSTER, 256, smem, (cudaStream_t)stream>>>(PRE, plan, WhhT);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_pmem(const int64_t* plan, int32_t n, int64_t max_len, const float* WmT, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  dim3 grid((unsigned)((max_len + 15) / 16), (unsigned)n);
  k_pmem<<<grid, 256, 0, (cudaStream_t)stream>>>(plan, WmT);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_mel_assemble(const int64_t* plan, int32_t n, int64_t max_rows, void* X0, int32_t ld,
                                 void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  k_mel_assemble<<<grid2(max_rows * ld, n), 256, 0, (cudaStream_t)stream>>>(plan, (__nv_bfloat16*)X0, ld);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_rowmap(const int64_t* plan, int32_t n, int64_t max_span, int32_t* row_out, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  k_rowmap<<<grid2(max_span, n), 256, 0, (cudaStream_t)stream>>>(plan, row_out);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_zero_halo(const int64_t* plan, int32_t n, int64_t max_halo, void* X, int32_t C,
                              void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  k_zero_halo<<<grid2(2 * max_halo * C, n), 256, 0, (cudaStream_t)stream>>>(plan, (__nv_bfloat16*)X, C);
  ITTS_RETURN_LAUNCH();
}

ITTS_API int itts_r_post_splice(const void* X4, const int64_t* plan, int32_t n, int64_t max_g,
                                const float* wpost, float bpost, const float* fade, int32_t overlap_frames,
                                int32_t overlap_samples, float* audio, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const int64_t work = max(max_g, (int64_t)overlap_frames * NMEL);
  k_post_splice<<<grid2(work, n), 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)X4, plan, wpost, bpost,
                                                                  fade, overlap_frames, overlap_samples, audio);
  ITTS_RETURN_LAUNCH();
}
