// the paper's BERT prosodic-structure frontend (PAPER.md:39 -- "the text is first
// passed through a shared BERT backbone ... three separate linear layers predict pw, pph, iph";
// the reference replaces it with a rule, src/frontend.py:174-188).  BERT-base encoder (12 layers,
// hidden 768, 12 heads, FFN 3072, post-LN, GELU) over the characters of a pooled batch of texts,
// packed without padding ([sum of lengths][768]); each text attends only to itself.
//
//   embed + LayerNorm        k_bert_embed_ln (one warp per row)
//   QKV / out / FFN GEMMs    tcgen05 implicit-GEMM conv with one tap (tc_conv.cu), bias and GELU
//                            fused in its epilogue
//   self-attention           k_bert_attn (per (text, head): K/V staged in shared memory)
//   residual + LayerNorm     k_bert_add_ln
//   three prosody heads      k_bert_heads (argmax of three 2-way linear layers)
//
// The whole sequence is issued from C++ (itts_bert_prosody) with programmatic dependent launch.
#include <cuda_bf16.h>

#include "common.cuh"

namespace {

constexpr int HB = 768, NH = 12, HD = 64, FF = 3072, NL = 12, MAXLEN = 256;

__device__ __forceinline__ void ln_row(const float* v, int lane, const float* g, const float* b, float* of,
                                       __nv_bfloat16* ob) {
  // v: 24 values per lane (columns lane + 32 i); two-pass mean / variance in fp32, eps 1e-12
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < HB / 32; ++i) s += v[i];
  const float mean = itts::warp_sum(s) * (1.0f / HB);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < HB / 32; ++i) q += (v[i] - mean) * (v[i] - mean);
  const float rstd = rsqrtf(itts::warp_sum(q) * (1.0f / HB) + 1e-12f);
#pragma unroll
  for (int i = 0; i < HB / 32; ++i) {
    const int c = lane + 32 * i;
    const float y = (v[i] - mean) * rstd * g[c] + b[c];
    of[c] = y;
    ob[c] = __float2bfloat16_rn(y);
  }
}

__global__ void __launch_bounds__(256) k_bert_embed_ln(const int32_t* __restrict__ ids, const int32_t* __restrict__ pos,
                                                       int64_t rows, const float* __restrict__ tok,
                                                       const float* __restrict__ pe, const float* __restrict__ g,
                                                       const float* __restrict__ b, float* __restrict__ xf,
                                                       __nv_bfloat16* __restrict__ xb) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float* t = tok + (int64_t)ids[r] * HB;
  const float* p = pe + (int64_t)pos[r] * HB;
  float v[HB / 32];
#pragma unroll
  for (int i = 0; i < HB / 32; ++i) v[i] = t[lane + 32 * i] + p[lane + 32 * i];
  ln_row(v, lane, g, b, xf + r * HB, xb + r * HB);
}

__global__ void __launch_bounds__(256) k_bert_add_ln(const float* __restrict__ y, int64_t rows,
                                                     const float* __restrict__ g, const float* __restrict__ b,
                                                     float* __restrict__ xf, __nv_bfloat16* __restrict__ xb) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  float v[HB / 32];
#pragma unroll
  for (int i = 0; i < HB / 32; ++i) v[i] = xf[r * HB + lane + 32 * i] + y[r * HB + lane + 32 * i];
  ln_row(v, lane, g, b, xf + r * HB, xb + r * HB);
}

// One CTA per (text, head): K and V of the head staged in shared memory (fp32), each warp takes
// queries w, w + 8, ...; lanes split the keys for the scores, then the head dims for the output.
__global__ void __launch_bounds__(256) k_bert_attn(const __nv_bfloat16* __restrict__ qkv,
                                                   const int64_t* __restrict__ plan, __nv_bfloat16* __restrict__ out) {
  itts::pdl_trigger();
  itts::pdl_wait();
  extern __shared__ float sm[];
  const int item = blockIdx.x, h = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = plan[2 * item];
  const int L = (int)plan[2 * item + 1];
  float* sK = sm;                       // [L][HD + 1]
  float* sV = sK + MAXLEN * (HD + 1);   // [L][HD]
  float* sP = sV + MAXLEN * HD;         // [8 warps][L] probabilities
  float* sQ = sP + 8 * MAXLEN;          // [8 warps][HD]
  for (int i = tid; i < L * HD; i += 256) {
    const int j = i / HD, d = i - j * HD;
    const __nv_bfloat16* row = qkv + (r0 + j) * (3 * HB);
    sK[j * (HD + 1) + d] = __bfloat162float(row[HB + h * HD + d]);
    sV[j * HD + d] = __bfloat162float(row[2 * HB + h * HD + d]);
  }
  __syncthreads();
  const float scale = 0.125f;  // 1 / sqrt(64)
  for (int qi = warp; qi < L; qi += 8) {
    const __nv_bfloat16* qrow = qkv + (r0 + qi) * (3 * HB) + h * HD;
    sQ[warp * HD + lane] = __bfloat162float(qrow[lane]) * scale;
    sQ[warp * HD + lane + 32] = __bfloat162float(qrow[lane + 32]) * scale;
    __syncwarp();
    float mx = -INFINITY;
    for (int j = lane; j < L; j += 32) {
      float sc = 0.f;
#pragma unroll 16
      for (int d = 0; d < HD; ++d) sc = fmaf(sQ[warp * HD + d], sK[j * (HD + 1) + d], sc);
      sP[warp * MAXLEN + j] = sc;
      mx = fmaxf(mx, sc);
    }
    mx = itts::warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < L; j += 32) {
      const float e = __expf(sP[warp * MAXLEN + j] - mx);
      sP[warp * MAXLEN + j] = e;
      sum += e;
    }
    const float inv = 1.0f / itts::warp_sum(sum);
    __syncwarp();
    float o0 = 0.f, o1 = 0.f;
    for (int j = 0; j < L; ++j) {
      const float p = sP[warp * MAXLEN + j];
      o0 = fmaf(p, sV[j * HD + lane], o0);
      o1 = fmaf(p, sV[j * HD + lane + 32], o1);
    }
    __nv_bfloat16* orow = out + (r0 + qi) * HB + h * HD;
    orow[lane] = __float2bfloat16_rn(o0 * inv);
    orow[lane + 32] = __float2bfloat16_rn(o1 * inv);
    __syncwarp();
  }
}

// Three 2-way heads per row: tokens[r][k] = argmax(W[2k..2k+1] . x + b) (ties -> 0).
__global__ void __launch_bounds__(256) k_bert_heads(const float* __restrict__ x, int64_t rows,
                                                    const float* __restrict__ W, const float* __restrict__ bh,
                                                    float* __restrict__ logits, int32_t* __restrict__ tokens) {
  itts::pdl_trigger();
  itts::pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int i = lane; i < HB; i += 32) {
    const float xv = x[r * HB + i];
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] = fmaf(W[k * HB + i], xv, acc[k]);
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) acc[k] = itts::warp_sum(acc[k]) + bh[k];
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      logits[r * 6 + 2 * k] = acc[2 * k];
      logits[r * 6 + 2 * k + 1] = acc[2 * k + 1];
      tokens[r * 3 + k] = acc[2 * k + 1] > acc[2 * k] ? 1 : 0;
    }
  }
}

}  // namespace

// weights: tok_emb fp32 [V][768], pos_emb fp32 [512][768], ln_g, ln_b, then per layer
// (Wqkv bf16 [1][2304][768], bqkv, Wo bf16 [1][768][768], bo, ln1_g, ln1_b, W1 bf16 [1][3072][768],
// b1, W2 bf16 [1][768][3072], b2, ln2_g, ln2_b) x 12, then Wh fp32 [6][768], bh [6] (150 pointers).
// ids / pos int32 [rows]; plan int64 [n][2] {first row, length <= 256}; row_map int32 [rows] =
// identity; work: xf fp32 / xb bf16 [rows][768], qkv bf16 [rows][2304], att bf16 [rows][768],
// y fp32 [rows][768], h bf16 [rows][3072]; outputs logits fp32 [rows][6], tokens int32 [rows][3].
ITTS_API int itts_bert_prosody(const int32_t* ids, const int32_t* pos, const int64_t* plan, int32_t n, int64_t rows,
                               int32_t max_len, const int64_t* weights, const int32_t* row_map, float* xf, void* xb,
                               void* qkv, void* att, float* y, void* h, float* logits, int32_t* tokens,
                               void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  if (!ids || !pos || !plan || !weights || !row_map || rows < 1 || max_len < 1) return ITTS_EINVAL;
  if (max_len > MAXLEN) return ITTS_EUNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  auto P = [&](int i) { return reinterpret_cast<const void*>(weights[i]); };
  auto F = [&](int i) { return reinterpret_cast<const float*>(weights[i]); };
  const dim3 rgrid((unsigned)((rows + 7) / 8));
  cudaError_t e = itts::launch_pdl_cls(itts::PDL_BERT, k_bert_embed_ln, rgrid, dim3(256), 0, st, ids, pos, rows, F(0), F(1), F(2), F(3),
                                   xf, (__nv_bfloat16*)xb);
  if (e != cudaSuccess) return (int)e;
  const size_t att_smem = sizeof(float) * (MAXLEN * (HD + 1) + MAXLEN * HD + 8 * MAXLEN + 8 * HD);
  static uint64_t configured = 0;
  if (!(configured & itts::device_bit())) {
    if ((e = cudaFuncSetAttribute(k_bert_attn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)att_smem)) !=
        cudaSuccess)
      return (int)e;
    configured |= itts::device_bit();
  }
  const int32_t off0 = 0;
  int r;
  for (int l = 0; l < NL; ++l) {
    const int w = 4 + 12 * l;
    // qkv = x Wqkv^T + b (bf16 out)
    if ((r = conv1d_tc_impl(xb, rows, HB, HB, P(w), 3 * HB, 1, &off0, F(w + 1), 3 * HB, row_map, nullptr, 1.0f,
                            nullptr, 1, nullptr, 0, qkv, 1.0f, 0, 0, 0, stream)))
      return r;
    if ((e = itts::launch_pdl_cls(itts::PDL_BERT, k_bert_attn, dim3(n, NH), dim3(256), att_smem, st, (const __nv_bfloat16*)qkv, plan,
                              (__nv_bfloat16*)att)) != cudaSuccess)
      return (int)e;
    // y = att Wo^T + bo (fp32); x = LN(x + y)
    if ((r = conv1d_tc_impl(att, rows, HB, HB, P(w + 2), HB, 1, &off0, F(w + 3), HB, row_map, nullptr, 1.0f, y, 1,
                            nullptr, 0, nullptr, 1.0f, 0, 0, 0, stream)))
      return r;
    if ((e = itts::launch_pdl_cls(itts::PDL_BERT, k_bert_add_ln, rgrid, dim3(256), 0, st, (const float*)y, rows, F(w + 4), F(w + 5), xf,
                              (__nv_bfloat16*)xb)) != cudaSuccess)
      return (int)e;
    // h = GELU(x W1^T + b1) (bf16); y = h W2^T + b2; x = LN(x + y)
    if ((r = conv1d_tc_impl(xb, rows, HB, HB, P(w + 6), FF, 1, &off0, F(w + 7), FF, row_map, nullptr, 1.0f, nullptr,
                            1, nullptr, 0, h, 1.0f, 0, 0, 2, stream)))
      return r;
    if ((r = conv1d_tc_impl(h, rows, FF, FF, P(w + 8), HB, 1, &off0, F(w + 9), HB, row_map, nullptr, 1.0f, y, 1,
                            nullptr, 0, nullptr, 1.0f, 0, 0, 0, stream)))
      return r;
    if ((e = itts::launch_pdl_cls(itts::PDL_BERT, k_bert_add_ln, rgrid, dim3(256), 0, st, (const float*)y, rows, F(w + 10), F(w + 11), xf,
                              (__nv_bfloat16*)xb)) != cudaSuccess)
      return (int)e;
  }
  e = itts::launch_pdl_cls(itts::PDL_BERT, k_bert_heads, rgrid, dim3(256), 0, st, (const float*)xf, rows, F(4 + 12 * NL),
                       F(5 + 12 * NL), logits, tokens);
  return e == cudaSuccess ? ITTS_OK : (int)e;
}
