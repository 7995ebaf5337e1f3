// Tier S: the reference's deterministic stand-in models, fp64, on the GPU.
//
//   K2 itts_s_encode        encode()        pkg/src/incrtts/acoustic.py:41-65
//                            seeded_vector() pkg/src/incrtts/domain.py:22-52
//   K3 itts_s_decode_chunk  decode_chunk()  pkg/src/incrtts/acoustic.py:136-219
//   K4 itts_s_vocode_chunk  vocode_chunk()  pkg/src/incrtts/vocoder.py:52-136
//
// Compiled with -fmad=false so every product and sum rounds exactly like
// the reference's separate numpy ops; reductions follow numpy's order where
// that is knowable (axis-0 means are sequential, 8-wide row means are
// numpy's pairwise block), so encoder rows and vocoder samples are
// bit-identical to the reference and decoder frames agree to ~1 ulp.
//
// All per-item addressing comes from a host-built int64 "plan" (absolute
// device pointers + sizes), so items may live anywhere in the ragged state
// arena and batches may be any subset in any order.

#include "common.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// seeded_vector(table, token, .)[d]: table<<56 | token<<16 | d, top 53 bits -> [-1, 1).
__device__ __forceinline__ double seeded(int table, int64_t token, int d) {
  const uint64_t key = ((uint64_t)(table & 0xFF) << 56) |
                       (((uint64_t)token & 0xFFFFFFFFFFull) << 16) | (uint64_t)(d & 0xFFFF);
  const uint64_t h = splitmix64(key) >> 11;
  return (double)h / 9007199254740992.0 * 2.0 - 1.0;
}

// numpy pairwise_sum for a short contiguous row (n <= 128 here).
template <int N>
__device__ __forceinline__ double np_pairwise_sum(const double* a) {
  if constexpr (N < 8) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) r += a[i];
    return r;
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    constexpr int body = N - (N % 8);
#pragma unroll
    for (int i = 8; i < body; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
    for (int i = body; i < N; ++i) res += a[i];
    return res;
  }
}

// ---------------------------------------------------------------- K2 encode
// plan[i] = {tok_off, L, feat_ptr, state_ptr}; tok4 = [4][total] int32.
template <int D>
__global__ void __launch_bounds__(kThreads) k_embed(const int32_t* __restrict__ tok4, int64_t total,
                                                    const int64_t* __restrict__ plan,
                                                    double* __restrict__ summed) {
  const int64_t* p = plan + 4 * blockIdx.y;
  const int64_t off = p[0], L = p[1];
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= L * D) return;
  const int64_t t = g / D;
  const int d = (int)(g % D);
  const int64_t idx = off + t;
  // ((phoneme + pw) + pph) + iph -- acoustic.py:52-59 evaluation order.
  const double v = ((seeded(0, tok4[idx], d) + seeded(1, tok4[total + idx], d)) +
                    seeded(2, tok4[2 * total + idx], d)) + seeded(3, tok4[3 * total + idx], d);
  summed[idx * D + d] = v;
}

template <int D>
__global__ void k_prefix(const int64_t* __restrict__ plan, const double* __restrict__ summed,
                         double* __restrict__ prefix) {
  const int64_t* p = plan + 4 * blockIdx.x;
  const int64_t off = p[0], L = p[1];
  const int d = threadIdx.x;
  if (d >= D) return;
  double s = 0.0;
  for (int64_t t = 0; t < L; ++t) {  // numpy axis-0 reduce: sequential from row 0
    s = s + summed[(off + t) * D + d];
    prefix[(off + t) * D + d] = s;
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_rows(const int64_t* __restrict__ plan,
                                                   const double* __restrict__ summed,
                                                   const double* __restrict__ prefix) {
  const int64_t* p = plan + 4 * blockIdx.y;
  const int64_t off = p[0], L = p[1];
  double* feat = reinterpret_cast<double*>(p[2]);
  double* state = reinterpret_cast<double*>(p[3]);
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  // Zero the initial decoder state (6 D-vectors + W + W_acc): acoustic.py:118-133.
  for (int64_t z = g; z < 6 * D + 2 * L; z += (int64_t)gridDim.x * kThreads) state[z] = 0.0;
  if (g >= L * D) return;
  const int64_t t = g / D;
  const int d = (int)(g % D);
  const double* x = summed + off * D + d;
  // suffix mean: summed[t:].mean(axis=0) sums forward from row t.
  double suf = 0.0;
  for (int64_t u = t; u < L; ++u) suf = suf + x[u * D];
  const double pre = prefix[(off + t) * D + d];
  feat[t * D + d] = ((x[t * D] + pre / (double)(t + 1)) + suf / (double)(L - t)) / 3.0;
}

// ---------------------------------------------------------------- K3 decode
// plan[i] = {feat_ptr, L, src_state_ptr, dst_state_ptr, steps, mel_ptr}.
// State region: [last, ctx, h_att, c_att, h_dec, c_dec] (6 x D), W[L], W_acc[L].
template <int D>
__global__ void __launch_bounds__(kThreads) k_decode(const int64_t* __restrict__ plan, double penalty) {
  const int64_t* p = plan + 6 * blockIdx.x;
  const double* __restrict__ rows = reinterpret_cast<const double*>(p[0]);
  const int64_t L = p[1];
  const double* src = reinterpret_cast<const double*>(p[2]);
  double* dst = reinterpret_cast<double*>(p[3]);
  const int steps = (int)p[4];
  double* mel = reinterpret_cast<double*>(p[5]);

  __shared__ double s_vec[6][D];  // last, ctx, h_att, c_att, h_dec, c_dec
  __shared__ double s_red[32];
  __shared__ double s_ctx[kThreads / 32][D];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 6 * D) s_vec[tid / D][tid % D] = src[tid];
  __syncthreads();

  double* W = dst + 6 * D;
  double* Wacc = W + L;
  const double* Wacc_src = src + 6 * D + L;

  for (int step = 0; step < steps; ++step) {
    const double* wacc_in = step == 0 ? Wacc_src : Wacc;
    if (tid < D) {  // attention cell: fold(tanh(M_last), A) -- acoustic.py:136-146, :165
      const double fold = tanh(s_vec[0][tid]) + s_vec[1][tid];
      const double c = tanh((0.5 * s_vec[3][tid] + 0.5 * fold) + 0.25 * s_vec[2][tid]);
      s_vec[3][tid] = c;
      s_vec[2][tid] = tanh(c);
    }
    __syncthreads();
    double h[D];
#pragma unroll
    for (int d = 0; d < D; ++d) h[d] = s_vec[2][d];
    // scores = rows @ h_att - lambda * W_acc
    double lmax = -INFINITY;
    for (int64_t t = tid; t < L; t += kThreads) {
      const double* r = rows + t * D;
      double s = r[0] * h[0];
#pragma unroll
      for (int d = 1; d < D; ++d) s = s + r[d] * h[d];
      s = s - penalty * wacc_in[t];
      W[t] = s;
      lmax = fmax(lmax, s);
    }
    const double M = itts::block_reduce<double, true>(lmax, s_red);
    double lsum = 0.0;
    for (int64_t t = tid; t < L; t += kThreads) {
      const double e = exp(W[t] - M);
      W[t] = e;
      lsum += e;
    }
    const double Z = itts::block_reduce<double, false>(lsum, s_red);
    double part[D];
#pragma unroll
    for (int d = 0; d < D; ++d) part[d] = 0.0;
    for (int64_t t = tid; t < L; t += kThreads) {
      const double w = W[t] / Z;
      W[t] = w;
      Wacc[t] = wacc_in[t] + w;
      const double* r = rows + t * D;
#pragma unroll
      for (int d = 0; d < D; ++d) part[d] = part[d] + w * r[d];
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double v = itts::warp_sum(part[d]);
      if (lane == 0) s_ctx[warp][d] = v;
    }
    __syncthreads();
    if (tid < D) {
      double ctx = s_ctx[0][tid];
      for (int w = 1; w < kThreads / 32; ++w) ctx = ctx + s_ctx[w][tid];
      s_vec[1][tid] = ctx;
      // decoder cell on cat(h_att, ctx), then frame = tanh(h_dec + ctx)
      const double fold = s_vec[2][tid] + ctx;
      const double c = tanh((0.5 * s_vec[5][tid] + 0.5 * fold) + 0.25 * s_vec[4][tid]);
      const double hd = tanh(c);
      s_vec[5][tid] = c;
      s_vec[4][tid] = hd;
      const double frame = tanh(hd + ctx);
      s_vec[0][tid] = frame;
      mel[(int64_t)step * D + tid] = frame;
    }
    __syncthreads();
  }
  if (tid < 6 * D) dst[tid] = s_vec[tid / D][tid % D];
}

// ---------------------------------------------------------------- K4 vocode
// plan[i] = {mel_ptr, m, flags(1=has_tail, 2=is_last), src_vs_ptr, dst_vs_ptr, out_off, 0}.
// Vocoder-state region: mel_tail [O][D], held [S].
template <int D>
__device__ __forceinline__ double frame_mean(const double* tail, const double* mel, int t_tail, int64_t f) {
  const double* row = f < t_tail ? tail + f * D : mel + (f - t_tail) * D;
  return np_pairwise_sum<D>(row) / (double)D;
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_vocode(const int64_t* __restrict__ plan, int O, int H,
                                                     const double* __restrict__ fade,
                                                     double* __restrict__ audio) {
  const int64_t* p = plan + 7 * blockIdx.y;
  const double* mel = reinterpret_cast<const double*>(p[0]);
  const int64_t m = p[1];
  const bool has_tail = p[2] & 1, is_last = p[2] & 2;
  const double* src = reinterpret_cast<const double*>(p[3]);
  double* dst = reinterpret_cast<double*>(p[4]);
  const int64_t out_off = p[5];
  const int64_t S = (int64_t)O * H;
  const int t_tail = has_tail ? O : 0;
  const int64_t G = (t_tail + m) * H;
  const int64_t count = is_last ? G : G - S;
  const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (j < count) {
    double v = frame_mean<D>(src, mel, t_tail, j / H);
    if (has_tail && j < S) v = fade[j] * v + fade[S + j] * src[(int64_t)O * D + j];  // Eq. 3
    audio[out_off + j] = v;
  }
  if (!is_last) {
    if (j < S) dst[(int64_t)O * D + j] = frame_mean<D>(src, mel, t_tail, (G - S + j) / H);
    if (j < (int64_t)O * D) dst[j] = mel[(m - O) * D + j];
  }
}

template <int D>
int launch_encode(const int32_t* tok4, int64_t total, const int64_t* plan, int n, int64_t max_len,
                  double* summed, double* prefix, cudaStream_t st) {
  dim3 grid((unsigned)((max_len * D + kThreads - 1) / kThreads), (unsigned)n);
  k_embed<D><<<grid, kThreads, 0, st>>>(tok4, total, plan, summed);
  k_prefix<D><<<n, 32, 0, st>>>(plan, summed, prefix);
  const int64_t zmax = 6 * D + 2 * max_len;
  dim3 grid2((unsigned)((max(max_len * D, zmax) + kThreads - 1) / kThreads), (unsigned)n);
  k_rows<D><<<grid2, kThreads, 0, st>>>(plan, summed, prefix);
  ITTS_RETURN_LAUNCH();
}

}  // namespace

#define ITTS_DISPATCH_D(dim, ...)                   \
  switch (dim) {                                    \
    case 4: { constexpr int D = 4; __VA_ARGS__; }          \
    case 8: { constexpr int D = 8; __VA_ARGS__; }          \
    case 16: { constexpr int D = 16; __VA_ARGS__; }        \
    case 32: { constexpr int D = 32; __VA_ARGS__; }        \
    default: return ITTS_EUNSUPPORTED;              \
  }

ITTS_API int itts_s_encode(const int32_t* tok4, int64_t total_tokens, const int64_t* plan,
                           int32_t n_items, int64_t max_len, int32_t dim, double* scratch,
                           void* stream) {
  if (n_items <= 0) return n_items == 0 ? ITTS_OK : ITTS_EINVAL;
  if (!tok4 || !plan || !scratch || max_len <= 0) return ITTS_EINVAL;
  double* summed = scratch;
  double* prefix = scratch + total_tokens * dim;
  cudaStream_t st = (cudaStream_t)stream;
  ITTS_DISPATCH_D(dim, return launch_encode<D>(tok4, total_tokens, plan, n_items, max_len, summed,
                                               prefix, st));
}

ITTS_API int itts_s_decode_chunk(const int64_t* plan, int32_t n_items, int32_t dim, double penalty,
                                 void* stream) {
  if (n_items <= 0) return n_items == 0 ? ITTS_OK : ITTS_EINVAL;
  if (!plan) return ITTS_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  ITTS_DISPATCH_D(dim, {
    k_decode<D><<<n_items, kThreads, 0, st>>>(plan, penalty);
    ITTS_RETURN_LAUNCH();
  });
}

ITTS_API int itts_s_vocode_chunk(const int64_t* plan, int32_t n_items, int32_t dim,
                                 int32_t overlap_frames, int32_t hop, int64_t max_samples,
                                 const double* fade, double* audio, void* stream) {
  if (n_items <= 0) return n_items == 0 ? ITTS_OK : ITTS_EINVAL;
  if (!plan || !fade || !audio || overlap_frames < 1 || hop < 1 || max_samples < 1) return ITTS_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t need = max(max_samples, (int64_t)overlap_frames * max(hop, dim));
  dim3 grid((unsigned)((need + kThreads - 1) / kThreads), (unsigned)n_items);
  ITTS_DISPATCH_D(dim, {
    k_vocode<D><<<grid, kThreads, 0, st>>>(plan, overlap_frames, hop, fade, audio);
    ITTS_RETURN_LAUNCH();
  });
}
