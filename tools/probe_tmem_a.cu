// Probe: tcgen05.mma kind::f16 with the A operand (M = 128 weight rows, K = 64) read from TMEM
// instead of shared memory.  A is written with tcgen05.st 32x32b (thread = lane = row, 32-bit
// column j = bf16 pair (k = 2j, 2j + 1), low half = even k); the result must equal the smem-A
// MMA bit for bit.  A second TMEM copy with the halves swapped shows the packing is not ignored.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2211_13939_b200/csrc tools/probe_tmem_a.cu -o /tmp/p
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "tcgen05.cuh"

constexpr int N = 16;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
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
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ int swz(int r, int k) { return r * 64 + ((((k >> 3) ^ (r & 7))) << 3) + (k & 7); }

__global__ void k_probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* out) {
  __shared__ __align__(1024) __nv_bfloat16 sA[128 * 64];
  __shared__ __align__(1024) __nv_bfloat16 sB[N * 64];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, q = t >> 5;
  for (int i = t; i < 128 * 64; i += 128) sA[swz(i / 64, i % 64)] = A[i];
  for (int i = t; i < N * 64; i += 128) sB[swz(i / 64, i % 64)] = B[i];
  if (q == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(tcg::smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    tcg::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  // A into TMEM: columns 64.. (natural packing) and 96.. (halves swapped), lane = row
  {
    const int r = t;
    uint32_t w[32], v[32];
    for (int j = 0; j < 32; ++j) {
      const uint16_t lo = __bfloat16_as_ushort(A[r * 64 + 2 * j]), hi = __bfloat16_as_ushort(A[r * 64 + 2 * j + 1]);
      w[j] = (uint32_t)lo | ((uint32_t)hi << 16);
      v[j] = (uint32_t)hi | ((uint32_t)lo << 16);
    }
    tmem_st32(tm + ((uint32_t)(32 * q) << 16) + 64, w);
    tmem_st32(tm + ((uint32_t)(32 * q) << 16) + 96, v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const uint32_t idesc = tcg::make_idesc<N>();
    const uint64_t da = tcg::make_desc<128>(tcg::smem_u32(sA)), db = tcg::make_desc<128>(tcg::smem_u32(sB));
    for (int kk = 0; kk < 4; ++kk) tcg::umma_bf16(tm + 0, da + 2 * kk, db + 2 * kk, idesc, kk != 0);
    for (int kk = 0; kk < 4; ++kk) umma_ts(tm + 16, tm + 64 + 8 * kk, db + 2 * kk, idesc, kk != 0);
    for (int kk = 0; kk < 4; ++kk) umma_ts(tm + 32, tm + 96 + 8 * kk, db + 2 * kk, idesc, kk != 0);
    tcg::umma_commit(&bar);
  }
  tcg::mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int v = 0; v < 3; ++v) {
    float d[16];
    tcg::tmem_ld16(tm + ((uint32_t)(32 * q) << 16) + 16 * v, d);
    for (int n = 0; n < 16; ++n) out[(v * 128 + t) * 16 + n] = d[n];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (q == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

int main() {
  std::vector<__nv_bfloat16> A(128 * 64), B(N * 64);
  std::vector<float> fa(A.size()), fb(B.size());
  srand(7);
  for (size_t i = 0; i < A.size(); ++i) { A[i] = __float2bfloat16((rand() % 2001 - 1000) / 1000.f); fa[i] = __bfloat162float(A[i]); }
  for (size_t i = 0; i < B.size(); ++i) { B[i] = __float2bfloat16((rand() % 2001 - 1000) / 1000.f); fb[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB;
  float* dO;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dO, 3 * 128 * 16 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  k_probe<<<1, 128>>>(dA, dB, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> o(3 * 128 * 16);
  cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
  double err[3] = {0, 0, 0};
  int diff_bits = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < 64; ++k) ref += (double)fa[m * 64 + k] * fb[n * 64 + k];
      for (int v = 0; v < 3; ++v) err[v] = fmax(err[v], fabs(o[(v * 128 + m) * 16 + n] - ref));
      diff_bits += o[(0 * 128 + m) * 16 + n] != o[(1 * 128 + m) * 16 + n];
    }
  printf("smem-A max err %.3g | tmem-A natural %.3g (bit differences vs smem-A: %d) | tmem-A swapped %.3g\n",
         err[0], err[1], diff_bits, err[2]);
  return 0;
}
