// Probe: can a tcgen05 K-major SWIZZLE_128B smem descriptor start at an arbitrary
// row (start address + s*128 B, s not a multiple of 8)?  If yes, a conv tile can
// load its A rows (+halo) ONCE and serve every tap by shifting the descriptor.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o gpurun_out/probe_desc tools/probe_desc.cu
//
// One CTA: A = 144 x 64 bf16 (rows x K), B = 64 x 64 (N x K), both written by
// threads in the 128B-swizzled layout TMA would produce (16-byte chunk c of row
// r at r*128 + ((c ^ (r & 7)) * 16)).  For each shift s in 0..15 and for
// base_offset mode {0, (addr>>7)&7}: D = A[s:s+128] * B^T (M128 N64 K64, 4 MMAs)
// -> compare with a host reference.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int SWZ>
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, int base_mode) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(((8 * SWZ) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  if (base_mode == 1) d |= (uint64_t)((saddr >> 7) & 7) << 49;
  d |= (SWZ == 128 ? 2ull : 4ull) << 61;
  return d;
}

template <int SWZ>
__global__ void k_probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* out, int shift, int base_mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // 144 rows * 128 B = 18432
  uint8_t* sB = smem + 18432 + 1024;  // 64 rows * 128 B (1024-aligned)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 8192);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x;
  constexpr int CH = SWZ / 16, KW = SWZ / 2;
  auto sw = [](int r, int c) { return SWZ == 128 ? (c ^ (r & 7)) : (c ^ ((r >> 1) & 3)); };
  for (int i = tid; i < 144 * CH; i += blockDim.x) {
    const int r = i / CH, c = i % CH;
    *reinterpret_cast<uint4*>(sA + r * SWZ + sw(r, c) * 16) = *reinterpret_cast<const uint4*>(A + r * KW + c * 8);
  }
  for (int i = tid; i < 64 * CH; i += blockDim.x) {
    const int r = i / CH, c = i % CH;
    *reinterpret_cast<uint4*>(sB + r * SWZ + sw(r, c) * 16) = *reinterpret_cast<const uint4*>(B + r * KW + c * 8);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = make_desc<SWZ>(smem_u32(sA + shift * SWZ), base_mode);
    const uint64_t db = make_desc<SWZ>(smem_u32(sB), 0);
    for (int kk = 0; kk < SWZ / 32; ++kk) {
      const uint32_t acc = kk != 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  }
  __syncwarp();
  {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = tid >> 5, lane = tid & 31;
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * 64 + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  std::vector<__nv_bfloat16> hA(144 * 64), hB(64 * 64);
  std::vector<float> fA(144 * 64), fB(64 * 64);
  srand(1);
  for (int i = 0; i < 144 * 64; ++i) { float v = (rand() % 17 - 8) / 8.0f; hA[i] = __float2bfloat16(v); fA[i] = v; }
  for (int i = 0; i < 64 * 64; ++i) { float v = (rand() % 17 - 8) / 8.0f; hB[i] = __float2bfloat16(v); fB[i] = v; }
  __nv_bfloat16 *dA, *dB; float* dO;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 18432 + 1024 + 8192 + 1024 + 64;
  cudaFuncSetAttribute(k_probe<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> o(128 * 64);
  for (int swz = 64; swz <= 128; swz *= 2)
  for (int mode = 0; mode < 2; ++mode) {
    const int KW = swz / 2;
    for (int s = 0; s < 16; ++s) {
      cudaMemset(dO, 0, 128 * 64 * 4);
      if (swz == 128) k_probe<128><<<1, 128, smem>>>(dA, dB, dO, s, mode); else k_probe<64><<<1, 128, smem>>>(dA, dB, dO, s, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("swz %d mode %d shift %d: CUDA error %s\n", swz, mode, s, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int k = 0; k < KW; ++k) ref += (double)fA[(m + s) * KW + k] * fB[n * KW + k];
          maxerr = fmax(maxerr, fabs(ref - o[m * 64 + n]));
        }
      printf("swz %d base_mode %d shift %2d: max|err| %.3g %s\n", swz, mode, s, maxerr, maxerr < 1e-3 ? "OK" : "WRONG");
    }
  }
  return 0;
}
