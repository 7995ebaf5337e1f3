// K5 recurrence on the tensor cores: the Tacotron2 encoder BiLSTM for a group of up to 32 items per
// 8-CTA cluster and direction (replaces one cluster per (item, direction) of k_bilstm in tier_r.cu for
// pooled encoder batches; reference encode_batch, src/acoustic.py:222-231, with the Tacotron2
// encoder of SURVEY Appendix B).
//
// CTA r of a cluster owns hidden units [32r, 32r+32), i.e. 128 gate rows ordered [unit][gate]. Per
// step: gates[128 rows][items] = Whh_slice[128 x 256] . h[items x 256]^T as ONE tcgen05 MMA chain
// (weights as M, resident in shared memory for the whole sequence; h split into bf16 hi + lo parts,
// so with bf16-exact weights the products Wh.(hh + hl) are fp32-level, fp32 accumulation in TMEM),
// then the LSTM cell per (unit, item) from the 4 gate rows of a TMEM lane quad, and the new h of
// the CTA's 32 units goes to every CTA of the cluster with st.async completing bytes on the
// receiver's mbarrier (double-buffered by step parity).  Items shorter than the group's longest step
// through as inactive (no output; their h bytes are still sent so the byte count stays fixed).
// Each item's arithmetic is independent of the other items of its group (MMA columns are
// independent): a request encodes to the same bits in any pooled batch.

#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "tcgen05.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int EH = 256, EMB = 512, EPLAN = 6, CL = 8, UNITS = EH / CL, ROWS = 4 * UNITS;  // 32 units, 128 rows
constexpr int MAXG = 32;                 // items per cluster
constexpr int NTHR = 256;
constexpr uint32_t W_BYTES = 4 * ROWS * 128;        // 4 K-chunks x [128 rows][64 bf16], 128B swizzle
constexpr uint32_t H_BYTES = 4 * MAXG * 128;        // 4 K-chunks x [32 items][64 bf16]

struct Smem {
  uint8_t w[W_BYTES];                   // A operand (resident)
  uint8_t hh[H_BYTES], hl[H_BYTES];     // B operand: bf16 high / low parts of h(s)
  float hs[2][MAXG][EH];                // received h (fp32), by step parity
  uint64_t wbar, hbar[2], mbar;
  uint32_t tmem;
  int64_t L[MAXG], row0[MAXG];
  float* out[MAXG];
};

__device__ __forceinline__ uint32_t map_rank(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ float sigm_f(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float tanh_f(float x) { return 1.0f - __fdividef(2.0f, 1.0f + __expf(2.0f * x)); }
// 128B-swizzled K-major tile element (row r, column c < 64), in bf16 elements
__device__ __forceinline__ int swz(int r, int c) { return r * 64 + ((((c >> 3) ^ (r & 7))) << 3) + (c & 7); }

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NTHR, 1)
    k_bilstm_tc(const float* __restrict__ PRE, const int64_t* __restrict__ plan, int n, int G,
                const __nv_bfloat16* __restrict__ Wt) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int pair = blockIdx.x / CL, grp = pair >> 1, dir = pair & 1;
  const int i0 = grp * G, ng = min(G, n - i0), npad = (ng + 15) / 16 * 16;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(tcg::align_smem_1024(smem_raw));
  itts::pdl_trigger();

  if (tid == 0) {
    tcg::mbar_init(&sm.wbar, 1);
    tcg::mbar_init(&sm.mbar, 1);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tcg::smem_u32(&sm.hbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tcg::smem_u32(&sm.hbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(tcg::smem_u32(&sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {  // this CTA's weight slice, pre-swizzled on the host: one bulk copy
    tcg::mbar_expect_tx(&sm.wbar, W_BYTES);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tcg::smem_u32(sm.w)),
                 "l"(Wt + ((int64_t)dir * CL + rank) * (W_BYTES / 2)), "r"(W_BYTES), "r"(tcg::smem_u32(&sm.wbar))
                 : "memory");
  }
  for (int i = tid; i < (int)(H_BYTES / 4); i += NTHR) {   // h(0) = 0 (and zero pad rows for good)
    reinterpret_cast<uint32_t*>(sm.hh)[i] = 0u;
    reinterpret_cast<uint32_t*>(sm.hl)[i] = 0u;
  }
  itts::pdl_wait();  // PRE (the input projection) comes from the previous kernel
  if (tid < ng) {
    const int64_t* p = plan + (int64_t)(i0 + tid) * EPLAN;
    sm.L[tid] = p[1];
    sm.row0[tid] = p[2];
    sm.out[tid] = reinterpret_cast<float*>(p[3]);
  }
  __syncthreads();
  int64_t maxL = 0;
  for (int g = 0; g < ng; ++g) maxL = max(maxL, sm.L[g]);
  const uint32_t hb0 = tcg::smem_u32(&sm.hbar[0]);
  const uint32_t xbytes = (uint32_t)(EH * 4 * ng);   // the group's h from the 8 CTAs
  auto expect = [&](int b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(hb0 + 8 * b), "r"(xbytes) : "memory");
  };
  if (tid == 0 && maxL > 1) expect(1);   // h(1) lands in buffer 1
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cluster.sync();   // barriers initialised and h(0) tiles zero everywhere before any remote write
  tcg::mbar_wait(&sm.wbar, 0);

  // epilogue ownership: warp w reads TMEM lanes 32 (w % 4).. (units 8 (w % 4) .. +8, 4 gates each)
  // for the items of half w / 4; the lane with gate index g owns the cells of items j = g mod 4
  const int qd = warp & 3, hf = warp >> 2, g4 = lane & 3;
  const int u = qd * 8 + (lane >> 2);          // local unit 0..31
  const int hw = npad / 2;                     // items per half (8 or 16)
  constexpr int OWN = MAXG / 2 / 4;            // cells per lane (items j = g4, g4 + 4, .. of the half)
  float cst[OWN], pre_n[OWN][4];
#pragma unroll
  for (int o = 0; o < OWN; ++o) cst[o] = 0.f;
  auto load_pre = [&](int64_t s) {
#pragma unroll
    for (int o = 0; o < OWN; ++o) {
      const int j = hf * hw + g4 + 4 * o;
      if (4 * o + g4 < hw && j < ng && s < sm.L[j]) {
        const int64_t t = dir ? sm.L[j] - 1 - s : s;
        const float* pr = PRE + (sm.row0[j] + t) * (8 * EH) + dir * 4 * EH + rank * UNITS + u;
#pragma unroll
        for (int q = 0; q < 4; ++q) pre_n[o][q] = pr[q * EH];
      }
    }
  };
  load_pre(0);
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(npad >> 3) << 17) | ((128u >> 4) << 24);
  for (int64_t s = 0; s < maxL; ++s) {
    const int cur = (int)(s & 1);
    if (s > 0) {
      wait_cluster(hb0 + 8 * cur, (uint32_t)((s - 1) >> 1) & 1u);   // h(s) from every CTA
      if (tid == 0 && s + 2 < maxL) expect(cur);                     // h(s+2) lands here next
      // h(s) fp32 -> bf16 high / low operand tiles (row = item, K column = unit)
      for (int e = tid; e < ng * EH; e += NTHR) {
        const int j = e / EH, k = e - j * EH;
        const float v = sm.hs[cur][j][k];
        const __nv_bfloat16 hi = __float2bfloat16_rn(v);
        const int off = (k >> 6) * (MAXG * 64) + swz(j, k & 63);
        reinterpret_cast<__nv_bfloat16*>(sm.hh)[off] = hi;
        reinterpret_cast<__nv_bfloat16*>(sm.hl)[off] = __float2bfloat16_rn(v - __bfloat162float(hi));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
    } else if (tid == 0 && maxL > 2) {
      expect(0);   // h(2)
    }
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const uint8_t* hsrc = part ? sm.hl : sm.hh;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          const uint64_t dw = tcg::make_desc<128>(tcg::smem_u32(sm.w + kc * ROWS * 128));
          const uint64_t dh = tcg::make_desc<128>(tcg::smem_u32(hsrc + kc * MAXG * 128));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)   // 8 independent accumulators (part, K chunk): short MMA chains
            tcg::umma_bf16(sm.tmem + (part * 4 + kc) * MAXG, dw + 2 * kk, dh + 2 * kk, idesc, kk != 0);
        }
      }
      tcg::umma_commit(&sm.mbar);
    }
    float pre_c[OWN][4];
#pragma unroll
    for (int o = 0; o < OWN; ++o)
#pragma unroll
      for (int q = 0; q < 4; ++q) pre_c[o][q] = pre_n[o][q];
    load_pre(s + 1);
    tcg::mbar_wait(&sm.mbar, (uint32_t)(s & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // gates = the 8 partial accumulators (hi part K-chunks 0..3, then lo part) summed in that order
    float x[16];
    tcg::tmem_ld16(sm.tmem + ((uint32_t)(qd * 32) << 16) + hf * hw, x);   // columns beyond npad unused
#pragma unroll
    for (int a8 = 1; a8 < 8; ++a8) {
      float y[16];
      tcg::tmem_ld16(sm.tmem + ((uint32_t)(qd * 32) << 16) + a8 * MAXG + hf * hw, y);
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] += y[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    const int nxt = cur ^ 1;
    // Gather: for each owned slot o, lane (quad q, gate g4) needs gates 0..3 of column c = 4 o + g4.
    // Lane with gate gq holds column c in x[c]; shuffle x[4 o + g] from lane (quad | gq) for every g:
    // the requested column index depends on the receiving lane's g4, so shuffle each of the 4
    // candidate columns and keep the matching one.
#pragma unroll
    for (int o = 0; o < OWN; ++o) {
      if (4 * o >= hw) break;
      float gsel[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int cg4 = 0; cg4 < 4; ++cg4) {
          const float v = __shfl_sync(0xffffffffu, x[4 * o + cg4], (lane & ~3) | q);
          if (cg4 == g4) gsel[q] = v;
        }
      }
      const int j = hf * hw + g4 + 4 * o;
      if (4 * o + g4 >= hw || j >= ng) continue;
      const int k = rank * UNITS + u;
      const bool act = s < sm.L[j];
      float hn = 0.f;
      if (act) {
        const float gi = gsel[0] + pre_c[o][0], gf = gsel[1] + pre_c[o][1];
        const float gg = gsel[2] + pre_c[o][2], go = gsel[3] + pre_c[o][3];
        const float c = sigm_f(gf) * cst[o] + sigm_f(gi) * tanh_f(gg);
        hn = sigm_f(go) * tanh_f(c);
        cst[o] = c;
        const int64_t t = dir ? sm.L[j] - 1 - s : s;
        sm.out[j][t * EMB + dir * EH + k] = hn;
      }
      if (s + 1 < maxL) {
        const uint32_t dst = tcg::smem_u32(&sm.hs[nxt][j][k]), bar = hb0 + 8 * nxt;
#pragma unroll
        for (int rr = 0; rr < CL; ++rr)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                           map_rank(dst, rr)),
                       "r"(__float_as_uint(hn)), "r"(map_rank(bar, rr))
                       : "memory");
      }
    }
    __syncthreads();   // TMEM read and the operand tiles free for the next step
  }
  cluster.sync();   // no CTA leaves while a peer may still address its shared memory
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(sm.tmem));
  }
}

}  // namespace

// Encoder BiLSTM for n items on the tensor cores.  Wt = bf16 [2 dir][8 rank][4 K-chunks][128 rows
// = 32 units x 4 gates][64] with the 128B swizzle (rows of rank r: gate g of unit 32 r + u at row
// 4 u + g; K = the 256 recurrent inputs), exactly the encoder's W_hh when it is bf16-exact;
// PRE / plan as itts_r_bilstm.
int bilstm_tc_launch(const float* PRE, const int64_t* plan, int32_t n, const void* Wt, void* stream) {
  if (n <= 0) return n == 0 ? ITTS_OK : ITTS_EINVAL;
  const int ngrp = (n + MAXG - 1) / MAXG, G = (n + ngrp - 1) / ngrp;   // balanced groups of <= 32
  const size_t smem = sizeof(Smem) + 1024;
  static uint64_t configured = 0;
  if (!(configured & itts::device_bit())) {
    const cudaError_t a = cudaFuncSetAttribute(k_bilstm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (a != cudaSuccess) return (int)a;
    configured |= itts::device_bit();
  }
  const cudaError_t e = itts::launch_pdl_cls(itts::PDL_BILSTM, k_bilstm_tc, dim3(ngrp * 2 * CL), dim3(NTHR), smem,
                                             (cudaStream_t)stream, PRE, plan, (int)n, G,
                                             (const __nv_bfloat16*)Wt);
  return e == cudaSuccess ? ITTS_OK : (int)e;
}

ITTS_API int itts_r_bilstm_tc(const float* PRE, const int64_t* plan, int32_t n, const void* Wt, void* stream) {
  if (!PRE || !plan || !Wt) return ITTS_EINVAL;
  return bilstm_tc_launch(PRE, plan, n, Wt, stream);
}
