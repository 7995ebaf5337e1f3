// Native launch sequence of the HiFi-GAN V1 stack for one pooled vocoder call
// (the conv stack of vocode_batch, reference src/vocoder.py:92-143, behind the
// vocoder_batch plugin boundary src/modules.py:77-90).
//
// Python used to issue the ~55 launches of a call one ctypes call at a time; at
// small pooled batches that host issue time (~20 us per launch) exceeded the
// GPU time of the stack.  Here the whole sequence -- spliced-mel assembly,
// conv_pre, the four transposed convs, 36 fused ResBlock1 layers with the three
// MRF branches of a stage on three streams and one merge pass per stage, halo
// re-zeroing -- is issued from
// C++ after one H2D copy of a packed plan that holds every row map and halo plan
// of the call.  Work buffers are owned here (grow-only).  The arithmetic and
// the order of every accumulation are those of the per-call path in tier_r.py
// (fused_mrf, native_vocoder=False).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace {

int g_fail_line = 0;
#define FAIL_AT(x) (g_fail_line = __LINE__, (x))

constexpr int kStages = 4;
constexpr int kUps[kStages] = {8, 8, 2, 2};
constexpr int kStageC[kStages] = {256, 128, 64, 32};
constexpr int kResK[3] = {3, 7, 11};
constexpr int kResDil[3] = {1, 3, 5};
constexpr int kMelHalo = 3;   // conv_pre k7
constexpr int kMrfHalo = 25;  // k11 dilation 5
constexpr int kNumWeights = 2 * (1 + kStages + kStages * 3 * 3 * 2);  // (w, bias) pairs
constexpr int kPlanPerItem = 9 * 5 + 4 * 3;                             // 9 row maps + 4 halo plans
constexpr int ACC_NONE = 0, ACC_STORE = 1;

struct Layout {
  std::vector<int64_t> rows, base;
  int64_t halo = 0, total = 0, max_span = 0;
  void build(const std::vector<int64_t>& r, int64_t h) {
    rows = r;
    halo = h;
    base.resize(r.size());
    total = 0;
    max_span = 0;
    for (size_t i = 0; i < r.size(); ++i) {
      base[i] = total;
      total += r[i] + 2 * h;
      max_span = std::max(max_span, r[i] + 2 * h);
    }
  }
  int64_t first(size_t i) const { return base[i] + halo; }
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  int ensure(size_t n) {
    if (n <= cap) return ITTS_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(n + n / 4, 1024);
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e != cudaSuccess) return (int)e;
    // debug / test: ITTS_VOC_POISON=1 fills fresh work buffers with 0xFF bytes (bf16 NaN), so a test
    // can show that no output depends on a row (e.g. a halo) the launch sequence did not write
    const char* poison = getenv("ITTS_VOC_POISON");
    if (poison && poison[0] == '1' && (e = cudaMemset(p, 0xFF, want * sizeof(T))) != cudaSuccess) return (int)e;
    cap = want;
    return ITTS_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct Vocoder {
  const void* w[kNumWeights / 2];
  const float* b[kNumWeights / 2];
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t ev_x = nullptr, ev_side[2] = {nullptr, nullptr}, ev_plan = nullptr;
  DevBuf<uint16_t> x0, act_in, b16[12];
  DevBuf<int32_t> rowmaps;
  DevBuf<int64_t> dplan;
  int64_t* hplan = nullptr;
  size_t hplan_cap = 0;
  bool plan_pending = false;

  // weight index helpers: 0 conv_pre, 1..4 ups, then res[s][j][m][c1/c2]
  static int res_id(int s, int j, int m, int c) { return 1 + kStages + ((s * 3 + j) * 3 + m) * 2 + c; }

  int grow_all(cudaStream_t stream, size_t rows0, size_t big, size_t rm_total, size_t plan_n) {
    bool need = x0.cap < rows0 * 128 || act_in.cap < rows0 * 512 || rowmaps.cap < rm_total || dplan.cap < plan_n;
    for (auto& t : b16) need |= t.cap < big;
    if (!need) return ITTS_OK;
    // buffers may still be read by queued work: drain before freeing
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return (int)e;
    for (auto s : side)
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return (int)e;
    int st;
    if ((st = x0.ensure(rows0 * 128))) return st;
    if ((st = act_in.ensure(rows0 * 512))) return st;
    for (auto& t : b16)
      if ((st = t.ensure(big))) return st;
    if ((st = rowmaps.ensure(rm_total))) return st;
    if ((st = dplan.ensure(plan_n))) return st;
    return ITTS_OK;
  }

  int stage_rows(const std::vector<int64_t>& Ts, size_t* rows0, size_t* big, size_t* rm_total) const {
    int64_t r0 = 0, b = 0, rm = 0, sumT = 0, mult = 1;
    for (int64_t T : Ts) r0 += T + 2 * kMelHalo, sumT += T;
    int64_t n = (int64_t)Ts.size();
    rm = 2 * r0;  // rm0 + rmT0 (both over the mel layout)
    for (int s = 0; s < kStages; ++s) {
      mult *= kUps[s];
      int64_t rows = sumT * mult + n * 2 * kMrfHalo;
      b = std::max(b, rows * kStageC[s]);
      rm += rows * (s + 1 < kStages ? 2 : 1);  // rm_s (+ rmT_{s+1} over the same layout)
    }
    *rows0 = (size_t)r0;
    *big = (size_t)b;
    *rm_total = (size_t)rm;
    return ITTS_OK;
  }

  int reserve(cudaStream_t stream, int n, int frames) {
    std::vector<int64_t> Ts(n, frames);
    size_t rows0, big, rm;
    stage_rows(Ts, &rows0, &big, &rm);
    int st = grow_all(stream, rows0, big, rm, (size_t)n * kPlanPerItem);
    if (st) return st;
    return host_plan((size_t)n * kPlanPerItem);
  }

  int host_plan(size_t n) {
    if (plan_pending) {  // the previous call's copy must have left the staging buffer
      cudaError_t e = cudaEventSynchronize(ev_plan);
      if (e != cudaSuccess) return (int)e;
      plan_pending = false;
    }
    if (n <= hplan_cap) return ITTS_OK;
    if (hplan) cudaFreeHost(hplan);
    hplan = nullptr;
    hplan_cap = 0;
    size_t want = std::max<size_t>(n + n / 4, 4096);
    cudaError_t e = cudaHostAlloc((void**)&hplan, want * sizeof(int64_t), cudaHostAllocDefault);
    if (e != cudaSuccess) return (int)e;
    hplan_cap = want;
    return ITTS_OK;
  }

  int conv(const void* x, int64_t rows, int c_in, int id, int n_total, int taps, int dil, int c_out,
           const int32_t* row_out, void* act_out, float slope, int zero_halo, cudaStream_t st) {
    int32_t offs[16];
    for (int j = 0; j < taps; ++j) offs[j] = dil * (j - (taps - 1) / 2);
    return itts_conv1d_tc(x, rows, c_in, c_in, w[id], n_total, taps, offs, b[id], c_out, row_out, nullptr, 1.0f,
                          nullptr, 1, nullptr, ACC_NONE, act_out, slope, zero_halo, 0, st);
  }

  int resblock(int s, int j, int m, const void* x, int64_t rows, const int32_t* rm, void* acc, int mode,
               void* act_out, float slope, cudaStream_t st) {
    const int C = kStageC[s], i1 = res_id(s, j, m, 0), i2 = res_id(s, j, m, 1);
    return itts_resblock_tc(x, rows, C, w[i1], w[i2], b[i1], b[i2], kResK[j], kResDil[m], rm, acc, mode, act_out,
                            slope, st);
  }

  int run(int n, const int32_t* Ts_in, const int64_t* d_mplan, int multi_stream, void** x4_out,
          cudaStream_t stream) {
    std::vector<int64_t> Ts(Ts_in, Ts_in + n);
    int64_t maxT = 0;
    for (int64_t T : Ts) {
      if (T < 1) return FAIL_AT(ITTS_EINVAL);
      maxT = std::max(maxT, T);
    }
    size_t rows0, big, rm_total;
    stage_rows(Ts, &rows0, &big, &rm_total);
    const size_t plan_n = (size_t)n * kPlanPerItem;
    int st = grow_all(stream, rows0, big, rm_total, plan_n);
    if (st) return FAIL_AT(st);
    if ((st = host_plan(plan_n))) return FAIL_AT(st);

    Layout lay[kStages + 1];
    lay[0].build(Ts, kMelHalo);
    int64_t mult = 1;
    for (int s = 0; s < kStages; ++s) {
      mult *= kUps[s];
      std::vector<int64_t> r(n);
      for (int i = 0; i < n; ++i) r[i] = Ts[i] * mult;
      lay[s + 1].build(r, kMrfHalo);
    }
    // packed plan: row maps rm0, (rmT_s, rm_s) x 4, then the four halo plans
    int64_t* hp = hplan;
    size_t rm_off[9];
    const int64_t* rm_plan[9];
    int64_t rm_span[9];
    size_t rm_cursor = 0;
    auto add_rowmap = [&](int k, const Layout& in, const Layout& out, int up) {
      int64_t* q = hp;
      for (int i = 0; i < n; ++i, q += 5) {
        q[0] = in.base[i];
        q[1] = in.rows[i];
        q[2] = in.halo;
        q[3] = out.first(i);
        q[4] = up;
      }
      rm_plan[k] = dplan.p + (hp - hplan);
      rm_span[k] = in.max_span;
      rm_off[k] = rm_cursor;
      rm_cursor += (size_t)in.total;
      hp = q;
    };
    add_rowmap(0, lay[0], lay[0], 1);
    for (int s = 0; s < kStages; ++s) {
      add_rowmap(1 + 2 * s, lay[s], lay[s + 1], kUps[s]);
      add_rowmap(2 + 2 * s, lay[s + 1], lay[s + 1], 1);
    }
    const int64_t* z_plan[kStages];
    for (int s = 0; s < kStages; ++s) {
      z_plan[s] = dplan.p + (hp - hplan);
      for (int i = 0; i < n; ++i, hp += 3) {
        hp[0] = lay[s + 1].base[i];
        hp[1] = lay[s + 1].rows[i];
        hp[2] = kMrfHalo;
      }
    }
    cudaError_t e = cudaMemcpyAsync(dplan.p, hplan, (size_t)(hp - hplan) * sizeof(int64_t), cudaMemcpyHostToDevice,
                                    stream);
    if (e != cudaSuccess) return FAIL_AT((int)e);
    if ((e = cudaEventRecord(ev_plan, stream)) != cudaSuccess) return FAIL_AT((int)e);
    plan_pending = true;

    int32_t* rm[9];
    for (int k = 0; k < 9; ++k) rm[k] = rowmaps.p + rm_off[k];
    if ((st = itts_r_rowmaps(9, rm_plan, rm, rm_span, n, stream))) return FAIL_AT(st);   // one launch
    // spliced mel -> conv_pre -> lrelu(0.1)
    if ((e = cudaMemsetAsync(x0.p, 0, (size_t)lay[0].total * 128 * sizeof(uint16_t), stream)) != cudaSuccess)
      return FAIL_AT((int)e);
    if ((st = itts_r_mel_assemble(d_mplan, n, maxT, x0.p, 128, stream))) return FAIL_AT(st);
    if ((st = conv(x0.p, lay[0].total, 128, 0, 512, 7, 1, 512, rm[0], act_in.p, 0.1f, 1, stream))) return FAIL_AT(st);

    const void* act = act_in.p;
    int c_prev = 512;
    for (int s = 0; s < kStages; ++s) {
      const int C = kStageC[s], u = kUps[s];
      const Layout& L = lay[s + 1];
      uint16_t *XA = b16[0].p, *YA = b16[1].p, *TB = b16[2].p, *ACC = b16[3].p, *OA = b16[4 + s % 2].p;
      // transposed conv: each input row -> u output rows, then re-zero the output halos
      if ((st = conv(act, lay[s].total, c_prev, 1 + s, u * C, 3, 1, C, rm[1 + 2 * s], XA, 0.1f, 0, stream)))
        return FAIL_AT(st);
      // (stages 1..3: re-zeroed by the previous stage's MRF merge launch)
      if (s == 0 && (st = itts_r_zero_halo(z_plan[s], n, kMrfHalo, XA, C, stream))) return FAIL_AT(st);
      const int32_t* rms = rm[2 + 2 * s];
      const float slope_out = s < 3 ? 0.1f : 0.01f;
      // MRF: three ResBlock1 branches, each writing its own y; one merge pass averages them.
      // With multi_stream, branches 1 and 2 run on side streams concurrently with branch 0.
      uint16_t* ya[3] = {YA, b16[6].p, b16[8].p};
      uint16_t* tb[3] = {TB, b16[7].p, b16[9].p};
      uint16_t* yo[3] = {ACC, b16[10].p, b16[11].p};
      if (multi_stream && (e = cudaEventRecord(ev_x, stream)) != cudaSuccess) return FAIL_AT((int)e);
      for (int j = 0; j < 3; ++j) {
        cudaStream_t sj = (j == 0 || !multi_stream) ? stream : side[j - 1];
        if (sj != stream && (e = cudaStreamWaitEvent(sj, ev_x, 0)) != cudaSuccess) return FAIL_AT((int)e);
        if ((st = resblock(s, j, 0, XA, L.total, rms, nullptr, ACC_NONE, ya[j], 0.1f, sj))) return FAIL_AT(st);
        if ((st = resblock(s, j, 1, ya[j], L.total, rms, nullptr, ACC_NONE, tb[j], 0.1f, sj))) return FAIL_AT(st);
        if ((st = resblock(s, j, 2, tb[j], L.total, rms, yo[j], ACC_STORE, nullptr, 0.f, sj))) return FAIL_AT(st);
        if (sj != stream && (e = cudaEventRecord(ev_side[j - 1], sj)) != cudaSuccess) return FAIL_AT((int)e);
      }
      if (multi_stream)
        for (int j = 0; j < 2; ++j)
          if ((e = cudaStreamWaitEvent(stream, ev_side[j], 0)) != cudaSuccess) return FAIL_AT((int)e);
      const bool more = s + 1 < kStages;   // the merge also re-zeroes the next stage's XA halos
      if ((st = mrf_combine_zero_halo(yo[0], yo[1], yo[2], L.total * C, slope_out, OA, more ? z_plan[s + 1] : nullptr,
                                      n, kMrfHalo, XA, more ? kStageC[s + 1] : 0, stream)))
        return FAIL_AT(st);
      act = OA;
      c_prev = C;
    }
    *x4_out = const_cast<void*>(act);
    return ITTS_OK;
  }

  void destroy() {
    for (auto s : side)
      if (s) cudaStreamSynchronize(s);
    x0.release();
    act_in.release();
    for (auto& t : b16) t.release();
    rowmaps.release();
    dplan.release();
    if (hplan) cudaFreeHost(hplan);
    for (auto s : side)
      if (s) cudaStreamDestroy(s);
    for (auto ev : {ev_x, ev_side[0], ev_side[1], ev_plan})
      if (ev) cudaEventDestroy(ev);
  }
};

}  // namespace

ITTS_API int itts_r_voc_create(void** handle, const int64_t* weights, int32_t count) {
  if (!handle || !weights || count != kNumWeights) return ITTS_EINVAL;
  Vocoder* v = new Vocoder();
  for (int k = 0; k < kNumWeights / 2; ++k) {
    v->w[k] = reinterpret_cast<const void*>(weights[2 * k]);
    v->b[k] = reinterpret_cast<const float*>(weights[2 * k + 1]);
    if (!v->w[k] || !v->b[k]) {
      delete v;
      return ITTS_EINVAL;
    }
  }
  cudaError_t e = cudaSuccess;
  for (auto& s : v->side)
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (auto* ev : {&v->ev_x, &v->ev_side[0], &v->ev_side[1], &v->ev_plan})
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    v->destroy();
    delete v;
    return (int)e;
  }
  *handle = v;
  return ITTS_OK;
}

ITTS_API int itts_r_voc_reserve(void* handle, int32_t n, int32_t frames, void* stream) {
  if (!handle || n < 1 || frames < 1) return ITTS_EINVAL;
  return static_cast<Vocoder*>(handle)->reserve((cudaStream_t)stream, n, frames);
}

ITTS_API int itts_r_voc_run(void* handle, int32_t n, const int32_t* frames, const int64_t* mel_plan,
                            int32_t multi_stream, void** x4_out, void* stream) {
  if (!handle || n < 1 || !frames || !mel_plan || !x4_out) return ITTS_EINVAL;
  const int st = static_cast<Vocoder*>(handle)->run(n, frames, mel_plan, multi_stream, x4_out, (cudaStream_t)stream);
  if (st && getenv("ITTS_DEBUG")) fprintf(stderr, "itts_r_voc_run: status %d at line %d\n", st, g_fail_line);
  return st;
}

ITTS_API int itts_r_voc_destroy(void* handle) {
  if (!handle) return ITTS_EINVAL;
  Vocoder* v = static_cast<Vocoder*>(handle);
  v->destroy();
  delete v;
  return ITTS_OK;
}
