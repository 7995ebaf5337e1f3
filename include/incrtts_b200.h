/*
 * incrtts_b200 -- C ABI of the B200-native incremental-TTS serving path.
 *
 * The reference (`incrtts`, pure Python) binds its models through the
 * PipelineModules plugin boundary (pkg/src/incrtts/scheduler.py:249-263),
 * four batched Python callables built by build_modules (:266-282).  The
 * drop-in replacement keeps that boundary in Python
 * (paper_2211_13939_b200/modules.py) and reaches the GPU only through the
 * functions below, loaded with ctypes.
 *
 * Conventions
 *   - Every function returns int: 0 on success, a cudaError_t value on a
 *     CUDA failure, or an ITTS_E* code for an argument error detected before
 *     anything is enqueued.  Nothing throws across this boundary.
 *   - All pointers are device pointers unless named host_*; `stream` is a
 *     cudaStream_t passed as void*.  Calls only enqueue work on `stream`.
 *   - Per-item addressing uses a device int64 "plan": one fixed-width row
 *     per batch item holding absolute device addresses and sizes, built by
 *     the host in batch order (= IterationReport.decoder_ids order).  The
 *     library never frees or retains caller memory.
 */
#ifndef INCRTTS_B200_H
#define INCRTTS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ITTS_OK 0
#define ITTS_EINVAL 10001
#define ITTS_EALIGN 10002
#define ITTS_EUNSUPPORTED 10003

int itts_version(void);

/* ---- K1: slot gather / scatter --------------------------------------
 * Replaces the per-item gather `[(item.dec_state, item.enc) for item in
 * dec_items]` and scatter `item.dec_state = out.state`
 * (scheduler.py:452-468, :485) for device-resident state: row i of the
 * contiguous batch buffer <-> the state row at src_ptrs[i] / dst_ptrs[i].
 * row_bytes and the contiguous buffer must be 16-byte aligned (128-bit
 * vector moves). */
int itts_gather_rows(void* dst, const int64_t* src_ptrs, int32_t n_rows, int64_t row_bytes,
                     void* stream);
int itts_scatter_rows(const int64_t* dst_ptrs, const void* src, int32_t n_rows, int64_t row_bytes,
                      void* stream);

/* ---- Tier S: the reference stand-in models in fp64 ------------------- */

/* K2. Replaces encode_batch + init_decoder_state (acoustic.py:222-231,
 * :118-133; scheduler.py:272-274).  tok4 = int32 [4][total_tokens]
 * (phoneme, pw, pph, iph streams of FrontendOutput, items concatenated);
 * plan = int64 [n_items][4] {tok_off, L, feat_ptr (double[L][dim]),
 * state_ptr (double[6*dim + 2L], zeroed)}; scratch = double[2*total*dim]. */
int itts_s_encode(const int32_t* tok4, int64_t total_tokens, const int64_t* plan, int32_t n_items,
                  int64_t max_len, int32_t dim, double* scratch, void* stream);

/* K3. Replaces decode_chunk_batch (acoustic.py:234-238, :204-219).
 * plan = int64 [n_items][6] {feat_ptr, L, src_state_ptr, dst_state_ptr,
 * steps, mel_ptr (double[steps][dim])}.  `steps` = min(chunk_frames,
 * target - emitted) is the reference's counter stop (acoustic.py:174-175,
 * :213-218), decided on the host.  src is read, dst written (value
 * semantics: the old state stays valid). */
int itts_s_decode_chunk(const int64_t* plan, int32_t n_items, int32_t dim, double penalty,
                        void* stream);

/* K4. Replaces vocode_batch (vocoder.py:139-143, :92-136) with the
 * stand-in generator (vocoder.py:52-60).  plan = int64 [n_items][7]
 * {mel_ptr, m, flags (1 = has tail, 2 = is_last), src_vs_ptr, dst_vs_ptr,
 * out_off, 0}; vocoder state = double[overlap*dim + overlap*hop]
 * (mel tail, held samples).  fade = double[2][overlap*hop] (sin, cos
 * ramps); audio = packed output, item i at audio[out_off]. */
int itts_s_vocode_chunk(const int64_t* plan, int32_t n_items, int32_t dim, int32_t overlap_frames,
                        int32_t hop, int64_t max_samples, const double* fade, double* audio,
                        void* stream);

/* ---- Tier R: Tacotron2 + HiFi-GAN V1 ---------------------------------- */

/* K7 core: one 1-D convolution layer as a persistent tcgen05 implicit GEMM
 * (bf16 operands, fp32 TMEM accumulation, TMA-fed).  Replaces the per-layer
 * work of the vocoder G inside vocode_chunk (vocoder.py:107/:124 `generate`;
 * HiFi-GAN V1 conv_pre / ConvTranspose / MRF convs) and
 * serves as the tensor-core GEMM of the encoder and the decoder gates.
 *   x      bf16 [rows][c_in] channels-last (row stride x_ld >= c_in), items
 *          packed with zero halos
 *   w      bf16 [n_taps][n_total][c_in]; host_tap_off[n_taps] row offsets
 *   out    n_total = phases * c_out columns; row_out[r] = output row of input
 *          row r (phase p goes to row_out[r] + p), -1 for halo rows
 *   epilogue: v = acc + bias (+ inv_lrelu(res_in, res_slope));
 *          f32_out = v (raw fp32; with ksplit > 1 each K slice z writes its
 *          partial at f32_out + z*rows*c_out and only slice 0 adds the bias);
 *          acc_mode 1 store / 2 add / 3 finalize v = (acc + v) / 3 on the bf16
 *          MRF accumulator; act_out = bf16(lrelu(v, slope)); zero_halo writes
 *          zeros into act_out halo rows.  0 <= slope <= 1, 0 < res_slope <= 1.
 * c_in and c_out must be multiples of 32; bn = N tile (32/64/128/256) or 0. */
int itts_conv1d_tc(const void* x, int64_t rows, int32_t c_in, int64_t x_ld, const void* w,
                   int32_t n_total, int32_t n_taps, const int32_t* host_tap_off, const float* bias,
                   int32_t c_out, const int32_t* row_out, const void* res_in, float res_slope,
                   float* f32_out, int32_t ksplit, void* acc, int32_t acc_mode, void* act_out,
                   float slope, int32_t zero_halo, int32_t bn, void* stream);

/* K7 fused HiFi-GAN ResBlock1 layer (one MRF branch step; replaces, with the
 * vocoder_batch stand-in src/vocoder.py:52-60, the pair of itts_conv1d_tc calls
 * c1 -> c2 of HiFi-GAN V1).  x = bf16 [rows][c] holding lrelu(x, 0.1), items
 * packed with zero halos >= 25 rows; w1/w2 = bf16 [taps][c][c] (K-major);
 * b1/b2 = fp32 [c]; row_out[r] < 0 marks halo rows.  y = x + c2(lrelu(c1(x)));
 * acc_mode 0: act_out = lrelu(y, slope); 1: acc = y; 2: acc += y;
 * 3: act_out = lrelu((acc + y) / 3, slope).  Exactly one output: act_out is given
 * for modes 0 / 3 and NULL for modes 1 / 2.  Halo rows of the output are written as
 * zeros.  c in {32, 64, 128, 256}, taps odd <= 11, dil <= 5, 0 <= slope <= 1.  act_out /
 * acc must not alias x. */
int itts_resblock_tc(const void* x, int64_t rows, int32_t c, const void* w1, const void* w2, const float* b1,
                     const float* b2, int32_t taps, int32_t dil, const int32_t* row_out, void* acc,
                     int32_t acc_mode, void* act_out, float slope, void* stream);
/* Profiling aid: per-CTA barrier-wait cycle counters of later itts_resblock_tc launches
 * ([grid][16] uint64 device buffer; NULL turns it off). */
int itts_resblock_debug_trace(void* buf);

/* K6 decoder-step chain (replaces decode_chunk_batch, acoustic.py:234-238,
 * with the Tacotron2 decoder, paper Eq. 2).  `state` = fp32 [B][4944] rows
 * gathered by itts_gather_rows: [p 256 | ctx 512 | att_h 1024 | dec_h 1024 |
 * att_c 1024 | dec_c 1024 | last_frame 80]; `xb` = bf16 [B][2816] operand
 * mirror of the first 2816 floats.  plan = int64 [B][8] {memory_ptr,
 * processed_memory_ptr, L, w_src_ptr (W|W_acc), w_dst_ptr, steps, mel_ptr,
 * gate_ptr}; items with step >= steps are left untouched (stop divergence).
 * The gate GEMMs between these calls are itts_conv1d_tc with one tap. */
/* K6P: the whole decoder chunk (nsteps steps) as one persistent, grid-synchronised kernel
 * (dec_persist.cu).  work = fp32 [B][4944] gathered state rows, plan as above; xb = bf16
 * scratch operand mirror, ceil(B/128) x 76 x 128 x 64 (UMMA-swizzled tiles); Wa / Wd = bf16
 * gate weights as [32 groups][K/64 chunks][128 rows = 32 units x 4 gates][64] swizzled tiles
 * (K = 1792 / 2560), ba / bd fp32 [32][128] in the same row order; Gp = fp32
 * [4][32][ceil16(B)][128] K-split partials;
 * W0T [80][256], W1T [256][256], WqT [1024][128], v [128], WpT [1536][81], bp [81] fp32;
 * WlocD [2][31][128] = the location conv composed with the location dense layer
 * (sum_f Wloc[f][c][k] WdT[f][a]).  Scratch: H1 [B][256], Q [32][B][128], P [33][B][81],
 * U [B][u_ld >= max L], AP [B][256][514], bar = 64 + B x u32 (zeroed by the call).  B <= 512, texts <= 8192 phonemes.
 * Split-bf16 parity mode: Wa_lo / Wd_lo = the low bf16 parts (W - bf16(W)) in the same layout;
 * the gate products are then Wh.Xh + Wh.Xl + Wl.Xh with fp32 accumulation (about 16 significant
 * bits per operand) and xb must hold 2 x the mirror (high parts, then low parts).  Both null: plain
 * bf16 products, or, with split_x != 0 (weights exactly representable in bf16, e.g. a bf16
 * checkpoint), Wh.Xh + Wh.Xl -- the same fp32-level products at the bf16 weight bytes. */
int itts_r_decode_persistent(int32_t B, int32_t nsteps, const int64_t* plan, float* work, void* xb,
                             const float* W0T, const float* W1T, const void* Wa, const float* ba,
                             const void* Wd, const float* bd, const float* WqT, const float* WlocD,
                             const float* v, const float* WpT, const float* bp,
                             float* Gp, float* H1, float* Q, float* P, float* U, int64_t u_ld, float* AP,
                             unsigned* bar, const void* Wa_lo, const void* Wd_lo, int32_t split_x,
                             void* stream);
/* Profiling aid: per-phase wall time of later persistent-decoder launches ([8] u64 ns). */
int itts_r_decode_debug_trace(void* buf);
int itts_r_dec_prepare(const float* state, void* xb, int32_t B, void* stream);
int itts_r_prenet(float* state, void* xb, const float* W0T, const float* W1T, const int64_t* plan,
                  float* H1, int32_t B, int32_t step, void* stream);
int itts_r_lstm_cell(const float* gates, int32_t nsplit, const float* bias, float* state, void* xb,
                     int32_t h_off, int32_t c_off, const int64_t* plan, int32_t B, int32_t step,
                     void* stream);
/* query partials: Q = fp32 [8][B][128] K-slices of Wq . att_h, summed (fixed order) by
 * itts_r_attention; proj partials = fp32 [8][B][81] scratch. */
int itts_r_query(const float* state, const float* WqT, float* Q, int32_t B, void* stream);
int itts_r_attention(float* state, void* xb, const int64_t* plan, int32_t B, int32_t max_len,
                     const float* Q, const float* Wloc, const float* WdT, const float* v, int32_t step,
                     void* stream);
int itts_r_proj(float* state, const int64_t* plan, int32_t B, const float* WpT, const float* bp,
                float* partials, int32_t step, void* stream);

/* K5 encoder (replaces encode_batch + init_decoder_state, acoustic.py:222-231,
 * :118-133, with the Tacotron2 encoder, paper Eq. 1).  plan = int64 [n][6]
 * {tok_off, L, first_row, memory_ptr (fp32 [L][512]), pm_ptr (fp32 [L][128]),
 * 0}; X = bf16 [rows][512] zero-haloed conv input; PRE = fp32 [rows][2048]
 * BiLSTM input projections (both directions, biases folded). */
int itts_r_enc_embed(const int32_t* tok4, int64_t total, const int64_t* plan, int32_t n,
                     int64_t max_len, const float* Eph, const float* Epw, const float* Epph,
                     const float* Eiph, void* X, void* stream);
int itts_r_bilstm(const float* PRE, const int64_t* plan, int32_t n, const float* WhhT, void* stream);
/* The whole encoder launch sequence above (embedding, 3 convs, input projection, BiLSTM,
 * processed memory, zeroed decoder-state rows) issued from C++ after one H2D copy: pack =
 * int32 tokens [4][total] (padded to 8 bytes), plan [n][6], row-map plan [n][5], state spans
 * [n][2] {ptr, floats}; weights = Eph, Epw, Epph, Eiph, (conv w, conv b) x 3, Wih, b_ih, WhhT, WmT;
 * xa / xb bf16 [rows][512], pre fp32 [rows][2048], rowmap int32 [rows] work buffers. */
int itts_r_encode(const void* pack, int64_t total, int32_t n, int64_t max_len, int64_t rows, int64_t max_span,
                  const int64_t* weights, int32_t conv_taps, void* xa, void* xb, float* pre, int32_t* rowmap,
                  void* stream);
/* The same encoder in the split-bf16 parity mode: every tensor-core product on [hi | lo | hi]
 * bf16 operands against [Wh | Wh | Wl] weights (Wh.Xh + Wh.Xl + Wl.Xh, fp32 accumulation), fp32
 * activations between layers.  weights3 = the itts_r_encode table with entries 4, 6, 8 (convs,
 * [5][512][1536]) and 10 (input projection, [1][2048][1536]) replaced; x3 bf16 [rows][1536],
 * f32 fp32 [rows][512] scratch.  Replaces the same reference functions as itts_r_encode.
 * parts = 3, or 2 when the weights are exact in bf16: entries [Wh | Wh] ([.][.][1024]) against the
 * first two operand thirds [hi | lo] (Wh.Xh + Wh.Xl). */
int itts_r_encode_split(const void* pack, int64_t total, int32_t n, int64_t max_len, int64_t rows,
                        int64_t max_span, const int64_t* weights3, int32_t conv_taps, void* x3, float* f32,
                        float* pre, int32_t* rowmap, int32_t parts, void* stream);
int itts_r_pmem(const int64_t* plan, int32_t n, int64_t max_len, const float* WmT, void* stream);
/* The same BiLSTM on the tensor cores (csrc/bilstm_tc.cu): one 8-CTA cluster per (direction,
 * group of <= 32 items), gates = W_hh . h as one tcgen05 MMA chain per step with h split into bf16
 * hi + lo parts (fp32-level for bf16-exact W_hh).  Wt = bf16 [2 dir][8 rank][4][128][64]: rank r's
 * 128 gate rows (unit 32 r + u, gate g at row 4 u + g) x 256 inputs as 128B-swizzled K-major tiles.
 * The encoder weight tables of itts_r_encode / itts_r_encode_split take it as entry 14 (0: SIMT). */
int itts_r_bilstm_tc(const float* PRE, const int64_t* plan, int32_t n, const void* Wt, void* stream);

/* K7 helpers around the HiFi-GAN conv stack (replaces vocode_batch,
 * vocoder.py:92-143): spliced-mel assembly, per-stage row maps, halo
 * re-zeroing, and conv_post + tanh fused with the Eq.-3 cross-fade /
 * hold-back epilogue writing the packed fp32 audio. */
int itts_r_mel_assemble(const int64_t* plan, int32_t n, int64_t max_rows, void* X0, int32_t ld,
                        void* stream);
int itts_r_rowmap(const int64_t* plan, int32_t n, int64_t max_span, int32_t* row_out, void* stream);
int itts_r_zero_halo(const int64_t* plan, int32_t n, int64_t max_halo, void* X, int32_t C, void* stream);
/* f3: chunk-local Tacotron2 PostNet over one decoder call's chunks (mel + PostNet(mel), 5 conv
 * k5 layers on the tensor cores, tanh after the first four, zero padding at chunk edges).
 * pack = mel-assembly plan [n][5] {0, mel_ptr, m, 0, first_row}, row-map plan [n][5], residual
 * plan [n][4] {mel_ptr, out_ptr, m, first_row}; weights = (w bf16 [5][c_out][c_in], b fp32) x 5,
 * the 80-wide ends padded to 96; x0 bf16 [rows][96], ya / yb bf16 [rows][512], post fp32
 * [rows][96], rowmap int32 [rows] work buffers. */
int itts_r_postnet(const int64_t* pack, int32_t n, int64_t max_m, int64_t rows, int64_t max_span,
                   const int64_t* weights, void* x0, void* ya, void* yb, float* post, int32_t* rowmap,
                   void* stream);
/* f4: BERT prosodic-structure frontend (12 layers, hidden 768, 12 heads, FFN 3072, post-LN,
 * GELU; three 2-way heads pw / pph / iph) over a pooled batch of texts packed without padding
 * (csrc/bert.cu).  ids / pos int32 [rows]; plan int64 [n][2] {first row, length <= 256};
 * weights = 150 device pointers (see bert.cu); row_map int32 [rows] = identity; work buffers
 * xf fp32 / xb bf16 [rows][768], qkv bf16 [rows][2304], att bf16 [rows][768], y fp32
 * [rows][768], h bf16 [rows][3072]; outputs logits fp32 [rows][6], tokens int32 [rows][3]. */
int itts_bert_prosody(const int32_t* ids, const int32_t* pos, const int64_t* plan, int32_t n, int64_t rows,
                      int32_t max_len, const int64_t* weights, const int32_t* row_map, float* xf, void* xb,
                      void* qkv, void* att, float* y, void* h, float* logits, int32_t* tokens, void* stream);
/* MRF merge of HiFi-GAN V1 (the xs / num_kernels average of the three ResBlock1 branches):
 * out = bf16(lrelu((y0 + y1 + y2) / 3, slope)) over n bf16 elements (n % 8 == 0). */
int itts_r_mrf_combine(const void* y0, const void* y1, const void* y2, int64_t n, float slope, void* out,
                       void* stream);
/* pcm16 (optional, may be NULL): int16 [total] 16-bit PCM of `audio` as the reference
 * pcm16_encode (src/vocoder.py:146-149), produced in the same pass.
 * nonfinite (optional): int32 [n], zeroed here, item i's count of non-finite emitted samples
 * (the finite-audio guard of AudioChunk, domain.py:_frozen_array, without a host scan). */
/* f1 wire format: per chunk i, base64 (RFC 4648, '=' padded) of the little-endian bytes of
 * pcm16[plan[3i] .. plan[3i] + plan[3i+1]) into out + plan[3i+2] (4 * ceil(2 count / 3) chars):
 * the reference server's encode_samples (src/server.py:78-79) on device. */
int itts_r_pcm16_b64(const void* pcm16, const int64_t* plan, int32_t n, int64_t max_samples, void* out,
                     void* stream);
int itts_r_post_splice(const void* X4, const int64_t* plan, int32_t n, int64_t max_g, const float* wpost,
                       float bpost, const float* fade, int32_t overlap_frames, int32_t overlap_samples,
                       float* audio, void* pcm16, int32_t* nonfinite, void* stream);

/* K7 native launch sequence: the whole HiFi-GAN V1 stack of one pooled vocoder
 * call (replaces the per-layer host loop over vocode_batch's conv stack,
 * src/vocoder.py:92-143) issued from C++ after a single H2D copy of a packed
 * plan.  weights = 154 device pointers, (w, bias) pairs in the order conv_pre,
 * ups[0..3], then res[stage][branch][layer][c1, c2] in the layouts
 * itts_conv1d_tc / itts_resblock_tc take.  run: frames = host int32 [n] spliced
 * frame counts T_i; mel_plan = the device plan of itts_r_mel_assemble;
 * multi_stream = 1 runs the three MRF branches of a stage on three streams
 * (same arithmetic); *x4_out receives the stage-4 activations (bf16
 * [rows][32], lrelu 0.01 applied) for itts_r_post_splice, valid until the next
 * run on the handle.  Work buffers are owned by the handle (grow-only;
 * itts_r_voc_reserve pre-sizes them so serving never allocates). */
int itts_r_voc_create(void** handle, const int64_t* weights, int32_t count);
int itts_r_voc_reserve(void* handle, int32_t n, int32_t frames, void* stream);
int itts_r_voc_run(void* handle, int32_t n, const int32_t* frames, const int64_t* mel_plan,
                   int32_t multi_stream, void** x4_out, void* stream);
int itts_r_voc_destroy(void* handle);

#ifdef __cplusplus
}
#endif

#endif /* INCRTTS_B200_H */
