"""Tier R GPU modules: random-init Tacotron2 + HiFi-GAN V1 behind PipelineModules.

Same three callables and the same handle/value semantics as Tier S
(``tier_s.py``), with the reference's stand-in arithmetic replaced by the
real networks (paper Eq. 1-3):

encoder_batch   K5: embedding sum -> 3 x tcgen05 conv(k5)+ReLU -> tcgen05
                BiLSTM input GEMM -> cluster BiLSTM recurrence -> memory,
                processed memory (FFMA).
decoder_batch   K1 gather of the fixed state rows -> K6 x steps: prenet,
                tcgen05 attention-LSTM gate GEMM (bf16, swap-free: batch rows
                x 4096 gates), cell, location-sensitive attention, tcgen05
                decoder-LSTM gate GEMM, cell, mel/gate projection -> K1
                scatter into the request's next state buffer.
vocoder_batch   K7: [mel_tail; mel] -> conv_pre -> 4 x (transposed conv as a
                3-tap phase GEMM, 3 MRF resblocks = 18 convs with fused
                bias / residual / MRF-average / leaky-ReLU epilogues) ->
                conv_post + tanh + cross-fade / hold-back (Eq. 3).

Stop is the reference's frame counter (``acoustic.py:174-175``): chunk
lengths, stop steps and sample offsets are decided on the host exactly as
in Tier S; the gate logit is computed and returned but not used.
"""

from __future__ import annotations

import ctypes
import functools
import os
import sys
import weakref

import numpy as np
import torch

from . import _native
from . import tc
from . import weights as W
from .arena import RaggedArena
from .audio import cached_curve
from .domain import AudioChunk, PipelineConfig, validate_config
from .handles import (DecodeChunkResult, DeviceDecoderState, DeviceEncodedFeatures, DeviceMelChunk,
                      DeviceRequest, DeviceVocoderState)

# decoder state row layout (floats) -- must match csrc/tier_r.cu
P_OFF, CTX_OFF, ATTH_OFF, DECH_OFF, ATTC_OFF, DECC_OFF, LAST_OFF, ROW = 0, 256, 768, 1792, 2816, 3840, 4864, 4944
XB_ROW = 2816
ENC_HALO = 2        # conv k5
ENC_TAPS = 5
POST_HALO = 2       # PostNet conv k5 (chunk-local zero padding)
POST_CP = 96        # PostNet mel channels padded for the tensor-core conv
MEL_HALO = 3        # conv_pre k7
MRF_HALO = 25       # k11 dilation 5
UPS = (8, 8, 2, 2)
STAGE_C = (256, 128, 64, 32)
DEC_KSPLIT = 4      # K-split of the decoder gate GEMMs (partials summed in fixed order by the cell kernel)
GRAPH_MAX_L = 8192  # attention smem is sized for this in captured graphs; longer texts run eagerly
HID = 1024
XB2 = 4864          # persistent decoder's bf16 mirror row (two banks of att_h / dec_h)
PERSIST_MAX_L = 8192  # 256 attention chunks of <= 32 positions
PERSIST_MAX_B = 512   # kernel limit (2 MMA N tiles, plan cache); larger pools decode in slices of <= 512
DEC_BAR_WORDS = 64 + PERSIST_MAX_B   # persistent-decoder counters: barrier / groups / contexts, then one per item


def _hifigan_macs_per_frame() -> int:
    """Algorithmic MACs of HiFi-GAN V1 per input mel frame (307,052,544)."""
    macs, rate, ch = W.N_MEL * W.HG_CH0 * 7, 1, W.HG_CH0
    for u, k in zip(W.HG_UP_RATES, W.HG_UP_KERNELS):
        macs += ch * (ch // 2) * k * rate      # transposed conv: every input sample hits k outputs
        rate, ch = rate * u, ch // 2
        macs += rate * 6 * ch * ch * sum(W.HG_RES_KERNELS)
    return macs + rate * ch * 7


HIFIGAN_MACS_PER_FRAME = _hifigan_macs_per_frame()
# Decoder-step weight bytes as stored here (bf16 gate GEMMs, fp32 elsewhere).
_DEC_GEMV_BYTES = (80 * 256 + 256 * 256 + 1024 * 128 + 32 * 62 + 32 * 128 + 128 + 1536 * 81 + 81) * 4
DEC_WEIGHT_BYTES = (4096 * 1792 + 4096 * 2560) * 2 + _DEC_GEMV_BYTES
# parity mode: the gate weights carry fp32-level values (high + low bf16 parts = 4 bytes per weight)
DEC_WEIGHT_BYTES_SPLIT = (4096 * 1792 + 4096 * 2560) * 4 + _DEC_GEMV_BYTES


def _on_device(fn):
    """Run a module entry point with the engine's device current (the calling thread may be on
    another device, e.g. a router worker or a test on cuda:1)."""
    @functools.wraps(fn)
    def wrapper(self, *args, **kw):
        with torch.cuda.device(self.device):
            return fn(self, *args, **kw)
    return wrapper


def _h2d(arr: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(arr)).pin_memory().to(device, non_blocking=True)


def _swizzle_tiles(w: torch.Tensor, rows: int = 32) -> torch.Tensor:
    """[N][K] bf16 (row groups of `rows`) -> [N/rows][K/64][rows][64] with the UMMA 128B swizzle
    (16-byte group j of row r stored at j ^ (r % 8)): each (group, 64-column chunk) stage of the
    persistent decoder's gate GEMM is one contiguous bulk copy."""
    n, k = w.shape
    t = w.reshape(n // rows, rows, k // 64, 8, 8).permute(0, 2, 1, 3, 4).contiguous()   # [grp][chunk][row][g][e]
    r = torch.arange(rows, device=w.device)[:, None]
    j = torch.arange(8, device=w.device)[None, :]
    src_grp = (j ^ (r % 8))          # stored group j holds logical group j ^ (r % 8)
    out = torch.gather(t, 3, src_grp[None, None, :, :, None].expand(t.shape))
    return out.reshape(n // rows, k // 64, rows, 64).contiguous()


class _Layout:
    """Packed rows of one activation stage: item i at [base_i, base_i + 2*halo + rows_i)."""

    def __init__(self, rows: list[int], halo: int):
        self.rows, self.halo = rows, halo
        spans = np.array(rows, dtype=np.int64) + 2 * halo
        self.base = np.concatenate([[0], np.cumsum(spans)[:-1]]).astype(np.int64)
        self.total = int(spans.sum())
        self.first = self.base + halo   # first valid row per item


class _Mark:
    __slots__ = ("engine", "kind", "units", "e0")

    def __init__(self, engine, kind, units):
        self.engine, self.kind, self.units = engine, kind, units

    def __enter__(self):
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e0.record(self.engine.stream)
        return self

    def __exit__(self, *exc):
        if exc[0] is None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(self.engine.stream)
            units = self.units() if callable(self.units) else self.units
            self.engine.timers.append((self.kind, self.e0, e1, units))
        return False


class _NoMark:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_NO_MARK = _NoMark()


class TierREngine:
    dtype = torch.float32

    def __init__(self, cfg: PipelineConfig, device=None, seed: int = 0, weights: dict | None = None,
                 postnet: bool = False, postnet_weights: dict | None = None):
        self.cfg = validate_config(cfg)
        if cfg.hop_samples != 256:
            raise ValueError("HiFi-GAN V1 upsamples by 256: hop_samples must be 256")
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type != "cuda":
            raise RuntimeError("Tier-R GPU modules need a CUDA device (no CPU fallback)")
        _native.lib()
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        # everything below -- torch allocations, the native vocoder's streams / events, its
        # cudaMalloc'd work buffers -- lives on self.device, whatever the calling thread's device
        with torch.cuda.device(self.device):
            self._init_on_device(seed, weights, postnet, postnet_weights)

    def _init_on_device(self, seed, weights, postnet, postnet_weights) -> None:
        cfg = self.cfg
        self.stream = torch.cuda.Stream(self.device)
        w = weights if weights is not None else W.tier_r_weights(seed)
        with torch.cuda.stream(self.stream):
            self._prepare_weights(w)
            # 2 GB up front: growing (re-allocate + copy) inside a serving window stalls an iteration
            self.arena = RaggedArena(self.dtype, self.device, 1 << 29, self.stream)
            curve = cached_curve(cfg.overlap_samples)
            self.fade = torch.from_numpy(np.concatenate([curve.fade_in, curve.fade_out])).float().to(self.device)
            self.iota = torch.arange(1 << 16, dtype=torch.int32, device=self.device)
        self.stream.synchronize()
        self.launches = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.timers: list | None = None  # set to [] to record (kind, ev0, ev1, units) per module call
        self.use_graphs = True           # CUDA-graph the 32-step decoder chunk per (batch, L) bucket
        self.fused_mrf = True            # one fused c1->c2 kernel per ResBlock1 layer (resblock_tc.cu)
        self.persistent_decoder = True   # whole decoder chunk in one grid-synchronised kernel (dec_persist.cu)
        # decoder gate products: "parity" = split bf16 (Wh.Xh + Wh.Xl + Wl.Xh, fp32 accumulate: fp32-level
        # mel, north_star's parity mode); "bf16" = single bf16 products (reported separately)
        self.precision = "parity"
        self.pcm16 = False               # also produce 16-bit PCM on device in the splice pass (f1)
        self.wire_b64 = False            # and its base64 wire text (server.encode_samples) on device (f1)
        self.mrf_streams = True          # run the 3 MRF branches of a stage on 3 streams (fused path)
        self.native_vocoder = True       # issue the fused HiFi-GAN stack from C++ (voc_run.cu)
        self.native_encoder = True       # issue the encoder launch sequence from C++ (itts_r_encode)
        # host work the scheduler loop runs while vocoder_batch waits on the GPU: idle_hook(done)
        # with done() -> True once the awaited work finished (set by SchedulerLoop)
        self.idle_hook = None
        self.diagnose = True             # on a non-finite chunk, record which inputs were already bad
        self.plan_staging = True         # decoder graph plans: rewrite only the rows that changed
        self.failures: list = []
        # diagnostics: keep the last decoder call's inputs / outputs so a non-finite chunk can be
        # traced to a transient (re-run differs) or an input fault (re-run reproduces it)
        self.keep_last_decoder = False
        self._last_dec = None
        self.poison_scratch = False          # debug: NaN-fill decoder scratch (eager path; True or a set of buffer names)
        self.bisect_dir: str | None = None   # with keep_last_decoder: shrink + dump failing decoder batches here
        self.speculate = True            # precompute the next decoder call's item fields during V waits
        self._spec_src = None            # continuing (state, features) of the last decoder call
        self._spec = None                # their precomputed plan fields (see _speculate_next_decoder)
        # pools of at least spec_launch_min continuing items launch their next decoder chunk during
        # the vocoder wait (0: off); small pools only precompute plan fields (a separate launch
        # for new items would cost their first chunk ~1.4 ms)
        self.spec_launch_min = 128
        # frontend outputs prefetched during a vocoder wait are encoded right then (pre_encode)
        self.pre_encode_enabled = True
        self._pre_enc: dict = {}
        self.pre_enc_hits = 0
        self._spec_out = None
        self._last_full_decode = True
        self.spec_hits = 0
        # f3: chunk-local Tacotron2 PostNet on the decoder's mel output (off: the reference's no-op)
        self.postnet = bool(postnet or postnet_weights is not None)
        if self.postnet:
            self._prepare_postnet(postnet_weights if postnet_weights is not None else W.postnet_weights(seed))
        enc_w = [*self.E]
        for wt, _, bias in self.enc_conv:
            enc_w += [wt, bias]
        enc_w += [self.enc_ih[0], self.enc_ih[2], self.enc_whhT, self.WmT]
        enc_p = [t.data_ptr() for t in enc_w] + [0 if self.enc_whh_tc is None else self.enc_whh_tc.data_ptr()]
        self._enc_ptrs = (ctypes.c_int64 * len(enc_p))(*enc_p)
        # parity mode: conv / input-projection weights as [Wh | Wh | Wl] along C_in (itts_r_encode_split)
        enc_p3 = list(enc_p)
        for i, t in enumerate(self._enc_split_w):
            enc_p3[4 + 2 * i] = t.data_ptr()
        self._enc_ptrs3 = (ctypes.c_int64 * len(enc_p3))(*enc_p3)
        self._voc = self._create_native_vocoder()
        self._side = [torch.cuda.Stream(self.device) for _ in range(2)]
        self._ev = [torch.cuda.Event() for _ in range(3)]
        self._dec_buckets: dict = {}
        self._pool: dict = {}
        self._pin_out = torch.empty(1 << 22, dtype=torch.float32, pin_memory=True)  # audio D2H (fallback)
        self._nf_pin = torch.empty(1024, dtype=torch.int32, pin_memory=True)     # per-chunk non-finite counts
        self._out_ring: list = [None] * 6    # pinned (tensor, ndarray) audio slots; chunks view them
        self._out_next = 0
        self.host_finite_check = False      # also scan the samples on the host (the device count is the guard)
        self._graph_warm = False

    PRECISIONS = ("parity", "bf16")

    def set_precision(self, mode: str) -> None:
        """Decoder gate-product arithmetic for later calls (drops captured decoder graphs)."""
        if mode not in self.PRECISIONS:
            raise ValueError(f"precision must be one of {self.PRECISIONS}")
        if mode != self.precision:
            self.stream.synchronize()
            self._dec_buckets = {}
            self._graph_warm = False
        self.precision = mode

    def precision_label(self) -> str:
        if self.precision == "parity":
            prod = ("bf16-grid weights x split-bf16 operands (x2)" if self.w_exact_bf16
                    else "split-bf16 (x3)")
            return (f"fp32-level decoder: {prod} tcgen05 gate products, fp32 accumulate / attention / "
                    "cells; bf16-operand encoder convs and HiFi-GAN (fp32 accumulate)")
        return "bf16 decoder gate products; bf16-operand encoder convs and HiFi-GAN (fp32 accumulate)"

    def _mark(self, kind: str, units):
        """Context manager recording CUDA events on the engine stream around a region (timers on);
        `units` may be a callable, evaluated only then."""
        return _Mark(self, kind, units) if self.timers is not None else _NO_MARK

    def _up(self, arr: np.ndarray) -> torch.Tensor:
        self.h2d_bytes += arr.nbytes
        return _h2d(arr, self.device)

    # ------------------------------------------------------------ weights
    def _prepare_weights(self, w: dict) -> None:
        d = self.device
        f32 = lambda t: t.detach().float().contiguous().to(d)
        self.E = [f32(w[f"emb.{k}"]) for k in ("phoneme", "pw", "pph", "iph")]
        self.enc_conv = []
        for i in range(3):
            wt, offs = tc.conv_weights(f32(w[f"enc.conv{i}.w"]))
            self.enc_conv.append((wt, offs, f32(w[f"enc.conv{i}.b"])))
        wih = torch.cat([w["enc.lstm_fwd.w_ih"], w["enc.lstm_bwd.w_ih"]], 0)          # [2048][512]
        self.enc_ih = (wih.to(d).to(torch.bfloat16)[None].contiguous(), [0],
                       f32(torch.cat([w["enc.lstm_fwd.b_ih"] + w["enc.lstm_fwd.b_hh"],
                                      w["enc.lstm_bwd.b_ih"] + w["enc.lstm_bwd.b_hh"]])))
        self.enc_whhT = f32(torch.stack([w["enc.lstm_fwd.w_hh"].T, w["enc.lstm_bwd.w_hh"].T]))  # [2][256][1024]
        # tensor-core BiLSTM (bilstm_tc.cu), OPT-IN (ITTS_BILSTM_TC=1): pooled encoder batches of >= 96
        # items then run the recurrence as tcgen05 MMAs (32 items per cluster; 2.05 vs 3.3 ms at 128
        # ragged items) but ~2x slower per step below that, and its arithmetic differs from the SIMT
        # recurrence, so a request's encoder bits would depend on the batch crossing the threshold
        # (batch transparency).  Needs bf16-exact W_hh; rows regrouped per direction as [rank r][unit u]
        # [gate g] (row g*256 + 32r + u), 128B-swizzled 128-row tiles.
        self.enc_whh_tc = None
        whh = [w["enc.lstm_fwd.w_hh"], w["enc.lstm_bwd.w_hh"]]
        if (os.environ.get("ITTS_BILSTM_TC") == "1"
                and all(bool((t.to(torch.bfloat16).float() == t).all()) for t in whh)):
            rows = (torch.arange(4)[None, None, :] * 256 + torch.arange(8)[:, None, None] * 32
                    + torch.arange(32)[None, :, None]).reshape(-1)
            self.enc_whh_tc = torch.stack([_swizzle_tiles(t.to(d).float()[rows.to(d)].to(torch.bfloat16), 128)
                                           for t in whh]).contiguous()

        # fp32 [k][C_out][C_in] -> bf16 [k][C_out][3 C_in] = [Wh | Wh | Wl], or [Wh | Wh] when every
        # encoder weight is exact in bf16 (Wl = 0: two products instead of three)
        enc_src = [f32(w[f"enc.conv{i}.w"]).permute(2, 0, 1) for i in range(3)] + [wih.to(d).float()[None]]
        self.enc_parts = 2 if all(bool((t.to(torch.bfloat16).float() == t).all()) for t in enc_src) else 3

        def split(t):
            hi = t.to(torch.bfloat16)
            lo = (t - hi.float()).to(torch.bfloat16)
            return torch.cat([hi, hi] + ([lo] if self.enc_parts == 3 else []), 2).contiguous()
        self._enc_split_w = [split(t) for t in enc_src]
        self.WmT = f32(w["att.memory_layer"].T)                                          # [512][128]
        # decoder
        self.W0T, self.W1T = f32(w["prenet.0"].T), f32(w["prenet.1"].T)
        wa = torch.cat([w["att_rnn.w_ih"], w["att_rnn.w_hh"]], 1)                       # [p|ctx|att_h]
        zeros = torch.zeros(4096, device=d)   # gate bias is added (once) by the cell kernel
        self.att_bias = f32(w["att_rnn.b_ih"] + w["att_rnn.b_hh"])
        self.att_gemm = (wa.to(d).to(torch.bfloat16)[None].contiguous(), [0], zeros)
        wih = w["dec_rnn.w_ih"]                                                          # cols [att_h | ctx]
        wd = torch.cat([wih[:, 1024:], wih[:, :1024], w["dec_rnn.w_hh"]], 1)             # [ctx|att_h|dec_h]
        self.dec_bias = f32(w["dec_rnn.b_ih"] + w["dec_rnn.b_hh"])
        self.dec_gemm = (wd.to(d).to(torch.bfloat16)[None].contiguous(), [0], zeros)
        # persistent decoder: gate rows regrouped per 32-unit group g as [unit u][gate q]
        # (row 128g + 4u + q <- original row q*1024 + 32g + u), then UMMA-swizzled 64-column tiles
        perm = lambda t: t.reshape(4, HID // 32, 32, -1).permute(1, 2, 0, 3).reshape(4 * HID, -1)
        # split-bf16 parity mode: W = Wh + Wl with Wh = bf16(W), Wl = bf16(W - Wh) (same layout)
        split = lambda t: (t.to(torch.bfloat16), (t - t.to(torch.bfloat16).float()).to(torch.bfloat16))
        wa_h, wa_l = split(perm(wa.to(d).float()))
        wd_h, wd_l = split(perm(wd.to(d).float()))
        # weights already on the bf16 grid (a bf16 checkpoint, or tier_r_weights' default): Wl = 0,
        # and the parity products reduce to Wh.Xh + Wh.Xl at the bf16 weight bytes
        self.w_exact_bf16 = not bool(wa_l.any()) and not bool(wd_l.any())
        self.Wa_p, self.Wd_p = _swizzle_tiles(wa_h, 128), _swizzle_tiles(wd_h, 128)
        self.Wal_p = self.Wdl_p = None
        if not self.w_exact_bf16:
            self.Wal_p, self.Wdl_p = _swizzle_tiles(wa_l, 128), _swizzle_tiles(wd_l, 128)
        self.ba_p = perm(self.att_bias[:, None]).reshape(-1).contiguous()
        self.bd_p = perm(self.dec_bias[:, None]).reshape(-1).contiguous()
        self.WqT = f32(w["att.query_layer"].T)                                           # [1024][128]
        self.Wloc = f32(w["att.location_conv"])                                          # [32][2][31]
        self.WdT = f32(w["att.location_dense"].T)                                        # [32][128]
        self.v = f32(w["att.v"][0])
        # location conv (32 x 2 x 31) composed with the location dense layer (32 -> 128): [2][31][128]
        self.WlocD = torch.einsum("fck,fa->cka", self.Wloc.double(), self.WdT.double()).float().contiguous()
        self.WpT = f32(torch.cat([w["proj.w"], w["gate.w"]], 0).T)                      # [1536][81]
        self.bp = f32(torch.cat([w["proj.b"], w["gate.b"]]))
        # HiFi-GAN
        wt, offs = tc.conv_weights(f32(w["hg.conv_pre.w"]), 1, c_in_pad=128)
        self.conv_pre = (wt, offs, f32(w["hg.conv_pre.b"]))
        self.ups, self.res = [], []
        for i, u in enumerate(UPS):
            wp, offs = tc.convt_weights(f32(w[f"hg.up{i}.w"]), u)
            self.ups.append((wp, offs, f32(w[f"hg.up{i}.b"])))
            blocks = []
            for j, k in enumerate(W.HG_RES_KERNELS):
                layers = []
                for m, dil in enumerate(W.HG_RES_DILATIONS):
                    key = f"hg.res{i}.{j}"
                    c1 = tc.conv_weights(f32(w[f"{key}.c1{m}.w"]), dil) + (f32(w[f"{key}.c1{m}.b"]),)
                    c2 = tc.conv_weights(f32(w[f"{key}.c2{m}.w"]), 1) + (f32(w[f"{key}.c2{m}.b"]),)
                    layers.append((c1, c2))
                blocks.append(layers)
            self.res.append(blocks)
        self.wpost = f32(w["hg.conv_post.w"][0])                                        # [32][7]
        self.bpost = float(w["hg.conv_post.b"][0])

    @_on_device
    def set_postnet(self, enabled: bool, weights: dict | None = None) -> None:
        """Turn the chunk-local PostNet (f3) on or off; weights default to postnet_weights(0)."""
        if enabled and (weights is not None or not hasattr(self, "_post_ptrs")):
            self._prepare_postnet(weights if weights is not None else W.postnet_weights(0))
        self.postnet = bool(enabled)

    def _prepare_postnet(self, pw: dict) -> None:
        """PostNet layers in tc_conv layout; the 80-channel ends padded to 96 (c_in, c_out % 32).
        Built on the engine stream (and waited for), so the first itts_r_postnet launch is ordered
        after these writes."""
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self._prepare_postnet_layers(pw)
        self.stream.synchronize()

    def _prepare_postnet_layers(self, pw: dict) -> None:
        d, layers = self.device, []
        for i in range(W.POSTNET_LAYERS):
            w = pw[f"post.conv{i}.w"].detach().float().to(d)
            b = pw[f"post.conv{i}.b"].detach().float().to(d)
            if w.shape[0] == W.N_MEL:   # last layer: 80 outputs -> 96 (zero rows)
                w = torch.cat([w, w.new_zeros(POST_CP - W.N_MEL, *w.shape[1:])], 0)
                b = torch.cat([b, b.new_zeros(POST_CP - W.N_MEL)])
            wt, _ = tc.conv_weights(w, 1, c_in_pad=POST_CP if w.shape[1] == W.N_MEL else None)
            layers += [wt, b.contiguous()]
        self._post_layers = layers   # keeps the tensors alive
        self._post_ptrs = (ctypes.c_int64 * len(layers))(*[t.data_ptr() for t in layers])

    def _apply_postnet(self, src_ptrs: np.ndarray, out_ptrs: np.ndarray, ms: list[int]) -> None:
        """out_i = mel_i + PostNet(mel_i) for n chunks of ms[i] frames (fp32 [m][80] at the given
        device addresses), one itts_r_postnet call on the engine stream."""
        n = len(ms)
        lay = _Layout(ms, POST_HALO)
        m_np = np.asarray(ms, np.int64)
        mplan = np.stack([np.zeros(n, np.int64), src_ptrs, m_np, np.zeros(n, np.int64), lay.first], 1)
        rm_plan = np.stack([lay.base, m_np, np.full(n, lay.halo, np.int64), lay.first, np.ones(n, np.int64)], 1)
        aplan = np.stack([src_ptrs, out_ptrs, m_np, lay.first], 1)
        pack = self._up(np.concatenate([mplan.reshape(-1), rm_plan.reshape(-1), aplan.reshape(-1)]))
        x0 = self._buf("post_x0", lay.total * POST_CP)
        ya = self._buf("post_ya", lay.total * W.POSTNET_CH)
        yb = self._buf("post_yb", lay.total * W.POSTNET_CH)
        post = self._buf("post_f32", lay.total * POST_CP, torch.float32)
        rm = self._buf("post_rm", lay.total, torch.int32)
        self._call("itts_r_postnet", pack.data_ptr(), n, max(ms), lay.total, max(ms) + 2 * lay.halo,
                   self._post_ptrs, x0.data_ptr(), ya.data_ptr(), yb.data_ptr(), post.data_ptr(), rm.data_ptr(),
                   self._st())
        self.launches += 7

    def _create_native_vocoder(self) -> int:
        """Handle of the C++ launch sequence (voc_run.cu) over this engine's HiFi-GAN weights."""
        ptrs = [self.conv_pre[0], self.conv_pre[2]]
        for wp, _, bias in self.ups:
            ptrs += [wp, bias]
        for blocks in self.res:
            for layers in blocks:
                for c1, c2 in layers:
                    ptrs += [c1[0], c1[2], c2[0], c2[2]]
        arr = (ctypes.c_int64 * len(ptrs))(*[t.data_ptr() for t in ptrs])
        h = ctypes.c_void_p()
        _native.call("itts_r_voc_create", ctypes.byref(h), arr, len(ptrs))
        weakref.finalize(self, _native.lib().itts_r_voc_destroy, h.value)
        return h.value

    # ------------------------------------------------------------ helpers
    def _st(self) -> int:
        return self.stream.cuda_stream

    def _call(self, name: str, *args) -> None:
        _native.call(name, *args)
        self.launches += 1

    def _conv(self, x, layer, c_out, row_out, **kw) -> None:
        wt, offs, bias = layer
        tc.conv1d_tc(x, wt, offs, bias, c_out, row_out, stream=self._st(), **kw)
        self.launches += 1

    def _resblock(self, x, c1, c2, dil, row_out, stream=None, **kw) -> None:
        st = self._st() if stream is None else stream.cuda_stream
        tc.resblock_tc(x, c1, c2, dil, row_out, stream=st, **kw)
        self.launches += 1

    def _buf(self, name: str, numel: int, dtype=torch.bfloat16, zero: bool = False) -> torch.Tensor:
        """Persistent grow-only work buffer (the first `numel` elements), so steady-state serving
        never reaches cudaMalloc.  All users run on the engine stream, so reuse is ordered."""
        t = self._pool.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(max(int(numel * 1.25), 1024), dtype=dtype, device=self.device)
            self._pool[name] = t
        v = t[:numel]
        if zero:
            v.zero_()
        return v

    def reserve_vocoder(self, max_batch: int, frames: int | None = None) -> None:
        """Grow the vocoder work buffers for `max_batch` chunks of `frames` (default O + C) frames."""
        T = frames or (self.cfg.overlap_frames + self.cfg.chunk_frames)
        rows0 = max_batch * (T + 2 * MEL_HALO)
        self._buf("x0", rows0 * 128)
        self._buf("act_in", rows0 * 512)
        biggest, mult = 0, 1
        for u, C in zip(UPS, STAGE_C):
            mult *= u
            biggest = max(biggest, max_batch * (T * mult + 2 * MRF_HALO) * C)
        if self.native_vocoder:
            self._call("itts_r_voc_reserve", self._voc, max_batch, T, self._st())
        else:
            for i in range(12):
                self._buf(f"b16_{i}", biggest)
        self._buf("audio", max_batch * T * self.cfg.hop_samples, torch.float32)
        for name, m in (("rm0", 1), ("rmT0", 1), ("rm_s0", 8), ("rmT1", 8), ("rm_s1", 64), ("rmT2", 64),
                        ("rm_s2", 128), ("rmT3", 128), ("rm_s3", 256)):
            self._buf(name, max_batch * (T * m + 2 * MRF_HALO), torch.int32)

    def prewarm_pinned(self, max_batch: int = 256) -> None:
        """Fill the caching host allocator with pinned blocks of every power-of-two size the
        serving path requests (plans up to the audio of `max_batch` chunks), so cudaHostAlloc --
        slow, and synchronising -- never runs inside a serving iteration."""
        top = max(4 * max_batch * (self.cfg.overlap_frames + self.cfg.chunk_frames) * self.cfg.hop_samples, 1 << 16)
        blocks = []
        for k in range(12, top.bit_length() + 1):
            for _ in range(4 if k < 20 else 3):
                blocks.append(torch.empty(1 << k, dtype=torch.uint8, pin_memory=True))
        del blocks

    def _iota(self, n: int) -> torch.Tensor:
        if n > self.iota.numel():
            self.iota = torch.arange(2 * n, dtype=torch.int32, device=self.device)
        return self.iota[:n]

    def _rowmap(self, layout: _Layout, out_first: np.ndarray, up: int, name: str | None = None) -> torch.Tensor:
        n = len(layout.rows)
        plan = np.stack([layout.base, np.array(layout.rows, np.int64), np.full(n, layout.halo, np.int64),
                         out_first.astype(np.int64), np.full(n, up, np.int64)], 1)
        rm = (self._buf(name, layout.total, torch.int32) if name is not None
              else torch.empty(layout.total, dtype=torch.int32, device=self.device))
        self._call("itts_r_rowmap", self._up(plan).data_ptr(), n,
                   int(max(layout.rows)) + 2 * layout.halo, rm.data_ptr(), self._st())
        return rm

    def state_size(self, L: int) -> int:
        return ROW + 2 * L

    def voc_size(self) -> int:
        return self.cfg.overlap_frames * W.N_MEL + self.cfg.overlap_samples

    # ------------------------------------------------------------ encoder
    @_on_device
    def pre_encode(self, fos) -> None:
        """Encode just-submitted requests' frontend outputs now (queued on the engine stream behind
        the vocoder call being waited on, so the work runs in the host gap between iterations);
        encoder_batch returns these results when the admitting iteration passes the same
        FrontendOutput objects.  Per-request results are independent of the batch they were
        computed in (batch transparency), so admission and outputs are unchanged."""
        if not self.pre_encode_enabled or not fos:
            return
        try:
            res = self._encode(list(fos))
        except Exception:  # noqa: BLE001 -- the admitting iteration encodes (and reports) itself
            return
        for fo, r in zip(fos, res):
            self._pre_enc[id(fo)] = (fo, r)
        while len(self._pre_enc) > 1024:   # requests never admitted (shutdown): forget the oldest
            self._pre_enc.pop(next(iter(self._pre_enc)))

    @_on_device
    def encoder_batch(self, fos) -> list:
        if self._pre_enc:
            hit = []
            for fo in fos:
                e = self._pre_enc.pop(id(fo), None)
                hit.append(e[1] if e is not None and e[0] is fo else None)
            if any(h is not None for h in hit):
                rest = [fo for fo, h in zip(fos, hit) if h is None]
                fresh = iter(self._encode(rest) if rest else [])
                self.pre_enc_hits += sum(h is not None for h in hit)
                return [h if h is not None else next(fresh) for h in hit]
        return self._encode(fos)

    def _encode(self, fos) -> list:
        n = len(fos)
        if n == 0:
            return []
        lens = [fo.seq_len for fo in fos]
        if min(lens) < 1:
            raise ValueError("frontend output needs at least one phoneme")
        total = sum(lens)
        tok = np.empty((4, total), dtype=np.int64)
        pos = 0
        for fo, L in zip(fos, lens):
            tok[:, pos:pos + L] = (fo.phonemes, fo.pw, fo.pph, fo.iph)
            pos += L
        if tok[0].max() >= W.N_SYMBOLS or tok[0].min() < 0:
            raise ValueError("phoneme id outside the embedding table")
        if tok[1:].max() > 1 or tok[1:].min() < 0:
            raise ValueError("prosody tokens must be 0/1")
        tok = tok.astype(np.int32)
        lay = _Layout(lens, ENC_HALO)
        reqs = []
        for L in lens:
            req = DeviceRequest(self, L)
            req.extra["mem_off"] = req.add_region(L * W.EMB)
            req.extra["pm_off"] = req.add_region(L * W.ATT_DIM)
            buf = req.claim(req.state_bufs, self.state_size(L), set())
            reqs.append((req, buf))
        a = self.arena
        tok_off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        plan = np.zeros((n, 6), dtype=np.int64)
        for i, (req, _) in enumerate(reqs):
            plan[i] = (tok_off[i], lens[i], lay.first[i], a.ptr(req.extra["mem_off"]),
                       a.ptr(req.extra["pm_off"]), 0)
        st = self._st()
        if self.native_encoder:
            return self._encode_native(tok, plan, lay, reqs, total, n, max(lens))
        with torch.cuda.stream(self.stream):
            d_tok, d_plan = self._up(tok), self._up(plan)
            mark = self._mark("encoder", total)
            mark.__enter__()
            xa = torch.zeros(lay.total, W.EMB, dtype=torch.bfloat16, device=self.device)
            xb = torch.empty_like(xa)
            self._call("itts_r_enc_embed", d_tok.data_ptr(), total, d_plan.data_ptr(), n, max(lens),
                       *[e.data_ptr() for e in self.E], xa.data_ptr(), st)
            rm = self._rowmap(lay, lay.first, 1)
            for i, layer in enumerate(self.enc_conv):
                src, dst = (xa, xb) if i % 2 == 0 else (xb, xa)
                self._conv(src, layer, W.EMB, rm, act_out=dst, slope=0.0)
            pre = torch.empty(lay.total, 2048, dtype=torch.float32, device=self.device)
            self._conv(xb, self.enc_ih, 2048, rm, f32_out=pre, bn=128)
            self._call("itts_r_bilstm", pre.data_ptr(), d_plan.data_ptr(), n, self.enc_whhT.data_ptr(), st)
            self._call("itts_r_pmem", d_plan.data_ptr(), n, max(lens), self.WmT.data_ptr(), st)
            for req, buf in reqs:
                a.tensor[buf.off:buf.off + self.state_size(req.seq_len)].zero_()
            mark.__exit__(None, None, None)
        fpp = self.cfg.frames_per_phoneme
        return [(DeviceEncodedFeatures(req), DeviceDecoderState(req, buf, 0, fpp * req.seq_len))
                for req, buf in reqs]

    def _encode_native(self, tok, plan, lay, reqs, total, n, max_len) -> list:
        """encoder_batch's launch sequence issued from C++ (itts_r_encode) after one H2D copy of
        tokens, item plan, row-map plan and the state rows to zero."""
        a = self.arena
        rm_plan = np.stack([lay.base, np.array(lay.rows, np.int64), np.full(n, lay.halo, np.int64),
                            lay.first.astype(np.int64), np.ones(n, np.int64)], 1)
        spans = np.array([(a.ptr(buf.off), self.state_size(req.seq_len)) for req, buf in reqs], np.int64)
        tok_words = np.zeros((4 * total + 1) // 2 * 2, np.int32)
        tok_words[:4 * total] = tok.reshape(-1)
        pack = np.concatenate([tok_words.view(np.int64), plan.reshape(-1), rm_plan.reshape(-1), spans.reshape(-1)])
        with torch.cuda.stream(self.stream):
            d_pack = self._up(pack)
            pre = self._buf("enc_pre", lay.total * 2048, torch.float32)
            rm = self._buf("enc_rm", lay.total, torch.int32)
            span = int(max(lay.rows)) + 2 * lay.halo
            with self._mark("encoder", total):
                if self.precision == "parity":
                    x3 = self._buf("enc_x3", lay.total * 3 * W.EMB)
                    f32 = self._buf("enc_f32", lay.total * W.EMB, torch.float32)
                    self._call("itts_r_encode_split", d_pack.data_ptr(), total, n, max_len, lay.total, span,
                               self._enc_ptrs3, ENC_TAPS, x3.data_ptr(), f32.data_ptr(), pre.data_ptr(),
                               rm.data_ptr(), self.enc_parts, self._st())
                    self.launches += 13  # embed, 4 splits, row map, 3 convs, input projection, BiLSTM, memory, zero
                else:
                    xa = self._buf("enc_xa", lay.total * W.EMB)
                    xb = self._buf("enc_xb", lay.total * W.EMB)
                    self._call("itts_r_encode", d_pack.data_ptr(), total, n, max_len, lay.total, span,
                               self._enc_ptrs, ENC_TAPS, xa.data_ptr(), xb.data_ptr(), pre.data_ptr(),
                               rm.data_ptr(), self._st())
                    self.launches += 9   # embed, row map, 3 convs, input projection, BiLSTM, memory, state zero
        fpp = self.cfg.frames_per_phoneme
        return [(DeviceEncodedFeatures(req), DeviceDecoderState(req, buf, 0, fpp * req.seq_len))
                for req, buf in reqs]

    # ------------------------------------------------------------ decoder
    def _dec_items(self, pairs, taken: set, cols=None, limits=None) -> list:
        """Per-item decoder plan fields (steps, L, dst buffer, mem / pm / src / dst offsets) --
        the host work between the previous vocoder wait and the decoder launch."""
        C = self.cfg.chunk_frames
        cols = cols if cols is not None else ([], [], [], [], [], [], [])
        steps, dsts, Ls, mem_off, pm_off, src_off, dst_off = cols
        for k, (state, enc) in enumerate(pairs):
            if type(state) is not DeviceDecoderState or type(enc) is not DeviceEncodedFeatures:
                if not isinstance(state, DeviceDecoderState) or not isinstance(enc, DeviceEncodedFeatures):
                    raise TypeError("Tier-R GPU decoder needs handles produced by its own encoder")
            req = state.req
            if req is not enc.req or req.engine is not self:
                raise ValueError("decoder state does not match encoded features")
            left = state.target_frames - state.frames_emitted
            if left <= 0:
                raise ValueError("decode past stop")
            n_steps = C if left > C else left
            if limits is not None:
                n_steps = min(n_steps, int(limits[k]))
                if n_steps < 1:
                    raise ValueError("step limit must be >= 1")
            steps.append(n_steps)
            L = req.seq_len
            Ls.append(L)
            d = req.claim(req.state_bufs, ROW + 2 * L, taken)
            dsts.append(d)
            ex = req.extra
            mem_off.append(ex["mem_off"])
            pm_off.append(ex["pm_off"])
            src_off.append(state.buf.off)
            dst_off.append(d.off)
        return cols

    def _speculate_next_decoder(self) -> None:
        """While the vocoder runs: the plan fields of the items that continue (the last decoder
        call's non-stopped results, in order -- the next call's batch prefix unless the
        scheduler drops an item).  decoder_batch uses them only if its pairs start with exactly
        these state / feature objects; the buffer claims are the ones it would make (the previous
        states are gone by now, so the free ping-pong buffer is determined)."""
        src, self._spec_src = self._spec_src, None
        self._spec = None
        self._spec_out = None
        if not src or not self.speculate:
            return
        if self.spec_launch_min and len(src) >= self.spec_launch_min and self._last_full_decode:
            # large pools: LAUNCH the continuing items' next chunk now, behind this vocoder call on
            # the engine stream, so the GPU does not idle while the host finishes this iteration
            # and prepares the next; decoder_batch returns these results for the matching pairs
            # (bit-identical: batch transparency) and decodes only the newly admitted items
            try:
                out = self._decode(src)
            except Exception:  # noqa: BLE001 -- the real call redoes (and retries) it
                return
            self._spec_out = (src, out)
            return
        taken: set = set()
        try:
            cols = self._dec_items(src, taken)
        except Exception:  # noqa: BLE001 -- the real call raises (and is retried per item) itself
            return
        self._spec = (src, taken, cols)

    @_on_device
    def decoder_steps(self, triples) -> list:
        """Step-granular decoding (the opt-in admission mode, ``scheduler.run_iteration_steps``):
        (state, features, limit) -> DecodeChunkResult of min(limit, frames left in the chunk) steps."""
        self._spec_out = None
        self._last_full_decode = False
        return self._decode([(s, e) for s, e, _ in triples], [lim for _, _, lim in triples])

    @_on_device
    def concat_mels(self, parts: list) -> DeviceMelChunk:
        """One mel chunk from consecutive partial decodes of the same request (engine stream)."""
        if len(parts) == 1:
            return parts[0]
        with torch.cuda.stream(self.stream):
            return DeviceMelChunk(torch.cat([m.data for m in parts], 0), parts[0].req)

    @_on_device
    def decoder_batch(self, pairs) -> list:
        self._last_full_decode = True
        so, self._spec_out = self._spec_out, None
        if so is None:
            return self._decode(pairs)
        # items whose next chunk was launched during the last vocoder wait (same state / feature
        # objects); the others -- normally just the newly admitted ones -- decode now
        done = {(id(st), id(enc)): r for (st, enc), r in zip(*so)}
        hit = [done.get((id(st), id(enc))) for st, enc in pairs]
        rest = [p for p, h in zip(pairs, hit) if h is None]
        fresh = iter(self._decode(rest) if rest else [])
        out = [h if h is not None else next(fresh) for h in hit]
        self._spec_src = [(r.state, enc) for r, (_, enc) in zip(out, pairs) if not r.stop]
        self.spec_hits += len(pairs) - len(rest)
        return out

    def _decode(self, pairs, limits=None) -> list:
        n = len(pairs)
        if n == 0:
            return []
        if n > PERSIST_MAX_B and self.persistent_decoder:
            # items are independent and the kernel is batch-invariant: balanced slices of <= 512 rows
            per = -(-n // -(-n // PERSIST_MAX_B))
            self._spec = None
            out = []
            for i in range(0, n, per):
                out += self._decode(pairs[i:i + per], None if limits is None else limits[i:i + per])
            self._spec_src = [(r.state, enc) for r, (_, enc) in zip(out, pairs) if not r.stop]
            return out
        C = self.cfg.chunk_frames
        a = self.arena
        spec, self._spec = self._spec, None
        if limits is not None:
            spec = None
            taken = set()
            cols = self._dec_items(pairs, taken, limits=limits)
        elif (spec is not None and len(spec[0]) <= n
                and all(p[0] is q[0] and p[1] is q[1] for p, q in zip(pairs, spec[0]))):
            taken, cols = spec[1], tuple(list(c) for c in spec[2])
            self._dec_items(pairs[len(spec[0]):], taken, cols)   # the newly admitted items
        else:
            taken = set()
            cols = self._dec_items(pairs, taken)
        steps, dsts, Ls, mem_off, pm_off, src_off, dst_off = cols
        base = a.ptr(0)
        max_L, max_steps = max(Ls), max(steps)
        steps_np = np.array(steps, dtype=np.int64)
        Ls_np = np.array(Ls, dtype=np.int64)
        src = base + 4 * np.array(src_off, dtype=np.int64)
        dstp = base + 4 * np.array(dst_off, dtype=np.int64)
        wbytes = DEC_WEIGHT_BYTES_SPLIT if self.precision == "parity" and not self.w_exact_bf16 else DEC_WEIGHT_BYTES
        dec_bytes = lambda: max_steps * wbytes + int(  # algorithmic bytes (timers only)
            (steps_np * (2 * 4 * ROW + Ls_np * (4 * 512 + 4 * 128 + 16) + 4 * 81)).sum())
        with torch.cuda.stream(self.stream):
            if self.use_graphs and max_steps == C and max_L <= GRAPH_MAX_L:
                bk = self._dec_bucket(n)
                B = bk.B
                hn = bk.host_np
                if bk.pending:  # the previous H2D out of the staging buffer must have finished
                    bk.copied.synchronize()
                if not self.plan_staging:   # whole template rewritten (A/B of the row-wise staging)
                    hn[:] = bk.template
                    bk.dirty = 0
                if bk.dirty > n:  # rows [n, dirty) go back to the idle template
                    for lo, hi in ((0, 8 * B), (8 * B, 9 * B), (9 * B, 10 * B)):
                        step = 8 if hi - lo == 8 * B else 1
                        hn[lo + n * step:lo + bk.dirty * step] = bk.template[lo + n * step:lo + bk.dirty * step]
                bk.dirty = n
                plan = hn[:8 * B].reshape(B, 8)
                plan[:n, 0] = base + 4 * np.array(mem_off, dtype=np.int64)
                plan[:n, 1] = base + 4 * np.array(pm_off, dtype=np.int64)
                plan[:n, 2] = Ls_np
                plan[:n, 3] = src + 4 * ROW
                plan[:n, 4] = dstp + 4 * ROW
                plan[:n, 5] = steps_np
                hn[8 * B:8 * B + n] = src
                hn[9 * B:9 * B + n] = dstp
                self.h2d_bytes += hn.nbytes
                bk.packed.copy_(bk.host, non_blocking=True)
                bk.copied.record(self.stream)
                bk.pending = True
                with self._mark("decoder", dec_bytes):
                    if bk.graph is None:
                        bk.capture(self)
                    bk.graph.replay()
                    self.launches += bk.launches
                mel_all, gate_all = bk.mel[:n].clone(), bk.gate[:n].clone()
                if self.postnet:
                    rows = mel_all.data_ptr() + 4 * W.N_MEL * C * np.arange(n, dtype=np.int64)
                    out = torch.empty_like(mel_all)
                    self._apply_postnet(rows, out.data_ptr() + (rows - mel_all.data_ptr()), steps)
                    mel_all = out
                mels = [DeviceMelChunk.row_of(mel_all, i, steps[i], st.req, gate_all)
                        for i, (st, _) in enumerate(pairs)]
            else:
                mel_off = np.concatenate([[0], np.cumsum(steps_np)]).astype(np.int64)
                mel = torch.empty(int(mel_off[-1]), W.N_MEL, dtype=torch.float32, device=self.device)
                gate = torch.empty(int(mel_off[-1]), dtype=torch.float32, device=self.device)
                if self.poison_scratch is True or (self.poison_scratch and "mel" in self.poison_scratch):
                    v = self.poison_scratch["mel"] if isinstance(self.poison_scratch, dict) else float("nan")
                    mel.fill_(v)
                    gate.fill_(v)
                plan = np.zeros((n, 8), dtype=np.int64)
                plan[:, 0] = base + 4 * np.array(mem_off, dtype=np.int64)
                plan[:, 1] = base + 4 * np.array(pm_off, dtype=np.int64)
                plan[:, 2] = Ls_np
                plan[:, 3] = src + 4 * ROW
                plan[:, 4] = dstp + 4 * ROW
                plan[:, 5] = steps_np
                plan[:, 6] = mel.data_ptr() + 4 * W.N_MEL * mel_off[:-1]
                plan[:, 7] = gate.data_ptr() + 4 * mel_off[:-1]
                packed = self._up(np.concatenate([plan.reshape(-1), src, dstp]))
                bufs = _DecBuffers(self, n, packed)
                if self.poison_scratch:
                    self._last_bufs = bufs   # debug: the scratch of the last poisoned call
                with self._mark("decoder", dec_bytes):
                    self._enqueue_decoder(bufs, max_L, max_steps)
                if self.postnet:
                    rows = mel.data_ptr() + 4 * W.N_MEL * mel_off[:-1]
                    out = torch.empty_like(mel)
                    self._apply_postnet(rows, out.data_ptr() + (rows - mel.data_ptr()), steps)
                    mel = out
                mels = [DeviceMelChunk(mel[int(mel_off[i]):int(mel_off[i + 1])], st.req)
                        for i, (st, _) in enumerate(pairs)]
                for i, m in enumerate(mels):
                    m._gate, m._row = gate[int(mel_off[i]):int(mel_off[i + 1])][None], 0
        out = []
        for (state, _), dst, k, m in zip(pairs, dsts, steps, mels):
            emitted = state.frames_emitted + k
            out.append(DecodeChunkResult(m, emitted >= state.target_frames,
                                         DeviceDecoderState(state.req, dst, emitted, state.target_frames)))
        self._spec_src = [(r.state, enc) for r, (_, enc) in zip(out, pairs) if not r.stop]
        if self.keep_last_decoder:
            self._last_dec = (list(pairs), out)
        return out

    def _enqueue_decoder(self, b: "_DecBuffers", max_L: int, nsteps: int) -> None:
        """K1 gather -> nsteps x (prenet, att GEMM, cell, query, attention, dec GEMM, cell, proj) -> K1 scatter."""
        st, n = self._st(), b.n
        self._call("itts_gather_rows", b.work.data_ptr(), b.d_src.data_ptr(), n, 4 * ROW, st)
        if self.persistent_decoder and max_L <= PERSIST_MAX_L and n <= PERSIST_MAX_B:
            split = self.precision == "parity"
            b.ensure_persistent(max_L, split)
            self._call("itts_r_decode_persistent", n, nsteps, b.d_plan.data_ptr(), b.work.data_ptr(),
                       b.xb2.data_ptr(), self.W0T.data_ptr(), self.W1T.data_ptr(), self.Wa_p.data_ptr(),
                       self.ba_p.data_ptr(), self.Wd_p.data_ptr(), self.bd_p.data_ptr(), self.WqT.data_ptr(),
                       self.WlocD.data_ptr(), self.v.data_ptr(), self.WpT.data_ptr(),
                       self.bp.data_ptr(), b.Gp.data_ptr(), b.H1.data_ptr(), b.Q.data_ptr(), b.P.data_ptr(),
                       b.U.data_ptr(),
                       b.U.shape[1], b.AP.data_ptr(), b.bar.data_ptr(),
                       self.Wal_p.data_ptr() if split and not self.w_exact_bf16 else 0,
                       self.Wdl_p.data_ptr() if split and not self.w_exact_bf16 else 0, int(split), st)
            self._call("itts_scatter_rows", b.d_dst.data_ptr(), b.work.data_ptr(), n, 4 * ROW, st)
            return
        self._call("itts_r_dec_prepare", b.work.data_ptr(), b.xbm.data_ptr(), n, st)
        rows = self._iota(n)
        x_att, x_dec = b.xbm[:, :1792], b.xbm[:, 256:]
        for step in range(nsteps):
            self._call("itts_r_prenet", b.work.data_ptr(), b.xbm.data_ptr(), self.W0T.data_ptr(),
                       self.W1T.data_ptr(), b.d_plan.data_ptr(), b.H1.data_ptr(), n, step, st)
            self._conv(x_att, self.att_gemm, 4096, rows, f32_out=b.G, ksplit=DEC_KSPLIT, bn=64)
            self._call("itts_r_lstm_cell", b.G.data_ptr(), DEC_KSPLIT, self.att_bias.data_ptr(), b.work.data_ptr(),
                       b.xbm.data_ptr(), ATTH_OFF, ATTC_OFF, b.d_plan.data_ptr(), n, step, st)
            self._call("itts_r_query", b.work.data_ptr(), self.WqT.data_ptr(), b.Q.data_ptr(), n, st)
            self._call("itts_r_attention", b.work.data_ptr(), b.xbm.data_ptr(), b.d_plan.data_ptr(), n, max_L,
                       b.Q.data_ptr(), self.Wloc.data_ptr(), self.WdT.data_ptr(), self.v.data_ptr(), step, st)
            self._conv(x_dec, self.dec_gemm, 4096, rows, f32_out=b.G, ksplit=DEC_KSPLIT, bn=64)
            self._call("itts_r_lstm_cell", b.G.data_ptr(), DEC_KSPLIT, self.dec_bias.data_ptr(), b.work.data_ptr(),
                       b.xbm.data_ptr(), DECH_OFF, DECC_OFF, b.d_plan.data_ptr(), n, step, st)
            self._call("itts_r_proj", b.work.data_ptr(), b.d_plan.data_ptr(), n, self.WpT.data_ptr(),
                       self.bp.data_ptr(), b.P.data_ptr(), step, st)
        self._call("itts_scatter_rows", b.d_dst.data_ptr(), b.work.data_ptr(), n, 4 * ROW, st)

    def _dec_bucket(self, n: int) -> "_DecBucket":
        B = -(-n // 16) * 16
        if B not in self._dec_buckets:
            self._dec_buckets[B] = _DecBucket(self, B, GRAPH_MAX_L)
        return self._dec_buckets[B]

    @_on_device
    def prepare_graphs(self, max_batch: int = 256) -> None:
        """Capture the decoder-chunk graph of every 16-row bucket up to ``max_batch`` now, and
        grow the vocoder work buffers for that batch, so no capture or cudaMalloc happens on
        the serving path."""
        self.prewarm_pinned(max_batch)
        with torch.cuda.stream(self.stream):
            self.reserve_vocoder(max_batch)
            for B in range(16, min(max_batch, PERSIST_MAX_B) + 1, 16):   # larger pools run in slices
                bk = self._dec_bucket(B)
                if bk.graph is None:
                    bk.idle_plan()
                    bk.capture(self)
        self.stream.synchronize()

    # ------------------------------------------------------------ vocoder
    @_on_device
    def vocoder_batch(self, triples) -> list:
        n = len(triples)
        if n == 0:
            return []
        O, H, S = self.cfg.overlap_frames, self.cfg.hop_samples, self.cfg.overlap_samples
        metas, host_mels = [], []
        for vstate, mel, is_last in triples:
            m = int(mel.frame_count)
            if not is_last and m < O:
                raise ValueError("non-final chunk shorter than the overlap window")
            has_tail = (vstate.has_tail if isinstance(vstate, DeviceVocoderState)
                        else vstate.mel_tail is not None)
            if not has_tail and not is_last and m * H <= S:
                raise ValueError("non-final chunk shorter than the overlap window")
            if isinstance(mel, DeviceMelChunk):
                if mel.width != W.N_MEL:
                    raise ValueError("mel chunk width must be 80")
            else:
                frames = np.asarray(mel.frames, dtype=np.float32)
                if frames.ndim != 2 or frames.shape[1] != W.N_MEL:
                    raise ValueError("mel chunk width must be 80")
                host_mels.append(frames)
            T = (O if has_tail else 0) + m
            metas.append((m, has_tail, bool(is_last), T, T * H, T * H if is_last else T * H - S))
        counts = [mt[5] for mt in metas]
        out_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        Ts = [mt[3] for mt in metas]
        a, st, dev = self.arena, self._st(), self.device
        keep, taken, results = [], set(), []
        with torch.cuda.stream(self.stream):
            if host_mels:
                hm = self._up(np.concatenate([f.reshape(-1) for f in host_mels]))
            hpos = 0
            lay0 = _Layout(Ts, MEL_HALO)
            stage4 = _Layout([T * 256 for T in Ts], MRF_HALO)
            owners = self._claim_voc(triples, [mt[2] for mt in metas], taken)  # before any a.ptr()
            # plan columns gathered per item, arrays built once (a numpy row store per item costs
            # more than the rest of the loop)
            tail_c, mel_c, dst_c = [], [], []
            for (vstate, mel, is_last), (m, has_tail, last, T, G, cnt), (req, dst) in zip(triples, metas, owners):
                if isinstance(mel, DeviceMelChunk):
                    mel_ptr = mel.ptr
                else:
                    mel_ptr = hm.data_ptr() + 4 * hpos
                    hpos += m * W.N_MEL
                tail_ptr = 0
                if has_tail:
                    if isinstance(vstate, DeviceVocoderState):
                        tail_ptr = a.ptr(vstate.buf.off)
                    else:
                        t = self._up(np.concatenate([np.asarray(vstate.mel_tail, np.float32).reshape(-1),
                                                     np.asarray(vstate.held_tail, np.float32).reshape(-1)]))
                        keep.append(t)
                        tail_ptr = t.data_ptr()
                tail_c.append(tail_ptr)
                mel_c.append(mel_ptr)
                dst_c.append(0 if dst is None else a.ptr(dst.off))
                results.append((req, dst, int(vstate.emitted_samples)))
            mt_arr = np.array(metas, dtype=np.int64)            # m, has_tail, last, T, G, cnt
            tail_a = np.array(tail_c, dtype=np.int64)
            mel_a = np.array(mel_c, dtype=np.int64)
            mplan = np.stack([tail_a, mel_a, mt_arr[:, 0], O * mt_arr[:, 1], lay0.first.astype(np.int64)], 1)
            pplan = np.stack([stage4.first.astype(np.int64), mt_arr[:, 4], mt_arr[:, 1] | 2 * mt_arr[:, 2],
                              np.where(mt_arr[:, 1] != 0, tail_a + 4 * O * W.N_MEL, 0),
                              np.array(dst_c, dtype=np.int64), out_off[:-1], mel_a, mt_arr[:, 0]], 1)
            d_mplan = self._up(mplan)
            d_pplan = self._up(pplan)
            audio = self._buf("audio", max(int(out_off[-1]), 1), torch.float32)
            with self._mark("vocoder", 2.0 * HIFIGAN_MACS_PER_FRAME * sum(Ts)):
                x4 = self._hifigan(Ts, lay0, d_mplan)
            want_pcm = self.pcm16 or self.wire_b64
            pcm = self._buf("pcm16", max(int(out_off[-1]), 1), torch.int16) if want_pcm else None
            nonfinite = self._buf("voc_nonfinite", n, torch.int32)
            self._call("itts_r_post_splice", x4 if isinstance(x4, int) else x4.data_ptr(), d_pplan.data_ptr(), n, max(mt[4] for mt in metas),
                       self.wpost.data_ptr(), self.bpost, self.fade.data_ptr(), O, S, audio.data_ptr(),
                       0 if pcm is None else pcm.data_ptr(), nonfinite.data_ptr(), st)
            if pcm is not None and self.pcm16:
                host_pcm = torch.empty(pcm.numel(), dtype=torch.int16, pin_memory=True)
                host_pcm.copy_(pcm, non_blocking=True)
            if self.wire_b64:   # base64 text of every chunk's PCM16, one kernel + one D2H
                b64_len = 4 * ((2 * np.asarray(counts, np.int64) + 2) // 3)
                b64_off = np.concatenate([[0], np.cumsum(b64_len)]).astype(np.int64)
                bplan = self._up(np.stack([out_off[:-1], np.asarray(counts, np.int64), b64_off[:-1]], 1))
                b64 = self._buf("b64", max(int(b64_off[-1]), 1), torch.uint8)
                self._call("itts_r_pcm16_b64", pcm.data_ptr(), bplan.data_ptr(), n, max(counts), b64.data_ptr(), st)
                host_b64 = torch.empty(max(int(b64_off[-1]), 1), dtype=torch.uint8, pin_memory=True)
                host_b64.copy_(b64[:host_b64.numel()], non_blocking=True)
            total = int(out_off[-1])
            # D2H straight into a pinned ring slot whose earlier chunks are all gone; the new chunks
            # are read-only views of it (no host copy).  No free slot (a client holding chunks of
            # several iterations): the persistent buffer, copied out after the wait.
            slot = self._out_slot(total)
            if slot is not None:
                host = slot[0][:total]
            else:
                if self._pin_out.numel() < total:   # grow-only persistent D2H buffer
                    self._pin_out = torch.empty(int(total * 1.5), dtype=torch.float32, pin_memory=True)
                host = self._pin_out[:total]
            host.copy_(audio[:total], non_blocking=True)
            if self._nf_pin.numel() < n:
                self._nf_pin = torch.empty(2 * n, dtype=torch.int32, pin_memory=True)
            nf_host = self._nf_pin[:n]
            nf_host.copy_(nonfinite, non_blocking=True)
        # result objects are built while the GPU works: the chunks are read-only views of `flat`
        flat = slot[1][:total] if slot is not None else np.empty(total, dtype=np.float32)
        out = []
        oo = out_off.tolist()
        for i, (req, dst, emitted) in enumerate(results):
            chunk = AudioChunk.trusted(flat[oo[i]:oo[i + 1]], emitted)
            out.append((chunk, DeviceVocoderState(req, dst, emitted + counts[i])))
        v_done = torch.cuda.Event()
        v_done.record(self.stream)        # this call's D2H copies are queued before this point
        self._speculate_next_decoder()    # may enqueue the next decoder chunk behind it
        if self.idle_hook is not None:
            self.idle_hook(v_done.query)
        v_done.synchronize()
        self.d2h_bytes += 4 * total + 4 * n
        if slot is None:
            np.copyto(flat, host.numpy())
        if nf_host.numpy().any() or (self.host_finite_check and not np.isfinite(flat).all()):
            if self.diagnose:
                self._diagnose_nonfinite(triples, flat, out_off)
            raise ValueError("array contains non-finite values")
        if self.wire_b64:
            raw = host_b64.numpy().tobytes()
            for i, (chunk, _) in enumerate(out):
                object.__setattr__(chunk, "_b64", raw[b64_off[i]:b64_off[i + 1]].decode("ascii"))
            self.d2h_bytes += int(b64_off[-1])
        if self.pcm16:
            pcm_np = host_pcm.numpy()
            for i, (chunk, _) in enumerate(out):
                object.__setattr__(chunk, "_pcm16", pcm_np[out_off[i]:out_off[i + 1]].astype("<i2").tobytes())
                self.d2h_bytes += 2 * counts[i]
        return out

    def _out_slot(self, total: int):
        """A pinned audio slot for `total` samples no live chunk views (None: all in use)."""
        ring = self._out_ring
        for _ in range(len(ring)):
            k = self._out_next
            self._out_next = (k + 1) % len(ring)
            if ring[k] is None or ring[k][0].numel() < total:
                if ring[k] is not None and sys.getrefcount(ring[k][1]) > 2:
                    continue   # too small AND still viewed: leave it to its chunks
                t = torch.empty(max(int(total * 1.25), 1 << 20), dtype=torch.float32, pin_memory=True)
                ring[k] = (t, t.numpy())
                return ring[k]
            if sys.getrefcount(ring[k][1]) == 2:   # only the ring (and the call) reference the array
                return ring[k]
        return None

    def _diagnose_nonfinite(self, triples, flat, out_off) -> None:
        """Failure path only: which inputs of the non-finite chunks are already non-finite."""
        import sys
        for i, (vstate, mel, last) in enumerate(triples):
            if np.isfinite(flat[out_off[i]:out_off[i + 1]]).all():
                continue
            req = getattr(mel, "req", None)
            info = {"item": i, "batch": len(triples), "frames": mel.frame_count, "last": bool(last),
                    "mel_finite": bool(np.isfinite(np.asarray(mel.frames)).all())}
            if req is not None:
                info["L"] = req.seq_len
                info["enc_finite"] = bool(np.isfinite(self.read_features(req)).all())
                info["pmem_finite"] = bool(np.isfinite(self.read_processed_memory(req)).all())
            self.failures.append(info)
            print("itts non-finite chunk:", info, file=sys.stderr, flush=True)
        if self._last_dec is not None and any(getattr(m, "req", None) is not None and
                                              any(m is r.mel for r in self._last_dec[1]) for _, m, _ in triples):
            info = self._rerun_last_decoder()
            self.failures.append(info)
            print("itts decoder re-run:", info, file=sys.stderr, flush=True)

    def _rerun_last_decoder(self) -> dict:
        """Failure path only: decode the last decoder call's inputs again (graph and eager) and
        compare bit for bit with what that call produced."""
        pairs, out = self._last_dec
        self._last_dec = None
        keep, spec_src, graphs = self.keep_last_decoder, self._spec_src, self.use_graphs
        self.keep_last_decoder = False
        bad = lambda fr: [i for i, f in enumerate(fr) if not np.isfinite(f).all()]
        info: dict = {"batch": len(pairs)}
        try:
            orig = [r.mel.frames for r in out]
            info["orig_nonfinite"] = bad(orig)
            info["src_nonfinite"] = [i for i, (st, _) in enumerate(pairs)
                                     if not np.isfinite(self._read(st.buf.off, self.state_size(st.req.seq_len))).all()]
            info["steps"] = [r.mel.frame_count for r in out]
            info["L"] = [st.req.seq_len for st, _ in pairs]
            for tag, use_graphs, poison in (("first", graphs, False), ("eager", False, False),
                                            ("eager_poisoned", False, True)):
                self.use_graphs, self.poison_scratch = use_graphs, poison
                try:
                    again = [r.mel.frames for r in self.decoder_batch(pairs)]
                finally:
                    self.poison_scratch = False
                info[f"{tag}_nonfinite"] = bad(again)
                info[f"{tag}_differs"] = [i for i, (a, b) in enumerate(zip(orig, again))
                                          if not np.array_equal(a, b, equal_nan=True)]
            if self.bisect_dir is not None and info.get("eager_nonfinite"):
                info["bisect"] = self._bisect_decoder(pairs)
        except Exception as exc:  # noqa: BLE001 -- diagnostics must not mask the failure
            info["error"] = repr(exc)
        finally:
            self.keep_last_decoder, self._spec_src, self.use_graphs = keep, spec_src, graphs
        return info

    # ------------------------------------------------------------ failure reproduction (debug only)
    def _bisect_decoder(self, pairs) -> dict:
        """Shrink a decoder batch whose eager re-run gives non-finite mel to a small failing subset
        (delta debugging on the item list), dump it with debug_dump_decoder_case."""
        import os
        self.use_graphs = False
        tries = {"n": 0}

        def fails(sub) -> bool:
            tries["n"] += 1
            return any(not np.isfinite(r.mel.frames).all() for r in self.decoder_batch(list(sub)))

        out: dict = {"solo_fails": [i for i in range(min(len(pairs), 8)) if fails([pairs[i]])]}
        cur, k = list(range(len(pairs))), 2
        while len(cur) > 1 and tries["n"] < 80:
            size = -(-len(cur) // k)
            parts = [cur[i:i + size] for i in range(0, len(cur), size)]
            for part in parts:   # a failing part
                if fails([pairs[i] for i in part]):
                    cur, k = part, 2
                    break
            else:
                for part in parts:   # a failing complement
                    rest = [i for i in cur if i not in part]
                    if len(parts) > 2 and fails([pairs[i] for i in rest]):
                        cur, k = rest, max(k - 1, 2)
                        break
                else:
                    if k >= len(cur):
                        break
                    k = min(len(cur), 2 * k)
        out["minimal"] = cur
        out["minimal_fails_again"] = [fails([pairs[i] for i in cur]) for _ in range(3)]
        out["tries"] = tries["n"]
        os.makedirs(self.bisect_dir, exist_ok=True)
        path = os.path.join(self.bisect_dir, f"dec_case_{len(self.failures)}.npz")
        self.debug_dump_decoder_case([pairs[i] for i in cur], path)
        out["dump"] = path
        return out

    def debug_dump_decoder_case(self, pairs, path: str) -> None:
        """Inputs of a decoder call (per item: state row + W / W_acc, memory, processed memory,
        counters) -> npz, replayable with debug_load_decoder_case on any engine."""
        arrs: dict = {"n": np.array(len(pairs))}
        for i, (st, enc) in enumerate(pairs):
            req = st.req
            arrs[f"state{i}"] = self._read(st.buf.off, self.state_size(req.seq_len))
            arrs[f"mem{i}"] = np.asarray(self.read_features(req))
            arrs[f"pm{i}"] = self.read_processed_memory(req)
            arrs[f"cnt{i}"] = np.array([st.frames_emitted, st.target_frames, req.seq_len])
        np.savez(path, **arrs)

    @_on_device
    def debug_load_decoder_case(self, path: str) -> list:
        """(state, features) handles holding exactly the dumped inputs."""
        from .frontend import FrontendOutput
        z = np.load(path)
        n = int(z["n"])
        Ls = [int(z[f"cnt{i}"][2]) for i in range(n)]
        fos = [FrontendOutput((1,) * L, (1,) * L, (0,) * L, (0,) * L, (0,) * L) for L in Ls]
        encs = self.encoder_batch(fos)
        self.stream.synchronize()
        pairs = []
        t = self.arena.tensor
        for i, (enc, st) in enumerate(encs):
            req = enc.req
            put = lambda off, arr: t[off:off + arr.size].copy_(torch.from_numpy(np.ascontiguousarray(arr.reshape(-1))))
            put(st.buf.off, z[f"state{i}"])
            put(req.extra["mem_off"], z[f"mem{i}"])
            put(req.extra["pm_off"], z[f"pm{i}"])
            fe, tf, _ = (int(v) for v in z[f"cnt{i}"])
            pairs.append((DeviceDecoderState(req, st.buf, fe, tf), enc))
        torch.cuda.synchronize(self.device)
        return pairs

    def _mrf_branches(self, s: int, XA, OA_next, scratch, outs, rm, slope_out: float) -> None:
        """One MRF stage: the three ResBlock1 branches each write their own y (last layer in
        ACC_STORE mode), then one merge pass writes lrelu((y0 + y1 + y2) / 3).  With mrf_streams,
        branches 1 and 2 run on side streams concurrently with branch 0 (same arithmetic): at small
        pooled batches a layer fills only part of the GPU, so the stage's critical path drops from
        9 layers to 3 plus the merge."""
        main = self.stream
        ev_x, ev_1, ev_2 = self._ev
        if self.mrf_streams:
            ev_x.record(main)
        for j, layers in enumerate(self.res[s]):
            ya, tb = scratch[j]
            st = main if j == 0 or not self.mrf_streams else self._side[j - 1]
            if st is not main:
                st.wait_event(ev_x)
            (c1a, c2a), (c1b, c2b), (c1c, c2c) = layers
            self._resblock(XA, c1a, c2a, W.HG_RES_DILATIONS[0], rm, stream=st, act_out=ya, slope=0.1)
            self._resblock(ya, c1b, c2b, W.HG_RES_DILATIONS[1], rm, stream=st, act_out=tb, slope=0.1)
            self._resblock(tb, c1c, c2c, W.HG_RES_DILATIONS[2], rm, stream=st, acc=outs[j],
                           acc_mode=tc.ACC_STORE, slope=0.0)
            if st is not main:
                (ev_1, ev_2)[j - 1].record(st)
        if self.mrf_streams:
            main.wait_event(ev_1)
            main.wait_event(ev_2)
        self._call("itts_r_mrf_combine", outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(),
                   outs[0].numel(), slope_out, OA_next.data_ptr(), self._st())

    def _hifigan(self, Ts: list[int], lay0: _Layout, d_mplan: torch.Tensor) -> torch.Tensor:
        """HiFi-GAN V1 over a packed batch of spliced chunks -> stage-4 bf16 act (lrelu 0.01 applied)."""
        dev, st, n = self.device, self._st(), len(Ts)
        if self.native_vocoder and self.fused_mrf:
            x4 = ctypes.c_void_p()
            frames = np.ascontiguousarray(Ts, np.int32)   # must outlive the call (raw pointer below)
            self._call("itts_r_voc_run", self._voc, n, frames.ctypes.data, d_mplan.data_ptr(),
                       int(self.mrf_streams), ctypes.byref(x4), st)
            self.launches += 55   # row maps, mel assembly, conv_pre, 4 x (convT, 9 ResBlock layers, merge), 1 halo pass
            return x4.value
        with torch.cuda.stream(self.stream):
            x0 = self._buf("x0", lay0.total * 128, zero=True).view(lay0.total, 128)
        self._call("itts_r_mel_assemble", d_mplan.data_ptr(), n, max(Ts), x0.data_ptr(), 128, st)
        rm0 = self._rowmap(lay0, lay0.first, 1, "rm0")
        act_in = self._buf("act_in", lay0.total * 512).view(lay0.total, 512)
        self._conv(x0, self.conv_pre, 512, rm0, act_out=act_in, slope=0.1)
        prev, mult, layouts = lay0, 1, []
        for u in UPS:
            mult *= u
            layouts.append(_Layout([T * mult for T in Ts], MRF_HALO))
        biggest = max(l.total * c for l, c in zip(layouts, STAGE_C))
        # bf16 only: the residual stream is kept as lrelu(y, 0.1) and inverted on load
        # xa ya tb acc oa oa' (+ ya/tb/y of MRF branches 1 and 2 in the fused path)
        b16 = [self._buf(f"b16_{i}", biggest) for i in range(12 if self.fused_mrf else 6)]
        for s, (u, lay) in enumerate(zip(UPS, layouts)):
            C = STAGE_C[s]
            view = lambda t: t[:lay.total * C].view(lay.total, C)
            XA, YA, TB, ACC = (view(t) for t in b16[:4])
            OA_next = view(b16[4 + s % 2])
            # transposed conv: each input row of the previous stage -> u output rows
            rmT = self._rowmap(prev, lay.first, u, f"rmT{s}")
            self._conv(act_in, self.ups[s], C, rmT, act_out=XA, slope=0.1, zero_halo=False)
            zplan = np.stack([lay.base, np.array(lay.rows, np.int64), np.full(n, lay.halo, np.int64)], 1)
            self._call("itts_r_zero_halo", self._up(zplan).data_ptr(), n, lay.halo, XA.data_ptr(), C, st)
            rm = self._rowmap(lay, lay.first, 1, f"rm_s{s}")
            slope_out = 0.1 if s < 3 else 0.01
            if self.fused_mrf:
                self._mrf_branches(s, XA, OA_next, [(YA, TB)] + [(view(b16[6 + 2 * j]), view(b16[7 + 2 * j]))
                                                                 for j in range(2)],
                                   [ACC, view(b16[10]), view(b16[11])], rm, slope_out)
                prev, act_in = lay, OA_next
                continue
            for j, layers in enumerate(self.res[s]):
                for m, (c1, c2) in enumerate(layers):
                    ya_in = XA if m == 0 else YA
                    self._conv(ya_in, c1, C, rm, act_out=TB, slope=0.1)
                    if m < 2:
                        self._conv(TB, c2, C, rm, res_in=ya_in, res_slope=0.1, act_out=YA, slope=0.1)
                    else:
                        mode = (tc.ACC_STORE, tc.ACC_ADD, tc.ACC_FINAL)[j]
                        self._conv(TB, c2, C, rm, res_in=YA, res_slope=0.1, acc=ACC, acc_mode=mode,
                                   act_out=OA_next if j == 2 else None, slope=slope_out)
            prev, act_in = lay, OA_next
        return act_in

    def _claim_voc(self, triples, lasts, taken) -> list:
        """(owning request, next vocoder-state buffer or None) per item; allocates up front."""
        owners = []
        for (vstate, mel, _), last in zip(triples, lasts):
            req = mel.req if isinstance(mel, DeviceMelChunk) else None
            if req is None:
                req = vstate.req if isinstance(vstate, DeviceVocoderState) else DeviceRequest(self, 0)
            owners.append((req, None if last else req.claim(req.voc_bufs, self.voc_size(), taken)))
        return owners

    # ------------------------------------------------------------ lazy reads (tests/debug)
    def _read(self, off: int, size: int) -> np.ndarray:
        self.stream.synchronize()
        return self.arena.tensor[off:off + size].to("cpu").numpy().copy()

    def read_features(self, req) -> np.ndarray:
        arr = self._read(req.extra["mem_off"], req.seq_len * W.EMB).reshape(req.seq_len, W.EMB)
        arr.setflags(write=False)
        return arr

    def read_processed_memory(self, req) -> np.ndarray:
        return self._read(req.extra["pm_off"], req.seq_len * W.ATT_DIM).reshape(req.seq_len, W.ATT_DIM)

    def read_state(self, req, buf) -> dict:
        L = req.seq_len
        raw = self._read(buf.off, self.state_size(L))
        out = {"last_frame": raw[LAST_OFF:LAST_OFF + 80], "attn_context": raw[CTX_OFF:CTX_OFF + 512],
               "attn_hidden": raw[ATTH_OFF:ATTH_OFF + 1024], "attn_cell": raw[ATTC_OFF:ATTC_OFF + 1024],
               "dec_hidden": raw[DECH_OFF:DECH_OFF + 1024], "dec_cell": raw[DECC_OFF:DECC_OFF + 1024],
               "attn_weights": raw[ROW:ROW + L], "attn_weights_sum": raw[ROW + L:ROW + 2 * L]}
        for v in out.values():
            v.setflags(write=False)
        return out

    def read_voc_state(self, req, buf):
        O = self.cfg.overlap_frames
        raw = self._read(buf.off, self.voc_size())
        return raw[:O * W.N_MEL].reshape(O, W.N_MEL), raw[O * W.N_MEL:]


class _ScratchPool:
    """Decoder scratch shared by every graph bucket of an engine: one flat buffer per name, sized
    for the largest bucket.  Decoder calls are serialised on the engine stream, so the buckets'
    captured graphs can all address the same memory (~0.4 GB at 512 rows, instead of per-bucket
    copies summing to several GB); a bucket's buffer is a view of the first numel elements."""

    def __init__(self, dev, poison):
        self.dev, self.poison, self.flat = dev, poison, {}

    def get(self, name: str, shape, dtype, max_numel: int) -> torch.Tensor:
        numel = int(np.prod(shape))
        t = self.flat.get(name)
        if t is None:
            t = torch.empty(max_numel, dtype=dtype, device=self.dev)
            if self.poison is True or (bool(self.poison) and name in self.poison):
                t.fill_(self.poison[name] if isinstance(self.poison, dict) else float("nan"))
            elif name == "xb2":
                t.zero_()
            self.flat[name] = t
        assert t.dtype == dtype and numel <= t.numel(), (name, shape)
        return t[:numel].view(shape)


class _DecBuffers:
    """Work buffers of one decoder call (n pooled rows); `packed` = plan | src ptrs | dst ptrs."""

    def __init__(self, eng: TierREngine, n: int, packed: torch.Tensor, pool: "_ScratchPool | None" = None):
        dev = eng.device
        self.dev = dev
        self.n = n
        self.packed = packed
        self.pool = pool
        self.d_plan, self.d_src, self.d_dst = packed[:8 * n], packed[8 * n:9 * n], packed[9 * n:10 * n]
        # scratch is never read before the kernels write it: eng.poison_scratch fills it with NaN
        # (debug / tests: the outputs must not change)
        self.poison = getattr(eng, "poison_scratch", False)
        self.work = self._empty((n, ROW), torch.float32, "work")
        self.xbm = self._empty((n, XB_ROW), torch.bfloat16, "xbm")
        self.G = self._empty((DEC_KSPLIT, n, 4096), torch.float32, "G")
        # query / projection partials: 8 K-slices (per-kernel chain) or 32 unit groups (+1 context
        # projection) in the persistent decoder
        self.Q = self._empty((32, n, 128), torch.float32, "Q")
        self.P = self._empty((33, n, 81), torch.float32, "P")
        self.H1 = self._empty((n, 256), torch.float32, "H1")
        self.dev, self.xb2, self.U, self.AP, self.bar, self.Gp = dev, None, None, None, None, None
        self.split = False

    def _poisoned(self, name: str) -> bool:
        return self.poison is True or (bool(self.poison) and name in self.poison)

    # per-row element counts of the scratch buffers at the pool's row limit
    _POOL_ROWS = PERSIST_MAX_B

    def _empty(self, shape, dtype, name: str) -> torch.Tensor:
        if self.pool is not None:   # a view of the engine-wide pool, sized for _POOL_ROWS rows
            numel = int(np.prod(shape))
            return self.pool.get(name, shape, dtype, numel // self.n * self._POOL_ROWS + 4096)
        t = torch.empty(shape, dtype=dtype, device=self.dev)
        if self._poisoned(name):   # True / a set: NaN; a dict: that buffer's fill value
            t.fill_(self.poison[name] if isinstance(self.poison, dict) else float("nan"))
        return t

    def ensure_persistent(self, max_L: int, split: bool = False) -> None:
        """Scratch of the persistent decoder kernel (allocated once per buffer set); the split-bf16
        mode keeps a second (low-part) operand mirror after the first."""
        if self.U is not None and self.U.shape[1] >= max_L and self.split == split:
            return
        self.split = split
        nblk = -(-self.n // 128)
        if self.pool is not None:   # pool views: sized for the largest bucket and the split layout
            self.xb2 = self.pool.get("xb2", (2 * nblk * (XB2 // 64) * 128 * 64,), torch.bfloat16,
                                     2 * (-(-self._POOL_ROWS // 128)) * (XB2 // 64) * 128 * 64)
            self.U = self.pool.get("U", (self.n, GRAPH_MAX_L), torch.float32, self._POOL_ROWS * GRAPH_MAX_L)
            self.AP = self.pool.get("AP", (self.n, 256, 2 + 512), torch.float32, self._POOL_ROWS * 256 * 514)
            self.bar = self.pool.get("bar", (DEC_BAR_WORDS,), torch.int32, DEC_BAR_WORDS)
            self.Gp = self.pool.get("Gp", (4 * 32 * (-(-self.n // 16) * 16) * 128,), torch.float32,
                                    4 * 32 * self._POOL_ROWS * 128)
            return
        self.xb2 = self._empty(((2 if split else 1) * nblk * (XB2 // 64) * 128 * 64,), torch.bfloat16, "xb2")
        if not self._poisoned("xb2"):
            self.xb2.zero_()
        self.U = self._empty((self.n, max(max_L, 256)), torch.float32, "U")
        self.AP = self._empty((self.n, 256, 2 + 512), torch.float32, "AP")
        self.bar = torch.zeros(DEC_BAR_WORDS, dtype=torch.int32, device=self.dev)
        self.Gp = self._empty((4 * 32 * (-(-self.n // 16) * 16) * 128,), torch.float32, "Gp")


class _DecBucket(_DecBuffers):
    """Fixed-address buffers + a CUDA graph of the full 32-step decoder chunk for <= B rows.

    Rows beyond the call's batch decode nothing (steps 0), gather a zero row
    and scatter into a private sink, so one graph serves every n <= B.
    """

    def __init__(self, eng: TierREngine, B: int, L: int):
        dev = eng.device
        if getattr(eng, "_scratch_pool", None) is None:
            eng._scratch_pool = _ScratchPool(dev, getattr(eng, "poison_scratch", False))
        super().__init__(eng, B, torch.empty(10 * B, dtype=torch.int64, device=dev), eng._scratch_pool)
        self.B, self.L = B, L
        C = eng.cfg.chunk_frames
        self.mel = self._empty((B, C, W.N_MEL), torch.float32, "bucket_mel")   # pool views (read right
        self.gate = self._empty((B, C), torch.float32, "bucket_gate")          # after each replay)
        self.zero_row = torch.zeros(ROW, dtype=torch.float32, device=dev)
        self.sink = self._empty((B, ROW), torch.float32, "sink")
        self.graph = None
        self.launches = 0
        # pinned staging of the packed plan [B][8] | src [B] | dst [B]: the per-call H2D source.
        # The idle template (rows decode nothing, gather the zero row, scatter into the sink) is
        # restored row by row, so a call only writes its own n rows.
        self.host = torch.empty(10 * B, dtype=torch.int64, pin_memory=True)
        self.host_np = self.host.numpy()
        self.template = np.concatenate([np.zeros(8 * B, np.int64), np.full(B, self.zero_row.data_ptr(), np.int64),
                                        self.sink.data_ptr() + 4 * ROW * np.arange(B, dtype=np.int64)])
        self.template[:8 * B].reshape(B, 8)[:, 6] = self.mel.data_ptr() + 4 * W.N_MEL * C * np.arange(B, dtype=np.int64)
        self.template[:8 * B].reshape(B, 8)[:, 7] = self.gate.data_ptr() + 4 * C * np.arange(B, dtype=np.int64)
        self.host_np[:] = self.template
        self.dirty = 0   # rows of host_np holding a previous call's plan
        self.copied = torch.cuda.Event()   # the last H2D out of `host` (reuse waits for it)
        self.pending = False

    def idle_plan(self) -> None:
        """Every row decodes nothing, gathers the zero row and scatters into its own sink."""
        B = self.B
        host = np.concatenate([np.zeros(8 * B, np.int64), np.full(B, self.zero_row.data_ptr(), np.int64),
                               self.sink.data_ptr() + 4 * ROW * np.arange(B, dtype=np.int64)])
        self.packed.copy_(torch.from_numpy(host))

    def capture(self, eng: TierREngine) -> None:
        C = eng.cfg.chunk_frames
        if not eng._graph_warm:  # one eager pass per engine sets kernel attributes before any capture
            eng._enqueue_decoder(self, self.L, C)
            eng._graph_warm = True
        g = torch.cuda.CUDAGraph()
        before = eng.launches
        with torch.cuda.graph(g, stream=eng.stream):
            eng._enqueue_decoder(self, self.L, C)
        self.launches = eng.launches - before
        eng.launches = before
        self.graph = g
