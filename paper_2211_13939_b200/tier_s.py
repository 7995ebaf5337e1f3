"""Tier S GPU modules: the reference stand-in models (fp64) behind PipelineModules.

Encoder, decoder and vocoder callables with exactly the reference's
signatures (``pkg/src/incrtts/scheduler.py:249-282``) whose arithmetic runs
in ``csrc/tier_s.cu`` through the C ABI.  Host work per call is O(batch):
validate handles, build one int64 plan, one H2D copy of the plan, one
launch; the vocoder adds one D2H copy of the packed audio.  Stop and chunk
lengths are counter-driven (``acoustic.py:174-175``) and therefore decided
on the host without a device round trip.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .audio import cached_curve
from .domain import AudioChunk, PipelineConfig, validate_config
from .handles import (DecodeChunkResult, DeviceDecoderState, DeviceEncodedFeatures, DeviceMelChunk,
                      DeviceRequest, DeviceVocoderState)
from .arena import RaggedArena


def _h2d(arr: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(arr)).pin_memory().to(device, non_blocking=True)


class TierSEngine:
    """Device state + launches for one GPU's Tier-S module set."""

    dtype = torch.float64

    def __init__(self, cfg: PipelineConfig, device: str | torch.device | None = None):
        self.cfg = validate_config(cfg)
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type != "cuda":
            raise RuntimeError("Tier-S GPU modules need a CUDA device (no CPU fallback)")
        _native.lib()  # fail loudly now if the extension is missing
        self.dim = cfg.feature_dim
        if self.dim not in (4, 8, 16, 32):
            raise ValueError(f"feature_dim {self.dim} unsupported by the GPU kernels (4/8/16/32)")
        self.stream = torch.cuda.Stream(self.device)
        with torch.cuda.stream(self.stream):
            self.arena = RaggedArena(self.dtype, self.device, 1 << 20, self.stream)
            curve = cached_curve(cfg.overlap_samples)
            self.fade = torch.from_numpy(np.concatenate([curve.fade_in, curve.fade_out])).to(self.device)
        self.launches = 0

    # ------------------------------------------------------------ sizes
    def state_size(self, L: int) -> int:
        return 6 * self.dim + 2 * L

    def voc_size(self) -> int:
        return self.cfg.overlap_frames * self.dim + self.cfg.overlap_samples

    # ------------------------------------------------------------ encoder
    def encoder_batch(self, fos) -> list:
        n = len(fos)
        if n == 0:
            return []
        lens = [fo.seq_len for fo in fos]
        if min(lens) < 1:
            raise ValueError("frontend output needs at least one phoneme")
        total = sum(lens)
        tok = np.empty((4, total), dtype=np.int32)
        pos = 0
        for fo, L in zip(fos, lens):
            tok[0, pos:pos + L] = fo.phonemes
            tok[1, pos:pos + L] = fo.pw
            tok[2, pos:pos + L] = fo.pph
            tok[3, pos:pos + L] = fo.iph
            pos += L
        reqs, plan = [], np.empty((n, 4), dtype=np.int64)
        pos = 0
        for i, L in enumerate(lens):
            req = DeviceRequest(self, L)
            feat_off = req.add_region(L * self.dim)
            req.extra["feat_off"] = feat_off
            buf = req.claim(req.state_bufs, self.state_size(L), set())
            reqs.append((req, buf))
            plan[i] = (pos, L, 0, 0)
            pos += L
        a = self.arena
        for i, (req, buf) in enumerate(reqs):
            plan[i, 2] = a.ptr(req.extra["feat_off"])
            plan[i, 3] = a.ptr(buf.off)
        with torch.cuda.stream(self.stream):
            d_tok, d_plan = _h2d(tok, self.device), _h2d(plan, self.device)
            scratch = torch.empty(2 * total * self.dim, dtype=self.dtype, device=self.device)
            _native.call("itts_s_encode", d_tok.data_ptr(), total, d_plan.data_ptr(), n, max(lens),
                         self.dim, scratch.data_ptr(), self.stream.cuda_stream)
        self.launches += 3
        fpp = self.cfg.frames_per_phoneme
        return [(DeviceEncodedFeatures(req), DeviceDecoderState(req, buf, 0, fpp * req.seq_len))
                for req, buf in reqs]

    # ------------------------------------------------------------ decoder
    def decoder_batch(self, pairs) -> list:
        n = len(pairs)
        if n == 0:
            return []
        C = self.cfg.chunk_frames
        steps, taken, dsts = [], set(), []
        for state, enc in pairs:
            if not isinstance(state, DeviceDecoderState) or not isinstance(enc, DeviceEncodedFeatures):
                raise TypeError("Tier-S GPU decoder needs handles produced by its own encoder")
            if state.req is not enc.req:
                raise ValueError("decoder state does not match encoded features")
            if state.frames_emitted >= state.target_frames:
                raise ValueError("decode past stop")
            steps.append(min(C, state.target_frames - state.frames_emitted))
        for state, _ in pairs:
            req = state.req
            dsts.append(req.claim(req.state_bufs, self.state_size(req.seq_len), taken))
        mel_off = np.concatenate([[0], np.cumsum(steps)]) * self.dim
        a = self.arena
        plan = np.empty((n, 6), dtype=np.int64)
        with torch.cuda.stream(self.stream):
            mel = torch.empty(int(mel_off[-1]), dtype=self.dtype, device=self.device)
            base = mel.data_ptr()
            for i, ((state, enc), dst) in enumerate(zip(pairs, dsts)):
                plan[i] = (a.ptr(enc.req.extra["feat_off"]), enc.seq_len, a.ptr(state.buf.off),
                           a.ptr(dst.off), steps[i], base + 8 * int(mel_off[i]))
            d_plan = _h2d(plan, self.device)
            _native.call("itts_s_decode_chunk", d_plan.data_ptr(), n, self.dim,
                         float(self.cfg.attention_penalty), self.stream.cuda_stream)
        self.launches += 1
        out = []
        for i, ((state, enc), dst) in enumerate(zip(pairs, dsts)):
            emitted = state.frames_emitted + steps[i]
            view = mel[int(mel_off[i]):int(mel_off[i + 1])].view(steps[i], self.dim)
            out.append(DecodeChunkResult(
                DeviceMelChunk(view, state.req), emitted >= state.target_frames,
                DeviceDecoderState(state.req, dst, emitted, state.target_frames)))
        return out

    # ------------------------------------------------------------ vocoder
    def vocoder_batch(self, triples) -> list:
        n = len(triples)
        if n == 0:
            return []
        cfg, O, H, S = self.cfg, self.cfg.overlap_frames, self.cfg.hop_samples, self.cfg.overlap_samples
        host_mels, metas = [], []
        for vstate, mel, is_last in triples:
            m = int(mel.frame_count)
            if not is_last and m < O:
                raise ValueError("non-final chunk shorter than the overlap window")
            has_tail = (vstate.has_tail if isinstance(vstate, DeviceVocoderState)
                        else vstate.mel_tail is not None)
            if not has_tail and not is_last and m * H <= S:
                raise ValueError("non-final chunk shorter than the overlap window")
            if not isinstance(mel, DeviceMelChunk):
                frames = np.asarray(mel.frames, dtype=np.float64)
                if frames.ndim != 2 or frames.shape[1] != self.dim:
                    raise ValueError("mel chunk width does not match feature_dim")
                host_mels.append(frames)
            elif mel.data.shape[1] != self.dim:
                raise ValueError("mel chunk width does not match feature_dim")
            G = ((O if has_tail else 0) + m) * H
            metas.append((m, has_tail, bool(is_last), G if is_last else G - S))
        counts = [mt[3] for mt in metas]
        out_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        plan = np.zeros((n, 7), dtype=np.int64)
        a = self.arena
        results_state = []
        keep = []  # temporaries that must outlive the launch
        taken = set()
        with torch.cuda.stream(self.stream):
            if host_mels:
                hm = _h2d(np.concatenate([f.reshape(-1) for f in host_mels]), self.device)
                keep.append(hm)
            hpos = 0
            owners = self._claim_voc(triples, [mt[2] for mt in metas], taken)  # before any a.ptr()
            for i, ((vstate, mel, is_last), (m, has_tail, last, cnt)) in enumerate(zip(triples, metas)):
                req, dst = owners[i]
                if isinstance(mel, DeviceMelChunk):
                    mel_ptr = mel.data.data_ptr()
                else:
                    mel_ptr = hm.data_ptr() + 8 * hpos
                    hpos += m * self.dim
                src_ptr = 0
                if has_tail:
                    if isinstance(vstate, DeviceVocoderState):
                        src_ptr = a.ptr(vstate.buf.off)
                    else:  # host VocoderState with tails: upload once
                        t = _h2d(np.concatenate([np.asarray(vstate.mel_tail, np.float64).reshape(-1),
                                                 np.asarray(vstate.held_tail, np.float64).reshape(-1)]),
                                 self.device)
                        keep.append(t)
                        src_ptr = t.data_ptr()
                plan[i] = (mel_ptr, m, int(has_tail) | (2 * int(last)), src_ptr,
                           0 if dst is None else a.ptr(dst.off), out_off[i], 0)
                results_state.append((req, dst, int(vstate.emitted_samples)))
            d_plan = _h2d(plan, self.device)
            audio = torch.empty(max(int(out_off[-1]), 1), dtype=self.dtype, device=self.device)
            max_g = max(((O if mt[1] else 0) + mt[0]) * H for mt in metas)
            _native.call("itts_s_vocode_chunk", d_plan.data_ptr(), n, self.dim, O, H, max_g,
                         self.fade.data_ptr(), audio.data_ptr(), self.stream.cuda_stream)
            host = torch.empty(audio.numel(), dtype=self.dtype, pin_memory=True)
            host.copy_(audio, non_blocking=True)
        self.launches += 1
        self.stream.synchronize()
        flat = host.numpy()
        if not np.isfinite(flat[:out_off[-1]]).all():
            raise ValueError("array contains non-finite values")
        out = []
        for i, (req, dst, emitted) in enumerate(results_state):
            samples = flat[out_off[i]:out_off[i + 1]]
            out.append((AudioChunk.trusted(samples, emitted),
                        DeviceVocoderState(req, dst, emitted + counts[i])))
        return out

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
        arr = self._read(req.extra["feat_off"], req.seq_len * self.dim).reshape(req.seq_len, self.dim)
        arr.setflags(write=False)
        return arr

    def read_state(self, req, buf) -> dict:
        D, L = self.dim, req.seq_len
        raw = self._read(buf.off, self.state_size(L))
        names = ("last_frame", "attn_context", "attn_hidden", "attn_cell", "dec_hidden", "dec_cell")
        out = {k: raw[j * D:(j + 1) * D] for j, k in enumerate(names)}
        out["attn_weights"] = raw[6 * D:6 * D + L]
        out["attn_weights_sum"] = raw[6 * D + L:6 * D + 2 * L]
        for v in out.values():
            v.setflags(write=False)
        return out

    def read_voc_state(self, req, buf):
        O, D = self.cfg.overlap_frames, self.dim
        raw = self._read(buf.off, self.voc_size())
        return raw[:O * D].reshape(O, D), raw[O * D:]
