"""GPU BERT prosodic-structure frontend (the paper's frontend).

G2P stays the reference's forward maximum matching on the host (``frontend.g2p``); prosody comes
from a BERT-base encoder over the text's characters with three 2-way linear heads (pw, pph, iph),
run on the GPU for the whole pooled batch by ``itts_bert_prosody`` (``csrc/bert.cu``), then
regulated by the per-character phoneme counts exactly like the rule-based path
(``frontend.regulate``).  Opt-in (``build_modules(..., frontend="bert")``): the reference's default
is the rule ``predict_prosody`` (``src/frontend.py:174-188``) and the weights here are random-init,
so this changes WHICH prosody tokens are produced, not how the pipeline schedules them.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _native
from .frontend import FrontendOutput, Lexicon, g2p, regulate

HIDDEN, HEADS, FFN, LAYERS, MAX_POS, MAX_LEN = 768, 12, 3072, 12, 512, 256
PAD_ID, UNK_ID = 0, 1


def char_vocab(lexicon: Lexicon) -> dict[str, int]:
    """Characters of the lexicon's phrase table, ids from 2 (0 = pad, 1 = unknown)."""
    chars = sorted({ch for phrase in lexicon.phrase_to_pinyin for ch in phrase})
    return {ch: i + 2 for i, ch in enumerate(chars)}


def bert_weights(vocab_size: int, seed: int = 0) -> dict[str, torch.Tensor]:
    """BERT-base shaped random init (normal 0.02, zero biases, unit LayerNorm), fp32 on the CPU."""
    g = torch.Generator().manual_seed(seed + 104729)
    nrm = lambda *shape: torch.randn(*shape, generator=g, dtype=torch.float64).mul_(0.02).float()
    w = {"tok": nrm(vocab_size, HIDDEN), "pos": nrm(MAX_POS, HIDDEN),
         "ln.g": torch.ones(HIDDEN), "ln.b": torch.zeros(HIDDEN)}
    for l in range(LAYERS):
        p = f"l{l}."
        w[p + "qkv.w"], w[p + "qkv.b"] = nrm(3 * HIDDEN, HIDDEN), torch.zeros(3 * HIDDEN)
        w[p + "o.w"], w[p + "o.b"] = nrm(HIDDEN, HIDDEN), torch.zeros(HIDDEN)
        w[p + "ln1.g"], w[p + "ln1.b"] = torch.ones(HIDDEN), torch.zeros(HIDDEN)
        w[p + "ff1.w"], w[p + "ff1.b"] = nrm(FFN, HIDDEN), torch.zeros(FFN)
        w[p + "ff2.w"], w[p + "ff2.b"] = nrm(HIDDEN, FFN), torch.zeros(HIDDEN)
        w[p + "ln2.g"], w[p + "ln2.b"] = torch.ones(HIDDEN), torch.zeros(HIDDEN)
    w["heads.w"], w["heads.b"] = nrm(6, HIDDEN), torch.zeros(6)   # rows 2k, 2k+1: head k (pw, pph, iph)
    return w


class BertProsody:
    """The encoder's weights on the device and the native call over a batch of texts."""

    def __init__(self, lexicon: Lexicon, device="cuda", seed: int = 0, weights: dict | None = None):
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise RuntimeError("the BERT frontend runs on a CUDA device (no CPU fallback)")
        _native.lib()
        self.lexicon = lexicon
        self.vocab = char_vocab(lexicon)
        self.weights = weights if weights is not None else bert_weights(len(self.vocab) + 2, seed)
        d = self.device
        f32 = lambda t: t.detach().float().contiguous().to(d)
        lin = lambda t: t.detach().to(d).to(torch.bfloat16)[None].contiguous()   # tc layout [1 tap][N][K]
        w = self.weights
        keep = [f32(w["tok"]), f32(w["pos"]), f32(w["ln.g"]), f32(w["ln.b"])]
        for l in range(LAYERS):
            p = f"l{l}."
            keep += [lin(w[p + "qkv.w"]), f32(w[p + "qkv.b"]), lin(w[p + "o.w"]), f32(w[p + "o.b"]),
                     f32(w[p + "ln1.g"]), f32(w[p + "ln1.b"]), lin(w[p + "ff1.w"]), f32(w[p + "ff1.b"]),
                     lin(w[p + "ff2.w"]), f32(w[p + "ff2.b"]), f32(w[p + "ln2.g"]), f32(w[p + "ln2.b"])]
        keep += [f32(w["heads.w"]), f32(w["heads.b"])]
        self._keep = keep
        self._ptrs = (ctypes.c_int64 * len(keep))(*[t.data_ptr() for t in keep])
        self.stream = torch.cuda.Stream(d)
        self._bufs: dict = {}

    def _buf(self, name, numel, dtype):
        t = self._bufs.get(name)
        if t is None or t.numel() < numel:
            t = torch.empty(max(int(numel * 1.25), 1024), dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t[:numel]

    def ids(self, text: str) -> list[int]:
        return [self.vocab.get(ch, UNK_ID) for ch in text]

    def run(self, texts: list[str]) -> tuple[np.ndarray, np.ndarray, list[int]]:
        """(logits [rows][6], tokens [rows][3], per-text row offsets) for the packed characters."""
        lens = [len(t) for t in texts]
        if min(lens) < 1:
            raise ValueError("empty input")
        if max(lens) > MAX_LEN:
            raise ValueError(f"BERT frontend texts are limited to {MAX_LEN} characters")
        rows = sum(lens)
        first = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        ids = np.fromiter((i for t in texts for i in self.ids(t)), np.int32, rows)
        pos = np.concatenate([np.arange(L, dtype=np.int32) for L in lens])
        plan = np.stack([first, np.asarray(lens, np.int64)], 1)
        with torch.cuda.stream(self.stream):
            d_ids = torch.from_numpy(ids).to(self.device, non_blocking=False)
            d_pos = torch.from_numpy(pos).to(self.device, non_blocking=False)
            d_plan = torch.from_numpy(plan.reshape(-1)).to(self.device, non_blocking=False)
            iota = torch.arange(rows, dtype=torch.int32, device=self.device)
            xf = self._buf("xf", rows * HIDDEN, torch.float32)
            xb = self._buf("xb", rows * HIDDEN, torch.bfloat16)
            qkv = self._buf("qkv", rows * 3 * HIDDEN, torch.bfloat16)
            att = self._buf("att", rows * HIDDEN, torch.bfloat16)
            y = self._buf("y", rows * HIDDEN, torch.float32)
            h = self._buf("h", rows * FFN, torch.bfloat16)
            logits = self._buf("logits", rows * 6, torch.float32)
            tokens = self._buf("tokens", rows * 3, torch.int32)
            _native.call("itts_bert_prosody", d_ids.data_ptr(), d_pos.data_ptr(), d_plan.data_ptr(), len(texts),
                         rows, max(lens), self._ptrs, iota.data_ptr(), xf.data_ptr(), xb.data_ptr(), qkv.data_ptr(),
                         att.data_ptr(), y.data_ptr(), h.data_ptr(), logits.data_ptr(), tokens.data_ptr(),
                         self.stream.cuda_stream)
            lg = logits.view(rows, 6).to("cpu")
            tk = tokens.view(rows, 3).to("cpu")
        self.stream.synchronize()
        return lg.numpy(), tk.numpy(), first.tolist()

    def frontend_batch(self, texts: list[str]) -> list[FrontendOutput]:
        """The frontend module: G2P on the host, BERT prosody on the GPU, regulated per text."""
        texts = list(texts)
        for t in texts:
            if not t:
                raise ValueError("empty input")
        g2ps = [g2p(t, self.lexicon) for t in texts]
        _, tokens, first = self.run(texts)
        out = []
        for (phonemes, counts), t, r0 in zip(g2ps, texts, first):
            tk = tokens[r0:r0 + len(t)]
            pw, pph, iph = (tk[:, k].tolist() for k in range(3))
            out.append(FrontendOutput(tuple(phonemes), tuple(counts), tuple(regulate(pw, counts)),
                                      tuple(regulate(pph, counts)), tuple(regulate(iph, counts))))
        return out
