"""TEST INFRASTRUCTURE ONLY -- torch-CPU fp32 oracle for Tier R (Tacotron2 + HiFi-GAN V1).

The reference contains no neural networks (``SPEC.md:8``),
so this oracle is the builder's own restatement of the public Tacotron2 /
HiFi-GAN V1 forward passes wired into the reference's
chunk semantics (Appendix A):

* ``encode`` -- paper Eq. 1: 4 summed embeddings -> 3 x (conv5 + folded BN +
  ReLU) -> BiLSTM (each direction starts at the request's true end) ->
  memory, processed memory.
* ``decoder_step`` -- paper Eq. 2 / Tacotron2 ``Decoder.decode``: prenet ->
  attention LSTMCell -> location-sensitive attention -> W_acc += W ->
  decoder LSTMCell -> mel/gate projection.  Stop is the reference's frame
  counter (``acoustic.py:174-175``); the gate logit is returned, not used.
* ``hifigan`` -- HiFi-GAN V1 generator on one spliced chunk with zero
  'same' padding at both chunk edges; ``vocode_chunk`` reuses the Tier-S
  splice (``oracle.tier_s.vocode_chunk``, reference ``vocoder.py:92-136``).

Parity: **unpinned by the reference** (nothing to pin against); the GPU is
checked against this oracle at mel max-abs <= 1e-3 and waveform SNR >= 40 dB.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from paper_2211_13939_b200 import weights as W

from . import tier_s


def _lstm_cell(x, h, c, w, prefix):
    gates = x @ w[prefix + ".w_ih"].T + w[prefix + ".b_ih"] + h @ w[prefix + ".w_hh"].T + w[prefix + ".b_hh"]
    i, f, g, o = gates.chunk(4, dim=-1)
    c = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(g)
    return torch.sigmoid(o) * torch.tanh(c), c


@torch.no_grad()
def encode(w, phonemes, pw, pph, iph):
    """-> (memory [L, 512], processed memory [L, 128])."""
    ids = [torch.as_tensor(np.asarray(v, dtype=np.int64)) for v in (phonemes, pw, pph, iph)]
    x = (w["emb.phoneme"][ids[0]] + w["emb.pw"][ids[1]] + w["emb.pph"][ids[2]] + w["emb.iph"][ids[3]])
    x = x.T.unsqueeze(0)  # [1, 512, L]
    for i in range(3):
        x = F.relu(F.conv1d(x, w[f"enc.conv{i}.w"], w[f"enc.conv{i}.b"], padding=2))
    x = x[0].T  # [L, 512]
    L = x.shape[0]
    outs = []
    for prefix, order in (("enc.lstm_fwd", range(L)), ("enc.lstm_bwd", range(L - 1, -1, -1))):
        h = torch.zeros(W.ENC_LSTM)
        c = torch.zeros(W.ENC_LSTM)
        out = torch.empty(L, W.ENC_LSTM)
        pre = x @ w[prefix + ".w_ih"].T + w[prefix + ".b_ih"] + w[prefix + ".b_hh"]
        for t in order:
            gates = pre[t] + h @ w[prefix + ".w_hh"].T
            i, f, g, o = gates.chunk(4)
            c = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(g)
            h = torch.sigmoid(o) * torch.tanh(c)
            out[t] = h
        outs.append(out)
    memory = torch.cat(outs, dim=1)
    return memory, memory @ w["att.memory_layer"].T


@dataclass
class RState:
    last_frame: torch.Tensor   # [80]
    context: torch.Tensor      # [512]
    att_h: torch.Tensor
    att_c: torch.Tensor
    dec_h: torch.Tensor
    dec_c: torch.Tensor
    weights: torch.Tensor      # [L]
    weights_cum: torch.Tensor  # [L]
    frames_emitted: int
    target_frames: int


def init_state(L: int, frames_per_phoneme: int) -> RState:
    z = torch.zeros
    return RState(z(W.N_MEL), z(W.EMB), z(W.ATT_RNN), z(W.ATT_RNN), z(W.DEC_RNN), z(W.DEC_RNN),
                  z(L), z(L), 0, frames_per_phoneme * L)


@torch.no_grad()
def decoder_step(w, s: RState, memory, pmem):
    """One frame; returns (mel [80], gate_logit, new state)."""
    p = F.relu(s.last_frame @ w["prenet.0"].T)
    p = F.relu(p @ w["prenet.1"].T)
    att_h, att_c = _lstm_cell(torch.cat([p, s.context]), s.att_h, s.att_c, w, "att_rnn")
    q = att_h @ w["att.query_layer"].T                                     # [128]
    loc = F.conv1d(torch.stack([s.weights, s.weights_cum]).unsqueeze(0), w["att.location_conv"],
                   padding=(W.LOC_KERNEL - 1) // 2)[0]                      # [32, L]
    loc = loc.T @ w["att.location_dense"].T                                 # [L, 128]
    e = torch.tanh(q + loc + pmem) @ w["att.v"][0]                          # [L]
    a = torch.softmax(e, dim=0)
    ctx = a @ memory                                                        # [512]
    dec_h, dec_c = _lstm_cell(torch.cat([att_h, ctx]), s.dec_h, s.dec_c, w, "dec_rnn")
    hc = torch.cat([dec_h, ctx])
    mel = hc @ w["proj.w"].T + w["proj.b"]
    gate = float(hc @ w["gate.w"][0] + w["gate.b"][0])
    n = s.frames_emitted + 1
    return mel, gate, RState(mel, ctx, att_h, att_c, dec_h, dec_c, a, s.weights_cum + a, n,
                             s.target_frames)


def decode_chunk(w, s: RState, memory, pmem, chunk_frames: int):
    """<= C steps, counter stop (reference ``acoustic.py:204-219``); -> (mel [m,80], stop, state, gates)."""
    if s.frames_emitted >= s.target_frames:
        raise ValueError("decode past stop")
    frames, gates = [], []
    for _ in range(chunk_frames):
        mel, gate, s = decoder_step(w, s, memory, pmem)
        frames.append(mel)
        gates.append(gate)
        if s.frames_emitted >= s.target_frames:
            return torch.stack(frames), True, s, gates
    return torch.stack(frames), False, s, gates


def postnet(pw, mel: np.ndarray | torch.Tensor) -> np.ndarray:
    """Chunk-local Tacotron2 PostNet: mel + PostNet(mel), 'same' zero padding at
    the chunk edges; 5 x conv k5 with tanh after the first four (batch norm folded into the
    weights of ``weights.postnet_weights``).  fp32 torch on the CPU."""
    x = torch.as_tensor(np.asarray(mel, np.float32)).T[None]          # [1][80][T]
    y = x
    for i in range(W.POSTNET_LAYERS):
        y = F.conv1d(y, pw[f"post.conv{i}.w"], pw[f"post.conv{i}.b"], padding=W.POSTNET_K // 2)
        if i < W.POSTNET_LAYERS - 1:
            y = torch.tanh(y)
    return (x + y)[0].T.numpy().astype(np.float64)


def _pad(k: int, d: int) -> int:
    return (k * d - d) // 2


@torch.no_grad()
def hifigan(w, mel: np.ndarray | torch.Tensor, hop: int = 256) -> np.ndarray:
    """HiFi-GAN V1 on one chunk: mel [T, 80] -> samples [T*256] (float64 array)."""
    assert hop == 256
    x = torch.as_tensor(np.asarray(mel, dtype=np.float32)).T.unsqueeze(0)  # [1, 80, T]
    x = F.conv1d(x, w["hg.conv_pre.w"], w["hg.conv_pre.b"], padding=3)
    for i, (u, k) in enumerate(zip(W.HG_UP_RATES, W.HG_UP_KERNELS)):
        x = F.leaky_relu(x, 0.1)
        x = F.conv_transpose1d(x, w[f"hg.up{i}.w"], w[f"hg.up{i}.b"], stride=u, padding=(k - u) // 2)
        acc = None
        for j, kr in enumerate(W.HG_RES_KERNELS):
            y = x
            for m, dil in enumerate(W.HG_RES_DILATIONS):
                key = f"hg.res{i}.{j}"
                t = F.leaky_relu(y, 0.1)
                t = F.conv1d(t, w[f"{key}.c1{m}.w"], w[f"{key}.c1{m}.b"], dilation=dil, padding=_pad(kr, dil))
                t = F.leaky_relu(t, 0.1)
                t = F.conv1d(t, w[f"{key}.c2{m}.w"], w[f"{key}.c2{m}.b"], padding=_pad(kr, 1))
                y = y + t
            acc = y if acc is None else acc + y
        x = acc / 3.0
    x = F.leaky_relu(x)  # default slope 0.01
    x = torch.tanh(F.conv1d(x, w["hg.conv_post.w"], w["hg.conv_post.b"], padding=3))
    return x[0, 0].double().numpy()


def vocode_chunk(w, state, mel, is_last, overlap_frames, hop=256):
    return tier_s.vocode_chunk(state, np.asarray(mel, dtype=np.float64), is_last, overlap_frames, hop,
                               gen=lambda m, h: hifigan(w, m, h))


def synthesize(w, phonemes, pw, pph, iph, *, frames_per_phoneme=8, chunk_frames=32,
               overlap_frames=4, hop=256, max_chunks=None):
    """Single-request incremental synthesis -> (list of (samples, offset), mel [F, 80], gates)."""
    memory, pmem = encode(w, phonemes, pw, pph, iph)
    s = init_state(memory.shape[0], frames_per_phoneme)
    v = tier_s.VocState(None, None, 0)
    chunks, mels, gates = [], [], []
    while True:
        mel, stop, s, g = decode_chunk(w, s, memory, pmem, chunk_frames)
        mels.append(mel)
        gates += g
        samples, off, v = vocode_chunk(w, v, mel.numpy(), stop, overlap_frames, hop)
        chunks.append((samples, off))
        if stop or (max_chunks is not None and len(chunks) >= max_chunks):
            return chunks, torch.cat(mels).numpy(), np.array(gates)


def snr_db(ref: np.ndarray, got: np.ndarray) -> float:
    noise = float(np.sum((np.asarray(ref, np.float64) - np.asarray(got, np.float64)) ** 2))
    sig = float(np.sum(np.asarray(ref, np.float64) ** 2))
    return float("inf") if noise == 0 else 10.0 * np.log10(sig / noise)
