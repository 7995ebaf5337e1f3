"""Seeded random-init weights for Tier R: Tacotron2 (512 enc, 1024 LSTM) + HiFi-GAN V1.

Not in the reference (it has no networks, ``SPEC.md:8``); the shapes follow
the public Tacotron2 / HiFi-GAN V1 definitions as restated in SURVEY
Appendix B.  Inference-time simplifications, all exact:

* encoder BatchNorm folded into the conv (random-init BN: gamma 1, beta 0,
  mean 0, var 1, eps 1e-5);
* HiFi-GAN weight-norm removed (at init ``g = ||v||`` so ``w = v``);
* prenet dropout off.

Initialisation mirrors the originals: Tacotron2 xavier-uniform with the
layer's gain (``LinearNorm`` / ``ConvNorm``), uniform(+-1/sqrt(H)) for the
LSTMs, the Tacotron2 embedding range; HiFi-GAN ``init_weights`` normal(0,
0.01) for ups / resblocks / conv_post, default conv init for conv_pre.
Every tensor is drawn from one ``torch.Generator(seed)`` in a fixed order,
so the CPU oracle and every GPU process see identical float32 values.

By default every parameter is then rounded to the nearest bfloat16 (kept as
float32): the weights are those of a bf16 checkpoint, the storage format of a
served model.  The oracle computes with exactly these values in fp32; the GPU
parity mode then needs no low-order weight parts (gate products Wh.(Xh + Xl),
fp32 accumulation) and streams half the weight bytes.  ``bf16_grid=False``
gives the unrounded float32 draw (the GPU parity mode then splits the weights
too: Wh.Xh + Wh.Xl + Wl.Xh).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

N_SYMBOLS = 148          # Tacotron2 symbol table size; the bundled lexicon uses ids < 61
EMB = 512                # encoder embedding / conv channels
ENC_LSTM = 256           # per direction
ATT_RNN = 1024
DEC_RNN = 1024
PRENET = 256
ATT_DIM = 128
LOC_FILTERS = 32
LOC_KERNEL = 31
N_MEL = 80
HG_UP_RATES = (8, 8, 2, 2)
HG_UP_KERNELS = (16, 16, 4, 4)
HG_CH0 = 512
HG_RES_KERNELS = (3, 7, 11)
HG_RES_DILATIONS = (1, 3, 5)
BN_EPS = 1e-5


@dataclass(frozen=True)
class TierRShapes:
    n_mel: int = N_MEL
    emb: int = EMB
    att_rnn: int = ATT_RNN
    dec_rnn: int = DEC_RNN
    prenet: int = PRENET
    att_dim: int = ATT_DIM
    hop: int = 256


def _gain(kind: str) -> float:
    return {"linear": 1.0, "relu": math.sqrt(2.0), "tanh": 5.0 / 3.0, "sigmoid": 1.0}[kind]


class _Draw:
    def __init__(self, seed: int):
        self.g = torch.Generator().manual_seed(seed)

    def uniform(self, shape, bound: float) -> torch.Tensor:
        return (torch.rand(shape, generator=self.g, dtype=torch.float64) * 2 - 1).mul_(bound).float()

    def normal(self, shape, std: float) -> torch.Tensor:
        return torch.randn(shape, generator=self.g, dtype=torch.float64).mul_(std).float()

    def xavier(self, shape, gain: str) -> torch.Tensor:
        rf = 1
        for s in shape[2:]:
            rf *= s
        fan_in, fan_out = shape[1] * rf, shape[0] * rf
        return self.uniform(shape, _gain(gain) * math.sqrt(6.0 / (fan_in + fan_out)))

    def bias(self, n: int, fan_in: int) -> torch.Tensor:
        return self.uniform((n,), 1.0 / math.sqrt(fan_in))


def _lstm(d: _Draw, w: dict, prefix: str, n_in: int, hidden: int) -> None:
    b = 1.0 / math.sqrt(hidden)
    w[prefix + ".w_ih"] = d.uniform((4 * hidden, n_in), b)   # gate order i, f, g, o
    w[prefix + ".w_hh"] = d.uniform((4 * hidden, hidden), b)
    w[prefix + ".b_ih"] = d.uniform((4 * hidden,), b)
    w[prefix + ".b_hh"] = d.uniform((4 * hidden,), b)


def _on_grid(w: dict[str, torch.Tensor], bf16_grid: bool) -> dict[str, torch.Tensor]:
    return {k: t.to(torch.bfloat16).float() for k, t in w.items()} if bf16_grid else w


def tier_r_weights(seed: int = 0, bf16_grid: bool = True) -> dict[str, torch.Tensor]:
    """All Tier-R parameters, float32 on the CPU, deterministic in ``seed`` (on the bf16 grid
    unless ``bf16_grid=False``)."""
    d, w = _Draw(seed), {}
    # --- encoder (paper Eq. 1: four embedding tables summed) -------------
    std = math.sqrt(2.0 / (N_SYMBOLS + EMB))
    w["emb.phoneme"] = d.uniform((N_SYMBOLS, EMB), math.sqrt(3.0) * std)
    for name in ("pw", "pph", "iph"):
        std2 = math.sqrt(2.0 / (2 + EMB))
        w[f"emb.{name}"] = d.uniform((2, EMB), math.sqrt(3.0) * std2)
    bn = 1.0 / math.sqrt(1.0 + BN_EPS)
    for i in range(3):
        w[f"enc.conv{i}.w"] = d.xavier((EMB, EMB, 5), "relu") * bn
        w[f"enc.conv{i}.b"] = d.bias(EMB, EMB * 5) * bn
    _lstm(d, w, "enc.lstm_fwd", EMB, ENC_LSTM)
    _lstm(d, w, "enc.lstm_bwd", EMB, ENC_LSTM)
    # --- decoder (paper Eq. 2) ------------------------------------------
    w["att.memory_layer"] = d.xavier((ATT_DIM, EMB), "tanh")
    w["prenet.0"] = d.xavier((PRENET, N_MEL), "linear")
    w["prenet.1"] = d.xavier((PRENET, PRENET), "linear")
    _lstm(d, w, "att_rnn", PRENET + EMB, ATT_RNN)
    w["att.query_layer"] = d.xavier((ATT_DIM, ATT_RNN), "tanh")
    w["att.v"] = d.xavier((1, ATT_DIM), "linear")
    w["att.location_conv"] = d.xavier((LOC_FILTERS, 2, LOC_KERNEL), "linear")
    w["att.location_dense"] = d.xavier((ATT_DIM, LOC_FILTERS), "tanh")
    _lstm(d, w, "dec_rnn", ATT_RNN + EMB, DEC_RNN)
    w["proj.w"] = d.xavier((N_MEL, DEC_RNN + EMB), "linear")
    w["proj.b"] = d.bias(N_MEL, DEC_RNN + EMB)
    w["gate.w"] = d.xavier((1, DEC_RNN + EMB), "sigmoid")
    w["gate.b"] = d.bias(1, DEC_RNN + EMB)
    # --- HiFi-GAN V1 generator -------------------------------------------
    b = 1.0 / math.sqrt(N_MEL * 7)
    w["hg.conv_pre.w"] = d.uniform((HG_CH0, N_MEL, 7), b)   # kaiming_uniform(a=sqrt 5) bound
    w["hg.conv_pre.b"] = d.uniform((HG_CH0,), b)
    ch = HG_CH0
    for i, (u, k) in enumerate(zip(HG_UP_RATES, HG_UP_KERNELS)):
        # ConvTranspose1d weight layout [C_in, C_out, k]
        w[f"hg.up{i}.w"] = d.normal((ch, ch // 2, k), 0.01)
        w[f"hg.up{i}.b"] = d.uniform((ch // 2,), 1.0 / math.sqrt(ch // 2 * k))
        ch //= 2
        for j, kr in enumerate(HG_RES_KERNELS):
            for m, dil in enumerate(HG_RES_DILATIONS):
                for which in (1, 2):
                    key = f"hg.res{i}.{j}.c{which}{m}"
                    w[key + ".w"] = d.normal((ch, ch, kr), 0.01)
                    w[key + ".b"] = d.uniform((ch,), 1.0 / math.sqrt(ch * kr))
    w["hg.conv_post.w"] = d.normal((1, ch, 7), 0.01)
    w["hg.conv_post.b"] = d.uniform((1,), 1.0 / math.sqrt(ch * 7))
    return _on_grid(w, bf16_grid)


POSTNET_CH, POSTNET_K, POSTNET_LAYERS = 512, 5, 5


def postnet_weights(seed: int = 0, bf16_grid: bool = True) -> dict[str, torch.Tensor]:
    """Tacotron2 PostNet: 5 x conv k5, 80 -> 512 -> 512 -> 512 -> 512 -> 80, batch
    norm folded (eval mode, unit running variance), tanh after the first four.  A separate stream
    (seed + 7919) so the main Tier-R weights do not change."""
    d, w = _Draw(seed + 7919), {}
    bn = 1.0 / math.sqrt(1.0 + BN_EPS)
    chans = [N_MEL] + [POSTNET_CH] * (POSTNET_LAYERS - 1) + [N_MEL]
    for i in range(POSTNET_LAYERS):
        gain = "tanh" if i < POSTNET_LAYERS - 1 else "linear"
        w[f"post.conv{i}.w"] = d.xavier((chans[i + 1], chans[i], POSTNET_K), gain) * bn
        w[f"post.conv{i}.b"] = d.bias(chans[i + 1], chans[i] * POSTNET_K) * bn
    return _on_grid(w, bf16_grid)


def parameter_count(w: dict[str, torch.Tensor], prefix: str = "") -> int:
    return sum(t.numel() for k, t in w.items() if k.startswith(prefix))
