"""CPU restatement of the BERT prosody frontend (test infrastructure).

Post-LN BERT encoder (Devlin et al. 2018, BERT-base shape) with GELU in its tanh form and three
2-way linear heads, per text (no padding, full self-attention within the text), torch fp32 on the
CPU, following ``paper_2211_13939_b200/csrc/bert.cu``'s operator order.  Parity is not pinned
by the reference (it replaces the BERT frontend with a rule, ``src/frontend.py:174-188``).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from paper_2211_13939_b200.bert_frontend import HEADS, HIDDEN, LAYERS


def _ln(x, g, b):
    return F.layer_norm(x, (HIDDEN,), g, b, eps=1e-12)


def _gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608 * (x + 0.044715 * x ** 3)))


def prosody_logits(w, ids: list[int]) -> np.ndarray:
    """[L][6] head logits for one text's character ids."""
    L = len(ids)
    x = _ln(w["tok"][torch.as_tensor(ids)] + w["pos"][:L], w["ln.g"], w["ln.b"])
    hd = HIDDEN // HEADS
    for l in range(LAYERS):
        p = f"l{l}."
        qkv = x @ w[p + "qkv.w"].T + w[p + "qkv.b"]
        q, k, v = (qkv[:, i * HIDDEN:(i + 1) * HIDDEN].reshape(L, HEADS, hd).transpose(0, 1) for i in range(3))
        att = torch.softmax((q / math.sqrt(hd)) @ k.transpose(1, 2), -1) @ v      # [H][L][hd]
        y = att.transpose(0, 1).reshape(L, HIDDEN) @ w[p + "o.w"].T + w[p + "o.b"]
        x = _ln(x + y, w[p + "ln1.g"], w[p + "ln1.b"])
        y = _gelu(x @ w[p + "ff1.w"].T + w[p + "ff1.b"]) @ w[p + "ff2.w"].T + w[p + "ff2.b"]
        x = _ln(x + y, w[p + "ln2.g"], w[p + "ln2.b"])
    return (x @ w["heads.w"].T + w["heads.b"]).numpy()
