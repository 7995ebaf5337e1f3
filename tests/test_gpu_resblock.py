"""Fused ResBlock1 layer (resblock_tc.cu) vs a plain PyTorch fp32 reference of the same op.

y = x + c2(lrelu(c1(lrelu x, 0.1), 0.1)) per item with 'same' zero padding at
the item edges, x stored as lrelu(x, 0.1) in bf16.  The kernel rounds the
intermediate lrelu(c1(.)) to bf16 (it is the c2 operand), so the reference
does the same; remaining differences are fp32 accumulation order and the bf16
output rounding: tolerance 1e-2 of the output scale.
"""

import pytest
import torch
import torch.nn.functional as F

from paper_2211_13939_b200 import tc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
HALO = 25


def layout(lengths):
    bases, pos = [], 0
    for T in lengths:
        bases.append(pos)
        pos += 2 * HALO + T
    row_out = torch.full((pos,), -1, dtype=torch.int32)
    for b, T in zip(bases, lengths):
        row_out[b + HALO:b + HALO + T] = torch.arange(b + HALO, b + HALO + T, dtype=torch.int32)
    return bases, pos, row_out


def bf(t):
    return t.to(torch.bfloat16).float()


def reference(y_items, w1, b1, w2, b2, k, dil):
    outs = []
    for y in y_items:
        xt = F.leaky_relu(y, 0.1).T[None]
        t = F.conv1d(xt, w1, b1, dilation=dil, padding=dil * (k - 1) // 2)
        t = bf(F.leaky_relu(t, 0.1))
        outs.append(y + F.conv1d(t, w2, b2, padding=(k - 1) // 2)[0].T)
    return outs


def make(C, k, lengths, seed):
    torch.manual_seed(seed)
    bases, rows, row_out = layout(lengths)
    # the stored activation is lrelu(y) in bf16; the residual is its exact inverse
    stored_items = [bf(F.leaky_relu(torch.randn(T, C), 0.1)) for T in lengths]
    y_items = [torch.where(s >= 0, s, s / 0.1) for s in stored_items]
    x = torch.zeros(rows, C)
    for s, b, T in zip(stored_items, bases, lengths):
        x[b + HALO:b + HALO + T] = s
    w1 = bf(torch.randn(C, C, k) / (C * k) ** 0.5)
    w2 = bf(torch.randn(C, C, k) / (C * k) ** 0.5)
    b1, b2 = torch.randn(C) * 0.1, torch.randn(C) * 0.1
    return bases, rows, row_out, x, y_items, w1, b1, w2, b2


@pytest.mark.parametrize("C,k,dil", [(256, 3, 1), (256, 11, 5), (128, 7, 3), (128, 3, 1), (64, 11, 5),
                                     (64, 7, 1), (32, 3, 3), (32, 11, 5)])
def test_resblock_layer_matches_torch(C, k, dil):
    lengths = [37, 300, 5, 128, 700]
    bases, rows, row_out, x, y_items, w1, b1, w2, b2 = make(C, k, lengths, seed=C + k + dil)
    c1 = tc.conv_weights(w1.to(DEV), dil) + (b1.to(DEV),)
    c2 = tc.conv_weights(w2.to(DEV), 1) + (b2.to(DEV),)
    xd = x.to(DEV).to(torch.bfloat16)
    out = torch.full((rows, C), 3.0, device=DEV, dtype=torch.bfloat16)
    tc.resblock_tc(xd, c1, c2, dil, row_out.to(DEV), act_out=out, slope=0.1)
    torch.cuda.synchronize()
    refs = reference(y_items, w1, b1, w2, b2, k, dil)
    got = out.float().cpu()
    for ref, b, T in zip(refs, bases, lengths):
        scale = ref.abs().max().item()
        err = (got[b + HALO:b + HALO + T] - F.leaky_relu(ref, 0.1)).abs().max().item()
        assert err <= 1e-2 * scale, (err, scale)
        assert torch.all(got[b:b + HALO] == 0) and torch.all(got[b + HALO + T:b + 2 * HALO + T] == 0)


@pytest.mark.parametrize("C", [128, 32])
def test_resblock_accumulator_modes(C):
    k, dil = 7, 3
    lengths = [90, 411]
    bases, rows, row_out, x, y_items, w1, b1, w2, b2 = make(C, k, lengths, seed=7)
    c1 = tc.conv_weights(w1.to(DEV), dil) + (b1.to(DEV),)
    c2 = tc.conv_weights(w2.to(DEV), 1) + (b2.to(DEV),)
    xd, ro = x.to(DEV).to(torch.bfloat16), row_out.to(DEV)
    acc0 = torch.randn(rows, C, device=DEV).to(torch.bfloat16)
    acc_store = torch.zeros(rows, C, device=DEV, dtype=torch.bfloat16)
    tc.resblock_tc(xd, c1, c2, dil, ro, acc=acc_store, acc_mode=tc.ACC_STORE)
    acc_add = acc0.clone()
    tc.resblock_tc(xd, c1, c2, dil, ro, acc=acc_add, acc_mode=tc.ACC_ADD)
    fin = torch.full((rows, C), 5.0, device=DEV, dtype=torch.bfloat16)
    tc.resblock_tc(xd, c1, c2, dil, ro, acc=acc0.clone(), acc_mode=tc.ACC_FINAL, act_out=fin, slope=0.01)
    torch.cuda.synchronize()
    refs = reference(y_items, w1, b1, w2, b2, k, dil)
    a0 = acc0.float().cpu()
    for ref, b, T in zip(refs, bases, lengths):
        sl = slice(b + HALO, b + HALO + T)
        scale = ref.abs().max().item()
        assert (acc_store.float().cpu()[sl] - ref).abs().max() <= 1e-2 * scale
        assert (acc_add.float().cpu()[sl] - (a0[sl] + ref)).abs().max() <= 1e-2 * scale
        want = F.leaky_relu((a0[sl] + ref) / 3.0, 0.01)
        assert (fin.float().cpu()[sl] - want).abs().max() <= 1e-2 * want.abs().max()
        assert torch.all(fin.float().cpu()[b:b + HALO] == 0)


def test_resblock_rejects_aliasing():
    C = 64
    x = torch.zeros(200, C, device=DEV, dtype=torch.bfloat16)
    w = torch.zeros(3, C, C, device=DEV, dtype=torch.bfloat16)
    b = torch.zeros(C, device=DEV)
    ro = torch.arange(200, dtype=torch.int32, device=DEV)
    with pytest.raises(RuntimeError, match="EINVAL"):
        tc.resblock_tc(x, (w, [-1, 0, 1], b), (w, [-1, 0, 1], b), 1, ro, act_out=x)
