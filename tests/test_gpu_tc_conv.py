"""tcgen05 implicit-GEMM conv kernel vs a plain PyTorch fp32 reference of the same op.

Inputs/weights are bf16-representable so the only difference is fp32
accumulation order: tolerance 2e-3 relative to the output scale.
"""

import pytest
import torch
import torch.nn.functional as F

from paper_2211_13939_b200 import tc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def layout(lengths, halo):
    """Packed rows: item b occupies [base, base+2*halo+T); valid rows map to themselves."""
    bases, pos = [], 0
    for T in lengths:
        bases.append(pos)
        pos += 2 * halo + T
    row_out = torch.full((pos,), -1, dtype=torch.int32)
    for b, T in zip(bases, lengths):
        row_out[b + halo:b + halo + T] = torch.arange(b + halo, b + halo + T, dtype=torch.int32)
    return bases, pos, row_out


def pack(items, bases, rows, halo, C):
    x = torch.zeros(rows, C)
    for it, b in zip(items, bases):
        x[b + halo:b + halo + it.shape[0]] = it
    return x


def bf(t):
    return t.to(torch.bfloat16).float()


@pytest.mark.parametrize("c_in,c_out,k,dil", [(256, 256, 3, 1), (128, 128, 11, 5), (64, 64, 7, 3),
                                              (32, 32, 3, 5), (128, 512, 7, 1), (64, 32, 5, 1)])
def test_conv_matches_torch(c_in, c_out, k, dil):
    torch.manual_seed(0)
    lengths, halo = [37, 128, 300, 5], 25
    bases, rows, row_out = layout(lengths, halo)
    items = [bf(torch.randn(T, c_in)) for T in lengths]
    w = bf(torch.randn(c_out, c_in, k) / (c_in * k) ** 0.5)
    bias = torch.randn(c_out)
    x = pack(items, bases, rows, halo, c_in).to(DEV).to(torch.bfloat16)
    wt, offs = tc.conv_weights(w.to(DEV), dil)
    out = torch.full((rows, c_out), 7.0, device=DEV)
    act = torch.full((rows, c_out), 7.0, device=DEV, dtype=torch.bfloat16)
    tc.conv1d_tc(x, wt, offs, bias.to(DEV), c_out, row_out.to(DEV), f32_out=out, act_out=act, slope=0.1)
    torch.cuda.synchronize()
    for it, b, T in zip(items, bases, lengths):
        ref = F.conv1d(it.T[None], w, bias, dilation=dil, padding=dil * (k - 1) // 2)[0].T
        got = out[b + halo:b + halo + T].cpu()
        scale = ref.abs().max().item()
        assert (got - ref).abs().max().item() <= 2e-3 * scale + 1e-5
        ref_act = F.leaky_relu(ref, 0.1).to(torch.bfloat16).float()
        got_act = act[b + halo:b + halo + T].float().cpu()
        assert (got_act - ref_act).abs().max().item() <= 1e-2 * scale + 1e-4
        assert torch.all(act[b:b + halo].float() == 0) and torch.all(act[b + halo + T:b + 2 * halo + T].float() == 0)


def test_residual_and_mrf_accumulate():
    """bf16 residual stream stored as lrelu(y, 0.1) and inverted on load; bf16 MRF accumulator."""
    torch.manual_seed(1)
    C, k, dil = 64, 5, 3
    lengths, halo = [100, 61], 25
    bases, rows, row_out = layout(lengths, halo)
    x = bf(torch.randn(rows, C)).to(DEV)
    for b, T in zip(bases, lengths):  # zero halos
        x[b:b + halo] = 0
        x[b + halo + T:b + 2 * halo + T] = 0
    w = bf(torch.randn(C, C, k) / (C * k) ** 0.5)
    bias = torch.randn(C).to(DEV)
    wt, offs = tc.conv_weights(w.to(DEV), dil)
    xb = x.to(torch.bfloat16)
    ro = row_out.to(DEV)
    y0 = torch.randn(rows, C, device=DEV)
    res = F.leaky_relu(y0, 0.1).to(torch.bfloat16)
    acc0 = torch.randn(rows, C, device=DEV).to(torch.bfloat16)
    conv = F.conv1d(x.T[None].cpu(), w, bias.cpu(), dilation=dil, padding=dil * (k - 1) // 2)[0].T
    y_in = torch.where(res.float() >= 0, res.float(), res.float() / 0.1).cpu()
    ref_y = y_in + conv
    valid = row_out >= 0
    scale = ref_y.abs().max()
    # residual add -> act_out (stored as lrelu(y))
    act = torch.zeros(rows, C, device=DEV, dtype=torch.bfloat16)
    tc.conv1d_tc(xb, wt, offs, bias, C, ro, res_in=res, res_slope=0.1, act_out=act, slope=0.1)
    # residual add -> accumulate
    acc = acc0.clone()
    tc.conv1d_tc(xb, wt, offs, bias, C, ro, res_in=res, res_slope=0.1, acc=acc, acc_mode=tc.ACC_ADD)
    # finalize (acc + y) / 3 -> lrelu 0.01
    fin_act = torch.zeros(rows, C, device=DEV, dtype=torch.bfloat16)
    tc.conv1d_tc(xb, wt, offs, bias, C, ro, res_in=res, res_slope=0.1, acc=acc0.clone(), acc_mode=tc.ACC_FINAL,
                 act_out=fin_act, slope=0.01)
    torch.cuda.synchronize()
    assert (act.float().cpu()[valid] - F.leaky_relu(ref_y, 0.1)[valid]).abs().max() < 1e-2 * scale
    assert (acc.float().cpu()[valid] - (acc0.float().cpu() + ref_y)[valid]).abs().max() < 1e-2 * scale
    fin = F.leaky_relu((acc0.float().cpu() + ref_y) / 3.0, 0.01)
    assert (fin_act.float().cpu()[valid] - fin[valid]).abs().max() < 1e-2 * fin.abs().max()


@pytest.mark.parametrize("B,K,ksplit", [(1, 1792, 4), (37, 2560, 4), (200, 1792, 1), (130, 2560, 2)])
def test_gemm_ksplit_on_column_slice(B, K, ksplit):
    """Decoder gate GEMM: x is a column slice of a wider bf16 row (ld 2816); K-split partials."""
    torch.manual_seed(3)
    full = bf(torch.randn(B, 2816)).to(DEV).to(torch.bfloat16)
    x = full[:, 2816 - K:]
    w = bf(torch.randn(4096, K) / K ** 0.5)
    out = torch.zeros(ksplit, B, 4096, device=DEV)
    rows = torch.arange(B, dtype=torch.int32, device=DEV)
    bias = torch.randn(4096, device=DEV)
    tc.conv1d_tc(x, w.to(DEV).to(torch.bfloat16)[None].contiguous(), [0], bias, 4096, rows, f32_out=out,
                 ksplit=ksplit, bn=64)
    torch.cuda.synchronize()
    ref = x.float().cpu() @ w.T + bias.cpu()
    got = out.sum(0).cpu()
    assert (got - ref).abs().max() <= 2e-3 * ref.abs().max()


@pytest.mark.parametrize("c_in,c_out,u", [(512, 256, 8), (256, 128, 8), (128, 64, 2), (64, 32, 2)])
def test_transposed_conv_matches_torch(c_in, c_out, u):
    torch.manual_seed(2)
    lengths, halo_in, halo_out = [36, 9, 33], 3, 25
    bases, rows, _ = layout(lengths, halo_in)
    out_bases, out_rows, _ = layout([T * u for T in lengths], halo_out)
    row_out = torch.full((rows,), -1, dtype=torch.int32)
    for b, ob, T in zip(bases, out_bases, lengths):
        row_out[b + halo_in:b + halo_in + T] = ob + halo_out + u * torch.arange(T, dtype=torch.int32)
    items = [bf(torch.randn(T, c_in)) for T in lengths]
    w = bf(torch.randn(c_in, c_out, 2 * u) * 0.05)
    bias = torch.randn(c_out)
    x = pack(items, bases, rows, halo_in, c_in).to(DEV).to(torch.bfloat16)
    wp, offs = tc.convt_weights(w.to(DEV), u)
    out = torch.zeros(out_rows, c_out, device=DEV)
    tc.conv1d_tc(x, wp, offs, bias.to(DEV), c_out, row_out.to(DEV), f32_out=out, zero_halo=False)
    torch.cuda.synchronize()
    for it, ob, T in zip(items, out_bases, lengths):
        ref = F.conv_transpose1d(it.T[None], w, bias, stride=u, padding=u // 2)[0].T
        got = out[ob + halo_out:ob + halo_out + T * u].cpu()
        assert got.shape == ref.shape
        assert (got - ref).abs().max().item() <= 2e-3 * ref.abs().max().item() + 1e-5
