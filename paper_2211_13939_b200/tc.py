"""Host wrappers for the tcgen05 implicit-GEMM conv (``csrc/tc_conv.cu``).

Weight re-layout helpers turn PyTorch-layout conv / transposed-conv weights
into the kernel's K-major ``Wt[tap][n][c_in]`` bf16 form, and
:func:`conv1d_tc` launches one layer through the C ABI.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native

ACC_NONE, ACC_STORE, ACC_ADD, ACC_FINAL = 0, 1, 2, 3


def conv_weights(w: torch.Tensor, dilation: int = 1, c_in_pad: int | None = None):
    """Conv1d weight [C_out][C_in][k] -> (Wt [k][C_out][C_in'] bf16, tap offsets)."""
    c_out, c_in, k = w.shape
    cp = c_in_pad or c_in
    wt = torch.zeros(k, c_out, cp, dtype=torch.float32, device=w.device)
    wt[:, :, :c_in] = w.permute(2, 0, 1)
    offs = [dilation * (j - (k - 1) // 2) for j in range(k)]
    return wt.to(torch.bfloat16).contiguous(), offs


def convt_weights(w: torch.Tensor, stride: int):
    """ConvTranspose1d weight [C_in][C_out][2u], padding u/2 -> 3-tap phase conv.

    out[u*q + r] = sum_s X[q + s] . W[:, :, r + p - u*s]  (s in -1, 0, 1) ->
    Wp[s+1][r*C_out + co][ci]; zero where the kernel index leaves [0, 2u).
    """
    c_in, c_out, k = w.shape
    u = stride
    assert k == 2 * u, "HiFi-GAN V1 upsampling uses kernel = 2 * stride"
    p = (k - u) // 2
    wp = torch.zeros(3, u * c_out, c_in, dtype=torch.float32, device=w.device)
    for s in (-1, 0, 1):
        for r in range(u):
            kk = r + p - u * s
            if 0 <= kk < k:
                wp[s + 1, r * c_out:(r + 1) * c_out, :] = w[:, :, kk].T
    return wp.to(torch.bfloat16).contiguous(), [-1, 0, 1]


def conv1d_tc(x: torch.Tensor, wt: torch.Tensor, offs, bias: torch.Tensor, c_out: int,
              row_out: torch.Tensor, *, res_in=None, res_slope: float = 1.0, f32_out=None, ksplit: int = 1,
              acc=None, acc_mode=ACC_NONE, act_out=None, slope: float = 1.0, zero_halo: bool = True,
              bn: int = 0, stream=None) -> None:
    """One conv layer: x bf16 [R][C_in] (row stride x.stride(0)) -> epilogue outputs (tc_conv.cu).

    res_in / acc / act_out are bf16; res_in holds lrelu(y, res_slope) and is
    inverted on load.  f32_out receives the raw fp32 result (K-split partial
    slices when ksplit > 1).
    """
    rows, c_in = x.shape
    assert x.stride(1) == 1
    taps, n_total, c_in_w = wt.shape
    assert c_in_w == c_in and len(offs) == taps
    offs_arr = (ctypes.c_int32 * len(offs))(*offs)
    ptr = lambda t: 0 if t is None else t.data_ptr()
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _native.call("itts_conv1d_tc", x.data_ptr(), rows, c_in, x.stride(0), wt.data_ptr(), n_total, taps,
                 offs_arr, bias.data_ptr(), c_out, row_out.data_ptr(), ptr(res_in), float(res_slope),
                 ptr(f32_out), int(ksplit), ptr(acc), acc_mode, ptr(act_out), float(slope), int(zero_halo),
                 int(bn), st)


def resblock_tc(x: torch.Tensor, c1, c2, dilation: int, row_out: torch.Tensor, *, acc=None, acc_mode=ACC_NONE,
                act_out=None, slope: float = 0.1, stream=None) -> None:
    """One fused ResBlock1 layer (resblock_tc.cu): y = x + c2(lrelu(c1(lrelu x))), then the
    accumulator / leaky-ReLU epilogue.  x holds lrelu(x, 0.1) in bf16 [R][C]; c1 / c2 are
    (Wt [k][C][C] bf16, tap offsets, bias) as made by :func:`conv_weights`.  Output buffers
    must not alias x (neighbouring tiles still read it)."""
    rows, c = x.shape
    assert x.is_contiguous() and x.dtype == torch.bfloat16
    (w1, offs1, b1), (w2, offs2, b2) = c1, c2
    taps = w1.shape[0]
    assert w1.shape == (taps, c, c) and w2.shape == (taps, c, c)
    ptr = lambda t: 0 if t is None else t.data_ptr()
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _native.call("itts_resblock_tc", x.data_ptr(), rows, c, w1.data_ptr(), w2.data_ptr(), b1.data_ptr(),
                 b2.data_ptr(), taps, int(dilation), row_out.data_ptr(), ptr(acc), acc_mode, ptr(act_out),
                 float(slope), st)
