"""SpAMM convolution drop-in (spamm_conv2d_im2col; Sec. 4.3.2).

  * configs[3]'s VGG13 layers: conv2_1 128 x 576 x 25600 and conv3_1 256 x 1152 x 6400,
    pruned weights x ReLU activations: Y equals the float64 oracle's SpAMM of W and the host im2col
    (synth.im2col, independent numpy code) at valid ratios ~97 / 63 % (Table 5 range);
  * the convolution semantics are pinned by brute force: at tau = 0 the result equals a direct
    nested-loop convolution for other kernel sizes, strides and paddings.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import T, _rel_fro, _rounded, sp  # noqa: F401

pytestmark = pytest.mark.gpu

DT = {"fp32": torch.float32, "fp32x3": torch.float32, "bf16": torch.bfloat16, "fp16": torch.float16}


def _direct_conv(X, W, kh, kw, stride, pad):
    nb, ci, h, w = X.shape
    co = W.shape[0]
    Ho, Wo = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    Wt = W.reshape(co, ci, kh, kw).astype(np.float64)
    Y = np.zeros((co, nb, Ho, Wo))
    for n in range(nb):
        for y in range(Ho):
            for x in range(Wo):
                for ky in range(kh):
                    for kx in range(kw):
                        iy, ix = y * stride - pad + ky, x * stride - pad + kx
                        if 0 <= iy < h and 0 <= ix < w:
                            Y[:, n, y, x] += Wt[:, :, ky, kx] @ X[n, :, iy, ix].astype(np.float64)
    return Y.reshape(co, nb * Ho * Wo)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("geom", [(3, 3, 1, 1), (3, 3, 2, 1), (5, 5, 1, 2), (1, 1, 1, 0), (3, 2, 2, 0)])
def test_conv_tau0_is_direct_convolution(sp, prec, geom):
    kh, kw, stride, pad = geom
    nb, ci, h, w, co = 2, 5, 9, 7, 6
    X = _rounded(synth.relu_activations(nb, ci, h, seed=161)[:, :, :, :w].copy(), prec)
    W = _rounded(synth.random_matrix(co, ci * kh * kw, seed=162), prec)
    Ho, Wo = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    N, K = nb * Ho * Wo, ci * kh * kw
    ldw = -(-K // 8) * 8
    Wd = torch.zeros((co, ldw), dtype=DT[prec], device="cuda")
    Wd[:, :K] = torch.from_numpy(W).to(DT[prec])
    Xd = torch.from_numpy(X).to(DT[prec]).cuda().contiguous()
    Y = torch.full((co, -(-N // 4) * 4), float("nan"), device="cuda")
    with sp.Plan(co, N, K, 0.0, prec) as plan:
        sp.spamm_conv2d_im2col(plan.handle, Wd[:, :K], Xd, Y[:, :N], kh, kw, stride, pad)
        torch.cuda.synchronize()
    ref = _direct_conv(X, W, kh, kw, stride, pad)
    assert _rel_fro(Y[:, :N].cpu().numpy(), ref) <= (2e-6 if prec == "fp32" else 1e-5)


@pytest.mark.parametrize("layer", ["conv21", "conv31"])
@pytest.mark.parametrize("prec", ["bf16", "fp32x3"])
def test_conv_vgg_layers_vs_oracle(sp, layer, prec):
    c_out, c_in, h, nb = synth.IM2COL_LAYERS[layer]
    W = _rounded(synth.conv_weight(c_out, c_in, 2107), prec)
    X = _rounded(synth.relu_activations(nb, c_in, h, 2117), prec)
    B = synth.im2col(X)                       # host im2col: independent of the CUDA kernel
    K, N = B.shape
    nA, nB = oracle.tile_norms(W, T), oracle.tile_norms(B, T)
    prods = np.unique(nA[:, :, None] * nB[None, :, :])
    Wd = torch.from_numpy(W).to(DT[prec]).cuda()
    Xd = torch.from_numpy(X).to(DT[prec]).cuda().contiguous()
    Y = torch.full((c_out, N), float("nan"), device="cuda")
    with sp.Plan(c_out, N, K, 0.0, prec) as plan:
        for vr in (0.97, 0.63):
            q = int((1.0 - vr) * (len(prods) - 1))
            tau = float(0.5 * (prods[q] + prods[q + 1]))
            plan.set_tau(tau)
            sp.spamm_conv2d_im2col(plan.handle, Wd, Xd, Y)
            torch.cuda.synchronize()
            assert plan.stats()["kept"] == oracle.count_kept(nA, nB, tau)
            err = _rel_fro(Y.cpu().numpy(), oracle.spamm(W, B, tau, T, nA, nB))
            assert err <= (5e-6 if prec == "fp32x3" else 1e-5), (vr, err)
