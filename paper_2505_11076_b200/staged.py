"""Staged-gradient consumers of the DBF forward on the GPU.

The reference computes, in float64 numpy, the gradients of the layer reconstruction loss through
the staged forward h0 = X*b, h1 = h0 B^T, h2 = h1*mid, h3 = h2 A^T, out = h3*a:

* ``channel_scores`` (budget.py:145-173): score_i = sum_batches (dL/dmid_i * mid_i)^2;
* ``staged_loss_grads`` (factorize.py:310-326, ``_staged_loss_grads``): loss and dL/da, dL/dmid,
  dL/db, including the TRANSPOSED sign products d_h2 = d_h3 A and d_h0 = (d_h2*mid) B;
* ``refine_scales`` (factorize.py:335-370): guarded gradient descent on (a, mid, b), signs frozen.

Here every sign product runs on the GPU through the C ABI: ``dbf_sign_gemm_f64`` (float64 on CUDA
cores -- the reference's tests check exact zeros and equalities, test_budget.py:97-145,
test_factorize.py:231-238, so these offline consumers keep float64) against the canonical words of
S and of S^T (``dbf_transpose_signs``, built once per sign matrix).  Element-wise products and
column sums are float64 torch ops on the device.  Host inputs/outputs keep the reference contract:
float64 numpy in, float64 numpy out, the same ValueError messages.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .bitcore import DbfLayer
from .validation import as_matrix, as_vector, check_shape


@dataclass(frozen=True)
class ChannelScores:
    """budget.py:57-65: per-middle-channel sensitivity scores of one layer."""

    name: str
    scores: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "scores", as_vector(self.scores, "scores"))
        if (self.scores < 0).any():
            raise ValueError("channel scores must be nonnegative")


def _signs(s):
    """Device canonical words of a host or device sign matrix (cached per object)."""
    from .kernel import as_device_signs

    return as_device_signs(s)


def sign_products_f64(ds, X):
    """X @ S^T for a float64 CUDA tensor X (batch x cols): out (batch x rows), float64."""
    import torch

    w = ds._need_words()
    X = X.contiguous()
    out = torch.empty((X.shape[0], ds.rows), dtype=torch.float64, device=X.device)
    _lib.check(
        _lib.lib.dbf_sign_gemm_f64(w.data_ptr(), ds.rows, ds.cols, w.shape[1], X.data_ptr(), X.stride(0),
                                   X.shape[0], out.data_ptr(), out.stride(0), _lib.stream_ptr()),
        "dbf_sign_gemm_f64",
    )
    return out


class _DeviceFactors:
    """Device float64 view of one layer's signs (S and S^T words) for the staged products."""

    def __init__(self, layer):
        self.A = _signs(layer.A)
        self.B = _signs(layer.B)
        self.At = self.A.transposed()  # k x n
        self.Bt = self.B.transposed()  # m x k


def _t(v):
    import torch

    return torch.as_tensor(np.array(v, dtype=np.float64)).cuda()


def _grads(f: _DeviceFactors, X, Y, a, mid, b, want_grads: bool = True):
    """factorize.py:310-326 on the device: (loss, grad_a, grad_mid, grad_b) as float64 tensors."""
    h0 = X * b[None, :]
    h1 = sign_products_f64(f.B, h0)          # h0 @ Bd^T
    h3 = sign_products_f64(f.A, h1 * mid[None, :])  # h2 @ Ad^T
    resid = h3 * a[None, :] - Y
    loss = (resid * resid).sum()
    if not want_grads:
        return loss, None, None, None
    d_h3 = 2.0 * resid * a[None, :]
    grad_a = 2.0 * (resid * h3).sum(0)
    d_h2 = sign_products_f64(f.At, d_h3)     # d_h3 @ Ad
    grad_mid = (d_h2 * h1).sum(0)
    d_h0 = sign_products_f64(f.Bt, d_h2 * mid[None, :])  # (d_h2 * mid) @ Bd
    grad_b = (d_h0 * X).sum(0)
    return loss, grad_a, grad_mid, grad_b


def staged_loss_grads(X, Y, layer):
    """factorize._staged_loss_grads for a layer: (loss, grad_a, grad_mid, grad_b), float64 numpy."""
    _lib.require_cuda()
    X = as_matrix(X, "X")
    Y = as_matrix(Y, "Y")
    check_shape(X, (X.shape[0], layer.m_dim), "X")
    check_shape(Y, (X.shape[0], layer.n), "Y")
    f = _DeviceFactors(layer)
    loss, ga, gm, gb = _grads(f, _t(X), _t(Y), _t(layer.a), _t(layer.mid), _t(layer.b))
    return float(loss.item()), ga.cpu().numpy(), gm.cpu().numpy(), gb.cpu().numpy()


def channel_scores(layer, X_batches, Y_batches, name: str = "layer") -> ChannelScores:
    """budget.channel_scores (budget.py:145-173) on the GPU."""
    X_batches = list(X_batches)
    Y_batches = list(Y_batches)
    if not X_batches or len(X_batches) != len(Y_batches):
        raise ValueError("need at least one (X, Y) batch pair")
    _lib.require_cuda()
    import torch

    f = _DeviceFactors(layer)
    a, mid, b = _t(layer.a), _t(layer.mid), _t(layer.b)
    scores = torch.zeros(layer.k, dtype=torch.float64, device="cuda")
    for X, Y in zip(X_batches, Y_batches):
        X = as_matrix(X, "X")
        Y = as_matrix(Y, "Y")
        if X.shape != (X.shape[0], layer.m_dim) or Y.shape != (X.shape[0], layer.n):
            raise ValueError(
                f"batch shapes {X.shape}/{Y.shape} do not match layer "
                f"{layer.n}x{layer.m_dim}"
            )
        Xd, Yd = _t(X), _t(Y)
        h1 = sign_products_f64(f.B, Xd * b[None, :])
        out = sign_products_f64(f.A, h1 * mid[None, :]) * a[None, :]
        d_h2 = sign_products_f64(f.At, 2.0 * (out - Yd) * a[None, :])
        grad = (d_h2 * h1).sum(0)
        scores += (grad * mid) ** 2
    return ChannelScores(name, scores.cpu().numpy())


def refine_scales(layer, X, Y, steps: int = 100, lr: float = 1e-3) -> DbfLayer:
    """factorize.refine_scales (factorize.py:335-370) on the GPU: guarded gradient descent on the
    scale vectors with the signs frozen; a step that increases the loss is halved up to 20 times,
    then skipped (the loss never increases)."""
    X = as_matrix(X, "X")
    Y = as_matrix(Y, "Y")
    check_shape(X, (X.shape[0], layer.m_dim), "X")
    check_shape(Y, (X.shape[0], layer.n), "Y")
    _lib.require_cuda()
    f = _DeviceFactors(layer)
    Xd, Yd = _t(X), _t(Y)
    a, mid, b = _t(layer.a), _t(layer.mid), _t(layer.b)
    for _ in range(steps):
        loss, g_a, g_mid, g_b = _grads(f, Xd, Yd, a, mid, b)
        loss = float(loss.item())
        if loss == 0.0:
            break
        step = lr
        accepted = False
        for _ in range(21):
            cand = (a - step * g_a, mid - step * g_mid, b - step * g_b)
            if float(_grads(f, Xd, Yd, *cand, want_grads=False)[0].item()) <= loss:
                a, mid, b = cand
                accepted = True
                break
            step *= 0.5
        if not accepted:
            break
    return DbfLayer(a=a.cpu().numpy(), A=layer.A, mid=mid.cpu().numpy(), B=layer.B, b=b.cpu().numpy())
