"""Layer math of the paper's workloads in fp64, NCHW layout (oracle, C1).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's CPU legs,
never by the product path.

The paper trains CNNs made of "convolutional layer, pooling layer,
Batch-Normalization (BN) layer, fully-connected layer" (Sec. 2.1) with
back-propagation: forward, backward, update. Each function below is
the textbook definition of one of those layers; backward functions are the
adjoints, written out directly (no autograd). Pinned by finite differences and
closed forms in tests/test_oracle_layers.py. Every function computes in the
dtype of its inputs (fp64 normally; the same code runs in fp32 for the oracle's
fp32 mode, which measures what plain fp32 arithmetic alone does to a result --
DESIGN.md Reading 28).
"""
from __future__ import annotations

import numpy as np

BN_EPS = 1e-5          # Reading 23 (paper silent)
SGD_MOMENTUM = 0.9     # Reading 23


# ---------------------------------------------------------------- TF32 operands
def _dt(*arrays):
    """Arithmetic type of a layer call: the inputs' (fp64 by default; fp32 when the oracle
    runs its fp32 mode, ``nets.forward_backward(precision="fp32")``)."""
    return np.result_type(*arrays)


def tf32(x):
    """Operand precision of the kernels' tensor-core contractions (BASELINE.json
    north_star: "TF32 in, FP32 accumulate"; DESIGN.md Reading 27): the value is
    rounded to fp32, then the 13 low mantissa bits are dropped (truncation, as
    measured on B200 -- tools/dbg_tf32.py). Returned as fp64. Used only when the
    oracle is asked to take decisions (ReLU masks, max-pool argmax) in the
    kernel's precision; the default oracle is exact fp64."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return u.view(np.float32).astype(np.float64)


# --------------------------------------------------------------------------- conv
def conv_out_hw(h: int, w: int, r: int, s: int, stride: int, pad: int):
    return (h + 2 * pad - r) // stride + 1, (w + 2 * pad - s) // stride + 1


def conv2d_fwd(x, w, stride=1, pad=0):
    """y[n,o,i,j] = sum_{c,u,v} x[n,c,s*i+u-p, s*j+v-p] * w[o,c,u,v] (zero padded)."""
    n, c, h, wd = x.shape
    o, c2, r, s = w.shape
    assert c == c2
    ho, wo = conv_out_hw(h, wd, r, s, stride, pad)
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    y = np.zeros((n, ho, wo, o), dtype=_dt(x, w))
    for u in range(r):
        for v in range(s):
            patch = xp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride]
            y += np.tensordot(patch, w[:, :, u, v], axes=([1], [1]))  # [n,ho,wo,o]
    return y.transpose(0, 3, 1, 2).copy()


def conv2d_dgrad(dy, w, x_shape, stride=1, pad=0):
    """dx = adjoint of conv2d_fwd w.r.t. x."""
    n, c, h, wd = x_shape
    o, _, r, s = w.shape
    _, _, ho, wo = dy.shape
    dxp = np.zeros((n, c, h + 2 * pad, wd + 2 * pad), dtype=_dt(dy, w))
    for u in range(r):
        for v in range(s):
            contrib = np.tensordot(dy, w[:, :, u, v], axes=([1], [0]))  # [n,ho,wo,c]
            dxp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride] += \
                contrib.transpose(0, 3, 1, 2)
    return dxp[:, :, pad:pad + h, pad:pad + wd].copy()


def conv2d_wgrad(x, dy, w_shape, stride=1, pad=0):
    """dw = adjoint of conv2d_fwd w.r.t. w."""
    o, c, r, s = w_shape
    _, _, ho, wo = dy.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    dw = np.zeros(w_shape, dtype=_dt(x, dy))
    for u in range(r):
        for v in range(s):
            patch = xp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride]
            dw[:, :, u, v] = np.tensordot(dy, patch, axes=([0, 2, 3], [0, 2, 3]))  # [o,c]
    return dw


# ------------------------------------------------------------------------- conv3d
# 3D workload of BASELINE.json config 4 ("3D U-Net-style, conv3d-BN-ReLU"; the paper's
# 3D-image motivation). NCDHW layout, cubic kernels.
def conv3d_out(d: int, k: int, stride: int, pad: int):
    return (d + 2 * pad - k) // stride + 1


def _win3(xp, u, v, t, stride, do, ho, wo):
    return xp[:, :, u:u + stride * (do - 1) + 1:stride, v:v + stride * (ho - 1) + 1:stride,
              t:t + stride * (wo - 1) + 1:stride]


def conv3d_fwd(x, w, stride=1, pad=0):
    """y[n,o,a,i,j] = sum_{c,u,v,t} x[n,c,s*a+u-p, s*i+v-p, s*j+t-p] * w[o,c,u,v,t] (zero padded)."""
    n, c, d, h, wd = x.shape
    o, c2, k, _, _ = w.shape
    assert c == c2
    do, ho, wo = (conv3d_out(e, k, stride, pad) for e in (d, h, wd))
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad), (pad, pad)))
    y = np.zeros((n, do, ho, wo, o), dtype=_dt(x, w))
    for u in range(k):
        for v in range(k):
            for t in range(k):
                y += np.tensordot(_win3(xp, u, v, t, stride, do, ho, wo), w[:, :, u, v, t], axes=([1], [1]))
    return y.transpose(0, 4, 1, 2, 3).copy()


def conv3d_dgrad(dy, w, x_shape, stride=1, pad=0):
    """dx = adjoint of conv3d_fwd w.r.t. x."""
    n, c, d, h, wd = x_shape
    o, _, k, _, _ = w.shape
    _, _, do, ho, wo = dy.shape
    dxp = np.zeros((n, c, d + 2 * pad, h + 2 * pad, wd + 2 * pad), dtype=_dt(dy, w))
    for u in range(k):
        for v in range(k):
            for t in range(k):
                contrib = np.tensordot(dy, w[:, :, u, v, t], axes=([1], [0]))  # [n,do,ho,wo,c]
                dxp[:, :, u:u + stride * (do - 1) + 1:stride, v:v + stride * (ho - 1) + 1:stride,
                    t:t + stride * (wo - 1) + 1:stride] += contrib.transpose(0, 4, 1, 2, 3)
    return dxp[:, :, pad:pad + d, pad:pad + h, pad:pad + wd].copy()


def conv3d_wgrad(x, dy, w_shape, stride=1, pad=0):
    """dw = adjoint of conv3d_fwd w.r.t. w."""
    o, c, k, _, _ = w_shape
    _, _, do, ho, wo = dy.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad), (pad, pad)))
    dw = np.zeros(w_shape, dtype=_dt(x, dy))
    for u in range(k):
        for v in range(k):
            for t in range(k):
                dw[:, :, u, v, t] = np.tensordot(dy, _win3(xp, u, v, t, stride, do, ho, wo),
                                                 axes=([0, 2, 3, 4], [0, 2, 3, 4]))
    return dw


def upconv3d_fwd(x, w):
    """Transposed convolution, kernel 2, stride 2 (the U-Net's up-sampling):
    y[n,o,2a+u,2i+v,2j+t] = sum_c x[n,c,a,i,j] * w[c,o,u,v,t]  -- every output voxel
    receives exactly one kernel tap. w is [Cin, Cout, 2, 2, 2]."""
    n, c, d, h, wd = x.shape
    c2, o = w.shape[:2]
    assert c == c2
    y = np.zeros((n, o, 2 * d, 2 * h, 2 * wd), dtype=_dt(x, w))
    for u in range(2):
        for v in range(2):
            for t in range(2):
                y[:, :, u::2, v::2, t::2] = np.tensordot(x, w[:, :, u, v, t], axes=([1], [0])).transpose(0, 4, 1, 2, 3)
    return y


def upconv3d_bwd(dy, x, w):
    """Adjoints of upconv3d_fwd: (dx, dw)."""
    dx = np.zeros_like(x, dtype=_dt(dy, x, w))
    dw = np.zeros(w.shape, dtype=_dt(dy, x, w))
    for u in range(2):
        for v in range(2):
            for t in range(2):
                g = dy[:, :, u::2, v::2, t::2]                                   # [n,o,d,h,w]
                dx += np.tensordot(g, w[:, :, u, v, t], axes=([1], [1])).transpose(0, 4, 1, 2, 3)
                dw[:, :, u, v, t] = np.tensordot(x, g, axes=([0, 2, 3, 4], [0, 2, 3, 4]))
    return dx, dw


def _pad3(x, pad, value=0.0):
    return np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad), (pad, pad)), constant_values=value) if pad else x


def maxpool3d_fwd(x, k=2, stride=2, pad=0):
    """Max over k^3 windows, -inf padding (the U-Net's 2^3 / 2 has none; ResNeXt-101 (3D)'s
    3^3 / 2 pads 1)."""
    n, c, d, h, w = x.shape
    do, ho, wo = (conv3d_out(e, k, stride, pad) for e in (d, h, w))
    xp = _pad3(x, pad, -np.inf)
    y = np.full((n, c, do, ho, wo), -np.inf, dtype=x.dtype)
    for u in range(k):
        for v in range(k):
            for t in range(k):
                y = np.maximum(y, _win3(xp, u, v, t, stride, do, ho, wo))
    return y


def maxpool3d_bwd(dy, x, k=2, stride=2, pad=0):
    """Gradient to the FIRST maximum in (u, v, t) row-major window order (Reading 25)."""
    n, c, d, h, w = x.shape
    _, _, do, ho, wo = dy.shape
    xp = _pad3(x, pad, -np.inf)
    best = np.full(dy.shape, -np.inf, dtype=x.dtype)
    arg = np.full(dy.shape, -1, dtype=np.int64)
    for u in range(k):
        for v in range(k):
            for t in range(k):
                win = _win3(xp, u, v, t, stride, do, ho, wo)
                better = win > best
                best = np.where(better, win, best)
                arg = np.where(better, (u * k + v) * k + t, arg)
    dxp = np.zeros(xp.shape, dtype=_dt(dy, x))
    for u in range(k):
        for v in range(k):
            for t in range(k):
                dxp[:, :, u:u + stride * (do - 1) + 1:stride, v:v + stride * (ho - 1) + 1:stride,
                    t:t + stride * (wo - 1) + 1:stride] += dy * (arg == (u * k + v) * k + t)
    return dxp[:, :, pad:pad + d, pad:pad + h, pad:pad + w].copy()


# ------------------------------------------------------ ResNeXt-101 (3D), SURVEY 8(f) f4
# "we computed ResNext101 (3D) [resnext] for various input data sizes with batch size of 1.
# ResNext101 (3D) is an extension of ResNext101 for video recognition based on [3dnn]"
# (Sec. 5.2). Its bottleneck's 3^3 convolution is GROUPED (ResNeXt's aggregated
# transformation, cardinality 32 [resnext]) and its stem strides (1, 2, 2) [3dnn]: a grouped
# convolution with a per-axis stride, written out below from its definition.
def _s3(stride):
    return (stride,) * 3 if isinstance(stride, int) else tuple(int(v) for v in stride)


def _win3s(xp, u, v, t, s3, do, ho, wo):
    sd, sh, sw = s3
    return xp[:, :, u:u + sd * (do - 1) + 1:sd, v:v + sh * (ho - 1) + 1:sh, t:t + sw * (wo - 1) + 1:sw]


def gconv3d_out(dhw, k, stride, pad):
    return tuple(conv3d_out(e, k, s, pad) for e, s in zip(dhw, _s3(stride)))


def gconv3d_fwd(x, w, stride=1, pad=0, groups=1):
    """Grouped 3D convolution, zero padded, stride (sd, sh, sw):
    y[n, g*Og+o, a, i, j] = sum_{c < Cg, u, v, t} x[n, g*Cg+c, sd*a+u-p, sh*i+v-p, sw*j+t-p]
                                                  * w[g*Og+o, c, u, v, t]
    with Cg = C / groups, Og = O / groups; w is [O, Cg, k, k, k] (groups = 1: conv3d_fwd)."""
    n, c, d, h, wd = x.shape
    o, cg, k, _, _ = w.shape
    assert c == cg * groups and o % groups == 0
    og = o // groups
    s3 = _s3(stride)
    do, ho, wo = gconv3d_out((d, h, wd), k, s3, pad)
    xp = _pad3(x, pad)
    y = np.zeros((n, o, do, ho, wo), dtype=_dt(x, w))
    for g in range(groups):
        xg = xp[:, g * cg:(g + 1) * cg]
        wg = w[g * og:(g + 1) * og]
        acc = np.zeros((n, do, ho, wo, og), dtype=y.dtype)
        for u in range(k):
            for v in range(k):
                for t in range(k):
                    acc += np.tensordot(_win3s(xg, u, v, t, s3, do, ho, wo), wg[:, :, u, v, t], axes=([1], [1]))
        y[:, g * og:(g + 1) * og] = acc.transpose(0, 4, 1, 2, 3)
    return y


def gconv3d_dgrad(dy, w, x_shape, stride=1, pad=0, groups=1):
    """dx = adjoint of gconv3d_fwd w.r.t. x."""
    n, c, d, h, wd = x_shape
    o, cg, k, _, _ = w.shape
    og = o // groups
    sd, sh, sw = _s3(stride)
    _, _, do, ho, wo = dy.shape
    dxp = np.zeros((n, c, d + 2 * pad, h + 2 * pad, wd + 2 * pad), dtype=_dt(dy, w))
    for g in range(groups):
        dyg = dy[:, g * og:(g + 1) * og]
        wg = w[g * og:(g + 1) * og]
        for u in range(k):
            for v in range(k):
                for t in range(k):
                    contrib = np.tensordot(dyg, wg[:, :, u, v, t], axes=([1], [0]))   # [n,do,ho,wo,cg]
                    dxp[:, g * cg:(g + 1) * cg, u:u + sd * (do - 1) + 1:sd, v:v + sh * (ho - 1) + 1:sh,
                        t:t + sw * (wo - 1) + 1:sw] += contrib.transpose(0, 4, 1, 2, 3)
    return dxp[:, :, pad:pad + d, pad:pad + h, pad:pad + wd].copy()


def gconv3d_wgrad(x, dy, w_shape, stride=1, pad=0, groups=1):
    """dw = adjoint of gconv3d_fwd w.r.t. w."""
    o, cg, k, _, _ = w_shape
    og = o // groups
    s3 = _s3(stride)
    _, _, do, ho, wo = dy.shape
    xp = _pad3(x, pad)
    dw = np.zeros(w_shape, dtype=_dt(x, dy))
    for g in range(groups):
        xg = xp[:, g * cg:(g + 1) * cg]
        dyg = dy[:, g * og:(g + 1) * og]
        for u in range(k):
            for v in range(k):
                for t in range(k):
                    dw[g * og:(g + 1) * og, :, u, v, t] = np.tensordot(
                        dyg, _win3s(xg, u, v, t, s3, do, ho, wo), axes=([0, 2, 3, 4], [0, 2, 3, 4]))
    return dw


# ----------------------------------------------------------------------------- BN
def _chan(v, ndim):
    """Per-channel vector broadcast against an N C spatial... array."""
    return v.reshape((1, -1) + (1,) * (ndim - 2))


def bn_fwd(x, gamma, beta, eps=BN_EPS):
    """Training-mode BN over (n, spatial...) per channel; biased variance."""
    ax = (0,) + tuple(range(2, x.ndim))
    mu = x.mean(axis=ax)
    var = ((x - _chan(mu, x.ndim)) ** 2).mean(axis=ax)
    invstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - _chan(mu, x.ndim)) * _chan(invstd, x.ndim)
    y = _chan(gamma, x.ndim) * xhat + _chan(beta, x.ndim)
    return y, (xhat, invstd)


def bn_bwd(dy, cache, gamma):
    """Closed form: dbeta = sum dy; dgamma = sum dy*xhat;
    dx = gamma*invstd*(dy - dbeta/N - xhat*dgamma/N)."""
    xhat, invstd = cache
    ax = (0,) + tuple(range(2, dy.ndim))
    m = dy.size // dy.shape[1]
    dbeta = dy.sum(axis=ax)
    dgamma = (dy * xhat).sum(axis=ax)
    dx = _chan(gamma * invstd, dy.ndim) * (dy - _chan(dbeta, dy.ndim) / m - xhat * _chan(dgamma, dy.ndim) / m)
    return dx, dgamma, dbeta


# --------------------------------------------------------------------------- ReLU
def relu_fwd(x):
    return np.maximum(x, 0.0)


def relu_bwd(dy, y):
    """dx = dy * [y > 0]  (ReLU'(0) = 0, Reading 26)."""
    return dy * (y > 0)


# ------------------------------------------------------------------------ pooling
def maxpool_fwd(x, k, stride, pad):
    """Max over k x k windows, -inf padding."""
    n, c, h, w = x.shape
    ho, wo = conv_out_hw(h, w, k, k, stride, pad)
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)), constant_values=-np.inf)
    y = np.full((n, c, ho, wo), -np.inf, dtype=x.dtype)
    for u in range(k):
        for v in range(k):
            y = np.maximum(y, xp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride])
    return y


def maxpool_bwd(dy, x, k, stride, pad):
    """Gradient to the FIRST maximum in row-major window order (Reading 25)."""
    n, c, h, w = x.shape
    _, _, ho, wo = dy.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)), constant_values=-np.inf)
    dxp = np.zeros_like(xp)
    best = np.full((n, c, ho, wo), -np.inf, dtype=x.dtype)
    arg = np.full((n, c, ho, wo), -1, dtype=np.int64)
    for u in range(k):
        for v in range(k):
            win = xp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride]
            better = win > best          # strict: first maximum wins
            best = np.where(better, win, best)
            arg = np.where(better, u * k + v, arg)
    for u in range(k):
        for v in range(k):
            sel = (arg == u * k + v)
            dxp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride] += dy * sel
    return dxp[:, :, pad:pad + h, pad:pad + w].copy()


def avgpool_fwd(x):
    """Global average pool: [n,c,h,w] (or [n,c,d,h,w]) -> [n,c]."""
    return x.mean(axis=tuple(range(2, x.ndim)))


def avgpool_bwd(dy, x_shape):
    sp = int(np.prod(x_shape[2:]))
    return np.broadcast_to(dy.reshape(dy.shape[:2] + (1,) * (len(x_shape) - 2)) / sp, x_shape).copy()


# ----------------------------------------------------------------------------- FC
def fc_fwd(x, w, b):
    """y = x W^T + b."""
    return x @ w.T + b[None, :]


def fc_bwd(dy, x, w):
    return dy @ w, dy.T @ x, dy.sum(axis=0)


# --------------------------------------------------------------------- softmax-CE
def softmax_ce(z, t):
    """loss = -mean_n log softmax(z_n)[t_n];  dz = (softmax(z) - onehot(t)) / B."""
    zmax = z.max(axis=1, keepdims=True)
    e = np.exp(z - zmax)
    p = e / e.sum(axis=1, keepdims=True)
    b = z.shape[0]
    loss = -np.mean(np.log(p[np.arange(b), t]))
    dz = p.copy()
    dz[np.arange(b), t] -= 1.0
    return loss, dz / b


# ---------------------------------------------------------------------------- SGD
def sgd_momentum(w, v, g, lr, mu=SGD_MOMENTUM, grad_scale=1.0):
    """v <- mu v + s g ; w <- w - lr v  (update step; s = 1/W under DP)."""
    v_new = mu * v + grad_scale * g
    return w - lr * v_new, v_new


# -------------------------------------------------------- AlexNet layers
# The paper's second image-recognition workload is AlexNet [alexnet] in
# Chainer's single-tower form: conv (+bias) -> ReLU -> local response normalisation -> max-pool,
# and fully-connected layers with ReLU and dropout.
LRN_N, LRN_K, LRN_ALPHA, LRN_BETA = 5, 2.0, 1e-4, 0.75   # Krizhevsky et al. / Chainer defaults


def conv2d_bias_fwd(x, w, b, stride=1, pad=0):
    """conv2d_fwd plus a per-output-channel bias."""
    return conv2d_fwd(x, w, stride, pad) + b.reshape(1, -1, 1, 1)


def lrn_fwd(x, n=LRN_N, k=LRN_K, alpha=LRN_ALPHA, beta=LRN_BETA):
    """Local response normalisation across channels (NCHW):
    y[c] = x[c] / (k + alpha / n * sum_{c' = c - n//2 .. c + n//2} x[c']^2) ** beta
    (channels outside [0, C) contribute nothing). Returns (y, s) with s the denominator base."""
    C = x.shape[1]
    sq = x * x
    s = np.zeros_like(x)
    for c in range(C):
        lo, hi = max(0, c - n // 2), min(C, c + n // 2 + 1)
        s[:, c] = sq[:, lo:hi].sum(axis=1)
    s = k + (alpha / n) * s
    return x * s ** (-beta), s


def lrn_bwd(dy, x, n=LRN_N, k=LRN_K, alpha=LRN_ALPHA, beta=LRN_BETA):
    """Adjoint of lrn_fwd: with s_j as above and t_j = dy_j x_j s_j^(-beta - 1),
    dx_c = dy_c s_c^(-beta) - (2 alpha beta / n) x_c sum_{j : |j - c| <= n//2} t_j."""
    _, s = lrn_fwd(x, n, k, alpha, beta)
    t = dy * x * s ** (-beta - 1.0)
    C = x.shape[1]
    acc = np.zeros_like(x)
    for c in range(C):
        lo, hi = max(0, c - n // 2), min(C, c + n // 2 + 1)
        acc[:, c] = t[:, lo:hi].sum(axis=1)
    return dy * s ** (-beta) - (2.0 * alpha * beta / n) * x * acc


def _fmix32(h):
    """MurmurHash3's 32-bit finaliser on uint32 arrays (wrap-around arithmetic)."""
    h = np.asarray(h, dtype=np.uint32).copy()
    h ^= h >> np.uint32(16)
    h *= np.uint32(0x85EBCA6B)
    h ^= h >> np.uint32(13)
    h *= np.uint32(0xC2B2AE35)
    h ^= h >> np.uint32(16)
    return h


def dropout_keep(shape, ratio, seed, step, task):
    """Counter-based dropout mask (the GPU implements the same generator; random numbers the
    method draws are a function of (seed, step, task, element index), so a recomputed forward
    reproduces its mask): key = fmix32(seed ^ fmix32(step * 0x9E3779B9 + task)), element i of the
    row-major [rows, cols] output is kept iff fmix32(key ^ fmix32(i)) >= floor(ratio * 2^32)."""
    with np.errstate(over="ignore"):
        key = _fmix32(np.uint32(seed) ^ _fmix32(np.uint32(step) * np.uint32(0x9E3779B9) + np.uint32(task)))
        idx = np.arange(int(np.prod(shape)), dtype=np.uint64).astype(np.uint32)
        u = _fmix32(key ^ _fmix32(idx))
    thresh = np.uint32(min(int(ratio * 4294967296.0), 4294967295))
    return (u >= thresh).reshape(shape)


def fc_relu_dropout_fwd(x, w, b, keep, ratio):
    """y = keep * relu(x W^T + b) / (1 - ratio)  (inverted dropout, ratio = drop probability)."""
    z = fc_fwd(x, w, b)
    return np.where(keep, np.maximum(z, 0.0) / (1.0 - ratio), 0.0), z


def fc_relu_dropout_bwd(dy, x, w, z, keep, ratio):
    """Adjoint of fc_relu_dropout_fwd: dz = dy * keep * [z > 0] / (1 - ratio); (dx, dW, db)."""
    dz = np.where(keep & (z > 0), dy / (1.0 - ratio), 0.0)
    return fc_bwd(dz, x, w)


# ------------------------------------------------ decisions taken in the kernel's precision
# Where floating point decides a discrete choice -- a ReLU mask, a max-pool winner -- the oracle
# can take that decision from the GPU's own tensors (its forward maps, read back) and compute
# everything else in fp64, so that both sides decide in the same precision and the comparison
# measures arithmetic, not the chaotic amplification of a flipped decision (DESIGN.md Reading 28).
def maxpool_argmax(xd, k, stride, pad):
    """Window index u*k+v of the FIRST maximum of every k x k window of xd (NCHW, -inf padding)."""
    n, c, h, w = xd.shape
    ho, wo = conv_out_hw(h, w, k, k, stride, pad)
    xp = np.pad(xd, ((0, 0), (0, 0), (pad, pad), (pad, pad)), constant_values=-np.inf)
    best = np.full((n, c, ho, wo), -np.inf, dtype=xd.dtype)
    arg = np.full((n, c, ho, wo), -1, dtype=np.int64)
    for u in range(k):
        for v in range(k):
            win = xp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride]
            better = win > best
            best = np.where(better, win, best)
            arg = np.where(better, u * k + v, arg)
    return arg


def maxpool_fwd_at(x, arg, k, stride, pad):
    """y = x at the window positions arg (from maxpool_argmax)."""
    n, c, h, w = x.shape
    _, _, ho, wo = arg.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)), constant_values=-np.inf)
    y = np.zeros(arg.shape, dtype=x.dtype)
    for u in range(k):
        for v in range(k):
            win = xp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride]
            y = np.where(arg == u * k + v, win, y)
    return y


def maxpool_bwd_at(dy, x_shape, arg, k, stride, pad):
    """dx: dy routed to the window positions arg."""
    n, c, h, w = x_shape
    _, _, ho, wo = dy.shape
    dxp = np.zeros((n, c, h + 2 * pad, w + 2 * pad), dtype=dy.dtype)
    for u in range(k):
        for v in range(k):
            dxp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride] += dy * (arg == u * k + v)
    return dxp[:, :, pad:pad + h, pad:pad + w].copy()


def maxpool3d_argmax(xd, k=2, stride=2, pad=0):
    n, c, d, h, w = xd.shape
    do, ho, wo = (conv3d_out(e, k, stride, pad) for e in (d, h, w))
    xp = _pad3(xd, pad, -np.inf)
    best = np.full((n, c, do, ho, wo), -np.inf, dtype=xd.dtype)
    arg = np.full((n, c, do, ho, wo), -1, dtype=np.int64)
    for u in range(k):
        for v in range(k):
            for t in range(k):
                win = _win3(xp, u, v, t, stride, do, ho, wo)
                better = win > best
                best = np.where(better, win, best)
                arg = np.where(better, (u * k + v) * k + t, arg)
    return arg


def maxpool3d_fwd_at(x, arg, k=2, stride=2, pad=0):
    _, _, do, ho, wo = arg.shape
    xp = _pad3(x, pad, -np.inf)
    y = np.zeros(arg.shape, dtype=x.dtype)
    for u in range(k):
        for v in range(k):
            for t in range(k):
                y = np.where(arg == (u * k + v) * k + t, _win3(xp, u, v, t, stride, do, ho, wo), y)
    return y


def maxpool3d_bwd_at(dy, x_shape, arg, k=2, stride=2, pad=0):
    _, _, do, ho, wo = dy.shape
    n, c, d, h, w = x_shape
    dxp = np.zeros((n, c, d + 2 * pad, h + 2 * pad, w + 2 * pad), dtype=dy.dtype)
    for u in range(k):
        for v in range(k):
            for t in range(k):
                dxp[:, :, u:u + stride * (do - 1) + 1:stride, v:v + stride * (ho - 1) + 1:stride,
                    t:t + stride * (wo - 1) + 1:stride] += dy * (arg == (u * k + v) * k + t)
    return dxp[:, :, pad:pad + d, pad:pad + h, pad:pad + w].copy()
