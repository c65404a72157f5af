"""Test-side glue between the oracle's parameter layout (OIHW, unpadded) and the
C ABI's (KRSC with Cin padded to 4, FC rows padded to a multiple of 4).
Pure re-layout (transpose / zero-pad / crop): no arithmetic of the method."""
import numpy as np


def to_pooch(name, arr, numel):
    a = np.asarray(arr, np.float32)
    if name.endswith(".w") and a.ndim in (4, 5):     # OI(D)HW -> K(T)RSC, pad C
        o, c = a.shape[:2]
        sp = a.shape[2:]
        cp = numel // (o * int(np.prod(sp)))
        out = np.zeros((o,) + sp + (cp,), np.float32)
        out[..., :c] = np.moveaxis(a, 1, -1)
        return out
    if name.endswith(".w") and a.ndim == 2:          # FC [classes, cin] -> [cpad, cin]
        k, cin = a.shape
        out = np.zeros((numel // cin, cin), np.float32)
        out[:k] = a
        return out
    if a.size != numel:                              # FC bias
        out = np.zeros(numel, np.float32)
        out[:a.size] = a.ravel()
        return out
    return a


def from_pooch(name, flat, ref_shape):
    """Pooch layout -> oracle layout of shape ref_shape."""
    ref_shape = tuple(ref_shape)
    if name.endswith(".w") and len(ref_shape) in (4, 5):
        o, c = ref_shape[:2]
        sp = ref_shape[2:]
        cp = flat.size // (o * int(np.prod(sp)))
        return np.moveaxis(flat.reshape((o,) + sp + (cp,))[..., :c], -1, 1)
    if name.endswith(".w") and len(ref_shape) == 2:
        k, cin = ref_shape
        return flat.reshape(-1, cin)[:k]
    return flat[:int(np.prod(ref_shape))].reshape(ref_shape)


def pad_input(x_nhwc, c=4):
    """Zero-pad the channel (last) axis of an N(D)HWC batch to c channels."""
    out = np.zeros(x_nhwc.shape[:-1] + (c,), np.float32)
    out[..., :x_nhwc.shape[-1]] = x_nhwc
    return out


def load_params(ctx, params):
    for i, (name, numel) in enumerate(ctx.params()):
        ctx.set_param(i, to_pooch(name, params[name], numel))


def read_params(ctx, params_ref, which):
    out = {}
    for i, (name, numel) in enumerate(ctx.params()):
        out[name] = from_pooch(name, ctx.get_param(i, which), np.shape(params_ref[name]))
    return out


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def global_rel(g, ref):
    """rel-L2 of the whole gradient (every parameter tensor concatenated)."""
    num = sum(float(np.sum((np.asarray(g[k], np.float64) - np.asarray(ref[k], np.float64)) ** 2)) for k in ref)
    den = sum(float(np.sum(np.asarray(ref[k], np.float64) ** 2)) for k in ref)
    return (num / max(den, 1e-300)) ** 0.5
