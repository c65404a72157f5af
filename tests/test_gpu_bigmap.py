"""Config 4 protection: the 3D U-Net's conv3d -> BN -> ReLU -> 2^3 max-pool chain (forward and
backward) on maps of MORE than 2^31 elements (config 4's 256^3 x 256-channel maps hold 4.3 G), through
the kernel-level C ABI the executor's launchers sit behind (pooch_op_conv_fwd with D > 0,
pooch_op_bn_finalize / bn_relu_fwd / bn_relu_bwd, pooch_op_maxpool3d_fwd / bwd).

Volume 416^3 x 32 channels = 2,303,721,472 elements per map (9.2 GB). Every check looks at elements
whose flat index is past 2^31 and compares with the fp64 oracle (oracle/layers.py) element by
element at sampled voxels -- conv outputs from their 3^3 x 32 input patch, pool windows, gradients --
and with whole-map fp64 reductions where the definition needs them (BN statistics, dgamma / dbeta),
plus the BN-backward invariants sum(gx) = 0 and sum(gx * xhat) = 0 per channel."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from oracle import layers as L  # noqa: E402

E, CH = 416, 32
ROWS = E ** 3
EPS = 1e-5


def _lib():
    from paper_1907_05013_b200 import _lib
    return _lib


def ptr(t):
    return C.c_void_p(t.data_ptr())


def _chan_sums(a, b=None, chunk=1 << 23):
    """Per-channel fp64 sums of a (or a * b) over the rows of [rows, CH] float32 host arrays."""
    out = np.zeros(a.shape[1])
    for i in range(0, a.shape[0], chunk):
        x = a[i:i + chunk].astype(np.float64)
        out += (x if b is None else x * b[i:i + chunk]).sum(axis=0)
    return out


@pytest.fixture(scope="module")
def chain():
    free, _ = torch.cuda.mem_get_info()
    if free < (60 << 30):
        pytest.skip("needs ~55 GB of free HBM")
    lib = _lib()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    x = torch.randn((E, E, E, CH), generator=gen, device="cuda")
    g = synthdata.rng(8)
    w = (g.standard_normal((CH, 3, 3, 3, CH)) * np.sqrt(2.0 / (27 * CH))).astype(np.float32)   # KTRSC
    gamma = g.uniform(0.5, 1.5, CH).astype(np.float32)
    beta = g.uniform(-0.2, 0.2, CH).astype(np.float32)
    d = lib.ConvDesc(1, E, E, CH, CH, 3, 3, 1, 1, 1, E, 0)
    tiles = lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
    wt, gt, bt = (torch.from_numpy(a).cuda() for a in (w, gamma, beta))
    y = torch.empty((E, E, E, CH), device="cuda")
    ts, tq = torch.empty((tiles, CH), device="cuda"), torch.empty((tiles, CH), device="cuda")
    lib.check(lib.lib.pooch_op_conv_fwd(C.byref(d), ptr(x), ptr(wt), ptr(y), ptr(ts), ptr(tq), None))
    mean, invstd, scale, shift = (torch.empty(CH, device="cuda") for _ in range(4))
    ws = torch.empty(lib.lib.pooch_op_bn_ws_bytes(CH) // 4 + 1, device="cuda")
    lib.check(lib.lib.pooch_op_bn_finalize(ptr(ts), ptr(tq), tiles, CH, ROWS, ptr(gt), ptr(bt), ptr(mean),
                                           ptr(invstd), ptr(scale), ptr(shift), ptr(ws), None))
    del ts, tq
    z = torch.empty_like(y)
    lib.check(lib.lib.pooch_op_bn_relu_fwd(ptr(y), ptr(scale), ptr(shift), ptr(z), ROWS, CH, None))
    pz = torch.empty((E // 2, E // 2, E // 2, CH), device="cuda")
    lib.check(lib.lib.pooch_op_maxpool3d_fwd(ptr(z), ptr(pz), E, E, E, CH, None))
    gp = torch.randn(pz.shape, generator=gen, device="cuda")
    gz = torch.empty_like(z)
    lib.check(lib.lib.pooch_op_maxpool3d_bwd(ptr(z), ptr(gp), ptr(gz), E, E, E, CH, 0, None))
    dgam, dbet = torch.empty(CH, device="cuda"), torch.empty(CH, device="cuda")
    gx = torch.empty_like(y)
    lib.check(lib.lib.pooch_op_bn_relu_bwd(ptr(y), ptr(gz), ptr(scale), ptr(shift), ptr(mean), ptr(invstd), ptr(gt),
                                           ptr(dgam), ptr(dbet), ptr(gx), ROWS, CH, ptr(ws), None))
    torch.cuda.synchronize()
    out = dict(w=w, gamma=gamma, beta=beta,
               x_tail=x[E - 17:].cpu().numpy(),                     # planes whose elements are past 2^31
               y=y.cpu().numpy().reshape(ROWS, CH), z=z.cpu().numpy().reshape(ROWS, CH),
               pz_tail=pz[E // 2 - 8:].cpu().numpy(), gp_tail=gp[E // 2 - 8:].cpu().numpy(),
               gz=gz.cpu().numpy().reshape(ROWS, CH), gx=gx.cpu().numpy().reshape(ROWS, CH),
               mean=mean.cpu().numpy(), invstd=invstd.cpu().numpy(), scale=scale.cpu().numpy(),
               shift=shift.cpu().numpy(), dgamma=dgam.cpu().numpy(), dbeta=dbet.cpu().numpy())
    del x, y, z, pz, gp, gz, gx
    torch.cuda.empty_cache()
    # oracle statistics of the conv output (Sec. 2.1 BN, biased variance), fp64 over all rows
    mu = _chan_sums(out["y"]) / ROWS
    var = np.zeros(CH)
    for i in range(0, ROWS, 1 << 23):
        var += ((out["y"][i:i + (1 << 23)].astype(np.float64) - mu) ** 2).sum(axis=0)
    out["mu64"], out["invstd64"] = mu, 1.0 / np.sqrt(var / ROWS + EPS)
    return out


def _samples():
    """Voxels (d, h, w) in the last 16 planes: flat element index (voxel * 32 + c) > 2^31."""
    g = synthdata.rng(9)
    v = [(E - 1, E - 1, E - 1), (E - 1, 0, 0), (E - 16, 1, E - 2)]
    for _ in range(40):
        v.append((int(g.integers(E - 16, E)), int(g.integers(0, E)), int(g.integers(0, E))))
    assert all(((a * E + b) * E + c) * CH > 2 ** 31 for a, b, c in v)
    return v


def test_conv3d_outputs_past_2_31(chain):
    xt = chain["x_tail"]                              # planes E-17 .. E-1
    w = np.moveaxis(chain["w"], -1, 1).astype(np.float64)   # [K, C, 3, 3, 3]
    got, ref = [], []
    for (a, b, c) in _samples():
        patch = np.zeros((3, 3, 3, CH))
        for i in range(3):
            for j in range(3):
                for k in range(3):
                    za, zb, zc = a + i - 1, b + j - 1, c + k - 1
                    if 0 <= za < E and 0 <= zb < E and 0 <= zc < E:
                        patch[i, j, k] = xt[za - (E - 17), zb, zc]
        ref.append(L.conv3d_fwd(np.moveaxis(patch, -1, 0)[None], w, 1, 0)[0, :, 0, 0, 0])
        got.append(chain["y"][(a * E + b) * E + c])
    got, ref = np.array(got, np.float64), np.array(ref)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 2e-5


def test_bn_statistics_over_2_31_elements(chain):
    np.testing.assert_allclose(chain["mean"], chain["mu64"], rtol=0, atol=1e-5 / chain["invstd64"].min())
    np.testing.assert_allclose(chain["invstd"], chain["invstd64"], rtol=1e-5)


def test_bn_relu_and_pool_past_2_31(chain):
    mu, inv, gam, bet = chain["mu64"], chain["invstd64"], chain["gamma"], chain["beta"]
    zt = chain["z"]
    for (a, b, c) in _samples():
        r = (a * E + b) * E + c
        ref = np.maximum(gam * (chain["y"][r].astype(np.float64) - mu) * inv + bet, 0.0)   # relu(BN(y))
        np.testing.assert_allclose(zt[r], ref, rtol=0, atol=2e-5)
    # pool windows over the last planes: exact (max is exact) and first-max routing of the gradient
    zv = zt.reshape(E, E, E, CH)
    g = synthdata.rng(10)
    for _ in range(40):
        pa, pb, pc = int(g.integers(E // 2 - 8, E // 2)), int(g.integers(0, E // 2)), int(g.integers(0, E // 2))
        win = np.moveaxis(zv[2 * pa:2 * pa + 2, 2 * pb:2 * pb + 2, 2 * pc:2 * pc + 2].astype(np.float64), -1, 0)[None]
        y_ref = L.maxpool3d_fwd(win)[0, :, 0, 0, 0]
        assert np.array_equal(chain["pz_tail"][pa - (E // 2 - 8), pb, pc].astype(np.float64), y_ref)
        gy = chain["gp_tail"][pa - (E // 2 - 8), pb, pc].astype(np.float64)[None, :, None, None, None]
        gx_ref = np.moveaxis(L.maxpool3d_bwd(gy, win)[0], 0, -1)
        gz = chain["gz"].reshape(E, E, E, CH)[2 * pa:2 * pa + 2, 2 * pb:2 * pb + 2, 2 * pc:2 * pc + 2]
        assert np.array_equal(gz.astype(np.float64), gx_ref)


def test_bn_backward_past_2_31(chain):
    mu, inv, gam = chain["mu64"], chain["invstd64"], chain["gamma"].astype(np.float64)
    y, z, gz, gx = chain["y"], chain["z"], chain["gz"], chain["gx"]
    dz_mask = (z > 0)
    dbeta = np.zeros(CH)
    dgamma = np.zeros(CH)
    sabs = np.zeros(CH)
    sgx = np.zeros(CH)
    sgx_xhat = np.zeros(CH)
    sgx_abs = np.zeros(CH)
    for i in range(0, ROWS, 1 << 23):
        dz = gz[i:i + (1 << 23)].astype(np.float64) * dz_mask[i:i + (1 << 23)]
        xh = (y[i:i + (1 << 23)].astype(np.float64) - mu) * inv
        dbeta += dz.sum(axis=0)
        dgamma += (dz * xh).sum(axis=0)
        sabs += np.abs(dz).sum(axis=0) + np.abs(dz * xh).sum(axis=0)
        g = gx[i:i + (1 << 23)].astype(np.float64)
        sgx += g.sum(axis=0)
        sgx_xhat += (g * xh).sum(axis=0)
        sgx_abs += np.abs(g).sum(axis=0) + np.abs(g * xh).sum(axis=0)
    # dgamma / dbeta: sums over 72 M voxels, compared against their conditioning (sum of |terms|)
    assert np.all(np.abs(chain["dbeta"] - dbeta) <= 1e-5 * sabs)
    assert np.all(np.abs(chain["dgamma"] - dgamma) <= 1e-5 * sabs)
    # BN-backward invariants: the input gradient has zero sum and is orthogonal to xhat per channel
    assert np.all(np.abs(sgx) <= 1e-5 * sgx_abs) and np.all(np.abs(sgx_xhat) <= 1e-5 * sgx_abs)
    # element values past 2^31: gx = gamma invstd (dz - dbeta / N - xhat dgamma / N)
    for (a, b, c) in _samples():
        r = (a * E + b) * E + c
        dz = gz[r].astype(np.float64) * (z[r] > 0)
        xh = (y[r].astype(np.float64) - mu) * inv
        ref = gam * inv * (dz - dbeta / ROWS - xh * dgamma / ROWS)
        np.testing.assert_allclose(gx[r], ref, rtol=0, atol=1e-5 * np.abs(gam * inv).max() * (np.abs(dz).max() + 1e-3))
