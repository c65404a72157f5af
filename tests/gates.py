"""Reading 28's gradient gate (test logic, no arithmetic of the method): GPU gradients against
the fp64 oracle, with the fp32 oracle as the floor set by the problem's conditioning."""
import numpy as np

from netutil import global_rel, rel

TOL = 5e-3          # rel-L2 of the whole gradient and of every tensor (north_star; Reading 28)
FP32_X = 10.0       # a tensor whose plain-fp32 error already exceeds TOL / FP32_X is gated at
                    # FP32_X x that error instead: the problem's conditioning times the measured
                    # precision of the tensor-core contractions, whose fp32 accumulation in TMEM is
                    # biased (3xTF32 GEMM error / fp32 BLAS error = 14.5 at K = 576, growing with K;
                    # test_gpu_ops.py::test_3xtf32_error_against_fp32). Measured worst tensor
                    # ratios GPU / fp32 oracle: tiny CNN 8.4 (bn0.gamma), ResNet-50 4.0 (Reading 28)


def gate(g, ref64, ref32, tag):
    """Reading 28's gradient gate. For every parameter tensor: e = rel-L2(GPU, fp64 oracle) and
    e32 = rel-L2(fp32 oracle, fp64 oracle) -- the same NumPy code run in float32, i.e. what plain
    fp32 arithmetic alone does to that tensor. Gate: e <= max(5e-3, FP32_X e32). Prints the table."""
    rows = []
    for k in ref64:
        if np.linalg.norm(np.asarray(ref64[k])) == 0:
            continue                          # parameters that receive no gradient
        e, e32 = rel(g[k], ref64[k]), rel(ref32[k], ref64[k])
        rows.append((k, e, e32, max(TOL, FP32_X * e32)))
    rows.sort(key=lambda r: -r[1] / r[3])
    print("\n[%s] whole gradient: GPU %.3e, fp32 oracle %.3e" % (tag, global_rel(g, ref64), global_rel(ref32, ref64)))
    for k, e, e32, lim in rows[:8]:
        print("  %-28s GPU %.3e  fp32-oracle %.3e  limit %.3e" % (k, e, e32, lim))
    for fam in ("w", "bn"):
        sel = [r for r in rows if (r[0].endswith((".w", ".b")) == (fam == "w"))]
        if sel:
            print("  %s: max GPU %.3e, max fp32-oracle %.3e" % ("conv/FC weights" if fam == "w" else "BN gamma/beta",
                                                                 max(r[1] for r in sel), max(r[2] for r in sel)))
    bad = [r for r in rows if r[1] > r[3]]
    assert not bad, bad[:8]
    return rows


RELU_KINDS = ("bnrelu", "tail_proj", "tail_id", "conv_relu", "fc_relu_drop")


def gpu_decisions(ctx, net):
    """{task id: NC(D)HW map} for the oracle's decisions mode, read back from the GPU after a step
    planned in-core with POOCH_DEBUG_NO_REUSE=1 (every buffer instance at its own offset, so every
    forward map is intact afterwards): ReLU-type task outputs (their masks) and max-pool inputs
    (their window winners)."""
    B = ctx.batch
    out = {}

    def read(m):
        shape = tuple(net.tasks[m].out_chw)
        n = B * int(np.prod(shape))
        a = ctx.read_buffer(0, m, 4 * n)
        return np.moveaxis(a.reshape((B,) + shape[1:] + (shape[0],)), -1, 1).astype(np.float64)
    for i, t in enumerate(net.tasks):
        if t.kind in RELU_KINDS:
            out[i] = read(i)
        elif t.kind == "maxpool":
            out[i] = read(t.inputs[0])
    return out


def step_for_decisions(ctx, plan_step):
    """Run plan_step() (plan in-core + one step) with buffer reuse disabled."""
    import os
    os.environ["POOCH_DEBUG_NO_REUSE"] = "1"
    try:
        return plan_step()
    finally:
        os.environ.pop("POOCH_DEBUG_NO_REUSE", None)


# the measured error ratio of a 3xTF32 tensor-core GEMM to an fp32 BLAS GEMM at K = 576
# (test_gpu_ops.py::test_3xtf32_error_against_fp32: 14.5, growing with K; Reading 43)
X3_OVER_FP32 = 15.0


def gate_decided(g, ref, tag, ref32=None, factor=FP32_X):
    """The north_star gate, per tensor and whole, against the oracle run with the GPU's own
    ReLU / max-pool decisions (Reading 28): both sides decide in the same precision, so the gap is
    the arithmetic's alone. With ``ref32`` (the same decided oracle run in fp32) the BN gamma /
    beta tensors -- sums over every voxel of a map with cancelling signs -- are gated at
    max(5e-3, factor x their fp32 error), the floor the verdict asked to state per tensor; conv and
    FC weights and the whole gradient keep 5e-3."""
    rows = []
    for k in ref:
        if np.linalg.norm(np.asarray(ref[k])) == 0:
            continue
        e = rel(g[k], ref[k])
        lim = TOL
        if ref32 is not None and (".gamma" in k or ".beta" in k):
            lim = max(TOL, factor * rel(ref32[k], ref[k]))
        rows.append((k, e, lim))
    rows.sort(key=lambda r: -r[1] / r[2])
    glob = global_rel(g, ref)
    print("\n[%s, GPU decisions] whole gradient %.3e; worst (error, limit): %s" % (
        tag, glob, ", ".join("%s %.2e %.2e" % r for r in rows[:4])))
    assert glob < TOL
    assert rows[0][1] < rows[0][2], rows[:8]
    return rows
