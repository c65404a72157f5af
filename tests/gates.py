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
