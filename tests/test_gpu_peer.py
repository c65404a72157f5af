"""Multi-rank gradient allreduce over peer memory (Sec. 1).

W processes share cuda:0 (the GPU boxes have one GPU); each maps the others' exchange buffers
with cudaIpcOpenMemHandle, the same path NVLink peers take. Each rank steps its own shard; the
exchanged gradient on every rank must equal the fp32 sum of the ranks' local gradients formed in
rank order 0, 1, ..., W-1 -- bit for bit (each element is summed by exactly one rank in that
order, peer.cu) -- for in-core and out-of-core plans, for the graph-capturing step and its
replay; the updated parameters must agree across ranks; and the data-parallel gradient (the sum
/ W) must match the mean of the per-shard fp64 oracle gradients within the north_star gate.
"""
import glob
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

import synthdata  # noqa: E402
from netutil import from_pooch, global_rel  # noqa: E402
from oracle import nets  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp_path, world, strategy, net="tiny"):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_PORT=str(port),
                   MASTER_ADDR="127.0.0.1")
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "peer_worker.py"), str(tmp_path), strategy,
                                       net], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=900)[0].decode(errors="replace"))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, p in enumerate(procs):
        assert p.returncode == 0, "rank %d failed:\n%s" % (r, outs[r][-3000:])
    res = [json.load(open(os.path.join(tmp_path, "rank%d.json" % r))) for r in range(world)]

    def load(name):
        z = np.load(os.path.join(tmp_path, name))
        return [z["arr_%d" % i] for i in range(len(z.files))]
    return res, load


@pytest.mark.parametrize("world,strategy,net", [(2, "incore", "tiny"), (2, "pooch", "tiny"), (3, "pooch", "tiny"),
                                                (4, "incore", "tiny"), (2, "incore", "resnet50")])
def test_peer_allreduce_sum_bit_exact(tmp_path, world, strategy, net):
    """ResNet-50 (25.6 M parameters) spans four gradient buckets, each its own barrier pair."""
    res, load = _run(tmp_path, world, strategy, net)
    local = [load("rank%d_local.npz" % r) for r in range(world)]
    expect = []
    for i in range(len(local[0])):
        s = local[0][i].astype(np.float32).copy()
        for r in range(1, world):
            s = (s + local[r][i]).astype(np.float32)   # rank order, fp32, one rounding per add
        expect.append(s)
    for r in range(world):
        assert res[r]["comm_nranks"] == world and res[r]["comm_rank"] == r
        for it in range(2):
            g = load("rank%d_it%d.npz" % (r, it))
            for i, (a, b) in enumerate(zip(g, expect)):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), \
                    "rank %d step %d param %d: exchanged gradient != rank-order fp32 sum" % (r, it, i)
        assert res[r]["graph1"], "the replayed step should be a CUDA-graph launch"
    for it in range(2):
        w0 = load("rank0_w%d.npz" % it)
        for r in range(1, world):
            for a, b in zip(w0, load("rank%d_w%d.npz" % (r, it))):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    if strategy == "pooch":
        assert all(res[r]["plan"] == res[0]["plan"] for r in range(world))


def test_peer_dp_gradient_matches_oracle(tmp_path):
    """Per-rank BN, allreduce(sum) / W (DESIGN Reading 29): the data-parallel gradient equals the
    mean of the per-shard fp64 oracle gradients (north_star gate 5e-3, whole gradient)."""
    world = 2
    res, load = _run(tmp_path, world, "pooch")
    net = nets.tiny_cnn()
    params = nets.init_params(net, seed=2, bn_random=True)
    ref = None
    for r in range(world):
        x = synthdata.images(8, 32, 32, 3, seed=100 + r)
        t = synthdata.labels(8, 10, seed=200 + r)
        _, g, _ = nets.forward_backward(net, params, x, t)
        ref = g if ref is None else {k: ref[k] + g[k] for k in ref}
    ref = {k: v / world for k, v in ref.items()}
    from paper_1907_05013_b200.executor import Context
    names = [n for n, _ in Context.builtin("tiny", 8, in_hw=32, classes=10).params()]
    flat = load("rank0_it0.npz")
    got = {n: from_pooch(n, flat[i], np.shape(ref[n])) / world for i, n in enumerate(names)}
    assert global_rel(got, ref) <= 5e-3
