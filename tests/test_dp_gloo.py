"""N>1 host-side path on CPU: two gloo ranks with different measured profiles
agree on one profile and therefore plan the identical classification through
the C ABI (pooch_plan_problem); DP semantics of the oracle (mean of per-shard
gradients with shard-local BN, Reading 29) checked against a direct sum."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synthdata
    from oracle import nets
    from paper_1907_05013_b200.dp import agree_profile
    from paper_1907_05013_b200.planning import PlanProblem
    net = nets.tiny_cnn()
    n = len(net.tasks)
    g = synthdata.rng(10 + rank)          # rank-specific measurements
    prof = {k: [int(v) for v in g.integers(1000, 50000, n)] for k in ("fwd", "bwd", "rec", "d2h", "h2d")}
    prof["tail"] = int(g.integers(100, 1000))
    prof.update(d2h_gbs=50.0 + rank, h2d_gbs=55.0 - rank, duplex_gbs=40.0 + 2 * rank)
    agreed = agree_profile(prof)
    nbytes = [8 * net.map_bytes_per_image(i) for i in range(n)]
    pp = PlanProblem(agreed["fwd"], agreed["bwd"], nbytes, agreed["d2h"], agreed["h2d"],
                     [[j for j in t.inputs if j >= 0] for t in net.tasks], [net.needs(i) for i in range(n)],
                     resident=0, budget=sum(nbytes) // 2, rec=agreed["rec"], tail=agreed["tail"],
                     duplex=(int(1000 * agreed["duplex_gbs"] / agreed["d2h_gbs"]),
                             int(1000 * agreed["duplex_gbs"] / agreed["h2d_gbs"])))
    cls, rep = pp.plan("pooch")
    link = (agreed["d2h_gbs"], agreed["h2d_gbs"], agreed["duplex_gbs"])
    q.put((rank, cls, agreed["fwd"][:3], prof["fwd"][:3], link))
    dist.destroy_process_group()


def test_two_ranks_agree_on_one_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    (r0, c0, a0, p0, l0), (r1, c1, a1, p1, l1) = res
    assert c0 is not None and c0 == c1
    assert l0 == l1 == (51.0, 55.0, 40.0)     # slowest link figures over the ranks (Reading 51)
    assert a0 == a1 == [max(x, y) for x, y in zip(p0, p1)]


def test_dp_gradient_is_mean_of_shards():
    """Reading 29: DP gradient = mean of per-shard gradients (shard-local BN)."""
    import synthdata
    from oracle import nets
    net = nets.tiny_cnn(width=4, in_hw=8)
    params = nets.init_params(net, seed=2, bn_random=True)
    shards = [(synthdata.images(2, 8, 8, 3, seed=r), synthdata.labels(2, 10, seed=1 + r)) for r in range(2)]
    gs = [nets.forward_backward(net, params, x, t)[1] for x, t in shards]
    w0 = {k: np.zeros_like(v) for k, v in params.items()}
    p_sum, _ = nets.sgd_step(params, w0, {k: gs[0][k] + gs[1][k] for k in params}, 0.1, grad_scale=0.5)
    p_mean, _ = nets.sgd_step(params, w0, {k: (gs[0][k] + gs[1][k]) / 2 for k in params}, 0.1)
    for k in params:
        np.testing.assert_allclose(p_sum[k], p_mean[k], rtol=1e-12, atol=1e-15)


def _ident_worker(rank, world, port, q, differ):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1907_05013_b200.dp import digest, ranks_identical
    arrs = [np.arange(1000, dtype=np.float32), np.ones(7, np.float32)]
    if differ and rank == 1:
        arrs[0][999] = np.nextafter(arrs[0][999], np.float32(2e3))   # one ulp on one rank
    q.put((rank, ranks_identical(digest(arrs))))
    dist.destroy_process_group()


@pytest.mark.parametrize("differ", [False, True])
def test_ranks_identical_checksum(differ):
    """bench.py's post-step rank-consistency check: every rank's parameter digest is gathered and
    compared; one ulp of difference on one rank is caught on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ident_worker, args=(r, 2, port, q, differ)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [ok for _, ok in res] == [not differ, not differ]


def test_numa_helpers_degrade_gracefully():
    from paper_1907_05013_b200.dp import node_cpus, pci_numa_node
    assert pci_numa_node("ffff:ff:1f.7") == -1          # no such device
    assert node_cpus(4096) == []                        # no such node
    c = node_cpus(0)
    assert c == [] or (all(isinstance(v, int) for v in c) and c == sorted(c))
