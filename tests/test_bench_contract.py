"""bench.py keeps the driver's contract: the committed cfg2 line carries every required key, and
the reference arm (the CPU oracle, this tier's reference) prints a valid line without a GPU."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..")
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline", "cpu_baseline"]


def test_committed_headline_line_has_the_contract_keys():
    """The committed default line (r02: BASELINE config 3, the metric's >HBM batch) carries every
    contract key plus the round-2 evidence: the full-size bit-exact check, a finite loss, the
    in-core comparison and the secondary cfg2 line checked against in-core."""
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_cfg3.json")))
    for k in REQUIRED:
        assert k in d, k
    assert d["config"]["workload"].startswith("cfg3")
    assert d["bitexact"]["bitexact"] is True and d["loss_finite"] is True
    assert d["incore"]["images_per_s"] > 0 and "overhead_vs_incore" in d
    assert d["cfg2"]["bitexact_vs_incore"] is True and d["cfg2"]["isolated_profile"]["bitexact_vs_incore"] is True
    assert d["config"]["L_O"] > 0 and d["config"]["L_I"] > 0 and d["config"]["profile_mode"] in ("isolated", "all_swap")
    assert d["warmup"] >= 3 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert 0 < d["roofline"]["frac"] <= 1
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k


def test_reference_arm_runs_on_cpu():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_gpus_n_without_launcher_relaunches_or_fails_loudly():
    """`bench.py --gpus 2` run by hand (no WORLD_SIZE) re-executes itself under
    torch.distributed.run; with fewer visible GPUs than asked it exits non-zero with a message
    instead of silently measuring one GPU."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 2, (r.returncode, r.stderr[-800:])
    assert "needs 2 visible GPUs" in r.stderr
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]


def test_relaunch_line_is_the_drivers():
    sys.path.insert(0, ROOT)
    from paper_1907_05013_b200.dp import relaunch_argv
    a = relaunch_argv("/x/bench.py", ["--gpus", "4", "--steps", "3"], 4, 29555)
    assert a[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in a and "--nnodes=1" in a
    assert a[a.index("--master-addr") + 1] == "127.0.0.1" and a[a.index("--master-port") + 1] == "29555"
    assert a[-5:] == ["/x/bench.py", "--gpus", "4", "--steps", "3"]
