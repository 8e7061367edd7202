"""``python -m paper_2201_12465_b200 bench`` (cli.py) against the reference's own ``bench``
subcommand (minml/cli.py:212-299): same synthetic blobs, models, optimizers and loss trajectory
(tests/golden/cli_bench.json, made by make_cli_golden.py), the reference's table / bench.json
layout and exit codes (minml/cli.py:34-48)."""
import json
import os

import numpy as np
import pytest

from paper_2201_12465_b200 import cli, registry

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "cli_bench.json")))


def _run(backend, key, tmp_path):
    argv = ["bench", "--backend", backend] + GOLD[key]["argv"] + ["--out", str(tmp_path)]
    assert cli.main(argv) == cli.EXIT_OK
    rep = json.load(open(tmp_path / "bench.json"))
    assert set(rep) == {"model", "batch", "iters", "warmup", "runs"}
    run = rep["runs"][0]
    assert set(run["phases"]) == {"data", "forward", "backward", "step"} and run["backend"] == backend
    got, want = np.array(run["losses"]), np.array(GOLD[key]["losses"])
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1.0)))


@pytest.fixture()
def oracle_backend():
    from oracle.backend import OracleBackend
    be = OracleBackend(name="oracle-cli")
    registry.register(be)
    yield be.name
    registry.unregister(be.name)


@pytest.mark.parametrize("key", sorted(GOLD))
def test_bench_matches_reference_cli_on_the_oracle(oracle_backend, key, tmp_path):
    assert _run(oracle_backend, key, tmp_path) <= 1e-5


def test_exit_codes(oracle_backend):
    assert cli.main(["bench", "--backend", "no-such-backend"]) == cli.EXIT_CONFIG
    assert cli.main(["bench", "--backend", oracle_backend, "--iters", "0"]) == cli.EXIT_CONFIG
    assert cli.main(["bench", "--backend", oracle_backend, "--alloc", "bogus"]) == cli.EXIT_CONFIG
    assert cli.main(["train"]) == cli.EXIT_CONFIG


def test_synth_blobs_match_reference_fixture():
    """The blob generator restated in cli.py against the reference's items stored in dp.npz."""
    d = np.load(os.path.join(HERE, "golden", "dp.npz"))
    xs, ys = cli.synth_blobs(320, seed=21, dim=784)
    assert np.array_equal(d["acc_images"], xs) and np.array_equal(d["acc_labels"], ys)


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(GOLD))
def test_bench_matches_reference_cli_on_the_gpu(key, tmp_path):
    """``python -m paper_2201_12465_b200 bench --backend gpu`` as its own process (the
    allocator policy is attached to a backend with no live blocks, as in the reference)."""
    import subprocess
    import sys
    root = os.path.dirname(HERE)
    argv = [sys.executable, "-m", "paper_2201_12465_b200", "bench", "--backend", "gpu"] + GOLD[key]["argv"] + [
        "--out", str(tmp_path)]
    r = subprocess.run(argv, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == cli.EXIT_OK, r.stderr[-2000:]
    assert r.stdout.splitlines()[0].split("\t")[0] == "backend"
    run = json.load(open(tmp_path / "bench.json"))["runs"][0]
    got, want = np.array(run["losses"]), np.array(GOLD[key]["losses"])
    assert float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1.0))) <= 1e-5
