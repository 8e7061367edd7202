"""World-size-2 data parallelism over real processes (gloo on CPU, oracle backend):
post-backward sync and the bucketed/overlapped DataParallel both reproduce the reference's
thread-rank run (tests/golden/models.json "dp_mlp"), and shape mismatches raise
CollectiveShapeError on every rank (minml/distributed.py:107-116)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from golden_util import models_meta, rel_err

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(world, mode, tmp_path, kind="oracle"):
    port = _port()
    env = dict(os.environ, PB_NO_AUTOREGISTER="1" if kind == "oracle" else "0", OMP_NUM_THREADS="1",
               OPENBLAS_NUM_THREADS="1")
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dp_worker.py"), str(r), str(world), str(port),
                               mode, str(tmp_path), kind], env=env) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    return [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]


@pytest.mark.parametrize("mode", ["sync", "bucketed"])
def test_two_rank_dp_matches_reference(mode, tmp_path):
    gold = models_meta()["dp_mlp"]
    res = launch(2, mode, tmp_path)
    for r in range(2):
        assert rel_err(res[r]["losses"], gold["losses"][r]) <= 1e-6, (res[r]["losses"], gold["losses"][r])
    assert rel_err(res[0]["param_sums"], gold["param_sums"]) <= 1e-6
    assert res[0]["param_sums"] == res[1]["param_sums"]  # replicas stay bit-identical
    if mode == "bucketed":
        assert res[0]["buckets"] > 1


def test_shape_mismatch_raises_on_every_rank(tmp_path):
    res = launch(2, "shape_error", tmp_path)
    assert [r["raised"] for r in res] == ["CollectiveShapeError"] * 2


def dp_meta():
    with open(os.path.join(HERE, "golden", "dp.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("mode", ["acceptance_sync", "acceptance_bucketed"])
def test_reference_dp_acceptance_fixture(mode, tmp_path):
    """The reference's own DP acceptance fixture (T/test_acceptance.py:394-440) on 4 process
    ranks: every rank's 50 losses equal the reference's thread-rank run (tests/golden/dp.json,
    made by make_dp_golden.py), the rank mean stays within 1e-3 of the single-rank run, and
    the metadata checks leave a bounded number of keys in the store."""
    gold = dp_meta()["acceptance"]
    res = launch(4, mode, tmp_path)
    for r in range(4):
        assert rel_err(res[r]["losses"], gold["ranks"][r]) <= 1e-5, r
    assert rel_err(res[0]["param_sums"], gold["param_sums"]) <= 1e-5
    assert all(res[r]["param_sums"] == res[0]["param_sums"] for r in range(4))
    gap = max(abs(float(np.mean([res[r]["losses"][k] for r in range(4)])) - gold["single"][k])
              for k in range(gold["steps"]))
    assert gap <= 1e-3, gap
    if mode == "acceptance_sync":  # 50 per-step checks, at most two checks' keys live per rank
        assert res[0]["store_keys"] <= 4 * 2 + 8, res[0]["store_keys"]


def test_batchnorm_dp_matches_reference_thread_ranks(tmp_path):
    """BatchNorm statistics stay per rank; a 2-rank ResNet run equals the
    reference's run_ranks on the same shards (losses, parameters, running statistics)."""
    gold = dp_meta()["bn"]
    res = launch(2, "bn", tmp_path)
    for r in range(2):
        assert rel_err(res[r]["losses"], gold["ranks"][r]) <= 1e-5, (r, res[r]["losses"], gold["ranks"][r])
        assert rel_err(res[r]["buffer_sums"], gold["buffer_sums"][r]) <= 1e-5
    assert rel_err(res[0]["param_sums"], gold["param_sums"][0]) <= 1e-4
    assert res[0]["buffer_sums"] != res[1]["buffer_sums"]  # per-rank statistics differ


def test_broadcast_accepts_none_and_any_placeholder_off_root(tmp_path):
    """minml's broadcast contract (test_broadcast_accepts_none_off_root): only the root's
    tensor matters; other ranks may pass None or a placeholder of another shape."""
    res = launch(2, "broadcast", tmp_path)
    want = (np.arange(6, dtype=np.float32).reshape(2, 3) + 10).tolist()
    assert all(r["a"] == want and r["b"] == want for r in res)
