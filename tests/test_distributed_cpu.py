"""World-size-2 data parallelism over real processes (gloo on CPU, oracle backend):
post-backward sync and the bucketed/overlapped DataParallel both reproduce the reference's
thread-rank run (tests/golden/models.json "dp_mlp"), and shape mismatches raise
CollectiveShapeError on every rank (minml/distributed.py:107-116)."""

import json
import os
import socket
import subprocess
import sys

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
