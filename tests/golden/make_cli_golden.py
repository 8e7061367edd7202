"""Golden losses of the REFERENCE's own ``bench`` subcommand (minml/cli.py:212-299), made in the
build container:  PB_NO_AUTOREGISTER=1 python tests/golden/make_cli_golden.py  -> cli_bench.json.
Both models, SGD and Adam, eager backend, 2 warm-up + 4 timed iterations."""
import json
import os
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
from minml import cli, figures  # noqa: E402

figures.bench_bars = lambda *a, **k: None  # matplotlib is not in this image; the JSON is what we keep

HERE = os.path.dirname(os.path.abspath(__file__))
out = {}
for model, opt, batch, lr in (("mlp", "sgd", 16, 0.05), ("cnn", "adam", 8, 1e-3)):
    d = tempfile.mkdtemp()
    argv = ["bench", "--backend", "eager", "--model", model, "--optim", opt, "--batch", str(batch), "--lr", str(lr),
            "--iters", "4", "--warmup", "2", "--seed", "5", "--out", d]
    assert cli.main(argv) == 0
    with open(os.path.join(d, "bench.json")) as f:
        rep = json.load(f)
    out[f"{model}-{opt}"] = {"argv": argv[3:-2], "losses": rep["runs"][0]["losses"]}
with open(os.path.join(HERE, "cli_bench.json"), "w") as f:
    json.dump(out, f, indent=1, sort_keys=True)
print(json.dumps(out))
