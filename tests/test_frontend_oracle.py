"""The product front end (Tensor/Variable/nn/optim) driven on the numpy oracle backend
reproduces the reference's own training trajectories (tests/golden/models.json)."""

import numpy as np
import pytest

from frontend_util import BUILDERS, run_trajectory
from golden_util import models_arrays, models_meta, rel_err
from oracle.backend import OracleBackend
from paper_2201_12465_b200 import registry

META = models_meta()


@pytest.fixture
def oracle_backend(request):
    be = OracleBackend(name=f"oracle-{request.node.name}")
    registry.register(be)
    yield be
    registry.unregister(be.name)


@pytest.mark.parametrize("name", sorted(BUILDERS))
def test_trajectory_matches_reference(name, oracle_backend):
    meta = META[name]
    losses, sums, model = run_trajectory(name, meta, oracle_backend)
    assert len(sums) == meta["n_params"]
    assert rel_err(losses, meta["losses"]) <= 1e-6, (losses, meta["losses"])
    assert rel_err(sums, meta["param_sums"]) <= 1e-5
    arrays = models_arrays()
    for i, p in enumerate(model.params()):
        key = f"{name}_p{i}"
        if key in arrays.files:
            assert rel_err(p.numpy(), arrays[key]) <= 1e-5, key


@pytest.mark.parametrize("name", ["mlp_full", "lenet_full"])
def test_fullsize_oracle_matches_reference(name, oracle_backend):
    """The oracle pinned at BASELINE size too (configs 1-2 at their real batch, 10 steps):
    the checker the GPU full-size tests are read against agrees with the reference run."""
    from fullsize_util import arrays, compare, meta, run
    m = meta()[name]
    losses, params = run(name, m, oracle_backend, "eager")
    err = compare(name, m, arrays(), losses, params)
    assert err["loss"] <= 1e-6 and err["sum"] <= 1e-6 and err["sampled"] <= 1e-6, err
