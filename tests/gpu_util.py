import pytest


def gpu_backend():
    import paper_2201_12465_b200 as pb
    from paper_2201_12465_b200 import registry
    if "gpu" not in registry.registered_ids():
        pytest.fail(f"GPU backend not registered: {registry._load_error}")
    return registry.get("gpu")
