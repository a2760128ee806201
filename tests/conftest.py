import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdh2.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


_CACHE = {}


def oracle_run(name, eps=None, mode="FROB_BLOCKREL", **over):
    """Build and recompress a named configuration with the oracle (memoised)."""
    from synth import get_config, mesh_for
    from oracle.structure import DH2Structure
    from oracle.recompress import Recompression

    cfg = get_config(name)
    cfg.update(over)
    key = (name, eps, mode, tuple(sorted(over.items())))
    if key not in _CACHE:
        xyz, tri = mesh_for(cfg)
        st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
        rc = Recompression(st, cfg["eps"] if eps is None else eps, mode).run()
        _CACHE[key] = rc
    return _CACHE[key]


@pytest.fixture(scope="session")
def oracle_cache():
    return oracle_run


def release_gpu_contexts():
    """Close the DH2 contexts other test modules cache (tests/test_gpu_parity.py _GPU,
    tests/test_gpu_lean.py _RUNS), so that a full-size configuration finds the device memory free."""
    import gc
    for mod in list(sys.modules.values()):
        for name in ("_GPU", "_RUNS"):
            cache = getattr(mod, name, None)
            if isinstance(cache, dict):
                for v in cache.values():
                    h = v[0] if isinstance(v, tuple) else v
                    if hasattr(h, "close"):
                        h.close()
                cache.clear()
    gc.collect()
