import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libparplan_cuda.so")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _impl_params():
    import oracle as O

    ps = [pytest.param("port", id="port")]
    if O.available("reference"):
        ps.append(pytest.param("reference", id="reference"))
    ps.append(pytest.param("gpu", id="gpu", marks=pytest.mark.gpu))
    return ps


_IMPLS = {}


def get_impl(name):
    import impls

    if name not in _IMPLS:
        _IMPLS[name] = impls.GpuImpl() if name == "gpu" else impls.OracleImpl(name)
    return _IMPLS[name]


@pytest.fixture(params=_impl_params())
def impl(request):
    return get_impl(request.param)


@pytest.fixture(scope="session")
def gpu():
    return get_impl("gpu")


@pytest.fixture(scope="session", autouse=True)
def _built_checkers():
    import oracle as O

    if not O.available("port"):
        O.build()
