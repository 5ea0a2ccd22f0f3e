import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


class _OptionPatch:
    """monkeypatch-style setter for the library's run-time options
    (sgb_set_option; the environment is read once per process, so tests switch
    knobs through the C API), restored on undo()."""

    def __init__(self):
        self._saved = []

    def setenv(self, key, value):
        from paper_1907_02818_b200 import api
        name = key[4:] if key.startswith("SGB_") else key
        self._saved.append((name, api.get_option(name)))
        api.set_option(name, int(value))

    def undo(self):
        from paper_1907_02818_b200 import api
        while self._saved:
            name, (v, was_set) = self._saved.pop()
            api.set_option(name, v if was_set else None)

    def context(self):
        import contextlib

        @contextlib.contextmanager
        def cm():
            p = _OptionPatch()
            try:
                yield p
            finally:
                p.undo()
        return cm()


import pytest  # noqa: E402


@pytest.fixture
def sgbopt():
    p = _OptionPatch()
    yield p
    p.undo()
