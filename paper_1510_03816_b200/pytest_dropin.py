"""pytest plugin: ``pytest -p paper_1510_03816_b200.pytest_dropin <geoshoot tests>``.

Installs the drop-in before test collection (test modules bind names such as
``from geoshoot import rhs`` at import time), so a geoshoot-based test suite
exercises the B200 path unmodified.
"""


def pytest_configure(config):
    from . import dropin

    dropin.install()


def pytest_unconfigure(config):
    from . import dropin

    dropin.uninstall()
