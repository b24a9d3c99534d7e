#!/usr/bin/env bash
# Run the reference's OWN test suite (geoshoot, 156 tests) against the B200 drop-in.
#
#   tools/run_reference_suite.sh prepare   # here (needs /root/reference): install the unmodified
#                                          # reference into the git-ignored baseline/_ref and copy
#                                          # its test files beside it (never committed)
#   tools/run_reference_suite.sh run       # on a GPU box (gpurun): pytest with the drop-in plugin
#
# The plugin (paper_1510_03816_b200.pytest_dropin) rebinds every alias of rhs / evolve / match /
# hamiltonian / analysis before collection, so the reference's test files run
# unmodified on the device path.
set -euo pipefail
cd "$(dirname "$0")/.."
case "${1:-run}" in
prepare)
    rm -rf /tmp/geoshoot_src && cp -r /root/reference/pkg /tmp/geoshoot_src
    python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
        --target baseline/_ref /tmp/geoshoot_src
    mkdir -p baseline/_ref/geoshoot_tests && cp /root/reference/pkg/tests/*.py baseline/_ref/geoshoot_tests/
    ;;
run)
    mkdir -p gpurun_out
    PYTHONPATH=baseline/_ref:. python -m pytest -p paper_1510_03816_b200.pytest_dropin -p no:cacheprovider \
        baseline/_ref/geoshoot_tests -q -rf --durations=15 2>&1 | tee gpurun_out/ref_suite_dropin.log
    ;;
esac
