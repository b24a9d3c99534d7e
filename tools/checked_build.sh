#!/usr/bin/env bash
# Build the checked library (device-side bounds / protocol asserts, -DGS_CHECKED) next to the
# product library: paper_1510_03816_b200/libgs_b200_checked.so.  Run the GPU suite against it with
#   GS_B200_LIB=$PWD/paper_1510_03816_b200/libgs_b200_checked.so python -m pytest tests -m gpu
set -euo pipefail
cd "$(dirname "$0")/.."
python -c "from paper_1510_03816_b200 import _build; print(_build.build(defines=['GS_CHECKED'], tag='checked'))"
