#!/usr/bin/env bash
# Build the CPU oracle (test infrastructure only) into oracle/libgs_oracle.so.
# -ffp-contract=off keeps the reference's separate multiply/add roundings.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
gcc -O3 -march=x86-64-v3 -ffp-contract=off -fopenmp -fPIC -shared \
    -o "$here/libgs_oracle.so" "$here/gs_oracle.c" -lm
