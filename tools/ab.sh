#!/usr/bin/env bash
# A/B of library variants on one GPU (run under gpurun).  Variants are built here first with
#   python -c "from paper_1510_03816_b200 import _build; _build.build(defines=['GS_CELL_MINB=6'], tag='m6')"
# then compared, each against the product library ("base"), on the RHS of the given configs:
#   tools/ab.sh "C5 C4" cell m6 m5        # tags of libgs_b200_<tag>.so
# Environment-variable knobs (GS_B200_CELL_SUB=3, GS_B200_SORT_SMALL_MAX=0, ...) go in front:
#   GS_B200_CELL_SUB=3 tools/ab.sh "C5" cell
# Every variant's (dq, dp) is compared with the base output (tools/ab_compare.py).
set -u
cfgs=${1:-C5}; path=${2:-cell}; shift 2 || true
for cfg in $cfgs; do
  for v in base "$@" base; do
    if [ "$v" = base ]; then L=paper_1510_03816_b200/libgs_b200.so; else L=paper_1510_03816_b200/libgs_b200_$v.so; fi
    printf "%s %s: " "$cfg" "$v"
    GS_B200_LIB=$PWD/$L python tools/profile_rhs.py --config "$cfg" --path "$path" --reps 5 \
      --save "gpurun_out/ab_${cfg}_$v.npz" 2>&1 | tail -n 1
  done
  for v in "$@"; do python tools/ab_compare.py "gpurun_out/ab_${cfg}_$v.npz" "gpurun_out/ab_${cfg}_base.npz"; done
done
rm -f gpurun_out/ab_*.npz
