#!/usr/bin/env bash
# compute-sanitizer evidence for every kernel family (run on one GPU through gpurun):
#   bash tools/sanitize.sh            -> gpurun_out/sanitizer/<tool>_<target>.log
# memcheck (out-of-bounds / misaligned accesses, leaks off), racecheck (shared-memory hazards),
# synccheck (barrier misuse), initcheck (reads of uninitialised device memory) on the small
# workloads of tools/sanitize_targets.py, plus the two-rank peer-exchange emulation under memcheck.
set -u
out=gpurun_out/sanitizer
mkdir -p $out
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
for tgt in small small1 sym partial cell verlet match batch velocity; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 $CS --tool $tool python tools/sanitize_targets.py $tgt > $out/${tool}_${tgt}.log 2>&1
    echo "$tool $tgt rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/${tool}_${tgt}.log | tail -1)"
  done
done
timeout 1200 $CS --tool memcheck python -m pytest tests/test_gpu_sharded.py -q -k "peer_exchange_two_ranks_emulated" \
  > $out/memcheck_p2p_emulation.log 2>&1
echo "memcheck p2p_emulation rc=$? $(grep -E 'ERROR SUMMARY' $out/memcheck_p2p_emulation.log | tail -1)"
timeout 1200 $CS --tool synccheck python -m pytest tests/test_gpu_sharded.py -q -k "peer_exchange_two_ranks_emulated" \
  > $out/synccheck_p2p_emulation.log 2>&1
echo "synccheck p2p_emulation rc=$? $(grep -E 'ERROR SUMMARY' $out/synccheck_p2p_emulation.log | tail -1)"
