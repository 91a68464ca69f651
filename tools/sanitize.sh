#!/usr/bin/env bash
# compute-sanitizer over the reduced-size GPU parity suite (every kernel of the
# encoder and decoder runs: K1 convert incl. the exact queue and its overflow
# re-pass, start/fit/refit incl. the cp.async prefetch slots and the global
# work-stealing counter, emit, entropy, and the whole decoder).
#   bash tools/sanitize.sh [tool ...]      (default: memcheck racecheck synccheck initcheck)
# Logs: gpurun_out/sanitize/<tool>.log
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
SEL=${STPC_SAN_SEL:-"golden or fuzz or edge or project or decode_errors or overlap or entropy or pipelined or gather_pipeline or intermediates or repeated or conftest_sensor"}
TOOLS=${*:-memcheck racecheck synccheck initcheck}
for t in $TOOLS; do
  extra=""
  [ "$t" = memcheck ] && extra="--leak-check full"
  timeout ${STPC_SAN_TIMEOUT:-1500} /usr/local/cuda/bin/compute-sanitizer --tool "$t" $extra --target-processes all \
    --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$SEL" \
    > "gpurun_out/sanitize/$t.log" 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize/$t.log | tail -3 | tr '\n' ' ')"
done
