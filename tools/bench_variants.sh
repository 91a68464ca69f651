#!/bin/bash
# Time the encode step of several library builds back to back (tuning aid).
#   tools/bench_variants.sh [lib.so ...]     ("product" = the in-tree library)
# Prints value and the fit stage times per build; BENCH_ARGS adds bench.py flags.
for v in "$@"; do
  if [ "$v" = product ]; then unset STPC_B200_LIB; else export STPC_B200_LIB=$v; fi
  timeout 300 python bench.py --no-e2e --no-cpu --no-decode --no-parity --steps 5 --warmup 3 $BENCH_ARGS 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());s=d['stage_ms'];print('$v', round(d['value']), 'fit_key', s['fit_key'], 'fit_p', s['fit_p'], 'start_p', s['start_p'], 'refit', s['refit'], 'convert', s['convert'], 'emit', s['emit'], 'pack', s['pack'])"
done
