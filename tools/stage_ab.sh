#!/bin/bash
# A/B the encode stages of several library builds on the bench workload.
#   tools/stage_ab.sh [lib.so|product ...]
for v in "$@"; do
  unset STPC_B200_LIB
  [ "$v" = product ] || export STPC_B200_LIB=$v
  timeout 300 python bench.py --no-e2e --no-cpu --no-decode --steps 5 --warmup 3 $BENCH_ARGS 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);s=d['stage_ms'];p=d.get('parity') or {};print('$v', round(d['value']), ' '.join(f'{k} {v:.2f}' for k,v in s.items()), 'parity', p.get('identical'), '/', p.get('groups_checked'))"
done
