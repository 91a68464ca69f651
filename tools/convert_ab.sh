#!/bin/bash
# A/B the convert stage of several library builds on the bench workload.
#   tools/convert_ab.sh [lib.so|product|regs ...]   (regs = product with STPC_CONVERT_REGS=1)
for v in "$@"; do
  unset STPC_CONVERT_REGS STPC_B200_LIB
  case $v in product) ;; regs) export STPC_CONVERT_REGS=1 ;; *) export STPC_B200_LIB=$v ;; esac
  timeout 300 python bench.py --no-e2e --no-cpu --no-decode --steps 5 --warmup 3 $BENCH_ARGS 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);s=d['stage_ms'];p=d.get('parity') or {};print('$v', round(d['value']), 'convert', s['convert'], 'bitmaps', s['bitmaps'], 'parity', p.get('identical'), '/', p.get('groups_checked'))"
done
