#!/bin/bash
# A/B the decoder of several library builds (tools/decode_diag.py phases, 1024 groups).
#   tools/decode_ab.sh [lib.so|product ...]
for v in "$@"; do
  unset STPC_B200_LIB
  [ "$v" = product ] || export STPC_B200_LIB=$v
  echo "== $v"; timeout 300 python tools/decode_diag.py ${DEC_GROUPS:-1024} 2>&1 | tail -2
done
