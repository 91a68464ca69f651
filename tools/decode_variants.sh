for v in "$@"; do
  STPC_B200_LIB=$v timeout 300 python tools/decode_diag.py 1024 2>&1 | tail -1 | sed "s|^|$v |"
done
