import ctypes, os, sys
sys.path.insert(0, os.getcwd())
sys.argv = [sys.argv[0], "64"]
import tools.decode_diag as dd
from paper_2008_06972_b200 import _native
L = _native.load()
dd.main()
st = (ctypes.c_ulonglong * 8)()
L.stpc_debug_huff_stats(st)
print("huff stats (3 decode reps x 64 blobs): symbols parsed", st[0], "rounds", st[1], "corrected threads", st[2])
