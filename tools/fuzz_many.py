"""Wide fuzz sweep of tests/test_gpu_parity.py::test_fuzz_small_configs_blob
(GPU; the test suite runs 12 seeds, this runs N).

    python tools/fuzz_many.py [N]
"""
import os
import sys
import warnings

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
warnings.simplefilter("ignore")

import test_gpu_parity as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
bad = []
for seed in range(n):
    try:
        T.test_fuzz_small_configs_blob(seed)
    except Exception as e:  # noqa: BLE001
        bad.append((seed, repr(e)[:300]))
print(f"fuzz: {n - len(bad)}/{n} seeds byte-identical")
for b in bad[:10]:
    print(b)
