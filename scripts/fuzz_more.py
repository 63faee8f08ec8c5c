#!/usr/bin/env python3
"""Run the randomized envelope test (tests/test_gpu_fuzz.py) over many more
seeds than the suite's 40 (development confidence runs on a B200).

    python scripts/fuzz_more.py [first_seed] [last_seed]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import test_gpu_fuzz as f  # noqa: E402

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 40
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 400
bad = []
for seed in range(lo, hi):
    try:
        f.test_fuzz_envelope(seed)
    except Exception as e:  # noqa: BLE001
        bad.append((seed, repr(e)[:300]))
print(f"seeds {lo}..{hi - 1}: {len(bad)} failures")
for b in bad[:20]:
    print(b)
