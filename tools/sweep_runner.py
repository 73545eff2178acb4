"""Run extra cases of tests/test_gpu_parity.py::test_seeded_sweep (bug hunting; not part of the suite)."""
import sys, traceback
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_gpu_parity as t
lo, hi = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for i in range(lo, hi):
    try:
        t.test_seeded_sweep(i)
    except Exception as e:
        bad += 1
        print("FAIL", i, t._fuzz_case(i)[:4], repr(e)[:300], flush=True)
print("done", lo, hi, "failures", bad)
