"""Run tests/test_gpu_fuzz.py on 40 more seeds (9..48): a longer soak of the
random programs than the suite's 8."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_fuzz as F
ok = 0
for seed in range(9, 49):
    F.test_random_programs(seed)
    ok += 1
print("fuzz seeds passed:", ok)
