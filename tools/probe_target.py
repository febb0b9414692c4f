"""ncu target: one launch set of the random-gather probe (4 B over 4 GiB)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2009_07174_b200 import api  # noqa: E402

print(api.gather_probe(0, 4 << 30, 4, 1))
