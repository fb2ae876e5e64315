"""Out-of-bounds writes (GPU). compute-sanitizer is not available on the GPU
pool; the library's guard mode (LAMG_GUARD=1: 256-byte pattern bands around
every device buffer, checked at release) and NaN poisoning of fresh buffers
(LAMG_POISON=1) run over the memory-safety workload -- the smoke solve, a
power-law THROUGHPUT solve from two contexts, a 32-column block through the
exact finest sweep and the cluster / slice tail -- and must find no overrun
while every result still matches its reference."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_bands_find_no_overrun():
    env = dict(os.environ, LAMG_GUARD="1", LAMG_POISON="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout + p.stderr
    m = re.search(r"guard bands: (\d+) buffers checked, (\d+) overruns", p.stdout)
    assert m and int(m.group(1)) > 100 and int(m.group(2)) == 0, p.stdout
    assert "[lamg guard]" not in p.stderr
