"""Matrix Market reader timing: the library (multi-threaded parse + sort/fold)
vs the unmodified reference reader (oracle/_ref/mm_ref) on the same file.

usage: python tools/mm_bench.py [cfg]   (default: config 2, 3D grid 128^3)
"""
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1108_1310_b200 import graphs as G  # noqa: E402
from paper_1108_1310_b200 import lamg as L  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a = G.make_config(cfg)
d = tempfile.mkdtemp()
path = os.path.join(d, "g.mtx")
t = time.time()
L.write_matrix_market(path, a)
tw = time.time() - t
t = time.time()
b, lap, _ = L.read_matrix_market(path)
tr = time.time() - t
assert np.array_equal(b.val, a.val) and np.array_equal(b.col, a.col)
t = time.time()
subprocess.run([os.path.join(ROOT, "oracle", "_ref", "mm_ref"), path, "0", "1", path + ".bin"], check=True)
tref = time.time() - t
print(json.dumps({"config": cfg, "n": a.n, "m": a.m, "file_mb": round(os.path.getsize(path) / 1e6, 1),
                  "write_s": round(tw, 2), "read_s": round(tr, 2), "reference_read_s": round(tref, 2),
                  "speedup": round(tref / tr, 1), "threads": os.cpu_count()}))
