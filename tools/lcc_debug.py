import sys; sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo')
import numpy as np
from test_gpu_gen import _disconnected
from paper_1108_1310_b200 import graphs as G
from paper_1108_1310_b200 import lamg as L
for seed in (1, 2, 3):
    full = _disconnected(seed)
    d = L.largest_component(full).download()
    sub, nodes = G.largest_component(full)
    print(seed, "gpu", d.n, d.m, "numpy", sub.n, sub.m, "eq", d.m == sub.m and np.array_equal(d.col, sub.col))
    # try all 300-node components
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    g = csr_matrix((np.ones(len(full.col)), full.col, full.row_ptr), shape=(full.n, full.n))
    nc, lab = connected_components(g, directed=False)
    for l in range(nc):
        nd = np.flatnonzero(lab == l)
        if len(nd) == d.n:
            print("   comp", l, "min node", nd.min(), "size", len(nd))
