import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_08233_b200 as bl
from blgen import grid_graph, uniform_coords
which = sys.argv[1]
g = grid_graph(int(sys.argv[2]), int(sys.argv[2]))
xy = uniform_coords(g.n, 1)
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d = torch.from_numpy(xy.copy()).cuda()
    t = time.time()
    if which == "eu": r = bl.bl_edge_uniformity(lay.h, d)
    if which == "st": r = bl.bl_stress(lay.h, d, np.arange(min(g.n, int(sys.argv[3])), dtype=np.int32))
    if which == "np": r = bl.bl_neighborhood_preservation(lay.h, d, np.arange(min(g.n, int(sys.argv[3])), dtype=np.int32))
    print(which, r, time.time() - t, flush=True)
