import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2009_00083_b200 as P
from oracle import lts_oracle as O
name = sys.argv[1]; sad = int(sys.argv[2])
z = np.load(f"tests/golden/{name}.npz")
dims = tuple(int(d) for d in z["dims"]); rank = z["F_rank"]
mesh = P.build_grid_triangulation(dims)
mn, mx = O.extrema(dims, rank)
keep = np.intersect1d(mx, z["pres_max"])
rp, rv = z["max_region_ptr"], z["max_region_verts"]
r = [i for i in range(len(rp)-1) if rv[rp[i]] == sad][0]
verts = rv[rp[r]:rp[r+1]]
print("region", verts.tolist(), "ranks", rank[verts].tolist())
for cap in (1, 2, 3, 4):
    loc, nit, st = O.localize(dims, np.array([0, verts.size]), verts, rank, cap)
    pr = P.remove_pass(mesh, P.order_from_ranks(rank), P.ConstraintSet(preserveMinima=mn, preserveMaxima=keep), "max", max_iterations=cap)
    ptr = pr.region_ptr.cpu().numpy(); gv = pr.region_verts.cpu().numpy()
    gr = [i for i in range(len(ptr)-1) if gv[ptr[i]] == sad][0]
    print("cap", cap, "ref", loc.tolist(), nit.tolist(), st.tolist(), "| gpu", gv[ptr[gr]:ptr[gr+1]].tolist() == verts.tolist(), pr.local_rank.cpu().numpy()[ptr[gr]:ptr[gr+1]].tolist(), int(pr.n_iters[gr]), int(pr.status[gr]))
