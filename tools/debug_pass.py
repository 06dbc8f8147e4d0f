"""Debug helper: compare one GPU maxima pass with the oracle on a golden case."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2009_00083_b200 as P
from oracle import lts_oracle as O
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_192"
z = np.load(f"tests/golden/{name}.npz")
dims = tuple(int(d) for d in z["dims"]); rank = z["F_rank"]
mesh = P.build_grid_triangulation(dims)
mn, mx = O.extrema(dims, rank)
keep = np.intersect1d(mx, z["pres_max"])
seeds = np.setdiff1d(mx, keep)
st, own, sad, park, tops, err = O.discover(dims, rank, seeds)
cl_ref = np.flatnonzero(st == 2)
pr = P.remove_pass(mesh, P.order_from_ranks(rank), P.ConstraintSet(preserveMinima=mn, preserveMaxima=keep), "max")
ptr = pr.region_ptr.cpu().numpy(); verts = pr.region_verts.cpu().numpy()
print("regions gpu", len(ptr) - 1, "ref", len(np.unique(own[cl_ref])), "claimed gpu", pr.report.claimed, "ref", cl_ref.size)
head = np.zeros(verts.size, bool); head[ptr[:-1]] = True
cl_gpu = np.sort(verts[~head])
print("claimed equal", np.array_equal(cl_gpu, cl_ref))
extra = np.setdiff1d(cl_gpu, cl_ref); missing = np.setdiff1d(cl_ref, cl_gpu)
print("extra", extra.size, extra[:10], "missing", missing.size, missing[:10])
print("dup slots", verts[~head].size - np.unique(verts[~head]).size)
# region compare by saddle
ref_reg = {}
for r in np.unique(own[cl_ref]):
    mem = np.sort(cl_ref[own[cl_ref] == r]); ref_reg[(int(sad[r]), int(tops[r]))] = mem
got_reg = {}
top = pr.topseed.cpu().numpy()
for r in range(len(ptr) - 1):
    seg = verts[ptr[r]:ptr[r+1]]
    got_reg[(int(seg[0]), int(top[r]))] = np.sort(seg[1:])
bad = [k for k in ref_reg if k not in got_reg or not np.array_equal(got_reg[k], ref_reg[k])]
print("bad regions", len(bad), "of", len(ref_reg))
for k in bad[:5]:
    g = [kk for kk in got_reg if kk[0] == k[0]]
    print(" ref", k, ref_reg[k].size, ref_reg[k][:8], "gpu same saddle:", [(kk, got_reg[kk].size) for kk in g][:3])
# check sortedness by rank within gpu regions
bad_sort = sum(1 for r in range(len(ptr)-1) if np.any(np.diff(rank[verts[ptr[r]+1:ptr[r+1]]]) <= 0))
print("regions not rank-sorted:", bad_sort)
