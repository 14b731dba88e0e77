"""Debug: a tiny case where phase 2 leaves excess; dump the arcs around it."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2601_17026_b200 import colgraph as cg
from synth import volumes as V
c, delta = V.tiny_case(1097)
X, Y, Z = c.shape
t = torch.from_numpy(np.ascontiguousarray(c)).cuda()
h = cg.colgraph_build(t, delta)
st, flow, _ = cg.maxflow_solve(h, None)
def state():
    a = torch.empty(8 * c.size, dtype=torch.int32, device="cuda")
    cg.lib().colgraph_export_state(h, a.data_ptr())
    return a.cpu().numpy().reshape(8, X, Y, Z)
pre = state()
st2, F = cg.maxflow_export_flow(h, t)
post = state()
cg.colgraph_free(h)
print("shape", c.shape, "delta", delta, "status", st2)
w = c.astype(np.int64).copy(); w[:, :, 0] = c[:, :, 0] - (c.sum(axis=2) + 1); w[:, :, 1:] = c[:, :, 1:] - c[:, :, :-1]
print("w", w.tolist())
for name, S in (("pre", pre), ("post", post)):
    print(name, "E", S[0].tolist()); print(name, "H", S[1].tolist()); print(name, "T", S[2].tolist()); print(name, "D", S[3].tolist())
    for d in range(4): print(name, "L%d" % d, S[4 + d].tolist())
