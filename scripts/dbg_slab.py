import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2601_17026_b200 import colgraph as cg
from synth import volumes as V
import oracle
from tests.test_gpu_parity import _certificate
c, delta = V.tiny_case(3023)
o = oracle.colgraph_solve(c, delta)
for ns in (1, 2, 3):
    for walk in (64, -1):
        t = torch.from_numpy(c).cuda()
        h = cg.colgraph_build_slabs(t, delta, ns)
        st, flow, stats = cg.maxflow_solve(h, cg.make_opts(walk_len=walk))
        out = torch.empty(8 * c.size, dtype=torch.int32, device='cuda')
        cg.colgraph_export_state(h, out); cg.colgraph_free(h)
        s = out.cpu().numpy()
        msg = 'ok'
        try: _certificate(c, delta, s)
        except AssertionError as e: msg = 'CERT FAIL: ' + str(e)[:200]
        X,Y,Z = c.shape; n=c.size
        E = s[:n].reshape(X,Y,Z); L = [s[(4+d)*n:(5+d)*n].reshape(X,Y,Z) for d in range(4)]
        print(ns, walk, st, flow, o['flow'], msg, 'minE', E.min(), 'minL', min(l.min() for l in L), 'minD', s[3*n:4*n].min())
