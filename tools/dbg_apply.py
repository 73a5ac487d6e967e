import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch, oracle as orc, paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs
for (m, n, b, s, k) in [(512,16,512,128,16),(1024,16,512,128,16),(1024,16,1024,128,16),(384,16,384,128,16),(2048,16,2048,128,16),(4096,16,512,96,16),(4096,16,512,64,16),(4096,32,512,128,16),(1024,16,512,128,64)]:
    At = inputs.gaussian(m, n, 0); A0 = inputs.to_numpy_colmajor(At).copy()
    Ad = At.cuda(); R, tree = T.factor(Ad, b, s)
    Ct = inputs.gaussian(m, k, 1); C0 = inputs.to_numpy_colmajor(Ct).copy(); Cd = Ct.cuda()
    T.apply_qt(tree, Cd); torch.cuda.synchronize()
    p = orc.plan(m, n, b, s, 1)
    f = orc.tsqr_factor(A0, p)
    Co = orc.tsqr_apply_qt(f, C0); Cg = inputs.to_numpy_colmajor(Cd)
    d = np.abs(Cg - Co).max(axis=1)
    bad = np.nonzero(d > 1e-10)[0]
    print(m, n, b, s, k, "tiles", p.ntiles, "err %.2e" % orc.rel_fro(Cg, Co), "bad rows", bad[:12], len(bad), "tile starts", p.tile_row0[:8])
