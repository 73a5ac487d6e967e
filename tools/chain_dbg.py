import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0808_2664_b200 as T
m, n = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator().manual_seed(0)
A0 = torch.randn((n, m), dtype=torch.float64, generator=g)
A = A0.cuda()
R, tree = T.factor(A, m, m)
torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/dbg_{m}_{n}.npz", A0=A0.numpy(), A=A.cpu().numpy(), R=R.cpu().numpy())
print("saved")
