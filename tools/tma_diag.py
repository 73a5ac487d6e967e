"""Which chain configurations run with TMA staging (diagnostic, not product code)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0808_2664_b200 as T
n = int(sys.argv[1]); m = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
b = int(sys.argv[3]) if len(sys.argv) > 3 else 700
A = torch.randn((n, m), dtype=torch.float64, device="cuda")
R, tree = T.factor(A, b, 0)
torch.cuda.synchronize()
print("ok", n, m, b, float(R.abs().sum()))
