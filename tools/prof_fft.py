import sys
sys.path.insert(0, ".")
import torch
from paper_2008_11607_b200 import inputs, rexi
D = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
p = rexi.Plan(D, 0.1, tol=1e-8)
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
for _ in range(3):
    F = p.forward(*f)
    out = p.inverse(F)
torch.cuda.synchronize()
print("ok")
