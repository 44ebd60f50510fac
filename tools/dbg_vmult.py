import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_09497_b200 as smg
k = int(sys.argv[1]); level = int(sys.argv[2]); dt = torch.float64 if (len(sys.argv) < 4 or sys.argv[3] == 'f64') else torch.float32
ctx = smg.Context(k, level)
x = torch.rand(ctx.sizes(level)[4], dtype=dt, device='cuda')
y = ctx.apply_stokes(level, x)
torch.cuda.synchronize()
print('ok', float(y.abs().sum()))
